"""Multi-rank host logic of bench.py on CPU (gloo, world_size 2).

The path does not shard (replicas only), so the only cross-rank step is
the job-time reduction: every rank times its own replica and rank 0 reports the max
(`bench.max_over_ranks`), with value = world_size x per-replica units / max time.
"""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import torch.distributed as dist
import bench
dist.init_process_group("gloo", init_method="env://")
r = dist.get_rank()
vals = [1.0 + r, 10.0 - r, 5.0]          # rank 0: [1, 10, 5]; rank 1: [2, 9, 5]
out = bench.max_over_ranks(vals, dist, "cpu")
assert out == [2.0, 10.0, 5.0], out
ws = dist.get_world_size()
# weak-scaling value: all replicas' units over the slowest rank's time
t = bench.max_over_ranks([0.5 + 0.25 * r], dist, "cpu")[0]
assert abs(ws * 300 / t - 2 * 300 / 0.75) < 1e-12
print("rank", r, "ok", flush=True)
dist.destroy_process_group()
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_max_over_ranks_gloo_two_ranks(tmp_path):
    w = tmp_path / "worker.py"
    w.write_text(WORKER)
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r),
                   WORLD_SIZE="2", LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, str(w), ROOT], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=120)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o
        assert "ok" in o


def test_single_rank_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks([3.0, 1.0]) == [3.0, 1.0]
