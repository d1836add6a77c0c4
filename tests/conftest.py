import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running oracle comparison")


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ---------------------------------------------------------------- parity log
# Every GPU parity comparison records (case, k_gpu, k_oracle, err, floor, tol) so the
# distances behind each green test are visible, not just pass/fail.  Written at the end of
# the session to $PARITY_LOG (default gpurun_out/parity_r02.json when a GPU ran).
PARITY_RECORDS = []


def record_parity(case, **kw):
    rec = {"case": case}
    for k, v in kw.items():
        try:
            import numpy as np
            if isinstance(v, (np.generic,)):
                v = v.item()
        except Exception:
            pass
        rec[k] = v
    PARITY_RECORDS.append(rec)
    return rec


def pytest_sessionfinish(session, exitstatus):
    if not PARITY_RECORDS:
        return
    import json
    path = os.environ.get("PARITY_LOG", os.path.join(ROOT, "gpurun_out", "parity_r02.json"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w") as f:
        json.dump({"records": PARITY_RECORDS, "exitstatus": int(exitstatus)}, f, indent=1)
