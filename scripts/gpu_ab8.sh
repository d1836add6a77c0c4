#!/bin/bash
TAG=${1:-ab8}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for E in "MSB_OLD_LEAF=1" "X=1"; do
  env $E timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr > $OUT/b.log 2>&1
  python - "$OUT/b.log" "$E" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    c5 = d.get('config5') or {}
    print(f"{sys.argv[2]:20s} iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f}) coarse {d['phase_ms']['t_coarse']:.2f} ms  c5 iter {c5.get('ms_per_iteration', 0)*1e3:7.1f} us ({c5.get('roofline_cycle', {}).get('frac', 0):.3f}) c5 coarse {c5.get('coarse_setup_ms',0):.1f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e, open(sys.argv[1]).read()[-800:])
PY
  env $E MSB_DYN_PROFILE=1 timeout 300 python scripts/run_config.py 3 >> $OUT/config3.txt 2>&1
done
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "cycle or schur or fgmres or dynamic or config3 or config2 or rap or constant or coarse or singular or error" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
cat $OUT/summary.txt $OUT/config3.txt; tail -2 $OUT/pytest.log
