#!/bin/bash
TAG=${1:-ab13}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for i in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr > $OUT/b.log 2>&1
  python - "$OUT/b.log" <<'PY' >> $OUT/summary.txt
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
c5 = d.get('config5') or {}
print(f"iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f}) sweep {d['hbm']['sweep_frac']:.3f} cycle_ms {d['phase_ms']['t_cycle']:.2f} c5 iter {c5.get('ms_per_iteration', 0)*1e3:7.1f} us ({c5.get('roofline_cycle', {}).get('frac', 0):.3f})")
PY
done
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "cycle or schur or fgmres or config2 or config5 or config4 or ilu or static or error or zero or fixed or reproducib" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
cat $OUT/summary.txt; tail -2 $OUT/pytest.log
