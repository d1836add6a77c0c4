#!/bin/bash
# Development call: new-path tests, then an A/B matrix of experiment knobs on the config-2
# bench and config 5.  usage: gpu_ab.sh TAG "ENV..." ...
TAG=${1:-ab}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_cpr.py -x -q > $OUT/pytest_cpr.log 2>&1; echo "rc=$?" >> $OUT/pytest_cpr.log
PARITY_LOG=$OUT/parity_cycle.json timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cycle or schur or symv or fgmres" > $OUT/pytest_cycle.log 2>&1; echo "rc=$?" >> $OUT/pytest_cycle.log
for E in "$@"; do
  env $E timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-config5 > $OUT/b.log 2>&1
  python - "$OUT/b.log" "$E" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    print(f"{sys.argv[2]:40s} sweep {d['ms_per_sweep']*1e3:7.2f} us ({d['hbm']['sweep_frac']:.3f})  iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f})  coarse {d['phase_ms']['t_coarse']:.1f} ms")
except Exception as e:
    print(sys.argv[2], "FAILED", e, open(sys.argv[1]).read()[-500:])
PY
done
for E in "MSB_X_SYMV=0" "MSB_X_SYMV=1"; do
  echo "== $E" >> $OUT/config5.txt
  env $E timeout 600 python scripts/run_config.py 5 >> $OUT/config5.txt 2>&1
done
cat $OUT/summary.txt
