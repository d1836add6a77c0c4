#!/bin/bash
# A/B matrix of env knobs on the config-2 bench (no CPU baseline).  usage: perf_matrix.sh tag "ENV1" "ENV2" ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
i=0
for E in "$@"; do
  env $E timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-config5 > $OUT/b$i.log 2>&1
  python - "$OUT/b$i.log" "$E" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    print(f"{sys.argv[2]:40s} sweep {d['ms_per_sweep']*1e3:7.2f} us ({d['hbm']['sweep_frac']:.3f})  iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f})  coarse {d['phase_ms']['t_coarse']:.1f} ms")
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  i=$((i+1))
done
cat $OUT/summary.txt
