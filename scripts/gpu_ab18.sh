#!/bin/bash
# A/B of compile-time streaming hints on the P loads of the Cartesian restriction and
# prolongation (-DMSB_PHINT=0 plain, 1 ld.global.cs, 2 createpolicy evict_first, 3 = 2 + hinted prefetch)
TAG=${1:-ab18}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in 0 1 2 3 0 2; do
  MSB_EXTRA_NVCC_FLAGS="-DMSB_PHINT=$v" timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
  timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr > $OUT/b.log 2>&1
  python - "$OUT/b.log" "PHINT=$v" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    c5 = d['config5']
    print(f"{sys.argv[2]:10s} iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f}) iters {d['iterations_per_step']} res {d['final_rel_residual']:.3e} sweep {d['hbm']['sweep_frac']:.3f} | c5 iter {c5['ms_per_iteration']*1e3:7.1f} us ({c5['roofline_cycle']['frac']:.3f}) res {c5['final_rel_residual']:.6e}")
except Exception as e:
    print(sys.argv[2], "FAILED", e); print(open(sys.argv[1]).read()[-1500:])
PY
done
cat $OUT/summary.txt
