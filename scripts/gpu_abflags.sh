#!/bin/bash
# Generic compile-time A/B: one build + bench per line of nvcc -D flags in the variants file.
#   bash scripts/gpu_abflags.sh TAG VARIANTS_FILE
TAG=${1:-abflags}
VAR=${2:-scripts/ab_variants.txt}
OUT=gpurun_out/$TAG
mkdir -p $OUT
while read -r flags; do
  [ -z "$flags" ] && continue
  [ "$flags" = "-" ] && flags=""
  MSB_EXTRA_NVCC_FLAGS="$flags" timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
  timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr $ABX > $OUT/b.log 2>&1
  python - "$OUT/b.log" "$flags" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    c5 = d['config5']
    print(f"{sys.argv[2]:44s} sweep {d['ms_per_sweep']*1e3:6.2f} us ({d['hbm']['sweep_frac']:.3f}) iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f}) iters {d['iterations_per_step']} res {d['final_rel_residual']:.3e} coarse {d['phase_ms']['t_coarse']:.1f} ms | c5 sweep {c5['ms_per_sweep']*1e3:6.1f} ({c5['roofline_sweep']['frac']:.3f}) iter {c5['ms_per_iteration']*1e3:7.1f} us ({c5['roofline_cycle']['frac']:.3f}) res {c5['final_rel_residual']:.6e}")
except Exception as e:
    print(sys.argv[2], "FAILED", e); print(open(sys.argv[1]).read()[-1500:])
PY
done < $VAR
cat $OUT/summary.txt
