#!/bin/bash
# A/B of the fused fixed-point Cartesian chain (k_resrestrict_fx + k_symv_tiles_fx +
# k_prolong_cart_fx) against the five-kernel chain: smoke, parity subset, config-2 bench.
TAG=${1:-ab15}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -20 $OUT/smoke.log; exit 1; }
run() {
  env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr --no-config5 > $OUT/b.log 2>&1
  python - "$OUT/b.log" "$*" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    print(f"{sys.argv[2]:28s} iter {d['ms_per_iteration']*1e3:7.2f} us ({d['hbm']['cycle_frac']:.3f}) iters {d['iterations_per_step']} res {d['final_rel_residual']:.3e} sweep {d['hbm']['sweep_frac']:.3f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e); print(open(sys.argv[1]).read()[-1500:])
PY
}
run MSB_X_FX=0
run MSB_X_UNR=2
run MSB_X_UNR=1
run MSB_X_UNR=4
run MSB_X_FX=0
run MSB_X_UNR=2
run5() {
  env "$@" timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-cpr > $OUT/b5.log 2>&1
  python - "$OUT/b5.log" "$*" <<'PY' >> $OUT/summary.txt
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][0])
    c5 = d['config5']
    print(f"{sys.argv[2]:28s} c5 iter {c5['ms_per_iteration']*1e3:7.1f} us ({c5['roofline_cycle']['frac']:.3f}) res {c5['final_rel_residual']:.6e} sweep {c5['roofline_sweep']['frac']:.3f}")
except Exception as e:
    print(sys.argv[2], "FAILED", e); print(open(sys.argv[1]).read()[-1500:])
PY
}
run5 MSB_X_FX=0
run5 MSB_X_UNR=2
run5 MSB_X_UNR=1
run5 MSB_X_UNR=4
cat $OUT/summary.txt
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "cycle or config2 or config4 or config5 or schur or error or zero or fixed or reproducib or import" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
