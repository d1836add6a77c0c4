#!/bin/bash
TAG=${1:-ab16}
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
run MSB_X_UNR=1 MSB_X_PF=1
run MSB_X_UNR=1 MSB_X_PF=0
run MSB_X_UNR=2 MSB_X_PF=0
run MSB_X_UNR=4 MSB_X_PF=0
cat $OUT/summary.txt
for v in "MSB_X_UNR=1 MSB_X_PF=0" "MSB_X_UNR=2 MSB_X_PF=0" "MSB_X_UNR=1 MSB_X_PF=1"; do
  n=$(echo $v | tr ' =' '__')
  env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$n.csv python scripts/profile_step.py > $OUT/ncu_$n.log 2>&1
  python scripts/ncu_summary.py launches $OUT/launches_$n.csv > $OUT/launches_$n.txt 2>&1
  echo "== $v"; head -12 $OUT/launches_$n.txt
done
