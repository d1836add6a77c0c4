#!/bin/bash
# ncu passes of the round evidence only (launch lists + --set full captures), see gpu_round.sh
TAG=${1:-ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/bench_plain.log 2>&1 &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
    --log-file $OUT/bench_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
    > $OUT/ncu_bench_launch.log 2>&1
timeout 300 python scripts/profile_step.py > $OUT/profile_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -c 1 \
    -o $OUT/sweep python scripts/profile_step.py > $OUT/ncu_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_jacobi|k_residual|k_restrict|k_symv|k_prolong|k_finalize" -s 35 -c 7 \
    -o $OUT/cycle python scripts/profile_step.py > $OUT/ncu_cycle.log 2>&1
echo done
