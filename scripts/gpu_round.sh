#!/bin/bash
# Round-evidence call: smoke, full GPU test suite, the default bench (with the CPU
# oracle baseline), the ncu launch list, and ncu --set full captures of the sweep and of
# one cycle iteration's kernels -> profiles/roofline_traffic.json input.
TAG=${1:-round}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { echo smoke failed; tail $OUT/smoke.log; exit 1; }
PARITY_LOG=$OUT/parity_r02.json timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 600 python scripts/run_config.py 5 > $OUT/config5.json 2>&1
timeout 900 python scripts/run_config.py 4 --steps 100 > $OUT/config4.json 2>&1
timeout 300 python scripts/run_config.py 3 > $OUT/config3.json 2>&1
timeout 600 python scripts/run_config.py 2 --cpr > $OUT/cpr.json 2>&1
# launch list of the bench command itself (one step, shares comparable with the bench's phases)
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
