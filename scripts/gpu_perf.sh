#!/bin/bash
# Perf experiment: smoke, bench with and without the L2-persisting coarse inverse, and one
# ncu --set full capture of the cycle kernels + sweep.  usage: bash scripts/gpu_perf.sh tag
TAG=${1:-perf}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { echo smoke failed; cat $OUT/smoke.log; exit 1; }
if [ "${RUN_TESTS:-0}" = "1" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "not config5" > $OUT/pytest.log 2>&1; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1
if [ -n "${BENCH2_ENV:-}" ]; then env $BENCH2_ENV timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench2.log 2>&1; fi
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 300 python scripts/profile_step.py > $OUT/profile_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_KERNELS:-k_restrict|k_prolong|k_jacobi|k_gemv|k_residual|k_sweep_tma}" -s ${NCU_SKIP:-20} -c ${NCU_COUNT:-7} \
      -o $OUT/full python scripts/profile_step.py > $OUT/ncu_full.log 2>&1
fi
echo done
