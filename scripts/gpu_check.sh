#!/bin/bash
# One gpurun round trip: smoke, GPU parity tests, a short bench, the ncu launch list and
# one `ncu --set full` capture of the hot kernels.  Output under gpurun_out/<tag>/.
# usage: gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag]
#   SKIP_NCU=1   skip both ncu passes;  SKIP_TESTS=1  skip pytest
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1
rc=$?; echo "smoke rc=$rc" >> $OUT/smoke.log
if [ $rc -ne 0 ]; then echo "smoke failed"; exit 1; fi
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 900 python bench.py --steps 3 --warmup 3 > $OUT/bench.log 2>&1
rc=$?; echo "bench rc=$rc" >> $OUT/bench.log
if [ $rc -ne 0 ]; then echo "bench failed"; exit 1; fi
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 300 python scripts/profile_step.py > $OUT/profile_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"${NCU_KERNELS:-k_sweep|k_restrict|k_prolong|k_jacobi|k_gemv|k_residual}" -c ${NCU_COUNT:-8} \
      -o $OUT/full python scripts/profile_step.py > $OUT/ncu_full.log 2>&1
fi
echo done
