#!/bin/bash
# One gpurun round trip: GPU parity tests, a short bench, the ncu launch list and
# one `ncu --set full` capture of the sweep and cycle kernels.  Output under gpurun_out/.
# usage: gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python scripts/profile_step.py > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep|k_res|k_prolong|k_jacobi|k_gemv" -c 6 -o $OUT/full \
    python scripts/profile_step.py > $OUT/ncu_full.log 2>&1
fi
echo done
