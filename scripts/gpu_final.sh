#!/bin/bash
# Short round-end check: smoke, full GPU suite, default bench, config 3 (no ncu passes).
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { echo smoke failed; tail $OUT/smoke.log; exit 1; }
PARITY_LOG=$OUT/parity_r02.json timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 300 python scripts/run_config.py 3 > $OUT/config3.json 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_reference.log 2>&1
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log; cut -c1-250 $OUT/config3.json
