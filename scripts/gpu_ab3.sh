#!/bin/bash
TAG=${1:-ab3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 300 python scripts/run_config.py 3 > $OUT/config3.json 2>&1
PARITY_LOG=$OUT/parity_dyn.json timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "dynamic or cycle or constant or fgmres or config3" > $OUT/pytest_dyn.log 2>&1; echo "rc=$?" >> $OUT/pytest_dyn.log
timeout 600 python scripts/run_config.py 2 --cpr > $OUT/cpr_config2.json 2>&1
for E in "MSB_AB_NOFUSE=0" "MSB_AB_NOFUSE=1"; do
  echo "== $E" >> $OUT/config5.txt
  if [ "$E" = "MSB_AB_NOFUSE=0" ]; then timeout 600 python scripts/run_config.py 5 >> $OUT/config5.txt 2>&1; else env $E timeout 600 python scripts/run_config.py 5 >> $OUT/config5.txt 2>&1; fi
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench.log 2>&1
cat $OUT/config3.json $OUT/cpr_config2.json; tail -2 $OUT/pytest_dyn.log
