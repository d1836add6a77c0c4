#!/bin/bash
TAG=${1:-ab29}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -20 $OUT/smoke.log; exit 1; }
tail -1 $OUT/smoke.log
for i in 1 2 3; do timeout 300 python scripts/run_config.py 3 >> $OUT/config3.json 2>&1; done
cat $OUT/config3.json | cut -c1-330
PARITY_LOG=$OUT/parity.json timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "dynamic or config3 or split or static or general or repro" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -4 $OUT/pytest.log
bash scripts/gpu_abflags.sh $TAG scripts/ab_variants.txt
