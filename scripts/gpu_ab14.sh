#!/bin/bash
TAG=${1:-ab14}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail $OUT/smoke.log; exit 1; }
timeout 300 python scripts/run_config.py 3 > $OUT/config3.json 2>&1
timeout 300 python scripts/run_config.py 3 >> $OUT/config3.json 2>&1
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "dynamic or config3 or cycle or fgmres or constant or repro or error or singular" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
cat $OUT/config3.json; tail -3 $OUT/smoke.log; tail -2 $OUT/pytest.log
