#!/bin/bash
TAG=${1:-ab26}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -20 $OUT/smoke.log; exit 1; }
tail -1 $OUT/smoke.log
bash scripts/gpu_abflags.sh $TAG scripts/ab_variants.txt
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
PARITY_LOG=$OUT/parity.json timeout 1200 python -m pytest tests/test_gpu_full.py -x -q -k "config5" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
