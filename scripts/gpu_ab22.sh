#!/bin/bash
TAG=${1:-ab22}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1 || { tail -20 $OUT/smoke.log; exit 1; }
tail -1 $OUT/smoke.log
PARITY_LOG=$OUT/parity.json timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -k "cycle or config2 or config4 or config5 or error or zero or fixed or reproducib or import" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
printf -- "-\n-DMSB_NOCHAIN\n-\n-DMSB_NOCHAIN\n" > $OUT/variants.txt
bash scripts/gpu_abflags.sh $TAG $OUT/variants.txt
