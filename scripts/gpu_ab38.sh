#!/bin/bash
TAG=${1:-ab38}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for flags in "-" "-DMSB_NO_WAVE" "-" "-DMSB_NO_WAVE"; do
  f=$flags; [ "$f" = "-" ] && f=""
  MSB_EXTRA_NVCC_FLAGS="$f" timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
  echo "== $flags" >> $OUT/config3.txt
  for i in 1 2; do timeout 300 python scripts/run_config.py 3 2>&1 | cut -c1-330 >> $OUT/config3.txt; done
done
cat $OUT/config3.txt
