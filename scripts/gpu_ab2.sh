#!/bin/bash
# Development call: config-3 dynamic-stage timing A/B and its launch list.
TAG=${1:-ab2}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for E in "$@"; do
  echo "== $E" >> $OUT/config3.txt
  env $E timeout 300 python scripts/run_config.py 3 >> $OUT/config3.txt 2>&1
done
timeout 300 python scripts/probes/profile_config3.py > $OUT/c3_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/c3_launches.csv python scripts/probes/profile_config3.py > $OUT/ncu_c3.log 2>&1
PARITY_LOG=$OUT/parity_dyn.json timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "dynamic or cycle or constant or fgmres" > $OUT/pytest_dyn.log 2>&1; echo "rc=$?" >> $OUT/pytest_dyn.log
cat $OUT/config3.txt
