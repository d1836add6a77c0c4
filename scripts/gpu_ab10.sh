#!/bin/bash
TAG=${1:-ab10}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 600 python scripts/run_config.py 5 > $OUT/config5.json 2>&1
timeout 600 python scripts/run_config.py 5 >> $OUT/config5.json 2>&1
timeout 300 python scripts/profile_step.py > $OUT/p_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ldl_inv_leaf|k_dgemm" -s 3 -c 6 \
    -o $OUT/leaf python scripts/profile_step.py > $OUT/ncu_leaf.log 2>&1
cat $OUT/config5.json | cut -c1-300
