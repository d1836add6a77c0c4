#!/bin/bash
TAG=${1:-ab4}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 300 python scripts/run_config.py 3 > $OUT/config3.json 2>&1
for E in A B A B; do
  if [ $E = A ]; then echo "== fused" >> $OUT/config5.txt; timeout 600 python scripts/run_config.py 5 >> $OUT/config5.txt 2>&1;
  else echo "== NOFUSE" >> $OUT/config5.txt; MSB_AB_NOFUSE=1 timeout 600 python scripts/run_config.py 5 >> $OUT/config5.txt 2>&1; fi
done
timeout 300 python scripts/profile_step.py 5 12 > $OUT/p5_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_symv_tiles_b|k_symv_reduce_b|k_schur_t|k_schur_u|k_restrict_cart|k_prolong_cart" -s 60 -c 8 \
    -o $OUT/c5schur python scripts/profile_step.py 5 12 > $OUT/ncu_c5.log 2>&1
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cpr.py -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.log 2>&1
cat $OUT/config3.json; grep -h "ms_per_iteration" $OUT/config5.txt | cut -c1-60; tail -2 $OUT/pytest.log
