#!/bin/bash
TAG=${1:-ab11}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 600 python scripts/run_config.py 5 > $OUT/config5.json 2>&1
timeout 600 python scripts/run_config.py 5 >> $OUT/config5.json 2>&1
PARITY_LOG=$OUT/parity.json timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
grep -o '"ms_per_iteration": [0-9.]*' $OUT/config5.json; tail -2 $OUT/pytest.log
