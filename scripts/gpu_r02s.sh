#!/bin/bash
# Round-2 GPU session S: small-problem launch lists; sanitizer test.
OUT=gpurun_out/r02s
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024 conv21 conv31; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$w.csv python scripts/small_one.py $w > /dev/null 2>&1
  python scripts/ncu_summary.py --launches $OUT/launches_$w.csv --tag r02s_$w | tail -7
done
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_sanitizers.py > $OUT/pytest_san.log 2>&1; tail -3 $OUT/pytest_san.log
