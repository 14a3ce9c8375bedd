#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
timeout 300 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e > $OUT/bench_p.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_umma -s 3 -c 1 -o $OUT/prof_umma2 -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skip_ -s 6 -c 3 -o $OUT/prof_skip -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
