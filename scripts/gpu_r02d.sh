#!/bin/bash
# Round-2 GPU session D: PDL + graph capture, blocked claim order restored.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py tests/test_gpu_parity.py > $OUT/pytest_d1.log 2>&1; tail -4 $OUT/pytest_d1.log
timeout 600 python bench.py --no-sweep --no-e2e --no-cpu-baseline > $OUT/bench_d.json 2> $OUT/bench_d.err; tail -3 $OUT/bench_d.err; head -c 1000 $OUT/bench_d.json; echo
timeout 600 python scripts/small_sizes.py > $OUT/small_d.json 2> $OUT/small_d.err; tail -3 $OUT/small_d.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_d.csv \
   python bench.py --n 8192 --lam 0.99 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
