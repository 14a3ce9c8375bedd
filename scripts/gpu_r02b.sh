#!/bin/bash
# Round-2 GPU session B: parity after the pyramid skip map / device partition refactor.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
timeout 180 python __graft_entry__.py smoke > $OUT/smoke_b.log 2>&1; tail -4 $OUT/smoke_b.log
timeout 900 python -m pytest tests -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py tests/test_gpu_tausearch.py > $OUT/pytest_b1.log 2>&1; tail -15 $OUT/pytest_b1.log
timeout 600 python bench.py --no-sweep --no-e2e --no-cpu-baseline > $OUT/bench_b.json 2> $OUT/bench_b.err; tail -3 $OUT/bench_b.err; head -c 900 $OUT/bench_b.json
timeout 1500 python -m pytest tests -q -m gpu tests/test_gpu_sweeps.py tests/test_gpu_configs.py > $OUT/pytest_b2.log 2>&1; tail -15 $OUT/pytest_b2.log
