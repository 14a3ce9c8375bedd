#!/bin/bash
# Round-end evidence (r01g): full GPU tests, smoke, bench line, reference arm, ncu launch list and
# --set full captures, all-config suite.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_final.log 2>&1; tail -2 $OUT/pytest_gpu_final.log
./scripts/gpu_final.sh
