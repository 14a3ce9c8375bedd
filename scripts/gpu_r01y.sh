#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_r01y.log 2>&1; tail -2 $OUT/pytest_gpu_r01y.log
for pr in bf16 fp32x3; do timeout 300 python bench.py --precision $pr --no-sweep --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['dtype'], d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
