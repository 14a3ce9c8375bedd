#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_r01s.log 2>&1; tail -3 $OUT/pytest_gpu_r01s.log
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
