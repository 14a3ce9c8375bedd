#!/bin/bash
# end-of-session check of the committed state: all GPU tests, smoke, bench line
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_r01i.log 2>&1; tail -1 $OUT/pytest_gpu_r01i.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r01i.log 2>&1; tail -3 $OUT/smoke_r01i.log
timeout 900 python bench.py > $OUT/bench_r01i.json 2> $OUT/bench_r01i.err; python -c "import json; d=json.load(open('$OUT/bench_r01i.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'])"
