#!/bin/bash
# r01e: full GPU suite with the 256x256 two-issuer kernel as the default tensor path, bench, suite
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_r01e.log 2>&1; tail -8 $OUT/pytest_gpu_r01e.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline'], d.get('clocks'))"
timeout 900 python scripts/suite.py --reps 5 --out $OUT/suite_r01e.json > $OUT/suite_r01e.log 2>&1; tail -5 $OUT/suite_r01e.log
