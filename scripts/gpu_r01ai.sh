#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32x3" 2>&1 | tail -1
timeout 300 python bench.py --precision fp32x3 --no-sweep --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
timeout 900 python scripts/suite.py --configs 3,5 --precs fp32x3 --reps 2 --out /tmp/s.json 2>&1 | grep -o '"config": "[^"]*"\|"valid_ratio": [0-9.]*\|"ms": [0-9.]*' | paste - - - 
