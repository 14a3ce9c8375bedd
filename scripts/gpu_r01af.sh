#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for o in 1 2; do echo "order $o"; SPAMM_DUAL_ORDER=$o timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
for o in 1 2; do echo "order $o N=16384 exp"; SPAMM_DUAL_ORDER=$o timeout 600 python scripts/suite.py --configs 2 --precs bf16 --reps 3 --out /tmp/s.json 2>&1 | grep -o '"config": "[^"]*"\|"valid_ratio": [0-9.]*\|"ms": [0-9.]*' | paste - - - | tail -6; done
