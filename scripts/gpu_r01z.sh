#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DUAL_ORDER=2 SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
for o in 1 2; do echo "order $o"; SPAMM_DUAL_ORDER=$o timeout 600 python scripts/suite.py --configs 5 --precs bf16 --reps 2 --out $OUT/suite_o$o.json 2>&1 | grep -o '"tau": [0-9e.-]*\|"ms": [0-9.]*\|"multiply_roofline_frac": [0-9.]*' | paste - - - ; done
