#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DUAL_ZF_CLAIM=4 SPAMM_TEST_VARIANTS=5 timeout 900 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
for c in 1 2 4 8; do echo "claim $c"; SPAMM_DUAL_ZF_CLAIM=$c timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
