#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>&1 | grep "dual tl\|dual prof\] issuer 0" | tail -2
