#!/bin/bash
# per-role cycle counters of the tensor multiply (SPAMM_DEBUG_UMMA_PROF) at the bench point
python -m paper_2103_13042_b200.build > /dev/null
for v in 0 1; do
echo "variant $v"
SPAMM_UMMA_VARIANT=$v SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -4
SPAMM_UMMA_VARIANT=$v timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"
done
