#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5,5:1 timeout 900 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for w in 0 1; do echo "wide $w"; SPAMM_DUAL_WIDE=$w timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -3
