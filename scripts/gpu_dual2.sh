#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=0,1,2,4,5 timeout 600 python -m pytest tests/test_gpu_variants.py -q > $OUT/pytest_variants.log 2>&1; tail -5 $OUT/pytest_variants.log
SPAMM_TEST_VARIANTS=3 timeout 600 python -m pytest tests/test_gpu_variants.py -q 2>&1 | grep -E "passed|failed|FAILED" | head -30
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e"
SPAMM_UMMA_VARIANT=5 SPAMM_DEBUG_UMMA_PROF=1 timeout 300 $B --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -3
