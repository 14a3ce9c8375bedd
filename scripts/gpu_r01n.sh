#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DEBUG_UMMA_PROF=1 SPAMM_DEBUG_UMMA_PROF_CTA=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 1 --warmup 3 > /dev/null 2> $OUT/dual_cta.log; grep "tiles:" $OUT/dual_cta.log | tail -8
