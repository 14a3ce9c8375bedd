#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
for m in 0 1; do SPAMM_DEBUG_DUAL_MODE=$m SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>&1 | grep "dual tl\|dual prof\] issuer 0" | tail -2; done
