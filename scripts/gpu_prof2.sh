#!/bin/bash
for m in 0 6 1 2; do
  echo "mode $m"
  SPAMM_DEBUG_UMMA_PROF=1 SPAMM_DEBUG_UMMA_MODE=$m timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "umma prof" | tail -2
done
