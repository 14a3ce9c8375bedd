#!/bin/bash
# debug modes of the tensor multiply (SPAMM_DEBUG_UMMA_MODE bits): 1 no data MMAs,
# 2 no TMA loads, 4 no C stores, 8 no epilogue
for m in ${MODES:-0 1 2 3 4 8 11 15}; do
  echo "mode $m"
  SPAMM_DEBUG_UMMA_MODE=$m timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms'])"
  SPAMM_DEBUG_UMMA_PROF=1 SPAMM_DEBUG_UMMA_MODE=$m timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "umma prof" | tail -4
done
