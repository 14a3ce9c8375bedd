#!/bin/bash
for m in 0; do
  echo "mode $m"
  SPAMM_DEBUG_UMMA_MODE=$m timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms'])"
done
