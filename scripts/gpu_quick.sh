#!/bin/bash
# quick check per tensor-path variant: parity subset + bench stage times + umma prof counters
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2}; do
  echo "== variant $v"
  export SPAMM_UMMA_VARIANT=$v
  timeout 400 python -m pytest tests -m gpu -x -q -k "spamm or macro or full" 2>&1 | tail -2
  timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 400 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d.get('clocks'))"
  SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "umma prof" | tail -2
done
