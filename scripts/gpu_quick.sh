#!/bin/bash
# quick check: GPU tests + bench stage times + tensor-kernel prof counters
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 400 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d.get('clocks'))"
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -2
