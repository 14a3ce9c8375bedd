#!/bin/bash
# r01d re-entry check: GPU tests, bench stage times, multiply + skip-map debug counters
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r01d.log 2>&1; tail -3 $OUT/pytest_gpu_r01d.log
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 > $OUT/bench_quick_r01d.json 2>&1; tail -c 1500 $OUT/bench_quick_r01d.json
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -3
SPAMM_DEBUG_SKIP_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep -i "skip" | tail -5
for m in 1 2 4 8 7; do echo "dbg $m"; SPAMM_DEBUG_UMMA_MODE=$m timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms'])"; done
