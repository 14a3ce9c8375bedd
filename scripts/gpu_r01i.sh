#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for m in 0 1 2 3; do echo "dual dbg $m"; SPAMM_DEBUG_DUAL_MODE=$m timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"; done
for m in 1 3; do SPAMM_DEBUG_DUAL_MODE=$m SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -3; done
for p in 1 2; do echo "pack $p 7-stage test skipped"; done
