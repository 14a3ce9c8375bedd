#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for z in 0 1 2 1000; do echo "zf $z"; SPAMM_DUAL_ZF=$z timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
echo "no zero-fill"; SPAMM_DEBUG_DUAL_MODE=1 timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
for z in 1 2; do SPAMM_DUAL_ZF=$z SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>&1 | grep "dual tl" | tail -1; done
