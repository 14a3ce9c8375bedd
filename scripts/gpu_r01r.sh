#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for cfg in "0 10000" "3000 10000" "2000 10000" "4000 20000" "1500 5000" "6000 0"; do set -- $cfg; echo "pace $1 delay $2"; SPAMM_DUAL_ZF_PACE_NS=$1 SPAMM_DUAL_ZF_DELAY_NS=$2 timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>&1 | grep "dual tl" | tail -1
