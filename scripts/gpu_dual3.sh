#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -3
SPAMM_DUAL_PACK=1 SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e"
for cfg in "0 2" "5 1" "5 2"; do set -- $cfg; echo "variant $1 pack $2"; SPAMM_DUAL_PACK=$2 SPAMM_UMMA_VARIANT=$1 timeout 300 $B --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'], d.get('clocks'))"; done
SPAMM_UMMA_VARIANT=5 SPAMM_DEBUG_UMMA_PROF=1 timeout 300 $B --steps 3 --warmup 3 2>&1 | grep "prof\]" | tail -3
