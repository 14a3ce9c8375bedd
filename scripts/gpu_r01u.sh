#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for cfg in "1 0" "2 0" "2 1" "2 2" "2 1000"; do set -- $cfg; echo "ef $1 zf $2"; SPAMM_DUAL_ZF_EF=$1 SPAMM_DUAL_ZF=$2 timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
