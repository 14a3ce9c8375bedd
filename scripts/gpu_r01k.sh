#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5 timeout 900 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for z in 0 1 2 4 1000; do echo "zf per wait $z"; SPAMM_DUAL_ZF=$z timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"; done
