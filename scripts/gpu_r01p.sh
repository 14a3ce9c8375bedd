#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -3
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for sp in 0 28 60; do echo "split $sp"; SPAMM_DUAL_SPLIT=$sp timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
for sp in 0 28; do SPAMM_DUAL_SPLIT=$sp SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 2 --warmup 3 2>&1 | grep "dual tl" | tail -1; done
