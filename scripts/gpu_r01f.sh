#!/bin/bash
# r01f: TMA ring probe, norm-kernel ring/box experiments, skip map with the bit-trick run encoder
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 120 ./scripts/probe_tma_rings > $OUT/probe_tma_rings.log 2>&1; cat $OUT/probe_tma_rings.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -2
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200"
for cfg in "4 8" "2 8" "2 16" "3 8" "3 16" "4 16" "2 4"; do set -- $cfg; echo "norm stages $1 bpc $2"; SPAMM_NORM_STAGES=$1 SPAMM_NORM_BPC=$2 timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'])"; done
SPAMM_DEBUG_SKIP_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep -i "skip prof" | tail -2
