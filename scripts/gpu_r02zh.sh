#!/bin/bash
# Round-2 GPU session ZH: per-k-step cost of the 128 x 128 kernel vs the number of CTAs (N = 1024: 64,
# N = 1536: 144) -- is the k-step bound per CTA or by CTAs sharing operand strips?
SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024:0.99 n1536:0.99 n1536:0.999; do timeout 120 python scripts/small_one.py $w 2>&1 | tail -3; done
