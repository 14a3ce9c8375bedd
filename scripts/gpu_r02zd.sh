#!/bin/bash
# Round-2 GPU session ZD: producer-side counters of the 128 x 128 kernel (profile build only).
SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024:0.9 n1024:0.99; do timeout 120 python scripts/small_one.py $w 2>&1 | tail -3; done
