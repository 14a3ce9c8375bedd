#!/bin/bash
# Round-2 GPU session V: timeline of the 128 x 128 BF16 kernel on configs[0] (-DSPAMM_PROFILE build).
OUT=gpurun_out/r02v
mkdir -p $OUT
SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024:0.99 n1024:0.9; do
  echo "== $w"; timeout 120 python scripts/small_one.py $w 2>&1 | tail -3
done
python -m paper_2103_13042_b200.build --force > /dev/null
