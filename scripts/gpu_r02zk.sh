#!/bin/bash
# Round-2 GPU session ZK: unroll depth of the SIMT k-slice loop (i-cache: the fully unrolled body
# is ~35 KB of SASS).
for u in 1 2 4 8; do
  SPAMM_NVCC_FLAGS=-DSPAMM_SIMT_QUNROLL=$u python -m paper_2103_13042_b200.build --force > /dev/null
  for t in 1e-10 1e-6; do echo "unroll $u"; python scripts/one_run.py 16384 0.99 $t fp32 3; done
  python scripts/one_run.py 1024 0.99 1e-4 fp32 5
done
