#!/bin/bash
# Round-2 GPU session Z: fused small path with register-resident lists; ncu --set full of the 128 x 128
# kernel on configs[0] (N = 1024, lambda = 0.99 / 0.9) to find its limiter; per-CTA timeline.
OUT=gpurun_out/r02z
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_fused.py > $OUT/pytest1.log 2>&1; tail -2 $OUT/pytest1.log
for w in n1024:0.99 n1024:0.9; do
  t=${w/:/_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_x3 -s 2 -c 1 -o $OUT/prof_x1_$t -f python scripts/small_one.py $w > $OUT/prof_$t.log 2>&1; echo "ncu $t rc=$?"
done
SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024:0.9 n1024:0.99; do timeout 120 python scripts/small_one.py $w 2>&1 | tail -3; done
