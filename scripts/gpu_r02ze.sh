#!/bin/bash
# Round-2 GPU session ZE: ncu --set full of the mid-size multiplies below their rooflines:
# FP32 SIMT and FP32X3 at the north-star N = 16384 (lambda 0.99, tau 1e-6), BF16 dual at configs[1] N = 8192.
OUT=gpurun_out/r02ze
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
python scripts/one_run.py 16384 0.99 1e-6 fp32 2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_simt -s 1 -c 1 -o $OUT/prof_simt_16384 -f python scripts/one_run.py 16384 0.99 1e-6 fp32 2 > $OUT/p1.log 2>&1; echo "simt rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_x3 -s 1 -c 1 -o $OUT/prof_x3_16384 -f python scripts/one_run.py 16384 0.99 1e-6 fp32x3 2 > $OUT/p2.log 2>&1; echo "x3 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 1 -c 1 -o $OUT/prof_dual_8192 -f python scripts/one_run.py 8192 0.99 1e-6 bf16 2 > $OUT/p3.log 2>&1; echo "dual rc=$?"
