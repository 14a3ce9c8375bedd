#!/bin/bash
# Round-2 GPU session ZQ: ncu --set full of the fused small-problem kernels on configs[0]
# (N = 1024, lambda = 0.99, tau = 1e-4): BF16 one-plane 128 x 128 kernel and FP32 SIMT.
OUT=gpurun_out/r02zq
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_x3 -s 2 -c 1 -o $OUT/prof_x1_n1024 -f python scripts/small_one.py n1024:0.99 > $OUT/p1.log 2>&1; echo "x1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_simt -s 2 -c 1 -o $OUT/prof_simt_n1024 -f python scripts/one_run.py 1024 0.99 1e-4 fp32 4 > $OUT/p2.log 2>&1; echo "simt rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_fp32.csv python scripts/one_run.py 1024 0.9 1e-4 fp32 4 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bf16.csv python scripts/small_one.py n1024:0.9 > /dev/null 2>&1
