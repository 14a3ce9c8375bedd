#!/bin/bash
# Round-2 GPU session ZJ: FP32 SIMT multiply with two C tiles per warp (8 x 8 register micro-tile,
# running sums in registers): parity, N = 16384 / 1024 timings, ncu.
OUT=gpurun_out/r02zj
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_mgpu_local.py tests/test_gpu_sweeps.py tests/test_gpu_configs.py tests/test_gpu_tausearch.py -k "fp32 and not fp32x3" > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
for t in 1e-10 1e-6 1e-2; do python scripts/one_run.py 16384 0.99 $t fp32 3; done
python scripts/one_run.py 1024 0.99 1e-4 fp32 5
python scripts/one_run.py 1024 0.9 1e-4 fp32 5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_simt -s 1 -c 1 -o $OUT/prof_simt_16384 -f python scripts/one_run.py 16384 0.99 1e-6 fp32 2 > $OUT/p1.log 2>&1; echo "simt rc=$?"
