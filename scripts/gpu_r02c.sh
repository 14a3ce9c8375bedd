#!/bin/bash
# Round-2 GPU session C: kstart claim order + im2col entry; sanitizers; N=65536 bench and dual ncu.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py tests/test_gpu_conv.py tests/test_gpu_parity.py > $OUT/pytest_c1.log 2>&1; tail -5 $OUT/pytest_c1.log
timeout 600 python bench.py --no-sweep --no-e2e --no-cpu-baseline > $OUT/bench_c.json 2> $OUT/bench_c.err; tail -3 $OUT/bench_c.err; head -c 1200 $OUT/bench_c.json; echo
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > $OUT/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -4 $OUT/sanitize_$tool.log
done
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual_65536_c -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_dual65c.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skip_pyr|pyramid" -s 6 -c 2 -o $OUT/prof_skip_65536_c -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_skip65c.log 2>&1
ls $OUT | tail -3
