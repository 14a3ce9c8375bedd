#!/bin/bash
# Round-2 GPU session A: FFMA peak, smoke, full GPU tests, N=65536 bench line, reference arm,
# ncu launch list and --set full captures at the sizes that matter (N=65536, N=16384).
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe_ffma scripts/probe_ffma.cu && ./scripts/probe_ffma > $OUT/ffma_peak.json
cat $OUT/ffma_peak.json
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used,memory.total --format=csv
timeout 180 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; tail -4 $OUT/smoke.log
timeout 1800 python -m pytest tests -q -m gpu -p no:randomly > $OUT/pytest_gpu.log 2>&1; tail -15 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err; head -c 1500 $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skip_fused|tile_norms" -s 6 -c 2 -o $OUT/prof_ns_65536 -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_ns.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual_16384 -f \
   python bench.py --n 16384 --lam 0.99 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_dual16.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual_65536 -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_dual65.log 2>&1
ls -la $OUT
