#!/bin/bash
# Round-2 final GPU session 3 (after the SIMT fused skip map): the committed state -- smoke, the whole GPU suite, the default bench line
# (configs[4] + sweeps incl. configs[2]) and the reference arm, the ncu launch list of the bench, ncu
# --set full of the headline multiply, small sizes.
OUT=gpurun_out/r02final3
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv
timeout 180 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; tail -4 $OUT/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; tail -4 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err; head -c 400 $OUT/bench.json; echo
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; head -c 300 $OUT/bench_ref.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual_65536 -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_dual65.log 2>&1; echo "ncu dual rc=$?"
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err
ls $OUT
