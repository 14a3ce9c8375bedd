#!/bin/bash
# Round-2 GPU session V1 (verification of the near-final state): smoke, the whole GPU suite, the
# default bench line + reference arm, the ncu launch list of the bench, small sizes.
OUT=gpurun_out/r02v1
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv
timeout 180 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; tail -4 $OUT/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; tail -4 $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err; head -c 400 $OUT/bench.json; echo
timeout 900 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; head -c 300 $OUT/bench_ref.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err
ls $OUT
