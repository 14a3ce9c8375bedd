#!/bin/bash
# One GPU session: smoke, bench line, reference arm, ncu launch list, ncu --set full of the top kernels.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build
timeout 120 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; tail -3 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err
timeout 300 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu_launch_bench.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_umma -s 3 -c 1 -o $OUT/prof_umma -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_norms|skip_" -s 4 -c 2 -o $OUT/prof_norms_skip -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_simt -s 3 -c 1 -o $OUT/prof_simt -f \
   python bench.py --precision fp32 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
