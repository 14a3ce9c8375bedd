#!/bin/bash
# ncu captures of the current kernels at the bench point + launch list
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
B="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_umma -s 3 -c 1 -o $OUT/prof_umma_b -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_norms|skip_fused" -s 6 -c 2 -o $OUT/prof_ns_b -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_simt -s 3 -c 1 -o $OUT/prof_simt_b -f python bench.py --precision fp32 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_b.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT/*.ncu-rep $OUT/launches_b.csv
