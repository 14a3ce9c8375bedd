#!/bin/bash
# Round-end evidence: full bench line (with sweep, e2e, cpu baseline), reference arm, smoke,
# ncu launch list and --set full captures of the three stage kernels at the bench point.
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_final.log 2>&1; tail -3 $OUT/smoke_final.log
timeout 900 python bench.py > $OUT/bench_final.json 2> $OUT/bench_final.err; tail -2 $OUT/bench_final.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_final.json 2> $OUT/bench_ref_final.err
B="python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_final.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual_final -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tile_norms|skip_fused" -s 6 -c 2 -o $OUT/prof_ns_final -f $B > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_x3 -s 3 -c 1 -o $OUT/prof_x3_final -f python bench.py --precision fp32x3 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT/*final*
for r in prof_dual_final prof_ns_final prof_x3_final; do ncu -i $OUT/$r.ncu-rep --page source --csv > $OUT/${r}_source.csv 2>/dev/null; done
timeout 1200 python scripts/suite.py --reps 5 --out $OUT/suite_final.json > $OUT/suite_final.log 2>&1; tail -2 $OUT/suite_final.log
