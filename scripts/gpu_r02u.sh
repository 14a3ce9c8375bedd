#!/bin/bash
# Round-2 GPU session U: where the small-problem time goes (configs[0] N = 1024 BF16, lambda 0.9 / 0.99).
OUT=gpurun_out/r02u
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
for w in n1024:0.9 n1024:0.99; do
  t=${w/:/_}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"spamm_mul_x3|skip_pyr|tile_norms" -s 3 -c 3 \
     -o $OUT/prof_$t -f python scripts/small_one.py $w > $OUT/prof_$t.log 2>&1
  ncu -i $OUT/prof_$t.ncu-rep --page details --csv > $OUT/prof_$t.csv 2>/dev/null
  ncu -i $OUT/prof_$t.ncu-rep --page source --csv -k regex:spamm_mul_x3 > $OUT/src_mul_$t.csv 2>/dev/null
  ncu -i $OUT/prof_$t.ncu-rep --page source --csv -k regex:skip_pyr > $OUT/src_skip_$t.csv 2>/dev/null
done
ls -la $OUT
