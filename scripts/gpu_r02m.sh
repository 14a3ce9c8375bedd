#!/bin/bash
# Round-2 GPU session L: super-block side 2-7 (two passes), DRAM bytes of 3-5.
OUT=gpurun_out/r02m
mkdir -p $OUT
for pass in 1 2; do
for S in 6 5 4 3 2 7; do
  SPAMM_NVCC_FLAGS="-DSPAMM_ORD_S=$S" python -m paper_2103_13042_b200.build --force > /dev/null
  timeout 300 python bench.py --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b$S.json 2> $OUT/b$S.err
  python -c "import json; d=json.load(open('$OUT/b$S.json')); print('S=$S', d['config']['N'], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'], round(d['stages_ms']['multiply']*d['clocks']['sm_mhz']/1000,1))"
done
done
for S in 5 4 3; do
SPAMM_NVCC_FLAGS="-DSPAMM_ORD_S=$S" python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1500 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spamm_mul_dual -s 3 -c 1 \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu$S.log 2>&1; echo S=$S; grep -E "dram__bytes|duration|hit_rate" $OUT/ncu$S.log
done
python -m paper_2103_13042_b200.build --force > /dev/null
