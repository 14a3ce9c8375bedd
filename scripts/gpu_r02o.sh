#!/bin/bash
# Round-2 GPU session O: rectangular super-blocks R x C of the many-tile claim order (two passes).
OUT=gpurun_out/r02o
mkdir -p $OUT
for pass in 1 2; do
for RC in "6 1" "4 1" "8 1" "12 1" "16 1" "6 2" "10 1"; do
  set -- $RC
  SPAMM_NVCC_FLAGS="-DSPAMM_ORD_R=$1 -DSPAMM_ORD_C=$2" python -m paper_2103_13042_b200.build --force > /dev/null
  timeout 300 python bench.py --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print('R=$1 C=$2', round(d['ms_per_step'],3), round(d['stages_ms']['multiply'],3), d['clocks']['sm_mhz'], round(d['stages_ms']['multiply']*d['clocks']['sm_mhz']/1000,1))"
done
done
python -m paper_2103_13042_b200.build --force > /dev/null
