#!/bin/bash
# Round-2 GPU session Q: LPT claim order keeps tile order within equal keys.
OUT=gpurun_out/r02q
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py > $OUT/pytest1.log 2>&1; tail -2 $OUT/pytest1.log
for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99"; do
  timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print(d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
done
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:spamm_mul_dual -s 3 -c 1 \
   python bench.py --n 16384 --lam 0.99 --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/ncu16.log 2>&1; grep -E "dram__bytes|duration" $OUT/ncu16.log
