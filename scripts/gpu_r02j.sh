#!/bin/bash
# Round-2 GPU session I: row-major order inside super-blocks (rank from 144-bit masks).
OUT=gpurun_out/r02j
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py tests/test_gpu_tausearch.py > $OUT/pytest1.log 2>&1; tail -2 $OUT/pytest1.log
for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99"; do
  timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print(d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_65536.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_8192.csv \
   python bench.py --n 8192 --lam 0.99 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_sweeps.py tests/test_gpu_configs.py tests/test_gpu_conv.py > $OUT/pytest2.log 2>&1; tail -2 $OUT/pytest2.log
