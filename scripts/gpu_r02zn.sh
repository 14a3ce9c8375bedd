#!/bin/bash
# Round-2 GPU session ZN: norm-kernel grid of 16 boxes per CTA when 8 would leave a nearly empty
# second wave (N = 8192 BF16): parity and stage times.
OUT=gpurun_out/r02zn
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_sweeps.py -k "norm or 8192 or toeplitz" > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
for cfg in "--n 8192 --lam 0.99" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99 --precision fp32x3"; do
  timeout 300 python bench.py $cfg --steps 10 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print(d['config']['N'], d['config']['precision'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d.get('roofline_norms',{}).get('frac'))"
done
