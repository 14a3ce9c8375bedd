#!/bin/bash
# Round-2 GPU session R: light side-stream zero-fill (1 / 2 / 4 warps per SM, LSU stores).
OUT=gpurun_out/r02r
mkdir -p $OUT
for pass in 1 2; do
for W in 0 1 2 4; do
  if [ $W = 0 ]; then F=""; else F="-DSPAMM_ZF_SIDE=$W"; fi
  SPAMM_NVCC_FLAGS="$F" python -m paper_2103_13042_b200.build --force > /dev/null
  for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99"; do
    timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
    python -c "import json; d=json.load(open('$OUT/b.json')); print('W=$W', d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
  done
done
done
SPAMM_NVCC_FLAGS="-DSPAMM_ZF_SIDE=2" python -m paper_2103_13042_b200.build --force > /dev/null
timeout 600 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_parity.py > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
python -m paper_2103_13042_b200.build --force > /dev/null
