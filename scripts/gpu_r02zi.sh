#!/bin/bash
# Round-2 GPU session ZI: zero-fill of empty macro-tiles interleaved with the accumulator waits,
# evict-first bulk stores (SPAMM_ZF_INTERLEAVE=1) vs zero-fill last (=0): timings at N = 65536 /
# 16384 / 8192, parity of the dual kernel.
OUT=gpurun_out/r02zi
mkdir -p $OUT
bench() {
  for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99" "--n 16384 --lam 0.99 --tau 1e-2"; do
    timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
    python -c "import json; d=json.load(open('$OUT/b.json')); print('$1', d['config']['N'], d['config']['tau'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
  done
}
SPAMM_NVCC_FLAGS=-DSPAMM_ZF_INTERLEAVE=0 python -m paper_2103_13042_b200.build --force > /dev/null
bench last
python -m paper_2103_13042_b200.build --force > /dev/null
bench interleaved
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_configs.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
