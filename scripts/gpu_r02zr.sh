#!/bin/bash
# Round-2 GPU session ZR: zero-fill of empty macro-tiles interleaved with the accumulator waits using
# LSU stores (not the TMA engine the operand loads use), always vs the default (bulk, ratio >= 2).
OUT=gpurun_out/r02zr
mkdir -p $OUT
bench() {
  for cfg in "--n 8192 --lam 0.99" "--n 16384 --lam 0.99" "--n 65536 --lam 0.999" "--n 8192 --lam 0.99 --tau 1e-2"; do
    timeout 300 python bench.py $cfg --steps 8 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
    python -c "import json; d=json.load(open('$OUT/b.json')); print('$1', d['config']['N'], d['config']['tau'], round(d['ms_per_step'],4), round(d['stages_ms']['multiply'],4), d['clocks']['sm_mhz'])"
  done
}
python -m paper_2103_13042_b200.build --force > /dev/null
bench default
SPAMM_NVCC_FLAGS="-DSPAMM_ZF_LSU=1 -DSPAMM_ZF_RATIO=0" python -m paper_2103_13042_b200.build --force > /dev/null
bench lsu-always
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_dual.py -k "band or parity" > $OUT/pytest1.log 2>&1; tail -1 $OUT/pytest1.log
SPAMM_NVCC_FLAGS="-DSPAMM_ZF_LSU=1 -DSPAMM_ZF_RATIO=2" python -m paper_2103_13042_b200.build --force > /dev/null
bench lsu-ratio2
