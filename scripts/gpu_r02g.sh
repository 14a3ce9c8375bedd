#!/bin/bash
# Round-2 GPU session G: warp-per-macro-tile skip map with list-based claim order; side-stream zero-fill.
OUT=gpurun_out/r02g
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1200 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py tests/test_gpu_tausearch.py tests/test_gpu_conv.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
run() {  # $1 = tag, $2 = nvcc flags
  SPAMM_NVCC_FLAGS="$2" python -m paper_2103_13042_b200.build --force > /dev/null
  for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99"; do
    timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/$1.json 2> $OUT/$1.err
    python -c "import json; d=json.load(open('$OUT/$1.json')); print('$1', d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
    grep -h "skip prof\|dual tl" $OUT/$1.err | tail -2
  done
}
run base ""
run zfside "-DSPAMM_ZF_SIDE"
run prof "-DSPAMM_PROFILE"
run prof_zf "-DSPAMM_PROFILE -DSPAMM_ZF_SIDE"
run base2 ""
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_sweeps.py tests/test_gpu_configs.py > $OUT/pytest2.log 2>&1; tail -3 $OUT/pytest2.log
