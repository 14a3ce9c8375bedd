#!/bin/bash
# Round-2 GPU session H: side-stream zero-fill with the SM carveout fix; skip-map ncu source capture.
OUT=gpurun_out/r02h
mkdir -p $OUT
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
run prof_zf "-DSPAMM_PROFILE -DSPAMM_ZF_SIDE"
run prof "-DSPAMM_PROFILE"
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_parity.py tests/test_gpu_dual.py tests/test_gpu_mgpu_local.py > $OUT/pytest1.log 2>&1; tail -2 $OUT/pytest1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"skip_pyr" -s 2 -c 1 -o $OUT/prof_skip_65536 -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/prof_skip.log 2>&1
ncu -i $OUT/prof_skip_65536.ncu-rep --page source --csv > $OUT/prof_skip_source.csv 2>/dev/null; ls -la $OUT | tail -3
