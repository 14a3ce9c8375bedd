#!/bin/bash
# Round-2 GPU session F: multiply experiments at N = 65536 / 16384 / 8192 -- L2 prefetch distance of
# the operand boxes (build-time -DSPAMM_PF_DIST), zero-fill on a side stream (-DSPAMM_ZF_SIDE), and the
# per-CTA issuer counters (-DSPAMM_PROFILE).
OUT=gpurun_out/r02f
mkdir -p $OUT
run() {  # $1 = tag, $2 = nvcc flags
  SPAMM_NVCC_FLAGS="$2" python -m paper_2103_13042_b200.build --force > /dev/null
  for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99"; do
    timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/$1.json 2>/dev/null
    python -c "import json; d=json.load(open('$OUT/$1.json')); print('$1', d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
  done
}
run base ""
run zfside "-DSPAMM_ZF_SIDE"
run pf4 "-DSPAMM_PF_DIST=4"
run pf8 "-DSPAMM_PF_DIST=8"
run pf16 "-DSPAMM_PF_DIST=16"
run zfside_pf8 "-DSPAMM_ZF_SIDE -DSPAMM_PF_DIST=8"
run base2 ""
SPAMM_NVCC_FLAGS="-DSPAMM_PROFILE" python -m paper_2103_13042_b200.build --force > /dev/null
timeout 300 python scripts/prof_n65536.py 1e-6 > $OUT/prof_counters_65536.log 2>&1; tail -6 $OUT/prof_counters_65536.log
for n in 8192 16384; do
  timeout 300 python bench.py --n $n --lam 0.99 --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2> $OUT/prof_counters_$n.log; tail -5 $OUT/prof_counters_$n.log
done
python -m paper_2103_13042_b200.build --force > /dev/null
