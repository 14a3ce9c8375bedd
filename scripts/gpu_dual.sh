#!/bin/bash
# variant 5 (256x256 two-issuer tensor multiply): parity, stage times vs variant 0, ncu capture
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_variants.py -x -q > $OUT/pytest_variants.log 2>&1; tail -15 $OUT/pytest_variants.log
B="python bench.py --no-sweep --no-cpu-baseline --no-e2e"
for v in 0 1 5; do echo "variant $v"; SPAMM_UMMA_VARIANT=$v timeout 300 $B --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'], d.get('clocks'))"; done
SPAMM_UMMA_VARIANT=5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spamm_mul_dual -s 3 -c 1 -o $OUT/prof_dual -f $B --steps 1 --warmup 3 > /dev/null 2>&1
ncu -i $OUT/prof_dual.ncu-rep --page raw --csv > $OUT/prof_dual_raw.csv 2>/dev/null; ls -la $OUT/prof_dual*
