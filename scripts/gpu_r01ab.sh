#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -x -k "65536" 2>&1 | tail -2
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python scripts/prof_n65536.py 1e-6 2>&1 | grep "dual prof\] issuer 0\|dual tl\|kept" | tail -3
timeout 900 python scripts/suite.py --configs 5 --precs bf16,fp32x3 --reps 2 --out $OUT/suite_c5.json 2>&1 | grep -o '"precision": "[a-z0-9]*"\|"valid_ratio": [0-9.]*\|"ms": [0-9.]*\|"multiply_roofline_frac": [0-9.]*' | paste - - - -
