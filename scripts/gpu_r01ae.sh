#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "water or config4" 2>&1 | tail -1
timeout 900 python scripts/suite.py --configs 4a --precs bf16 --reps 3 --out $OUT/suite_4a.json 2>&1 | grep -o '"valid_ratio": [0-9.]*\|"ms": [0-9.]*\|"multiply_roofline_frac": [0-9.]*' | paste - - -
