#!/bin/bash
OUT=gpurun_out
mkdir -p $OUT
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DUAL_ORDER=2 SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -1
for o in 1 2; do echo "order $o"; SPAMM_DUAL_ORDER=$o timeout 900 python scripts/suite.py --configs 5 --precs bf16 --reps 2 --out $OUT/suite_c5_o$o.json 2>&1 | grep -o '"valid_ratio": [0-9.]*\|"ms": [0-9.]*\|"multiply_roofline_frac": [0-9.]*' | paste - - -; done
