#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_X3_ORDER=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32x3" 2>&1 | tail -1
for o in 1 2; do echo "x3 order $o"; SPAMM_X3_ORDER=$o timeout 900 python scripts/suite.py --configs 5 --precs fp32x3 --reps 2 --out /tmp/s$o.json 2>&1 | grep -o '"valid_ratio": [0-9.]*\|"ms": [0-9.]*\|"multiply_roofline_frac": [0-9.]*' | paste - - -; done
