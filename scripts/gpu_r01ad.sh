#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DUAL_ORDER=2 SPAMM_TEST_VARIANTS=5 timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -2
