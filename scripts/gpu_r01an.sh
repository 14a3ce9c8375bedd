#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "blocked" 2>&1 | tail -1
