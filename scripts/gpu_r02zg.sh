#!/bin/bash
# Round-2 GPU session ZG: FP32 SIMT with LDS and the original lane mapping (g = lane & 7).
python -m paper_2103_13042_b200.build --force > /dev/null
for t in 1e-10 1e-6 1e-2; do python scripts/one_run.py 16384 0.99 $t fp32 3; done
python scripts/one_run.py 1024 0.99 1e-4 fp32 5
