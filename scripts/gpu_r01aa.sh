#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
SPAMM_DEBUG_UMMA_PROF=1 timeout 300 python scripts/prof_n65536.py 1e-6 2>&1 | grep "dual prof\] issuer 0\|dual tl\|kept" | tail -3
