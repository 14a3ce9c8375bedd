#!/bin/bash
# multiply-kernel variants at the bench point (stage times, 50 steps each)
python -m paper_2103_13042_b200.build > /dev/null
run() { echo -n "$1: "; env $2 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"; }
run "variant 0 (2 CTAs/SM)            " "SPAMM_UMMA_VARIANT=0"
run "variant 4 (1 CTA/SM split, 32)   " "SPAMM_UMMA_VARIANT=4"
run "variant 2 (1 CTA/SM split, 64)   " "SPAMM_UMMA_VARIANT=2"
run "variant 1 (2 CTAs/SM, 64)        " "SPAMM_UMMA_VARIANT=1"
