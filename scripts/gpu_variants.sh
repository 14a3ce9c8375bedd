#!/bin/bash
# multiply-kernel experiments at the bench point (stage times, 50 steps each)
python -m paper_2103_13042_b200.build > /dev/null
run() { echo -n "$1: "; env $2 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"; }
run "B 128-byte rows (default)" "X=1"
run "B 64-byte rows, 3-D      " "SPAMM_UMMA_BMODE=1"
run "B128 variant 1 (64-deep) " "SPAMM_UMMA_VARIANT=1"
run "B128 stream-K            " "SPAMM_STREAMK=1"
