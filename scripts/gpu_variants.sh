#!/bin/bash
# multiply-kernel scheduling experiments at the bench point (stage times, 50 steps each)
python -m paper_2103_13042_b200.build > /dev/null
run() { echo -n "$1: "; env $2 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,1), {k: round(v*1e3,1) for k,v in d['stages_ms'].items()})"; }
run "default (dynamic LPT, empty tiles via pipeline)" "X=1"
run "dynamic, epilogue zero-fill in waits         " "SPAMM_DEBUG_UMMA_MODE=32"
run "stream-K weighted, zero-fill in waits         " "SPAMM_STREAMK=1"
run "default variant 1                            " "SPAMM_UMMA_VARIANT=1"
