#!/bin/bash
python -m paper_2103_13042_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tausearch.py -q -x 2>&1 | tail -1
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"
SPAMM_DEBUG_SKIP_PROF=1 timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep -i "skip prof" | tail -1
