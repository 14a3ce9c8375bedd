#!/bin/bash
# skip-map kernel: stage times + one ncu --set full capture
timeout 300 python bench.py --no-sweep --no-cpu-baseline --no-e2e --steps 100 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['stages_ms'])"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"skip_fused|tile_norms" -s 4 -c 2 -o gpurun_out/prof_skip -f \
   python bench.py --steps 1 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > /dev/null 2>&1
