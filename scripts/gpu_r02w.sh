#!/bin/bash
# Round-2 GPU session W: 128 x 128 kernel changes (runs encoded by the producer, no TMEM chunking
# for one plane) -- parity of the affected paths, small-size timings, launch lists.
OUT=gpurun_out/r02w
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1200 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_parity.py tests/test_gpu_mgpu_local.py tests/test_gpu_conv.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err; tail -2 $OUT/small_sizes.err
python - <<'PY'
import json
for r in json.load(open("gpurun_out/r02w/small_sizes.json")):
    print(r["case"], r["precision"], "graph %.4f cublas %.4f x%.2f" % (r["graph_ms"], r["cublas_ms"], r["speedup_graph_vs_cublas"]), {k: round(v, 4) for k, v in r["stages_ms"].items()})
PY
for w in n1024:0.9 n1024:0.99; do
  t=${w/:/_}
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$t.csv python scripts/small_one.py $w > /dev/null 2>&1
  python scripts/ncu_summary.py --launches $OUT/launches_$t.csv --tag r02w_$t | tail -4
done
