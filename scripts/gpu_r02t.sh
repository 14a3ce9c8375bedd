#!/bin/bash
# Round-2 GPU session T: small-problem path (128 x 128 BF16 tiles, inline order, no pyramid for small K).
OUT=gpurun_out/r02t
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 180 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 1200 python -m pytest -q -m gpu -x tests/test_gpu_dual.py tests/test_gpu_parity.py tests/test_gpu_mgpu_local.py tests/test_gpu_conv.py tests/test_gpu_tausearch.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err; tail -2 $OUT/small_sizes.err
python - <<'PY'
import json
for r in json.load(open("gpurun_out/r02t/small_sizes.json")):
    print(r["case"], r["precision"], "graph %.4f cublas %.4f x%.2f" % (r["graph_ms"], r["cublas_ms"], r["speedup_graph_vs_cublas"]))
PY
for w in n1024 conv21; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$w.csv python scripts/small_one.py $w > /dev/null 2>&1
  python scripts/ncu_summary.py --launches $OUT/launches_$w.csv --tag r02t_$w | tail -6
done
for cfg in "--n 65536 --lam 0.999" "--n 16384 --lam 0.99" "--n 8192 --lam 0.99" "--n 2048 --lam 0.99"; do
  timeout 300 python bench.py $cfg --steps 6 --warmup 3 --no-sweep --no-e2e --no-cpu-baseline > $OUT/b.json 2> $OUT/b.err
  python -c "import json; d=json.load(open('$OUT/b.json')); print(d['config']['N'], round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms'].items()}, d['clocks']['sm_mhz'])"
done
timeout 1800 python -m pytest -q -m gpu tests/test_gpu_sweeps.py tests/test_gpu_configs.py tests/test_gpu_sanitizers.py > $OUT/pytest2.log 2>&1; tail -3 $OUT/pytest2.log
