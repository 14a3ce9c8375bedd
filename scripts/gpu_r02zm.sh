#!/bin/bash
# Round-2 GPU session ZM: two k-steps per stage in the one-plane 128 x 128 kernel
OUT=gpurun_out/r02zm
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1500 python -m pytest -q -m gpu -x tests/test_gpu_fused.py tests/test_gpu_dual.py tests/test_gpu_parity.py tests/test_gpu_conv.py tests/test_gpu_mgpu_local.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err; tail -2 $OUT/small_sizes.err
python - <<'PY'
import json
for r in json.load(open("gpurun_out/r02zm/small_sizes.json")):
    print(r["case"], r["precision"], "graph %.4f staged %.4f cublas %.4f x%.2f" % (r["graph_ms"], r["graph_staged_ms"], r["cublas_ms"], r["speedup_graph_vs_cublas"]))
PY
SPAMM_NVCC_FLAGS=-DSPAMM_PROFILE python -m paper_2103_13042_b200.build --force > /dev/null
for w in n1024:0.9 n1024:0.99; do timeout 120 python scripts/small_one.py $w 2>&1 | tail -3; done
