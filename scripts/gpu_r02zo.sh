#!/bin/bash
# Round-2 GPU session ZO: fused skip map in the FP32 SIMT kernel -- parity (fused vs staged bitwise,
# oracle), the FP32 suites, small sizes.
OUT=gpurun_out/r02zo
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 1800 python -m pytest -q -m gpu -x tests/test_gpu_fused.py tests/test_gpu_parity.py tests/test_gpu_mgpu_local.py tests/test_gpu_conv.py tests/test_gpu_dual.py > $OUT/pytest1.log 2>&1; tail -3 $OUT/pytest1.log
timeout 1800 python -m pytest -q -m gpu -x tests/test_gpu_sweeps.py tests/test_gpu_configs.py tests/test_gpu_tausearch.py -k "fp32" > $OUT/pytest2.log 2>&1; tail -3 $OUT/pytest2.log
timeout 600 python scripts/small_sizes.py > $OUT/small_sizes.json 2> $OUT/small_sizes.err; tail -2 $OUT/small_sizes.err
python - <<'PY'
import json
for r in json.load(open("gpurun_out/r02zo/small_sizes.json")):
    print(r["case"], r["precision"], "graph %.4f staged %.4f cublas %.4f x%.2f" % (r["graph_ms"], r["graph_staged_ms"], r["cublas_ms"], r["speedup_graph_vs_cublas"]))
PY
