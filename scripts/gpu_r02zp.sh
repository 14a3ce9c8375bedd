#!/bin/bash
# Round-2 GPU session ZP: ring depth of the one-plane 128 x 128 kernel -- 4 stages + TMA-store staging
# (default) vs 6 stages with register-store epilogue; small sizes and a parity subset.
OUT=gpurun_out/r02zp
mkdir -p $OUT
for st in 6 4; do
  SPAMM_NVCC_FLAGS=-DSPAMM_X1_STAGES=$st python -m paper_2103_13042_b200.build --force > /dev/null
  echo "stages $st"
  timeout 900 python -m pytest -q -m gpu -x tests/test_gpu_fused.py -k "bf16 or fp16" > $OUT/pytest_$st.log 2>&1; tail -1 $OUT/pytest_$st.log
  timeout 600 python scripts/small_sizes.py > $OUT/small_sizes_$st.json 2> $OUT/small_sizes.err
  python - <<PY
import json
for r in json.load(open("gpurun_out/r02zp/small_sizes_$st.json")):
    if r["precision"] == "bf16": print(r["case"], "graph %.4f x%.2f" % (r["graph_ms"], r["speedup_graph_vs_cublas"]))
PY
done
