#!/bin/bash
# Round-2 GPU session ZL: bench sweep with the configs[2] algebraic Table-1 block.
OUT=gpurun_out/r02zl
mkdir -p $OUT
python -m paper_2103_13042_b200.build --force > /dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; tail -3 $OUT/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r02zl/bench.json"))
for r in d["sweep"]["points"]:
    print(r.get("workload"), r["N"], r["precision"], r["tau"], "%.4f ms vr %.4f" % (r["ms"], r["valid_ratio"]), "x%.2f" % r.get("speedup_vs_cublas", 0), r.get("multiply_roofline", {}).get("frac"))
print(d["sweep"]["cublas"])
PY
