#!/usr/bin/env python
"""Summarise ncu reports / launch lists into profiles/ (text + ncu_traffic.json).

  python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --tag r02a [--workload "<bench config.workload>"]
  python scripts/ncu_summary.py --launches gpurun_out/launches.csv --tag r01
"""
import argparse
import csv
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def to_bytes(val, unit):
    v = float(str(val).replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def summarise_rep(rep, tag, workload):
    rows, units = raw_rows(rep)
    lines = [f"# ncu --set full summary of {os.path.basename(rep)} ({tag})"]
    traffic = {}
    for r in rows:
        name = r.get("Kernel Name", "?")
        lines.append(f"\n## {name[:160]}")
        for k in KEYS:
            if k in r:
                lines.append(f"{k} = {r[k]} {units.get(k, '')}")
        if "dram__bytes_read.sum" in r and "dram__bytes_write.sum" in r:
            t = to_bytes(r["dram__bytes_read.sum"], units["dram__bytes_read.sum"]) + \
                to_bytes(r["dram__bytes_write.sum"], units["dram__bytes_write.sum"])
            lines.append(f"traffic (dram read+write) = {t:.4g} B")
            base = re.search(r"(\w+)(?:<[^()]*>)?\(", name)
            kname = base.group(1) if base else name
            key = "multiply" if "spamm_mul" in name else ("norms" if "tile_norms" in name else "skipmap_" + kname)
            traffic[key] = t   # one capture per kernel per step
    base = os.path.splitext(os.path.basename(rep))[0]
    with open(os.path.join(ROOT, "profiles", f"{tag}_{base}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(tp)) if os.path.exists(tp) else {}
    if workload:   # keyed by bench.py's config.workload string: the bench uses it only for that workload
        d.setdefault(workload, {}).update(traffic)
    json.dump(d, open(tp, "w"), indent=1)
    print("\n".join(lines[:40]))


def summarise_launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, iid = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID")
    recs = [(int(r[iid]), r[ik], float(r[iv].replace(",", ""))) for r in rows[hi + 1:] if len(r) > iv]
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none launch list ({tag}); ns per launch",
           "id,kernel,ns"]
    out += [f"{i},{k[:120].replace(',', ';')},{v:.0f}" for i, k, v in recs]
    # share of the last complete step (from the last tile_norms pair to the end)
    starts = [j for j, (_, k, _) in enumerate(recs) if "tile_norms" in k]
    if starts:
        step = recs[starts[-1]:]
        flush = lambda k: "FillFunctor" in k or "reduce_kernel" in k   # noqa: E731  (L2 flush write + read)
        tot = sum(v for _, k, v in step if not flush(k))
        out.append("\n# share of one step (L2-flush kernels excluded)")
        for _, k, v in step:
            if flush(k):
                continue
            out.append(f"{k.split('(')[0][:80]}: {v / 1e3:.1f} us ({100 * v / tot:.1f} %)")
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out[-12:]))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--workload", default=None, help="bench.py config.workload of the captured run")
    a = ap.parse_args()
    if a.rep:
        summarise_rep(a.rep, a.tag, a.workload)
    if a.launches:
        summarise_launches(a.launches, a.tag)
