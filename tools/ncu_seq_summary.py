"""Summarise the `ncu --set full` capture of bench.py's headline step (tools/prof_seq.py:
the 4 decode launches of one layer step -- qkv, o, gate_up, down) into
profiles/<tag>_seq_ncu.md (runs HERE over gpurun_out/).

    python tools/ncu_seq_summary.py --rep gpurun_out/prof_seq_r2c.ncu-rep --tag r2"""
import argparse
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_program_summary import SCALE, WANT, stalls  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]


def alg_bytes(m, n, k):
    return n * k // 2 + 4 * n + 2 * m * k + 2 * m * n + 4 * m


ap = argparse.ArgumentParser()
ap.add_argument("--rep", required=True)
ap.add_argument("--tag", default="r2")
ap.add_argument("--m", type=int, default=16)
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]


def val(r, metric):
    i = hdr.index(metric)
    v = float(r[i].replace(",", ""))
    u = units[i]
    if u in SCALE:
        return v * SCALE[u]
    if u == "ns":
        return v * 1e-3
    if u == "usecond":
        return v
    if u == "msecond":
        return v * 1e3
    return v


lines = [f"# Headline step, ncu --set full ({args.tag})", "",
         f"Command: `ncu --set full --clock-control none --import-source on -k regex:w4a8_decode_dyn -s 4 -c 4 "
         f"python tools/prof_seq.py` -- the 4 decode launches of ONE step of bench.py's headline (the LLaMA-13B "
         f"layer as 4 dependent launches at M={args.m}: act quant + one-linear w4a8_decode_dyn_kernel each; only "
         f"the decode kernels are captured).  Serialised, cold L2, unlocked clocks: compare bytes and shares, "
         f"not absolute times.", ""]
cols = ["linear", "alg MB"] + [name for _, name in WANT if name not in ("grid", "block")] + ["grid"]
lines.append("| " + " | ".join(cols) + " |")
lines.append("|" + "---|" * len(cols))
tot_dram = tot_alg = 0.0
for (name, n, k), r in zip(LAYERS, data):
    a = alg_bytes(args.m, n, k)
    cells = [name, f"{a / 1e6:.2f}"]
    dr = 0.0
    for metric, label in WANT:
        if label in ("grid", "block"):
            continue
        try:
            v = val(r, metric)
        except (ValueError, IndexError):
            cells.append("-")
            continue
        if label.startswith("DRAM read") or label.startswith("DRAM write"):
            dr += v
        if "bytes" in metric or label == "L2 traffic":
            cells.append(f"{v / 1e6:.2f} MB")
        elif label == "duration":
            cells.append(f"{v:.2f} us")
        else:
            cells.append(f"{v:.1f}")
    cells.append(r[hdr.index("launch__grid_size")])
    tot_dram += dr
    tot_alg += a
    lines.append("| " + " | ".join(cells) + " |")
lines += ["", f"DRAM read+write over the 4 launches: {tot_dram / 1e6:.2f} MB against {tot_alg / 1e6:.2f} MB "
          f"algorithmic ({tot_dram / tot_alg:.3f} x): every weight byte is fetched once.", ""]
st = stalls(args.rep)
if st:
    lines += ["Top warp-stall reasons (source page, all 4 launches):", "", "| reason | samples | share |", "|---|---|---|"]
    lines += [f"| {k} | {v} | {s:.1%} |" for k, v, s in st]
path = os.path.join(ROOT, "profiles", f"{args.tag}_seq_ncu.md")
open(path, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
