"""Summarise ncu captures into profiles/ (runs HERE, on the CPU box, over gpurun_out/).

    python tools/ncu_summary.py --rep gpurun_out/prof_gemm_r1.ncu-rep \
        --launches gpurun_out/launches_r1.csv --tag r1 --m 16

Writes profiles/<tag>_gemm_ncu.md (per-launch metrics of the FastGEMM for the four
LLaMA-13B layer shapes), profiles/<tag>_launches.md (the launch list of one bench run,
device time per kernel family and share) and profiles/ncu_gemm_traffic.json (the DRAM
bytes bench.py reports as roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = {(120, 15360): "qkv", (120, 5120): "o", (148, 27648): "gate_up"}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "Kbyte/block": 1e3}


def to_num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * SCALE.get(unit, 1)


def gemm_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = r[0], r[1], r[2:]
    res = []
    for row in rows:
        d = {"kernel": row[hdr.index("Kernel Name")], "grid": row[hdr.index("Grid Size")]}
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                d[w] = to_num(row[i], units[i])
                d[w + ".unit"] = units[i]
        res.append(d)
    return res


def layer_of(d, order):
    return order


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--m", type=int, default=16)
    args = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if args.rep:
        rows = gemm_rows(args.rep)
        names = ["qkv", "o", "gate_up", "down"]  # tools/prof_gemm.py launch order
        alg = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824)}
        m = args.m
        lines = [f"# FastGEMM ncu --set full, M={m} ({args.tag})", "",
                 "Command: `ncu --set full --clock-control none --import-source on -k regex:w4a8_gemm_kernel "
                 "-s 8 -c 4 python tools/prof_gemm.py` (one launch per LLaMA-13B layer shape, cold L2,"
                 " serialised -- compare bytes and shares, not absolute times).", "",
                 "| layer | grid | cluster | time us | DRAM read MB | DRAM write MB | algorithmic MB | DRAM/alg |"
                 " DRAM thr % | SM thr % | tensor % | regs | smem KB |",
                 "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
        tot_dram = tot_alg = 0.0
        per = {}
        for nm, d in zip(names, rows):
            n, k = alg[nm]
            a = n * k // 2 + m * k + 4 * n + 4 * m + 2 * m * n
            dr = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            tot_dram += dr
            tot_alg += a
            per[nm] = {"dram_bytes": dr, "algorithmic_bytes": a, "time_us": d.get("gpu__time_duration.sum")}
            lines.append(
                f"| {nm} | {d['grid']} | {d.get('launch__cluster_dim_x')} | {d.get('gpu__time_duration.sum'):.2f} | "
                f"{d.get('dram__bytes_read.sum', 0) / 1e6:.2f} | {d.get('dram__bytes_write.sum', 0) / 1e6:.3f} | "
                f"{a / 1e6:.2f} | {dr / a:.3f} | "
                f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                f"{d.get('launch__registers_per_thread')} | {d.get('launch__shared_mem_per_block_dynamic', 0) / 1e3:.1f} |")
        lines += ["", f"Sum over the 4 launches: DRAM {tot_dram / 1e6:.2f} MB vs algorithmic {tot_alg / 1e6:.2f} MB "
                  f"(ratio {tot_dram / tot_alg:.3f}): no weight byte is fetched twice; outputs stay in L2."]
        with open(os.path.join(prof, f"{args.tag}_gemm_ncu.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        tj = os.path.join(prof, "ncu_gemm_traffic.json")
        d = json.load(open(tj)) if os.path.exists(tj) else {}
        d[f"M{m}"] = round(tot_dram)  # bytes over one launch of each of the 4 layer GEMMs
        d[f"M{m}_per_layer"] = per
        d[f"M{m}_source"] = f"profiles/{args.tag}_gemm_ncu.md"
        with open(tj, "w") as f:
            json.dump(d, f, indent=1)
    if args.launches:
        rows = list(csv.reader(open(args.launches)))
        hdr = next(r for r in rows if "Kernel Name" in r)
        data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
        agg = collections.OrderedDict()
        for d in data:
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            nm = d["Kernel Name"].split("(")[0].replace("void ", "")
            key = (nm[:70], d.get("Grid Size", ""))
            scale = SCALE.get(d.get("Metric Unit", "ns"), 1)
            agg.setdefault(key, []).append(float(d["Metric Value"].replace(",", "")) * scale)
        ours = {k: v for k, v in agg.items() if "odyb200" in k[0]}
        tot = sum(sum(v) for v in ours.values())
        lines = [f"# Launch list of `python bench.py --steps 20 --warmup 3 --no-cpu` under ncu ({args.tag})", "",
                 "`ncu --metrics gpu__time_duration.sum --clock-control none -c 300` -- serialised, cold-cache"
                 " per-launch device times; only the SHARE of each kernel family is meaningful.", "",
                 "| kernel | grid | launches | mean us | share of our device time |", "|---|---|---|---|---|"]
        for (nm, grid), v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{nm}` | {grid} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v) / tot * 100:.1f}% |")
        other = {k: v for k, v in agg.items() if "odyb200" not in k[0]}
        lines += ["", f"Other (torch setup: RNG / casts / fills) launches: {sum(len(v) for v in other.values())}."]
        with open(os.path.join(prof, f"{args.tag}_launches.md"), "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
