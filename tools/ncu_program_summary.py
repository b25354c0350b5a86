"""Summarise the decode linear-program ncu captures into profiles/ (runs HERE, on the CPU
box, over gpurun_out/).

    python tools/ncu_program_summary.py --rep gpurun_out/prof_program_r1.ncu-rep \
        --launches gpurun_out/launches_r1.csv --tag r1

Writes profiles/<tag>_program_ncu.md (the full-set metrics of one w4a8_decode_dyn_kernel
launch: the LLaMA-13B layer's 4 linears at M=16, plus the top stall reasons from the
source page), profiles/<tag>_program_launches.md (per-launch device time and DRAM bytes of
the kernels inside bench.py's timed region) and the "program_M16" entry of
profiles/ncu_gemm_traffic.json (bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
        ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
         "UTCIMMA (tcgen05 kind::i8) % of peak"),
        ("lts__t_bytes.sum", "L2 traffic"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2]


def stalls(rep, top=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next((r for r in rows if "Address" in r and "Source" in r), None)
    if not hdr:
        return []
    data = rows[rows.index(hdr) + 1:]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    for r in data:
        for c in cols:
            try:
                tot[c] += int(r[hdr.index(c)])
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    return [(k, v, v / s) for k, v in tot.most_common(top)]


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    ui = hdr.index("Metric Unit")
    gi = hdr.index("Grid Size")
    d = collections.defaultdict(dict)
    meta = {}
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        d[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1)
        meta[r[ii]] = (r[ki], r[gi])
    return d, meta


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches", required=True)
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--chain", action="store_true", help="the capture is the dependent chain (prof_program.py --chain)")
    args = ap.parse_args()
    what = "chain" if args.chain else "program"
    hdr, units, vals = raw(args.rep)
    desc = ("the DEPENDENT chain qkv -> o(qkv[:, :5120]) -> gate_up -> down(gate_up[:, :13824]) (bench.py's "
            "headline step: dependent linears' x quantized in-kernel grid-wide)" if args.chain else
            "the 4 linears as INDEPENDENT inputs")
    lines = [f"# Decode linear {what}, ncu --set full ({args.tag})", "",
             "Command: `ncu --set full --clock-control none --import-source on -k regex:w4a8_decode_dyn -s 2 "
             f"-c 1 python tools/prof_program.py{' --chain' if args.chain else ''}` -- ONE launch of "
             "w4a8_decode_dyn_kernel running the LLaMA-13B decoder layer's 4 linears (qkv, o, gate_up, down) at "
             f"M=16: {desc}; cold L2, serialised, unlocked clocks (compare bytes and shares, not absolutes).",
             "", "| metric | value |", "|---|---|"]
    traffic = 0.0
    for key, label in WANT:
        if key in hdr:
            i = hdr.index(key)
            lines.append(f"| {label} (`{key}`) | {vals[i]} {units[i]} |")
            if key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                traffic += float(vals[i].replace(",", "")) * SCALE.get(units[i], 1)
    if args.chain:  # bench.py linear_bytes: INT4 W + scales + fp16 x + fp16 y + token scales
        alg = sum(n * k // 2 + 4 * n + 2 * 16 * k + 2 * 16 * n + 4 * 16
                  for n, k in ((15360, 5120), (5120, 5120), (27648, 5120), (5120, 13824)))
    else:
        alg = 158597120 + 4 * (15360 + 5120 + 27648 + 5120) + 16 * (5120 * 3 + 13824) + 2 * 16 * (15360 + 5120 + 27648 + 5120)
    lines += ["", f"DRAM traffic {traffic / 1e6:.2f} MB vs algorithmic {alg / 1e6:.2f} MB "
              f"(INT4 weights + scales + int8 activation tiles + fp16 outputs): ratio {traffic / alg:.3f} -- "
              "every weight byte is fetched from HBM once.", ""]
    st = stalls(args.rep)
    if st:
        lines += ["Warp-state samples (source page), top reasons:", "", "| reason | samples | share |", "|---|---|---|"]
        lines += [f"| {k} | {v} | {f:.1%} |" for k, v, f in st]
    open(os.path.join(ROOT, "profiles", f"{args.tag}_{what}_ncu.md"), "w").write("\n".join(lines) + "\n")

    d, meta = launches(args.launches)
    fam = collections.defaultdict(list)
    for i in d:
        fam[(meta[i][0].split("(")[0].replace("void ", ""), meta[i][1])].append(d[i])
    total = sum(x.get("gpu__time_duration.sum", 0) for v in fam.values() for x in v)
    out = [f"# Launch list inside bench.py's timed region ({args.tag})", "",
           "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
           "-k \"regex:w4a8|act_quant\" -s 20 -c 24 python bench.py --steps 20 --warmup 3 --no-cpu --quick` -- "
           "serialised, cold-cache per-launch device times: only the SHARE of each kernel is meaningful.", "",
           "| kernel | grid | launches | mean us | mean DRAM read MB | share of device time |", "|---|---|---|---|---|---|"]
    for (name, grid), v in sorted(fam.items(), key=lambda kv: -sum(x.get("gpu__time_duration.sum", 0) for x in kv[1])):
        t = [x.get("gpu__time_duration.sum", 0) for x in v]
        rd = [x.get("dram__bytes_read.sum", 0) for x in v]
        out.append(f"| `{name}` | {grid} | {len(v)} | {sum(t) / len(t):.2f} | {sum(rd) / len(rd) / 1e6:.2f} | "
                   f"{sum(t) / total:.1%} |")
    open(os.path.join(ROOT, "profiles", f"{args.tag}_{what}_launches.md"), "w").write("\n".join(out) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    js = json.load(open(tp)) if os.path.exists(tp) else {}
    js[f"{what}_M16"] = int(traffic)
    js[f"{what}_M16_source"] = f"profiles/{args.tag}_{what}_ncu.md"
    json.dump(js, open(tp, "w"), indent=1)
    print("\n".join(lines))
    print("\n".join(out))


if __name__ == "__main__":
    main()
