"""Summarise the ncu captures of the prefill FastGEMM into profiles/ (runs HERE, on the CPU
box, over gpurun_out/).

    python tools/ncu_prefill_summary.py --rep gpurun_out/prof_prefill_r1b.ncu-rep \
        --launches gpurun_out/prefill_launches.csv --tag r1

Writes profiles/<tag>_prefill_ncu.md: per-launch metrics of w4a8_prefill_kernel for the
four LLaMA-13B layer shapes at M = 1024 (tools/prof_gemm.py --m 1024) and the device-time
launch list of the same command."""
import argparse
import csv
import io
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
M = 1024
SHAPES = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]
WANT = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__cluster_dim_x"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(WANT)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def launches(path):
    if not path or not os.path.exists(path):
        return []
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = []
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            out.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit", "")))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r1")
    a = ap.parse_args()
    rows, units = raw(a.rep)
    md = [f"# {a.tag}: ncu --set full of the prefill FastGEMM (M = {M}, LLaMA-13B layer shapes)", "",
          "Command (GPU box): `ncu --set full --clock-control none --import-source on -k regex:w4a8_prefill "
          "-s 4 -c 4 python tools/prof_gemm.py --m 1024` -- one launch per shape after warm-up. "
          "ncu serialises launches with a cold L2; `bench.py`'s `prefill` key holds the live CUDA-event "
          "times. Algorithmic ops per launch = 2*M*N*K; peak = 4.5 POPS dense INT8 (datasheet).", "",
          "| shape | N | K | grid | cluster | regs | smem KiB | time us | SM GHz | TOPS | frac 4.5P | tensor pipe % | "
          "SM % | L1 % | L2 % | issue % | DRAM rd MB | DRAM wr MB |",
          "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for (name, n, k), r in zip(SHAPES, rows):
        t = float(r["gpu__time_duration.sum"])
        tu = units["gpu__time_duration.sum"]
        us = t / 1000.0 if tu == "ns" else (t * 1000.0 if tu == "ms" else t)
        tops = 2.0 * M * n * k / (us * 1e-6) / 1e12

        def mb(key):
            v = float(r[key])
            u = units[key]
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)

        md.append(f"| {name} | {n} | {k} | {r['launch__grid_size']} | {r['launch__cluster_dim_x']} | "
                  f"{r['launch__registers_per_thread']} | {float(r['launch__shared_mem_per_block_dynamic']):.0f} | "
                  f"{us:.1f} | {float(r['sm__cycles_elapsed.avg.per_second']):.2f} | {tops:.0f} | {tops / 4500:.3f} | "
                  f"{float(r['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                  f"{float(r['sm__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                  f"{float(r['l1tex__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                  f"{float(r['lts__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                  f"{float(r['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
                  f"{mb('dram__bytes_read.sum'):.1f} | {mb('dram__bytes_write.sum'):.1f} |")
    md += ["", "Reading: no unit is saturated (tensor pipe <= 66% of the cycles at the clock ncu saw, "
           "1.67-1.81 GHz under this power draw; L2 and L1 well below peak; DRAM ~ the weights once + the fp16 output) -- the "
           "per-k-block pipeline is bound by shared-memory traffic (B bulk-copy write + widened A tile "
           "write + both MMA operand reads, ~64 KiB per k-block per SM; W comes from L2 straight into "
           "the converter warps' registers) and the stage round trip. "
           "DESIGN.md section 4.5 lists the variants measured.", ""]
    ls = launches(a.launches)
    if ls:
        md += ["## Launch list (`ncu --metrics gpu__time_duration.sum`, same command)", "",
               "| # | kernel | us |", "|---|---|---|"]
        for i, (kn, v, u) in enumerate(ls):
            us = v / 1000.0 if u == "ns" else (v * 1000.0 if u == "ms" else v)
            md.append(f"| {i} | {kn[:90]} | {us:.1f} |")
        md.append("")
    out = os.path.join(ROOT, "profiles", f"{a.tag}_prefill_ncu.md")
    with open(out, "w") as f:
        f.write("\n".join(md))
    print(out)


if __name__ == "__main__":
    main()
