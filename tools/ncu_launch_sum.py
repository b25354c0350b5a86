"""Per-step DRAM traffic and device-time shares from an ncu launch list of bench.py's
timed region (runs HERE over gpurun_out/):

    python tools/ncu_launch_sum.py gpurun_out/launches_r2s.csv --tag r2 --per-step 4

Writes profiles/<tag>_seq_launches.md and the "seq_M16" entry of
profiles/ncu_gemm_traffic.json (bench.py's roofline.traffic: DRAM read + write of the
step's decode-program launches)."""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_program_summary import launches  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--tag", default="r2")
    ap.add_argument("--per-step", type=int, default=4, help="decode-program launches per step")
    a = ap.parse_args()
    d, meta = launches(a.csv)
    fam = collections.defaultdict(list)
    for i in d:
        fam[meta[i][0].split("(")[0].replace("void ", "")].append(d[i])
    total = sum(x.get("gpu__time_duration.sum", 0) for v in fam.values() for x in v)
    dyn = [x for k, v in fam.items() if "decode_dyn" in k for x in v]
    per_launch = sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in dyn) / len(dyn)
    traffic = per_launch * a.per_step
    out = [f"# Launch list inside bench.py's timed region ({a.tag}, headline step = 4 dependent launches)", "",
           "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
           "-k \"regex:w4a8|act_quant\" -s 40 -c 32 python bench.py --steps 20 --warmup 3 --no-cpu --quick` -- "
           "serialised, cold-cache per-launch device times: only the SHARE of each kernel is meaningful.", "",
           "| kernel | launches | mean us | mean DRAM read+write MB | share of device time |", "|---|---|---|---|---|"]
    for name, v in sorted(fam.items(), key=lambda kv: -sum(x.get("gpu__time_duration.sum", 0) for x in kv[1])):
        t = [x.get("gpu__time_duration.sum", 0) for x in v]
        b = [x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in v]
        out.append(f"| `{name}` | {len(v)} | {sum(t) / len(t):.2f} | {sum(b) / len(b) / 1e6:.2f} | "
                   f"{sum(t) / total:.1%} |")
    out += ["", f"Decode-program DRAM traffic per step ({a.per_step} launches): {traffic / 1e6:.2f} MB "
            f"(algorithmic 161.45 MB)."]
    open(os.path.join(ROOT, "profiles", f"{a.tag}_seq_launches.md"), "w").write("\n".join(out) + "\n")
    tp = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    js = json.load(open(tp)) if os.path.exists(tp) else {}
    js["seq_M16"] = int(traffic)
    js["seq_M16_source"] = f"profiles/{a.tag}_seq_launches.md"
    json.dump(js, open(tp, "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
