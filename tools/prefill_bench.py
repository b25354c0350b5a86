"""Prefill-shape (M = 1024) W4A8 GEMM throughput on the LLaMA-13B layer shapes: TOPS
against the INT8 dense tensor peak (diagnostics; GPU box only).  Times the FastGEMM on
pre-quantized activations (the GEMM-only kernel) and the whole linear (act quant + GEMM)."""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]


def timed(fn, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(reps):
        g.replay()
    e.record(st)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--peak", type=float, default=4500.0, help="INT8 dense TOPS denominator")
    args = ap.parse_args()
    m = args.m
    res = {}
    for name, n, k in LAYERS:
        ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _ in range(2)]
        x = (torch.randn((m, k), device="cuda") * 2).half()
        a = dev.act_quant(x)
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        gws = dev.Workspace.get(m, n, k, "cuda")
        ms = timed(lambda: [dev.w4a8_gemm(a, w, out=out, workspace=gws) for w in ws]) / len(ws)
        ms_lin = timed(lambda: [dev.w4a8_linear(x, w, out=out) for w in ws]) / len(ws)
        ops = 2.0 * m * n * k
        res[name] = {"M": m, "N": n, "K": k, "gemm_us": round(ms * 1e3, 2),
                     "gemm_TOPS": round(ops / (ms * 1e-3) / 1e12, 1),
                     "frac_of_peak": round(ops / (ms * 1e-3) / 1e12 / args.peak, 3),
                     "linear_us": round(ms_lin * 1e3, 2),
                     "linear_TOPS": round(ops / (ms_lin * 1e-3) / 1e12, 1)}
        print(name, res[name], flush=True)
    print(json.dumps({"prefill": res, "peak_tops": args.peak}))


if __name__ == "__main__":
    main()
