"""FastGEMM consumption rate with weights L2-resident vs HBM-streamed (diagnostics).

If the L2-resident rate is far above HBM, the kernel's pipeline can catch up after a
stall (L2 prefetch pays); if it is near the HBM rate, the pipeline itself is the bound."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402


def timed(fn, reps=50):
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
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=0)
    args = ap.parse_args()
    m = args.m
    for name, n, k in [("o", 5120, 5120), ("qkv", 15360, 5120), ("down", 5120, 13824),
                       ("gate_up", 27648, 5120)]:
        ncopy = 6
        ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _ in range(ncopy)]
        x = (torch.randn((m, k), device="cuda") * 2).half()
        a = dev.act_quant(x)
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        wsb = dev.Workspace.get_linear(m, n, k, "cuda")
        reps_in = 8
        hot = timed(lambda: [dev.w4a8_gemm(a, ws[0], out=out, workspace=wsb, pdl=bool(args.pdl))
                             for _ in range(reps_in)]) / reps_in
        cold = timed(lambda: [dev.w4a8_gemm(a, w, out=out, workspace=wsb, pdl=bool(args.pdl))
                              for w in ws]) / ncopy
        b = n * k / 2
        print(f"{name:8s} M={m} N={n} K={k}: L2-hot {hot*1e3:7.2f} us ({b/hot/1e6:7.0f} GB/s)   "
              f"HBM {cold*1e3:7.2f} us ({b/cold/1e6:7.0f} GB/s)")
        del ws


if __name__ == "__main__":
    main()
