"""Timeline of back-to-back bench steps in the program lowering (batched act quant + one
w4a8_decode_dyn_kernel launch per step, PDL-chained, replayed from a CUDA graph): per
launch, CTA entry / producer-done / exit spreads relative to the first step (diagnostics;
GPU box only)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--pdl", type=int, default=1)
    args = ap.parse_args()
    m = args.m
    xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (5120, 13824)}
    progs = []
    for _ in range(args.copies):
        calls = [dev.LinearCall(xs[k], dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1),
                                torch.empty((m, n), dtype=torch.float16, device="cuda")) for _, n, k in LAYERS]
        progs.append(dev.Program(calls))
    bufs = [torch.zeros(148 * 32 + 512, dtype=torch.int64, device="cuda") for _ in progs]
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        for p in progs:
            p.run(pdl=bool(args.pdl), stream=st)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for p, b in zip(progs, bufs):
            lib().ody_dev_set_trace(b.data_ptr())
            p.run(pdl=bool(args.pdl), stream=st)
        lib().ody_dev_set_trace(None)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        g.replay()
        e.record(st)
    torch.cuda.synchronize()
    print(f"{args.copies} steps: {s.elapsed_time(e) * 1e3 / args.copies:.2f} us/step (pdl={args.pdl})")
    ts = [b[:148 * 32].view(148, 32).cpu().numpy() for b in bufs]
    base = min(t[t[:, 0] > 0, 0].min() for t in ts)
    for i, t in enumerate(ts):
        t = t[t[:, 0] > 0]
        f = lambda c: (t[:, c] - base) / 1e3  # noqa: E731
        print(f"step {i}: entry {f(0).min():6.2f}..{f(0).max():6.2f}  producer done {np.median(f(6)):6.2f} "
              f"(max {f(6).max():6.2f})  exit {f(5).min():6.2f} / {np.median(f(5)):6.2f} / {f(5).max():6.2f}")


if __name__ == "__main__":
    main()
