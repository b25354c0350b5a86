"""Timeline of one bench step in the decode lowering (4 x w4a8_decode_kernel, PDL-chained,
next-weight L2 prefetch hints) from the kernels' %globaltimer stamps, replayed as the
same CUDA graph bench.py times (diagnostics, GPU box only)."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

HIDDEN, INTER = 5120, 13824
LAYERS = [("qkv", 3 * HIDDEN, HIDDEN), ("o", HIDDEN, HIDDEN), ("gate_up", 2 * INTER, HIDDEN),
          ("down", HIDDEN, INTER)]
COLS = [("entry", 0), ("setup", 1), ("pdl_rel", 8), ("localmax", 9), ("exch", 10), ("scaled", 13),
        ("quant", 14), ("bready", 11), ("mma0", 2), ("mmaN", 3), ("epi", 4), ("exit", 5), ("prod", 6)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--prefetch", type=int, default=1)
    ap.add_argument("--copies", type=int, default=4)
    args = ap.parse_args()
    m = args.m
    lib().ody_dev_set_linear_mode(2)
    copies = [[dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _, n, k in LAYERS]
              for _ in range(args.copies)]
    xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (HIDDEN, INTER)}
    outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _ in LAYERS]
    st = torch.cuda.Stream()
    tr = [[torch.zeros(148 * 32, dtype=torch.int64, device="cuda") for _ in LAYERS] for _ in copies]

    def step(c, trace):
        seq = copies[c]
        for i, (w, (_, n, k)) in enumerate(zip(seq, LAYERS)):
            nxt = seq[i + 1] if i + 1 < len(seq) else copies[(c + 1) % len(copies)][0]
            lib().ody_dev_set_trace(tr[c][i].data_ptr() if trace else None)
            dev.w4a8_linear(xs[k], w, out=outs[i], pdl=bool(args.pdl), stream=st,
                            prefetch_next=nxt if args.prefetch else None)
        lib().ody_dev_set_trace(None)

    with torch.cuda.stream(st):
        for c in range(len(copies)):
            step(c, False)
    torch.cuda.synchronize()
    graphs = []
    for c in range(len(copies)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step(c, True)
        graphs.append(g)
    with torch.cuda.stream(st):
        for r in range(8):
            graphs[r % len(copies)].replay()
    torch.cuda.synchronize()
    for c in tr:
        for t in c:
            t.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        s.record(st)
        for r in range(len(copies)):
            graphs[r].replay()
        e.record(st)
    torch.cuda.synchronize()
    print(f"M={m} pdl={args.pdl} prefetch={args.prefetch}: {s.elapsed_time(e) * 1e3 / len(copies):.2f} us/step")
    c = len(copies) - 1  # a step in the middle of a back-to-back sequence
    data = [tr[c][i].view(148, 32).cpu().numpy() for i in range(len(LAYERS))]
    base = min(d[d[:, 0] > 0, 0].min() for d in data)
    print("median (max) us from the step's first entry:")
    print(f"{'linear':9s}" + "".join(f"{n:>14s}" for n, _ in COLS))
    for (name, _, _), d in zip(LAYERS, data):
        d = d[d[:, 0] > 0]
        row = []
        for _, ci in COLS:
            v = d[:, ci]
            v = v[v > 0]
            row.append(f"{np.median((v - base) / 1e3):6.2f}({(v.max() - base) / 1e3:6.2f})" if len(v) else " " * 14)
        print(f"{name:9s}" + "".join(f"{x:>14s}" for x in row))
    print("per-tile epilogue of the owner thread (median/max us): d_full, peers' partials in, stored, slot recycled")
    for (name, _, _), d in zip(LAYERS, data):
        d = d[d[:, 0] > 0]
        for i in range(4):
            cols = d[:, 16 + 4 * i:20 + 4 * i]
            if not (cols[:, 0] > 0).any():
                continue
            row = []
            for j in range(4):
                v = cols[:, j]
                v = v[v > 0]
                row.append(f"{np.median((v - base) / 1e3):6.2f}/{(v.max() - base) / 1e3:6.2f}" if len(v) else "-")
            print(f"   {name:8s} tile {i}: " + "   ".join(row))


if __name__ == "__main__":
    main()
