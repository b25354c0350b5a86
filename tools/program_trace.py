"""Per-CTA timeline of ONE linear-program launch (the LLaMA-13B layer's 4 linears,
pre-quantized activations): for every linear, when each CTA issued its first MMA and
finished its epilogue (diagnostics, GPU box only)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("ODY_PLAN_LOG", "1")
from paper_2311_09550_b200 import _lib as _l  # noqa: E402
_l.use_diag_library()  # ODY_PLAN_LOG needs the -DODY_DIAG build
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--layers", default="qkv,o,gate_up,down")
    args = ap.parse_args()
    sel = [l for l in LAYERS if l[0] in args.layers.split(",")]
    m = args.m
    calls = []
    for name, n, k in sel:
        w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
        x = (torch.randn((m, k), device="cuda") * 2).half()
        calls.append(dev.LinearCall(x, w, torch.empty((m, n), dtype=torch.float16, device="cuda")))
    prog = dev.Program(calls)
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    buf = torch.zeros(148 * 32 + 512, dtype=torch.int64, device="cuda")
    lib().ody_dev_set_trace(buf.data_ptr())
    prog.run()
    lib().ody_dev_set_trace(None)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        prog.run()
    e.record()
    torch.cuda.synchronize()
    print(f"program of {len(sel)} linears: {s.elapsed_time(e) * 1e3 / 20:.2f} us/launch (incl. act quant)")
    t = buf[:148 * 32].view(148, 32).cpu().numpy()
    ut = buf[148 * 32:].view(64, 8).cpu().numpy()
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()

    def stat(col):
        v = t[:, col]
        v = v[v > 0]
        if not len(v):
            return "      -      "
        v = (v - base) / 1e3
        return f"{v.min():6.2f}/{np.median(v):6.2f}/{v.max():6.2f}"
    print(f"CTAs {len(t)}  (min/median/max us from the first CTA entry)")
    for nm, col in [("entry", 0), ("setup", 1), ("producer done", 6), ("exit", 5)]:
        print(f"  {nm:14s} {stat(col)}")
    for i, (name, _, _) in enumerate(sel):
        print(f"  {name:8s} first MMA {stat(10 + 4 * i)}   epilogue done {stat(11 + 4 * i)}")
    full = buf[:148 * 32].view(148, 32).cpu().numpy()
    ex = [(b, (full[b, 5] - base) / 1e3) for b in range(148) if full[b, 0] > 0]
    ex.sort(key=lambda z: -z[1])
    print("slowest CTAs (block, exit us, per-linear epilogue done):",
          [(b, round(e, 1), [round((full[b, 11 + 4 * i] - base) / 1e3, 1) for i in range(len(sel))]) for b, e in ex[:12]])
    print("fastest CTAs:", [(b, round(e, 1)) for b, e in ex[-6:]])
    ub = ut[ut > 0].min() if (ut > 0).any() else 0
    print("CTA 0 units (cycles): conv start, conv done, MMA ready, MMA issued, prod at unit, prod slot free, W issued, B issued")
    for u in range(64):
        if ut[u].max() == 0:
            continue
        print("  %3d " % u + " ".join("%8d" % ((v - ub) if v > 0 else -1) for v in ut[u]))


if __name__ == "__main__":
    main()
