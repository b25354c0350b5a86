"""Per-CTA timeline of ONE dependent-chain program launch (the LLaMA-13B layer
qkv -> o -> gate_up -> down, slices as attention / SiLU stand-ins) on the dynamic
kernel: per linear, each CTA's first MMA, dependency release and last epilogue
(diagnostics, GPU box only)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import os  # noqa: E402
if os.environ.get("ODY_USE_DIAG"):
    from paper_2311_09550_b200 import _lib as _l  # noqa: E402
    _l.use_diag_library()
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

H, I = 5120, 13824
LAYERS = [("qkv", 3 * H, H), ("o", H, H), ("gate_up", 2 * I, H), ("down", H, I)]


def main(m=16, single=None):
    if single:  # one linear (n, k) as a program of one
        n, k = single
        w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
        x = (torch.randn((m, k), device="cuda") * 2).half()
        prog = dev.Program([dev.LinearCall(x, w, torch.empty((m, n), dtype=torch.float16, device="cuda"))])
    else:
        ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _, n, k in LAYERS]
        x = (torch.randn((m, H), device="cuda") * 2).half()
        outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _ in LAYERS]
        prog = dev.Program([dev.LinearCall(x, ws[0], outs[0]),
                            dev.LinearCall(outs[0][:, :H], ws[1], outs[1], dep=0),
                            dev.LinearCall(outs[1], ws[2], outs[2], dep=1),
                            dev.LinearCall(outs[2][:, :I], ws[3], outs[3], dep=2)])
    buf = torch.zeros(148 * 32 + 512 + 512, dtype=torch.int64, device="cuda")
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    # traced launch right behind an untraced one: no other kernel in between (any other
    # kernel leaves the SM instruction caches cold, tools/icache_probe.cu)
    prog.run()
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
    print(f"M={m} chain program: {s.elapsed_time(e) * 1e3 / 20:.2f} us/launch (incl. act quant)")
    t = buf[:148 * 32].view(148, 32).cpu().numpy()
    t = t[t[:, 0] > 0]
    base = t[:, 0].min()

    def stat(col):
        v = t[:, col]
        v = v[v > 0]
        if not len(v):
            return "        -          "
        v = (v - base) / 1e3
        return f"{v.min():6.2f}/{np.median(v):6.2f}/{v.max():6.2f} n={len(v):3d}"
    print(f"CTAs {len(t)}  (min/median/max us from the first CTA entry)")
    for nm, col in [("entry", 0), ("setup", 1), ("producer in", 2), ("item id", 3), ("first item", 30), ("first W issued", 31), ("producer done", 6), ("epilogues done", 4), ("exit", 5)]:
        print(f"  {nm:14s} {stat(col)}")
    for i, (name, _, _) in enumerate(LAYERS):
        print(f"  {name:8s} first MMA {stat(10 + 4 * i)}  dep released {stat(12 + 4 * i)}  last epilogue {stat(11 + 4 * i)}")
        print(f"  {'':8s} x quantized {stat(13 + 4 * i)}  producer saw qdone {stat(26 + i)}")
    if not single:
        tt = buf[:148 * 32].view(148, 32).cpu().numpy()
        for i, (name, _, k) in enumerate(LAYERS):
            if i == 0:
                continue
            kb = (k + 127) // 128
            q = (tt[:, 13 + 4 * i] - base) / 1e3
            r = (tt[:, 12 + 4 * i] - base) / 1e3
            quant = np.arange(148) < kb
            d = q - r
            order = np.argsort(-d)
            print(f"  {name}: quantizing CTAs {quant.sum()}: release->quantized us median {np.median(d[quant]):.2f} "
                  f"max {d[quant].max():.2f}; slowest CTAs " +
                  ", ".join(f"{c}({d[c]:.2f})" for c in order[:5]) +
                  f"; non-quantizing max {d[~quant].max() if (~quant).any() else 0:.2f}")
    et = buf[148 * 32 + 512:].view(32, 16).cpu().numpy()[:, :11]
    print("last CTA, per item epilogue (us): d_full, tmem ld, scales, atom, reduced, stored, amax, done, after-bar, "
          "fields, token 8")
    for j2 in range(32):
        row = et[j2]
        if row.max() == 0:
            continue
        print("  %3d " % j2 + " ".join("%7.2f" % ((v - base) / 1e3) if v > 0 else "      -" for v in row))
    ut = buf[148 * 32:148 * 32 + 512].view(64, 8).cpu().numpy()
    print("last CTA, per unit (us from first CTA entry): W issued, MMA saw a_full, B-quant saw x, B done, "
          "conv saw W, conv done, MMA saw b_full")
    for u in range(64):
        row = ut[u]
        if row.max() == 0:
            continue
        print("  %3d " % u + " ".join("%7.2f" % ((v - base) / 1e3) if v > 0 else "      -" for v in row[:8]))
    print("  last x issue: %.2f" % ((ut[63, 7] - base) / 1e3 if ut[63, 7] > 0 else -1))


if __name__ == "__main__":
    if len(sys.argv) > 2:  # chain_trace.py N K [M]: one linear
        main(int(sys.argv[3]) if len(sys.argv) > 3 else 16, (int(sys.argv[1]), int(sys.argv[2])))
    else:
        for m in (1, 16):
            main(m)
