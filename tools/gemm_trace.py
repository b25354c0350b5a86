"""Per-CTA timeline of the FastGEMM kernel (diagnostics; run on the GPU box).

Uses ody_dev_set_trace: every CTA writes %globaltimer at entry, after setup, when the
first stage lands at the MMA warp, at its last MMA commit, when its epilogue is done,
at exit, and when its producer has issued every copy."""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

SLOTS = ["entry", "setup", "first_data", "last_mma", "epi_done", "exit", "prod_done"]


def trace_one(name, m, n, k, pdl, reps=3):
    x = (torch.randn((m, k), device="cuda") * 2).half()
    w = torch.randn((n, k), device="cuda") * 0.1
    wq = dev.W4Weight.quantize(w)
    a = dev.act_quant(x)
    buf = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    for _ in range(reps):
        dev.w4a8_gemm(a, wq, out=out, pdl=pdl)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(buf.data_ptr())
    dev.act_quant(x, out=a, pdl=pdl)
    dev.w4a8_gemm(a, wq, out=out, pdl=pdl)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(None)
    t = buf.view(148, 8).cpu().numpy()
    live = t[:, 0] > 0
    t = t[live]
    base = t[:, 0].min()
    rel = (t[:, :7] - base) / 1000.0  # us
    meta = t[:, 7]
    units = meta & 0xFFFFFFFF
    segs = meta >> 32
    print(f"== {name}: M={m} N={n} K={k} pdl={pdl} CTAs={live.sum()} units/CTA "
          f"{units.min()}..{units.max()} segs {segs.min()}..{segs.max()}")
    for i, s in enumerate(SLOTS):
        col = rel[:, i]
        print(f"   {s:>10}: min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
    span = rel[:, 5].max()
    print(f"   kernel span (first entry -> last exit) {span:.2f} us; "
          f"weights {n * k / 2 / 1e6:.1f} MB -> {n * k / 2 / (span * 1e-6) / 1e9:.0f} GB/s")


def fused_trace(m=16, n=15360, k=5120):
    x = (torch.randn((m, k), device="cuda") * 2).half()
    wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    dbg0 = 148 * 8 + 64 * 4 + 148 * 16 + 256
    buf = torch.zeros(dbg0 + 148 * 8, dtype=torch.int64, device="cuda")
    dev.w4a8_linear(x, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(buf.data_ptr())
    dev.w4a8_linear(x, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(None)
    cta = buf[:148 * 8].view(148, 8).cpu().numpy()
    live = cta[:, 0] > 0
    base = cta[live, 0].min()
    d = buf[dbg0:].view(148, 8).cpu().numpy()[live]
    rel = lambda v: (v - base) / 1000.0
    print(f"fused {m}x{n}x{k}: CTAs {live.sum()}")
    for i, nm in [(0, "loads issued"), (1, "local max"), (4, "max sent"), (5, "max recv"),
                  (2, "scales done"), (6, "codes stored"), (3, "pushes issued"), (7, "b_ready")]:
        col = d[:, i]
        if (col == 0).all():
            continue
        col = rel(col)
        print(f"   {nm:>14}: min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
    for i, nm in [(1, "setup"), (2, "first_data"), (3, "last_mma"), (5, "exit")]:
        col = rel(cta[live, i])
        print(f"   {nm:>14}: min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=0)
    ap.add_argument("--units", action="store_true")
    ap.add_argument("--epi", action="store_true")
    ap.add_argument("--fused", action="store_true")
    ap.add_argument("--layer", default="o")
    args = ap.parse_args()
    if args.units:
        unit_trace(args.m)
        return
    if args.fused:
        shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824)}
        for nm in (shapes if args.layer == "all" else [args.layer if args.layer in shapes else "qkv"]):
            fused_trace(args.m, *shapes[nm])
        return
    if args.epi:
        n, k = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120),
                "down": (5120, 13824)}[args.layer]
        epi_trace(args.m, n, k)
        return
    for name, n, k in [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120),
                       ("down", 5120, 13824)]:
        trace_one(name, args.m, n, k, bool(args.pdl))



def unit_trace(m=16, n=27648, k=5120):
    """clock64 per unit of CTA 0: conv start, a_empty ok, st done, MMA a_full ok."""
    x = (torch.randn((m, k), device="cuda") * 2).half()
    wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    a = dev.act_quant(x)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    buf = torch.zeros(148 * 8 + 64 * 4 + 148 * 16 + 64 * 4, dtype=torch.int64, device="cuda")
    dev.w4a8_gemm(a, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(buf.data_ptr())
    dev.w4a8_gemm(a, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(None)
    u = buf[148 * 8:148 * 8 + 256].view(64, 4).cpu().numpy()
    mm = buf[148 * 8 + 256 + 148 * 16:].view(64, 4).cpu().numpy()
    base = u[u > 0].min()
    print("unit  conv_start  a_empty_ok  st_done  mma_go | mma: loop_top  wfull_ok  issued")
    for i in range(64):
        if u[i].max() == 0:
            continue
        r = [(v - base) if v > 0 else -1 for v in u[i]]
        q = [(v - base) if v > 0 else -1 for v in mm[i]]
        print(f"{i:4d} {r[0]:10d} {r[1]:10d} {r[2]:9d} {r[3]:8d} | {q[0]:8d} {q[1]:9d} {q[2]:7d}")



def epi_trace(m=16, n=5120, k=5120):
    x = (torch.randn((m, k), device="cuda") * 2).half()
    wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    a = dev.act_quant(x)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    buf = torch.zeros(148 * 8 + 64 * 4 + 148 * 16 + 256 + 148 * 4, dtype=torch.int64, device="cuda")
    dev.w4a8_gemm(a, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(buf.data_ptr())
    dev.w4a8_gemm(a, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(None)
    cta = buf[:148 * 8].view(148, 8).cpu().numpy()
    base = cta[:, 0][cta[:, 0] > 0].min()
    e16 = buf[148 * 8 + 256:148 * 8 + 256 + 148 * 16].view(148, 16).cpu().numpy()
    fix = e16[:, 15].copy()
    e16[:, 12:] = 0
    e = e16.reshape(148, 4, 4)
    fin = (e[:, :, 3] >> 63) & 1
    e[:, :, 3] &= (1 << 63) - 1
    rows = []
    for b in range(148):
        for j in range(4):
            if e[b, j, 0] == 0:
                continue
            r = [(v - base) / 1000 if v > 0 else -1 for v in e[b, j]]
            rows.append((b, j, *r, fin[b, j], (cta[b, 3] - base) / 1000,
                         (fix[b] - base) / 1000 if fix[b] > 0 else -1))
    dbg = buf[148 * 8 + 256 + 148 * 16 + 256:].view(148, 4).cpu().numpy()
    d = dbg[dbg[:, 0] > 0]
    if len(d):
        print("epilogue clock deltas (cycles, median/max over CTAs): ld->adds %d/%d adds->stores %d/%d "
              "stores->arrive %d/%d" % (np.median(d[:, 1] - d[:, 0]), (d[:, 1] - d[:, 0]).max(),
                                      np.median(d[:, 2] - d[:, 1]), (d[:, 2] - d[:, 1]).max(),
                                      np.median(d[:, 3] - d[:, 2]), (d[:, 3] - d[:, 2]).max()))
    rows.sort(key=lambda r: -max(r[2:6]))
    print("cta seg  dfull  stored  fixok  done  owner last_mma fixup_done  (us, slowest first)")
    for r in rows[:20]:
        print("%3d %3d %6.2f %7.2f %7.2f %6.2f %4d %8.2f %8.2f" % r)


if __name__ == "__main__":
    main()
