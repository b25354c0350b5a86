"""Timeline of one bench step (4 x [act_quant -> FastGEMM]) from in-kernel %globaltimer
stamps, replayed as the same CUDA graph bench.py times (diagnostics, GPU box only)."""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=1)
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--fused", action="store_true")
    args = ap.parse_args()
    m = args.m
    lib().ody_dev_set_linear_mode(1 if args.fused else 0)
    ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _, n, k in LAYERS]
    xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (HIDDEN, INTER)}
    a_buf = {k: dev.act_quant(xs[k]) for k in (HIDDEN, INTER)}
    outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _ in LAYERS]
    wsb = dev.Workspace.for_shapes([(m, n, k) for _, n, k in LAYERS], "cuda")
    for _, n, k in LAYERS:
        wsb = dev.Workspace.get_linear(m, n, k, "cuda")
    st = torch.cuda.Stream()
    gtr = [torch.zeros(148 * 8 + 4096, dtype=torch.int64, device="cuda") for _ in LAYERS]
    atr = [torch.zeros(8 * 1024, dtype=torch.int64, device="cuda") for _ in LAYERS]

    def step(trace):
        for i, (w, (_, n, k)) in enumerate(zip(ws, LAYERS)):
            lib().ody_dev_set_act_trace(atr[i].data_ptr() if trace else None)
            lib().ody_dev_set_trace(gtr[i].data_ptr() if trace else None)
            if not args.fused:
                dev.act_quant(xs[k], out=a_buf[k], pdl=bool(args.pdl), stream=st)
                dev.w4a8_gemm(a_buf[k], w, out=outs[i], pdl=bool(args.pdl), stream=st, workspace=wsb)
            else:
                dev.w4a8_linear(xs[k], w, out=outs[i], pdl=bool(args.pdl), stream=st, workspace=wsb)
        lib().ody_dev_set_act_trace(None)
        lib().ody_dev_set_trace(None)

    with torch.cuda.stream(st):
        for _ in range(3):
            step(False)
    torch.cuda.synchronize()
    if args.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            step(True)
        for _ in range(5):
            with torch.cuda.stream(st):
                g.replay()
        torch.cuda.synchronize()
        for t in gtr + atr:
            t.zero_()
        with torch.cuda.stream(st):
            g.replay()
    else:
        with torch.cuda.stream(st):
            step(True)
    torch.cuda.synchronize()
    ev = []
    act_detail = []
    for i, (name, n, k) in enumerate(LAYERS):
        a8 = atr[i][: 8 * 1024].view(1024, 8).cpu().numpy()
        a8 = a8[a8[:, 0] > 0]
        if len(a8) == 0:
            a8 = np.zeros((1, 8), np.int64)
        a = a8[:, :2]
        act_detail.append((name, a8))
        t = gtr[i][: 148 * 8].view(148, 8).cpu().numpy()
        ev.append((f"act_quant[{name}]", a[:, 0], a[:, 1], None))
        ev.append((f"gemm[{name}] {n}x{k}", t[:, 0], t[:, 5], t))
    base = min(e[1][e[1] > 0].min() for e in ev if (e[1] > 0).any())
    print(f"M={m} pdl={args.pdl} graph={args.graph}  (us from first kernel entry)")
    print(f"{'kernel':32s} {'entry0':>8s} {'entry_max':>9s} {'exit_min':>8s} {'exit_max':>8s}  extra")
    for name, ent, ex, t in ev:
        if not (ent > 0).any():
            continue
        ent = (ent[ent > 0] - base) / 1e3
        ex = (ex[ex > 0] - base) / 1e3
        extra = ""
        if t is not None:
            t = t[t[:, 0] > 0]
            fd = (t[:, 2] - base) / 1e3
            lm = (t[:, 3] - base) / 1e3
            extra = f"first_data med {np.median(fd):6.2f}  last_mma med {np.median(lm):6.2f} max {lm.max():6.2f}"
        print(f"{name:32s} {ent.min():8.2f} {ent.max():9.2f} {ex.min():8.2f} {ex.max():8.2f}  {extra}")
    print("act_quant phases (median us from base): entry, pdl_wait done, loaded+local max, cluster sync 2, exit")
    for name, a8 in act_detail:
        cols = [0, 2, 3, 4, 1]
        med = [np.median((a8[:, c][a8[:, c] > 0] - base) / 1e3) if (a8[:, c] > 0).any() else -1 for c in cols]
        print(f"   {name:10s} " + "  ".join(f"{v:7.2f}" for v in med))


if __name__ == "__main__":
    main()

