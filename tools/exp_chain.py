"""Decode lowering comparison on the LLaMA-13B layer (diagnostics, GPU box only):
independent-linear program vs the dependent chain qkv -> o -> gate_up -> down (slices as
attention / SiLU stand-ins) vs per-linear launches; graphs over rotating weight copies."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

H, I = 5120, 13824
LAYERS = [("qkv", 3 * H, H), ("o", H, H), ("gate_up", 2 * I, H), ("down", H, I)]


def lin_bytes(m, n, k):
    return n * k // 2 + 4 * n + 2 * m * k + 2 * m * n + 4 * m


def gtime(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    copies = 4
    for m in (1, 16):
        ws = [[dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _, n, k in LAYERS]
              for _ in range(copies)]
        byts = sum(lin_bytes(m, n, k) for _, n, k in LAYERS)
        x = (torch.randn((m, H), device="cuda") * 2).half()
        xi = (torch.randn((m, I), device="cuda") * 2).half()
        outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _ in LAYERS]
        # independent program
        ind = [dev.Program([dev.LinearCall(x if k == H else xi, w, o) for (_, n, k), w, o in zip(LAYERS, wc, outs)])
               for wc in ws]
        # chain program
        chain = []
        for wc in ws:
            calls = [dev.LinearCall(x, wc[0], outs[0]),
                     dev.LinearCall(outs[0][:, :H], wc[1], outs[1], dep=0),
                     dev.LinearCall(outs[1], wc[2], outs[2], dep=1),
                     dev.LinearCall(outs[2][:, :I], wc[3], outs[3], dep=2)]
            chain.append(dev.Program(calls))
        print(f"M={m}: chain fused={chain[0].fused} independent fused={ind[0].fused}")
        for name, progs in (("independent", ind), ("chain", chain)):
            for pdl in (False, True):
                ms = gtime(lambda s, progs=progs, pdl=pdl: [p.run(pdl=pdl, stream=s) for p in progs]) / copies
                print(f"  {name:12s} pdl={pdl}: {ms*1e3:7.2f} us/layer  {byts/ms/1e6:7.1f} GB/s")
        # per-linear launches (chain semantics), each through w4a8_linear
        wsl = dev.Workspace.get_linear(m, 27648, 13824, "cuda")

        def per_linear(s, pdl):
            for wc in ws:
                dev.w4a8_linear(x, wc[0], out=outs[0], stream=s, pdl=pdl, workspace=wsl)
                dev.w4a8_linear(outs[0][:, :H], wc[1], out=outs[1], stream=s, pdl=pdl, workspace=wsl)
                dev.w4a8_linear(outs[1], wc[2], out=outs[2], stream=s, pdl=pdl, workspace=wsl)
                dev.w4a8_linear(outs[2][:, :I], wc[3], out=outs[3], stream=s, pdl=pdl, workspace=wsl)
        for pdl in (False, True):
            ms = gtime(lambda s, pdl=pdl: per_linear(s, pdl)) / copies
            print(f"  per-linear   pdl={pdl}: {ms*1e3:7.2f} us/layer  {byts/ms/1e6:7.1f} GB/s")
        # each linear alone (rotating copies)
        for li, (nm, n, k) in enumerate(LAYERS):
            xx = x if k == H else xi
            ms = gtime(lambda s, li=li, xx=xx: [dev.w4a8_linear(xx, wc[li], out=outs[li], stream=s, pdl=True,
                                                                workspace=wsl) for wc in ws]) / copies
            print(f"    {nm:8s} alone (pdl chain of copies): {ms*1e3:7.2f} us  {lin_bytes(m, n, k)/ms/1e6:7.1f} GB/s")
        del ws, ind, chain
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
