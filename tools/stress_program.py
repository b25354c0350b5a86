"""Stress: decode-program and two-kernel linears at decode widths, repeated, fresh objects
each trial; reports any output that differs from the first trial (diagnostics; GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

L = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824)}


def two_kernel(x, w):
    dev.lib().ody_dev_set_linear_mode(0)
    try:
        return dev.w4a8_linear(x, w, torch.float16)
    finally:
        dev.lib().ody_dev_set_linear_mode(2)


def main():
    ms = [int(a) for a in sys.argv[1:]] or [64]
    for m in ms:
        ws, xs = [], []
        for i, (name, (n, k)) in enumerate(L.items()):
            ws.append(dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.05))
            xs.append((torch.randn((m, k), device="cuda") * (1 + i)).half())
        base = [two_kernel(x, w) for x, w in zip(xs, ws)]
        bad_ref, bad_prog = {}, {}
        for it in range(60):
            for x, w, b, name in zip(xs, ws, base, L):
                r = two_kernel(x, w)
                if not torch.equal(r, b):
                    d = (r != b).nonzero()
                    bad_ref.setdefault(name, []).append((it, len(d), sorted(set(d[:, 0].tolist()))[:6],
                                                         int(d[:, 1].min()), int(d[:, 1].max())))
            outs = [torch.zeros_like(b) for b in base]
            prog = dev.Program([dev.LinearCall(x, w, o) for x, w, o in zip(xs, ws, outs)])
            prog.run()
            torch.cuda.synchronize()
            for o, b, name in zip(outs, base, L):
                if not torch.equal(o, b):
                    d = (o != b).nonzero()
                    bad_prog.setdefault(name, []).append((it, len(d), sorted(set(d[:, 0].tolist()))[:6],
                                                          int(d[:, 1].min()), int(d[:, 1].max())))
        print("M", m, "ref:", {k: (len(v), v[:2]) for k, v in bad_ref.items()},
              "prog:", {k: (len(v), v[:2]) for k, v in bad_prog.items()}, flush=True)


if __name__ == "__main__":
    main()
