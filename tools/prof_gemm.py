"""Launch the FastGEMM once per LLaMA-13B layer shape (after warm-up) -- the command
profiled by `ncu --set full` for profiles/ (diagnostics, GPU box only)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

HIDDEN, INTER = 5120, 13824
LAYERS = [("qkv", 3 * HIDDEN, HIDDEN), ("o", HIDDEN, HIDDEN), ("gate_up", 2 * INTER, HIDDEN),
          ("down", HIDDEN, INTER)]

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
m = args.m
ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _, n, k in LAYERS]
xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (HIDDEN, INTER)}
a = {k: dev.act_quant(xs[k]) for k in (HIDDEN, INTER)}
outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _ in LAYERS]
for _ in range(args.reps):
    for w, o, (_, n, k) in zip(ws, outs, LAYERS):
        dev.w4a8_gemm(a[k], w, out=o)
torch.cuda.synchronize()
print("ok")
