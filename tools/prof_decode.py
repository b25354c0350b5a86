"""Launch the decode-width linear kernel on one LLaMA-13B layer shape a few times -- the
command profiled by ncu for profiles/ (diagnostics, GPU box only)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

SHAPES = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824)}
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--layer", default="o")
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
names = list(SHAPES) if args.layer == "all" else [args.layer]
dev.lib().ody_dev_set_linear_mode(2)
for name in names:
    n, k = SHAPES[name]
    x = (torch.randn((args.m, k), device="cuda") * 2).half()
    w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    out = torch.empty((args.m, n), dtype=torch.float16, device="cuda")
    for _ in range(args.reps):
        dev.w4a8_linear(x, w, out=out)
torch.cuda.synchronize()
print("ok")
