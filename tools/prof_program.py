"""Run the LLaMA-13B decoder-layer linear program (4 linears, one launch + the batched
act quant) a few times -- the command profiled by ncu for profiles/ (GPU box only)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]
ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--chain", action="store_true", help="the dependent chain qkv -> o -> gate_up -> down")
args = ap.parse_args()
calls = []
outs = []
for i, (name, n, k) in enumerate(LAYERS):
    w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    out = torch.empty((args.m, n), dtype=torch.float16, device="cuda")
    if args.chain and i > 0:
        x = outs[-1][:, :k]
        calls.append(dev.LinearCall(x, w, out, dep=i - 1))
    else:
        x = (torch.randn((args.m, k), device="cuda") * 2).half()
        calls.append(dev.LinearCall(x, w, out))
    outs.append(out)
prog = dev.Program(calls)
for _ in range(args.reps):
    prog.run()
torch.cuda.synchronize()
print("ok", prog.fused)
