"""Run bench.py's headline step (the LLaMA-13B decoder layer as 4 dependent launches:
act quant + one-linear decode program each, M = 16) a few times -- the command profiled by
`ncu --set full` for profiles/ (GPU box only).  Launch order per step: act quant(qkv),
decode(qkv), act quant(o), decode(o), ... so `-k regex:w4a8_decode_dyn -s 4 -c 4` captures
the 4 decode launches of the second step."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
ws = [dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 + i)) for i, (_, n, k) in enumerate(bench.LAYERS)]
x = (torch.randn((args.m, bench.HIDDEN), device="cuda") * 2).half()
layer = bench.SeqLayer(dev, ws, x)
for _ in range(args.reps):
    layer.run(pdl=True)
torch.cuda.synchronize()
print("ok")
