"""The dependent LLaMA-13B layer (M = 16) as ONE chain program vs FOUR single-linear
programs in stream order (each quantizing its input with the batched act quant), CUDA
graph of 4 steps over 4 weight copies, PDL --
bench.py's headline timing (GPU box)."""
import os
import sys

import torch

sys.path.insert(0, ".")
if os.environ.get("ODY_USE_DIAG"):
    from paper_2311_09550_b200 import _lib as _l
    _l.use_diag_library()
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
stream = torch.cuda.Stream()
copies = [[dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in
           enumerate(bench.LAYERS)] for c in range(4)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
chains = [bench.ChainLayer(dev, cw, x) for cw in copies]


seqs = [bench.SeqLayer(dev, cw, x) for cw in copies]
runs = [("chain program", chains), ("4 launches", seqs)] * 2
for name, objs in runs:
    if not objs:
        continue
    ms = bench._graph_time(lambda objs=objs: [o.run(pdl=True, stream=stream) for o in objs], stream, reps=50) / 4
    print(f"{name:14s} {ms * 1e3:7.2f} us/layer  {bench.step_bytes(m) / (ms * 1e-3) / 1e9:7.1f} GB/s")
