"""The dependent LLaMA-13B layer (M = 16) as ONE chain program vs FOUR single-linear
programs in stream order (each quantizing its input with the batched act quant), CUDA
graph of 4 steps over 4 weight copies, PDL -- bench.py's headline timing (GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
stream = torch.cuda.Stream()
copies = [[dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in
           enumerate(bench.LAYERS)] for c in range(4)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
chains = [bench.ChainLayer(dev, cw, x) for cw in copies]


class Seq:
    def __init__(self, ws):
        self.outs = [torch.empty((m, w.n), dtype=torch.float16, device="cuda") for w in ws]
        o, d = ws[1], ws[3]
        ins = [x, self.outs[0][:, :o.k], self.outs[1], self.outs[2][:, :d.k]]
        self.progs = [dev.Program([dev.LinearCall(i, w, y)]) for i, w, y in zip(ins, ws, self.outs)]

    def run(self, pdl=True, stream=None):
        for p in self.progs:
            p.run(pdl=pdl, stream=stream)


seqs = [Seq(cw) for cw in copies]
for name, objs in (("chain program", chains), ("4 launches", seqs), ("chain program", chains), ("4 launches", seqs)):
    ms = bench._graph_time(lambda objs=objs: [o.run(pdl=True, stream=stream) for o in objs], stream, reps=50) / 4
    print(f"{name:14s} {ms * 1e3:7.2f} us/layer  {bench.step_bytes(m) / (ms * 1e-3) / 1e9:7.1f} GB/s")
