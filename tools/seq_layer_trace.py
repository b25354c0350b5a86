"""Timeline of the headline step (the dependent layer as 4 launches, M = 16, PDL, CUDA
graph): per launch, CTA entry, first MMA, last epilogue and exit from %globaltimer, relative
to the first launch's first CTA entry (GPU box, diagnostics)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
stream = torch.cuda.Stream()
ws = [dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 + i)) for i, (_, n, k) in enumerate(bench.LAYERS)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
bufs = [torch.zeros(148 * 32 + 1024 + 512, dtype=torch.int64, device="cuda") for _ in range(4)]
layer = bench.SeqLayer(dev, ws, x)
# bake one trace buffer into each program's launch (the pointer is read at launch time)
with torch.cuda.stream(stream):
    layer.run(pdl=True, stream=stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for p, b in zip(layer.progs, bufs):
        lib().ody_dev_set_trace(b.data_ptr())
        p.run(pdl=True, stream=stream)
    lib().ody_dev_set_trace(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
for b in bufs:
    b.zero_()
g.replay()
torch.cuda.synchronize()
t = [b[:148 * 32].view(148, 32).cpu().numpy() for b in bufs]
base = min(tt[:, 0][tt[:, 0] > 0].min() for tt in t)
for (name, _, _), tt in zip(bench.LAYERS, t):
    v = tt[tt[:, 0] > 0]
    f = lambda a: (a - base) / 1e3  # noqa: E731
    print(f"{name:8s} CTAs {len(v):3d} entry {f(v[:, 0].min()):6.2f}-{f(v[:, 0].max()):6.2f}  first MMA med "
          f"{f(np.median(v[:, 10])):6.2f}  last epilogue med {f(np.median(v[:, 11])):6.2f} max {f(v[:, 11].max()):6.2f}"
          f"  exit max {f(v[:, 5].max()):6.2f}")
