"""Timeline of the headline step (the dependent layer as 4 launches, M = 16, PDL, CUDA
graph): per launch, CTA entry, first MMA, last epilogue and exit from %globaltimer, relative
to the first launch's first CTA entry (GPU box, diagnostics)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
if os.environ.get("ODY_USE_DIAG"):
    from paper_2311_09550_b200 import _lib as _l
    _l.use_diag_library()
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
    pw = v[:, 8][v[:, 8] > 0]
    fb = v[:, 9][v[:, 9] > 0]
    print(f"{'':8s} GEMM pdl_wait returned "
          f"med {f(np.median(pw)) if len(pw) else -1:6.2f} min {f(pw.min()) if len(pw) else -1:6.2f}"
          f"  first B landed med {f(np.median(fb)):6.2f} max {f(fb.max()):6.2f}")

print("per unit of the LAST CTA (us): W issued, MMA saw a_full, conv q1, conv q2, -, conv saw W(q0), "
      "MMA saw b_full, conv q3")
for (name, _, _), bb in zip(bench.LAYERS, bufs):
    ut = bb[148 * 32:148 * 32 + 512].view(64, 8).cpu().numpy()
    print(name)
    for u in range(64):
        row = ut[u]
        if row.max() == 0:
            continue
        print("  %3d " % u + " ".join("%7.2f" % ((v - base) / 1e3) if v > 0 else "      -" for v in row))
