"""Timeline of the headline layer as chain links (ody_dev_w4a8_linear_chain, M = 16, PDL,
CUDA graph): per link, CTA entry, pdl_wait, the B-quantizers' start / qdone release, the
producer warp's qdone acquire, first B landed, first MMA, last epilogue and exit from
%globaltimer (diagnostics library, GPU box).  Run with ODY_USE_DIAG=1."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import _lib as _l  # noqa: E402
_l.use_diag_library()
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
links = len(sys.argv) <= 2 or sys.argv[2] != "0"
stream = torch.cuda.Stream()
ws = [dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 + i)) for i, (_, n, k) in enumerate(bench.LAYERS)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
layer = bench.SeqLayer(dev, ws, x, links=links)
blk = 148 * 32 + 1536
buf = torch.zeros(4 * blk, dtype=torch.int64, device="cuda")
with torch.cuda.stream(stream):
    layer.run(pdl=True, stream=stream)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    if links:
        lib().ody_dev_set_trace(buf.data_ptr())
        layer.run(pdl=True, stream=stream)
    else:
        for i, p in enumerate(layer.progs):
            lib().ody_dev_set_trace(buf[i * blk:].data_ptr())
            p.run(pdl=True, stream=stream)
    lib().ody_dev_set_trace(None)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
buf.zero_()
g.replay()
torch.cuda.synchronize()
t = [buf[i * blk:i * blk + 148 * 32].view(148, 32).cpu().numpy() for i in range(4)]
base = min(tt[:, 0][tt[:, 0] > 0].min() for tt in t)
f = lambda a: (a - base) / 1e3  # noqa: E731


def st(a):
    a = a[a > 0]
    return f"{f(np.median(a)):6.2f}/{f(a.max()):6.2f}" if len(a) else "     -/     -"


print("med/max us:   entry         pdl_wait      quant start   chunk0 quant  quant done    bar done      "
      "qdone rel     qdone acq     first B       first MMA     last epi      exit")
for (name, _, _), tt in zip(bench.LAYERS, t):
    v = tt[tt[:, 0] > 0]
    print(f"{name:8s} {len(v):3d} " + "  ".join(st(v[:, c]) for c in (0, 8, 12, 14, 15, 16, 13, 26, 9, 10, 11, 5)))

if not links:
    print("act quant (16 CTAs): entry / wait returned / loads landed / row max / scale / codes / done, med/max us")
    for i, (name, _, _) in enumerate(bench.LAYERS):
        a = buf[i * blk + 148 * 32 + 512:i * blk + 148 * 32 + 512 + 8 * 64].view(64, 8).cpu().numpy()
        a = a[3:16]  # CTAs 0-2's slots overlap another trace region (8 slots per CTA)
        a = a[a[:, 0] > 0]
        print(f"{name:8s} {len(a):3d} " + "  ".join(st(a[:, c]) for c in (0, 1, 3, 4, 5, 6, 2)))
if not links and len(sys.argv) > 3:
    for i, (name, _, _) in enumerate(bench.LAYERS):
        a = buf[i * blk + 148 * 32 + 512:i * blk + 148 * 32 + 512 + 8 * 64].view(64, 8).cpu().numpy()
        print(name, [(round(f(r[0]), 2), round(f(r[1]), 2), round(f(r[2]), 2)) for r in a[a[:, 0] > 0]])
