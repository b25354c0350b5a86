"""Headline step time (the dependent layer as 4 launches, graph of 4 steps over 4 weight
copies, PDL) on the DIAGNOSTICS library, so ODY_* knobs set by the caller apply; argv[1]
= M (default 16).  Usage: ODY_REST_PF=1 python tools/seq_ab.py 16 (GPU box)."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import _lib as _l  # noqa: E402
_l.use_diag_library()
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
stream = torch.cuda.Stream()
copies = [[dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in enumerate(bench.LAYERS)]
          for c in range(4)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
layers = [bench.SeqLayer(dev, cw, x) for cw in copies]
ts = [bench._graph_time(lambda: [l.run(pdl=True, stream=stream) for l in layers], stream, reps=200) / 4 * 1e3
      for _ in range(3)]
knobs = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("ODY_"))
print(f"M={m} {knobs or '(defaults)'}: " + " ".join(f"{t:.2f}" for t in ts) + " us/step")
