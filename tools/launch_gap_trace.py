"""Gap between consecutive single-linear programs (M = 16, eager, PDL): per-CTA entry /
exit of launch i and i+1 of w4a8_decode_dyn_kernel from %globaltimer (GPU box)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = 16
ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _ in range(4)]
x = (torch.randn((m, k), device="cuda") * 2).half()
out = torch.empty((m, n), dtype=torch.float16, device="cuda")
progs = [dev.Program([dev.LinearCall(x, w, out)]) for w in ws]
for _ in range(3):
    for p in progs:
        p.run(pdl=True)
torch.cuda.synchronize()
bufs = [torch.zeros(148 * 32 + 1024 + 512, dtype=torch.int64, device="cuda") for _ in progs]
for p, b in zip(progs, bufs):
    lib().ody_dev_set_trace(b.data_ptr())
    p.run(pdl=True)
lib().ody_dev_set_trace(None)
torch.cuda.synchronize()
t = [b[:148 * 32].view(148, 32).cpu().numpy() for b in bufs]
base = t[0][:, 0][t[0][:, 0] > 0].min()
for i, tt in enumerate(t):
    v = tt[tt[:, 0] > 0]
    ent, setup, exit_ = v[:, 0], v[:, 1], v[:, 5]
    ep = v[:, 4]
    print(f"launch {i}: CTAs {len(v)} entry {(ent.min() - base) / 1e3:7.2f}-{(ent.max() - base) / 1e3:7.2f}  "
          f"setup med {(np.median(setup) - base) / 1e3:7.2f}  epilogues done med {(np.median(ep) - base) / 1e3:7.2f} "
          f"max {(ep.max() - base) / 1e3:7.2f}  exit max {(exit_.max() - base) / 1e3:7.2f} us")
