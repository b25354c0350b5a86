"""A/B of single decode linears (one launch each, M = 16, 6 rotating weight copies) timed
like bench.py's per_shape (CUDA graph, PDL; diagnostics: ODY_USE_DIAG + ODY_PROGRAM_DYN=0
selects the static cluster kernel with in-kernel K1)."""
import os
import sys

import torch

sys.path.insert(0, ".")
if os.environ.get("ODY_USE_DIAG"):
    from paper_2311_09550_b200 import _lib as _l
    _l.use_diag_library()
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

res = {}
stream = torch.cuda.Stream()
for n, k in ((4096, 4096), (5120, 5120), (15360, 5120), (27648, 5120), (5120, 13824)):
    m = 16
    ws = [dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1) for _ in range(6)]
    x = (torch.randn((m, k), device="cuda") * 2).half()
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    wsl = dev.Workspace.get_linear(m, n, k, "cuda")
    ms = bench._graph_time(lambda: [dev.w4a8_linear(x, w, out=out, stream=stream, pdl=True, workspace=wsl)
                                    for w in ws], stream, reps=30) / len(ws)
    res[f"{n}x{k}"] = round(ms * 1e3, 2)
print(os.environ.get("ODY_PROGRAM_DYN", "dyn"), res)
