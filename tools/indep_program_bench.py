"""The LLaMA-13B layer's 4 linears on INDEPENDENT inputs as one program launch (M = 16),
graph of the 4 weight copies, PDL -- bench.py's roofline.independent_linears_program."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

m = 16
stream = torch.cuda.Stream()
copies = [[dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in
           enumerate(bench.LAYERS)] for c in range(4)]
xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (bench.HIDDEN, bench.INTER)}
ind = [dev.Program([dev.LinearCall(xs[w.k], w, torch.empty((m, w.n), dtype=torch.float16, device="cuda"))
                    for w in cw]) for cw in copies]
for _ in range(3):
    ms = bench._graph_time(lambda: [p.run(pdl=True, stream=stream) for p in ind], stream, reps=50) / len(ind)
    print(f"independent program {ms * 1e3:.2f} us  {bench.step_bytes(m) / (ms * 1e-3) / 1e9:.1f} GB/s")
