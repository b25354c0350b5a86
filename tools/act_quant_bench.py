"""K1 (per-token act quant) device time per launch, CUDA-graph replay (diagnostics; GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

for m, k in [(16, 5120), (256, 5120), (1024, 5120), (1024, 13824)]:
    x = (torch.randn((m, k), device="cuda") * 2).half()
    a = dev.act_quant(x)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            dev.act_quant(x, out=a, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(20):
            dev.act_quant(x, out=a, stream=st)
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    with torch.cuda.stream(st):
        for _ in range(10):
            g.replay()
    e.record(st)
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / 200 * 1e3
    b = m * k * 3 + 4 * m
    print(f"act_quant {m}x{k}: {us:.2f} us/launch, {b / us / 1e3:.0f} GB/s")
