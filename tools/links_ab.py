"""A/B of the headline step's two lowerings of the dependent layer (M = 16 unless argv[1]):
four one-linear programs each behind its own act-quant kernel, vs the chain as links
(ody_dev_w4a8_linear_chain: one act quant, dependent x quantized in-kernel); graph of 4
steps over 4 weight copies, PDL, CUDA events (GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
stream = torch.cuda.Stream()
copies = [[dev.W4Weight.quantize(bench._weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in enumerate(bench.LAYERS)]
          for c in range(4)]
x = (torch.randn((m, bench.HIDDEN), device="cuda") * 2).half()
res = {}
for links in (False, True, False, True):
    layers = [bench.SeqLayer(dev, cw, x, links=links) for cw in copies]
    t = bench._graph_time(lambda: [l.run(pdl=True, stream=stream) for l in layers], stream, reps=200) / 4
    res.setdefault(links, []).append(t * 1e3)
    outs = [l.y.clone() for l in layers]
    if links:
        ref = [bench.SeqLayer(dev, cw, x, links=False) for cw in copies]
        for r in ref:
            r.run(pdl=True, stream=stream)
        torch.cuda.synchronize()
        for r, l in zip(ref, layers):
            for a, b in zip(r.outs, l.outs):
                assert torch.equal(a, b), "links differ from the 4-program step"
    del layers
for k, v in res.items():
    print(f"M={m} links={k}: " + " ".join(f"{u:.2f}" for u in v) + " us/step")
