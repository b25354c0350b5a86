"""Stress: the 2-SM prefill GEMM repeated on the LLaMA-13B shapes (M = 1024) and ragged
shapes; every repeat must be bit-identical to the first (diagnostics; GPU box)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402

SHAPES = [(1024, 15360, 5120), (1024, 5120, 5120), (1024, 27648, 5120), (1024, 5120, 13824),
          (300, 384, 1000), (1537, 256, 384), (512, 1000, 2048)]


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    for m, n, k in SHAPES:
        x = torch.randn((m, k), device="cuda").half()
        w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.05)
        aq = dev.act_quant(x)
        base = dev.w4a8_gemm(aq, w, accumulators=True)
        y0 = dev.w4a8_gemm(aq, w, torch.float16)
        bad = 0
        for _ in range(reps):
            if not torch.equal(dev.w4a8_gemm(aq, w, accumulators=True), base):
                bad += 1
            if not torch.equal(dev.w4a8_gemm(aq, w, torch.float16), y0):
                bad += 1
        print(f"{m}x{n}x{k}: {bad} mismatching repeats of {2 * reps}", flush=True)


if __name__ == "__main__":
    main()
