"""Diagnostic probe for the GEMM layouts (run on the GPU box; prints, never asserts).

Structured inputs make layout bugs legible: with one-hot activation rows and weight
codes that encode (row, k), each accumulator names the element it picked up."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402


def main():
    print(lib().ody_b200_version().decode())
    torch.manual_seed(0)
    for (m, n, k) in [(16, 128, 128), (1, 128, 128), (16, 256, 256), (3, 5, 7), (64, 384, 1024),
                      (128, 256, 512), (200, 300, 700)]:
        x = torch.randn((m, k), device="cuda")
        w = torch.randn((n, k), device="cuda") * 0.1
        aq = dev.act_quant(x)
        wq = dev.W4Weight.quantize(w)
        acc = dev.w4a8_gemm(aq, wq, accumulators=True).cpu().numpy().astype(np.int64)
        codes = aq.codes().cpu().numpy().astype(np.int64)
        flat = wq.to_flat().cpu().numpy().astype(np.int64)
        idx = np.arange(n * k)
        nib = np.where(idx % 2 == 0, flat[idx // 2] & 0xF, flat[idx // 2] >> 4)
        wc = np.where(nib >= 8, nib - 16, nib).reshape(n, k)
        want = 16 * (codes @ wc.T)
        ok = np.array_equal(acc, want)
        print(f"m={m} n={n} k={k}: {'OK' if ok else 'MISMATCH'}")
        if not ok:
            bad = np.argwhere(acc != want)
            print("  mismatches", len(bad), "of", acc.size, "first", bad[:6].tolist())
            print("  got ", acc[0, :8].tolist())
            print("  want", want[0, :8].tolist())
    # one-hot probe: a row t has a single 1 at column c -> acc[t, j] = 16 * w[j, c] * code
    m, n, k = 16, 128, 128
    a = np.zeros((m, k), np.float32)
    for t in range(m):
        a[t, (t * 9) % k] = 1.0
    w = np.zeros((n, k), np.float32)
    rs = np.random.default_rng(1)
    wcodes = rs.integers(-8, 8, (n, k))
    w[:] = wcodes * 0.1
    w[:, 0] = 0.7  # pin per-row scale to 0.1
    aq = dev.act_quant(torch.from_numpy(a).cuda())
    wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda())
    acc = dev.w4a8_gemm(aq, wq, accumulators=True).cpu().numpy()
    wc = np.rint(w / 0.1).astype(np.int64)
    for t in range(4):
        c = (t * 9) % k
        want = 16 * 127 * wc[:8, c]
        print(f"one-hot t={t} col={c}: got {acc[t, :8].tolist()} want {want.tolist()}")
        if not np.array_equal(acc[t, :8], want):
            # which column did we pick up?
            for cc in range(k):
                if np.array_equal(acc[t, :32], 16 * 127 * wc[:32, cc]):
                    print(f"   -> matches weight column {cc}")
                    break


if __name__ == "__main__":
    main()
