"""Per-k-block timeline of the 2-SM prefill FastGEMM, CTA pair 0 (diagnostics; GPU box).

Slots per k-block u: producer past empty[s], converter past full[s], converter arrived
on the leader's ready[s], leader MMA past ready[s]; per tile: epilogue start / end."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

K_TR = 256


def main():
    m, n, k = 1024, int(sys.argv[1]) if len(sys.argv) > 1 else 15360, 5120
    x = (torch.randn((m, k), device="cuda") * 2).half()
    wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
    a = dev.act_quant(x)
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    for _ in range(3):
        dev.w4a8_gemm(a, wq, out=out)
    buf = torch.zeros(2 * K_TR * 4 + 64 + 40, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(buf.data_ptr())
    dev.w4a8_gemm(a, wq, out=out)
    torch.cuda.synchronize()
    lib().ody_dev_set_trace(None)
    t = buf.cpu().numpy()
    kb = t[:2 * K_TR * 4].reshape(2, K_TR, 4)
    ep = t[2 * K_TR * 4:2 * K_TR * 4 + 64].reshape(2, 16, 2)
    ph = t[2 * K_TR * 4 + 64:].reshape(8, 5)
    print("epilogue tile 0, CTA 0, clk per chunk: ld+wait, stage, bar1, store, (to next chunk)")
    for c in range(8):
        nxt = ph[c + 1, 0] if c < 7 else ph[c, 4]
        print("  chunk", c, ph[c, 1] - ph[c, 0], ph[c, 2] - ph[c, 1], ph[c, 3] - ph[c, 2], ph[c, 4] - ph[c, 3], nxt - ph[c, 4])
    base = kb[kb > 0].min()
    rel = np.where(kb > 0, (kb - base) / 1000.0, np.nan)
    print("u  | cta0: prod conv_in conv_out mma | cta1: prod conv_in conv_out")
    for u in list(range(0, 12)) + list(range(36, 46)) + list(range(120, 126)):
        r0, r1 = rel[0, u], rel[1, u]
        print(f"{u:3d} | " + " ".join(f"{v:8.3f}" for v in r0) + " | " + " ".join(f"{v:8.3f}" for v in r1[:3]))
    mma = rel[0, :, 3]
    d = np.diff(mma[~np.isnan(mma)])
    print("MMA k-block cadence us: median %.3f mean %.3f max %.3f" % (np.median(d), d.mean(), d.max()))
    epr = np.where(ep > 0, (ep - base) / 1000.0, np.nan)
    for c in range(2):
        print("cta%d epilogue (start,end):" % c, [(round(a_, 2), round(b_, 2)) for a_, b_ in epr[c] if not np.isnan(a_)])


if __name__ == "__main__":
    main()
