"""Per-CTA timeline of the decode-width linear kernel (w4a8_decode_kernel), one launch per
LLaMA-13B layer shape (diagnostics; GPU box only).  Slots (globaltimer, us from the first
CTA entry): entry, setup done, first MMA issued, last MMA issued, epilogue done, exit,
producer done."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("ODY_PLAN_LOG", "1")
from paper_2311_09550_b200 import _lib as _l  # noqa: E402
_l.use_diag_library()  # ODY_PLAN_LOG needs the -DODY_DIAG build
from paper_2311_09550_b200 import device as dev  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

SLOTS = ["entry", "setup", "first_mma", "last_mma", "epi_done", "exit", "prod_done", None, "q_waited", "q_localmax", "q_exchanged", "q_bready", "mma_bready", "q_scaled", "q_quantized"]
LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--pdl", type=int, default=0)
    args = ap.parse_args()
    lib().ody_dev_set_linear_mode(2)
    for name, n, k in LAYERS:
        m = args.m
        x = (torch.randn((m, k), device="cuda") * 2).half()
        wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.1)
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
        for _ in range(3):
            dev.w4a8_linear(x, wq, out=out)
        torch.cuda.synchronize()
        lib().ody_dev_set_trace(buf.data_ptr())
        dev.w4a8_linear(x, wq, out=out, pdl=bool(args.pdl))
        torch.cuda.synchronize()
        lib().ody_dev_set_trace(None)
        t = buf.view(148, 32).cpu().numpy()
        live = t[:, 0] > 0
        t = t[live]
        base = t[:, 0].min()
        rel = (t[:, :15] - base) / 1000.0
        meta = t[:, 7]
        print(f"== {name}: M={m} N={n} K={k} CTAs={live.sum()} tiles/CTA {(meta & 0xFFFFFFFF).min()}.."
              f"{(meta & 0xFFFFFFFF).max()} S={meta[0] >> 32}")
        for i, s in enumerate(SLOTS):
            if s is None or (t[:, i] == 0).all():
                continue
            col = rel[:, i]
            print(f"   {s:>10}: min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
        span = rel[:, 5].max()
        print(f"   span {span:.2f} us -> {n * k / 2 / (span * 1e-6) / 1e9:.0f} GB/s of weights")


if __name__ == "__main__":
    main()
