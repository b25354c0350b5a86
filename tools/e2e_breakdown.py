"""Host-side time of each reference-ABI call in bench.py's e2e step (GPU box)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2311_09550_b200 import api  # noqa: E402
from paper_2311_09550_b200._lib import lib  # noqa: E402

LAYERS = [("qkv", 15360, 5120), ("o", 5120, 5120), ("gate_up", 27648, 5120), ("down", 5120, 13824)]
rs = np.random.default_rng(7)
wq = [api.quantize_weights((rs.standard_normal((n, k), dtype=np.float32) * 0.1)) for _, n, k in LAYERS]
x = rs.standard_normal((16, 5120), dtype=np.float32) * 2


def measure(threads, iters=30):
    lib().ody_set_threads(threads)
    acc, tot = {}, 0.0
    for it in range(iters):
        h = x
        t_step = time.perf_counter()
        for (name, n, k), w in zip(LAYERS, wq):
            t0 = time.perf_counter()
            hs = h[:, :k]  # row-strided view: ody_tensor_create_strided
            t1 = time.perf_counter()
            t = api.Tensor(hs)
            t2 = time.perf_counter()
            aq = api.quantize_activations_per_token(t)
            t3 = time.perf_counter()
            h = api.gemm_w4a8_fast(aq, w)
            t4 = time.perf_counter()
            if it >= 5:
                for key, v in (("slice", t1 - t0), ("tensor_create", t2 - t1), ("quantize_act", t3 - t2),
                               ("gemm", t4 - t3)):
                    acc[key] = acc.get(key, 0) + v * 1e6 / (iters - 5)
        if it >= 5:
            tot += (time.perf_counter() - t_step) * 1e6 / (iters - 5)
    return acc, tot


for threads in (1, 0, 0):
    acc, tot = measure(threads)
    print(f"threads={threads}: step {tot:7.1f} us  " + "  ".join(f"{k} {v:6.1f}" for k, v in acc.items()))
