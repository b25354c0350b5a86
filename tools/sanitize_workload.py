"""One small invocation of every kernel family of libodyssey_b200.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck) runs (GPU box only):

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck python tools/sanitize_workload.py

Kernels: act_quant_kernel / act_quant_rows_kernel (K1), w_scale + w4_quant_prepack (K2),
w4a8_gemm_kernel (tile GEMM, decode + stream-K widths), w4a8_prefill_kernel (2-SM),
w4a8_decode_dyn_kernel (independent program, dependency chain at BN 16/32/64 as one program
and as chain links, one-linear ody_gemm path storing into host-mapped memory), the engine kernels (W8A8 / ASYM / FINE incl. regroup / W4A16), LWC."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2311_09550_b200 import api  # noqa: E402
from paper_2311_09550_b200 import device as dev  # noqa: E402


def main():
    torch.cuda.set_device(0)
    rs = np.random.default_rng(3)
    # host ABI: quantize + FAST at decode (dyn kernel) and tile/prefill widths
    for m, n, k in ((5, 256, 384), (80, 384, 512), (256, 512, 640)):
        a = rs.standard_normal((m, k), dtype=np.float32)
        w = rs.standard_normal((n, k), dtype=np.float32) * 0.1
        aq = api.quantize_activations_per_token(a)
        wq = api.quantize_weights(w)
        api.gemm_w4a8_fast(aq, wq)
        api.gemm_w4a8_fast_accumulators(aq, wq)
        api.dequantize(wq)
    # comparison engines
    m, n, k = 9, 200, 384
    a = rs.standard_normal((m, k), dtype=np.float32)
    w = rs.standard_normal((n, k), dtype=np.float32) * 0.1
    aq = api.quantize_activations_per_token(a)
    api.run_engine(4, None, aq, api.quantize_weights(w, 8, 1, 128))
    api.run_engine(2, None, aq, api.quantize_weights(w))
    api.run_engine(1, None, aq, api.quantize_weights(w, 4, 3, 64))
    api.run_engine(1, None, aq, api.quantize_weights(w, 4, 3, 48))  # regroup path
    api.run_engine(0, a, None, api.quantize_weights(w, 4, 3, 64))
    api.optimize_clipping(w[:8, :128], 4)
    # device API: linear (tile + decode), independent program, chains at BN 16/32/64
    for mm in (3, 16, 40, 64):
        dims = [(768, 512), (512, 384), (640, 512), (512, 640)]
        ws = [dev.W4Weight.quantize(torch.randn((nn, kk), device="cuda") * 0.1) for nn, kk in dims]
        x = (torch.randn((mm, 512), device="cuda") * 2).half()
        outs = [torch.empty((mm, nn), dtype=torch.float16, device="cuda") for nn, _ in dims]
        chain = dev.Program([dev.LinearCall(x, ws[0], outs[0]),
                             dev.LinearCall(outs[0][:, :384], ws[1], outs[1], dep=0),
                             dev.LinearCall(outs[1], ws[2], outs[2], dep=1),
                             dev.LinearCall(outs[2][:, :640], ws[3], outs[3], dep=2)])
        chain.run(pdl=True)
        links = dev.Program(chain.calls, links=True)  # the chain as one launch per linear
        assert links.fused
        links.run(pdl=True)
        links.run(pdl=True)
        xs = {kk: (torch.randn((mm, kk), device="cuda") * 2).half() for _, kk in dims}
        ind = dev.Program([dev.LinearCall(xs[kk], wq, torch.empty((mm, nn), dtype=torch.float16, device="cuda"))
                           for (nn, kk), wq in zip(dims, ws)])
        ind.run(pdl=True)
        dev.w4a8_linear(xs[512], ws[0])
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
