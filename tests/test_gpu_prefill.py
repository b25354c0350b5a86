"""GPU parity of the prefill-width FastGEMM (prefill_kernel.cu: 2-SM cta_group::2 MMAs,
256 weight rows x 256 tokens per CTA pair) against the pinned C oracle, and against the
1-SM tile GEMM on the same inputs.  Bar: bit-exact int32 accumulators and f32 outputs;
f16/bf16 equal to round-to-nearest conversion of the exact f32 result."""
import os

import numpy as np
import pytest

from tests.helpers import bits_of

pytestmark = pytest.mark.gpu

THREADS = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def dev():
    from paper_2311_09550_b200 import device
    device.lib().ody_dev_set_prefill_min_m(65)
    return device


def _oracle_case(oracle, m, n, k, seed):
    r = oracle.rng(seed)
    a = oracle.gaussian_fill(r, (m, k))
    w = oracle.gaussian_fill(r, (n, k), 0.1)
    codes, sa = oracle.quantize_activations(a)
    _, packed, sw = oracle.quantize_weights(w)
    return a, w, oracle.fast_gemm(codes, sa, packed, sw, m, n, k, threads=THREADS)


# ragged shapes: odd 128-row tile counts (a pair's second CTA has no weights), token
# counts that leave a half or whole empty 128-token half tile, K not a multiple of 128
@pytest.mark.parametrize("m,n,k", [(65, 256, 384), (100, 640, 520), (128, 384, 1024), (200, 1000, 640),
                                   (96, 250, 256), (320, 300, 384),  # output rows not 16-byte aligned
                                   (256, 128, 128), (300, 384, 1000), (384, 200, 640),
                                   (640, 1000, 2048), (1024, 640, 520), (1537, 256, 384)])
def test_prefill_vs_oracle(m, n, k, oracle, torch_cuda, dev):
    torch = torch_cuda
    a, w, want = _oracle_case(oracle, m, n, k, 7000 + m + n + k)
    aq = dev.act_quant(torch.from_numpy(a).cuda())
    wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda())
    got = dev.w4a8_gemm(aq, wq, torch.float32).cpu().numpy()
    bad = np.argwhere(bits_of(got) != bits_of(want))
    assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:4].tolist()}"
    assert torch.equal(dev.w4a8_gemm(aq, wq, torch.float16).cpu(), torch.from_numpy(want).half())
    assert torch.equal(dev.w4a8_gemm(aq, wq, torch.bfloat16).cpu(),
                       torch.from_numpy(want).to(torch.bfloat16))


@pytest.mark.parametrize("layer,n,k", [("qkv", 15360, 5120), ("o", 5120, 5120),
                                       ("gate_up", 27648, 5120), ("down", 5120, 13824)])
def test_prefill_llama_equals_tile_gemm(layer, n, k, torch_cuda, dev):
    """LLaMA-13B prefill shapes (M=1024): the 2-SM kernel's int32 accumulators and fp16
    outputs equal the 1-SM tile GEMM's (itself pinned to the oracle at these shapes)."""
    torch = torch_cuda
    g = torch.Generator(device="cuda").manual_seed(n + k)
    x = torch.randn((1024, k), device="cuda", generator=g, dtype=torch.float16)
    w = torch.randn((n, k), device="cuda", generator=g) * 0.05
    aq, wq = dev.act_quant(x), dev.W4Weight.quantize(w)
    acc = dev.w4a8_gemm(aq, wq, accumulators=True)
    y = dev.w4a8_gemm(aq, wq, torch.float16)
    dev.lib().ody_dev_set_prefill_min_m(0)
    try:
        acc_ref = dev.w4a8_gemm(aq, wq, accumulators=True)
        y_ref = dev.w4a8_gemm(aq, wq, torch.float16)
    finally:
        dev.lib().ody_dev_set_prefill_min_m(65)
    assert torch.equal(acc, acc_ref)
    assert torch.equal(y, y_ref)


def test_prefill_cluster_count_invariance(torch_cuda, dev):
    """Any number of persistent CTA pairs gives identical results (tile order changes)."""
    torch = torch_cuda
    x = torch.randn((1024, 2048), device="cuda")
    w = torch.randn((3000, 2048), device="cuda") * 0.05
    aq, wq = dev.act_quant(x), dev.W4Weight.quantize(w)
    base = dev.w4a8_gemm(aq, wq, accumulators=True)
    for ctas in (2, 6, 50, 148):
        assert torch.equal(dev.w4a8_gemm(aq, wq, accumulators=True, max_ctas=ctas), base), ctas
