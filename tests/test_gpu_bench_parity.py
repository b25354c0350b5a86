"""GPU parity of exactly what bench.py times, against the oracle -- never CUDA vs CUDA.

* the decode step: one LLaMA-13B decoder layer's 4 linears at M = 16 as ONE linear
  program (batched K1 + w4a8_decode_dyn_kernel), fp16 x = 2 N(0,1), W = 0.1 N(0,1);
* the dependent chain qkv -> o -> gate_up -> down (slices as attention / SiLU stand-ins);
* prefill: all four LLaMA-13B shapes at M = 1024 through the 2-SM prefill kernel, every
  output compared (no sampling);
* config 1 (M = 16, N = K = 4096) through the reference C ABI;
* the reference acceptance sweep (acceptance.cpp:65-105) replayed through the C ABI;
* ody_dequantize bit-exact against quantize.cpp:134-146.

The full-size reference results come from Oracle.exact_accumulators / exact_epilogue
(f64 BLAS over the integer codes -- exact, pinned to the C restatement on CPU)."""
import numpy as np
import pytest

from tests.helpers import bits_of
from tests.test_oracle_golden import acceptance_trials

pytestmark = pytest.mark.gpu

H, I = 5120, 13824
LAYERS = [("qkv", 3 * H, H), ("o", H, H), ("gate_up", 2 * I, H), ("down", H, I)]


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def dev():
    from paper_2311_09550_b200 import device
    return device


@pytest.fixture(scope="module")
def layer(oracle, torch_cuda, dev):
    """The bench layer: host f32 weights, quantized by BOTH sides from the same values."""
    torch = torch_cuda
    rs = np.random.default_rng(2024)
    out = []
    for name, n, k in LAYERS:
        w = (rs.standard_normal((n, k), dtype=np.float32) * np.float32(0.1)).astype(np.float32)
        wcodes, _, sw = oracle.quantize_weights(w)
        wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda())
        assert np.array_equal(bits_of(wq.s.cpu().numpy()), bits_of(sw)), name
        out.append((name, n, k, wq, wcodes, sw))
        del w
    return out


def _want_f16(oracle, x_f16, wcodes, sw):
    codes, sa = oracle.quantize_activations(x_f16.astype(np.float32))
    y = oracle.exact_fast_gemm(codes, sa, wcodes, sw)
    return y.astype(np.float16), sa


def test_bench_program_vs_oracle(layer, oracle, torch_cuda, dev):
    """The bench step (independent linears, one program launch) bit-exact vs the oracle."""
    torch = torch_cuda
    m = 16
    rs = np.random.default_rng(7)
    xs = {k: (rs.standard_normal((m, k), dtype=np.float32) * 2).astype(np.float16) for k in (H, I)}
    xd = {k: torch.from_numpy(v).cuda() for k, v in xs.items()}
    outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _, *_ in layer]
    prog = dev.Program([dev.LinearCall(xd[k], wq, o) for (_, n, k, wq, _, _), o in zip(layer, outs)])
    assert prog.fused
    for pdl in (False, True):
        for o in outs:
            o.fill_(0)
        prog.run(pdl=pdl)
        torch.cuda.synchronize()
        for (name, n, k, wq, wcodes, sw), o in zip(layer, outs):
            want, _ = _want_f16(oracle, xs[k], wcodes, sw)
            got = o.cpu().numpy()
            assert np.array_equal(got.view(np.uint16), want.view(np.uint16)), (name, pdl)


@pytest.mark.parametrize("links", [False, True])
def test_dependent_chain_vs_oracle(links, layer, oracle, torch_cuda, dev):
    """qkv -> o -> gate_up -> down as a dependency chain in one program: each linear's
    input is the previous linear's fp16 output (column slices as the attention / SiLU
    stand-ins), quantized per token inside the launch.  Bit-exact vs the oracle run
    step by step on the same fp16 intermediates.  links: bench.py's headline step, the
    chain as one launch per linear (each dependent x quantized in-kernel)."""
    torch = torch_cuda
    for m in (1, 16):
        rs = np.random.default_rng(70 + m)
        x = (rs.standard_normal((m, H), dtype=np.float32) * 2).astype(np.float16)
        xd = torch.from_numpy(x).cuda()
        outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for _, n, _, *_ in layer]
        w = [t[3] for t in layer]
        prog = dev.Program([dev.LinearCall(xd, w[0], outs[0]),
                            dev.LinearCall(outs[0][:, :H], w[1], outs[1], dep=0),
                            dev.LinearCall(outs[1], w[2], outs[2], dep=1),
                            dev.LinearCall(outs[2][:, :I], w[3], outs[3], dep=2)], links=links)
        assert prog.fused
        for _ in range(2):  # the second run starts from the state the first left behind
            prog.run(pdl=True)
        torch.cuda.synchronize()
        cur = x
        for li, (name, n, k, wq, wcodes, sw) in enumerate(layer):
            want, _ = _want_f16(oracle, np.ascontiguousarray(cur[:, :k]), wcodes, sw)
            got = outs[li].cpu().numpy()
            assert np.array_equal(got.view(np.uint16), want.view(np.uint16)), (m, name)
            cur = got


@pytest.mark.parametrize("li", range(4))
def test_prefill_m1024_full_vs_oracle(li, layer, oracle, torch_cuda, dev):
    """configs[2]: M = 1024 through the 2-SM prefill kernel, EVERY output bit-exact."""
    torch = torch_cuda
    name, n, k, wq, wcodes, sw = layer[li]
    m = 1024
    rs = np.random.default_rng(100 + li)
    x = (rs.standard_normal((m, k), dtype=np.float32) * 2).astype(np.float16)
    aq = dev.act_quant(torch.from_numpy(x).cuda())
    codes, sa = oracle.quantize_activations(x.astype(np.float32))
    assert np.array_equal(aq.codes().cpu().numpy(), codes)
    acc = dev.w4a8_gemm(aq, wq, accumulators=True).cpu().numpy()
    want_acc = oracle.exact_accumulators(codes, wcodes)
    assert np.array_equal(acc, want_acc), (name, int((acc != want_acc).sum()))
    want = oracle.exact_epilogue(want_acc, sa, sw)
    got = dev.w4a8_gemm(aq, wq, torch.float16).cpu().numpy()
    assert np.array_equal(got.view(np.uint16), want.astype(np.float16).view(np.uint16)), name
    got32 = dev.w4a8_gemm(aq, wq, torch.float32).cpu().numpy()
    assert np.array_equal(bits_of(got32), bits_of(want)), name


def test_config1_c_abi_vs_oracle(oracle):
    """configs[0]: M = 16, N = K = 4096 (the reference bench.cpp inputs) through the C ABI."""
    from paper_2311_09550_b200 import api
    m, n, k = 16, 4096, 4096
    a, w = oracle.bench_inputs(1, m, n, k)
    aq = api.quantize_activations_per_token(a)
    wq = api.quantize_weights(w)
    out = api.gemm_w4a8_fast(aq, wq)
    codes, sa = oracle.quantize_activations(a)
    wcodes, _, sw = oracle.quantize_weights(w)
    assert np.array_equal(bits_of(out), bits_of(oracle.exact_fast_gemm(codes, sa, wcodes, sw)))


@pytest.mark.parametrize("m,n,k", [(16, 27648, 5120), (5, 20544, 2048)])
def test_c_abi_over_one_wave_vs_oracle(oracle, m, n, k):
    """ody_gemm at decode widths with more 128-row tiles than SMs (gate_up's 216; 161):
    the partial last wave runs k-split (split2 2 / 4); bit-exact vs the oracle."""
    from paper_2311_09550_b200 import api
    a, w = oracle.bench_inputs(7, m, n, k)
    aq = api.quantize_activations_per_token(a)
    wq = api.quantize_weights(w)
    out = api.gemm_w4a8_fast(aq, wq)
    codes, sa = oracle.quantize_activations(a)
    wcodes, _, sw = oracle.quantize_weights(w)
    assert np.array_equal(bits_of(out), bits_of(oracle.exact_fast_gemm(codes, sa, wcodes, sw)))


def test_acceptance_sweep_c_abi(oracle):
    """acceptance.cpp:65-105 replayed on the GPU through the C ABI: 100 random matrices
    (Rng(101), w 0.2 N(0,1)): acc % 16 == 0, acc >> 4 == the int code dot, and the whole
    accumulator matrix bit-equal to the oracle's."""
    from paper_2311_09550_b200 import api
    for t, (m, n, k, a, w) in enumerate(acceptance_trials(oracle)):
        aq = api.quantize_activations_per_token(a)
        wq = api.quantize_weights(w)
        acc = api.gemm_w4a8_fast_accumulators(aq, wq)
        codes, _ = oracle.quantize_activations(a)
        wcodes, packed, _ = oracle.quantize_weights(w)
        assert np.all(acc % 16 == 0), t
        assert np.array_equal(acc >> 4, codes.astype(np.int64) @ wcodes.astype(np.int64).T), t
        assert np.array_equal(acc, oracle.fast_accumulators(codes, packed, m, n, k)), t


def test_dequantize_bit_exact(oracle):
    """ody_dequantize (GPU) == ref quantize.cpp:134-146 float(code) * scale, bit for bit,
    for per-token activations and per-channel weights (odd K: ragged nibble tail)."""
    from paper_2311_09550_b200 import api
    r = oracle.rng(909)
    for m, n, k in ((3, 5, 7), (16, 130, 333), (64, 257, 1000)):
        a = oracle.gaussian_fill(r, (m, k)) * 4
        w = oracle.gaussian_fill(r, (n, k), 0.1)
        codes, sa = oracle.quantize_activations(a)
        wcodes, _, sw = oracle.quantize_weights(w)
        da = api.dequantize(api.quantize_activations_per_token(a))
        dw = api.dequantize(api.quantize_weights(w))
        assert np.array_equal(bits_of(da), bits_of(oracle.dequantize_rows(codes, sa)))
        assert np.array_equal(bits_of(dw), bits_of(oracle.dequantize_rows(wcodes, sw)))
