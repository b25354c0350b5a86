"""GPU parity of the decode-width W4A8 linear kernel (csrc/decode_kernel.cu): per-token
INT8 quantization of each CTA's k-slice fused into the cluster split-K FastGEMM, with a
DSMEM reduce-scatter epilogue.  Everything is bit-exact against the pinned CPU oracle
(ref quantize.cpp:113-132 + gemm.cpp:251-279), for every cluster split the planner can
pick, odd shapes, strides, dtypes, zero rows and rounding-boundary activations."""
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
    device.lib().ody_dev_set_linear_mode(2)
    return device


def _weights(torch, dev, n, k, seed, scale=0.1):
    rs = np.random.default_rng(seed)
    wq = dev.W4Weight.quantize(torch.from_numpy(rs.standard_normal((n, k), dtype=np.float32) * scale).cuda())
    return wq, wq.to_flat().cpu().numpy(), wq.s.cpu().numpy()


def _want(oracle, x32, flat, sw, m, n, k):
    codes, sa = oracle.quantize_activations(x32)
    return oracle.fast_gemm(codes, sa, flat, sw, m, n, k, threads=THREADS), sa


def _assert_bits(got, want):
    g = got.cpu().float().numpy() if hasattr(got, "cpu") else got
    if not np.array_equal(bits_of(np.ascontiguousarray(g, np.float32)), bits_of(want)):
        bad = np.argwhere(g != want)
        pytest.fail(f"{len(bad)} of {want.size} outputs differ, first {bad[:4].tolist()}")


@pytest.mark.parametrize("m,n,k", [
    (1, 128, 128), (3, 130, 1000), (16, 1000, 4100), (7, 384, 64), (2, 257, 2049),
    (16, 5120, 14336), (3, 640, 16384),  # largest K the batched act quant holds: 256 x 4 x 16
    (5, 15360, 5120), (16, 27648, 5120), (11, 5120, 13824), (1, 5120, 5120),
    (17, 640, 1536), (33, 5120, 5120), (64, 2048, 13824), (48, 130, 1000),  # BN 32 / 64 kernels
    (3, 20544, 2048), (40, 27648, 5120),  # > 148 tiles: the partial last wave k-split (split2 4 / 2)
])
def test_decode_linear_vs_oracle(m, n, k, oracle, torch_cuda, dev):
    torch = torch_cuda
    assert dev.lib().ody_dev_linear_is_fused(m, n, k) == 1
    wq, flat, sw = _weights(torch, dev, n, k, seed=n + k + m)
    x16 = (torch.randn((m, k), generator=torch.Generator().manual_seed(m * 7 + k)) * 1.7).half()
    want, sa = _want(oracle, x16.float().numpy(), flat, sw, m, n, k)
    sa_out = torch.empty(m, dtype=torch.float32, device="cuda")
    got = dev.w4a8_linear(x16.cuda(), wq, torch.float32, sa_out=sa_out)
    assert np.array_equal(bits_of(sa_out.cpu().numpy()), bits_of(sa))
    _assert_bits(got, want)


def test_decode_plan_invariance(torch_cuda, dev):
    """Any CTA budget (cluster split S, cluster count C, or the two-kernel fallback when no
    plan fits) gives the same bits -- the int32 reduce-scatter is order-free."""
    torch = torch_cuda
    m, n, k = 16, 5120, 5120
    wq, _, _ = _weights(torch, dev, n, k, seed=5)
    x = (torch.randn((m, k), device="cuda") * 2).half()
    base = dev.w4a8_linear(x, wq, torch.float32)
    for ctas in (1, 3, 7, 16, 21, 37, 100, 147, 148):
        got = dev.w4a8_linear(x, wq, torch.float32, max_ctas=ctas)
        assert torch.equal(got, base), ctas


def test_decode_dtypes_strides_zero_rows(oracle, torch_cuda, dev):
    torch = torch_cuda
    m, n, k = 9, 640, 1536
    wq, flat, sw = _weights(torch, dev, n, k, seed=9)
    for xdt in (torch.float16, torch.bfloat16):
        wide = (torch.randn((m, k + 64), device="cuda") * 4).to(xdt)
        wide[2].zero_()                      # all-zero token: S = 2^-24, codes 0 (ref tensor.hpp:14)
        x = wide[:, :k]                      # row stride k + 64
        want, sa = _want(oracle, x.float().cpu().numpy(), flat, sw, m, n, k)
        assert sa[2] == np.float32(2.0 ** -24)
        for odt in (torch.float32, torch.float16, torch.bfloat16):
            got = dev.w4a8_linear(x, wq, odt)
            assert torch.equal(got.cpu(), torch.from_numpy(want).to(odt)), (xdt, odt)


@pytest.mark.parametrize("xdt", ["f16", "bf16"])
def test_decode_rounding_boundaries(xdt, oracle, torch_cuda, dev):
    """16-bit activations on and next to x/S = j + 1/2, where the reciprocal fast path must
    defer to IEEE division (ref quantize.cpp:44 divides)."""
    torch = torch_cuda
    tdt = torch.float16 if xdt == "f16" else torch.bfloat16
    rs = np.random.default_rng(3)
    m, k, n = 16, 1024, 256
    rows = []
    for _ in range(m):
        amax = float(torch.tensor(rs.uniform(0.05, 60.0)).to(tdt))
        S = np.float32(np.float32(amax) / np.float32(127.0))
        half = (np.arange(-127, 127, dtype=np.float32) + np.float32(0.5)) * S
        near = torch.from_numpy(half).to(tdt)
        up = torch.nextafter(near, torch.tensor(np.inf, dtype=tdt))
        dn = torch.nextafter(near, torch.tensor(-np.inf, dtype=tdt))
        rnd = torch.from_numpy(rs.uniform(-amax, amax, k).astype(np.float32)).to(tdt)
        row = torch.cat([near, up, dn, rnd])[:k].float().clamp(-amax, amax).to(tdt)
        row[5] = amax
        rows.append(row)
    x = torch.stack(rows)
    wq, flat, sw = _weights(torch, dev, n, k, seed=1)
    want, _ = _want(oracle, x.float().numpy(), flat, sw, m, n, k)
    _assert_bits(dev.w4a8_linear(x.cuda(), wq, torch.float32), want)


def test_decode_tiny_bf16_rows(oracle, torch_cuda, dev):
    """bf16 rows of magnitude ~1e-39: S = max/127 is an f32 subnormal and 1/S overflows,
    so the whole row takes the IEEE-division path (no FTZ anywhere)."""
    torch = torch_cuda
    m, k, n = 3, 512, 128
    x = (torch.randn((m, k)) * 1e-39).to(torch.bfloat16)
    x[1] = (torch.randn(k) * 1e-3).to(torch.bfloat16)
    wq, flat, sw = _weights(torch, dev, n, k, seed=2)
    want, sa = _want(oracle, x.float().numpy(), flat, sw, m, n, k)
    sa_out = torch.empty(m, dtype=torch.float32, device="cuda")
    got = dev.w4a8_linear(x.cuda(), wq, torch.float32, sa_out=sa_out)
    assert np.array_equal(bits_of(sa_out.cpu().numpy()), bits_of(sa))
    _assert_bits(got, want)


def test_decode_pdl_chain_and_graph(torch_cuda, dev):
    """x of each linear is the previous linear's output: with PDL the weight stream starts
    before griddepcontrol.wait and only the activation loads wait -- results must equal
    the serialised launches, eagerly and replayed from a CUDA graph."""
    torch = torch_cuda
    m, d = 4, 2048
    ws = [_weights(torch, dev, d, d, seed=s, scale=0.02)[0] for s in range(4)]
    x0 = (torch.randn((m, d), device="cuda")).half()

    def chain(pdl, outs):
        h = x0
        for w, o in zip(ws, outs):
            h = dev.w4a8_linear(h, w, torch.float16, out=o, pdl=pdl)
        return h

    ref_outs = [torch.empty((m, d), dtype=torch.float16, device="cuda") for _ in ws]
    ref = chain(False, ref_outs).clone()
    st = torch.cuda.Stream()
    outs = [torch.empty((m, d), dtype=torch.float16, device="cuda") for _ in ws]
    with torch.cuda.stream(st):
        got = chain(True, outs)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        chain(True, outs)
    for o in outs:
        o.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(outs[-1], ref)


LLAMA13B = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120), "down": (5120, 13824)}


def _two_kernel(dev, torch, x, w, odt):
    """Reference lowering: act-quant kernel + FastGEMM (pinned to the oracle elsewhere)."""
    dev.lib().ody_dev_set_linear_mode(0)
    try:
        return dev.w4a8_linear(x, w, odt)
    finally:
        dev.lib().ody_dev_set_linear_mode(2)


@pytest.mark.parametrize("m", [1, 3, 16, 32, 64])
def test_program_independent_layer(m, torch_cuda, dev):
    """The 4 LLaMA-13B layer linears as ONE launch (independent inputs): every output is
    bit-identical to the same linear run alone."""
    torch = torch_cuda
    calls, refs = [], []
    for i, (name, (n, k)) in enumerate(LLAMA13B.items()):
        w, _, _ = _weights(torch, dev, n, k, seed=100 + i)
        x = (torch.randn((m, k), device="cuda") * (1 + i)).half()
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        calls.append(dev.LinearCall(x, w, out))
        refs.append(_two_kernel(dev, torch, x, w, torch.float16))
    prog = dev.Program(calls)
    assert prog.fused
    for _ in range(3):  # replays: the program leaves its workspace reusable
        for c in calls:
            c.out.zero_()
        prog.run()
        torch.cuda.synchronize()
        for c, ref, name in zip(calls, refs, LLAMA13B):
            assert torch.equal(c.out, ref), name


@pytest.mark.parametrize("links", [False, True])
@pytest.mark.parametrize("m", [1, 16, 17, 32, 48, 64])
def test_program_dependency_chain(torch_cuda, dev, m, links):
    """x of each linear is (a column slice of) an earlier linear's output inside the same
    launch: grid-wide completion counters order them; bit-identical to sequential runs,
    eagerly, back to back and from a CUDA graph.  Every decode width (BN = 16/32/64), in
    a workspace of exactly the queried size.  links: the same chain as one launch per
    linear (ody_dev_w4a8_linear_chain, dependent x quantized in-kernel)."""
    torch = torch_cuda
    dims = [(3072, 1024), (1024, 2048), (2048, 1024), (1024, 2048)]  # (n, k); x1 = out0[:, :2048]
    ws = [_weights(torch, dev, n, k, seed=200 + i, scale=0.03)[0] for i, (n, k) in enumerate(dims)]
    x0 = torch.randn((m, 1024), device="cuda").half()
    outs = [torch.empty((m, n), dtype=torch.float16, device="cuda") for n, _ in dims]
    calls = [dev.LinearCall(x0, ws[0], outs[0]),
             dev.LinearCall(outs[0][:, :2048], ws[1], outs[1], dep=0),
             dev.LinearCall(outs[1], ws[2], outs[2], dep=1),
             dev.LinearCall(outs[2], ws[3], outs[3], dep=2)]
    h = x0
    refs = []
    for i, w in enumerate(ws):
        y = _two_kernel(dev, torch, h, w, torch.float16)
        refs.append(y)
        h = y[:, :2048] if i == 0 else y
    prog = dev.Program(calls, links=links)
    assert prog.fused
    st = torch.cuda.Stream()
    for pdl in (False, True):
        for o in outs:
            o.zero_()
        with torch.cuda.stream(st):
            for _ in range(3):
                prog.run(pdl=pdl, stream=st)
        torch.cuda.synchronize()
        for i, (o, r) in enumerate(zip(outs, refs)):
            assert torch.equal(o, r), (pdl, i)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        prog.run(pdl=True, stream=st)
    for o in outs:
        o.zero_()
    for _ in range(4):
        g.replay()
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)


def test_program_fallback_and_errors(torch_cuda, dev):
    """M > 64 falls back to one launch per linear (same results); a forward dependency
    is rejected with EINVAL like the reference's argument checks."""
    torch = torch_cuda
    from paper_2311_09550_b200._lib import OdyError
    w, _, _ = _weights(torch, dev, 256, 512, seed=7)
    x = torch.randn((80, 512), device="cuda").half()
    out = torch.empty((80, 256), dtype=torch.float16, device="cuda")
    prog = dev.Program([dev.LinearCall(x, w, out)])
    assert not prog.fused
    prog.run()
    assert torch.equal(out, _two_kernel(dev, torch, x, w, torch.float16))
    x2 = torch.randn((4, 512), device="cuda").half()
    o2 = torch.empty((4, 256), dtype=torch.float16, device="cuda")
    with pytest.raises(OdyError):
        dev.Program([dev.LinearCall(x2, w, o2, dep=0)]).run()


@pytest.mark.parametrize("links", [False, True])
@pytest.mark.parametrize("m,xdt", [(1, "f16"), (16, "bf16"), (32, "f16"), (64, "bf16")])
def test_program_chain_vs_oracle(m, xdt, links, oracle, torch_cuda, dev):
    """Dependency chain on the dynamic kernel (producer epilogues accumulate the consumer's
    per-token row max; the consumer quantizes its B tiles in-kernel): every linear's
    output bit-exact vs the oracle applied step by step to the same 16-bit intermediates.
    Includes a split-K producer (K = 13824) and a ragged N."""
    torch = torch_cuda
    dt = torch.float16 if xdt == "f16" else torch.bfloat16
    dims = [(3000, 1024), (13824, 1000), (1000, 13824), (640, 1000)]  # x1 = out0[:, 8:1008]
    ws = [_weights(torch, dev, n, k, seed=300 + i, scale=0.05) for i, (n, k) in enumerate(dims)]
    x0 = (torch.randn((m, 1024), device="cuda") * 2).to(dt)
    outs = [torch.empty((m, n), dtype=dt, device="cuda") for n, _ in dims]
    calls = [dev.LinearCall(x0, ws[0][0], outs[0]),
             dev.LinearCall(outs[0][:, 8:1008], ws[1][0], outs[1], dep=0),
             dev.LinearCall(outs[1], ws[2][0], outs[2], dep=1),
             dev.LinearCall(outs[2], ws[3][0], outs[3], dep=2)]
    prog = dev.Program(calls, links=links)
    assert prog.fused
    for rep in range(3):
        for o in outs:
            o.zero_()
        prog.run(pdl=rep > 0)
        torch.cuda.synchronize()
        h = x0.float().cpu().numpy()
        for i, ((n, k), (_, flat, sw), o) in enumerate(zip(dims, ws, outs)):
            xin = np.ascontiguousarray(h[:, 8:1008]) if i == 1 else h
            want, _ = _want(oracle, xin, flat, sw, m, n, k)
            got = o.float().cpu().numpy()
            want16 = torch.from_numpy(want).to(dt).float().numpy()
            assert np.array_equal(bits_of(got), bits_of(want16)), (rep, i, int((got != want16).sum()))
            h = got


def test_program_row_parallel_shards(oracle, torch_cuda, dev):
    """Row-parallel TP building block: two K-shards of one linear in ONE program, each
    quantized with the FULL row's max (absmax_in) and emitting int32 pre-shift partials
    (acc_out).  partial_0 + partial_1 == the unsharded accumulators bit for bit, and the
    K4 epilogue of the sum == the unsharded linear."""
    torch = torch_cuda
    for m in (1, 16, 48):
        n, k = 1000, 2048
        rs = np.random.default_rng(m)
        w = torch.from_numpy(rs.standard_normal((n, k), dtype=np.float32) * 0.05).cuda()
        x = (torch.randn((m, k), device="cuda") * 2).half()
        full = dev.W4Weight.quantize(w)
        shards = [dev.W4Weight.quantize_with_scales(w[:, :k // 2].contiguous(), full.s),
                  dev.W4Weight.quantize_with_scales(w[:, k // 2:].contiguous(), full.s)]
        amax = dev.row_absmax(x)
        accs = [torch.empty((m, n), dtype=torch.int32, device="cuda") for _ in range(2)]
        xs = [x[:, :k // 2].contiguous(), x[:, k // 2:].contiguous()]
        prog = dev.Program([dev.LinearCall(xs[i], shards[i], None, absmax_in=amax, acc_out=accs[i])
                            for i in range(2)])
        assert prog.fused
        prog.run()
        aq = dev.act_quant(x)
        want_acc = dev.w4a8_gemm(aq, full, accumulators=True)
        codes = aq.codes().cpu().numpy()
        flat = full.to_flat().cpu().numpy()
        assert np.array_equal(want_acc.cpu().numpy(), oracle.fast_accumulators(codes, flat, m, n, k, THREADS))
        assert torch.equal(accs[0] + accs[1], want_acc), m
        y = dev.dequant_epilogue(accs[0] + accs[1], aq.s, full.s, torch.float16)
        assert torch.equal(y, dev.w4a8_gemm(aq, full, torch.float16)), m

