"""GPU parity: the sm_100a path against the reference's golden vectors and the pinned
CPU oracle, through the C ABI.  Bar: bit-exact codes, scales, packed nibbles, int32
accumulators and f32 outputs; f16/bf16 outputs bit-exact against round-to-nearest
conversion of the exact f32 result (so within 2^-11 / 2^-8 relative of it)."""
import os

import numpy as np
import pytest

from tests.helpers import bits_of, case_inputs, f32_from_bits, hex_bytes

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
    return device


def hot_cases(golden):
    return [c for c in golden if c["kind"] == "hot_path"]


def test_library_is_b200_native():
    from paper_2311_09550_b200._lib import lib
    v = lib().ody_b200_version().decode()
    assert "sm_100a" in v and "B200" in v, v


def test_act_quant_matches_reference(golden, oracle, torch_cuda, dev):
    torch = torch_cuda
    for c in hot_cases(golden):
        a, _, _, _ = case_inputs(oracle, c)
        aq = dev.act_quant(torch.from_numpy(a).cuda())
        codes = aq.codes().cpu().numpy()
        assert codes.reshape(-1).tolist() == c["a_codes"], c["name"]
        assert np.array_equal(bits_of(aq.s.cpu().numpy()), np.asarray(c["a_scales_bits"], np.uint32))


def test_weight_quant_matches_reference(golden, oracle, torch_cuda, dev):
    torch = torch_cuda
    for c in hot_cases(golden):
        _, w, g, b = case_inputs(oracle, c)
        wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda(),
                                   torch.from_numpy(g).cuda() if g is not None else None,
                                   torch.from_numpy(b).cuda() if b is not None else None)
        flat = wq.to_flat().cpu().numpy()
        assert np.array_equal(flat, hex_bytes(c["w_packed"])), c["name"]
        assert np.array_equal(bits_of(wq.s.cpu().numpy()), np.asarray(c["w_scales_bits"], np.uint32))


def test_gemm_matches_reference_golden(golden, oracle, torch_cuda, dev):
    torch = torch_cuda
    for c in hot_cases(golden):
        a, w, g, b = case_inputs(oracle, c)
        aq = dev.act_quant(torch.from_numpy(a).cuda())
        wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda(),
                                   torch.from_numpy(g).cuda() if g is not None else None,
                                   torch.from_numpy(b).cuda() if b is not None else None)
        acc = dev.w4a8_gemm(aq, wq, accumulators=True).cpu().numpy()
        want = np.asarray(c["acc16"], np.int64).astype(np.int32).reshape(c["m"], c["n"])
        if not np.array_equal(acc, want):
            bad = np.argwhere(acc != want)
            pytest.fail(f"{c['name']}: {len(bad)} accumulator mismatches, first {bad[:4].tolist()} "
                        f"got {acc[tuple(bad[0])]} want {want[tuple(bad[0])]}")
        out = dev.w4a8_gemm(aq, wq, torch.float32).cpu().numpy()
        assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c["out_bits"], np.uint32)), c["name"]


def test_c_abi_host_path_matches_reference(golden, oracle):
    """ody_quantize_* + ody_gemm(ODY_ENGINE_FAST) with host buffers (the drop-in)."""
    from paper_2311_09550_b200 import api
    for c in hot_cases(golden):
        a, w, g, b = case_inputs(oracle, c)
        aq = api.quantize_activations_per_token(a)
        wq = api.quantize_weights(w, clip_gamma=g, clip_beta=b)
        out, counters = api.gemm_w4a8_fast(aq, wq, with_counters=True)
        assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c["out_bits"], np.uint32)), c["name"]
        assert [counters[k] for k in ("int8_mac_ops", "dequant_events", "zero_point_sub_ops",
                                      "final_scale_ops")] == c["counters"]
        codes, sa = aq.export()
        assert codes.reshape(-1).tolist() == c["a_codes"]
        flat, sw = wq.export()
        assert np.array_equal(flat, hex_bytes(c["w_packed"]))
        acc = api.gemm_w4a8_fast_accumulators(aq, wq)
        assert np.array_equal(acc.reshape(-1), np.asarray(c["acc16"], np.int64).astype(np.int32))


def test_c_abi_capi_example():
    """test_capi.cpp:121-165: FAST vs matmul_f32(dequant a, dequant w) <= 1e-4 rel."""
    from paper_2311_09550_b200 import api
    m, n, k = 3, 4, 8
    av = np.array([0.125 * ((i * 7 % 23) - 11) for i in range(m * k)], np.float32).reshape(m, k)
    wv = np.array([0.03 * ((i * 5 % 17) - 8) for i in range(n * k)], np.float32).reshape(n, k)
    aq = api.quantize_activations_per_token(av)
    wq = api.quantize_weights(wv)
    out, counters = api.gemm_w4a8_fast(aq, wq, with_counters=True)
    assert counters["int8_mac_ops"] == m * n * k and counters["dequant_events"] == m * n
    ref = api.dequantize(aq) @ api.dequantize(wq).T
    assert np.all(np.abs(out - ref) <= 1e-4 * np.maximum(1.0, np.abs(ref)))


def test_bench_config_checksums(golden, oracle):
    """cfg1 (M=16, N=K=4096) and LLaMA o-proj M=1: every intermediate's FNV-1a equals
    the reference's, through the C ABI."""
    from paper_2311_09550_b200 import api
    for c in (x for x in golden if x["kind"] == "checksum"):
        a, w = oracle.bench_inputs(c["seed"], c["m"], c["n"], c["k"])
        aq = api.quantize_activations_per_token(a)
        wq = api.quantize_weights(w)
        out = api.gemm_w4a8_fast(aq, wq)
        codes, sa = aq.export()
        flat, sw = wq.export()
        assert str(oracle.fnv1a(codes)) == c["fnv_a_codes"], c["name"]
        assert str(oracle.fnv1a(sa)) == c["fnv_a_scales"], c["name"]
        assert str(oracle.fnv1a(flat)) == c["fnv_w_packed"], c["name"]
        assert str(oracle.fnv1a(sw)) == c["fnv_w_scales"], c["name"]
        assert str(oracle.fnv1a(out)) == c["fnv_out"], c["name"]


LLAMA13B = {"qkv": (15360, 5120), "o": (5120, 5120), "gate_up": (27648, 5120),
            "down": (5120, 13824)}


@pytest.mark.parametrize("m", [1, 2, 16, 33, 64, 100, 1024])
@pytest.mark.parametrize("layer", ["o", "down"])
def test_llama_shapes_vs_oracle(m, layer, oracle, torch_cuda, dev):
    torch = torch_cuda
    n, k = LLAMA13B[layer]
    r = oracle.rng(1000 + m)
    a = oracle.gaussian_fill(r, (m, k))
    w = oracle.gaussian_fill(r, (n, k), 0.1)
    codes, sa = oracle.quantize_activations(a)
    wcodes, packed, sw = oracle.quantize_weights(w)
    if m >= 256:  # full-size: the exact f64-BLAS checker (pinned to the C restatement)
        want = oracle.exact_fast_gemm(codes, sa, wcodes, sw)
    else:
        want = oracle.fast_gemm(codes, sa, packed, sw, m, n, k, threads=THREADS)
    aq = dev.act_quant(torch.from_numpy(a).cuda())
    wq = dev.W4Weight.quantize(torch.from_numpy(w).cuda())
    got = dev.w4a8_gemm(aq, wq, torch.float32).cpu().numpy()
    assert np.array_equal(bits_of(got), bits_of(want))
    got16 = dev.w4a8_gemm(aq, wq, torch.float16).cpu()
    assert torch.equal(got16, torch.from_numpy(want).to(torch.float16))
    gotbf = dev.w4a8_gemm(aq, wq, torch.bfloat16).cpu()
    assert torch.equal(gotbf, torch.from_numpy(want).to(torch.bfloat16))


@pytest.mark.parametrize("layer", ["qkv", "gate_up", "down"])
@pytest.mark.parametrize("m", [1, 64, 1024])
def test_llama_full_size_sampled(layer, m, oracle, torch_cuda, dev):
    """Full-size shapes: exact int64 dots on 256 sampled outputs + row-slice invariance
    (the first 8 rows computed alone equal the same rows of the full batch)."""
    torch = torch_cuda
    n, k = LLAMA13B[layer]
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n)
    x = torch.randn((m, k), device="cuda", generator=g, dtype=torch.bfloat16)
    w = torch.randn((n, k), device="cuda", generator=g) * 0.05
    aq = dev.act_quant(x)
    wq = dev.W4Weight.quantize(w)
    acc = dev.w4a8_gemm(aq, wq, accumulators=True)
    codes = aq.codes().cpu().numpy().astype(np.int64)
    flat = wq.to_flat().cpu().numpy()
    rs = np.random.default_rng(m + n)
    ti = rs.integers(0, m, 256)
    ni = rs.integers(0, n, 256)
    acc_np = acc.cpu().numpy()
    for t, j in zip(ti.tolist(), ni.tolist()):
        idx = np.arange(j * k, j * k + k)          # flat element indices of weight row j
        b = flat[idx // 2].astype(np.int64)
        nib = np.where(idx % 2 == 0, b & 0xF, b >> 4)
        wc = np.where(nib >= 8, nib - 16, nib)     # ref tensor.cpp:42-47 sign extension
        assert acc_np[t, j] == 16 * int(codes[t] @ wc), (t, j)
    mm = min(m, 8)
    aq_head = dev.act_quant(x[:mm])
    acc_head = dev.w4a8_gemm(aq_head, wq, accumulators=True)
    assert torch.equal(acc_head, acc[:mm])


def test_split_invariance(oracle, torch_cuda, dev):
    """Results identical for any CTA count (stream-K split points move; int32 sums are
    exact) -- the GPU analogue of test_gemm.cpp:289-308 thread-count invariance."""
    torch = torch_cuda
    x = torch.randn((16, 5120), device="cuda")
    w = torch.randn((5120, 5120), device="cuda") * 0.05
    aq, wq = dev.act_quant(x), dev.W4Weight.quantize(w)
    base = dev.w4a8_gemm(aq, wq, accumulators=True)
    for ctas in (1, 3, 37, 100, 148, 296):
        assert torch.equal(dev.w4a8_gemm(aq, wq, accumulators=True, max_ctas=ctas), base), ctas


def test_input_dtypes_bit_exact(oracle, torch_cuda, dev):
    torch = torch_cuda
    for dt in (torch.float16, torch.bfloat16):
        x = (torch.randn((37, 1000), device="cuda") * 3).to(dt)
        aq = dev.act_quant(x)
        codes, sa = oracle.quantize_activations(x.float().cpu().numpy())
        assert np.array_equal(aq.codes().cpu().numpy(), codes)
        assert np.array_equal(bits_of(aq.s.cpu().numpy()), bits_of(sa))


def test_act_quant_rounding_boundaries(oracle, torch_cuda, dev):
    """Adversarial K1 inputs: x/S lands on / next to every half-integer, where the
    reciprocal fast path must defer to IEEE division to stay bit-exact."""
    torch = torch_cuda
    rs = np.random.default_rng(11)
    rows = []
    for r in range(64):
        absmax = np.float32(rs.uniform(0.01, 100.0))
        S = np.float32(absmax / np.float32(127.0))
        half = (np.arange(-127, 127, dtype=np.float32) + np.float32(0.5)) * S
        row = np.concatenate([half, np.nextafter(half, np.float32(np.inf)),
                              np.nextafter(half, np.float32(-np.inf)),
                              rs.uniform(-absmax, absmax, 256).astype(np.float32)])
        row = np.clip(row, -absmax, absmax).astype(np.float32)
        row[0] = absmax
        rows.append(row)
    x = np.stack(rows).astype(np.float32)
    codes, sa = oracle.quantize_activations(x)
    aq = dev.act_quant(torch.from_numpy(x).cuda())
    assert np.array_equal(bits_of(aq.s.cpu().numpy()), bits_of(sa))
    got = aq.codes().cpu().numpy()
    assert np.array_equal(got, codes), int((got != codes).sum())


def test_absmax_override_row_parallel(oracle, torch_cuda, dev):
    """K-sharded row quantized with the global max gives the full-row codes."""
    torch = torch_cuda
    x = torch.randn((5, 512), device="cuda")
    full = dev.act_quant(x)
    amax = dev.row_absmax(x)
    left = dev.act_quant(x[:, :256].contiguous(), absmax=amax)
    right = dev.act_quant(x[:, 256:].contiguous(), absmax=amax)
    fc = full.codes()
    assert torch.equal(torch.cat([left.codes(), right.codes()], 1), fc)
    assert torch.equal(left.s, full.s)


def test_prepack_roundtrip_and_import(golden, oracle, torch_cuda, dev):
    torch = torch_cuda
    for c in hot_cases(golden)[:8]:
        flat = torch.from_numpy(hex_bytes(c["w_packed"])).cuda()
        sw = torch.from_numpy(f32_from_bits(c["w_scales_bits"])).cuda()
        wq = dev.W4Weight.from_flat(flat, sw, c["n"], c["k"])
        assert torch.equal(wq.to_flat(), flat)


def test_negative_control_corrupted_tile(oracle, torch_cuda, dev):
    """pipeline.cpp:204-210 analogue: one flipped nibble in the prepacked tile breaks parity."""
    torch = torch_cuda
    x = torch.randn((4, 256), device="cuda")
    w = torch.randn((130, 256), device="cuda") * 0.1
    aq, wq = dev.act_quant(x), dev.W4Weight.quantize(w)
    good = dev.w4a8_gemm(aq, wq, accumulators=True)
    wq.packed[1234] ^= 0x10
    bad = dev.w4a8_gemm(aq, wq, accumulators=True)
    assert not torch.equal(good, bad)


def test_workspace_reuse_across_shapes(torch_cuda, dev):
    """Stream-K counters are left at zero by every launch: interleaving shapes that
    share one workspace never leaks partial sums between launches."""
    torch = torch_cuda
    shapes = [(16, 15360, 5120), (16, 5120, 13824), (3, 5120, 5120), (64, 27648, 5120)]
    ws = torch.zeros(max(dev.lib().ody_dev_workspace_bytes(*s) for s in shapes), dtype=torch.uint8,
                     device="cuda")
    ops = []
    for m, n, k in shapes:
        aq = dev.act_quant(torch.randn((m, k), device="cuda"))
        wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.05)
        ops.append((aq, wq))
    first = [dev.w4a8_gemm(a, w, accumulators=True, workspace=ws) for a, w in ops]
    for _ in range(2):
        for (a, w), ref in zip(reversed(ops), reversed(first)):
            assert torch.equal(dev.w4a8_gemm(a, w, accumulators=True, workspace=ws), ref)


def test_error_paths_match_reference():
    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import ODY_EINVAL, OdyError
    aq = api.quantize_activations_per_token(np.ones((2, 8), np.float32))
    wq = api.quantize_weights(np.ones((3, 12), np.float32))
    with pytest.raises(OdyError) as e:  # test_gemm.cpp:310-318
        api.gemm_w4a8_fast(aq, wq)
    assert e.value.status == ODY_EINVAL and "inner dims disagree" in e.value.message
    with pytest.raises(OdyError) as e:
        api.run_engine(1, None, aq, wq)
    assert e.value.status == ODY_EINVAL


@pytest.fixture(params=[0, 1, 2], ids=["two_kernel", "fused_prologue", "decode"])
def linear_mode(request, dev):
    """Every lowering of w4a8_linear: act-quant kernel + GEMM, K1 fused into the GEMM
    prologue (cluster code all-gather), and the cluster split-K decode kernel (default)."""
    dev.lib().ody_dev_set_linear_mode(request.param)
    yield request.param
    dev.lib().ody_dev_set_linear_mode(2)


@pytest.mark.parametrize("m", [1, 3, 16, 17, 64])
@pytest.mark.parametrize("layer", ["qkv", "o", "gate_up", "down"])
def test_fused_linear_matches_oracle(m, layer, linear_mode, oracle, torch_cuda, dev):
    """w4a8_linear (either lowering) == oracle act quant + FastGEMM, bit for bit,
    including the per-token scales it exports."""
    torch = torch_cuda
    n, k = LLAMA13B[layer]
    r = oracle.rng(77 + m)
    a16 = oracle.gaussian_fill(r, (m, k), 1.5).astype(np.float16)  # fp16 x: the fused path
    a = a16.astype(np.float32)
    codes, sa = oracle.quantize_activations(a)
    rs = np.random.default_rng(m + n)
    wt = torch.from_numpy((rs.standard_normal((n, k), dtype=np.float32) * 0.1)).cuda()
    wq = dev.W4Weight.quantize(wt)
    flat = wq.to_flat().cpu().numpy()
    sw = wq.s.cpu().numpy()
    want = oracle.fast_gemm(codes, sa, flat, sw, m, n, k, threads=THREADS)
    sa_out = torch.empty(m, dtype=torch.float32, device="cuda")
    got = dev.w4a8_linear(torch.from_numpy(a16).cuda(), wq, torch.float32, sa_out=sa_out)
    assert np.array_equal(bits_of(sa_out.cpu().numpy()), bits_of(sa))
    got_np = got.cpu().numpy()
    if not np.array_equal(bits_of(got_np), bits_of(want)):
        bad = np.argwhere(got_np != want)
        pytest.fail(f"{len(bad)} mismatches, first {bad[:4].tolist()}")
    fused_upto = {0: 0, 1: 16, 2: 64}[linear_mode]  # decode program: M <= 64
    assert dev.lib().ody_dev_linear_is_fused(m, n, k) == (1 if m <= fused_upto else 0)


def test_fused_linear_input_dtypes(linear_mode, oracle, torch_cuda, dev):
    torch = torch_cuda
    m, n, k = 16, 5120, 5120
    wq = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.05)
    flat, sw = wq.to_flat().cpu().numpy(), wq.s.cpu().numpy()
    for dt in (torch.float16, torch.bfloat16, torch.float32):
        x = (torch.randn((m, k), device="cuda") * 3).to(dt)
        codes, sa = oracle.quantize_activations(x.float().cpu().numpy())
        want = oracle.fast_gemm(codes, sa, flat, sw, m, n, k, threads=THREADS)
        got = dev.w4a8_linear(x, wq, torch.float16)
        assert torch.equal(got.cpu(), torch.from_numpy(want).to(torch.float16))


@pytest.mark.parametrize("m", [24, 48, 64])
def test_repeated_gemm_is_deterministic(m, torch_cuda, dev):
    """Regression for a converter-ring race: two converter groups alternating units over
    an odd-length stage ring could wait one mbarrier phase ahead, pass on the previous
    phase and widen stale weights (whole wrong 128-row tiles, ~1 run in 20 at BN = 64).
    Groups now own ring stages; 40 repeats of each shape must be bit-identical."""
    torch = torch_cuda
    for n, k in ((27648, 5120), (5120, 13824)):
        x = torch.randn((m, k), device="cuda").half()
        w = dev.W4Weight.quantize(torch.randn((n, k), device="cuda") * 0.05)
        aq = dev.act_quant(x)
        base = dev.w4a8_gemm(aq, w, accumulators=True)
        for _ in range(40):
            assert torch.equal(dev.w4a8_gemm(aq, w, accumulators=True), base)
