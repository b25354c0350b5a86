"""Pins the CPU oracle (oracle/odyssey_oracle.c) to the reference.

Sources of truth, in order:
  1. golden vectors the REFERENCE produced (tests/golden/reference_golden.json,
     made by oracle/gen_golden.cpp compiled from /root/reference/proj/src);
  2. the known-answer tests of the reference's own suite
     (proj/tests/test_gemm.cpp:55-127, test_quantizer.cpp:9-119, pipeline.cpp:149-232);
  3. when oracle/_ref/libodyssey_ref.so exists, the reference C ABI run side by side.
"""
import os

import numpy as np
import pytest

from tests.helpers import bits_of, case_inputs, f32_from_bits, hex_bytes


def test_rng_matches_reference_inputs(oracle, golden):
    """splitmix64 + Box-Muller stream == the reference's (rng.hpp:10-52)."""
    seen = 0
    for case in golden:
        if case["kind"] != "hot_path" or "a_bits" not in case:
            continue
        a, w, _, _ = case_inputs(oracle, case)
        assert np.array_equal(bits_of(a).reshape(-1), np.asarray(case["a_bits"], np.uint32))
        assert np.array_equal(bits_of(w).reshape(-1), np.asarray(case["w_bits"], np.uint32))
        seen += 1
    assert seen >= 20


def test_symmetric_known_answers(oracle, golden):
    """test_quantizer.cpp:31-42, 108-119: codes [7,-4,2], clip -> [7,-8], 1.27 -> 127, zero row."""
    cases = {c["name"]: c for c in golden if c["kind"] == "symmetric"}
    for name, c in cases.items():
        x = f32_from_bits(c["x_bits"])
        g = float(f32_from_bits([c["gamma_bits"]])[0])
        b = float(f32_from_bits([c["beta_bits"]])[0])
        codes, s = oracle.quantize_symmetric(x, c["bits"], g, b)
        assert codes.tolist() == c["codes"], name
        assert int(np.float32(s).view(np.uint32)) == c["scale_bits"], name
    assert cases["w3_bits4"]["codes"] == [7, -4, 2]
    assert cases["clip_half_bits4"]["codes"] == [7, -8]
    assert cases["row_1p27_bits8"]["codes"] == [127, 127, 127]
    assert cases["zero_row_bits8"]["scale_bits"] == int(np.float32(2.0 ** -24).view(np.uint32))


def test_high_nibble_pins(oracle):
    """test_gemm.cpp:55-77: -7 -> -112, 5 -> 80, -8 -> -128, 7 -> 112, -1 -> -16; nibble 0x9."""
    packed = oracle.pack_int4(np.array([-7, 5, -8, 7, 0, -1], np.int8))
    lanes = [oracle.high_nibble_lane(packed, i) for i in range(6)]
    assert lanes == [-112, 80, -128, 112, 0, -16]
    assert packed[0] & 0x0F == 0x09
    allv = np.arange(-8, 8, dtype=np.int8)
    p16 = oracle.pack_int4(allv)
    for i, v in enumerate(allv):
        lane = oracle.high_nibble_lane(p16, i)
        assert lane == v * 16 and (lane >> 4) == v
        assert oracle.int4_get(p16, i) == v


def test_packing_odd_tail(oracle):
    """test_tensor_otf.cpp:82-89: 5 int4 elements -> 3 bytes, last high nibble 0."""
    p = oracle.pack_int4(np.array([1, -1, 7, -8, 3], np.int8))
    assert p.size == 3 and (p[2] >> 4) == 0


def test_scalar_example(oracle):
    """test_gemm.cpp:91-101 / SPEC.md:372: a=[3,-2], w=[-7,5] -> -496, >>4 = -31."""
    a = np.array([[3, -2]], np.int8)
    w = oracle.pack_int4(np.array([-7, 5], np.int8))
    acc = oracle.fast_accumulators(a, w, 1, 1, 2)
    assert acc[0, 0] == -496 and (acc[0, 0] >> 4) == -31
    out = oracle.fast_gemm(a, np.ones(1, np.float32), w, np.ones(1, np.float32), 1, 1, 2)
    assert out[0, 0] == -31.0


def test_exhaustive_scalar_sweep(oracle):
    """pipeline.cpp:152-167: all 16 x 256 (w, a) pairs, (a*lane)>>4 == a*w."""
    for wv in range(-8, 8):
        lane = oracle.high_nibble_lane(oracle.pack_int4(np.array([wv], np.int8)), 0)
        for av in range(-128, 128):
            assert (av * lane) >> 4 == av * wv


@pytest.mark.parametrize("idx", range(25))
def test_hot_path_cases_bit_exact(oracle, golden, idx):
    cases = [c for c in golden if c["kind"] == "hot_path"]
    if idx >= len(cases):
        pytest.skip("fewer cases")
    c = cases[idx]
    a, w, gamma, beta = case_inputs(oracle, c)
    m, n, k = c["m"], c["n"], c["k"]
    codes, sa = oracle.quantize_activations(a)
    assert codes.reshape(-1).tolist() == c["a_codes"]
    assert np.array_equal(bits_of(sa), np.asarray(c["a_scales_bits"], np.uint32))
    wcodes, packed, sw = oracle.quantize_weights(w, gamma, beta)
    assert np.array_equal(packed, hex_bytes(c["w_packed"]))
    assert np.array_equal(bits_of(sw), np.asarray(c["w_scales_bits"], np.uint32))
    acc = oracle.fast_accumulators(codes, packed, m, n, k, threads=2)
    assert np.array_equal(acc.reshape(-1), np.asarray(c["acc16"], np.int64).astype(np.int32))
    assert np.all(acc % 16 == 0)
    # >>4 equals the int64 dot of the codes (test_gemm.cpp:110-127)
    dot = codes.astype(np.int64) @ wcodes.astype(np.int64).T
    assert np.array_equal(acc >> 4, dot)
    out = oracle.fast_gemm(codes, sa, packed, sw, m, n, k, threads=3)
    assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c["out_bits"], np.uint32))
    assert c["counters"] == [m * n * k, m * n, 0, m * n]


def test_bench_generator_checksums(oracle, golden):
    """bench.cpp:78-113 inputs, checksums of every intermediate == the reference's."""
    for c in (x for x in golden if x["kind"] == "checksum"):
        m, n, k = c["m"], c["n"], c["k"]
        a, w = oracle.bench_inputs(c["seed"], m, n, k)
        codes, sa = oracle.quantize_activations(a)
        _, packed, sw = oracle.quantize_weights(w)
        assert str(oracle.fnv1a(codes)) == c["fnv_a_codes"], c["name"]
        assert str(oracle.fnv1a(sa)) == c["fnv_a_scales"], c["name"]
        assert str(oracle.fnv1a(packed)) == c["fnv_w_packed"], c["name"]
        assert str(oracle.fnv1a(sw)) == c["fnv_w_scales"], c["name"]
        out = oracle.fast_gemm(codes, sa, packed, sw, m, n, k, threads=8)
        assert str(oracle.fnv1a(out)) == c["fnv_out"], c["name"]


def test_negative_control_fault_is_detected(oracle):
    """pipeline.cpp:204-210: one flipped nibble must break the accumulator check."""
    r = oracle.rng(5)
    a = oracle.gaussian_fill(r, (7, 40))
    w = oracle.gaussian_fill(r, (9, 40), 0.1)
    codes, _ = oracle.quantize_activations(a)
    wcodes, packed, _ = oracle.quantize_weights(w)
    good = oracle.fast_accumulators(codes, packed, 7, 9, 40)
    bad_packed = packed.copy()
    idx = (7 * 9) % (9 * 40)
    v = oracle.int4_get(bad_packed, idx)
    nv = -8 if v == 7 else v + 1
    byte = bad_packed[idx // 2]
    nib = nv & 0xF
    bad_packed[idx // 2] = (byte & 0xF0) | nib if idx % 2 == 0 else (byte & 0x0F) | (nib << 4)
    bad = oracle.fast_accumulators(codes, bad_packed, 7, 9, 40)
    assert not np.array_equal(good, bad)


REF_SO = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref",
                      "libodyssey_ref.so")


@pytest.mark.skipif(not os.path.exists(REF_SO), reason="reference .so not built here")
def test_oracle_matches_reference_capi(oracle):
    """Side by side with the reference's own C ABI on seeded random shapes."""
    from oracle.oracle import RefCAPI
    ref = RefCAPI()
    r = oracle.rng(77)
    for _ in range(6):
        m, n, k = (oracle.uniform_int(r, 1, 40), oracle.uniform_int(r, 1, 70),
                   oracle.uniform_int(r, 1, 300))
        a = oracle.gaussian_fill(r, (m, k))
        w = oracle.gaussian_fill(r, (n, k), 0.1)
        ah, wh = ref.tensor(a), ref.tensor(w)
        aq, wq = ref.quantize_activations(ah), ref.quantize_weights(wh)
        want = ref.gemm_fast(aq, wq, m, n)
        codes, sa = oracle.quantize_activations(a)
        _, packed, sw = oracle.quantize_weights(w)
        got = oracle.fast_gemm(codes, sa, packed, sw, m, n, k)
        assert np.array_equal(bits_of(got), bits_of(want))
        for h in (aq, wq):
            ref.free_qtensor(h)
        for h in (ah, wh):
            ref.free_tensor(h)


def test_exact_blas_checker_matches_restatement(oracle, golden):
    """The numpy full-size checker (f64 BLAS over integer codes, exact below 2^53) equals
    the C restatement bit for bit: on every golden hot-path case and on a LLaMA-wide row
    block with K = 13824 (the longest reduction the path runs)."""
    for c in (x for x in golden if x["kind"] == "hot_path"):
        a, w, gamma, beta = case_inputs(oracle, c)
        codes, sa = oracle.quantize_activations(a)
        wcodes, packed, sw = oracle.quantize_weights(w, gamma, beta)
        acc = oracle.exact_accumulators(codes, wcodes)
        assert np.array_equal(acc.reshape(-1), np.asarray(c["acc16"], np.int64).astype(np.int32))
        out = oracle.exact_fast_gemm(codes, sa, wcodes, sw)
        assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c["out_bits"], np.uint32))
    r = oracle.rng(4242)
    m, n, k = 5, 96, 13824
    a = oracle.gaussian_fill(r, (m, k)) * 3
    w = oracle.gaussian_fill(r, (n, k), 0.1)
    codes, sa = oracle.quantize_activations(a)
    wcodes, packed, sw = oracle.quantize_weights(w)
    want = oracle.fast_gemm(codes, sa, packed, sw, m, n, k, threads=4)
    assert np.array_equal(bits_of(oracle.exact_fast_gemm(codes, sa, wcodes, sw)), bits_of(want))


def acceptance_trials(oracle, trials=100):
    """proj/tests/acceptance.cpp:80-86: Rng(101); per trial m, n, k = uniform_int(1, 64)
    then a = N(0,1) m x k, w = 0.2 N(0,1) n x k (random_tensor, :49-53)."""
    r = oracle.rng(101)
    out = []
    for _ in range(trials):
        m, n, k = (oracle.uniform_int(r, 1, 64) for _ in range(3))
        a = oracle.gaussian_fill(r, (m, k))
        w = oracle.gaussian_fill(r, (n, k), 0.2)
        out.append((m, n, k, a, w))
    return out


def test_acceptance_matrix_cases_oracle(oracle):
    """acceptance.cpp:65-105 on the oracle: 100 random matrices, acc % 16 == 0 and
    acc >> 4 == the int code dot."""
    for m, n, k, a, w in acceptance_trials(oracle):
        codes, _ = oracle.quantize_activations(a)
        wcodes, packed, _ = oracle.quantize_weights(w)
        acc = oracle.fast_accumulators(codes, packed, m, n, k)
        assert np.all(acc % 16 == 0)
        assert np.array_equal(acc >> 4, codes.astype(np.int64) @ wcodes.astype(np.int64).T)


def _engine_inputs(oracle, c):
    r = oracle.rng(c["seed"])
    a = oracle.gaussian_fill(r, (c["m"], c["k"]))
    w = oracle.gaussian_fill(r, (c["n"], c["k"]), 0.1)
    return a, w


def test_comparison_engines_vs_reference(oracle, golden):
    """gemm.cpp:105-311 restated (W8A8, fine-grained, asymmetric, W4A16) == the
    reference's outputs bit for bit on its own seeded inputs (gen_golden engine_case)."""
    cs = [c for c in golden if c["kind"] == "engines"]
    assert len(cs) >= 3
    for c in cs:
        a, w = _engine_inputs(oracle, c)
        g = c["group"]
        codes, sa = oracle.quantize_activations(a)
        w8, _, s8 = oracle.quantize_weights(w, bits=8)
        assert w8.reshape(-1).tolist() == c["w8_codes"]
        assert np.array_equal(bits_of(s8), np.asarray(c["w8_scales_bits"], np.uint32))
        wg, sg = oracle.quantize_weights_per_group(w, g)
        assert np.array_equal(oracle.pack_int4(wg.reshape(-1)), hex_bytes(c["wg_packed"]))
        assert np.array_equal(bits_of(sg).reshape(-1), np.asarray(c["wg_scales_bits"], np.uint32))
        w4, _, s4 = oracle.quantize_weights(w)
        got = {"w8a8": oracle.gemm_w8a8(codes, sa, w8, s8),
               "finegrained": oracle.gemm_finegrained(codes, sa, wg, sg, g),
               "asymmetric": oracle.gemm_asymmetric(codes, sa, w4, s4),
               "w4a16": oracle.gemm_w4a16(a, wg, sg, g)}
        for key, out in got.items():
            assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c[key + "_out_bits"], np.uint32)), (c["name"], key)
        # FastGEMM == asymmetric bit for bit (test_gemm.cpp:129-149)
        assert c["fast_out_bits"] == c["asymmetric_out_bits"]


def test_lwc_grid_search_vs_reference(oracle, golden):
    """clip.cpp:55-103 restated == the reference's (gamma, beta, mse) bit for bit."""
    for c in (x for x in golden if x["kind"] == "lwc"):
        w = f32_from_bits(c["w_bits"]).reshape(c["n"], c["k"])
        gmin = float(f32_from_bits([c["gmin_bits"]])[0])
        gstep = float(f32_from_bits([c["gstep_bits"]])[0])
        g, b, mb, ma = oracle.optimize_clipping(w, c["bits"], gmin, gstep)
        for got, key in ((g, "gamma_bits"), (b, "beta_bits"), (mb, "mse_before_bits"), (ma, "mse_after_bits")):
            assert np.array_equal(bits_of(got), np.asarray(c[key], np.uint32)), (c["name"], key)
