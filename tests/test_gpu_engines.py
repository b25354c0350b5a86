"""GPU parity of the comparison engines (ref gemm.cpp:100-311) run
through ody_gemm -- W8A8, ASYMMETRIC (UINT4 + 8 with the zero-point subtract),
FINEGRAINED (per-group float accumulation) and W4A16 -- against

* the REFERENCE's own outputs and counters on its seeded inputs (tests/golden, made by
  oracle/gen_golden.cpp linked against the reference sources): bit for bit;
* the C restatement (oracle/) on acceptance-style random shapes and LLaMA-sized ones:
  bit for bit, counters by the reference's formulas;
* the reference's cross-engine agreement (acceptance.cpp:147-191): FAST == ASYMMETRIC bit
  for bit (test_gemm.cpp:129-149) and FINEGRAINED(g=K) / W8A8 within 1e-5 relative;
* the reference's validation errors (EINVAL) and the OTF round trip of the new formats."""
import numpy as np
import pytest

from tests.helpers import bits_of

pytestmark = pytest.mark.gpu

W4A16, FINE, ASYM, FAST, W8A8 = range(5)
PER_CHANNEL, PER_GROUP = 1, 3


def _inputs(oracle, seed, m, n, k, wstd=0.1):
    r = oracle.rng(seed)
    return oracle.gaussian_fill(r, (m, k)), oracle.gaussian_fill(r, (n, k), wstd)


def _run(api, engine, a, aq, wq):
    return api.run_engine(engine, a, aq, wq, with_counters=True)


def test_engines_vs_reference_golden(oracle, golden):
    from paper_2311_09550_b200 import api
    cs = [c for c in golden if c["kind"] == "engines"]
    assert len(cs) >= 3
    for c in cs:
        r = oracle.rng(c["seed"])
        a = oracle.gaussian_fill(r, (c["m"], c["k"]))
        w = oracle.gaussian_fill(r, (c["n"], c["k"]), 0.1)
        g = c["group"]
        aq = api.quantize_activations_per_token(a)
        w8 = api.quantize_weights(w, 8, PER_CHANNEL, 128)
        wg = api.quantize_weights(w, 4, PER_GROUP, g)
        w4 = api.quantize_weights(w, 4, PER_CHANNEL, 128)
        codes8, s8 = w8.export()
        assert codes8.reshape(-1).tolist() == c["w8_codes"], c["name"]
        assert np.array_equal(bits_of(s8), np.asarray(c["w8_scales_bits"], np.uint32)), c["name"]
        flat_g, sg = wg.export()
        assert flat_g.tobytes().hex() == c["wg_packed"], c["name"]
        assert np.array_equal(bits_of(sg), np.asarray(c["wg_scales_bits"], np.uint32)), c["name"]
        for key, engine, wq, dense in (("w8a8", W8A8, w8, None), ("finegrained", FINE, wg, None),
                                       ("asymmetric", ASYM, w4, None), ("fast", FAST, w4, None),
                                       ("w4a16", W4A16, wg, a)):
            out, cnt = _run(api, engine, dense, aq if engine != W4A16 else None, wq)
            assert np.array_equal(bits_of(out).reshape(-1), np.asarray(c[key + "_out_bits"], np.uint32)), \
                (c["name"], key)
            assert [cnt[f] for f in ("int8_mac_ops", "dequant_events", "zero_point_sub_ops", "final_scale_ops")] \
                == c[key + "_counters"], (c["name"], key)


SHAPES = [(1, 7, 96), (5, 40, 64), (17, 130, 384), (33, 257, 512), (64, 640, 1024), (100, 300, 640),
          (16, 4096, 4096), (200, 512, 256)]


@pytest.mark.parametrize("m,n,k", SHAPES)
def test_integer_engines_vs_oracle(oracle, m, n, k):
    """W8A8 and ASYMMETRIC bit-exact vs the restatement at decode and prefill widths
    (split-K engaged for the small-M shapes); counters by formula."""
    from paper_2311_09550_b200 import api
    a, w = _inputs(oracle, 1000 + m + n + k, m, n, k)
    codes, sa = oracle.quantize_activations(a)
    aq = api.quantize_activations_per_token(a)
    c8, _, s8 = oracle.quantize_weights(w, bits=8)
    c4, _, s4 = oracle.quantize_weights(w)
    out, cnt = _run(api, W8A8, None, aq, api.quantize_weights(w, 8, PER_CHANNEL, 128))
    assert np.array_equal(bits_of(out), bits_of(oracle.gemm_w8a8(codes, sa, c8, s8)))
    assert cnt == {"int8_mac_ops": m * n * k, "dequant_events": m * n, "zero_point_sub_ops": 0,
                   "final_scale_ops": m * n}
    out, cnt = _run(api, ASYM, None, aq, api.quantize_weights(w))
    want = oracle.gemm_asymmetric(codes, sa, c4, s4)
    assert np.array_equal(bits_of(out), bits_of(want))
    assert cnt == {"int8_mac_ops": m * n * k, "dequant_events": m * n, "zero_point_sub_ops": n * k,
                   "final_scale_ops": m * n}
    # FAST and ASYMMETRIC agree bit for bit on the same codes (ref test_gemm.cpp:129-149)
    assert np.array_equal(bits_of(api.gemm_w4a8_fast(aq, api.quantize_weights(w))), bits_of(want))


@pytest.mark.parametrize("m,n,k,g", [(5, 40, 64, 16), (3, 7, 96, 32), (16, 130, 384, 128), (17, 200, 1024, 64),
                                     (64, 256, 768, 96), (40, 300, 4096, 128), (16, 4096, 4096, 128), (2, 9, 75, 75),
                                     (7, 33, 120, 40)])
def test_finegrained_vs_oracle(oracle, m, n, k, g):
    """Per-group float accumulation in the reference's group order, bit-exact; groups that
    are not a multiple of the MMA's 32-k step take the re-laid-out path."""
    from paper_2311_09550_b200 import api
    a, w = _inputs(oracle, 2000 + m + k + g, m, n, k)
    codes, sa = oracle.quantize_activations(a)
    cg, sg = oracle.quantize_weights_per_group(w, g)
    wg = api.quantize_weights(w, 4, PER_GROUP, g)
    flat, got_sg = wg.export()
    assert np.array_equal(flat, oracle.pack_int4(cg.reshape(-1)))
    assert np.array_equal(bits_of(got_sg), bits_of(sg).reshape(-1))
    out, cnt = _run(api, FINE, None, api.quantize_activations_per_token(a), wg)
    assert np.array_equal(bits_of(out), bits_of(oracle.gemm_finegrained(codes, sa, cg, sg, g)))
    assert cnt == {"int8_mac_ops": m * n * k, "dequant_events": m * n * (k // g), "zero_point_sub_ops": 0,
                   "final_scale_ops": 0}
    # per-channel weights through the fine-grained engine: g = K (ref gemm.cpp:128)
    c4, _, s4 = oracle.quantize_weights(w)
    out, _ = _run(api, FINE, None, api.quantize_activations_per_token(a), api.quantize_weights(w))
    assert np.array_equal(bits_of(out), bits_of(oracle.gemm_finegrained(codes, sa, c4, s4.reshape(n, 1), k)))


@pytest.mark.parametrize("m,n,k,g", [(1, 7, 96, 32), (5, 40, 64, 16), (16, 64, 1024, 128), (3, 50, 200, 200)])
def test_w4a16_vs_oracle(oracle, m, n, k, g):
    from paper_2311_09550_b200 import api
    a, w = _inputs(oracle, 3000 + m + k, m, n, k)
    cg, sg = oracle.quantize_weights_per_group(w, g)
    out, cnt = _run(api, W4A16, a, None, api.quantize_weights(w, 4, PER_GROUP, g))
    assert np.array_equal(bits_of(out), bits_of(oracle.gemm_w4a16(a, cg, sg, g)))
    assert cnt["dequant_events"] == m * n * k and cnt["int8_mac_ops"] == 0


def test_cross_engine_agreement_acceptance(oracle):
    """ref acceptance.cpp:147-191: 50 trials (seed 303, m,n in [1,48], k in [1,96], w
    sigma 0.2): fine-grained(g=K), asymmetric and W8A8 (on the widened INT4 codes) agree
    with FAST within 1e-5 relative -- here through the GPU engines."""
    import os
    import tempfile
    from paper_2311_09550_b200 import api
    r = oracle.rng(303)
    for trial in range(50):
        m = oracle.uniform_int(r, 1, 48)
        n = oracle.uniform_int(r, 1, 48)
        k = oracle.uniform_int(r, 1, 96)
        a = oracle.gaussian_fill(r, (m, k))
        w = oracle.gaussian_fill(r, (n, k), 0.2)
        aq = api.quantize_activations_per_token(a)
        w4 = api.quantize_weights(w)
        fast = api.gemm_w4a8_fast(aq, w4)
        fg, _ = _run(api, FINE, None, aq, w4)
        asym, _ = _run(api, ASYM, None, aq, w4)
        # W8A8 on the widened INT4 codes: an OTF 8-bit per-channel tensor with the same scales
        codes, _, s4 = oracle.quantize_weights(w)  # == the GPU's codes (bit-exact quantizer)
        with tempfile.TemporaryDirectory() as d:
            _write_w8_otf(os.path.join(d, "w8"), codes, s4)
            w8 = api.read_qtensor(os.path.join(d, "w8"))
        w8out, _ = _run(api, W8A8, None, aq, w8)
        tol = 1e-5 * max(1.0, float(np.abs(fast).max()))
        assert np.array_equal(bits_of(asym), bits_of(fast)), trial
        assert np.abs(fg - fast).max() <= tol, trial
        assert np.abs(w8out - fast).max() <= tol, trial


def _write_w8_otf(d, codes, scales):
    import os
    os.makedirs(d, exist_ok=True)
    n, k = codes.shape

    def raw(dtype, dims, payload):
        return (b"OTF1" + bytes([dtype, len(dims)]) + b"".join(int(x).to_bytes(8, "little") for x in dims) +
                payload)
    with open(os.path.join(d, "payload.otf"), "wb") as f:
        f.write(raw(1, (n, k), codes.astype(np.int8).tobytes()))
    with open(os.path.join(d, "scales.otf"), "wb") as f:
        f.write(raw(0, (n, 1), np.asarray(scales, np.float32).tobytes()))
    with open(os.path.join(d, "scheme.txt"), "w") as f:
        f.write("bits=8\nsymmetric=1\ngranularity=per_channel\ngroup_size=128\n")


def test_engine_errors_map_like_the_reference(oracle):
    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import OdyError
    a, w = _inputs(oracle, 7, 4, 8, 64)
    aq = api.quantize_activations_per_token(a)
    w4, wg, w8 = (api.quantize_weights(w), api.quantize_weights(w, 4, PER_GROUP, 32),
                  api.quantize_weights(w, 8, PER_CHANNEL, 128))
    for engine, dense, q, wq in ((W8A8, None, aq, w4),       # gemm_w8a8: per-channel 8-bit only
                                 (ASYM, None, aq, wg),       # asymmetric: per-channel 4-bit only
                                 (ASYM, None, aq, w8),
                                 (FINE, None, aq, w8),       # fine-grained: 4-bit weights
                                 (W4A16, a, None, w8),       # w4a16: 4-bit weights
                                 (FAST, None, aq, w8),       # fast: per-channel 4-bit
                                 (FAST, None, aq, wg),
                                 (W8A8, None, w4, w8)):      # activations must be per-token INT8
        with pytest.raises(OdyError) as e:
            api.run_engine(engine, dense, q, wq)
        assert e.value.status == 1
    with pytest.raises(OdyError) as e:  # inner dims disagree
        api.run_engine(W8A8, None, api.quantize_activations_per_token(a[:, :32]), w8)
    assert e.value.status == 1
    with pytest.raises(OdyError):  # group size must divide K (QuantScheme::validate)
        api.quantize_weights(w, 4, PER_GROUP, 48)


def test_new_formats_otf_round_trip_and_dequantize(oracle, tmp_path):
    """ody_qtensor_write / _read of per-group INT4 and per-channel INT8 weights (ref
    otf.cpp:121-202: scales rows x groups, group_size in scheme.txt) and ody_dequantize
    (ref quantize.cpp:134-146) against the restatement's q * S."""
    from paper_2311_09550_b200 import api
    a, w = _inputs(oracle, 11, 6, 40, 256)
    aq = api.quantize_activations_per_token(a)
    for bits, gran, gs, engine in ((4, PER_GROUP, 64, FINE), (8, PER_CHANNEL, 128, W8A8)):
        q = api.quantize_weights(w, bits, gran, gs)
        d = str(tmp_path / f"w{bits}")
        q.write(d)
        with open(d + "/scheme.txt") as f:
            txt = f.read()
        assert f"bits={bits}" in txt and f"group_size={gs}" in txt
        assert ("per_group" if gran == PER_GROUP else "per_channel") in txt
        q2 = api.read_qtensor(d)
        assert q2.scheme == q.scheme
        c1, s1 = q.export()
        c2, s2 = q2.export()
        assert np.array_equal(c1, c2) and np.array_equal(bits_of(s1), bits_of(s2))
        o1, _ = _run(api, engine, None, aq, q)
        o2, _ = _run(api, engine, None, aq, q2)
        assert np.array_equal(bits_of(o1), bits_of(o2))
        deq = api.dequantize(q)
        if bits == 8:
            codes = c1.astype(np.float32)
            want = (codes * s1[:, None]).astype(np.float32)
        else:
            cg, sg = oracle.quantize_weights_per_group(w, gs)
            want = (cg.astype(np.float32) * np.repeat(sg, gs, axis=1)).astype(np.float32)
        assert np.array_equal(bits_of(deq), bits_of(want))
