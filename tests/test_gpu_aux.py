"""GPU parity of the reference's neighbours of the hot path (SURVEY §8f rows 3-4 and the
float oracle), against vectors the REFERENCE produced (tests/golden, oracle/gen_golden.cpp):

* ody_optimize_clipping -- the LWC grid search (ref clip.cpp:55-103) on the GPU: gamma,
  beta, mse_before, mse_after bit-exact, including an outlier and an all-zero channel;
* ody_qtensor_write -- byte-identical OTF files (ref otf.cpp:121-153);
* ody_qtensor_read -- an OTF directory ingested straight into the prepacked device
  layout (ref otf.cpp:164-202), then through the FastGEMM; its error statuses (EIO,
  EPARSE) as the reference maps them (capi.cpp:32-43);
* ody_matmul_f32 -- the fixed-order f32 matmul (ref tensor.cpp:176-196), and the
  reference's C-API agreement test (test_capi.cpp:121-165) replayed through it."""
import os

import numpy as np
import pytest

from tests.helpers import bits_of, f32_from_bits, hex_bytes

pytestmark = pytest.mark.gpu


def cases(golden, kind):
    return [c for c in golden if c["kind"] == kind]


def test_lwc_grid_search_vs_reference(golden):
    from paper_2311_09550_b200 import api
    cs = cases(golden, "lwc")
    assert len(cs) >= 3
    for c in cs:
        w = f32_from_bits(c["w_bits"]).reshape(c["n"], c["k"])
        gmin = float(f32_from_bits([c["gmin_bits"]])[0])
        gstep = float(f32_from_bits([c["gstep_bits"]])[0])
        g, b, before, after = api.optimize_clipping(w, c["bits"], gmin, gstep)
        assert np.array_equal(bits_of(g), np.asarray(c["gamma_bits"], np.uint32)), c["name"]
        assert np.array_equal(bits_of(b), np.asarray(c["beta_bits"], np.uint32)), c["name"]
        assert np.array_equal(bits_of(before), np.asarray(c["mse_before_bits"], np.uint32)), c["name"]
        assert np.array_equal(bits_of(after), np.asarray(c["mse_after_bits"], np.uint32)), c["name"]


def test_lwc_clipped_quantization_feeds_the_kernel(golden, oracle):
    """The searched (gamma, beta) go into ody_quantize_weights; the clipped per-channel
    codes and scales equal the oracle's, and the MSE improved (mse_after <= mse_before)."""
    from paper_2311_09550_b200 import api
    c = cases(golden, "lwc")[0]
    w = f32_from_bits(c["w_bits"]).reshape(c["n"], c["k"])
    g, b, before, after = api.optimize_clipping(w, 4)
    assert np.all(after <= before)
    flat, sw = api.quantize_weights(w, clip_gamma=g, clip_beta=b).export()
    _, packed, want_sw = oracle.quantize_weights(w, g, b)
    assert np.array_equal(flat, packed)
    assert np.array_equal(bits_of(sw), bits_of(want_sw))


def test_otf_write_is_byte_identical(golden, tmp_path):
    from paper_2311_09550_b200 import api
    c = cases(golden, "otf")[0]
    w = f32_from_bits(c["w_bits"]).reshape(3, 5)
    q = api.quantize_weights(w, 4, 1, 128)  # the reference's per_channel(4): group_size 128 in scheme.txt
    d = str(tmp_path / "w.q")
    q.write(d)
    for fname, key in (("payload.otf", "payload_otf"), ("scales.otf", "scales_otf"), ("scheme.txt", "scheme_txt")):
        with open(os.path.join(d, fname), "rb") as f:
            assert np.array_equal(np.frombuffer(f.read(), np.uint8), hex_bytes(c[key])), fname


def test_otf_read_ingests_into_the_kernel(golden, oracle, tmp_path):
    """Reference-written OTF files -> device prepack -> FastGEMM == the oracle."""
    from paper_2311_09550_b200 import api
    c = cases(golden, "otf")[0]
    d = tmp_path / "ref.q"
    d.mkdir()
    for fname, key in (("payload.otf", "payload_otf"), ("scales.otf", "scales_otf"), ("scheme.txt", "scheme_txt")):
        (d / fname).write_bytes(hex_bytes(c[key]).tobytes())
    q = api.read_qtensor(str(d))
    assert q.shape == (3, 5)
    flat, sw = q.export()
    w = f32_from_bits(c["w_bits"]).reshape(3, 5)
    wcodes, packed, want_sw = oracle.quantize_weights(w)
    assert np.array_equal(flat, packed) and np.array_equal(bits_of(sw), bits_of(want_sw))
    r = oracle.rng(9)
    a = oracle.gaussian_fill(r, (4, 5))
    out = api.gemm_w4a8_fast(api.quantize_activations_per_token(a), q)
    codes, sa = oracle.quantize_activations(a)
    assert np.array_equal(bits_of(out), bits_of(oracle.fast_gemm(codes, sa, packed, want_sw, 4, 3, 5)))
    # a round trip of a LLaMA-width weight through disk keeps every byte
    big = oracle.gaussian_fill(r, (640, 5120), 0.1)
    qb = api.quantize_weights(big)
    qb.write(str(tmp_path / "big.q"))
    back = api.read_qtensor(str(tmp_path / "big.q"))
    f1, s1 = qb.export()
    f2, s2 = back.export()
    assert np.array_equal(f1, f2) and np.array_equal(bits_of(s1), bits_of(s2))


def test_otf_errors_map_like_the_reference(tmp_path):
    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import OdyError
    with pytest.raises(OdyError) as e:
        api.read_qtensor(str(tmp_path / "missing"))
    assert e.value.status == 2  # ODY_EIO
    d = tmp_path / "bad"
    d.mkdir()
    (d / "scheme.txt").write_text("bits=4\nsymmetric=1\ngranularity=per_channel\ngroup_size=0\n")
    (d / "payload.otf").write_bytes(b"NOPE garbage")
    with pytest.raises(OdyError) as e:
        api.read_qtensor(str(d))
    assert e.value.status == 3  # ODY_EPARSE (bad magic)
    (d / "payload.otf").write_bytes(b"OTF1\x02\x02" + (3).to_bytes(8, "little") + (5).to_bytes(8, "little") + b"\x00")
    with pytest.raises(OdyError) as e:
        api.read_qtensor(str(d))
    assert e.value.status == 3  # truncated payload
    # dense f32 tensors round-trip too (ody_tensor_write / _read)
    x = np.arange(12, dtype=np.float32).reshape(3, 4) / 7
    api.write_tensor(x, str(tmp_path / "x.otf"))
    assert np.array_equal(api.read_tensor(str(tmp_path / "x.otf")), x)


def test_matmul_f32_bit_exact_and_capi_agreement(oracle):
    """ody_matmul_f32 == the oracle's fixed-order matmul bit for bit; then the reference's
    test_capi.cpp:121-165 (FAST vs matmul_f32 of the dequantized operands, <= 1e-4 rel)."""
    from paper_2311_09550_b200 import api
    r = oracle.rng(31337)
    for m, n, k in ((3, 4, 8), (17, 65, 300), (1, 1, 1)):
        a = oracle.gaussian_fill(r, (m, k))
        b = oracle.gaussian_fill(r, (n, k))
        want = np.empty((m, n), np.float32)
        for i in range(m):  # ref tensor.cpp:189-190, sequential f32
            for j in range(n):
                acc = np.float32(0)
                for kk in range(k):
                    acc = np.float32(acc + np.float32(a[i, kk] * b[j, kk]))
                want[i, j] = acc
        assert np.array_equal(bits_of(api.matmul_f32(a, b)), bits_of(want))
    m, n, k = 3, 4, 8
    av = np.array([0.125 * ((i * 7 % 23) - 11) for i in range(m * k)], np.float32).reshape(m, k)
    wv = np.array([0.03 * ((i * 5 % 17) - 8) for i in range(n * k)], np.float32).reshape(n, k)
    aq, wq = api.quantize_activations_per_token(av), api.quantize_weights(wv)
    out = api.gemm_w4a8_fast(aq, wq)
    ref = api.matmul_f32(api.dequantize(aq), api.dequantize(wq))
    assert np.all(np.abs(out - ref) <= 1e-4 * np.maximum(1.0, np.abs(ref)))


def test_device_w4_quantize_rejects_bad_clip_factors():
    """ody_dev_w4_quantize with device gamma/beta outside (0, 1] returns EINVAL (as the
    reference's QuantScheme::validate / compute_scale_symmetric reject them) instead of
    faulting, and the context stays usable; valid factors give the same scales as the
    host ABI path."""
    import torch

    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200 import device as dev
    from paper_2311_09550_b200._lib import OdyError
    rs = np.random.default_rng(11)
    w = rs.standard_normal((64, 256), dtype=np.float32)
    wd = torch.from_numpy(w).cuda()
    for g, b in ((0.0, 1.0), (1.0, 1.5), (-0.5, 0.5), (float("nan"), 1.0)):
        gd = torch.full((64,), g, device="cuda")
        bd = torch.full((64,), b, device="cuda")
        with pytest.raises(OdyError) as e:
            dev.W4Weight.quantize(wd, gamma=gd, beta=bd)
        assert e.value.status == 1, (g, b)
    ok_g = np.linspace(0.5, 1.0, 64, dtype=np.float32)
    ok_b = np.linspace(1.0, 0.6, 64, dtype=np.float32)
    q = dev.W4Weight.quantize(wd, gamma=torch.from_numpy(ok_g).cuda(), beta=torch.from_numpy(ok_b).cuda())
    torch.cuda.synchronize()
    _, sw = api.quantize_weights(w, clip_gamma=ok_g, clip_beta=ok_b).export()
    assert np.array_equal(bits_of(q.s.cpu().numpy()), bits_of(sw))
