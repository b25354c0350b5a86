"""The C-ABI library loads and exports every symbol include/odyssey_b200.h declares;
host-side argument validation behaves like the reference ABI (no GPU needed)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2311_09550_b200 import _lib
from paper_2311_09550_b200._lib import ODY_EINVAL, OdyError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "odyssey_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ody_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build_library()
    return _lib.lib()


def test_header_symbols_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} missing from the ctypes signature table"


def test_reference_hot_path_subset_present():
    """Every hot-path entry of ref odyssey.h keeps its name."""
    ref_hot = ["ody_last_error", "ody_string_free", "ody_set_threads", "ody_tensor_create",
               "ody_tensor_free", "ody_tensor_dims", "ody_tensor_data", "ody_qtensor_free",
               "ody_qtensor_dims", "ody_quantize_weights", "ody_quantize_activations",
               "ody_dequantize", "ody_gemm"]
    assert set(ref_hot) <= set(declared_symbols())


def test_status_and_enum_values_match_reference():
    assert (_lib.ODY_OK, _lib.ODY_EINVAL, _lib.ODY_EIO, _lib.ODY_EPARSE, _lib.ODY_ENUMERIC) == (0, 1, 2, 3, 4)
    assert _lib.ODY_ENGINE_FAST == 3 and _lib.ODY_PER_CHANNEL == 1


def test_null_arguments_einval(L):
    h = ctypes.c_void_p()
    assert L.ody_gemm(3, None, None, None, None, ctypes.byref(h)) == ODY_EINVAL
    assert b"null argument" in L.ody_last_error()
    assert L.ody_quantize_activations(None, ctypes.byref(h)) == ODY_EINVAL
    assert L.ody_quantize_weights(None, 4, 1, 0, None, None, ctypes.byref(h)) == ODY_EINVAL
    assert L.ody_tensor_create(2, 2, None, ctypes.byref(h)) == ODY_EINVAL


def test_host_tensor_roundtrip_and_finite_check():
    from paper_2311_09550_b200.api import Tensor
    x = np.arange(12, dtype=np.float32).reshape(3, 4) / 7
    t = Tensor(x)
    assert t.shape == (3, 4)
    assert np.array_equal(t.numpy(), x)
    bad = x.copy()
    bad[1, 2] = np.nan
    with pytest.raises(OdyError) as e:
        Tensor(bad)
    assert e.value.status == ODY_EINVAL and "non-finite" in e.value.message


def test_weight_scheme_validation_before_device():
    """ref quantize.cpp:75-83 / tensor.cpp:86-110 order; rejected without touching a GPU."""
    from paper_2311_09550_b200.api import quantize_weights
    w = np.ones((4, 6), np.float32)
    with pytest.raises(OdyError, match="bits must be 4 or 8"):
        quantize_weights(w, bits=3)
    with pytest.raises(OdyError, match="does not divide"):
        quantize_weights(w, bits=4, granularity=_lib.ODY_PER_GROUP, group_size=4)
    with pytest.raises(OdyError, match="clip_gamma outside"):
        quantize_weights(w, clip_gamma=np.array([1, 1, 0, 1], np.float32))
    with pytest.raises(OdyError, match="granularity"):
        quantize_weights(w, granularity=_lib.ODY_PER_TOKEN)
    with pytest.raises(OdyError, match="empty tensor"):
        quantize_weights(np.zeros((0, 6), np.float32))


def test_device_layout_sizes(L):
    assert L.ody_dev_a8_bytes(1, 1) == 128 * 128
    assert L.ody_dev_a8_bytes(130, 5120) == 256 * 5120
    assert L.ody_dev_w4_bytes(5120, 5120) == 5120 * 5120 // 2
    assert L.ody_dev_w4_bytes(1, 129) == 128 * 256 // 2
    assert L.ody_dev_workspace_bytes(16, 4096, 4096) > 0


def test_gpu_entry_points_fail_loudly_without_device(L):
    """No CPU fallback: device work without a GPU is an error, never a silent result."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    from paper_2311_09550_b200.api import Tensor, quantize_activations_per_token
    with pytest.raises(OdyError) as e:
        quantize_activations_per_token(Tensor(np.ones((2, 8), np.float32)))
    assert e.value.status == _lib.ODY_EDEVICE


def test_tensor_create_large_copy_and_finite_check():
    """ody_tensor_create (ref tensor.cpp:21-27 + capi.cpp:149): a multi-MB tensor is
    copied exactly (fused copy + finite scan), and a NaN/Inf anywhere -- first, middle,
    last element -- is rejected with EINVAL."""
    import numpy as np

    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import OdyError
    x = np.random.default_rng(0).standard_normal((1024, 1000), dtype=np.float32)
    assert np.array_equal(api.Tensor(x).numpy(), x)
    for pos, bad in ((0, np.inf), (512_000, np.nan), (1_023_999, -np.inf)):
        y = x.copy().reshape(-1)
        y[pos] = bad
        with pytest.raises(OdyError) as e:
            api.Tensor(y.reshape(1024, 1000))
        assert e.value.status == 1


@pytest.mark.parametrize("threads", [1, 3, 0])
def test_tensor_create_strided_and_threads(threads):
    """ody_tensor_create_strided (a column slice, no intermediate copy) == ody_tensor_create
    of the contiguous copy, for every host-pool size (ody_set_threads); a non-finite value
    inside the slice is rejected at any position and piece boundary, one in the columns
    the slice skips is not."""
    import numpy as np

    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import OdyError, lib
    lib().ody_set_threads(threads)
    try:
        big = np.random.default_rng(1).standard_normal((64, 15360), dtype=np.float32)
        for cols in (5120, 13824, 1, 15360):
            sl = big[:, :cols]
            assert np.array_equal(api.Tensor(sl).numpy(), np.ascontiguousarray(sl)), cols
        sl = big[3:40, 100:6100]
        assert np.array_equal(api.Tensor(sl).numpy(), np.ascontiguousarray(sl))
        outside = big.copy()
        outside[:, 6000] = np.nan  # skipped by the slice
        assert np.array_equal(api.Tensor(outside[:, :5120]).numpy(), big[:, :5120])
        for r, c in ((0, 0), (31, 2559), (32, 0), (63, 5119), (17, 4000)):
            y = big.copy()
            y[r, c] = np.inf
            with pytest.raises(OdyError) as e:
                api.Tensor(y[:, :5120])
            assert e.value.status == 1, (r, c)
        flat = np.random.default_rng(2).standard_normal((16, 65536), dtype=np.float32)
        for pos in (0, 131071, 131072, 16 * 65536 - 1):
            y = flat.copy().reshape(-1)
            y[pos] = np.nan
            with pytest.raises(OdyError):
                api.Tensor(y.reshape(16, 65536))
        assert np.array_equal(api.Tensor(flat).numpy(), flat)
    finally:
        lib().ody_set_threads(0)
