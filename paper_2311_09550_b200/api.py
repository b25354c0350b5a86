"""Host-side mirror of the reference's hot-path interface, over the C ABI.

Names, argument meaning and error behaviour follow the reference
(ref proj/src/core/quantize.hpp:31-34, gemm.hpp:70-85, capi.cpp:146-296):

    quantize_activations_per_token(a)          -> QTensor   (per-token INT8, GPU)
    quantize_weights(w, bits=4, per_channel)   -> QTensor   (per-channel INT4, GPU prepack)
    gemm_w4a8_fast(a_q, w_q)                   -> f32 M x N (FastGEMM, GPU)
    gemm_w4a8_fast_accumulators(a_q, w_q)      -> int32 M x N, before the >>4
    run_engine(engine, a_dense, a_q, w_q)      -> only ENGINE_FAST; others raise EINVAL
    dequantize(q)                              -> f32

Every call goes through libodyssey_b200.so; numpy arrays are host buffers.  Errors
raise :class:`OdyError` with the same status the reference ABI returns.
"""
from __future__ import annotations

from ctypes import POINTER, byref, c_float, c_int, c_size_t, c_void_p, cast

import numpy as np

from ._lib import (ODY_ENGINE_ASYMMETRIC, ODY_ENGINE_FAST, ODY_ENGINE_FINEGRAINED,  # noqa: F401
                   ODY_ENGINE_W4A16, ODY_ENGINE_W8A8, ODY_PER_CHANNEL, ODY_PER_GROUP, ODY_PER_TOKEN, OdyError,
                   check, lib, ody_gemm_counters)

__all__ = ["Tensor", "QTensor", "quantize_activations_per_token", "quantize_weights",
           "gemm_w4a8_fast", "gemm_w4a8_fast_accumulators", "run_engine", "dequantize",
           "import_w4", "import_a8", "counters_fast", "matmul_f32", "optimize_clipping",
           "write_tensor", "read_tensor", "write_qtensor", "read_qtensor", "OdyError"]


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(POINTER(c_float))


class Tensor:
    """ody_tensor: a host row-major f32 matrix (ref tensor.hpp:17-41)."""

    def __init__(self, data, _handle=None):
        if _handle is not None:
            self._h = _handle
            return
        arr = np.asarray(data, dtype=np.float32)
        if arr.ndim != 2:
            raise ValueError("Tensor expects a 2-D array")
        h = c_void_p()
        if arr.shape[0] > 1 and arr.strides[1] == 4 and arr.strides[0] % 4 == 0 and arr.strides[0] >= 4 * arr.shape[1]:
            # row-strided (e.g. a column slice): ody_tensor_create_strided copies it straight
            # into the tensor, no intermediate contiguous copy
            check(lib().ody_tensor_create_strided(arr.shape[0], arr.shape[1], arr.strides[0] // 4, _fptr(arr),
                                                  byref(h)))
        else:
            arr = np.ascontiguousarray(arr)
            check(lib().ody_tensor_create(arr.shape[0], arr.shape[1], _fptr(arr), byref(h)))
        self._h = h

    @property
    def shape(self):
        r, c = c_size_t(), c_size_t()
        check(lib().ody_tensor_dims(self._h, byref(r), byref(c)))
        return (r.value, c.value)

    def numpy(self, copy: bool = True) -> np.ndarray:
        """The tensor's data.  copy=False returns a zero-copy view of the (pinned) buffer
        that ody_tensor_data borrows (odyssey.h:68-69); the view keeps this Tensor -- and so
        the buffer -- alive for as long as it exists."""
        rows, cols = self.shape
        p = POINTER(c_float)()
        check(lib().ody_tensor_data(self._h, byref(p)))
        if rows * cols == 0:
            return np.zeros((rows, cols), np.float32)
        if copy:
            return np.ctypeslib.as_array(p, shape=(rows, cols)).copy()
        buf = (c_float * (rows * cols)).from_address(cast(p, c_void_p).value)
        buf._owner = self  # the view's base holds the handle
        return np.frombuffer(buf, dtype=np.float32).reshape(rows, cols)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ody_tensor_free(h)
            self._h = None


class QTensor:
    """ody_qtensor: device-resident codes + scales in the kernel layouts."""

    def __init__(self, handle, kind: str = ""):
        self._h = handle
        self.kind = kind  # informational; the scheme is read from the handle

    @property
    def shape(self):
        r, c = c_size_t(), c_size_t()
        check(lib().ody_qtensor_dims(self._h, byref(r), byref(c)))
        return (r.value, c.value)

    @property
    def scheme(self):
        """(bits, granularity, group_size) -- ref QuantScheme (tensor.hpp:76-90)."""
        b, g, gs = c_int(), c_int(), c_size_t()
        check(lib().ody_qtensor_scheme(self._h, byref(b), byref(g), byref(gs)))
        return b.value, g.value, gs.value

    def export(self):
        """(codes, scales) in the REFERENCE layouts: 8-bit -> int8 [rows, cols];
        4-bit -> flat PackedInt4Buffer bytes ((rows*cols+1)//2,) (ref tensor.hpp:43-64);
        scales f32 [rows * groups_per_row]."""
        rows, cols = self.shape
        bits, gran, gs = self.scheme
        groups = cols // gs if gran == ODY_PER_GROUP else 1
        scales = np.empty(rows * groups, np.float32)
        if bits == 8:
            codes = np.empty((rows, cols), np.int8)
        else:
            codes = np.empty((rows * cols + 1) // 2, np.uint8)
        check(lib().ody_qtensor_export(self._h, codes.ctypes.data_as(c_void_p),
                                       scales.ctypes.data_as(c_void_p)))
        return codes, scales

    def write(self, directory: str) -> None:
        """ody_qtensor_write: the reference's OTF directory (otf.cpp:121-153)."""
        check(lib().ody_qtensor_write(self._h, directory.encode()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().ody_qtensor_free(h)
            self._h = None


def _as_tensor(x) -> Tensor:
    return x if isinstance(x, Tensor) else Tensor(x)


def quantize_activations_per_token(a, bits: int = 8) -> QTensor:
    """ref quantize.cpp:113-132 (INT8 only, as ody_quantize_activations)."""
    if bits != 8:
        raise OdyError(1, "quantize_activations_per_token: the C ABI quantizes INT8 only")
    t = _as_tensor(a)
    h = c_void_p()
    check(lib().ody_quantize_activations(t._h, byref(h)))
    return QTensor(h, "a8")


def quantize_weights(w, bits: int = 4, granularity: int = ODY_PER_CHANNEL, group_size: int = 0,
                     clip_gamma=None, clip_beta=None) -> QTensor:
    """ref quantize.cpp:75-111 through ody_quantize_weights (capi.cpp:207-221)."""
    t = _as_tensor(w)
    g = b = None
    if clip_gamma is not None:
        g = np.ascontiguousarray(clip_gamma, np.float32)
    if clip_beta is not None:
        b = np.ascontiguousarray(clip_beta, np.float32)
    h = c_void_p()
    check(lib().ody_quantize_weights(t._h, bits, granularity, group_size,
                                     _fptr(g) if g is not None else None,
                                     _fptr(b) if b is not None else None, byref(h)))
    return QTensor(h, "w8" if bits == 8 else ("w4g" if granularity == ODY_PER_GROUP else "w4"))


def run_engine(engine: int, a_dense, a_q: QTensor | None, w_q: QTensor, with_counters=False):
    """ref gemm.cpp:313-333 via ody_gemm; returns f32 [M, N] (and counters)."""
    dense = _as_tensor(a_dense) if a_dense is not None else None
    counters = ody_gemm_counters()
    h = c_void_p()
    check(lib().ody_gemm(engine, dense._h if dense else None, a_q._h if a_q else None, w_q._h,
                         byref(counters), byref(h)))
    out = Tensor(None, _handle=h).numpy(copy=False)  # the result buffer itself, no extra copy
    if with_counters:
        return out, {f: getattr(counters, f) for f, _ in ody_gemm_counters._fields_}
    return out


def gemm_w4a8_fast(a_q: QTensor, w_q: QTensor, with_counters=False):
    """ref gemm.cpp:251-279."""
    return run_engine(ODY_ENGINE_FAST, None, a_q, w_q, with_counters)


def gemm_w4a8_fast_accumulators(a_q: QTensor, w_q: QTensor) -> np.ndarray:
    """ref gemm.cpp:229-249: int32 sum a*(16w) per output, before the >>4."""
    m, _ = a_q.shape
    n, _ = w_q.shape
    acc = np.empty((m, n), np.int32)
    check(lib().ody_gemm_accumulators(a_q._h, w_q._h, acc.ctypes.data_as(c_void_p)))
    return acc


def dequantize(q: QTensor) -> np.ndarray:
    """ref quantize.cpp:134-146 via ody_dequantize."""
    h = c_void_p()
    check(lib().ody_dequantize(q._h, byref(h)))
    return Tensor(None, _handle=h).numpy()


def import_w4(n: int, k: int, flat_nibbles: np.ndarray, scales: np.ndarray) -> QTensor:
    """Reference-layout packed INT4 payload + scales -> device prepacked qtensor."""
    flat = np.ascontiguousarray(flat_nibbles, np.uint8)
    sc = np.ascontiguousarray(scales, np.float32)
    if flat.size != (n * k + 1) // 2 or sc.size != n:
        raise OdyError(1, "import_w4: payload or scales size mismatch")
    h = c_void_p()
    check(lib().ody_qtensor_import_w4(n, k, flat.ctypes.data_as(c_void_p),
                                      sc.ctypes.data_as(c_void_p), byref(h)))
    return QTensor(h, "w4")


def import_a8(codes: np.ndarray, scales: np.ndarray) -> QTensor:
    """Reference-layout per-token INT8 codes + scales -> device qtensor."""
    c = np.ascontiguousarray(codes, np.int8)
    sc = np.ascontiguousarray(scales, np.float32)
    if c.ndim != 2 or sc.size != c.shape[0]:
        raise OdyError(1, "import_a8: codes/scales shape mismatch")
    h = c_void_p()
    check(lib().ody_qtensor_import_a8(c.shape[0], c.shape[1], c.ctypes.data_as(c_void_p),
                                      sc.ctypes.data_as(c_void_p), byref(h)))
    return QTensor(h, "a8")


def counters_fast(m: int, n: int, k: int) -> dict:
    """The fast engine's counter formulas (ref gemm.cpp:270-272, test_gemm.cpp:262-267)."""
    return {"int8_mac_ops": m * n * k, "dequant_events": m * n, "zero_point_sub_ops": 0,
            "final_scale_ops": m * n}



def matmul_f32(a, b_transposed) -> np.ndarray:
    """ref tensor.cpp:176-196 (fixed-order f32 dots) via ody_matmul_f32."""
    ta, tb = _as_tensor(a), _as_tensor(b_transposed)
    h = c_void_p()
    check(lib().ody_matmul_f32(ta._h, tb._h, byref(h)))
    return Tensor(None, _handle=h).numpy()


def optimize_clipping(w, bits: int = 4, grid_min: float = 0.5, grid_step: float = 0.01):
    """ref clip.cpp:55-103 LWC grid search (GPU) via ody_optimize_clipping:
    -> (gamma, beta, mse_before, mse_after), one value per channel."""
    t = _as_tensor(w)
    n = t.shape[0]
    outs = [np.empty(n, np.float32) for _ in range(4)]
    check(lib().ody_optimize_clipping(t._h, bits, grid_min, grid_step, *[_fptr(o) for o in outs]))
    return tuple(outs)


def write_tensor(t, path: str) -> None:
    h = _as_tensor(t)  # held: the handle must outlive the call
    check(lib().ody_tensor_write(h._h, path.encode()))


def read_tensor(path: str) -> np.ndarray:
    h = c_void_p()
    check(lib().ody_tensor_read(path.encode(), byref(h)))
    return Tensor(None, _handle=h).numpy()


def write_qtensor(q: QTensor, directory: str) -> None:
    q.write(directory)


def read_qtensor(directory: str) -> QTensor:
    """ody_qtensor_read: an `odyssey quantize` output directory straight into the device
    layouts (ref otf.cpp:164-202): per-channel / per-group INT4 and per-channel INT8
    weights, per-token INT8 activations."""
    h = c_void_p()
    check(lib().ody_qtensor_read(directory.encode(), byref(h)))
    q = QTensor(h)
    bits, gran, _ = q.scheme
    q.kind = "a8" if gran == ODY_PER_TOKEN else ("w8" if bits == 8 else ("w4g" if gran == ODY_PER_GROUP else "w4"))
    return q
