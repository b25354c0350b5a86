"""Python handle on the CPU parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs import this module.  The product package never does.

    Oracle    -- ctypes over _build/libody_oracle.so, the C restatement
                 (odyssey_oracle.c) of the reference hot path.
    RefCAPI   -- ctypes over _ref/libodyssey_ref.so, the reference itself compiled
                 from /root/reference/proj/src (prebuilt in the dev container).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, byref, c_double, c_float, c_int, c_int64, c_size_t, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libody_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libodyssey_ref.so")


def build(ref: bool = True) -> None:
    """Build the port (and the reference .so when /root/reference is present)."""
    subprocess.run(["make", "-C", HERE, "all" if ref else "port"], check=True,
                   capture_output=True, text=True)


class _Rng(ctypes.Structure):
    _fields_ = [("state", c_uint64), ("spare", c_double), ("have_spare", c_int)]


class Oracle:
    """The C restatement of the reference path (odyssey_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        L.oracle_rng_gaussian.restype = c_double
        L.oracle_rng_uniform.restype = c_double
        L.oracle_rng_uniform_int.restype = c_int64
        L.oracle_rng_uniform_int.argtypes = [POINTER(_Rng), c_int64, c_int64]
        L.oracle_rng_next_u64.restype = c_uint64
        L.oracle_rng_init.argtypes = [POINTER(_Rng), c_uint64]
        L.oracle_rng_fill_gaussian.argtypes = [POINTER(_Rng), c_void_p, c_size_t, c_double]
        L.oracle_compute_scale_symmetric.argtypes = [c_void_p, c_size_t, c_int, c_float, c_float, c_void_p]
        L.oracle_quantize_symmetric.argtypes = [c_void_p, c_size_t, c_int, c_float, c_float, c_void_p, c_void_p]
        L.oracle_quantize_activations_per_token.argtypes = [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]
        L.oracle_quantize_weights_per_channel.argtypes = [c_void_p, c_size_t, c_size_t, c_int, c_void_p,
                                                          c_void_p, c_void_p, c_void_p]
        L.oracle_pack_int4.argtypes = [c_void_p, c_size_t, c_void_p]
        L.oracle_int4_get.argtypes = [c_void_p, c_size_t]
        L.oracle_int4_get.restype = ctypes.c_int8
        L.oracle_unpack_sint4_as_high_nibble.argtypes = [c_void_p, c_size_t]
        L.oracle_unpack_sint4_as_high_nibble.restype = ctypes.c_int8
        L.oracle_gemm_w4a8_fast_accumulators.argtypes = [c_void_p, c_void_p, c_size_t, c_size_t,
                                                         c_size_t, c_int, c_void_p]
        L.oracle_gemm_w4a8_fast.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                            c_size_t, c_size_t, c_int, c_void_p]
        L.oracle_dequantize_rows.argtypes = [c_void_p, c_void_p, c_size_t, c_size_t, c_void_p]
        L.oracle_quantize_with_scale.argtypes = [c_void_p, c_size_t, c_int, c_float, c_void_p]
        L.oracle_quantize_weights_per_group.argtypes = [c_void_p, c_size_t, c_size_t, c_size_t, c_int,
                                                        c_void_p, c_void_p]
        for nm in ("oracle_gemm_w8a8", "oracle_gemm_asymmetric"):
            getattr(L, nm).argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_size_t,
                                       c_void_p]
            getattr(L, nm).restype = None
        L.oracle_gemm_finegrained.argtypes = [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t,
                                              c_size_t, c_size_t, c_void_p]
        L.oracle_gemm_finegrained.restype = None
        L.oracle_gemm_w4a16.argtypes = [c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_size_t, c_size_t,
                                        c_void_p]
        L.oracle_gemm_w4a16.restype = None
        L.oracle_optimize_clipping.argtypes = [c_void_p, c_size_t, c_size_t, c_int, c_float, c_float, c_void_p,
                                               c_void_p, c_void_p, c_void_p]
        L.oracle_fnv1a.argtypes = [c_void_p, c_size_t]
        L.oracle_fnv1a.restype = c_uint64
        self.L = L

    def fnv1a(self, buf) -> int:
        """ref bench.cpp:14-22 over the raw bytes of a numpy array."""
        a = np.ascontiguousarray(buf)
        return int(self.L.oracle_fnv1a(a.ctypes.data, a.nbytes))

    # ---- rng (ref rng.hpp) ----
    def rng(self, seed: int) -> _Rng:
        r = _Rng()
        self.L.oracle_rng_init(byref(r), seed)
        return r

    def gaussian_fill(self, rng: _Rng, shape, stddev: float = 1.0) -> np.ndarray:
        out = np.empty(shape, np.float32)
        self.L.oracle_rng_fill_gaussian(byref(rng), out.ctypes.data, out.size, stddev)
        return out

    def uniform_int(self, rng: _Rng, lo: int, hi: int) -> int:
        return int(self.L.oracle_rng_uniform_int(byref(rng), lo, hi))

    def uniform(self, rng: _Rng) -> float:
        return float(self.L.oracle_rng_uniform(byref(rng)))

    def bench_inputs(self, seed: int, m: int, n: int, k: int):
        """ref bench.cpp:78-83: Rng(seed ^ 0x9d2c5680), a ~ N(0,1) then w ~ 0.1 N(0,1)."""
        r = self.rng(seed ^ 0x9D2C5680)
        a = self.gaussian_fill(r, (m, k), 1.0)
        w = self.gaussian_fill(r, (n, k), 0.1)
        return a, w

    # ---- quantizers ----
    def quantize_symmetric(self, x: np.ndarray, bits: int, gamma=1.0, beta=1.0):
        x = np.ascontiguousarray(x, np.float32)
        codes = np.empty(x.size, np.int8)
        s = c_float()
        rc = self.L.oracle_quantize_symmetric(x.ctypes.data, x.size, bits, gamma, beta,
                                              codes.ctypes.data, byref(s))
        if rc:
            raise ValueError("oracle_quantize_symmetric: invalid argument")
        return codes, np.float32(s.value)

    def quantize_with_scales(self, x: np.ndarray, scales: np.ndarray, bits: int) -> np.ndarray:
        """Per-row codes clamp(round(x/S_r)) under given scales."""
        x = np.ascontiguousarray(x, np.float32)
        codes = np.empty(x.shape, np.int8)
        for r in range(x.shape[0]):
            self.L.oracle_quantize_with_scale(x[r].ctypes.data, x.shape[1], bits, float(scales[r]),
                                              codes[r].ctypes.data)
        return codes

    def quantize_activations(self, a: np.ndarray):
        a = np.ascontiguousarray(a, np.float32)
        m, k = a.shape
        codes = np.empty((m, k), np.int8)
        s = np.empty(m, np.float32)
        if self.L.oracle_quantize_activations_per_token(a.ctypes.data, m, k, codes.ctypes.data,
                                                        s.ctypes.data):
            raise ValueError("oracle: invalid activation tensor")
        return codes, s

    def quantize_weights(self, w: np.ndarray, gamma=None, beta=None, bits: int = 4):
        """-> (codes int8 [n,k], packed bytes ((n*k+1)//2,), scales [n])."""
        w = np.ascontiguousarray(w, np.float32)
        n, k = w.shape
        codes = np.empty((n, k), np.int8)
        s = np.empty(n, np.float32)
        g = np.ascontiguousarray(gamma, np.float32) if gamma is not None else None
        b = np.ascontiguousarray(beta, np.float32) if beta is not None else None
        rc = self.L.oracle_quantize_weights_per_channel(
            w.ctypes.data, n, k, bits, g.ctypes.data if g is not None else None,
            b.ctypes.data if b is not None else None, codes.ctypes.data, s.ctypes.data)
        if rc:
            raise ValueError("oracle: invalid weight tensor / clip")
        return codes, (self.pack_int4(codes.reshape(-1)) if bits == 4 else None), s

    def pack_int4(self, codes: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.int8).reshape(-1)
        out = np.empty((codes.size + 1) // 2, np.uint8)
        if self.L.oracle_pack_int4(codes.ctypes.data, codes.size, out.ctypes.data):
            raise ValueError("oracle_pack_int4: value out of [-8,7]")
        return out

    def int4_get(self, packed: np.ndarray, i: int) -> int:
        return int(self.L.oracle_int4_get(np.ascontiguousarray(packed).ctypes.data, i))

    def high_nibble_lane(self, packed: np.ndarray, i: int) -> int:
        return int(self.L.oracle_unpack_sint4_as_high_nibble(np.ascontiguousarray(packed).ctypes.data, i))

    # ---- FastGEMM ----
    def fast_accumulators(self, a_codes, w_packed, m, n, k, threads: int = 1) -> np.ndarray:
        a_codes = np.ascontiguousarray(a_codes, np.int8)
        w_packed = np.ascontiguousarray(w_packed, np.uint8)
        acc = np.empty((m, n), np.int32)
        if self.L.oracle_gemm_w4a8_fast_accumulators(a_codes.ctypes.data, w_packed.ctypes.data,
                                                     m, n, k, threads, acc.ctypes.data):
            raise ValueError("oracle: invalid gemm shape")
        return acc

    def fast_gemm(self, a_codes, sa, w_packed, sw, m, n, k, threads: int = 1) -> np.ndarray:
        a_codes = np.ascontiguousarray(a_codes, np.int8)
        w_packed = np.ascontiguousarray(w_packed, np.uint8)
        sa = np.ascontiguousarray(sa, np.float32)
        sw = np.ascontiguousarray(sw, np.float32)
        out = np.empty((m, n), np.float32)
        if self.L.oracle_gemm_w4a8_fast(a_codes.ctypes.data, sa.ctypes.data, w_packed.ctypes.data,
                                        sw.ctypes.data, m, n, k, threads, out.ctypes.data):
            raise ValueError("oracle: invalid gemm shape")
        return out

    # ---- comparison engines + LWC (ref gemm.cpp:105-311, clip.cpp:55-103) ----
    def quantize_weights_per_group(self, w: np.ndarray, g: int, bits: int = 4):
        """-> (codes int8 [n,k], scales f32 [n, k/g])."""
        w = np.ascontiguousarray(w, np.float32)
        n, k = w.shape
        codes = np.empty((n, k), np.int8)
        s = np.empty((n, k // g), np.float32)
        if self.L.oracle_quantize_weights_per_group(w.ctypes.data, n, k, g, bits, codes.ctypes.data, s.ctypes.data):
            raise ValueError("oracle: invalid per-group quantization")
        return codes, s

    def _eng(self, fn, *arrays_and_dims):
        return fn(*arrays_and_dims)

    def gemm_w8a8(self, a_codes, sa, w_codes, sw):
        a, w = np.ascontiguousarray(a_codes, np.int8), np.ascontiguousarray(w_codes, np.int8)
        sa, sw = np.ascontiguousarray(sa, np.float32), np.ascontiguousarray(sw, np.float32)
        m, k = a.shape
        n = w.shape[0]
        out = np.empty((m, n), np.float32)
        self.L.oracle_gemm_w8a8(a.ctypes.data, sa.ctypes.data, w.ctypes.data, sw.ctypes.data, m, n, k,
                                out.ctypes.data)
        return out

    def gemm_asymmetric(self, a_codes, sa, w_codes, sw):
        a, w = np.ascontiguousarray(a_codes, np.int8), np.ascontiguousarray(w_codes, np.int8)
        sa, sw = np.ascontiguousarray(sa, np.float32), np.ascontiguousarray(sw, np.float32)
        m, k = a.shape
        n = w.shape[0]
        out = np.empty((m, n), np.float32)
        self.L.oracle_gemm_asymmetric(a.ctypes.data, sa.ctypes.data, w.ctypes.data, sw.ctypes.data, m, n, k,
                                      out.ctypes.data)
        return out

    def gemm_finegrained(self, a_codes, sa, w_codes, wscales, g):
        a, w = np.ascontiguousarray(a_codes, np.int8), np.ascontiguousarray(w_codes, np.int8)
        sa, ws = np.ascontiguousarray(sa, np.float32), np.ascontiguousarray(wscales, np.float32)
        m, k = a.shape
        n = w.shape[0]
        out = np.empty((m, n), np.float32)
        self.L.oracle_gemm_finegrained(a.ctypes.data, sa.ctypes.data, w.ctypes.data, ws.ctypes.data, g, m, n, k,
                                       out.ctypes.data)
        return out

    def gemm_w4a16(self, a, w_codes, wscales, g):
        a, w = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(w_codes, np.int8)
        ws = np.ascontiguousarray(wscales, np.float32)
        m, k = a.shape
        n = w.shape[0]
        out = np.empty((m, n), np.float32)
        self.L.oracle_gemm_w4a16(a.ctypes.data, w.ctypes.data, ws.ctypes.data, g, m, n, k, out.ctypes.data)
        return out

    def optimize_clipping(self, w, bits=4, gmin=0.5, gstep=0.01):
        w = np.ascontiguousarray(w, np.float32)
        n, k = w.shape
        outs = [np.empty(n, np.float32) for _ in range(4)]
        if self.L.oracle_optimize_clipping(w.ctypes.data, n, k, bits, gmin, gstep, *[o.ctypes.data for o in outs]):
            raise ValueError("oracle: invalid clip grid")
        return tuple(outs)

    # ---- full-size checker (numpy, exact) ----
    @staticmethod
    def exact_accumulators(a_codes: np.ndarray, w_codes: np.ndarray) -> np.ndarray:
        """ref gemm.cpp:229-249 at full LLaMA sizes: acc16[i,j] = sum_k a[i,k]*(16 w[j,k]).

        Evaluated as a float64 BLAS matmul of the integer codes: every partial sum is an
        integer of magnitude <= 128*8*2^17 < 2^53, so each f64 product and addition is
        exact in any order and the result equals the reference's int32 sum bit for bit
        (pinned against the C restatement in tests/test_oracle_golden.py)."""
        a = np.ascontiguousarray(a_codes, np.int8).astype(np.float64)
        w = np.ascontiguousarray(w_codes, np.int8).astype(np.float64)
        dot = (a @ w.T).astype(np.int64)
        return (dot * 16).astype(np.int32)

    @staticmethod
    def exact_epilogue(acc16: np.ndarray, sa: np.ndarray, sw: np.ndarray) -> np.ndarray:
        """ref gemm.cpp:269-273: float(acc >> 4) * (sa * sw[j]), each an IEEE f32 RN op."""
        sh = (np.asarray(acc16, np.int32) >> 4).astype(np.float32)
        scale = np.asarray(sa, np.float32)[:, None] * np.asarray(sw, np.float32)[None, :]
        return sh * scale

    def exact_fast_gemm(self, a_codes, sa, w_codes, sw) -> np.ndarray:
        return self.exact_epilogue(self.exact_accumulators(a_codes, w_codes), sa, sw)

    def dequantize_rows(self, codes: np.ndarray, scales: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, np.int8)
        scales = np.ascontiguousarray(scales, np.float32)
        r, c = codes.shape
        out = np.empty((r, c), np.float32)
        self.L.oracle_dequantize_rows(codes.ctypes.data, scales.ctypes.data, r, c, out.ctypes.data)
        return out


class RefCAPI:
    """The reference's own C ABI (libodyssey.so built from its sources)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
        L.ody_tensor_create.argtypes = [c_size_t, c_size_t, c_void_p, POINTER(c_void_p)]
        L.ody_tensor_free.argtypes = [c_void_p]
        L.ody_tensor_data.argtypes = [c_void_p, POINTER(c_void_p)]
        L.ody_qtensor_free.argtypes = [c_void_p]
        L.ody_quantize_activations.argtypes = [c_void_p, POINTER(c_void_p)]
        L.ody_quantize_weights.argtypes = [c_void_p, c_int, c_int, c_size_t, c_void_p, c_void_p,
                                           POINTER(c_void_p)]
        L.ody_gemm.argtypes = [c_int, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_void_p)]
        L.ody_set_threads.argtypes = [c_int]
        L.ody_last_error.restype = ctypes.c_char_p
        self.L = L

    def tensor(self, arr: np.ndarray):
        arr = np.ascontiguousarray(arr, np.float32)
        h = c_void_p()
        rc = self.L.ody_tensor_create(arr.shape[0], arr.shape[1], arr.ctypes.data, byref(h))
        if rc:
            raise RuntimeError(self.L.ody_last_error())
        return h

    def quantize_activations(self, a_h):
        h = c_void_p()
        if self.L.ody_quantize_activations(a_h, byref(h)):
            raise RuntimeError(self.L.ody_last_error())
        return h

    def quantize_weights(self, w_h):
        h = c_void_p()
        if self.L.ody_quantize_weights(w_h, 4, 1, 0, None, None, byref(h)):
            raise RuntimeError(self.L.ody_last_error())
        return h

    def gemm_fast(self, aq_h, wq_h, m: int, n: int) -> np.ndarray:
        h = c_void_p()
        if self.L.ody_gemm(3, None, aq_h, wq_h, None, byref(h)):
            raise RuntimeError(self.L.ody_last_error())
        p = c_void_p()
        self.L.ody_tensor_data(h, byref(p))
        out = np.ctypeslib.as_array(ctypes.cast(p, POINTER(c_float)), shape=(m, n)).copy()
        self.L.ody_tensor_free(h)
        return out

    def free_tensor(self, h):
        self.L.ody_tensor_free(h)

    def free_qtensor(self, h):
        self.L.ody_qtensor_free(h)
