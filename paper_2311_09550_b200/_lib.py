"""ctypes binding of libodyssey_b200.so (include/odyssey_b200.h).

The shared library is built in-tree (``make -C paper_2311_09550_b200`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing or
cannot be loaded, :func:`lib` raises, so no caller can silently run on the CPU.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from ctypes import POINTER, c_char_p, c_float, c_int, c_size_t, c_void_p

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libodyssey_b200.so")

# ody_status (odyssey_b200.h part 1; codes 0-4 identical to ref odyssey.h:21-27)
ODY_OK, ODY_EINVAL, ODY_EIO, ODY_EPARSE, ODY_ENUMERIC, ODY_EDEVICE = range(6)
STATUS_NAMES = {0: "ODY_OK", 1: "ODY_EINVAL", 2: "ODY_EIO", 3: "ODY_EPARSE", 4: "ODY_ENUMERIC",
                5: "ODY_EDEVICE"}
# ody_granularity / ody_engine (ref odyssey.h:29-42)
ODY_PER_TENSOR, ODY_PER_CHANNEL, ODY_PER_TOKEN, ODY_PER_GROUP = range(4)
ODY_ENGINE_W4A16, ODY_ENGINE_FINEGRAINED, ODY_ENGINE_ASYMMETRIC, ODY_ENGINE_FAST, ODY_ENGINE_W8A8 = range(5)
# ody_dtype
ODY_DTYPE_F32, ODY_DTYPE_F16, ODY_DTYPE_BF16 = range(3)


class ody_gemm_counters(ctypes.Structure):
    _fields_ = [("int8_mac_ops", ctypes.c_uint64), ("dequant_events", ctypes.c_uint64),
                ("zero_point_sub_ops", ctypes.c_uint64), ("final_scale_ops", ctypes.c_uint64)]


class ody_linear_desc(ctypes.Structure):
    """include/odyssey_b200.h ody_linear_desc (one linear of a linear program)."""
    _fields_ = [("x", c_void_p), ("x_dtype", c_int), ("ldx", c_size_t), ("w_packed", c_void_p),
                ("s_w", c_void_p), ("m", c_size_t), ("n", c_size_t), ("k", c_size_t), ("out", c_void_p),
                ("out_dtype", c_int), ("s_a_out", c_void_p), ("dep", c_int), ("absmax_in", c_void_p),
                ("acc_out", c_void_p)]


# name -> (restype, argtypes); the complete exported surface of odyssey_b200.h
SIGNATURES = {
    "ody_last_error": (c_char_p, []),
    "ody_string_free": (None, [c_void_p]),
    "ody_set_threads": (None, [c_int]),
    "ody_tensor_create": (c_int, [c_size_t, c_size_t, POINTER(c_float), POINTER(c_void_p)]),
    "ody_tensor_create_strided": (c_int, [c_size_t, c_size_t, c_size_t, POINTER(c_float), POINTER(c_void_p)]),
    "ody_tensor_free": (None, [c_void_p]),
    "ody_tensor_dims": (c_int, [c_void_p, POINTER(c_size_t), POINTER(c_size_t)]),
    "ody_tensor_data": (c_int, [c_void_p, POINTER(POINTER(c_float))]),
    "ody_qtensor_free": (None, [c_void_p]),
    "ody_qtensor_dims": (c_int, [c_void_p, POINTER(c_size_t), POINTER(c_size_t)]),
    "ody_quantize_weights": (c_int, [c_void_p, c_int, c_int, c_size_t, POINTER(c_float),
                                     POINTER(c_float), POINTER(c_void_p)]),
    "ody_quantize_activations": (c_int, [c_void_p, POINTER(c_void_p)]),
    "ody_dequantize": (c_int, [c_void_p, POINTER(c_void_p)]),
    "ody_gemm": (c_int, [c_int, c_void_p, c_void_p, c_void_p, POINTER(ody_gemm_counters),
                         POINTER(c_void_p)]),
    "ody_dev_a8_bytes": (c_size_t, [c_size_t, c_size_t]),
    "ody_dev_w4_bytes": (c_size_t, [c_size_t, c_size_t]),
    "ody_dev_workspace_bytes": (c_size_t, [c_size_t, c_size_t, c_size_t]),
    "ody_dev_act_quant": (c_int, [c_void_p, c_int, c_size_t, c_size_t, c_size_t, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_int, c_void_p]),
    "ody_dev_row_absmax": (c_int, [c_void_p, c_int, c_size_t, c_size_t, c_size_t, c_void_p, c_void_p]),
    "ody_dev_w4_quantize": (c_int, [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p]),
    "ody_dev_w4_quantize_with_scales": (c_int, [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p,
                                                c_void_p]),
    "ody_dev_dequant_epilogue": (c_int, [c_void_p, c_void_p, c_void_p, c_size_t, c_size_t, c_int,
                                         c_void_p, c_void_p]),
    "ody_dev_w4_prepack": (c_int, [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]),
    "ody_dev_w4_unpack": (c_int, [c_void_p, c_size_t, c_size_t, c_void_p, c_void_p]),
    "ody_dev_w4a8_gemm": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_size_t,
                                  c_size_t, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_int,
                                  c_int, c_void_p]),
    "ody_dev_workspace_init": (c_int, [c_void_p, c_size_t, c_void_p]),
    "ody_dev_w4a8_linear": (c_int, [c_void_p, c_int, c_size_t, c_void_p, c_void_p, c_size_t, c_size_t,
                                    c_size_t, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_int,
                                    c_int, c_void_p]),
    "ody_dev_w4a8_linear_pf": (c_int, [c_void_p, c_int, c_size_t, c_void_p, c_void_p, c_size_t, c_size_t,
                                       c_size_t, c_int, c_void_p, c_void_p, c_void_p, c_size_t, c_int,
                                       c_int, c_void_p, c_size_t, c_void_p]),
    "ody_dev_linear_workspace_bytes": (c_size_t, [c_size_t, c_size_t, c_size_t]),
    "ody_dev_program_workspace_bytes": (c_size_t, [c_void_p, c_int]),
    "ody_dev_w4a8_linear_program": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_int, c_int, c_void_p,
                                            c_size_t, c_void_p]),
    "ody_dev_program_is_fused": (c_int, [c_void_p, c_int]),
    "ody_dev_w4a8_linear_chain": (c_int, [c_void_p, c_int, c_void_p, c_size_t, c_int, c_int, c_void_p]),
    "ody_dev_chain_is_links": (c_int, [c_void_p, c_int]),
    "ody_dev_linear_is_fused": (c_int, [c_size_t, c_size_t, c_size_t]),
    "ody_dev_set_linear_mode": (None, [c_int]),
    "ody_dev_set_prefill_min_m": (None, [c_int]),
    "ody_dev_set_trace": (None, [c_void_p]),
    "ody_dev_set_act_trace": (None, [c_void_p]),
    "ody_dev_a8_unpack": (c_int, [c_void_p, c_void_p, c_size_t, c_size_t, c_void_p, c_void_p,
                                  c_void_p]),
    "ody_qtensor_export": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ody_qtensor_import_w4": (c_int, [c_size_t, c_size_t, c_void_p, c_void_p, POINTER(c_void_p)]),
    "ody_qtensor_import_a8": (c_int, [c_size_t, c_size_t, c_void_p, c_void_p, POINTER(c_void_p)]),
    "ody_gemm_dev": (c_int, [c_int, c_void_p, c_size_t, c_void_p, c_void_p, c_void_p, POINTER(ody_gemm_counters),
                             c_void_p]),
    "ody_qtensor_scheme": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int), POINTER(c_size_t)]),
    "ody_gemm_accumulators": (c_int, [c_void_p, c_void_p, c_void_p]),
    "ody_b200_version": (c_char_p, []),
    "ody_tensor_write": (c_int, [c_void_p, c_char_p]),
    "ody_tensor_read": (c_int, [c_char_p, POINTER(c_void_p)]),
    "ody_matmul_f32": (c_int, [c_void_p, c_void_p, POINTER(c_void_p)]),
    "ody_qtensor_write": (c_int, [c_void_p, c_char_p]),
    "ody_qtensor_read": (c_int, [c_char_p, POINTER(c_void_p)]),
    "ody_optimize_clipping": (c_int, [c_void_p, c_int, c_float, c_float, POINTER(c_float), POINTER(c_float),
                                      POINTER(c_float), POINTER(c_float)]),
    "ody_comm_unique_id": (c_int, [c_void_p]),
    "ody_comm_init": (c_int, [c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "ody_comm_free": (c_int, [c_void_p]),
    "ody_comm_dims": (c_int, [c_void_p, POINTER(c_int), POINTER(c_int)]),
    "ody_tp_linear_workspace_bytes": (c_size_t, [c_int, c_size_t, c_size_t, c_size_t]),
    "ody_tp_linear": (c_int, [c_void_p, c_int, c_void_p, c_int, c_size_t, c_void_p, c_void_p, c_size_t,
                              c_size_t, c_size_t, c_int, c_void_p, c_void_p, c_size_t, c_void_p]),
}

_lock = threading.Lock()
_lib = None
_path = LIB_PATH
DIAG_LIB_PATH = os.path.join(PKG_DIR, "libodyssey_b200_diag.so")


def use_diag_library() -> None:
    """tools/ only: load the -DODY_DIAG build (``make -C paper_2311_09550_b200 diag``),
    whose kernels honour the ODY_* ablation / plan-log environment knobs.  Must be
    called before the first lib().  The product library never reads the environment."""
    global _path
    if _lib is not None:
        raise RuntimeError("use_diag_library() after the library was loaded")
    _path = DIAG_LIB_PATH


class OdyError(RuntimeError):
    """A non-OK ody_status, carrying the library's thread-local message.

    Mirrors the reference's ``ody::Error`` as surfaced through its C ABI
    (ref proj/src/capi/capi.cpp:32-58)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


def build_library(quiet: bool = True) -> str:
    """Compile libodyssey_b200.so for sm_100a with nvcc (no GPU needed)."""
    out = subprocess.run(["make", "-C", PKG_DIR, "-j4"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libodyssey_b200.so failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)
    return LIB_PATH


def lib() -> ctypes.CDLL:
    """The loaded library.  Raises if it is missing -- never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_path):
                raise RuntimeError(
                    f"{_path} is missing: the W4A8 path has no CPU fallback. "
                    "Build it with `make -C paper_2311_09550_b200` or __graft_entry__.build().")
            handle = ctypes.CDLL(_path, mode=ctypes.RTLD_LOCAL)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int) -> None:
    if status != ODY_OK:
        msg = lib().ody_last_error()
        raise OdyError(status, msg.decode() if msg else "")
