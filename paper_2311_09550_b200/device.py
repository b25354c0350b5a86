"""Device-resident, stream-ordered API (torch tensors as HBM buffers).

PyTorch is only plumbing here: it allocates HBM and owns the streams; every
arithmetic step is one of libodyssey_b200.so's sm_100a kernels, called through the
C ABI (include/odyssey_b200.h part 2) with raw pointers.

    a = act_quant(x)                     # K1: per-token INT8 (ref quantize.cpp:113-132)
    w = W4Weight.quantize(w_f32)         # K2: per-channel INT4 + prepack (ref quantize.cpp:75-111)
    y = w4a8_gemm(a, w, torch.float16)   # K3+K4: FastGEMM + dequant epilogue (ref gemm.cpp:251-279)
    lin = W4A8Linear.from_float(w_f32); y = lin(x)
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from ._lib import (ODY_DTYPE_BF16, ODY_DTYPE_F16, ODY_DTYPE_F32, OdyError, check, lib,
                   ody_linear_desc)

_DT = {torch.float32: ODY_DTYPE_F32, torch.float16: ODY_DTYPE_F16, torch.bfloat16: ODY_DTYPE_BF16}
K_MAX = 1 << 17  # ref gemm.cpp:14


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _require_cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise OdyError(1, f"{name} must be a CUDA tensor (the W4A8 path has no CPU fallback)")


@dataclass
class A8:
    """Per-token INT8 activations in the a8 k-block layout (csrc/layout.h)."""
    q: torch.Tensor        # uint8/int8 buffer of ody_dev_a8_bytes(m, k)
    s: torch.Tensor        # f32 [m]
    m: int
    k: int

    def codes(self, stream=None) -> torch.Tensor:
        """Row-major int8 [m, k] (reference layout) -- inspection only."""
        out = torch.empty((self.m, self.k), dtype=torch.int8, device=self.q.device)
        check(lib().ody_dev_a8_unpack(self.q.data_ptr(), self.s.data_ptr(), self.m, self.k,
                                      out.data_ptr(), None, _stream(stream)))
        return out


@dataclass
class W4Weight:
    """Per-channel INT4 weights prepacked in the w4 tile layout (csrc/layout.h)."""
    packed: torch.Tensor   # uint8 buffer of ody_dev_w4_bytes(n, k)
    s: torch.Tensor        # f32 [n]
    n: int
    k: int

    @staticmethod
    def quantize(w: torch.Tensor, gamma=None, beta=None, stream=None) -> "W4Weight":
        """K2 on the device: f32 [n, k] -> codes clamp(round(w/S), -8, 7) + scales."""
        _require_cuda(w, "w")
        w = w.contiguous().float()
        n, k = w.shape
        if n == 0 or k == 0:
            raise OdyError(1, "quantize_weights: empty tensor")
        packed = torch.empty(lib().ody_dev_w4_bytes(n, k), dtype=torch.uint8, device=w.device)
        s = torch.empty(n, dtype=torch.float32, device=w.device)
        g = gamma.contiguous().float() if gamma is not None else None
        b = beta.contiguous().float() if beta is not None else None
        check(lib().ody_dev_w4_quantize(w.data_ptr(), n, k, g.data_ptr() if g is not None else None,
                                        b.data_ptr() if b is not None else None, packed.data_ptr(),
                                        s.data_ptr(), _stream(stream)))
        return W4Weight(packed, s, n, k)

    @staticmethod
    def quantize_with_scales(w: torch.Tensor, scales: torch.Tensor, stream=None) -> "W4Weight":
        """Codes of ``w`` under given per-row scales (a K-shard of a row-parallel layer
        quantized with its FULL row's scale)."""
        _require_cuda(w, "w")
        w = w.contiguous().float()
        n, k = w.shape
        s = scales.contiguous().float().clone()
        packed = torch.empty(lib().ody_dev_w4_bytes(n, k), dtype=torch.uint8, device=w.device)
        check(lib().ody_dev_w4_quantize_with_scales(w.data_ptr(), n, k, s.data_ptr(),
                                                    packed.data_ptr(), _stream(stream)))
        return W4Weight(packed, s, n, k)

    @staticmethod
    def from_flat(flat: torch.Tensor, scales: torch.Tensor, n: int, k: int,
                  stream=None) -> "W4Weight":
        """Reference PackedInt4Buffer bytes ((n*k+1)//2) + scales -> prepacked."""
        _require_cuda(flat, "flat")
        if flat.numel() != (n * k + 1) // 2 or scales.numel() != n:
            raise OdyError(1, "from_flat: payload or scales size mismatch")
        packed = torch.empty(lib().ody_dev_w4_bytes(n, k), dtype=torch.uint8, device=flat.device)
        check(lib().ody_dev_w4_prepack(flat.contiguous().data_ptr(), n, k, packed.data_ptr(),
                                       _stream(stream)))
        return W4Weight(packed, scales.contiguous().float(), n, k)

    def to_flat(self, stream=None) -> torch.Tensor:
        flat = torch.empty((self.n * self.k + 1) // 2, dtype=torch.uint8, device=self.packed.device)
        check(lib().ody_dev_w4_unpack(self.packed.data_ptr(), self.n, self.k, flat.data_ptr(),
                                      _stream(stream)))
        return flat


def act_quant(x: torch.Tensor, absmax: torch.Tensor | None = None, export_absmax: bool = False,
              pdl: bool = False, stream=None, out: A8 | None = None):
    """K1: per-token symmetric INT8 of a [m, k] f32/f16/bf16 CUDA tensor.

    ``absmax`` (f32 [m]) overrides the row max (row-parallel TP passes the
    all-reduced global max).  Returns an :class:`A8` (and the row max if asked)."""
    _require_cuda(x, "x")
    if x.dim() != 2:
        raise OdyError(1, "act_quant expects a 2-D tensor")
    if x.dtype not in _DT:
        raise OdyError(1, f"act_quant: unsupported dtype {x.dtype}")
    if x.stride(1) != 1:
        x = x.contiguous()
    m, k = x.shape
    if out is None:
        q = torch.empty(lib().ody_dev_a8_bytes(m, k), dtype=torch.uint8, device=x.device)
        s = torch.empty(m, dtype=torch.float32, device=x.device)
        out = A8(q, s, m, k)
    amax_out = torch.empty(m, dtype=torch.float32, device=x.device) if export_absmax else None
    check(lib().ody_dev_act_quant(
        x.data_ptr(), _DT[x.dtype], x.stride(0), m, k, out.q.data_ptr(), out.s.data_ptr(),
        absmax.data_ptr() if absmax is not None else None,
        amax_out.data_ptr() if amax_out is not None else None, int(pdl), _stream(stream)))
    return (out, amax_out) if export_absmax else out


def row_absmax(x: torch.Tensor, stream=None) -> torch.Tensor:
    _require_cuda(x, "x")
    x = x if x.stride(1) == 1 else x.contiguous()
    m, k = x.shape
    out = torch.empty(m, dtype=torch.float32, device=x.device)
    check(lib().ody_dev_row_absmax(x.data_ptr(), _DT[x.dtype], x.stride(0), m, k, out.data_ptr(),
                                   _stream(stream)))
    return out


class Workspace:
    """Stream-K workspace: per-tile counters (zero-initialised; every launch leaves them
    zero) and contributor slots for int32 partial sums."""

    _per_device: dict = {}

    @classmethod
    def for_shapes(cls, shapes, device) -> torch.Tensor:
        """One buffer large enough for every (m, n, k) in `shapes`."""
        ws = None
        for m, n, k in shapes:
            ws = cls.get(m, n, k, device)
        return ws

    _per_device_linear: dict = {}

    @classmethod
    def get_linear(cls, m: int, n: int, k: int, device) -> torch.Tensor:
        """Workspace for w4a8_linear (decode-program counters and split-K sums, GEMM
        stream-K state, a8 scratch).  A separate buffer from ``get``'s: the two layouts
        keep different regions zero."""
        dev = torch.device(device)
        need = lib().ody_dev_linear_workspace_bytes(m, n, k)
        ws = cls._per_device_linear.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
            cls._per_device_linear[dev] = ws
        return ws

    @classmethod
    def get(cls, m: int, n: int, k: int, device) -> torch.Tensor:
        dev = torch.device(device)
        need = lib().ody_dev_workspace_bytes(m, n, k)
        ws = cls._per_device.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
            cls._per_device[dev] = ws
        return ws


def w4a8_gemm(a: A8, w: W4Weight, out_dtype=torch.float16, out: torch.Tensor | None = None,
              accumulators: bool = False, max_ctas: int = 0, pdl: bool = False, stream=None,
              workspace: torch.Tensor | None = None):
    """K3+K4: y[m, n] = float((sum a*16w) >> 4) * (sa*sw), written as out_dtype.

    With ``accumulators=True`` returns the int32 pre-shift accumulators instead
    (ref gemm_w4a8_fast_accumulators, gemm.cpp:229-249)."""
    if a.k != w.k:
        raise OdyError(1, "gemm_w4a8_fast: inner dims disagree")
    if w.k > K_MAX:
        raise OdyError(1, "GEMM: K exceeds the 32-bit accumulator safety bound 2^17")
    dev = a.q.device
    ws = workspace if workspace is not None else Workspace.get(a.m, w.n, w.k, dev)
    acc = None
    if accumulators:
        acc = torch.empty((a.m, w.n), dtype=torch.int32, device=dev)
        y_ptr = None
    else:
        if out is None:
            out = torch.empty((a.m, w.n), dtype=out_dtype, device=dev)
        y_ptr = out.data_ptr()
        out_dtype = out.dtype
    check(lib().ody_dev_w4a8_gemm(
        a.q.data_ptr(), a.s.data_ptr(), w.packed.data_ptr(), w.s.data_ptr(), a.m, w.n, w.k,
        _DT[out_dtype], y_ptr, acc.data_ptr() if acc is not None else None, ws.data_ptr(),
        ws.numel(), max_ctas, int(pdl), _stream(stream)))
    return acc if accumulators else out


def dequant_epilogue(acc: torch.Tensor, sa: torch.Tensor, sw: torch.Tensor, out_dtype=torch.float16,
                     stream=None) -> torch.Tensor:
    """K4 alone on int32 accumulators: float(acc >> 4) * (sa[i] * sw[j])."""
    _require_cuda(acc, "acc")
    m, n = acc.shape
    out = torch.empty((m, n), dtype=out_dtype, device=acc.device)
    check(lib().ody_dev_dequant_epilogue(acc.contiguous().data_ptr(), sa.data_ptr(), sw.data_ptr(),
                                         m, n, _DT[out_dtype], out.data_ptr(), _stream(stream)))
    return out


def w4a8_linear(x: torch.Tensor, w: W4Weight, out_dtype=torch.float16,
                out: torch.Tensor | None = None, sa_out: torch.Tensor | None = None,
                max_ctas: int = 0, pdl: bool = False, stream=None,
                workspace: torch.Tensor | None = None,
                prefetch_next: "W4Weight | None" = None) -> torch.Tensor:
    """The whole W4A8 linear y = x W^T from unquantized x (K1 + K3 + K4).

    Decode widths (m <= 16) run as ONE kernel: the per-token INT8 quantization happens
    inside the GEMM (codes stay in shared memory).  Bit-identical to
    ``w4a8_gemm(act_quant(x), w)``.  ``prefetch_next``: the weights of the linear launched
    next on this stream, L2-prefetched once this kernel's own loads are issued (a hint)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.shape[1] != w.k:
        raise OdyError(1, "gemm_w4a8_fast: inner dims disagree")
    if x.stride(1) != 1:
        x = x.contiguous()
    m, k = x.shape
    if out is None:
        out = torch.empty((m, w.n), dtype=out_dtype, device=x.device)
    if workspace is None:
        workspace = Workspace.get_linear(m, w.n, k, x.device)
    nxt = prefetch_next.packed if prefetch_next is not None else None
    check(lib().ody_dev_w4a8_linear_pf(
        x.data_ptr(), _DT[x.dtype], x.stride(0), w.packed.data_ptr(), w.s.data_ptr(), m, w.n, k,
        _DT[out.dtype], out.data_ptr(), sa_out.data_ptr() if sa_out is not None else None,
        workspace.data_ptr(), workspace.numel(), max_ctas, int(pdl),
        nxt.data_ptr() if nxt is not None else None, nxt.numel() if nxt is not None else 0,
        _stream(stream)))
    return out


@dataclass
class LinearCall:
    """One linear of a program: out = x @ w^T.  ``dep``: index of an earlier linear of
    the same program whose ``out`` is (or contains) this ``x``, or -1."""
    x: torch.Tensor
    w: "W4Weight"
    out: torch.Tensor | None
    dep: int = -1
    sa_out: torch.Tensor | None = None
    absmax_in: torch.Tensor | None = None  # row-parallel TP: the all-reduced per-token max
    acc_out: torch.Tensor | None = None    # int32 [m, n] pre-shift accumulators instead of out


class Program:
    """A reusable linear program (ody_dev_w4a8_linear_program): up to 8 W4A8 linears in ONE
    persistent kernel launch when all are decode-width (m <= 16).  The descriptor array
    is built once; ``run`` launches it (also inside CUDA-graph capture)."""

    def __init__(self, calls: list, workspace: torch.Tensor | None = None,
                 prefetch_next: "W4Weight | None" = None, max_ctas: int = 0, links: bool = False):
        if not 1 <= len(calls) <= 8:
            raise OdyError(1, "a linear program holds 1..8 linears")
        self.calls = list(calls)
        descs = (ody_linear_desc * len(calls))()
        for d, c in zip(descs, self.calls):
            _require_cuda(c.x, "x")
            if c.x.dim() != 2 or c.x.shape[1] != c.w.k or c.x.stride(1) != 1:
                raise OdyError(1, "linear program: x must be [m, k] with unit column stride")
            m = c.x.shape[0]
            tgt = c.acc_out if c.acc_out is not None else c.out
            if tgt is None or tuple(tgt.shape) != (m, c.w.n) or not tgt.is_contiguous():
                raise OdyError(1, "linear program: out (or acc_out) must be a contiguous [m, n] tensor")
            if c.acc_out is not None and c.acc_out.dtype != torch.int32:
                raise OdyError(1, "linear program: acc_out must be int32")
            d.x, d.x_dtype, d.ldx = c.x.data_ptr(), _DT[c.x.dtype], c.x.stride(0)
            d.w_packed, d.s_w = c.w.packed.data_ptr(), c.w.s.data_ptr()
            d.m, d.n, d.k = m, c.w.n, c.w.k
            d.out = c.out.data_ptr() if c.out is not None else None
            d.out_dtype = _DT[c.out.dtype] if c.out is not None else _DT[torch.float16]
            d.s_a_out = c.sa_out.data_ptr() if c.sa_out is not None else None
            d.dep = c.dep
            d.absmax_in = c.absmax_in.data_ptr() if c.absmax_in is not None else None
            d.acc_out = c.acc_out.data_ptr() if c.acc_out is not None else None
        self.descs = descs
        need = lib().ody_dev_program_workspace_bytes(descs, len(calls))
        if workspace is None or workspace.numel() < need:
            workspace = torch.zeros(need, dtype=torch.uint8, device=self.calls[0].x.device)
        self.workspace = workspace
        self.prefetch_next = prefetch_next
        self.max_ctas = max_ctas
        # links: a dependency chain as one launch per linear (ody_dev_w4a8_linear_chain),
        # each dependent launch quantizing its x in-kernel
        self.links = links

    @property
    def fused(self) -> bool:
        if self.links:
            return bool(lib().ody_dev_chain_is_links(self.descs, len(self.calls)))
        return bool(lib().ody_dev_program_is_fused(self.descs, len(self.calls)))

    def run(self, pdl: bool = False, stream=None):
        if self.links:
            check(lib().ody_dev_w4a8_linear_chain(self.descs, len(self.calls), self.workspace.data_ptr(),
                                                  self.workspace.numel(), self.max_ctas, int(pdl),
                                                  _stream(stream)))
            return [c.acc_out if c.acc_out is not None else c.out for c in self.calls]
        nxt = self.prefetch_next.packed if self.prefetch_next is not None else None
        check(lib().ody_dev_w4a8_linear_program(
            self.descs, len(self.calls), self.workspace.data_ptr(), self.workspace.numel(), self.max_ctas,
            int(pdl), nxt.data_ptr() if nxt is not None else None, nxt.numel() if nxt is not None else 0,
            _stream(stream)))
        return [c.acc_out if c.acc_out is not None else c.out for c in self.calls]


class W4A8Linear:
    """A linear layer on the FastGEMM path: y = x @ W^T with W4 per-channel weights
    and dynamic per-token A8 activations (the paper's W4A8 linear)."""

    def __init__(self, weight: W4Weight, out_dtype=torch.float16):
        self.weight = weight
        self.out_dtype = out_dtype

    @classmethod
    def from_float(cls, w: torch.Tensor, out_dtype=torch.float16, gamma=None, beta=None):
        return cls(W4Weight.quantize(w, gamma, beta), out_dtype)

    @property
    def in_features(self):
        return self.weight.k

    @property
    def out_features(self):
        return self.weight.n

    def __call__(self, x: torch.Tensor, pdl: bool = False) -> torch.Tensor:
        return w4a8_linear(x, self.weight, self.out_dtype, pdl=pdl)


# ------------------------------------------------------------------ tensor parallelism
ODY_TP_COLUMN, ODY_TP_ROW = 0, 1
COMM_ID_BYTES = 128


class Comm:
    """An ody_comm (C ABI part 4): an NCCL communicator over this rank's current device.
    Rank 0 makes ``unique_id()``; every rank passes the same bytes to ``Comm(...)``."""

    def __init__(self, nranks: int, rank: int, uid: bytes):
        import ctypes
        if len(uid) != COMM_ID_BYTES:
            raise OdyError(1, "ody_comm_init: the unique id is 128 bytes")
        self._uid = ctypes.create_string_buffer(uid, COMM_ID_BYTES)
        h = ctypes.c_void_p()
        check(lib().ody_comm_init(nranks, rank, self._uid, ctypes.byref(h)))
        self.handle = h
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        import ctypes
        buf = ctypes.create_string_buffer(COMM_ID_BYTES)
        check(lib().ody_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Bootstrap over an initialised torch.distributed group (the id travels as an
        object broadcast from rank 0)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
        return cls(world, rank, box[0])

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            check(lib().ody_comm_free(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TPWorkspace:
    """Per-device workspace for ody_tp_linear (zeroed once, reused)."""

    _per_device: dict = {}

    @classmethod
    def get(cls, kind: int, m: int, n: int, k_local: int, device) -> torch.Tensor:
        dev = torch.device(device)
        need = lib().ody_tp_linear_workspace_bytes(kind, m, n, k_local)
        ws = cls._per_device.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 1 << 20), dtype=torch.uint8, device=dev)
            cls._per_device[dev] = ws
        return ws


def tp_linear(comm: Comm, kind: int, x: torch.Tensor, w: W4Weight, out_dtype=torch.float16,
              out: torch.Tensor | None = None, workspace: torch.Tensor | None = None, stream=None):
    """One Megatron shard through ody_tp_linear: COLUMN (this rank's N rows, no
    collective) or ROW (this rank's K columns; MAX + exact int32 SUM all-reduces)."""
    _require_cuda(x, "x")
    if x.dim() != 2 or x.shape[1] != w.k or x.stride(1) != 1:
        raise OdyError(1, "ody_tp_linear: x must be [m, k_local] with unit column stride")
    m = x.shape[0]
    if out is None:
        out = torch.empty((m, w.n), dtype=out_dtype, device=x.device)
    if workspace is None:
        workspace = TPWorkspace.get(kind, m, w.n, w.k, x.device)
    check(lib().ody_tp_linear(comm.handle, kind, x.data_ptr(), _DT[x.dtype], x.stride(0), w.packed.data_ptr(),
                              w.s.data_ptr(), m, w.n, w.k, _DT[out.dtype], out.data_ptr(), workspace.data_ptr(),
                              workspace.numel(), _stream(stream)))
    return out
