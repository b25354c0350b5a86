"""Megatron-style tensor parallelism for the W4A8 linear.

Column-parallel (qkv, gate/up): W split along N.  Per-channel scales are row-local,
so each rank's shard quantizes exactly as the unsharded weight; activations are
replicated and every rank runs K1 on the same input, giving identical codes.  No
collective -- the N-sharded output feeds the following row-parallel layer.

Row-parallel (o, down): W and x split along K.
  1. local row max|x| (K1 pass 1) -> all_reduce(MAX) of M floats, so every rank
     quantizes its K-slice with the scale of the FULL row (ref quantize.cpp:113-132);
  2. the weight K-shards are quantized with the FULL rows' scales (computed before
     sharding), so the shards concatenate to the unsharded codes;
  3. each rank's FastGEMM emits int32 pre-shift partial accumulators;
  4. all_reduce(SUM) on int32 -- integer addition is exact and order-free, so the
     sum equals the unsharded accumulator bit for bit;
  5. the dequantizing epilogue (K4) runs once on the reduced accumulators.
The result is bit-identical to the single-GPU layer (and to the reference).

Two transports, one arithmetic:
  * ``comm=device.Comm`` (the product path on GPUs): each shard is ONE ody_tp_linear call
    of the C ABI -- K1, the K-shard FastGEMM, NCCL MAX/SUM all-reduces and K4 all
    stream-ordered in the library (CUDA-graph capturable);
  * ``comm=None``: the same steps orchestrated here over torch.distributed with a
    backend for the arithmetic (default: the sm_100a kernels through the C ABI; the CPU
    tests drive it over gloo with the oracle's arithmetic).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class DeviceBackend:
    """The product backend: libodyssey_b200.so kernels on the current CUDA device."""

    def __init__(self, out_dtype=torch.float16):
        from . import device
        self.d = device
        self.out_dtype = out_dtype

    def quantize(self, w):
        return self.d.W4Weight.quantize(w)

    def full_row_scales(self, w):
        return self.d.W4Weight.quantize(w).s

    def quantize_with_scales(self, w, s):
        return self.d.W4Weight.quantize_with_scales(w, s)

    def row_absmax(self, x):
        return self.d.row_absmax(x)

    def act_quant(self, x, absmax=None):
        return self.d.act_quant(x, absmax=absmax)

    def scales_of(self, a):
        return a.s

    def gemm(self, a, w):
        return self.d.w4a8_gemm(a, w, self.out_dtype)

    def gemm_acc(self, a, w):
        return self.d.w4a8_gemm(a, w, accumulators=True)

    def epilogue(self, acc, sa, w):
        return self.d.dequant_epilogue(acc, sa, w.s, self.out_dtype)


def _rank_world(group):
    if group is None and not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _split(total: int, world: int, rank: int):
    if total % world:
        raise ValueError(f"dimension {total} is not divisible by the TP size {world}")
    step = total // world
    return rank * step, (rank + 1) * step


class ColumnParallelW4A8Linear:
    """y[:, shard] = x @ W[shard, :]^T ; output stays N-sharded."""

    def __init__(self, w_full, group=None, backend=None, comm=None, out_dtype=torch.float16):
        self.group = group
        self.comm = comm
        self.out_dtype = out_dtype
        self.rank, self.world = (comm.rank, comm.nranks) if comm is not None else _rank_world(group)
        self.backend = backend or DeviceBackend(out_dtype)
        n = w_full.shape[0]
        self.n0, self.n1 = _split(n, self.world, self.rank)
        self.weight = self.backend.quantize(w_full[self.n0:self.n1].contiguous())

    def __call__(self, x, out=None, stream=None):
        if self.comm is not None:
            from . import device
            return device.tp_linear(self.comm, device.ODY_TP_COLUMN, x, self.weight, self.out_dtype, out=out,
                                    stream=stream)
        a = self.backend.act_quant(x)
        return self.backend.gemm(a, self.weight)


class RowParallelW4A8Linear:
    """y = sum_r x[:, Kr] @ W[:, Kr]^T, reduced exactly in int32 before the epilogue."""

    def __init__(self, w_full, group=None, backend=None, comm=None, out_dtype=torch.float16):
        self.group = group
        self.comm = comm
        self.out_dtype = out_dtype
        self.rank, self.world = (comm.rank, comm.nranks) if comm is not None else _rank_world(group)
        self.backend = backend or DeviceBackend(out_dtype)
        k = w_full.shape[1]
        self.k0, self.k1 = _split(k, self.world, self.rank)
        scales = self.backend.full_row_scales(w_full)  # scale of the FULL row, pre-sharding
        self.weight = self.backend.quantize_with_scales(w_full[:, self.k0:self.k1].contiguous(),
                                                        scales)

    def __call__(self, x_local, out=None, stream=None):
        """x_local: this rank's K-slice [M, K/P] of the activations."""
        if self.comm is not None:
            from . import device
            return device.tp_linear(self.comm, device.ODY_TP_ROW, x_local, self.weight, self.out_dtype, out=out,
                                    stream=stream)
        amax = self.backend.row_absmax(x_local)
        if self.world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=self.group)
        a = self.backend.act_quant(x_local, absmax=amax)
        acc = self.backend.gemm_acc(a, self.weight)
        if self.world > 1:
            dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        return self.backend.epilogue(acc, self.backend.scales_of(a), self.weight)


class TPDecoderLinears:
    """The four linears of one LLaMA decoder layer under TP (config 4/5 of BASELINE.json):
    qkv and gate_up column-parallel, o and down row-parallel.  Attention, norm and SiLU
    are stand-ins (slices), never part of the GEMM metric."""

    def __init__(self, w_qkv, w_o, w_gate_up, w_down, group=None, backend=None, comm=None):
        self.qkv = ColumnParallelW4A8Linear(w_qkv, group, backend, comm)
        self.o = RowParallelW4A8Linear(w_o, group, backend, comm)
        self.gate_up = ColumnParallelW4A8Linear(w_gate_up, group, backend, comm)
        self.down = RowParallelW4A8Linear(w_down, group, backend, comm)
        self.comm = comm
        self._bufs = None

    def shapes(self):
        """(kind, n, k_local) of this rank's four shards, in layer order."""
        return [(0, self.qkv.weight.n, self.qkv.weight.k), (1, self.o.weight.n, self.o.weight.k),
                (0, self.gate_up.weight.n, self.gate_up.weight.k), (1, self.down.weight.n, self.down.weight.k)]

    def __call__(self, x, stream=None):
        if self.comm is not None:
            return self._forward_comm(x, stream)
        qkv = self.qkv(x)                                  # [M, 3H/P] local heads
        h_local = qkv[:, : self.o.k1 - self.o.k0]          # stand-in for local attention
        h = self.o(h_local.contiguous())                   # [M, H] replicated
        gu = self.gate_up(h)                               # [M, 2I/P]
        act_local = gu[:, : self.down.k1 - self.down.k0]   # stand-in for SiLU(g)*u
        return self.down(act_local.contiguous())           # [M, H]

    def _forward_comm(self, x, stream):
        """Preallocated outputs (CUDA-graph friendly): the stand-in slices are views with
        the producer's row stride, read in place by the next shard."""
        m = x.shape[0]
        if self._bufs is None or self._bufs[0].shape[0] != m:
            mk = lambda n: torch.empty((m, n), dtype=torch.float16, device=x.device)  # noqa: E731
            self._bufs = (mk(self.qkv.weight.n), mk(self.o.weight.n), mk(self.gate_up.weight.n),
                          mk(self.down.weight.n))
        qkv, h, gu, y = self._bufs
        self.qkv(x, out=qkv, stream=stream)
        self.o(qkv[:, : self.o.k1 - self.o.k0], out=h, stream=stream)
        self.gate_up(h, out=gu, stream=stream)
        self.down(gu[:, : self.down.k1 - self.down.k0], out=y, stream=stream)
        return y
