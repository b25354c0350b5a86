"""Tensor-parallel orchestration (paper_2311_09550_b200/tp.py) over gloo, world_size 2,
on CPU.  The arithmetic comes from an oracle-backed test backend; the sharding, the
MAX all-reduce of the per-token row max, the full-row weight scales and the exact
int32 SUM all-reduce are the product code under test.  Bar: the TP layer output is
bit-identical to the unsharded oracle layer."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleBackend:
    """CPU stand-in with the kernels' exact semantics (test infrastructure)."""

    def __init__(self):
        from oracle.oracle import Oracle
        self.o = Oracle()

    def _w(self, codes, scales):
        codes = np.ascontiguousarray(codes, np.int8)
        return {"codes": codes, "packed": self.o.pack_int4(codes.reshape(-1)),
                "s": np.ascontiguousarray(scales, np.float32), "n": codes.shape[0],
                "k": codes.shape[1]}

    def quantize(self, w):
        codes, _, s = self.o.quantize_weights(w.numpy())
        return self._w(codes, s)

    def full_row_scales(self, w):
        return self.o.quantize_weights(w.numpy())[2]

    def quantize_with_scales(self, w, s):
        codes = self.o.quantize_with_scales(w.numpy(), s, 4)
        return self._w(np.clip(codes, -8, 7), s)

    def row_absmax(self, x):
        return torch.from_numpy(np.abs(x.numpy()).max(axis=1).astype(np.float32))

    def act_quant(self, x, absmax=None):
        xn = x.numpy().astype(np.float32)
        if absmax is None:
            codes, s = self.o.quantize_activations(xn)
        else:
            s = (absmax.numpy().astype(np.float32) / np.float32(127.0)).astype(np.float32)
            s = np.where(s > 0, s, np.float32(2.0 ** -24)).astype(np.float32)
            codes = self.o.quantize_with_scales(xn, s, 8)
        return {"codes": codes, "s": s}

    def scales_of(self, a):
        return a["s"]

    def gemm(self, a, w):
        m, k = a["codes"].shape
        return torch.from_numpy(self.o.fast_gemm(a["codes"], a["s"], w["packed"], w["s"], m,
                                                 w["n"], k))

    def gemm_acc(self, a, w):
        m, k = a["codes"].shape
        return torch.from_numpy(self.o.fast_accumulators(a["codes"], w["packed"], m, w["n"], k))

    def epilogue(self, acc, sa, w):
        acc = acc.numpy()
        sh = (acc >> 4).astype(np.float32)
        scale = (sa[:, None].astype(np.float32) * w["s"][None, :].astype(np.float32)).astype(np.float32)
        return torch.from_numpy((sh * scale).astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_09550_b200.tp import ColumnParallelW4A8Linear, RowParallelW4A8Linear
        be = OracleBackend()
        r = be.o.rng(2024)
        m, n, k = 5, 12, 64
        x = torch.from_numpy(be.o.gaussian_fill(r, (m, k)))
        w = torch.from_numpy(be.o.gaussian_fill(r, (n, k), 0.1))
        row = RowParallelW4A8Linear(w, backend=be)
        y_row = row(x[:, row.k0:row.k1].contiguous())
        col = ColumnParallelW4A8Linear(w, backend=be)
        y_col = col(x)
        gathered = [torch.empty_like(y_col) for _ in range(world)]
        dist.all_gather(gathered, y_col)
        result_q.put((rank, y_row.numpy(), torch.cat(gathered, 1).numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_tp_world2_bit_exact_vs_unsharded():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=150) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    be = OracleBackend()
    r = be.o.rng(2024)
    m, n, k = 5, 12, 64
    x = be.o.gaussian_fill(r, (m, k))
    w = be.o.gaussian_fill(r, (n, k), 0.1)
    codes, sa = be.o.quantize_activations(x)
    _, packed, sw = be.o.quantize_weights(w)
    want = be.o.fast_gemm(codes, sa, packed, sw, m, n, k)
    for rank, y_row, y_col in results:
        assert np.array_equal(y_row.view(np.uint32), want.view(np.uint32)), rank
        assert np.array_equal(y_col.view(np.uint32), want.view(np.uint32)), rank


def test_split_rejects_indivisible():
    from paper_2311_09550_b200.tp import _split
    with pytest.raises(ValueError):
        _split(10, 3, 0)
    assert _split(12, 3, 2) == (8, 12)


def _decoder_ref(o, x, ws, h, inter, world):
    """Unsharded oracle chain with the TP stand-ins (each rank's first width/world
    columns of its own column block), f32 intermediates like OracleBackend."""
    def lin(xx, w):
        codes, sa = o.quantize_activations(np.ascontiguousarray(xx, np.float32))
        _, packed, sw = o.quantize_weights(w)
        return o.fast_gemm(codes, sa, packed, sw, xx.shape[0], w.shape[0], xx.shape[1])

    def cols(y, width):
        blk, wd = y.shape[1] // world, width // world
        return np.concatenate([y[:, r * blk: r * blk + wd] for r in range(world)], 1)
    q = lin(x, ws[0])
    hh = lin(cols(q, h), ws[1])
    gu = lin(hh, ws[2])
    return lin(cols(gu, inter), ws[3])


def _decoder_worker(rank, world, port, result_q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2311_09550_b200.tp import TPDecoderLinears
        be = OracleBackend()
        r = be.o.rng(77)
        h, inter, m = 32, 48, 5
        x = be.o.gaussian_fill(r, (m, h))
        ws = [be.o.gaussian_fill(r, s, 0.1) for s in ((3 * h, h), (h, h), (2 * inter, h), (h, inter))]
        layer = TPDecoderLinears(*[torch.from_numpy(w) for w in ws], backend=be)
        y = layer(torch.from_numpy(x))
        result_q.put((rank, y.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_tp_decoder_layer_world2():
    """The four-linear TP decoder layer (column qkv -> row o -> column gate_up -> row
    down) over gloo, world 2: every rank's output equals the unsharded oracle chain."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_decoder_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=150) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    be = OracleBackend()
    r = be.o.rng(77)
    h, inter, m = 32, 48, 5
    x = be.o.gaussian_fill(r, (m, h))
    ws = [be.o.gaussian_fill(r, s, 0.1) for s in ((3 * h, h), (h, h), (2 * inter, h), (h, inter))]
    want = _decoder_ref(be.o, x, ws, h, inter, world)
    for rank, y in results:
        assert np.array_equal(y.view(np.uint32), want.view(np.uint32)), rank
