"""GPU parity of the tensor-parallel device path (paper_2311_09550_b200/tp.py,
C ABI part 4), bit-exact against the unsharded oracle:

* ody_tp_linear through an NCCL ody_comm at world = 1 (COLUMN and ROW), eager and from a
  CUDA graph;
* TPDecoderLinears on the comm (C-ABI) transport at world = 1 vs the oracle chain;
* the torch.distributed transport with the product DeviceBackend at world = 1 and at
  world = 2 over gloo, two processes sharing cuda:0 (NCCL refuses two ranks on one GPU);
* the TP building blocks alone: ody_dev_w4_quantize_with_scales and
  ody_dev_dequant_epilogue vs the oracle."""
import os
import socket

import numpy as np
import pytest

from tests.helpers import bits_of

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def dev():
    from paper_2311_09550_b200 import device
    return device


@pytest.fixture(scope="module")
def comm1(dev):
    c = dev.Comm(1, 0, dev.Comm.unique_id())
    yield c
    c.close()


def _oracle_linear(oracle, x32, w32):
    codes, sa = oracle.quantize_activations(x32)
    wcodes, _, sw = oracle.quantize_weights(w32)
    return oracle.exact_fast_gemm(codes, sa, wcodes, sw)


def test_quantize_with_scales_and_epilogue_vs_oracle(oracle, torch_cuda, dev):
    torch = torch_cuda
    r = oracle.rng(55)
    m, n, k = 9, 300, 1000
    x = oracle.gaussian_fill(r, (m, k)) * 3
    w = oracle.gaussian_fill(r, (n, k), 0.1)
    wcodes, _, sw = oracle.quantize_weights(w)
    # K-shard [256, 1000) quantized with the FULL rows' scales == the full codes' columns
    shard = dev.W4Weight.quantize_with_scales(torch.from_numpy(np.ascontiguousarray(w[:, 256:])).cuda(),
                                              torch.from_numpy(sw).cuda())
    flat = shard.to_flat().cpu().numpy()
    want_flat = oracle.pack_int4(np.ascontiguousarray(wcodes[:, 256:]).reshape(-1))
    assert np.array_equal(flat, want_flat)
    assert np.array_equal(oracle.quantize_with_scales(w[:, 256:], sw, 4), wcodes[:, 256:])
    # K4 alone on int32 accumulators
    codes, sa = oracle.quantize_activations(x)
    acc = oracle.exact_accumulators(codes, wcodes)
    want = oracle.exact_epilogue(acc, sa, sw)
    for dt, npdt in ((torch.float32, np.float32), (torch.float16, np.float16), (torch.bfloat16, None)):
        got = dev.dequant_epilogue(torch.from_numpy(acc).cuda(), torch.from_numpy(sa).cuda(),
                                   torch.from_numpy(sw).cuda(), dt)
        ref = torch.from_numpy(want).to(dt)
        assert torch.equal(got.cpu(), ref), dt


@pytest.mark.parametrize("m", [1, 16, 64, 200])
def test_tp_linear_world1_vs_oracle(m, oracle, torch_cuda, dev, comm1):
    torch = torch_cuda
    rs = np.random.default_rng(m)
    n, k = 1280, 2048
    x = (rs.standard_normal((m, k), dtype=np.float32) * 2).astype(np.float16)
    w = (rs.standard_normal((n, k), dtype=np.float32) * 0.05).astype(np.float32)
    want = _oracle_linear(oracle, x.astype(np.float32), w).astype(np.float16)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    wq = dev.W4Weight.quantize(wd)
    for kind in (dev.ODY_TP_COLUMN, dev.ODY_TP_ROW):
        y = dev.tp_linear(comm1, kind, xd, wq)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy().view(np.uint16), want.view(np.uint16)), (m, kind)
    # stream-ordered and graph-capturable (NCCL inside the capture)
    st = torch.cuda.Stream()
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    with torch.cuda.stream(st):
        dev.tp_linear(comm1, dev.ODY_TP_ROW, xd, wq, out=out, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        dev.tp_linear(comm1, dev.ODY_TP_ROW, xd, wq, out=out, stream=st)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint16), want.view(np.uint16))


def _decoder_weights(rs, h, inter):
    mk = lambda n, k: (rs.standard_normal((n, k), dtype=np.float32) * 0.05).astype(np.float32)  # noqa: E731
    return [mk(3 * h, h), mk(h, h), mk(2 * inter, h), mk(h, inter)]


def _local_cols(y, width, world):
    """The TP stand-ins read each rank's first `width / world` columns of its own column
    block: unsharded, that is the concatenation over ranks of those slices."""
    blk, w = y.shape[1] // world, width // world
    return np.ascontiguousarray(np.concatenate([y[:, r * blk: r * blk + w] for r in range(world)], 1))


def _oracle_decoder(oracle, x16, ws, h, inter, world=1):
    """The unsharded TPDecoderLinears chain on the oracle with fp16 intermediates."""
    q = _oracle_linear(oracle, x16.astype(np.float32), ws[0]).astype(np.float16)
    hh = _oracle_linear(oracle, _local_cols(q, h, world).astype(np.float32), ws[1]).astype(np.float16)
    gu = _oracle_linear(oracle, hh.astype(np.float32), ws[2]).astype(np.float16)
    return _oracle_linear(oracle, _local_cols(gu, inter, world).astype(np.float32), ws[3]).astype(np.float16)


@pytest.mark.parametrize("transport", ["comm", "torch"])
def test_tp_decoder_world1_vs_oracle(transport, oracle, torch_cuda, dev, comm1):
    torch = torch_cuda
    from paper_2311_09550_b200.tp import DeviceBackend, TPDecoderLinears
    h, inter, m = 512, 1024, 16
    rs = np.random.default_rng(31)
    ws = _decoder_weights(rs, h, inter)
    x = (rs.standard_normal((m, h), dtype=np.float32) * 2).astype(np.float16)
    want = _oracle_decoder(oracle, x, ws, h, inter)
    wd = [torch.from_numpy(w).cuda() for w in ws]
    if transport == "comm":
        layer = TPDecoderLinears(*wd, comm=comm1)
    else:
        layer = TPDecoderLinears(*wd, backend=DeviceBackend(torch.float16))
    y = layer(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy().view(np.uint16), want.view(np.uint16))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2311_09550_b200.tp import DeviceBackend, TPDecoderLinears
        h, inter, m = 512, 1024, 16
        rs = np.random.default_rng(31)
        ws = [torch.from_numpy(w).cuda() for w in _decoder_weights(rs, h, inter)]
        x = (rs.standard_normal((m, h), dtype=np.float32) * 2).astype(np.float16)
        layer = TPDecoderLinears(*ws, backend=DeviceBackend(torch.float16))
        y = layer(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        q.put((rank, y.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_tp_decoder_world2_gloo_on_one_gpu(oracle):
    """Two ranks (processes) on cuda:0, collectives over gloo on CUDA tensors: the sharded
    layer (column/row split, MAX + int32 SUM all-reduces) equals the unsharded oracle."""
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, inter, m = 512, 1024, 16
    rs = np.random.default_rng(31)
    ws = _decoder_weights(rs, h, inter)
    x = (rs.standard_normal((m, h), dtype=np.float32) * 2).astype(np.float16)
    want = _oracle_decoder(oracle, x, ws, h, inter, world)
    for rank, y in res:
        assert np.array_equal(y.view(np.uint16), want.view(np.uint16)), rank
