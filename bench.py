"""bench.py -- W4A8 FastGEMM on B200 (OdysseyLLM's FastGEMM linear, arXiv 2311.09550).

HEADLINE (BASELINE.json configs[1]; the metric's "LLaMA-13B layer latency"): one STEP is
one LLaMA-13B decoder layer's linear stack at decode batch M (default 16), run as the
DEPENDENT chain a real layer executes (not four independent linears):
    x[M,5120] -> qkv (15360x5120) -> o (5120x5120) on qkv[:, :5120]   (attention stand-in)
              -> gate_up (27648x5120) -> down (5120x13824) on gate_up[:, :13824] (SiLU stand-in)
Each linear quantizes its input per token (K1), runs the W4A8 FastGEMM (K3) and the
dequantizing epilogue (K4), fp16 in / fp16 out.  At N = 1 the step is FOUR dependent
launches in stream order (per linear: the batched act-quant kernel + a one-linear program
on the persistent w4a8_decode_dyn_kernel, PDL between them) -- measured faster than the
same layer as one chain program, which is reported beside it (roofline.chain_program).  At N > 1
the same layer runs Megatron-TP over N GPUs through ody_tp_linear (column qkv/gate_up,
row o/down with the MAX + exact int32 SUM NCCL all-reduces), one CUDA graph per step;
strong scaling (the layer is fixed, its shards shrink).

value  = the step's algorithmic HBM bytes (all ranks) / device step time (CUDA events,
         CUDA-graph replay, max over ranks), GB/s.  Bytes per linear = N*K/2 (INT4
         weights) + 4N (channel scales) + 2MK (fp16 x) + 2MN (fp16 y) + 4M (token scales).
e2e    = the same bytes / wall time through the reference-facing C ABI with HOST f32
         buffers (ody_tensor_create -> ody_quantize_activations -> ody_gemm(FAST) ->
         host f32, chained), H2D and D2H inside the timed region.
L2     : each step streams 158.6 MB of weights (> 126 MB L2) and steps rotate over 4
         distinct weight copies, so no timed weight byte is an L2 hit.
Other BASELINE configs ride in the same JSON line (N = 1 unless stated):
  config1   configs[0]: single GEMM M=16, N=K=4096 (one ody_dev_w4a8_linear per step)
  sweep_M   configs[1]: the chain step at M = 1..64
  prefill   configs[2]: the four 13B GEMMs at M = 1024 (INT8 tensor-pipe bound)
  tp70b     configs[3]: LLaMA-2-70B decoder-layer linears, TP = N (all ranks)
  stack13b  configs[4]: 40 LLaMA-13B layers, 1024-token prefill + 128 decode steps, TP = N
--impl reference: the reference's own CPU engine (oracle/_ref/libodyssey_ref.so, its C
         ABI: ody_quantize_activations + ody_gemm(ODY_ENGINE_FAST)) on the host cores.
--gpus N without torchrun: re-launches itself under torch.distributed.run, N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HIDDEN, INTER = 5120, 13824
LAYERS = [("qkv", 3 * HIDDEN, HIDDEN), ("o", HIDDEN, HIDDEN), ("gate_up", 2 * INTER, HIDDEN),
          ("down", HIDDEN, INTER)]
H70, I70, KV70 = 8192, 28672, 1024  # LLaMA-2-70B: hidden, intermediate, GQA kv width
LAYERS70 = [("qkv", H70 + 2 * KV70, H70), ("o", H70, H70), ("gate_up", 2 * I70, H70), ("down", H70, I70)]
METRIC = "W4A8 GEMM HBM GB/s (LLaMA-13B decoder-layer linear chain, decode)"
INT8_PEAK_TOPS = 4500.0  # B200 dense INT8 (datasheet); MEASURED_PEAKS.json has no INT8 figure


def linear_bytes(m, n, k):
    """Algorithmic HBM bytes of one W4A8 linear from fp16 x: packed INT4
    weights, per-channel scales, fp16 activations in, fp16 outputs out, token scales."""
    return n * k // 2 + 4 * n + 2 * m * k + 2 * m * n + 4 * m


def gemm_bytes(m, n, k):
    """One W4A8 GEMM on pre-quantized A (the reference CPU path's unit)."""
    return n * k // 2 + m * k + 4 * n + 4 * m + 2 * m * n


def actq_bytes(m, k):
    return 2 * m * k + m * k + 4 * m


def step_bytes(m, layers=LAYERS):
    return sum(linear_bytes(m, n, k) for _, n, k in layers)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def i8_peak():
    """Measured whole-GPU dense INT8 peak (tools/i8_peak.cu; profiles/i8_peak.json)."""
    p = os.path.join(ROOT, "profiles", "i8_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("i8_dense_tops_measured")
    return None


def bf16_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("bf16_tflops")
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._ready = threading.Event()  # set once the first sample is in (or sampling failed)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:  # NVML: ~1 ms per query, so even a short timed region gets many samples
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                    ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                    ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                    ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap)]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(sm), str(mx), hex(r)] +
                                 ["Active" if r & b else "Not Active" for _, b in bits])
                self._ready.set()
                self._stop.wait(0.002)
            return
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        self._ready.wait(timeout=30)  # the timed region starts with the sampler running
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "error": getattr(self, "err", None)}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}




# --------------------------------------------------------------------- B200 arm
def _graph_time(fn, stream, reps, warm=3):
    """Average device time of fn() (CUDA-graph replay, CUDA events on `stream`), ms."""
    import torch
    with torch.cuda.stream(stream):
        for _ in range(warm):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    with torch.cuda.stream(stream):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s.record(stream)
        for _ in range(reps):
            g.replay()
        e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def _max_over_ranks(ms, world):
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _weights_f32(n, k, seed):
    """Synthetic 0.1 N(0,1) f32 weights, identical on every rank (seeded generator)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn((n, k), device="cuda", generator=g) * 0.1


class ChainLayer:
    """One decoder layer's linears as the dependent chain qkv -> o -> gate_up -> down,
    ONE linear program (batched act quant + one persistent w4a8_decode_dyn_kernel; each
    dependent linear's input is quantized in-kernel once its producer completed).  The
    attention / SiLU stand-ins are column slices read in place.  M > 64 (prefill) lowers
    to one act-quant + FastGEMM pair per linear, in stream order."""

    def __init__(self, dev, ws, x, workspace=None):
        import torch
        m = x.shape[0]
        self.x = x
        self.outs = [torch.empty((m, w.n), dtype=torch.float16, device=x.device) for w in ws]
        o, d = ws[1], ws[3]
        self.prog = dev.Program([dev.LinearCall(x, ws[0], self.outs[0]),
                                 dev.LinearCall(self.outs[0][:, :o.k], o, self.outs[1], dep=0),
                                 dev.LinearCall(self.outs[1], ws[2], self.outs[2], dep=1),
                                 dev.LinearCall(self.outs[2][:, :d.k], d, self.outs[3], dep=2)],
                                workspace=workspace)
        self.y = self.outs[3]

    def run(self, pdl=True, stream=None):
        self.prog.run(pdl=pdl, stream=stream)
        return self.y


class SeqLayer:
    """One decoder layer's linears as FOUR dependent launches in stream order (each: the
    batched act quant of its input + a one-linear program on the dynamic kernel, PDL
    between launches): qkv -> o(qkv[:, :5120]) -> gate_up -> down(gate_up[:, :13824]),
    the slices read in place.  The headline step at N = 1: measured faster than the
    one-launch chain program (tools/layer_launch_ab.py).  Shares one
    workspace across its programs (stream-ordered)."""

    def __init__(self, dev, ws, x, workspace=None, links=False):
        import torch
        m = x.shape[0]
        self.outs = [torch.empty((m, w.n), dtype=torch.float16, device=x.device) for w in ws]
        o, d = ws[1], ws[3]
        ins = [x, self.outs[0][:, :o.k], self.outs[1], self.outs[2][:, :d.k]]
        self.progs = []
        if links:
            calls = [dev.LinearCall(i, w, y, dep=li - 1) for li, (i, w, y) in enumerate(zip(ins, ws, self.outs))]
            self.progs.append(dev.Program(calls, workspace=workspace, links=True))
            workspace = self.progs[-1].workspace
        for i, w, y in ([] if links else zip(ins, ws, self.outs)):
            self.progs.append(dev.Program([dev.LinearCall(i, w, y)], workspace=workspace))
            workspace = self.progs[-1].workspace
        self.workspace = workspace
        self.y = self.outs[3]

    def run(self, pdl=True, stream=None):
        for p in self.progs:
            p.run(pdl=pdl, stream=stream)
        return self.y


class TPLayer:
    """The same layer under Megatron TP over an ody_comm (ody_tp_linear per shard)."""

    def __init__(self, dims, comm, seed):
        from paper_2311_09550_b200.tp import TPDecoderLinears
        ws = [_weights_f32(n, k, seed + i) for i, (_, n, k) in enumerate(dims)]
        self.layer = TPDecoderLinears(*ws, comm=comm)
        del ws

    def run(self, x, stream=None):
        return self.layer(x, stream=stream)

    def local_bytes(self, m):
        return sum(linear_bytes(m, n, k) for _, n, k in self.layer.shapes())


def headline(args, dev, world, rank, comm, stream):
    """The metric's step: one 13B decoder layer chain at M, rotating weight copies."""
    import torch
    m = args.m
    x = (torch.randn((m, HIDDEN), device="cuda", generator=torch.Generator(device="cuda").manual_seed(7)) *
         2).half()
    if comm is None:
        copies = []
        for c in range(args.copies):
            copies.append([dev.W4Weight.quantize(_weights_f32(n, k, 1000 * c + i)) for i, (_, n, k) in
                           enumerate(LAYERS)])
        ws_shared = None
        layers = []
        for c in range(args.copies):
            layers.append(SeqLayer(dev, copies[c], x, workspace=ws_shared))
            ws_shared = layers[-1].workspace
        step = lambda c: layers[c].run(pdl=True, stream=stream)  # noqa: E731
        launches = 8  # 4 x (batched act quant + one-linear decode program)
        local_b = step_bytes(m)
    else:
        copies = None
        layers = [TPLayer(LAYERS, comm, 1000 * c) for c in range(args.copies)]
        step = lambda c: layers[c].run(x, stream=stream)  # noqa: E731
        launches = 12  # per rank: column 2 + row 4 (absmax, act quant, program, epilogue), x2
        local_b = layers[0].local_bytes(m)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(max(args.warmup, 1)):
            step(i % args.copies)
    torch.cuda.synchronize()
    graphs = []
    for c in range(args.copies):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(c)
        graphs.append(g)
    multi = torch.cuda.CUDAGraph()  # the steady-state decode loop: `copies` steps per graph
    with torch.cuda.graph(multi, stream=stream):
        for c in range(args.copies):
            step(c)
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            graphs[i % args.copies].replay()
        multi.replay()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        with torch.cuda.stream(stream):
            start.record(stream)
            for _ in range(args.steps // args.copies):
                multi.replay()
            for i in range(args.steps % args.copies):
                graphs[i].replay()
            end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    ms = _max_over_ranks(start.elapsed_time(end), world)
    return {"layers": layers, "copies": copies, "x": x, "ms": ms, "clk": clk.summary(),
            "launches": launches, "local_bytes": local_b, "graphs": graphs}


def roofline(args, dev, h, stream):
    """Dominant kernel at N = 1: the one-linear decode program (act_quant_rows_kernel +
    w4a8_decode_dyn_kernel<16, 0, 4>), four dependent launches per step, timed alone over
    graph replays of the weight copies back to back (no PDL: each launch starts on an
    idle GPU); achieved = the layer's algorithmic bytes / the step's launch time.  Also:
    the same dependent layer as ONE chain program, the four linears as INDEPENDENT inputs
    in one launch, and each linear alone."""
    import torch
    hbm, kind = peaks()
    m = args.m
    layers = h["layers"]

    def seq():
        for l in layers:
            l.run(pdl=False, stream=stream)

    ms = _graph_time(seq, stream, reps=50) / len(layers)
    achieved = step_bytes(m) / (ms * 1e-3) / 1e9
    xs = {k: (torch.randn((m, k), device="cuda") * 2).half() for k in (HIDDEN, INTER)}
    ind = [dev.Program([dev.LinearCall(xs[w.k], w, torch.empty((m, w.n), dtype=torch.float16, device="cuda"))
                        for w in cw]) for cw in h["copies"]]
    ms_ind = _graph_time(lambda: [p.run(pdl=True, stream=stream) for p in ind], stream, reps=50) / len(ind)
    del ind
    chains = [ChainLayer(dev, cw, h["x"]) for cw in h["copies"]]
    ms_chain = _graph_time(lambda: [c.run(pdl=True, stream=stream) for c in chains], stream, reps=50) / len(chains)
    del chains
    links = [SeqLayer(dev, cw, h["x"], links=True) for cw in h["copies"]]
    ms_links = _graph_time(lambda: [c.run(pdl=True, stream=stream) for c in links], stream, reps=50) / len(links)
    del links
    torch.cuda.empty_cache()
    per = {}
    wsl = dev.Workspace.get_linear(m, 27648, 13824, "cuda")
    for li, (name, n, k) in enumerate(LAYERS):
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        ws = [cw[li] for cw in h["copies"]]
        t = _graph_time(lambda ws=ws, k=k, out=out: [dev.w4a8_linear(xs[k], w, out=out, stream=stream, pdl=True,
                                                                      workspace=wsl) for w in ws],
                        stream, reps=100) / len(ws)
        b = linear_bytes(m, n, k)
        per[name] = {"N": n, "K": k, "us": round(t * 1e3, 3), "GB/s": round(b / (t * 1e-3) / 1e9, 1),
                     "frac": round(b / (t * 1e-3) / 1e9 / hbm, 4)}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(f"seq_M{m}")
        except Exception:
            traffic = None
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic, "peak_kind": kind,
            "kernel": "act_quant_rows_kernel + w4a8_decode_dyn_kernel<16, 0, 4> per linear (4 dependent launches "
                      "per step; bytes and time per step)",
            "launch_us": round(ms * 1e3, 3), "algorithmic_bytes_per_launch": step_bytes(m),
            "chain_program": {"us": round(ms_chain * 1e3, 3),
                              "GB/s": round(step_bytes(m) / (ms_chain * 1e-3) / 1e9, 1),
                              "frac": round(step_bytes(m) / (ms_chain * 1e-3) / 1e9 / hbm, 4),
                              "note": "the same dependent layer as ONE program launch (in-kernel grid-wide "
                                      "quantization of each dependent x), PDL"},
            "chain_links": {"us": round(ms_links * 1e3, 3),
                            "GB/s": round(step_bytes(m) / (ms_links * 1e-3) / 1e9, 1),
                            "frac": round(step_bytes(m) / (ms_links * 1e-3) / 1e9 / hbm, 4),
                            "note": "the same dependent layer as one launch per linear, each dependent x "
                                    "quantized from the row maxima its producer launch's epilogues "
                                    "accumulated (ody_dev_w4a8_linear_chain, act_quant_premax_kernel), PDL"},
            "independent_linears_program": {"us": round(ms_ind * 1e3, 3),
                                            "GB/s": round(step_bytes(m) / (ms_ind * 1e-3) / 1e9, 1),
                                            "frac": round(step_bytes(m) / (ms_ind * 1e-3) / 1e9 / hbm, 4),
                                            "note": "same 4 linears on independent inputs (no dependencies), PDL"},
            "per_shape": per, "per_shape_kernel": "one ody_dev_w4a8_linear launch per linear, PDL between copies"}


def config1(args, dev, stream):
    """configs[0]: single W4A8 linear M=16, N=K=4096 from fp16 x (K1+K3+K4), 24 rotating
    weight copies (201 MB > L2), one launch each."""
    import torch
    hbm, _ = peaks()
    m, n, k = 16, 4096, 4096
    ws = [dev.W4Weight.quantize(_weights_f32(n, k, 77 + c)) for c in range(24)]
    x = (torch.randn((m, k), device="cuda") * 2).half()
    out = torch.empty((m, n), dtype=torch.float16, device="cuda")
    wsl = dev.Workspace.get_linear(m, n, k, "cuda")
    ms = _graph_time(lambda: [dev.w4a8_linear(x, w, out=out, stream=stream, pdl=True, workspace=wsl) for w in ws],
                     stream, reps=50) / len(ws)
    b = linear_bytes(m, n, k)
    return {"M": m, "N": n, "K": k, "us": round(ms * 1e3, 3), "GB/s": round(b / (ms * 1e-3) / 1e9, 1),
            "frac": round(b / (ms * 1e-3) / 1e9 / hbm, 4), "TOPS": round(2 * m * n * k / (ms * 1e-3) / 1e12, 2),
            "kernel": "act_quant_rows_kernel + w4a8_decode_dyn_kernel<16> (program of one linear)"}


def engines_ablation(args, stream):
    """The paper's dequantization-scheme ablation (Fig. 7) on B200: the
    reference's engines (ref gemm.cpp:100-311) through ody_gemm_dev on pre-quantized
    activations, one 13B o-proj-sized GEMM (N = K = 5120) at decode M = 16 and prefill
    M = 1024.  FAST = the FastGEMM kernels; ASYMMETRIC / FINEGRAINED (g = 128) / W8A8 =
    engine_kernel.cu (ASYMMETRIC re-packs to UINT4+8 every call, as the reference does);
    W4A16 = the reference's sequential-f32 engine (decode only).  Rotating weight copies
    (> L2 at decode); CUDA-event time per call on the stream."""
    import numpy as np
    import torch

    from paper_2311_09550_b200 import api
    from paper_2311_09550_b200._lib import lib
    hbm, _ = peaks()
    res = {}
    rs = np.random.default_rng(11)
    n = k = 5120
    for m, copies in ((16, 8), (1024, 2)):
        a = (rs.standard_normal((m, k), dtype=np.float32) * 2).astype(np.float32)
        aq = api.quantize_activations_per_token(a)
        a_dev = torch.from_numpy(a).cuda()
        wf = [(rs.standard_normal((n, k), dtype=np.float32) * 0.1).astype(np.float32) for _ in range(copies)]
        ws = {"fast": (3, [api.quantize_weights(w) for w in wf]),
              "asymmetric": (2, [api.quantize_weights(w) for w in wf]),
              "finegrained_g128": (1, [api.quantize_weights(w, 4, 3, 128) for w in wf]),
              "w8a8": (4, [api.quantize_weights(w, 8, 1, 128) for w in wf])}
        if m == 16:
            ws["w4a16_g128"] = (0, ws["finegrained_g128"][1])
        del wf
        out = torch.empty((m, n), dtype=torch.float32, device="cuda")
        row = {}
        for name, (eng, wl) in ws.items():
            def call(w, eng=eng):
                rc = lib().ody_gemm_dev(eng, a_dev.data_ptr() if eng == 0 else None, m, None if eng == 0 else aq._h,
                                        w._h, out.data_ptr(), None, stream.cuda_stream)
                if rc:
                    raise RuntimeError(f"ody_gemm_dev({name}) failed: {lib().ody_last_error()}")
            with torch.cuda.stream(stream):
                for w in wl:
                    call(w)
            torch.cuda.synchronize()
            reps = 10 if (m == 1024 or eng == 0) else 40
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                s0.record(stream)
                for _ in range(reps):
                    for w in wl:
                        call(w)
                e0.record(stream)
            torch.cuda.synchronize()
            us = s0.elapsed_time(e0) * 1e3 / (reps * len(wl))
            wbytes = n * k if name == "w8a8" else n * k // 2
            byts = wbytes + m * k + 4 * n + 4 * m + 4 * m * n
            row[name] = {"us": round(us, 2), "GB/s": round(byts / (us * 1e-6) / 1e9, 1),
                         "frac_hbm": round(byts / (us * 1e-6) / 1e9 / hbm, 3),
                         "TOPS": round(2.0 * m * n * k / (us * 1e-6) / 1e12, 1)}
        res[f"M{m}"] = row
        del ws, aq
        torch.cuda.empty_cache()
    return {"shape": {"N": n, "K": k}, "per_M": res, "out": "f32 (the reference's engines return f32)",
            "note": "ody_gemm_dev per call incl. launch; ASYMMETRIC includes its per-call UINT4+8 repack"}


def decode_sweep(args, dev, h, stream):
    """configs[1] sweep: the headline step (the dependent layer, 4 launches) at M = 1..64."""
    import torch
    hbm, _ = peaks()
    res = {}
    for m in (1, 2, 4, 8, 16, 32, 64):
        x = (torch.randn((m, HIDDEN), device="cuda") * 2).half()
        ls = [SeqLayer(dev, cw, x) for cw in h["copies"]]
        ms = _graph_time(lambda ls=ls: [l.run(pdl=True, stream=stream) for l in ls], stream, reps=20) / len(ls)
        gbs = step_bytes(m) / (ms * 1e-3) / 1e9
        res[f"M{m}"] = {"us_per_step": round(ms * 1e3, 2), "GB/s": round(gbs, 1), "frac": round(gbs / hbm, 3),
                        "fused": all(p.fused for p in ls[0].progs)}
        del ls
    return res


def prefill_roofline(args, dev, h, stream, m=1024):
    """configs[2]: the 13B layer GEMMs at M = 1024 -- INT8 tensor-pipe bound.  Dominant
    kernel: w4a8_prefill_kernel (2-SM cta_group::2 FastGEMM) on pre-quantized
    activations, CUDA-event time over graph replays rotating the weight copies."""
    import torch
    res = {}
    tot_ops = tot_ms = 0.0
    bf16 = bf16_peak()
    for li, (name, n, k) in enumerate(LAYERS):
        x = (torch.randn((m, k), device="cuda") * 2).half()
        a = dev.act_quant(x)
        out = torch.empty((m, n), dtype=torch.float16, device="cuda")
        gws = dev.Workspace.get(m, n, k, "cuda")
        ws = [cw[li] for cw in h["copies"]]
        ms = _graph_time(lambda ws=ws, a=a, out=out, gws=gws: [dev.w4a8_gemm(a, w, out=out, stream=stream,
                                                                             workspace=gws) for w in ws],
                         stream, reps=10) / len(ws)
        ops = 2.0 * m * n * k
        tops = ops / (ms * 1e-3) / 1e12
        res[name] = {"N": n, "K": k, "us": round(ms * 1e3, 2), "TOPS": round(tops, 1),
                     "frac": round(tops / INT8_PEAK_TOPS, 3)}
        tot_ops += ops
        tot_ms += ms
    tops = tot_ops / (tot_ms * 1e-3) / 1e12
    i8m = i8_peak()
    if i8m:
        for v in res.values():
            v["frac_measured"] = round(v["TOPS"] / i8m, 3)
    return {"bound": "tensor", "M": m, "achieved": round(tops, 1), "peak": INT8_PEAK_TOPS, "unit": "TOP/s",
            "frac": round(tops / INT8_PEAK_TOPS, 3),
            "peak_measured": i8m, "frac_measured": round(tops / i8m, 3) if i8m else None,
            "peak_measured_source": "tools/i8_peak.cu (profiles/r2_i8_peak.md): sustained, power-capped ~1.59 GHz",
            "frac_of_2x_measured_bf16": round(tops / (2 * bf16), 3) if bf16 else None,
            "kernel": "w4a8_prefill_kernel (2-SM tcgen05 kind::i8, 256 weight rows x BT tokens per CTA pair)",
            "layer_us": round(tot_ms * 1e3, 1), "per_shape": res, "traffic": "profiles/r2_prefill_ncu.md"}


def tp70b(args, dev, world, comm, stream):
    """configs[3]: LLaMA-2-70B decoder-layer linears (hidden 8192, inter 28672, GQA kv
    1024) at TP = N: column qkv/gate_up, row o/down (MAX + int32 SUM all-reduces).  At
    N = 1 the unsharded layer runs as the headline step (4 dependent launches).  Decode M in {1, 16, 64} (2
    rotating weight copies, 856 MB); prefill M = 1024 once."""
    import torch
    hbm, _ = peaks()
    copies = 2
    if comm is None:
        cws = [[dev.W4Weight.quantize(_weights_f32(n, k, 7000 + 100 * c + i)) for i, (_, n, k) in
                enumerate(LAYERS70)] for c in range(copies)]
    else:
        tls = [TPLayer(LAYERS70, comm, 7000 + 100 * c) for c in range(copies)]
    res = {}
    for m in (1, 16, 64, 1024):
        x = (torch.randn((m, H70), device="cuda", generator=torch.Generator(device="cuda").manual_seed(m)) *
             2).half()
        if comm is None:
            ls = [SeqLayer(dev, cw, x) for cw in cws]
            fn = lambda ls=ls: [l.run(pdl=True, stream=stream) for l in ls]  # noqa: E731
            local = step_bytes(m, LAYERS70)
        else:
            fn = lambda x=x: [t.run(x, stream=stream) for t in tls]  # noqa: E731
            local = tls[0].local_bytes(m)
        ms = _max_over_ranks(_graph_time(fn, stream, reps=5 if m == 1024 else 30) / copies, world)
        tot = step_bytes(m, LAYERS70)
        ops = 2.0 * m * sum(n * k for _, n, k in LAYERS70)
        res[f"M{m}"] = {"us_per_layer": round(ms * 1e3, 2), "GB/s": round(tot / (ms * 1e-3) / 1e9, 1),
                        "TOPS": round(ops / (ms * 1e-3) / 1e12, 1),
                        "per_rank_frac_hbm": round(local / (ms * 1e-3) / 1e9 / hbm, 3)}
    return {"tp": world, "dims": {nm: [n, k] for nm, n, k in LAYERS70},
            "path": "4 dependent one-linear launches" if comm is None else "ody_tp_linear x4 (NCCL), one CUDA graph per layer",
            "per_M": res}


def stack13b(args, dev, world, comm, stream, n_layers=40, prompt=1024, gen=128):
    """configs[4]: 40 LLaMA-13B layers' linear stacks: a 1024-token prefill, then 128
    decode steps at batch args.stack_m (default 1), each decode step = ONE CUDA graph of
    the 40 layers (N = 1: 160 one-linear decode programs + their batched act quants, the
    headline step's launch form, PDL-chained; N > 1: ody_tp_linear shards).  The layer output feeds the next layer; the last
    layer's output feeds the next step (synthetic stand-in for the LM head + sampling)."""
    import torch
    hbm, _ = peaks()
    mb = args.stack_m
    w_bytes = n_layers * sum(n * k // 2 for _, n, k in LAYERS)
    if comm is None:
        ws = [[dev.W4Weight.quantize(_weights_f32(n, k, 90000 + 10 * L + i)) for i, (_, n, k) in enumerate(LAYERS)]
              for L in range(n_layers)]
    else:
        tls = [TPLayer(LAYERS, comm, 90000 + 10 * L) for L in range(n_layers)]
    torch.cuda.synchronize()

    def build(m):
        x0 = (torch.randn((m, HIDDEN), device="cuda") * 2).half()
        if comm is None:
            chain, x, wsp = [], x0, None
            for L in range(n_layers):
                chain.append(SeqLayer(dev, ws[L], x, workspace=wsp))
                wsp = chain[-1].workspace
                x = chain[-1].y
            def run():
                for c in chain:
                    c.run(pdl=True, stream=stream)
                return chain[-1].y
            return x0, run
        def run():
            x = x0
            for t in tls:
                x = t.run(x, stream=stream)
            return x
        return x0, run

    # prefill: M = 1024 through every layer (act quant + prefill FastGEMM per linear)
    x0p, runp = build(prompt)
    ms_p = _max_over_ranks(_graph_time(runp, stream, reps=3, warm=1), world)
    # decode: one graph per step; the step's output is copied into its input
    x0d, rund = build(mb)
    with torch.cuda.stream(stream):
        for _ in range(3):
            rund()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        y = rund()
        x0d.copy_(y)
    with torch.cuda.stream(stream):
        g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        s.record(stream)
        for _ in range(gen):
            g.replay()
        e.record(stream)
    torch.cuda.synchronize()
    ms_d = _max_over_ranks(s.elapsed_time(e) / gen, world)
    floor_ms = w_bytes / (hbm * 1e9) * 1e3 / world
    ops_p = 2.0 * prompt * n_layers * sum(n * k for _, n, k in LAYERS)
    return {"layers": n_layers, "tp": world, "prefill_tokens": prompt, "decode_steps": gen, "decode_batch": mb,
            "weight_bytes": w_bytes, "prefill_ms": round(ms_p, 3),
            "prefill_TOPS": round(ops_p / (ms_p * 1e-3) / 1e12, 1),
            "decode_ms_per_step": round(ms_d, 4), "decode_tokens_per_s": round(mb * 1e3 / ms_d, 1),
            "decode_GB/s": round(w_bytes / (ms_d * 1e-3) / 1e9, 1),
            "decode_hbm_floor_ms": round(floor_ms, 4), "decode_frac_of_floor": round(floor_ms / ms_d, 3),
            "total_ms_1024in_128out": round(ms_p + gen * ms_d, 2),
            "reference_paper_a100_13b_ms": 1139}


def e2e_c_abi(args, m):
    """Through the reference-facing C ABI with HOST buffers (api.py over ody_*): the layer
    chain, each linear's host f32 output feeding the next (slices as the stand-ins)."""
    import numpy as np

    from paper_2311_09550_b200 import api
    rs = np.random.default_rng(7)
    wq = []
    for _, n, k in LAYERS:  # offline weight quantization (not timed, as in the reference flow)
        w = (rs.standard_normal((n, k), dtype=np.float32) * 0.1).astype(np.float32)
        wq.append(api.quantize_weights(w))
        del w
    x = rs.standard_normal((m, HIDDEN), dtype=np.float32) * 2
    h2d = sum(m * k * 4 for _, _, k in LAYERS)
    d2h = sum(m * n * 4 for _, n, _ in LAYERS)

    def one():
        h = x
        for (_, n, k), w in zip(LAYERS, wq):
            aq = api.quantize_activations_per_token(api.Tensor(h[:, :k]))  # row-strided: no copy
            h = api.gemm_w4a8_fast(aq, w)

    for _ in range(max(args.warmup, 3)):
        one()
    reps = max(5, min(args.steps, 50))
    t0 = time.perf_counter()
    for _ in range(reps):
        one()
    dt = (time.perf_counter() - t0) / reps
    return {"value": round(step_bytes(m) / dt / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 4),
            "path": "C ABI ody_tensor_create/ody_quantize_activations/ody_gemm(FAST), host f32 in/out, chained",
            "timing": "host wall clock (the C-ABI calls are synchronous)"}


def e2e_tp(args, h, stream, world):
    """N > 1 (or --tp): end to end through the repo's TP API (TPDecoderLinears over an
    ody_comm) with the step's activations copied in from pinned host memory and the
    layer output copied back every step, host wall clock, max over ranks."""
    import torch
    m = args.m
    x_host = (torch.randn((m, HIDDEN)) * 2).half().pin_memory()
    y_host = torch.empty((m, HIDDEN), dtype=torch.float16).pin_memory()
    layer, xdev = h["layers"][0], h["x"]

    def one():
        with torch.cuda.stream(stream):
            xdev.copy_(x_host, non_blocking=True)
            y = layer.run(xdev, stream=stream)
            y_host.copy_(y, non_blocking=True)
        stream.synchronize()

    for _ in range(5):
        one()
    reps = 50
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(reps):
        one()
    dt = _max_over_ranks((time.perf_counter() - t0) / reps * 1e3, world) * 1e-3
    return {"value": round(step_bytes(m) / dt / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": m * HIDDEN * 2,
            "d2h_bytes_per_step": m * HIDDEN * 2, "ms_per_step": round(dt * 1e3, 4),
            "path": "TPDecoderLinears(comm) eager: pinned H2D x -> 4 ody_tp_linear -> D2H y, per rank",
            "timing": "host wall clock, max over ranks"}


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2311_09550_b200 import device as dev

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = dev.Comm.from_process_group() if world > 1 else (dev.Comm(1, 0, dev.Comm.unique_id()) if args.tp
                                                            else None)
    stream = torch.cuda.Stream()
    h = headline(args, dev, world, rank, comm, stream)
    m = args.m
    ms_step = h["ms"] / args.steps
    value = step_bytes(m) / (ms_step * 1e-3) / 1e9
    hbm, kind = peaks()
    result = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "s8 x s4(widened to s8) -> s32 accum, fp16 io",
        "data": "synthetic: x fp16 2*N(0,1), W f32 0.1*N(0,1) quantized on device",
        "config": {"workload": "llama13b_decoder_layer_linear_chain_decode", "M": m,
                   "layers": {nm: [n, k] for nm, n, k in LAYERS}, "hidden": HIDDEN, "intermediate": INTER,
                   "chain": "qkv -> o(qkv[:, :5120]) -> gate_up -> down(gate_up[:, :13824])",
                   "step": "4 dependent launches (act quant + one-linear decode program each), PDL",
                   "parallelism": f"tp{world}" if (world > 1 or comm is not None) else "single",
                   "weight_bytes_per_step": sum(n * k // 2 for _, n, k in LAYERS),
                   "l2": "inputs larger than L2 (158.6 MB weights/step, 4 rotating copies)",
                   "cuda_graph": "one graph per 4 steps (the 4 weight copies)", "pdl": True,
                   "step_latency_us": round(ms_step * 1e3, 2)},
        "clocks": h["clk"],
        "gpu_launches": h["launches"] * args.steps,
    }
    if world > 1 or comm is not None:
        result["roofline"] = {"bound": "hbm", "per_rank": True, "achieved": round(
            h["local_bytes"] / (ms_step * 1e-3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(h["local_bytes"] / (ms_step * 1e-3) / 1e9 / hbm, 4), "traffic": None,
            "kernel": "per rank: 4 x ody_tp_linear (act quant + w4a8_decode_dyn_kernel; row shards add row "
                      "absmax, NCCL MAX + int32 SUM all-reduces, K4 epilogue)",
            "local_bytes_per_step": h["local_bytes"]}
    if world > 1 or comm is not None:
        result["e2e"] = e2e_tp(args, h, stream, world)
    if world == 1 and comm is None and not args.quick:
        result["roofline"] = roofline(args, dev, h, stream)
        result["config1"] = config1(args, dev, stream)
        result["sweep_M"] = decode_sweep(args, dev, h, stream)
        result["prefill"] = prefill_roofline(args, dev, h, stream)
        result["engines"] = engines_ablation(args, stream)
    h = None
    torch.cuda.empty_cache()
    if not args.quick:
        result["tp70b"] = tp70b(args, dev, world, comm, stream)
        torch.cuda.empty_cache()
        result["stack13b"] = stack13b(args, dev, world, comm, stream)
        torch.cuda.empty_cache()
    if rank == 0 and world == 1:
        result["e2e"] = e2e_c_abi(args, m)
        if not args.no_cpu:
            result["cpu_baseline"] = cpu_baseline(args, m)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


# --------------------------------------------------------------- CPU reference
class CpuReference:
    """The reference's CPU engine on the layer shapes, inputs prepared once.

    kind "reference": oracle/_ref/libodyssey_ref.so (the reference compiled from its
    own sources, driven through its C ABI); else "port": the pinned C restatement."""

    def __init__(self, m, threads, layers):
        from oracle.oracle import REF_SO, Oracle, RefCAPI
        self.m, self.threads = m, threads
        self.orc = Oracle()
        self.ref = RefCAPI() if os.path.exists(REF_SO) else None
        self.kind = "reference" if self.ref is not None else "port"
        os.environ["ODYSSEY_THREADS"] = str(threads)
        if self.ref is not None:
            self.ref.L.ody_set_threads(threads)
        self.prep = {}
        for name, n, k in LAYERS:
            if name not in layers:
                continue
            a, w = self.orc.bench_inputs(1, m, n, k)
            if self.ref is not None:
                ah, wh = self.ref.tensor(a), self.ref.tensor(w)
                wq = self.ref.quantize_weights(wh)  # offline, untimed
                self.ref.free_tensor(wh)
                self.prep[name] = (n, k, ah, wq)
            else:
                _, packed, sw = self.orc.quantize_weights(w)
                self.prep[name] = (n, k, a, (packed, sw))

    def run(self, name):
        """One act quant + FAST GEMM of layer `name`; returns (bytes, seconds)."""
        n, k, a, wq = self.prep[name]
        m = self.m
        if self.ref is not None:
            t0 = time.perf_counter()
            aq = self.ref.quantize_activations(a)
            self.ref.gemm_fast(aq, wq, m, n)
            dt = time.perf_counter() - t0
            self.ref.free_qtensor(aq)
        else:
            packed, sw = wq
            t0 = time.perf_counter()
            codes, sa = self.orc.quantize_activations(a)
            self.orc.fast_gemm(codes, sa, packed, sw, m, n, k, threads=self.threads)
            dt = time.perf_counter() - t0
        return gemm_bytes(m, n, k) + actq_bytes(m, k), dt


def cpu_model():
    """`lscpu` model name (BASELINE.md §4 asks for it next to the core count)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_baseline(args, m, reps=5, warmup=2):
    """BASELINE.md §4 / SURVEY §8(d): the reference CPU engine on the bench layer, 2
    warm-ups then the median of `reps` timed passes (ref bench.cpp:158-178), all host
    threads (ODYSSEY_THREADS = nproc).  A pass = the layer's 4 linears (act quant + FAST
    GEMM each), the same step the GPU arm times."""
    threads = os.cpu_count() or 1
    names = [nm for nm, _, _ in LAYERS]
    cpu = CpuReference(m, threads, names)

    def one_pass():
        b = s = 0
        for nm in names:
            bb, ss = cpu.run(nm)
            b += bb
            s += ss
        return b, s

    for _ in range(warmup):
        one_pass()
    runs = [one_pass() for _ in range(reps)]
    med = statistics.median(s for _, s in runs)
    b = runs[0][0]
    return {"value": round(b / med / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": cpu.kind,
            "cpu_model": cpu_model(),
            "sample": f"the layer's 4 linears (act quant + FAST GEMM each) at M={m}, f32 host inputs, "
                      f"ODYSSEY_THREADS={threads}; {warmup} warm-ups then the median of {reps} passes "
                      f"(ref bench.cpp:158-178). The reference parallelises over M rows only and "
                      f"unpacks nibbles serially (ref gemm.cpp:219-225)",
            "ms_per_pass_median": round(med * 1e3, 3),
            "ms_per_pass_all": [round(s * 1e3, 3) for _, s in runs]}


def run_reference(args):
    """The reference's own CPU engine (oracle/_ref: the reference compiled from its sources,
    driven through its C ABI) on the same step: the layer's 4 linears, all host threads.
    Rank 0 only under torchrun.  A bounded (~2 minute) sample of the requested steps."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    m = args.m
    threads = os.cpu_count() or 1
    cpu = CpuReference(m, threads, [nm for nm, _, _ in LAYERS])
    kind = cpu.kind

    def one_step():
        b = s = 0
        for nm, _, _ in LAYERS:
            bb, ss = cpu.run(nm)
            b += bb
            s += ss
        return b, s

    t_w = time.perf_counter()
    for _ in range(args.warmup):
        one_step()
    per_step = (time.perf_counter() - t_w) / max(args.warmup, 1)
    timed = min(args.steps, max(5, int(120.0 / max(per_step, 1e-3))))
    runs = [one_step() for _ in range(timed)]
    secs = sum(s for _, s in runs)
    value = sum(b for b, _ in runs) / secs / 1e9
    sample = (f"each step = the layer's 4 linears (act quant + FAST GEMM each, M={m}), reference C ABI on "
              f"{threads} host threads; {timed} of the {args.steps} requested steps timed (a bounded ~2-minute "
              f"sample; median step {statistics.median(s for _, s in runs) * 1e3:.1f} ms)")
    out = {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(secs / timed * 1e3, 3), "timed_steps": timed, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "s8 x s4 -> s32 (CPU)",
           "data": "synthetic: ref Rng(seed^0x9d2c5680) a~N(0,1), w~0.1 N(0,1)",
           "config": {"workload": "llama13b_decoder_layer_linear_chain_decode", "M": m,
                      "layers": {nm: [n, k] for nm, n, k in LAYERS}},
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": kind,
                            "cpu_model": cpu_model(), "sample": sample},
           "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--m", type=int, default=16, help="decode batch (tokens) per step")
    ap.add_argument("--copies", type=int, default=4, help="distinct weight copies rotated")
    ap.add_argument("--stack-m", type=int, default=1, help="decode batch of the 40-layer stack (configs[4])")
    ap.add_argument("--tp", action="store_true", help="N = 1: run the TP (ody_tp_linear / NCCL) path anyway")
    ap.add_argument("--quick", action="store_true", help="headline only")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
