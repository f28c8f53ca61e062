"""Benchmark: QuartetLinear fwd+bwd at Llama-7B shapes (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--tokens T]

One step = forward + backward of the Quartet linear layer (Alg. 1) for each of the three Llama-7B
projection shapes (4096->4096, 4096->11008, 11008->4096) on T tokens per GPU, through the
reference-mirroring functional API (paper_2505_14669_b200.forward / backward -> C ABI -> sm_100a
kernels).  Inputs are synthetic and resident in HBM; every input tensor is larger than L2 (126 MB
for x / dy at T=16384), so no L2 flush is needed between steps.

Multi-GPU (torchrun): data-parallel, weak scaling; each rank runs its own T tokens and the dW of
every shape is all-reduced in bf16 over NCCL (the only exchange step in DP training).

--impl reference times the reference itself (mx4train.qlinear from baseline/_ref, native backend) on the
host CPU, one worker process per core, on bounded token slices of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QuartetLinear fwd+bwd TFLOPS vs BF16 (Llama-7B shapes); train tok/s @1–8 GPU"
SHAPES = [(4096, 4096), (4096, 11008), (11008, 4096)]   # (d_in, d_out)


def flops_per_step(tokens: int) -> float:
    return float(sum(6 * tokens * di * do for di, do in SHAPES))


# --------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML (in-process, no nvidia-smi fork) every
    `period` seconds from a background thread while the timed region runs."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples = []
        self._stop = threading.Event()
        self._thread = None
        self.smax = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()

    def _run(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            self._stop.wait(self.period)

    def stop(self) -> dict:
        if self._thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self._thread.join()
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        sm = [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax, "reasons": reasons,
                "samples": len(sm), "source": "NVML nvmlDeviceGetClockInfo / CurrentClocksEventReasons"}


# ------------------------------------------------------------------------------ helpers
def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"], "source": "MEASURED_PEAKS.json"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic() -> dict:
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The unmodified reference (mx4train) as pip-installed into baseline/_ref, native (Cython) backend:
    the CPU implementation of the path this bench's reference arm and cpu_baseline time.  Test/measurement
    infrastructure only -- nothing on the GPU path imports it."""
    if not os.path.isdir(os.path.join(REF_DIR, "mx4train")):
        raise RuntimeError(f"reference not installed in {REF_DIR} (python -m pip install --no-index "
                           "--no-build-isolation --no-deps --target baseline/_ref <copy of /root/reference/pkg>)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    os.environ["MX4TRAIN_BACKEND"] = "native"
    from mx4train import qlinear
    from mx4train._backend import BACKEND

    if BACKEND != "native":
        raise RuntimeError(f"reference backend is {BACKEND!r}, expected the compiled 'native' kernels")
    return qlinear


def _bf16_valued(a):
    """Round an fp32 array to bf16-representable values (RNE), like the GPU arm's bf16 inputs."""
    import numpy as np

    b = a.astype(np.float32).view(np.uint32)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return b.view(np.float32)


def ref_inputs(tokens: int, d_in: int, d_out: int, seed: int):
    """Synthetic inputs of one shape (x, dy ~ N(0,1) bf16-valued; W ~ N(0, 1/d_in) fp32)."""
    import numpy as np

    r = np.random.default_rng(seed)
    x = _bf16_valued(r.standard_normal((tokens, d_in), dtype=np.float32))
    w = (r.standard_normal((d_out, d_in), dtype=np.float32) / np.float32(np.sqrt(d_in))).astype(np.float32)
    dy = _bf16_valued(r.standard_normal((tokens, d_out), dtype=np.float32))
    return x, w, dy


def cpu_baseline_sample(tokens: int = 128) -> dict:
    """cpu_baseline: the reference itself (mx4train.qlinear.forward + backward, native backend, one core --
    its kernels are single-threaded) on a bounded sample of the bench workload: one fwd+bwd of each of the
    three Llama-7B shapes on `tokens` tokens (of the 16384)."""
    ql = import_reference()
    total_flop, total_s = 0.0, 0.0
    for i, (d_in, d_out) in enumerate(SHAPES):
        x, w, dy = ref_inputs(tokens, d_in, d_out, seed=i)
        t0 = time.perf_counter()
        _, ctx = ql.forward(x, w)
        ql.backward(dy, ctx, 7)
        total_s += time.perf_counter() - t0
        total_flop += 6.0 * tokens * d_in * d_out
    return {"flop": total_flop, "seconds": total_s}


def kernel_table(qt, data, dev, reps=10):
    """Average device time of every hot-path kernel of one step (per shape): each kernel is launched
    `reps` times back to back between two CUDA events on the launching stream, with the operands the
    step produces (inputs of each shape exceed L2 except W)."""
    import torch

    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import gemm, quant_dual, quant_fused, sign_bits

    op = 0.5 + 1 / 32          # bytes per element of one MXFP4 operand (codes + E8M0 scales)
    RH, RT = _lib.QT_TRANSFORM_HADAMARD, _lib.QT_TRANSFORM_RANDOMIZED
    rows = []

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) * 1e3 / reps

    for (x, w, dy) in data:
        T, d_in = x.shape
        d_out = w.shape[0]
        _, ctx = qt.forward(x, w, out_dtype=torch.bfloat16, check_finite=False, bwd_xi=7)
        xt_q, wt_q = ctx.eager.xt_q, ctx.eager.wt_q
        t_signs, d_signs = ctx.eager.t_signs, ctx.eager.d_signs
        g_q, gt_q = quant_dual(dy, _lib.QT_ROUND_RTN, transform=RT, signs=d_signs, col_signs=t_signs, prescale=0.75)
        fl = 2.0 * T * d_in * d_out
        QQ, RTN = _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN
        cases = [
            # X -> X_q (+ trust mask) and X_t from one read of X; same for the fp32 master W
            ("quant_fused_x", lambda: quant_fused(x, QQ, RTN, transform=RH, col_transform=RT, col_signs=t_signs),
             T * d_in * (2 + 2 * op + 1 / 8), 0),
            ("quant_fused_w", lambda: quant_fused(w, QQ, RTN, transform=RH, col_transform=RT, col_signs=d_signs),
             d_out * d_in * (4 + 2 * op + 1 / 8), 0),
            ("quant_dual_dy", lambda: quant_dual(dy, RTN, transform=RT, signs=d_signs, col_signs=t_signs,
                                                 prescale=0.75),
             T * d_out * (2 + 2 * op), 0),
            ("gemm_fwd", lambda: gemm(ctx.x_q, ctx.w_q, out_dtype=torch.bfloat16), 0, fl),
            ("gemm_dx", lambda: gemm(g_q, wt_q, out_dtype=torch.bfloat16, mask=ctx.x_q.mask, scale=16 / 9), 0, fl),
            ("gemm_dw", lambda: gemm(gt_q, xt_q, out_dtype=torch.float32, mask=ctx.w_q.mask, scale=16 / 9), 0, fl),
        ]
        for name, fn, nbytes, flop in cases:
            us = timeit(fn)
            r = {"kernel": name, "shape": f"{d_in}->{d_out}", "us": round(us, 2), "kind": "gemm" if flop else "quant"}
            if flop:
                r.update(flop=flop, tflops=round(flop / (us * 1e-6) / 1e12, 1))
            else:
                r.update(bytes=nbytes, gbs=round(nbytes / (us * 1e-6) / 1e9, 1))
            rows.append(r)
    return rows


# ---------------------------------------------------------------------------- our arm
def johnson_order(a, b):
    """Two-machine flow-shop order (Johnson's rule) for jobs with upload times a and download times b:
    jobs with a < b first by increasing a, then the rest by decreasing b."""
    first = sorted((i for i in range(len(a)) if a[i] < b[i]), key=lambda i: a[i])
    rest = sorted((i for i in range(len(a)) if a[i] >= b[i]), key=lambda i: -b[i])
    return first + rest


def e2e_pipeline(qt, data, dev, steps, outs_sink=None, world=1, rank=0):
    """End to end through the public API with host buffers: every step uploads each shape's x and dy
    from pinned host memory and downloads its dx (bf16) and dw (fp32).  Three streams -- uploads,
    compute, downloads -- so PCIe runs both directions at once (full duplex, measured 92 GB/s
    aggregate vs 55 GB/s one way; tools/pcie_probe.py): shape i's upload overlaps shape i-1's
    compute and shape i-2's download, and step k+1's uploads overlap step k's last downloads.
    Device input buffers are double-buffered by step parity; shapes run in Johnson order
    (upload-light / download-heavy first), which minimises the two-stage makespan."""
    import torch
    import torch.distributed as dist

    T = data[0][0].shape[0]
    host = [(x.cpu().pin_memory(), dy.cpu().pin_memory()) for (x, _, dy) in data]
    outs = [(torch.empty(x.shape, dtype=torch.bfloat16).pin_memory(),
             torch.empty(w.shape, dtype=torch.float32).pin_memory()) for (x, w, _) in data]
    bufs = [[(torch.empty_like(x), torch.empty_like(dy)) for (x, _, dy) in data] for _ in range(2)]
    up, down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    comp = torch.cuda.current_stream(dev)
    freed = [[None] * len(data) for _ in range(2)]   # compute done with bufs[parity][i]
    up_b = [hx.numel() * 2 + hdy.numel() * 2 for hx, hdy in host]
    down_b = [ox.numel() * 2 + ow.numel() * 4 for ox, ow in outs]
    order = johnson_order(up_b, down_b)

    def e2e_step(k, xi):
        par = k & 1
        for i in order:
            (hx, hdy), (ox, ow), (bx, bdy) = host[i], outs[i], bufs[par][i]
            with torch.cuda.stream(up):
                if freed[par][i] is not None:
                    up.wait_event(freed[par][i])
                bx.copy_(hx, non_blocking=True)
                bdy.copy_(hdy, non_blocking=True)
                ready = torch.cuda.Event()
                ready.record(up)
            comp.wait_event(ready)
            kw = dict(token_offset=rank * T, total_tokens=world * T) if world > 1 else {}
            y, ctx = qt.forward(bx, data[i][1], out_dtype=torch.bfloat16, check_finite=False, bwd_xi=xi * 3 + i, **kw)
            dx, dw = qt.backward(bdy, ctx, xi=xi * 3 + i, dx_dtype=torch.bfloat16, check_finite=False, **kw)
            if world > 1:   # the data-parallel exchange of the step: bf16 all-reduce of dW before it goes down
                buf = dw.to(torch.bfloat16)
                dist.all_reduce(buf, async_op=True).wait()
                dw.copy_(buf)
            done = torch.cuda.Event()
            done.record(comp)
            freed[par][i] = done
            with torch.cuda.stream(down):
                down.wait_event(done)
                ox.copy_(dx, non_blocking=True)
                ow.copy_(dw, non_blocking=True)
            dx.record_stream(down)
            dw.record_stream(down)
        return sum(up_b), sum(down_b)

    for k in range(2):
        e2e_step(k, k)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(comp)
    for k in range(steps):
        h2d, d2h = e2e_step(k, 100 + k)
    comp.wait_stream(up)
    comp.wait_stream(down)
    e.record(comp)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if outs_sink is not None:      # tests: the host results of the last step (xi = 100 + steps - 1)
        outs_sink.extend(outs)
    return {"value": round(world * flops_per_step(T) / (ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "paper_2505_14669_b200.forward/backward (C ABI), eager; pinned host x/dy in, dx/dw out; "
                    "upload / compute / download streams (PCIe full duplex), double-buffered inputs; "
                    + ("bytes per rank, dW all-reduced (bf16) before download" if world > 1 else "one GPU")}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2505_14669_b200 as qt

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    qt.load()
    T = args.tokens
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    data = []
    for d_in, d_out in SHAPES:
        x = torch.randn(T, d_in, device=dev, generator=g).to(torch.bfloat16)
        w = torch.randn(d_out, d_in, device=dev, generator=g) / (d_in ** 0.5)
        dy = torch.randn(T, d_out, device=dev, generator=g).to(torch.bfloat16)
        data.append((x, w, dy))

    def shape_step(i, xi, rounding="rtn"):
        x, w, dy = data[i]
        # the step's backward seed is known at forward time (train.py:346-348), so X_t / W_t come
        # out of the forward read of X / W (qt_quant_fused)
        # rank r holds tokens [r T, (r + 1) T) of the global batch: global sign / SR offsets make its
        # operands exact slices of the single-GPU operands (dp.py)
        y, ctx = qt.forward(x, w, out_dtype=torch.bfloat16, check_finite=False, bwd_xi=xi * 3 + i,
                            bwd_rounding=rounding, token_offset=rank * T, total_tokens=world * T)
        dx, dw = qt.backward(dy, ctx, xi=xi * 3 + i, rounding=rounding, dx_dtype=torch.bfloat16,
                             dw_dtype=torch.float32, check_finite=False, token_offset=rank * T,
                             total_tokens=world * T)
        return dw

    def step(xi, rounding="rtn", graphs=None):
        pending = []
        for i in range(len(data)):
            if graphs is not None:
                graphs[i][0].replay()
                dw = graphs[i][1]
            else:
                dw = shape_step(i, xi, rounding)
            if world > 1:  # data parallel: the token-sum of dW is the only exchange (bf16, NCCL); it runs
                # asynchronously on NCCL's stream while the next shape computes, and is waited for at step end
                buf = dw.to(torch.bfloat16)
                pending.append((dist.all_reduce(buf, async_op=True), buf, dw))
        for work, buf, dw in pending:
            work.wait()
            dw.copy_(buf)

    def capture(fn):
        g_ = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cap):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g_, stream=cap):
                out = fn()
        torch.cuda.current_stream().wait_stream(cap)
        return g_, out

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    graph = graphs = None
    if not args.no_graph and world == 1:
        # capture one full step (all shapes, fwd + bwd) once; every replay re-executes every kernel
        graph, _ = capture(lambda: step(args.warmup + 1))
    elif not args.no_graph:
        # N > 1: each shape's compute is one captured graph (the same kernels as the N = 1 graph); the
        # bf16 dW all-reduces are launched between the replays so they overlap the next shape's compute
        graphs = [capture(lambda i=i: shape_step(i, args.warmup + 1)) for i in range(len(data))]
    for _ in range(2):
        if graph is not None:
            graph.replay()
        else:
            step(args.warmup, graphs=graphs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local_rank) if rank == 0 and not args.no_clocks else None
    if sampler:
        sampler.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for i in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step(args.warmup + i, graphs=graphs)
    end.record()
    torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # the same step with stochastic-rounding backward operands (qlinear.py:168-175, rounding="sr"): the SR
    # quantizers run on the CUDA cores (the tensor-core dual quantizer is RTN-only)
    sr = {}
    if world == 1 and not args.no_graph:
        for mode, what in (("sr", "same step, backward rounding 'sr' (G, G_t, W_t, X_t by SR on the reference's "
                                  "splitmix64 stream, bit-exact)"),
                           ("sr_fast", "same step, backward rounding 'sr_fast' (B200 extension: SR to the same "
                                       "neighbours by the hardware conversion cvt.rs.e2m1x4, P(up) = floor(p 2^16) / 2^16; "
                                       "not the reference's draws)")):
            g_sr, _ = capture(lambda m=mode: step(args.warmup + 2, rounding=m))
            g_sr.replay()
            torch.cuda.synchronize()
            s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(args.steps):
                g_sr.replay()
            e0.record()
            torch.cuda.synchronize()
            sr_ms = s0.elapsed_time(e0) / args.steps
            sr[mode] = {"value": round(flops_per_step(T) / (sr_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                        "ms_per_step": round(sr_ms, 4), "what": what}
            del g_sr
    # end to end at N GPUs: every rank streams its own shard through its own PCIe link; max over ranks
    if world > 1:
        dist.barrier()
    e2e = e2e_pipeline(qt, data, dev, args.steps, world=world, rank=rank)
    if rank != 0:
        return None
    table = kernel_table(qt, data, dev, reps=10)

    # bf16 cuBLAS comparator on the same shapes (3 GEMMs per shape: y, dx, dw)
    mats = [(x, w.to(torch.bfloat16), dy) for (x, w, dy) in data]

    def bf16_step():
        for x, wb, dy in mats:
            torch.matmul(x, wb.t())
            torch.matmul(dy, wb)
            torch.matmul(dy.t(), x)
    for _ in range(3):
        bf16_step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        bf16_step()
    e.record()
    torch.cuda.synchronize()
    bf16_ms = s.elapsed_time(e) / args.steps


    peaks = measured_peaks()
    fp4_peak = 4.0 * peaks["bf16_tflops"]
    value = world * flops_per_step(T) / (ms * 1e-3) / 1e12
    gemm_rows = [r for r in table if r["kind"] == "gemm"]
    quant_rows = [r for r in table if r["kind"] == "quant"]
    gemm_us = sum(r["us"] for r in gemm_rows)
    gemm_tflops = sum(r["flop"] for r in gemm_rows) / (gemm_us * 1e-6) / 1e12
    q_us = sum(r["us"] for r in quant_rows)
    q_gbs = sum(r["bytes"] for r in quant_rows) / (q_us * 1e-6) / 1e9
    traffic = ncu_traffic().get("gemm_dram_bytes_per_launch")
    return {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "TFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "mxfp4-e2m1 x e2m1 (E8M0 block-32 scales), fp32 accumulate",
        "data": "synthetic (x, dy ~ N(0,1) bf16; W ~ N(0,1/d_in) fp32 master)",
        "config": {"workload": "QuartetLinear fwd+bwd, Llama-7B projection shapes (BASELINE configs[2])",
                   "shapes_din_dout": SHAPES, "tokens_per_gpu": T, "global_tokens": T * world,
                   "scheme": "quest fwd / rtn bwd, hadamard g=32", "parallelism": f"dp{world}",
                   "l2": "inputs larger than L2 (x/dy 128-344 MB per shape); no flush needed",
                   "launch": ("CUDA graph replay of one captured step" if graph is not None else
                              "one CUDA graph per shape, bf16 dW NCCL all-reduces launched between replays"
                              if graphs is not None else "eager")},
        "tokens_per_s": round(world * T * len(SHAPES) / (ms * 1e-3), 1),
        "bf16_cublas": {"value": round(flops_per_step(T) / (bf16_ms * 1e-3) / 1e12, 2), "unit": "TFLOP/s",
                        "ms_per_step": round(bf16_ms, 4), "speedup_ours": round(bf16_ms / ms, 3),
                        "what": "torch.matmul bf16: y = x W^T, dx = dy W, dw = dy^T x per shape"},
        "roofline": {"kernel": "k_gemm_mxf4_2sm (tcgen05.mma.cta_group::2.kind::mxf4, 2-CTA pairs; 1-CTA k_gemm_mxf4 for other shapes)", "bound": "tensor",
                     "achieved": round(gemm_tflops, 1), "peak": round(fp4_peak, 1), "unit": "TFLOP/s",
                     "frac": round(gemm_tflops / fp4_peak, 4), "traffic": traffic,
                     "peak_source": f"4 x bf16_tflops of {peaks['source']} (dense FP4 = 4x dense BF16 on B200); "
                                    "spec 9000 TFLOP/s",
                     "flop_per_launch_avg": sum(r["flop"] for r in gemm_rows) / len(gemm_rows),
                     "launches_per_step": len(gemm_rows), "share_of_step": round(gemm_us * 1e-3 / ms, 4),
                     "method": "CUDA events around 10 back-to-back launches of each GEMM of the step, "
                               "right after the timed region"},
        "quantizer_roofline": {"bound": "hbm", "achieved": round(q_gbs, 1), "peak": peaks["hbm_gbs"],
                               "unit": "GB/s", "frac": round(q_gbs / peaks["hbm_gbs"], 4),
                               "share_of_step": round(q_us * 1e-3 / ms, 4)},
        "kernels": table,
        "sr_backward": sr.get("sr"),
        "sr_fast_backward": sr.get("sr_fast"),
        "e2e": e2e,
        # per step and shape: 2 sign bitmaps + 2 fused forward quantizers + 1 GEMM; 1 dual quantizer + 2 GEMMs
        # per shape: signs pair, fused X, fused W, GEMM, dual dy, 2 GEMMs, and the zero-fill of the dW GEMM's
        # split last-wave blocks (all three bench dW GEMMs split their tail: 34 / 22 / 22 tiles)
        "gpu_launches": 8 * len(SHAPES) * args.steps,
        "clocks": clocks,
    }


def run_train(rank, world, local_rank):
    """BASELINE configs 2 / 4 / 5 through the Llama-Quartet stack (all linears MXFP4): Llama-200M data-parallel
    training throughput (64 x 512 tokens per GPU, bf16 NCCL gradient all-reduce), one Llama-30M training step,
    and one Llama-7B-dims transformer block fwd+bwd at 8k sequence x batch 4 (per GPU)."""
    import torch

    from paper_2505_14669_b200 import llama
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
    from train_llama import run

    dev = torch.device("cuda", local_rank)
    out = {"data": "synthetic token streams (no datasets offline)",
           "optimizer": "AdamW 0.9/0.95 wd 0.1, clip 1.0, warmup+cosine (train.py:58-85, 325-382)"}
    for key, args in (("llama200m_dp", ("200m", 64, 5, 3, False)), ("llama30m", ("30m", 64, 5, 3, False)),
                      ("block7b_8k_b4", ("7b", 4, 3, 1, True))):
        q = run(llama, *args, dev, world, rank, "quartet")
        torch.cuda.empty_cache()
        b = run(llama, *args, dev, world, rank, "bf16")   # comparator: same model/glue/optimizer, bf16 linears
        torch.cuda.empty_cache()
        q["bf16_arm"] = {k: b[k] for k in ("ms_per_step", "tokens_per_s", "linear_tflops", "loss") if k in b}
        q["speedup_vs_bf16"] = round(b["ms_per_step"] / q["ms_per_step"], 3)
        out[key] = q
    return out


_REF = {}   # inherited by the forked reference workers: module, inputs, start barrier


def _ref_worker(job):
    """One reference worker's share of a step: its own token slice through the unmodified
    mx4train.qlinear.forward / backward (data-parallel decomposition: every worker re-quantizes W, as
    every data-parallel rank must).  Returns (start, end) on the host's monotonic clock."""
    shape, k, xi = job
    ql = _REF["ql"]
    x, w, dy = _REF["data"][shape]
    T = _REF["tokens"]
    xs, dys = x[k * T:(k + 1) * T], dy[k * T:(k + 1) * T]
    _REF["barrier"].wait()
    t0 = time.perf_counter()
    _, ctx = ql.forward(xs, w)
    ql.backward(dys, ctx, xi)
    return t0, time.perf_counter()


def run_reference(args, rank, world):
    """Reference arm: the reference's own CPU implementation of the path -- mx4train.qlinear.forward +
    backward (QuEST forward, RTN backward, hadamard=True; native Cython kernels) from baseline/_ref -- on the
    host cores.  The reference's kernels are single-threaded, so it uses every core as one worker process
    per core (bounded by host memory), each running its own --ref-tokens token slice of the same shape
    (data parallel, W re-quantized per worker as per data-parallel rank).  A step = one fwd+bwd of one of
    the three Llama-7B shapes (cycling) on every worker; value = FLOP of all workers / step wall time
    (first start to last end), summed over the timed steps.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return None
    import multiprocessing as mp

    ql = import_reference()
    cores = os.cpu_count() or 1
    try:
        import psutil

        avail_gb = psutil.virtual_memory().available / 2**30
    except Exception:
        avail_gb = 64.0
    # the 11008 x 4096 shapes hold a few f32 / f64 copies of W per worker (~2 GB transient)
    P = max(1, min(cores, args.ref_workers or cores, int(avail_gb // 3)))
    T = args.ref_tokens
    _REF.update(ql=ql, tokens=T, data=[ref_inputs(P * T, d_in, d_out, seed=i) for i, (d_in, d_out) in
                                       enumerate(SHAPES)])
    ctx = mp.get_context("fork")
    _REF["barrier"] = ctx.Barrier(P)
    flop = sec = 0.0
    done = 0
    budget = args.ref_budget_s
    with ctx.Pool(P) as pool:
        def one(i):
            s = i % len(SHAPES)
            ts = pool.map(_ref_worker, [(s, k, 7 + i) for k in range(P)], chunksize=1)
            d_in, d_out = SHAPES[s]
            return 6.0 * P * T * d_in * d_out, max(e for _, e in ts) - min(b for b, _ in ts)

        t_all = time.perf_counter()
        for i in range(min(args.warmup, 1)):
            one(i)
        for i in range(args.steps):
            f, t = one(i)
            flop += f
            sec += t
            done += 1
            if time.perf_counter() - t_all > budget:  # keep the whole arm within a few minutes
                break
    v = flop / sec / 1e12
    return {
        "impl": "reference", "metric": METRIC, "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "steps_timed": done, "warmup": min(args.warmup, 1), "ms_per_step": round(1e3 * sec / done, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (fp32 work dtype; MXFP4 simulated in f64 quantizers, as the reference)",
        "data": "synthetic (x, dy ~ N(0,1) bf16-valued; W ~ N(0,1/d_in) fp32)",
        "config": {"workload": "QuartetLinear fwd+bwd, Llama-7B projection shapes (BASELINE configs[2])",
                   "shapes_din_dout": SHAPES, "tokens_per_worker": T, "workers": P,
                   "scheme": "quest fwd / rtn bwd, hadamard g=32", "implementation":
                   "mx4train.qlinear.forward/backward from baseline/_ref (unmodified reference, native backend)"},
        "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "cores": P, "kind": "reference",
                         "sample": f"per step one fwd+bwd of one shape (cycling) on {P} worker processes x {T} "
                                   f"tokens (of the GPU arm's 16384), {done} steps timed"},
        "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--ref-tokens", type=int, default=256, help="reference arm: tokens per worker and step")
    ap.add_argument("--ref-workers", type=int, default=0, help="reference arm: worker processes (0 = all cores)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0, help="reference arm: wall-clock budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel from Python each step")
    ap.add_argument("--no-train", action="store_true", help="skip the Llama training-throughput section")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # test hook: QT_BENCH_ONE_GPU=1 puts every rank on cuda:0 (with QT_BENCH_BACKEND=gloo) so the multi-rank
    # code path can be exercised on a one-GPU box; the driver's runs use one GPU per rank over NCCL
    if os.environ.get("QT_BENCH_ONE_GPU"):
        local_rank = 0

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch.distributed as dist

    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        backend = os.environ.get("QT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    out = run_ours(args, rank, world, local_rank)
    if not args.no_train:
        tr = run_train(rank, world, local_rank)
        if out is not None:
            out["train"] = tr
    if out is not None and world == 1 and not args.no_cpu_baseline:
        r = cpu_baseline_sample(128)
        out["cpu_baseline"] = {"value": round(r["flop"] / r["seconds"] / 1e12, 6), "unit": "TFLOP/s", "cores": 1,
                               "kind": "reference", "sample": "128 tokens x 3 shapes, one fwd+bwd each through the "
                               "unmodified mx4train.qlinear (baseline/_ref, native backend, single-threaded)",
                               "seconds": round(r["seconds"], 2)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if out is not None:
        # contract keys first, the long per-kernel table and the train section last (a truncated log tail still
        # shows the headline fields)
        head = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "e2e", "roofline", "cpu_baseline", "bf16_cublas",
                "quantizer_roofline", "gpu_launches", "clocks", "tokens_per_s", "sr_backward", "sr_fast_backward")
        tail = ("train", "kernels")
        ordered = {k: out[k] for k in head if k in out}
        ordered.update({k: v for k, v in out.items() if k not in head and k not in tail})
        ordered.update({k: out[k] for k in tail if k in out})
        print(json.dumps(ordered), flush=True)


if __name__ == "__main__":
    main()
