#!/usr/bin/env python
"""Benchmark of the Atom W4A4 hot path on B200 (one JSON line on rank 0).

A step = one pass of the whole hot path over one batch: a1 atom_reorder_quantize of the
activations + a2-a5 atom_w4a4_gemm (+ the tensor-parallel collective when N > 1).  Weights are
quantized once, offline (a0), outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--shard n|k]
  python bench.py --impl reference ...     # the CPU oracle as the reference arm

Metric (BASELINE.json): W4A4 mixed GEMM effective TOPS = 2*M*N*K / t_step, K counting the 128
outlier channels.  Multi-GPU (torchrun, one rank per GPU, NCCL): tensor parallel, N-shard
(all-gather of fp16 column blocks) or K-shard (all-reduce of fp32 partials), strong scaling;
time = max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import synth  # noqa: E402

CONFIGS = {
    # name: (M tokens, N out features, K in features incl. 128 outliers, description)
    "cfg1": (16, 1024, 1024, "single W4A4 linear, M=16, K=1024, N=1024"),
    "cfg2": (256, 4096, 4096, "Llama-7B q/k/v/o projection, M=256, K=N=4096"),
    "cfg3_up": (1024, 11008, 4096, "Llama-7B MLP up/gate, M=1024, K=4096, N=11008"),
    "cfg3_down": (1024, 4096, 11008, "Llama-7B MLP down, M=1024, K=11008, N=4096"),
    "cfg4": (512, 13824, 5120, "Llama-13B linear, M=512, K=5120, N=13824"),
    "cfg5": (1024, 28672, 8192, "Llama-70B MLP, M=1024, K=8192, N=28672"),
}
# BASELINE config 3 is a batch sweep (Fig 8a): the memory- to compute-bound crossover of the
# Llama-7B MLP up/gate (K=4096 -> N=11008) and down (K=11008 -> N=4096) projections
for _m in (8, 16, 32, 64, 128, 256, 512, 1024):
    CONFIGS[f"cfg3_up_m{_m}"] = (_m, 11008, 4096, f"Llama-7B MLP up/gate, M={_m}, K=4096, N=11008")
    CONFIGS[f"cfg3_down_m{_m}"] = (_m, 4096, 11008, f"Llama-7B MLP down, M={_m}, K=11008, N=4096")
METRIC = "W4A4 mixed GEMM effective TOPS and % roofline at Llama-7B/70B shapes, 1/2/4/8 B200"
UNIT = "TOPS"
K_OUT = 128


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def algorithmic_bytes(M, N, K, c_bytes=2):
    """Bytes the method must move: packed W + packed A (INT4 + INT8 + fp32
    scales) + C."""
    per_row = (K - K_OUT) // 2 + K_OUT + (K // 128) * 4
    return N * per_row + M * per_row + M * N * c_bytes


def quant_bytes(M, K):
    """a1 as timed: read X fp16 + perm, write the GEMM operand form (one byte per code, and the
    per-row (alpha, beta) pairs) and the scales (include/atom.h a_f8, a_ab, scales)."""
    return M * K * 2 + K * 4 + M * K + M * (K // 128) * 12


# ------------------------------------------------------------------------------------------------
# clocks (NVML, sampled during the timed region)
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.ok = [], set(), False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------------
# CPU oracle baseline (bounded sample)
# ------------------------------------------------------------------------------------------------
def oracle_setup(M, N, K, seed=0):
    import oracle
    X, perm = synth.activations(M, K, seed), synth.perm_for(K, seed)
    W = synth.weights(N, K, seed)
    w4, w8, ws = oracle.quantize_rows(W, perm, K, K_OUT, 0.85, 1.0)      # offline (a0), untimed
    return X, perm, (w4, w8, ws)


def oracle_step(X, perm, wpack, N, K, rows):
    """One oracle step on a sample of token rows: a1 quantize + a2-a5 outputs for those rows."""
    import oracle
    a4, a8, as_ = oracle.quantize_rows(X[rows], perm, K, K_OUT, 0.9, 1.0)
    w4, w8, ws = wpack
    return oracle.output_rows(a4, a8, as_, w4, w8, ws, len(rows), N, K, K_OUT,
                              np.arange(len(rows)))


def cpu_baseline(M, N, K, target_s=12.0, setup=None):
    import oracle
    X, perm, wpack = setup if setup is not None else oracle_setup(M, N, K)
    cores = oracle.max_threads()
    # calibrate on a small sample, then size the sample to ~target_s
    t0 = time.perf_counter()
    oracle_step(X, perm, wpack, N, K, np.arange(min(2, M)))
    dt = (time.perf_counter() - t0) / min(2, M)
    R = int(max(1, min(M, target_s / max(dt, 1e-6))))
    R = max(cores, (R // cores) * cores) if R >= cores else R
    R = min(R, M)
    rows = np.linspace(0, M - 1, R).astype(np.int64)
    t0 = time.perf_counter()
    oracle_step(X, perm, wpack, N, K, rows)
    t = time.perf_counter() - t0
    return {"value": 2.0 * R * N * K / t / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{R} of {M} token rows of the workload (quantize those rows + their full "
                      f"output rows, N={N}, K={K}); {t:.2f} s on {cores} host threads"}


# ------------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ------------------------------------------------------------------------------------------------
def run_reference(args, M, N, K, cfg_name, world, rank):
    if rank != 0:
        return
    import oracle
    setup = oracle_setup(M, N, K)
    X, perm, wpack = setup
    cores = oracle.max_threads()
    t0 = time.perf_counter()
    oracle_step(X, perm, wpack, N, K, np.arange(1))
    t_row = time.perf_counter() - t0
    budget = 150.0 / max(1, args.steps + args.warmup)      # whole run within a few minutes
    R = int(max(1, min(M, budget / max(t_row, 1e-6))))
    rows_all = [np.sort(np.random.default_rng(i).choice(M, R, replace=False))
                for i in range(args.steps + args.warmup)]
    for i in range(args.warmup):
        oracle_step(X, perm, wpack, N, K, rows_all[i])
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        oracle_step(X, perm, wpack, N, K, rows_all[args.warmup + i])
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = 2.0 * R * N * K / step_s / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (synth/: Llama-like activations with 128 x100 outlier channels, "
                "N(0,0.02^2) weights, seed 0)",
        "config": {"workload": cfg_name, "M": M, "N": N, "K": K, "k_outlier": K_OUT,
                   "group": 128, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"each step: {R} random token rows of {M} (quantize + full "
                                   f"output rows), N={N}, K={K}, {cores} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# the CUDA path
# ------------------------------------------------------------------------------------------------
def run_atom(args, M, N, K, cfg_name, world, rank, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2310_19102_b200 as atom
    from paper_2310_19102_b200 import build
    if rank == 0 or not (ROOT / "paper_2310_19102_b200" / "libatom.so").exists():
        build.build()
    if world > 1:
        dist.barrier()
    atom.load()
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    P, shard = world, args.shard
    G = K // 128

    # ---------------- inputs (synthetic, seeded; identical bytes on every rank) ----------------
    from paper_2310_19102_b200 import tp
    X = synth.activations(M, K, args.seed)
    perm = synth.perm_for(K, args.seed)
    if shard == "n":
        n0, n1 = tp.n_shard_rows(N, P, rank)
        W = synth.weights(N, K, args.seed, rows=(n0, n1))   # this rank's rows only
    else:
        W = synth.weights(N, K, args.seed)
        n0, n1 = 0, N
    Nr = n1 - n0
    xd = torch.from_numpy(X).to(dev)
    layer = tp.TensorParallelLinear(torch.from_numpy(W).to(dev), torch.from_numpy(perm).to(dev),
                                    K, shard)                  # a0: weights quantized offline
    K_r = layer.K
    del W
    aq = layer.quantize(xd)                                    # output buffers reused below
    c_loc = layer.gemm(aq)
    c_all = (torch.empty((P, M, Nr), dtype=torch.float16, device=dev) if shard == "n"
             else torch.empty((M, N), dtype=torch.float16, device=dev)) if P > 1 else None
    torch.cuda.synchronize()

    launches = [0]

    def step(x_in):
        layer.quantize(x_in, out=aq)
        launches[0] += atom.last_launch_count()
        layer.gemm(aq, out=c_loc)
        launches[0] += atom.last_launch_count()

    def collective():
        return layer.combine(c_loc, c_all)

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * l2 + (64 << 20), dtype=torch.uint8, device=dev)

    def flush_l2():
        flush.zero_()

    # spin up clocks (untimed), then W warm-up steps
    t_end = time.perf_counter() + args.spinup
    while time.perf_counter() < t_end:
        for _ in range(20):
            step(xd)
        torch.cuda.synchronize()
    for _ in range(args.warmup):
        flush_l2()
        step(xd)
        collective()
    torch.cuda.synchronize()

    # ---------------- the step's two kernels as CUDA graphs (no host launch gaps) ----------------
    # The device-timed region measures the kernels, not Python/ctypes launch latency (which the
    # e2e number below includes).  Each graph holds one ABI call; their kernels read and write
    # the same buffers every replay (the GEMM's workspace counters are self-cleaning).
    # The step graph holds both kernels: the GEMM is launched with programmatic dependent launch
    # (its prologue and first weight loads overlap the end of the quantize kernel); the
    # per-kernel graphs time each kernel alone.
    g_quant, g_gemm, g_step = None, None, None
    per_step_launches = 0
    if not args.no_graph:
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            g_quant, g_gemm, g_step = (torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph(),
                                       torch.cuda.CUDAGraph())
            with torch.cuda.graph(g_quant, stream=side):
                layer.quantize(xd, out=aq)
            per_step_launches += atom.last_launch_count()
            with torch.cuda.graph(g_gemm, stream=side):
                layer.gemm(aq, out=c_loc)
            per_step_launches += atom.last_launch_count()
            with torch.cuda.graph(g_step, stream=side):
                layer.quantize(xd, out=aq)
                layer.gemm(aq, out=c_loc)
        torch.cuda.current_stream().wait_stream(side)
        for _ in range(3):
            g_quant.replay()
            g_gemm.replay()
            g_step.replay()
        torch.cuda.synchronize()

    # ---------------- timed region: exactly K steps ----------------
    E = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    launches[0] = 0
    sampler = ClockSampler(torch.cuda.current_device())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for i in range(args.steps):
            if not args.no_flush:
                flush_l2()
            E[i][0].record()
            if g_step is not None:
                g_step.replay()
                launches[0] += per_step_launches
            else:
                layer.quantize(xd, out=aq)
                E[i][1].record()
                layer.gemm(aq, out=c_loc)
                launches[0] += 2
            E[i][2].record()
            collective()
            E[i][3].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    last = 3 if P > 1 else 2          # no collective at P = 1
    step_ms = [E[i][0].elapsed_time(E[i][last]) for i in range(args.steps)]
    c_ms = [E[i][2].elapsed_time(E[i][3]) if P > 1 else 0.0 for i in range(args.steps)]
    if g_step is not None:
        # each kernel alone (same flush, same graphs minus the step's overlap), for the roofline
        for i in range(args.steps):
            if not args.no_flush:
                flush_l2()
            E[i][0].record()
            g_quant.replay()
            E[i][1].record()
            g_gemm.replay()
            E[i][2].record()
        torch.cuda.synchronize()
    q_ms = [E[i][0].elapsed_time(E[i][1]) for i in range(args.steps)]
    g_ms = [E[i][1].elapsed_time(E[i][2]) for i in range(args.steps)]
    stats = torch.tensor([sum(step_ms) / args.steps, sum(q_ms) / args.steps,
                          sum(g_ms) / args.steps, sum(c_ms) / args.steps], device=dev,
                         dtype=torch.float64)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    step_avg, q_avg, g_avg, c_avg = stats.tolist()
    gpu_launches = launches[0]

    # ---------------- e2e through the public API with host buffers ----------------
    e2e = None
    if not args.no_e2e:
        x_h = torch.from_numpy(X).pin_memory()
        out_shape = c_all.shape if (P > 1) else c_loc.shape
        out_dtype = torch.float16
        c_h = torch.empty(out_shape, dtype=out_dtype).pin_memory()
        xin = torch.empty_like(xd)
        EE = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
        for i in range(max(1, args.warmup)):
            xin.copy_(x_h, non_blocking=True)
            step(xin)
            c = collective()
            c_h.copy_(c if c.dtype == out_dtype else c.half(), non_blocking=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # P = 1: the step is pipelined over token chunks through the same public calls -- the
        # H2D copy of chunk i+1 and the D2H copy of chunk i-1 overlap the quantize + GEMM of
        # chunk i on three streams (the transfers are the bound: 75 MB per step over PCIe);
        # every step still moves all of its inputs and outputs inside the timed region
        nch = max(1, min(args.e2e_chunks, M // 64)) if P == 1 else 1
        bounds = [(M * j // nch, M * (j + 1) // nch) for j in range(nch)]
        s_in, s_cmp, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
        aqs = [layer.quantize(xin[a:b]) for a, b in bounds] if nch > 1 else None
        torch.cuda.synchronize()

        def piped_step(ev0):
            ev_in = [torch.cuda.Event() for _ in bounds]
            ev_c = [torch.cuda.Event() for _ in bounds]
            s_in.wait_event(ev0)
            for j, (a, b) in enumerate(bounds):
                with torch.cuda.stream(s_in):
                    xin[a:b].copy_(x_h[a:b], non_blocking=True)
                    ev_in[j].record(s_in)
                s_cmp.wait_event(ev_in[j])
                with torch.cuda.stream(s_cmp):
                    layer.quantize(xin[a:b], out=aqs[j])
                    layer.gemm(aqs[j], out=c_loc[a:b])
                    ev_c[j].record(s_cmp)
                s_out.wait_event(ev_c[j])
                with torch.cuda.stream(s_out):
                    c_h[a:b].copy_(c_loc[a:b], non_blocking=True)
            torch.cuda.current_stream().wait_stream(s_out)

        if nch > 1:                                   # untimed warm-up of the pipelined step
            for _ in range(2):
                ev = torch.cuda.Event()
                ev.record()
                piped_step(ev)
            torch.cuda.synchronize()
        for i in range(args.steps):
            if not args.no_flush:
                flush_l2()
            EE[i][0].record()
            if nch > 1:
                piped_step(EE[i][0])
            else:
                xin.copy_(x_h, non_blocking=True)
                step(xin)
                c = collective()
                c_h.copy_(c if c.dtype == out_dtype else c.half(), non_blocking=True)
            EE[i][1].record()
        torch.cuda.synchronize()
        e_ms = torch.tensor([sum(EE[i][0].elapsed_time(EE[i][1]) for i in range(args.steps))
                             / args.steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        e_ms = float(e_ms.item())
        e2e = {"value": 2.0 * M * N * K / (e_ms * 1e-3) / 1e12, "unit": UNIT,
               "h2d_bytes_per_step": int(P * X.nbytes),
               "d2h_bytes_per_step": int(P * c_h.numel() * c_h.element_size()),
               "ms_per_step": e_ms,
               "pipeline": f"{nch} token chunks: H2D / quantize+GEMM / D2H on 3 streams"
                           if nch > 1 else "sequential"}

    # ---------------- NEXT-1: the fused RMSNorm + reorder + quantize kernel (not in the step) ----
    norm_us = None
    if not args.no_graph and P == 1:
        gamma = torch.from_numpy(
            (1 + 0.1 * np.random.default_rng(args.seed).standard_normal(K)).astype(np.float16)).to(dev)
        g_norm = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            atom.rmsnorm_reorder_quantize(xd, gamma, layer.perm, out=aq)
            with torch.cuda.graph(g_norm, stream=side):
                atom.rmsnorm_reorder_quantize(xd, gamma, layer.perm, out=aq)
        torch.cuda.current_stream().wait_stream(side)
        en = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(10)]
        for i in range(10):
            flush_l2()
            en[i][0].record()
            g_norm.replay()
            en[i][1].record()
        torch.cuda.synchronize()
        norm_us = 1e3 * sum(a.elapsed_time(b) for a, b in en) / len(en)

    # ---------------- NEXT-4 piece: fused SwiGLU + reorder + quantize of the down projection's
    # input (gate / up outputs of width N, as the up/gate GEMM of this config produces) ----------
    swiglu_us, swiglu_bytes = None, None
    if not args.no_graph and P == 1 and N % 128 == 0:
        rng = np.random.default_rng(args.seed + 7)
        gate = torch.from_numpy(synth.activations(M, N, args.seed + 7)).to(dev)
        upp = torch.from_numpy(rng.standard_normal((M, N)).astype(np.float16)).to(dev)
        perm_i = torch.from_numpy(synth.perm_for(N, args.seed + 7)).to(dev)
        hq = atom.silu_mul_reorder_quantize(gate, upp, perm_i)
        g_swi = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            atom.silu_mul_reorder_quantize(gate, upp, perm_i, out=hq, stream=side)
            with torch.cuda.graph(g_swi, stream=side):
                atom.silu_mul_reorder_quantize(gate, upp, perm_i, out=hq, stream=side)
        torch.cuda.current_stream().wait_stream(side)
        es = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(10)]
        for i in range(10):
            flush_l2()
            es[i][0].record()
            g_swi.replay()
            es[i][1].record()
        torch.cuda.synchronize()
        swiglu_us = 1e3 * sum(a.elapsed_time(b) for a, b in es) / len(es)
        swiglu_bytes = quant_bytes(M, N) + M * N * 2        # a second fp16 input row

    # ---------------- NEXT-2: Atom (FP) on the MX format, same workload (not the headline) ----------
    mx = None
    if not args.no_graph and not args.no_mx and P == 1:
        mx = time_atom_fp(atom, xd, layer.perm, M, N, K, args, dev, flush_l2)

    # ---------------- NEXT-3: INT4 KV cache decode attention (Llama-7B decode, batch 128) -------
    kv = None
    if not args.no_graph and not args.no_kv and P == 1:
        kv = time_kv_attention(atom, dev, flush_l2, args)

    # the box's INT8 tensor peak, measured in this run: cuBLAS int8 GEMM (torch._int_mm, 8192^3)
    int8_meas = None
    if rank == 0 and not args.no_peak:
        try:
            a8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev)
            b8 = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev)
            for _ in range(3):
                torch._int_mm(a8, b8)
            ep = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ep[0].record()
            for _ in range(10):
                torch._int_mm(a8, b8)
            ep[1].record()
            torch.cuda.synchronize()
            int8_meas = 2.0 * 8192 ** 3 / (ep[0].elapsed_time(ep[1]) / 10 * 1e-3) / 1e12
            del a8, b8
        except Exception as ex:   # report, never fail the bench on it
            int8_meas = f"unavailable: {type(ex).__name__}"

    if rank != 0:
        return
    peaks, peak_src = load_peaks()
    ops = 2.0 * M * N * K
    value = ops / (step_avg * 1e-3) / 1e12
    # dominant kernel: the GEMM (int8 tensor-core contraction).  Peak for its own dtype: the
    # measured bf16 burst peak x the nominal int8/bf16 ratio (4.5 / 2.25 = 2).
    gemm_ops_launch = 2.0 * M * Nr * K_r
    achieved = gemm_ops_launch / (g_avg * 1e-3) / 1e12
    peak_int8 = 2.0 * peaks["bf16_tflops"]
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(f"{cfg_name}:gemm:P{P}{shard}")
    t_roof_spec = max(2.0 * M * Nr * K_r / 4.5e15, algorithmic_bytes(M, Nr, K_r) / 8e12)
    qb = quant_bytes(M, K_r)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_avg, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (synth/: Llama-like activations with 128 x100 outlier channels, "
                "N(0,0.02^2) weights, seed 0)",
        "config": {"workload": cfg_name, "desc": CONFIGS[cfg_name][3], "M": M, "N": N, "K": K,
                   "k_outlier": K_OUT, "group": 128,
                   "parallelism": "single" if P == 1 else f"tp{P}-{shard}shard",
                   "l2": "flushed before every timed step (write of 2xL2+64MiB)"
                         if not args.no_flush else "warm",
                   "launch": "CUDA graph replay of the step (GEMM programmatic dependent launch)" if not args.no_graph else "direct"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_int8,
                     "unit": "TFLOP/s", "frac": achieved / peak_int8, "traffic": traffic,
                     "kernel": "atom::w4a4_gemm_kernel",
                     "peak_source": f"{peak_src} bf16 burst {peaks['bf16_tflops']} x 2 "
                                    f"(int8/bf16 nominal ratio)"},
        "roofline_spec": {"t_roof_us": t_roof_spec * 1e6, "t_gemm_us": g_avg * 1e3,
                          "frac": t_roof_spec / (g_avg * 1e-3),
                          "bound": "tensor" if 2.0 * M * Nr * K_r / 4.5e15 >=
                                   algorithmic_bytes(M, Nr, K_r) / 8e12 else "hbm",
                          "model": "max(2MNK/4.5e15, bytes/8e12) per GPU (BASELINE.json)"},
        "int8_peak_in_run": None if int8_meas is None else {
            "TOPS": int8_meas, "how": "torch._int_mm int8 8192^3, 10 back-to-back calls",
            "gemm_frac": achieved / int8_meas if isinstance(int8_meas, float) else None},
        "kernels": {
            "reorder_quantize": {"us": q_avg * 1e3, "GB/s": qb / (q_avg * 1e-3) / 1e9,
                                 "frac_hbm": qb / (q_avg * 1e-3) / 1e9 / peaks["hbm_gbs"]},
            "w4a4_gemm": {"us": g_avg * 1e3, "TOPS": achieved},
            "rmsnorm_reorder_quantize": None if norm_us is None else {
                "us": norm_us, "GB/s": qb / (norm_us * 1e-6) / 1e9,
                "note": "NEXT-1 fused RMSNorm + a1 (same bytes as reorder_quantize); not part of "
                        "the step"},
            "silu_mul_reorder_quantize": None if swiglu_us is None else {
                "us": swiglu_us, "GB/s": swiglu_bytes / (swiglu_us * 1e-6) / 1e9,
                "shape": [M, N],
                "note": "NEXT-4 piece: SwiGLU of gate/up [M][N] fused with a1 for the down "
                        "projection; not part of the step"},
            "collective": {"us": c_avg * 1e3},
        },
        "gpu_launches": gpu_launches,
        "atom_fp": None if mx is None else dict(mx, roofline={
            "bound": "tensor", "achieved": ops / (mx["gemm_us"] * 1e-6) / 1e12,
            "peak": 4.0 * peaks["bf16_tflops"], "unit": "TFLOP/s",
            "frac": ops / (mx["gemm_us"] * 1e-6) / 1e12 / (4.0 * peaks["bf16_tflops"]),
            "kernel": "atom::mx_gemm_kernel",
            "peak_source": f"{peak_src} bf16 burst {peaks['bf16_tflops']} x 4 (fp4/bf16 nominal "
                           f"ratio, 9 / 2.25 PFLOP/s)"}),
        "kv_attention": None if kv is None else dict(kv, roofline={
            "bound": "hbm", "achieved": kv["GB/s"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": kv["GB/s"] / peaks["hbm_gbs"], "kernel": "atom::decode_attention_kernel",
            "peak_source": f"{peak_src} HBM copy bandwidth"}),
        "clocks": sampler.summary(),
        "e2e": e2e,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(M, N, K, target_s=args.cpu_seconds)
    print(json.dumps(line), flush=True)


def time_atom_fp(atom, xd, perm, M, N, K, args, dev, flush_l2):
    """NEXT-2: the same layer as Atom (FP) -- MXFP4 E2M1 blocks of 32 + MXFP8 E4M3 outliers
    with UE8M0 scales on tcgen05 block-scaled MMAs.  Weights MX-quantized offline (untimed); the
    step (activation quantize + GEMM) and each kernel alone timed as CUDA graphs, L2 flushed
    before every replay."""
    import torch
    W = torch.from_numpy(synth.weights(N, K, args.seed)).to(dev)
    wq = atom.mx_quantize(W, perm)
    del W
    aq = atom.mx_quantize(xd, perm)
    c = atom.mx_gemm(aq, wq)
    graphs = {}
    atom.mx_quantize(xd, perm, out=aq)
    n_launch = atom.last_launch_count()
    atom.mx_gemm(aq, wq, out=c)
    n_launch += atom.last_launch_count()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for name, fn in (("quant", lambda: atom.mx_quantize(xd, perm, out=aq, stream=side)),
                         ("gemm", lambda: atom.mx_gemm(aq, wq, out=c, stream=side)),
                         ("step", lambda: (atom.mx_quantize(xd, perm, out=aq, stream=side),
                                           atom.mx_gemm(aq, wq, out=c, stream=side)))):
            fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                fn()
            graphs[name] = g
    torch.cuda.current_stream().wait_stream(side)
    out = {}
    n = max(5, args.steps // 2)
    for name, g in graphs.items():
        for _ in range(3):
            g.replay()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n)]
        for i in range(n):
            if not args.no_flush:
                flush_l2()
            ev[i][0].record()
            g.replay()
            ev[i][1].record()
        torch.cuda.synchronize()
        out[f"{name}_us"] = 1e3 * sum(a.elapsed_time(b) for a, b in ev) / n
    ops = 2.0 * M * N * K
    out["TOPS_step"] = ops / (out["step_us"] * 1e-6) / 1e12
    out["TOPS_gemm"] = ops / (out["gemm_us"] * 1e-6) / 1e12
    out["format"] = "MXFP4 E2M1 (blocks of 32) + 128 MXFP8 E4M3 outlier channels, UE8M0 scales"
    out["gpu_launches_per_step"] = n_launch
    return out


def time_kv_attention(atom, dev, flush_l2, args, B=128, L=1024, H=32):
    """NEXT-3: one decode step of Llama-7B attention (32 heads x 128) at batch 128
    (the paper's Fig 8b batch) with 1024 cached tokens per sequence, over the INT4 paged cache;
    the cache is built (quantized) untimed, the attention timed as a CUDA graph after an L2
    flush.  Algorithmic bytes: K and V codes + (s, mn) per (token, head) = 2 x 72 B."""
    import torch
    rng = np.random.default_rng(args.seed)
    pages = (L + 15) // 16
    bt = torch.from_numpy(rng.permutation(B * pages).reshape(B, pages).astype(np.int32)).to(dev)
    k, v = atom.KvCache.empty(B * pages, H, dev), atom.KvCache.empty(B * pages, H, dev)
    slots = (bt[:, :, None] * 16 + torch.arange(16, device=dev)).reshape(B, -1)[:, :L].int()
    gen = torch.Generator(device=dev).manual_seed(args.seed)
    for b in range(B):
        x = torch.randn((L, H * 128), device=dev, generator=gen).half()
        atom.kv_quantize(x, slots[b].contiguous(), k)
        atom.kv_quantize(x * 0.5, slots[b].contiguous(), v)
    q = torch.randn((B, H, 128), device=dev, generator=gen).half()
    sl = torch.full((B,), L, dtype=torch.int32, device=dev)
    out = atom.decode_attention(q, k, v, bt, sl, L)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        atom.decode_attention(q, k, v, bt, sl, L, out=out, stream=side)
        launches = atom.last_launch_count()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            atom.decode_attention(q, k, v, bt, sl, L, out=out, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    n = max(5, args.steps // 2)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n)]
    for i in range(n):
        if not args.no_flush:
            flush_l2()
        ev[i][0].record()
        g.replay()
        ev[i][1].record()
    torch.cuda.synchronize()
    us = 1e3 * sum(a.elapsed_time(b) for a, b in ev) / n
    nbytes = 2 * B * L * H * (64 + 8)
    return {"us": us, "GB/s": nbytes / (us * 1e-6) / 1e9, "bytes": nbytes,
            "shape": {"batch": B, "seq_len": L, "heads": H, "head_dim": 128},
            "format": "INT4 asymmetric per (token, head), 16-token pages",
            "gpu_launches_per_step": launches}


def _spawn_ranks(args) -> int:
    """`python bench.py --gpus N` (N > 1) without a torchrun environment: re-launch this script
    as N ranks on this node (torch.distributed.run, one process per GPU, rendezvous on
    127.0.0.1), exactly the launch the driver uses, and return the launcher's exit code."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def run_dry(args, M, N, K, cfg_name, world, rank):
    """--dry-run: the multi-rank plumbing without a GPU (gloo on CPU): every rank derives its
    shard, the shard table is all-gathered, rank 0 prints it as one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2310_19102_b200 import tp
    if args.shard == "n":
        lo, hi = tp.n_shard_rows(N, world, rank)
    else:
        g0, g1 = tp.k_shard_groups(K, world, rank)
        lo, hi = g0 * 128, g1 * 128
    mine = torch.tensor([rank, lo, hi], dtype=torch.int64)
    table = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_gather(table, mine)
    else:
        table = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "config": {"workload": cfg_name},
                          "shard": args.shard,
                          "ranks": [[int(v) for v in t.tolist()] for t in table]}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["atom", "reference"], default="atom")
    ap.add_argument("--config", choices=list(CONFIGS), default="cfg5")
    ap.add_argument("--shard", choices=["n", "k"], default="n")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--spinup", type=float, default=0.5, help="seconds of untimed clock spin-up")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the step's kernels directly instead of replaying CUDA graphs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-peak", action="store_true", help="skip the in-run int8 peak measurement")
    ap.add_argument("--no-mx", action="store_true", help="skip the NEXT-2 Atom (FP) MX timing")
    ap.add_argument("--no-kv", action="store_true", help="skip the NEXT-3 KV attention timing")
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="token chunks of the pipelined e2e step (1 = sequential)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="multi-rank plumbing only (gloo, no GPU work): prints the shard table")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "W >= 3 warm-up steps"

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    M, N, K, _ = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, M, N, K, args.config, world, rank)
        return
    if args.dry_run:
        import torch.distributed as dist
        if world > 1:
            dist.init_process_group("gloo")
        try:
            run_dry(args, M, N, K, args.config, world, rank)
        finally:
            if world > 1:
                dist.destroy_process_group()
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # communicator setup (ring / NVLS) is logged per rank beside the bench output
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", str(ROOT / "gpurun_out" / "nccl.%h.%p.log"))
        (ROOT / "gpurun_out").mkdir(exist_ok=True)
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_atom(args, M, N, K, args.config, world, rank, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
