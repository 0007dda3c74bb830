#!/usr/bin/env python
"""flute-b200 benchmark — LUT-GEMM µs & effective HBM GB/s (BASELINE.json).

Workloads (``--workload``; ``config.workload`` names the one measured):

* ``headline`` (default) — BASELINE.json configs[0] + configs[1], the W3/W4
  g128 M=1–32 cases the metric is quoted on: W4 NF g128 K=N=4096 (LLaMA-3-8B
  q_proj) at M=1 and M=16, and W3 NF g128 on the LLaMA-3-8B MLP shapes
  (K,N) = (4096,14336), (14336,4096) at M = 1, 4, 16, 32.  One *step* = one
  pass over those 10 GEMMs.
* ``sweep`` — configs[2]: W2/W3/W4 x g32/64/128/256 on K=N=8192, M = 1, 4,
  16, 32 (48 GEMMs per step), every case next to cuBLAS fp16.
* ``tc`` — configs[4]: W4 g128 M = 64…512 on 4096² and 8192² (tcgen05/TMEM
  kernel), TFLOP/s next to cuBLAS fp16.
* ``70b`` — configs[3]: the LLaMA-3-70B layer K=8192 N=28672 W4 g128 M=1,
  N-sharded over the ranks + output all-gather (strong scaling).

L2: every weight shape has R replicas (R = max(8, ceil(2.5 x L2 / bytes)))
rotated with one counter PER SHAPE, so a replica is reused only after more
than 2.5x the 126 MB L2 of other weights has streamed through.

value  = algorithmic bytes of a step (each byte once) / step
         time: K steps replayed from CUDA graphs (exactly K: full 16-step
         graphs plus a remainder graph), CUDA events on the launching stream,
         max over ranks.
e2e    = the same metric through the public C ABI with HOST buffers:
         flute_host_batch_run per step (H2D of every X, the GEMMs, D2H of
         every Y), wall clock.

``--impl reference`` times the reference's own CPU engine (flutesim::execute,
compiled from the reference sources into oracle/_ref/) on the box's host
cores over the same step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LUT-GEMM µs & effective HBM GB/s (W3/W4 g128, M=1–32) vs 8 TB/s peak"
L2_BYTES = 126 * 1024 * 1024  # replaced by the device's own figure at run time
G = 16                        # steps per captured CUDA graph


def workload_cases(name):
    """[(bits, group, m, k, n)] of one step."""
    if name == "headline":
        c = [(4, 128, m, 4096, 4096) for m in (1, 16)]
        c += [(3, 128, m, k, n) for m in (1, 4, 16, 32) for (k, n) in ((4096, 14336), (14336, 4096))]
        return c
    if name == "sweep":
        return [(b, g, m, 8192, 8192) for b in (2, 3, 4) for g in (32, 64, 128, 256)
                for m in (1, 4, 16, 32)]
    if name == "tc":
        return [(4, 128, m, s, s) for s in (4096, 8192) for m in (64, 128, 256, 512)]
    raise ValueError(name)


WORKLOAD_DESC = {
    "headline": "BASELINE configs[0]+[1]: W4 NF g128 K=N=4096 M=1,16 + W3 NF g128 LLaMA-3-8B MLP "
                "(K,N)=(4096,14336),(14336,4096) M=1,4,16,32; 10 GEMMs/step",
    "sweep": "BASELINE configs[2]: W2/W3/W4 x g32/64/128/256, K=N=8192, M=1,4,16,32; 48 GEMMs/step",
    "tc": "BASELINE configs[4]: W4 NF g128 M=64,128,256,512 on 4096^2 and 8192^2 (tcgen05/TMEM); "
          "8 GEMMs/step",
}


def algo_bytes(m, k, n, bits, group):
    return (k * n * bits + 7) // 8 + (k * n // group) * 2 + m * k * 2 + m * n * 2 + (1 << bits) * 2


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s burst, kind) — MEASURED_PEAKS.json (driver-
    written) else the profiling guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU arm (test infrastructure: oracle/_ref, else the C oracle port)
# ---------------------------------------------------------------------------

class _CpuStep:
    """One workload step on the host cores through the reference's own
    flutesim::execute (oracle/_ref) — or the C oracle port when the reference
    library is absent.  Inputs are prepared once (outside the timed region)."""

    def __init__(self, cases):
        from oracle import Oracle, RefLib
        self.cores = os.cpu_count() or 1
        os.environ.setdefault("OMP_NUM_THREADS", str(self.cores))
        if RefLib.available():
            self.lib, self.kind = RefLib(), "reference"
        else:
            self.lib, self.kind = Oracle(), "port"
        self.cases = cases
        self.inputs = {}
        for i, (bits, group, m, k, n) in enumerate(cases):
            key = (bits, group, k, n)
            if key not in self.inputs:
                rng = np.random.default_rng(100 + i)
                w = rng.standard_normal((k, n), dtype=np.float32)
                idx, scales = self.lib.quantize(w, bits, group)
                self.inputs[key] = (self.lib.pack(idx, bits), scales, self.lib.nf_table(bits))
        rng = np.random.default_rng(7)
        self.xs = {(m, k): (rng.standard_normal((m, k)) * 0.5).astype(np.float16).view(np.uint16)
                   for (_, _, m, k, _) in cases}
        self.step_bytes = sum(algo_bytes(m, k, n, b, g) for (b, g, m, k, n) in cases)

    def run(self):
        per = []
        for (bits, group, m, k, n) in self.cases:
            slices, scales, table = self.inputs[(bits, group, k, n)]
            t0 = time.perf_counter()
            self.lib.execute(self.xs[(m, k)], slices, k, n, bits, group, scales, table,
                             workers=self.cores)
            per.append(time.perf_counter() - t0)
        return per

    def sample_desc(self, per=None):
        s = (f"flutesim::execute ({'reference library oracle/_ref' if self.kind == 'reference' else 'C oracle port'}), "
             f"workers = {self.cores} OpenMP threads, layout 16,64,64,16,8,16")
        if per is not None:
            s += "; one full step: " + "; ".join(
                f"W{b}g{g} M={m} K={k} N={n}: {t * 1e3:.0f} ms"
                for (b, g, m, k, n), t in zip(self.cases, per))
        return s


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cases = workload_cases(args.workload if args.workload != "70b" else "headline")
    steps = args.steps if args.steps is not None else 5
    warmup = args.warmup if args.warmup is not None else 3
    cpu = _CpuStep(cases)
    t_wall = time.perf_counter()
    for _ in range(warmup):
        cpu.run()
    secs, last = [], None
    for _ in range(steps):
        last = cpu.run()
        secs.append(sum(last))
    value = cpu.step_bytes * steps / sum(secs) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 5), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": round(1e3 * sum(secs) / steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC[args.workload if args.workload != "70b" else "headline"],
                   "step_bytes": cpu.step_bytes,
                   "step": "the same GEMMs as the GPU arm's step, reference CPU engine"},
        "cpu_baseline": {"value": round(value, 5), "unit": "GB/s", "cores": cpu.cores, "kind": cpu.kind,
                         "sample": f"{steps} full steps; " + cpu.sample_desc(last)},
        "e2e": {"value": round(value, 5), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_wall, 2),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def _replicas(bytes_):
    return max(8, math.ceil(2.5 * L2_BYTES / bytes_))


def _make_weights(F, cases, rank):
    """{(bits, group, k, n): [DeviceWeights] * R} — R per shape, see module doc."""
    weights = {}
    for i, (bits, group, m, k, n) in enumerate(cases):
        key = (bits, group, k, n)
        if key in weights:
            continue
        rng = np.random.default_rng(1000 * rank + i)
        w = rng.standard_normal((k, n), dtype=np.float32)
        idx, scales = F.quantize_matrix(w, bits, group)
        table = F.build_nf_table(bits)
        r = _replicas(algo_bytes(1, k, n, bits, group))
        # pack once on the host, upload R copies of the device layout
        packed = F.pack_device(idx, bits, group)
        sdev = F.scales_device(scales, k, n, group)
        vl = F.make_vectorized_lut(table, bits)
        weights[key] = [F.DeviceWeights.from_device_layout(packed, sdev, vl, k, n, bits, group)
                        for _ in range(r)]
    return weights


class Rotor:
    """Per-shape replica counters (a replica is reused only after all R of its
    shape have been used)."""

    def __init__(self, weights):
        self.w = weights
        self.c = {k: 0 for k in weights}

    def next(self, key):
        reps = self.w[key]
        dw = reps[self.c[key] % len(reps)]
        self.c[key] += 1
        return dw


def _time_graph(torch, graph, stream, reps, div):
    with torch.cuda.stream(stream):
        for _ in range(2):
            graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps):
            graph.replay()
        e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * div)  # µs per item


def per_case_table(torch, F, cases, weights, xs, ys, stream, peak_gbs, peak_tf):
    """Per-GEMM µs (graph of L launches rotating the shape's replicas) next to
    cuBLAS fp16 (torch.matmul, same shape, same replica rotation)."""
    out = []
    dense_cache = {}
    for (bits, group, m, k, n) in cases:
        key = (bits, group, k, n)
        reps = weights[key]
        L = max(30, 2 * len(reps))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for r in range(L):
                reps[r % len(reps)].gemm(xs[(m, k)], ys[(m, n)], stream=stream.cuda_stream)
        us = _time_graph(torch, g, stream, 10, L)
        del g
        if (k, n) not in dense_cache:
            dense_cache.clear()
            nd = max(3, math.ceil(2.5 * L2_BYTES / (k * n * 2)))
            dense_cache[(k, n)] = [torch.randn(k, n, dtype=torch.float16, device="cuda") for _ in range(nd)]
        wd = dense_cache[(k, n)]
        gc = torch.cuda.CUDAGraph()
        Lc = max(30, 2 * len(wd))
        with torch.cuda.graph(gc, stream=stream):
            for r in range(Lc):
                torch.matmul(xs[(m, k)], wd[r % len(wd)], out=ys[(m, n)])
        cub = _time_graph(torch, gc, stream, 10, Lc)
        del gc
        b = algo_bytes(m, k, n, bits, group)
        gbs = b / us / 1e3
        out.append({"bits": bits, "group": group, "m": m, "k": k, "n": n, "us": round(us, 3),
                    "gbs": round(gbs, 1), "frac": round(gbs / peak_gbs, 4),
                    "tflops": round(2.0 * m * n * k / us / 1e6, 3),
                    "cublas_fp16_us": round(cub, 3),
                    "speedup_vs_cublas": round(cub / us, 3)})
    dense_cache.clear()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F
    global L2_BYTES

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L2_BYTES = torch.cuda.get_device_properties(local).L2_cache_size or L2_BYTES
    steps = args.steps if args.steps is not None else 2000
    warmup = max(3, args.warmup if args.warmup is not None else 32)
    peak_gbs, peak_tf, peak_kind = peaks()

    cases = workload_cases(args.workload)
    step_bytes = sum(algo_bytes(m, k, n, b, g) for (b, g, m, k, n) in cases)
    step_flops = sum(2 * m * n * k for (b, g, m, k, n) in cases)
    weights = _make_weights(F, cases, rank)
    rng = np.random.default_rng(7 + rank)
    xs, ys = {}, {}
    for (b, g, m, k, n) in cases:
        if (m, k) not in xs:
            xs[(m, k)] = torch.from_numpy((rng.standard_normal((m, k)) * 0.5).astype(np.float16)).cuda()
        if (m, n) not in ys:
            ys[(m, n)] = torch.empty((m, n), dtype=torch.float16, device="cuda")
    for reps in weights.values():  # per-handle workspaces for every row class (not capturable)
        for dw in reps:
            dw.reserve(max(m for (_, _, m, _, _) in cases))

    stream = torch.cuda.Stream()
    rotor = Rotor(weights)

    def launch_step():
        for (b, g, m, k, n) in cases:
            rotor.next((b, g, k, n)).gemm(xs[(m, k)], ys[(m, n)], stream=stream.cuda_stream)

    with torch.cuda.stream(stream):
        for _ in range(2):
            launch_step()
    stream.synchronize()

    def capture(nsteps):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            for _ in range(nsteps):
                launch_step()
        return gr

    # exactly `steps` timed steps: full G-step graphs + one remainder graph
    # (the remainder graph continues the same per-shape rotation)
    g_full = capture(G)
    rem = steps % G
    g_rem = capture(rem) if rem else None
    stream.synchronize()

    per_case = []
    torch.matmul(xs[(cases[0][2], cases[0][3])],
                 torch.zeros((cases[0][3], cases[0][4]), dtype=torch.float16, device="cuda"))
    torch.cuda.synchronize()  # the cuBLAS handle outside graph capture
    if not args.quick:
        per_case = per_case_table(torch, F, cases, weights, xs, ys, stream, peak_gbs, peak_tf)

    # ---- warm-up: exactly `warmup` steps, eager (same kernels, same rotation) ----
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            launch_step()
        g_full.replay()  # graph upload outside the timed region
        if g_rem is not None:
            g_rem.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(steps // G):
            g_full.replay()
        if g_rem is not None:
            g_rem.replay()
        e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    elapsed_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / steps
    value = world * step_bytes / (ms_per_step * 1e-3) / 1e9

    # ---- end to end through the C ABI with (pinned) host buffers ----
    e2e = run_e2e(torch, dist, F, cases, weights, xs, stream, world, step_bytes, steps)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cs = _CpuStep(cases if args.workload != "sweep" else cases[::4])
            per = cs.run()
            cpu = {"value": round(cs.step_bytes / sum(per) / 1e9, 5), "unit": "GB/s", "cores": cs.cores,
                   "kind": cs.kind, "sample": ("one full step of the workload; " if args.workload != "sweep"
                                               else "every 4th GEMM of the step (M=1 cases); ")
                   + cs.sample_desc(per)}
        achieved = value / world
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": round(ms_per_step, 6),
            "us_per_gemm": round(ms_per_step * 1e3 / len(cases), 3),
            "tflops": round(world * step_flops / (ms_per_step * 1e-3) / 1e12, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (N(0,1) weights NF-quantized, N(0,0.25) activations)",
            "config": {"workload": WORKLOAD_DESC[args.workload],
                       "l2": "inputs larger than L2: per-shape weight replica rotation, "
                             + ", ".join(f"W{b}g{g} {k}x{n}: {len(v)} replicas"
                                         for (b, g, k, n), v in weights.items()),
                       "parallelism": f"weak: {world} GPU(s) each run the full per-GPU workload",
                       "step_bytes": step_bytes,
                       "timing": f"CUDA graphs of {G} steps (+ a {rem}-step remainder graph), "
                                 "events on the launching stream"},
            "roofline": {"bound": "hbm" if args.workload != "tc" else "tensor",
                         "achieved": round(achieved, 1) if args.workload != "tc"
                         else round(step_flops / (ms_per_step * 1e-3) / 1e12, 2),
                         "peak": peak_gbs if args.workload != "tc" else peak_tf,
                         "unit": "GB/s" if args.workload != "tc" else "TFLOP/s",
                         "frac": round(achieved / peak_gbs, 4) if args.workload != "tc"
                         else round(step_flops / (ms_per_step * 1e-3) / 1e12 / peak_tf, 4),
                         "peak_kind": peak_kind,
                         # ncu dram__bytes_read.sum + dram__bytes_write.sum of one
                         # W3 M=1 4096x14336 launch (profiles/); its algorithmic
                         # bytes are 22,974,480 (no re-reads)
                         "traffic": 23003904 if args.workload == "headline" else None,
                         "traffic_case": ("W3 g128 M=1 K=4096 N=14336, DRAM bytes per launch (ncu)"
                                          if args.workload == "headline" else None),
                         "kernel": ("qgemm_tc_kernel<4,BN> (+ splitk_reduce_kernel) = every launch "
                                    "of the step (achieved = step FLOPs / step time)"
                                    if args.workload == "tc" else
                                    "qgemm_mma_kernel<BITS,BM,...> = every launch of the step "
                                    "(achieved = step bytes / step time)")},
            "e2e": e2e,
            "gpu_launches": steps * len(cases),
            "clocks": clocks,
            "cases": per_case,
        }
        if args.workload == "headline" and per_case:
            c1 = [c for c in per_case if c["bits"] == 4 and c["k"] == 4096 and c["n"] == 4096]
            out["north_star"] = {
                "config": "BASELINE configs[0]: W4 NF g128 K=N=4096 (target: >=70% of HBM peak at M=1, "
                          ">=2.5x cuBLAS fp16 at M<=16)",
                "target_us_70pct": round(algo_bytes(1, 4096, 4096, 4, 128) / (0.7 * peak_gbs) / 1e3, 3),
                "cases": c1}
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_e2e(torch, dist, F, cases, weights, xs, stream, world, step_bytes, steps):
    """One flute_host_batch_run per step: every GEMM's X copied in from pinned
    host memory and its Y copied back (captured once per replica set as a
    CUDA graph by the library), wall clock, median of 5 rounds."""
    e2e_steps = max(5, min(200, steps // 10))
    # Johnson's rule for the copy-in -> copy-out flow shop: items whose input
    # is no larger than their output first (ascending input), then the rest
    # (descending output); inputs back to back in one pinned buffer and outputs
    # in another, in that order, so each copy group is a single transfer.
    order = sorted(cases, key=lambda c: (0, c[2] * c[3]) if c[3] <= c[4] else (1, -c[2] * c[4]))
    x_arena = torch.empty(sum(m * k for (_, _, m, k, _) in order), dtype=torch.float16).pin_memory()
    y_arena = torch.empty(sum(m * n for (_, _, m, _, n) in order), dtype=torch.float16).pin_memory()
    x_host, y_host = [], []
    xo = yo = 0
    for (b, g, m, k, n) in order:
        xh = x_arena[xo:xo + m * k].numpy().view(np.uint16).reshape(m, k)
        xh[...] = xs[(m, k)].cpu().numpy().view(np.uint16)
        x_host.append(xh)
        y_host.append(y_arena[yo:yo + m * n].numpy().view(np.uint16).reshape(m, n))
        xo += m * k
        yo += m * n
    rot = Rotor(weights)
    nb = max(len(v) for v in weights.values())
    batches = []
    for _ in range(nb):  # one host batch per replica set, prepared once
        items = [(rot.next((b, g, k, n)), x_host[i], y_host[i]) for i, (b, g, m, k, n) in enumerate(order)]
        batches.append(F.HostBatch(items))
    for _ in range(2):
        for bt in batches:
            bt.run(stream.cuda_stream)

    def rounds(fn, nrounds=5):
        per = max(4, e2e_steps // nrounds)
        out = []
        for r in range(nrounds):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            fn(r * per, per)
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t.item())
            out.append(dt / per)
        return out

    def run_batches(s0, count):
        for s_ in range(s0, s0 + count):
            batches[s_ % nb].run(stream.cuda_stream)

    rs = rounds(run_batches)
    val = world * step_bytes / statistics.median(rs) / 1e9
    h2d = sum(m * k * 2 for (_, _, m, k, _) in cases)
    d2h = sum(m * n * 2 for (_, _, m, _, n) in cases)
    return {"value": round(val, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "flute_host_batch_run (C ABI; the library captures the batch once as a CUDA graph): "
                    "per step every GEMM's X copied in from pinned host memory and Y copied out, "
                    "pipelined with the GEMMs; wall clock, one synchronous call per step, median of 5 rounds",
            "steps": 5 * max(4, e2e_steps // 5),
            "rounds_gbs": [round(world * step_bytes / t / 1e9, 1) for t in rs]}


def run_sharded_70b(args):
    """BASELINE.json configs[3]: one LLaMA-3-70B MLP layer (K=8192, N=28672, W4
    NF g128, M=1), N-sharded over the ranks; a step = each rank's shard GEMM +
    the output all-gather (NCCL, or the fused peer-store epilogue with
    --allgather peer).  Strong scaling: the layer is fixed as N grows."""
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F
    from paper_2407_10960_b200.sharded import NativeShardedWeights, NcclComm

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local))
    steps = args.steps if args.steps is not None else 400
    warmup = max(3, args.warmup if args.warmup is not None else 20)
    k, n, bits, group, m = 8192, 28672, 4, 128, 1
    rng = np.random.default_rng(70)
    w = rng.standard_normal((k, n), dtype=np.float32)
    idx, scales = F.quantize_matrix(w, bits, group)
    table = F.build_nf_table(bits)
    shard_bytes = F.shard_range(k, n, bits, group, world, rank).w_bytes
    reps = max(2, int(np.ceil(3 * 126e6 / shard_bytes)))
    comm = NcclComm(rank, world)  # C++ communicator (NCCL loaded by the library)
    sws = [NativeShardedWeights(comm, idx, scales, table, bits, group, max_m=m)
           for _ in range(min(reps, 24))]
    x = torch.from_numpy((rng.standard_normal((m, k)) * 0.5).astype(np.float16)).cuda()
    y = torch.empty((m, n), dtype=torch.float16, device="cuda")
    layer_bytes = algo_bytes(m, k, n, bits, group)
    stream = torch.cuda.current_stream().cuda_stream

    def step(i):
        if args.allgather == "peer":
            sws[i % len(sws)].gemm_fused(x, stream=stream)
        else:
            sws[i % len(sws)].gemm(x, y, stream=stream)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        step(i)
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    peak, _, peak_kind = peaks()
    if rank == 0:
        per_gpu = (shard_bytes + F.shard_range(k, n, bits, group, world, 0).s_bytes + m * k * 2
                   + m * (n // world) * 2) / (ms * 1e-3) / 1e9
        print(json.dumps({
            "metric": METRIC, "value": round(layer_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": round(ms, 6),
            "us_per_layer": round(ms * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic (N(0,1) weights NF4 g128)",
            "config": {"workload": "BASELINE configs[3]: LLaMA-3-70B layer K=8192 N=28672 W4 g128 "
                                   "M=1, N-sharded + output all-gather",
                       "allgather": args.allgather + (" (flute_sharded_gemm: shard GEMM + ncclAllGather)"
                                                      if args.allgather == "nccl" else
                                                      " (flute_sharded_gemm_fused: peer-store epilogue + "
                                                      "device flag barrier)"),
                       "layer_bytes": layer_bytes,
                       "l2": f"{len(sws)} weight replicas rotated (>= 3x L2 per rank)"},
            "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_gpu / peak, 4), "peak_kind": peak_kind,
                         "note": "per-GPU shard bytes / step time (includes the all-gather)"},
            "gpu_launches": steps, "clocks": clocks}), flush=True)
    dist.barrier()
    del sws
    comm.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip the per-case table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--workload", default="headline", choices=["headline", "sweep", "tc", "70b"])
    ap.add_argument("--allgather", default="nccl", choices=["nccl", "peer"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "70b":
        if "MASTER_ADDR" not in os.environ:
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29531", RANK="0", WORLD_SIZE="1",
                              LOCAL_RANK="0")
        return run_sharded_70b(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
