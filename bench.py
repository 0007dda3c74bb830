#!/usr/bin/env python
"""flute-b200 benchmark — LUT-GEMM µs & effective HBM GB/s (BASELINE.json).

Workload (config.workload): BASELINE.json configs[1] — W3 NF-LUT g128 on the
LLaMA-3-8B MLP shapes (K,N) = (4096,14336) and (14336,4096) at M = 1, 4, 16,
32.  One *step* = one pass over those 8 GEMMs.  Each GEMM launch reads a
different weight replica (3 per shape, rotated per call) so every launch
streams its weights from HBM (>= 2x the 126 MB L2 between reuses).

value  = algorithmic bytes of a step (each byte once) / step
         time, whole job, device-timed with CUDA events around K graph-replayed
         steps, max over ranks.
e2e    = the same metric through the public C ABI with HOST buffers
         (flute_gemm_host: H2D of X, GEMM, D2H of Y, synchronised per call).

`--impl reference` times the reference's own CPU engine (flutesim::execute,
compiled from the reference sources into oracle/_ref/) on the box's host cores.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LUT-GEMM µs & effective HBM GB/s (W3/W4 g128, M=1–32) vs 8 TB/s peak"
SHAPES = [(4096, 14336), (14336, 4096)]
MS = [1, 4, 16, 32]
BITS, GROUP = 3, 128
REPLICAS = 6


def algo_bytes(m, k, n, bits=BITS, group=GROUP):
    return (k * n * bits + 7) // 8 + (k * n // group) * 2 + m * k * 2 + m * n * 2 + (1 << bits) * 2


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
# reference CPU arm
# ---------------------------------------------------------------------------

def _ref_inputs(ref, k, n, m, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n), dtype=np.float32)
    idx, scales = ref.quantize(w, BITS, GROUP)
    slices = ref.pack(idx, BITS)
    table = ref.nf_table(BITS)
    x16 = (rng.standard_normal((m, k)) * 0.5).astype(np.float16).view(np.uint16)
    return x16, slices, scales, table


def cpu_reference_sample(cases, max_seconds=20.0, reps=None):
    """Time the reference's own execute (oracle/_ref) — or the C oracle port
    when the reference .so is absent — on a bounded sample of the workload."""
    from oracle import Oracle, RefLib
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    if RefLib.available():
        lib, kind = RefLib(), "reference"
    else:
        lib, kind = Oracle(), "port"
    tot_bytes, tot_s, done = 0, 0.0, []
    t_start = time.perf_counter()
    for i, (m, k, n) in enumerate(cases):
        x16, slices, scales, table = _ref_inputs(lib if kind == "reference" else RefLibShim(lib),
                                                 k, n, m, 100 + i)
        t0 = time.perf_counter()
        if kind == "reference":
            lib.execute(x16, slices, k, n, BITS, GROUP, scales, table, workers=cores)
        else:
            lib.execute(x16, slices, k, n, BITS, GROUP, scales, table, workers=cores)
        dt = time.perf_counter() - t0
        tot_bytes += algo_bytes(m, k, n)
        tot_s += dt
        done.append(f"M={m} K={k} N={n}: {dt * 1e3:.0f} ms")
        if reps is None and time.perf_counter() - t_start > max_seconds:
            break
    return {"value": tot_bytes / tot_s / 1e9, "unit": "GB/s", "cores": cores, "kind": kind,
            "sample": f"flutesim::execute W{BITS}g{GROUP}, workers=OMP threads={cores}, layout "
                      f"16,64,64,16,8,16; " + "; ".join(done)}


class RefLibShim:
    """Input producer for the oracle-port CPU baseline (same API subset)."""

    def __init__(self, orc):
        self.o = orc

    def quantize(self, w, bits, group):
        return self.o.quantize(w, bits, group)

    def pack(self, idx, bits):
        return self.o.pack(idx, bits)

    def nf_table(self, bits):
        return self.o.nf_table(bits)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cases = [(m, k, n) for m in MS for (k, n) in SHAPES]
    vals, secs = [], []
    total_bytes = 0
    t0 = time.perf_counter()
    for step in range(args.warmup + args.steps):
        m, k, n = cases[step % len(cases)]
        s = cpu_reference_sample([(m, k, n)], reps=1)
        if step >= args.warmup:
            vals.append(s["value"])
            secs.append(algo_bytes(m, k, n) / (s["value"] * 1e9))
            total_bytes += algo_bytes(m, k, n)
            kind, cores = s["kind"], s["cores"]
    value = total_bytes / sum(secs) / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(secs) / len(secs), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": "BASELINE configs[1]: W3 g128 LLaMA-3-8B MLP shapes, M=1,4,16,32",
                   "step": "one GEMM of the 8-case workload per step (rotating), reference CPU engine"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": f"{args.steps} GEMMs of the workload, flutesim::execute with "
                                   f"workers = {cores} OpenMP threads"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def make_case_weights(F, k, n, seed):
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((k, n), dtype=np.float32)
    idx, scales = F.quantize_matrix(w, BITS, GROUP)
    table = F.build_nf_table(BITS)
    return idx, scales, table


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    # weights: REPLICAS per shape (weak scaling: every rank owns its own copy of
    # the per-GPU workload)
    weights = {}
    for si, (k, n) in enumerate(SHAPES):
        idx, scales, table = make_case_weights(F, k, n, 1000 * rank + si)
        weights[(k, n)] = [F.DeviceWeights(idx, scales, table, BITS, GROUP) for _ in range(REPLICAS)]
    rng = np.random.default_rng(7 + rank)
    xs = {}
    for m in MS:
        for (k, n) in SHAPES:
            x = torch.from_numpy((rng.standard_normal((m, k)) * 0.5).astype(np.float16)).cuda()
            xs[(m, k)] = x
    ys = {(m, n): torch.empty((m, n), dtype=torch.float16, device="cuda")
          for m in MS for (_, n) in SHAPES}
    # load-time autotuning (public API; outside the timed region): pick the
    # work decomposition per weight handle and row class
    tuned = {}
    if args.autotune:
        for (k, n), reps in weights.items():
            for m in MS:
                for dw in reps:
                    r = dw.autotune(m)
                tuned[f"M={m} K={k} N={n}"] = min(
                    (ln for ln in r.splitlines() if ln.strip()),
                    key=lambda ln: float(ln.split(":")[-1].split()[0]))
    cases = [(m, k, n) for m in MS for (k, n) in SHAPES]
    step_bytes = sum(algo_bytes(m, k, n) for (m, k, n) in cases)

    stream = torch.cuda.Stream()
    counter = [0]

    def launch_step():
        for (m, k, n) in cases:
            dw = weights[(k, n)][counter[0] % REPLICAS]
            counter[0] += 1
            dw.gemm(xs[(m, k)], ys[(m, n)], stream=stream.cuda_stream)

    # ---- capture G steps into one CUDA graph (launch-overhead free replay) ----
    G = 16
    with torch.cuda.stream(stream):
        for _ in range(3):
            launch_step()
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for _ in range(G):
            launch_step()
    stream.synchronize()
    reps_warm = max(1, (args.warmup + G - 1) // G)
    reps = max(1, (args.steps + G - 1) // G)
    steps = reps * G

    # ---- per-case microbenchmarks (ours + cuBLAS fp16), not the headline ----
    torch.matmul(xs[(1, SHAPES[0][0])], torch.zeros(SHAPES[0], dtype=torch.float16, device="cuda"))
    torch.cuda.synchronize()  # create the cuBLAS handle outside graph capture
    per_case = []
    if not args.quick:
        for (m, k, n) in cases:
            gcase = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gcase, stream=stream):
                for r in range(30):
                    weights[(k, n)][r % REPLICAS].gemm(xs[(m, k)], ys[(m, n)], stream=stream.cuda_stream)
            wd = [torch.randn(k, n, dtype=torch.float16, device="cuda") for _ in range(REPLICAS)]
            gcb = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gcb, stream=stream):
                for r in range(30):
                    torch.matmul(xs[(m, k)], wd[r % REPLICAS], out=ys[(m, n)])
            res = {}
            for name, gr in (("ours", gcase), ("cublas_fp16", gcb)):
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        gr.replay()
                torch.cuda.synchronize()  # warm replays must not spill into the timed ones
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record()
                    for _ in range(10):
                        gr.replay()
                    e1.record()
                e1.synchronize()
                res[name] = e0.elapsed_time(e1) * 1e3 / 300.0
            del wd
            b = algo_bytes(m, k, n)
            per_case.append({"m": m, "k": k, "n": n, "us": round(res["ours"], 3),
                             "gbs": round(b / res["ours"] / 1e3, 1),
                             "cublas_fp16_us": round(res["cublas_fp16"], 3),
                             "speedup_vs_cublas": round(res["cublas_fp16"] / res["ours"], 2)})

    # ---- timed region ----
    with torch.cuda.stream(stream):
        for _ in range(reps_warm):
            graph.replay()
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
        for _ in range(reps):
            graph.replay()
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

    # ---- end-to-end through the C ABI with (pinned) host buffers ----
    e2e_steps = max(3, min(200, args.steps // 20))
    # The step's 8 GEMMs are independent, so the host batch runs them in the
    # order that best overlaps the copies with the GEMMs — Johnson's rule for
    # the copy-in -> copy-out flow shop: items whose input is no larger than
    # their output first (ascending input), then the rest (descending output).
    # Their inputs sit back to back in one pinned buffer and their outputs in
    # another, in that order, so each copy group is a single transfer.
    e2e_order = sorted(cases, key=lambda c: (0, c[0] * c[1]) if c[1] <= c[2] else (1, -c[0] * c[2]))
    x_arena = torch.empty(sum(m * k for (m, k, _) in cases), dtype=torch.float16).pin_memory()
    y_arena = torch.empty(sum(m * n for (m, _, n) in cases), dtype=torch.float16).pin_memory()
    x_host, y_host = {}, {}
    xo = yo = 0
    for (m, k, n) in e2e_order:
        x_host[(m, k)] = x_arena[xo:xo + m * k].numpy().view(np.uint16).reshape(m, k)
        x_host[(m, k)][...] = xs[(m, k)].cpu().numpy().view(np.uint16)
        y_host[(m, n)] = y_arena[yo:yo + m * n].numpy().view(np.uint16).reshape(m, n)
        xo += m * k
        yo += m * n
    # one step = one flute_gemm_host_batch call over the step's 8 GEMMs: every
    # input copied in from pinned host memory and every output copied back,
    # pipelined with the GEMMs; the call returns with all outputs on the host
    def e2e_items(step):
        return [(weights[(k, n)][(step * len(cases) + i) % REPLICAS], x_host[(m, k)],
                 y_host[(m, n)]) for i, (m, k, n) in enumerate(e2e_order)]

    batches = [F.HostBatch(e2e_items(s_)) for s_ in range(REPLICAS)]  # prepared once
    for _ in range(4):  # warm (first replays upload the graphs)
        for b in batches:
            b.run(stream.cuda_stream)
    def timed_rounds(fn, rounds=5):
        """wall seconds per step of each round (max over ranks); the median is
        reported, so one host hiccup does not decide the number"""
        per = max(4, e2e_steps // rounds)
        out = []
        for r in range(rounds):
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
            batches[s_ % REPLICAS].run(stream.cuda_stream)

    def run_single(s0, count):
        cnt = s0 * len(cases)
        for _ in range(count):
            for (m, k, n) in cases:
                weights[(k, n)][cnt % REPLICAS].gemm_host(x_host[(m, k)], out=y_host[(m, n)])
                cnt += 1

    e2e_rounds = timed_rounds(run_batches)
    single_rounds = timed_rounds(run_single)
    e2e_value = world * step_bytes / statistics.median(e2e_rounds) / 1e9
    e2e_single = world * step_bytes / statistics.median(single_rounds) / 1e9
    h2d = sum(m * k * 2 for (m, k, n) in cases)
    d2h = sum(m * n * 2 for (m, k, n) in cases)

    peak, peak_kind = peaks()
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_reference_sample([(1, 4096, 14336), (1, 14336, 4096), (4, 4096, 14336)],
                                       max_seconds=15.0)
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": steps, "warmup": reps_warm * G, "ms_per_step": round(ms_per_step, 6),
            "us_per_gemm": round(ms_per_step * 1e3 / len(cases), 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (N(0,1) weights NF3-quantized g128, N(0,0.25) activations)",
            "config": {"workload": "BASELINE configs[1]: W3 NF-LUT g128, LLaMA-3-8B MLP "
                                   "(K,N)=(4096,14336),(14336,4096), M=1,4,16,32; 8 GEMMs/step",
                       "l2": f"inputs larger than L2: {REPLICAS} weight replicas per shape "
                             "rotated per launch",
                       "parallelism": f"weak: {world} GPU(s) each run the full per-GPU workload",
                       "step_bytes": step_bytes, "timing": "CUDA graph of 16 steps, events",
                       "autotune": tuned or "off"},
            "roofline": {"bound": "hbm", "achieved": round(value / world, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(value / world / peak, 4),
                         "peak_kind": peak_kind,
                         # ncu dram__bytes_read.sum + dram__bytes_write.sum of one
                         # W3 M=1 4096x14336 launch (profiles/r1/ncu_full_r1m.txt);
                         # its algorithmic bytes are 22,974,480 (no re-reads)
                         "traffic": 23003136,
                         "traffic_case": "W3 g128 M=1 K=4096 N=14336, bytes per launch",
                         "kernel": "qgemm_mma_kernel<3,BM> (all 8 launches of a step)"},
            "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "flute_host_batch_run (C ABI, CUDA graph captured once): per "
                            "step the 8 GEMMs' X copied in from pinned host memory and Y copied "
                            "out (grouped copies on two copy streams, pipelined with the GEMMs); "
                            "wall clock, one synchronous call per step, median of 5 rounds",
                    "steps": e2e_steps,
                    "rounds_gbs": [round(world * step_bytes / t / 1e9, 1) for t in e2e_rounds],
                    "per_call_value": round(e2e_single, 2),
                    "per_call_path": "flute_gemm_host, one synchronous call per GEMM"},
            "gpu_launches": steps * len(cases),
            "clocks": clocks,
            "cases": per_case,
        }
        if cpu is not None:
            out["cpu_baseline"] = cpu
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded_70b(args):
    """BASELINE.json configs[3]: one LLaMA-3-70B MLP layer (K=8192, N=28672, W4
    NF g128, M=1), N-sharded over the ranks; a step = each rank's shard GEMM +
    the output all-gather (NCCL, or the fused peer-store epilogue with
    --allgather peer).  Strong scaling: the layer is fixed as N grows."""
    import torch
    import torch.distributed as dist
    import paper_2407_10960_b200 as F
    from paper_2407_10960_b200.sharded import ShardedWeights

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local))
    k, n, bits, group, m = 8192, 28672, 4, 128, 1
    rng = np.random.default_rng(70)
    w = rng.standard_normal((k, n), dtype=np.float32)
    idx, scales = F.quantize_matrix(w, bits, group)
    table = F.build_nf_table(bits)
    shard_bytes = F.shard_range(k, n, bits, group, world, rank).w_bytes
    reps = max(2, int(np.ceil(3 * 126e6 / shard_bytes)))
    sws = [ShardedWeights(idx, scales, table, bits, group, rank, world, mode=args.allgather)
           for _ in range(min(reps, 24))]
    x = torch.from_numpy((rng.standard_normal((m, k)) * 0.5).astype(np.float16)).cuda()
    layer_bytes = algo_bytes(m, k, n, bits, group)
    for i in range(args.warmup):
        sws[i % len(sws)].gemm(x)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        y = sws[i % len(sws)].gemm(x)
    e1.record()
    e1.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = sampler.stop()
    t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    peak, peak_kind = peaks()
    if rank == 0:
        per_gpu = (shard_bytes + F.shard_range(k, n, bits, group, world, 0).s_bytes + m * k * 2
                   + m * (n // world) * 2) / (ms * 1e-3) / 1e9
        print(json.dumps({
            "metric": METRIC, "value": round(layer_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 6),
            "us_per_layer": round(ms * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic (N(0,1) weights NF4 g128)",
            "config": {"workload": "BASELINE configs[3]: LLaMA-3-70B layer K=8192 N=28672 W4 g128 "
                                   "M=1, N-sharded + output all-gather",
                       "allgather": args.allgather, "layer_bytes": layer_bytes,
                       "l2": f"{len(sws)} weight replicas rotated (>= 3x L2 per rank)"},
            "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(per_gpu / peak, 4), "peak_kind": peak_kind,
                         "note": "per-GPU shard bytes / step time (includes the all-gather)"},
            "gpu_launches": args.steps, "clocks": clocks}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4000)
    ap.add_argument("--warmup", type=int, default=32)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--quick", action="store_true", help="skip per-case micro-benchmarks")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--autotune", action="store_true",
                    help="run DeviceWeights.autotune per handle and row class at load time "
                         "(isolated cold-launch criterion; the heuristic matches it on this workload)")
    ap.add_argument("--workload", default="mlp8b", choices=["mlp8b", "70b"],
                    help="mlp8b: configs[1] (default, weak scaling); 70b: configs[3] N-sharded")
    ap.add_argument("--allgather", default="nccl", choices=["nccl", "peer"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
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
