#!/usr/bin/env python
"""Benchmark of the fused MBCI chain (BASELINE.json metric) — one JSON line on rank 0.

Default workload (N = 1): BASELINE.json configs[1], BERT-base self-attention chain,
batch 8 x 12 heads, seq 512, head_dim 64, fp16, scale 1/8 + softmax.
A "step" is one fused-chain launch over the whole batch (every §8(a) row on the path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {cuda,reference}]
                    [--config C2|C3|C4-16|...|C6] [--no-cpu-baseline]

Multi-GPU (one rank per GPU; `--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset): rank r owns the contiguous β range [r·b/g, (r+1)·b/g) of the global batch
(SURVEY §8(e)).  `--scaling strong` (default for C2 and C5) splits the config's batch over the
ranks; `--scaling weak` gives every rank the full per-GPU batch.  No collective on the data
path; NCCL only for the barrier, the MAX over ranks of device time, the SUM of bytes and,
after timing, an all-gather of E that the cpu_baseline leg checks against the oracle on rank 0.

Timing: inputs resident in HBM; `rot` sets of (A, B, D, E) used round-robin so the
working set between reuses exceeds 2x L2 (126 MB) — no step hits L2-resident inputs;
the K steps are captured once in a CUDA graph and replayed on a dedicated stream,
bracketed by CUDA events on that stream (plus barrier + synchronize); max over ranks.
`e2e` times mbci_chain_run_host (pinned host buffers, H2D inputs + D2H E every step).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same
workload (rank 0 only).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-chain µs and HBM GB/s (% of B200 peak), BERT-base attn, 1/2/4/8 GPU"

# name: (dtype, batch x heads, M, N, K, L, op, description)
CONFIGS = {
    "C1": ("f32", 1, 128, 128, 16, 16, "none", "fp32 chain E=(A.B).D, batch 1, M=N=128, K=L=16, no inter-op"),
    "C2": ("f16", 96, 512, 512, 64, 64, "softmax",
           "BERT-base self-attention chain fp16: batch 8 x 12 heads, seq 512, head_dim 64, scale 1/8 + softmax"),
    "C3": ("bf16", 128, 1024, 1024, 64, 64, "softmax",
           "BERT-large attention chain bf16: batch 8 x 16 heads, seq 1024, head_dim 64, scale+softmax"),
    "C4-16": ("bf16", 64, 2048, 2048, 16, 16, "none", "plain chain bf16: batch 64, M=N=2048, K=L=16"),
    "C4-32": ("bf16", 64, 2048, 2048, 32, 32, "none", "plain chain bf16: batch 64, M=N=2048, K=L=32"),
    "C4-64": ("bf16", 64, 2048, 2048, 64, 64, "none", "plain chain bf16: batch 64, M=N=2048, K=L=64"),
    "C4-128": ("bf16", 64, 2048, 2048, 128, 128, "none", "plain chain bf16: batch 64, M=N=2048, K=L=128"),
    "C5": ("bf16", 512, 4096, 4096, 128, 128, "softmax",
           "long-sequence attention chain bf16: batch 32 x 16 heads, seq 4096, head_dim 128"),
    "C6": ("f16", 96, 256, 256, 64, 64, "softmax", "ViT-base attention chain fp16: batch 8 x 12 heads, seq 256, d 64"),
}

L2_BYTES = 126 * 1024 * 1024


def peaks():
    p = {"hbm_gbs": None, "bf16_tflops": None, "bf16_tflops_sustained": None, "src": "fallback"}
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            j = json.load(f)
        p.update({k: j.get(k) for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained")})
        p["src"] = "measured (MEASURED_PEAKS.json)"
    if p["hbm_gbs"] is None:   # B200_PROFILING.md fallback
        p.update(hbm_gbs=6650.0, bf16_tflops=1590.0, bf16_tflops_sustained=1400.0, src="fallback (B200_PROFILING.md)")
    return p


def cfg_numbers(name):
    dtype, b, M, N, K, L, op, desc = CONFIGS[name]
    s = 4 if dtype == "f32" else 2
    bytes_ = b * (M * K + K * N + N * L + M * L) * s       # A, B, D, E only
    flops = 2.0 * b * M * N * (K + L)
    exps = b * M * N if op == "softmax" else 0
    return dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu_id)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 <= t <= t1 + 0.15] or [r for (_, r) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in rows if len(r) > 2 and num(r[1]) is not None]
        smax = [num(r[2]) for r in rows if len(r) > 2 and num(r[2]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max((num(r[3]) or 0.0) for r in rows) if rows else None}


# ---------------------------------------------------------------------------- CPU oracle
def time_oracle(name, min_seconds, max_slices=None, seed=0):
    """Oracle on a bounded sample (a few β slices of the workload); returns (GB/s, sample, cores, secs)."""
    import mbci_inputs as gen
    import oracle
    dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps = cfg_numbers(name)
    per_slice = (M * K + K * N + N * L + M * L) * s
    cores = oracle.max_threads()
    nsl = max_slices or max(1, min(b, cores))
    inp = gen.make_chain_inputs(seed, dtype, nsl, M, N, K, L, 1 if op == "softmax" else 0)
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    oracle.chain(inp, op, sc)                      # warm (page-in)
    t0 = time.perf_counter()
    reps = 0
    while True:
        oracle.chain(inp, op, sc)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds:
            break
    sec_per = el / reps
    gbs = nsl * per_slice / sec_per / 1e9
    sample = f"{nsl} of {b} batch x head slices of {name} per step (fp64 unfused chain, {reps} reps, {el:.1f} s)"
    return gbs, sample, cores, sec_per


def gather_check(name, seed, E_all, slices, rows_per_slice=32):
    """cpu_baseline leg, rank 0: sampled rows of the gathered E (every rank's shard) against the
    oracle, each slice's inputs regenerated from the seeded generator (batch_start = β)."""
    import numpy as np
    import mbci_inputs as gen
    import oracle
    dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps = cfg_numbers(name)
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    sig = (1.0, 1.0, 1.0) if op == "softmax" else (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N))
    rng = np.random.default_rng(seed + 17)
    worst = 0.0
    nrows = 0
    for beta in slices:
        inp = gen.make_chain_inputs(seed, dtype, 1, M, N, K, L, 1 if op == "softmax" else 0, sigmas=sig,
                                    batch_start=int(beta))
        ms = np.unique(np.concatenate([[0, M - 1], rng.integers(0, M, rows_per_slice - 2)])).astype(np.int64)
        rows = np.stack([np.zeros_like(ms), ms], axis=1)
        ref = oracle.chain(inp, op, sc, rows=rows)
        got = gen.bits_to_f64_numpy(np.ascontiguousarray(E_all[int(beta)][ms]), dtype)
        worst = max(worst, oracle.row_max_error(got, ref))
        nrows += len(ms)
    tol = 1e-5 if dtype == "f32" else 2e-2
    return {"slices": [int(x) for x in slices], "rows": nrows, "max_row_err": worst, "tol": tol, "ok": worst <= tol}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on rank 0 only."""
    if rank != 0:
        return
    name = args.config
    dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps = cfg_numbers(name)
    import mbci_inputs as gen
    import oracle
    cores = oracle.max_threads()
    nsl = max(1, min(b, cores))           # bounded sample per step
    per_slice = (M * K + K * N + N * L + M * L) * s
    inp = gen.make_chain_inputs(0, dtype, nsl, M, N, K, L, 1 if op == "softmax" else 0)
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    for _ in range(args.warmup):
        oracle.chain(inp, op, sc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.chain(inp, op, sc)
    el = time.perf_counter() - t0
    ms = el / args.steps * 1e3
    gbs = nsl * per_slice / (el / args.steps) / 1e9
    sample = f"{nsl} of {b} batch x head slices of {name} per step (fp64 unfused chain)"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "name": name, "batch_heads": b, "M": M, "N": N, "K": K, "L": L, "op": op,
                   "sample_batch_heads_per_step": nsl, "parallelism": "host cores (OpenMP)"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- CUDA path
_ORIG_AFFINITY = None


def pin_to_gpu_cpus(local_rank):
    """Bind this process to the CPU cores NVML reports as local to its GPU, so the pinned host
    buffers of the e2e leg are first-touched on the GPU's NUMA node (a remote node measured 12 vs
    54 GB/s H2D on one box).  Returns the core count, or None when NVML is unavailable."""
    try:
        import pynvml
        global _ORIG_AFFINITY
        _ORIG_AFFINITY = os.sched_getaffinity(0)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local_rank)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        return None
    return None


def run_cuda(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import mbci_inputs as gen
    from paper_2506_22169_b200 import mbci, sharding

    name = args.config
    dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps = cfg_numbers(name)
    numa = pin_to_gpu_cpus(local_rank)   # before any host allocation: pinned buffers land GPU-local
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dtype]
    b_layout = 1 if op == "softmax" else 0
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    sig = (1.0, 1.0, 1.0) if op == "softmax" else (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N))

    # this rank's shard: strong scaling splits the config's batch, weak scaling keeps b per rank
    global_b = b if args.scaling == "strong" else b * world
    lo, hi = sharding.shard_range(global_b, rank, world)
    counts = [sharding.shard_range(global_b, r, world)[1] - sharding.shard_range(global_b, r, world)[0]
              for r in range(world)]
    nb = hi - lo
    inp = gen.make_chain_inputs(args.seed, dtype, nb, M, N, K, L, b_layout, sigmas=sig, batch_start=lo)

    def to_t(bits):
        x = torch.from_numpy(bits.view(np.int32 if dtype == "f32" else np.int16))
        return x.view(tdt)

    hA, hB, hD = to_t(inp.A), to_t(inp.B), to_t(inp.D)
    step_bytes = nb * (M * K + K * N + N * L + M * L) * s
    rot = max(2, math.ceil(2 * L2_BYTES / step_bytes) + 1)
    rot = min(rot, max(2, int(0.5 * torch.cuda.mem_get_info(dev)[0] // max(step_bytes, 1))))
    sets = []
    for r in range(rot):
        A, B, D = hA.to(dev), hB.to(dev), hD.to(dev)
        E = torch.empty(nb, M, L, dtype=tdt, device=dev)
        sets.append((A, B, D, E))
    forced = None
    if args.plan:
        forced = mbci.mbci_plan_t()
        forced.kernel = 0
        parts = [int(x) for x in args.plan.split(":")]
        if len(parts) == 3:
            parts = [0] + parts
        forced.kernel, forced.BN, forced.TL, forced.stages = parts
    ch = mbci.Chain(nb, M, N, K, L, dtype, op, sc, b_layout=b_layout, device=local_rank, tune=args.tune,
                    plan=forced)
    plan = ch.plan()
    launches = ch.launches_per_run()
    stream = torch.cuda.Stream(dev)

    def step(i):
        A, B, D, E = sets[i % rot]
        ch.run_ptr(A.data_ptr(), B.data_ptr(), D.data_ptr(), E.data_ptr(), 0, stream.cuda_stream)

    # warm-up (eager), then capture exactly K steps in one graph
    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    stream.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(args.steps):
            step(i)
    # sustained pre-run (not timed) so the clock sampler sees the kernel under load
    sampler = ClockSampler(_gpu_id(local_rank))
    sampler.start()
    time.sleep(0.3)
    t_load0 = time.time()
    pre_t0 = time.perf_counter()
    while time.perf_counter() - pre_t0 < args.sustain:
        with torch.cuda.stream(stream):
            g.replay()
        stream.synchronize()
    # the timed region: the K-step graph replayed `repeats` times, each bracketed by CUDA events on
    # the launch stream (barrier + synchronize on both sides); value = the median replay, max over ranks
    reps_ms = []
    for _ in range(max(1, args.repeats)):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            g.replay()
        ev1.record(stream)
        ev1.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reps_ms.append(sharding.max_over_ranks(ev0.elapsed_time(ev1)))
    t_load1 = time.time()
    time.sleep(0.25)
    sampler.stop()
    ms = statistics.median(reps_ms)
    ms_per_step = ms / args.steps
    total_bytes = sharding.sum_over_ranks(step_bytes)
    gbs = total_bytes / (ms_per_step * 1e-3) / 1e9
    clocks = sampler.summary(t_load0, t_load1)

    # ---- e2e through the public host entry point (pinned host buffers)
    pA, pB, pD = hA.pin_memory(), hB.pin_memory(), hD.pin_memory()
    pE = torch.empty(nb, M, L, dtype=tdt).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    for _ in range(2):
        ch.run_host(pA, pB, pD, pE, stream=stream)
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        ch.run_host(pA, pB, pD, pE, stream=stream)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = sharding.max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    h2d = (hA.numel() + hB.numel() + hD.numel()) * s
    d2h = pE.numel() * s
    e2e_gbs = total_bytes / (e2e_ms * 1e-3) / 1e9

    # ---- after timing: gather E of every shard to rank 0 (NCCL), checked in the cpu_baseline leg
    A0, B0, D0, E0 = sets[0]
    with torch.cuda.stream(stream):
        ch.run_ptr(A0.data_ptr(), B0.data_ptr(), D0.data_ptr(), E0.data_ptr(), 0, stream.cuda_stream)
    stream.synchronize()
    E_bits = E0.view(torch.int32 if dtype == "f32" else torch.int16)
    E_all = sharding.gather_shards(E_bits, counts) if world > 1 else E_bits
    E_all = E_all.cpu().numpy().view(np.uint32 if dtype == "f32" else np.uint16) if rank == 0 else None

    if rank != 0:
        return
    pk = peaks()
    tflops = world * nb / b * flops / (ms_per_step * 1e-3) / 1e12 if b else 0.0
    frac = gbs / (pk["hbm_gbs"] * world)
    traffic = _traffic(name, world)
    roofline = {"bound": "hbm", "achieved": gbs / world, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": frac, "traffic": traffic, "peak_src": pk["src"],
                "kernel": {0: "k_chain_tc", 1: "k_chain_simt", 4: "k_chain_tc4", 5: "k_chain_tc5"}.get(plan.kernel, "?"),
                "per_launch_bytes": step_bytes, "per_launch_us": ms_per_step * 1e3,
                "tensor_tflops": tflops / world, "tensor_frac": tflops / world / pk["bf16_tflops"],
                "ex2_per_s": (exps * nb / b) / (ms_per_step * 1e-3) if exps else 0.0}
    gcheck = None
    if _ORIG_AFFINITY:   # the oracle legs use every host core again
        os.sched_setaffinity(0, _ORIG_AFFINITY)
    if not args.no_cpu_baseline:
        # one slice from each end of every rank's shard, at most 16 in all
        sl = sorted({x for r in range(world) for x in (sharding.shard_range(global_b, r, world)[0],
                                                         sharding.shard_range(global_b, r, world)[1] - 1)})
        sl = sl[:: max(1, len(sl) // 16)][:16]
        gcheck = gather_check(name, args.seed, E_all, sl)
    if not args.no_cpu_baseline and world == 1:
        cgbs, sample, cores, _ = time_oracle(name, args.cpu_seconds)
        cpu = {"value": cgbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample}
    else:
        cpu = None
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "us_per_chain": ms_per_step * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "mbci_env": {k: v for k, v in sorted(os.environ.items()) if k.startswith("MBCI_")},
        "config": {"workload": desc, "name": name, "batch_heads_per_gpu": nb, "global_batch_heads": global_b,
                   "M": M, "N": N, "K": K, "L": L, "op": op, "scale": sc, "b_layout": b_layout,
                   "l2": f"{rot} rotating input sets ({rot * step_bytes / 2**20:.0f} MiB) > 2x L2 between reuses",
                   "timing": f"K steps in one CUDA graph, CUDA events on the launch stream, max over ranks, "
                             f"median of {len(reps_ms)} replays",
                   "replay_us_per_step": [round(x / args.steps * 1e3, 3) for x in reps_ms],
                   "parallelism": f"dp{world} (batch x head sharding, no data-path collective)",
                   "plan": ch.describe(), "env": {k: v for k, v in os.environ.items() if k.startswith("MBCI_")}},
        "hbm_frac_of_8TBps": gbs / (8000.0 * world),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_gbs, "unit": "GB/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "api": "mbci_chain_run_host", "gpu_local_cpus": numa},
        "gpu_launches": launches * args.steps, "timed_replays": len(reps_ms),
        "clocks": clocks,
        "gather_check": gcheck,
    }
    print(json.dumps(line), flush=True)
    ch.close()


def run_split(args, rank, world, local_rank):
    """--split-n P: the key axis cut into P ranges.  world > 1: ranks form
    world / P groups of P consecutive ranks; a group shares a β range (strong / weak as usual), each
    rank runs mbci_chain_run_partial on its key range (B, D strided views at the range's first key),
    the group all-gathers the partial E and row log-sum-exp over NCCL and mbci_merge_partials reduces
    them — the path's one exchange step, inside the timed region (eager launches: the NCCL calls are
    not graph-captured).  world == 1: the P partial launches run back to back on one GPU, then the
    merge (graph-captured) — the cost of split-N against the single fused launch."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import mbci_inputs as gen
    from paper_2506_22169_b200 import mbci, sharding

    P = args.split_n
    if world > 1 and world % P:
        raise SystemExit("--split-n must divide the number of ranks")
    name = args.config
    dtype, b, M, N, K, L, op, desc, s, bytes_, flops, exps = cfg_numbers(name)
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    tdt = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}[dtype]
    b_layout = 1 if op == "softmax" else 0
    sc = 1.0 / math.sqrt(K) if op == "softmax" else 1.0
    sig = (1.0, 1.0, 1.0) if op == "softmax" else (1.0, 1.0 / math.sqrt(K), 1.0 / math.sqrt(N))
    groups = world // P if world > 1 else 1
    grp, part = sharding.split_grid(rank, world, P) if world > 1 else (0, None)
    global_b = b if args.scaling == "strong" else b * groups
    lo, hi = sharding.shard_range(global_b, grp, groups)
    nb = hi - lo
    inp = gen.make_chain_inputs(args.seed, dtype, nb, M, N, K, L, b_layout, sigmas=sig, batch_start=lo)
    mine = [part] if world > 1 else list(range(P))
    spans = [sharding.key_range(N, p, P) for p in range(P)]

    def to_t(bits):
        return torch.from_numpy(bits.view(np.int32 if dtype == "f32" else np.int16)).view(tdt)
    hA, hB, hD = to_t(inp.A), to_t(inp.B), to_t(inp.D)
    step_bytes = nb * (M * K + K * N + N * L + M * L) * s // (P if world > 1 else 1)
    rot = max(2, math.ceil(2 * L2_BYTES / max(1, nb * (M * K + K * N + N * L + M * L) * s)) + 1)
    sets = [(hA.to(dev), hB.to(dev), hD.to(dev)) for _ in range(rot)]
    strides = ({"ld_b": K, "bs_b": N * K} if b_layout == 1 else {"ld_b": N, "bs_b": K * N})
    strides.update(ld_d=L, bs_d=N * L)
    chs = [mbci.Chain(nb, M, spans[p][1] - spans[p][0], K, L, dtype, op, sc, b_layout=b_layout, device=local_rank,
                      strides=strides) for p in mine]
    E_parts = torch.empty(len(mine), nb, M, L, dtype=tdt, device=dev)
    lse = torch.empty(len(mine), nb, M, dtype=torch.float32, device=dev)
    E = torch.empty(nb, M, L, dtype=tdt, device=dev)
    sub = None
    if world > 1:
        for ranks in sharding.key_groups(world, P):   # every rank creates every group, same order
            gh = dist.new_group(ranks)
            if rank in ranks:
                sub = gh
    stream = torch.cuda.Stream(dev)

    def step(i):
        A, B, D = sets[i % rot]
        for j, p in enumerate(mine):
            n0, n1 = spans[p]
            Bv = B[:, n0:n1, :] if b_layout == 1 else B[:, :, n0:n1]
            chs[j].run_partial(A, Bv, D[:, n0:n1, :], E_parts[j], lse[j] if op == "softmax" else None, None, n0,
                               stream=stream)
        if world > 1:
            Ea, la = sharding.gather_partials(E_parts[0], lse[0] if op == "softmax" else None, group=sub)
        else:
            Ea, la = E_parts, (lse if op == "softmax" else None)
        mbci.merge_partials(Ea, la, E, op, stream=stream)

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            step(i)
    stream.synchronize()
    graph = None
    if world == 1:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(args.steps):
                step(i)
    sampler = ClockSampler(_gpu_id(local_rank))
    sampler.start()
    time.sleep(0.3)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_load0 = time.time()
    ev0.record(stream)
    with torch.cuda.stream(stream):
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(i)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_load1 = time.time()
    time.sleep(0.25)
    sampler.stop()
    ms_per_step = sharding.max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    total_bytes = sharding.sum_over_ranks(step_bytes)
    gbs = total_bytes / (ms_per_step * 1e-3) / 1e9
    # after timing: the merged rows of every β group against the oracle (rank 0)
    with torch.cuda.stream(stream):
        step(0)
    stream.synchronize()
    E_bits = E.view(torch.int32 if dtype == "f32" else torch.int16)
    if world > 1:
        counts = [sharding.shard_range(global_b, r // P, groups)[1] - sharding.shard_range(global_b, r // P, groups)[0]
                  for r in range(world)]
        allE = sharding.gather_shards(E_bits, counts)
        offs = np.cumsum([0] + counts)
        E_all = torch.cat([allE[offs[g * P]: offs[g * P] + counts[g * P]] for g in range(groups)]) if rank == 0 else None
    else:
        E_all = E_bits
    if rank != 0:
        return
    E_all = E_all.cpu().numpy().view(np.uint32 if dtype == "f32" else np.uint16)
    sl = sorted({0, global_b - 1} | {sharding.shard_range(global_b, g, groups)[0] for g in range(groups)})[:16]
    gcheck = gather_check(name, args.seed, E_all, sl) if not args.no_cpu_baseline else None
    clocks = sampler.summary(t_load0, t_load1)
    pk = peaks()
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "us_per_chain": ms_per_step * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "mbci_env": {k: v for k, v in sorted(os.environ.items()) if k.startswith("MBCI_")},
        "config": {"workload": desc, "name": name, "split_n": P, "beta_groups": groups, "global_batch_heads": global_b,
                   "batch_heads_per_group": nb, "key_ranges": spans, "M": M, "N": N, "K": K, "L": L, "op": op,
                   "parallelism": f"dp{groups} x split-N {P} (all-gather of partial E + lse, merge kernel)",
                   "timing": ("K steps in one CUDA graph" if world == 1 else "K eager steps (NCCL inside)")
                             + ", CUDA events on the launch stream, max over ranks",
                   "plans": [c.describe() for c in chs]},
        "roofline": {"bound": "hbm", "achieved": gbs / world, "peak": pk["hbm_gbs"], "unit": "GB/s",
                     "frac": gbs / world / pk["hbm_gbs"], "traffic": None, "peak_src": pk["src"]},
        "cpu_baseline": None, "e2e": None,
        "gpu_launches": (len(mine) + 1) * args.steps, "clocks": clocks, "gather_check": gcheck,
    }
    print(json.dumps(line), flush=True)
    for c in chs:
        c.close()


def _gpu_id(local_rank):
    try:
        import torch
        u = str(torch.cuda.get_device_properties(local_rank).uuid)
        return u if u.startswith("GPU-") else "GPU-" + u
    except Exception:
        return local_rank


def _traffic(name, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as f:
            j = json.load(f)
        v = j.get(name)
        return v.get("dram_bytes_per_launch") if isinstance(v, dict) else v
    except Exception:
        return None


def _free_port() -> int:
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    return port


def relaunch_cmd(argv, n_gpus, port):
    """`bench.py --gpus N` without WORLD_SIZE: the torch.distributed.run command that starts one
    rank per GPU on this node (rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def default_scaling(config: str) -> str:
    """C2 and C5 split the global batch over the ranks (strong scaling)."""
    return "strong" if config in ("C2", "C5") else "weak"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["cuda", "reference"], default="cuda")
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="strong: split the config's batch over the ranks; weak: full batch per rank")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--tune", type=int, default=0)
    ap.add_argument("--plan", default="", help="force a plan kernel:BN:TL:stages (tensor-core path)")
    ap.add_argument("--sustain", type=float, default=1.0, help="seconds of untimed load for the clock sampler")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--repeats", type=int, default=5, help="timed replays of the K-step graph (median reported)")
    ap.add_argument("--split-n", type=int, default=1,
                    help="cut the key axis into P ranges (SURVEY f1): groups of P ranks all-gather and merge")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.scaling is None:
        args.scaling = default_scaling(args.config)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(subprocess.call(relaunch_cmd(sys.argv[1:], args.gpus, _free_port())))
    if os.environ.get("MBCI_T4_DEBUG") or os.environ.get("MBCI_LIB") == "trace":
        print(json.dumps({"error": "MBCI_T4_DEBUG / MBCI_LIB=trace are diagnostics builds; bench refuses them"}))
        sys.exit(2)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        print(f"[bench] warning: --gpus {args.gpus} but WORLD_SIZE {world}; using {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        t = torch.ones(1, device="cuda")
        dist.all_reduce(t)   # creates the NCCL communicator now, not inside the timed region
        print(f"[bench] rank {rank}/{world} (local {local_rank}, {torch.cuda.get_device_name(local_rank)}): "
              f"NCCL communicator ready, nranks={int(t.item())}, nccl {'.'.join(map(str, torch.cuda.nccl.version()))}",
              file=sys.stderr, flush=True)
    try:
        if args.split_n > 1:
            return run_split(args, rank, world, local_rank)
        run_cuda(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
