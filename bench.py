"""Benchmark of the PDGraph scoring hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload is BASELINE config 2 ("100k queued apps, depth-8 PDGraphs,
256-bin demand histograms, full re-score on 1 B200"); under torchrun each rank
re-scores its own 100k-app shard (weak scaling) and the packed (key, arrival
position) pairs are all-gathered over NCCL for the global order (config 3's
exchange step).

A step = full re-score of the queue: K1b Gittins scorer over every resident
histogram row (+ overrun penalty + packed sort key) followed by the global
order (radix sort of the packed keys).  Synthetic data (seeded) -- there is
no dataset; histograms are multinomial draws of n=512 samples over 256
equal-width buckets, ages span the whole support (some rows exhausted).

Timing: W warm-up steps, then K timed steps; each step is bracketed by CUDA
events on the launching stream; L2 is flushed (256 MiB write) between steps,
outside the events.  The step time is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDGraph Gittins-index apps scored/sec at 1/2/4/8 B200; p50 scheduling latency"
UNIT = "apps/s"
N_APPS = 100_000
N_BINS = 256
N_SAMP = 512
PENALTY = 2.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--apps", type=int, default=N_APPS)
    ap.add_argument("--bins", type=int, default=N_BINS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling run: skip CUPTI launch counting, e2e and CPU legs")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# synthetic workload (host numpy; identical generator for both arms)
# ---------------------------------------------------------------------------

def make_rows(n, b, seed):
    rng = np.random.default_rng(seed)
    lo = rng.uniform(0.0, 600.0, n)
    w = rng.lognormal(-0.5, 1.0, n)
    est = rng.uniform(0.0, 300.0, n)
    # each row: a mixture of two bumps over the bucket grid, n=512 samples
    j = np.arange(b)
    c1 = rng.uniform(0, b, n)[:, None]
    c2 = rng.uniform(0, b, n)[:, None]
    s1 = rng.uniform(2, b / 4, n)[:, None]
    s2 = rng.uniform(2, b / 4, n)[:, None]
    mix = rng.uniform(0.2, 0.8, n)[:, None]
    pr = mix * np.exp(-0.5 * ((j - c1) / s1) ** 2) + (1 - mix) * np.exp(-0.5 * ((j - c2) / s2) ** 2)
    pr /= pr.sum(axis=1, keepdims=True)
    cdf = np.cumsum(pr, axis=1)
    cdf[:, -1] = 1.0
    off = np.arange(n, dtype=np.float64)[:, None]
    u = rng.random((n, N_SAMP))
    flat = np.searchsorted((cdf + off).ravel(), (u + off).ravel(), side="right")
    idx = np.minimum(flat.reshape(n, N_SAMP) - (np.arange(n) * b)[:, None], b - 1)
    counts = np.zeros((n, b), dtype=np.int64)
    np.add.at(counts, (np.repeat(np.arange(n), N_SAMP), idx.ravel()), 1)
    nb = np.full(n, b)
    age = est + rng.uniform(0.0, 1.05, n) * (b * w)
    return dict(lo=lo, width=w, est_age=est, nbins=nb, nsamp=np.full(n, N_SAMP),
                counts=counts, age=age)


def oracle_values(rows):
    b = rows["counts"].shape[1]
    j = np.arange(b, dtype=np.float64)
    lo, w = rows["lo"][:, None], rows["width"][:, None]
    v = ((lo + j * w) + (lo + (j + 1.0) * w)) / 2.0 + rows["est_age"][:, None]
    return v, rows["counts"] / rows["nsamp"][:, None].astype(np.float64)


# ---------------------------------------------------------------------------
# CPU (oracle port) timing: used by the cpu_baseline object and --impl reference
# ---------------------------------------------------------------------------

def _cpu_chunk(args):
    rows, reps = args
    from oracle import pdg_oracle as O
    v, p = oracle_values(rows)
    t0 = time.perf_counter()
    for _ in range(reps):
        r = O.gittins_rank_batch(v, p, rows["age"])
        r = np.where(np.isnan(r), rows["age"] * PENALTY, r)
        np.lexsort((np.arange(len(r)), r))
    return (time.perf_counter() - t0) / reps


def cpu_rate(sample_rows, procs):
    """apps/s of the oracle port over `sample_rows`, sharded over `procs` processes."""
    n = len(sample_rows["lo"])
    if procs <= 1:
        return n / _cpu_chunk((sample_rows, 1))
    import multiprocessing as mp
    parts = np.array_split(np.arange(n), procs)
    chunks = [({k: v[p] for k, v in sample_rows.items()}, 1) for p in parts]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        t0 = time.perf_counter()
        pool.map(_cpu_chunk, chunks)
        dt = time.perf_counter() - t0
    return n / dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    sample = min(args.apps, 20_000)
    rows = make_rows(sample, args.bins, seed=1)
    for _ in range(max(args.warmup, 1)):
        cpu_rate(rows, procs)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_rate(rows, procs)
        times.append(time.perf_counter() - t0)
    ms = float(np.median(times)) * 1e3
    val = sample / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2: full Gittins re-score of a 256-bucket queue",
                   "apps": args.apps, "bins": args.bins, "samples_per_hist": N_SAMP},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{sample} apps per step (of {args.apps}), numpy "
                                   f"gittins_rank_batch + penalty + lexsort, {procs} procs"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(kernel):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d[kernel]["dram_bytes_per_launch"], d[kernel].get("apps_per_launch")
    except (OSError, KeyError, ValueError):
        return None, None


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2506_14851_b200 import _lib
    from paper_2506_14851_b200.queue import HistQueue

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    L = _lib.lib()
    n, b = args.apps, args.bins

    rows = make_rows(n, b, seed=1000 + rank)
    q = HistQueue(n, b)
    gtb = (rank * n + np.arange(n)).astype(np.int64)          # global arrival position
    q.load_rows(rows["lo"], rows["width"], rows["est_age"], rows["nbins"], rows["nsamp"],
                rows["counts"], age=rows["age"], tiebreak=gtb)
    stream = torch.cuda.current_stream()
    gathered = torch.empty(world * n, dtype=torch.int64, device=dev)
    gslots = torch.arange(world * n, dtype=torch.int32, device=dev)
    out_keys = torch.empty_like(gathered)
    out_slots = torch.empty_like(gslots)
    tb = int(L.pdg_order_temp_bytes(world * n))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    k1_ev = []

    def step(record_k1=False):
        if record_k1:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        q.score(PENALTY)
        if record_k1:
            e1.record(stream)
            k1_ev.append((e0, e1))
        if world > 1:
            dist.all_gather_into_tensor(gathered, q.keys[:n])
            src = gathered
        else:
            src = q.keys[:n]
        _lib.check(L.pdg_order(_lib.ptr(src), _lib.ptr(out_keys), _lib.ptr(gslots),
                               _lib.ptr(out_slots), world * n, 32, _lib.ptr(temp),
                               temp.numel(), _lib.stream_ptr(stream)), "pdg_order")

    # kernels per step (CUPTI count of one step, outside the timed region)
    launches = None if args.ncu else count_launches(step)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    # keep the GPU busy ~0.4 s before the timed steps so nvidia-smi samples
    # the clocks under load; the timed steps run inside that sampled window
    t_end = time.perf_counter() + 0.4
    while time.perf_counter() < t_end:
        step()
        torch.cuda.synchronize()
    step_ev = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(record_k1=True)
        e1.record(stream)
        step_ev.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_end = time.perf_counter() + 0.3
    while time.perf_counter() < t_end:
        step()
        torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = np.array([a.elapsed_time(b_) for a, b_ in step_ev])
    k1_ms = np.array([a.elapsed_time(b_) for a, b_ in k1_ev])
    tot = torch.tensor([step_ms.sum(), np.median(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot[0].item()) / args.steps
    p50 = float(tot[1].item())
    value = world * n / (ms_per_step / 1e3)

    # e2e: through the public queue API with pinned HOST buffers -- each step
    # uploads that refresh's attained-service vector (the per-refresh input)
    # and reads back the global order and keys.
    if args.ncu:
        if rank == 0:
            print(json.dumps({"ncu_run": True, "ms_per_step": ms_per_step}), flush=True)
        return
    h_age = torch.from_numpy(rows["age"]).pin_memory()
    h_order = torch.empty(world * n, dtype=torch.int32).pin_memory()
    h_keys = torch.empty(n, dtype=torch.float32).pin_memory()
    for _ in range(2):
        q.age[:n].copy_(h_age, non_blocking=True)
        step()
        h_order.copy_(out_slots, non_blocking=True)
        h_keys.copy_(q.key_f32[:n], non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q.age[:n].copy_(h_age, non_blocking=True)
        step()
        h_order.copy_(out_slots, non_blocking=True)
        h_keys.copy_(q.key_f32[:n], non_blocking=True)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2t = torch.tensor([float(np.sum(e2e_ms)), float(np.median(e2e_ms))], dtype=torch.float64,
                       device=dev)
    if world > 1:
        dist.all_reduce(e2t, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(e2t[0].item()) / args.steps
    e2e = {"value": world * n / (e2e_ms_step / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(h_age.numel() * 8),
           "d2h_bytes_per_step": int(h_order.numel() * 4 + h_keys.numel() * 4),
           "ms_per_step": e2e_ms_step, "p50_latency_ms": float(e2t[1].item()),
           "path": "HistQueue.age <- pinned host; score+order; order/keys -> pinned host"}

    # roofline of the dominant kernel (K1b), algorithmic bytes per app
    bytes_per_app = 2 * b + 4 * 8 + 4 + 4 + 4 + 1 + 8
    k1_avg = float(k1_ms.mean())
    achieved = bytes_per_app * n / (k1_avg / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    traffic, _ = ncu_traffic("gittins_hist_kernel")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": "gittins_hist_kernel<1>",
                "bytes_per_app": bytes_per_app, "avg_launch_ms": k1_avg,
                "share_of_step": k1_avg / float(np.mean(step_ms)), "peak_source": peak_src}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "p50_latency_ms": p50, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64/f32/u16 (f64 support, f32 scan, u16 counts)",
        "data": "synthetic (seeded multinomial histograms, n=512 per app)",
        "config": {"workload": "config2: full Gittins re-score of a 100k-app 256-bucket queue + global order",
                   "apps_per_gpu": n, "bins": b, "samples_per_hist": N_SAMP,
                   "parallelism": f"shard-by-app x{world}, NCCL all_gather of 8 B keys",
                   "l2": "flushed between steps (256 MiB write, outside the step events)"},
        "gpu_launches": None if launches is None else launches * args.steps,
        "gpu_launches_per_step": launches,
        "e2e": e2e, "roofline": roofline, "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(n, 20_000)
        sub = {k: v[:sample] for k, v in rows.items()}
        rate = cpu_rate(sub, 1)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{sample} of {n} apps, oracle numpy "
                                          f"gittins_rank_batch + penalty + lexsort, 1 process"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def count_launches(step):
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    ours = [nm for nm in names if ("pdg" in nm or "gittins" in nm or "cub" in nm.lower()
                                   or "Radix" in nm)]
    return len(ours)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
