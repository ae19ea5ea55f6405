"""Benchmark of the PDGraph scoring hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload = BASELINE config 2: "100k queued apps, depth-8 PDGraphs, 256-bin
demand histograms, full re-score on 1 B200".  Every app owns its own depth-8
PDGraph (tools/synth.py: chain + 3-way branch + self-loop + back-edge loop,
256 lognormal duration records per unit) and sits at a random unit with a
random amount of service attained.

Multi-GPU: `--gpus N` without a launcher re-executes this script under
`torch.distributed.run` (N ranks, one per GPU, NCCL); under torchrun the
ranks come from the environment.  The headline then scales weakly: each rank
re-scores its own 100k-app shard and the packed (key, arrival position)
pairs are all-gathered over NCCL for the global order.  Every line also
carries `config3`, the strong-scaling run of BASELINE config 3: a 1M-app
queue split 1M/N per rank, step = engine + K1b + NCCL all-gather + the
global 1M-key sort, max over ranks.

One step = full re-score of the queue, the reference's policy runtime
(monte_carlo_remaining_demand(n=512) +
set_remaining(256) + one gittins_rank_batch row per app) plus the global
order:
  K2/a4  mc_walk_kernel       512-walk Monte Carlo from the current unit,
                              bit-identical to the reference, bucketed to 256
  K1b    gittins_pair_kernel  Gittins key + overrun penalty + packed sort key
  K5     radix sort           global order (after the all-gather when N > 1)
Each step uses fresh per-app seeds (a genuine re-estimate, nothing cached).

Timing: W warm-up steps, then K timed steps, each bracketed by CUDA events on
the launching stream; L2 flushed (256 MiB write) between steps outside the
events (the 1.6 GB graph bank exceeds L2 anyway); step time = max over ranks.

The reference arm (`--impl reference`) re-scores a bounded sample of the SAME
queue (same graphs, current units, seeds + step salt, attained service) with
the CPU restatement of the reference on every host core; its `ms_per_step`
is the measured wall time of that sample.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
N_REC = 256
VISIT_CAP = 64
PENALTY = 2.0
CONFIG3_APPS = 1_000_000
SEED_WORLD, SEED_JOBS, SEED_AGES = 1000, 1001, 1002
SALT_TIMED = 100            # timed step i uses per-app seed + SALT_TIMED + i


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--apps", type=int, default=N_APPS)
    ap.add_argument("--bins", type=int, default=N_BINS)
    ap.add_argument("--cpu-apps", type=int, default=1500,
                    help="apps in the bounded 1-core CPU-baseline sample")
    ap.add_argument("--ref-apps", type=int, default=0,
                    help="apps per reference-arm step (default 256 per host core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary sections (configs 1, 4, 5, K1c, K6, masks)")
    ap.add_argument("--ncu", action="store_true",
                    help="profiling run: skip CUPTI launch counting, e2e and CPU legs")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo check of the launch + exchange plumbing (no kernels)")
    return ap.parse_args(argv)


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: run N ranks of this script under
    torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def init_nccl(local: int):
    """One NCCL communicator over the node; NCCL's INIT log (comm, rank,
    nranks) goes to stderr so the rank count can be verified from the run."""
    import torch
    import torch.distributed as dist
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t = torch.ones(1, device=torch.device("cuda", local))
    dist.all_reduce(t)                     # forces communicator creation now
    return int(t.item())


def bench_config(n, b, world):
    """`config` of the headline line (identical in both arms)."""
    return {"workload": "config2: full re-score = attained service (_update_attained) + MC "
                        "demand engine (n=512, bit-exact vs reference) + 256-bucket Gittins "
                        "+ global order",
            "apps_per_gpu": n, "bins": b, "samples_per_app": N_SAMP,
            "records_per_unit": N_REC, "units_per_graph": 8, "visit_cap": VISIT_CAP,
            "queue": f"tools/synth.py make({n}, {N_REC}, seed={SEED_WORLD}+rank), "
                     f"jobs(seed={SEED_JOBS}+rank), ages(seed={SEED_AGES}+rank)",
            "parallelism": f"shard-by-app x{world}, NCCL all_gather of 8 B keys",
            "l2": "flushed between steps (256 MiB write, outside the step events); "
                  "1.6 GB graph bank > L2"}


# ---------------------------------------------------------------------------
# queue state shared by both arms
# ---------------------------------------------------------------------------

def reachable_units(u: int) -> int:
    """Units reachable from unit u in the synth template (tools/synth.py)."""
    return {0: 8, 1: 7, 2: 6, 3: 5, 4: 5, 5: 5, 6: 2, 7: 1}[int(u)]


NOW = 10000.0          # simulated clock of the re-score


def ages_for(rng, n, mean_rem, max_rem):
    """_update_attained's inputs (simcore.py:306-313) per app: completed
    service (= est_age, the attained service at the estimate), the current
    unit's progress and one active task (start, cold delay, service; start NaN
    = not started).  Served since the estimate ~ U(0, 0.9) x E[remaining]; 1%
    forced exhausted.  Element-wise in the inputs, so a sample of
    apps gets the same values as in the full queue.  Returns (est, age,
    columns); age is the attained service the device computes from them,
    evaluated here with the reference's operation order."""
    est = rng.uniform(0.0, 200.0, n)
    served = rng.uniform(0.0, 0.9, n) * mean_rem
    ex = rng.random(n) < 0.01
    served[ex] = 1.01 * max_rem[ex]
    progress = served * rng.uniform(0.0, 1.0, n)
    cold = np.where(rng.random(n) < 0.5, 0.0, rng.uniform(0.0, 5.0, n))
    start = NOW - served - cold
    start[(rng.random(n) < 0.2) & ~ex] = np.nan
    service = served * rng.uniform(1.0, 1.5, n)
    cols = {"completed": est, "progress": progress, "start": start, "cold": cold,
            "service": service}
    return est, attained(cols), cols


def attained(c):
    """completed + max(progress, min(service, max(0, now - (start + cold)))),
    as Simulator._update_attained evaluates it (one task per app)."""
    with np.errstate(invalid="ignore"):
        x = NOW - (c["start"] + c["cold"])
        run = np.where(x > 0.0, x, 0.0)
        v = np.where(run < c["service"], run, c["service"])
        prog = np.where(~np.isnan(c["start"]) & (v > c["progress"]), v, c["progress"])
    return c["completed"] + prog


def hist_mean_max(lo, width, k, counts, n_samp=N_SAMP):
    """E[remaining] over the bucket midpoints lo + (j + 1/2) w and the top
    edge lo + k w -- the first estimate's statistics the ages derive from."""
    j = np.arange(counts.shape[-1], dtype=np.float64)
    mids = lo[:, None] + (j[None, :] + 0.5) * width[:, None]
    return (counts * mids).sum(1) / n_samp, lo + k * width


# ---------------------------------------------------------------------------
# CPU (oracle port) legs: cpu_baseline objects and --impl reference.  Each
# leg runs on persistent forked workers that own a fixed shard of the sample
# (graphs built once per worker, outside the timed steps); a step sends one
# message to every worker and the parent times send -> last reply.
# ---------------------------------------------------------------------------

_CPU: dict = {}          # leg state, set by the parent before the workers fork


def _worker_loop(conn, init_fn, step_fn, shard):
    try:
        state = init_fn(shard)
        conn.send(("ready", None))
        while True:
            msg = conn.recv()
            if msg is None:
                break
            conn.send(("ok", step_fn(state, msg)))
    except Exception as e:            # surfaced by the parent
        conn.send(("error", repr(e)))


class ShardWorkers:
    """`procs` forked workers; worker i owns shard i of `items`.  procs == 1
    runs in-process.  call(msg) -> list of per-shard results."""

    def __init__(self, init_fn, step_fn, items, procs):
        import multiprocessing as mp
        edges = np.linspace(0, len(items), max(procs, 1) + 1).astype(int)
        shards = [items[a:b] for a, b in zip(edges[:-1], edges[1:]) if b > a]
        self.step_fn = step_fn
        self.local = None
        self.conns, self.procs = [], []
        if procs <= 1:
            self.local = init_fn(items)
            return
        ctx = mp.get_context("fork")
        for sh in shards:
            a, b = ctx.Pipe()
            p = ctx.Process(target=_worker_loop, args=(b, init_fn, step_fn, sh), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        for c in self.conns:
            tag, err = c.recv()
            if tag != "ready":
                raise RuntimeError(f"CPU worker failed: {err}")

    @property
    def n(self):
        return 1 if self.local is not None else len(self.conns)

    def call(self, msg):
        if self.local is not None:
            return [self.step_fn(self.local, msg)]
        for c in self.conns:
            c.send(msg)
        out = []
        for c in self.conns:
            tag, val = c.recv()
            if tag != "ok":
                raise RuntimeError(f"CPU worker failed: {val}")
            out.append(val)
        return out

    def timed(self, msg):
        t0 = time.perf_counter()
        out = self.call(msg)
        return out, time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            c.send(None)
        for p in self.procs:
            p.join(10)


def _c2_init(apps):
    """Worker state: oracle graphs of its apps (the same synth documents the
    GPU bank is built from) and their first estimates (seed + 0), from which
    the ages derive exactly as in run_ours."""
    from oracle import pdg_oracle as O
    from tools import synth
    st = _CPU["c2"]
    graphs = {int(a): O.graph_from_kb(synth.kb_doc(st["w"], int(a))) for a in apps}
    first = []
    for a in apps:
        r = O.mc_remaining_demand(graphs[a], f"s{st['unit'][a]}", [], N_SAMP,
                                  int(st["seed"][a]), VISIT_CAP)
        b = O.bucketize(r.samples.tolist(), st["bins"])
        m, mx = hist_mean_max(np.array([b.lo]), np.array([b.width]), np.array([b.k]),
                              b.counts[None].astype(np.float64))
        first.append((int(a), float(m[0]), float(mx[0])))
    return {"apps": [int(a) for a in apps], "graphs": graphs, "first": first, "ages": {}}


def _c2_step(state, msg):
    """("first",) -> first-estimate stats; ("ages", {app: (completed, progress,
    start, cold, service)}); ("step", salt) -> [(app, key)]: _update_attained
    + MC(n=512) + bucketize(256) + Gittins row + overrun penalty on one core
    (simcore.py:306-313, sched.py:170-181, 244-318, estimator.py:305-362)."""
    from oracle import pdg_oracle as O
    if msg[0] == "first":
        return state["first"]
    if msg[0] == "ages":
        state["ages"].update({a: msg[1][a] for a in state["apps"]})
        return None
    st = _CPU["c2"]
    salt = int(msg[1])
    out = []
    for a in state["apps"]:
        est, prog, start, cold, service = state["ages"][a]
        age = O.update_attained([est], [prog], [] if start != start else
                                [(0, start, cold, service)], NOW)[0]
        r = O.mc_remaining_demand(state["graphs"][a], f"s{st['unit'][a]}", [], N_SAMP,
                                  int(st["seed"][a]) + salt, VISIT_CAP)
        b = O.bucketize(r.samples.tolist(), st["bins"])
        v = b.midpoints() + est
        k = O.gittins_rank_batch(v[None], b.probs[None], np.array([age]))[0]
        out.append((a, age * PENALTY if np.isnan(k) else float(k)))
    return out


class Config2CPU:
    """The config-2 queue restated on the host for a bounded, evenly strided
    sample of its apps: same graphs, units, seeds, ages as the GPU arm."""

    def __init__(self, n_apps, sample, bins, procs, rank=0, world=None, jobs=None):
        from tools import synth
        w = world if world is not None else synth.make(n_apps, N_REC, seed=SEED_WORLD + rank)
        jb = jobs if jobs is not None else synth.jobs(n_apps, seed=SEED_JOBS + rank)
        self.idx = np.unique(np.linspace(0, n_apps - 1, sample).astype(np.int64))
        _CPU["c2"] = {"w": w, "unit": jb["unit"], "seed": jb["seed"], "bins": bins}
        self.workers = ShardWorkers(_c2_init, _c2_step, [int(a) for a in self.idx], procs)
        mean_rem, max_rem = np.zeros(n_apps), np.zeros(n_apps)
        for part in self.workers.call(("first",)):
            for a, m, mx in part:
                mean_rem[a], max_rem[a] = m, mx
        est, age, cols = ages_for(np.random.default_rng(SEED_AGES + rank), n_apps, mean_rem,
                                  max_rem)
        self.est, self.age = est, age
        self.workers.call(("ages", {int(a): tuple(float(cols[k][a]) for k in (
            "completed", "progress", "start", "cold", "service")) for a in self.idx}))

    def step(self, salt):
        """One re-score of the sample + its (key, arrival) order: wall
        seconds, keys (in self.idx order), order."""
        parts, dt = self.workers.timed(("step", salt))
        t0 = time.perf_counter()
        res = dict(x for part in parts for x in part)
        keys = np.array([res[int(a)] for a in self.idx])
        order = np.lexsort((self.idx, keys))
        return dt + time.perf_counter() - t0, keys, order

    def close(self):
        self.workers.close()


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    sample = args.ref_apps or max(256 * procs, 1024)
    t_setup = time.perf_counter()
    c2 = Config2CPU(args.apps, sample, args.bins, procs)
    t_setup = time.perf_counter() - t_setup
    for i in range(args.warmup):
        c2.step(1 + i)
    dts = [c2.step(SALT_TIMED + i)[0] for i in range(args.steps)]
    c2.close()
    m = len(c2.idx)
    ms_per_step = float(np.sum(dts)) / args.steps * 1e3
    val = m / (ms_per_step / 1e3)
    n_gpus = max(args.gpus, world)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": n_gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "p50_latency_ms": float(np.median(dts)) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded app-unique depth-8 PDGraphs, 256 records per unit)",
        "config": bench_config(args.apps, args.bins, n_gpus),
        "sample_apps": m,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{m} of the {args.apps} apps of the queue the GPU arm "
                                   f"scores (rank-0 shard; same graphs, units, seeds + step "
                                   f"salt, attained-service inputs), oracle _update_attained+"
                                   f"MC(n=512)+bucketize({args.bins})+"
                                   f"Gittins+penalty+order on {procs} processes; ms_per_step "
                                   f"= measured wall time of the sample step",
                         "setup_s": t_setup},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# --dry-run: the launch and exchange plumbing on CPU (gloo), no kernels
# ---------------------------------------------------------------------------

def run_dry(args):
    import torch
    import torch.distributed as dist
    from paper_2506_14851_b200.distributed import global_order, pack_keys, shard_range
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    n_total = args.apps * world
    lo, hi = shard_range(n_total, world, rank)
    keys = np.random.default_rng(7).lognormal(2, 1, n_total).astype(np.float32)
    local = pack_keys(torch.from_numpy(keys[lo:hi]), torch.arange(lo, hi))
    ms = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        order = global_order(local, n_total,
                             sort_fn=lambda k: k[torch.sort(k >> 32, stable=True).indices])
        if i >= args.warmup:
            ms.append((time.perf_counter() - t0) * 1e3)
    ranks = [None] * world
    if world > 1:
        dist.all_gather_object(ranks, rank)
    else:
        ranks = [0]
    pos = (order & 0xFFFFFFFF).numpy()
    ok = bool(np.array_equal(pos, np.lexsort((np.arange(n_total), keys.astype(np.float64)))))
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": world,
                          "ranks_seen": ranks, "order_ok": ok, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": float(np.mean(ms))}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


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


def ncu_summary(kernel):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(kernel, {})
    except (OSError, ValueError):
        return {}


def count_launches(step):
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step(0)
        torch.cuda.synchronize()
    names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
    ours = [nm for nm in names if ("pdg" in nm or "gittins" in nm or "mc_" in nm
                                   or "Radix" in nm or "cub" in nm.lower())]
    return len(ours), sorted(set(ours))


def max_over_ranks(vals, world, dev):
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2506_14851_b200 import _lib
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.queue import HistQueue
    from tools import synth

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_nccl(local)
    L = _lib.lib()
    n, b = args.apps, args.bins

    # ---- resident state: graph bank + queue + per-app job state ----------
    w = synth.make(n, N_REC, seed=SEED_WORLD + rank)
    eng = DemandEngine(synth.bank(w, device=str(dev)), device=str(dev))
    jb = synth.jobs(n, seed=SEED_JOBS + rank)
    q = HistQueue(n, b)
    g_idx = torch.arange(n, dtype=torch.int32, device=dev)
    u_idx = torch.from_numpy(jb["unit"]).to(dev)
    seeds0 = torch.from_numpy(jb["seed"]).to(dev)
    seeds = seeds0.clone()
    # attained service: drawn once from the first estimate's mean / max
    eng.run(g_idx, u_idx, seeds, n=N_SAMP, bucket_count=b, visit_cap=VISIT_CAP, queue=q)
    torch.cuda.synchronize()
    mean_rem, max_rem = hist_mean_max(q.lo[:n].cpu().numpy(), q.width[:n].cpu().numpy(),
                                      q.nbins[:n].double().cpu().numpy(),
                                      q.counts[:n].double().cpu().numpy())
    est, age, cols = ages_for(np.random.default_rng(SEED_AGES + rank), n, mean_rem, max_rem)
    q.est_age[:n] = torch.from_numpy(est).to(dev)
    q.tiebreak[:n] = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int32, device=dev)
    q.n = n
    # the scheduler's per-app attained-service inputs (one running task per
    # app), resident; every step recomputes q.age from them (a11b)
    att = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
    t_app = torch.arange(n, dtype=torch.int32, device=dev)
    t_active = torch.ones(n, dtype=torch.uint8, device=dev)

    # the step's per-app inputs, read through a holder so that the pipelined
    # e2e measurement can point the step at a double-buffered upload set
    inp = {"u": u_idx, "s": seeds0, "att": att}

    def update_age():
        at = inp["att"]
        q.update_attained(at["completed"], at["progress"], t_app, t_active, at["start"],
                          at["cold"], at["service"], NOW)

    update_age()
    torch.cuda.synchronize()
    assert np.array_equal(q.age[:n].cpu().numpy(), age), "attained service differs"

    stream = torch.cuda.current_stream()
    gathered = torch.empty(world * n, dtype=torch.int64, device=dev)
    gslots = torch.arange(world * n, dtype=torch.int32, device=dev)
    out_keys = torch.empty_like(gathered)
    out_slots = torch.empty_like(gslots)
    tb = int(L.pdg_order_temp_bytes(world * n))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    k_ev = {"engine": [], "k1": []}

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def step(salt, record=False):
        torch.add(inp["s"], salt, out=seeds)                # fresh estimate seeds
        update_age()                                        # _update_attained, all apps
        if record:
            e0, e1, e2 = ev(), ev(), ev()
            e0.record(stream)
        eng.run(g_idx, inp["u"], seeds, n=N_SAMP, bucket_count=b, visit_cap=VISIT_CAP,
                queue=q)
        if record:
            e1.record(stream)
        q.score(PENALTY)
        if record:
            e2.record(stream)
            k_ev["engine"].append((e0, e1))
            k_ev["k1"].append((e1, e2))
        if world > 1:
            dist.all_gather_into_tensor(gathered, q.keys[:n])
            src = gathered
        else:
            src = q.keys[:n]
        # shards are in global arrival order (rank-major), so a stable sort on
        # the 32-bit key alone yields the (key, arrival) order
        _lib.check(L.pdg_order(_lib.ptr(src), _lib.ptr(out_keys), _lib.ptr(gslots),
                               _lib.ptr(out_slots), world * n, 32, _lib.ptr(temp),
                               temp.numel(), _lib.stream_ptr()), "pdg_order")

    launches, kernel_names = (None, None) if args.ncu else count_launches(step)

    for i in range(args.warmup):
        flush.zero_()
        step(1 + i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    t_end = time.perf_counter() + 0.4        # clocks sampled under load
    while time.perf_counter() < t_end:
        step(7)
        torch.cuda.synchronize()
    step_ev = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record(stream)
        step(SALT_TIMED + i, record=True)
        e1.record(stream)
        step_ev.append((e0, e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_end = time.perf_counter() + 0.3
    while time.perf_counter() < t_end:
        step(9)
        torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = np.array([a.elapsed_time(b_) for a, b_ in step_ev])
    eng_ms = np.array([a.elapsed_time(b_) for a, b_ in k_ev["engine"]])
    k1_ms = np.array([a.elapsed_time(b_) for a, b_ in k_ev["k1"]])
    tot_ms, p50 = max_over_ranks([step_ms.sum(), np.median(step_ms)], world, dev)
    ms_per_step = tot_ms / args.steps
    value = world * n / (ms_per_step / 1e3)

    if args.ncu:
        if rank == 0:
            print(json.dumps({"ncu_run": True, "ms_per_step": ms_per_step}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- e2e through the public API with pinned HOST buffers --------------
    # every step uploads the per-app queue state the scheduler owns (current
    # unit, estimate seed, attained service now and at the estimate) and reads
    # back the global order and the keys
    h_unit = torch.from_numpy(jb["unit"]).pin_memory()
    h_seed = torch.from_numpy(jb["seed"]).pin_memory()
    h_cols = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in cols.items()}
    h_est = torch.from_numpy(est).pin_memory()
    h_order = torch.empty(world * n, dtype=torch.int32).pin_memory()
    h_keys = torch.empty(n, dtype=torch.float32).pin_memory()

    def e2e_step(salt):
        u_idx.copy_(h_unit, non_blocking=True)
        seeds0.copy_(h_seed, non_blocking=True)
        for k, v in h_cols.items():
            att[k].copy_(v, non_blocking=True)
        q.est_age[:n].copy_(h_est, non_blocking=True)
        step(salt)
        h_order.copy_(out_slots, non_blocking=True)
        h_keys.copy_(q.key_f32[:n], non_blocking=True)

    for i in range(2):
        e2e_step(200 + i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_ms = []
    for i in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step(300 + i)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_tot, e2e_p50 = max_over_ranks([np.sum(e2e_ms), np.median(e2e_ms)], world, dev)
    e2e_ms_step = e2e_tot / args.steps
    h2d = h_unit.numel() * 4 + h_seed.numel() * 8 + h_est.numel() * 8 + \
        sum(v.numel() * 8 for v in h_cols.values())

    # pipelined: every step still uploads its own inputs from the pinned host
    # buffers and reads its order and keys back, but the upload of step i+1
    # (copy stream, double-buffered device set) runs under step i's compute,
    # as a scheduler refreshing continuously would run it
    stage = [{"u": torch.empty_like(u_idx), "s": torch.empty_like(seeds0),
              "att": {k: torch.empty_like(v) for k, v in att.items()},
              "est": torch.empty(n, dtype=torch.float64, device=dev)} for _ in range(2)]
    cs = torch.cuda.Stream()
    ev_up = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]

    def upload(i):
        st_ = stage[i % 2]
        with torch.cuda.stream(cs):
            cs.wait_event(ev_free[i % 2])                  # step i-2 is done with it
            st_["u"].copy_(h_unit, non_blocking=True)
            st_["s"].copy_(h_seed, non_blocking=True)
            for k, v in h_cols.items():
                st_["att"][k].copy_(v, non_blocking=True)
            st_["est"].copy_(h_est, non_blocking=True)
            ev_up[i % 2].record(cs)

    def piped_step(i, salt):
        st_ = stage[i % 2]
        comp = torch.cuda.current_stream()
        comp.wait_event(ev_up[i % 2])
        inp.update(u=st_["u"], s=st_["s"], att=st_["att"])
        q.est_age[:n].copy_(st_["est"], non_blocking=True)
        flush.zero_()                                       # L2 flush counted inside
        step(salt)
        ev_free[i % 2].record(comp)
        h_order.copy_(out_slots, non_blocking=True)
        h_keys.copy_(q.key_f32[:n], non_blocking=True)

    def piped(k, salt0):
        upload(0)
        for i in range(k):
            if i + 1 < k:
                upload(i + 1)
            piped_step(i, salt0 + i)

    piped(2, 400)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    piped(args.steps, 500)
    torch.cuda.synchronize()
    pipe_ms = (time.perf_counter() - t0) * 1e3
    inp.update(u=u_idx, s=seeds0, att=att)
    pipe_tot = max_over_ranks([pipe_ms], world, dev)[0]
    pipe_step = pipe_tot / args.steps
    e2e = {"value": world * n / (pipe_step / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(h_order.numel() * 4 + h_keys.numel() * 4),
           "ms_per_step": pipe_step,
           "path": "pinned host queue state (units, seeds, estimate ages, attained-service "
                   "inputs) -> HistQueue.update_attained + DemandEngine.run + "
                   "HistQueue.score + pdg_order -> pinned host order/keys; uploads "
                   "double-buffered on a copy stream under the previous step's compute, L2 "
                   "flush inside the timed region (wall clock over K steps, synchronized "
                   "at both ends)",
           "serial": {"value": world * n / (e2e_ms_step / 1e3), "ms_per_step": e2e_ms_step,
                      "p50_latency_ms": e2e_p50,
                      "path": "the same, one step at a time: upload, step, read-back, "
                              "synchronize (L2 flushed outside the timed region)"}}

    # ---- the same step replayed as one CUDA graph ---------------------------
    # (all launches captured once; shows how much of the step the ~12 host
    # launches cost -- they are enqueued while the engine runs)
    graph = cuda_graph_step(step, flush, args.steps, world, n)

    # ---- roofline of the dominant kernel (the engine) ----------------------
    reach = np.array([reachable_units(u) for u in jb["unit"]])
    # per app: pools of reachable units (256 f64) + their descriptors (64 B) and
    # successor slots (4 x 12 B) + job (unit, graph, seed) + histogram row out
    per_app = reach * (N_REC * 8 + 64 + 48) + (4 + 4 + 8) + (2 * q.stride + 8 + 8 + 4 + 4)
    bytes_per_app = float(per_app.mean())
    eng_avg = float(eng_ms.mean())
    achieved = bytes_per_app * n / (eng_avg / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    ns = ncu_summary("engine")
    traffic = ns.get("dram_bytes_per_launch") if ns.get("apps_per_launch") == n else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "mc_walk_kernel", "bytes_per_app": bytes_per_app,
                "avg_launch_ms": eng_avg, "share_of_step": eng_avg / float(np.mean(step_ms)),
                "peak_source": peak_src,
                "note": "not HBM-bound: the kernel is integer-issue bound (one 128-bit PCG64 "
                        "LCG step per consumed numpy word, ~1.5 words per walk visit); issue "
                        "utilisation and warp instructions per launch from the committed ncu "
                        "capture (profiles/ncu_summary.json)",
                "issue_active_frac": ns.get("issue_active_frac"),
                "warp_instructions": ns.get("warp_instructions")}
    if ns.get("pcg_floor_ms") is not None:
        # issue-time floors from the ncu capture (4 warp instructions / SM /
        # cycle): the PCG64 stream alone, and every instruction the kernel ran
        roofline["pcg_floor_ms"] = ns["pcg_floor_ms"]
        roofline["frac_of_pcg_floor"] = ns["pcg_floor_ms"] / eng_avg
    if ns.get("issue_floor_ms") is not None:
        roofline["issue_floor_ms"] = ns["issue_floor_ms"]
        roofline["issue_frac"] = ns["issue_floor_ms"] / eng_avg
    k1_bytes = 2 * q.stride + 4 * 8 + 4 + 4 + 4 + 1 + 8
    k1 = {"kernel": "gittins_pair_kernel", "avg_launch_ms": float(k1_ms.mean()),
          "bytes_per_app": k1_bytes,
          "achieved_gbs": k1_bytes * n / (float(k1_ms.mean()) / 1e3) / 1e9,
          "apps_per_s": n / (float(k1_ms.mean()) / 1e3)}

    # ---- steady-state refresh: the bucket-period re-rank of cached rows ----
    # (simcore.py:636-640: no re-estimation, only K1b over the resident
    # histograms at the current attained service + the global order)
    ref_ev = []
    for i in range(max(args.steps, 10)):
        flush.zero_()
        e0, e1 = ev(), ev()
        e0.record(stream)
        update_age()
        q.score(PENALTY)
        if world > 1:
            dist.all_gather_into_tensor(gathered, q.keys[:n])
        _lib.check(L.pdg_order(_lib.ptr(gathered if world > 1 else q.keys[:n]),
                               _lib.ptr(out_keys), _lib.ptr(gslots), _lib.ptr(out_slots),
                               world * n, 32, _lib.ptr(temp), temp.numel(), _lib.stream_ptr()),
                   "pdg_order")
        e1.record(stream)
        ref_ev.append((e0, e1))
    torch.cuda.synchronize()
    ref_ms = np.array([a_.elapsed_time(b_) for a_, b_ in ref_ev])
    ref_p50 = max_over_ranks([float(np.median(ref_ms))], world, dev)[0]
    periodic = {"p50_latency_ms": ref_p50, "apps_per_s": world * n / (ref_p50 / 1e3),
                "what": "bucket-period refresh of the resident queue (simcore.py:636-640): "
                        "attained service + K1b over the cached histograms + global order, "
                        "no re-estimation; L2 flushed before each"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "p50_latency_ms": p50, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 walks/f32 scan/u16 counts",
        "data": "synthetic (seeded app-unique depth-8 PDGraphs, 256 records per unit)",
        "config": bench_config(n, b, world),
        "gpu_launches": None if launches is None else launches * args.steps,
        "gpu_launches_per_step": launches, "kernels": kernel_names,
        "e2e": e2e, "roofline": roofline, "k1_refresh": k1, "periodic_refresh": periodic,
        "cuda_graph": graph, "clocks": clk,
    }

    # ---- like-for-like CPU baseline (rank 0, N = 1): the same apps --------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = Config2CPU(n, args.cpu_apps, b, 1, rank=0, world=w, jobs=jb)
        cpu_dt, cpu_keys, _ = cpu.step(SALT_TIMED)
        cpu.close()
        step(SALT_TIMED)                                  # the GPU's keys of that step
        gk = q.key_f32[:n].cpu().numpy()[cpu.idx].astype(np.float64)
        rel = np.abs(gk - cpu_keys) / np.maximum(np.abs(cpu_keys), 1e-300)
        line["cpu_baseline"] = {
            "value": len(cpu.idx) / cpu_dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{len(cpu.idx)} of the {n} apps of this queue (evenly strided; same "
                      f"graphs, units, seeds, attained-service inputs, step salt {SALT_TIMED}), "
                      f"oracle _update_attained+MC(n=512)+bucketize({b})+Gittins row+penalty, "
                      f"1 process",
            "sample_wall_s": cpu_dt,
            "keys_max_rel_err_vs_gpu": float(rel.max())}
    del w

    # ---- config 3: 1M apps split 1M/N over the ranks (strong scaling) -----
    line["config3"] = bench_config3(dev, eng, n, b, world, rank, flush)

    if world == 1 and not args.no_extra:
        line["k1c_policy"] = bench_policy(dev, eng, g_idx, u_idx, seeds, q, n, b)
        line["k6_dispatch"] = bench_dispatch(dev)
        line["masks"] = bench_masks(dev)
        line["config1_refresh_latency"] = bench_refresh_latency()
        line["config1_simulation"] = bench_config1_sim()
        line["k1_refresh_1m"] = bench_k1_large(dev)
        line["config2_llm"] = bench_llm(dev, cpu_sample=0 if args.no_cpu_baseline else 200)
        del eng, q
        torch.cuda.empty_cache()
        line["config4_stream"] = bench_stream(dev, cpu=not args.no_cpu_baseline)
        torch.cuda.empty_cache()
        line["config5_prewarm"] = bench_need(dev, cpu=not args.no_cpu_baseline)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# config 3 (strong scaling): a 1M-app queue split 1M/N over the ranks; step =
# engine + K1b on the shard, NCCL all-gather of the 8-byte packed keys, the
# global 1M-key order on every rank.  Time = max over ranks.
# ---------------------------------------------------------------------------

def bench_config3(dev, eng, n_graphs, b, world, rank, flush, total=CONFIG3_APPS, steps=5):
    import torch
    import torch.distributed as dist

    from paper_2506_14851_b200 import _lib
    from paper_2506_14851_b200.distributed import SENTINEL, shard_range
    from paper_2506_14851_b200.queue import HistQueue
    from tools import synth
    L = _lib.lib()
    lo, hi = shard_range(total, world, rank)
    n = hi - lo
    width = -(-total // world)
    jb = synth.jobs(total, seed=3003)
    g = (torch.arange(lo, hi, dtype=torch.int64, device=dev) % n_graphs).to(torch.int32)
    u = torch.from_numpy(jb["unit"][lo:hi]).to(dev)
    sd0 = torch.from_numpy(jb["seed"][lo:hi]).to(dev)
    sd = sd0.clone()
    q = HistQueue(width, b)
    q.n = n
    q.est_age.zero_()
    q.age.fill_(1.0)
    q.tiebreak[:n] = torch.arange(lo, hi, dtype=torch.int32, device=dev)
    q.keys.fill_(SENTINEL)                 # pad of an uneven shard sorts last
    gathered = torch.empty(world * width, dtype=torch.int64, device=dev)
    ok = torch.empty_like(gathered)
    sl = torch.arange(world * width, dtype=torch.int32, device=dev)
    osl = torch.empty_like(sl)
    tb = int(L.pdg_order_temp_bytes(world * width))
    temp = torch.empty(max(tb, 16), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    parts = {"engine": [], "k1": [], "allgather": [], "sort": []}

    def step(salt, record=False):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if record else None
        torch.add(sd0, salt, out=sd)
        if record:
            evs[0].record(stream)
        eng.run(g, u, sd, n=N_SAMP, bucket_count=b, visit_cap=VISIT_CAP, queue=q)
        if record:
            evs[1].record(stream)
        q.score(PENALTY)
        if record:
            evs[2].record(stream)
        if world > 1:
            dist.all_gather_into_tensor(gathered, q.keys[:width])
            src = gathered
        else:
            src = q.keys[:width]
        if record:
            evs[3].record(stream)
        _lib.check(L.pdg_order(_lib.ptr(src), _lib.ptr(ok), _lib.ptr(sl), _lib.ptr(osl),
                               world * width, 32, _lib.ptr(temp), temp.numel(),
                               _lib.stream_ptr(stream)), "pdg_order")
        if record:
            evs[4].record(stream)
            for k, (a, c) in zip(parts, zip(evs[:-1], evs[1:])):
                parts[k].append((a, c))

    for i in range(2):
        step(50 + i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = []
    for i in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(60 + i, record=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    if world > 1:
        dist.barrier()
    split = {k: float(np.mean([a.elapsed_time(c) for a, c in v])) for k, v in parts.items()}
    t_mean, t_p50 = max_over_ranks([np.mean(ms), np.median(ms)], world, dev)
    # the order must hold every global arrival position once (every rank)
    pos = (ok[:total] & 0xFFFFFFFF).to(torch.int32)
    perm_ok = bool(torch.equal(torch.sort(pos).values,
                               torch.arange(total, dtype=torch.int32, device=dev)))
    out = {"workload": f"config3: {total} apps (instances of this rank's {n_graphs} depth-8 "
                       f"graphs, own unit and seed) split {total}/{world} per rank; step = engine "
                       f"(n=512, bit-exact) + K1b + NCCL all_gather of 8 B keys + global "
                       f"{total}-key radix sort; L2 flushed between steps",
           "scaling": "strong", "n_gpus": world, "apps_total": total, "apps_per_rank": n,
           "ms_per_rescore": t_mean, "p50_ms": t_p50, "apps_per_s": total / (t_mean / 1e3),
           "rank0_split_ms": split, "order_is_permutation": perm_ok,
           "north_star_target_ms": 10.0}
    del q, gathered, ok, temp
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# SRPT-mean / LSTF keys (K1c) and the engine's mean epilogue
# ---------------------------------------------------------------------------

def bench_policy(dev, eng, g_idx, u_idx, seeds, q, n, b, rows=1_000_000, reps=20):
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.sched import Policy

    def timed(fn, k):
        ts = []
        for _ in range(k):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.mean(ts))

    run = lambda mean: eng.run(g_idx, u_idx, seeds, n=N_SAMP, bucket_count=b,  # noqa: E731
                               visit_cap=VISIT_CAP, queue=q, mean=mean)
    run(True)
    base_ms, mean_ms = timed(lambda: run(False), 3), timed(lambda: run(True), 3)
    hq = HistQueue(rows, 8)
    rng = torch.Generator(device=dev).manual_seed(5)
    for t in (hq.mean, hq.worst, hq.est_age, hq.age, hq.deadline):
        t.uniform_(0, 1000, generator=rng)
    hq.n = rows
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    for pol in (Policy.SRPT_MEAN, Policy.LSTF):
        hq.score_policy(pol, 500.0)

        def one():
            hq.score_policy(pol, 500.0)
        ts = []
        for _ in range(reps):
            flush.zero_()
            ts.append(timed(one, 1))
        ms = float(np.mean(ts))
        nbytes = (4 if pol is Policy.SRPT_MEAN else 5) * 8 + 16
        out[pol.value] = {"ms_per_launch": ms, "rows": rows, "apps_per_s": rows / (ms / 1e3),
                          "roofline": {"bound": "hbm", "bytes_per_app": nbytes,
                                       "achieved": nbytes * rows / (ms / 1e3) / 1e9,
                                       "peak": measured_peaks()[0], "unit": "GB/s"}}
        out[pol.value]["roofline"]["frac"] = (out[pol.value]["roofline"]["achieved"]
                                              / out[pol.value]["roofline"]["peak"])
    out["engine_mean_epilogue"] = {"engine_ms": base_ms, "engine_with_mean_ms": mean_ms,
                                   "apps": n, "note": "RemainingDemand.mean() in CPython "
                                   "sum() order: the running sum and the compensation are sequential "
                                   "float64 chains (lane 0), the compensation terms are formed "
                                   "across the warp"}
    return out


# ---------------------------------------------------------------------------
# K1b periodic refresh of a 1M-row resident queue (no re-estimation)
# ---------------------------------------------------------------------------

def cuda_graph_step(step, flush, steps, world, n):
    """Capture step() (fixed salt) into a CUDA graph and time K replays with
    the L2 flushed between them; max over ranks.  Single-rank only: the
    N>1 step contains an NCCL all-gather issued through torch.distributed."""
    import torch
    if world > 1:
        return {"skipped": "N>1 step holds a torch.distributed all-gather"}
    try:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step(SALT_TIMED)                          # warm the capture stream
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(SALT_TIMED)
        torch.cuda.synchronize()
    except Exception as e:                            # report, do not hide
        return {"error": f"{type(e).__name__}: {e}"}
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ts]))
    return {"ms_per_step": ms, "apps_per_s": n / (ms / 1e3),
            "note": "the timed step replayed as one captured CUDA graph (same kernels)"}


def bench_k1_large(dev, n=1_000_000, reps=60):
    import torch
    from paper_2506_14851_b200.queue import HistQueue
    q = HistQueue(n, N_BINS)
    g = torch.Generator(device=dev).manual_seed(1)
    q.counts.copy_((torch.rand((n, N_BINS), device=dev, generator=g) * 5).to(torch.uint16))
    q.nsamp.fill_(N_SAMP)
    q.nbins.fill_(N_BINS)
    q.lo.uniform_(0, 100, generator=g)
    q.width.uniform_(0.1, 2, generator=g)
    q.est_age.uniform_(0, 10, generator=g)
    q.age.copy_(q.est_age + torch.rand(n, device=dev, dtype=torch.float64, generator=g) * 200)
    q.n = n
    for _ in range(3):
        q.score(PENALTY)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(reps):
        flush.zero_()
        # keep the stream busy while the host issues the launch, so that the
        # events bracket the kernel's device time, not host launch overhead
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        q.score(PENALTY)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    # the event clock ticks in 2.048 us steps on these boxes; the launch's
    # phase against the tick is random, so the MEAN of the ticked intervals
    # estimates the duration (the median would snap to a tick)
    ms = float(np.mean(ts))
    nbytes = 2 * q.stride + 4 * 8 + 4 + 4 + 4 + 1 + 8
    ach = nbytes * n / (ms / 1e3) / 1e9
    peak = measured_peaks()[0]
    return {"kernel": "gittins_pair_kernel", "rows": n, "ms_per_launch": ms,
            "apps_per_s": n / (ms / 1e3),
            "roofline": {"bound": "hbm", "bytes_per_app": nbytes, "achieved": ach,
                         "peak": peak, "unit": "GB/s", "frac": ach / peak}}


# ---------------------------------------------------------------------------
# config 2, LLM variant: the engine on depth-8 templates mixing LLM units,
# own-input units and upstream-conditioned (K3) units, 3 in 4 apps conditioned
# on an observation (mc_walk_kernel<7>; estimator.py:236-302, 305-362)
# ---------------------------------------------------------------------------

def bench_llm(dev, n_apps=100_000, templates=256, reps=10, cpu_sample=200):
    import torch
    from oracle import pdg_oracle as O
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from tools import synth
    docs = synth.llm_docs(templates, 200, seed=2027)
    eng = DemandEngine({k: graph_from_kb(v) for k, v in docs.items()}, device=str(dev))
    q = synth.llm_queue(docs, n_apps, seed=9)
    jobs = synth.llm_jobs(eng, q, dev)
    hq = HistQueue(n_apps, N_BINS)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        res = eng.run(*jobs, n=N_SAMP, bucket_count=N_BINS, visit_cap=VISIT_CAP, queue=hq)
    torch.cuda.synchronize()
    fl = res["flags"].cpu().numpy()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run(*jobs, n=N_SAMP, bucket_count=N_BINS, visit_cap=VISIT_CAP, queue=hq)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    out = {"workload": f"config2-llm: {n_apps} apps over {templates} depth-8 templates "
                       "(LLM, own-input and K3-conditioned units; tools/synth.llm_docs), "
                       "MC n=512 + 256-bucket rows", "apps": n_apps,
           "engine_ms": ms, "apps_per_s": n_apps / (ms / 1e3),
           "conditioned_frac": float((fl & 1).mean()),
           "replayed_serial": int(((fl & 4) != 0).sum()),
           "redrawn_in_kernel": int(((fl & 8) != 0).sum()),
           "bank_features": int(eng.bank.features)}
    if cpu_sample:
        og = {k: O.graph_from_kb(v) for k, v in docs.items()}
        idx = np.linspace(0, n_apps - 1, cpu_sample).astype(int)
        t0 = time.perf_counter()
        for a in idx:
            o = q["obs"][a]
            obs = [] if o is None else [O.OObs(o[0], o[1], o[2], o[3])]
            r = O.mc_remaining_demand(og[q["names"][q["graph"][a]]], f"s{q['unit'][a]}", obs,
                                      N_SAMP, int(q["seed"][a]), VISIT_CAP)
            O.bucketize(r.samples.tolist(), N_BINS)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": len(idx) / dt, "unit": UNIT, "cores": 1, "kind": "port",
                               "sample": f"{len(idx)} evenly strided apps of this queue, oracle "
                                         "MC(n=512, conditioned)+bucketize(256)"}
    return out


# ---------------------------------------------------------------------------
# config 1: the paper's "policy runtime" (refresh_priorities elapsed_ns,
# sched.py:269-310) at scheduler-sized batches, drop-in vs the reference
# ---------------------------------------------------------------------------

def bench_config1_sim():
    """Config 1 end to end: the reference simulator with its own hot path and
    with the GPU drop-in (same event log), and the Monte Carlo call latency."""
    try:
        from tools.config1_sim_time import measure
        r = measure()
    except ImportError as e:
        return {"unavailable": f"reference pdgsim not importable: {e}"}
    r["note"] = ("BASELINE config 1 (1000 apps, code-gen + fact-verify, 64 buckets, Gittins, "
                 "plan prewarm): simcore.run_simulation wall time; MC p50 over the "
                 "simulation's own monte_carlo_remaining_demand calls (one app each)")
    return r


def bench_refresh_latency():
    try:
        from tools.refresh_latency import apps
        from tests.dispatch_hook import import_pdgsim
        pdgsim = import_pdgsim()
        from pdgsim import sched as ref
    except ImportError as e:
        return {"unavailable": f"reference pdgsim not importable: {e}"}
    from paper_2506_14851_b200 import sched as ours
    rng = np.random.default_rng(0)
    out = {"note": "median RefreshResult.elapsed_ns over 300 forced refreshes; the reference "
                   "timed on this host's CPU, ours through the drop-in (host arrays in/out)"}
    for m, b in ((47, 64), (1000, 10)):
        live = apps(pdgsim, m, b, rng)
        for name, fn in (("ours", ours.refresh_priorities), ("reference", ref.refresh_priorities)):
            for _ in range(30):
                fn(live, 0.0, 1.0, force=True)
            ts = [fn(live, 0.0, 1.0, force=True).elapsed_ns for _ in range(300)]
            out[f"{name}_apps{m}_bins{b}_p50_us"] = float(np.median(ts)) / 1e3
    return out


# ---------------------------------------------------------------------------
# correlation masks (estimator.py:62-142)
# ---------------------------------------------------------------------------

def bench_masks(dev, copies=256, cpu_copies=2):
    """build_masks over `copies` x the 8 reference archetype graphs of the
    golden set (one pdg_pearson_flags launch incl. host gather), and the
    oracle (the reference's own arithmetic) on a bounded sample."""
    import copy
    import gzip

    from oracle import pdg_oracle as O
    from paper_2506_14851_b200.graphs import build_masks, graph_from_kb
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    base = {k: docs[k] for k in STREAM_TEMPLATES}
    graphs = {f"{k}#{i}": graph_from_kb(copy.deepcopy(v)) for i in range(copies)
              for k, v in base.items()}
    build_masks(graphs)
    tm = {}
    t0 = time.perf_counter()
    res = build_masks(graphs, timing=tm)
    gpu_ms = (time.perf_counter() - t0) * 1e3
    n_jobs = sum(len(m) for g in res.values() for m in g.values())
    t0 = time.perf_counter()
    for _ in range(cpu_copies):
        for v in base.values():
            O.build_masks(O.graph_from_kb(v))
    cpu_ms = (time.perf_counter() - t0) * 1e3 / cpu_copies * copies
    return {"graphs": len(graphs), "pearson_jobs": n_jobs, "ms": gpu_ms,
            "kernel_ms": tm.get("kernel_ms"), "cpu_port_ms_extrapolated": cpu_ms,
            "note": "wall clock incl. the host-side join of records (Python) and the copy back"}


# ---------------------------------------------------------------------------
# dispatch / preemption plan (K6)
# ---------------------------------------------------------------------------

def bench_dispatch(dev, n_tasks=1_000_000, slots=(64, 32, 32), reps=10, cpu_tasks=20_000):
    """One PriorityRefresh's preemption + dispatch decisions over a 1M-task
    table on 3 backends (device), and the reference's min()/max() scans
    (oracle restatement of simcore.py:512-516, 652-687) on a bounded sample."""
    import torch
    from oracle import pdg_oracle as O
    from paper_2506_14851_b200.dispatch import DispatchPlanner
    rng = np.random.default_rng(11)

    def table(n):
        be = rng.integers(0, len(slots), n)
        act = np.zeros(n, dtype=np.int64)
        for b, s in enumerate(slots):
            idx = np.flatnonzero(be == b)[:s]
            act[idx] = 1
        return {"backend": be, "active": act, "key": rng.lognormal(3, 2, n),
                "app_rank": rng.permutation(n), "stage": rng.integers(0, 4, n),
                "request": rng.integers(0, 3, n)}
    t = table(n_tasks)
    d = (torch.tensor(t["backend"], dtype=torch.int32, device=dev),
         torch.tensor(t["active"], dtype=torch.uint8, device=dev),
         torch.tensor(t["key"], dtype=torch.float64, device=dev),
         torch.tensor(t["app_rank"], dtype=torch.int32, device=dev),
         torch.tensor(t["stage"], dtype=torch.int32, device=dev),
         torch.tensor(t["request"], dtype=torch.int32, device=dev))
    pl = DispatchPlanner(device=str(dev))
    ev = pl.plan(*d, list(slots))
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pl.plan(*d, list(slots))                  # includes the event read-back
        ts.append((time.perf_counter() - t0) * 1e3)
    c = table(cpu_tasks)
    t0 = time.perf_counter()
    O.plan_dispatch(c["backend"].tolist(), c["active"].tolist(), c["key"].tolist(),
                    c["app_rank"].tolist(), c["stage"].tolist(), c["request"].tolist(),
                    list(slots), 1.5)
    cpu_ms = (time.perf_counter() - t0) * 1e3
    return {"tasks": n_tasks, "backends": len(slots), "slots": list(slots),
            "events": len(ev), "ms_per_plan_p50": float(np.median(ts)),
            "tasks_per_s": n_tasks / (float(np.median(ts)) / 1e3),
            "cpu_port_ms": cpu_ms, "cpu_sample_tasks": cpu_tasks,
            "note": "wall clock incl. event read-back; the CPU port's min()/max() scans "
                    "grow with tasks x slots"}


# ---------------------------------------------------------------------------
# BASELINE config 4 (refinement stream) and config 5 (prewarm need grid)
# ---------------------------------------------------------------------------

STREAM_TEMPLATES = ["code-gen", "fact-verify", "verify-chain-bimodal", "bimodal",
                    "plan-execute", "react-loop", "fanout-reduce", "cond"]
STREAM_ATTAINED = 5.0


def _c4_init(events):
    from oracle import pdg_oracle as O
    st = _CPU["c4"]
    return {"ev": list(events), "ogs": {k: O.graph_from_kb(st["docs"][k]) for k in st["names"]}}


def _c4_step(state, msg):
    """The reference's per-event path, restated: _complete_unit -> _estimate
    (monte_carlo_remaining_demand with the observation, simcore.py:562-587,
    317-325) -> set_remaining(256) -> _refresh([app], force=True) (one
    Gittins row + penalty, simcore.py:327-337)."""
    from oracle import pdg_oracle as O
    st = _CPU["c4"]
    out = []
    for e in state["ev"]:
        a = st["app"][e]
        nm = st["names"][st["graph"][a]]
        og = state["ogs"][nm]
        order_u = st["orders"][nm]
        ob = st["obs"][e]
        obs = [O.OObs(order_u[st["completed"][e]], float(ob[0]), float(ob[1]), int(ob[2]))]
        r = O.mc_remaining_demand(og, order_u[st["next"][e]], obs, N_SAMP, int(st["seed"][e]),
                                  VISIT_CAP)
        bz = O.bucketize(r.samples.tolist(), N_BINS)
        v = bz.midpoints() + STREAM_ATTAINED
        k = O.gittins_rank_batch(v[None], bz.probs[None], np.array([STREAM_ATTAINED]))[0]
        out.append((int(e), STREAM_ATTAINED * PENALTY if np.isnan(k) else float(k)))
    return out


def cpu_leg(init_fn, step_fn, items, procs, reps=1):
    """Events (or jobs) per second of a CPU leg over `items` on `procs`
    processes: best of `reps` timed passes after one warm pass."""
    wk = ShardWorkers(init_fn, step_fn, items, procs)
    try:
        res = wk.call(("run",))
        dts = [wk.timed(("run",))[1] for _ in range(reps)]
    finally:
        wk.close()
    return len(items) / min(dts), min(dts), [x for part in res for x in part]


def bench_stream(dev, n_apps=1_000_000, n_events=100_000, batch=1000, cpu=True):
    """Config 4: 1M-app queue of template PDGraphs (the reference's own
    archetypes, with correlation masks); 100k unit-completion events with
    observations, applied in micro-batches: K3+K2 re-estimate, K1 re-score of
    the touched rows, K5b merge into the global order.  Device-timed.  CPU
    legs: the reference's per-event path on a bounded sample of the same
    events, 1 core and all cores."""
    import gzip
    import torch
    from paper_2506_14851_b200.estimator import DemandEngine
    from paper_2506_14851_b200.graphs import graph_from_kb
    from paper_2506_14851_b200.queue import HistQueue
    from paper_2506_14851_b200.stream import RefinementStream
    from tools import synth
    with gzip.open(os.path.join(ROOT, "tests", "golden", "graphs.json.gz"), "rt") as fh:
        docs = json.load(fh)
    graphs = {k: graph_from_kb(docs[k]) for k in STREAM_TEMPLATES}
    q = synth.template_queue(graphs, n_apps, seed=41)
    ev = synth.events(graphs, q, n_events, seed=42)
    eng = DemandEngine(graphs, device=str(dev))
    hq = HistQueue(n_apps, N_BINS)
    gi = torch.from_numpy(q["graph"]).to(dev)
    ui = torch.from_numpy(q["unit"].copy()).to(dev)
    seeds = torch.arange(n_apps, dtype=torch.int64, device=dev) * 1000003
    eng.run(gi, ui, seeds, n=N_SAMP, bucket_count=N_BINS, queue=hq)
    hq.est_age[:n_apps] = 0.0
    hq.age[:n_apps] = 0.0
    hq.n = n_apps
    hq.score()
    st = RefinementStream(eng, hq, gi, ui, bucket_count=N_BINS)
    st.order()
    # pinned host event buffers; each batch is uploaded inside its timed span
    h = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
         for k, v in (("app", ev["app"]), ("next", ev["next"]), ("comp", ev["completed"]),
                      ("obs", ev["obs"]), ("seed", ev["seed"]))}
    h["att"] = torch.full((n_events,), STREAM_ATTAINED, dtype=torch.float64).pin_memory()
    d = {k: torch.empty(v.shape, dtype=v.dtype, device=dev) for k, v in h.items()}
    stream = torch.cuda.current_stream()
    nb = n_events // batch

    def run_batch(i, evs=None):
        sl = slice(i * batch, (i + 1) * batch)
        for k in h:
            d[k][sl].copy_(h[k][sl], non_blocking=True)
        if evs:
            evs[0].record(stream)
        st.process(d["app"][sl], d["next"][sl], d["seed"][sl], d["comp"][sl], d["obs"][sl],
                   d["att"][sl], resort=True)

    run_batch(0)                                       # warm-up (re-applies batch 0)
    torch.cuda.synchronize()
    launches, names = count_launches(lambda _: run_batch(1))
    marks = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(nb)]
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(nb):
        sub = torch.cuda.Event(enable_timing=True)
        run_batch(i, [sub])
        marks[i] = (sub, torch.cuda.Event(enable_timing=True))
        marks[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    total_ms = t0.elapsed_time(t1)
    lat = np.array([a.elapsed_time(b) for a, b in marks])
    keys = hq.key_f32[:n_apps].cpu().numpy()
    # algorithmic bytes per batch: event records in (app, next, completed,
    # seed, obs[3], attained = 52 B), histogram rows out (2 B/bucket + 40 B),
    # K1 over the touched rows (row in + 25 B out), and the K5b merge of the
    # resident order (1M x (8 B key + 4 B slot) read and written) + mark bytes
    row = 2 * hq.stride + 40
    bpb = batch * (52 + row + row + 25) + n_apps * (2 * 12 + 1)
    peak, _ = measured_peaks()
    ms_b = float(np.mean(lat))
    out = {"workload": f"config4: {n_apps} queued template apps ({len(STREAM_TEMPLATES)} "
                       f"reference archetypes), {n_events} refinement events in batches of "
                       f"{batch}; per batch K3+K2+a4 re-estimate, K1 re-score, K5b merge into "
                       f"the global order",
           "events_per_s": n_events / (total_ms / 1e3), "batch": batch,
           "batch_latency_ms_p50": float(np.median(lat)),
           "batch_latency_ms_p99": float(np.percentile(lat, 99)),
           "launches_per_batch": launches, "kernels": names,
           "roofline": {"bound": "hbm", "bytes_per_batch": bpb,
                        "achieved": bpb / (ms_b / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": bpb / (ms_b / 1e3) / 1e9 / peak,
                        "note": "launch-latency bound at 1000-event batches: the batch's "
                                "algorithmic bytes are dominated by the K5b merge over the "
                                "resident 1M-app order"},
           "note": "latency = batch upload issued -> global order visible (device events); "
                   "at 100k events/s a 1000-event batch is 10 ms of arrivals"}
    if cpu:
        _CPU["c4"] = {"docs": {k: docs[k] for k in STREAM_TEMPLATES}, "names": q["names"],
                      "orders": q["orders"], "graph": q["graph"], "app": ev["app"],
                      "next": ev["next"], "completed": ev["completed"], "obs": ev["obs"],
                      "seed": ev["seed"]}
        procs = os.cpu_count() or 1
        r1, dt1, res1 = cpu_leg(_c4_init, _c4_step, list(range(300)), 1)
        rn, dtn, _ = cpu_leg(_c4_init, _c4_step, list(range(min(150 * procs, n_events))), procs)
        # the last batch holding each sampled event decides the app's key: the
        # events are on distinct apps, so compare every sampled key
        rel = max(abs(float(keys[ev["app"][e]]) - k) / max(abs(k), 1e-300) for e, k in res1)
        out["cpu_baseline"] = {
            "kind": "port", "unit": "events/s",
            "value_1core": r1, "sample_1core": 300, "wall_s_1core": dt1,
            "value_all_cores": rn, "cores": procs, "sample_all_cores": min(150 * procs, n_events),
            "wall_s_all_cores": dtn,
            "path": "per event: oracle MC(n=512) with the observation (K3 conditioning) + "
                    "bucketize(256) + one Gittins row + penalty (simcore.py:562-587 -> "
                    "_estimate 317-325 -> _refresh([app], force=True) 327-337)",
            "keys_max_rel_err_vs_gpu": rel}
    return out


def _c5_init(jobs):
    return {"jobs": list(jobs)}


def _c5_step(state, msg):
    """plan_prewarm per (app, successor) (prewarm.py:42-96 via
    _plan_prewarms, simcore.py:450-487) and the need grid per app."""
    from oracle import pdg_oracle as O
    st = _CPU["c5"]
    U, S = st["U"], st["SLOT"]
    out = []
    for a in state["jobs"]:
        g_, u_ = int(st["g"][a]), int(st["u"][a])
        now = float(st["now"][a])
        svc = st["svc"][g_ * U + u_]
        comp = [now + s for s in svc]
        base = (g_ * U + u_) * S
        plans, succ = [], []
        for slot in range(int(st["s_len"][g_ * U + u_])):
            ty = int(st["utype"][g_ * U + int(st["s_nxt"][base + slot])])
            p = float(st["s_p"][base + slot])
            succ.append((p, ty))
            plans.append(O.plan_prewarm(comp, N_BINS, p, float(st["warm"][ty]), st["knob"], now)
                         if ty >= 0 else None)
        if msg[0] == "need":
            out.append((a, O.need_grid(svc, succ, now, st["win"], st["T"])))
        else:
            out.append((a, plans))
    return out


def bench_need(dev, n_apps=1_000_000, n_templates=1024, steps=10, cpu=True):
    """Config 5: need probability for 16 backend types x 32 windows over 1M
    apps (templates: depth-8 synth graphs, unit types random in [0,16)), and
    the latest-safe trigger per (app, successor).  CPU legs: plan_prewarm per
    (app, successor) and the need grid per app on bounded samples of the same
    jobs, 1 core and all cores."""
    import torch
    from paper_2506_14851_b200.prewarm import PrewarmTables
    from tools import synth
    w = synth.make(n_templates, N_REC, seed=77)
    rng = np.random.default_rng(78)
    A, U, R = n_templates, synth.U, N_REC
    svc = np.sort(w["dur"], axis=2).reshape(-1)
    counts = np.zeros((A, U, U))
    for v in range(U):
        counts[:, :, v] = np.count_nonzero(w["nxt"] == v, axis=2)
    s_off = np.arange(A * U) * synth.SLOT
    s_len = w["succ_len"].reshape(-1)
    s_nxt = w["succ_nxt"].reshape(-1)
    s_p = np.zeros(A * U * synth.SLOT)
    for a_u in range(A * U):
        a, u = divmod(a_u, U)
        for q in range(s_len[a_u]):
            s_p[a_u * synth.SLOT + q] = counts[a, u, s_nxt[a_u * synth.SLOT + q]] / R
    utype = rng.integers(0, 16, A * U)
    tb = PrewarmTables(svc_sorted=svc, svc_off=np.arange(A * U) * R, svc_len=np.full(A * U, R),
                       graph_base=np.arange(A) * U, succ_off=s_off, succ_len=s_len,
                       succ_nxt=s_nxt, succ_p=s_p, unit_type=utype, n_types=16,
                       device=str(dev))
    gv = rng.integers(0, A, n_apps).astype(np.int32)
    uv = rng.integers(0, U, n_apps).astype(np.int32)
    nowv = rng.uniform(0, 100, n_apps)
    g = torch.from_numpy(gv).to(dev)
    u = torch.from_numpy(uv).to(dev)
    now = torch.from_numpy(nowv).to(dev)
    winv = np.linspace(2.0, 64.0, 32)
    win = torch.from_numpy(winv).to(dev)
    need = torch.empty((n_apps, 16, 32), dtype=torch.float32, device=dev)
    for _ in range(3):
        tb.need(g, u, now, win, out=need)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    for e0, e1 in ev:
        e0.record()
        tb.need(g, u, now, win, out=need)
        e1.record()
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    # the per-successor latest-safe triggers (plan_prewarm per (app, successor))
    knob = 0.3
    warmv = rng.uniform(1.0, 30.0, 16)
    warm = torch.from_numpy(warmv).to(dev)
    tb.triggers(g, u, now, warm, knob, N_BINS)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    has, trig, pe = tb.triggers(g, u, now, warm, knob, N_BINS)
    e1.record()
    torch.cuda.synchronize()
    trig_ms = e0.elapsed_time(e1)
    jobs = int((s_len.reshape(A, U)[gv, uv]).sum())
    trig_out = {"ms": trig_ms, "plans": int(has.sum().item()), "app_successor_jobs": jobs,
                "jobs_per_s": jobs / (trig_ms / 1e3),
                "note": f"plan_prewarm (bit-exact) for every (app, successor), knob {knob}, "
                        f"{N_BINS} buckets, warm-up per backend type U(1, 30) s"}
    # algorithmic bytes per app: dense need row out + job (graph, unit, now)
    bytes_app = 16 * 32 * 4 + 4 + 4 + 8
    peak, _ = measured_peaks()
    out = {"workload": f"config5: need[{n_apps},16,32] float32 + [16,32] aggregate over "
                       f"{n_apps} apps ({n_templates} depth-8 templates)",
           "apps_per_s": n_apps / (ms / 1e3), "ms_per_launch": ms, "triggers": trig_out,
           "roofline": {"bound": "hbm", "bytes_per_app": bytes_app,
                        "achieved": bytes_app * n_apps / (ms / 1e3) / 1e9, "peak": peak,
                        "unit": "GB/s",
                        "frac": bytes_app * n_apps / (ms / 1e3) / 1e9 / peak}}
    if cpu:
        _CPU["c5"] = {"U": U, "SLOT": synth.SLOT, "g": gv, "u": uv, "now": nowv,
                      "svc": svc.reshape(A * U, R), "s_len": s_len, "s_nxt": s_nxt, "s_p": s_p,
                      "utype": utype, "warm": warmv, "knob": knob, "win": winv, "T": 16}
        procs = os.cpu_count() or 1
        sample = np.random.default_rng(79).choice(n_apps, 400, replace=False).tolist()
        wide = np.random.default_rng(80).choice(n_apps, 100 * procs, replace=False).tolist()
        jobs_of = lambda apps: int(s_len.reshape(A, U)[gv[apps], uv[apps]].sum())  # noqa
        t1, dt1, res = cpu_leg(_c5_init, lambda s, m: _c5_step(s, ("plan",)), sample, 1)
        tn, dtn, _ = cpu_leg(_c5_init, lambda s, m: _c5_step(s, ("plan",)), wide, procs)
        n1, ndt1, nres = cpu_leg(_c5_init, lambda s, m: _c5_step(s, ("need",)), sample, 1)
        # cross-check the sample against the device results
        hs, tr, pv = has.cpu().numpy(), trig.cpu().numpy(), pe.cpu().numpy()
        mism = 0
        for a, plans in res:
            for slot, p in enumerate(plans):
                want = p is not None
                if bool(hs[a, slot]) != want or (want and (tr[a, slot] != p[0]
                                                          or pv[a, slot] != p[1])):
                    mism += 1
        nd = need[torch.tensor([a for a, _ in nres], device=dev)].cpu().numpy()
        nerr = float(max(np.max(np.abs(nd[i] - x)) for i, (_, x) in enumerate(nres)))
        js1, jsn = jobs_of(np.array(sample)), jobs_of(np.array(wide))
        out["cpu_baseline"] = {
            "kind": "port", "cores": procs,
            "plan_prewarm_jobs_per_s_1core": js1 / dt1,
            "plan_prewarm_jobs_per_s_all_cores": jsn / dtn,
            "need_apps_per_s_1core": len(sample) / ndt1,
            "sample": f"plan_prewarm: {len(sample)} apps ({js1} app x successor jobs) on 1 "
                      f"core, {len(wide)} apps ({jsn} jobs) on {procs}; need grid: "
                      f"{len(sample)} apps on 1 core; same jobs as the device run",
            "triggers_mismatches_vs_gpu": mism, "need_max_abs_err_vs_gpu": nerr}
        del t1, tn, n1
    return out


def main():
    args = parse()
    world, _, _ = dist_env()
    if args.dry_run:
        if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
            sys.exit(spawn_ranks(args))
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
