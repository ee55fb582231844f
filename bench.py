#!/usr/bin/env python
"""Benchmark of the restricted-PCG energy-minimisation hot path on B200.

One STEP = one pass of the whole hot path over the
synthetic workload, through the C ABI: emin_setup from device-resident inputs
(validation, index prep, halo plan, Alg. 2, r0, E0) -> emin_iterate(k) (k
restricted-PCG steps, CUDA graph) -> emin_energy -> emin_get_P (into a device
buffer) -> emin_destroy.  ``value`` = P-nonzero updates per second =
nnz(W) * k * K / (device time of the K timed steps), max over ranks.

Default workload: BASELINE config 3 (FV lognormal 128^3, 40 iterations), the
configuration BASELINE.json's metric ("... at 1/2/4/8 GPU") is quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl reference]

--gpus N without a torchrun environment launches N ranks itself (one process
per GPU, NCCL); it fails if fewer than N GPUs are visible.  Each rank passes
emin_setup only its own rows of A, P and B (partition.rank_slice).
--impl reference runs the CPU oracle (the tier's reference arm) on the host.
--dry-run (CPU, gloo): the launcher and the partition without a GPU (tests).
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "P-nonzero updates/sec per restricted-PCG iter; HBM GB/s vs peak at 1/2/4/8 GPU"
UNIT = "P-nonzero updates/s"
WORKLOADS = {
    "1": "config1: 2D Poisson 5-pt 32^2, equal-weight start, 20 it",
    "2": "config2: 3D 7-pt aniso (1,1,1e-3) 64^3, least-norm start, 30 it",
    "3": "config3: FV lognormal diffusion 128^3 (log10 k in [-6,6], corr 8), least-norm start, 40 it",
    "4": "config4: Q1 elasticity 48^3, E=1, nu=0.3, bottom clamped, 6 RBMs, 30 it",
    "5": "config5: Q1 elasticity 160^3, 8 layers E in 10^U(-2,2), nu=0.25, 6 RBMs, 40 it",
}
KEYS = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload_name(args):
    w = WORKLOADS.get(args.config, args.config)
    return w if args.size is None else f"{w} [reduced size {args.size}]"


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def spgemm_algorithmic_bytes(prob, nnzW, nnzAFF, nF):
    """bytes the masked SpGEMM (+ projection) must move per
    launch: A_FF values + column ids (12 B/entry), row pointers (4 B/row at
    int32), and per W entry the y value + column id read, yb written and
    the Q_i row read (8 + 4 + 8 + 8 nv B)."""
    return 12 * nnzAFF + 4 * (nF + 1) + nnzW * (20 + 8 * prob.nv)


def iteration_algorithmic_bytes(prob, nnzW, nnzAFF, nF):
    """SURVEY §8d B_iter (fused two-stage schedule): 12 nnz(A_FF) + 4 (n_F+1)
    + nnz(W) (84 + 8 nv)."""
    return 12 * nnzAFF + 4 * (nF + 1) + nnzW * (84 + 8 * prob.nv)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region.
    The sampler process is started before the warm-up (its start-up -- NVML
    initialisation -- must not fall inside the timed region) and keeps
    sampling every 200 ms (the profiling recipe's period); summary() keeps the samples whose timestamps lie
    in the timed region (mark_begin / mark_end), falling back to all samples
    if the region was shorter than the sampling period."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0, period_ms=200):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.period = int(period_ms)
        self.p = None
        self.t0 = self.t1 = None

    def __enter__(self):
        if self.period <= 0:          # diagnostics only (--clock-ms 0): no sampler
            return self
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", str(self.period)],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def wait_first(self, timeout=10.0):
        """block until the sampler has written its first line"""
        t = time.time()
        while self.p is not None and time.time() - t < timeout:
            self.f.flush()
            if os.path.getsize(self.f.name) > 0:
                return
            time.sleep(0.02)

    def mark_begin(self):
        self.t0 = datetime.datetime.now()

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        with open(self.f.name) as fh:
            rows = [l.strip().split(",") for l in fh.read().splitlines() if l.strip()]
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 10]

        def ts(r):
            try:
                return datetime.datetime.strptime(r[0], "%Y/%m/%d %H:%M:%S.%f")
            except ValueError:
                return None
        inside = [r for r in rows if self.t0 and self.t1 and ts(r) and self.t0 <= ts(r) <= self.t1]
        rows = inside or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        rows = [r[1:] for r in rows]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows), "samples_in_region": len(inside),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                                   default=None)}


# ---------------------------------------------------------------------------
# the CPU oracle legs (reference arm, cpu_baseline): the only places bench.py
# executes oracle/
# ---------------------------------------------------------------------------

def oracle_iterate_counted(o, k):
    """o.iterate(k), returning the steps taken even if the unguarded run
    meets round-off curvature (y'Ky < 0, EMIN_ERR_BREAKDOWN) before k."""
    from oracle import OracleError
    if k <= 0:
        return 0
    before = o.k_total
    try:
        kd, _ = o.iterate(k)
        return kd
    except OracleError:
        return o.k_total - before


def oracle_step_rate(prob, threads, budget_s):
    """One oracle step of ``prob`` (setup + k iterations + energy + P out) on
    ``threads`` host threads, the iteration count bounded so the step takes
    about ``budget_s``.  Returns (updates/s, description, seconds, k_used)."""
    import oracle
    from oracle import Oracle
    oracle.set_threads(threads)
    k = prob.iters
    t0 = time.perf_counter()
    o = Oracle(prob, stagnation_rel=0.0)      # the GPU arm's setting: all k steps, guard off
    t_setup = time.perf_counter() - t0
    t1 = time.perf_counter()
    kd1, _ = o.iterate(1)
    t_it = time.perf_counter() - t1
    k_s = max(0, min(k - 1, int((budget_s - t_setup) / max(t_it, 1e-4)) - 1))
    t1 = time.perf_counter()
    kd2 = oracle_iterate_counted(o, k_s)
    t_its = time.perf_counter() - t1
    o.energy()
    o.get_P()
    tot = time.perf_counter() - t0
    iters = kd1 + kd2
    v = prob.nnz_W * iters / tot
    desc = (f"setup {t_setup:.2f} s + {iters} of {k} iterations ({(t_it + t_its) / max(iters, 1):.3f} s/it) "
            f"+ energy + P = {tot:.1f} s on {threads} thread(s)")
    return v, desc, tot, iters


def cpu_baseline(prob, args):
    """The oracle as it stands on this host: all cores, and 1 thread (SURVEY
    §8d / BASELINE.md §3), each a bounded sample of the same workload (one
    step, iterations capped to ~15 s per leg).  Config 5 is sampled at the
    generator's 40^3 size (the full oracle needs ~1 min per iteration)."""
    import oracle
    nproc = os.cpu_count() or 1
    sample_prob, note = prob, ""
    if args.config == "5" and prob.n > 3_000_000:
        from workloads.problems import make_config
        sample_prob = make_config("5", size=40)
        note = f"same generator at 40^3 elements ({sample_prob.n} dofs): "
    v_all, d_all, _, _ = oracle_step_rate(sample_prob, nproc, 15.0)
    v_one, d_one, _, _ = oracle_step_rate(sample_prob, 1, 15.0)
    oracle.set_threads(nproc)
    return {"value": v_all, "unit": UNIT, "cores": nproc, "kind": "oracle",
            "sample": note + "one oracle step of the workload: " + d_all,
            "cpu_model": cpu_model(), "nproc": nproc,
            "single_thread": {"value": v_one, "cores": 1, "sample": note + d_one}}


def run_reference(args, rank):
    """The tier's reference arm: the CPU oracle as it stands, all host cores,
    rank 0 only (the other ranks exit without work)."""
    if rank != 0:
        return None
    from workloads.problems import make_config
    prob = make_config(args.config, size=args.size)
    nproc = os.cpu_count() or 1
    k = prob.iters
    steps, warm = args.steps, args.warmup
    # bounded: each step at most ~240 s / (steps + warmup) of CPU time
    budget = 240.0 / max(1, steps + warm)
    v, desc, _, k_step = oracle_step_rate(prob, nproc, budget)
    times = []
    for s in range(warm + steps):
        import oracle
        from oracle import Oracle
        oracle.set_threads(nproc)
        t0 = time.perf_counter()
        o = Oracle(prob, stagnation_rel=0.0)
        kd = oracle_iterate_counted(o, k_step)
        o.energy()
        o.get_P()
        dt = time.perf_counter() - t0
        k_step = min(k_step, kd) if kd else k_step
        if s >= warm:
            times.append(dt)
    tot = sum(times)
    v = prob.nnz_W * k_step * steps / tot
    sample = (f"{workload_name(args)}: full oracle step (setup + {k_step} of {k} iterations + energy + P) "
              f"per step, C + OpenMP on {nproc} threads ({cpu_model()}), {steps} timed steps")
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * tot / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(args), "iters": k_step},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ---------------------------------------------------------------------------
# launcher: --gpus N without torchrun spawns the N ranks itself
# ---------------------------------------------------------------------------

def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    n = args.gpus
    if not args.dry_run:
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < n:
            print(json.dumps({"error": f"--gpus {n} needs {n} visible GPUs, found {have}", "n_gpus": n}),
                  flush=True)
            log(f"[bench] --gpus {n}: only {have} GPU(s) visible; refusing to time fewer ranks than asked")
            return 2
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        out = None if r == 0 else subprocess.DEVNULL
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=out))
    rcs = [p.wait() for p in procs]
    return max(rcs)


def dry_run(args, world, rank):
    """CPU-only check of the launcher and the partition: every rank builds
    its slice, the ranks agree over gloo, rank 0 prints a summary line."""
    import torch
    import torch.distributed as dist
    from paper_2208_02995_b200.partition import partition_rows, plane_rows, rank_slice
    from workloads.problems import make_config
    prob = make_config(args.config, size=args.size)
    if world > 1:
        dist.init_process_group("gloo")
    ranges = partition_rows(prob.P_rowptr, prob.is_coarse, world, plane=plane_rows(prob))
    rb, re_ = ranges[rank]
    a = rank_slice(prob, rb, re_)
    mine = torch.tensor([rb, re_, int(a["P_rowptr"][-1]), int(a["A_rowptr"][-1]), os.getpid()], dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    if world > 1:
        dist.all_gather(allv, mine)
    else:
        allv = [mine]
    allv = [t.tolist() for t in allv]
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    covers = allv[0][0] == 0 and allv[-1][1] == prob.n and all(allv[i][1] == allv[i + 1][0] for i in range(world - 1))
    print(json.dumps({"dry_run": True, "n_gpus": world, "ranges": [v[:2] for v in allv],
                      "nnz_P_per_rank": [v[2] for v in allv], "nnz_A_per_rank": [v[3] for v in allv],
                      "pids": [v[4] for v in allv], "covers": bool(covers),
                      "nnz_P_total_ok": sum(v[2] for v in allv) == int(prob.P_rowptr[-1]),
                      "workload": workload_name(args)}), flush=True)
    return 0


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--clock-ms", type=int, default=200,
                    help="nvidia-smi sampling period during the timed region (0: no sampler, diagnostics only)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("EMIN_BENCH_CONFIG", "3"))
    ap.add_argument("--size", type=int, default=None, help="reduced generator size (tests only; not a bench line)")
    ap.add_argument("--impl", default="emin", choices=["emin", "reference"])
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo check of the launcher and partition")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--precond", default="jacobi", choices=["jacobi", "sgs"],
                    help="Alg. 3 preconditioner: Jacobi M_1 (default, the headline) or projected SGS M_2")
    ap.add_argument("--sgs-key", default="color", choices=["color", "natural"],
                    help="SGS visiting order (reading A23): a grid colouring or the natural row order")
    ap.add_argument("--profile-steps", type=int, default=2,
                    help="timed steps (the last ones) that record per-kernel CUDA events (0 = all); "
                         "the kernel times of the roofline come from these steps.  The event "
                         "nodes cost ~1.5 ms per config-3 step, so by default only 2 steps carry "
                         "them and the others run as a user runs them")
    ap.add_argument("--start", default="given", choices=["given", "maxvol"],
                    help="W^ start: the workload's (least-norm) or Alg. 1's max-vol tentative start")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if args.dry_run:
        return dry_run(args, world, rank)
    if world != args.gpus:
        log(f"[bench] WORLD_SIZE={world} but --gpus {args.gpus}: timing {world} rank(s)")

    from workloads.problems import make_config
    t0 = time.perf_counter()
    prob = make_config(args.config, size=args.size)
    log(f"[bench] rank {rank}: generated {prob.name}: n={prob.n} nF={prob.n_F} nnzW={prob.nnz_W} "
        f"in {time.perf_counter() - t0:.1f}s")

    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2208_02995_b200 import build as _build
    if rank == 0:
        _build()
    if world > 1:
        dist.barrier()
    from paper_2208_02995_b200 import emin as E
    from paper_2208_02995_b200.partition import partition_rows, plane_rows, rank_slice

    stream = torch.cuda.current_stream()
    # row partition (contiguous z-slabs balanced by nnz(W)); each rank gets its
    # own rows only (rebased row pointers), plus the global is_coarse and B_c
    comm = None
    rb, re_ = 0, prob.n
    if world > 1:
        rb, re_ = partition_rows(prob.P_rowptr, prob.is_coarse, world, plane=plane_rows(prob))[rank]
        comm = E.nccl_comm_from_torch()
    host = rank_slice(prob, rb, re_)
    key = None
    if args.precond == "sgs":
        from workloads.problems import sgs_key
        key = sgs_key(prob, args.sgs_key)[rb:re_]
    host["sgs_key"] = key
    dev = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)).cuda()) for k, v in host.items()}
    nnzP = int(host["P_rowptr"][-1])
    out_dev = torch.empty(nnzP, dtype=torch.float64, device="cuda")
    k_it = prob.iters
    nnzW_global = prob.nnz_W

    def setup(arrs):
        return E.emin_setup(prob.n, prob.nc, arrs["A_rowptr"], arrs["A_col"], arrs["A_val"], arrs["is_coarse"],
                            arrs["P_rowptr"], arrs["P_col"], arrs["P_val"], prob.nv, arrs["B"], arrs["Bc"],
                            block_size=prob.block_size, stagnation_rel=0.0, stream=stream.cuda_stream,
                            nccl_comm=comm, row_begin=rb, row_end=re_, precond=args.precond, start=args.start,
                            sgs_key=arrs["sgs_key"])

    stats = {"launches": 0, "spgemm_ms": 0.0, "spgemm_n": 0, "stage_ms": [0.0, 0.0], "scalar_ms": 0.0,
             "k_done": [], "E": None, "report": None}

    def step(arrs, out, profile):
        h = setup(arrs)
        if profile:
            E.emin_set_profiling(h, 1)
        E.emin_iterate(h, k_it)
        stats["E"] = E.emin_energy(h)
        E.emin_get_P(h, out)
        rep = E.emin_report(h)
        stats["launches"] += rep["launches"]
        stats["k_done"].append(rep["k_total"])
        stats["report"] = rep
        if profile:
            kt = E.emin_kernel_times(h)
            stats["spgemm_ms"] += kt["spgemm"][0]
            stats["spgemm_n"] += kt["spgemm"][1]
            stats["stage_ms"][0] += kt["stage1"][0]
            stats["stage_ms"][1] += kt["stage2"][0]
            stats["scalar_ms"] += kt["scalar"][0]
        E.emin_destroy(h)

    # the clock sampler starts before the warm-up (its start-up stays out of
    # the timed region; only samples inside the region are summarised)
    clk = ClockSampler(local_rank, args.clock_ms)
    clk.__enter__()
    # warm-up (untimed): the W requested steps, then -- only while the last
    # steps are not yet steady (a box just freed by a large process was seen
    # to run every step 3.5x slower for ~0.5 s) -- up to 40 more, about 0.3 s
    # of extra warm-up at most on config 3
    wt = []
    for w_i in range(args.warmup + (40 if world == 1 else 0)):    # ranks step in lockstep (collectives)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        step(dev, out_dev, w_i < args.warmup)
        eb.record(stream)
        torch.cuda.synchronize()
        wt.append(ea.elapsed_time(eb))
        if w_i + 1 >= args.warmup and len(wt) >= 4 and max(wt[-3:]) <= 1.2 * min(wt[1:]):
            break
    if len(wt) > args.warmup:
        log(f"[bench] rank {rank}: {len(wt) - args.warmup} extra warm-up steps until steady ({wt[-1]:.2f} ms)")
    clk.wait_first()
    stats.update(launches=0, spgemm_ms=0.0, spgemm_n=0, stage_ms=[0.0, 0.0], scalar_ms=0.0, k_done=[])

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: K whole-path steps, device-resident inputs
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    nprof = args.steps if args.profile_steps <= 0 else min(args.profile_steps, args.steps)
    clk.mark_begin()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev0.record(stream)
    evs[0].record(stream)
    for it in range(args.steps):
        step(dev, out_dev, it >= args.steps - nprof)
        evs[it + 1].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    seq = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    per = sorted(seq)
    step_stats = {"min": per[0], "median": per[len(per) // 2], "max": per[-1],
                  "above_1p5x_median": sum(t > 1.5 * per[len(per) // 2] for t in seq)}
    log(f"[bench] rank {rank}: per-step ms min {per[0]:.3f} median {per[len(per) // 2]:.3f} max {per[-1]:.3f}; "
        f"steps above 1.5x median: {sum(t > 1.5 * per[len(per) // 2] for t in seq)}")
    log("[bench] per-step ms: " + " ".join(f"{t:.2f}" for t in seq))
    clk.__exit__(None, None, None)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches_timed = stats["launches"]
    clocks = clk.summary()
    rep = stats["report"]
    nnzW, nnzAFF, nF = rep["nnz_W"], rep["nnz_AFF"], rep["n_fine"]
    # updates actually performed: the CG steps each timed step took (never the
    # requested ones; 0 if the CG stopped at once).  Value-independent kernels
    # make every step take the same number (stagnation guard off).
    kd_steps = stats["k_done"]
    k_eff = min(min(kd_steps), k_it)
    if len(set(kd_steps)) != 1:
        log(f"[bench] warning: k_done differs between steps: {sorted(set(kd_steps))}; counting the minimum")
    updates = nnzW_global * k_eff * args.steps
    value = updates / (ms / 1e3)

    # ---- iteration-only rate (setup excluded, SURVEY §8d definition)
    h = setup(dev)
    E.emin_iterate(h, k_it)
    torch.cuda.synchronize()
    ia, ib = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(1, args.steps // 2)
    it_ms = []
    for _ in range(reps):
        E.emin_reset(h)
        barrier()
        ia.record(stream)
        E.emin_iterate(h, k_it)
        ib.record(stream)
        torch.cuda.synchronize()
        it_ms.append(ia.elapsed_time(ib))
    E.emin_destroy(h)
    it_ms_med = max_over_ranks(statistics.median(it_ms))

    # ---- roofline of the dominant kernel (masked SpGEMM), from the timed region
    peak, peak_src = measured_peak()
    sp_avg_ms = stats["spgemm_ms"] / max(1, stats["spgemm_n"])
    sp_bytes = spgemm_algorithmic_bytes(prob, nnzW, nnzAFF, nF)
    achieved = sp_bytes / (sp_avg_ms / 1e3) / 1e9 if sp_avg_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": "masked SpGEMM + Pi_B (yb = Pi K y)", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": sp_bytes,
                "avg_launch_ms": sp_avg_ms, "launches": stats["spgemm_n"],
                "share_of_step": (stats["spgemm_ms"] / nprof / (ms / args.steps)) if ms > 0 else None,
                "profiled_steps": nprof, "rank": rank}

    # ---- e2e: the same metric through the C ABI with HOST buffers: every
    # step passes pinned host pointers to emin_setup (the library copies them
    # to the device inside the call) and emin_get_P writes P into a host
    # buffer; all of it inside the timed region.  e2e_pipelined: the same
    # step with the H2D of step s+1 and the D2H of step s overlapped with step
    # s's compute by the caller (torch copies on side streams into device
    # buffers, device pointers into the C ABI).
    e2e = e2e_pipe = None
    if not args.no_e2e:
        pin_t = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)).pin_memory())
                 for k, v in host.items()}
        pin = {k: (None if v is None else v.numpy()) for k, v in pin_t.items()}
        out_host_t = torch.empty(nnzP, dtype=torch.float64).pin_memory()
        out_host = out_host_t.numpy()
        h2d = sum(v.nbytes for v in pin.values() if v is not None)
        d2h = out_host.nbytes + 8
        n_e2e = max(1, args.steps // 2)

        def whole_job_bytes(b):
            if world == 1:
                return int(b)
            import torch.distributed as dist
            t = torch.tensor([b], device="cuda", dtype=torch.int64)
            dist.all_reduce(t)
            return int(t.item())

        h2d_all, d2h_all = whole_job_bytes(h2d), whole_job_bytes(d2h)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # (a) serial C-ABI calls with host pointers
        step(pin, out_host, False)
        barrier()
        torch.cuda.synchronize()
        ea.record(stream)
        for _ in range(n_e2e):
            step(pin, out_host, False)
        eb.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(ea.elapsed_time(eb))
        e2e = {"value": nnzW_global * k_eff * n_e2e / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h_all,
               "h2d_bytes_per_step_per_rank": int(h2d), "ms_per_step": e_ms / n_e2e, "steps": n_e2e,
               "mode": "serial C-ABI calls with pinned host pointers (emin_setup copies the inputs, "
                       "emin_get_P writes P to host memory)"}
        # (b) caller-pipelined
        cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
        bufs = [{k: (None if v is None else torch.empty(v.shape, dtype=v.dtype, device="cuda"))
                 for k, v in pin_t.items()} for _ in range(2)]
        outs = [torch.empty(nnzP, dtype=torch.float64, device="cuda") for _ in range(2)]
        mk = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        h2d_done, in_free, out_free, p_ready = mk(), mk(), mk(), mk()

        def enqueue_h2d(s):
            b = s % 2
            with torch.cuda.stream(cs):
                if s >= 2:
                    cs.wait_event(in_free[b])
                for k, v in pin_t.items():
                    if v is not None:
                        bufs[b][k].copy_(v, non_blocking=True)
                h2d_done[b].record(cs)

        def pstep(s, n):
            b = s % 2
            stream.wait_event(h2d_done[b])
            if s + 1 < n:
                enqueue_h2d(s + 1)
            hh = setup(bufs[b])
            in_free[b].record(stream)
            E.emin_iterate(hh, k_it)
            stats["E"] = E.emin_energy(hh)
            if s >= 2:
                stream.wait_event(out_free[b])
            E.emin_get_P(hh, outs[b])
            p_ready[b].record(stream)
            with torch.cuda.stream(ds):
                ds.wait_event(p_ready[b])
                out_host_t.copy_(outs[b], non_blocking=True)
                out_free[b].record(ds)
            E.emin_destroy(hh)

        def run(n):
            cs.wait_stream(stream)
            enqueue_h2d(0)
            for s_ in range(n):
                pstep(s_, n)
            stream.wait_stream(ds)
            stream.wait_stream(cs)

        run(2)                                     # untimed warm-up of the pipeline
        barrier()
        torch.cuda.synchronize()
        ea.record(stream)
        run(n_e2e)
        eb.record(stream)
        torch.cuda.synchronize()
        p_ms = max_over_ranks(ea.elapsed_time(eb))
        e2e_pipe = {"value": nnzW_global * k_eff * n_e2e / (p_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d_all, "d2h_bytes_per_step": d2h_all,
                    "ms_per_step": p_ms / n_e2e, "steps": n_e2e,
                    "mode": "caller-pipelined: H2D of step s+1 and D2H of step s overlap step s's compute "
                            "(pinned host buffers, two device buffer sets)"}

    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(prob, args)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "error": str(ex)}
    it_bytes = iteration_algorithmic_bytes(prob, nnzW, nnzAFF, nF)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args), "iters_per_step": k_it, "nnz_W": nnzW_global,
                   "nnz_A_FF_rank0": nnzAFF, "n_F_rank0": nF, "nv": prob.nv,
                   "step": "emin_setup(device inputs) + emin_iterate(k) + emin_energy + emin_get_P + emin_destroy",
                   "l2": "inputs larger than L2 (per-iteration working set %.2f GB > 126 MB)" % (it_bytes / 1e9),
                   "parallelism": f"rows{world} (z-slab row partition, NCCL halo + allreduce)" if world > 1
                   else "single GPU",
                   "kernel_path": E.KERNEL_PATHS.get(rep["kernel_path"]),
                   "precond": args.precond if args.precond == "jacobi" else
                   f"sgs ({args.sgs_key} order, {rep['sgs_levels']} levels per sweep)",
                   "start": args.start,
                   "halo_rank0": {"rows": rep["n_halo_rows"], "entries": rep["n_halo_entries"],
                                  "sent_entries": rep["n_send_entries"]} if world > 1 else None,
                   "step_ms_rank0": step_stats},
        "roofline": roofline,
        "iter_only": {"value": nnzW_global * k_eff / (it_ms_med / 1e3) if k_eff else 0.0, "unit": UNIT,
                      "ms_per_iter": it_ms_med / max(k_eff, 1),
                      "GBps_vs_B_iter_rank0": it_bytes / (it_ms_med / max(k_eff, 1) / 1e3) / 1e9,
                      "frac_of_peak_rank0": it_bytes / (it_ms_med / max(k_eff, 1) / 1e3) / 1e9 / peak},
        "kernel_ms_per_step": {"spgemm": stats["spgemm_ms"] / nprof,
                               "stage1": stats["stage_ms"][0] / nprof,
                               "stage2": stats["stage_ms"][1] / nprof,
                               "scalar": stats["scalar_ms"] / nprof},
        "cpu_baseline": cpu, "e2e": e2e, "e2e_pipelined": e2e_pipe,
        "gpu_launches": launches_timed, "clocks": clocks,
        "energy": stats["E"], "k_done": k_eff,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
