#!/usr/bin/env python
"""Benchmark of the restricted-PCG energy-minimisation hot path on B200.

One STEP = one pass of the whole hot path over the
synthetic workload, through the C ABI: emin_setup from device-resident inputs
(validation, index prep, Alg. 2, r0, E0) -> emin_iterate(k) (k restricted-PCG
steps, CUDA graph) -> emin_energy -> emin_get_P (into a device buffer) ->
emin_destroy.  ``value`` = P-nonzero updates per second = nnz(W) * k * K /
(device time of the K timed steps), max over ranks.

Default workload: BASELINE config 3 (FV lognormal 128^3, 40 iterations), the
configuration BASELINE.json's metric ("... at 1/2/4/8 GPU") is quoted on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl reference]

--impl reference runs the CPU oracle (the tier's reference arm) on the host.
"""
from __future__ import annotations

import argparse
import json
import os
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


def log(*a):
    print(*a, file=sys.stderr, flush=True)


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


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.gpu = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [l.strip().split(",") for l in self.f.read().splitlines() if l.strip()]
        rows = [[c.strip() for c in r] for r in rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()),
                                   default=None)}


def run_reference(args, prob, rank):
    """The tier's reference arm: the CPU oracle as it stands, one thread."""
    if rank != 0:
        return None
    from oracle import Oracle
    k = prob.iters
    nnzW = prob.nnz_W
    steps, warm = args.steps, args.warmup
    # one step = one whole oracle pass (setup + k iterations + energy + P out);
    # bounded: fewer iterations per step if the full run would exceed ~4 min
    t0 = time.perf_counter()
    o = Oracle(prob)
    o.iterate(1)
    t_probe = time.perf_counter() - t0
    est = t_probe + (k - 1) * 0.25 * t_probe
    k_step = k
    budget = 240.0 / max(1, steps + warm)
    if est > budget:
        k_step = max(1, int(k * budget / est))
    times = []
    for s in range(warm + steps):
        t0 = time.perf_counter()
        o = Oracle(prob)
        kd, _ = o.iterate(k_step)
        o.energy()
        o.get_P()
        dt = time.perf_counter() - t0
        if s >= warm:
            times.append(dt)
    tot = sum(times)
    v = nnzW * k_step * steps / tot
    sample = (f"{WORKLOADS[args.config]}: full oracle step (setup + {k_step} of {k} iterations + "
              f"energy + P) per step, single-threaded C, {steps} timed steps")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * tot / steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOADS[args.config], "iters": k_step},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def cpu_baseline(prob, args):
    """Oracle timed on the host, bounded sample (one full step, ~10-20 s).
    For the large configs (4, 5) the sample is the same generator at a
    reduced size (the oracle needs ~1 min per iteration at 160^3)."""
    from oracle import Oracle
    if args.config in ("4", "5") and prob.n > 400000:
        from workloads.problems import make_config
        small = make_config(args.config, size=24)
        res = cpu_baseline(small, argparse.Namespace(config="small"))
        res["sample"] = f"same generator at 24^3 elements ({small.n} dofs): " + res["sample"]
        return res
    k = prob.iters
    t0 = time.perf_counter()
    o = Oracle(prob)
    t_setup = time.perf_counter() - t0
    # bound the sample to ~25 s of CPU work
    t1 = time.perf_counter()
    o.iterate(1)
    t_it = time.perf_counter() - t1
    k_s = max(1, min(k - 1, int(20.0 / max(t_it, 1e-3))))
    t1 = time.perf_counter()
    kd, _ = o.iterate(k_s)
    t_its = time.perf_counter() - t1
    o.energy()
    o.get_P()
    tot = time.perf_counter() - t0
    iters = 1 + kd
    v = prob.nnz_W * iters / tot
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"one oracle step of the same workload: setup ({t_setup:.2f} s) + {iters} of "
                      f"{k} iterations ({(t_it + t_its) / iters:.3f} s/it) + energy + P, "
                      f"single-threaded C (-O2), {tot:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("EMIN_BENCH_CONFIG", "3"))
    ap.add_argument("--impl", default="emin", choices=["emin", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true",
                    help="e2e without the copy/compute pipeline (host pointers into emin_setup, steps back to back)")
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

    from workloads.problems import make_config
    t0 = time.perf_counter()
    prob = make_config(args.config)
    log(f"[bench] generated {prob.name}: n={prob.n} nF={prob.n_F} nnzW={prob.nnz_W} "
        f"in {time.perf_counter() - t0:.1f}s")

    if args.impl == "reference":
        line = run_reference(args, prob, rank)
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0

    import torch
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

    stream = torch.cuda.current_stream()
    keys = ["A_rowptr", "A_col", "A_val", "is_coarse", "P_rowptr", "P_col", "P_val", "B", "Bc"]
    host = {k: getattr(prob, k) for k in keys}
    dev = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)).cuda()) for k, v in host.items()}
    # row partition (contiguous z-slabs balanced by nnz(W)); NCCL communicator
    comm = None
    rb, re_ = 0, prob.n
    if world > 1:
        from paper_2208_02995_b200.partition import partition_rows
        dims = prob.meta["dims"]
        plane = dims[0] * dims[1] * (3 if prob.block_size == 3 else 1)
        rb, re_ = partition_rows(prob.P_rowptr, prob.is_coarse, world, plane=plane)[rank]
        comm = E.nccl_comm_from_torch()
    nnzP = int(prob.P_rowptr[re_] - prob.P_rowptr[rb])
    out_dev = torch.empty(nnzP, dtype=torch.float64, device="cuda")
    k_it = prob.iters
    nnzW_global = prob.nnz_W

    key = None
    if args.precond == "sgs":
        from workloads.problems import sgs_key
        key = sgs_key(prob, args.sgs_key)
    host["sgs_key"] = key
    dev["sgs_key"] = None if key is None else torch.from_numpy(key).cuda()

    def setup(arrs):
        nv = prob.nv
        kk = arrs["sgs_key"]
        return E.emin_setup(prob.n, prob.nc, arrs["A_rowptr"][rb:re_ + 1], arrs["A_col"], arrs["A_val"],
                            arrs["is_coarse"], arrs["P_rowptr"][rb:re_ + 1], arrs["P_col"], arrs["P_val"],
                            nv, arrs["B"][rb:re_], arrs["Bc"], block_size=prob.block_size,
                            stagnation_rel=0.0, stream=stream.cuda_stream, nccl_comm=comm,
                            row_begin=rb, row_end=re_, precond=args.precond, start=args.start,
                            sgs_key=None if kk is None else kk[rb:re_])

    stats = {"launches": 0, "spgemm_ms": 0.0, "spgemm_n": 0, "stage_ms": [0.0, 0.0], "scalar_ms": 0.0,
             "k_done": 0, "E": None, "report": None}

    def step(arrs, out, profile):
        h = setup(arrs)
        if profile:
            E.emin_set_profiling(h, 1)
        E.emin_iterate(h, k_it)
        stats["E"] = E.emin_energy(h)
        E.emin_get_P(h, out)
        rep = E.emin_report(h)
        stats["launches"] += rep["launches"]
        stats["k_done"] = rep["k_total"]
        stats["report"] = rep
        if profile:
            kt = E.emin_kernel_times(h)
            stats["spgemm_ms"] += kt["spgemm"][0]
            stats["spgemm_n"] += kt["spgemm"][1]
            stats["stage_ms"][0] += kt["stage1"][0]
            stats["stage_ms"][1] += kt["stage2"][0]
            stats["scalar_ms"] += kt["scalar"][0]
        E.emin_destroy(h)

    # warm-up (untimed)
    for _ in range(args.warmup):
        step(dev, out_dev, True)
    for k in list(stats):
        if isinstance(stats[k], (int, float)) and k not in ("E",):
            stats[k] = 0 if isinstance(stats[k], int) else 0.0
    stats["stage_ms"] = [0.0, 0.0]

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- timed region: K whole-path steps, device-resident inputs
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    nprof = args.steps if args.profile_steps <= 0 else min(args.profile_steps, args.steps)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for it in range(args.steps):
            step(dev, out_dev, it >= args.steps - nprof)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = clk.summary()
    nnzW = stats["report"]["nnz_W"]
    nnzAFF = stats["report"]["nnz_AFF"]
    nF = stats["report"]["n_fine"]
    # updates actually performed: if the CG ever stopped before k_it (gamma or
    # y'Ky at zero), count only the steps it took (never the requested ones)
    k_eff = stats["k_done"] if 0 < stats["k_done"] < k_it else k_it
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
        ia.record(stream)
        E.emin_iterate(h, k_it)
        ib.record(stream)
        torch.cuda.synchronize()
        it_ms.append(ia.elapsed_time(ib))
    E.emin_destroy(h)
    it_ms_med = statistics.median(it_ms)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([it_ms_med], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        it_ms_med = float(t.item())

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
                "kernel": "masked SpGEMM + Pi_B (ŷ = Pi K y)", "peak_source": peak_src,
                "algorithmic_bytes_per_launch": sp_bytes,
                "avg_launch_ms": sp_avg_ms, "launches": stats["spgemm_n"],
                "share_of_step": (stats["spgemm_ms"] / nprof / (ms / args.steps)) if ms > 0 else None,
                "profiled_steps": nprof}

    # ---- e2e: same metric through the public API from HOST buffers (pinned):
    # every step copies its inputs host -> device and reads P back inside the
    # timed region.  Default: pipelined over two device buffer sets -- step
    # s+1's inputs are copied on a copy stream while step s computes (device
    # inputs to emin_setup), P goes back on a third stream (PCIe is full
    # duplex).  --e2e-serial: the plain C-ABI call with host pointers (the
    # library copies), steps back to back.
    e2e = None
    if not args.no_e2e:
        pin_t = {k: (None if v is None else torch.from_numpy(np.ascontiguousarray(v)).pin_memory())
                 for k, v in host.items()}
        pin = {k: (None if v is None else v.numpy()) for k, v in pin_t.items()}
        out_host_t = torch.empty(nnzP, dtype=torch.float64).pin_memory()
        out_host = out_host_t.numpy()
        h2d = sum(v.nbytes for v in pin.values() if v is not None)
        d2h = out_host.nbytes + 8
        n_e2e = max(1, args.steps // 2)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if args.e2e_serial:
            step(pin, out_host, False)
            barrier()
            torch.cuda.synchronize()
            ea.record(stream)
            for _ in range(n_e2e):
                step(pin, out_host, False)
            eb.record(stream)
        else:
            cs, ds = torch.cuda.Stream(), torch.cuda.Stream()
            bufs = [{k: (None if v is None else torch.empty(v.shape, dtype=v.dtype, device="cuda"))
                     for k, v in pin_t.items()} for _ in range(2)]
            outs = [torch.empty(nnzP, dtype=torch.float64, device="cuda") for _ in range(2)]
            ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
            h2d_done, in_free, out_free, p_ready = ev(), ev(), ev(), ev()

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
                h = setup(bufs[b])
                in_free[b].record(stream)
                E.emin_iterate(h, k_it)
                stats["E"] = E.emin_energy(h)
                if s >= 2:
                    stream.wait_event(out_free[b])
                E.emin_get_P(h, outs[b])
                p_ready[b].record(stream)
                with torch.cuda.stream(ds):
                    ds.wait_event(p_ready[b])
                    out_host_t.copy_(outs[b], non_blocking=True)
                    out_free[b].record(ds)
                E.emin_destroy(h)

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
        e_ms = ea.elapsed_time(eb)
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": nnzW_global * k_eff * n_e2e / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_ms / n_e2e, "steps": n_e2e,
               "mode": "serial (host pointers into the C ABI)" if args.e2e_serial else
                       "pipelined (H2D of step s+1 and D2H of step s overlap step s's compute; pinned host buffers)"}

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
        "scaling": "strong" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "iters_per_step": k_it, "nnz_W": nnzW_global,
                   "nnz_A_FF": nnzAFF, "n_F": nF, "nv": prob.nv,
                   "step": "emin_setup(device inputs) + emin_iterate(k) + emin_energy + emin_get_P + emin_destroy",
                   "l2": "inputs larger than L2 (per-iteration working set %.2f GB > 126 MB)" % (it_bytes / 1e9),
                   "parallelism": f"rows{world}" if world > 1 else "single GPU",
                   "kernel_path": E.KERNEL_PATHS.get(stats["report"]["kernel_path"]),
                   "precond": args.precond if args.precond == "jacobi" else
                   f"sgs ({args.sgs_key} order, {stats['report']['sgs_levels']} levels per sweep)",
                   "start": args.start},
        "roofline": roofline,
        "iter_only": {"value": nnzW_global * k_eff / (it_ms_med / 1e3), "unit": UNIT,
                      "ms_per_iter": it_ms_med / k_eff,
                      "GBps_vs_B_iter": it_bytes / (it_ms_med / k_eff / 1e3) / 1e9,
                      "frac_of_peak": it_bytes / (it_ms_med / k_eff / 1e3) / 1e9 / peak},
        "kernel_ms_per_step": {"spgemm": stats["spgemm_ms"] / nprof,
                               "stage1": stats["stage_ms"][0] / nprof,
                               "stage2": stats["stage_ms"][1] / nprof,
                               "scalar": stats["scalar_ms"] / nprof},
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": stats["launches"], "clocks": clocks,
        "energy": stats["E"], "k_done": stats["k_done"],
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
