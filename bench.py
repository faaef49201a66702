#!/usr/bin/env python
"""Benchmark of the AsyFLEXA hot path on B200 (BASELINE.json metric:
"block updates/sec and HBM GB/s vs peak; time to rel. objective err 1e-6").

One step = one asynchronous solve of BASELINE configs[1] (dense LASSO,
10000 x 20000 fp64, blocks of 32) from x0 = 0 until the relative objective
error (F - F*)/|F*| <= 1e-6, checked every few sweeps from the maintained
residual, followed by one stationarity evaluation (fresh residual, Eq. 5).
`value` = block updates / s over the timed steps (device time, CUDA events,
max over ranks); `ms_per_step` = time to rel. err 1e-6.

--impl reference times the oracle (oracle/, plain fp64 CPU) on the host cores
as the reference arm.  Multi-GPU: replicas only (independent instances, one
per rank, seeds base+rank) -- the method has no data-path exchange.
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

TARGET = 1e-6


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--schedule", default="cyclic", choices=["cyclic", "random"])
    ap.add_argument("--check-every", type=int, default=5, help="sweeps between objective checks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--panel-rows", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--workers", type=int, default=0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(P, schedule):
    return (f"configs[{P.meta.get('config_idx', '?')}] {P.name} {P.m}x{P.n} fp64 "
            f"{'CSC' if P.kind == 'csc' else 'dense col-major'}, blocks of {P.block}, "
            f"async {schedule}, gamma {P.gamma}")


def make_problem(idx, seed):
    from paper_1701_04900_b200 import inputs
    P = inputs.config(idx, seed=seed)
    P.meta["config_idx"] = idx
    return P


def bytes_per_sweep(P):
    """Algorithmic HBM bytes of one sweep of block updates:
    dense: A once (8 m n) + x read/write (16 n); CSC: vals+rowidx once
    (12 nnz) + colptr (8 n) + x read/write (16 n)."""
    if P.kind == "dense":
        return 8.0 * P.m * P.n + 16.0 * P.n
    return 12.0 * P.vals.size + 8.0 * P.n + 16.0 * P.n


class ClockSampler:
    def __init__(self, idx):
        self.idx, self.rows, self.proc = idx, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def traffic_for(P):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p)).get(P.name)
        if not d:
            return None
        return d["dram_bytes_per_sweep"] + d.get("dram_write_bytes_per_sweep", 0.0)  # read + write
    except Exception:
        return None


def reduce_over_ranks(ms: float, units: float, world: int, device="cpu"):
    """Replica timing (replicas only): the job time is the MAX of the
    ranks' device times, the work is the SUM of their units."""
    if world <= 1:
        return ms, units
    import torch
    import torch.distributed as dist
    mx = torch.tensor([ms], dtype=torch.float64, device=device)
    sm = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return mx.item(), sm.item()


# ----------------------------------------------------------------------------- oracle arms
def oracle_rate(P, seconds, x0=None):
    """Sequential Algorithm 1 (d = 0) of the oracle, as it stands, on host cores:
    block updates/s over a bounded sample (whole sweeps prefixes)."""
    from oracle import asyflexa_oracle as O
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        cores = os.cpu_count()
    x = None if x0 is None else x0.copy()
    done, t0 = 0, time.perf_counter()
    chunk = max(1, min(P.nblocks, 64))
    k = 0
    while time.perf_counter() - t0 < seconds:
        sched = [(k + i) % P.nblocks for i in range(chunk)]
        x, _ = O.run_sequential(P, P.gamma, sched, x0=x)
        k += chunk
        done += chunk
    dt = time.perf_counter() - t0
    return done / dt, cores, done, dt


# ----------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch
    from paper_1701_04900_b200 import asyflexa as A

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    P = make_problem(args.config, seed=rank)
    stream = torch.cuda.Stream()
    S = A.Solver(P, device=local, mem="device", stream=stream.cuda_stream)
    sched = A.ASY_SCHED_CYCLIC if args.schedule == "cyclic" else A.ASY_SCHED_RANDOM
    kw = dict(schedule=sched, seed=1234 + rank, panel_rows=args.panel_rows, stages=args.stages,
              workers=args.workers)

    # F* (untimed): run until the objective stops changing [PAPER.md:434]
    S.solve(sweeps=50, reset=True, **kw)
    Fprev = S.objective()
    for _ in range(200):
        S.solve(sweeps=25, **kw)
        F = S.objective()
        if abs(Fprev - F) <= 1e-15 * abs(F):
            break
        Fprev = F
    st_star = S.stationarity()
    Fstar = st_star.objective

    def solve_to_target(solver_kw_reset):
        updates, launches, kms, sweeps = 0, 0, 0.0, 0
        st = S.solve(sweeps=args.check_every, reset=True, **kw, **solver_kw_reset)
        while True:
            updates += st.block_updates
            launches += st.launches
            kms += st.kernel_ms
            sweeps += args.check_every
            if (st.objective - Fstar) / abs(Fstar) <= TARGET or sweeps >= 5000:
                break
            st = S.solve(sweeps=args.check_every, **kw)
        stat = S.stationarity()
        return updates, launches + 6, kms, sweeps, stat, st.kernel, st.delay, st.delay_observed

    for _ in range(args.warmup):
        solve_to_target({})
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    res = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            ev[i][0].record(stream)
            res.append(solve_to_target({}))
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    updates = sum(r[0] for r in res)
    launches = sum(r[1] for r in res)
    kernel_ms = sum(r[2] for r in res)
    sweeps = sum(r[3] for r in res)
    tot_ms_all, updates_all = reduce_over_ranks(tot_ms, updates, world, device=f"cuda:{local}")

    # roofline of the fused async kernel: algorithmic bytes / its device time
    hbm_peak, peak_kind = peaks()
    achieved = bytes_per_sweep(P) * sweeps / (kernel_ms * 1e-3) / 1e9
    traffic = traffic_for(P)
    if traffic is not None:
        traffic = traffic * args.check_every  # per launch (one launch = check_every sweeps), like `achieved`
    last_stat = res[-1][4]

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Sh = A.Solver(P, device=local, mem="host", stream=stream.cuda_stream, pinned=True)
        pstruct = Sh.problem_struct(P)  # pinned host arrays kept alive by Sh
        xout = torch.empty(P.n, dtype=torch.float64).pin_memory()
        h2d = (8 * P.m * P.n if P.kind == "dense" else 12 * P.vals.size + 8 * (P.n + 1)) + 8 * P.m + 8 * P.n

        def e2e_step():
            A.asy_set_problem(Sh.h, pstruct)
            u, checks = 0, 0
            st = Sh.solve(sweeps=args.check_every, reset=True, **kw)
            while True:
                u += st.block_updates
                checks += 1
                if (st.objective - Fstar) / abs(Fstar) <= TARGET or checks * args.check_every >= 5000:
                    break
                st = Sh.solve(sweeps=args.check_every, **kw)
            A.asy_get_x(Sh.h, xout.data_ptr(), A.ASY_MEM_HOST)
            return u, checks

        e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eu, echecks = 0, 0
        for _ in range(args.steps):
            u, c = e2e_step()
            eu += u
            echecks += c
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": eu / (ems * 1e-3), "unit": "block_updates/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(8 * P.n + 8 * echecks / args.steps),
               "ms_per_step": ems / args.steps}
        Sh.close()

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, cores, done, dt = oracle_rate(P, args.cpu_seconds)
        cpu = {"value": rate, "unit": "block_updates/s", "cores": cores, "kind": "oracle",
               "sample": f"{done} sequential block updates (Algorithm 1, d=0) of the same instance from x0=0, "
                         f"{dt:.1f} s, numpy/BLAS fp64"}

    if rank == 0:
        line = {
            "metric": "block updates/sec (async AsyFLEXA) | HBM GB/s vs peak | time to rel. objective err 1e-6",
            "value": updates_all / (tot_ms_all * 1e-3),
            "unit": "block_updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_ms_all / args.steps,
            "time_to_rel_err_1e-6_ms": tot_ms_all / args.steps,
            "sweeps_per_step": sweeps / args.steps,
            "hbm_gbs": achieved,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded recipe of BASELINE configs, DESIGN.md)",
            "config": {"workload": workload_name(P, args.schedule), "m": P.m, "n": P.n, "block": P.block,
                       "gamma": P.gamma, "lambda": P.lam, "check_every_sweeps": args.check_every,
                       "target_rel_err": TARGET, "parallelism": f"replicas x{world}",
                       "l2": "inputs larger than L2 (A = %.2f GB vs 126 MB)" % (bytes_per_sweep(P) / 1e9)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                         "traffic": traffic, "kernel": A.KERNEL_NAMES.get(res[-1][5], "?"),
                         "enforced_delay": res[-1][6],
                         "observed_delay": res[-1][7] if res[-1][7] >= 0 else None,
                         "bytes_per_sweep": bytes_per_sweep(P), "kernel_ms": kernel_ms / args.steps},
            "final": {"rel_err": (res[-1][4].objective - Fstar) / abs(Fstar), "mf_norm2": last_stat.mf_norm2,
                      "merit_inf": last_stat.merit_inf, "Fstar": Fstar, "Fstar_mf_norm2": st_star.mf_norm2},
            "clocks": clk.summary(),
            "gpu_launches": int(launches),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    S.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def run_reference(args, rank, world):
    if rank != 0:
        return
    P = make_problem(args.config, seed=0)
    rate0, cores, _, _ = oracle_rate(P, 2.0)  # warm-up + size the sample
    per_step = max(1.0, min(20.0, 60.0 / max(1, args.steps)))
    for _ in range(args.warmup):
        oracle_rate(P, min(2.0, per_step))
    t0 = time.perf_counter()
    done_all = 0
    for _ in range(args.steps):
        rate, cores, done, dt = oracle_rate(P, per_step)
        done_all += done
    tot = time.perf_counter() - t0
    value = done_all / tot
    line = {"impl": "reference",
            "metric": "block updates/sec (async AsyFLEXA) | HBM GB/s vs peak | time to rel. objective err 1e-6",
            "value": value, "unit": "block_updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(P, args.schedule), "m": P.m, "n": P.n, "block": P.block},
            "cpu_baseline": {"value": value, "unit": "block_updates/s", "cores": cores, "kind": "oracle",
                             "sample": f"{done_all} sequential block updates (Algorithm 1, d=0), "
                                       f"{per_step:.0f} s per step"},
            "e2e": {"value": value, "unit": "block_updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
