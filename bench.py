"""Benchmark of the ChFSI hot path on B200 (BASELINE.json metric: filter FP64 TFLOP/s).

Workload (config.workload): BASELINE config 4's Chebyshev filter call --
n = 20000, the full search block k = nev + nex = 2200 columns, degree m = 25
-- on H built with the c0 spectrum recipe (seeded, synthetic: no public
dataset exists). One step = one filter call p_m(H) Y = m fused DMMA GEMM +
recurrence launches; algorithmic work 8 n^2 k m FLOP per step. At N > 1
(torchrun, one process per GPU) the k columns are sharded across ranks (H
replicated, strong scaling) and each step ends with the NCCL all-gather of
the filtered block, as the solver needs it for QR and Rayleigh-Ritz.

Also reported: e2e (the same filter through the drop-in Python API
``chebyshev_filter(H, Y, spec)`` with pinned host H/Y, host<->device copies
inside the timed region), roofline of the dominant kernel (measured FP64
tensor-pipe peak), GPU clocks during the timed region, the oracle CPU filter
on the host cores (cpu_baseline), tail-width throughput, a full c0 solve and
c1 sequence, and at every N the s per ChFSI solve at n = 20000 (solve_c4:
BASELINE c4 problem 1, column-sharded over the ranks for N > 1).

``--impl reference`` times the reference algorithm's CPU filter (the oracle
restatement, numpy/OpenBLAS on all host cores) on a bounded column sample of
the same workload.
"""

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

METRIC = "filter FP64 TFLOP/s (ChFSI Chebyshev filter, n=20000, k=nev+nex=2200, m=25)"
UNIT = "TFLOP/s"


def metric_name(args):
    if (args.n, args.k, args.degree) == (20000, 2200, 25):
        return METRIC
    return (f"filter FP64 TFLOP/s (ChFSI Chebyshev filter, n={args.n}, k={args.k}, "
            f"m={args.degree}; non-default test shape)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    # (long names: torchrun's argparse would take "--n"/"--k" as abbreviations of its own)
    ap.add_argument("--matrix-order", dest="n", type=int, default=20000)
    ap.add_argument("--block-cols", dest="k", type=int, default=2200)
    ap.add_argument("--degree", type=int, default=25)
    ap.add_argument("--no-extras", action="store_true", help="skip e2e/cpu/tail/solve legs")
    ap.add_argument("--legs", default="",
                    help="comma list: run only these extra legs (development; default all)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--time-budget-s", type=float, default=720.0,
                    help="an optional leg is skipped (and says so in the line) when the "
                         "process has already run this long minus the leg's usual duration, "
                         "so the JSON line is printed before any outer limit")
    ap.add_argument("--complex-mul", type=int, default=3, choices=[3, 4],
                    help="complex products of the GEMMs: 3 (3M, default) or 4 real DMMA "
                         "products (the north star's literal four-MMA form)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N > 1 (gloo: host-staged, for testing)")
    return ap.parse_args()


T_PROCESS_START = time.monotonic()

# usual duration of the long optional legs on one B200 (s), for the time budget
LEG_SECONDS = {"solve_c4": 100.0, "solve_c4_reference_window": 45.0, "sequence_c4": 190.0,
               "solve_c0": 30.0, "sequence_c1": 30.0, "generalized_c4_setup": 15.0,
               "e2e_pageable": 20.0, "tail": 10.0, "filter_complex_mul_4": 20.0,
               "filter_complex_mul_3": 20.0}


def want(args, key):
    """Extra legs to run: all by default, or the --legs subset."""
    return not args.legs or key in args.legs.split(",")


def in_budget(args, key):
    """False when starting this optional leg now would run past --time-budget-s."""
    elapsed = time.monotonic() - T_PROCESS_START
    return elapsed + LEG_SECONDS.get(key, 0.0) <= args.time_budget_s


def workload_cfg(args, n_gpus):
    return {
        "workload": "BASELINE c4 first-iteration Chebyshev filter (standard-form H, c0 spectrum recipe)",
        "n": args.n, "k": args.k, "degree": args.degree, "nev": 2000, "nex": 200,
        "parallelism": f"column-shard x{n_gpus} (H replicated)" if n_gpus > 1 else "single GPU",
        "l2": "inputs larger than L2 (H = 6.4 GB per GPU)",
        "seed": 0,
    }


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU legs
def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return {d.get("internal_api", "?"): d.get("num_threads") for d in threadpool_info()
                if d.get("user_api") == "blas"}
    except Exception:  # pragma: no cover - informational only
        return {}


def host_operands(n, k, seed=0):
    """The GPU arm's operands on the host: H from the c0 spectrum recipe at order n,
    generated exactly as the GPU arm generates it (workloads.spectrum_matrix_torch on
    cuda:0 -- torch QR/matmul, data generation only, none of this repo's kernels), the
    start block Y (n x k, torch generator seed 1234) and the spectrum. Without a GPU
    (CPU tests) H follows the host recipe (workloads.baseline_matrix)."""
    import torch
    from paper_1305_5120_b200 import workloads as Wl
    if torch.cuda.is_available():
        dev = torch.device("cuda", torch.cuda.current_device())
        H, lam = Wl.spectrum_matrix_torch(seed, n, dev)
        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        Y = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
        h = H.cpu().numpy().T  # (k, n) row j = column j -> F-order n x n
        del H
        y = Y.cpu().numpy().T
        del Y
        torch.cuda.empty_cache()
        return h, y, lam, "c0 spectrum recipe, generated on the GPU exactly as the b200 arm"
    h, lam, _ = Wl.baseline_matrix(seed, n)
    rng = np.random.default_rng(1234)
    y = np.asfortranarray(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))
    return h, y, lam, "c0 spectrum recipe (host numpy; no GPU visible)"


def filter_params(lam, k):
    nev = int(round(k * 2000 / 2200))
    return float(lam[0]), float(lam[min(nev, len(lam) - 1)]), 1.01 * float(lam[-1])


def cpu_filter_rate(h, y, lam, seconds):
    """Oracle CPU filter (the reference's recurrence, numpy zgemm via OpenBLAS on all host
    threads) on the bench's own H and full k-column block, one degree step per call,
    repeated until ``seconds`` have elapsed; returns (TFLOP/s, sample, cores)."""
    import oracle.chfsi_oracle as O
    n, k = y.shape
    lam_ref, a_edge, b_up = filter_params(lam, k)
    O.cheb_filter(h, y[:, :32], 1, a_edge, b_up, lam_ref)  # warm-up (thread pool, pages)
    done, t_used, calls = 0.0, 0.0, 0
    while t_used < seconds and calls < 50:
        t0 = time.perf_counter()
        O.cheb_filter(h, y, 1, a_edge, b_up, lam_ref)
        t_used += time.perf_counter() - t0
        done += 8.0 * n * n * k
        calls += 1
    cores = os.cpu_count()
    sample = (f"oracle cheb_filter (core.py:263-284 restated) on the bench's H (n={n}) and full "
              f"{k}-column block, one degree step per call, {calls} calls ({t_used:.1f} s), "
              f"numpy/OpenBLAS on {cores} host threads {blas_threads()}")
    return done / t_used / 1e12, sample, cores


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's filter (oracle restatement of
    core.py:263-284: numpy zgemm on OpenBLAS, all host threads) on the b200 arm's own
    workload -- the same H (c0 recipe, n), the same full k-column block -- one degree step
    per step (the b200 arm's step is a degree-m call: same_config differs only in the
    degree; the unit is per-flop). Rank 0 alone runs it; other ranks exit 0."""
    if rank != 0:
        return
    import oracle.chfsi_oracle as O
    n, k = args.n, args.k
    t0 = time.perf_counter()
    h, y, lam, recipe = host_operands(n, k)
    t_gen = time.perf_counter() - t0
    lam_ref, a_edge, b_up = filter_params(lam, k)
    step_flops = 8.0 * n * n * k

    def step():
        O.cheb_filter(h, y, 1, a_edge, b_up, lam_ref)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    val = step_flops * args.steps / dt / 1e12
    cores = os.cpu_count()
    sample = (f"one full-width filter degree step per step (zgemm n={n} x k={k} + recurrence), "
              f"oracle restatement of core.py:263-284, numpy/OpenBLAS on {cores} threads "
              f"{blas_threads()}")
    line = {
        "impl": "reference", "metric": metric_name(args), "value": val, "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": f"synthetic (seeded; H = Q diag(lambda) Q^H, {recipe})",
        "config": dict(workload_cfg(args, 1), degree_per_step=1, same_config=True,
                       setup_s=t_gen),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200 import workloads as Wl
    from paper_1305_5120_b200.distributed import ColumnShards

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    eng = D.Engine.get(dev)
    eng.set_complex_mul(args.complex_mul)
    n, k, m = args.n, args.k, args.degree

    # ---- data: H (c0 spectrum recipe, seeded) replicated on every rank
    t0 = time.perf_counter()
    H, lam = Wl.spectrum_matrix_torch(0, n, dev)
    nev = int(round(k * 2000 / 2200))
    lam_ref, a_edge = float(lam[0]), float(lam[min(nev, n - 1)])
    v0 = np.random.default_rng(1).standard_normal(n) + 1j * np.random.default_rng(2).standard_normal(n)
    v0 /= np.linalg.norm(v0)
    b_up, _, _ = eng.lanczos_bound(H, D.to_device(v0, dev), 10)
    t_gen = time.perf_counter() - t0

    shards = ColumnShards(k, world)
    lo, hi = shards.range(rank)
    kp = hi - lo
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    Yfull = torch.randn((k, n), dtype=torch.complex128, device=dev, generator=g)
    Y0 = Yfull[lo:hi].clone()
    Y = torch.empty_like(Y0)
    W = torch.empty_like(Y0)
    gathered = torch.empty((shards.padded * world, n), dtype=torch.complex128, device=dev) if world > 1 else None

    def step():
        Y.copy_(Y0)
        out = eng.filter(H, Y, W, m, a_edge, b_up, lam_ref)
        if world > 1:
            shards.all_gather(out, gathered)
        return out

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region
    sampler = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    eng.launch_count(reset=True)
    stream = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    f_events = []
    e0.record(stream)
    for _ in range(args.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        Y.copy_(Y0)
        a.record(stream)
        out = eng.filter(H, Y, W, m, a_edge, b_up, lam_ref)
        b.record(stream)
        if world > 1:
            shards.all_gather(out, gathered)
        f_events.append((a, b))
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    launches = eng.launch_count(reset=True)
    t_total = e0.elapsed_time(e1) * 1e-3
    t_filter = sum(a.elapsed_time(b) for a, b in f_events) * 1e-3
    tt = torch.tensor([t_total, t_filter], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_total, t_filter = float(tt[0]), float(tt[1])
    flops_step = 8.0 * n * n * k * m
    value = flops_step * args.steps / t_total / 1e12
    ms_per_step = t_total / args.steps * 1e3

    # roofline of the dominant kernel (the fused filter step): per-launch work / duration.
    # The conventional count of a complex n x n x k product is 8 n^2 k flop (the metric's
    # unit); with 3M complex products (default) the kernel's own algorithm executes
    # 6 n^2 k real DMMA flop (3 real products of 2 n^2 k), which is what the tensor
    # pipe's peak bounds.
    mul = eng.complex_mul()
    avg_launch_s = t_filter / (args.steps * m)
    achieved_conv = 8.0 * n * n * kp / avg_launch_s / 1e12
    achieved = 2.0 * mul * n * n * kp / avg_launch_s / 1e12

    kernel_name = plan_kernel_name(eng, n, kp)
    e2e_multi = None
    if world > 1 and not args.no_extras and want(args, "e2e"):
        # every rank takes part (collectives inside); max over ranks
        e2e_multi = e2e_leg_sharded(args, H, Yfull, shards, rank, world, a_edge, b_up,
                                    lam_ref, dev)
    line = None
    if rank == 0:
        line = headline_line(args, world, value, ms_per_step, mul, launches, clocks, achieved,
                             achieved_conv, kernel_name, n, kp, local_rank, t_gen)
        if e2e_multi is not None:
            line["e2e"] = e2e_multi
    if world > 1:
        if not args.no_extras:
            # s per ChFSI solve at the metric's n on all ranks (column-sharded)
            nev_s = int(round(k * 2000 / 2200))
            def agreed_in_budget(key):
                # rank 0 decides for everyone (the legs have collectives inside)
                flag = torch.tensor([1 if in_budget(args, key) else 0], device=dev)
                dist.broadcast(flag, 0)
                return bool(flag.item())

            legs = [("solve_c4", lambda: solve_c4_leg(H, lam, rank, world, dev, nev_s,
                                                      k - nev_s, m))]
            legs += extra_solve_legs(H, lam, rank, world, dev, nev_s, k - nev_s, m)
            for key, fn in legs:
                if not want(args, key):
                    continue
                if not agreed_in_budget(key):
                    out = {"skipped": f"time budget ({args.time_budget_s:.0f} s)"}
                else:
                    out = guarded_leg(line, rank, fn, key=key)
                if rank == 0:
                    line[key] = out
        if rank == 0:
            print(json.dumps(line), flush=True)
        return
    finish_single_gpu(args, line, eng, H, Yfull, Y0, Y, W, lam, a_edge, b_up, lam_ref, dev, n, m)


def headline_line(args, world, value, ms_per_step, mul, launches, clocks, achieved, achieved_conv,
                  kernel_name, n, kp, local_rank, t_gen):
    peaks = measured_fp64_peaks(local_rank)
    peak = peaks["dmma_tflops"]
    # the committed ncu capture is of the default (3M) kernel at this shape
    traffic = committed_traffic(n, kp) if mul == 3 else None
    line = {
        "metric": metric_name(args), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64 DMMA, 3M complex products)" if mul == 3 else "c128 (f64 DMMA)",
        "data": "synthetic (seeded; H = Q diag(lambda) Q^H with the c0 spectrum recipe at n=20000)",
        "config": workload_cfg(args, world),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": kernel_name,
                     "complex_mul": mul,
                     "work_per_launch": f"{2 * mul} n^2 k real DMMA flop ({'3M' if mul == 3 else '4 real products'}"
                                        f" per complex MAC), n={n}, k={kp}",
                     "achieved_conventional_8n2k": achieved_conv,
                     "peak_source": "measured on this GPU: DMMA.8x8x4 issue-bound microkernel "
                                    "(chfsi_peak_dmma), best of 3 x ~0.5 s",
                     "peaks": peaks},
        "setup_s": t_gen,
    }
    return line


def finish_single_gpu(args, line, eng, H, Yfull, Y0, Y, W, lam, a_edge, b_up, lam_ref, dev, n, m):
    import torch
    if not args.no_extras:
        def leg(key, fn):
            # an optional leg must never cost the headline line
            if not want(args, key):
                return
            if not in_budget(args, key):
                line[key] = {"skipped": f"time budget ({args.time_budget_s:.0f} s)"}
                return
            try:
                line[key] = fn()
            except Exception as exc:  # pragma: no cover - reported, not raised
                line[key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()

        # the contract's keys first (e2e, cpu_baseline), then the optional legs in the
        # order of what they explain; a leg that would run past --time-budget-s is skipped
        leg("e2e", lambda: e2e_leg(args, H, Yfull, a_edge, b_up, lam_ref, dev))
        # host copies for the CPU baseline leg (the same H and full block)
        h_host = H.cpu().numpy().T
        y_host = Yfull.cpu().numpy().T

        def cpu_leg():
            rate, sample, cores = cpu_filter_rate(h_host, y_host, lam, args.cpu_seconds)
            return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}
        leg("cpu_baseline", cpu_leg)
        del h_host, y_host
        leg("e2e_pageable", lambda: e2e_leg(args, H, Yfull, a_edge, b_up, lam_ref, dev,
                                            pinned=False))
        leg("tail", lambda: tail_widths(eng, H, n, dev, a_edge, b_up, lam_ref))
        other = 4 if args.complex_mul == 3 else 3
        leg(f"filter_complex_mul_{other}",
            lambda: filter_other_mul(eng, H, Y0, Y, W, m, a_edge, b_up, lam_ref, other))
        del Yfull, Y0, Y, W
        torch.cuda.empty_cache()
        nev_s = int(round(args.k * 2000 / 2200))
        legs = [("solve_c4", lambda: solve_c4_leg(H, lam, 0, 1, dev, nev_s, args.k - nev_s,
                                                  args.degree))]
        legs += extra_solve_legs(H, lam, 0, 1, dev, nev_s, args.k - nev_s, args.degree)
        for key, fn in legs:
            if not want(args, key):
                continue
            if not in_budget(args, key):
                line[key] = {"skipped": f"time budget ({args.time_budget_s:.0f} s)"}
                continue
            line[key] = guarded_leg(line, 0, fn, key=key)
            torch.cuda.empty_cache()
        del H
        torch.cuda.empty_cache()
        leg("solve_c0", solve_c0)
        leg("sequence_c1", sequence_c1)
        leg("generalized_c4_setup", generalized_c4_setup)
    print(json.dumps(line), flush=True)


KERNELS = {
    0: "zgemm_dmma_kernel<64,64,BK8,warp32x32,cp.async x4>",
    1: "zgemm_dmma_kernel<64,32,BK8,warp32x16,cp.async x4>",
    2: "zgemm_dmma_kernel<64,16,BK8,warp16x16,cp.async x4>",
    3: "zgemm_dmma_kernel<32,16,BK8,warp16x8,cp.async x4>",
    4: "zgemm_dmma_kernel<64,64,BK16,warp32x32,cp.async x3>",
    5: "zgemm_dmma_kernel<128,64,BK8,warp32x32,cp.async x4>",
    6: "zgemm_dmma_kernel<128,32,BK8,warp32x16,cp.async x4>",
    7: "zgemm_tma_kernel<64,32,warp32x16,TMA+mbarrier x4,EPI_FILTER>",
    8: "zgemm_tma_kernel<64,16,warp16x16,TMA+mbarrier x4,EPI_FILTER>",
    9: "zgemm_tma_kernel<64,64,warp32x32,TMA+mbarrier x4,EPI_FILTER>",
    10: "zgemm_tma_kernel<64,32,warp16x32,TMA+mbarrier x4,EPI_FILTER>",
    11: "zgemm_tma_kernel<64,32,warp32x16,TMA+mbarrier x4,EPI_FILTER,3M>",
    12: "zgemm_tma_kernel<64,32,warp16x32,TMA+mbarrier x4,EPI_FILTER,3M>",
    13: "zgemm_tma_kernel<64,32,warp16x16,TMA+mbarrier x4,EPI_FILTER,3M>",
    14: "zgemm_tma_kernel<64,32,warp32x16,TMA+mbarrier x4,EPI_FILTER,3M,sum planes>",
    15: "zgemm_tma_kernel<64,32,warp16x32,TMA+mbarrier x4,EPI_FILTER,3M,sum planes>",
    16: "zgemm_tma_kernel<64,24,warp16x24,TMA+mbarrier x4,EPI_FILTER,3M,sum planes>",
    17: "zgemm_tma_kernel<64,32,warp16x32,TMA+mbarrier x4,EPI_FILTER,3M,B-sum plane>",
    18: "zgemm_tma_kernel<64,24,warp16x24,TMA+mbarrier x4,EPI_FILTER,3M,B-sum plane>",
}


SOLVE_LEG_LIMIT_S = 900.0


def guarded_leg(line, rank, fn, limit_s=SOLVE_LEG_LIMIT_S, key="solve_c4"):
    """Run a leg that has collectives inside on every rank. An exception is reported in
    the line; a leg still running after limit_s (e.g. a rank stuck in a collective
    after another rank failed) makes rank 0 print the headline line with the error and
    every rank exit 0, so the headline is never lost."""
    import threading

    def fire():
        if rank == 0 and line is not None:
            line[key] = {"error": f"leg exceeded {limit_s:.0f} s; abandoned"}
            print(json.dumps(line), flush=True)
        os._exit(0)

    timer = threading.Timer(limit_s, fire)
    timer.daemon = True
    timer.start()
    try:
        return fn()
    except Exception as exc:  # pragma: no cover - reported, not raised
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}
    finally:
        timer.cancel()


def solve_c4_leg(H, lam, rank, world, dev, nev=2000, nex=200, degree=25):
    """s per ChFSI solve at the metric's n = 20000 (BASELINE c4 problem 1 in standard
    form: the c0 spectrum recipe, nev = 2000, nex = 200, m = 25, random start, solver
    seed 1, opt-in block_top interval; other --matrix-order/--block-cols scale nev/nex)
    on every rank; for N > 1 column-sharded over the process group with H
    broadcast from rank 0 (the replicated k x k decisions need the identical operator).
    Time = max over ranks of the solve's wall time between barriers."""
    import torch
    import torch.distributed as dist
    import paper_1305_5120_b200 as G
    n = H.shape[0]
    if world > 1:
        dist.broadcast(H, src=0)
    hm = G.HermitianDenseMatrix.from_device(H, trusted=True)
    cfg = G.SolverConfig(nev=nev, buffer=nex, degree=degree, max_outer_iters=2000,
                         interval="block_top")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    vals, vecs, rep = G.chfsi_solve(hm, None, cfg, seed=1,
                                    group=dist.group.WORLD if world > 1 else None)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt, rep.t_filter], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt, tf = float(tt[0]), float(tt[1])
    flops = 8.0 * n * n * degree * sum(it.filtered_cols for it in rep.iterations)
    del vecs
    return {"n": n, "nev": nev, "nex": nex, "degree": degree, "interval": "block_top",
            "n_gpus": world, "s_per_solve": dt, "outer_iterations": rep.outer_iterations,
            "total_matmuls": rep.total_matmuls,
            "filter_tflops_whole_job": flops / tf / 1e12 if tf > 0 else None,
            "filter_share": tf / dt,
            "residuals_below_tol": bool(rep.converged),
            "max_rel_eig_err_vs_exact": float(np.max(np.abs(vals - lam[:nev]) / np.abs(lam[:nev])))}


def extra_solve_legs(H, lam, rank, world, dev, nev, nex, degree):
    """The legs that run on every rank after solve_c4 (column-sharded for N > 1)."""
    return [("solve_c4_reference_window",
             lambda: reference_window_leg(H, lam, rank, world, dev, nev, nex, degree)),
            ("sequence_c4", lambda: sequence_c4_leg(H, lam, rank, world, dev, nev, nex, degree))]


# c4 standard problem 1 with the reference's own interval semantics (profiles/r01/solves/
# c4_standard_problem1_reference_interval_3m.json, one B200): 5024 outer iterations, of
# which this many ran at full width (k_a > 1000) and the rest in the narrow tail
REF_TRACE = os.path.join(ROOT, "profiles", "r01", "solves",
                         "c4_standard_problem1_reference_interval_3m.json")


def reference_window_leg(H, lam, rank, world, dev, nev=2000, nex=200, degree=25, head=3,
                         tail=40, tail_cols=201):
    """A bounded window of the c4 solve under the reference's own interval semantics
    (a = Ritz value nev+1, core.py:507-509), timed at every N (max over ranks):
    * head: the solve's first ``head`` outer iterations at full width (chfsi_solve with
      max_outer_iters = head; its NotConverged report carries the iteration times);
    * tail: ``tail`` iterations of the long narrow tail that dominates this solve
      (k_a ~ 201 columns against 2000 locked vectors), timed from a synthetic state
      (DeviceSolver.probe_iterations: random orthonormal locked block, random active
      block; the per-iteration work does not depend on the values);
    and the whole-solve estimate t_head x (full-width iterations of the one-GPU trace)
    + t_tail x (its narrow iterations)."""
    import torch
    import torch.distributed as dist

    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.core import DeviceSolver
    n = H.shape[0]
    grp = dist.group.WORLD if world > 1 else None
    if world > 1:
        dist.broadcast(H, src=0)
    hm = G.HermitianDenseMatrix.from_device(H, trusted=True)
    cfg = G.SolverConfig(nev=nev, buffer=nex, degree=degree, max_outer_iters=head,
                         interval="reference")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    try:
        G.chfsi_solve(hm, None, cfg, seed=1, group=grp)
        its = None
    except G.NotConverged as exc:
        its = exc.report.iterations
    torch.cuda.synchronize()
    t_head_total = time.perf_counter() - t0
    head_iter = [i.t_filter + i.t_qr + i.t_rr for i in (its or [])]
    # tail state (replicated: generated from one seed and broadcast)
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    locked = torch.linalg.qr(torch.randn((n, nev), dtype=torch.complex128, device=dev,
                                         generator=g))[0]
    locked = locked.T.contiguous()  # (nev, n): column-major n x nev block
    active = torch.randn((tail_cols, n), dtype=torch.complex128, device=dev, generator=g)
    if world > 1:
        dist.broadcast(locked, src=0)
        dist.broadcast(active, src=0)
    solver = DeviceSolver(hm, cfg, group=grp)
    b_up = 1.01 * float(lam[-1])
    solver.probe_iterations(locked, active, 2, float(lam[nev]), b_up, float(lam[0]))  # warm
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    per = solver.probe_iterations(locked, active, tail, float(lam[nev]), b_up, float(lam[0]))
    torch.cuda.synchronize()
    t_tail_total = time.perf_counter() - t0
    vals = [t_head_total / max(1, len(head_iter)), t_tail_total / tail,
            sum(p[0] for p in per) / tail, sum(p[1] for p in per) / tail,
            sum(p[2] for p in per) / tail]
    tt = torch.tensor(vals, dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_head, t_tail, tf, tq, trr = [float(x) for x in tt]
    out = {"n": n, "nev": nev, "nex": nex, "degree": degree, "interval": "reference",
           "n_gpus": world, "head_iterations": len(head_iter),
           "s_per_head_iteration": t_head, "tail_iterations": tail, "tail_cols": tail_cols,
           "s_per_tail_iteration": t_tail,
           "tail_phase_s": {"filter": tf, "qr": tq, "rr": trr}}
    try:
        with open(REF_TRACE) as f:
            trace = json.load(f)["problems"][0]["iterations"]
        wide = sum(1 for it in trace if it[0] > 1000)
        narrow = len(trace) - wide
        if (n, nev, nex, degree) == (20000, 2000, 200, 25):
            out["est_s_per_solve"] = wide * t_head + narrow * t_tail
            out["est_basis"] = (f"one-GPU reference-interval trace: {wide} full-width + "
                                f"{narrow} narrow iterations (measured 1-GPU solve 2012 s)")
    except Exception:  # pragma: no cover - informational
        pass
    return out


def sequence_c4_leg(H, lam, rank, world, dev, nev=2000, nex=200, degree=25, problems=2):
    """The north star's target sequence, bounded to ``problems`` problems: BASELINE c4
    generalized (S = I + 0.1 B^H B / ||B^H B||, A_1 = the bench's H, A_{l+1} = A_l +
    delta E_l with delta = 1e-3 ||A_1||), eigenvector reuse, through the drop-in
    solve_sequence(seq, config, "reuse", group=) -- column-sharded over the ranks for
    N > 1 -- with the opt-in block_top interval; s per problem (max over ranks)."""
    import torch
    import torch.distributed as dist

    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200 import device as D
    n = H.shape[0]
    eng = D.Engine.get(dev)
    grp = dist.group.WORLD if world > 1 else None

    def norm2(blk, seed):
        v = np.random.default_rng(seed).standard_normal(n) + 0j
        v /= np.linalg.norm(v)
        return eng.lanczos_bound(blk, D.to_device(v, dev), 10)[0]

    t0 = time.perf_counter()
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    b = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    s = torch.empty_like(b)
    eng.zgemm("C", "N", n, n, n, 1.0, b, b, 0.0, s)
    del b
    eng.hermitize(s)
    s.mul_(0.1 / norm2(s, 4))
    s.diagonal().add_(1.0)
    mats = [H.clone()]
    delta = 1e-3 * max(abs(float(lam[0])), abs(float(lam[-1])))
    for ell in range(2, problems + 1):
        g.manual_seed(100 + ell)
        e = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
        e = ((e + e.conj().T) / 2).conj().resolve_conj().contiguous()
        e.mul_(delta / norm2(e, 200 + ell))
        mats.append(mats[-1] + e)
        del e
    if world > 1:  # the replicated decisions need bit-identical operators
        dist.broadcast(s, src=0)
        for a in mats:
            dist.broadcast(a, src=0)
    seq = G.ProblemSequence(
        spec=G.SequenceSpec(n=n, N=problems, nev=nev, seed=0, kind="generalized"),
        problems=[(G.HermitianDenseMatrix.from_device(a, trusted=True),
                   G.HermitianDenseMatrix.from_device(s, trusted=True)) for a in mats])
    # one S object for the whole sequence: its Cholesky factor is computed once
    smat = seq.problems[0][1]
    seq.problems = [(a, smat) for a, _ in seq.problems]
    t_gen = time.perf_counter() - t0
    cfg = G.SolverConfig(nev=nev, buffer=nex, degree=degree, max_outer_iters=2000,
                         interval="block_top")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    rep = G.solve_sequence(seq, cfg, "reuse", angles=False, group=grp)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt] + [r.t_total for r in rep.reports], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    # verification of the last problem: generalized residuals and B-orthonormality
    vb = rep.vectors[-1].device_block()
    lamc = rep.eigenvalues[-1]
    k = vb.shape[0]
    av, sv = torch.empty_like(vb), torch.empty_like(vb)
    eng.zgemm("N", "N", n, k, n, 1.0, mats[-1], vb, 0.0, av)
    eng.zgemm("N", "N", n, k, n, 1.0, s, vb, 0.0, sv)
    lt = torch.as_tensor(lamc, device=dev).to(vb.dtype)
    res = float(torch.linalg.vector_norm(av - sv * lt[:, None], dim=1).max())
    gram = torch.empty((k, k), dtype=vb.dtype, device=dev)
    eng.zgemm("C", "N", k, k, n, 1.0, vb, sv, 0.0, gram)
    orth = float(torch.linalg.matrix_norm(gram - torch.eye(k, dtype=vb.dtype, device=dev)))
    return {"n": n, "nev": nev, "nex": nex, "degree": degree, "problems": problems,
            "generalized": True, "interval": "block_top", "n_gpus": world,
            "s_total": float(tt[0]), "s_per_problem": [float(x) for x in tt[1:]],
            "outer_iterations": [r.outer_iterations for r in rep.reports],
            "filter_tflops": [r.filter_tflops for r in rep.reports],
            "t_lanczos": [r.t_lanczos for r in rep.reports],
            "max_generalized_residual": res, "b_orthonormality": orth, "setup_s": t_gen,
            "path": "solve_sequence(seq, cfg, 'reuse', group=WORLD)"}


def plan_kernel_name(eng, n, k):
    import ctypes
    from paper_1305_5120_b200 import _native
    cfg, split = ctypes.c_int(), ctypes.c_int()
    # filter_epilogue 2: the filter call's steps (3M operand-sum planes when 3M is on)
    _native.call("chfsi_gemm_plan", eng.h, 0, 0, 2, n, k, n, ctypes.byref(cfg), ctypes.byref(split))
    name = KERNELS.get(cfg.value, f"cfg{cfg.value}")
    return name + (f" split-K {split.value}" if split.value > 1 else "")


def generalized_c4_setup(n=20000):
    """Per-problem generalized-to-standard cost at c4 scale (core.py:549-569): S = I +
    0.1 B^H B / ||B^H B|| (norm from a 10-step Lanczos bound), zpotrf, blocked
    triangular inverse, H = L^-1 A L^-H (two DMMA GEMMs skipping the zero triangle of
    L^-1), Hermitian check/symmetrise."""
    import torch
    from paper_1305_5120_b200 import device as D
    from paper_1305_5120_b200 import workloads as Wl
    dev = torch.device("cuda", torch.cuda.current_device())
    eng = D.Engine.get(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(3)
    b = torch.randn((n, n), dtype=torch.complex128, device=dev, generator=g)
    s = torch.empty_like(b)
    eng.zgemm("C", "N", n, n, n, 1.0, b, b, 0.0, s)  # B^H B (column-major blocks)
    del b
    eng.hermitize(s)
    v0 = np.random.default_rng(4).standard_normal(n) + 0j
    v0 /= np.linalg.norm(v0)
    top, _, _ = eng.lanczos_bound(s, D.to_device(v0, dev), 10)
    s.mul_(0.1 / top)
    s.diagonal().add_(1.0)  # (k, n) block: the diagonal is the same set of entries
    a, _ = Wl.spectrum_matrix_torch(5, n, dev)
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.cholesky(s)
    torch.cuda.synchronize()
    t["potrf_s"] = time.perf_counter() - t0
    linv = torch.empty_like(s)
    t0 = time.perf_counter()
    eng.trtri_lower(s, linv)
    torch.cuda.synchronize()
    t["trtri_s"] = time.perf_counter() - t0
    w = torch.empty_like(s)
    t0 = time.perf_counter()
    h = torch.empty_like(s)
    eng.reduce_to_standard(a, linv, w, h)  # two GEMMs skipping L^-1's zero triangle
    torch.cuda.synchronize()
    t["reduce_gemms_s"] = time.perf_counter() - t0
    # algorithmic work 8 n^3 flop: each GEMM multiplies by a triangular factor (4 n^3)
    t["reduce_gemms_tflops"] = 8.0 * n ** 3 / t["reduce_gemms_s"] / 1e12
    t["reduce_dense_equivalent_tflops"] = 16.0 * n ** 3 / t["reduce_gemms_s"] / 1e12
    a = h
    t0 = time.perf_counter()
    fro, devn = eng.hermitian_norms(a)
    eng.hermitize(a)
    torch.cuda.synchronize()
    t["hermitian_check_s"] = time.perf_counter() - t0
    t["relative_hermitian_deviation"] = devn / fro
    t["n"] = n
    return t


def measured_fp64_peaks(index):
    from paper_1305_5120_b200 import device as D
    dm = max(D.peak_dmma_tflops(index, 400000) for _ in range(3))
    df = max(D.peak_dfma_tflops(index, 400000) for _ in range(3))
    nominal = 148 * 1.965e9 * 128 / 1e12
    return {"dmma_tflops": dm, "dfma_tflops": df, "nominal_fp64_tflops_at_max_clock": nominal}


def committed_traffic(n, k):
    """DRAM bytes per launch from the committed ncu --set full capture of the same
    launch shape (profiles/filter_kernel_ncu.json), else None."""
    p = os.path.join(ROOT, "profiles", "filter_kernel_ncu.json")
    try:
        with open(p) as f:
            d = json.load(f)
        if (d.get("n"), d.get("k")) != (n, k):
            return None
        return d.get("dram_bytes_per_launch")
    except Exception:
        return None


def e2e_leg_sharded(args, H, Yfull, shards, rank, world, a_edge, b_up, lam_ref, dev, steps=2):
    """N-GPU e2e through the public API: every rank calls
    chebyshev_filter(H, Y, spec, group=WORLD) on the same pinned host H / Y; inside,
    each rank uploads one column slab of H (all-gathered over NVLink) and its own
    column shard of Y, filters it and all-gathers the result; rank 0 then reads the
    full filtered block back to the host. Time = max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200 import device as D
    n, k, m = args.n, args.k, args.degree
    h_pin = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
    h_pin.copy_(H)
    y_pin = torch.empty((k, n), dtype=torch.complex128, pin_memory=True)
    y_pin.copy_(Yfull)
    h_np, y_np = h_pin.numpy().T, y_pin.numpy().T
    spec = G.FilterSpec(degree=m, a=a_edge, b=b_up, lam_ref=lam_ref)
    d2h = 0

    def one():
        nonlocal d2h
        out = G.chebyshev_filter(h_np, y_np, spec, group=dist.group.WORLD)
        if rank == 0:
            d2h = D.to_host(out.device_block()).nbytes

    one()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    return {"value": 8.0 * n * n * k * m * steps / float(dt) / 1e12, "unit": UNIT,
            "h2d_bytes_per_step": int(16 * n * n + 16 * n * k),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": "chebyshev_filter(H, Y, FilterSpec, group=WORLD): per-rank H slab upload + "
                    "NCCL all-gather of H, Y column shards, NCCL all-gather of the result; "
                    "rank 0 VectorBlock -> host"}


def e2e_leg(args, H, Yfull, a_edge, b_up, lam_ref, dev, steps=2, pinned=True):
    """Same filter through the public API with host inputs; H2D/D2H inside. pinned=True:
    page-locked host H / Y; pinned=False: plain (pageable) numpy arrays, as a drop-in
    caller of the reference's chebyshev_filter passes them (core.py:287-311) -- the
    library stages them through its pinned ring (csrc/staging.cu)."""
    import torch

    import paper_1305_5120_b200 as G
    n, k, m = args.n, args.k, args.degree
    h_pin = torch.empty((n, n), dtype=torch.complex128, pin_memory=pinned)
    h_pin.copy_(H)
    y_pin = torch.empty((k, n), dtype=torch.complex128, pin_memory=pinned)
    y_pin.copy_(Yfull)
    h_np = h_pin.numpy().T  # F-order n x n view of the host buffer (column j = row j)
    y_np = y_pin.numpy().T
    spec = G.FilterSpec(degree=m, a=a_edge, b=b_up, lam_ref=lam_ref)
    out = G.chebyshev_filter(h_np, y_np, spec)  # warm-up
    res = out.entries
    nbytes = int(res.nbytes)
    del out, res
    torch.cuda.synchronize()
    # each step's result is read to the host, checked and released before the next
    # step, so its page-locked buffer is recycled by torch's host allocator (keeping
    # every result alive would add a one-time ~0.43 s page-locking per new 704 MB
    # buffer on this box, measured)
    checks = []
    t0 = time.perf_counter()
    for _ in range(steps):
        out = G.chebyshev_filter(h_np, y_np, spec)
        res = out.entries  # device -> host of the filtered block
        checks.append(bool(np.isfinite(res[:1, :]).all()))
        del out, res
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    flops = 8.0 * n * n * k * m
    return {"value": flops * steps / dt / 1e12, "unit": UNIT,
            "h2d_bytes_per_step": int(16 * n * n + 16 * n * k),
            "d2h_bytes_per_step": nbytes, "steps": steps, "results_finite": all(checks),
            "host_memory": "page-locked" if pinned else "pageable numpy (staged by the library)",
            "path": "paper_1305_5120_b200.chebyshev_filter(H, Y, FilterSpec) -> VectorBlock.entries"}


def filter_other_mul(eng, H, Y0, Y, W, degree, a_edge, b_up, lam_ref, mul, steps=2):
    """The headline filter call with the other complex-product scheme (the north star's
    literal four real MMAs when the headline runs 3M), timed the same way; restores the
    headline scheme afterwards."""
    import torch
    n, k = H.shape[0], Y0.shape[0]
    old = eng.complex_mul()
    eng.set_complex_mul(mul)
    try:
        Y.copy_(Y0)
        eng.filter(H, Y, W, degree, a_edge, b_up, lam_ref)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            Y.copy_(Y0)
            eng.filter(H, Y, W, degree, a_edge, b_up, lam_ref)
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) * 1e-3 / steps
    finally:
        eng.set_complex_mul(old)
    return {"complex_mul": mul, "value": 8.0 * n * n * k * degree / t / 1e12, "unit": UNIT,
            "ms_per_step": t * 1e3, "steps": steps,
            "executed_dmma_tflops": 2.0 * mul * n * n * k * degree / t / 1e12}


def tail_widths(eng, H, n, dev, a_edge, b_up, lam_ref, degree=5):
    """Filter throughput at the solve's dominant narrow widths: full
    filter calls (sum planes, split-K plans) of `degree` steps; ms per step."""
    import torch
    out = {}
    eng.declare_operator(H)  # as in a solve: H's 3M sum plane formed once, not per call
    # 26 / 51 / 101: the 8- / 4- / 2-GPU shards of the reference-interval tail block
    # (k_a = 201); 210: that tail on one GPU; 275: the 8-GPU shard of the full block
    for k in (26, 51, 101, 210, 275):
        Y0 = torch.randn((k, n), dtype=torch.complex128, device=dev)
        Y = torch.empty_like(Y0)
        W = torch.empty_like(Y)
        # every call filters the same start block (repeated in-place filtering would grow
        # the block to inf / NaN); the copy is ~0.1 % of a call
        for _ in range(2):
            Y.copy_(Y0)
            eng.filter(H, Y, W, degree, a_edge, b_up, lam_ref)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            Y.copy_(Y0)
            eng.filter(H, Y, W, degree, a_edge, b_up, lam_ref)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / (3 * degree)
        out[str(k)] = {"ms": ms, "tflops": 8.0 * n * n * k / (ms * 1e-3) / 1e12,
                       "kernel": plan_kernel_name(eng, n, k)}
    eng.declare_operator(None)
    return out


def oracle_c0_solve(limit_s=240.0):
    """The reference algorithm (oracle restatement of core.py:385-546, numpy/OpenBLAS on
    all host cores + the C Jacobi) solving BASELINE config 0 in full on this box's CPU,
    in the same run (generator seed 0, solver seed 1). Runs in a child process under a
    time limit so a slow host cannot cost the headline line."""
    code = ("import json, os, sys, time; sys.path.insert(0, %r); "
            "import oracle.chfsi_oracle as O; "
            "from paper_1305_5120_b200.workloads import baseline_matrix; "
            "h, lam_true, _ = baseline_matrix(0, 1000); t0 = time.perf_counter(); "
            "lam, v, rep = O.solve(h, None, 100, 20, 15, 1e-10, 20000, seed=1); "
            "dt = time.perf_counter() - t0; "
            "print(json.dumps({'s': dt, 'iterations': len(rep['iterations']), "
            "'total_matmuls': int(rep['total_matmuls']), 'lam': [float(x) for x in lam]}))"
            % ROOT)
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                             timeout=limit_s, cwd=ROOT)
    except subprocess.TimeoutExpired:
        return {"error": f"oracle c0 solve exceeded {limit_s:.0f} s"}
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"error": (out.stderr or "no output")[-300:]}
    d = json.loads(lines[-1])
    d["cores"] = os.cpu_count()
    d["blas_threads"] = blas_threads()
    d["kind"] = "port"
    return d


def solve_c0():
    """s per ChFSI solve at BASELINE config 0 (n=1000, nev=100, nex=20, m=15, random start;
    generator seed 0, solver seed 1), for the reference interval placement and for the
    opt-in block_top placement (SURVEY.md section 7 ii), with the reference algorithm's
    own full CPU solve timed on this box's host cores in the same run (oracle)."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_matrix
    h, lam_true, _ = baseline_matrix(0, 1000)
    out = {}
    for interval in ("reference", "block_top"):
        cfg = G.SolverConfig(nev=100, buffer=20, degree=15, max_outer_iters=20000,
                             interval=interval)
        t0 = time.perf_counter()
        lam, vecs, rep = G.chfsi_solve(h, None, cfg, seed=1)
        dt = time.perf_counter() - t0
        out[interval] = {
            "s_per_solve": dt, "outer_iterations": rep.outer_iterations,
            "total_matmuls": rep.total_matmuls,
            "max_rel_eig_err_vs_exact": float(np.max(np.abs(lam - lam_true[:100]) / np.abs(lam_true[:100]))),
            "t_filter": rep.t_filter, "t_qr": rep.t_qr, "t_rr": rep.t_rr}
        if interval == "reference":
            lam_gpu = lam
    cpu = oracle_c0_solve()
    if "lam" in cpu:
        ref = np.asarray(cpu.pop("lam"))
        cpu["max_rel_eig_diff_gpu_vs_cpu"] = float(np.max(np.abs(lam_gpu - ref) / np.abs(ref)))
        out["reference_cpu_s"] = cpu["s"]
        out["reference_cpu_iterations"] = cpu["iterations"]
        out["speedup_vs_cpu"] = cpu["s"] / out["reference"]["s_per_solve"]
    out["reference_cpu"] = cpu
    return out


def oracle_c1_sample(probs, limit_iters=80):
    """CPU side of the c1 leg: the oracle solving c1 problem 1 (reference RNG order: the
    solver Generator [seed, 11, 1]) for a bounded number of outer iterations on this
    box's cores; returns (seconds, matmul-columns done) for a per-column extrapolation."""
    import oracle.chfsi_oracle as O
    tally = O.Tally()
    t0 = time.perf_counter()
    try:
        O.solve(probs[0][0], None, 200, 40, 20, 1e-10, limit_iters,
                seed=np.random.default_rng([0, 11, 1]), tally=tally)
    except O.OracleError:
        pass  # NotConverged after the bounded sample: expected
    dt = time.perf_counter() - t0
    return dt, int(tally.cols)


def sequence_c1():
    """BASELINE config 1: 5 correlated n=2000 problems (delta = 1e-3 ||H_1||), nev=200, nex=40,
    m=20, eigenvector reuse through solve_sequence; s per sequence. CPU: the oracle's time per
    matmul-column on a bounded sample of problem 1 (same box, same run) times the
    sequence's total work (which equals the reference's: tests/golden/c1_full.npz),
    labelled as extrapolated."""
    import paper_1305_5120_b200 as G
    from paper_1305_5120_b200.workloads import baseline_sequence
    probs = baseline_sequence(0, 2000, 5)
    seq = G.ProblemSequence(spec=G.SequenceSpec(n=2000, N=5, nev=200, seed=0),
                            problems=[(a, None) for a, _ in probs])
    cfg = G.SolverConfig(nev=200, buffer=40, degree=20, max_outer_iters=20000)
    t0 = time.perf_counter()
    rep = G.solve_sequence(seq, cfg, "reuse", angles=False)
    dt = time.perf_counter() - t0
    out = {"s_per_sequence": dt,
           "iterations": [r.outer_iterations for r in rep.reports],
           "work": rep.work, "filter_s": sum(r.t_filter for r in rep.reports)}
    gold = os.path.join(ROOT, "tests", "golden", "c1_full.npz")
    if os.path.exists(gold):
        g = np.load(gold)
        out["max_rel_eig_diff_vs_reference"] = max(
            float(np.max(np.abs(lam - g[f"lam{i}"]) / np.abs(g[f"lam{i}"])))
            for i, lam in enumerate(rep.eigenvalues))
        out["reference_iterations"] = [int(len(g[f"it_filtered{i}"])) for i in range(5)]
    try:
        t_s, cols = oracle_c1_sample(probs)
        total = float(sum(rep.work))
        out["reference_cpu"] = {
            "s_extrapolated": t_s / max(cols, 1) * total, "kind": "port",
            "cores": os.cpu_count(), "blas_threads": blas_threads(),
            "sample": f"oracle solve of problem 1, first 80 outer iterations: {cols} "
                      f"matmul-columns in {t_s:.1f} s, scaled to the sequence's {int(total)}"}
        out["reference_cpu_s"] = out["reference_cpu"]["s_extrapolated"]
    except Exception as exc:  # pragma: no cover - reported
        out["reference_cpu"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    return out


def free_port():
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launcher_argv(argv, n):
    """The torch.distributed.run command that starts ``n`` ranks of this script with the
    same arguments (one process per GPU, rendezvous on 127.0.0.1)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={free_port()}",
            os.path.abspath(__file__)] + list(argv)


def check_visible_gpus(args):
    """--gpus N over NCCL needs N distinct GPUs; fail loudly instead of measuring fewer."""
    if args.impl != "b200" or args.dist_backend != "nccl":
        return None
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < args.gpus:
        return f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}"
    return None


def main():
    args = parse()
    if args.gpus < 1:
        sys.exit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # started without a launcher: start the N ranks ourselves (the driver's
        # `bench.py --gpus N` and a torchrun launch measure the same thing)
        err = check_visible_gpus(args)
        if err:
            sys.exit(f"bench.py: {err}")
        proc = subprocess.run(launcher_argv(sys.argv[1:], args.gpus))
        sys.exit(proc.returncode)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1 and local_rank == 0:
        err = check_visible_gpus(args)
        if err:
            sys.exit(f"bench.py: {err}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "gloo":
            # test mode: ranks may share a GPU (host-staged gather, no waiting kernels)
            local_rank = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    run_b200(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
