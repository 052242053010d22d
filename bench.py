#!/usr/bin/env python
"""randUTV benchmark: BASELINE.json's metric on BASELINE.json's config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One "step" = one full randUTV factorization (every row of SURVEY §8(a)) of the
config-3 matrix: 10000 x 10000 fp64, S-shaped spectrum, b = 256, q = 2, in the
paper's "no orthonormal matrices" mode (U = V = NULL) that the flop formula
(5+2q) m n^2 - (3+2q) n^3/3 of PAPER.md:1203-1207 counts.  value = that flop
count / device time, whole job (N independent replicas: DESIGN.md "Multi-GPU").
The input (800 MB) is larger than L2 (126 MB) and is re-read from HBM every
step; T is rewritten from A inside each step.

Extra keys: e2e (same metric through the C ABI on pinned HOST buffers, H2D of A
and D2H of T inside the timed region), roofline (dominant kernel class = the
DMMA GEMMs, CUDA-event timed per launch inside the library), cpu_baseline (the
oracle on a bounded sample, rank 0, N = 1), clocks, gpu_launches, utv (the
same factorization with U and V formed, for context).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "randUTV fp64 GFLOP/s & time-to-factor n=10k, 1/2/4/8 B200, % of FP64 peak"
UNIT = "GFLOP/s"
# FP64 DMMA peak measured on this pool's B200 by tools/fp64_peaks.cu (profiles/r01_fp64_peaks.md);
# MEASURED_PEAKS.json carries no fp64 entry.
FP64_DMMA_PEAK_TFLOPS = 37.0
FP64_CUBLAS_DGEMM_TFLOPS = 35.46


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-utv", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed (NCCL, block-cyclic) path even at N=1")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = c3 recipe at n = 10000 N^(1/3) (fixed flops per GPU); strong = fixed c3")
    return ap.parse_args()


# The paper's own n = 10000, q = 2 numbers (CPU, b = 64,
# matrix values unstated): context only -- another machine, another block size,
# so vs_baseline stays null.
PAPER_CONTEXT = {
    "hardware": "Intel Xeon E5-2695 v3 (Haswell), 14 cores, 2.3 GHz, MKL 11.2.3",
    "workload": "n=10000, b=64, q=2, no U,V", "t_randutv_s": 36.2, "t_mkl_dgesvd_s": 155.0,
    "speedup_over_dgesvd": 4.28, "derived_gflops": 184.0, "source": "PAPER.md:1706 via BASELINE.md",
}


def workload_desc(case, m, n):
    return {
        "workload": f"{case.name}: {m}x{n} fp64, b={case.b}, q={case.q}, T-only (U=V=NULL), full factorization"
        if case.name != "c5" else f"c5: {m}x{n}, b={case.b}, q={case.q}, k_stop={case.k_stop}",
        "m": m, "n": n, "b": case.b, "q": case.q, "reortho": True, "mode": "T",
        "flops_formula": "(5+2q)mn^2-(3+2q)n^3/3 (PAPER.md:1205)",
        "l2": ("inputs larger than L2 (A = %.0f MB > 126 MB), re-read every step" % (m * n * 8 / 1e6))
        if m * n * 8 > 126e6 else ("A = %.1f MB fits in L2 (not flushed; a parity-size config, not the "
                                   "driver's bench line)" % (m * n * 8 / 1e6)),
    }


def flops_for(case, m, n):
    from paper_1703_00998_b200 import flops
    if case.k_stop:
        return flops.flops_T_steps(m, n, case.b, case.q, case.k_stop)
    return flops.flops_T(m, n, case.q)


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


def oracle_sample(A_host, case, reps=1):
    """The oracle as it stands on this host: the first randomized step of the
    workload (k_stop = b, T-only).  Returns (GFLOP/s, seconds, flops, cores)."""
    import numpy as np
    from oracle import randutv as oracle_randutv
    from paper_1703_00998_b200 import flops
    m, n = A_host.shape
    f = flops.flops_T_steps(m, n, case.b, case.q, k_stop=case.b)
    try:
        from threadpoolctl import threadpool_info
        cores = max([d.get("num_threads", 1) for d in threadpool_info()] or [os.cpu_count()])
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle_randutv(A_host, case.b, case.q, case.seed, k_stop=case.b, build_ortho=False)
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    del np
    return f / t / 1e9, t, f, cores


def critical_path(tl):
    """Breakdown of the critical (first-used) stream of one profiled
    factorization (per-launch (class, stream slot, start, end) from the
    library's event timeline): busy time by class, idle time (waits on side
    streams and launch gaps), and the latency-bound QR-chain time that no GEMM
    on another stream overlaps (exposed)."""
    if not tl:
        return None
    main = sorted((a, e, c) for c, s, a, e in tl if s == 0)
    span = max(e for _, _, _, e in tl) - min(a for _, _, a, _ in tl)
    busy = {}
    for a, e, c in main:
        busy[c] = busy.get(c, 0.0) + (e - a)
    others = sorted((a, e) for c, s, a, e in tl if s != 0 and c.startswith("gemm_"))

    def covered(a, e):  # length of [a, e] covered by other-stream GEMMs
        tot, cur_a, cur_e = 0.0, None, None
        for x, y in others:
            if y <= a or x >= e:
                continue
            x, y = max(x, a), min(y, e)
            if cur_e is None or x > cur_e:
                if cur_e is not None:
                    tot += cur_e - cur_a
                cur_a, cur_e = x, y
            else:
                cur_e = max(cur_e, y)
        if cur_e is not None:
            tot += cur_e - cur_a
        return tot
    chain = [(a, e) for a, e, c in main if c in ("qr_small", "gemm_panel_qr")]
    chain_ms = sum(e - a for a, e in chain)
    exposed = sum((e - a) - covered(a, e) for a, e in chain)
    # stricter: span time in which no big GEMM (sketch / right / left apply) runs on
    # ANY stream -- the exposed latency-bound chains wherever they run, plus the tail
    # after the last big GEMM (the last SVD chunk and the folds)
    big = sorted((a, e) for c, s, a, e in tl if c in ("gemm_sketch", "gemm_right_apply", "gemm_left_apply"))
    t0 = min(a for _, _, a, _ in tl)
    t1 = max(e for _, _, _, e in tl)
    union, cur = 0.0, None
    for a, e in big:
        if cur is None or a > cur[1]:
            if cur is not None:
                union += cur[1] - cur[0]
            cur = [a, e]
        else:
            cur[1] = max(cur[1], e)
    if cur is not None:
        union += cur[1] - cur[0]
    last_big = max((e for _, e in big), default=t0)
    return {"factorization_span": round(span, 3), "main_busy": round(sum(busy.values()), 3),
            "no_big_gemm": round((t1 - t0) - union, 3), "tail_after_last_big_gemm": round(t1 - last_big, 3),
            "main_idle": round(span - sum(busy.values()), 3),
            "main_by_class": {k: round(v, 3) for k, v in sorted(busy.items(), key=lambda t: -t[1])},
            "qr_chain_main": round(chain_ms, 3), "qr_chain_main_exposed": round(exposed, 3),
            "note": "one profiled (eager, per-launch event-timed) factorization; idle = waits for side-stream "
                    "work (trailing update, panel QR, look-ahead left update, last SVD chunk) and launch gaps"}


def make_input(case_name, device, rank, scale=1.0):
    import testmat
    At, case = testmat.device_config(case_name, device=device, scale=scale)
    return At, case


def run_reference(args):
    """--impl reference: the oracle (CPU) on the same config, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import numpy as np
    import torch
    import testmat
    case_name = args.config
    # the same workload as our arm at this N (weak scaling: n = 10000 N^(1/3))
    scale = world ** (1.0 / 3.0) if (world > 1 and args.scaling == "weak") else 1.0
    if torch.cuda.is_available():
        At, case = testmat.device_config(case_name, device="cuda", scale=scale)
        A_host = np.asfortranarray(At.t().cpu().numpy())
        del At
        torch.cuda.empty_cache()
    else:
        c = testmat.config(case_name, scale=scale)
        A_host, case = c.A, c
    m, n = A_host.shape
    # warm-up samples (thread pools, page faults), capped at ~20 s of CPU time
    warm, t_warm = 0, 0.0
    while warm < args.warmup and t_warm < 20.0:
        _, t, _, _ = oracle_sample(A_host, case)
        warm += 1
        t_warm += t
    vals, ts = [], []
    for _ in range(args.steps):
        v, t, f, cores = oracle_sample(A_host, case)
        vals.append(v)
        ts.append(t)
    value = statistics.median(vals)
    sample = f"first randomized step of {case_name} (k_stop=b={case.b}, q={case.q}, T-only) on the full {m}x{n} input"
    cfg = workload_desc(case, m, n)
    cfg["workload"] = (f"{case_name}: {m}x{n} fp64, b={case.b}, q={case.q}, T-only -- FIRST RANDOMIZED STEP ONLY "
                       f"(k_stop = b = {case.b}; a bounded sample of the full factorization, rate in the same unit)")
    cfg["sample_flops"] = f
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": warm, "ms_per_step": round(1e3 * statistics.median(ts), 3),
        "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import paper_1703_00998_b200 as P
    from paper_1703_00998_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_dist = world > 1 or args.dist
    dist = None
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if use_dist:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    scaling = args.scaling if world > 1 else "weak"
    scale = world ** (1.0 / 3.0) if (world > 1 and scaling == "weak") else 1.0

    At, case = make_input(args.config, dev, rank, scale)
    A = At.t()
    m, n = A.shape
    F = flops_for(case, m, n)
    stream = torch.cuda.current_stream(dev)
    if use_dist:
        comm = D.nccl_from_torch()
        S = D.shard(A, case.b, rank, world)
        A_host_src = S
        del A, At
        torch.cuda.empty_cache()
        Tsh = [P.empty_cm(m, S.shape[1], dev)]

        def step(with_uv=False, out=None):
            return D.factor(comm, [S], m, n, case.b, case.q, case.seed, k_stop=case.k_stop, tol=case.tol, out=Tsh)
    else:
        T = P.empty_cm(m, n, dev)

        def step(with_uv=False, out=None):
            return P.randutv(A, case.b, case.q, case.seed, k_stop=case.k_stop, tol=case.tol, with_uv=with_uv,
                             out=out if out is not None else (None, T, None))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize(dev)

    # ---------------------------------------------------------------- timed region
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.3)
    l0 = P.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    launches = P.launch_count() - l0
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if dist:
        t = torch.tensor([ms, float(launches)], device=dev, dtype=torch.float64)
        tl = t.clone()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        ms, launches = float(t[0].item()), int(tl[1].item())
    value = F / (ms * 1e-3) / 1e9  # whole-job flops (the factorization's flop count) / time

    # ---------------------------------------------------------------- roofline of the dominant kernel
    # One profiled factorization (per-launch CUDA events on each launch's own
    # stream, inside the library; graph replay is off while profiling).  The
    # dominant kernel is the sketch DGEMM class (Y = X^T G, Z = X Y, Y = X^T Z:
    # ~51 % of the flops and the largest share of device time); its launches
    # run on the critical stream, mostly alone.  The other GEMM roles run
    # concurrently on side streams, so their per-launch event durations include
    # sharing the SMs -- listed in by_class, not used as the headline.
    P.profile_begin()
    step()
    prof = P.profile_end()
    tl = P.profile_timeline()
    gemm = {k: v for k, v in prof.items() if k.startswith("gemm_")}
    g_ms = sum(v["ms"] for v in gemm.values())
    g_n = sum(v["launches"] for v in gemm.values())
    tot_ms = sum(v["ms"] for v in prof.values())
    sk = prof["gemm_sketch"]
    achieved = sk["flops"] / (sk["ms"] * 1e-3) / 1e12 if sk["ms"] > 0 else 0.0
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get("bytes_per_launch")
            traffic_src = "stored_ncu: " + tj.get("source", "profiles/gemm_traffic.json") + " (not measured in this run)"
        except Exception:  # noqa: BLE001
            traffic = None
    # the method's algorithmic bytes of one sketch launch Y = X^T G at step 1: X and G read, Y written
    alg_bytes = 8 * (m * n + m * case.b + n * case.b)
    roofline = {
        "bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": round(achieved / FP64_DMMA_PEAK_TFLOPS, 4), "traffic": traffic, "traffic_source": traffic_src,
        "algorithmic_bytes_step1_launch": alg_bytes,
        "kernel": "dgemm_kernel, sketch role (X^T G, X Y, X^T Z; FP64 DMMA m8n8k4, incl. its split-K reduce)",
        "flops_per_launch": "2 m_i n_i b (sum over the class: (2+4q) sum_i m_i n_i b, SURVEY 8(d))",
        "peak_source": "measured DMMA peak, tools/fp64_peaks.cu (profiles/r01_fp64_peaks.md); "
                       "MEASURED_PEAKS.json has no fp64 entry",
        "sketch_launches": sk["launches"], "sketch_ms": round(sk["ms"], 3),
        "all_gemm": {"launches": g_n, "event_ms": round(g_ms, 3),
                     "tflops_per_event_time": round(sum(v["flops"] for v in gemm.values()) / (g_ms * 1e-3) / 1e12, 3)
                     if g_ms > 0 else None,
                     "share_of_event_time": round(g_ms / tot_ms, 4) if tot_ms else None},
        "by_class": {k: {"ms": round(v["ms"], 3), "tflops": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2)
                         if v["ms"] > 0 and v["flops"] > 0 else None, "launches": v["launches"]}
                     for k, v in prof.items()},
    }
    if use_dist:
        roofline["note"] = "rank 0's kernels; per-class event times include waits on collectives"
    critical = critical_path(tl)

    # ---------------------------------------------------------------- U,V formed (context, single GPU)
    utv = None
    if not args.no_utv and not use_dist:
        U = P.empty_cm(m, m, dev)
        V = P.empty_cm(n, n, dev)
        step(True, (U, T, V))
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(True, (U, T, V))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        tu = e0.elapsed_time(e1)
        utv = {"ms": round(tu, 3), "gflops_credited_FT": round(F / (tu * 1e-3) / 1e9, 3),
               "gflops_executed": round((F + P.flops.flops_UV(m, n)) / (tu * 1e-3) / 1e9, 3)}
        del U, V
        torch.cuda.empty_cache()

    # ---------------------------------------------------------------- end to end, host buffers in the timed region
    e2e = None
    if not args.no_e2e:
        reps = max(1, min(args.steps, 3))
        if use_dist:
            # per rank: pinned host shard -> device, distributed factorization, T shard -> host
            nl = A_host_src.shape[1]
            Ah = torch.empty(nl, m, dtype=torch.float64, pin_memory=True)
            Ah.copy_(A_host_src.t())
            Th = torch.empty(nl, m, dtype=torch.float64, pin_memory=True)
            Sd = P.empty_cm(m, nl, dev)

            def e2e_step():
                Sd.t().copy_(Ah, non_blocking=True)
                D.factor(comm, [Sd], m, n, case.b, case.q, case.seed, k_stop=case.k_stop, tol=case.tol, out=Tsh)
                Th.copy_(Tsh[0].t(), non_blocking=True)
                torch.cuda.synchronize(dev)
            e2e_step()
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                e2e_step()
            te = (time.perf_counter() - t0) / reps
            t = torch.tensor([te], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
            hb = tb = m * nl * 8
            del Ah, Th, Sd
        else:
            Ah = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
            Ah.copy_(At)
            Th = torch.empty(n, m, dtype=torch.float64, pin_memory=True)
            torch.cuda.synchronize(dev)
            P.factor_raw(m, n, Ah.data_ptr(), m, case.b, case.q, case.seed, case.k_stop, None, Th.data_ptr(), None)
            t0 = time.perf_counter()
            for _ in range(reps):
                rc = P.factor_raw(m, n, Ah.data_ptr(), m, case.b, case.q, case.seed, case.k_stop, None,
                                  Th.data_ptr(), None)
                assert rc == 0, rc
            te = (time.perf_counter() - t0) / reps
            hb = tb = m * n * 8
            del Ah, Th
        e2e = {"value": round(F / te / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": hb,
               "d2h_bytes_per_step": tb, "ms_per_step": round(te * 1e3, 3),
               "timer": "host wall clock (max over ranks) around H2D of A, the factorization and D2H of T"
                        + (" (per-rank shards, bytes per rank)" if use_dist else " (randutv_factor on pinned host A, T)")}

    # ---------------------------------------------------------------- CPU oracle baseline (rank 0, N = 1)
    cpu = None
    if not args.no_cpu_baseline and world == 1 and rank == 0 and not use_dist:
        A_host = np.asfortranarray(A.cpu().numpy())
        v, t, f, cores = oracle_sample(A_host, case)
        cpu = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first randomized step of {case.name} (k_stop=b={case.b}, q={case.q}, T-only) "
                         f"on the same {m}x{n} input: {f:.3e} flops in {t:.2f} s"}

    if rank == 0:
        if use_dist:
            par = f"block-cyclic columns (b={case.b}) x{world}, NCCL"
        else:
            par = "single"
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": scaling if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_desc(case, m, n), parallelism=par),
            "pct_fp64_peak": round(100 * value / world / 1e3 / FP64_DMMA_PEAK_TFLOPS, 2),
            "pct_cublas_dgemm": round(100 * value / world / 1e3 / FP64_CUBLAS_DGEMM_TFLOPS, 2),
            "time_to_factor_s": round(ms * 1e-3, 4),
            "roofline": roofline, "critical_path_ms": critical, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches,
            "utv": utv,
            "paper_context": PAPER_CONTEXT if case.name == "c3" else None,
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
