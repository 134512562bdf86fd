#!/usr/bin/env python
"""bench.py -- FPE multi-point evaluation throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fpe|reference] [--config 3] [--fp32]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL)

A step is one pass of the whole hot path -- fpe_evaluate: classification (lambda, k_lambda,
[l, r]) and window evaluation of every point -- over one batch of synthetic points
already resident in HBM.  Workload (default): BASELINE.json configs[2], complex fp64,
d = 2^20 - 1, |a_k| = 2^(200 sin(pi k/d) + N(0,4)), 2^26 points uniform on the Riemann
sphere per rank (weak scaling: every rank evaluates its own 2^26-point batch; the
preconditioned polynomial is replicated once with an NCCL broadcast, untimed).
--config 5 [--fp32] is BASELINE.json configs[4], the scaling run: complex fp64 (or fp32)
d = 2^22 - 1, N = 2^28 points in total, each rank evaluating its contiguous shard of
ceil(N/G) points (strong scaling; every rank generates exactly its slice of the seeded
sequence).  Points exceed the 126 MB L2, so no flush is needed between steps.
Prints ONE JSON line on rank 0.
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

METRIC = "polynomial evals/sec (fp64 complex, d=2^20) at 1/2/4/8 B200; % of roofline"
FP64_FMA_PEAK = 148 * 64 * 1.965e9      # SMs x fp64 FMA lanes/clk/SM x max SM clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fpe", choices=["fpe", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--fp32", action="store_true", help="the fp32 variant (coefficients and points rounded)")
    ap.add_argument("--points", type=int, default=0,
                    help="override points per rank (weak scaling) or in total (--config 5, strong scaling)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the context measurements (full Horner, the other BASELINE configs)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0:
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if args.impl == "fpe":
        torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if args.impl == "fpe":   # bind the NCCL communicator to this rank's GPU (eager init)
            dist.init_process_group(backend="nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend="gloo")
        pg = dist
    return world, rank, local, pg


def reduce_max(pg, v: float, device) -> float:
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(pg, v: float, device) -> float:
    if pg is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def algorithmic_fma(diag_fields, cplx: bool, parts: bool = False):
    """sum over points of c (K + 2 ceil(log2 l) [l > 0]): the paper's count (PAPER.md:1621-1627,
    1321-1324), c = 4 fp64 FMAs per complex multiply-add, 1 for real.  parts=True returns the window
    part c K (the Horner over the kept terms: the evaluator kernels) and the power part c 2 ceil(log2 l)
    (z^l: applied by k_unsort's epilogue) separately."""
    import torch
    K = diag_fields["kept"].double()
    l = diag_fields["l"].double()
    pw = torch.where(l > 0, 2.0 * torch.ceil(torch.log2(torch.clamp(l, min=1.0))), torch.zeros_like(l))
    c = 4.0 if cplx else 1.0
    if parts:
        return float((c * K).sum()), float((c * pw).sum())
    return float((c * (K + pw)).sum())


def cpu_baseline(cfg: int, sample: int, fp32: bool = False):
    """The oracle as it stands (oracle/, binary128, OpenMP over all host cores), timed on a
    bounded sample of the same workload: classification + Q_lambda for `sample` points."""
    import numpy as np

    import oracle
    import workloads
    a = workloads.coefficients(cfg)
    if fp32:
        a = workloads.to_fp32(a)
    t0 = time.perf_counter()
    P = oracle.OraclePoly(a)
    t_pre = time.perf_counter() - t0
    pts = workloads.points(cfg, sample, shard=977)
    if fp32:
        pts = workloads.to_fp32(pts)
    t0 = time.perf_counter()
    c = P.classify(pts)
    P.fpe_eval(pts, c)
    dt = time.perf_counter() - t0
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": sample / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
            "sample": f"{sample} points of cfg{cfg} (same distribution, shard 977): binary128 classify + "
                      f"Q_lambda; preconditioning {t_pre:.2f}s not included",
            "seconds": dt}


def _time_ms(fn, steps: int, warmup: int) -> float:
    """Mean device time of fn() in ms (CUDA events on the current stream, synchronised)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def extra_context(device: int, steps: int = 3):
    """Context numbers on 1 GPU (north_star): the full-Horner kernel on the headline workload, and the
    other BASELINE configs (evals/s through fpe_evaluate, algorithmic fp64/fp32 FMA rate from a
    2^20-point diagnostic subsample).  Each entry is independent; a failure is recorded, not raised."""
    import numpy as np
    import torch

    import paper_2211_06320_b200 as fpe
    import workloads
    dev = torch.device("cuda", device)
    out = {}
    try:   # full Horner, cfg3 polynomial (d = 2^20 - 1), 2^20 sphere points (3.5 waves of the persistent warps)
        poly = fpe.precondition(workloads.coefficients(3), device=device)
        pts = torch.from_numpy(workloads.points(3, 1 << 20, shard=5)).to(dev)
        ms = _time_ms(lambda: poly.horner(pts), 2, 1)
        fma = 4.0 * (poly.info["k_max"] - poly.info["k_min"] + 1) * pts.numel()
        out["full_horner_cfg3"] = {"evals_per_s": pts.numel() / (ms * 1e-3), "ms": ms, "points": pts.numel(),
                                   "fma_per_s": fma / (ms * 1e-3)}
        del poly, pts
    except Exception as e:  # noqa: BLE001
        out["full_horner_cfg3"] = {"error": repr(e)[:200]}
    # preconditioning (§8(f) row 3): host path (coefficients copied to the host, precondition.cpp, upload)
    # vs the device preconditioner (precondition_gpu.cu), coefficients resident on the GPU; wall clock
    for cfg in (3, 5, 4):
        try:
            a = torch.from_numpy(workloads.coefficients(cfg)).to(dev)

            def wall(f, reps=5):   # the call only: the handle is released outside the timed region
                ts = []
                for _ in range(reps):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    h = f()
                    torch.cuda.synchronize()
                    ts.append(time.perf_counter() - t0)
                    h.close()
                return 1e3 * sorted(ts)[len(ts) // 2]
            fpe.precondition_gpu(a).close()
            ms_host = wall(lambda: fpe.precondition(a))
            ms_gpu = wall(lambda: fpe.precondition_gpu(a))
            out[f"precondition_cfg{cfg}"] = {"coefficients": a.numel(), "host_ms": ms_host, "gpu_ms": ms_gpu,
                                             "speedup": ms_host / ms_gpu}
            del a
        except Exception as e:  # noqa: BLE001
            out[f"precondition_cfg{cfg}"] = {"error": repr(e)[:200]}
    # the BASELINE configs, then the second point sets of SURVEY 8(f) row 4 on the cfg5 / cfg2 polynomials
    specs = [(1, None, False, None), (2, None, False, None), (4, None, False, None), (5, None, False, None),
             (5, None, True, None), (5, 1 << 24, False, "disk"), (2, None, False, "rbar")]
    for cfg, n, fp32, pset in specs:
        name = f"cfg{cfg}" + ("_fp32" if fp32 else "") + (f"_{pset}" if pset else "")
        try:
            c = workloads.CONFIGS[cfg]
            n = n or c["n_points"]
            a = workloads.coefficients(cfg)
            if pset == "disk":
                p = workloads.disk_points(cfg, n)
            elif pset == "rbar":
                p = workloads.rbar_points(cfg, n)
            else:
                p = workloads.points(cfg, n)
            if fp32:
                a, p = workloads.to_fp32(a), workloads.to_fp32(p)
            poly = fpe.precondition(a, device=device)
            pts = torch.from_numpy(p).to(dev)
            del p
            sub = pts[: min(n, 1 << 20)]
            _, _, dg = poly.evaluate(sub, exps=True, diag=True)
            D = fpe.diag_fields(dg)
            cplx = np.iscomplexobj(a)
            wwin, wpow = algorithmic_fma(D, cplx, parts=True)
            # dense: the evaluator kernels do the window sums (z^l in k_unsort); sparse: k_eval_sparse_coop
            # forms every term's power itself
            work_pt = (wwin + (wpow if poly.info["sparse"] else 0.0)) / sub.numel()
            meanK = float(D["kept"].double().mean())
            del dg, D
            vals = torch.empty(n, dtype=(torch.complex64 if cplx else torch.float32) if fp32 else
                               (torch.complex128 if cplx else torch.float64), device=dev)
            ms = _time_ms(lambda: poly.evaluate(pts, exps=True, out=vals), steps, 2)
            poly.set_profiling(True)
            poly.evaluate(pts, exps=True, out=vals)
            stages = dict(poly.last_stage_ms())
            poly.set_profiling(False)
            peak = FP64_FMA_PEAK * (2 if fp32 else 1)
            ev_ms = sum(v for k, v in stages.items() if k in ("eval_mma", "eval_tiled", "eval_overflow")) or \
                max(stages.values())
            out[name] = {"workload": c["name"] + (f" at {pset} points" if pset else ""), "points": n,
                         "evals_per_s": n / (ms * 1e-3), "ms_per_step": ms,
                         "mean_kept_terms": meanK, "stages_ms": stages,
                         "eval_kernel_fma_frac": work_pt * n / (ev_ms * 1e-3) / peak,
                         "sparse": bool(poly.info["sparse"]), "dtype": "f32" if fp32 else "f64"}
            del poly, pts, vals
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001
            out[name] = {"error": repr(e)[:200]}
    return out


def run_reference(args):
    """--impl reference: the oracle (CPU) on rank 0, each step a bounded sample."""
    world, rank, local, pg = dist_setup(args)
    if rank != 0:
        return
    import oracle
    import workloads
    cfg = args.config
    sample = args.cpu_sample or 8192
    a = workloads.coefficients(cfg)
    pts = workloads.points(cfg, sample, shard=977)
    if args.fp32:
        a, pts = workloads.to_fp32(a), workloads.to_fp32(pts)
    P = oracle.OraclePoly(a)
    for _ in range(args.warmup):
        P.fpe_eval(pts[:64], P.classify(pts[:64]))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        P.fpe_eval(pts, P.classify(pts))
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    val = sample / (ms * 1e-3)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    line = {"metric": METRIC, "value": val, "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if cfg == 5 else "weak",
            "vs_baseline": None, "dtype": "f128", "data": "synthetic", "impl": "reference",
            "config": {"workload": workloads.CONFIGS[cfg]["name"] + ("_fp32" if args.fp32 else ""),
                       "points_per_step": sample, "sample": True},
            "cpu_baseline": {"value": val, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "sample": f"{sample} points of cfg{cfg} per step (binary128 oracle)"},
            "e2e": {"value": val, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def profiled_traffic(prefixes=("void k_eval_tiled", "k_eval_mma", "void k_eval_mma", "void k_eval_overflow")):
    """DRAM bytes (read + write) per step of the kernels whose names start with `prefixes` (default: the window
    evaluator, k_eval_mma + k_eval_tiled [+ the overflow kernel]) from the committed ncu --set full summary of
    the same cfg3 workload (round 2: profiles/r02_ncu_cfg3_all_kernels.json, in bytes; round 1's file was in
    GB); None if absent."""
    for name, scale in (("r02_ncu_cfg3_all_kernels.json", 1.0), ("r01_ncu_eval_tiled_cfg3.json", 1e9)):
        path = os.path.join(ROOT, "profiles", name)
        try:
            with open(path) as f:
                tot, seen = 0.0, False
                for k in json.load(f):
                    if k.get("kernel", "").startswith(prefixes):
                        tot += scale * (k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"])
                        seen = True
                if seen:
                    return {"bytes": tot, "source": os.path.relpath(path, ROOT)}
        except (OSError, ValueError, KeyError):
            continue
    return None


def run_fpe(args):
    import numpy as np
    import torch

    import paper_2211_06320_b200 as fpe
    import workloads
    from paper_2211_06320_b200 import dist as fdist

    world, rank, local, pg = dist_setup(args)
    dev = torch.device("cuda", local)
    cfg = args.config
    c = workloads.CONFIGS[cfg]
    fp32 = bool(args.fp32)
    strong = cfg == 5   # BASELINE configs[4]: N points in total, sharded by point
    if strong:
        n_total = args.points or c["n_points"]
        lo, hi = fdist.shard_range(n_total, rank, world)
        n = hi - lo
        pts_np = workloads.points(cfg, n, start=lo)
    else:
        n = args.points or c["n_points"]
        pts_np = workloads.points(cfg, n, shard=rank)
    if fp32:
        pts_np = workloads.to_fp32(pts_np)
    # -- replicate the preconditioned polynomial (rank 0 builds, NCCL broadcast; untimed) --
    poly = None
    if rank == 0:
        a = workloads.coefficients(cfg)
        poly = fpe.precondition(workloads.to_fp32(a) if fp32 else a, device=local)
    poly = fdist.replicate(poly, src=0, device=local) if pg is not None else poly
    cplx = c["dtype"].startswith("c")
    pts = torch.from_numpy(pts_np).to(dev)
    vdt = (torch.complex64 if cplx else torch.float32) if fp32 else (torch.complex128 if cplx else torch.float64)
    vals = torch.empty(n, dtype=vdt, device=dev)
    exps = torch.empty(n, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    ws = poly.workspace(n, stream)

    def step():
        poly.evaluate(pts, exps=True, out=vals, workspace=ws)

    # algorithmic work from one untimed diagnostic pass
    _, _, dg = poly.evaluate(pts, exps=True, diag=True)
    D = fpe.diag_fields(dg)
    fma_window, fma_power = algorithmic_fma(D, cplx, parts=True)
    fma_total = fma_window + fma_power
    meanK = float(D["kept"].double().mean())
    kq = torch.quantile(D["kept"].double()[:: max(1, D["kept"].numel() // (1 << 22))], torch.tensor([0.5, 0.99], dtype=torch.float64, device=D["kept"].device))
    kept_stats = {"median": float(kq[0]), "p99": float(kq[1]), "max": int(D["kept"].max())}
    hard = int(D["hard"].sum())
    del dg, D
    torch.cuda.empty_cache()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # -- timed region ------------------------------------------------------------------------
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = reduce_max(pg, ms_local, dev)
    total_points = reduce_sum(pg, float(n), dev)
    value = total_points / (ms * 1e-3)
    launches = poly.last_stats()["launches"]
    counters = poly.workspace_stats(ws, stream)
    in_bytes = n * pts.element_size()

    # -- per-kernel durations, live, on the launch stream (profiling events) --------------------
    poly.set_profiling(True)
    stage_acc = {}
    for _ in range(max(3, min(args.steps, 5))):
        step()
        for name, t in poly.last_stage_ms():
            stage_acc.setdefault(name, []).append(t)
    poly.set_profiling(False)
    stages = {k: statistics.mean(v) for k, v in stage_acc.items()}
    # the window evaluator: the tensor-core pieces (k_eval_mma) and the vector Horner (k_eval_tiled)
    # together do the algorithmic work, so the roofline takes their summed duration
    ev_keys = [k for k in ("eval_mma", "eval_tiled", "eval_overflow") if k in stages]
    dom = "+".join(ev_keys) if ev_keys else max(stages, key=stages.get)
    dom_ms = sum(stages[k] for k in ev_keys) if ev_keys else stages[dom]
    # the evaluator kernels do the window sums (c K per point); z^l is applied by k_unsort's epilogue, so
    # its 2 ceil(log2 l) multiplications are not credited to them
    achieved = 2.0 * fma_window / (dom_ms * 1e-3) / 1e12        # TFLOP/s (2 flops per FMA)
    peak = 2.0 * FP64_FMA_PEAK * (2 if fp32 else 1) / 1e12   # fp32: 128 FMA lanes / SM / clk

    # -- end to end through the public API with host buffers (pinned) ---------------------------
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(pts_np).pin_memory()
        hv = torch.empty(n, dtype=vals.dtype).pin_memory()
        he = torch.empty(n, dtype=torch.int64).pin_memory()
        pdt = (3 if cplx else 2) if fp32 else (1 if cplx else 0)
        poly.evaluate_host_ptr(hp.data_ptr(), pdt, n, hv.data_ptr(), he.data_ptr())
        if pg is not None:
            pg.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            poly.evaluate_host_ptr(hp.data_ptr(), pdt, n, hv.data_ptr(), he.data_ptr())
        dt = (time.perf_counter() - t0) / args.e2e_steps
        dt = reduce_max(pg, dt, dev)
        e2e = {"value": total_points / dt, "unit": "evals/s", "h2d_bytes_per_step": int(in_bytes),
               "d2h_bytes_per_step": int(n * (vals.element_size() + 8)), "ms_per_step": dt * 1e3}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(cfg, args.cpu_sample or 65536, fp32)
    context = None
    if not args.no_extra and world == 1:
        del pts, vals, exps, ws
        torch.cuda.empty_cache()
        context = extra_context(local)
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f32" if fp32 else "f64", "data": "synthetic",
        "config": {"workload": c["name"] + ("_fp32" if fp32 else ""), "points_per_gpu": n,
                   "points_total": int(total_points), "degree": c["d"],
                   "parallelism": f"points x{world}" + (" (contiguous shards of N)" if strong else ""),
                   "l2": f"inputs ({in_bytes / 2**30:.2f} GiB/rank) larger than L2; no flush",
                   "mean_kept_terms": meanK, "kept_terms": kept_stats, "hard_lambdas": hard,
                   "counters": counters},
        "roofline": {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak,
                     "traffic": (profiled_traffic() or {}).get("bytes") if (cfg == 3 and not fp32) else None,
                     "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the evaluator kernels "
                                     f"({(profiled_traffic() or {}).get('source')}): they read the 32-B bucket-order "
                                     f"records and write a 32-B accumulator per point at its input index "
                                     f"({64 * n / 1e9:.2f} GB); the path's algorithmic bytes are 40 B/pt = "
                                     f"{40 * n / 1e9:.2f} GB (points in, values and exponents out, the latter written "
                                     "by k_unsort); step_traffic = every kernel of the step",
                     "step_traffic": (profiled_traffic(("void k_", "k_")) or {}).get("bytes")
                     if (cfg == 3 and not fp32) else None,
                     "peak_note": ("fp32 FMA: 148 SM x 128 lanes x 1.965 GHz x 2; " if fp32 else "") +
                                  "fp64 FMA: 148 SM x 64 lanes x 1.965 GHz x 2 (guide unit counts/clock); the FP64 "
                                  "tensor cores (DMMA, k_eval_mma) run on the same datapath: 18.5T FMA/s measured "
                                  "(profiles/r01_dmma_vs_dfma.json)",
                     "algorithmic_fma_per_launch": fma_window, "algorithmic_fma_step": fma_total,
                     "algorithmic_note": "window sums c*K over the kept terms (the evaluator kernels); the step also "
                                         "applies z^l (c*2*ceil(log2 l) per point) in k_unsort",
                     "kernel_ms": dom_ms, "stages_ms": stages},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches * args.steps),
        "clocks": clk.summary(),
        "context": context,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_fpe(args)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
