#!/usr/bin/env python
"""Benchmark of the B200 P_N solve path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload: config 4 (P7, 256^3, 1.07e9 unknowns, fp64) -- the largest
single-GPU configuration, the strong-scaling config of BASELINE.json.  A step
is one operator apply (alternating A u and A^T u, the two sparse products of
a CGNR iteration) on device-resident vectors; value = unknowns * K / time
(Gunknowns/s, whole job).  Every vector is 8.6 GB, far above the 126 MB L2,
so no L2 flush is needed between steps.  Extra keys report the full fused CG
iteration, time-to-residual 1e-6 on config 2, the end-to-end solve from host
fields (e2e), the HBM roofline of the apply kernel, and the CPU oracle
(C port of the reference path) timed on the host cores as the baseline.

--impl reference times the reference's CPU implementation of the path (the C
port under oracle/, all host threads) on a bounded sample of the same
workload: the first 8 z-planes of config 4 (256 x 256 x 8, P7).
Multi-GPU (torchrun): z-slabs of config 4, NCCL halos; timing is the max over
ranks of CUDA-event time.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "P_N operator applies: Gunknowns/s (1/2/4/8 GPU) and time-to-residual 1e-6"
UNIT = "Gunk/s"
SAMPLE_PLANES = 8


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic():
    """dram bytes per apply launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_apply_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        time.sleep(0.15)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def sample_spec(cfg_spec, planes=SAMPLE_PLANES):
    """First `planes` z-planes of a config (same h, same fields)."""
    from paper_1807_00410_b200.problems import ProblemSpec
    nx, ny, nz = cfg_spec.res
    f = {}
    for k, v in cfg_spec.fields.items():
        f[k] = v if np.ndim(v) == 0 else np.ascontiguousarray(np.asarray(v)[:, :, :planes])
    h = cfg_spec.h
    return ProblemSpec(dim=3, origin=cfg_spec.origin, extent=(nx * h, ny * h, planes * h), res=(nx, ny, planes),
                       fields=f, bc="dirichlet", name=cfg_spec.name + f"_z{planes}")


def cpu_oracle_rate(cfg, steps=None, budget_s=12.0, warmup=1):
    """The C port of the reference operator (oracle/, OpenMP over rows) on the
    bounded sample; returns (Gunk/s, per-step seconds list, sample R, cores)."""
    from oracle.oracle import StencilOracle
    from paper_1807_00410_b200.program import build_tables
    spec = sample_spec(cfg.spec)
    o = StencilOracle(build_tables(cfg.N), spec)
    x = np.random.default_rng(0).normal(size=o.R)
    for k in range(warmup):
        o.apply(x, transpose=bool(k & 1))
    times = []
    t_start = time.perf_counter()
    k = 0
    while True:
        t0 = time.perf_counter()
        o.apply(x, transpose=bool(k & 1))
        times.append(time.perf_counter() - t0)
        k += 1
        if steps is not None and k >= steps:
            break
        if steps is None and time.perf_counter() - t_start > budget_s and k >= 3:
            break
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return o.R * len(times) / sum(times) / 1e9, times, o.R, cores


# The only published P_N solve times: the
# paper's C++/Eigen CPU runtime (not shipped, hardware unstated), context only.
PAPER_RUNS = (
    ("checkerboard 71^2 P1", "cb", 1, 1e-10, 0.27),
    ("checkerboard 71^2 P5", "cb", 5, 1e-10, 25.0),
    ("point source 80^3 P1", "ps", 1, 1e-10, 600.0),
    ("point source 80^3 P5", "ps", 5, 1e-10, 2700.0),
)


def paper_workloads(device):
    """Time to normal residual 1e-10 (the paper's "10e-10") on the paper's own
    problems, device-resident inputs after a warm-up solve: the 2-D checkerboard
    (tables from the committed reference fixtures tests/golden/tables_N*_2d.json)
    and the 3-D point source (80^3, sigma_t 8, albedo 0.9)."""
    import torch
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.program import build_tables, from_json
    from paper_1807_00410_b200.run import make_pointsource
    from paper_1807_00410_b200.solver import PnContext
    out = {}
    for name, kind, N, tol, paper_s in PAPER_RUNS:
        if kind == "cb":
            t = from_json(json.loads((ROOT / "tests" / "golden" / f"tables_N{N}_2d.json").read_text()))
            spec = make_checkerboard(71)
        else:
            t = build_tables(N)
            spec = make_pointsource(80)
        c = PnContext(t, spec.res, spec.h, device=device)
        c.set_fields(spec)
        c.solve(tol=tol, max_iter=5)
        torch.cuda.synchronize()
        # median of 3 timed solves for the millisecond-scale problems (one sample
        # of a 3 ms solve swings by 2x with host scheduling)
        secs = []
        while len(secs) < 3:
            t0 = time.perf_counter()
            _, rep = c.solve(tol=tol, max_iter=200000)
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - t0)
            if secs[0] > 1.0:
                break
        sec = float(np.median(secs))
        out[name] = {"seconds": sec, "timed_solves": len(secs), "iterations": rep.iterations, "converged": rep.converged, "tol": tol,
                     "unknowns": c.R_local, "paper_cpu_seconds": paper_s, "paper_over_ours": paper_s / sec}
        del c
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1807_00410_b200.configs import make_config
    cfg = make_config(4)
    rate, times, R, cores = cpu_oracle_rate(cfg, steps=args.steps, warmup=args.warmup)
    sample = f"cfg4 first {SAMPLE_PLANES} z-planes (256x256x{SAMPLE_PLANES}, P7, {R} unknowns), one apply per step"
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4 P7 256^3 (bounded CPU sample)", "sample": sample},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1807_00410_b200 import _lib
    from paper_1807_00410_b200.configs import make_config, solve_spec
    from paper_1807_00410_b200.program import build_tables
    from paper_1807_00410_b200.solver import PnContext

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"note: --gpus {args.gpus} but WORLD_SIZE {world}; using WORLD_SIZE")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allmax(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_gen = time.perf_counter()
    cfg = make_config(4)
    spec = cfg.spec
    N = cfg.N
    nx, ny, nz = spec.res
    U = (N + 1) ** 2
    R = nx * ny * nz * U
    nzl = nz // world
    z0 = rank * nzl
    tables = build_tables(N)
    log(f"[rank {rank}] config generated in {time.perf_counter() - t_gen:.1f}s; R={R}")
    nccl_id = None
    if world > 1:
        buf = [None]
        if rank == 0:
            L = _lib.load()
            cbuf = np.zeros(128, np.uint8)
            _lib.check(L.pn_nccl_unique_id(cbuf.ctypes.data))
            buf[0] = bytes(cbuf)
        dist.broadcast_object_list(buf, src=0)
        nccl_id = buf[0]
    ctx = PnContext(tables, spec.res, spec.h, device=local, z0=z0, nz_local=nzl, rank=rank, world=world,
                    nccl_id=nccl_id)
    t0 = time.perf_counter()
    ctx.set_fields(spec)
    log(f"[rank {rank}] fields + setup {time.perf_counter() - t0:.2f}s")

    # ---- warm-up + timed applies (CUDA events inside pn_bench, max over ranks)
    ctx.bench(0, max(args.warmup, 3))
    barrier()
    launches0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        ms_apply = ctx.bench(0, args.steps)
        barrier()
    launches = ctx.kernel_launches() - launches0
    t_total_s = allmax(ms_apply * args.steps / 1e3)
    value = R * args.steps / t_total_s / 1e9
    ms_step = 1e3 * t_total_s / args.steps

    # ---- fused CG iteration (2 applies + updates + reductions)
    ctx.bench(1, 3)
    barrier()
    ms_iter = allmax(ctx.bench(1, max(5, args.steps // 2)))

    # ---- roofline of the apply kernel (per GPU, algorithmic bytes per launch)
    nvox_l = nx * ny * nzl
    bytes_apply = 8 * nvox_l * (2 * U + 2)
    peak, peak_src = measured_peak()
    achieved = bytes_apply / (ms_step / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": profile_traffic(), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_apply,
                "bytes_formula": "8*nvox*(2U+2): read u, write A u, read sigma_t and sigma_s"}

    # algorithmic bytes of one fused iteration (per GPU): two applies, r -= alpha w
    # (read r, w; write r) and x += alpha p; p = z + beta p (read x, p, z; write x, p)
    it_bytes = 2 * bytes_apply + 8 * 8 * nvox_l * U

    # ---- the other single-GPU configurations' apply throughput (rank 0, context)
    others = None
    if rank == 0 and not args.skip_others:
        others = {}
        for idx in (1, 2, 3):
            co = make_config(idx)
            ctx_o = PnContext(build_tables(co.N), co.spec.res, co.spec.h, device=local)
            ctx_o.set_fields(co.spec)
            ctx_o.bench(0, 5)
            ms_o = ctx_o.bench(0, 50)
            U_o = (co.N + 1) ** 2
            nv_o = int(np.prod(co.spec.res))
            gbs = 8 * nv_o * (2 * U_o + 2) / (ms_o / 1e3) / 1e9
            others[f"cfg{idx}"] = {"apply_ms": ms_o, "gunk_s": nv_o * U_o / (ms_o / 1e3) / 1e9,
                                   "achieved_gbs": gbs, "frac": gbs / peak,
                                   "note": "L2-resident working set" if idx <= 2 else "HBM-bound"}
            del ctx_o

    # ---- time-to-residual 1e-6 on configs 2 and 3 (single GPU, rank 0; config 3
    # with the sigma_t floor tau = 1 its vacuum needs, configs.solve_spec)
    ttr = None
    if rank == 0 and not args.skip_ttr:
        ttr = {}
        for idx, ref_it in ((2, 259), (3, None)):
            co = make_config(idx)
            so = solve_spec(co)
            ctx_t = PnContext(build_tables(co.N), so.res, so.h, device=local)
            ctx_t.set_fields(so)
            ctx_t.solve(tol=co.tol, max_iter=5)          # warm-up: graph capture, lazy loading
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep_t = ctx_t.solve(tol=co.tol, max_iter=co.max_iter)
            torch.cuda.synchronize()
            ttr[f"cfg{idx}"] = {"config": f"cfg{idx} P{co.N} {so.res[0]}^3", "tol": co.tol,
                                "seconds": time.perf_counter() - t0, "iterations": rep_t.iterations,
                                "converged": rep_t.converged, "sigma_t_floor": co.floor,
                                "reference_iterations": ref_it, "device_resident_inputs": True}
            del ctx_t
        torch.cuda.empty_cache()

    # ---- the paper's own problems (rank 0): time to residual 1e-10
    paper = None
    if rank == 0 and not args.skip_paper:
        paper = paper_workloads(local)
        torch.cuda.empty_cache()

    # ---- e2e: public API from host fields to host solution, fixed iterations
    e2e = None
    if not args.skip_e2e:
        iters = args.e2e_iters
        h2d = sum(np.asarray(v).nbytes for v in spec.fields.values() if np.ndim(v) > 0)
        d2h = 8 * R // world
        host_out = torch.empty(ctx.R_local, dtype=torch.float64, pin_memory=True)
        times = []
        for k in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            ctx.set_fields(spec)                                  # H2D fields + assembly
            x, rep = ctx.solve(tol=1e-300, max_iter=iters)        # CGNR on device
            host_out.copy_(x)                                     # D2H solution
            torch.cuda.synchronize()
            dt = allmax(time.perf_counter() - t0)
            if k > 0:
                times.append(dt)
            del x
        t_e2e = float(np.mean(times))
        e2e = {"value": 2 * R * iters / t_e2e / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d * world),
               "d2h_bytes_per_step": int(d2h * world), "seconds_per_step": t_e2e,
               "what": f"set_fields (H2D + assembly) + solve_normal_cg fixed {iters} iterations + D2H of x; "
                       f"value counts 2 applies per iteration"}

    # ---- CPU baseline (rank 0, N=1): the C port of the reference operator
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        rate, times, Rs, cores = cpu_oracle_rate(cfg, budget_s=args.cpu_budget)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"cfg4 first {SAMPLE_PLANES} z-planes (256x256x{SAMPLE_PLANES}, P7, {Rs} unknowns), "
                         f"{len(times)} applies, oracle/pn_oracle.c OpenMP"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg4: P7 (64 coeffs) 256^3 fp64, 4-octave cloud sigma_t<=100, albedo 0.99, "
                                   "HG g=0.8, one operator apply (A / A^T alternating) per step",
                       "unknowns": R, "parallelism": f"z-slab x{world}",
                       "l2": "inputs larger than L2 (8.6 GB per vector), no flush"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cg_iteration": {"ms": ms_iter, "gunk_s_2_applies": 2 * R / (ms_iter / 1e3) / 1e9,
                             "algorithmic_bytes": it_bytes, "achieved_gbs": it_bytes / (ms_iter / 1e3) / 1e9,
                             "frac": it_bytes / (ms_iter / 1e3) / 1e9 / peak,
                             "bytes_formula": "2 applies + 8 vector passes of 8R bytes (r -= alpha w: 3, "
                                              "x += alpha p; p = z + beta p: 5), per GPU",
                             "what": "one fused CGNR iteration: A p + ww, alpha, x/r update + rr, A^T r + zz/zzt, "
                                     "beta, p update"},
            "time_to_residual": ttr,
            "paper_workloads": paper,
            "other_configs_apply": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--skip-ttr", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-others", action="store_true")
    ap.add_argument("--skip-paper", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        log("warm-up raised to 3 (contract minimum)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
