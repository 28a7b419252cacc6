#!/usr/bin/env python
"""Benchmark of the B200 P_N solve path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--weak]

Workload (default, strong scaling): config 4 (P7, 256^3, 1.07e9 unknowns,
fp64) -- the largest single-GPU configuration and BASELINE.json's
strong-scaling config, z-slabs over N GPUs.  A step is one operator apply
(alternating A u and A^T u, the two sparse products of a CGNR iteration) on
device-resident dense pseudo-random vectors; value = global unknowns * K /
time (Gunknowns/s, whole job, max over ranks of CUDA-event time).  Every
vector is 8.6 GB, far above the 126 MB L2, so no L2 flush is needed.

Extra keys: a sustained apply figure (>= 2.5 s of applies, the board at its
power cap), the fused CG iteration against SURVEY.md s8d's two-sweep bytes,
config-4 time to residual 1e-6 on the N GPUs, a rank-count-independent solve
checksum (50 fixed iterations: sha256 over per-plane digests of x and of the
residual history -- identical for every N), config 5 (P5 512^3, 200 fixed
iterations) when N = 8, the end-to-end drop-in call solve_pn() from pinned
host fields to the host collocated grid, and at N = 1 the other configs, time
to residual on configs 1-3 and the paper's own problems.

--weak: the config-5 weak-scaling companion, a (256, 256, 256 N) P5 box on N
GPUs (one 256^3 slab each), applies as above.

--impl reference times the reference itself (baseline/_ref: pnrte installed
from /root/reference, its own assemble + scipy csr_matvec products) on the
box's host cores: a bounded sample of config 4 (its first 2 z-planes as a
256 x 256 x 2 problem, A and A^T alternating), plus BASELINE.md s3's config-2
companion (median A@x, time to residual 1e-6, 200 fixed iterations).
Without baseline/_ref it falls back to the C port of the reference operator
(oracle/), labelled kind "port".  Under torchrun only rank 0 works.

--gpus N without torchrun re-launches itself under torch.distributed.run.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import pathlib
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "P_N operator applies: Gunknowns/s (1/2/4/8 GPU) and time-to-residual 1e-6"
UNIT = "Gunk/s"
REF_DIR = ROOT / "baseline" / "_ref"
REF_SAMPLE_PLANES = 2
NCU_TRAFFIC = "profiles/ncu_apply_summary.json"


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
    """dram bytes per apply launch from the committed ncu --set full capture."""
    p = ROOT / NCU_TRAFFIC
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_launch"), d.get("source", NCU_TRAFFIC)
        except Exception:
            pass
    return None, None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during a timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

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
        sm, pw, mx, reasons = [], [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                pw.append(float(parts[6]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": float(np.median(pw)) if pw else None}


def cpu_info():
    model = None
    try:
        for ln in pathlib.Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def blas_info():
    try:
        from threadpoolctl import threadpool_info
        return [{k: i.get(k) for k in ("internal_api", "version", "num_threads", "architecture")}
                for i in threadpool_info()]
    except Exception as e:   # informational only
        return [{"error": str(e)}]


# --------------------------------------------------------------------------
# reference arm (CPU): the installed reference, else the C port
# --------------------------------------------------------------------------

def have_reference():
    return (REF_DIR / "pnrte" / "solver.py").exists()


def _import_reference():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import pnrte.solver as rs
    from pnrte.equations import build_pn
    from pnrte.problems import ProblemSpec as RefSpec
    from pnrte.stencil import compile_program
    return rs, build_pn, compile_program, RefSpec


def _ref_spec(RefSpec, spec, res):
    """A reference ProblemSpec with the given fields (same h, origin -1)."""
    h = spec.h
    fields = {k: (np.ascontiguousarray(v) if np.ndim(v) else v) for k, v in spec.fields.items()}
    return RefSpec(dim=3, origin=(-1.0,) * 3, extent=tuple(r * h for r in res), res=tuple(res), fields=fields)


def reference_cfg4_sample(steps, warmup, budget_s=None):
    """pnrte.solver.assemble + scipy products (A, A^T alternating, as in
    solve_normal_cg) on the first REF_SAMPLE_PLANES z-planes of config 4."""
    from paper_1807_00410_b200.configs import make_config
    rs, build_pn, compile_program, RefSpec = _import_reference()
    cfg = make_config(4, planes=(0, REF_SAMPLE_PLANES))
    spec = _ref_spec(RefSpec, cfg.spec, (256, 256, REF_SAMPLE_PLANES))
    t0 = time.perf_counter()
    system = rs.assemble(compile_program(build_pn(7, 3)), spec)
    t_asm = time.perf_counter() - t0
    A = system.A
    At = A.T.tocsr()
    R = A.shape[0]
    x = np.random.default_rng(0).normal(size=R)
    for k in range(warmup):
        (At if k & 1 else A) @ x
    times = []
    t_start = time.perf_counter()
    k = 0
    while True:
        t1 = time.perf_counter()
        (At if k & 1 else A) @ x
        times.append(time.perf_counter() - t1)
        k += 1
        if steps is not None and k >= steps:
            break
        if steps is None and (time.perf_counter() - t_start > budget_s and k >= 4):
            break
    sample = (f"cfg4 first {REF_SAMPLE_PLANES} z-planes as a 256x256x{REF_SAMPLE_PLANES} P7 problem "
              f"({R} unknowns, {A.nnz} stored entries), pnrte.solver.assemble + scipy csr_matvec, "
              f"A and A^T alternating, {len(times)} products (assembly {t_asm:.1f} s, untimed)")
    return R * len(times) / sum(times) / 1e9, times, sample


def reference_cfg2_companion(iters=200):
    """config 2 through the reference -- median A@x, time to
    residual 1e-6, and a fixed-iteration solve (the config-5 companion)."""
    from paper_1807_00410_b200.configs import make_config
    rs, build_pn, compile_program, RefSpec = _import_reference()
    cfg = make_config(2)
    spec = _ref_spec(RefSpec, cfg.spec, cfg.spec.res)
    t0 = time.perf_counter()
    system = rs.assemble(compile_program(build_pn(cfg.N, 3)), spec)
    t_asm = time.perf_counter() - t0
    A = system.A
    x = np.random.default_rng(0).normal(size=A.shape[0])
    ts = []
    for _ in range(6):
        t1 = time.perf_counter()
        A @ x
        ts.append(time.perf_counter() - t1)
    med = float(np.median(ts[1:]))
    t1 = time.perf_counter()
    _, rep = rs.solve_normal_cg(system, tol=cfg.tol, max_iter=cfg.max_iter)
    ttr = time.perf_counter() - t1
    t1 = time.perf_counter()
    _, rep2 = rs.solve_normal_cg(system, tol=1e-300, max_iter=iters)
    fixed = time.perf_counter() - t1
    R = A.shape[0]
    return {"config": "cfg2 P3 64^3", "assemble_s": t_asm, "apply_median_ms": 1e3 * med,
            "apply_gunk_s": R / med / 1e9,
            "time_to_residual": {"tol": cfg.tol, "seconds": ttr, "iterations": rep.iterations,
                                 "converged": rep.converged},
            f"fixed_{iters}_iterations": {"seconds": fixed, "iterations": rep2.iterations,
                                          "ms_per_iteration": 1e3 * fixed / max(rep2.iterations, 1)}}


def port_cfg4_sample(steps=None, budget_s=12.0, warmup=1, planes=8):
    """The C port of the reference operator (oracle/pn_oracle.c, OpenMP over
    rows, all host threads) on the first `planes` z-planes of config 4."""
    from oracle.oracle import StencilOracle
    from paper_1807_00410_b200.configs import make_config
    from paper_1807_00410_b200.problems import ProblemSpec
    from paper_1807_00410_b200.program import build_tables
    cfg = make_config(4, planes=(0, planes))
    h = cfg.spec.h
    f = {k: (np.ascontiguousarray(v) if np.ndim(v) else v) for k, v in cfg.spec.fields.items()}
    spec = ProblemSpec(dim=3, origin=(-1.0,) * 3, extent=(256 * h, 256 * h, planes * h), res=(256, 256, planes),
                       fields=f)
    o = StencilOracle(build_tables(7), spec)
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
    sample = f"cfg4 first {planes} z-planes (256x256x{planes}, P7, {o.R} unknowns), {len(times)} applies, " \
             f"oracle/pn_oracle.c OpenMP"
    return o.R * len(times) / sum(times) / 1e9, times, cores, sample


def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return
    # all host threads (torchrun sets OMP_NUM_THREADS=1 per rank; only rank 0 works here)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(os.cpu_count() or 1)
    except Exception:
        pass
    if have_reference():
        rate, times, sample = reference_cfg4_sample(args.steps, args.warmup)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
               "note": "scipy csr_matvec is single-threaded (sparsetools); OpenBLAS threads serve the "
                       "solver's dot products only", "host": cpu_info(), "threadpool_info": blas_info()}
        extra = {}
        if not args.skip_cfg2:
            extra["cfg2_companion"] = reference_cfg2_companion()
        port_rate, _, port_cores, port_sample = port_cfg4_sample(budget_s=6.0)
        extra["port"] = {"value": port_rate, "unit": UNIT, "cores": port_cores, "kind": "port",
                         "sample": port_sample}
    else:
        rate, times, cores, sample = port_cfg4_sample(steps=args.steps, warmup=args.warmup)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
               "note": "baseline/_ref (the installed reference) not present"}
        extra = {}
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4 P7 256^3 (bounded CPU sample)", "sample": cpu["sample"]},
        "cpu_baseline": cpu,
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **extra,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

class Dist:
    def __init__(self):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def allmax(self, v):
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out


def slab_planes(nz, world, rank):
    from paper_1807_00410_b200.distributed import slab_bounds
    z0, nzl = slab_bounds(nz, world, rank)
    return z0, nzl, (z0, min(z0 + nzl + 1, nz))


def plane_digests(x, nzl):
    """sha256 of every local z-plane of a reference-layout slab vector."""
    a = (x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)).reshape(nzl, -1)
    return [hashlib.sha256(a[k].tobytes()).hexdigest() for k in range(nzl)]


def global_digest(parts):
    """sha256 over the plane digests of all ranks in rank (= global plane) order."""
    return hashlib.sha256("".join(d for part in parts for d in part).encode()).hexdigest()


def solve_checksum(D, ctx, nzl, iters=50):
    """Fixed-iteration fast solve; sha256 over the per-plane digests of x in
    global plane order and over the residual history -- independent of the
    rank count when the solve is (slab reductions in plane order)."""
    x, rep = ctx.solve(tol=1e-300, max_iter=iters)
    h = global_digest(D.gather(plane_digests(x, nzl)))
    hist = hashlib.sha256(np.asarray(rep.normal_history, np.float64).tobytes()).hexdigest()
    return {"iterations": rep.iterations, "x_plane_digest_sha256": h, "normal_history_sha256": hist,
            "normal_history_last": rep.normal_history[-1] if rep.normal_history else None,
            "what": f"fast CGNR, {iters} fixed iterations from x0 = 0 on the floored config-4 system; "
                    "must be identical for every GPU count"}


def apply_bench(D, ctx, steps, warmup, clocks_index):
    ctx.bench(0, max(warmup, 3))
    D.barrier()
    l0 = ctx.kernel_launches()
    with ClockSampler(clocks_index) as clk:
        D.barrier()
        ms = ctx.bench(0, steps)
        D.barrier()
    launches = ctx.kernel_launches() - l0
    return D.allmax(ms), launches, clk.summary()


def pinned_spec(spec):
    """The same spec with its array fields in pinned host memory (the e2e
    inputs are copied from pinned buffers every step)."""
    import torch
    from dataclasses import replace
    f = {}
    keep = []
    for k, v in spec.fields.items():
        if np.ndim(v) == 0:
            f[k] = v
            continue
        t = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
        keep.append(t)
        f[k] = t.numpy()
    return replace(spec, fields=f), keep


def e2e_through_api(D, cfg, spec, iters, steps):
    """solve_pn() -- the north-star entry point -- from pinned host fields to
    the host collocated grid, fixed iterations; max over ranks of wall time."""
    import torch
    from paper_1807_00410_b200.solver import solve_pn
    pspec, keep = pinned_spec(spec)
    nx, ny, nz = spec.res
    nzl = nz // D.world
    U = (cfg.N + 1) ** 2
    out = torch.empty((nx, ny, nzl, U), dtype=torch.float64, pin_memory=True).numpy()
    h2d = sum(np.asarray(v).nbytes for v in pspec.fields.values() if np.ndim(v) > 0)
    times = []
    for k in range(steps + 1):
        D.barrier()
        t0 = time.perf_counter()
        _, rep = solve_pn(cfg.N, pspec, tol=1e-300, max_iter=iters, world=D.world, rank=D.rank, device=D.local,
                          out=out)
        torch.cuda.synchronize()
        dt = D.allmax(time.perf_counter() - t0)
        if k > 0:
            times.append(dt)
        torch.cuda.empty_cache()
    t = float(np.mean(times))
    R = nx * ny * nz * U
    return {"value": 2 * R * iters / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(D.allmax(h2d) * D.world),
            "d2h_bytes_per_step": int(out.nbytes * D.world), "seconds_per_step": t, "steps": len(times),
            "what": f"solver.solve_pn(N, spec, world, rank): pinned host fields -> H2D + assembly -> CGNR "
                    f"{iters} fixed iterations -> unstagger -> D2H of the collocated (nx, ny, nz/N, U) grid; "
                    f"value counts 2 applies per iteration"}


def run_ours(args):
    import torch
    from paper_1807_00410_b200.configs import make_config, solve_spec, weak_config
    from paper_1807_00410_b200.distributed import make_rank_context, share_nccl_id
    from paper_1807_00410_b200.program import build_tables

    D = Dist()
    world, rank = D.world, D.rank
    peak, peak_src = measured_peak()
    t_gen = time.perf_counter()
    if args.weak:
        nz_g = 256 * world
        z0, nzl, planes = slab_planes(nz_g, world, rank)
        cfg = weak_config(world, planes=planes)
    else:
        z0, nzl, planes = slab_planes(256, world, rank)
        cfg = make_config(4, planes=planes)
    spec = cfg.spec
    N = cfg.N
    nx, ny, nz = spec.res
    U = (N + 1) ** 2
    R = nx * ny * nz * U
    tables = build_tables(N)
    log(f"[rank {rank}] {spec.name} planes {planes} generated in {time.perf_counter() - t_gen:.1f}s; R={R}")
    nccl_id = share_nccl_id(rank, world) if world > 1 else None
    t0 = time.perf_counter()
    ctx = make_rank_context(tables, spec, rank, world, device=D.local, nccl_id=nccl_id)
    log(f"[rank {rank}] context + fields + setup {time.perf_counter() - t0:.2f}s")

    # ---- headline: K timed applies (A / A^T alternating), dense inputs
    ms_step, launches, clocks = apply_bench(D, ctx, args.steps, args.warmup, D.local)
    value = R / (ms_step / 1e3) / 1e9

    # ---- roofline of the apply kernel (per GPU, algorithmic bytes per launch)
    nvox_l = nx * ny * nzl
    bytes_apply = 8 * nvox_l * (2 * U + 2)
    achieved = bytes_apply / (ms_step / 1e3) / 1e9
    traffic, traffic_src = profile_traffic() if not args.weak else (None, None)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src and f"from_profile: {traffic_src}",
                "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_apply,
                "bytes_formula": "8*nvox*(2U+2) per GPU: read u, write A u, read sigma_t and sigma_s",
                "frac_of_nominal_8tbs": achieved / 8000.0}

    # ---- sustained: >= 2.5 s of applies (the board reaches its power cap)
    reps = max(args.steps, int(math.ceil(args.sustain_s * 1e3 / ms_step)))
    with ClockSampler(D.local) as clk_s:
        D.barrier()
        ms_sus = D.allmax(ctx.bench(0, reps))
        D.barrier()
    sustained = {"value": R / (ms_sus / 1e3) / 1e9, "unit": UNIT, "applies": reps, "ms_per_apply": ms_sus,
                 "seconds": reps * ms_sus / 1e3, "frac": bytes_apply / (ms_sus / 1e3) / 1e9 / peak,
                 "clocks": clk_s.summary()}

    # ---- fused CG iteration (2 applies + updates + reductions)
    ctx.bench(1, 3)
    D.barrier()
    ms_iter = D.allmax(ctx.bench(1, max(5, args.steps // 2)))
    fused_bytes = 88 * nvox_l * U + 32 * nvox_l           # two fused sweeps
    unfused_bytes = 2 * bytes_apply + 8 * 8 * nvox_l * U  # as launched: 2 applies + 8 vector passes
    gbs_fused = fused_bytes / (ms_iter / 1e3) / 1e9
    cg = {"ms": ms_iter, "gunk_s_2_applies": 2 * R / (ms_iter / 1e3) / 1e9,
          "frac": gbs_fused / peak, "achieved_gbs": gbs_fused, "algorithmic_bytes": fused_bytes,
          "bytes_formula": "88R + 32 nvox per GPU (SURVEY.md s8d: two fused sweeps, 11 vector passes + sigma)",
          "frac_as_launched": unfused_bytes / (ms_iter / 1e3) / 1e9 / peak,
          "bytes_as_launched": unfused_bytes,
          "as_launched_formula": "2 applies + 8 vector passes of 8R (r -= alpha w: 3; x += alpha p; p = z + beta p: 5)",
          "what": "one fused CGNR iteration: A p + ww, alpha, r update + rr, A^T r + zz, beta, x/p update"}

    # ---- converging solves on the floored system (sigma_t >= 1)
    check = ttr_main = None
    if not args.weak:
        ctx.set_fields(solve_spec(cfg))
        check = solve_checksum(D, ctx, nzl)
        if not args.skip_ttr4:
            ctx.solve(tol=cfg.tol, max_iter=5)        # graph capture, lazy allocations
            D.barrier()
            t0 = time.perf_counter()
            _, rep = ctx.solve(tol=cfg.tol, max_iter=cfg.max_iter)
            torch.cuda.synchronize()
            secs = D.allmax(time.perf_counter() - t0)
            ttr_main = {"config": f"cfg4 P7 256^3, {world} GPU(s)", "tol": cfg.tol, "seconds": secs,
                        "iterations": rep.iterations, "converged": rep.converged,
                        "normal_residual": rep.normal_residual, "sigma_t_floor": cfg.floor,
                        "ms_per_iteration": 1e3 * secs / max(rep.iterations, 1),
                        "device_resident_inputs": True}
    else:
        ctx.solve(tol=1e-300, max_iter=5)
        D.barrier()
        t0 = time.perf_counter()
        _, rep = ctx.solve(tol=1e-300, max_iter=cfg.max_iter)
        torch.cuda.synchronize()
        secs = D.allmax(time.perf_counter() - t0)
        ttr_main = {"config": f"weak P5 256x256x{256 * world}, {world} GPU(s)", "fixed_iterations": rep.iterations,
                    "seconds": secs, "ms_per_iteration": 1e3 * secs / max(rep.iterations, 1),
                    "solve_gunk_s_2_applies": 2 * R * rep.iterations / secs / 1e9}
    del ctx
    torch.cuda.empty_cache()

    # ---- e2e: the drop-in entry point from host fields to host grid
    e2e = None
    if not args.skip_e2e and not args.weak:
        e2e = e2e_through_api(D, cfg, spec, args.e2e_iters, args.e2e_steps)
        torch.cuda.empty_cache()

    # ---- config 5 (P5 512^3, 200 fixed iterations): 8 GPUs (38.7 GB per vector)
    cfg5 = None
    if (world == 8 or args.cfg5) and not args.weak:
        cfg5 = run_cfg5(D, peak, args.cfg5_n)

    # ---- single-GPU context: other configs, time to residual, paper problems
    others = ttr = paper = None
    if world == 1 and not args.weak:
        if not args.skip_others:
            others = other_configs(D.local, peak)
        if not args.skip_ttr:
            ttr = small_ttr(D.local)
        if not args.skip_paper:
            paper = paper_workloads(D.local)
        torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N = 1): the reference itself when installed
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        if have_reference():
            rate, times, sample = reference_cfg4_sample(None, 1, budget_s=args.cpu_budget)
            cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "reference", "sample": sample,
                   "host": cpu_info()}
        else:
            rate, times, cores, sample = port_cfg4_sample(budget_s=args.cpu_budget)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        tag = "weak" if args.weak else "strong"
        if args.weak:
            workload = (f"weak: P5 (36 coeffs) 256x256x{256 * world} fp64 (one 256^3 slab per GPU), config-3 "
                        f"cloud generator, one operator apply (A / A^T alternating) per step")
        else:
            workload = ("cfg4: P7 (64 coeffs) 256^3 fp64, 4-octave cloud sigma_t<=100, albedo 0.99, HG g=0.8, "
                        "one operator apply (A / A^T alternating) per step, dense pseudo-random inputs")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": tag,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "unknowns": R, "parallelism": f"z-slab x{world} (NCCL halos)",
                       "l2": "inputs larger than L2 (8.6 GB per vector at 1 GPU), no flush"},
            "roofline": roofline,
            "sustained": sustained,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "cg_iteration": cg,
            "solve_check": check,
            ("fixed_200_iterations" if args.weak else "time_to_residual_cfg4"): ttr_main,
            "cfg5": cfg5,
            "time_to_residual": ttr,
            "paper_workloads": paper,
            "other_configs_apply": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        D.dist.barrier()
        D.dist.destroy_process_group()


def run_cfg5(D, peak, n=512):
    """Config 5: P5 512^3 (4.83e9 unknowns), each rank generating only its
    planes; per-apply Gunk/s and the fixed 200-iteration CGNR.  (n < 512:
    the same code path on a smaller grid, for validation on fewer GPUs.)"""
    import torch
    from paper_1807_00410_b200.configs import make_config
    from paper_1807_00410_b200.distributed import make_rank_context, share_nccl_id
    from paper_1807_00410_b200.program import build_tables
    z0, nzl, planes = slab_planes(n, D.world, D.rank)
    t0 = time.perf_counter()
    cfg = make_config(5, n=n, planes=planes)
    nccl_id = share_nccl_id(D.rank, D.world) if D.world > 1 else None
    ctx = make_rank_context(build_tables(cfg.N), cfg.spec, D.rank, D.world, device=D.local, nccl_id=nccl_id)
    t_setup = D.allmax(time.perf_counter() - t0)
    nx, ny, nz = cfg.spec.res
    U = (cfg.N + 1) ** 2
    R = nx * ny * nz * U
    ms, _, clk = apply_bench(D, ctx, 20, 3, D.local)
    ctx.solve(tol=1e-300, max_iter=5)
    D.barrier()
    t0 = time.perf_counter()
    _, rep = ctx.solve(tol=1e-300, max_iter=cfg.max_iter)
    torch.cuda.synchronize()
    secs = D.allmax(time.perf_counter() - t0)
    bytes_apply = 8 * nx * ny * nzl * (2 * U + 2)
    out = {"config": f"cfg5 P5 {n}^3 on {D.world} GPUs", "unknowns": R, "setup_s": t_setup,
           "apply_ms": ms, "apply_gunk_s": R / (ms / 1e3) / 1e9,
           "roofline_per_gpu": {"achieved": bytes_apply / (ms / 1e3) / 1e9, "peak": peak,
                                "frac": bytes_apply / (ms / 1e3) / 1e9 / peak, "unit": "GB/s"},
           "fixed_iterations": rep.iterations, "solve_seconds": secs,
           "solve_gunk_s_2_applies": 2 * R * rep.iterations / secs / 1e9, "clocks": clk}
    del ctx
    torch.cuda.empty_cache()
    return out


def other_configs(device, peak):
    from paper_1807_00410_b200.configs import make_config
    from paper_1807_00410_b200.program import build_tables
    from paper_1807_00410_b200.solver import PnContext
    out = {}
    for idx in (1, 2, 3):
        co = make_config(idx)
        c = PnContext(build_tables(co.N), co.spec.res, co.spec.h, device=device)
        c.set_fields(co.spec)
        c.bench(0, 5)
        ms = c.bench(0, 50)
        U = (co.N + 1) ** 2
        nv = int(np.prod(co.spec.res))
        gbs = 8 * nv * (2 * U + 2) / (ms / 1e3) / 1e9
        out[f"cfg{idx}"] = {"apply_ms": ms, "gunk_s": nv * U / (ms / 1e3) / 1e9, "achieved_gbs": gbs,
                            "frac": gbs / peak, "note": "L2-resident working set" if idx <= 2 else "HBM-bound"}
        del c
    return out


def small_ttr(device):
    """Time to residual 1e-6 on configs 1-3 (device-resident inputs, after a
    5-iteration warm-up solve); the reference's iteration counts beside."""
    import torch
    from paper_1807_00410_b200.configs import make_config, solve_spec
    from paper_1807_00410_b200.program import build_tables
    from paper_1807_00410_b200.solver import PnContext
    gold = ROOT / "tests" / "golden"
    ref_it = {}
    try:
        cj = json.loads((gold / "configs.json").read_text())
        ref_it = {1: cj["cfg1"]["iterations"], 2: cj["cfg2"]["iterations"]}
        fs = json.loads((gold / "fullsize.json").read_text())
        if "cfg3" in fs:
            ref_it[3] = fs["cfg3"]["iterations"]
    except Exception:
        pass
    out = {}
    for idx in (1, 2, 3):
        co = make_config(idx)
        so = solve_spec(co)
        c = PnContext(build_tables(co.N), so.res, so.h, device=device)
        c.set_fields(so)
        c.solve(tol=co.tol, max_iter=5)
        torch.cuda.synchronize()
        secs = []
        while len(secs) < 3:
            t0 = time.perf_counter()
            _, rep = c.solve(tol=co.tol, max_iter=co.max_iter)
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - t0)
            if secs[0] > 1.0:
                break
        out[f"cfg{idx}"] = {"config": f"cfg{idx} P{co.N} {so.res[0]}^3", "tol": co.tol,
                            "seconds": float(np.median(secs)), "timed_solves": len(secs),
                            "iterations": rep.iterations, "converged": rep.converged, "sigma_t_floor": co.floor,
                            "reference_iterations": ref_it.get(idx),
                            "reference_iterations_source": {1: "live reference", 2: "live reference",
                                                            3: "C oracle (bit-identical restatement)"}[idx]}
        del c
    return out


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
    problems, device-resident inputs after a warm-up solve: the 2-D
    checkerboard and the 3-D point source (80^3, sigma_t 8, albedo 0.9)."""
    import torch
    from paper_1807_00410_b200.problems import make_checkerboard
    from paper_1807_00410_b200.program import build_tables
    from paper_1807_00410_b200.run import make_pointsource
    from paper_1807_00410_b200.solver import PnContext
    out = {}
    for name, kind, N, tol, paper_s in PAPER_RUNS:
        if kind == "cb":
            t = build_tables(N, dim=2)
            spec = make_checkerboard(71)
        else:
            t = build_tables(N)
            spec = make_pointsource(80)
        c = PnContext(t, spec.res, spec.h, device=device)
        c.set_fields(spec)
        c.solve(tol=tol, max_iter=5)
        torch.cuda.synchronize()
        secs = []
        while len(secs) < 3:
            t0 = time.perf_counter()
            _, rep = c.solve(tol=tol, max_iter=200000)
            torch.cuda.synchronize()
            secs.append(time.perf_counter() - t0)
            if secs[0] > 1.0:
                break
        sec = float(np.median(secs))
        out[name] = {"seconds": sec, "timed_solves": len(secs), "iterations": rep.iterations,
                     "converged": rep.converged, "tol": tol, "unknowns": c.R_local, "paper_cpu_seconds": paper_s,
                     "paper_over_ours": paper_s / sec}
        del c
    return out


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--weak", action="store_true", help="256x256x(256 N) P5 box, one 256^3 slab per GPU")
    ap.add_argument("--cfg5", action="store_true", help="config 5 at any N (needs >= 4 GPUs of memory)")
    ap.add_argument("--cfg5-n", type=int, default=512, help="config-5 grid edge (validation runs on fewer GPUs)")
    ap.add_argument("--e2e-iters", type=int, default=50)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--sustain-s", type=float, default=2.5)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--skip-ttr", action="store_true")
    ap.add_argument("--skip-ttr4", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-others", action="store_true")
    ap.add_argument("--skip-paper", action="store_true")
    ap.add_argument("--skip-cfg2", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(pathlib.Path(__file__).resolve()),
               *sys.argv[1:]]
        log("launching: " + " ".join(cmd))
        sys.exit(subprocess.call(cmd))
    if args.warmup < 3 and args.impl == "ours":
        log("warm-up raised to 3 (contract minimum)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        if args.gpus != int(os.environ.get("WORLD_SIZE", "1")):
            log(f"note: --gpus {args.gpus} but WORLD_SIZE {os.environ.get('WORLD_SIZE', '1')}")
        run_ours(args)


if __name__ == "__main__":
    main()
