"""Sustained CG iteration rate on config 4: consecutive fixed-length solves
(500 iterations each, ~70 s in total) with nvidia-smi sampled alongside
(SM / memory clocks, power, temperatures, throttle reasons), to separate a
sustained-load clock effect from solver-loop overhead."""
import json, pathlib, subprocess, sys, threading, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext

Q = ("timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,"
     "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
     "clocks_event_reasons.hw_thermal_slowdown")
lines = []
proc = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={Q}", "--format=csv,noheader,nounits", "-lms", "1000"],
                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
threading.Thread(target=lambda: [lines.append(l.strip()) for l in proc.stdout], daemon=True).start()

cfg = make_config(4)
spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h)
c.set_fields(spec)
c.solve(tol=1e-300, max_iter=5)
torch.cuda.synchronize()
x = None
for chunk in range(8):
    t0 = time.perf_counter()
    x, rep = c.solve(tol=1e-300, max_iter=500, x0=x)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"chunk": chunk, "iterations": rep.iterations, "seconds": dt,
                      "ms_per_iteration": 1e3 * dt / rep.iterations, "t_since_start_s": time.perf_counter()}), flush=True)
time.sleep(1.5)
proc.terminate()
for l in lines:
    print("smi", l, flush=True)
