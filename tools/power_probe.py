"""Config-4 apply: dense vs all-zero operands, short burst vs sustained, with
SM clock and board power sampled by NVML every ~5 ms -- separates a
power-cap effect from a kernel effect (round-1 headline ran on the RHS, which
is zero outside 32 of 1.07e9 entries).

    python tools/power_probe.py [--config 4] > profiles/r02_power_probe.jsonl
"""
import argparse
import json
import pathlib
import sys
import threading
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1807_00410_b200.configs import make_config  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402


class Nvml:
    def __init__(self, index=0, period=0.005):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.period = period
        self.samples = []
        self.on = False

    def __enter__(self):
        self.on = True
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        nv, h = self.nv, self.h
        while self.on:
            try:
                self.samples.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetPowerUsage(h) / 1e3))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.on = False
        self.t.join()

    def window(self, t0, t1):
        s = [x for x in self.samples if t0 <= x[0] <= t1]
        if not s:
            return {}
        clk = [x[1] for x in s]
        pw = [x[2] for x in s]
        return {"n": len(s), "sm_mhz_median": float(np.median(clk)), "sm_mhz_min": min(clk),
                "power_w_median": float(np.median(pw)), "power_w_max": max(pw)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    a = ap.parse_args()
    cfg = make_config(a.config)
    c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h)
    c.set_fields(cfg.spec)
    R = c.R_local
    c.bench(0, 5)
    with Nvml() as mon:
        for data in ("dense", "zero", "dense"):
            c.bench(7 if data == "dense" else 6, 0)
            for reps in (40, 800):
                time.sleep(1.0)   # cool down / leave the cap
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                ms = c.bench(0, reps)
                t1 = time.perf_counter()
                print(json.dumps({"config": a.config, "data": data, "applies": reps, "ms_per_apply": ms,
                                  "gunk_s": R / (ms / 1e3) / 1e9, **mon.window(t0, t1)}), flush=True)
        c.bench(7, 0)
        for what, name in ((1, "cg_iteration"), (4, "r_update"), (5, "xp_update"), (2, "apply_fused_red")):
            time.sleep(1.0)
            c.bench(what, 3)
            t0 = time.perf_counter()
            ms = c.bench(what, 40)
            t1 = time.perf_counter()
            print(json.dumps({"config": a.config, "what": name, "ms": ms, **mon.window(t0, t1)}), flush=True)


if __name__ == "__main__":
    main()
