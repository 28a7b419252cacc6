"""Time set_fields (H2D of the fields + device assembly) on a config."""
import argparse, pathlib, sys, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
a = ap.parse_args()
cfg = make_config(a.config)
c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h)
for k in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    c.set_fields(cfg.spec)
    torch.cuda.synchronize()
    print(f"cfg{a.config} set_fields: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
