import sys, pathlib
sys.path.insert(0, "/root/repo")
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(2); spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h); c.set_fields(spec)
c.solve(tol=1e-300, max_iter=20)
torch.cuda.synchronize()
