import sys; sys.path.insert(0,'/root/repo')
import torch
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(2); t = build_tables(cfg.N)
ctx = PnContext(t, cfg.spec.res, cfg.spec.h); ctx.set_fields(cfg.spec)
csr, q = ctx.assemble_csr("dirichlet")
x = torch.randn(csr.R_local, dtype=torch.float64, device="cuda")
for _ in range(3): csr.apply(x)
torch.cuda.synchronize()
