import sys; sys.path.insert(0,'/root/repo')
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(4, n=128)
c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h); c.set_fields(cfg.spec)
c.bench(0, 2); c.bench(2, 2)
