import sys; sys.path.insert(0,'/root/repo')
from paper_1807_00410_b200.configs import make_config
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(4)
c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h); c.set_fields(cfg.spec)
for what in (0, 2, 3, 0, 2, 3):
    c.bench(what, 4); ms = c.bench(what, 20)
    print("what", what, f"{ms*1e3:.1f} us")
