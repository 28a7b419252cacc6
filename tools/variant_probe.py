"""A/B of library builds (PNRTE_LIB=variants/<v>/libpnrte_b200.so): config-4
apply on dense operands (40-apply burst, 800-apply sustained with NVML clocks),
on all-zero operands (unthrottled kernel), the fused CG iteration, and the
sha256 of a bulk-path apply on a small grid (variants must agree bit for bit).

    for v in base priv; do PNRTE_LIB=variants/$v/libpnrte_b200.so python tools/variant_probe.py $v; done
"""
import hashlib
import json
import os
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tools"))
import torch  # noqa: E402

from cases import probe_vector, rand_spec  # noqa: E402
from paper_1807_00410_b200.configs import make_config  # noqa: E402
from paper_1807_00410_b200.program import build_tables  # noqa: E402
from paper_1807_00410_b200.solver import PnContext  # noqa: E402
from power_probe import Nvml  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("PNRTE_LIB", "default")
    out = {"variant": name}
    os.environ["PNRTE_SEG_BULK"] = "1"
    digests = []
    for N in (3, 5, 7):
        spec = rand_spec(N, (64, 9, 6), 40 + N)
        c = PnContext(build_tables(N), spec.res, spec.h)
        c.set_fields(spec)
        x = probe_vector(c.R_local)
        for tr in (0, 1):
            digests.append(hashlib.sha256(c.apply(x, tr).cpu().numpy().tobytes()).hexdigest()[:16])
        del c
    os.environ.pop("PNRTE_SEG_BULK")
    out["bulk_apply_sha"] = digests
    cfg = make_config(4)
    c = PnContext(build_tables(cfg.N), cfg.spec.res, cfg.spec.h)
    c.set_fields(cfg.spec)
    R = c.R_local
    c.bench(0, 5)
    with Nvml() as mon:
        for label, what, reps in (("dense_burst", 7, 40), ("dense_sustained", 7, 800), ("zero_burst", 6, 40),
                                  ("zero_sustained", 6, 400)):
            c.bench(what, 0)
            time.sleep(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ms = c.bench(0, reps)
            t1 = time.perf_counter()
            out[label] = {"ms": ms, "gunk_s": R / ms / 1e6, **mon.window(t0, t1)}
        c.bench(7, 0)
        time.sleep(1.0)
        c.bench(1, 3)
        t0 = time.perf_counter()
        out["cg_iteration_ms"] = c.bench(1, 40)
        out["cg_iteration_clock"] = mon.window(t0, time.perf_counter())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
