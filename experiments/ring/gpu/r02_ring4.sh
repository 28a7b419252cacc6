mkdir -p gpurun_out
for v in ringy ringy74; do
  PNRTE_LIB=variants/$v/libpnrte_b200.so timeout 600 python experiments/ring/ring_probe.py --rings 1 > gpurun_out/r02_ring4_$v.jsonl 2> gpurun_out/r02_ring4_$v.err
  echo "$v rc=$?"
  grep -c '"same": true' gpurun_out/r02_ring4_$v.jsonl; grep '"same": false' gpurun_out/r02_ring4_$v.jsonl
  tail -n 1 gpurun_out/r02_ring4_$v.jsonl | cut -c1-700
  tail -n 3 gpurun_out/r02_ring4_$v.err
done
export PNRTE_LIB=variants/ringy/libpnrte_b200.so
PNRTE_SEG_RING=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_seg_ring -s 2 -c 2 -o gpurun_out/r02_ring4_ncu python tools/profile_apply.py --config 4 --reps 4 > gpurun_out/r02_ring4_ncu.log 2>&1
echo "ncu rc=$?"
unset PNRTE_LIB
python - <<'P'
import sys, json, pathlib
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import torch
from paper_1807_00410_b200.configs import make_config, solve_spec
from paper_1807_00410_b200.program import build_tables
from paper_1807_00410_b200.solver import PnContext
cfg = make_config(3); spec = solve_spec(cfg)
c = PnContext(build_tables(cfg.N), spec.res, spec.h); c.set_fields(spec)
def rel(a, b): return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))
xs, rep = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=8, blas_kernel=0)
out = {"ref_iterations": rep.iterations}
for T, k in ((8, 2), (8, 1), (64, 0), (1, 2)):
    xa, ra = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="faithful", blas_threads=T, blas_kernel=k)
    out[f"delta_T{T}_k{k}"] = [ra.iterations, rel(xa, xs)]
    print(json.dumps(out), flush=True)
xf, rf = c.solve(tol=cfg.tol, max_iter=cfg.max_iter, mode="fast")
out["fast"] = [rf.iterations, rel(xf, xs)]
xt, rt = c.solve(tol=1e-9, max_iter=cfg.max_iter, mode="fast")
out["tight_1e-9"] = [rt.iterations, rt.converged]
out["ref_vs_tight"] = rel(xs, xt); out["fast_vs_tight"] = rel(xf, xt)
print(json.dumps(out), flush=True)
pathlib.Path("gpurun_out/r02_cfg3_delta_probe.json").write_text(json.dumps(out))
P
