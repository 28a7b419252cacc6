"""Time the fast operator apply of several configs for each library variant."""
import os, subprocess, sys, json, pathlib
ROOT = pathlib.Path(__file__).resolve().parents[1]
variants = sys.argv[1].split(",")
cases = [("4", "128"), ("3", "128"), ("2", "0"), ("1", "0"), ("4", "256")]
for v in variants:
    for cfg, n in cases:
        env = dict(os.environ, PNRTE_LIB=str(ROOT / "variants" / v / "libpnrte_b200.so"))
        args = [sys.executable, str(ROOT / "tools" / "profile_apply.py"), "--config", cfg, "--reps", "20"]
        if n != "0": args += ["--n", n]
        out = subprocess.run(args, env=env, capture_output=True, text=True)
        line = (out.stdout.strip().splitlines() or ["ERR " + out.stderr[-300:]])[-1]
        print(v, line, flush=True)
