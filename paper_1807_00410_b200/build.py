"""Build the sm_100a shared library libpnrte_b200.so in-tree (nvcc, no torch JIT).

Translation units compile in parallel; the faithful-arithmetic unit
(pn_kernels.cu) is compiled with -fmad=false so no multiply-add is ever
contracted (numpy / scipy sparsetools round every product).
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent
CSRC = HERE / "csrc"
OUT_DIR = pathlib.Path(os.environ.get("PNRTE_BUILD_DIR", HERE / "_lib"))
EXTRA = os.environ.get("PNRTE_NVCC_FLAGS", "").split()
LIB = OUT_DIR / "libpnrte_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        inc = pathlib.Path(base) / "nccl" / "include"
        lib = pathlib.Path(base) / "nccl" / "lib"
        if (inc / "nccl.h").exists() and lib.exists():
            return inc, lib
    return pathlib.Path("/usr/include"), pathlib.Path("/usr/lib/x86_64-linux-gnu")


def sources():
    units = [CSRC / "pn_kernels.cu", CSRC / "pn_runtime.cu", CSRC / "pn_seg.cu", CSRC / "pn_csr.cu", CSRC / "pn_post.cu"]
    units += sorted((CSRC / "generated").glob("pn_seg_N*.cu"))
    return units


def _flags(src, inc):
    f = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", str(CSRC), "-I", str(inc), *ARCH]
    f += EXTRA
    if src.name in ("pn_kernels.cu", "pn_csr.cu", "pn_post.cu"):
        f += ["-fmad=false", "-Xcompiler", "-ffp-contract=off"]   # device and host twins (k_setup constants)
    return f


def build(verbose=False, force=False):
    from . import codegen
    codegen.generate()
    inc, libdir = _nccl_dirs()
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    deps = list(CSRC.glob("*.cuh")) + list((CSRC / "generated").glob("*.cuh")) + list((CSRC / "generated").glob("*.h"))
    newest_dep = max(p.stat().st_mtime for p in deps)
    for src in sources():
        obj = OUT_DIR / (src.stem + ".o")
        objs.append(obj)
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_dep):
            jobs.append([NVCC, *_flags(src, inc), "-c", str(src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        list(ex.map(run, jobs))
    if jobs or not LIB.exists():
        nccl_so = next(iter(sorted(libdir.glob("libnccl.so*"))), None)
        link = [NVCC, "-shared", *ARCH, "-o", str(LIB), *map(str, objs), "-lcudart_static"]
        if nccl_so is not None:
            link += ["-L", str(libdir), f"-Xlinker=-l:{nccl_so.name}", f"-Xlinker=-rpath={libdir}"]
        else:
            link += ["-lnccl"]
        run(link)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
