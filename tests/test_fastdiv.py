"""The multiply-high division behind the segmented kernel's CTA -> row-block
map (FastDiv in csrc/pn_seg_types.cuh): the host-side magic numbers, with the
device's __umulhi emulated in 64-bit, give n / d exactly for 0 <= n < 2^31.
Compiled with g++ from the header itself (no GPU)."""

import pathlib
import shutil
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
CSRC = ROOT / "paper_1807_00410_b200" / "csrc"

SRC = r"""
#define __host__
#define __device__
typedef struct CUstream_st *cudaStream_t;
#include <cstdint>
#include <cstdio>
#include <random>
#include "pn_seg_types.cuh"
static unsigned fdiv_host(unsigned n, const pn::FastDiv &f) {
    return f.m ? (unsigned)(((unsigned long long)n * f.m) >> 32) >> f.s : n;
}
int main() {
    std::mt19937_64 rng(7);
    long long checked = 0;
    auto check = [&](unsigned n, unsigned d, const pn::FastDiv &f) {
        ++checked;
        if (fdiv_host(n, f) != n / d) { std::printf("FAIL n=%u d=%u\n", n, d); return false; }
        return true;
    };
    for (unsigned d = 1; d < 70000 + 2000; ++d) {
        const unsigned dd = d < 70000 ? d : (unsigned)(rng() % 0x7fffffffu) + 1u;
        const pn::FastDiv f = pn::make_fastdiv(dd);
        if (f.d != dd) { std::printf("FAIL d field\n"); return 1; }
        const unsigned edge[] = {0u, 1u, dd - 1, dd, dd + 1, 2 * dd - 1, 0x7fffffffu, 0x7ffffffeu};
        for (unsigned n : edge)
            if (n <= 0x7fffffffu && !check(n, dd, f)) return 1;
        for (int k = 0; k < 64; ++k)
            if (!check((unsigned)(rng() & 0x7fffffffu), dd, f)) return 1;
    }
    std::printf("OK %lld\n", checked);
    return 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_fastdiv_exact(tmp_path):
    src = tmp_path / "fastdiv.cpp"
    src.write_text(SRC)
    exe = tmp_path / "fastdiv"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", str(CSRC), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK")
