// Host side of the segmented fast operator: eligibility, parameter blocks,
// launch dispatch per order N, and the reference <-> segmented layout
// conversion (a 32 x U transpose inside each 32-voxel row).
#include <cuda_runtime.h>

#include <cmath>
#include <algorithm>
#include <cstring>
#include <cstdlib>

#include "generated/pn_seg_wmap.h"
#include "pn_seg.cuh"
#include "pn_seg_types.cuh"

namespace pn {

struct SegCtx {
    SegParams *pa = nullptr, *pt = nullptr;   // host parameter blocks (A, A^T)
    SegGeo g{};
    bool ok = false;
    double *sig_pad = nullptr;                // padded sigma_t / sigma_s slabs (nx % 32 != 0)
    size_t sig_pad_n = 0;                     // doubles per field
    FuseSched fr{};                           // fused residual update + A^T apply
    bool fr_ok = false;
};

static bool seg_padded(const pn_context *c) { return c->g.nx % 32 != 0; }

static bool seg_geometry_ok(const pn_context *c) {
    // a partial last row is zero-padded in the solve layout (single-slab contexts)
    return (c->g.nx % 32 == 0 || c->splane != c->g.plane) && c->N >= 1 && c->N <= 7 && c->canonical_diag &&
           c->U <= 64;
}

int pn_seg_red_blocks(const pn_context *c) {
    if (!seg_geometry_ok(c)) return 0;
    // one reduction partial per warp: segments x row blocks x warps per CTA
    const int warps = seg_rows(c->N) * (seg_pair(c->N) ? 2 : 1);
    return ((c->g.nx + 31) / 32) * ((c->g.ny + seg_rows(c->N) - 1) / seg_rows(c->N)) * warps;
}

// sigma slab ((nzl+1) planes, rows of nx) -> rows of sx >= nx, edge-replicated in x
__global__ void k_sig_pad(const double *__restrict__ src, double *__restrict__ dst, int nx, int sx, long long rows) {
    const long long n = rows * sx;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
        const long long row = t / sx;
        const int i = (int)(t - row * sx);
        dst[t] = src[row * nx + min(i, nx - 1)];
    }
}

// The generated code hard-wires the stencil structure of build_tables(N): every
// table entry must match it (target / source comp, direction, diagonal flag,
// |w| class and sign), otherwise the table operator runs instead.
static bool seg_structure_ok(const pn_context *c) {
    if ((int)c->h_par.size() != c->U) return false;
    for (int trans = 0; trans < 2; ++trans) {
        const int *sig = seg_sig(c->N, trans);
        int nw = 0;
        const int *rep = seg_wrep(c->N, trans, &nw);
        if (!sig || !rep || sig[0] != c->U) return false;
        const int U = sig[0], n = sig[1];
        const int *ptr = sig + 2, *oth = ptr + U + 1, *dir = oth + n, *dg = dir + n, *code = dg + n, *par = code + n;
        const std::vector<int> &hp = trans ? c->h_tptr : c->h_aptr, &ho = trans ? c->h_tsrc : c->h_atgt,
                               &hd = trans ? c->h_tdir : c->h_adir, &hg = trans ? c->h_tdiag : c->h_adiag;
        const std::vector<double> &hw = trans ? c->h_tw : c->h_aw;
        if ((int)ho.size() != n || (int)hw.size() != n || (int)hp.size() != U + 1) return false;
        for (int q = 0; q <= U; ++q)
            if (hp[q] != ptr[q]) return false;
        for (int q = 0; q < U; ++q)
            if (c->h_par[q] != par[q]) return false;
        for (int e = 0; e < n; ++e) {
            if (ho[e] != oth[e] || hd[e] != dir[e] || (hg[e] != 0) != (dg[e] != 0)) return false;
            if (dg[e]) continue;
            const int u = code[e] >> 1, neg = code[e] & 1;
            if (u >= nw || rep[u] >= n) return false;
            if (std::fabs(hw[e]) != std::fabs(hw[rep[u]]) || (int)std::signbit(hw[e]) != neg || hw[e] == 0.0) return false;
        }
    }
    return true;
}

bool pn_seg_ok(const pn_context *c) { return c->seg && ((SegCtx *)c->seg)->ok; }
bool pn_seg_fused_r_ok(const pn_context *c) { return pn_seg_ok(c) && ((SegCtx *)c->seg)->fr_ok; }

// Ticket schedule of k_seg_fr (pn_seg_types.cuh FuseSched).  Single slab, bulk
// path, orders whose CTAs have the 256 threads the residual update is blocked
// for; PNRTE_SEG_FUSE_R=0/1 forces.
static int seg_fuse_prepare(pn_context *c, SegCtx *sc, cudaStream_t s) {
    sc->fr_ok = false;
    const SegGeo &g = sc->g;
    const int rows = seg_rows(c->N), threads = 32 * rows * (seg_pair(c->N) ? 2 : 1);
    // default for P7 (measured: config 4, 17.13 -> 16.61 ms per iteration, time to 1e-6 68.5 -> 66.5 s,
    // same bits); the other orders' chunks are smaller than the register path of the embedded
    // update and stay on the launch chain unless forced
    // (and only where every chunk is four whole P7 rows, the shape the embedded register path takes:
    // ny a multiple of the rows per CTA; other extents run the slower block update and were not timed)
    const long long chunk0 = (g.plane + c->vec_bx - 1) / c->vec_bx;
    bool want = c->N == 7 && chunk0 == 8192 && g.plane % chunk0 == 0;
    if (const char *e = getenv("PNRTE_SEG_FUSE_R")) want = atoi(e) != 0;
    if (!want || !g.bulk || threads != 256 || c->world > 1 || g.nz < 3 || c->vec_bx < 1) return PN_OK;
    const int ntiles = (g.nyb + g.tyb - 1) / g.tyb;
    if (ntiles > FUSE_MAX_TILES) return PN_OK;
    FuseSched &f = sc->fr;
    unsigned *ctl = f.ctl, *flags = f.flags;
    const size_t nflags = (size_t)g.nz * c->vec_bx;
    // counter and flags start together: epoch 1 over all-zero flags (a re-set field comes
    // through here again with the epoch advanced, so both are rewound, not only the flags)
    if (!ctl) PN_CUDA(cudaMalloc(&ctl, 4 * sizeof(unsigned)));
    if (flags) cudaFree(flags);
    flags = nullptr;
    PN_CUDA(cudaMalloc(&flags, nflags * sizeof(unsigned)));
    const unsigned init[4] = {0u, 1u, 0u, 0u};   // 64-bit counter: ticket (low word), epoch (high word)
    PN_CUDA(cudaMemcpyAsync(ctl, init, sizeof(init), cudaMemcpyHostToDevice, s));
    PN_CUDA(cudaMemsetAsync(flags, 0, nflags * sizeof(unsigned), s));
    PN_CUDA(cudaStreamSynchronize(s));   // setup time; the solve may run on another stream
    f = FuseSched{};
    f.ctl = ctl;
    f.flags = flags;
    f.ntiles = ntiles;
    // planes the residual update runs ahead of the apply: far enough that an apply
    // unit's chunks were drawn more than a device-full of CTAs earlier
    f.D = 4;
    if (const char *e = getenv("PNRTE_SEG_FUSE_D")) f.D = std::max(2, atoi(e));
    if (f.D > g.nz - 1) f.D = g.nz - 1;
    f.vec_bx = c->vec_bx;
    f.chunk = (g.plane + c->vec_bx - 1) / c->vec_bx;
    const long long rowlen = (long long)c->U * 32;
    unsigned long long t = 0;
    int c_prev = -1;
    for (int T = 0; T < ntiles; ++T) {
        const int jb0 = T * g.tyb, jb1 = std::min(g.nyb, jb0 + g.tyb);
        const int j_halo = std::min(jb1 * rows, g.ny - 1);   // one row line beyond the tile
        long long c_hi = (((long long)j_halo + 1) * g.nseg * rowlen - 1) / f.chunk;
        if (T == ntiles - 1 || c_hi > c->vec_bx - 1) c_hi = c->vec_bx - 1;
        f.tile_start[T] = (unsigned)t;
        f.c_lo[T] = c_prev + 1;
        f.n_u[T] = (int)(c_hi - c_prev);
        f.n_a[T] = g.nseg * (jb1 - jb0);
        c_prev = (int)c_hi;
        t += (unsigned long long)f.D * f.n_u[T] + (unsigned long long)g.nz * f.n_a[T];
    }
    if (t >= (1ULL << 31)) return PN_OK;
    f.tile_start[ntiles] = (unsigned)t;
    sc->fr_ok = true;
    return PN_OK;
}

int pn_seg_prepare(pn_context *c, cudaStream_t s) {
    SegCtx *sc = (SegCtx *)c->seg;
    if (!sc) {
        sc = new SegCtx();
        c->seg = sc;
    }
    sc->ok = false;
    if (!seg_geometry_ok(c) || !c->uniform_phase || c->red_bx < pn_seg_red_blocks(c)) return PN_OK;
    if (c->f.kind[0] != 2 || c->f.kind[1] != 2) return PN_OK;   // sigma arrays (uniform ones are materialised)
    if (!seg_structure_ok(c)) return PN_OK;
    if (!sc->pa) {
        sc->pa = new SegParams();
        sc->pt = new SegParams();
    }
    memset(sc->pa, 0, sizeof(SegParams));
    memset(sc->pt, 0, sizeof(SegParams));
    // distinct weight magnitudes: |w_e * h^-1| of a representative entry e
    for (int trans = 0; trans < 2; ++trans) {
        int nw = 0;
        const int *rep = seg_wrep(c->N, trans, &nw);
        const std::vector<double> &tw = trans ? c->h_tw : c->h_aw;
        SegParams *pp = trans ? sc->pt : sc->pa;
        if (!rep || nw > SEG_MAXW) return PN_OK;
        for (int u = 0; u < nw; ++u) {
            if (rep[u] >= (int)tw.size()) return PN_OK;
            pp->w[u] = std::fabs(tw[rep[u]]);
        }
    }
    std::vector<double> lamp(c->U);
    PN_CUDA(cudaMemcpy(lamp.data(), c->tb.lamp, c->U * sizeof(double), cudaMemcpyDeviceToHost));
    for (int q = 0; q < c->U; ++q) sc->pa->lamp[q] = sc->pt->lamp[q] = lamp[q];
    SegGeo &g = sc->g;
    g.U = c->U; g.nx = c->g.nx; g.ny = c->g.ny; g.nz = c->g.nz; g.z0 = c->g.z0; g.nzl = c->g.nzl;
    g.nseg = (c->g.nx + 31) / 32;
    g.sx = seg_padded(c) ? g.nseg * 32 : c->g.nx;
    g.nyb = (c->g.ny + seg_rows(c->N) - 1) / seg_rows(c->N);
    // planes above ~12 MB: march in z inside y-tiles of ~32 rows so the z
    // neighbour rows stay in L2; smaller planes: plain (x, y, z) order
    const double plane_mb = (double)c->g.plane * sizeof(double) / 1e6;
    g.tyb = plane_mb > 12.0 ? std::min(g.nyb, std::max(1, 32 / seg_rows(c->N))) : g.nyb;
    g.plane = c->splane;   // solve layout (== c->g.plane unless padded)
    g.pvox = c->g.pvox;
    if (seg_padded(c)) {
        const long long rows = (long long)(c->g.nzl + 1) * c->g.ny;
        const size_t n = (size_t)rows * g.sx;
        if (sc->sig_pad_n != n) {
            if (sc->sig_pad) cudaFree(sc->sig_pad);
            sc->sig_pad = nullptr;
            PN_CUDA(cudaMalloc(&sc->sig_pad, 2 * n * sizeof(double)));
            sc->sig_pad_n = n;
        }
        for (int f = 0; f < 2; ++f) {
            k_sig_pad<<<1184, 256, 0, s>>>(c->f.data[f], sc->sig_pad + f * n, c->g.nx, g.sx, rows);
            PN_CUDA(cudaGetLastError());
        }
    }
    // bulk (TMA) staging + in-CTA y neighbours where the vector streams from
    // HBM (measured +2-4 % at 128^3 and 256^3); cp.async where it sits in L2
    // (64^3: the bulk path measured ~10 % slower).  PNRTE_SEG_BULK=0/1 forces.
    const double vec_mb = (double)c->g.nzl * c->g.plane * sizeof(double) / 1e6;
    g.bulk = vec_mb > 96.0;
    if (const char *e = getenv("PNRTE_SEG_BULK")) g.bulk = atoi(e) != 0;
    sc->ok = true;
    PN_TRY(seg_fuse_prepare(c, sc, s));
    return PN_OK;
}

int pn_seg_apply(pn_context *c, int trans, const double *x, double *y, int red, const double *minv, double *zt,
                 bool gated, cudaStream_t s, int kl0, int npl, int kst) {
    SegCtx *sc = (SegCtx *)c->seg;
    SegGeo g = sc->g;
    g.kl0 = kl0;
    g.kst = kst;
    g.npl = npl < 0 ? c->g.nzl : npl;
    if (g.npl <= 0) return PN_OK;
    const SegParams &prm = trans ? *sc->pt : *sc->pa;
    const long long stride = (long long)c->g.nz * c->red_bx;
    const State *st = gated ? c->state : nullptr;
    const double *sig_t = c->f.data[0], *sig_s = c->f.data[1];
    if (sc->sig_pad) {
        sig_t = sc->sig_pad;
        sig_s = sc->sig_pad + sc->sig_pad_n;
    }
    int rc;
    switch (c->N) {
#define PN_N(n)                                                                                                 \
    case n:                                                                                                     \
        rc = seg_launch<n>(prm, g, trans, red, minv != nullptr, x, y, minv, zt, sig_t, sig_s, c->partials, \
                           stride, c->red_bx, st, s);                                                           \
        break;
        PN_N(1) PN_N(2) PN_N(3) PN_N(4) PN_N(5) PN_N(6) PN_N(7)
#undef PN_N
        default: set_error("segmented kernel: unsupported order"); return PN_ERR_UNSUPPORTED;
    }
    c->launches++;
    return rc;
}

// r -= alpha w ; z = A^T r with the fused reductions, one launch (k_seg_fr)
int pn_seg_apply_fused_r(pn_context *c, double *r, const double *w, double *z, const double *minv, double *zt,
                         cudaStream_t s) {
    SegCtx *sc = (SegCtx *)c->seg;
    SegGeo g = sc->g;
    g.kl0 = 0;
    g.kst = 1;
    g.npl = c->g.nzl;
    const long long stride = (long long)c->g.nz * c->red_bx;
    const double *sig_t = c->f.data[0], *sig_s = c->f.data[1];
    if (sc->sig_pad) {
        sig_t = sc->sig_pad;
        sig_s = sc->sig_pad + sc->sig_pad_n;
    }
    int rc;
    switch (c->N) {
#define PN_N(n)                                                                                                  \
    case n:                                                                                                      \
        rc = seg_launch_fused_r<n>(*sc->pt, g, sc->fr, minv != nullptr, r, w, z, minv, zt, sig_t, sig_s,        \
                                   c->partials, stride, c->red_bx, c->state, s);                                 \
        break;
        PN_N(1) PN_N(2) PN_N(3) PN_N(4) PN_N(5) PN_N(6) PN_N(7)
#undef PN_N
        default: set_error("fused kernel: unsupported order"); return PN_ERR_UNSUPPORTED;
    }
    c->launches++;
    return rc;
}

// dir 0: reference layout (voxel-major, comp-minor) -> segmented; 1: back.
// One block per 32-voxel row; a partial last row (w < 32 voxels, nx % 32 != 0)
// is zero-filled beyond w in the segmented layout and its padding is dropped
// on the way back.
__global__ void k_seg_convert(int dir, int U, int nx, int nseg, const double *__restrict__ src,
                              double *__restrict__ dst) {
    extern __shared__ double tile[];   // 32 x (U+1)
    const long long row = blockIdx.x;  // (kl, j) line * nseg + seg
    const long long line = row / nseg;
    const int seg = (int)(row - line * nseg);
    const int w = min(32, nx - seg * 32);
    const long long rbase = (line * nx + seg * 32) * U;   // reference layout
    const long long sbase = row * 32 * U;                 // segmented layout
    const int n = 32 * U;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        int l, c;
        double v;
        if (dir == 0) {
            l = t / U; c = t - l * U;
            v = l < w ? src[rbase + t] : 0.0;
        } else {
            c = t >> 5; l = t & 31;
            v = src[sbase + t];
        }
        tile[l * (U + 1) + c] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        int l, c;
        if (dir == 0) {
            c = t >> 5; l = t & 31;
            dst[sbase + t] = tile[l * (U + 1) + c];
        } else {
            l = t / U; c = t - l * U;
            if (l < w) dst[rbase + t] = tile[l * (U + 1) + c];
        }
    }
}

int pn_seg_convert(pn_context *c, int dir, const double *src, double *dst, cudaStream_t s) {
    if (src == dst) { set_error("pn_seg_convert: in-place"); return PN_ERR_INVALID; }
    const int nseg = (c->g.nx + 31) / 32;
    long long rows = (long long)c->g.nzl * c->g.ny * nseg;
    size_t sm = (size_t)32 * (c->U + 1) * sizeof(double);
    k_seg_convert<<<(unsigned)rows, 256, sm, s>>>(dir, c->U, c->g.nx, nseg, src, dst);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

void pn_seg_release(pn_context *c) {
    SegCtx *sc = (SegCtx *)c->seg;
    if (!sc) return;
    delete sc->pa;
    delete sc->pt;
    if (sc->sig_pad) cudaFree(sc->sig_pad);
    if (sc->fr.ctl) cudaFree(sc->fr.ctl);
    if (sc->fr.flags) cudaFree(sc->fr.flags);
    delete sc;
    c->seg = nullptr;
}

}  // namespace pn
