// Generic sm_100a kernels of the P_N solve path: field upload, assembly of
// the diagonal / RHS, the faithful (scipy-order) operator, the table-driven
// fast operator for grids the segmented kernel does not cover, elementwise
// CG updates, deterministic reductions, the OpenBLAS ddot emulation used by
// the faithful mode, the solver scalar steps and unstagger.
//
// Reference behaviour mirrored (pkg/src/pnrte/):
//   assemble            solver.py:96-186   (k_setup: diag/RHS in tree order, pinned rows)
//   csr_matvec          solver.py:209-255  (k_apply_table: ascending column order, no FMA)
//   solve_normal_cg     solver.py:189-257  (k_vec + k_scalar)
//   unstagger           solver.py:275-296  (k_unstagger)
// This file is compiled with -fmad=false: faithful arithmetic must never be
// contracted into FMAs (numpy / sparsetools do mul then add).  Kernels that
// may use FMA live in pn_seg.cu.
#include <atomic>
#include <cuda_runtime.h>
#include <cstdint>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <cooperative_groups.h>

#include "pn_internal.cuh"
#include "pn_vec.cuh"
#include "pn_seg_types.cuh"

namespace pn {

namespace cg = cooperative_groups;

__device__ __forceinline__ bool stopped(const State *st) { return *(volatile const int *)&st->done != 0; }

// ------------------------------------------------------------ field slab --
// src: [i][j][k] C-order global field.  dst: planes kl = 0..nzl (global
// k = min(z0+kl, nz-1), the +1 plane is the edge-replicated sample of
// solver.py:62-64), x fastest.  32x32 smem transpose per j.
__global__ void k_field_slab(const double *__restrict__ src, double *__restrict__ dst, int nx, int ny, int nz,
                             int z0, int nplanes, int src_k0, int src_nk) {
    __shared__ double tile[32][33];
    const int j = blockIdx.z;
    const int i0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {
        int i = i0 + r, kl = k0 + threadIdx.x;
        if (i < nx && kl < nplanes) {
            int kg = min(z0 + kl, nz - 1);
            tile[r][threadIdx.x] = src[((long long)i * ny + j) * src_nk + (kg - src_k0)];
        }
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        int kl = k0 + r, i = i0 + threadIdx.x;
        if (i < nx && kl < nplanes) dst[((long long)kl * ny + j) * nx + i] = tile[threadIdx.x][r];
    }
}

int launch_field_slab(pn_context *c, int slot, const double *src, double *dst, cudaStream_t s, int src_k0,
                      int src_nk) {
    const Geo &g = c->g;
    int nplanes = g.nzl + 1;
    if (src_nk <= 0) { src_k0 = 0; src_nk = g.nz; }   // the global field
    dim3 grid((g.nx + 31) / 32, (nplanes + 31) / 32, g.ny), block(32, 8);
    k_field_slab<<<grid, block, 0, s>>>(src, dst, g.nx, g.ny, g.nz, g.z0, nplanes, src_k0, src_nk);
    PN_CUDA(cudaGetLastError());
    return PN_OK;
}

__global__ void k_fill(double *p, long long n, double v) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_fill_hash(double *p, long long n, long long offset, unsigned long long seed) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + 0x9E3779B97F4A7C15ULL * (unsigned long long)(offset + i + 1);   // splitmix64
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        z ^= z >> 31;
        p[i] = (double)(z >> 11) * 0x1.0p-52 - 1.0;
    }
}

int launch_fill_hash(double *p, long long n, long long offset, unsigned long long seed, cudaStream_t s) {
    k_fill_hash<<<1184, 256, 0, s>>>(p, n, offset, seed);
    PN_CUDA(cudaGetLastError());
    return PN_OK;
}

int launch_fill(double *p, long long n, double v, cudaStream_t s) {
    k_fill<<<1184, 256, 0, s>>>(p, n, v);
    PN_CUDA(cudaGetLastError());
    return PN_OK;
}

// ---------------------------------------------------------------- setup --
__device__ __forceinline__ double fsample(const Fields &F, const Geo &g, int slot, int i, int j, int kl, int site) {
    int kd = F.kind[slot];
    if (kd == 0) return 0.0;
    if (kd == 1) return F.scalar[slot];
    int ii = min(i + (site & 1), g.nx - 1);
    int jj = min(j + ((site >> 1) & 1), g.ny - 1);
    int kk = kl + ((site >> 2) & 1);   // plane nzl exists (clamped at upload)
    return F.data[slot][(long long)kk * g.pvox + (long long)jj * g.nx + ii];
}

__device__ double eval_terms(const Tables &T, const Fields &F, const Geo &g, int t0, int t1, int i, int j, int kl) {
    double acc = 0.0;
    for (int t = t0; t < t1; ++t) {
        int nf = T.nf[t], f = 0;
        double v;
        if (T.hascoef[t]) v = T.tcoef[t];
        else { v = fsample(F, g, T.tf[2 * t], i, j, kl, T.tsite[2 * t]); f = 1; }
        for (; f < nf; ++f) v = __dmul_rn(v, fsample(F, g, T.tf[2 * t + f], i, j, kl, T.tsite[2 * t + f]));
        acc = (t == t0) ? v : __dadd_rn(acc, v);
    }
    return acc;
}

__device__ __forceinline__ int boundary_bits(const Geo &g, int i, int j, int kg) {
    return (i == g.nx - 1) | ((j == g.ny - 1) << 1) | ((kg == g.nz - 1) << 2);
}

// one thread per (local voxel, comp): diag (optional) and RHS (solver.py:136-181);
// pin = 0 for Neumann (no pinned rows, solver.py:133-135)
// Grid (row blocks of a plane, planes): index arithmetic stays 32-bit inside a
// plane (a plane holds < 2^31 rows), 64-bit divisions per row made the kernel
// integer-bound (8.6 GB of RHS in 35 ms at config 4).
__global__ void k_setup(Tables T, Fields F, Geo g, double *diag, double *rhs, int pin, const int *__restrict__ rmode,
                        const double *__restrict__ rconst) {
    const int kl = blockIdx.y;
    const unsigned rp = blockIdx.x * blockDim.x + threadIdx.x;   // row within the plane
    if (rp >= (unsigned)g.plane) return;
    const unsigned v = rp / (unsigned)g.U;
    const int c = (int)(rp - v * (unsigned)g.U);
    const int i = (int)(v % (unsigned)g.nx);
    const int j = (int)(v / (unsigned)g.nx);
    const long long row = (long long)kl * g.plane + rp;
    int bb = boundary_bits(g, i, j, g.z0 + kl);
    if (diag) diag[row] = eval_terms(T, F, g, T.d_ptr[c], T.d_ptr[c + 1], i, j, kl);
    if (rhs) {
        double r = 0.0;
        if (rmode[c]) r = rconst[c];
        else if (T.r_ptr[c + 1] > T.r_ptr[c]) r = -eval_terms(T, F, g, T.r_ptr[c], T.r_ptr[c + 1], i, j, kl);
        rhs[row] = (pin && (T.par[c] & bb)) ? 0.0 : r;
    }
}

// Host twin of eval_terms for comps whose factors are all constants (missing
// or uniform fields): the same multiplies and adds in the same order, IEEE
// double on both sides (this unit is compiled without contraction), so the
// constant equals what every thread would compute.
static void rhs_constants(pn_context *c) {
    const int U = c->U;
    c->h_rmode.assign(U, 0);
    c->h_rconst.assign(U, 0.0);
    for (int comp = 0; comp < U; ++comp) {
        const int t0 = c->h_rptr[comp], t1 = c->h_rptr[comp + 1];
        bool konst = true;
        double acc = 0.0;
        for (int t = t0; t < t1 && konst; ++t) {
            auto fs = [&](int slot, bool &ok) {
                const int kd = c->f.kind[slot];
                if (kd == 2) ok = false;
                return kd == 1 ? c->f.scalar[slot] : 0.0;
            };
            const int nf = c->h_nf[t];
            int f = 0;
            double v;
            if (c->h_hascoef[t]) v = c->h_tcoef[t];
            else { v = fs(c->h_tf[2 * t], konst); f = 1; }
            for (; f < nf; ++f) v = v * fs(c->h_tf[2 * t + f], konst);
            acc = (t == t0) ? v : acc + v;
        }
        if (!konst) continue;
        c->h_rmode[comp] = 1;
        c->h_rconst[comp] = t1 > t0 ? -acc : 0.0;
    }
}

int launch_setup(pn_context *c, bool want_diag, bool want_rhs, cudaStream_t s, double *rhs_out, int pin) {
    int bs = 256;
    if (c->g.plane >= (1LL << 31)) { set_error("setup: z-plane too large"); return PN_ERR_UNSUPPORTED; }
    dim3 grid((unsigned)((c->g.plane + bs - 1) / bs), (unsigned)c->g.nzl);
    double *rhs = want_rhs ? (rhs_out ? rhs_out : c->b.p) : nullptr;
    if (want_rhs) {
        rhs_constants(c);
        PN_CUDA(cudaMemcpyAsync(c->d_rmode, c->h_rmode.data(), c->U * sizeof(int), cudaMemcpyHostToDevice, s));
        PN_CUDA(cudaMemcpyAsync(c->d_rconst, c->h_rconst.data(), c->U * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    k_setup<<<grid, bs, 0, s>>>(c->tb, c->f, c->g, want_diag ? c->diag : nullptr, rhs, pin, c->d_rmode, c->d_rconst);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

// ------------------------------------------------------ table operator --
__constant__ int c_dx[7] = {0, -1, 1, 0, 0, 0, 0};
__constant__ int c_dy[7] = {0, 0, 0, -1, 1, 0, 0};
__constant__ int c_dz[7] = {0, 0, 0, 0, 0, -1, 1};

// red: 0 none, 1 = sum y^2 -> slot 0, 2 = z/zt: sum z*zt -> slot 2, sum z^2 -> slot 1
// faithful: sequential mul-then-add in table order starting from 0 (scipy
// csr_matvec); otherwise FMA and the recomputed or stored diagonal.
template <bool FAITHFUL, bool RECOMPUTE_DIAG>
__global__ void __launch_bounds__(256) k_apply_table(Tables T, Fields F, Geo g, int trans, int squared,
                                                     const double *__restrict__ x, double *__restrict__ y,
                                                     const double *__restrict__ diag, int red, const double *minv,
                                                     double *zt, double *partials, long long slot_stride, int rb,
                                                     const State *st, int kl0, int kst, int pst, FastDiv du,
                                                     FastDiv dnx) {
    if (st && stopped(st)) return;
    extern __shared__ unsigned char smem_raw[];
    const int U = g.U;
    const int ne = trans ? T.n_t : T.n_a;
    double *sw = (double *)smem_raw;
    int *sptr = (int *)(sw + ne);
    int *soth = sptr + U + 1, *sdir = soth + ne, *sisd = sdir + ne;
    int *spar = sisd + ne;
    double *slamp = (double *)(((uintptr_t)(spar + U) + 15) & ~(uintptr_t)15);
    int *sdg = (int *)(slamp + U);   // fast path: the diagonal entry of each row, -1 if none
    {
        const int *p_ = trans ? T.t_ptr : T.a_ptr;
        const int *o_ = trans ? T.t_src : T.a_tgt;
        const int *d_ = trans ? T.t_dir : T.a_dir;
        const int *i_ = trans ? T.t_diag : T.a_diag;
        const double *w_ = trans ? T.t_w : T.a_w;
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            sw[e] = w_[e]; soth[e] = o_[e]; sdir[e] = d_[e]; sisd[e] = i_[e];
        }
        for (int e = threadIdx.x; e <= U; e += blockDim.x) sptr[e] = p_[e];
        for (int e = threadIdx.x; e < U; e += blockDim.x) { spar[e] = T.par[e]; slamp[e] = T.lamp[e]; }
        for (int cc = threadIdx.x; cc < U; cc += blockDim.x) {
            int dg = -1;
            for (int e = p_[cc]; e < p_[cc + 1]; ++e)
                if (i_[e]) dg = e;
            sdg[cc] = dg;
        }
    }
    __syncthreads();
    const int kl = kl0 + blockIdx.y * kst;
    const long long chunk = (g.plane + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(g.plane, r0 + chunk);
    double acc_r[2] = {0.0, 0.0};
    const int kg = g.z0 + kl;
    for (long long rp = r0 + threadIdx.x; rp < r1; rp += blockDim.x) {
        const long long row = (long long)kl * g.plane + rp;
        // (voxel, comp) and (i, j) by multiply-high division (plane < 2^31, checked at launch)
        const unsigned vp = fdiv((unsigned)rp, du);
        const int c = (int)((unsigned)rp - vp * (unsigned)U);
        const unsigned jq = fdiv(vp, dnx);
        const int i = (int)(vp - jq * (unsigned)g.nx), j = (int)jq;
        const int bb = boundary_bits(g, i, j, kg);
        const bool pinned_c = (spar[c] & bb) != 0;
        double sum = 0.0;
        if (!FAITHFUL && sdg[c] >= 0) {
            // fast: the diagonal term once per row, ahead of the (lane-divergent)
            // entry loop, instead of whenever some lane of the warp reaches it
            double a;
            if (RECOMPUTE_DIAG) {
                const int pc = spar[c];
                double st_ = 0.0, ss_ = 0.0;
                int n = 0;
                for (int s = 0; s < 8; ++s) {
                    if (s & ~pc) continue;
                    st_ += fsample(F, g, 0, i, j, kl, s);
                    ss_ += fsample(F, g, 1, i, j, kl, s);
                    ++n;
                }
                const double inv = 1.0 / n;
                a = st_ * inv - slamp[c] * (ss_ * inv);
            } else {
                a = diag[row];
            }
            sum = a * x[row];
        }
        for (int e = sptr[c]; e < sptr[c + 1]; ++e) {
            const int o = soth[e];
            double a, xv;
            if (sisd[e]) {
                if (!FAITHFUL) continue;   // done above
                if (RECOMPUTE_DIAG) {
                    // avg over the staggered site set, then diag = avg_t - lamp*avg_s
                    const int pc = spar[c];
                    double st_ = 0.0, ss_ = 0.0;
                    int n = 0;
                    for (int s = 0; s < 8; ++s) {
                        if (s & ~pc) continue;
                        st_ += fsample(F, g, 0, i, j, kl, s);
                        ss_ += fsample(F, g, 1, i, j, kl, s);
                        ++n;
                    }
                    const double inv = 1.0 / n;
                    a = st_ * inv - slamp[c] * (ss_ * inv);
                } else {
                    a = diag[row];
                }
                xv = x[row];
            } else {
                const int d = sdir[e];
                const int ii = i + c_dx[d], jj = j + c_dy[d], kk = kg + c_dz[d];
                if (pinned_c || ii < 0 || jj < 0 || kk < 0 || ii >= g.nx || jj >= g.ny || kk >= g.nz) continue;
                const int nbb = (ii == g.nx - 1) | ((jj == g.ny - 1) << 1) | ((kk == g.nz - 1) << 2);
                if (spar[o] & nbb) continue;
                a = sw[e];
                xv = x[((long long)(kk - g.z0) * g.pvox + (long long)jj * g.nx + ii) * U + o];
            }
            if (FAITHFUL) {
                if (squared) a = __dmul_rn(a, a);
                sum = __dadd_rn(sum, __dmul_rn(a, xv));
            } else {
                sum = fma(a, xv, sum);
            }
        }
        y[row] = sum;
        if (red == 1) {
            acc_r[0] = fma(sum, sum, acc_r[0]);
        } else if (red == 2) {
            double t = minv ? sum * minv[row] : sum;
            if (zt) zt[row] = t;
            acc_r[0] = fma(sum, t, acc_r[0]);
            acc_r[1] = fma(sum, sum, acc_r[1]);
        }
    }
    if (red) {
        const long long idx = (long long)kg * pst + blockIdx.x;
        if (red == 1) {
            double v[1] = {acc_r[0]};
            const int sl[1] = {0};
            block_partials<1>(v, partials, sl, slot_stride, idx);
        } else {
            double v[2] = {acc_r[0], acc_r[1]};
            const int sl[2] = {2, 1};
            block_partials<2>(v, partials, sl, slot_stride, idx);
        }
    }
}

static size_t table_smem(const pn_context *c, int trans) {
    int ne = trans ? c->tb.n_t : c->tb.n_a;
    size_t b = (size_t)ne * 8 + (size_t)(c->U + 1) * 4 + (size_t)ne * 12 + (size_t)c->U * 4;
    b = (b + 15) & ~(size_t)15;
    return b + (size_t)c->U * 8 + (size_t)c->U * 4 + 16;
}

static long long slot_stride(const pn_context *c) { return (long long)c->g.nz * c->red_bx; }

int launch_apply_table(pn_context *c, int trans, int faithful, int squared, const double *x, double *y, int red,
                       const double *minv, double *zt, cudaStream_t s, bool gated, int kl0, int npl, int kst) {
    if (npl < 0) npl = c->g.nzl;
    if (npl <= 0) return PN_OK;
    dim3 grid(c->vec_bx, npl);
    size_t sm = table_smem(c, trans);
    const State *st = gated ? c->state : nullptr;
    bool recompute = !faithful && c->canonical_diag && c->uniform_phase;
    if (!recompute && !c->diag_ready) { set_error("internal: diagonal not assembled"); return PN_ERR_INVALID; }
    if (c->g.plane >= (1LL << 31)) { set_error("table operator: z-plane too large"); return PN_ERR_UNSUPPORTED; }
    const FastDiv du = make_fastdiv((unsigned)c->U), dnx = make_fastdiv((unsigned)c->g.nx);
    if (faithful) {
        k_apply_table<true, false><<<grid, 256, sm, s>>>(c->tb, c->f, c->g, trans, squared, x, y, c->diag, red, minv,
                                                         zt, c->partials, slot_stride(c), c->vec_bx, st, kl0, kst, c->red_bx, du, dnx);
    } else if (recompute) {
        k_apply_table<false, true><<<grid, 256, sm, s>>>(c->tb, c->f, c->g, trans, 0, x, y, c->diag, red, minv, zt,
                                                         c->partials, slot_stride(c), c->vec_bx, st, kl0, kst, c->red_bx, du, dnx);
    } else {
        k_apply_table<false, false><<<grid, 256, sm, s>>>(c->tb, c->f, c->g, trans, 0, x, y, c->diag, red, minv, zt,
                                                          c->partials, slot_stride(c), c->vec_bx, st, kl0, kst, c->red_bx, du, dnx);
    }
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

int launch_apply_faithful(pn_context *c, int trans, int squared, const double *x, double *y, cudaStream_t s,
                          bool gated) {
    return launch_apply_table(c, trans, 1, squared, x, y, 0, nullptr, nullptr, s, gated, 0, -1, 1);
}

// ----------------------------------------------------------- vector ops --
// geometry of the vectors the current operation works on: the segmented solve
// layout (x padded to whole rows) during fast segmented solves, else the
// reference layout
static Geo vgeo(const pn_context *c) {
    Geo g = c->g;
    g.plane = c->vplane();
    return g;
}

__global__ void __launch_bounds__(256) k_vec(int op, Geo g, double *y, const double *a, const double *b, State *st,
                                             double *partials, long long slot_stride, int rb, int gated) {
    if (gated && stopped(st)) return;
    const int kl = blockIdx.y;
    const long long chunk = (g.plane + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(g.plane, r0 + chunk);
    const long long base = (long long)kl * g.plane;
    const double alpha = st ? st->alpha : 0.0, beta = st ? st->beta : 0.0;
    for (long long rp = r0 + threadIdx.x; rp < r1; rp += blockDim.x) {
        const long long i = base + rp;
        switch (op) {
            case V_COPY: y[i] = a[i]; break;
            case V_ZERO: y[i] = 0.0; break;
            case V_FILL_ONE: y[i] = 1.0; break;
            case V_SUB: y[i] = __dsub_rn(a[i], b[i]); break;
            case V_MUL: y[i] = __dmul_rn(a[i], b[i]); break;
            case V_RECIP_DIAG: { double d = a[i]; y[i] = __ddiv_rn(1.0, d == 0.0 ? 1.0 : d); } break;
            case V_AXPY_ALPHA: y[i] = __dadd_rn(y[i], __dmul_rn(alpha, a[i])); break;
            case V_AXMY_ALPHA: y[i] = __dsub_rn(y[i], __dmul_rn(alpha, a[i])); break;
            case V_P_UPDATE: y[i] = __dadd_rn(a[i], __dmul_rn(beta, y[i])); break;
        }
    }
}

// fast r -= alpha w with ||r||^2 partials (slot 3); x is updated later,
// fused with the p update (k_xp), with the same alpha and p (bitwise equal)
__global__ void __launch_bounds__(256) k_r(Geo g, double *__restrict__ r, const double *__restrict__ w,
                                           const State *st, double *partials, long long slot_stride, int rb, int pst) {
    if (stopped(st)) return;
    r_update_block<false>(g.plane, (g.plane + rb - 1) / rb, (int)blockIdx.x, (int)blockIdx.y, g.z0, r, w, st->alpha,
                          partials, slot_stride, pst);
}

// fast x += alpha p_old ; p = zt + beta p_old (p only while not stopped).
// Runs after the stop test of the iteration, gated on st->xupd, which the
// iteration's beta step sets and the next alpha step clears.
__global__ void __launch_bounds__(256) k_xp(Geo g, double *__restrict__ x, double *__restrict__ p,
                                            const double *__restrict__ zt, const State *st, int rb) {
    if (*(volatile const int *)&st->xupd == 0) return;
    const bool upd_p = !stopped(st);
    const int kl = blockIdx.y;
    const long long chunk = (g.plane + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(g.plane, r0 + chunk);
    const long long base = (long long)kl * g.plane;
    const double alpha = st->alpha, beta = st->beta;
    long long i0 = base + r0, i1 = base + r1;
#ifndef PN_VEC_SCALAR
    const bool paired = !(g.plane & 1) && !((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(p) |
                                             reinterpret_cast<uintptr_t>(zt)) & 15);
    if (paired && (i0 & 1) && i0 < i1) {
        if (threadIdx.x == 0) {
            const double pv = p[i0];
            x[i0] = fma(alpha, pv, x[i0]);
            if (upd_p) p[i0] = fma(beta, pv, zt[i0]);
        }
        ++i0;
    }
    const long long np = paired ? (i1 - i0) >> 1 : 0;
    double2 *x2 = reinterpret_cast<double2 *>(x + i0);
    double2 *p2 = reinterpret_cast<double2 *>(p + i0);
    const double2 *z2 = reinterpret_cast<const double2 *>(zt + i0);
    if (upd_p) {
#pragma unroll 4
        for (long long q = threadIdx.x; q < np; q += blockDim.x) {
            const double2 pv = p2[q], zv = z2[q];
            double2 xv = x2[q];
            xv.x = fma(alpha, pv.x, xv.x);
            xv.y = fma(alpha, pv.y, xv.y);
            x2[q] = xv;
            p2[q] = make_double2(fma(beta, pv.x, zv.x), fma(beta, pv.y, zv.y));
        }
    } else {
#pragma unroll 4
        for (long long q = threadIdx.x; q < np; q += blockDim.x) {
            const double2 pv = p2[q];
            double2 xv = x2[q];
            xv.x = fma(alpha, pv.x, xv.x);
            xv.y = fma(alpha, pv.y, xv.y);
            x2[q] = xv;
        }
    }
    i0 += 2 * np;
#endif
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double pv = p[i];
        x[i] = fma(alpha, pv, x[i]);
        if (upd_p) p[i] = fma(beta, pv, zt[i]);
    }
}

// deterministic dot products into slot (per plane-block partials)
__global__ void __launch_bounds__(256) k_dot(Geo g, const double *__restrict__ a, const double *__restrict__ b,
                                             int slot, double *partials, long long slot_stride, int rb,
                                             const State *st, int pst) {
    if (st && stopped(st)) return;
    const int kl = blockIdx.y;
    const long long chunk = (g.plane + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(g.plane, r0 + chunk);
    const long long base = (long long)kl * g.plane;
    double acc = 0.0;
    for (long long rp = r0 + threadIdx.x; rp < r1; rp += blockDim.x) acc = fma(a[base + rp], b[base + rp], acc);
    double v[1] = {acc};
    const int sl[1] = {slot};
    block_partials<1>(v, partials, sl, slot_stride, (long long)(g.z0 + kl) * pst + blockIdx.x);
}

int launch_vec(pn_context *c, int op, double *y, const double *a, const double *b, cudaStream_t s, bool gated) {
    dim3 grid(c->vec_bx, c->g.nzl);
    k_vec<<<grid, 256, 0, s>>>(op, vgeo(c), y, a, b, c->state, c->partials, slot_stride(c), c->vec_bx, gated ? 1 : 0);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

int launch_r_update(pn_context *c, cudaStream_t s) {
    dim3 grid(c->vec_bx, c->g.nzl);
    k_r<<<grid, 256, 0, s>>>(vgeo(c), c->r.p, c->w.p, c->state, c->partials, slot_stride(c), c->vec_bx, c->red_bx);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

int launch_xp_update(pn_context *c, const double *zt, cudaStream_t s) {
    dim3 grid(c->vec_bx, c->g.nzl);
    k_xp<<<grid, 256, 0, s>>>(vgeo(c), c->x.p, c->p.p, zt, c->state, c->vec_bx);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

int launch_dot(pn_context *c, const double *a, const double *b, int slot, cudaStream_t s, bool gated) {
    dim3 grid(c->vec_bx, c->g.nzl);
    k_dot<<<grid, 256, 0, s>>>(vgeo(c), a, b, slot, c->partials, slot_stride(c), c->vec_bx, gated ? c->state : nullptr,
                               c->red_bx);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

// ------------------------------------------------- OpenBLAS ddot emulation --
// OpenBLAS 0.3.30 ddot (numpy's x @ y and np.linalg.norm):
// T-way chunking width = ceil(rem/(T-t)) when n > 10000, chunk results
// summed in order from 0.0.  Per chunk, SkylakeX kernel: 4x8-lane FMA
// accumulators over 32-blocks, fold hi+lo to 4x4 lanes, 4x4-lane FMA over
// the 16-block remainder, lanewise ((a0+a1)+a2)+a3, (s0+s2)+(s1+s3), FMA
// scalar tail.  Haswell kernel: 4x4-lane FMA over 16-blocks, fold to 2 lanes,
// (h0+h1)+(h2+h3), lane sum, mul-then-add tail.  One block per chunk; its
// warp 0 carries the lane accumulators.
__device__ __forceinline__ void chunk_range(long long n, int T, int t, long long &off, long long &width) {
    long long rem = n;
    off = 0;
    width = 0;
    for (int q = 0; q <= t; ++q) {
        width = (rem + (T - q) - 1) / (T - q);
        if (width > rem) width = rem;
        if (q < t) { off += width; rem -= width; }
    }
}

// The lane accumulators are sequential FMA chains (that order IS the result), so
// the speed comes from keeping the chain fed: all DD_THREADS threads of the
// block stream the chunk through a DD_STAGES-deep cp.async ring of DD_TILE-element
// tiles in shared memory, and warp 0 runs the chain over each landed tile
// (one dependent DFMA per 32 / 16 elements, operands from shared memory).  A
// one-warp version that loaded straight from HBM ran ~0.5 us per chain step:
// 0.15 s per dot product at config 3 (75.5 M elements, 8 chunks).
__device__ __forceinline__ double tree256(double *sh);

constexpr int DD_TILE = 2048, DD_STAGES = 5, DD_THREADS = 256;
constexpr size_t DD_SMEM = (size_t)DD_STAGES * 2 * DD_TILE * sizeof(double);

__device__ __forceinline__ void dd_cp8(double *dst_smem, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst_smem)),
                 "l"(src));
}

// acc = fma(x[i + lane], y[i + lane], acc) for i = 0, W, 2W, ... < nm (nm % W == 0), lanes < W of warp 0
template <int W>
__device__ __forceinline__ double dd_chain(const double *__restrict__ x, const double *__restrict__ y, long long nm,
                                           double *sm) {
    const int tid = threadIdx.x;
    const long long ntiles = (nm + DD_TILE - 1) / DD_TILE;
    auto issue = [&](long long t) {
        if (t < ntiles) {
            const long long base = t * DD_TILE;
            const int cnt = (int)min((long long)DD_TILE, nm - base);
            double *xs = sm + (size_t)(t % DD_STAGES) * 2 * DD_TILE, *ys = xs + DD_TILE;
            for (int e = tid; e < cnt; e += DD_THREADS) {
                dd_cp8(xs + e, x + base + e);
                dd_cp8(ys + e, y + base + e);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    for (int t = 0; t < DD_STAGES - 1; ++t) issue(t);
    double acc = 0.0;
    for (long long t = 0; t < ntiles; ++t) {
        issue(t + DD_STAGES - 1);   // refills the buffer consumed in iteration t - 1
        asm volatile("cp.async.wait_group %0;\n" ::"n"(DD_STAGES - 1));
        __syncthreads();
        if (tid < W) {
            const int cnt = (int)min((long long)DD_TILE, nm - t * DD_TILE);
            const double *xs = sm + (size_t)(t % DD_STAGES) * 2 * DD_TILE + tid, *ys = xs + DD_TILE;
#pragma unroll 8
            for (int i = 0; i < cnt; i += W) acc = fma(xs[i], ys[i], acc);
        }
        __syncthreads();
    }
    return acc;
}

__global__ void __launch_bounds__(DD_THREADS) k_ddot_emul(const double *__restrict__ x, const double *__restrict__ y,
                                                          long long n, int T, int kernel, double *out,
                                                          const State *st) {
    extern __shared__ __align__(16) double dd_sm[];
    if (st && stopped(st)) return;
    const int lane = threadIdx.x & 31;
    long long off, w;
    if (n <= 10000 || T <= 1) { off = 0; w = n; }
    else chunk_range(n, T, blockIdx.x, off, w);
    x += off;
    y += off;
    double dot = 0.0;
    if (kernel == 0) {
        const long long n32 = w & ~31LL, n16 = w & ~15LL;
        const int q = lane >> 3, l8 = lane & 7;
        // a8[q][l8] += x[i + 8 q + l8] * y[...] over the 32-blocks (8 q + l8 == lane)
        const double a8 = dd_chain<32>(x, y, n32, dd_sm);
        if (threadIdx.x >= 32) return;
        // fold to 4 lanes per accumulator: a4[q][l] = a8[q][l] + a8[q][l+4]
        double hi = __shfl_down_sync(0xffffffffu, a8, 4);
        double a4 = __dadd_rn(a8, hi);   // valid for l8 < 4
        if (n32 < n16 && l8 < 4) a4 = fma(x[n32 + 4 * q + l8], y[n32 + 4 * q + l8], a4);
        // lanewise ((a0+a1)+a2)+a3 over q, lane l8<4 of each q group
        double a_1 = __shfl_sync(0xffffffffu, a4, 8 + (lane & 3));
        double a_2 = __shfl_sync(0xffffffffu, a4, 16 + (lane & 3));
        double a_3 = __shfl_sync(0xffffffffu, a4, 24 + (lane & 3));
        double s = __dadd_rn(__dadd_rn(__dadd_rn(a4, a_1), a_2), a_3);   // valid at lanes 0..3
        double s0 = __shfl_sync(0xffffffffu, s, 0), s1 = __shfl_sync(0xffffffffu, s, 1);
        double s2 = __shfl_sync(0xffffffffu, s, 2), s3 = __shfl_sync(0xffffffffu, s, 3);
        if (lane == 0) {
            dot = n16 ? __dadd_rn(__dadd_rn(s0, s2), __dadd_rn(s1, s3)) : 0.0;
            for (long long i = n16; i < w; ++i) dot = fma(y[i], x[i], dot);
        }
    } else if (kernel == 2) {
        // not an OpenBLAS kernel: a pairwise-style order (thread-strided FMA partials,
        // 256-leaf tree) for measuring the reference's own sensitivity to the dot
        // order (SURVEY.md s8c protocol 3: "a different (pairwise) dot order")
        __shared__ double sh[DD_THREADS];
        double a = 0.0;
        for (long long i = threadIdx.x; i < w; i += DD_THREADS) a = fma(x[i], y[i], a);
        sh[threadIdx.x] = a;
        __syncthreads();
        dot = tree256(sh);
    } else {
        const long long n16 = w & ~15LL;
        // a4[q][l4] over the 16-blocks (4 q + l4 == lane, lanes 0..15)
        const double a4 = dd_chain<16>(x, y, n16, dd_sm);
        if (threadIdx.x >= 32) return;
        double hi = __shfl_down_sync(0xffffffffu, a4, 2);
        double h = __dadd_rn(a4, hi);   // valid at l4 < 2
        double h1 = __shfl_sync(0xffffffffu, h, 4 + (lane & 1));
        double h2 = __shfl_sync(0xffffffffu, h, 8 + (lane & 1));
        double h3 = __shfl_sync(0xffffffffu, h, 12 + (lane & 1));
        double t = __dadd_rn(__dadd_rn(h, h1), __dadd_rn(h2, h3));   // lanes 0,1
        double t0 = __shfl_sync(0xffffffffu, t, 0), t1 = __shfl_sync(0xffffffffu, t, 1);
        if (lane == 0) {
            dot = n16 ? __dadd_rn(t0, t1) : 0.0;
            for (long long i = n16; i < w; ++i) dot = __dadd_rn(dot, __dmul_rn(y[i], x[i]));
        }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = dot;
}

int launch_ddot_emul(pn_context *c, const double *a, const double *b, long long n, int slot, int threads, int kernel,
                     cudaStream_t s, bool gated) {
    int nb = (n <= 10000 || threads <= 1) ? 1 : threads;
    if (nb > 64) { set_error("blas_threads > 64"); return PN_ERR_INVALID; }
    static std::atomic<unsigned long long> cfg_mask{0};   // the attribute is per device
    const unsigned long long bit = 1ULL << (c->device & 63);
    if (!(cfg_mask.load() & bit)) {
        PN_CUDA(cudaFuncSetAttribute(k_ddot_emul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DD_SMEM));
        cfg_mask.fetch_or(bit);
    }
    k_ddot_emul<<<nb, DD_THREADS, DD_SMEM, s>>>(a, b, n, threads, kernel, c->ddot_chunks + slot * 64,
                                                gated ? c->state : nullptr);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

// Tree sum of sh[0..255] (blockDim.x == 256, sh written and synchronised) in
// the order of `for o = 128..1: sh[t] += sh[t + o]`; the steps o <= 16 run in
// warp 0's registers (shfl_down gives lane t the same two operands), so the
// result is bit-identical with 3 block barriers instead of 8.  Valid in
// thread 0; sh may be rewritten after the next __syncthreads.
__device__ __forceinline__ double tree256(double *sh) {
    for (int o = 128; o >= 32; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + o]);
        __syncthreads();
    }
    double a = 0.0;
    if (threadIdx.x < 32) {
        a = sh[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
    }
    return a;
}

// ---------------------------------------------------------- plane sums --
// Level 1 of every fast reduction: the block partials of one z-plane are
// summed in a fixed order into plane_sums[slot][kg].  The scalar kernels sum
// the nz plane values (level 2); multi-GPU ranks all-gather plane sums, so
// the result does not depend on the slab decomposition.
__global__ void __launch_bounds__(256) k_plane_sums(const double *__restrict__ partials, double *__restrict__ plane_sums,
                                                    long long slot_stride, int rb, int nz, int z0, int mask, int cnt) {
    const int slot = blockIdx.y;
    if (!(mask >> slot & 1)) return;
    const int kg = z0 + blockIdx.x;
    const double *p = partials + slot * slot_stride + (long long)kg * rb;
    __shared__ double sh[256];
    double acc = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) acc = __dadd_rn(acc, p[i]);
    sh[threadIdx.x] = acc;
    __syncthreads();
    const double t = tree256(sh);
    if (threadIdx.x == 0) plane_sums[slot * nz + kg] = t;
}

int launch_plane_sums(pn_context *c, int mask, int cnt, cudaStream_t s) {
    dim3 grid(c->g.nzl, RED_SLOTS);
    k_plane_sums<<<grid, 256, 0, s>>>(c->partials, c->plane_sums, slot_stride(c), c->red_bx, c->g.nz, c->g.z0, mask,
                                      cnt);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

// -------------------------------------------------------- scalar steps --
// One block: fixed-order sums of the plane-block partials (fast) or the
// in-order combination of ddot chunks (faithful), then the CGNR scalar logic
// of solver.py:231-253 on thread 0.
struct ScalarArgs {
    const double *partials;
    long long n_part;            // entries per slot (nz * rb)
    const double *chunks;
    int faithful, nchunks;
    double *hist_n, *hist_p;
    long long hist_len;
};

__device__ double sum_slot(const ScalarArgs &a, int slot, double *sh) {
    const double *p = a.partials + slot * a.n_part;   // plane sums of the slot
    double acc = 0.0;
    // L2 loads: in the fused plane-sum step the values were written by other blocks of the same grid
    for (long long i = threadIdx.x; i < a.n_part; i += blockDim.x) acc = __dadd_rn(acc, __ldcg(p + i));
    sh[threadIdx.x] = acc;
    __syncthreads();
    const double r = tree256(sh);   // blockDim.x == 256 (k_scalar, k_plane_sums_scalar); thread 0 uses it
    __syncthreads();
    return r;
}

__device__ double chunk_sum(const ScalarArgs &a, int slot) {
    const double *c = a.chunks + slot * 64;
    if (a.nchunks == 1) return c[0];
    double d = 0.0;
    for (int t = 0; t < a.nchunks; ++t) d = __dadd_rn(d, c[t]);
    return d;
}

__device__ void scalar_step(int which, const ScalarArgs &a, State *st, double *sh) {
    if (which == S_ALPHA && threadIdx.x == 0) st->xupd = 0;   // previous iteration's x update has run
    if ((which == S_ALPHA || which == S_BETA) && stopped(st)) return;
    // slots each step consumes: 0 generic / ww, 1 zz, 2 zzt, 3 rr
    int mask = 0;
    switch (which) {
        case S_NORMB: case S_NORMATB: case S_ALPHA: mask = 1; break;
        case S_RHO: mask = 4; break;
        case S_BETA: mask = 2 | 4 | 8; break;
        case S_FINAL: mask = 1 | 8; break;
    }
    double v[4] = {0, 0, 0, 0};
    for (int q = 0; q < 4; ++q)
        if (mask >> q & 1) v[q] = a.faithful ? chunk_sum(a, q) : sum_slot(a, q, sh);
    if (threadIdx.x != 0) return;
    switch (which) {
        case S_NORMB: st->norm_b = __dsqrt_rn(v[0]); break;
        case S_NORMATB: st->norm_atb = __dsqrt_rn(v[0]); break;
        case S_RHO: st->rho = v[2]; break;
        case S_ALPHA: {
            const double ww = v[0];
            st->ww = ww;
            if (ww == 0.0) { st->done = 1; st->zero_ww = 1; break; }
            st->alpha = __ddiv_rn(st->rho, ww);
            break;
        }
        case S_BETA: {
            const double zz = v[1], zzt = v[2];
            st->rr = v[3];
            const long long it = st->it + 1;
            const double normal_rel = __ddiv_rn(__dsqrt_rn(zz), st->norm_atb);
            const double primal_rel = __ddiv_rn(__dsqrt_rn(v[3]), st->norm_b);
            if (it - 1 < a.hist_len) { a.hist_n[it - 1] = normal_rel; a.hist_p[it - 1] = primal_rel; }
            st->it = it;
            st->zz = zz;
            st->zzt = zzt;
            st->xupd = 1;
            if (normal_rel <= st->tol && (st->primal_tol < 0.0 || primal_rel <= st->primal_tol)) {
                st->converged = 1;
                st->done = 1;
                break;
            }
            st->beta = st->rho != 0.0 ? __ddiv_rn(zzt, st->rho) : 0.0;
            st->rho = zzt;
            if (it >= st->max_iter) st->done = 1;
            break;
        }
        case S_FINAL: st->zz = v[0]; st->rr = v[3]; break;
    }
}

__global__ void __launch_bounds__(256) k_scalar(int which, ScalarArgs a, State *st) {
    __shared__ double sh[256];
    scalar_step(which, a, st, sh);
}

// Single-slab fast solves: the level-1 plane sums of the masked slots (slot 3
// with its own partial count) and, in the block that finishes last, the
// scalar step -- one launch instead of two (three at the beta step), with the
// same fixed summation trees, so the result is bit-identical to the separate
// kernels.  counter returns to 0 for the next launch.
__global__ void __launch_bounds__(256) k_plane_sums_scalar(const double *__restrict__ partials, double *plane_sums,
                                                           long long slot_stride, int rb, int nz, int z0, int mask,
                                                           int cnt, int cnt3, int which, ScalarArgs a, State *st,
                                                           unsigned *counter) {
    __shared__ double sh[256];
    __shared__ bool last;
    const int slot = blockIdx.y;
    if (mask >> slot & 1) {
        const int kg = z0 + blockIdx.x;
        const double *p = partials + slot * slot_stride + (long long)kg * rb;
        const int n = slot == 3 ? cnt3 : cnt;
        double acc = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) acc = __dadd_rn(acc, p[i]);
        sh[threadIdx.x] = acc;
        __syncthreads();
        const double t = tree256(sh);
        if (threadIdx.x == 0) plane_sums[slot * nz + kg] = t;
        __syncthreads();   // sh is reused by the scalar step
    }
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned done = atomicAdd(counter, 1u);
        last = done == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    scalar_step(which, a, st, sh);
    if (threadIdx.x == 0) *counter = 0u;
}

static ScalarArgs scalar_args(pn_context *c, int faithful, int blas_threads) {
    ScalarArgs a;
    a.partials = c->plane_sums;
    a.n_part = c->g.nz;
    a.chunks = c->ddot_chunks;
    a.faithful = faithful;
    a.nchunks = (c->R_l() <= 10000 || blas_threads <= 1) ? 1 : blas_threads;
    a.hist_n = c->hist_n;
    a.hist_p = c->hist_p;
    a.hist_len = c->hist_len;
    return a;
}

int launch_plane_sums_scalar(pn_context *c, int mask, int cnt, int cnt3, int which, cudaStream_t s) {
    dim3 grid(c->g.nzl, RED_SLOTS);
    k_plane_sums_scalar<<<grid, 256, 0, s>>>(c->partials, c->plane_sums, slot_stride(c), c->red_bx, c->g.nz, c->g.z0,
                                             mask, cnt, cnt3, which, scalar_args(c, 0, 1), c->state, c->counter);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

int launch_scalar(pn_context *c, int which, int faithful, int blas_threads, cudaStream_t s) {
    ScalarArgs a;
    a.partials = c->plane_sums;
    a.n_part = c->g.nz;
    a.chunks = c->ddot_chunks;
    a.faithful = faithful;
    a.nchunks = (c->R_l() <= 10000 || blas_threads <= 1) ? 1 : blas_threads;
    a.hist_n = c->hist_n;
    a.hist_p = c->hist_p;
    a.hist_len = c->hist_len;
    k_scalar<<<1, 256, 0, s>>>(which, a, c->state);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

// ------------------------------------------------- small-system CGNR --
// Fast CGNR (solver.py:231-253) for systems whose working set is a few MB:
// there the graph-replayed chain of six launches per iteration is latency
// bound (config 1: ~30 us per iteration).  One cooperative launch runs the
// whole iteration loop: reference layout, the table operator (both A and A^T
// tables resident in shared memory for the whole solve), grid barriers
// between the four phases w = A p | x, r update | z = A^T r | p update.  Every
// block sums the block partials in the same fixed order, so all blocks take
// the same scalar decisions; block 0 writes the histories and, at the end,
// the solver state.
struct SmallTab {
    double *w;
    int *ptr, *oth, *dir, *isd, *dg;
};

__device__ void small_load_tab(const Tables &T, int trans, int U, const SmallTab &s) {
    const int *p_ = trans ? T.t_ptr : T.a_ptr;
    const int *o_ = trans ? T.t_src : T.a_tgt;
    const int *d_ = trans ? T.t_dir : T.a_dir;
    const int *i_ = trans ? T.t_diag : T.a_diag;
    const double *w_ = trans ? T.t_w : T.a_w;
    const int ne = p_[U];
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        s.w[e] = w_[e]; s.oth[e] = o_[e]; s.dir[e] = d_[e]; s.isd[e] = i_[e];
    }
    for (int e = threadIdx.x; e <= U; e += blockDim.x) s.ptr[e] = p_[e];
    for (int cc = threadIdx.x; cc < U; cc += blockDim.x) {
        int dg = -1;
        for (int e = p_[cc]; e < p_[cc + 1]; ++e)
            if (i_[e]) dg = e;
        s.dg[cc] = dg;
    }
}

// operand of a phase, formed on the fly: v[i] = fma(s, a[i], b[i])
// (p_new = zt + beta p_old in the A phase, r_new = r_old - alpha w in the A^T phase)
struct SmallIn {
    const double *a, *b;
    double s;
    __device__ __forceinline__ double operator()(long long i) const { return fma(s, a[i], b[i]); }
};

// one row of the fast table operator (as k_apply_table<false, RECOMPUTE>)
template <bool RECOMPUTE>
__device__ __forceinline__ double small_row(const SmallTab &s, const int *spar, const double *slamp, const Fields &F,
                                            const Geo &g, const double *diag, const SmallIn &x, unsigned row,
                                            double xrow, const FastDiv &du, const FastDiv &dnx, const FastDiv &dny) {
    const int U = g.U;
    const unsigned vox = fdiv(row, du);
    const int c = (int)(row - vox * (unsigned)U);
    const unsigned q = fdiv(vox, dnx);
    const int i = (int)(vox - q * (unsigned)g.nx);
    const unsigned k = fdiv(q, dny);
    const int j = (int)(q - k * (unsigned)g.ny), kg = (int)k;
    const bool pinned_c = (spar[c] & boundary_bits(g, i, j, kg)) != 0;
    double sum = 0.0;
    if (s.dg[c] >= 0) {
        double a;
        if (RECOMPUTE) {
            const int pc = spar[c];
            double st_ = 0.0, ss_ = 0.0;
            int n = 0;
            for (int t = 0; t < 8; ++t) {
                if (t & ~pc) continue;
                st_ += fsample(F, g, 0, i, j, kg, t);
                ss_ += fsample(F, g, 1, i, j, kg, t);
                ++n;
            }
            const double inv = 1.0 / n;
            a = st_ * inv - slamp[c] * (ss_ * inv);
        } else {
            a = diag[row];
        }
        sum = a * xrow;
    }
    if (pinned_c) return sum;
    for (int e = s.ptr[c]; e < s.ptr[c + 1]; ++e) {
        if (s.isd[e]) continue;
        const int d = s.dir[e], o = s.oth[e];
        const int ii = i + c_dx[d], jj = j + c_dy[d], kk = kg + c_dz[d];
        if (ii < 0 || jj < 0 || kk < 0 || ii >= g.nx || jj >= g.ny || kk >= g.nz) continue;
        const int nbb = (ii == g.nx - 1) | ((jj == g.ny - 1) << 1) | ((kk == g.nz - 1) << 2);
        if (spar[o] & nbb) continue;
        sum = fma(s.w[e], x(((long long)kk * g.pvox + (long long)jj * g.nx + ii) * U + o), sum);
    }
    return sum;
}

// block tree of up to 2 values -> parts[slot * cap + blockIdx.x]
__device__ __forceinline__ void small_block_sum(double a, double b, int nv, double *parts, int s0, int s1, int cap,
                                                double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
        if (nv > 1) b = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, o));
    }
    if (lane == 0) { red[wid] = a; red[32 + wid] = b; }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        a = lane < nw ? red[lane] : 0.0;
        b = lane < nw ? red[32 + lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
            if (nv > 1) b = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, o));
        }
        if (lane == 0) {
            parts[s0 * cap + blockIdx.x] = a;
            if (nv > 1) parts[s1 * cap + blockIdx.x] = b;
        }
    }
    __syncthreads();
}

// fixed-order sums of the nb partials of NS slots s0, s0+1, ... in one pass
// (identical in every block)
template <int NS>
__device__ __forceinline__ void small_grid_sum(const double *parts, int s0, int cap, double *red, double *out) {
    double a[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) a[q] = 0.0;
    for (int t = threadIdx.x; t < (int)gridDim.x; t += blockDim.x)
#pragma unroll
        for (int q = 0; q < NS; ++q) a[q] = __dadd_rn(a[q], __ldcg(parts + (s0 + q) * cap + t));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        for (int o = 16; o > 0; o >>= 1) a[q] = __dadd_rn(a[q], __shfl_xor_sync(0xffffffffu, a[q], o));
        if (lane == 0) red[64 + q * 8 + wid] = a[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        double r = 0.0;
        for (int w_ = 0; w_ < nw; ++w_) r = __dadd_rn(r, red[64 + q * 8 + w_]);
        out[q] = r;
    }
    __syncthreads();
}

static size_t small_smem(const pn_context *c) {
    const size_t na = c->tb.n_a, nt = c->tb.n_t, U = c->U;
    return (na + nt + U + 96) * sizeof(double) + (2 * (U + 1) + 3 * (na + nt) + 3 * U) * sizeof(int);
}

template <bool RECOMPUTE>
__global__ void __launch_bounds__(256, 4) k_cg_small(Tables T, Fields F, Geo g, const double *diag, double *x, double *r,
                                                  double *p, double *w, double *z, double *zt, const double *minv,
                                                  double *p2, double *r2, double *parts, int cap, State *st, double *hist_n, double *hist_p,
                                                  long long hist_len, FastDiv du, FastDiv dnx, FastDiv dny) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int U = g.U, na = T.n_a, nt = T.n_t;
    double *dp = (double *)smem_raw;
    SmallTab ta, tt;
    ta.w = dp; tt.w = dp + na;
    double *slamp = dp + na + nt, *red = slamp + U;
    int *ip = (int *)(red + 96);
    ta.ptr = ip; ta.oth = ta.ptr + U + 1; ta.dir = ta.oth + na; ta.isd = ta.dir + na; ta.dg = ta.isd + na;
    tt.ptr = ta.dg + U; tt.oth = tt.ptr + U + 1; tt.dir = tt.oth + nt; tt.isd = tt.dir + nt; tt.dg = tt.isd + nt;
    int *spar = tt.dg + U;
    small_load_tab(T, 0, U, ta);
    small_load_tab(T, 1, U, tt);
    for (int e = threadIdx.x; e < U; e += blockDim.x) { spar[e] = T.par[e]; slamp[e] = T.lamp[e]; }
    __syncthreads();

    const unsigned R = (unsigned)(g.plane * g.nzl);
    const unsigned nth = gridDim.x * blockDim.x, tid = blockIdx.x * blockDim.x + threadIdx.x;
    const double *ZT = zt ? zt : z;
    double rho = st->rho, alpha = st->alpha, beta = 0.0, ww = st->ww, zz = st->zz, zzt = st->zzt, rr = st->rr;
    const double tol = st->tol, primal_tol = st->primal_tol, norm_atb = st->norm_atb, norm_b = st->norm_b;
    long long it = st->it;
    const long long max_iter = st->max_iter;
    int converged = 0, zero_ww = 0;
    // p and r double-buffered: each phase forms its operand on the fly from the
    // previous buffer and writes the updated vector of its own rows to the other,
    // so an iteration is two phases and two grid barriers.  p starts as zt
    // (fma(0, p, zt) = zt).
    double *pa = p, *pb = p2, *ra = r, *rb = r2;
    while (true) {
        // p = zt + beta p ; w = A p ; ww
        double a0 = 0.0;
        const SmallIn inp{pa, ZT, beta};
        for (unsigned row = tid; row < R; row += nth) {
            const double pn = inp(row);
            pb[row] = pn;
            const double v = small_row<RECOMPUTE>(ta, spar, slamp, F, g, diag, inp, row, pn, du, dnx, dny);
            w[row] = v;
            a0 = fma(v, v, a0);
        }
        small_block_sum(a0, 0.0, 1, parts, 0, 0, cap, red);
        grid.sync();
        small_grid_sum<1>(parts, 0, cap, red, &ww);
        if (ww == 0.0) { zero_ww = 1; break; }
        alpha = rho / ww;
        // x += alpha p ; r -= alpha w ; z = A^T r ; zt = z * minv ; zz, z.zt, rr
        double a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const SmallIn inr{w, ra, -alpha};
        for (unsigned row = tid; row < R; row += nth) {
            x[row] = fma(alpha, pb[row], x[row]);
            const double rn = inr(row);
            rb[row] = rn;
            a3 = fma(rn, rn, a3);
            const double v = small_row<RECOMPUTE>(tt, spar, slamp, F, g, diag, inr, row, rn, du, dnx, dny);
            z[row] = v;
            const double t = minv ? v * minv[row] : v;
            if (zt) zt[row] = t;
            a2 = fma(v, t, a2);
            a1 = fma(v, v, a1);
        }
        small_block_sum(a1, a2, 2, parts, 1, 2, cap, red);
        small_block_sum(a3, 0.0, 1, parts, 3, 3, cap, red);
        grid.sync();
        double sums[3];
        small_grid_sum<3>(parts, 1, cap, red, sums);
        zz = sums[0];
        zzt = sums[1];
        rr = sums[2];
        ++it;
        const double normal_rel = sqrt(zz) / norm_atb, primal_rel = sqrt(rr) / norm_b;
        if (blockIdx.x == 0 && threadIdx.x == 0 && it - 1 < hist_len) {
            hist_n[it - 1] = normal_rel;
            hist_p[it - 1] = primal_rel;
        }
        if (normal_rel <= tol && (primal_tol < 0.0 || primal_rel <= primal_tol)) { converged = 1; break; }
        beta = rho != 0.0 ? zzt / rho : 0.0;
        rho = zzt;
        if (it >= max_iter) break;
        double *t0 = pa; pa = pb; pb = t0;
        double *t1 = ra; ra = rb; rb = t1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->rho = rho; st->alpha = alpha; st->beta = beta;
        st->ww = ww; st->zz = zz; st->zzt = zzt; st->rr = rr;
        st->it = it;
        st->converged = converged;
        st->zero_ww = zero_ww;
        st->done = 1;
        st->xupd = 0;
    }
}

// rows the one-launch solve covers with one row per resident thread (its
// per-iteration time doubles beyond that; profiles/r01_coop_probe.jsonl)
int cg_small_capacity(pn_context *c, long long *rows) {
    auto kern = k_cg_small<false>;   // the solve assembles the stored diagonal first
    const size_t sm = small_smem(c);
    int optin = 0;
    PN_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
    if (sm > (size_t)optin) { *rows = 0; return PN_OK; }   // tables do not fit: the chain runs instead
    if (sm > 48 * 1024) PN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 0, nsm = 0;
    PN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, sm));
    PN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    *rows = (long long)std::min(per_sm * nsm, SMALL_MAX_BLOCKS) * 256;
    return PN_OK;
}

int launch_cg_small(pn_context *c, bool jacobi, cudaStream_t s) {
    const Geo g = c->g;
    const long long R = g.plane * g.nzl;
    if (R >= (1LL << 31) || g.nzl != g.nz) { set_error("internal: small solve needs one slab < 2^31 rows"); return PN_ERR_INVALID; }
    // the stored diagonal (assembled once, k_setup): one load per row instead of
    // up to 16 site samples of sigma_t / sigma_s (12-18 % per iteration)
    if (!c->diag_ready) { set_error("internal: diagonal not assembled"); return PN_ERR_INVALID; }
    auto kern = k_cg_small<false>;
    const size_t sm = small_smem(c);
    if (sm > 48 * 1024) PN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 0, nsm = 0;
    PN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, sm));
    PN_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    if (per_sm < 1) { set_error("small solve: kernel does not fit on an SM"); return PN_ERR_UNSUPPORTED; }
    int nb = (int)std::min<long long>((long long)per_sm * nsm, (R + 255) / 256);
    if (const char *e = getenv("PNRTE_SMALL_GRID")) nb = atoi(e);   // test hook: force a grid size
    nb = std::max(1, std::min(nb, SMALL_MAX_BLOCKS));
    Tables T = c->tb;
    Fields F = c->f;
    const double *diag = c->diag;
    double *x = c->x.p, *r = c->r.p, *p = c->p.p, *w = c->w.p, *z = c->z.p;
    double *zt = jacobi ? c->zt.p : nullptr;
    const double *minv = jacobi ? c->minv.p : nullptr;
    double *p2 = c->small_vecs, *r2 = c->small_vecs + R;
    double *parts = c->small_parts;
    int cap = SMALL_MAX_BLOCKS;
    State *st = c->state;
    double *hn = c->hist_n, *hp = c->hist_p;
    long long hl = c->hist_len;
    FastDiv du = make_fastdiv((unsigned)c->U), dnx = make_fastdiv((unsigned)g.nx), dny = make_fastdiv((unsigned)g.ny);
    void *args[] = {&T, &F, (void *)&g, &diag, &x, &r, &p, &w, &z, &zt, &minv, &p2, &r2, &parts, &cap, &st, &hn, &hp, &hl,
                    &du, &dnx, &dny};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, nb, 256, args, sm, s);
    if (e == cudaErrorCooperativeLaunchTooLarge) {
        // SMs taken by other work (MPS, green contexts): the caller runs the launch chain
        cudaGetLastError();
        set_error("cooperative launch too large");
        return PN_ERR_UNSUPPORTED;
    }
    PN_CUDA(e);
    c->launches++;
    return PN_OK;
}

// ------------------------------------------------------------ unstagger --
// out [i][j][kl][c] (local slab, C-order); nested 0.5*(g + g_lower) in axis
// order x, y, z with the lower sample replicated at global index 0.
__global__ void k_unstagger(const int *__restrict__ par, Geo g, const double *__restrict__ u, double *__restrict__ out) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)g.nx * g.ny * g.nzl * g.U;
    if (q >= total) return;
    const int c = (int)(q % g.U);
    const long long vox = q / g.U;
    const int kl = (int)(vox % g.nzl);
    const int j = (int)((vox / g.nzl) % g.ny);
    const int i = (int)(vox / ((long long)g.nzl * g.ny));
    const int pc = par[c];
    int ax[3], na = 0;
    for (int a = 0; a < 3; ++a)
        if (pc >> a & 1) ax[na++] = a;
    const int n = 1 << na;
    double gv[8];
    for (int s = 0; s < n; ++s) {
        int ii = i, jj = j, kk = g.z0 + kl;
        for (int b = 0; b < na; ++b)
            if (s >> b & 1) {
                if (ax[b] == 0) ii = ii > 0 ? ii - 1 : 0;
                if (ax[b] == 1) jj = jj > 0 ? jj - 1 : 0;
                if (ax[b] == 2) kk = kk > 0 ? kk - 1 : 0;
            }
        gv[s] = u[((long long)(kk - g.z0) * g.pvox + (long long)jj * g.nx + ii) * g.U + c];
    }
    for (int b = 0; b < na; ++b)
        for (int s = 0; s < n; ++s)
            if (!(s >> b & 1)) gv[s] = __dmul_rn(0.5, __dadd_rn(gv[s], gv[s | (1 << b)]));
    out[q] = gv[0];
}

int launch_unstagger(pn_context *c, const double *u, double *out, cudaStream_t s) {
    // CSR systems assembled from a stencil program keep its grid and parities
    const Geo &g = c->is_csr ? c->csr.ug : c->g;
    const int *par = c->is_csr ? c->csr.upar : c->tb.par;
    long long total = (long long)g.nx * g.ny * g.nzl * g.U;
    k_unstagger<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(par, g, u, out);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

}  // namespace pn
