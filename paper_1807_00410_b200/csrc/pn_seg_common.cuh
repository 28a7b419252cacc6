// Device side of the segmented fast operator (included by the generated
// per-order translation units pn_seg_N*.cu).
//
// Layout ("segmented", AoSoA): a local-slab vector is a sequence of rows
// (kl, j, seg) of 32 consecutive voxels along x; inside a row the 32*U
// doubles are component-major, lane-minor: element (c, lane) at c*32 + lane.
// The row base equals the reference layout's row base, so z-planes stay
// contiguous (halo exchange is unchanged) and conversion is a 32 x U
// transpose inside each row.
//
// One warp owns one row; lane = voxel.  Every load is a coalesced 256 B row
// chunk, every weight is warp-uniform (constant bank).  Dirichlet masks of
// assemble() (solver.py:151-163) are applied to loaded values: a sample on the
// last face of its staggered axis reads as 0 off the diagonal, and a pinned
// row keeps only diag * x.
#pragma once
#include <atomic>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "pn_internal.cuh"
#include "pn_seg_types.cuh"
#include "pn_vec.cuh"

namespace pn {


struct SegRow {
    const double *xs;                       // own row staged in shared memory, + lane
    const double *eprev, *enext;            // shared: x-edge values of the adjacent segments [U]
    const double *sig;                      // shared: sigma_t / sigma_s rows [2][4][34]
    const double *Xym, *Xyp, *Xzm, *Xzp;    // neighbour rows in global memory + lane (null outside)
    double *Y;                              // output row + lane
    const double *minv;                     // Jacobi inverse diag row + lane
    double *zt;                             // z * minv row + lane
    const double *diag;                     // stored diagonal row + lane (DIAG_ARRAY)
    int lane;
    bool bx, bx_p, by, bz, by_p, bz_p;      // last-face flags: own voxel, x+1, y+1 row, z+1 row
    static constexpr bool ysm = false;      // y-neighbour rows always in global memory
    static constexpr bool padx = false;     // no zero-padded lanes
};
// bulk path: a y-neighbour row may be a staged row of this CTA (shared memory)
struct SegRowY : SegRow {
    static constexpr bool ysm = true;
};
// nx % 32 != 0: the last row of each x-line is zero-padded; its padding lanes
// (xpad) output 0 (separate instantiation, so unpadded grids pay nothing)
template <class Base>
struct SegRowPad : Base {
    bool xpad;
    static constexpr bool padx = true;
};

struct RedAcc {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
};

__device__ __forceinline__ bool seg_stopped(const State *st) { return *(volatile const int *)&st->done != 0; }

template <int PS>
__device__ __forceinline__ bool pinned(const SegRow &r) {
    return ((PS & 1) && r.bx) || ((PS & 2) && r.by) || ((PS & 4) && r.bz);
}

template <int PS>
__device__ __forceinline__ bool pinned_yz(const SegRow &r) {
    return ((PS & 2) && r.by) || ((PS & 4) && r.bz);
}

__device__ __forceinline__ void cp_async16(void *dst_smem, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst_smem)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async8(void *dst_smem, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst_smem)),
                 "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Bulk (TMA) copy of the own row: one thread arms an mbarrier with the byte
// count and issues a single cp.async.bulk of the 32*U doubles (the row is
// contiguous in the segmented layout); the row's warps wait on the barrier.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n) : "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(phase)
        : "memory");
}

// own-voxel value of comp s as an off-diagonal input (0 on its last face).
// BND = false: interior row, no face can be hit, no masks are evaluated.
template <int PS, bool BND>
__device__ __forceinline__ double ld_own(const SegRow &r, int s) {
    const double v = r.xs[s * 32];
    return (BND && pinned<PS>(r)) ? 0.0 : v;
}

// x neighbour (lane -+ 1) from the staged row, segment edges from eprev/enext
// (zero-filled outside the domain)
template <int PS, int SIDE, bool BND>
__device__ __forceinline__ double nb_x(const SegRow &r, int s) {
    if (BND && pinned_yz<PS>(r)) return 0.0;
    if (SIDE < 0) {
        return r.lane == 0 ? r.eprev[s] : r.xs[s * 32 - 1];
    } else {
        const double n = r.lane == 31 ? r.enext[s] : r.xs[s * 32 + 1];
        return (BND && (PS & 1) && r.bx_p) ? 0.0 : n;
    }
}

template <bool YSM>
__device__ __forceinline__ double ld_row(const double *p) {
    if constexpr (YSM) return *p;   // generic load: shared (row of this CTA) or global
    else return __ldg(p);
}

template <int PS, int SIDE, bool BND, class Row>
__device__ __forceinline__ double nb_y(const Row &r, int s) {
    const double *p = SIDE < 0 ? r.Xym : r.Xyp;
    if (!BND) return ld_row<Row::ysm>(p + s * 32);
    if (!p) return 0.0;
    const double v = ld_row<Row::ysm>(p + s * 32);
    const bool pin = ((PS & 1) && r.bx) || ((PS & 2) && SIDE > 0 && r.by_p) || ((PS & 4) && r.bz);
    return pin ? 0.0 : v;
}

template <int PS, int SIDE, bool BND>
__device__ __forceinline__ double nb_z(const SegRow &r, int s) {
    const double *p = SIDE < 0 ? r.Xzm : r.Xzp;
    if (!BND) return __ldg(p + s * 32);
    if (!p) return 0.0;
    const double v = __ldg(p + s * 32);
    const bool pin = ((PS & 1) && r.bx) || ((PS & 2) && r.by) || ((PS & 4) && SIDE > 0 && r.bz_p);
    return pin ? 0.0 : v;
}

// average of sigma_t / sigma_s over the staggered site set of class P
// (shared rows q = sy + 2 sz, 34-double stride: 32 lanes + the x+1 sample of lane 31)
template <int P>
__device__ __forceinline__ void class_avg(const SegRow &r, double &at, double &as) {
    double t_ = 0.0, s_ = 0.0;
#pragma unroll
    for (int sz = 0; sz < ((P & 4) ? 2 : 1); ++sz)
#pragma unroll
        for (int sy = 0; sy < ((P & 2) ? 2 : 1); ++sy) {
            const int q = sy + 2 * sz;
            t_ += r.sig[q * 34];
            s_ += r.sig[136 + q * 34];
            if (P & 1) {
                t_ += r.sig[q * 34 + 1];
                s_ += r.sig[136 + q * 34 + 1];
            }
        }
    constexpr int n = 1 << (((P >> 0) & 1) + ((P >> 1) & 1) + ((P >> 2) & 1));
    constexpr double inv = 1.0 / n;
    at = t_ * inv;
    as = s_ * inv;
}

template <int RED, bool JAC>
__device__ __forceinline__ void store_out(const SegRow &r, RedAcc &ra, int c, double a) {
    r.Y[c * 32] = a;
    if (RED == 2 && JAC) {   // Jacobi: zt = z * minv, z.zt and z.z per output
        const double t = a * __ldg(r.minv + c * 32);
        r.zt[c * 32] = t;
        ra.s2 = fma(a, t, ra.s2);
        ra.s1 = fma(a, a, ra.s1);
    }
}

// class-level reduction without Jacobi: RED 1 -> w.w, RED 2 -> z.z (= z.zt)
template <int RED>
__device__ __forceinline__ void seg_red_add(RedAcc &ra, double sq) {
    if (RED == 1) ra.s0 += sq;
    if (RED == 2) ra.s1 += sq;
}
template <int RED>
__device__ __forceinline__ void seg_red_sq(RedAcc &ra, double a) {
    if (RED == 1) ra.s0 = fma(a, a, ra.s0);
    if (RED == 2) ra.s1 = fma(a, a, ra.s1);
}

#define W(e) prm.w[e]
#define DIAG(at, as, c) (DIAG_ARRAY ? __ldg(r.diag + (c) * 32) : fma(-prm.lamp[c], (as), (at)))
#define STORE(c, a) store_out<RED, JAC>(r, ra, (c), (a))

}  // namespace pn

#include "generated/pn_seg_gen.cuh"

namespace pn {

template <int N> struct SegTune {
    static constexpr int rows = seg_rows(N), minb = seg_minb(N);
    static constexpr bool pair = seg_pair(N);
    static constexpr int wpr = pair ? 2 : 1;         // warps per row
    static constexpr int threads = 32 * rows * wpr;
};

template <int N>
__host__ __device__ constexpr size_t seg_smem_per_warp() {
    // own row, segment edges, sigma rows, the row's mbarrier (16 B); rounded
    // up to 128 B so every staged row starts on a shared-memory wavefront
    // (a misaligned row costs a third wavefront per 256 B warp load)
    return sizeof(double) * (((size_t)32 * (N + 1) * (N + 1) + 2 * (N + 1) * (N + 1) + 2 * 4 * 34 + 2 + 15) / 16 * 16);
}

template <int N>
__device__ __forceinline__ unsigned long long *seg_bar(double *xs) {
    constexpr int U = (N + 1) * (N + 1);
    return reinterpret_cast<unsigned long long *>(xs + 32 * U + 2 * U + 2 * 4 * 34);
}

// one row of one CTA row-group ("virtual block" vb of the tiled traversal):
// CTAs march in z inside y-tiles of g.tyb row blocks, so the z-neighbour rows
// (k-1, k+1) are still in L2 when read
struct SegItem {
    int seg, jb, kl, j, kg;
    long long rowbase;
};

template <int N>
__device__ __forceinline__ SegItem seg_item(const SegGeo &g, unsigned vb, int rw) {
    constexpr long long rowlen = (long long)(N + 1) * (N + 1) * 32;
    SegItem it;
    unsigned q = fdiv(vb, g.dseg);
    it.seg = (int)(vb - q * g.dseg.d);
    vb = q;
    q = fdiv(vb, g.dtyb);
    const int jb_in = (int)(vb - q * g.dtyb.d);
    vb = q;
    q = fdiv(vb, g.dnpl);
    it.kl = g.kl0 + (int)(vb - q * g.dnpl.d) * g.kst;
    it.jb = (int)q * (int)g.dtyb.d + jb_in;
    it.j = it.jb < g.nyb ? it.jb * SegTune<N>::rows + rw : g.ny;
    it.kg = g.z0 + it.kl;
    it.rowbase = (((long long)it.kl * g.ny + it.j) * g.nseg + it.seg) * rowlen;
    return it;
}

// issue the row's copies into buffer xs (split over the warps of the row):
// the own row (32*U doubles), the four sigma_t / sigma_s rows of the
// staggered site sets, the x+1 sample of lane 31, and the segment-edge values
// of the neighbours.  Everything from HBM goes through L2 only.  TMA: the own
// row is one bulk copy completing on the row's mbarrier (initialised by the
// kernel before the CTA barrier); otherwise cp.async by all the row's lanes.
template <int N, bool TMA>
__device__ __forceinline__ void seg_stage(const SegGeo &g, const SegItem &it, double *xs, const double *__restrict__ X,
                                          const double *__restrict__ st, const double *__restrict__ ss, int lane,
                                          int half) {
    constexpr int U = (N + 1) * (N + 1);
    constexpr int WPR = SegTune<N>::wpr;
    constexpr long long rowlen = (long long)U * 32;
    double *ep = xs + 32 * U, *en = ep + U, *sg = en + U;
    const double *Xrow = X + it.rowbase;
    const bool has_prev = it.seg > 0, has_next = it.seg < g.nseg - 1;
    if constexpr (TMA) {
        if (half == 0 && lane == 0) {
            unsigned long long *bar = seg_bar<N>(xs);
            mbar_expect_tx(bar, (unsigned)(rowlen * sizeof(double)));
            bulk_g2s(xs, Xrow, (unsigned)(rowlen * sizeof(double)), bar);
        }
    } else {
#pragma unroll 4
        for (int q = lane + 32 * half; q < 16 * U; q += 32 * WPR) cp_async16(xs + 2 * q, Xrow + 2 * q);
    }
    for (int q = lane + 32 * half; q < 128; q += 32 * WPR) {
        const int rowq = q >> 4, part = (q & 15) * 2, fld = rowq >> 2, r4 = rowq & 3;
        const int jj = min(it.j + (r4 & 1), g.ny - 1);
        const int kk = it.kl + (r4 >> 1);   // plane nzl exists (edge-replicated at upload)
        const long long vb = ((long long)kk * g.ny + jj) * g.sx + it.seg * 32;
        cp_async16(sg + fld * 136 + r4 * 34 + part, (fld ? ss : st) + vb + part);
    }
    if (half == WPR - 1) {
        if (lane < 8) {   // x+1 sample of lane 31 per sigma row, edge-replicated at nx-1
            const int fld = lane >> 2, r4 = lane & 3;
            const int jj = min(it.j + (r4 & 1), g.ny - 1);
            const int kk = it.kl + (r4 >> 1);
            const long long vb = ((long long)kk * g.ny + jj) * g.sx + it.seg * 32 + (has_next ? 32 : 31);
            cp_async8(sg + fld * 136 + r4 * 34 + 32, (fld ? ss : st) + vb);
        }
        for (int c = lane; c < U; c += 32) {
            if (has_prev) cp_async8(ep + c, Xrow - rowlen + c * 32 + 31);
            else ep[c] = 0.0;
            if (has_next) cp_async8(en + c, Xrow + rowlen + c * 32);
            else en[c] = 0.0;
        }
    }
}

template <int N>
__device__ __forceinline__ void seg_pair_sync(int rw) {
    if (SegTune<N>::wpr == 1) __syncwarp();
    else asm volatile("bar.sync %0, %1;\n" ::"r"(1 + rw), "r"(32 * SegTune<N>::wpr) : "memory");
}

// compute one staged row: outputs (and fused reduction terms) of this warp's classes
template <int N, int TRANS, int RED, bool JAC, bool TMA, bool PAD>
__device__ __forceinline__ void seg_compute(const SegParams &prm, const SegGeo &g, const SegItem &it,
                                            const double *xs, const double *__restrict__ X, double *__restrict__ Y,
                                            int rw,
                                            const double *__restrict__ minv, double *__restrict__ zt, int lane,
                                            int half, RedAcc &ra) {
    constexpr int U = (N + 1) * (N + 1);
    constexpr long long rowlen = (long long)U * 32;
    const int i = it.seg * 32 + lane;
    using RowB = std::conditional_t<TMA, SegRowY, SegRow>;
    std::conditional_t<PAD, SegRowPad<RowB>, RowB> r;
    r.lane = lane;
    r.xs = xs + lane;
    r.eprev = xs + 32 * U;
    r.enext = r.eprev + U;
    r.sig = r.enext + U + lane;
    const double *Xl = X + it.rowbase + lane;
    r.Xym = it.j > 0 ? Xl - g.nseg * rowlen : nullptr;
    r.Xyp = it.j < g.ny - 1 ? Xl + g.nseg * rowlen : nullptr;
    if constexpr (TMA) {   // y neighbours inside the CTA: the adjacent staged rows
        constexpr int SW = (int)(seg_smem_per_warp<N>() / sizeof(double));
        if (rw > 0) r.Xym = xs - SW + lane;
        if (rw < SegTune<N>::rows - 1 && r.Xyp) r.Xyp = xs + SW + lane;
    }
    r.Xzm = it.kg > 0 ? Xl - g.plane : nullptr;
    r.Xzp = it.kg < g.nz - 1 ? Xl + g.plane : nullptr;
    r.Y = Y + it.rowbase + lane;
    r.minv = minv ? minv + it.rowbase + lane : nullptr;
    r.zt = zt ? zt + it.rowbase + lane : nullptr;
    r.diag = nullptr;
    if constexpr (PAD) r.xpad = i >= g.nx;
    r.bx = i == g.nx - 1;
    r.bx_p = i + 1 == g.nx - 1;
    r.by = it.j == g.ny - 1;
    r.bz = it.kg == g.nz - 1;
    r.by_p = it.j + 1 == g.ny - 1;
    r.bz_p = it.kg + 1 == g.nz - 1;
    // warp-uniform: rows away from the last faces and the y/z domain
    // ends take the mask-free code path
    const bool interior = it.seg != g.nseg - 1 && it.j >= 1 && it.j <= g.ny - 3 && it.kg >= 1 && it.kg <= g.nz - 3;
    if (SegTune<N>::wpr == 1) {
        if (interior) seg_row<N, TRANS, RED, JAC, false, false>(r, prm, ra);
        else seg_row<N, TRANS, RED, JAC, false, true>(r, prm, ra);
    } else if (half == 0) {
        if (interior) seg_half<N, TRANS, 0, RED, JAC, false, false>(r, prm, ra);
        else seg_half<N, TRANS, 0, RED, JAC, false, true>(r, prm, ra);
    } else {
        if (interior) seg_half<N, TRANS, 1, RED, JAC, false, false>(r, prm, ra);
        else seg_half<N, TRANS, 1, RED, JAC, false, true>(r, prm, ra);
    }
}

// one reduction partial per warp and row group (fixed slot): warp tree, lane 0 stores
template <int N, int RED, bool JAC>
__device__ __forceinline__ void seg_partial(const SegGeo &g, const SegItem &it, const RedAcc &ra, int lane, int warp,
                                            double *partials, long long slot_stride, int rb) {
    if (!RED) return;
    constexpr int W = SegTune<N>::rows * SegTune<N>::wpr;
    double v0 = ra.s0, v1 = ra.s1, v2 = ra.s2;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {   // only the sums this reduction writes
        if (RED == 1) v0 += __shfl_down_sync(0xffffffffu, v0, o);
        if (RED == 2) v1 += __shfl_down_sync(0xffffffffu, v1, o);
        if (RED == 2 && JAC) v2 += __shfl_down_sync(0xffffffffu, v2, o);
    }
    if (RED == 2 && !JAC) v2 = v1;
    if (lane == 0 && it.jb < g.nyb) {
        const long long idx = (long long)it.kg * rb + ((long long)it.seg * g.nyb + it.jb) * W + warp;
        if (RED == 1) partials[idx] = v0;
        if (RED == 2) { partials[1 * slot_stride + idx] = v1; partials[2 * slot_stride + idx] = v2; }
    }
}

#ifdef PN_SEG_MAXNREG
#define PN_SEG_BOUNDS(N) __maxnreg__(PN_SEG_MAXNREG)
#else
#define PN_SEG_BOUNDS(N) __launch_bounds__(SegTune<N>::threads, SegTune<N>::minb)
#endif

#ifndef PN_SEG_PF
#define PN_SEG_PF 148   // L2 prefetch distance in CTAs (bulk path); 0 disables
#endif

// TMA = true ("bulk" path, HBM-sized slabs): own rows by cp.async.bulk on
// per-row mbarriers, y neighbours inside the CTA read from the adjacent staged
// rows, and the row of the CTA PN_SEG_PF places ahead prefetched into L2.
// TMA = false (L2-resident slabs, where the bulk path measured slower):
// cp.async staging, all y/z neighbours from L2.
template <int N, int TRANS, int RED, bool JAC, bool TMA, bool PAD>
__global__ void PN_SEG_BOUNDS(N) k_seg(
    const __grid_constant__ SegParams prm, SegGeo g, const double *__restrict__ X, double *__restrict__ Y,
    const double *__restrict__ minv, double *__restrict__ zt, const double *__restrict__ st,
    const double *__restrict__ ss, double *__restrict__ partials, long long slot_stride, int rb, const State *state) {
    extern __shared__ __align__(16) double smem[];
    constexpr int WPR = SegTune<N>::wpr;
    constexpr int SW = (int)(seg_smem_per_warp<N>() / sizeof(double));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rw = warp / WPR, half = warp % WPR;   // row within the CTA, class half
    const SegItem it = seg_item<N>(g, blockIdx.x, rw);
    double *xs = smem + rw * SW;
    if constexpr (TMA) {   // every row's barrier exists before any warp waits on it
        if (threadIdx.x < SegTune<N>::rows) mbar_init(seg_bar<N>(smem + threadIdx.x * SW), 1);
        __syncthreads();
    }
    if (it.j < g.ny) {
        seg_stage<N, TMA>(g, it, xs, X, st, ss, lane, half);
        cp_async_commit();
    }
    if constexpr (TMA && PN_SEG_PF > 0) {
        // warm L2 with the row the CTA PN_SEG_PF places later will stage
        // (about half a CTA lifetime ahead at two resident CTAs per SM)
        if (lane == 0 && half == WPR - 1 && blockIdx.x + PN_SEG_PF < gridDim.x) {
            const SegItem nx = seg_item<N>(g, blockIdx.x + PN_SEG_PF, rw);
            if (nx.j < g.ny) bulk_prefetch_l2(X + nx.rowbase, (unsigned)((N + 1) * (N + 1) * 32 * sizeof(double)));
        }
    }
    // predicated on the solver's stop flag (CTA-uniform), read while the copies are in flight
    if (state && seg_stopped(state)) {
        cp_async_wait<0>();
        if (TMA && it.j < g.ny && half == 0 && lane == 0) mbar_wait(seg_bar<N>(xs), 0);   // no copy outlives the CTA
        return;
    }
    RedAcc ra;
    if (it.j < g.ny) {
        cp_async_wait<0>();
        seg_pair_sync<N>(rw);
        if constexpr (TMA) {   // own row, and the CTA's adjacent rows serving as y neighbours
            mbar_wait(seg_bar<N>(xs), 0);
            if (rw > 0) mbar_wait(seg_bar<N>(xs - SW), 0);
            if (rw < SegTune<N>::rows - 1 && it.j + 1 < g.ny) mbar_wait(seg_bar<N>(xs + SW), 0);
        }
        seg_compute<N, TRANS, RED, JAC, TMA, PAD>(prm, g, it, xs, X, Y, rw, minv, zt, lane, half, ra);
    }
    seg_partial<N, RED, JAC>(g, it, ra, lane, warp, partials, slot_stride, rb);
}

// ---------------------------------------------------------------------------
#ifndef PN_FR_TICKET
#define PN_FR_TICKET 1   // 1: work units drawn by atomic ticket; 0: the block index is the ticket
#endif
// Fused residual update + A^T apply: one launch does r -= alpha w (the k_r
// blocks, same arithmetic and partial slots) and z = A^T r with the fused
// reductions (the k_seg row groups), so the apply reads the new r from L2
// instead of HBM and the streaming update fills the apply's latency gaps.
// Work units are drawn by ticket in the order of FuseSched; an update unit
// publishes its chunk with a release store of the launch epoch, an apply unit
// acquires the chunks its rows, y / z neighbour rows and segment edges lie in.
// Every unit a CTA can wait for has a smaller ticket, i.e. belongs to a CTA
// that is already running and never waits itself: no deadlock.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <int N, bool JAC, bool PAD>
__global__ void PN_SEG_BOUNDS(N) k_seg_fr(
    const __grid_constant__ SegParams prm, const __grid_constant__ SegGeo g, const __grid_constant__ FuseSched f,
    double *__restrict__ R, const double *__restrict__ W, double *__restrict__ Z, const double *__restrict__ minv,
    double *__restrict__ zt, const double *__restrict__ st, const double *__restrict__ ss,
    double *__restrict__ partials, long long slot_stride, int rb, const State *state) {
    extern __shared__ __align__(16) double smem[];
    static_assert(SegTune<N>::threads == 256, "fused path: the residual update is blocked for 256 threads");
    constexpr int WPR = SegTune<N>::wpr, ROWS = SegTune<N>::rows;
    constexpr int SW = (int)(seg_smem_per_warp<N>() / sizeof(double));
    constexpr long long rowlen = (long long)(N + 1) * (N + 1) * 32;
    __shared__ unsigned long long s_ticket;
    if (seg_stopped(state)) return;   // CTA-uniform; no ticket is drawn by a stopped launch
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // one 64-bit counter: launch epoch in the high word, next ticket in the low one.  The CTA
    // that draws the last ticket rewinds it for the next launch (nobody else touches it again)
#if PN_FR_TICKET
    if (threadIdx.x == 0) {
        const unsigned long long tk = atomicAdd(reinterpret_cast<unsigned long long *>(f.ctl), 1ULL);
        s_ticket = tk;
        if ((unsigned)tk == gridDim.x - 1)
            *reinterpret_cast<volatile unsigned long long *>(f.ctl) = ((tk >> 32) + 1ULL) << 32;
    }
    if (threadIdx.x < ROWS) mbar_init(seg_bar<N>(smem + threadIdx.x * SW), 1);
    __syncthreads();
    const unsigned t = (unsigned)s_ticket, epoch = (unsigned)(s_ticket >> 32);
#else
    // the block index is the ticket (CTAs of a 1-D grid are dispatched in index order);
    // the host zeroes the flags before every launch, so "published" is simply 1
    if (threadIdx.x < ROWS) mbar_init(seg_bar<N>(smem + threadIdx.x * SW), 1);
    __syncthreads();
    const unsigned t = blockIdx.x, epoch = 1u;
    (void)s_ticket;
#endif
    // ---- decode the ticket.  Per tile: D update-only steps (planes 0..D-1), then nz steps of
    // nA apply units; the unit of plane k and index i also updates chunk i (and i + nA, for the
    // few chunks beyond nA) of plane k + D while its own rows are on their way.
    int T = 0;
    while (T + 1 < f.ntiles && t >= f.tile_start[T + 1]) ++T;
    unsigned u = t - f.tile_start[T];
    const unsigned nU = (unsigned)f.n_u[T], nA = (unsigned)f.n_a[T], D = (unsigned)f.D, nz = (unsigned)g.nz;
    const unsigned want = 8u * epoch;   // a chunk is published by eight warp-level increments per launch
    if (u < D * nU) {
        // ---- update-only unit: chunk c of this plane (k_r block (c, plane))
        const unsigned plane = u / nU, idx = u - plane * nU;
        const int c = f.c_lo[T] + (int)idx;
        r_update_block<true>(g.plane, f.chunk, c, (int)plane, 0, R, W, state->alpha, partials, slot_stride, rb);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(f.flags + (size_t)plane * f.vec_bx + c, 8u);
        }
        return;
    }
    u -= D * nU;
    const unsigned plane = u / nA, idx = u - plane * nA;
    const unsigned uplane = plane + D;
    const int rw = warp / WPR, half = warp % WPR;
    SegItem it;
    it.seg = (int)(idx % (unsigned)g.nseg);
    it.jb = T * g.tyb + (int)(idx / (unsigned)g.nseg);
    it.kl = (int)plane;
    it.kg = (int)plane;
    it.j = it.jb * ROWS + rw;
    if (it.j >= g.ny) it.j = g.ny;
    it.rowbase = (((long long)it.kl * g.ny + it.j) * g.nseg + it.seg) * rowlen;
    __shared__ double s_wsum[8];
    __shared__ long long s_pidx;
    const int tid = threadIdx.x;
    // ---- the embedded update, first chunk: the operands of its first half go in flight now and
    // stay in registers across the flag polling and the staging of the unit's own rows
    bool did_update = false;
    int c_first = 0;
    double2 wv[8], rv[8];
    double2 *r2 = nullptr;
    const double2 *w2 = nullptr;
    unsigned long long pf = 0, pl = 0;
    if (idx < nU && uplane < nz) {
        c_first = f.c_lo[T] + (int)idx;
        const long long r0 = (long long)c_first * f.chunk, r1 = min(g.plane, r0 + f.chunk);
        const long long i0 = (long long)uplane * g.plane + r0;
        did_update = !(g.plane & 1) && !(i0 & 1) && (r1 - r0) == 8192 &&
                     !((reinterpret_cast<uintptr_t>(R) | reinterpret_cast<uintptr_t>(W)) & 15);
        if (did_update) {
            pf = l2_policy_evict_first();
            pl = l2_policy_evict_last();
            r2 = reinterpret_cast<double2 *>(R + i0);
            w2 = reinterpret_cast<const double2 *>(W + i0);
#pragma unroll
            for (int e = 0; e < 8; ++e) wv[e] = ldv2<true>(w2 + tid + 256 * e, pf);
#pragma unroll
            for (int e = 0; e < 8; ++e) rv[e] = ldv2<true>(r2 + tid + 256 * e, pf);
        }
    }
    // ---- chunks to acquire: threads 0..17 the rows (j0 - 1 .. j0 + ROWS, seg - 1 .. seg + 1) of
    // this plane, 18 + .. the group's rows of the planes below and above
    {
        const int j0 = it.jb * ROWS;
        int pj = -1, ps = 0, pk = (int)plane;
        if (tid < 3 * (ROWS + 2)) {
            pj = j0 - 1 + tid / 3;
            ps = it.seg - 1 + tid % 3;
        } else if (tid < 3 * (ROWS + 2) + 2 * ROWS) {
            const int q = tid - 3 * (ROWS + 2);
            pj = j0 + q % ROWS;
            ps = it.seg;
            pk = (int)plane + (q < ROWS ? -1 : 1);
        }
        if (pj >= 0 && pj < g.ny && ps >= 0 && ps < g.nseg && pk >= 0 && pk < g.nz) {
            const long long off = ((long long)pj * g.nseg + ps) * rowlen;
            const long long c0 = off / f.chunk, c1 = (off + rowlen - 1) / f.chunk;
            for (long long c = c0; c <= c1; ++c) {
                const unsigned *fl = f.flags + (size_t)pk * f.vec_bx + c;
                while ((int)(ld_acquire_u32(fl) - want) < 0) __nanosleep(64);
            }
        }
    }
    __syncthreads();
    asm volatile("fence.proxy.async;\n" ::: "memory");   // the bulk copies read what other SMs just wrote
    double *xs = smem + rw * SW;
    if (it.j < g.ny) {
        seg_stage<N, true>(g, it, xs, R, st, ss, lane, half);
        cp_async_commit();
    }
    // ---- finish the update while the rows land
    if (did_update) {
        const double alpha = state->alpha;
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            rv[e].x = fma(-alpha, wv[e].x, rv[e].x);
            rv[e].y = fma(-alpha, wv[e].y, rv[e].y);
            stv2<true>(r2 + tid + 256 * e, rv[e], pl);
            acc = fma(rv[e].x, rv[e].x, acc);
            acc = fma(rv[e].y, rv[e].y, acc);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) wv[e] = ldv2<true>(w2 + 2048 + tid + 256 * e, pf);
#pragma unroll
        for (int e = 0; e < 8; ++e) rv[e] = ldv2<true>(r2 + 2048 + tid + 256 * e, pf);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            rv[e].x = fma(-alpha, wv[e].x, rv[e].x);
            rv[e].y = fma(-alpha, wv[e].y, rv[e].y);
            stv2<true>(r2 + 2048 + tid + 256 * e, rv[e], pl);
            acc = fma(rv[e].x, rv[e].x, acc);
            acc = fma(rv[e].y, rv[e].y, acc);
        }
        // publish per warp (no CTA barrier in front of the apply); the block sum of
        // ||r||^2 is finished at the end of the unit in block_partials' order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        __syncwarp();
        if (lane == 0) {
            s_wsum[warp] = acc;
            __threadfence();
            atomicAdd(f.flags + (size_t)uplane * f.vec_bx + c_first, 1u);
        }
        if (tid == 0) s_pidx = (long long)uplane * rb + c_first;
    }
    RedAcc ra;
    if (it.j < g.ny) {
        cp_async_wait<0>();
        seg_pair_sync<N>(rw);
        mbar_wait(seg_bar<N>(xs), 0);
        if (rw > 0) mbar_wait(seg_bar<N>(xs - SW), 0);
        if (rw < ROWS - 1 && it.j + 1 < g.ny) mbar_wait(seg_bar<N>(xs + SW), 0);
        seg_compute<N, 1, 2, JAC, true, PAD>(prm, g, it, xs, R, Z, rw, minv, zt, lane, half, ra);
    }
    seg_partial<N, 2, JAC>(g, it, ra, lane, warp, partials, slot_stride, rb);
    if (did_update) {   // second level of block_partials
        __syncthreads();
        if (warp == 0) {
            double a = lane < 8 ? s_wsum[lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
            if (lane == 0) partials[3 * slot_stride + s_pidx] = a;
        }
    }
    // chunks the register path did not take: odd sizes, and the few chunks beyond nA (one row line
    // past the tile); nothing in this tile's remaining steps waits for them sooner than D planes on
    for (unsigned ci = did_update ? idx + nA : idx; ci < nU && uplane < nz; ci += nA) {
        const int c = f.c_lo[T] + (int)ci;
        __syncthreads();
        r_update_block<true>(g.plane, f.chunk, c, (int)uplane, 0, R, W, state->alpha, partials, slot_stride, rb);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(f.flags + (size_t)uplane * f.vec_bx + c, 8u);
        }
    }
}

template <int N>
int seg_launch_fused_r(const SegParams &prm, const SegGeo &g, const FuseSched &f, bool jac, double *r, const double *w,
                       double *z, const double *minv, double *zt, const double *st, const double *ss,
                       double *partials, long long slot_stride, int rb, const State *state, cudaStream_t s) {
    if constexpr (SegTune<N>::threads != 256) {
        set_error("fused residual update: unsupported order");
        return PN_ERR_UNSUPPORTED;
    } else {
        const size_t smem = SegTune<N>::rows * seg_smem_per_warp<N>();
        const unsigned nblk = f.tile_start[f.ntiles];
        int dev = 0;
        PN_CUDA(cudaGetDevice(&dev));
#define PN_FR_GO(J, P)                                                                                         \
    do {                                                                                                       \
        static std::atomic<unsigned long long> cfg_mask{0};                                                    \
        const unsigned long long bit_ = 1ULL << (dev & 63);                                                    \
        if (!(cfg_mask.load() & bit_)) {                                                                       \
            PN_CUDA(cudaFuncSetAttribute(k_seg_fr<N, J, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                         (int)smem));                                                          \
            cfg_mask.fetch_or(bit_);                                                                           \
        }                                                                                                      \
        if (!PN_FR_TICKET) PN_CUDA(cudaMemsetAsync(f.flags, 0, (size_t)g.nz * f.vec_bx * sizeof(unsigned), s));        \
        k_seg_fr<N, J, P><<<nblk, 256, smem, s>>>(prm, g, f, r, w, z, minv, zt, st, ss, partials, slot_stride, \
                                                  rb, state);                                                  \
    } while (0)
        const bool pad = g.sx != g.nx;
        if (jac) { if (pad) PN_FR_GO(true, true); else PN_FR_GO(true, false); }
        else { if (pad) PN_FR_GO(false, true); else PN_FR_GO(false, false); }
#undef PN_FR_GO
        PN_CUDA(cudaGetLastError());
        return PN_OK;
    }
}

template <int N>
int seg_launch(const SegParams &prm, const SegGeo &g0, int trans, int red, bool jac, const double *x, double *y,
               const double *minv, double *zt, const double *st, const double *ss, double *partials,
               long long slot_stride, int rb, const State *state, cudaStream_t s) {
    constexpr int rows = SegTune<N>::rows;
    SegGeo g = g0;
    const long long ytiles = (g.nyb + g.tyb - 1) / g.tyb;
    const long long nblk = (long long)g.nseg * g.tyb * g.npl * ytiles;
    if (nblk >= (1LL << 31) - PN_SEG_PF) { set_error("segmented launch: grid too large"); return PN_ERR_INVALID; }
    g.dseg = make_fastdiv((unsigned)g.nseg);
    g.dtyb = make_fastdiv((unsigned)std::min(g.tyb, g.nyb));
    g.dnpl = make_fastdiv((unsigned)g.npl);
    dim3 grid((unsigned)nblk), block(SegTune<N>::threads);
    const size_t smem = rows * seg_smem_per_warp<N>();
    if (g.nyb != (g.ny + rows - 1) / rows) { set_error("segmented launch: row blocking mismatch"); return PN_ERR_INVALID; }
    int dev = 0;
    PN_CUDA(cudaGetDevice(&dev));
#define PN_SEG_GO3(T, R, J, B, P)                                                                                 \
    do {                                                                                                          \
        /* the attribute is per device: one bit per device ordinal */                                           \
        static std::atomic<unsigned long long> cfg_mask{0};                                                       \
        const unsigned long long bit_ = 1ULL << (dev & 63);                                                       \
        if (!(cfg_mask.load() & bit_)) {                                                                          \
            PN_CUDA(cudaFuncSetAttribute(k_seg<N, T, R, J, B, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                         (int)smem));                                                             \
            cfg_mask.fetch_or(bit_);                                                                              \
        }                                                                                                         \
        k_seg<N, T, R, J, B, P><<<grid, block, smem, s>>>(prm, g, x, y, minv, zt, st, ss, partials, slot_stride,  \
                                                          rb, state);                                             \
    } while (0)
#define PN_SEG_GO2(T, R, J, B)                        \
    do {                                              \
        if (g.sx != g.nx) PN_SEG_GO3(T, R, J, B, true); \
        else PN_SEG_GO3(T, R, J, B, false);           \
    } while (0)
#define PN_SEG_GO(T, R, J)                     \
    do {                                       \
        if (g.bulk) PN_SEG_GO2(T, R, J, true); \
        else PN_SEG_GO2(T, R, J, false);       \
    } while (0)
    if (!trans) {
        if (red == 1) PN_SEG_GO(0, 1, false);
        else PN_SEG_GO(0, 0, false);
    } else {
        if (red == 2) {
            if (jac) PN_SEG_GO(1, 2, true);
            else PN_SEG_GO(1, 2, false);
        } else {
            PN_SEG_GO(1, 0, false);
        }
    }
#undef PN_SEG_GO2
#undef PN_SEG_GO3
#undef PN_SEG_GO
    PN_CUDA(cudaGetLastError());
    return PN_OK;
}

}  // namespace pn
