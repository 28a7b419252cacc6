// Device pieces shared by the vector kernels (pn_kernels.cu) and the fused
// apply (pn_seg_common.cuh): the fixed-tree block reduction and the body of
// the fast residual update, so both produce the same bits.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pn {

// Block reduction of up to 3 per-thread values into partials (fixed tree).
template <int NV>
__device__ __forceinline__ void block_partials(double (&v)[NV], double *partials, const int *slots, long long slot_stride,
                                               long long idx) {
    __shared__ double red[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double a = v[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
        if (lane == 0) red[q][wid] = a;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double a = lane < nw ? red[q][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, o));
            if (lane == 0) partials[slots[q] * slot_stride + idx] = a;
        }
    }
}

// CG (fused apply): operands bypass L1 and are marked evict-first in L2 (they
// are streamed once), the new r is stored evict-last (the apply reads it back
// a few planes later)
__device__ __forceinline__ unsigned long long l2_policy_evict_first() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
template <bool CG>
__device__ __forceinline__ double ldv(const double *p, unsigned long long pol) {
    if (!CG) return *p;
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
template <bool CG>
__device__ __forceinline__ double2 ldv2(const double2 *p, unsigned long long pol) {
    if (!CG) return *p;
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
template <bool CG>
__device__ __forceinline__ void stv(double *p, double v, unsigned long long pol) {
    if (!CG) { *p = v; return; }
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
template <bool CG>
__device__ __forceinline__ void stv2(double2 *p, double2 v, unsigned long long pol) {
    if (!CG) { *p = v; return; }
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// r -= alpha w over chunk bx of local plane kl (chunk doubles per block, 256
// threads), ||r||^2 partial into slot 3 at (z0 + kl) * pst + bx.  CG: loads
// bypass L1 (the fused apply reads the new r on the same SM afterwards).
template <bool CG>
__device__ __forceinline__ void r_update_block(long long plane, long long chunk, int bx, int kl, int z0,
                                               double *__restrict__ r, const double *__restrict__ w, double alpha,
                                               double *partials, long long slot_stride, int pst) {
    const long long r0 = (long long)bx * chunk;
    const long long r1 = min(plane, r0 + chunk);
    const long long base = (long long)kl * plane;
    double acc = 0.0;
    long long i0 = base + r0, i1 = base + r1;
    const unsigned long long pf = CG ? l2_policy_evict_first() : 0ULL, pl = CG ? l2_policy_evict_last() : 0ULL;
#ifndef PN_VEC_SCALAR
    // paired (16 B) accesses when every z-plane starts 16 B-aligned (even plane
    // length, aligned buffers): the element-to-thread map then depends on the
    // plane-local index only, so the partial sums do not depend on the slab
    // decomposition.  A leading odd element is done first.
    const bool paired = !(plane & 1) && !((reinterpret_cast<uintptr_t>(r) | reinterpret_cast<uintptr_t>(w)) & 15);
    if (paired && (i0 & 1) && i0 < i1) {
        if (threadIdx.x == 0) {
            const double rv = fma(-alpha, ldv<CG>(w + i0, pf), ldv<CG>(r + i0, pf));
            stv<CG>(r + i0, rv, pl);
            acc = fma(rv, rv, acc);
        }
        ++i0;
    }
    const long long np = paired ? (i1 - i0) >> 1 : 0;
    double2 *r2 = reinterpret_cast<double2 *>(r + i0);
    const double2 *w2 = reinterpret_cast<const double2 *>(w + i0);
    if (CG) {
        // eight pairs of each operand in flight per thread (the unit is latency-bound:
        // one CTA, 64 KB per operand); same per-thread order of the sum
        long long q = threadIdx.x;
        for (; q + 7 * (long long)blockDim.x < np; q += 8 * (long long)blockDim.x) {
            double2 wv[8], rv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) wv[e] = ldv2<CG>(w2 + q + e * (long long)blockDim.x, pf);
#pragma unroll
            for (int e = 0; e < 8; ++e) rv[e] = ldv2<CG>(r2 + q + e * (long long)blockDim.x, pf);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                rv[e].x = fma(-alpha, wv[e].x, rv[e].x);
                rv[e].y = fma(-alpha, wv[e].y, rv[e].y);
                stv2<CG>(r2 + q + e * (long long)blockDim.x, rv[e], pl);
                acc = fma(rv[e].x, rv[e].x, acc);
                acc = fma(rv[e].y, rv[e].y, acc);
            }
        }
        for (; q < np; q += blockDim.x) {
            const double2 wv = ldv2<CG>(w2 + q, pf);
            double2 rv = ldv2<CG>(r2 + q, pf);
            rv.x = fma(-alpha, wv.x, rv.x);
            rv.y = fma(-alpha, wv.y, rv.y);
            stv2<CG>(r2 + q, rv, pl);
            acc = fma(rv.x, rv.x, acc);
            acc = fma(rv.y, rv.y, acc);
        }
    } else {
#pragma unroll 4
        for (long long q = threadIdx.x; q < np; q += blockDim.x) {
            const double2 wv = w2[q];
            double2 rv = r2[q];
            rv.x = fma(-alpha, wv.x, rv.x);
            rv.y = fma(-alpha, wv.y, rv.y);
            r2[q] = rv;
            acc = fma(rv.x, rv.x, acc);
            acc = fma(rv.y, rv.y, acc);
        }
    }
    i0 += 2 * np;
#endif
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double rv = fma(-alpha, ldv<CG>(w + i, pf), ldv<CG>(r + i, pf));
        stv<CG>(r + i, rv, pl);
        acc = fma(rv, rv, acc);
    }
    double v[1] = {acc};
    const int sl[1] = {3};
    block_partials<1>(v, partials, sl, slot_stride, (long long)(z0 + kl) * pst + bx);
}

}  // namespace pn
