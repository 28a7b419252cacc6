// Generic CSR operator for solve_normal_cg on arbitrary sparse systems
// (pkg/src/pnrte/solver.py:189-257 accepts any SparseSystem; the reference's
// own tests solve identity / dense / Jacobi systems, test_solver.py:99-145).
//
// A is kept as given (scipy csr_matvec iterates the stored order); A^T is
// built on the device exactly like A.T.tocsr() (solver.py:203): a stable sort
// of the entries by column keeps, inside every transposed row, ascending
// original row order and stored order among duplicates.
// Stencil systems can also be assembled into this form on the device
// (k_stencil_csr): the export behind StencilOperator.to_scipy() and the
// operator of Neumann-boundary systems, whose redirected writes the
// matrix-free kernels do not model.
// This file is compiled with -fmad=false (faithful sums are mul-then-add).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "pn_internal.cuh"

namespace pn {

__global__ void k_csr_keys(long long n, const long long *__restrict__ ap, const int *__restrict__ aj,
                           unsigned long long *keys, long long *vals) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (long long e = ap[i]; e < ap[i + 1]; ++e) {
        keys[e] = (unsigned long long)aj[e] * (unsigned long long)n + (unsigned long long)i;
        vals[e] = e;
    }
}

__global__ void k_csr_scatter(long long nnz, long long n, const unsigned long long *keys, const long long *perm,
                              const double *__restrict__ ax, int *tj, double *tx, long long *cnt) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nnz) return;
    const unsigned long long k = keys[e];
    tj[e] = (int)(k % (unsigned long long)n);   // original row
    tx[e] = ax[perm[e]];
    atomicAdd((unsigned long long *)&cnt[k / (unsigned long long)n], 1ULL);
}

// y = A x / A^T x over CSR, one thread per row, in stored order.
// faithful: sum = 0; sum += a*x (no FMA); fast: FMA.  red: 1 -> sum y^2 in
// slot 0, 2 -> z.zt / z.z in slots 2 / 1 (same partial layout as k_vec).
template <bool FAITHFUL>
__global__ void __launch_bounds__(256) k_csr_apply(long long n, const long long *__restrict__ p,
                                                   const int *__restrict__ j, const double *__restrict__ a,
                                                   int squared, const double *__restrict__ x, double *__restrict__ y,
                                                   int red, const double *minv, double *zt, double *partials,
                                                   long long slot_stride, int rb, const State *st) {
    if (st && *(volatile const int *)&st->done) return;
    const long long chunk = (n + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(n, r0 + chunk);
    double acc0 = 0.0, acc1 = 0.0;
    for (long long r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        double sum = 0.0;
        for (long long e = p[r]; e < p[r + 1]; ++e) {
            double v = a[e];
            if (FAITHFUL) {
                if (squared) v = __dmul_rn(v, v);
                sum = __dadd_rn(sum, __dmul_rn(v, x[j[e]]));
            } else {
                sum = fma(v, x[j[e]], sum);
            }
        }
        y[r] = sum;
        if (red == 1) acc0 = fma(sum, sum, acc0);
        if (red == 2) {
            const double t = minv ? sum * minv[r] : sum;
            if (zt) zt[r] = t;
            acc0 = fma(sum, t, acc0);
            acc1 = fma(sum, sum, acc1);
        }
    }
    if (!red) return;
    __shared__ double sh[2][256];
    sh[0][threadIdx.x] = acc0;
    sh[1][threadIdx.x] = acc1;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sh[0][threadIdx.x] = __dadd_rn(sh[0][threadIdx.x], sh[0][threadIdx.x + o]);
            sh[1][threadIdx.x] = __dadd_rn(sh[1][threadIdx.x], sh[1][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (red == 1) partials[blockIdx.x] = sh[0][0];
        else {
            partials[2 * slot_stride + blockIdx.x] = sh[0][0];
            partials[1 * slot_stride + blockIdx.x] = sh[1][0];
        }
    }
}

// Fast-mode CSR product: CSR_SUB lanes per row, each striding the row's
// entries by CSR_SUB (a lane group reads consecutive entries: full 32 B
// sectors), partial sums folded by xor shuffles.  Row sums differ from the
// stored-order sum only by rounding (fast mode); the faithful product keeps
// one thread per row in stored order (k_csr_apply<true>).
#ifndef PN_CSR_SUB
#define PN_CSR_SUB 2
#endif
constexpr int CSR_SUB = PN_CSR_SUB;

__global__ void __launch_bounds__(256) k_csr_apply_sub(long long n, const long long *__restrict__ p,
                                                       const int *__restrict__ j, const double *__restrict__ a,
                                                       const double *__restrict__ x, double *__restrict__ y, int red,
                                                       const double *minv, double *zt, double *partials,
                                                       long long slot_stride, int rb, const State *st) {
    if (st && *(volatile const int *)&st->done) return;
    const int lane = threadIdx.x & 31, sub = lane % CSR_SUB;
    const int ngrp = blockDim.x / CSR_SUB;
    const long long chunk = (n + rb - 1) / rb;
    const long long r0 = (long long)blockIdx.x * chunk;
    const long long r1 = min(n, r0 + chunk);
    const long long wbase = r0 + (threadIdx.x >> 5) * (32 / CSR_SUB);
    double acc0 = 0.0, acc1 = 0.0;
    for (long long rb0 = wbase; rb0 < r1; rb0 += ngrp) {   // warp-uniform trip count
        const long long r = rb0 + (lane / CSR_SUB);
        const bool has = r < r1;
        double sum = 0.0;
        if (has) {
            const long long ee = p[r + 1];
#pragma unroll 2
            for (long long e = p[r] + sub; e < ee; e += CSR_SUB) sum = fma(a[e], __ldg(x + j[e]), sum);
        }
#pragma unroll
        for (int o = CSR_SUB / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (has && sub == 0) {
            y[r] = sum;
            if (red == 1) acc0 = fma(sum, sum, acc0);
            if (red == 2) {
                const double t = minv ? sum * minv[r] : sum;
                if (zt) zt[r] = t;
                acc0 = fma(sum, t, acc0);
                acc1 = fma(sum, sum, acc1);
            }
        }
    }
    if (!red) return;
    __shared__ double sh[2][256];
    sh[0][threadIdx.x] = acc0;
    sh[1][threadIdx.x] = acc1;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sh[0][threadIdx.x] = __dadd_rn(sh[0][threadIdx.x], sh[0][threadIdx.x + o]);
            sh[1][threadIdx.x] = __dadd_rn(sh[1][threadIdx.x], sh[1][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (red == 1) partials[blockIdx.x] = sh[0][0];
        else {
            partials[2 * slot_stride + blockIdx.x] = sh[0][0];
            partials[1 * slot_stride + blockIdx.x] = sh[1][0];
        }
    }
}

int csr_build(pn_context *c, long long n, long long nnz, const long long *h_ap, const int *h_aj, const double *h_ax) {
    CsrOp &o = c->csr;
    o.n = n;
    o.nnz = nnz;
    PN_CUDA(cudaMalloc(&o.ap, (n + 1) * sizeof(long long)));
    PN_CUDA(cudaMalloc(&o.aj, std::max<long long>(nnz, 1) * sizeof(int)));
    PN_CUDA(cudaMalloc(&o.ax, std::max<long long>(nnz, 1) * sizeof(double)));
    PN_CUDA(cudaMalloc(&o.tp, (n + 1) * sizeof(long long)));
    PN_CUDA(cudaMalloc(&o.tj, std::max<long long>(nnz, 1) * sizeof(int)));
    PN_CUDA(cudaMalloc(&o.tx, std::max<long long>(nnz, 1) * sizeof(double)));
    // host or device sources (unified addressing decides the direction)
    PN_CUDA(cudaMemcpy(o.ap, h_ap, (n + 1) * sizeof(long long), cudaMemcpyDefault));
    if (nnz) {
        PN_CUDA(cudaMemcpy(o.aj, h_aj, nnz * sizeof(int), cudaMemcpyDefault));
        PN_CUDA(cudaMemcpy(o.ax, h_ax, nnz * sizeof(double), cudaMemcpyDefault));
    }
    PN_CUDA(cudaMemset(o.tp, 0, (n + 1) * sizeof(long long)));
    if (nnz == 0) return PN_OK;
    // A^T: stable radix sort of (col * n + row) keys carrying the entry index
    unsigned long long *k_in, *k_out;
    long long *v_in, *v_out, *cnt;
    PN_CUDA(cudaMalloc(&k_in, nnz * 8));
    PN_CUDA(cudaMalloc(&k_out, nnz * 8));
    PN_CUDA(cudaMalloc(&v_in, nnz * 8));
    PN_CUDA(cudaMalloc(&v_out, nnz * 8));
    PN_CUDA(cudaMalloc(&cnt, (n + 1) * 8));
    PN_CUDA(cudaMemset(cnt, 0, (n + 1) * 8));
    k_csr_keys<<<(unsigned)((n + 255) / 256), 256>>>(n, o.ap, o.aj, k_in, v_in);
    PN_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)n * (unsigned long long)n >> end_bit)) ++end_bit;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, v_out, (int)nnz, 0, end_bit);
    void *tmp;
    PN_CUDA(cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)));
    PN_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, v_out, (int)nnz, 0, end_bit));
    k_csr_scatter<<<(unsigned)((nnz + 255) / 256), 256>>>(nnz, n, k_out, v_out, o.ax, o.tj, o.tx, cnt);
    PN_CUDA(cudaGetLastError());
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, o.tp, (int)(n + 1));
    void *stmp;
    PN_CUDA(cudaMalloc(&stmp, std::max<size_t>(scan_bytes, 1)));
    PN_CUDA(cub::DeviceScan::ExclusiveSum(stmp, scan_bytes, cnt, o.tp, (int)(n + 1)));
    PN_CUDA(cudaDeviceSynchronize());
    cudaFree(k_in); cudaFree(k_out); cudaFree(v_in); cudaFree(v_out); cudaFree(cnt); cudaFree(tmp); cudaFree(stmp);
    return PN_OK;
}

// ---------------------------------------------------------------------------
// Device assembly (solver.py:96-186).  One thread per row (v, c): walk the
// row's table entries in program order, map each to its column -- Dirichlet:
// dropped when the target is outside the domain, on the last face sample of
// its staggered axis, or the row is pinned (:151-163); Neumann: target index
// clipped into the domain (:146-147) -- and insert it into a per-row sorted
// list, summing entries that land on the same column.  The result is
// coo_matrix(...).tocsr(): ascending columns, duplicates summed (a row sees
// at most two writes per column -- a staggered target is reached along one
// axis only -- so the sum is order independent), explicit zeros kept.
// Pass 1 (ap == nullptr) writes per-row counts, pass 2 fills.
__constant__ int a_dx[7] = {0, -1, 1, 0, 0, 0, 0};
__constant__ int a_dy[7] = {0, 0, 0, -1, 1, 0, 0};
__constant__ int a_dz[7] = {0, 0, 0, 0, 0, -1, 1};

__global__ void k_stencil_csr(Tables T, Geo g, const double *__restrict__ diag, int neumann, long long *cnt,
                              const long long *__restrict__ ap, int *aj, double *ax) {
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long R = (long long)g.nz * g.plane;
    if (row >= R) return;
    const int U = g.U;
    const long long v = row / U;
    const int c = (int)(row - v * U);
    const int i = (int)(v % g.nx), j = (int)((v / g.nx) % g.ny), k = (int)(v / g.pvox);
    const int bb = (i == g.nx - 1) | ((j == g.ny - 1) << 1) | ((k == g.nz - 1) << 2);
    const bool pinned = !neumann && (T.par[c] & bb);
    int col[ASM_MAX];
    double val[ASM_MAX];
    int n = 0;
    for (int e = T.a_ptr[c]; e < T.a_ptr[c + 1]; ++e) {
        int cc;
        double a;
        if (T.a_diag[e]) {
            cc = (int)row;
            a = diag[row];
        } else {
            const int o = T.a_tgt[e], d = T.a_dir[e];
            int ii = i + a_dx[d], jj = j + a_dy[d], kk = k + a_dz[d];
            if (neumann) {
                ii = min(max(ii, 0), g.nx - 1);
                jj = min(max(jj, 0), g.ny - 1);
                kk = min(max(kk, 0), g.nz - 1);
            } else {
                if (pinned || ii < 0 || jj < 0 || kk < 0 || ii >= g.nx || jj >= g.ny || kk >= g.nz) continue;
                const int nbb = (ii == g.nx - 1) | ((jj == g.ny - 1) << 1) | ((kk == g.nz - 1) << 2);
                if (T.par[o] & nbb) continue;
            }
            cc = (int)(((long long)kk * g.pvox + (long long)jj * g.nx + ii) * U + o);
            a = T.a_w[e];
        }
        int p = n;
        while (p > 0 && col[p - 1] > cc) --p;
        if (p > 0 && col[p - 1] == cc) {
            val[p - 1] = __dadd_rn(val[p - 1], a);
            continue;
        }
        for (int q = n; q > p; --q) { col[q] = col[q - 1]; val[q] = val[q - 1]; }
        col[p] = cc;
        val[p] = a;
        ++n;
    }
    if (!ap) {
        cnt[row] = n;
        return;
    }
    const long long base = ap[row];
    for (int q = 0; q < n; ++q) { aj[base + q] = col[q]; ax[base + q] = val[q]; }
}

int stencil_csr_assemble(pn_context *c, int neumann, cudaStream_t s, long long **ap_out, int **aj_out,
                         double **ax_out, long long *nnz_out) {
    const Geo &g = c->g;
    const long long R = (long long)g.nz * g.plane;
    long long *cnt = nullptr, *ap = nullptr;
    int *aj = nullptr;
    double *ax = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    long long nnz = 0;
    const unsigned nb = (unsigned)((R + 127) / 128);
    int st = PN_OK;
    auto fail = [&](int code) { cudaFree(cnt); cudaFree(ap); cudaFree(aj); cudaFree(ax); cudaFree(tmp); return code; };
    if (cudaMalloc(&cnt, (R + 1) * 8) != cudaSuccess || cudaMalloc(&ap, (R + 1) * 8) != cudaSuccess)
        return fail(PN_ERR_NOMEM);
    if (cudaMemsetAsync(cnt, 0, (R + 1) * 8, s) != cudaSuccess) return fail(PN_ERR_CUDA);
    k_stencil_csr<<<nb, 128, 0, s>>>(c->tb, g, c->diag, neumann, cnt, nullptr, nullptr, nullptr);
    if (cudaGetLastError() != cudaSuccess) return fail(PN_ERR_CUDA);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, ap, (int)(R + 1), s);
    if (cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)) != cudaSuccess) return fail(PN_ERR_NOMEM);
    if (cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, ap, (int)(R + 1), s) != cudaSuccess) return fail(PN_ERR_CUDA);
    if (cudaMemcpyAsync(&nnz, ap + R, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(PN_ERR_CUDA);
    if (cudaMalloc(&aj, std::max<long long>(nnz, 1) * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&ax, std::max<long long>(nnz, 1) * sizeof(double)) != cudaSuccess)
        return fail(PN_ERR_NOMEM);
    k_stencil_csr<<<nb, 128, 0, s>>>(c->tb, g, c->diag, neumann, nullptr, ap, aj, ax);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return fail(PN_ERR_CUDA);
    c->launches += 2;
    cudaFree(cnt);
    cudaFree(tmp);
    *ap_out = ap; *aj_out = aj; *ax_out = ax; *nnz_out = nnz;
    return st;
}

// ---------------------------------------------------------------------------
// General programs (field-dependent coefficients, e.g. CDA): every entry,
// diagonal and residual is a postfix program (general.py) evaluated per
// voxel with the reference's numpy arithmetic -- one IEEE op per array
// operation (this file is built with -fmad=false), reciprocal for ** -1.
// st: caller-owned evaluation stack (GEN_STACK doubles).  It is declared in
// the kernel on purpose: as a local of this (inlined) function NVVM's stack
// colouring placed it on top of the caller's live val[] array.
__device__ double gen_eval(const GenProg &P, int pc, int i, int j, int k, double *st) {
    int sp = 0;
    for (;; ++pc) {
        const int op = P.ops[2 * pc], arg = P.ops[2 * pc + 1];
        switch (op) {
        case G_END: return st[0];
        case G_NUM: st[sp++] = P.consts[arg]; break;
        case G_FIELD: {
            const int f = P.s_slot[arg];
            double v = 0.0;
            if (P.f_kind[f] == 1) v = P.f_scalar[f];
            else if (P.f_kind[f] == 2) {
                const int ii = min(max(i + P.s_dx[arg], 0), P.nx - 1);
                const int jj = min(max(j + P.s_dy[arg], 0), P.ny - 1);
                const int kk = min(max(k + P.s_dz[arg], 0), P.nz - 1);
                v = P.f_data[f][((long long)ii * P.ny + jj) * P.nz + kk];
            }
            st[sp++] = v;
            break;
        }
        case G_ADD: --sp; st[sp - 1] = __dadd_rn(st[sp - 1], st[sp]); break;
        case G_MUL: --sp; st[sp - 1] = __dmul_rn(st[sp - 1], st[sp]); break;
        case G_RECIP: st[sp - 1] = __ddiv_rn(1.0, st[sp - 1]); break;
        case G_SQUARE: st[sp - 1] = __dmul_rn(st[sp - 1], st[sp - 1]); break;
        case G_SQRT: st[sp - 1] = __dsqrt_rn(st[sp - 1]); break;
        case G_ONE: st[sp - 1] = 1.0; break;
        default: return __longlong_as_double(0x7ff8000000000000LL);
        }
    }
}

// one thread per row (v, c): entries in program order -> masked (Dirichlet,
// solver.py:151-163) or clipped (Neumann, :146-147) columns, insertion-sorted
// and duplicate-summed as in k_stencil_csr; RHS = -(residual), pinned rows 0
__global__ void k_general_csr(GenProg P, int neumann, long long *cnt, const long long *__restrict__ ap, int *aj,
                              double *ax, double *rhs) {
    const long long pvox = (long long)P.nx * P.ny;
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= pvox * P.nz * P.U) return;
    const long long v = row / P.U;
    const int c = (int)(row - v * P.U);
    const int i = (int)(v % P.nx), j = (int)((v / P.nx) % P.ny), k = (int)(v / pvox);
    const int bb = (i == P.nx - 1) | ((j == P.ny - 1) << 1) | ((k == P.nz - 1) << 2);
    const bool pinned = !neumann && (P.par[c] & bb);
    double st[GEN_STACK];
    if (rhs) {
        const double r = -gen_eval(P, P.r_code[c], i, j, k, st);
        rhs[row] = pinned ? 0.0 : r;
        return;
    }
    int col[ASM_MAX];
    double val[ASM_MAX];
    int n = 0;
    for (int e = P.e_ptr[c]; e < P.e_ptr[c + 1]; ++e) {
        const int o = P.e_tgt[e];
        int ii = i + P.e_dx[e], jj = j + P.e_dy[e], kk = k + P.e_dz[e];
        const bool in = ii >= 0 && jj >= 0 && kk >= 0 && ii < P.nx && jj < P.ny && kk < P.nz;
        if (!neumann) {
            if (!in) continue;
            if (!P.e_diag[e]) {
                const int nbb = (ii == P.nx - 1) | ((jj == P.ny - 1) << 1) | ((kk == P.nz - 1) << 2);
                if (pinned || (P.par[o] & nbb)) continue;
            }
        }
        ii = min(max(ii, 0), P.nx - 1);
        jj = min(max(jj, 0), P.ny - 1);
        kk = min(max(kk, 0), P.nz - 1);
        const int cc = (int)(((long long)kk * pvox + (long long)jj * P.nx + ii) * P.U + o);
        const double a = gen_eval(P, P.e_code[e], i, j, k, st);
        int p = n;
        while (p > 0 && col[p - 1] > cc) --p;
        if (p > 0 && col[p - 1] == cc) {
            val[p - 1] = __dadd_rn(val[p - 1], a);
            continue;
        }
        for (int q = n; q > p; --q) { col[q] = col[q - 1]; val[q] = val[q - 1]; }
        col[p] = cc;
        val[p] = a;
        ++n;
    }
    if (!ap) {
        cnt[row] = n;
        return;
    }
    const long long base = ap[row];
    for (int q = 0; q < n; ++q) { aj[base + q] = col[q]; ax[base + q] = val[q]; }
}

int general_csr_assemble(const GenProg &P, int neumann, double *rhs, cudaStream_t s, long long **ap_out,
                         int **aj_out, double **ax_out, long long *nnz_out) {
    const long long R = (long long)P.nx * P.ny * P.nz * P.U;
    long long *cnt = nullptr, *ap = nullptr;
    int *aj = nullptr;
    double *ax = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    long long nnz = 0;
    const unsigned nb = (unsigned)((R + 127) / 128);
    auto fail = [&](int code) { cudaFree(cnt); cudaFree(ap); cudaFree(aj); cudaFree(ax); cudaFree(tmp); return code; };
    if (rhs) {
        k_general_csr<<<nb, 128, 0, s>>>(P, neumann, nullptr, nullptr, nullptr, nullptr, rhs);
        if (cudaGetLastError() != cudaSuccess) return fail(PN_ERR_CUDA);
    }
    if (cudaMalloc(&cnt, (R + 1) * 8) != cudaSuccess || cudaMalloc(&ap, (R + 1) * 8) != cudaSuccess)
        return fail(PN_ERR_NOMEM);
    if (cudaMemsetAsync(cnt, 0, (R + 1) * 8, s) != cudaSuccess) return fail(PN_ERR_CUDA);
    k_general_csr<<<nb, 128, 0, s>>>(P, neumann, cnt, nullptr, nullptr, nullptr, nullptr);
    if (cudaGetLastError() != cudaSuccess) return fail(PN_ERR_CUDA);
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, ap, (int)(R + 1), s);
    if (cudaMalloc(&tmp, std::max<size_t>(tmp_bytes, 1)) != cudaSuccess) return fail(PN_ERR_NOMEM);
    if (cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, ap, (int)(R + 1), s) != cudaSuccess) return fail(PN_ERR_CUDA);
    if (cudaMemcpyAsync(&nnz, ap + R, 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(PN_ERR_CUDA);
    if (cudaMalloc(&aj, std::max<long long>(nnz, 1) * sizeof(int)) != cudaSuccess ||
        cudaMalloc(&ax, std::max<long long>(nnz, 1) * sizeof(double)) != cudaSuccess)
        return fail(PN_ERR_NOMEM);
    k_general_csr<<<nb, 128, 0, s>>>(P, neumann, nullptr, ap, aj, ax, nullptr);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) return fail(PN_ERR_CUDA);
    cudaFree(cnt);
    cudaFree(tmp);
    *ap_out = ap; *aj_out = aj; *ax_out = ax; *nnz_out = nnz;
    return PN_OK;
}

void csr_release(pn_context *c) {
    CsrOp &o = c->csr;
    for (void *p : {(void *)o.ap, (void *)o.aj, (void *)o.ax, (void *)o.tp, (void *)o.tj, (void *)o.tx, (void *)o.upar})
        if (p) cudaFree(p);
    o = CsrOp{};
}

int launch_csr_apply(pn_context *c, int trans, int faithful, int squared, const double *x, double *y, int red,
                     const double *minv, double *zt, cudaStream_t s, bool gated) {
    const CsrOp &o = c->csr;
    const long long *p = trans ? o.tp : o.ap;
    const int *j = trans ? o.tj : o.aj;
    const double *a = trans ? o.tx : o.ax;
    const State *st = gated ? c->state : nullptr;
    const long long stride = (long long)c->g.nz * c->red_bx;
    if (faithful)
        k_csr_apply<true><<<c->vec_bx, 256, 0, s>>>(o.n, p, j, a, squared, x, y, red, minv, zt, c->partials, stride,
                                                    c->red_bx, st);
    else if (squared)
        k_csr_apply<false><<<c->vec_bx, 256, 0, s>>>(o.n, p, j, a, squared, x, y, red, minv, zt, c->partials, stride,
                                                     c->red_bx, st);
    else
        k_csr_apply_sub<<<c->vec_bx, 256, 0, s>>>(o.n, p, j, a, x, y, red, minv, zt, c->partials, stride, c->red_bx,
                                                  st);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

}  // namespace pn
