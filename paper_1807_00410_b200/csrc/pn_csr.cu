// Generic CSR operator for solve_normal_cg on arbitrary sparse systems
// (pkg/src/pnrte/solver.py:189-257 accepts any SparseSystem; the reference's
// own tests solve identity / dense / Jacobi systems, test_solver.py:99-145).
//
// A is kept as given (scipy csr_matvec iterates the stored order); A^T is
// built on the device exactly like A.T.tocsr() (solver.py:203): a stable sort
// of the entries by column keeps, inside every transposed row, ascending
// original row order and stored order among duplicates.
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
    PN_CUDA(cudaMemcpy(o.ap, h_ap, (n + 1) * sizeof(long long), cudaMemcpyHostToDevice));
    if (nnz) {
        PN_CUDA(cudaMemcpy(o.aj, h_aj, nnz * sizeof(int), cudaMemcpyHostToDevice));
        PN_CUDA(cudaMemcpy(o.ax, h_ax, nnz * sizeof(double), cudaMemcpyHostToDevice));
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

void csr_release(pn_context *c) {
    CsrOp &o = c->csr;
    for (void *p : {(void *)o.ap, (void *)o.aj, (void *)o.ax, (void *)o.tp, (void *)o.tj, (void *)o.tx})
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
    else
        k_csr_apply<false><<<c->vec_bx, 256, 0, s>>>(o.n, p, j, a, squared, x, y, red, minv, zt, c->partials, stride,
                                                     c->red_bx, st);
    PN_CUDA(cudaGetLastError());
    c->launches++;
    return PN_OK;
}

}  // namespace pn
