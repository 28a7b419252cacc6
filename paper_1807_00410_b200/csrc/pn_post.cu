// Post-processing of the collocated solution on the device
// (pkg/src/pnrte/solver.py:299-343):
//   pn_fluence      sqrt(4 pi) * L00                      solver.py:299-301
//   pn_trilinear    clamped trilinear interpolation       solver.py:304-327
//   pn_reconstruct  radiance at points x directions       solver.py:330-343
// The interpolation restates the reference's scalar arithmetic op for op
// (bit-identical); the real SH basis (sh.py:33-101) is evaluated with the
// device libm (acos / atan2 / cos / sin), so radiance agrees to rounding.
// Built with -fmad=false: interpolation weights and sums must not contract.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "pn_internal.cuh"

namespace pn {

constexpr int POST_MAX_U = 64;

__global__ void k_fluence(const double *__restrict__ coll, long long nvox, int U, double *__restrict__ out) {
    const double s4pi = 3.5449077018110318;   // math.sqrt(4 * math.pi)
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < nvox;
         v += (long long)gridDim.x * blockDim.x)
        out[v] = __dmul_rn(s4pi, coll[v * U]);
}

struct PostGrid {
    int dim, U;
    int res[3];
    double origin[3];
    double h;
};

// coef[p][q] = trilinear(coll[..., q], x_p) for q < U (solver.py:304-327)
__global__ void k_trilinear(const double *__restrict__ coll, PostGrid G, long long npts, const double *__restrict__ pts,
                            double *__restrict__ coef) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npts) return;
    int i0[3] = {0, 0, 0};
    double t[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < G.dim; ++k) {
        double s = __dsub_rn(__ddiv_rn(__dsub_rn(pts[p * G.dim + k], G.origin[k]), G.h), 0.5);
        s = fmin(fmax(s, 0.0), (double)G.res[k] - 1.0);
        const int base = G.res[k] > 1 ? min((int)floor(s), G.res[k] - 2) : 0;
        i0[k] = base;
        t[k] = __dsub_rn(s, (double)base);
    }
    for (int q = 0; q < G.U; ++q) {
        double acc = 0.0;
        for (int corner = 0; corner < (1 << G.dim); ++corner) {
            double w = 1.0;
            long long off = 0;
            for (int k = 0; k < G.dim; ++k) {
                const int bit = (corner >> k) & 1;
                w = __dmul_rn(w, bit ? t[k] : __dsub_rn(1.0, t[k]));
                off = off * G.res[k] + min(i0[k] + bit, G.res[k] - 1);
            }
            acc = __dadd_rn(acc, __dmul_rn(w, coll[off * G.U + q]));
        }
        coef[p * G.U + q] = acc;
    }
}

// Y[d][q] = real_sh(l_q, m_q, theta_d, phi_d) (sh.py:33-101: phase-free
// associated Legendre recurrence, sqrt(2) N cos(m phi) for m > 0,
// sqrt(2) N sin(|m| phi) for m < 0)
struct LmTable {
    int U;
    int l[POST_MAX_U], m[POST_MAX_U];
    double norm[POST_MAX_U];   // sqrt((2l+1)/(4pi) (l-|m|)!/(l+|m|)!), host-computed
};

__global__ void k_basis(LmTable T, long long ndirs, const double *__restrict__ dirs, double *__restrict__ Y) {
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= ndirs) return;
    const double ox = dirs[3 * d], oy = dirs[3 * d + 1], oz = dirs[3 * d + 2];
    const double nrm = sqrt(ox * ox + oy * oy + oz * oz);
    const double z = oz / nrm;
    const double theta = acos(fmax(-1.0, fmin(1.0, z)));
    const double phi = atan2(oy / nrm, ox / nrm);
    const double x = fmax(-1.0, fmin(1.0, cos(theta)));
    const double somx2 = sqrt(1.0 - x * x);
    for (int q = 0; q < T.U; ++q) {
        const int l = T.l[q], am = abs(T.m[q]);
        double pmm = 1.0, fact = 1.0;
        for (int r = 0; r < am; ++r) { pmm *= fact * somx2; fact += 2.0; }
        double plm = pmm;
        if (l > am) {
            double pmmp1 = x * (2 * am + 1) * pmm;
            for (int ll = am + 2; ll <= l; ++ll) {
                const double pll = (x * (2 * ll - 1) * pmmp1 - (ll + am - 1) * pmm) / (ll - am);
                pmm = pmmp1;
                pmmp1 = pll;
            }
            plm = pmmp1;
        }
        double v = T.norm[q] * plm;
        if (T.m[q] > 0) v *= 1.4142135623730951 * cos(am * phi);
        if (T.m[q] < 0) v *= 1.4142135623730951 * sin(am * phi);
        Y[d * T.U + q] = v;
    }
}

// out[p][d] = sum_q coef[p][q] * Y[d][q], q ascending (solver.py:340-342)
__global__ void k_radiance(const double *__restrict__ coef, const double *__restrict__ Y, int U, long long npts,
                           long long ndirs, double *__restrict__ out) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= npts * ndirs) return;
    const long long p = idx / ndirs, d = idx - p * ndirs;
    double val = 0.0;
    for (int q = 0; q < U; ++q) val = __dadd_rn(val, __dmul_rn(coef[p * U + q], Y[d * U + q]));
    out[idx] = val;
}

static int post_grid(PostGrid &G, int32_t dim, const int32_t *res, int32_t U, const double *origin, double h) {
    if (dim < 1 || dim > 3 || !res || !origin || U < 1 || !(h > 0)) return PN_ERR_INVALID;
    G.dim = dim;
    G.U = U;
    for (int k = 0; k < 3; ++k) {
        G.res[k] = k < dim ? res[k] : 1;
        G.origin[k] = k < dim ? origin[k] : 0.0;
        if (G.res[k] < 1) return PN_ERR_INVALID;
    }
    G.h = h;
    return PN_OK;
}

}  // namespace pn

using namespace pn;

extern "C" {

int pn_fluence(const double *coll, int64_t nvox, int32_t U, double *out, void *stream) {
    if (!coll || !out || nvox < 0 || U < 1) { set_error("invalid arguments"); return PN_ERR_INVALID; }
    if (nvox == 0) return PN_OK;
    const long long nb = std::min<long long>((nvox + 255) / 256, 148LL * 16);
    k_fluence<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(coll, nvox, U, out);
    return cudaGetLastError() == cudaSuccess ? PN_OK : PN_ERR_CUDA;
}

int pn_trilinear(const double *coll, int32_t dim, const int32_t *res, int32_t U, const double *origin, double h,
                 int64_t npts, const double *pts, double *out, void *stream) {
    PostGrid G;
    if (post_grid(G, dim, res, U, origin, h) != PN_OK || npts < 0 || (npts && (!coll || !pts || !out))) {
        set_error("invalid arguments");
        return PN_ERR_INVALID;
    }
    if (npts == 0) return PN_OK;
    k_trilinear<<<(unsigned)((npts + 127) / 128), 128, 0, (cudaStream_t)stream>>>(coll, G, npts, pts, out);
    return cudaGetLastError() == cudaSuccess ? PN_OK : PN_ERR_CUDA;
}

int pn_reconstruct(const double *coll, int32_t dim, const int32_t *res, int32_t U, const int32_t *lm,
                   const double *origin, double h, int64_t npts, const double *pts, int64_t ndirs, const double *dirs,
                   double *out, void *stream) {
    PostGrid G;
    if (post_grid(G, dim, res, U, origin, h) != PN_OK || U > POST_MAX_U || !lm || npts < 0 || ndirs < 0) {
        set_error("invalid arguments");
        return PN_ERR_INVALID;
    }
    if (npts == 0 || ndirs == 0) return PN_OK;
    if (!coll || !pts || !dirs || !out) { set_error("invalid arguments"); return PN_ERR_INVALID; }
    LmTable T;
    T.U = U;
    const double pi = 3.141592653589793;
    for (int q = 0; q < U; ++q) {
        const int l = lm[2 * q], m = lm[2 * q + 1], am = m < 0 ? -m : m;
        if (l < 0 || am > l) { set_error("|m| > l in the unknown list"); return PN_ERR_INVALID; }
        double ratio = 1.0;   // (l-|m|)! / (l+|m|)!
        for (int r = l - am + 1; r <= l + am; ++r) ratio /= r;
        T.l[q] = l;
        T.m[q] = m;
        T.norm[q] = sqrt((2 * l + 1) / (4 * pi) * ratio);
    }
    cudaStream_t s = (cudaStream_t)stream;
    double *coef = nullptr, *Y = nullptr;
    if (cudaMallocAsync(&coef, (size_t)npts * U * sizeof(double), s) != cudaSuccess) return PN_ERR_NOMEM;
    if (cudaMallocAsync(&Y, (size_t)ndirs * U * sizeof(double), s) != cudaSuccess) {
        cudaFreeAsync(coef, s);
        return PN_ERR_NOMEM;
    }
    k_trilinear<<<(unsigned)((npts + 127) / 128), 128, 0, s>>>(coll, G, npts, pts, coef);
    k_basis<<<(unsigned)((ndirs + 127) / 128), 128, 0, s>>>(T, ndirs, dirs, Y);
    const long long n = npts * ndirs;
    k_radiance<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(coef, Y, U, npts, ndirs, out);
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(coef, s);
    cudaFreeAsync(Y, s);
    return e == cudaSuccess ? PN_OK : PN_ERR_CUDA;
}

}  // extern "C"
