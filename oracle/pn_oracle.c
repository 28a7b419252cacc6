/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by, or called
 * from the product path (paper_1807_00410_b200/).  Only tests/, bench.py's
 * cpu_baseline / --impl reference legs and __graft_entry__.smoke() use it, as
 * the checker.
 *
 * A plain-C restatement of the reference's solve path (pnrte, Python):
 *
 *   or_setup        diagonal + RHS of assemble()      solver.py:96-186, cas.py:465-517
 *   or_csr          the assembled CSR, scipy order     solver.py:129-185 (coo->csr)
 *   or_csr_bc       same with the boundary condition: Neumann redirects
 *                   writes into the domain (solver.py:133-135,146-147) and
 *                   tocsr() sums the duplicates (solver.py:182-185)
 *   or_apply        y = A x / A^T x, scipy csr_matvec order (sequential,
 *                   ascending column, mul then add, no FMA)   solver.py:209,226-227,232,239
 *   or_jacobi_diag  colsum(A o A), ascending row order solver.py:218-223
 *   or_ddot         numpy x@y / np.linalg.norm through OpenBLAS 0.3.30 ddot:
 *                   T-way chunk split + SkylakeX / Haswell kernel emulation
 *                   (numpy 2.3.5 + libscipy_openblas 0.3.30, the reference's
 *                   pinned third-party arithmetic)
 *   or_cgnr         solve_normal_cg, op for op      solver.py:189-257
 *   or_unstagger    unstagger                       solver.py:275-296
 *
 * Compiled with -ffp-contract=off so every a*b+c stays two roundings, like
 * numpy and scipy's sparsetools.  The fast paths (OpenMP over rows) are bit
 * identical to the sequential ones because rows are independent.
 *
 * Layout: solution index = (i + nx*(j + ny*k))*U + comp (solver.py:4-6,87-93).
 * Fields are x-fastest voxel arrays (the Python wrapper transposes the
 * reference's [i,j,k] C-order fields once).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t U, nx, ny, nz;
    const int32_t *par;                                   /* [U] parity bits x|y<<1|z<<2 */
    const int32_t *a_ptr, *a_tgt, *a_dir, *a_diag; const double *a_w;
    const int32_t *t_ptr, *t_src, *t_dir, *t_diag; const double *t_w;
    const int32_t *d_ptr, *r_ptr, *term_hascoef, *term_nf, *term_f, *term_site;
    const double *term_coef;
} or_tables;

/* field slot s: kind 0 absent (zero), 1 uniform scalar, 2 array (x-fastest) */
typedef struct {
    int32_t n;
    const int32_t *kind;
    const double *scalar;
    const double *const *data;
} or_fields;

static const int DX[7] = {0, -1, 1, 0, 0, 0, 0};
static const int DY[7] = {0, 0, 0, -1, 1, 0, 0};
static const int DZ[7] = {0, 0, 0, 0, 0, -1, 1};

static inline int boundary_bits(const or_tables *T, int i, int j, int k) {
    return (i == T->nx - 1) | ((j == T->ny - 1) << 1) | ((k == T->nz - 1) << 2);
}

/* field sample at voxel (i,j,k)+site, edge-replicated (solver.py:62-64,118-123) */
static inline double fsample(const or_tables *T, const or_fields *F, int slot, int i, int j, int k, int site) {
    int kd = F->kind[slot];
    if (kd == 0) return 0.0;
    if (kd == 1) return F->scalar[slot];
    int ii = i + (site & 1), jj = j + ((site >> 1) & 1), kk = k + ((site >> 2) & 1);
    if (ii > T->nx - 1) ii = T->nx - 1;
    if (jj > T->ny - 1) jj = T->ny - 1;
    if (kk > T->nz - 1) kk = T->nz - 1;
    return F->data[slot][(int64_t)ii + (int64_t)T->nx * (jj + (int64_t)T->ny * kk)];
}

/* sum of product terms in expression-tree order (cas.py:494-503) */
static double eval_terms(const or_tables *T, const or_fields *F, int t0, int t1, int i, int j, int k) {
    double acc = 0.0;
    for (int t = t0; t < t1; ++t) {
        double v;
        int nf = T->term_nf[t];
        int f = 0;
        if (T->term_hascoef[t]) v = T->term_coef[t];
        else { v = fsample(T, F, T->term_f[2 * t], i, j, k, T->term_site[2 * t]); f = 1; }
        for (; f < nf; ++f) v = v * fsample(T, F, T->term_f[2 * t + f], i, j, k, T->term_site[2 * t + f]);
        acc = (t == t0) ? v : acc + v;
    }
    return acc;
}

/* diag[R], rhs[R]; pinned rows keep their diagonal and get rhs 0 (solver.py:136-141,179-180) */
void or_setup_bc(const or_tables *T, const or_fields *F, int pin, double *diag, double *rhs) {
    const int U = T->U;
    const int64_t nvox = (int64_t)T->nx * T->ny * T->nz;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvox; ++v) {
        int i = (int)(v % T->nx), j = (int)((v / T->nx) % T->ny), k = (int)(v / ((int64_t)T->nx * T->ny));
        int bb = boundary_bits(T, i, j, k);
        for (int c = 0; c < U; ++c) {
            diag[v * U + c] = eval_terms(T, F, T->d_ptr[c], T->d_ptr[c + 1], i, j, k);
            double r = 0.0;
            if (T->r_ptr[c + 1] > T->r_ptr[c]) r = -eval_terms(T, F, T->r_ptr[c], T->r_ptr[c + 1], i, j, k);
            rhs[v * U + c] = (pin && (T->par[c] & bb)) ? 0.0 : r;
        }
    }
}

void or_setup(const or_tables *T, const or_fields *F, double *diag, double *rhs) { or_setup_bc(T, F, 1, diag, rhs); }

/* neighbour voxel along direction code d, or -1 when outside the domain */
static inline int64_t neighbour(const or_tables *T, int i, int j, int k, int d, int *bb) {
    int ii = i + DX[d], jj = j + DY[d], kk = k + DZ[d];
    if (ii < 0 || jj < 0 || kk < 0 || ii >= T->nx || jj >= T->ny || kk >= T->nz) return -1;
    *bb = boundary_bits(T, ii, jj, kk);
    return (int64_t)ii + (int64_t)T->nx * (jj + (int64_t)T->ny * kk);
}

/*
 * y = A x (transpose=0) or A^T x (transpose=1), scipy csr_matvec order:
 * sum = 0; for each stored entry in ascending column order: sum += a*x.
 * Dirichlet masks (solver.py:151-163): an off-diagonal entry survives iff its
 * target voxel is in the domain, the target sample is not on the last face
 * of its staggered axis, and the row is not pinned.  For A^T the same
 * predicate is evaluated on the (row, column) pair of A.
 * mode 1 = squared coefficients (used by or_jacobi_diag with x = 1).
 */
static void apply_impl(const or_tables *T, const double *diag, int transpose, int squared,
                       const double *x, double *y) {
    const int U = T->U;
    const int64_t nvox = (int64_t)T->nx * T->ny * T->nz;
    const int32_t *ptr = transpose ? T->t_ptr : T->a_ptr;
    const int32_t *oth = transpose ? T->t_src : T->a_tgt;
    const int32_t *dir = transpose ? T->t_dir : T->a_dir;
    const int32_t *isd = transpose ? T->t_diag : T->a_diag;
    const double *w = transpose ? T->t_w : T->a_w;
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < nvox; ++v) {
        int i = (int)(v % T->nx), j = (int)((v / T->nx) % T->ny), k = (int)(v / ((int64_t)T->nx * T->ny));
        int bb = boundary_bits(T, i, j, k);
        for (int c = 0; c < U; ++c) {
            double sum = 0.0;
            int pinned_c = (T->par[c] & bb) != 0;
            for (int e = ptr[c]; e < ptr[c + 1]; ++e) {
                int o = oth[e];
                double a, xv;
                if (isd[e]) {
                    a = diag[v * U + c];
                    xv = x[v * U + c];
                } else {
                    int nbb = 0;
                    int64_t u = neighbour(T, i, j, k, dir[e], &nbb);
                    if (u < 0 || pinned_c || (T->par[o] & nbb)) continue;
                    a = w[e];
                    xv = x[u * U + o];
                }
                if (squared) a = a * a;
                sum = sum + a * xv;
            }
            y[v * U + c] = sum;
        }
    }
}

void or_apply(const or_tables *T, const double *diag, int transpose, const double *x, double *y) {
    apply_impl(T, diag, transpose, 0, x, y);
}

/* A.multiply(A).sum(axis=0): per column, squares added in ascending row order */
void or_jacobi_diag(const or_tables *T, const double *diag, double *out) {
    const int64_t R = (int64_t)T->nx * T->ny * T->nz * T->U;
    double *ones = (double *)malloc(sizeof(double) * R);
    for (int64_t r = 0; r < R; ++r) ones[r] = 1.0;
    apply_impl(T, diag, 1, 1, ones, out);
    free(ones);
}

/* CSR of A exactly as scipy's coo->csr leaves it: ascending columns, explicit
 * zeros kept.  Returns nnz; pass NULL buffers to count only. */
int64_t or_csr(const or_tables *T, const double *diag, int64_t *indptr, int32_t *indices, double *data) {
    const int U = T->U;
    const int64_t nvox = (int64_t)T->nx * T->ny * T->nz;
    int64_t nnz = 0;
    if (indptr) indptr[0] = 0;
    for (int64_t v = 0; v < nvox; ++v) {
        int i = (int)(v % T->nx), j = (int)((v / T->nx) % T->ny), k = (int)(v / ((int64_t)T->nx * T->ny));
        int bb = boundary_bits(T, i, j, k);
        for (int c = 0; c < U; ++c) {
            int pinned_c = (T->par[c] & bb) != 0;
            for (int e = T->a_ptr[c]; e < T->a_ptr[c + 1]; ++e) {
                int o = T->a_tgt[e];
                int64_t col;
                double a;
                if (T->a_diag[e]) { col = v * U + c; a = diag[v * U + c]; }
                else {
                    int nbb = 0;
                    int64_t u = neighbour(T, i, j, k, T->a_dir[e], &nbb);
                    if (u < 0 || pinned_c || (T->par[o] & nbb)) continue;
                    col = u * U + o; a = T->a_w[e];
                }
                if (indices) { indices[nnz] = (int32_t)col; data[nnz] = a; }
                ++nnz;
            }
            if (indptr) indptr[v * U + c + 1] = nnz;
        }
    }
    return nnz;
}

/*
 * Neumann CSR: every entry of row (v, c) is written, its target index
 * clipped into the domain; tocsr() then orders each row by column and sums
 * entries that share one (sum_duplicates).  Per row: collect (col, value) in
 * program order, stable insertion sort by column, sum equal neighbours left
 * to right.  neumann = 0 gives or_csr.
 */
int64_t or_csr_bc(const or_tables *T, const double *diag, int neumann, int64_t *indptr, int32_t *indices,
                  double *data) {
    if (!neumann) return or_csr(T, diag, indptr, indices, data);
    const int U = T->U;
    const int64_t nvox = (int64_t)T->nx * T->ny * T->nz;
    int64_t nnz = 0;
    int64_t cols[256];
    double vals[256];
    if (indptr) indptr[0] = 0;
    for (int64_t v = 0; v < nvox; ++v) {
        int i = (int)(v % T->nx), j = (int)((v / T->nx) % T->ny), k = (int)(v / ((int64_t)T->nx * T->ny));
        for (int c = 0; c < U; ++c) {
            int n = 0;
            for (int e = T->a_ptr[c]; e < T->a_ptr[c + 1]; ++e) {
                int64_t col;
                double a;
                if (T->a_diag[e]) { col = v * U + c; a = diag[v * U + c]; }
                else {
                    int d = T->a_dir[e];
                    int ii = i + DX[d], jj = j + DY[d], kk = k + DZ[d];
                    ii = ii < 0 ? 0 : (ii >= T->nx ? T->nx - 1 : ii);
                    jj = jj < 0 ? 0 : (jj >= T->ny ? T->ny - 1 : jj);
                    kk = kk < 0 ? 0 : (kk >= T->nz ? T->nz - 1 : kk);
                    col = ((int64_t)ii + (int64_t)T->nx * (jj + (int64_t)T->ny * kk)) * U + T->a_tgt[e];
                    a = T->a_w[e];
                }
                int p = n;
                while (p > 0 && cols[p - 1] > col) { cols[p] = cols[p - 1]; vals[p] = vals[p - 1]; --p; }
                cols[p] = col; vals[p] = a; ++n;
            }
            for (int q = 0; q < n; ++q) {
                double acc = vals[q];
                while (q + 1 < n && cols[q + 1] == cols[q]) acc += vals[++q];
                if (indices) { indices[nnz] = (int32_t)cols[q]; data[nnz] = acc; }
                ++nnz;
            }
            if (indptr) indptr[v * U + c + 1] = nnz;
        }
    }
    return nnz;
}

/* ------------------------------------------------------------------------ */
/* OpenBLAS 0.3.30 ddot emulation (kernel/x86_64/ddot.c driver + microkernels) */
/* ------------------------------------------------------------------------ */

/* SkylakeX: 4x8-lane FMA over 32-blocks, fold to 4x4 lanes, 4x4-lane FMA over
 * 16-blocks, lanewise ((a0+a1)+a2)+a3, (s0+s2)+(s1+s3), FMA scalar tail. */
static double ddot_skx(int64_t n, const double *x, const double *y) {
    double a8[4][8], a4[4][4];
    memset(a8, 0, sizeof a8);
    int64_t i = 0, n32 = n & ~(int64_t)31, n16 = n & ~(int64_t)15;
    for (; i < n32; i += 32)
        for (int q = 0; q < 4; ++q)
            for (int l = 0; l < 8; ++l) a8[q][l] = fma(x[i + 8 * q + l], y[i + 8 * q + l], a8[q][l]);
    for (int q = 0; q < 4; ++q)
        for (int l = 0; l < 4; ++l) a4[q][l] = a8[q][l] + a8[q][l + 4];
    for (; i < n16; i += 16)
        for (int q = 0; q < 4; ++q)
            for (int l = 0; l < 4; ++l) a4[q][l] = fma(x[i + 4 * q + l], y[i + 4 * q + l], a4[q][l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = ((a4[0][l] + a4[1][l]) + a4[2][l]) + a4[3][l];
    double dot = n16 ? (s[0] + s[2]) + (s[1] + s[3]) : 0.0;
    for (i = n16; i < n; ++i) dot = fma(y[i], x[i], dot);
    return dot;
}

/* Haswell: 4x4-lane FMA over 16-blocks, fold to 2 lanes, (h0+h1)+(h2+h3),
 * lane sum, mul-then-add scalar tail. */
static double ddot_hsw(int64_t n, const double *x, const double *y) {
    double a4[4][4];
    memset(a4, 0, sizeof a4);
    int64_t i = 0, n16 = n & ~(int64_t)15;
    for (; i < n16; i += 16)
        for (int q = 0; q < 4; ++q)
            for (int l = 0; l < 4; ++l) a4[q][l] = fma(x[i + 4 * q + l], y[i + 4 * q + l], a4[q][l]);
    double t[2];
    for (int l = 0; l < 2; ++l) {
        double h0 = a4[0][l] + a4[0][l + 2], h1 = a4[1][l] + a4[1][l + 2];
        double h2 = a4[2][l] + a4[2][l + 2], h3 = a4[3][l] + a4[3][l + 2];
        t[l] = (h0 + h1) + (h2 + h3);
    }
    double dot = n16 ? t[0] + t[1] : 0.0;
    for (i = n16; i < n; ++i) dot = dot + y[i] * x[i];
    return dot;
}

/* kernel: 0 = SkylakeX, 1 = Haswell; threads = OpenBLAS thread count */
double or_ddot(int64_t n, const double *x, const double *y, int threads, int kernel) {
    double (*kern)(int64_t, const double *, const double *) = kernel ? ddot_hsw : ddot_skx;
    if (n <= 0) return 0.0;
    if (n <= 10000 || threads <= 1) return kern(n, x, y);
    double dot = 0.0;
    int64_t rem = n, off = 0;
    for (int t = 0; t < threads && rem > 0; ++t) {
        int64_t width = (rem + (threads - t) - 1) / (threads - t);
        if (width > rem) width = rem;
        dot = dot + kern(width, x + off, y + off);
        off += width;
        rem -= width;
    }
    return dot;
}

/* ------------------------------------------------------------------------ */
/* CGNR (solver.py:189-257), numpy semantics op for op                       */
/* ------------------------------------------------------------------------ */

typedef struct {
    double tol;
    int64_t max_iter;
    double primal_tol;     /* < 0 means None */
    int32_t jacobi;
    int32_t blas_threads, blas_kernel;
} or_cg_opts;

typedef struct {
    int64_t iterations;
    int32_t converged;
    double normal_residual, primal_residual;
} or_cg_report;

/* generic operator: stencil tables or a CSR matrix (and its transpose) */
typedef struct {
    const or_tables *T;
    const double *diag;
    int64_t n;
    const int64_t *ap; const int32_t *aj; const double *ax;     /* A   (CSR) */
    const int64_t *tp; const int32_t *tj; const double *tx;     /* A^T (CSR) */
} or_op;

static void csr_matvec(int64_t n, const int64_t *p, const int32_t *j, const double *a, const double *x, double *y) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        double s = 0.0;
        for (int64_t e = p[r]; e < p[r + 1]; ++e) s = s + a[e] * x[j[e]];
        y[r] = s;
    }
}

static void op_apply(const or_op *op, int transpose, const double *x, double *y) {
    if (op->T) apply_impl(op->T, op->diag, transpose, 0, x, y);
    else if (transpose) csr_matvec(op->n, op->tp, op->tj, op->tx, x, y);
    else csr_matvec(op->n, op->ap, op->aj, op->ax, x, y);
}

/* minv supplied by the caller when jacobi (diag with 0 -> 1, then 1/diag) */
int or_cgnr(const or_op *op, const double *b, const double *x0, const double *minv,
            const or_cg_opts *o, double *x, or_cg_report *rep,
            double *normal_hist, double *primal_hist) {
    const int64_t n = op->n;
    const int th = o->blas_threads, kn = o->blas_kernel;
    rep->iterations = 0; rep->converged = 0;
    rep->normal_residual = INFINITY; rep->primal_residual = INFINITY;
    double *r = malloc(8 * n), *z = malloc(8 * n), *zt = malloc(8 * n), *p = malloc(8 * n), *w = malloc(8 * n);
    double *tmp = malloc(8 * n);
    double norm_b = sqrt(or_ddot(n, b, b, th, kn));
    op_apply(op, 1, b, tmp);
    double norm_atb = sqrt(or_ddot(n, tmp, tmp, th, kn));
    if (norm_atb == 0.0 || norm_b == 0.0) {
        for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
        rep->converged = 1; rep->normal_residual = 0.0; rep->primal_residual = 0.0;
        free(r); free(z); free(zt); free(p); free(w); free(tmp);
        return 0;
    }
    for (int64_t i = 0; i < n; ++i) x[i] = x0 ? x0[i] : 0.0;
    op_apply(op, 0, x, tmp);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - tmp[i];
    op_apply(op, 1, r, z);
    const double *ztp = z;
    if (minv) { for (int64_t i = 0; i < n; ++i) zt[i] = z[i] * minv[i]; ztp = zt; }
    memcpy(p, ztp, 8 * n);
    double rho = or_ddot(n, z, ztp, th, kn);
    for (int64_t it = 1; it <= o->max_iter; ++it) {
        op_apply(op, 0, p, w);
        double ww = or_ddot(n, w, w, th, kn);
        if (ww == 0.0) break;
        double alpha = rho / ww;
        for (int64_t i = 0; i < n; ++i) x[i] = x[i] + alpha * p[i];
        for (int64_t i = 0; i < n; ++i) r[i] = r[i] - alpha * w[i];
        op_apply(op, 1, r, z);
        if (minv) for (int64_t i = 0; i < n; ++i) zt[i] = z[i] * minv[i];
        double rho_new = or_ddot(n, z, ztp, th, kn);
        double normal_rel = sqrt(or_ddot(n, z, z, th, kn)) / norm_atb;
        double primal_rel = sqrt(or_ddot(n, r, r, th, kn)) / norm_b;
        if (normal_hist) normal_hist[it - 1] = normal_rel;
        if (primal_hist) primal_hist[it - 1] = primal_rel;
        rep->iterations = it;
        if (normal_rel <= o->tol && (o->primal_tol < 0 || primal_rel <= o->primal_tol)) {
            rep->converged = 1;
            break;
        }
        double beta = rho != 0.0 ? rho_new / rho : 0.0;
        for (int64_t i = 0; i < n; ++i) p[i] = ztp[i] + beta * p[i];
        rho = rho_new;
    }
    op_apply(op, 0, x, tmp);
    for (int64_t i = 0; i < n; ++i) tmp[i] = tmp[i] - b[i];
    op_apply(op, 1, tmp, w);
    rep->normal_residual = sqrt(or_ddot(n, w, w, th, kn)) / norm_atb;
    rep->primal_residual = sqrt(or_ddot(n, tmp, tmp, th, kn)) / norm_b;
    free(r); free(z); free(zt); free(p); free(w); free(tmp);
    return 0;
}

/* (*res, U) C-order collocated grid: nested 0.5*(g + g_lower) along each
 * staggered axis in x, y, z order, sample 0 replicated (solver.py:275-296) */
void or_unstagger(const or_tables *T, const double *u, double *out) {
    const int U = T->U, nx = T->nx, ny = T->ny, nz = T->nz;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < (int64_t)nx * ny * nz; ++q) {
        int i = (int)(q / ((int64_t)ny * nz)), j = (int)((q / nz) % ny), k = (int)(q % nz);
        for (int c = 0; c < U; ++c) {
            int par = T->par[c];
            /* value at the sample set: process axes in order, each averaging
             * with the lower neighbour (clamped) of the already-averaged grid */
            double g[8];
            /* the 2^popcount lower-corner samples, bit b = lower along ax[b] */
            int ax[3], na = 0;
            for (int a = 0; a < 3; ++a) if (par >> a & 1) ax[na++] = a;
            int n = 1 << na;
            for (int s = 0; s < n; ++s) {
                int ii = i, jj = j, kk = k;
                for (int b = 0; b < na; ++b) if (s >> b & 1) {
                    if (ax[b] == 0) ii = ii > 0 ? ii - 1 : 0;
                    if (ax[b] == 1) jj = jj > 0 ? jj - 1 : 0;
                    if (ax[b] == 2) kk = kk > 0 ? kk - 1 : 0;
                }
                g[s] = u[((int64_t)ii + (int64_t)nx * (jj + (int64_t)ny * kk)) * U + c];
            }
            /* combine axis b: g[s] = 0.5*(g[s] + g[s | bit]) for s without bit */
            for (int b = 0; b < na; ++b)
                for (int s = 0; s < n; ++s)
                    if (!(s >> b & 1)) g[s] = 0.5 * (g[s] + g[s | (1 << b)]);
            out[q * U + c] = g[0];
        }
    }
}
