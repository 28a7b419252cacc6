/*
 * pnrte_b200 — C ABI of the B200 (sm_100a) P_N solve path.
 *
 * Drop-in boundary for the reference's runtime functions (pnrte):
 *   assemble(program, spec)            pkg/src/pnrte/solver.py:96      -> pn_create + pn_set_field + pn_setup
 *   solve_normal_cg(system, tol, max_iter, primal_tol, jacobi, x0)
 *                                      pkg/src/pnrte/solver.py:189-190 -> pn_solve
 *   A @ x, A.T @ x (csr_matvec)        pkg/src/pnrte/solver.py:209,226-227,232,239 -> pn_apply
 *   unstagger(u, program, res)         pkg/src/pnrte/solver.py:275     -> pn_unstagger
 *   SparseSystem.A / .Q (debug parity) pkg/src/pnrte/solver.py:182-186 -> pn_export_diag_rhs
 *   A.multiply(A).sum(axis=0)          pkg/src/pnrte/solver.py:219     -> pn_jacobi_diag
 * The reference has no formal plugin ABI; its Python entry points are the
 * boundary.  The Python mirror in paper_1807_00410_b200/solver.py
 * binds these symbols with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Plain pointers and sizes, no torch types.  Unless a name says _host,
 *    vector pointers are DEVICE pointers on the context's device, stream
 *    ordered on the `stream` argument (a cudaStream_t, NULL = legacy default).
 *  - Vectors use the reference layout: index (i + nx*(j + ny*k))*U + comp,
 *    comp = l(l+1)+m, over the context's local z-slab [z0, z0+nz_local).
 *  - Every call returns PN_OK or an error code; pn_last_error() gives the
 *    message.  Non-convergence is NOT an error (report.converged), exactly
 *    like the reference (solver.py:247-250).
 *  - A context is single-stream and not thread safe; use one per GPU/rank.
 */
#ifndef PNRTE_B200_H
#define PNRTE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PN_OK 0
#define PN_ERR_INVALID 1      /* ValueError in the reference (e.g. tol <= 0, solver.py:200-201) */
#define PN_ERR_CUDA 2
#define PN_ERR_UNSUPPORTED 3  /* program outside the matrix-free P_N form */
#define PN_ERR_NCCL 4
#define PN_ERR_NOMEM 5

typedef struct pn_context pn_context;

/* Flat stencil tables (paper_1807_00410_b200/program.py:pack_tables), copied
 * at create.  a_* = rows of A in ascending column order, t_* = rows of A^T in
 * ascending column order, dir codes 0 same voxel, 1/2 -x/+x, 3/4 -y/+y, 5/6 -z/+z.
 * Term programs evaluate diag/RHS coefficients in expression-tree order. */
typedef struct {
    int32_t N, U;
    int32_t nx, ny, nz;          /* global grid */
    int32_t z0, nz_local;        /* this context's z-slab */
    double h;
    int32_t device;
    int32_t n_fields;            /* sigma_t, sigma_s, p_0..p_N, Q by comp */
    const int32_t *par;          /* [U] staggered parity bits x|y<<1|z<<2 */
    const double *lam;           /* [U] lambda_l of each comp */
    const int32_t *lidx;         /* [U] l of each comp */
    int32_t n_a, n_t, n_terms;
    const int32_t *a_ptr, *a_tgt, *a_dir, *a_diag; const double *a_w;
    const int32_t *t_ptr, *t_src, *t_dir, *t_diag; const double *t_w;
    const int32_t *d_ptr, *r_ptr, *term_hascoef, *term_nf, *term_f, *term_site;
    const double *term_coef;
    int32_t canonical_diag;      /* 1: diag = avg(st) - lam*p*avg(ss) form (program.canonical_diag) */
    /* multi-GPU: NCCL unique id bytes (128) or NULL for a single GPU */
    const void *nccl_id;
    int32_t rank, world;
} pn_desc;

int pn_create(const pn_desc *desc, pn_context **out);

/* Generic sparse system (any SparseSystem.A, solver.py:189 accepts them):
 * host CSR arrays (scipy layout), copied to the device; A^T is built on the
 * device in A.T.tocsr() order.  Usable with pn_apply / pn_jacobi_diag /
 * pn_solve (b required); stencil-only entry points return PN_ERR_UNSUPPORTED. */
int pn_create_csr(int64_t n, int64_t nnz, const int64_t *indptr, const int32_t *indices, const double *data,
                  int32_t device, pn_context **out);
int pn_destroy(pn_context *ctx);
const char *pn_last_error(void);

/* Assemble a single-GPU stencil context (fields set) into an explicit
 * device CSR system, exactly as assemble() builds it (solver.py:96-186):
 * bc 0 = Dirichlet (dropped writes, pinned rows), 1 = Neumann (writes
 * redirected to the nearest in-domain sample, solver.py:133-135,146-147;
 * duplicates summed, columns ascending, explicit zeros kept, i.e.
 * coo_matrix(...).tocsr() at solver.py:182-185).  Returns a new CSR context
 * (pn_create_csr semantics) and, when rhs is non-NULL, writes Q (device
 * buffer of R doubles; Neumann rows are not pinned). */
int pn_assemble_csr(pn_context *ctx, int32_t bc, double *rhs, pn_context **out, void *stream);

/* General stencil program (coefficients that depend on fields, e.g. the CDA
 * system of equations.py:213-237): every entry coefficient, diagonal and
 * residual is a postfix program (paper_1807_00410_b200/general.py) that
 * pn_assemble_general evaluates per voxel on the device with numpy's
 * arithmetic, then assembles the CSR exactly as pn_assemble_csr does
 * (bc 0 Dirichlet / 1 Neumann).  All arrays are HOST arrays except the field
 * data (DEVICE, the reference's [i,j,k] C-order grids; 2-D: nz = 1).  Ops are
 * (opcode, argument) pairs: 0 end, 1 push consts[a], 2 push sample a (field
 * s_slot[a] at voxel + (s_dx, s_dy, s_dz)[a], clamped to the grid), 3 add,
 * 4 mul, 5 reciprocal, 6 square, 7 sqrt, 8 ones.  The returned CSR context
 * keeps the grid and row parities, so pn_unstagger works on it. */
typedef struct {
    int32_t U, nx, ny, nz;
    int32_t device;
    const int32_t *par;          /* [U] row location parity bits (x | y<<1 | z<<2) */
    const int32_t *e_ptr;        /* [U+1] */
    const int32_t *e_tgt, *e_dx, *e_dy, *e_dz, *e_diag, *e_code;   /* per entry, program order */
    const int32_t *r_code;       /* [U] residual program (RHS = -value) */
    const int32_t *ops; int32_t n_ops;          /* n_ops pairs */
    const double *consts; int32_t n_consts;
    const int32_t *s_slot, *s_dx, *s_dy, *s_dz; int32_t n_samples;
    int32_t n_fields;            /* <= 32 */
    const int32_t *f_kind;       /* 0 absent (zero), 1 uniform scalar, 2 device array */
    const double *f_scalar;
    const double *const *f_data;
} pn_general_desc;

int pn_assemble_general(const pn_general_desc *desc, int32_t bc, double *rhs, pn_context **out, void *stream);

/* Download a CSR context's A in scipy layout into HOST buffers (the
 * assembled system's A.indptr / A.indices / A.data).  NULL arrays: only
 * *nnz is written. */
int pn_csr_export(pn_context *csr, int64_t *nnz, int64_t *indptr, int32_t *indices, double *data);

/* Field slot s (order of desc): kind 0 = absent (zero), 1 = uniform scalar,
 * 2 = array.  Arrays are the reference's [i,j,k] C-order global field
 * (z fastest) in DEVICE memory; the context transposes its slab (+1 plane).
 * Fields are consumed by pn_setup and may be freed afterwards. */
int pn_set_field(pn_context *ctx, int32_t slot, int32_t kind, double scalar,
                 const double *data, void *stream);

/* Same for a z-range of the field: `data` holds the [i,j,k] C-order planes
 * [k0, k0 + n_planes) of the global field (shape nx x ny x n_planes), which
 * must cover the context's slab [z0, z0 + nz_local) and its +1 plane
 * (clamped at nz).  One rank of a slab decomposition then never holds the
 * global field (config 5: 1.07 GB per field at 512^3). */
int pn_set_field_planes(pn_context *ctx, int32_t slot, int32_t kind, double scalar,
                        const double *data, int32_t k0, int32_t n_planes, void *stream);

/* Evaluate diagonal (when needed) and RHS Q from the fields (assemble()). */
int pn_setup(pn_context *ctx, void *stream);

/* Copy the assembled diagonal and RHS into caller buffers (parity/debug). */
int pn_export_diag_rhs(pn_context *ctx, double *diag, double *rhs, void *stream);

/* y = A x (transpose = 0) or A^T x (transpose = 1).
 * mode 0 = fast (B200 kernel), 1 = faithful (scipy csr_matvec order, no FMA). */
int pn_apply(pn_context *ctx, int32_t transpose, int32_t mode, const double *x, double *y, void *stream);

/* colsum(A o A) with 0 kept (the reference replaces 0 by 1 afterwards). */
int pn_jacobi_diag(pn_context *ctx, double *out, void *stream);

typedef struct {
    double tol;                  /* > 0 */
    int64_t max_iter;
    double primal_tol;           /* < 0 means None */
    int32_t jacobi;
    int32_t mode;                /* 0 fast, 1 faithful */
    int32_t blas_threads;        /* faithful: OpenBLAS thread count to emulate */
    int32_t blas_kernel;         /* faithful: 0 SkylakeX, 1 Haswell; 2 = pairwise order (noise-floor probe, no OpenBLAS twin) */
    int32_t check_every;         /* host polls the device stop flag every k iterations (0 = auto) */
} pn_solve_opts;

typedef struct {
    int64_t iterations;
    int32_t converged;
    double normal_residual;      /* ||A^T(Ax-b)|| / ||A^T b|| */
    double primal_residual;      /* ||Ax-b|| / ||b|| */
    double wall_time;            /* seconds, device events around the solve */
} pn_report;

/* CGNR (solve_normal_cg).  b = NULL uses the assembled RHS.  x0 may be NULL.
 * x is written (local slab).  Histories are HOST buffers of hist_cap entries
 * (may be NULL).  Synchronises the stream before returning the report. */
int pn_solve(pn_context *ctx, const pn_solve_opts *opts, const double *b, const double *x0,
             double *x, pn_report *report, double *normal_hist, double *primal_hist,
             int64_t hist_cap, void *stream);

/* Collocated coefficients (*res, U) C-order for the local slab (unstagger()).
 * Reads the k-1 plane of z-staggered comps from the lower neighbour on
 * multi-GPU.  out: [nx][ny][nz_local][U]. */
int pn_unstagger(pn_context *ctx, const double *u, double *out, void *stream);

/* Context-free unstagger for any program (row parities par[U], host):
 * u and out are device buffers as in pn_unstagger (single GPU). */
int pn_unstagger_grid(const int32_t *par, int32_t U, int32_t nx, int32_t ny, int32_t nz, const double *u,
                      double *out, void *stream);

/* Post-processing of collocated coefficients (DEVICE arrays; grids are the
 * (*res, U) C-order output of pn_unstagger):
 *   pn_fluence      out[v] = sqrt(4 pi) * coll[v, 0]                 solver.py:299-301
 *   pn_trilinear    out[p, q] = trilinear(coll[..., q], pts[p])      solver.py:304-327
 *   pn_reconstruct  out[p, d] = radiance at pts[p] in direction dirs[d]
 *                   (trilinear coefficients . real SH basis)        solver.py:330-343
 * pts: [npts][dim] world positions inside the domain (the caller checks,
 * as the reference raises OutOfDomainError); dirs: [ndirs][3], any length;
 * lm: HOST [U][2] (l, m) per component (unknown_order). */
int pn_fluence(const double *coll, int64_t nvox, int32_t U, double *out, void *stream);
int pn_trilinear(const double *coll, int32_t dim, const int32_t *res, int32_t U, const double *origin, double h,
                 int64_t npts, const double *pts, double *out, void *stream);
int pn_reconstruct(const double *coll, int32_t dim, const int32_t *res, int32_t U, const int32_t *lm,
                   const double *origin, double h, int64_t npts, const double *pts, int64_t ndirs,
                   const double *dirs, double *out, void *stream);

/* Host-buffer composite (e2e): host fields already set, host x out. */
int pn_solve_host(pn_context *ctx, const pn_solve_opts *opts, double *x_host,
                  pn_report *report, double *normal_hist, double *primal_hist, int64_t hist_cap);

/* Number of fast-path kernels launched by this context since creation. */
int64_t pn_kernel_launches(pn_context *ctx);

/* NCCL unique id (128 bytes) for multi-GPU creation (rank 0 calls it). */
int pn_nccl_unique_id(void *out128);

/* One-rank check of the NCCL call patterns of the slab path on `device`
 * (communicator, grouped send/recv, in-place all-gather, captured into a CUDA
 * graph on a forked stream and replayed) over n doubles; PN_OK or an error. */
int pn_nccl_selftest(int device, int n);

/* Loopback slab group: several contexts on ONE device whose halos and
 * partial sums are exchanged by device copies instead of NCCL (tests of the
 * slab decomposition on one GPU).  Contexts must be created with world > 1,
 * nccl_id = NULL, ranks 0..n-1 in order. */
int pn_group_solve(pn_context **ctxs, int32_t n, const pn_solve_opts *opts, double **x,
                   pn_report *report, double *normal_hist, double *primal_hist, int64_t hist_cap,
                   void *stream);
int pn_group_apply(pn_context **ctxs, int32_t n, int32_t transpose, int32_t mode,
                   const double **x, double **y, void *stream);

/* Kernel-level timing hooks for bench.py: run `reps` back-to-back fast
 * operations on internal buffers and return the average device time per
 * launch in milliseconds.  what: 0 applies (A / A^T alternating), 1 fused CG
 * iterations, 2 applies with the fused reductions, 3 applies predicated on the
 * stop flag, 4 the r update (r -= alpha w, ||r||^2), 5 the x / p update. */
int pn_bench(pn_context *ctx, int32_t what, int32_t reps, double *ms_per, void *stream);

#ifdef __cplusplus
}
#endif
#endif
