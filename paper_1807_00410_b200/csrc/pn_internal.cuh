// Internal types of the B200 P_N runtime (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pnrte_b200.h"

namespace pn {

// ---------------------------------------------------------------- errors --
void set_error(const std::string &msg);
#define PN_CUDA(call)                                                              \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            ::pn::set_error(std::string(#call) + ": " + cudaGetErrorString(e_));   \
            return PN_ERR_CUDA;                                                    \
        }                                                                          \
    } while (0)
#define PN_TRY(call)            \
    do {                        \
        int s_ = (call);        \
        if (s_ != PN_OK) return s_; \
    } while (0)

// --------------------------------------------------------- device tables --
// Everything a kernel needs to know about the operator, passed by value.
struct Geo {
    int U, nx, ny, nz;      // global grid
    int z0, nzl;            // slab
    long long plane;        // doubles per z-plane of a vector = nx*ny*U
    long long pvox;         // voxels per plane = nx*ny
};

struct Tables {
    const int *par;         // [U] parity bits
    const double *lamp;     // [U] lambda_l * p_l (uniform phase fields)
    const int *a_ptr, *a_tgt, *a_dir, *a_diag; const double *a_w;
    const int *t_ptr, *t_src, *t_dir, *t_diag; const double *t_w;
    const int *d_ptr, *r_ptr, *hascoef, *nf, *tf, *tsite; const double *tcoef;
    int n_a, n_t;
};

constexpr int MAX_FIELDS = 2 + 8 + 64 + 8;
struct Fields {
    int n;
    int kind[MAX_FIELDS];
    double scalar[MAX_FIELDS];
    const double *data[MAX_FIELDS];   // slab arrays, (nzl+1) planes, x fastest
};

// device-resident solver scalars (one struct, updated by scalar kernels)
struct State {
    double rho, alpha, beta;
    double norm_b, norm_atb;
    double ww, zz, zzt, rr;
    double tol, primal_tol;
    long long it;           // completed iterations
    long long max_iter;
    int done;               // stop flag: all iteration kernels become no-ops
    int converged;
    int zero_ww;
    int xupd;               // fast path: x += alpha p still pending for this iteration
};

// number of fast-reduction partial slots per (plane, block)
constexpr int RED_SLOTS = 4;   // 0: ww / zzt, 1: zz, 2: rr, 3: spare

struct Comm;   // halo + partial exchange (NCCL or loopback)

// generic CSR operator (pn_csr.cu): A as given, A^T as A.T.tocsr()
struct CsrOp {
    long long n = 0, nnz = 0;
    long long *ap = nullptr, *tp = nullptr;
    int *aj = nullptr, *tj = nullptr;
    double *ax = nullptr, *tx = nullptr;
    // grid of the stencil program the system was assembled from (unstagger)
    int *upar = nullptr;
    Geo ug{};
};

// general stencil program (pn_csr.cu, pn_assemble_general): postfix
// coefficient programs over field samples, device copies of pn_general_desc
enum GenOp { G_END = 0, G_NUM, G_FIELD, G_ADD, G_MUL, G_RECIP, G_SQUARE, G_SQRT, G_ONE };
constexpr int GEN_STACK = 16;
constexpr int GEN_FIELDS = 32;
struct GenProg {
    int U, nx, ny, nz;
    const int *par, *e_ptr, *e_tgt, *e_dx, *e_dy, *e_dz, *e_diag, *e_code, *r_code, *ops;
    const double *consts;
    const int *s_slot, *s_dx, *s_dy, *s_dz;
    int f_kind[GEN_FIELDS];
    double f_scalar[GEN_FIELDS];
    const double *f_data[GEN_FIELDS];   // reference [i][j][k] C-order arrays
};

// ------------------------------------------------------------- context --
struct Buf {
    double *alloc = nullptr;  // includes one halo plane each side
    double *p = nullptr;      // interior base (plane 0 of the slab)
};

}  // namespace pn

struct pn_context {
    int N = 0, U = 0;
    pn::Geo g{};
    double h = 0;
    int device = 0;
    int rank = 0, world = 1;
    int canonical_diag = 0;
    int uniform_phase = 1;
    int n_fields = 0;

    // tables (device)
    std::vector<void *> dev_allocs;
    pn::Tables tb{};
    std::vector<int> h_par, h_lidx;
    std::vector<double> h_lam;

    // fields
    pn::Fields f{};
    std::vector<double *> field_alloc;

    // assembled operator state
    double *diag = nullptr;       // [R_l] (faithful / non-canonical path)
    pn::Buf b;                    // RHS
    bool setup_done = false;
    bool diag_ready = false;

    // Krylov vectors (padded with z-halo planes)
    pn::Buf x, r, p, z, zt, w, tmp, minv;
    bool vecs_ready = false;
    bool bench_ready = false;

    // reductions
    int red_bx = 0;               // partial slots per plane (stride of the partials array)
    int vec_bx = 0;               // blocks per plane of the vector / table / dot kernels
    double *partials = nullptr;   // [RED_SLOTS][nz][red_bx] block partials (global plane index)
    double *plane_sums = nullptr; // [RED_SLOTS][nz] level-1 sums (all-gathered across ranks)
    unsigned *counter = nullptr;  // finished-block count of the fused plane-sum / scalar launch
    double *small_parts = nullptr;// [4][SMALL_MAX_BLOCKS] block partials of the one-launch small solve
    double *small_vecs = nullptr; // [2][R_l] second p and r buffers of the one-launch small solve
    double *ddot_chunks = nullptr;// faithful ddot chunk results [4][64]
    pn::State *state = nullptr;   // device
    pn::State *h_state = nullptr; // pinned host mirror
    double *hist_n = nullptr, *hist_p = nullptr;  // device histories
    long long hist_len = 0;

    // comm
    pn::Comm *comm = nullptr;
    void *nccl = nullptr;         // ncclComm_t

    long long launches = 0;

    // multi-slab: halo exchange on its own stream, overlapped with interior planes
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t cev_ready = nullptr, cev_halo = nullptr;

    // CUDA graph of a batch of CGNR iterations (single context, no NCCL)
    cudaStream_t gstream = nullptr;
    cudaEvent_t gev0 = nullptr, gev1 = nullptr;
    cudaGraphExec_t gexec = nullptr;
    long long gkey = -1;           // (mode, jacobi, seg, batch) the graph was captured for
    long long graph_launches = 0;  // kernels per graph replay
    long long gen = 0;             // bumped whenever captured arguments may change (drop_graph)
    std::vector<std::pair<pn_context *, long long>> gmembers;   // (context, gen) the graph captured

    // segmented fast path (pn_seg.cu)
    void *seg = nullptr;
    pn::Buf bs;                   // RHS in the solve layout
    std::vector<double> h_aw, h_tw;
    std::vector<int> h_aptr, h_atgt, h_adir, h_adiag, h_tptr, h_tsrc, h_tdir, h_tdiag;   // structure checks
    // residual (RHS) term program on the host: comps whose terms use only
    // constant factors get their value once per setup (k_setup skips them)
    std::vector<int> h_rptr, h_hascoef, h_nf, h_tf;
    std::vector<double> h_tcoef;
    std::vector<int> h_rmode;       // per comp: 1 = constant RHS
    std::vector<double> h_rconst;   // per comp: that constant (exact device arithmetic)
    int *d_rmode = nullptr;
    double *d_rconst = nullptr;

    // generic CSR system instead of a stencil (pn_create_csr)
    bool is_csr = false;
    pn::CsrOp csr;

    long long R_l() const { return (long long)g.nzl * g.plane; }
    // solve layout of the segmented operator: rows of 32 voxels along x, the
    // last one zero-padded when nx % 32 != 0 (single-slab contexts only);
    // splane doubles per z-plane (== g.plane without padding)
    long long splane = 0;
    bool seg_active = false;      // a fast segmented solve / bench is running: vector kernels use splane
    long long R_s() const { return (long long)g.nzl * splane; }
    long long vplane() const { return seg_active ? splane : g.plane; }
    long long nvox_l() const { return (long long)g.nzl * g.pvox; }
};

namespace pn {

// kernels (pn_kernels.cu)
int launch_fill(double *p, long long n, double v, cudaStream_t s);
// p[i] = uniform [-1, 1) from a hash of (seed, offset + i): dense deterministic
// bench inputs, identical for any slab decomposition (offset = global index)
int launch_fill_hash(double *p, long long n, long long offset, unsigned long long seed, cudaStream_t s);
// src: [i,j,k] C-order planes [src_k0, src_k0 + src_nk) of the field (src_nk <= 0: all nz planes)
int launch_field_slab(pn_context *c, int slot, const double *src, double *dst, cudaStream_t s, int src_k0 = 0,
                      int src_nk = 0);
int launch_setup(pn_context *c, bool want_diag, bool want_rhs, cudaStream_t s, double *rhs_out = nullptr, int pin = 1);
int launch_apply_table(pn_context *c, int trans, int faithful, int squared, const double *x, double *y, int red,
                       const double *minv, double *zt, cudaStream_t s, bool gated, int kl0 = 0, int npl = -1,
                       int kst = 1);
int launch_apply_faithful(pn_context *c, int trans, int squared, const double *x, double *y,
                          cudaStream_t s, bool gated = false);
int launch_r_update(pn_context *c, cudaStream_t s);
int launch_xp_update(pn_context *c, const double *zt, cudaStream_t s);
int launch_plane_sums(pn_context *c, int mask, int cnt, cudaStream_t s);
// single-slab: plane sums of `mask` (slot 3 with cnt3 partials) + scalar step `which` in one launch
int launch_plane_sums_scalar(pn_context *c, int mask, int cnt, int cnt3, int which, cudaStream_t s);
int launch_dot(pn_context *c, const double *a, const double *b, int slot, cudaStream_t s, bool gated = false);
int launch_ddot_emul(pn_context *c, const double *a, const double *b, long long n, int slot, int threads,
                     int kernel, cudaStream_t s, bool gated = false);
int launch_unstagger(pn_context *c, const double *u, double *out, cudaStream_t s);

// generic CSR (pn_csr.cu)
int csr_build(pn_context *c, long long n, long long nnz, const long long *ap, const int *aj, const double *ax);
// device assembly of a stencil context into canonical CSR (caller frees);
// rows may hold at most ASM_MAX table entries (P7: 21)
constexpr int ASM_MAX = 48;
int stencil_csr_assemble(pn_context *c, int neumann, cudaStream_t s, long long **ap, int **aj, double **ax,
                         long long *nnz);
int general_csr_assemble(const GenProg &P, int neumann, double *rhs, cudaStream_t s, long long **ap, int **aj,
                         double **ax, long long *nnz);
void csr_release(pn_context *c);
int launch_csr_apply(pn_context *c, int trans, int faithful, int squared, const double *x, double *y, int red,
                     const double *minv, double *zt, cudaStream_t s, bool gated);

// elementwise ops, see pn_kernels.cu for the op codes
int launch_vec(pn_context *c, int op, double *y, const double *a, const double *b, cudaStream_t s,
               bool gated = false);

enum VecOp {
    V_COPY = 0,        // y = a
    V_ZERO,            // y = 0
    V_SUB,             // y = a - b
    V_MUL,             // y = a * b
    V_RECIP_DIAG,      // y = 1/(a == 0 ? 1 : a)
    V_AXPY_ALPHA,      // y = y + (alpha * a)           (numpy: x += alpha*p)
    V_AXMY_ALPHA,      // y = y - (alpha * a)           (numpy: r -= alpha*w)
    V_P_UPDATE,        // y = a + (beta * y)            (numpy: p = zt + beta*p)
    V_FILL_ONE,        // y = 1
};

// reduction slots: 0 generic / ww, 1 zz, 2 z.zt, 3 rr (fast partials and
// faithful ddot chunks use the same numbering)
enum Scalar {
    S_NORMB = 0,       // norm_b = sqrt(slot 0)
    S_NORMATB,         // norm_atb = sqrt(slot 0)
    S_RHO,             // rho = slot 2
    S_ALPHA,           // ww = slot 0 -> alpha (or stop without counting)
    S_BETA,            // zz, zzt, rr -> history, stop test, beta, rho
    S_FINAL,           // zz = slot 0, rr = slot 3 (true residuals)
};
int launch_scalar(pn_context *c, int which, int faithful, int blas_threads, cudaStream_t s);

// Small single-slab fast solves: the whole CGNR iteration loop in one
// cooperative launch (reference layout, table operator).
constexpr int SMALL_MAX_BLOCKS = 2048;
int launch_cg_small(pn_context *c, bool jacobi, cudaStream_t s);
int cg_small_capacity(pn_context *c, long long *rows);

}  // namespace pn
