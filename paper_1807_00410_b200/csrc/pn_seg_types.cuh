// Host/device shared types of the segmented fast operator.
#pragma once

namespace pn {

constexpr int SEG_MAXW = 128;   // distinct |weight| values per table (80 for P7)
// Launch shape per order N: warps (32-voxel rows along y) per CTA and the
// CTAs per SM the register budget targets.  Shared memory holds one staged
// row per warp (32*U doubles + edges + sigma rows).
#ifdef PN_SEG_ROWS_OVERRIDE
__host__ __device__ constexpr int seg_rows(int) { return PN_SEG_ROWS_OVERRIDE; }
__host__ __device__ constexpr int seg_minb(int) { return PN_SEG_MINB_OVERRIDE; }
__host__ __device__ constexpr bool seg_pair(int) { return PN_SEG_PAIR_OVERRIDE; }
#else
// pair: two warps share one staged row, each computing half of the classes.
// P5 (config 3): one warp per row, 4 CTAs of 4 rows per SM at 128 registers
// (no spills) measured 328 vs 322 Gunk/s for warp pairs at 80 registers
// (profiles/r01_sweep_p5_shape.log); P7 cannot hold 4 CTAs of staged rows.
__host__ __device__ constexpr bool seg_pair(int N) { return N >= 3 && N != 5; }
__host__ __device__ constexpr int seg_rows(int N) { return N <= 2 ? 8 : 4; }
__host__ __device__ constexpr int seg_minb(int N) { return N <= 2 ? 4 : (N == 5 ? 4 : (N <= 6 ? 3 : 2)); }
#endif

struct SegParams {
    double w[SEG_MAXW];   // distinct |a_w| (or |t_w|) magnitudes, exact reference values
    double lamp[64];      // lambda_l * p_l per comp
};

// n / d for 0 <= n < 2^31 by multiply-high and shift (m = ceil(2^(31+l) / d),
// l = ceil(log2 d)); d = 1 passes n through.  Replaces the 64-bit division
// of the CTA -> row-block map (about 40 instructions each, three per CTA).
struct FastDiv {
    unsigned d, m, s;
};
inline FastDiv make_fastdiv(unsigned d) {
    FastDiv f{d, 0u, 0u};
    if (d <= 1) return f;
    unsigned l = 0;
    while ((1ull << l) < d) ++l;
    f.m = (unsigned)(((1ull << (31 + l)) + d - 1) / d);
    f.s = l - 1;
    return f;
}
#ifdef __CUDACC__
__device__ __forceinline__ unsigned fdiv(unsigned n, const FastDiv &f) { return f.m ? (__umulhi(n, f.m) >> f.s) : n; }
#endif

struct SegGeo {
    int U, nx, ny, nz, z0, nzl, nseg, nyb;
    int tyb;                 // row blocks per y-tile of the CTA traversal
    int kl0, npl, kst;       // local planes kl0 + i*kst, i < npl, computed by one launch
    int sx;                  // row stride of the sigma slabs the kernel reads (nx, or nseg*32 when padded)
    int bulk;                // 1: bulk (TMA) staging path, for slabs far larger than L2
    long long plane, pvox;
    FastDiv dseg, dtyb, dnpl;   // set per launch by seg_launch (nseg, min(tyb, nyb), npl)
};

// Schedule of the fused residual update + A^T apply (k_seg_fr): work units are
// handed out by ticket.  Per y-tile T of the z-marching traversal and step s:
// the residual-update chunks (k_r blocks) of plane s that overlap the tile and
// one row line beyond it, then the row groups of plane s - D of the tile.
constexpr int FUSE_MAX_TILES = 64;
struct FuseSched {
    int ntiles, D, vec_bx, pad_;
    long long chunk;                             // doubles per residual-update chunk
    unsigned tile_start[FUSE_MAX_TILES + 1];     // first ticket of tile T
    int c_lo[FUSE_MAX_TILES], n_u[FUSE_MAX_TILES], n_a[FUSE_MAX_TILES];
    unsigned *ctl;                               // {next ticket, CTAs finished, epoch}
    unsigned *flags;                             // [nz][vec_bx]: epoch of the chunk's last update
};

struct State;

template <int N>
int seg_launch(const SegParams &prm, const SegGeo &g, int trans, int red, bool jac, const double *x, double *y,
               const double *minv, double *zt, const double *st, const double *ss, double *partials,
               long long slot_stride, int rb, const State *state, cudaStream_t s);

// fused r -= alpha w ; z = A^T r (+ reductions): single slab, bulk path, 256-thread CTAs
template <int N>
int seg_launch_fused_r(const SegParams &prm, const SegGeo &g, const FuseSched &f, bool jac, double *r, const double *w,
                       double *z, const double *minv, double *zt, const double *st, const double *ss,
                       double *partials, long long slot_stride, int rb, const State *state, cudaStream_t s);

}  // namespace pn
