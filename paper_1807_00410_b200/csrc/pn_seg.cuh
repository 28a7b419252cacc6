// Segmented (32-voxel AoSoA) fast path of the P_N operator: host interface.
#pragma once
#include "pn_internal.cuh"

namespace pn {
// true when the fast solve can run in the segmented layout for this context
bool pn_seg_ok(const pn_context *c);
// one-time preparation after pn_setup (parameter blocks, layout checks)
int pn_seg_prepare(pn_context *c, cudaStream_t s);
// y = A x or A^T x on segmented-layout vectors (padded, local slab)
int pn_seg_apply(pn_context *c, int trans, const double *x, double *y, int red, const double *minv, double *zt,
                 bool gated, cudaStream_t s, int kl0 = 0, int npl = -1, int kst = 1);
// true when the fused residual update + A^T apply is available for this context
bool pn_seg_fused_r_ok(const pn_context *c);
// r -= alpha w (with its ||r||^2 partials) ; z = A^T r (with the z reductions), one launch
int pn_seg_apply_fused_r(pn_context *c, double *r, const double *w, double *z, const double *minv, double *zt,
                         cudaStream_t s);
// layout conversion of one local-slab vector: dir 0 = reference -> segmented, 1 = back
int pn_seg_convert(pn_context *c, int dir, const double *src, double *dst, cudaStream_t s);
void pn_seg_release(pn_context *c);
// reduction blocks per plane the segmented kernel produces (0 when unused)
int pn_seg_red_blocks(const pn_context *c);
}  // namespace pn
