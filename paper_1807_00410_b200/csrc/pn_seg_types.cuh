// Host/device shared types of the segmented fast operator.
#pragma once

namespace pn {

constexpr int SEG_MAXW = 1024;
constexpr int SEG_ROWS = 8;   // warps (rows along y) per CTA

struct SegParams {
    double w[SEG_MAXW];   // table weights (a_w or t_w), exact reference values
    double lamp[64];      // lambda_l * p_l per comp
};

struct SegGeo {
    int U, nx, ny, nz, z0, nzl, nseg, nyb;
    long long plane, pvox;
};

struct State;

template <int N>
int seg_launch(const SegParams &prm, const SegGeo &g, int trans, int red, bool jac, const double *x, double *y,
               const double *minv, double *zt, const double *st, const double *ss, double *partials,
               long long slot_stride, int rb, const State *state, cudaStream_t s);

}  // namespace pn
