// z-marching variant of the segmented operator (included by pn_seg_common.cuh).
//
// A CTA owns ZM_ROWS consecutive 32-voxel rows (same segment, rows j0..) and
// marches a chunk of z-planes.  Every operand of a step lives in shared
// memory and is fetched one step ahead with cp.async:
//   * own rows: 4-slot plane ring (planes k-1, k, k+1 in use, k+2 landing);
//     the z neighbours are the ring slots k-1 / k+1 of the same row;
//   * y neighbours: the CTA's other rows, plus a double-buffered halo row
//     holding the y-bit-1 components of row j0-1 and the y-bit-0 components of
//     row j0+R (exactly the components the outer rows read);
//   * sigma rows (3-plane ring) and segment-edge values (double-buffered).
// Four warps share a row, each computing a quarter of the parity classes.
// Outside the domain the staged values are zero-filled (boundary rows take the
// masked code path, as in k_seg).
#pragma once

namespace pn {

constexpr int ZM_ROWS = 1;     // rows per CTA
constexpr int ZM_WPR = 8;      // warps per row (one parity class each)
constexpr int ZM_KZ = 16;      // z-planes per CTA chunk

template <int N>
struct ZmLayout {
    static constexpr int U = (N + 1) * (N + 1);
    static constexpr int ROW = 32 * U;                          // doubles per staged row
    static constexpr int OWN = 0;                               // [4][ZM_ROWS][ROW]
    static constexpr int HALO = OWN + 4 * ZM_ROWS * ROW;        // [2][ROW]
    static constexpr int SIG = HALO + 2 * ROW;                  // [3][2 fields][ZM_ROWS+1][34]
    static constexpr int SIGF = (ZM_ROWS + 1) * 34;             // field stride
    static constexpr int SIGP = 2 * SIGF;                       // plane stride
    static constexpr int EDGE = SIG + 3 * SIGP;                 // [2][ZM_ROWS][2][U]
    static constexpr int EDGEP = ZM_ROWS * 2 * U;
    static constexpr int TOTAL = EDGE + 2 * EDGEP;
    static constexpr size_t BYTES = sizeof(double) * (size_t)TOTAL;
};

template <int N>
__device__ __forceinline__ void zm_zero(double *dst, int n, int tid, int nthr) {
    for (int q = tid; q < n; q += nthr) dst[q] = 0.0;
}

// stage the ZM_ROWS own rows of local plane kl into ring slot `slot`
template <int N>
__device__ __forceinline__ void zm_stage_rows(double *sm, const SegGeo &g, const double *X, int seg, int j0, int kl,
                                              int slot, int tid, int nthr) {
    using L = ZmLayout<N>;
    const int kg = g.z0 + kl;
    const long long rowlen = (long long)L::ROW;
    for (int r = 0; r < ZM_ROWS; ++r) {
        double *dst = sm + L::OWN + (slot * ZM_ROWS + r) * L::ROW;
        const int j = j0 + r;
        if (kg < 0 || kg >= g.nz || j >= g.ny) {
            zm_zero<N>(dst, L::ROW, tid, nthr);
            continue;
        }
        const double *src = X + (((long long)kl * g.ny + j) * g.nseg + seg) * rowlen;
        for (int q = tid; q < L::ROW / 2; q += nthr) cp_async16(dst + 2 * q, src + 2 * q);
    }
}

// halo row of local plane kl: y-bit-1 comps from row j0-1, y-bit-0 comps from row j0+R
template <int N>
__device__ __forceinline__ void zm_stage_halo(double *sm, const int *par, const SegGeo &g, const double *X, int seg,
                                              int j0, int kl, int slot, int tid, int nthr) {
    using L = ZmLayout<N>;
    const int kg = g.z0 + kl;
    double *dst = sm + L::HALO + slot * L::ROW;
    const bool zok = kg >= 0 && kg < g.nz;
    const long long rowlen = (long long)L::ROW;
    for (int q = tid; q < L::U * 16; q += nthr) {
        const int c = q >> 4, part = (q & 15) * 2;
        const int j = (par[c] & 2) ? j0 - 1 : j0 + ZM_ROWS;
        if (!zok || j < 0 || j >= g.ny) {
            dst[c * 32 + part] = 0.0;
            dst[c * 32 + part + 1] = 0.0;
        } else {
            const double *src = X + (((long long)kl * g.ny + j) * g.nseg + seg) * rowlen + c * 32 + part;
            cp_async16(dst + c * 32 + part, src);
        }
    }
}

// sigma rows j0 .. j0+R (clamped) of field plane kl (plane nzl exists; kl <= nzl)
template <int N>
__device__ __forceinline__ void zm_stage_sig(double *sm, const SegGeo &g, const double *st, const double *ss, int seg,
                                             int j0, int kl, int slot, int tid, int nthr) {
    using L = ZmLayout<N>;
    double *dst = sm + L::SIG + slot * L::SIGP;
    const bool has_next = seg < g.nseg - 1;
    const int rows = ZM_ROWS + 1;
    for (int q = tid; q < 2 * rows * 16; q += nthr) {
        const int fld = q / (rows * 16), rr = (q / 16) % rows, part = (q & 15) * 2;
        const int jj = min(j0 + rr, g.ny - 1);
        const long long vb = ((long long)kl * g.ny + jj) * g.nx + seg * 32;
        cp_async16(dst + fld * L::SIGF + rr * 34 + part, (fld ? ss : st) + vb + part);
    }
    for (int q = tid; q < 2 * rows; q += nthr) {   // x+1 sample of lane 31 (edge-replicated at nx-1)
        const int fld = q / rows, rr = q % rows;
        const int jj = min(j0 + rr, g.ny - 1);
        const long long vb = ((long long)kl * g.ny + jj) * g.nx + seg * 32 + (has_next ? 32 : 31);
        cp_async8(dst + fld * L::SIGF + rr * 34 + 32, (fld ? ss : st) + vb);
    }
}

// segment-edge values (lane 31 of the previous segment, lane 0 of the next) of plane kl
template <int N>
__device__ __forceinline__ void zm_stage_edge(double *sm, const SegGeo &g, const double *X, int seg, int j0, int kl,
                                              int slot, int tid, int nthr) {
    using L = ZmLayout<N>;
    const int kg = g.z0 + kl;
    double *dst = sm + L::EDGE + slot * L::EDGEP;
    const long long rowlen = (long long)L::ROW;
    const bool has_prev = seg > 0, has_next = seg < g.nseg - 1;
    for (int q = tid; q < ZM_ROWS * 2 * L::U; q += nthr) {
        const int r = q / (2 * L::U), side = (q / L::U) & 1, c = q % L::U;
        const int j = j0 + r;
        const bool ok = kg >= 0 && kg < g.nz && j < g.ny && (side ? has_next : has_prev);
        double *d = dst + (r * 2 + side) * L::U + c;
        if (!ok) {
            *d = 0.0;
        } else {
            const double *row = X + (((long long)kl * g.ny + j) * g.nseg + seg) * rowlen;
            cp_async8(d, side ? row + rowlen + c * 32 : row - rowlen + c * 32 + 31);
        }
    }
}

template <int N, int TRANS, int RED, bool JAC>
__global__ void __launch_bounds__(32 * ZM_ROWS * ZM_WPR, 2) k_zm(
    const __grid_constant__ SegParams prm, SegGeo g, const double *__restrict__ X, double *__restrict__ Y,
    const double *__restrict__ minv, double *__restrict__ zt, const double *__restrict__ st,
    const double *__restrict__ ss, double *__restrict__ partials, long long slot_stride, int rb, const State *state,
    const int *__restrict__ par) {
    using L = ZmLayout<N>;
    constexpr int NT = 32 * ZM_ROWS * ZM_WPR;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rw = warp / ZM_WPR, quarter = warp % ZM_WPR;
    long long bid = blockIdx.x;
    const int seg = (int)(bid % g.nseg);
    bid /= g.nseg;
    const int nyb = (g.ny + ZM_ROWS - 1) / ZM_ROWS;
    const int jb = (int)(bid % nyb);
    const int zc = (int)(bid / nyb);
    const int j0 = jb * ZM_ROWS, j = j0 + rw;
    const int kz0 = g.kl0 + zc * ZM_KZ, kz1 = min(kz0 + ZM_KZ, g.kl0 + g.npl);
    if (state && seg_stopped(state)) return;   // CTA-uniform

    // prologue: planes kz0-1, kz0, kz0+1 (+ halo / sigma / edges of kz0) | plane kz0+2, halo kz0+1, ...
    auto slot4 = [&](int kl) { return ((kl - kz0) % 4 + 4) % 4; };
    auto slot3 = [&](int kl) { return ((kl - kz0) % 3 + 3) % 3; };
    auto slot2 = [&](int kl) { return ((kl - kz0) % 2 + 2) % 2; };
    zm_stage_rows<N>(sm, g, X, seg, j0, kz0 - 1, slot4(kz0 - 1), tid, NT);
    zm_stage_rows<N>(sm, g, X, seg, j0, kz0, slot4(kz0), tid, NT);
    zm_stage_rows<N>(sm, g, X, seg, j0, kz0 + 1, slot4(kz0 + 1), tid, NT);
    zm_stage_halo<N>(sm, par, g, X, seg, j0, kz0, slot2(kz0), tid, NT);
    zm_stage_sig<N>(sm, g, st, ss, seg, j0, kz0, slot3(kz0), tid, NT);
    zm_stage_sig<N>(sm, g, st, ss, seg, j0, kz0 + 1, slot3(kz0 + 1), tid, NT);
    zm_stage_edge<N>(sm, g, X, seg, j0, kz0, slot2(kz0), tid, NT);
    cp_async_commit();
    if (kz0 + 2 <= kz1) zm_stage_rows<N>(sm, g, X, seg, j0, kz0 + 2, slot4(kz0 + 2), tid, NT);
    if (kz0 + 1 < kz1) {
        zm_stage_halo<N>(sm, par, g, X, seg, j0, kz0 + 1, slot2(kz0 + 1), tid, NT);
        zm_stage_edge<N>(sm, g, X, seg, j0, kz0 + 1, slot2(kz0 + 1), tid, NT);
    }
    if (kz0 + 2 <= kz1) zm_stage_sig<N>(sm, g, st, ss, seg, j0, kz0 + 2, slot3(kz0 + 2), tid, NT);
    cp_async_commit();

    const int i = seg * 32 + lane;
    for (int kl = kz0; kl < kz1; ++kl) {
        const int kg = g.z0 + kl;
        cp_async_wait<1>();
        __syncthreads();
        RedAcc ra;
        if (j < g.ny) {
            SegRow r;
            r.lane = lane;
            const double *own = sm + L::OWN + (slot4(kl) * ZM_ROWS) * L::ROW;
            r.xs = own + rw * L::ROW + lane;
            const double *halo = sm + L::HALO + slot2(kl) * L::ROW + lane;
            r.ys_m = rw == 0 ? halo : own + (rw - 1) * L::ROW + lane;
            r.ys_p = rw == ZM_ROWS - 1 ? halo : own + (rw + 1) * L::ROW + lane;
            r.zs_m = sm + L::OWN + (slot4(kl - 1) * ZM_ROWS + rw) * L::ROW + lane;
            r.zs_p = sm + L::OWN + (slot4(kl + 1) * ZM_ROWS + rw) * L::ROW + lane;
            r.sig0 = sm + L::SIG + slot3(kl) * L::SIGP + rw * 34 + lane;
            r.sig1 = sm + L::SIG + slot3(kl + 1) * L::SIGP + rw * 34 + lane;
            r.sgf = L::SIGF;
            const double *edge = sm + L::EDGE + slot2(kl) * L::EDGEP + rw * 2 * L::U;
            r.eprev = edge;
            r.enext = edge + L::U;
            const long long rowbase = (((long long)kl * g.ny + j) * g.nseg + seg) * (long long)L::ROW;
            r.Y = Y + rowbase + lane;
            r.minv = minv ? minv + rowbase + lane : nullptr;
            r.zt = zt ? zt + rowbase + lane : nullptr;
            r.diag = nullptr;
            r.bx = i == g.nx - 1;
            r.bx_p = i + 1 == g.nx - 1;
            r.by = j == g.ny - 1;
            r.bz = kg == g.nz - 1;
            r.by_p = j + 1 == g.ny - 1;
            r.bz_p = kg + 1 == g.nz - 1;
            const bool interior = seg != g.nseg - 1 && j >= 1 && j <= g.ny - 3 && kg >= 1 && kg <= g.nz - 3;
#define PN_ZM_Q(Q)                                                                          \
    if (quarter == Q) {                                                                     \
        if (interior) seg_group<N, TRANS, ZM_WPR, Q, RED, JAC, false, false, 1>(r, prm, ra); \
        else seg_group<N, TRANS, ZM_WPR, Q, RED, JAC, false, true, 1>(r, prm, ra);          \
    }
            PN_ZM_Q(0) PN_ZM_Q(1) PN_ZM_Q(2) PN_ZM_Q(3) PN_ZM_Q(4) PN_ZM_Q(5) PN_ZM_Q(6) PN_ZM_Q(7)
#undef PN_ZM_Q
        }
        if (RED) {
            constexpr int W = ZM_ROWS * ZM_WPR;
            double v0 = ra.s0, v1 = ra.s1, v2 = (RED == 2 && !JAC) ? ra.s1 : ra.s2;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 += __shfl_down_sync(0xffffffffu, v0, o);
                v1 += __shfl_down_sync(0xffffffffu, v1, o);
                v2 += __shfl_down_sync(0xffffffffu, v2, o);
            }
            if (lane == 0) {
                const long long idx = (long long)kg * rb + ((long long)seg * nyb + jb) * W + warp;
                if (RED == 1) partials[idx] = v0;
                if (RED == 2) { partials[1 * slot_stride + idx] = v1; partials[2 * slot_stride + idx] = v2; }
            }
        }
        __syncthreads();   // slots of plane kl-1, halo / sigma / edges of kl are free
        if (kl + 3 <= kz1) zm_stage_rows<N>(sm, g, X, seg, j0, kl + 3, slot4(kl + 3), tid, NT);
        if (kl + 2 < kz1) {
            zm_stage_halo<N>(sm, par, g, X, seg, j0, kl + 2, slot2(kl + 2), tid, NT);
            zm_stage_edge<N>(sm, g, X, seg, j0, kl + 2, slot2(kl + 2), tid, NT);
        }
        if (kl + 3 <= kz1) zm_stage_sig<N>(sm, g, st, ss, seg, j0, kl + 3, slot3(kl + 3), tid, NT);
        cp_async_commit();
    }
    cp_async_wait<0>();
}

template <int N>
int zm_launch(const SegParams &prm, const SegGeo &g, int trans, int red, bool jac, const double *x, double *y,
              const double *minv, double *zt, const double *st, const double *ss, double *partials,
              long long slot_stride, int rb, const State *state, const int *par, cudaStream_t s) {
    using L = ZmLayout<N>;
    const int nyb = (g.ny + ZM_ROWS - 1) / ZM_ROWS;
    const long long chunks = (g.npl + ZM_KZ - 1) / ZM_KZ;
    if (g.kst != 1) { set_error("z-march launch: strided plane sets unsupported"); return PN_ERR_INVALID; }
    dim3 grid((unsigned)((long long)g.nseg * nyb * chunks)), block(32 * ZM_ROWS * ZM_WPR);
#define PN_ZM_GO(T, R, J)                                                                                       \
    do {                                                                                                        \
        static bool cfg_done = false;                                                                           \
        if (!cfg_done) {                                                                                        \
            cudaFuncSetAttribute(k_zm<N, T, R, J>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::BYTES); \
            cfg_done = true;                                                                                    \
        }                                                                                                       \
        k_zm<N, T, R, J><<<grid, block, L::BYTES, s>>>(prm, g, x, y, minv, zt, st, ss, partials, slot_stride, rb, \
                                                       state, par);                                            \
    } while (0)
    if (!trans) {
        if (red == 1) PN_ZM_GO(0, 1, false);
        else PN_ZM_GO(0, 0, false);
    } else {
        if (red == 2) {
            if (jac) PN_ZM_GO(1, 2, true);
            else PN_ZM_GO(1, 2, false);
        } else {
            PN_ZM_GO(1, 0, false);
        }
    }
#undef PN_ZM_GO
    PN_CUDA(cudaGetLastError());
    return PN_OK;
}

}  // namespace pn
