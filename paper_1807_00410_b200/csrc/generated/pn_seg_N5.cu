// GENERATED translation unit: segmented fast operator kernels for P5.
#include "../pn_seg_common.cuh"
namespace pn {
template int seg_launch<5>(const SegParams &, const SegGeo &, int, int, bool, const double *, double *,
                            const double *, double *, const double *, const double *, double *, long long, int,
                            const State *, cudaStream_t);
template int seg_launch_fused_r<5>(const SegParams &, const SegGeo &, const FuseSched &, bool, double *, const double *,
                                    double *, const double *, double *, const double *, const double *, double *,
                                    long long, int, const State *, cudaStream_t);
}
