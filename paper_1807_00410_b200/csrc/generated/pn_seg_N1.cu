// GENERATED translation unit: segmented fast operator kernels for P1.
#include "../pn_seg_common.cuh"
namespace pn {
template int seg_launch<1>(const SegParams &, const SegGeo &, int, int, bool, const double *, double *,
                            const double *, double *, const double *, const double *, double *, long long, int,
                            const State *, cudaStream_t);
}
