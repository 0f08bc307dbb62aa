// bb_launch_f64.cu -- kernels and launch sequence for double storage.
#include "bb_launch.cuh"

namespace bbhost {
template bb_status launch_all<double>(const Plan &, const void *, int64_t, int64_t, int64_t, void *, int64_t, void *,
                                   int64_t, void *, cudaStream_t);
} // namespace bbhost
