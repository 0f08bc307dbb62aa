// bb_launch_f32.cu -- kernels and launch sequence for float storage.
#include "bb_launch.cuh"

namespace bbhost {
template bb_status launch_all<float>(const Plan &, const void *, int64_t, int64_t, int64_t, void *, int64_t, void *,
                                   int64_t, void *, cudaStream_t);
} // namespace bbhost
