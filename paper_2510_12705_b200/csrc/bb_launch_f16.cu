// bb_launch_f16.cu -- kernels and launch sequence for __half storage.
#include "bb_launch.cuh"

namespace bbhost {
template bb_status launch_all<__half>(const Plan &, const void *, int64_t, int64_t, int64_t, void *, int64_t, void *,
                                   int64_t, void *, cudaStream_t);
} // namespace bbhost
