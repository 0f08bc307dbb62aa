// bb_plan.h -- host-side plan of one call (shared by the C ABI translation
// unit and the per-dtype launch translation units).  Host logic only.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

#include "bandbidiag.h"

namespace bbhost {

constexpr size_t kAlign = 256;
constexpr int kSmemOptinFallback = 227 * 1024;

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline int round_odd(int x) { return (x & 1) ? x : x + 1; }

inline size_t elem_size(bb_dtype dt)
{
    switch (dt) {
    case BB_F16: return 2;
    case BB_F32: return 4;
    case BB_F64: return 8;
    }
    return 0;
}
inline size_t compute_size(bb_dtype dt) { return dt == BB_F64 ? 8 : 4; }

struct PassPlan {
    int c, t, s;
    int nsweeps;     // non-empty sweeps: r in [0, nsweeps)
    int cycles;      // max_r (s*r + J_r)
    int LT, LW;
    size_t smem;     // dynamic shared memory bytes
    int threads;
    // register kernel (bb_pass_v2.cuh)
    bool v2 = false;
    int mt = 0, ntc = 0, a0 = 0, b0 = 0, LW2 = 0;
    size_t smem2 = 0;
    // multi-sweep kernel (bb_pass_v4.cuh)
    int g4 = 0, nt4 = 0, LDT4 = 0, LDW4 = 0, NS4 = 0, slot4 = 0, ntmax4 = 0, tp4 = 0, pw4 = 0;
    int a4 = 0, b4 = 0; // v4 half-step wait offsets (refined for target bandwidth < 4, tools/depcheck.py)
    size_t smem4 = 0;
    // unit kernel (bb_pass_v5.cuh): G sweeps per CTA advanced one step at a time
    int g5 = 0, nt5 = 0, LA5 = 0, LB5 = 0, a5 = 0, b5 = 0, b5t = 0, ngroups5 = 0;
    size_t smem5 = 0;
    // segment-ring kernel (bb_pass_v6.cuh): target bandwidth 1, G sweeps per CTA
    int g6 = 0, r6 = 0, nt6 = 0, ngroups6 = 0;
    size_t smem6 = 0;
    // progress flags of this pass: offset (ints) into the flag region, stride
    // (ints) between consecutive flags -- one L2 line per group flag for the
    // unit / segment-ring kernels (neighbouring groups' flags sharing a line
    // are written and polled concurrently), 1 for the per-sweep kernels
    int64_t flag_off = 0;
    int fstride = 1;
};

struct Plan {
    int64_t n = 0, b_eff = 0, batch = 0;
    int tw = 0;
    int64_t ldw = 0, ku = 0, mat_stride = 0;
    bb_config cfg{};
    std::vector<PassPlan> passes;
    size_t band_bytes = 0, flag_bytes = 0, counter_bytes = 0, total = 0;
};

struct DeviceInfo {
    int sms = 0;
    int smem_optin = 0;
    bool ok = false;
};

inline int64_t sweep_len_h(int64_t n, int64_t c, int64_t t, int64_t r)
{
    int64_t first = r + c - t;
    return first > n - 2 ? 0 : (n - 2 - first) / c + 1;
}

bool device_info(DeviceInfo &out);
bb_status make_plan(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg_in, Plan &P);

// one call's device work (pack -> passes -> extract) for storage type S;
// explicitly instantiated in bb_launch_f16.cu / bb_launch_f32.cu / bb_launch_f64.cu
template <class S>
bb_status launch_all(const Plan &P, const void *band, int64_t ldband, int64_t stride_band, int64_t b_in,
                     void *d_out, int64_t stride_d, void *e_out, int64_t stride_e, void *ws, cudaStream_t st);

} // namespace bbhost
