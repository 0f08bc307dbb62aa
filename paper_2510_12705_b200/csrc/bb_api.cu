// bb_api.cu -- C ABI (include/bandbidiag.h) of the B200 band -> bidiagonal
// reduction: argument validation, pass plan (Alg. 1 line 1), workspace
// carving, and the launch sequence pack -> one launch per pass -> extract.
//
// Host logic only; every arithmetic step of the method runs in the kernels of
// bb_kernels.cuh.  No CPU fallback exists: without a usable CUDA device every
// compute entry point returns BB_ERR_CUDA.
#include "bb_plan.h"
#include "bb_pass_v4.cuh" // constants of the multi-sweep kernel's plan (no kernel is instantiated here)
#include "bandbidiag.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace bbhost {

int default_tw(bb_dtype dt)
{
    // P:315 found one 128-byte cache line optimal on its GPUs: 32 (FP32), 16
    // (FP64).  On B200 with the v4 kernel tw = 32 is faster for FP64 too
    // (n = 32768, b = 128: 2.2 s vs 2.6 s): the number of
    // passes -- each a chain of ~n sweep hand-offs -- halves.
    (void)dt;
    return 32;
}


bb_status make_plan(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg_in, Plan &P)
{
    if (elem_size(dtype) == 0) return BB_ERR_NOT_SUPPORTED;
    if (n < 0 || b < 0 || batch < 0) return BB_ERR_INVALID_VALUE;
    bb_config cfg{};
    if (cfg_in) cfg = *cfg_in;
    if (cfg.tw < 0 || cfg.threads_per_block < 0 || cfg.max_blocks_per_sm < 0 || cfg.dep_distance < 0 ||
        cfg.schedule < 0 || cfg.schedule > BB_SCHED_CYCLE)
        return BB_ERR_INVALID_VALUE;
    if (cfg.threads_per_block && (cfg.threads_per_block % 32 || cfg.threads_per_block > 512))
        return BB_ERR_INVALID_VALUE;
    if (cfg.num_timing_events < 0) return BB_ERR_INVALID_VALUE;
    if (cfg.schedule == BB_SCHED_AUTO) cfg.schedule = BB_SCHED_FLAGS;
    if (cfg.tw == 0 && elem_size(dtype) == 8) {
        // default tilewidth 32, unless a pass window would not fit one SM's shared
        // memory even for the generic kernel (very wide fp64 bands, b >~ 400):
        // then the paper's fp64 value 16
        bb_config c32 = cfg;
        c32.tw = 32;
        Plan probe;
        if (make_plan(n, b, dtype, batch, &c32, probe) == BB_ERR_NOT_SUPPORTED) cfg.tw = 16;
    }
    P.n = n;
    P.batch = batch;
    P.b_eff = n > 0 ? std::min<int64_t>(b, n - 1) : 0;
    int tw = cfg.tw ? cfg.tw : default_tw(dtype);
    // the headroom only needs the largest tilewidth any pass uses
    tw = (int)std::max<int64_t>(1, std::min<int64_t>(tw, std::max<int64_t>(P.b_eff - 1, 1)));
    cfg.tw = tw;
    P.tw = tw;
    {
        // band + twice the tilewidth (reading Q11): the diagonal at storage
        // row ku >= b_eff + tw, tw rows below it.  TMA column boxes (bb_pass_v6.cuh)
        // need 16-byte aligned box starts and column strides: ku + 1 and ldw are
        // rounded up to multiples of 16 / elem (the box of the last pass, c in
        // {16, 32}, starts at row ku - (2c - 1)); a few extra zero rows at most
        const int64_t q = 16 / (int64_t)elem_size(dtype);
        P.ku = P.b_eff + tw;
        while ((P.ku + 1) % q) ++P.ku;
        P.ldw = P.ku + tw + 1;
        while (P.ldw % q) ++P.ldw;
        P.mat_stride = n * P.ldw;
    }
    P.passes.clear();
    if (n > 2 && P.b_eff > 1) {
        int64_t c = P.b_eff;
        while (c > 1) {
            int64_t t = std::min<int64_t>(tw, c - 1);
            PassPlan pp{};
            pp.c = (int)c;
            pp.t = (int)t;
            int s_auto = (c - t == 1) ? 3 : 2; // reading Q4
            pp.s = std::max(s_auto, (int)cfg.dep_distance);
            int64_t ns = std::max<int64_t>(0, (n - 2) - (c - t) + 1);
            pp.nsweeps = (int)ns;
            int64_t cyc = 0;
            for (int64_t r = 0; r < ns; ++r) cyc = std::max(cyc, pp.s * r + sweep_len_h(n, c, t, r));
            pp.cycles = (int)cyc;
            pp.LT = round_odd((int)(c + t + 1));
            pp.LW = round_odd((int)(t + 1));
            size_t cs = compute_size(dtype);
            pp.smem = ((size_t)pp.LT * (t + 1) + (size_t)pp.LW * c + (t + 1) + 8) * cs;
            if (pp.smem > (size_t)kSmemOptinFallback) return BB_ERR_NOT_SUPPORTED;
            int thr = cfg.threads_per_block;
            if (!thr) thr = (int)std::min<int64_t>(256, std::max<int64_t>(64, (c + t + 31) / 32 * 32));
            pp.threads = thr;
            // register kernel: reflector length t+1 <= 33, c + t + 1 + 64 <= 1024 threads
            const int tb = (int)(c - t);
            pp.a0 = tb >= 4 ? 2 : (tb >= 2 ? 4 : 6);
            pp.b0 = tb >= 4 ? 3 : pp.a0;
            if (pp.s > (tb == 1 ? 3 : 2)) pp.a0 = pp.b0 = 2 * pp.s; // user asked for a larger distance
            pp.mt = t + 1 <= 9 ? 9 : (t + 1 <= 17 ? 17 : (t + 1 <= 33 ? 33 : 0));
            pp.ntc = (int)((c + t + 1 + 31) / 32 * 32);
            pp.LW2 = round_odd(pp.mt);
            pp.smem2 = cs * (size_t)(2 * pp.mt + 4 + (size_t)pp.LW2 * (c + t + 1)) + 16;
            pp.v2 = pp.mt > 0 && pp.ntc + 64 <= 512 && !(cfg.flags & BB_FLAG_GENERIC_KERNEL) &&
                    pp.smem2 <= (size_t)kSmemOptinFallback;
            // multi-sweep CTA (bb_pass_v4.cuh): G warp-groups of nt4 threads + producer and
            // release warps; needs reflector length t + 1 in {16, 17, 32, 33} (compiled), and
            // c - t >= max(4, 2G) for G > 1 (bb_pass_v4.cuh header)
            {
                const int MT4 = (int)t + 1;
                const bool mt_ok = MT4 == 16 || MT4 == 17 || MT4 == 32 || MT4 == 33;
                pp.nt4 = (int)((c + t + 31) / 32 * 32);
                // instantiated thread bounds: 576 (96 registers); fp64 with t >= 31
                // needs more registers per thread: 384 (168 registers) or 512 (128)
                // (the 512 variant spills; measured no faster than G = 1, so fp64 t >= 31
                // stays within 384 threads)
                const int ntlim = (cs == 8 && MT4 > 17) ? 384 : 576;
                int gmax = 4; // measured: G <= 4 is as fast as larger G (tools/gsweep.py)
                if (const char *e = getenv("BB_V4_G")) gmax = std::max(0, std::min(gmax, atoi(e)));
                if (cfg.flags & BB_FLAG_GENERIC_KERNEL) gmax = 0;
                int G = mt_ok ? gmax : 0;
                for (; G > 0; --G) {
                    if (G > 1 && (c - t < 4 || c - t < 2 * G)) continue;
                    const int nthr = G * pp.nt4 + 32 * (bb::V4_PW + 1);
                    if (nthr > ntlim) continue;
                    pp.ntmax4 = (cs == 8 && MT4 > 17) ? (nthr <= 384 ? 384 : 512) : 576;
                    // slot = T (c + G rows, row-major) + W (c columns), both with a
                    // compile-time odd pitch TP >= t + G (bb_pass_v4.cuh): (MT | 1) + 8, or
                    // (MT | 1) + 2 for fp64 t >= 31 (smaller slots: G = 2 fits 227 KB)
                    const bool tight = cs == 8 && MT4 >= 32 && (int)t + G <= (MT4 | 1) + 2;
                    if (cs == 8 && MT4 >= 32 && !tight) continue;
                    const int TP = (MT4 | 1) + (tight ? 2 : 8);
                    pp.tp4 = TP;
                    pp.LDT4 = (int)c + G;
                    pp.LDW4 = TP;
                    pp.slot4 = (pp.LDT4 + (int)c) * TP;
                    pp.slot4 += pp.slot4 & 1;
                    // dynamic budget leaves room for the kernel's static shared memory
                    // (progress counters + mbarrier rings, ~2.4 KB)
                    const size_t budget = (size_t)kSmemOptinFallback - 4096;
                    for (pp.NS4 = G + 2; pp.NS4 >= G + 1; --pp.NS4) {
                        pp.smem4 = cs * (size_t)pp.slot4 * pp.NS4;
                        if (pp.smem4 <= budget) break;
                    }
                    if (pp.smem4 <= budget && pp.NS4 + 4 <= bb::V4_RING) break;
                }
                pp.g4 = G;
                // producer warps: 2, or -- when shared memory already limits the SM to
                // one CTA -- as many as the thread bound leaves, up to 6 (fills are on
                // the cross-CTA critical path)
                pp.pw4 = bb::V4_PW;
                if (G > 0 && pp.smem4 > (size_t)kSmemOptinFallback / 2) {
                    const int left = pp.ntmax4 - G * pp.nt4 - 32;
                    pp.pw4 = std::max(bb::V4_PW, std::min(6, left / 32));
                }
                // half-step rule of the v4 kernel (every pair of conflicting phases
                // ordered, tools/depcheck.py): target bandwidth >= 4: A(j) waits for
                // progress[r-1] >= 2j+2, B(j) for >= 2j+3; 2..3: 2j+2 / 2j+4 (whole
                // step s = 2 would be 2j+4 / 2j+4); 1: 2j+4 / 2j+5 (s = 3: 2j+6 / 2j+6)
                pp.a4 = tb >= 2 ? 2 : 4;
                pp.b4 = tb >= 4 ? 3 : (tb >= 2 ? 4 : 5);
                if (pp.s > (tb == 1 ? 3 : 2)) pp.a4 = pp.b4 = 2 * pp.s; // user asked for a larger distance
            }
            // unit kernel (bb_pass_v5.cuh): reflector length t + 1 in {17, 33}, G a
            // multiple of 8 with G <= c - t (only exactly commuting reflector pairs are
            // reordered), one unit window + reflector panels in shared memory
            {
                const int MT5 = (int)t + 1;
                const bool ok5 = (MT5 == 17 || MT5 == 33) && !(cfg.flags & (BB_FLAG_GENERIC_KERNEL | BB_FLAG_NO_UNIT_KERNEL)) &&
                                 pp.s == (tb == 1 ? 3 : 2);
                int gcap = 32;
                if (const char *e = getenv("BB_V5_G")) gcap = std::max(0, std::min(32, atoi(e)));
                // compiled group sizes 32, 16, 8: the largest with 2G <= c - t (the
                // cheaper wait rule), else the largest with G <= c - t; halved until
                // the unit window fits shared memory
                int G = 0;
                const int VP = (MT5 + 2) & ~1;
                const bool wide = getenv("BB_V5_WIDE") != nullptr; // experiments: largest G <= c - t
                if (ok5) {
                    for (int Gc : {32, 16, 8})
                        if (!wide && Gc <= gcap && 2 * Gc <= c - t) {
                            G = Gc;
                            break;
                        }
                    if (!G)
                        for (int Gc : {32, 16, 8})
                            if (Gc <= gcap && Gc <= c - t) {
                                G = Gc;
                                break;
                            }
                }
                for (; G >= 8; G /= 2) {
                    const int W = (int)t + G;
                    const int LA = round_odd((int)c + W), LB = round_odd(W);
                    const size_t sm = compute_size(dtype) * ((size_t)W * LA + (size_t)c * LB + 2 * (size_t)G * VP + 2 * (MT5 + 1)) + 16;
                    if (sm <= (size_t)kSmemOptinFallback - 1024) {
                        pp.g5 = G;
                        pp.LA5 = LA;
                        pp.LB5 = LB;
                        pp.smem5 = sm;
                        break;
                    }
                }
                if (pp.g5 > 0) {
                    // inter-group rule of the unit kernel: exact hazard search over its
                    // load / write-back rectangles (tools/v5_rules.py,
                    // tests/test_unit_schedule.py): A half waits for progress[k-1] >=
                    // 2j + a5, B half for >= 2j + b5 -- (2, 3) when 3G <= c - t, with
                    // 2j + 4 while the predecessor's unit j+1 is its last one (that unit
                    // writes back its whole H region); (2, 4) when 2G <= c - t; else (4, 5)
                    const int G5 = pp.g5;
                    if (3 * G5 <= c - t) {
                        pp.a5 = 2;
                        pp.b5 = 3;
                        pp.b5t = 4;
                    } else if (2 * G5 <= c - t) {
                        pp.a5 = 2;
                        pp.b5 = pp.b5t = 4;
                    } else {
                        pp.a5 = 4;
                        pp.b5 = pp.b5t = 5;
                    }
                    pp.nt5 = (int)std::min<int64_t>(256, std::max<int64_t>(64, (c + t + 31) / 32 * 32));
                    pp.ngroups5 = (int)((ns + pp.g5 - 1) / pp.g5);
                }
            }
            // segment-ring kernel (bb_pass_v6.cuh) for target bandwidth 1: reflector
            // length t + 1 = c in {16, 32}; G sweeps per CTA (one WG of 2c threads
            // each); a ring of R column chunks (c columns x 3c rows, the TMA box)
            if (tb == 1 && (c == 16 || c == 32) && pp.g5 == 0 && pp.s == 3 && P.ku + c + 1 <= P.ldw &&
                !(cfg.flags & (BB_FLAG_GENERIC_KERNEL | BB_FLAG_NO_SEGMENT_KERNEL))) {
                const int cc = (int)c;
                const int nt = 2 * cc;
                const int ntmax = cs == 8 ? (cc == 32 ? 384 : 448) : (cc == 32 ? 512 : 576); // bb_launch.cuh instantiations
                // default cap 4: measured best for fp64 (the ring allows at most 4) and
                // fp32 (n = 32768: 428 -> 395 ms, 16384: 183 -> 170, 8192: 74 -> 70,
                // 1024: 6.8 -> 6.5 ms against the thread-bound G = 7,
                // profiles/r02/v6_group_size_f32.txt); BB_V6_G overrides (up to 16)
                int gcap = 4;
                if (const char *e = getenv("BB_V6_G")) gcap = std::max(0, std::min(16, atoi(e)));
                const size_t chunk = cs * (size_t)cc * (size_t)(3 * cc); // TMA box: 3c rows x c columns
                // ring budget: the 196 KB shared-memory carve-out (static: barriers, counters,
                // x staging ~10 KB) -- the kernel is measurably faster with >= 60 KB of L1 left
                // than at the 228 KB carve-out (fp64, c = 32: G = 3 / R = 7 at 181 KB: 297 ms,
                // G = 3 / R = 8 at 206 KB: 312 ms, G = 4 / R = 9 at 230 KB: 309 ms;
                // profiles/r02/v6_group_ring_sweep.txt); falls back to the full opt-in size
                const size_t budget_l1 = (size_t)196 * 1024 - 10240;
                const size_t budget_max = (size_t)kSmemOptinFallback - 10240;
                const bool env_g = getenv("BB_V6_G") != nullptr; // experiments / tests ask for a group size
                for (size_t budget : {env_g ? budget_max : budget_l1, budget_max}) {
                if (pp.g6 > 0) break;
                for (int G = std::min(std::min(gcap, 14), cc); G >= 1; --G) { // named barriers 1 + g <= 15; G <= c
                    // (the writer's finality rule, tests/test_v6_protocol.py)
                    if (G * nt + 64 > ntmax) continue;
                    // WG g trails WG g-1 by ~2 steps in steady state; the ring holds
                    // the chunks from the last WG's position to WG 0's B window,
                    // as many as shared memory allows (slack absorbs jitter)
                    const int rmin = 3 + 2 * (G - 1);
                    int R = (int)std::min<size_t>(std::min<size_t>(budget / chunk, (size_t)rmin + 4), 48); // < V6_FRING;
                    // slack 4: larger rings measured slower for fp32 (smaller L1 carve-out)
                    if (const char *e = getenv("BB_V6_R")) R = std::max(rmin, std::min(R, atoi(e))); // experiments
                    if (R < rmin) continue;
                    pp.g6 = G;
                    pp.r6 = R;
                    pp.nt6 = G * nt + 64;
                    pp.smem6 = (size_t)R * chunk + 128; // + alignment of the ring to 128 bytes
                    pp.ngroups6 = (int)((ns + G - 1) / G);
                    break;
                }
                }
            }
            P.passes.push_back(pp);
            c -= t;
        }
    }
    if (cfg.timing_events && cfg.num_timing_events < (int)P.passes.size() + 3) return BB_ERR_INVALID_VALUE;
    P.cfg = cfg;
    size_t es = elem_size(dtype);
    P.band_bytes = align_up((size_t)batch * (size_t)P.mat_stride * es);
    {
        // flags: per pass batch x (groups or sweeps) x stride ints; group flags one
        // per 128-byte line unless that would exceed 1/8 of the band storage
        int stride = 32;
        for (;; stride /= 2) {
            int64_t off = 0;
            for (PassPlan &pp : P.passes) {
                const bool grp = pp.g5 > 0 || pp.g6 > 0;
                const int64_t nf = grp ? (pp.g5 > 0 ? pp.ngroups5 : pp.ngroups6) : n;
                pp.fstride = grp ? stride : 1;
                pp.flag_off = off;
                off += (int64_t)batch * std::max<int64_t>(nf, 1) * pp.fstride;
            }
            P.flag_bytes = align_up((size_t)off * sizeof(int));
            if (stride == 1 || P.flag_bytes * 8 <= (size_t)batch * (size_t)P.mat_stride * elem_size(dtype)) break;
        }
    }
    P.counter_bytes = align_up(std::max<size_t>(1, P.passes.size()) * sizeof(int));
    P.total = P.band_bytes + P.flag_bytes + P.counter_bytes;
    return BB_SUCCESS;
}


bool device_info(DeviceInfo &out)
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    static std::mutex mu;
    static std::vector<DeviceInfo> cache;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)cache.size() <= dev) cache.resize(dev + 1);
    if (!cache[dev].ok) {
        DeviceInfo di;
        if (cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&di.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        di.ok = true;
        cache[dev] = di;
    }
    out = cache[dev];
    return true;
}

bb_status validate(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band, int64_t ldband,
                   int64_t stride_band, const void *d_out, int64_t stride_d, const void *e_out, int64_t stride_e)
{
    if (elem_size(dtype) == 0) return BB_ERR_NOT_SUPPORTED;
    if (n < 0 || b < 0 || batch < 0) return BB_ERR_INVALID_VALUE;
    if (ldband < b + 1) return BB_ERR_INVALID_VALUE;
    if (n == 0 || batch == 0) return BB_SUCCESS;
    if (!band || !d_out || (n > 1 && !e_out)) return BB_ERR_INVALID_VALUE;
    if (batch > 1) {
        if (stride_band < n * ldband || stride_d < n || stride_e < n - 1) return BB_ERR_INVALID_VALUE;
    }
    if (n > INT32_MAX / 4 || ldband > INT32_MAX || b > INT32_MAX / 4) return BB_ERR_NOT_SUPPORTED;
    return BB_SUCCESS;
}

bb_status run_ex(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band, int64_t ldband,
                 int64_t stride_band, void *d_out, int64_t stride_d, void *e_out, int64_t stride_e,
                 const bb_config *cfg, void *ws, size_t ws_bytes, cudaStream_t st)
{
    bb_status v = validate(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e);
    if (v != BB_SUCCESS) return v;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    if (n == 0 || batch == 0) return BB_SUCCESS;
    if (!ws || ws_bytes < P.total) return BB_ERR_INVALID_VALUE;
    switch (dtype) {
    case BB_F16: return launch_all<__half>(P, band, ldband, stride_band, b, d_out, stride_d, e_out, stride_e, ws, st);
    case BB_F32: return launch_all<float>(P, band, ldband, stride_band, b, d_out, stride_d, e_out, stride_e, ws, st);
    case BB_F64: return launch_all<double>(P, band, ldband, stride_band, b, d_out, stride_d, e_out, stride_e, ws, st);
    }
    return BB_ERR_NOT_SUPPORTED;
}

bb_status run_alloc(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band, int64_t ldband,
                    int64_t stride_band, void *d_out, int64_t stride_d, void *e_out, int64_t stride_e,
                    const bb_config *cfg, cudaStream_t st)
{
    bb_status v = validate(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e);
    if (v != BB_SUCCESS) return v;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    if (n == 0 || batch == 0) return BB_SUCCESS;
    void *ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, P.total, st);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return BB_ERR_OUT_OF_MEMORY;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return BB_ERR_CUDA;
    }
    s = run_ex(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e, cfg, ws, P.total, st);
    if (cudaFreeAsync(ws, st) != cudaSuccess && s == BB_SUCCESS) s = BB_ERR_CUDA;
    return s;
}

} // namespace bbhost

using namespace bbhost;
extern "C" {

bb_status bb_band_to_bidiag(int64_t n, int64_t b, bb_dtype dtype, const void *band, int64_t ldband, void *d_out,
                            void *e_out, void *stream)
{
    return run_alloc(n, b, dtype, 1, band, ldband, n * ldband, d_out, n, e_out, n - 1, nullptr,
                     reinterpret_cast<cudaStream_t>(stream));
}

bb_status bb_band_to_bidiag_batched(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band,
                                    int64_t ldband, int64_t stride_band, void *d_out, int64_t stride_d, void *e_out,
                                    int64_t stride_e, void *stream)
{
    return run_alloc(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e, nullptr,
                     reinterpret_cast<cudaStream_t>(stream));
}

bb_status bb_band_to_bidiag_ex(int64_t n, int64_t b, bb_dtype dtype, const void *band, int64_t ldband, void *d_out,
                               void *e_out, const bb_config *cfg, void *workspace, size_t workspace_bytes,
                               void *stream)
{
    return run_ex(n, b, dtype, 1, band, ldband, n * ldband, d_out, n, e_out, n - 1, cfg, workspace, workspace_bytes,
                  reinterpret_cast<cudaStream_t>(stream));
}

bb_status bb_band_to_bidiag_batched_ex(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band,
                                       int64_t ldband, int64_t stride_band, void *d_out, int64_t stride_d,
                                       void *e_out, int64_t stride_e, const bb_config *cfg, void *workspace,
                                       size_t workspace_bytes, void *stream)
{
    return run_ex(n, b, dtype, batch, band, ldband, stride_band, d_out, stride_d, e_out, stride_e, cfg, workspace,
                  workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

bb_status bb_band_to_bidiag_host(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const void *band_host,
                                 int64_t ldband, int64_t stride_band, void *d_host, int64_t stride_d, void *e_host,
                                 int64_t stride_e, const bb_config *cfg, void *stream)
{
    if (batch == 1) {
        stride_band = n * ldband;
        stride_d = n;
        stride_e = n - 1;
    }
    bb_status v = validate(n, b, dtype, batch, band_host, ldband, stride_band, d_host, stride_d, e_host, stride_e);
    if (v != BB_SUCCESS) return v;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    if (n == 0 || batch == 0) return BB_SUCCESS;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t es = elem_size(dtype);
    const size_t band_b = align_up((size_t)batch * stride_band * es);
    const size_t d_b = align_up((size_t)batch * stride_d * es);
    const size_t e_b = align_up((size_t)batch * std::max<int64_t>(stride_e, 1) * es);
    const size_t total = band_b + d_b + e_b + P.total;
    // per-device staging buffer, kept between calls (grown on demand) so the
    // host path does not pay an allocation per call; calls serialise on it
    static std::mutex mu;
    static std::vector<std::pair<void *, size_t>> cache;
    std::lock_guard<std::mutex> lk(mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return BB_ERR_CUDA;
    }
    if ((int)cache.size() <= dev) cache.resize(dev + 1, {nullptr, 0});
    if (cache[dev].second < total) {
        if (cache[dev].first) {
            if (cudaStreamSynchronize(st) != cudaSuccess) return BB_ERR_CUDA;
            cudaFree(cache[dev].first);
            cache[dev] = {nullptr, 0};
        }
        void *p = nullptr;
        cudaError_t e = cudaMalloc(&p, total);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return e == cudaErrorMemoryAllocation ? BB_ERR_OUT_OF_MEMORY : BB_ERR_CUDA;
        }
        cache[dev] = {p, total};
    }
    unsigned char *buf = reinterpret_cast<unsigned char *>(cache[dev].first);
    void *dband = buf, *dd = buf + band_b, *de = buf + band_b + d_b, *ws = buf + band_b + d_b + e_b;
    const size_t in_bytes = (size_t)((batch - 1) * stride_band + n * ldband) * es;
    if (cudaMemcpyAsync(dband, band_host, in_bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) s = BB_ERR_CUDA;
    if (s == BB_SUCCESS)
        s = run_ex(n, b, dtype, batch, dband, ldband, stride_band, dd, stride_d, de, stride_e, cfg, ws, P.total, st);
    if (s == BB_SUCCESS) {
        const size_t dn = (size_t)((batch - 1) * stride_d + n) * es;
        if (cudaMemcpyAsync(d_host, dd, dn, cudaMemcpyDeviceToHost, st) != cudaSuccess) s = BB_ERR_CUDA;
        if (n > 1) {
            const size_t en = (size_t)((batch - 1) * stride_e + (n - 1)) * es;
            if (cudaMemcpyAsync(e_host, de, en, cudaMemcpyDeviceToHost, st) != cudaSuccess) s = BB_ERR_CUDA;
        }
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && s == BB_SUCCESS) s = BB_ERR_CUDA;
    return s;
}

bb_status bb_workspace_size(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg, size_t *bytes)
{
    if (!bytes) return BB_ERR_INVALID_VALUE;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    *bytes = P.total;
    return BB_SUCCESS;
}

bb_status bb_plan(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg, bb_plan_stats *out)
{
    if (!out) return BB_ERR_INVALID_VALUE;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    std::memset(out, 0, sizeof(*out));
    out->passes = (int64_t)P.passes.size();
    out->tw = P.tw;
    out->ldw = P.ldw;
    out->ku = P.ku;
    out->mat_stride = P.mat_stride;
    out->workspace_bytes = P.total;
    if (!P.passes.empty()) { // threads per CTA the first pass launches
        const PassPlan &p0 = P.passes[0];
        out->threads_per_block = p0.g5 > 0   ? p0.nt5
                                 : p0.g6 > 0 ? p0.nt6
                                 : p0.g4 > 0 ? p0.g4 * p0.nt4 + 32 * (p0.pw4 + 1)
                                 : p0.v2     ? p0.ntc + 64
                                             : p0.threads;
    }
    double elems = 0, flops = 0;
    int64_t steps = 0, crit = 0;
    for (const PassPlan &pp : P.passes) {
        crit += pp.cycles;
        const int64_t c = pp.c, t = pp.t;
        auto one = [&](int64_t r, int64_t j) {
            int64_t p = r + (c - t) + j * c;
            int64_t q = j ? p - c : r;
            int64_t hi = std::min<int64_t>(p + t, n - 1);
            int64_t ce = std::min<int64_t>(hi + c, n - 1);
            int64_t m = hi - p + 1;
            elems += (double)(m * ((hi - q + 1) + (ce - p + 1) - m));
            flops += (double)(4 * m * (hi - q) + 4 * m * (ce - p) + 6 * m);
        };
        // interior steps (j >= 1, window unclipped: p + t + c <= n - 1) all move
        // (t+1)(2c+t+1) elements and 8(t+1)(c+t) + 6(t+1) flops; the first step
        // and the clipped tail of each sweep are counted one by one
        const double e_int = (double)((t + 1) * (2 * c + t + 1));
        const double f_int = (double)(8 * (t + 1) * (c + t) + 6 * (t + 1));
        for (int64_t r = 0; r < pp.nsweeps; ++r) {
            const int64_t J = sweep_len_h(n, c, t, r);
            steps += J;
            if (J == 0) continue;
            one(r, 0);
            // last j with r + (c - t) + j c + t + c <= n - 1
            const int64_t num = n - 1 - r - 2 * c;
            int64_t jint = num >= 0 ? num / c : 0;
            jint = std::min<int64_t>(jint, J - 1);
            if (jint >= 1) {
                elems += e_int * (double)jint;
                flops += f_int * (double)jint;
            }
            for (int64_t j = std::max<int64_t>(1, jint + 1); j < J; ++j) one(r, j);
        }
    }
    out->steps = steps;
    out->critical_cycles = crit;
    out->alg_elements = elems;
    out->alg_bytes = 2.0 * (double)elem_size(dtype) * elems;
    out->alg_flops = flops;
    return BB_SUCCESS;
}

bb_status bb_launch_count(int64_t n, int64_t b, bb_dtype dtype, int64_t batch, const bb_config *cfg,
                          int64_t *launches)
{
    if (!launches) return BB_ERR_INVALID_VALUE;
    Plan P;
    bb_status s = make_plan(n, b, dtype, batch, cfg, P);
    if (s != BB_SUCCESS) return s;
    if (n == 0 || batch == 0) {
        *launches = 0;
        return BB_SUCCESS;
    }
    int64_t L = 2; // pack + extract
    for (const PassPlan &pp : P.passes)
        L += (P.cfg.schedule == BB_SCHED_CYCLE) ? pp.cycles : (pp.nsweeps > 0 ? 1 : 0);
    *launches = L;
    return BB_SUCCESS;
}

const char *bb_status_string(bb_status s)
{
    switch (s) {
    case BB_SUCCESS: return "BB_SUCCESS";
    case BB_ERR_INVALID_VALUE: return "BB_ERR_INVALID_VALUE: invalid argument";
    case BB_ERR_NOT_SUPPORTED: return "BB_ERR_NOT_SUPPORTED: unsupported dtype or configuration";
    case BB_ERR_OUT_OF_MEMORY: return "BB_ERR_OUT_OF_MEMORY: device allocation failed";
    case BB_ERR_CUDA: return "BB_ERR_CUDA: CUDA runtime or launch failure";
    case BB_ERR_INTERNAL: return "BB_ERR_INTERNAL: internal invariant violated";
    }
    return "unknown bb_status";
}

int32_t bb_version(void) { return BB_VERSION; }

} // extern "C"
