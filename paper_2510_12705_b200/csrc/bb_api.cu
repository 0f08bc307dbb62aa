// bb_api.cu -- C ABI (include/bandbidiag.h) of the B200 band -> bidiagonal
// reduction: argument validation, pass plan (Alg. 1 line 1), workspace
// carving, and the launch sequence pack -> one launch per pass -> extract.
//
// Host logic only; every arithmetic step of the method runs in the kernels of
// bb_kernels.cuh.  No CPU fallback exists: without a usable CUDA device every
// compute entry point returns BB_ERR_CUDA.
#include "bb_kernels.cuh"
#include "bb_pass_v2.cuh"
#include "bb_pass_v4.cuh"

#include <cudaTypedefs.h>
#include "bandbidiag.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace {

constexpr size_t kAlign = 256;
constexpr int kSmemOptinFallback = 227 * 1024;

inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
inline int round_odd(int x) { return (x & 1) ? x : x + 1; }

size_t elem_size(bb_dtype dt)
{
    switch (dt) {
    case BB_F16: return 2;
    case BB_F32: return 4;
    case BB_F64: return 8;
    }
    return 0;
}
size_t compute_size(bb_dtype dt) { return dt == BB_F64 ? 8 : 4; }

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
};

struct Plan {
    int64_t n = 0, b_eff = 0, batch = 0;
    int tw = 0;
    int64_t ldw = 0, ku = 0, mat_stride = 0;
    bb_config cfg{};
    std::vector<PassPlan> passes;
    size_t band_bytes = 0, flag_bytes = 0, counter_bytes = 0, total = 0;
};

int default_tw(bb_dtype dt)
{
    // P:315 found one 128-byte cache line optimal on its GPUs: 32 (FP32), 16
    // (FP64).  On B200 with the v4 kernel tw = 32 is faster for FP64 too
    // (n = 32768, b = 128: 2.2 s vs 2.6 s): the number of
    // passes -- each a chain of ~n sweep hand-offs -- halves.
    (void)dt;
    return 32;
}

int64_t sweep_len_h(int64_t n, int64_t c, int64_t t, int64_t r)
{
    int64_t first = r + c - t;
    return first > n - 2 ? 0 : (n - 2 - first) / c + 1;
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
    P.ku = P.b_eff + tw;
    P.ldw = P.b_eff + 2 * tw + 1; // band + twice the tilewidth (reading Q11)
    {
        // TMA diagonal view: (ldw - 1) * elem must be a multiple of 16 bytes
        const int64_t q = 16 / (int64_t)elem_size(dtype);
        while ((P.ldw - 1) % q) ++P.ldw;
        P.mat_stride = (n * P.ldw + q - 1) / q * q;
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
            P.passes.push_back(pp);
            c -= t;
        }
    }
    if (cfg.timing_events && cfg.num_timing_events < (int)P.passes.size() + 3) return BB_ERR_INVALID_VALUE;
    P.cfg = cfg;
    size_t es = elem_size(dtype);
    P.band_bytes = align_up((size_t)batch * (size_t)P.mat_stride * es);
    P.flag_bytes = align_up((size_t)P.passes.size() * (size_t)batch * (size_t)n * sizeof(int));
    P.counter_bytes = align_up(std::max<size_t>(1, P.passes.size()) * sizeof(int));
    P.total = P.band_bytes + P.flag_bytes + P.counter_bytes;
    return BB_SUCCESS;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder()
{
    static std::once_flag once;
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    });
    return fn;
}

struct DeviceInfo {
    int sms = 0;
    int smem_optin = 0;
    bool ok = false;
};

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

template <class S>
bb_status launch_all(const Plan &P, const void *band, int64_t ldband, int64_t stride_band, int64_t b_in,
                     void *d_out, int64_t stride_d, void *e_out, int64_t stride_e, void *ws, cudaStream_t st)
{
    DeviceInfo di;
    if (!device_info(di)) return BB_ERR_CUDA;
    unsigned char *base = reinterpret_cast<unsigned char *>(ws);
    S *W = reinterpret_cast<S *>(base);
    int *flags = reinterpret_cast<int *>(base + P.band_bytes);
    int *counters = reinterpret_cast<int *>(base + P.band_bytes + P.flag_bytes);
    const int64_t mat_stride = P.mat_stride;
    const int n = (int)P.n;
    const int batch = (int)P.batch;

    cudaEvent_t *ev = reinterpret_cast<cudaEvent_t *>(P.cfg.timing_events);
    auto mark = [&](int k) { if (ev) cudaEventRecord(ev[k], st); };
    if (!P.passes.empty()) {
        if (cudaMemsetAsync(flags, 0, P.flag_bytes + P.counter_bytes, st) != cudaSuccess) return BB_ERR_CUDA;
    }
    mark(0);
    {
        int64_t total = (int64_t)batch * mat_stride;
        int thr = 256;
        int64_t blocks = std::min<int64_t>((total + thr - 1) / thr, (int64_t)di.sms * 16);
        bb::pack_kernel<S><<<(unsigned)std::max<int64_t>(blocks, 1), thr, 0, st>>>(
            reinterpret_cast<const S *>(band), ldband, stride_band, (int)b_in, (int)P.b_eff, W, mat_stride,
            (int)P.ldw, (int)P.ku, n, batch);
    }
    mark(1);
    size_t npasses = P.passes.size();
    if (const char *dp = getenv("BB_DEBUG_PASSES")) npasses = std::min(npasses, (size_t)atoi(dp)); // debug only
    for (size_t pi = 0; pi < npasses; ++pi) {
        const PassPlan &pp = P.passes[pi];
        if ((int)pp.smem > di.smem_optin) return BB_ERR_NOT_SUPPORTED;
        bb::PassArgs a{};
        a.W = W;
        a.mat_stride = mat_stride;
        a.ldw = (int)P.ldw;
        a.ku = (int)P.ku;
        a.n = n;
        a.c = pp.c;
        a.t = pp.t;
        a.s = pp.s;
        a.batch = batch;
        a.nsweeps = pp.nsweeps;
        a.progress = flags + (int64_t)pi * batch * n;
        a.counter = counters + pi;
        a.LT = pp.LT;
        a.LW = pp.LW;
        if (P.cfg.schedule == BB_SCHED_CYCLE) {
            auto kern = bb::pass_cycle_kernel<S>;
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem) != cudaSuccess)
                return BB_ERR_CUDA;
            int maxT = pp.cycles;
            if (const char *dbg = getenv("BB_DEBUG_MAX_CYCLES")) maxT = std::min(maxT, atoi(dbg)); // debug only
            for (int T = 0; T < maxT; ++T) {
                a.cycle_T = T;
                int rmax = std::min(T / pp.s + 1, pp.nsweeps);
                dim3 grid((unsigned)std::max(rmax, 1), (unsigned)batch);
                kern<<<grid, pp.threads, pp.smem, st>>>(a);
            }
        } else if (pp.g4 > 0) {
            const int G = pp.g4;
            bb::PassArgsV4 a4{};
            a4.W = W;
            a4.mat_stride = mat_stride;
            a4.ldw = (int)P.ldw;
            a4.ku = (int)P.ku;
            a4.n = n;
            a4.c = pp.c;
            a4.t = pp.t;
            a4.a0 = pp.a4;
            a4.b0 = pp.b4;
            a4.batch = batch;
            a4.nsweeps = pp.nsweeps;
            a4.G = G;
            a4.ngroups = (pp.nsweeps + G - 1) / G;
            a4.progress = a.progress;
            a4.counter = a.counter;
            a4.NT = pp.nt4;
            a4.LDT = pp.LDT4;
            a4.LDW = pp.LDW4;
            a4.NS = pp.NS4;
            a4.slot_elems = pp.slot4;
            a4.pw = pp.pw4;
            int nt = G * pp.nt4 + 32 * (pp.pw4 + 1);
            void (*kern)(bb::PassArgsV4) = nullptr;
            constexpr bool F64 = sizeof(typename bb::ComputeOf<S>::type) == 8;
            switch (pp.t + 1) {
            case 16: kern = bb::pass_v4_kernel<S, 16, 576, 25>; break;
            case 17: kern = bb::pass_v4_kernel<S, 17, 576, 25>; break;
            case 32:
                kern = !F64 ? bb::pass_v4_kernel<S, 32, 576, 41>
                            : (pp.ntmax4 <= 384 ? bb::pass_v4_kernel<S, 32, 384, 35> : bb::pass_v4_kernel<S, 32, 512, 35>);
                break;
            default:
                kern = !F64 ? bb::pass_v4_kernel<S, 33, 576, 41>
                            : (pp.ntmax4 <= 384 ? bb::pass_v4_kernel<S, 33, 384, 35> : bb::pass_v4_kernel<S, 33, 512, 35>);
                break;
            }
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem4) != cudaSuccess)
                return BB_ERR_CUDA;
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, pp.smem4) != cudaSuccess)
                return BB_ERR_CUDA;
            if (occ < 1) return BB_ERR_NOT_SUPPORTED;
            if (occ >= 2 && a4.pw > 1) {
                // several CTAs per SM (small c): resident groups bound the wavefront
                // (each CTA holds its sweeps for ~n/c steps), so trade a producer warp
                // for occupancy when that admits more CTAs per SM
                int occ1 = 0;
                const int nt1 = nt - 32 * (a4.pw - 1);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, kern, nt1, pp.smem4) == cudaSuccess &&
                    occ1 > occ) {
                    occ = occ1;
                    a4.pw = 1;
                    nt = nt1;
                }
            }
            if (P.cfg.max_blocks_per_sm > 0) occ = std::min(occ, (int)P.cfg.max_blocks_per_sm);
            else if (pp.c - pp.t == 1 && pp.c >= 32 && batch == 1) occ = 1; // measured: the sweep chain of the
            // target-bandwidth-1 pass (c >= 32) runs faster with one CTA per SM (tools/maxb_sweep.py)
            int64_t tasks = (int64_t)a4.ngroups * batch;
            int64_t grid = std::min<int64_t>(tasks, (int64_t)occ * di.sms);
            const char *tf = getenv("BB_TRACE_FILE");
            const char *tp = getenv("BB_TRACE_PASS");
            unsigned long long *tbuf = nullptr;
            if (tf && (int)pi == (tp ? atoi(tp) : 0)) {
                a4.trace_sweeps = std::min(pp.nsweeps, 1024);
                a4.trace_steps = (int)sweep_len_h(n, pp.c, pp.t, 0);
                size_t tb = (size_t)a4.trace_sweeps * a4.trace_steps * 16 * sizeof(unsigned long long);
                if (cudaMalloc(&tbuf, tb) == cudaSuccess) {
                    cudaMemsetAsync(tbuf, 0, tb, st);
                    a4.trace = tbuf;
                }
            }
            if (grid >= 1) kern<<<(unsigned)grid, nt, pp.smem4, st>>>(a4);
            if (tbuf) {
                size_t cnt = (size_t)a4.trace_sweeps * a4.trace_steps * 16;
                std::vector<unsigned long long> h(cnt);
                cudaMemcpyAsync(h.data(), tbuf, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                if (FILE *f = fopen(tf, "wb")) {
                    int hdr[6] = {a4.trace_sweeps, a4.trace_steps, pp.c, pp.t, G, (int)grid};
                    fwrite(hdr, sizeof(int), 6, f);
                    fwrite(h.data(), sizeof(unsigned long long), cnt, f);
                    fclose(f);
                }
                cudaFree(tbuf);
            }
        } else if (pp.v2) {
            bb::PassArgsV2 a2{};
            a2.W = W;
            a2.mat_stride = mat_stride;
            a2.ldw = (int)P.ldw;
            a2.ku = (int)P.ku;
            a2.n = n;
            a2.c = pp.c;
            a2.t = pp.t;
            a2.a0 = pp.a0;
            a2.b0 = pp.b0;
            a2.batch = batch;
            a2.nsweeps = pp.nsweeps;
            a2.progress = a.progress;
            a2.counter = a.counter;
            a2.ntc = pp.ntc;
            a2.LW = pp.LW2;
            void (*kern)(bb::PassArgsV2) = nullptr;
            const int nt = pp.ntc + 64;
            if (nt <= 256) {
                kern = pp.mt == 9 ? bb::pass_v2_kernel<S, 9, 256>
                                  : (pp.mt == 17 ? bb::pass_v2_kernel<S, 17, 256> : bb::pass_v2_kernel<S, 33, 256>);
            } else {
                kern = pp.mt == 9 ? bb::pass_v2_kernel<S, 9, 512>
                                  : (pp.mt == 17 ? bb::pass_v2_kernel<S, 17, 512> : bb::pass_v2_kernel<S, 33, 512>);
            }
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem2) != cudaSuccess)
                return BB_ERR_CUDA;
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, pp.smem2) != cudaSuccess)
                return BB_ERR_CUDA;
            if (P.cfg.max_blocks_per_sm > 0) occ = std::min(occ, (int)P.cfg.max_blocks_per_sm);
            occ = std::max(occ, 1);
            int64_t tasks = (int64_t)pp.nsweeps * batch;
            int64_t grid = std::min<int64_t>(tasks, (int64_t)occ * di.sms);
            const char *tf = getenv("BB_TRACE_FILE");
            const char *tp = getenv("BB_TRACE_PASS");
            unsigned long long *tbuf = nullptr;
            if (tf && (int)pi == (tp ? atoi(tp) : 0)) {
                a2.trace_sweeps = std::min(pp.nsweeps, 1024);
                a2.trace_steps = (int)sweep_len_h(n, pp.c, pp.t, 0);
                size_t tb = (size_t)a2.trace_sweeps * a2.trace_steps * 16 * sizeof(unsigned long long);
                if (cudaMalloc(&tbuf, tb) == cudaSuccess) {
                    cudaMemsetAsync(tbuf, 0, tb, st);
                    a2.trace = tbuf;
                }
            }
            if (grid >= 1) kern<<<(unsigned)grid, nt, pp.smem2, st>>>(a2);
            if (tbuf) {
                size_t cnt = (size_t)a2.trace_sweeps * a2.trace_steps * 16;
                std::vector<unsigned long long> h(cnt);
                cudaMemcpyAsync(h.data(), tbuf, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                if (FILE *f = fopen(tf, "wb")) {
                    int hdr[6] = {a2.trace_sweeps, a2.trace_steps, pp.c, pp.t, pp.s, (int)grid};
                    fwrite(hdr, sizeof(int), 6, f);
                    fwrite(h.data(), sizeof(unsigned long long), cnt, f);
                    fclose(f);
                }
                cudaFree(tbuf);
            }
        } else {
            auto kern = bb::pass_flags_kernel<S>;
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem) != cudaSuccess)
                return BB_ERR_CUDA;
            int occ = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, pp.threads, pp.smem) != cudaSuccess)
                return BB_ERR_CUDA;
            if (P.cfg.max_blocks_per_sm > 0) occ = std::min(occ, (int)P.cfg.max_blocks_per_sm);
            occ = std::max(occ, 1);
            int64_t tasks = (int64_t)pp.nsweeps * batch;
            int64_t grid = std::min<int64_t>(tasks, (int64_t)occ * di.sms);
            // debug tracing (BB_TRACE_FILE, BB_TRACE_PASS): per-step timestamps of
            // matrix 0's first sweeps in one pass, dumped after that pass
            const char *tf = getenv("BB_TRACE_FILE");
            const char *tp = getenv("BB_TRACE_PASS");
            unsigned long long *tbuf = nullptr;
            if (tf && (int)pi == (tp ? atoi(tp) : 0)) {
                a.trace_sweeps = std::min(pp.nsweeps, 1024);
                a.trace_steps = (int)sweep_len_h(n, pp.c, pp.t, 0);
                size_t tb = (size_t)a.trace_sweeps * a.trace_steps * 4 * sizeof(unsigned long long);
                if (cudaMalloc(&tbuf, tb) == cudaSuccess) {
                    cudaMemsetAsync(tbuf, 0, tb, st);
                    a.trace = tbuf;
                }
            }
            if (grid >= 1) kern<<<(unsigned)grid, pp.threads, pp.smem, st>>>(a);
            if (tbuf) {
                size_t cnt = (size_t)a.trace_sweeps * a.trace_steps * 4;
                std::vector<unsigned long long> h(cnt);
                cudaMemcpyAsync(h.data(), tbuf, cnt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                if (FILE *f = fopen(tf, "wb")) {
                    int hdr[6] = {a.trace_sweeps, a.trace_steps, pp.c, pp.t, pp.s, (int)grid};
                    fwrite(hdr, sizeof(int), 6, f);
                    fwrite(h.data(), sizeof(unsigned long long), cnt, f);
                    fclose(f);
                }
                cudaFree(tbuf);
            }
        }
        if (getenv("BB_DEBUG_SYNC")) { // debug: surface asynchronous kernel errors per pass
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) {
                fprintf(stderr, "bandbidiag: pass %d (c=%d t=%d g4=%d v2=%d) failed: %s\n", (int)pi, pp.c, pp.t,
                        pp.g4, (int)pp.v2, cudaGetErrorString(e));
                return BB_ERR_CUDA;
            }
        }
        if (cudaGetLastError() != cudaSuccess) return BB_ERR_CUDA;
        mark(2 + (int)pi);
    }
    {
        int64_t total = (int64_t)batch * n;
        int thr = 256;
        int64_t blocks = std::min<int64_t>((total + thr - 1) / thr, (int64_t)di.sms * 8);
        bb::extract_kernel<S><<<(unsigned)std::max<int64_t>(blocks, 1), thr, 0, st>>>(
            W, mat_stride, (int)P.ldw, (int)P.ku, n, batch, reinterpret_cast<S *>(d_out), stride_d,
            reinterpret_cast<S *>(e_out), stride_e, (P.cfg.flags & BB_FLAG_NONNEG_OUTPUT) ? 1 : 0);
    }
    mark(2 + (int)P.passes.size());
    if (cudaGetLastError() != cudaSuccess) return BB_ERR_CUDA;
    return BB_SUCCESS;
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

} // namespace

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
    unsigned char *buf = nullptr;
    const size_t total = band_b + d_b + e_b + P.total;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&buf), total, st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return e == cudaErrorMemoryAllocation ? BB_ERR_OUT_OF_MEMORY : BB_ERR_CUDA;
    }
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
    if (cudaFreeAsync(buf, st) != cudaSuccess && s == BB_SUCCESS) s = BB_ERR_CUDA;
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
    out->threads_per_block = P.passes.empty() ? 0 : P.passes[0].threads;
    double elems = 0, flops = 0;
    int64_t steps = 0, crit = 0;
    for (const PassPlan &pp : P.passes) {
        crit += pp.cycles;
        for (int64_t r = 0; r < pp.nsweeps; ++r) {
            int64_t J = sweep_len_h(n, pp.c, pp.t, r);
            for (int64_t j = 0; j < J; ++j) {
                int64_t p = r + (pp.c - pp.t) + j * pp.c;
                int64_t q = j ? p - pp.c : r;
                int64_t hi = std::min<int64_t>(p + pp.t, n - 1);
                int64_t ce = std::min<int64_t>(hi + pp.c, n - 1);
                int64_t m = hi - p + 1;
                elems += (double)(m * ((hi - q + 1) + (ce - p + 1) - m));
                flops += (double)(4 * m * (hi - q) + 4 * m * (ce - p) + 6 * m);
                ++steps;
            }
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
