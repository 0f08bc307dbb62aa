// bb_pass_v6.cuh -- segment-ring kernel for the passes whose target bandwidth
// is 1 (c - t == 1: the last pass of Alg. 1), sm_100a.
//
// In such a pass the dependency distance is the paper's "three-cycle
// separation" (reading Q4): sweep r may do A(j) (row
// reflector + right application) only after sweep r-1 finished step j+1, and
// B(j) (column reflector + left application) only after sweep r-1 finished
// A(j+2).  The unit kernel (bb_pass_v5.cuh) cannot be used (its reorder needs
// G <= c - t), and round 1's multi-sweep kernel ran ONE sweep per CTA here, so
// every sweep-to-sweep hand-off crossed CTAs through L2 flags and refills
// (~25 us per sweep, 39 % of the headline run).
//
// This kernel gives one CTA a GROUP of G consecutive sweeps r0 .. r0+G-1, one
// warp-group (WG, NT = 2c threads: one row / one column per thread)
// per sweep, executing the steps in exactly the oracle's arithmetic (bitwise
// equal to the one-sweep-per-CTA kernel), and keeps the band segment the group
// is working on RESIDENT in shared memory as a ring of column CHUNKS:
//
//   chunk m of the group = columns [P_m, P_m + c), P_m = r0 + 1 + m*c
//   (sweep r0's step-m base column), all live rows of each column: band
//   offsets x - i in [-t, c + t] (the fill bound, reading Q11): 3c - 1
//   elements per column, stored with pitch P = 3c at
//   ring[(x - r0 - 1) mod NB][off], off = i - x + c + t, NB = R*c columns.
//
// Data moves between HBM/L2 and the ring exactly once per group:
//   PRODUCER warp: loads chunk m once the previous group's last sweep has
//     finished step m+1 (its progress >= 2m + 4: no sweep of that group
//     touches chunk m afterwards) and the ring slot is free -- ONE TMA box
//     copy (cp.async.bulk.tensor, 3c rows x c columns, completion counted in
//     bytes on the chunk's mbarrier) issued by one thread (fp16 storage: a
//     warp converts to fp32 through registers);
//   WRITER warp: after this group's last sweep s finished step j, every
//     column x < s + 1 + (j+1)c is final for the group (every earlier sweep of
//     the group is ahead of s); it writes those columns back and publishes
//     progress 2j + 2 for the group at gpu scope (release); the final value
//     (2 J_s) only after every WG finished and the rest of the ring is flushed.
// Inside the CTA, WG g waits for WG g-1 with the same rule (A(j): >= 2j + 4,
// B(j): >= 2j + 5) on shared-memory counters with sleeping mbarrier waits
// (bb_pass_v4.cuh's SyncV4 machinery).  WG g trails WG g-1 by 3 half-steps,
// so the ring needs R >= 2 + floor(1.5 (G - 1)) chunks (host: bb_api.cu).
//
// Only one hand-off in G crosses CTAs, and no sweep of the group reloads its
// window from L2.
#pragma once

#include "bb_pass_v4.cuh"

#include <cuda.h>

#include <type_traits>

namespace bb {

#ifndef BB_V6_POLL
#define BB_V6_POLL 20 // ns between polls of a chunk barrier (0: suspended try_wait)
#endif
constexpr int V6_GMAX = 16;
// chunk-loaded events: the producer runs up to R chunks ahead of WG 0, so the
// ring of "chunk m loaded" mbarriers must be longer than R (a phase seen
// twice would hang the waiter); the host caps R below this
constexpr int V6_FRING = 64;
// wait for a chunk-loaded phase: polled with test_wait + a short sleep (a
// suspended try_wait is not reliably woken by TMA complete_tx; measured
// multi-microsecond late wake-ups)
__device__ __forceinline__ bool mb_test_wait(uint64_t *b, unsigned par)
{
    unsigned ok;
    asm volatile("{\n\t.reg .pred P1;\n\t"
                 "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par)
                 : "memory");
    return ok != 0;
}
__device__ __forceinline__ void chunk_wait(uint64_t *b, unsigned par)
{
    if (BB_V6_POLL) {
        while (!mb_test_wait(b, par)) __nanosleep(BB_V6_POLL);
    } else {
        mb_wait(b, par);
    }
}
__device__ __forceinline__ uint64_t *fring_slot(uint64_t *ring, int K, unsigned &par)
{
    par = (unsigned)(K / V6_FRING) & 1u;
    return ring + (K % V6_FRING);
}

struct PassArgsV6 {
    void *W;
    int64_t mat_stride;
    int ldw, ku, n;
    int c, t, G, R;
    int batch, nsweeps, ngroups;
    int *progress; // [batch][ngroups] x fstride: half-steps of each group's last sweep
    int fstride;   // ints between consecutive group flags
    int *counter;
    unsigned long long *trace;
    int trace_groups, trace_steps;
    int trace_ring; // slots 8..15 hold ring-latency clocks (writer / producer / WG0 / last WG) instead of step probes
};

#define TRACE6(slot_, j_)                                                                                  \
    do {                                                                                                   \
        if (a.trace && mat == 0 && k < a.trace_groups && (j_) < a.trace_steps)                            \
            a.trace[((int64_t)k * a.trace_steps + (j_)) * 16 + (slot_)] = gtimer();                        \
    } while (0)
// ring-latency probes (a.trace_ring): clock64 of one SM, slots 8..15
#define TRACE6R(slot_, j_)                                                                                 \
    do {                                                                                                   \
        if (a.trace && a.trace_ring && mat == 0 && k < a.trace_groups && (j_) < a.trace_steps)            \
            a.trace[((int64_t)k * a.trace_steps + (j_)) * 16 + (slot_)] = clock64();                       \
    } while (0)

// ---- TMA (bulk tensor copies) ---------------------------------------------
__device__ __forceinline__ void mb_expect_tx(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// box (3c rows, c columns, 1 matrix) at (row, col, mat) of the working band
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                 "%4}], [%5];" ::"r"(su32(dst)),
                 "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, int c0, int c1, int c2, const void *src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(su32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// every bulk store of this thread complete (its writes performed)
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// every bulk store of this thread has finished READING its shared-memory source
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// generic-proxy accesses (flag acquire, shared-memory reads of a ring slot)
// ordered before the async-proxy (TMA) accesses that follow
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Row access in the ring: element k of row i over columns p + k lives at
// base + k*(P - 1) while the column index does not wrap; past the wrap point
// kw (uniform over the WG) the address drops by NB*P.
template <class C, int MT, bool FULL, bool WRAP, int STR>
__device__ __forceinline__ void ld_row6(const C *b, int m, int kw, int wrapd, C (&v)[MT])
{
#pragma unroll
    for (int k = 0; k < MT; ++k)
        if (FULL || k < m) v[k] = b[k * STR - ((WRAP && k >= kw) ? wrapd : 0)];
}
template <class S, class C, int MT, bool FULL, bool WRAP, int STR>
__device__ __forceinline__ void st_row6(C *b, int m, int kw, int wrapd, const C (&v)[MT])
{
#pragma unroll
    for (int k = 0; k < MT; ++k)
        if (FULL || k < m) b[k * STR - ((WRAP && k >= kw) ? wrapd : 0)] = StoreRound<S, C>::r(v[k]);
}

// One step (r0 + g, j).  FULL: m == MT; WRAP: the step's columns p .. p+t may
// wrap around the ring (then the row-reflector source is staged contiguously).
template <class S, int MT, bool FULL, bool WRAP>
__device__ __forceinline__ void step_v6(const PassArgsV6 &a, typename ComputeOf<S>::type *ring,
                                        typename ComputeOf<S>::type *xstage, int r0, int g, int j, int Jprev,
                                        const SyncV4 &y, int tid, int bar, int NT, unsigned long long *tr)
{
    using C = typename ComputeOf<S>::type;
    constexpr int P = 3 * MT; // column pitch: 3c - 1 live rows (+1 pad: the TMA box)
    constexpr int OFF0 = 2 * MT - 1; // c + t
    const int n = a.n, c = MT;
    const int NB = a.R * MT;
    const int r = r0 + g;
    const int p = r + 1 + j * c;
    const int q = j ? p - c : r;
    const int hi = min(p + MT - 1, n - 1);
    const int ce = min(hi + c, n - 1);
    const int m = FULL ? MT : hi - p + 1;
    const int lane = tid & 31, warp = tid >> 5;
    int xb = (p - r0 - 1) % NB; // ring column of p
    const int kw = NB - xb;      // first k whose column wraps (>= MT: none)
    const int wrapd = NB * P;

    // ---------------------------------------------------------------- A wait
    if (warp == 0) {
        if (g == 0) {
            unsigned par;
            uint64_t *b = fring_slot(y.barF, y.fbase + j, par); // chunk j loaded
            chunk_wait(b, par);
        } else {
            wait_prog(y, g - 1, min(2 * j + 4, 2 * Jprev));
        }
    }
    nbar_sync(bar, NT);
    if (tr && tid == 0) tr[g == 0 ? 4 : 7] = gtimer();
#define PROBE6(i_) do { if (tr && !a.trace_ring && tid == 0 && g == 0) tr[i_] = clock64(); } while (0)
    PROBE6(8);

    // ---------------------------------------------------------------- right application (A)
    // x = A[q][p..hi]; rows q+1..hi, one per thread
    C *xrow = ring + xb * P + (q - p + OFF0); // element k at k*(P-1) (before the wrap)
    if (WRAP) {
        // stage x contiguously (its columns may wrap around the ring)
        if (tid < m) xstage[tid] = xrow[tid * (P - 1) - (tid >= kw ? wrapd : 0)];
        nbar_sync(bar, NT);
    }
    const int nR = hi - q;
    C beta1;
    {
        C av[MT];
        const bool mine = tid < nR;
        C *rb = ring + xb * P + (q + 1 + tid - p + OFF0);
        if (mine) ld_row6<C, MT, FULL, WRAP, P - 1>(rb, m, kw, wrapd, av);
        else {
#pragma unroll
            for (int k = 0; k < MT; ++k) av[k] = C(0);
        }
        if constexpr (WRAP) beta1 = refl_apply<C, MT, FULL, 1>(xstage, m, av, mine);
        else beta1 = refl_apply<C, MT, FULL, P - 1>(xrow, m, av, mine);
        PROBE6(9);
        if (mine) st_row6<S, C, MT, FULL, WRAP, P - 1>(rb, m, kw, wrapd, av);
    }
    PROBE6(10);
    nbar_sync(bar, NT);
    PROBE6(11);
    if (warp == 0) {
        // x row -> (beta, 0, ..., 0): exact zeros in the annihilated slots
        beta1 = StoreRound<S, C>::r(beta1);
        if (lane < m) xrow[lane * (P - 1) - ((WRAP && lane >= kw) ? wrapd : 0)] = lane ? C(0) : beta1;
        __syncwarp();
        if (lane == 0) post_prog(y, g, 2 * j + 1);
    }

    // ---------------------------------------------------------------- B wait
    if (warp == 0) {
        if (g == 0) {
            if (p + c <= n - 1) { // chunk j+1 exists: loaded?
                unsigned par;
                uint64_t *b = fring_slot(y.barF, y.fbase + j + 1, par);
                chunk_wait(b, par);
            }
        } else {
            wait_prog(y, g - 1, min(2 * j + 5, 2 * Jprev));
        }
    }
    nbar_sync(bar, NT);
    if (tr && tid == 0 && g == 0) tr[5] = gtimer();
    PROBE6(12);
    if (tr && a.trace_ring && tid == 0 && g == 0) tr[12] = clock64(); // WG0: chunk j+1 here

    // ---------------------------------------------------------------- left application (B)
    // y = A[p..hi][p], contiguous; columns p+1..ce, one per thread
    C *ycol = ring + xb * P + OFF0;
    const int nL = ce - p;
    C beta2;
    {
        C bv[MT];
        const bool mine = tid < nL;
        int xc = xb + 1 + tid;
        if (xc >= NB) xc -= NB;
        C *cb = ring + xc * P + (OFF0 - 1 - tid); // row p of column p + 1 + tid
        if (mine) ld_vec<1, C, MT, FULL>(cb, m, bv);
        else {
#pragma unroll
            for (int k = 0; k < MT; ++k) bv[k] = C(0);
        }
        beta2 = refl_apply<C, MT, FULL, 1>(ycol, m, bv, mine);
        PROBE6(13);
        if (mine) st_vec<1, S, C, MT, FULL>(cb, m, bv);
    }
    PROBE6(14);
    nbar_sync(bar, NT);
    PROBE6(15);
    if (warp == 0) {
        beta2 = StoreRound<S, C>::r(beta2);
        if (lane < m) ycol[lane] = lane ? C(0) : beta2;
        __syncwarp();
        if (lane == 0) post_prog(y, g, 2 * j + 2);
    }
}

// clipped steps (matrix end): out of line, so the hot code stays small
template <class S, int MT>
__device__ __noinline__ void step_v6_tail(const PassArgsV6 &a, typename ComputeOf<S>::type *ring,
                                          typename ComputeOf<S>::type *xstage, int r0, int g, int j, int Jprev,
                                          const SyncV4 &y, int tid, int bar, int NT, unsigned long long *tr)
{
    step_v6<S, MT, false, true>(a, ring, xstage, r0, g, j, Jprev, y, tid, bar, NT, tr);
}

// fp16 storage: ring columns [x0, x1) loaded by one warp, widened to fp32
// through registers (all 3c - 1 live offsets of each column: one contiguous
// run of the column in HBM)
template <int MT>
__device__ __forceinline__ void v6_load_cols_h(const __half *__restrict__ Wg, int ku, int64_t ldw, int xr0, int NB,
                                               int x0, int x1, float *ring, int lane)
{
    constexpr int P = 3 * MT, OFF0 = 2 * MT - 1, NV = (P - 1 + 31) / 32;
    int xc = xr0;
    for (int x = x0; x < x1; ++x) {
        const __half *src = Wg + (ku - OFF0) + (int64_t)x * ldw;
        float v[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int off = lane + 32 * u;
            v[u] = off < P - 1 ? ldg_cg(src + off) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int off = lane + 32 * u;
            if (off < P - 1) ring[xc * P + off] = v[u];
        }
        if (++xc == NB) xc = 0;
    }
}

// write-back of ring columns [x0, x1) (x < n): all live offsets of each column
template <class S, int MT>
__device__ __forceinline__ void v6_store_cols(S *__restrict__ Wg, int ku, int64_t ldw, int r0, int NB, int x0, int x1,
                                              const typename ComputeOf<S>::type *ring, int lane)
{
    using C = typename ComputeOf<S>::type;
    constexpr int P = 3 * MT, OFF0 = 2 * MT - 1, NV = (P - 1 + 31) / 32;
    if (x1 <= x0) return;
    int xc = (x0 - r0 - 1) % NB;
    for (int x = x0; x < x1; ++x) {
        S *dst = Wg + (ku - OFF0) + (int64_t)x * ldw;
        C v[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int off = lane + 32 * u;
            if (off < P - 1) v[u] = ring[xc * P + off];
        }
#pragma unroll
        for (int u = 0; u < NV; ++u) {
            const int off = lane + 32 * u;
            if (off < P - 1) stg(dst + off, v[u]);
        }
        if (++xc == NB) xc = 0;
    }
}

// G compute WGs of NT = 2c threads, one producer warp, one writer warp.
template <class S, int MT, int NTMAX>
__global__ void __launch_bounds__(NTMAX, 1) pass_v6_kernel(PassArgsV6 a, const __grid_constant__ CUtensorMap tmap)
{
    using C = typename ComputeOf<S>::type;
    constexpr int NT = 2 * MT;
    constexpr int P = 3 * MT;
    constexpr bool TMA = std::is_same<S, C>::value; // fp16 storage widens through registers
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // TMA destinations: 128-byte aligned (the host adds 128 bytes of slack)
    C *ring = reinterpret_cast<C *>(smem_raw + ((128 - (su32(smem_raw) & 127)) & 127));
    __shared__ int s_task;
    __shared__ int prog_s[V6_GMAX];
    __shared__ __align__(8) uint64_t bars[2 * V6_GMAX * V4_RING + V6_FRING];
    __shared__ int ebase_s[V6_GMAX];
    __shared__ int fbase_s;
    __shared__ volatile int wb_s; // chunks written back (ring slots free)
    __shared__ C xstage_s[V6_GMAX][MT + 1];
    constexpr int NBAR = 2 * V6_GMAX * V4_RING + V6_FRING;

    const int G = a.G, n = a.n, c = MT, t = MT - 1;
    const int NB = a.R * MT;
    const int ncomp = G * NT;
    const int total = a.batch * a.ngroups;
    for (int i = threadIdx.x; i < NBAR; i += blockDim.x)
        mb_init(bars + i, (i >= 2 * V6_GMAX * V4_RING && !TMA) ? 32u : 1u);
    fence_mbarrier_init();
    if (threadIdx.x < V6_GMAX) ebase_s[threadIdx.x] = 0;
    if (threadIdx.x == 0) fbase_s = 0;
    int prev_r0 = -1, prev_M = 0;

    for (;;) {
        __syncthreads(); // the previous task is complete
        if (threadIdx.x == 0) {
            s_task = atomicAdd(a.counter, 1);
            wb_s = 0;
        }
        if (threadIdx.x < V6_GMAX) {
            prog_s[threadIdx.x] = 0;
            if (prev_r0 >= 0 && prev_r0 + (int)threadIdx.x < a.nsweeps)
                ebase_s[threadIdx.x] += sweep_len(n, c, t, prev_r0 + threadIdx.x);
        }
        if (threadIdx.x == 0 && prev_r0 >= 0) fbase_s += prev_M;
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int k = task / a.batch;
        const int r0 = k * G;
        const int glast = min(G, a.nsweeps - r0) - 1;
        // chunks of the group: columns [r0 + 1 + m c, ...) inside the matrix
        const int M = (r0 + 1 <= n - 1) ? (n - 1 - (r0 + 1)) / c + 1 : 0;
        prev_r0 = r0;
        prev_M = M;
        const SyncV4 y{prog_s, bars, bars + V6_GMAX * V4_RING, bars + 2 * V6_GMAX * V4_RING, ebase_s, fbase_s};
        S *Wg = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;
        const int64_t ldw = a.ldw;
        const int ku = a.ku;
        int *gprog = a.progress + (int64_t)mat * a.ngroups * a.fstride;
        const int fs = a.fstride;

        if ((int)threadIdx.x < ncomp) {
            // ------------------------------------------------ compute WGs
            const int g = threadIdx.x / NT;
            const int tid = threadIdx.x - g * NT;
            if (g <= glast) {
                const int r = r0 + g;
                const int J = sweep_len(n, c, t, r);
                const int Jprev = g > 0 ? sweep_len(n, c, t, r - 1) : 0;
                for (int j = 0; j < J; ++j) {
                    const int p = r + 1 + j * c;
                    const int xb = (p - r0 - 1) % NB;
                    const bool full = p + MT - 1 <= n - 1;
                    if (g == 0 && tid == 0) TRACE6(0, j);
                    unsigned long long *tr = (a.trace && g <= 1 && mat == 0 && k < a.trace_groups && j < a.trace_steps)
                                                 ? a.trace + ((int64_t)k * a.trace_steps + j) * 16
                                                 : nullptr;
                    if (full && xb + MT <= NB)
                        step_v6<S, MT, true, false>(a, ring, &xstage_s[g][0], r0, g, j, Jprev, y, tid, 1 + g, NT, tr);
                    else if (full) // the row access wraps the ring (once per R steps for WG g > 0): inline,
                                   // an out-of-line call saved / restored ~600 B of registers per thread
                                   // through local memory
                        step_v6<S, MT, true, true>(a, ring, &xstage_s[g][0], r0, g, j, Jprev, y, tid, 1 + g, NT, tr);
                    else
                        step_v6_tail<S, MT>(a, ring, &xstage_s[g][0], r0, g, j, Jprev, y, tid, 1 + g, NT, tr);
                    if (g == 0 && tid == 0) TRACE6(6, j);
                    if (g == glast && tid == 0) TRACE6(1, j);
                    if (g == glast && tid == 0) TRACE6R(13, j); // last WG finished step j
                }
            }
        } else if ((int)threadIdx.x < ncomp + 32) {
            // ------------------------------------------------ PRODUCER warp: chunk loads
            const int lane = threadIdx.x & 31;
            const int Jp = r0 > 0 ? sweep_len(n, c, t, r0 - 1) : 0;
            const int *pprev = k > 0 ? gprog + (int64_t)(k - 1) * fs : nullptr;
            for (int mm = 0; mm < M; ++mm) {
                if (lane == 0) {
                    // ring slot of chunk mm - R free (written back)
                    if (mm >= a.R)
                        while (wb_s < mm - a.R + 1) __nanosleep(64);
                    TRACE6R(10, mm); // ring slot free
                    // the previous group's last sweep finished step mm + 1 (and wrote it back)
                    if (pprev) wait_geq_v4(pprev, min(2 * mm + 4, 2 * Jp), 2 * mm);
                    TRACE6(2, mm);
                }
                const int x0 = r0 + 1 + mm * c;
                C *slot = ring + (size_t)(mm % a.R) * c * P;
                unsigned par;
                uint64_t *fb = fring_slot(y.barF, y.fbase + mm, par);
                if constexpr (TMA) {
                    if (lane == 0) {
                        fence_proxy_async(); // acquired global data and freed slot -> async proxy
                        mb_expect_tx(fb, (unsigned)(c * P * sizeof(C)));
                        tma_load_3d(slot, &tmap, ku - (2 * MT - 1), x0, mat, fb);
                        TRACE6R(11, mm); // load issued
                    }
                } else {
                    __syncwarp();
                    v6_load_cols_h<MT>(reinterpret_cast<const __half *>(Wg), ku, ldw, (mm % a.R) * c, NB, x0,
                                       min(x0 + c, n), reinterpret_cast<float *>(ring), lane);
                    mb_arrive(fb);
                }
            }
        } else if ((int)threadIdx.x < ncomp + 64) {
            // ------------------------------------------------ WRITER warp: write-back + publish
            // chunk m is final for the group once its last sweep s finished step
            // m (every column < s + 1 + (m+1)c is); the next group's chunk m' needs
            // our columns < r0 + G + (m'+1)c, i.e. chunk m'+1: published 2(m'+1)+2
            const int lane = threadIdx.x & 31;
            const int s = r0 + glast;
            const int Js = sweep_len(n, c, t, s);
            auto write_chunk = [&](int mm) {
                const int x0 = r0 + 1 + mm * c;
                const C *slot = ring + (size_t)(mm % a.R) * c * P;
                if constexpr (TMA) {
                    if (lane == 0) {
                        fence_proxy_async(); // WG writes of the slot -> async-proxy reads
                        tma_store_3d(&tmap, ku - (2 * MT - 1), x0, mat, slot);
                    }
                } else {
                    v6_store_cols<S, MT>(Wg, ku, ldw, r0, NB, x0, min(x0 + c, n), ring, lane);
                }
            };
            auto publish = [&](int v, int wb) {
                if constexpr (TMA) {
                    if (lane == 0) tma_store_wait_all();
                }
                __syncwarp();
                if (lane == 0) {
                    fence_proxy_async(); // async-proxy global writes -> generic release
                    fence_acq_rel();
                    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(gprog + (int64_t)k * fs), "r"(v) : "memory");
                    wb_s = wb;
                }
            };
            // Batched: every step the last WG has finished since the previous
            // round is written back in one go (one completion wait per round, not
            // per chunk -- a serial store + wait per chunk capped the group at one
            // step per write-back latency, ~2 us); ring slots are released as soon
            // as the stores have READ them, before the global writes complete.
            int wb = 0; // chunks written back
            int j = 0;  // steps [0, j) handled
            while (j < Js - 1) {
                int have = 0;
                if (lane == 0) {
                    wait_prog(y, glast, 2 * j + 2);
                    have = lds_acquire_v(y.prog + glast);
                }
                have = __shfl_sync(0xffffffffu, have, 0);
                const int jend = min(Js - 1, have >> 1); // steps [0, jend) of the last WG done
                if (lane == 0)
                    for (int jj = j; jj < jend; ++jj) TRACE6R(8, jj); // writer saw step jj done
                for (; j < jend; ++j)
                    if (j < M) {
                        write_chunk(j);
                        wb = j + 1;
                    }
                if constexpr (TMA) {
                    if (lane == 0) {
                        tma_store_wait_read();
                        wb_s = wb; // slots free for the producer
                        for (int jj = 0; jj < 64 && jend - 1 - jj >= 0; ++jj) {
                            if (a.trace && a.trace_ring && mat == 0 && k < a.trace_groups && jend - 1 - jj < a.trace_steps) {
                                unsigned long long *q = a.trace + ((int64_t)k * a.trace_steps + (jend - 1 - jj)) * 16 + 9;
                                if (*q) break;
                                *q = clock64(); // slot of chunk freed
                            } else break;
                        }
                    }
                }
                publish(2 * jend, wb);
                if (lane == 0) TRACE6(3, jend - 1);
            }
            // every WG finished: flush the rest of the ring, publish the final value
            if (lane == 0)
                for (int g = 0; g <= glast; ++g) wait_prog(y, g, 2 * sweep_len(n, c, t, r0 + g));
            __syncwarp();
            for (int mm = wb; mm < M; ++mm) write_chunk(mm);
            publish(2 * Js, M);
        }
    }
}

} // namespace bb
