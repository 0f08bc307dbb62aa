// bb_pass_v4.cuh -- multi-sweep persistent pass kernel, latency-optimised step
// (sm_100a).
//
// A pass (Alg. 1 lines 2-12) is a chain of ~n sweep-to-sweep
// hand-offs: sweep r+1 may do step j only after sweep r did (part of) step
// j+1 (refined rule of bb_pass_v2.cuh).  The time of a pass is
// therefore ~n x (step latency + hand-off latency).  This kernel attacks both:
//
//  * G CONSECUTIVE sweeps per CTA, one warp-group (WG) each ("software-level
//    loop unrolling: a single block is assigned multiple tasks", with
//    the tasks overlapped).  Their step windows at step j differ by a shift of
//    one row and one column, so the union lives in ONE shared-memory slot; a
//    WG -> WG hand-off is a shared-memory progress counter and no data moves.
//    Only every G-th hand-off crosses CTAs (global progress flags + L2).
//  * PRODUCER warps (2..6, a.pw) fill slot j from L2 with flattened cp.async
//    copies as soon as the previous group allows it (their own global waits):
//    the T part first (all WG 0's right application needs, signalled on its
//    own mbarrier), then the early W columns, then -- after the B wait -- the
//    late W columns;
//  * the step (Alg. 2) with a short critical path: every thread of the WG
//    loads the reflector source vector x (row q) itself and computes the
//    reflector scalars redundantly (beta, tau, rho = 1/(alpha - beta); no
//    broadcast barrier), and the dot products are taken against x directly,
//        w_i = tau * (A[i][p] + rho * sum_{k>=1} A[i][p+k] x_k),
//        A[i][p+k] -= w_i * v_k,  v_0 = 1, v_k = rho * x_k,
//    so they overlap the norm reduction (same reflector as LAPACK dlarfg,
//    reading Q7; identity iff x[1:] == 0 exactly, reading Q8).  The left
//    application is the same with the column y = A[p..hi][p].  Two WG
//    barriers per step.  With G = 1 the right-application rows are also
//    written through to the band from registers.
//  * write-back by the LAST MODIFIER: the "closer" of step j (the last WG of
//    the group that has a step j) copies the group's whole step-j union to
//    the working band: the right-application region after its A half (before
//    progress 2j+1 is published) and the left-application region after its B
//    half (before 2j+2).  Cells of the union that no WG touched are copied
//    unchanged; nobody else writes them in between (c - t >= 2G, see below).
//
// SLOT j (sweep r0's geometry p0 = r0 + (c - t) + j*c, q0 = (j ? p0 - c : r0),
// WT = t + G, trow0 = (j ? q0 + WT : r0)) holds, in the compute type C, with
// a compile-time odd pitch TP >= WT (see "Shared-memory layout" below):
//   T: rows [trow0, trow0 + c + G) x cols [p0, p0 + WT), row-major
//   W: rows [p0, p0 + WT) x cols [p0 + WT, p0 + WT + c), column-major
// Rows [q0, q0 + WT) of cols [p0, p0 + WT) belong to slot j-1's W (its right
// end), so every cell has exactly one home.  Only cells with band offset
// col - row in [-t, c + t] (the fill-in bound, reading Q11) are ever loaded,
// used or written back.
//
// ORDERING.  Inside the CTA: WG g waits for WG g-1 with the half-step rule
// (A(j): progress >= 2j + a0, B(j): >= 2j + b0; a0/b0 by target bandwidth,
// bb_api.cu), on shared-memory counters (CTA-scope release/acquire) with
// mbarrier-based sleeping waits.  Across CTAs (previous group -> WG 0 through
// the producer): the T part and the early W columns of slot j are loaded
// after the previous group's last sweep published 2j + a0; the late W columns
// (those the phase awaited by B can still modify) after 2j + b0.
// The RELEASE warp republishes the group's last sweep's counter at gpu scope
// (fence + store); the final value (sweep finished) is only published once
// every WG of the group finished, so data written back by earlier WGs at the
// matrix end is covered.  With c - t >= 2G no other group writes a cell of a
// slot between its fill and its write-back (v4 section).
#pragma once

#include "bb_pass_v2.cuh"

#include <cstdio>

namespace bb {

#ifndef BB_V4_WATCHDOG
#define BB_V4_WATCHDOG 0 // debug: print a message when a wait exceeds 2 s (hang diagnosis)
#endif

constexpr int V4_GMAX = 8;
constexpr int V4_PW = 2; // producer warps (minimum; the launch may add more: a.pw)

struct PassArgsV4 {
    void *W;
    int64_t mat_stride;
    int ldw, ku, n;
    int c, t;
    int a0, b0;
    int batch, nsweeps;
    int G, ngroups;
    int *progress; // [batch][n]
    int *counter;
    int NT;         // threads per WG (multiple of 32, >= c + t)
    int LDT, LDW;   // slot pitches (odd)
    int NS;         // slots in the ring (>= G + 1)
    int slot_elems; // elements per slot: LDT*WT (T) then LDW*c (W)
    int pw;         // producer warps (>= V4_PW)
    unsigned long long *trace;
    int trace_sweeps, trace_steps;
};

__device__ __forceinline__ int lds_volatile(const int *p)
{
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void lds_acquire(const int *p)
{
    asm volatile("{\n\t.reg .b32 t;\n\tld.acquire.cta.shared.b32 t, [%0];\n\t}" ::"r"((unsigned)__cvta_generic_to_shared(p))
                 : "memory");
}
__device__ __forceinline__ int lds_acquire_v(const int *p)
{
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void sts_release(int *p, int v)
{
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
// ---- intra-CTA signalling: progress counters + mbarriers -------------------
// The counters (prog_s[g] = completed half-steps of WG g) are the truth; a
// ring of V4_RING mbarriers per WG and per half (arrival count 1) lets the
// waiters SLEEP in hardware (mbarrier.try_wait) instead of spinning on shared
// memory -- spinning warps flood the LSU and slow every other warp's memory
// traffic several-fold (measured: fills and write-backs 4-8x slower).  A
// waiter re-checks the counter after every (time-bounded) try_wait, so ring
// aliasing can never deadlock it.
constexpr int V4_RING = 16;

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
// make mbarrier initialisations visible before first use (by other threads)
__device__ __forceinline__ void fence_mbarrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mb_inval(uint64_t *b)
{
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_cp_async_arrive(uint64_t *b)
{
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(b)) : "memory");
}
// true once the phase with parity `par` has completed; sleeps up to ~hint ns
__device__ __forceinline__ bool mb_try_wait(uint64_t *b, unsigned par, unsigned hint_ns)
{
    unsigned ok;
    asm volatile("{\n\t.reg .pred P1;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\t"
                 "selp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par), "r"(hint_ns)
                 : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mb_wait(uint64_t *b, unsigned par)
{
    unsigned long long t0 = 0;
    while (!mb_try_wait(b, par, 1000000u)) {
        if (BB_V4_WATCHDOG) {
            const unsigned long long now = gtimer();
            if (!t0) t0 = now;
            if (now - t0 > 2000000000ull && t0 != 1) {
                if ((threadIdx.x & 31) == 0)
                    printf("v4 watchdog: mb_wait block %d thread %d\n", (int)blockIdx.x, (int)threadIdx.x);
                t0 = 1;
            }
        }
    }
}

// The barriers are initialised once per launch and never re-initialised: event
// k of the current task is event base + k of the barrier's lifetime (the bases
// advance by the number of steps of each finished task), which fixes its ring
// slot and phase parity.
struct SyncV4 {
    int *prog;        // [V4_GMAX] completed half-steps per WG (reset per task)
    uint64_t *barA;   // [V4_GMAX][V4_RING]: A(k) of WG g done
    uint64_t *barS;   // [V4_GMAX][V4_RING]: step k of WG g done
    uint64_t *barF;   // [2][V4_RING]: slot k filled (0: T + early W, 1: late W)
    const int *ebase; // [V4_GMAX] lifetime event base per WG
    int fbase;        // lifetime fill base
};
__device__ __forceinline__ uint64_t *ring_slot(uint64_t *ring, int K, unsigned &par)
{
    par = (unsigned)(K / V4_RING) & 1u;
    return ring + (K % V4_RING);
}

// wait until prog[g] >= need (need >= 1 half-steps).  Completion of the
// awaited event's mbarrier phase implies the counter (written before the
// arrive) has reached `need`, so a successful try_wait ends the wait; the
// try_wait result MUST be consumed -- otherwise the compiler drops the
// conditional suspend and the loop spins on shared memory, stealing issue
// slots from every working warp (ncu: 1.9e9 spin iterations in one pass).
// A ring slot that has advanced two phases (waiter far behind) makes
// try_wait time out; the counter re-check then ends the wait.
__device__ __forceinline__ void wait_prog(const SyncV4 &y, int g, int need)
{
    const int *cnt = y.prog + g;
    if (lds_volatile(cnt) < need) {
        const int k = (need - 1) >> 1; // step index of the awaited half
        unsigned par;
        uint64_t *b = ring_slot(((need & 1) ? y.barA : y.barS) + g * V4_RING, y.ebase[g] + k, par);
        unsigned long long t0 = 0;
        while (lds_volatile(cnt) < need) {
            if (mb_try_wait(b, par, 20000u)) break;
            if (BB_V4_WATCHDOG && !t0) t0 = gtimer();
            if (BB_V4_WATCHDOG && t0 != 1 && gtimer() - t0 > 2000000000ull) {
                if ((threadIdx.x & 31) == 0)
                    printf("v4 watchdog: wait_prog g %d need %d have %d block %d thread %d\n", g, need,
                           lds_volatile(cnt), (int)blockIdx.x, (int)threadIdx.x);
                t0 = 1;
            }
        }
    }
    lds_acquire(cnt);
}
// publish prog[g] = v (caller: one thread, after the WG's barrier)
__device__ __forceinline__ void post_prog(const SyncV4 &y, int g, int v)
{
    sts_release(y.prog + g, v);
    const int k = (v - 1) >> 1;
    unsigned par;
    mb_arrive(ring_slot(((v & 1) ? y.barA : y.barS) + g * V4_RING, y.ebase[g] + k, par));
}

template <class C> __device__ __forceinline__ void cp_async_elem(C *dst, const C *src);
template <> __device__ __forceinline__ void cp_async_elem<double>(double *dst, const double *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
template <> __device__ __forceinline__ void cp_async_elem<float>(float *dst, const float *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// element copy global -> shared slot (async where the storage and compute
// types agree; fp16 storage widens to fp32 through registers)
template <class S, class C> struct Fill {
    static __device__ __forceinline__ void elem(C *dst, const S *src) { cp_async_elem<C>(dst, src); }
    static constexpr bool async = true;
};
template <> struct Fill<__half, float> {
    static __device__ __forceinline__ void elem(float *dst, const __half *src) { *dst = ldg_cg(src); }
    static constexpr bool async = false;
};
// every producer thread arrives once per fill phase: on completion of its
// cp.async copies (async) or after its plain stores
template <class S, class C> __device__ __forceinline__ void fill_arrive(uint64_t *b)
{
    if (Fill<S, C>::async) mb_cp_async_arrive(b);
    else mb_arrive(b);
}

// Values stored into a slot are rounded to the storage precision, so data a
// warp-group hands to the next one in shared memory is exactly what a round
// trip through the fp16 band would give (reading Q13: fp16 storage, fp32
// arithmetic, RNE on every store) and the result does not depend on G.
template <class S, class C> struct StoreRound {
    static __device__ __forceinline__ C r(C v) { return v; }
};
template <> struct StoreRound<__half, float> {
    static __device__ __forceinline__ float r(float v) { return __half2float(__float2half_rn(v)); }
};

#define TRACE4(r_, j_, slot)                                                                                  \
    do {                                                                                                      \
        if (a.trace && mat == 0 && (r_) < a.trace_sweeps && (j_) < a.trace_steps)                             \
            a.trace[((int64_t)(r_) * a.trace_steps + (j_)) * 16 + (slot)] = gtimer();                         \
    } while (0)

// Reflector scalars from x0 = alpha and x[1..m-1] (dlarfg convention):
// beta = -sign(alpha) ||x||, tau = (beta - alpha) / beta, rho = 1 / (alpha - beta).
// Returns false when the plain sum of squares is outside the safe range; the
// caller then takes the scaled slow path.  ident: x[1:] == 0 exactly.
// Reciprocal and reciprocal square root: hardware approximation + Newton
// steps (inline, no slow-path call, so no register spills around a call).
// Arguments are in the safe range [1e-280, 1e280] (fp64) / [1e-25, 1e25]
// (fp32) by construction; results are within ~1 ulp.
template <class C> struct V4Math;
template <> struct V4Math<double> {
    static __device__ __forceinline__ double rsq(double x)
    {
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        const double hx = 0.5 * x;
        y = y * fma(-hx * y, y, 1.5);
        y = y * fma(-hx * y, y, 1.5);
        return y;
    }
    static __device__ __forceinline__ double rcp(double d)
    {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
        double e = fma(-d, r, 1.0);
        r = fma(r, e, r);
        e = fma(-d, r, 1.0);
        return fma(r, e, r);
    }
};
template <> struct V4Math<float> {
    static __device__ __forceinline__ float rsq(float x)
    {
        float y;
        asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y * fmaf(-0.5f * x * y, y, 1.5f);
    }
    static __device__ __forceinline__ float rcp(float d)
    {
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
        return fmaf(r, fmaf(-d, r, 1.0f), r);
    }
};

// Safe-range test of a sum of squares, tot in [NormRange::lo, NormRange::hi],
// as an integer compare of the bit pattern (non-negative finite values order
// like their bit patterns; NaN, inf and -0 fall outside): identical to the
// floating-point test, but an integer compare is ~5 cycles on B200 where a
// dependent fp64 compare is ~30 (tools/ubench/lat5.cu)
template <class C> struct RangeBits;
template <> struct RangeBits<double> {
    static __device__ __forceinline__ bool in(double v)
    {
        const long long b = __double_as_longlong(v);
        return b >= 0x05CD0B15A491EB84ll /* 1e-280 */ && b <= 0x7A11A0FC668AAC70ll /* 1e280 */;
    }
};
template <> struct RangeBits<float> {
    static __device__ __forceinline__ bool in(float v)
    {
        const int b = __float_as_int(v);
        return b >= 0x15F79688 /* 1e-25f */ && b <= 0x69045951 /* 1e25f */;
    }
};

template <class C>
__device__ __forceinline__ bool refl_scalars(C alpha, C ssq1, C &tau, C &rho, C &beta)
{
    const C tot = fma(alpha, alpha, ssq1);
    if (!RangeBits<C>::in(tot)) return false;
    const C rn = V4Math<C>::rsq(tot);
    const C nrm = tot * rn;
    beta = alpha >= C(0) ? -nrm : nrm;
    tau = fma(fabs(alpha), rn, C(1));
    rho = V4Math<C>::rcp(alpha - beta);
    return true;
}

// Out-of-line slow path of refl_apply (sum of squares outside the safe
// range): the same reflector from x scaled by an exact power of two 2^-e
// (e = exponent of max|x_k|), so no intermediate under/overflows.
template <class C>
__device__ __noinline__ C refl_apply_scaled(const C *xb, int xs, int m, C *av, bool has_vec)
{
    const C alpha = xb[0];
    C amax = fabs(alpha);
    for (int k = 1; k < m; ++k) amax = fmax(amax, fabs(xb[k * xs]));
    const int e = ilogb(amax);
    C ss = 0;
    for (int k = 0; k < m; ++k) {
        const C yk = scalbn(xb[k * xs], -e);
        ss = fma(yk, yk, ss);
    }
    const C ay = scalbn(alpha, -e);
    const C nrm_y = sqrt(ss);
    const C beta_y = ay >= C(0) ? -nrm_y : nrm_y;
    const C tau = C(1) + fabs(ay) / nrm_y;
    const C rd = C(1) / (ay - beta_y); // |ay - beta_y| >= nrm_y >= 1
    if (has_vec) {
        C sd = av[0];
        for (int k = 1; k < m; ++k) sd = fma(av[k], scalbn(xb[k * xs], -e) * rd, sd);
        const C w = tau * sd;
        av[0] -= w;
        for (int k = 1; k < m; ++k) av[k] = fma(-w, scalbn(xb[k * xs], -e) * rd, av[k]);
    }
    return scalbn(beta_y, e);
}

// Apply the reflector of the source vector x (shared memory, xb[k*xs],
// length m; FULL: m == MT) to the register vector av: av -= tau (v . av) v,
// v_0 = 1, v_k = rho x_k (LAPACK dlarfg reflector, readings Q7/Q8).  The dot
// product is taken against x while the norm accumulates, and every caller
// computes the scalars from the same x in the same order, so all threads
// agree bitwise.  x is re-read for the update (keeps the register peak at
// one vector).  Sum of squares outside the safe range: the same reflector
// from x scaled by an exact power of two 2^-e (e = exponent of max|x_k|), so
// no intermediate under/overflows.  Returns beta.
template <class C, int MT, bool FULL, int xs>
__device__ __forceinline__ C refl_apply(const C *xb, int m, C (&av)[MT], bool has_vec)
{
    C q4[4] = {0, 0, 0, 0}, s4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 1; k < MT; ++k) {
        if (FULL || k < m) {
            const C xk = xb[k * xs];
            q4[k & 3] = fma(xk, xk, q4[k & 3]);
            s4[k & 3] = fma(av[k], xk, s4[k & 3]);
        }
    }
    const C alpha = xb[0];
    const C ssq1 = (q4[0] + q4[1]) + (q4[2] + q4[3]);
    // identity iff x[1:] == 0 exactly (reading Q8): decided from the sum of
    // squares (one compare instead of a chain of m dependent fp compares);
    // only a zero sum (every square underflowed, or x[1:] == 0) looks at x
    bool nz = ssq1 > C(0);
    if (!nz) {
        for (int k = 1; k < m; ++k) nz |= (xb[k * xs] != C(0));
    }
    if (!nz) return alpha; // identity: nothing to annihilate
    C tau, rho, beta;
    asm volatile("" ::: "memory"); // re-read x below (register peak)
    if (refl_scalars<C>(alpha, ssq1, tau, rho, beta)) {
        if (has_vec) {
            const C w = tau * fma(rho, (s4[0] + s4[1]) + (s4[2] + s4[3]), av[0]);
            const C wr = w * rho;
            av[0] -= w;
#pragma unroll
            for (int k = 1; k < MT; ++k)
                if (FULL || k < m) av[k] = fma(-wr, xb[k * xs], av[k]);
        }
        return beta;
    }
    // scaled slow path (out of line: keeps the hot code small for the I-cache)
    C tmp[MT];
#pragma unroll
    for (int k = 0; k < MT; ++k) tmp[k] = av[k];
    beta = refl_apply_scaled<C>(xb, xs, m, tmp, has_vec);
#pragma unroll
    for (int k = 0; k < MT; ++k) av[k] = tmp[k];
    return beta;
}

struct GeoV4 {
    int p0, q0, trow0, p, q, hi, ce, m;
};
__device__ __forceinline__ GeoV4 geo_v4(int n, int c, int t, int G, int r0, int g, int j)
{
    GeoV4 s;
    s.p0 = r0 + (c - t) + j * c;
    s.q0 = j ? s.p0 - c : r0;
    s.trow0 = j ? s.q0 + t + G : r0;
    s.p = s.p0 + g;
    s.q = s.q0 + g;
    s.hi = min(s.p + t, n - 1);
    s.ce = min(s.hi + c, n - 1);
    s.m = s.hi - s.p + 1;
    return s;
}

// Visit the cells (row, col) of a rectangle rows [i0, i0+nr) x cols [c0, c0+nc)
// that lie in the matrix and in the band offsets [-t, c+t], distributing the
// elements over nthr threads, consecutive threads on consecutive rows of a
// column (coalesced in the column-major band).
template <class F>
__device__ __forceinline__ void for_rect(int i0, int nr, int c0, int nc, int n, int lo_off, int hi_off, int tid,
                                         int nthr, F &&f)
{
    const int tot = nr * nc;
    if (nr <= 0 || nc <= 0) return;
    int e = tid;
    int k = e / nr, ii = e - k * nr;
    const int dk = nthr / nr, dii = nthr - dk * nr;
    for (; e < tot; e += nthr) {
        const int i = i0 + ii, jc = c0 + k;
        const int off = jc - i;
        if (i < n && jc < n && off >= lo_off && off <= hi_off) f(ii, k, i, jc);
        ii += dii;
        k += dk;
        if (ii >= nr) {
            ii -= nr;
            ++k;
        }
    }
}

// One step (r0 + g, j) of a compute WG.  FULL: m == MT.
// Shared-memory layout of a slot (compute type C), pitch TP (odd, >= t + G;
// (MT | 1) + 8 by default, (MT | 1) + 2 for fp64 t >= 31, a compile-time pitch so every hot loop addresses
// shared memory as base + immediate):
//   T: ROW-major,    row i - trow0 (LDT = c + G rows), element jc - p0 (< WT)
//   W: COLUMN-major, column jc - p0 - WT (c columns),  element i - p0 (< WT)
// A right-application row is contiguous in T (stride 1) or strided by TP in
// the previous slot's W; a left-application column is strided by TP in T or
// contiguous in W.  Odd TP keeps both thread-per-row and thread-per-column
// accesses bank-conflict free.
// default pitch (room for G <= 8); the host may pick a tighter odd pitch >= t + G
template <int MT> struct TPitch {
    static constexpr int value = (MT | 1) + 8;
};

template <int ST, class C, int MT, bool FULL>
__device__ __forceinline__ void ld_vec(const C *b, int m, C (&v)[MT])
{
#pragma unroll
    for (int k = 0; k < MT; ++k)
        if (FULL || k < m) v[k] = b[k * ST];
}
template <int ST, class S, class C, int MT, bool FULL>
__device__ __forceinline__ void st_vec(C *b, int m, const C (&v)[MT])
{
#pragma unroll
    for (int k = 0; k < MT; ++k)
        if (FULL || k < m) b[k * ST] = StoreRound<S, C>::r(v[k]);
}

// global progress wait of the producer (relaxed polling, acquire fence)
__device__ __forceinline__ void wait_geq_v4(const int *p, int need, int dbg_tag, const int *prog_s = nullptr,
                                            int r0 = 0, int glast = 0)
{
    int v = ld_relaxed(p);
    if (v < need) {
        const unsigned long long t0 = BB_V4_WATCHDOG ? gtimer() : 0ull;
        while (v < need) {
            __nanosleep(poll_ns(v, need, 4)); // far behind (> 2 steps): sleep ~1 us
            v = ld_relaxed(p);
            if (BB_V4_WATCHDOG && gtimer() - t0 > 2000000000ull) {
                printf("v4 watchdog: global wait need %d have %d tag %d block %d r0 %d glast %d prog %d %d %d\n", need,
                       v, dbg_tag, (int)blockIdx.x, r0, glast, prog_s ? prog_s[0] : -1,
                       prog_s ? prog_s[1] : -1, prog_s ? prog_s[2] : -1);
                while (ld_relaxed(p) < need) __nanosleep(1000);
                break;
            }
        }
    }
    (void)ld_acquire(p); // acquire (no full fence: the producer has no stores to drain)
}

template <class S, int MT, int TP, bool FULL, bool JP>
__device__ __forceinline__ void step_v4(const PassArgsV4 &a, S *Wg, int mat, int r0, int g, int j, int Jprev,
                                        bool closer, bool own_next, const SyncV4 &y,
                                        typename ComputeOf<S>::type *slots, int tid, int bar)
{
    using C = typename ComputeOf<S>::type;
    const int n = a.n, c = a.c, t = a.t, G = a.G, NT = a.NT;
    const int WT = t + G;
    const int ku = a.ku;
    const int64_t ldw = a.ldw;
    const int lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
    const GeoV4 s = geo_v4(n, c, t, G, r0, g, j);
    const int m = FULL ? MT : s.m;
    const int r = r0 + g;
    C *curT = slots + (size_t)(j % a.NS) * a.slot_elems;
    C *curW = curT + a.LDT * TP;
    C *prvW = slots + (size_t)((j + a.NS - 1) % a.NS) * a.slot_elems + a.LDT * TP;
    const bool jp = JP || j > 0; // JP: the hot instantiation (full step, j > 0)
    // home of cell (i, jc), jc in [p0, p0 + WT): previous slot's W (rows < trow0) or T
    auto tcell = [&](int i, int jc) -> C * {
        if (jp && i < s.trow0) return prvW + (jc - s.q0 - WT) * TP + (i - s.q0);
        return curT + (i - s.trow0) * TP + (jc - s.p0);
    };

    // ---------------------------------------------------------------- A wait
    // one warp waits (hardware-suspended try_wait), the others block on the
    // WG barrier: waiting warps must not steal issue slots from working ones
    if (warp == 0) {
        if (g == 0) {
            unsigned par;
            uint64_t *b = ring_slot(y.barF, y.fbase + j, par);
            mb_wait(b, par);
        } else {
            wait_prog(y, g - 1, min(2 * j + a.a0, 2 * Jprev));
        }
    }
    nbar_sync(bar, NT);
    if (tid == 0) TRACE4(r, j, 0);

    // ---------------------------------------------------------------- right application
    // x = A[q][p..hi] (row reflector source): in the previous slot's W
    // (stride TP) for j > 0, in T (stride 1) for j == 0; rows q+1..hi
    C *xb = tcell(s.q, s.p);
    const int nR = s.hi - s.q;
    C beta1;
    {
        C av[MT];
        C *rb = nullptr;
        const bool mine = tid < nR;
        const int i = s.q + 1 + tid;
        const bool rprev = jp && i < s.trow0;
        if (mine) {
            rb = tcell(i, s.p);
            if (rprev) ld_vec<TP, C, MT, FULL>(rb, m, av);
            else ld_vec<1, C, MT, FULL>(rb, m, av);
        } else {
#pragma unroll
            for (int k = 0; k < MT; ++k) av[k] = C(0);
        }
        if (JP) beta1 = refl_apply<C, MT, FULL, TP>(xb, m, av, mine);
        else beta1 = jp ? refl_apply<C, MT, FULL, TP>(xb, m, av, mine) : refl_apply<C, MT, FULL, 1>(xb, m, av, mine);
        if (mine) {
            if (rprev) st_vec<TP, S, C, MT, FULL>(rb, m, av);
            else st_vec<1, S, C, MT, FULL>(rb, m, av);
            if (G == 1) {
                // one sweep per CTA: the union is this step's window, so write the
                // row through from registers (coalesced across the WG for each k)
                S *grow = Wg + (ku + i) + (int64_t)s.p * (ldw - 1);
#pragma unroll
                for (int k = 0; k < MT; ++k)
                    if (FULL || k < m) stg(grow + (int64_t)k * (ldw - 1), av[k]);
            }
        }
    }
    nbar_sync(bar, NT);
    beta1 = StoreRound<S, C>::r(beta1);
    if (tid == 0) {
        // x row -> (beta, 0, ..., 0): exact zeros in the annihilated slots
        const int xs = jp ? TP : 1;
        xb[0] = beta1;
        for (int k = 1; k < m; ++k) xb[k * xs] = C(0);
        if (G == 1) {
            S *gx = Wg + (ku + s.q) + (int64_t)s.p * (ldw - 1);
            for (int k = 0; k < m; ++k) stg(gx + (int64_t)k * (ldw - 1), k == 0 ? beta1 : C(0));
        }
        TRACE4(r, j, 1);
    }
    if (closer && G > 1) {
        // A write-back of the union's right-application region: rows
        // [q0, p0 + WT) x cols [p0, p0 + WT), band offsets [-t, c + t]; one
        // warp per column (coalesced).  This WG's own x row is taken from
        // registers (tid 0 writes it to shared memory concurrently).
        for (int k = warp; k < WT; k += nwarps) {
            const int jc = s.p0 + k;
            if (jc >= n) break;
            const int rlo = max(s.q0, jc - c - t), rhi = min(min(s.p0 + WT - 1, jc + t), n - 1);
            S *gcol = Wg + (ku - jc) + (int64_t)jc * ldw;
            for (int i = rlo + lane; i <= rhi; i += 32) {
                // this WG's own x row is being rewritten by tid 0: take it from beta1
                // without reading the cell (no read-write race on shared memory)
                const bool xrow = i == s.q && jc >= s.p && jc <= s.hi;
                const C v = xrow ? ((jc == s.p) ? beta1 : C(0)) : *tcell(i, jc);
                stg(gcol + i, v);
            }
        }
        nbar_sync(bar, NT);
    }
    if (tid == 0) {
        post_prog(y, g, 2 * j + 1);
        TRACE4(r, j, 2);
    }

    // ---------------------------------------------------------------- B wait
    if (warp == 0) {
        if (g == 0) {
            unsigned par;
            uint64_t *b = ring_slot(y.barF + V4_RING, y.fbase + j, par);
            mb_wait(b, par);
        } else {
            wait_prog(y, g - 1, min(2 * j + a.b0, 2 * Jprev));
        }
    }
    nbar_sync(bar, NT);
    if (tid == 0) TRACE4(r, j, 3);

    // ---------------------------------------------------------------- left application
    // y = A[p..hi][p] (column reflector source), in T (stride TP);
    // columns p+1..ce: in T (stride TP) below p0 + WT, else in W (stride 1)
    C *yb = curT + (s.p - s.trow0) * TP + (s.p - s.p0);
    const int nL = s.ce - s.p;
    C beta2;
    {
        C bv[MT];
        C *cb = nullptr;
        const bool mine = tid < nL;
        const int jc = s.p + 1 + tid;
        const bool inT = jc < s.p0 + WT;
        if (mine) {
            if (inT) {
                cb = curT + (s.p - s.trow0) * TP + (jc - s.p0);
                ld_vec<TP, C, MT, FULL>(cb, m, bv);
            } else {
                cb = curW + (jc - s.p0 - WT) * TP + (s.p - s.p0);
                ld_vec<1, C, MT, FULL>(cb, m, bv);
            }
        } else {
#pragma unroll
            for (int k = 0; k < MT; ++k) bv[k] = C(0);
        }
        beta2 = refl_apply<C, MT, FULL, TP>(yb, m, bv, mine);
        if (mine) {
            if (inT) st_vec<TP, S, C, MT, FULL>(cb, m, bv);
            else st_vec<1, S, C, MT, FULL>(cb, m, bv);
        }
    }
    nbar_sync(bar, NT);
    beta2 = StoreRound<S, C>::r(beta2);
    if (tid == 0) {
        yb[0] = beta2;
        for (int k = 1; k < m; ++k) yb[k * TP] = C(0);
        TRACE4(r, j, 4);
    }
    if (closer) {
        // B write-back of the union's left-application region: rows
        // [p0, p0 + WT) x cols [p0, p0 + WT + c).  Columns >= p0 + c are the
        // top rows of step j+1's right-application region: when this WG has a
        // step j+1 its A write-back there (program order) covers them;
        // otherwise every other WG's A(j+1) write-back happened before (chain)
        // and this copy is the last one.  Own y column from registers.
        // flattened over the WG: every lane busy (one warp per 19-row column
        // segment was measured 3x slower, tools/ubench/wbfill.cu)
        const int ncol = own_next ? c : WT + c;
        const int tot = WT * ncol, dk = NT / WT, dii = NT - dk * WT;
        int k = tid / WT, ii = tid - k * WT;
        for (int e = tid; e < tot; e += NT) {
            const int i = s.p0 + ii, jc = s.p0 + k, off = jc - i;
            if (i < n && jc < n && off >= -t && off <= c + t) {
                const bool ycol = jc == s.p && i >= s.p && i <= s.hi; // own y column: from beta2
                const C v = ycol ? ((i == s.p) ? beta2 : C(0))
                                 : (k < WT ? curT[(i - s.trow0) * TP + k] : curW[(k - WT) * TP + ii]);
                stg(Wg + (ku + i) + (int64_t)jc * (ldw - 1), v);
            }
            ii += dii;
            k += dk;
            if (ii >= WT) {
                ii -= WT;
                ++k;
            }
        }
        nbar_sync(bar, NT);
    }
    if (tid == 0) {
        post_prog(y, g, 2 * j + 2);
        TRACE4(r, j, 5);
    }
}

// Clipped steps at the matrix end (m < MT) and every sweep's first step
// (j = 0, x in T): out of line, so the hot code (one full step with j > 0)
// stays small enough for the instruction cache.
template <class S, int MT, int TP>
__device__ __noinline__ void step_v4_tail(const PassArgsV4 &a, S *Wg, int mat, int r0, int g, int j, int Jprev,
                                          bool closer, bool own_next, const SyncV4 &y,
                                          typename ComputeOf<S>::type *slots, int tid, int bar)
{
    step_v4<S, MT, TP, false, false>(a, Wg, mat, r0, g, j, Jprev, closer, own_next, y, slots, tid, bar);
}

// G compute WGs of NT threads, a.pw producer warps, one release warp.
template <class S, int MT, int NTMAX, int TP>
__global__ void __launch_bounds__(NTMAX, 1) pass_v4_kernel(PassArgsV4 a)
{
    using C = typename ComputeOf<S>::type;
    static_assert(TP % 2 == 1 && TP >= MT, "slot pitch: odd, >= t + G");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *slots = reinterpret_cast<C *>(smem_raw);
    __shared__ int s_task;
    __shared__ int prog_s[V4_GMAX];
    __shared__ __align__(8) uint64_t bars[(2 * V4_GMAX + 2) * V4_RING];
    __shared__ int ebase_s[V4_GMAX];
    __shared__ int fbase_s;
    constexpr int NBAR = (2 * V4_GMAX + 2) * V4_RING;

    const int G = a.G, NT = a.NT;
    const int n = a.n, c = a.c, t = a.t;
    const int WT = t + G;
    const int ncomp = G * NT;
    const int npt = 32 * a.pw;
    const int total = a.batch * a.ngroups;
    for (int i = threadIdx.x; i < NBAR; i += blockDim.x)
        mb_init(bars + i, i >= 2 * V4_GMAX * V4_RING ? (unsigned)npt : 1u);
    fence_mbarrier_init();
    if (threadIdx.x < V4_GMAX) ebase_s[threadIdx.x] = 0;
    if (threadIdx.x == 0) fbase_s = 0;
    int prev_r0 = -1;

    for (;;) {
        __syncthreads(); // the previous task is complete
        if (threadIdx.x == 0) s_task = atomicAdd(a.counter, 1);
        if (threadIdx.x < V4_GMAX) {
            prog_s[threadIdx.x] = 0;
            // every event of the previous task was consumed: advance the lifetime bases
            if (prev_r0 >= 0 && prev_r0 + (int)threadIdx.x < a.nsweeps)
                ebase_s[threadIdx.x] += sweep_len(n, c, t, prev_r0 + threadIdx.x);
        }
        if (threadIdx.x == 0 && prev_r0 >= 0) fbase_s += sweep_len(n, c, t, prev_r0);
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int r0 = (task / a.batch) * G;
        prev_r0 = r0;
        const int glast = min(G, a.nsweeps - r0) - 1;
        const SyncV4 y{prog_s, bars, bars + V4_GMAX * V4_RING, bars + 2 * V4_GMAX * V4_RING, ebase_s, fbase_s};
        if (BB_V4_WATCHDOG > 1 && threadIdx.x == 0) printf("task %d block %d r0 %d\n", task, (int)blockIdx.x, r0);
        int *gprog = a.progress + (int64_t)mat * n;
        S *Wg = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;

        if ((int)threadIdx.x < ncomp) {
            // ------------------------------------------------ compute warp-groups
            const int g = threadIdx.x / NT;
            const int tid = threadIdx.x - g * NT;
            if (g <= glast) {
                const int r = r0 + g;
                const int J = sweep_len(n, c, t, r);
                const int Jprev = g > 0 ? sweep_len(n, c, t, r - 1) : 0;
                const int Jnext = g < glast ? sweep_len(n, c, t, r + 1) : 0;
                for (int j = 0; j < J; ++j) {
                    const bool closer = (g == glast) || (j >= Jnext);
                    const bool own_next = j + 1 < J;
                    const int p = r + (c - t) + j * c;
                    if (j > 0 && min(p + t, n - 1) - p + 1 == MT)
                        step_v4<S, MT, TP, true, true>(a, Wg, mat, r0, g, j, Jprev, closer, own_next, y, slots, tid, 1 + g);
                    else
                        step_v4_tail<S, MT, TP>(a, Wg, mat, r0, g, j, Jprev, closer, own_next, y, slots, tid, 1 + g);
                }
            }
        } else if ((int)threadIdx.x < ncomp + npt) {
            // ------------------------------------------------ PRODUCER warps: fill slot j for the group
            const int ptid = threadIdx.x - ncomp;
            const int pbar = 1 + V4_GMAX; // named barrier of the producer warps
            const int J0 = sweep_len(n, c, t, r0);
            const int Jp = r0 > 0 ? sweep_len(n, c, t, r0 - 1) : 0;
            const int *pprev = r0 > 0 ? gprog + (r0 - 1) : nullptr;
            // first late W column index: the columns the previous group's phase
            // awaited by B (and not by A) can still modify.  Refined rule (b0 = 3):
            // its A(j+1), cols >= p0 + c - G; b0 = 4 (target bandwidth 2..3, G = 1):
            // its step j+1, cols >= p0 + c - 1; b0 = 5 (target bandwidth 1, G = 1):
            // its A(j+2), cols >= p0 + 2c - 1.  Equal waits: no late part.
            const int kLate = (a.b0 == a.a0) ? c : (a.b0 == 5 ? 2 * c - 1 - WT : c - t - 2 * G);
            const int ku = a.ku;
            const int64_t ldw = a.ldw;
            // flattened copy of rows [i0, i0+nr) x cols [c0, c0+nc) (band offsets
            // [-t, c+t], inside the matrix) to dst[ii*drs + k*dcs]: consecutive
            // threads on consecutive rows (coalesced), every lane busy
            auto fill_rect = [&](int i0, int nr, int c0, int nc, C *dst, int drs, int dcs) {
                if (nr <= 0 || nc <= 0) return;
                const int tot = nr * nc, dk = npt / nr, dii = npt - dk * nr;
                int k = ptid / nr, ii = ptid - k * nr;
                if (Fill<S, C>::async) {
                    for (int e = ptid; e < tot; e += npt) {
                        const int i = i0 + ii, jc = c0 + k, off = jc - i;
                        if (i < n && jc < n && off >= -t && off <= c + t)
                            Fill<S, C>::elem(dst + ii * drs + k * dcs, Wg + (ku + i) + (int64_t)jc * (ldw - 1));
                        ii += dii;
                        k += dk;
                        if (ii >= nr) {
                            ii -= nr;
                            ++k;
                        }
                    }
                } else {
                    // fp16 storage (widened to fp32 through registers): batches of 8
                    // loads in flight, then their shared-memory stores
                    constexpr int U = 8;
                    for (int e = ptid; e < tot; e += U * npt) {
                        C v[U];
                        int so[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            so[u] = -1;
                            const int i = i0 + ii, jc = c0 + k, off = jc - i;
                            if (e + u * npt < tot && i < n && jc < n && off >= -t && off <= c + t) {
                                v[u] = ldg_cg(Wg + (ku + i) + (int64_t)jc * (ldw - 1));
                                so[u] = ii * drs + k * dcs;
                            }
                            ii += dii;
                            k += dk;
                            if (ii >= nr) {
                                ii -= nr;
                                ++k;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (so[u] >= 0) dst[so[u]] = v[u];
                    }
                }
            };
            for (int j = 0; j < J0; ++j) {
                const GeoV4 s = geo_v4(n, c, t, G, r0, 0, j);
                C *curT = slots + (size_t)(j % a.NS) * a.slot_elems;
                C *curW = curT + a.LDT * TP;
                unsigned par;
                uint64_t *fA = ring_slot(y.barF, y.fbase + j, par), *fB = ring_slot(y.barF + V4_RING, y.fbase + j, par);
                if (ptid == 0) {
                    // slot reuse: every WG finished A(j - NS + 1) (the last reader of slot j - NS)
                    if (j >= a.NS)
                        for (int g = 0; g <= glast; ++g)
                            wait_prog(y, g, min(2 * (j - a.NS + 1) + 1, 2 * sweep_len(n, c, t, r0 + g)));
                    if (pprev) wait_geq_v4(pprev, min(2 * j + a.a0, 2 * Jp), 2 * j, prog_s, r0, glast);
                    TRACE4(r0, j, 6);
                }
                nbar_sync(pbar, npt);
                // T part first (all WG 0's A phase needs): rows [trow0, p0 + WT) x
                // cols [p0, p0 + WT), row-major in shared memory
                fill_rect(s.trow0, s.p0 + WT - s.trow0, s.p0, WT, curT, TP, 1);
                fill_arrive<S, C>(fA); // completes when every producer thread's copies landed
                if (ptid == 0) TRACE4(r0, j, 7);
                // early W columns [p0 + WT, p0 + WT + kLate): only needed by B phases
                fill_rect(s.p0, WT, s.p0 + WT, kLate, curW, 1, TP);
                if (pprev && a.b0 > a.a0) {
                    if (ptid == 0) wait_geq_v4(pprev, min(2 * j + a.b0, 2 * Jp), 2 * j + 1, prog_s, r0, glast);
                    nbar_sync(pbar, npt);
                }
                if (ptid == 0) TRACE4(r0, j, 8);
                fill_rect(s.p0, WT, s.p0 + WT + kLate, c - kLate, curW + kLate * TP, 1, TP);
                fill_arrive<S, C>(fB);
                if (ptid == 0) TRACE4(r0, j, 9);
            }
            if (Fill<S, C>::async) cp_async_wait_all();
        } else if ((threadIdx.x & 31) == 0) {
            // ------------------------------------------------ RELEASE warp (lane 0)
            // republish the group's last sweep's progress at gpu scope; the
            // final value waits until every WG of the group finished.
            const int rl = r0 + glast;
            const int target = 2 * sweep_len(n, c, t, rl);
            int published = 0;
            while (published < target) {
                wait_prog(y, glast, published + 1);
                int v = lds_volatile(y.prog + glast);
                if (v >= target) {
                    for (int g = 0; g < glast; ++g) wait_prog(y, g, 2 * sweep_len(n, c, t, r0 + g));
                    v = target;
                }
                fence_acq_rel();
                asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(gprog + rl), "r"(v) : "memory");
                published = v;
            }
        }
    }
}

} // namespace bb
