// bb_pass_v5.cuh -- blocked "unit" pass kernel for passes whose target
// bandwidth c - t is at least G >= 2 (sm_100a).
//
// A pass (Alg. 1) is a chain of ~n sweeps, sweep r+1 following
// sweep r through the band.  Round 1 ran one sweep per
// warp-group and paid a hand-off (the "cycle" of P:145) per sweep.  This
// kernel gives one CTA a GROUP of G consecutive sweeps r0 .. r0+G-1 and
// advances them together, one UNIT (step j of all G sweeps) at a time:
//
//   A half: the G row reflectors of step j, g = 0..G-1 (Alg. 2 lines 5-13)
//   B half: the G column reflectors of step j, g = 0..G-1 (lines 15-20)
//
// The oracle runs A_0 B_0 A_1 B_1 ... and finishes sweep r0 before sweep
// r0+1 starts.  The unit order only swaps pairs that commute EXACTLY:
//   * A_g(j) and B_g'(j), g' < g: B_g' touches rows [p+g', p+g'+t] only, A_g
//     columns [p+g, p+g+t] only; neither touches the other's reflector source
//     (row q_g = p-c+g, column p+g'), and each one's range covers the other's
//     output inside the overlap -- so H_L (A H_R) = (H_L A) H_R;
//   * B_g(j) and A_g'(j+1), g > g' (same argument one step further);
// and it requires G <= c - t so that no NON-commuting pair (two right or two
// left reflectors of different units on shared rows/columns) is reordered.
// The result is therefore the same orthogonal equivalence in exact
// arithmetic (reading Q20); tools/v5_proto.py checks it in fp64.
//
// With the G reflectors of a half known one after another, each half is
//   PANEL  (warp 0): the chain -- reflector g is generated from the panel
//          row/column g after reflectors 0..g-1 were applied to it (LQ / QR
//          of a G x (t+G) staircase), v_g and tau_g go to shared memory;
//   BULK   (all threads): every other row (A) / column (B) of the window is
//          held in registers and receives the G reflectors in chunks of U,
//          so shared memory is read and written once per U reflectors, not
//          once per reflector (P:175-180's "rows in registers", widened).
//
// Window of unit j (p = r0 + (c-t) + j*c, q0 = r0 for j = 0 else p - c,
// dq = p - q0, W = t + G), compute type C, column-major in shared memory:
//   Win[(x-p)*LA + (i-q0)]   cols [p, p+W)      rows [q0, p+W)   (V region)
//   Hr [(x-p-W)*LB + (i-p)]  cols [p+W, p+W+c)  rows [p, p+W)    (rest of H)
// Only cells inside the matrix with band offset x - i in [-t, c+t] (the fill
// bound, reading Q11) are loaded or written back; the others are zero.
// The H-region columns [p+c, p+c+W) rows [p, p+W) are the next unit's V rows
// [q0', q0'+W): they stay in shared memory (CARRY) and are not re-read.
//
// Global memory protocol per unit (half-units published in progress[k]):
//   wait progress[k-1] >= 2j+a0;  load V rows ([q0+W, p+W) for j > 0)
//   A half; write back rows [q0, p) of the V region; publish 2j+1
//   wait progress[k-1] >= 2j+b0;  load Hr
//   B half; write back rows [p, p+W) x cols [p, p+c) (last unit: all);
//   publish 2j+2; carry.
// (a0, b0) are chosen on the host by an exact hazard search over these
// rectangles (tools/v5_rules.py; bb_api.cu v5_rule()).
#pragma once

#include "bb_pass_v4.cuh"

#include <type_traits>

namespace bb {

struct PassArgsV5 {
    void *W;
    int64_t mat_stride;
    int ldw, ku, n;
    int c, t, G;
    int a0, b0, b0t; // B wait 2j + b0, or 2j + b0t while the predecessor's unit j+1 is its last
    int batch, nsweeps, ngroups;
    int *progress; // [batch][ngroups] x fstride, half-units
    int fstride;   // ints between consecutive group flags
    int *counter;
    int LA, LB; // shared pitches (odd, in elements of C)
    unsigned long long *trace;
    int trace_groups, trace_units;
};

// Reflector scalars by the scaled slow path (sum of squares outside the safe
// range): x scaled by the exact power of two 2^-e, e = exponent of max|x_k|,
// so no intermediate under/overflows (reading Q8).  Returns tau,
// beta, e and rd = 1 / (alpha' - beta') in the scaled domain; the caller forms
// v_k = (x_k 2^-e) rd directly -- 1 / (alpha - beta) itself can overflow when
// x is denormal-scale (fp32).
template <class C>
__device__ __noinline__ void v5_scalars_scaled(const C *xb, int xs, int m, C &tau, C &beta, int &e, C &rd)
{
    C amax = 0;
    for (int k = 0; k < m; ++k) amax = fmax(amax, fabs(xb[k * xs]));
    e = ilogb(amax);
    C ss = 0;
    for (int k = 0; k < m; ++k) {
        const C yk = scalbn(xb[k * xs], -e);
        ss = fma(yk, yk, ss);
    }
    const C ay = scalbn(xb[0], -e);
    const C nrm_y = sqrt(ss);
    const C beta_y = ay >= C(0) ? -nrm_y : nrm_y;
    tau = C(1) + fabs(ay) / nrm_y;
    rd = C(1) / (ay - beta_y); // |ay - beta_y| >= nrm_y >= 1
    beta = scalbn(beta_y, e);
}

// One panel link: x = source (shared, stride xs), m = MT (cells outside the
// matrix are zero, which leaves the reflector unchanged).  Every lane
// computes the scalars redundantly from the same x in the same order.  On
// return v_k = rho * x[k] for k >= 1 (the slow path stores v_k in x[k] and
// sets rho = 1).
template <class C, int MT>
__device__ __forceinline__ void v5_link_scalars(const C *xb, int xs, C (&x)[MT], C &tau, C &rho, C &beta, bool &ident)
{
    C q4[4] = {0, 0, 0, 0};
    bool nz = false;
#pragma unroll
    for (int k = 0; k < MT; ++k) x[k] = xb[k * xs];
#pragma unroll
    for (int k = 1; k < MT; ++k) {
        nz |= (x[k] != C(0));
        q4[k & 3] = fma(x[k], x[k], q4[k & 3]);
    }
    ident = !nz;
    const C alpha = x[0];
    if (ident) {
        tau = 0;
        rho = 0;
        beta = alpha;
        return;
    }
    if (!refl_scalars<C>(alpha, (q4[0] + q4[1]) + (q4[2] + q4[3]), tau, rho, beta)) {
        int e;
        C rd;
        v5_scalars_scaled<C>(xb, xs, MT, tau, beta, e, rd);
#pragma unroll
        for (int k = 1; k < MT; ++k) x[k] = scalbn(x[k], -e) * rd;
        rho = C(1);
    }
}

// Flattened masked copy global -> shared of rows [i0, i0+nr) x cols [x0, x0+nc)
// into s[(x-x0)*ls + (i-i0)]; cells outside the matrix / band offsets
// [-t, c+t] are zero.  Consecutive threads on consecutive rows (coalesced).
// Storage = compute type (fp32, fp64): cp.async with zero-fill, every copy in
// flight at once (one L2 round trip; caller waits with v5_load_wait).  fp16
// storage widens through registers (batches of 4 loads in flight).
template <class C> __device__ __forceinline__ void v5_cp_async(C *dst, const C *src, bool valid);
template <> __device__ __forceinline__ void v5_cp_async<double>(double *dst, const double *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}
template <> __device__ __forceinline__ void v5_cp_async<float>(float *dst, const float *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void v5_load_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <class S, class C>
__device__ __forceinline__ void v5_load(const S *__restrict__ Wg, int ku, int64_t ldw1, int n, int c, int t, int i0,
                                        int nr, int x0, int nc, C *__restrict__ s, int ls, int tid, int nthr)
{
    const int tot = nr * nc;
    if (nr <= 0 || nc <= 0) return;
    int e = tid;
    int k = e / nr, ii = e - k * nr;
    const int dk = nthr / nr, dii = nthr - dk * nr;
    if constexpr (std::is_same<S, C>::value) {
        for (; e < tot; e += nthr) {
            const int i = i0 + ii, x = x0 + k, off = x - i;
            const bool ok = i < n && x < n && off >= -t && off <= c + t;
            v5_cp_async<C>(s + k * ls + ii, ok ? Wg + (ku + i) + (int64_t)x * ldw1 : Wg, ok);
            ii += dii;
            k += dk;
            if (ii >= nr) {
                ii -= nr;
                ++k;
            }
        }
    } else {
        constexpr int UL = 4;
        while (e < tot) {
            C buf[UL];
            int so[UL];
#pragma unroll
            for (int u = 0; u < UL; ++u) {
                so[u] = -1;
                if (e < tot) {
                    const int i = i0 + ii, x = x0 + k, off = x - i;
                    so[u] = k * ls + ii;
                    buf[u] = (i < n && x < n && off >= -t && off <= c + t)
                                 ? ldg_cg(Wg + (ku + i) + (int64_t)x * ldw1)
                                 : C(0);
                }
                e += nthr;
                ii += dii;
                k += dk;
                if (ii >= nr) {
                    ii -= nr;
                    ++k;
                }
            }
#pragma unroll
            for (int u = 0; u < UL; ++u)
                if (so[u] >= 0) s[so[u]] = buf[u];
        }
    }
}

template <class S, class C>
__device__ __forceinline__ void v5_store(S *__restrict__ Wg, int ku, int64_t ldw1, int n, int c, int t, int i0, int nr,
                                         int x0, int nc, const C *__restrict__ s, int ls, int tid, int nthr)
{
    const int tot = nr * nc;
    if (nr <= 0 || nc <= 0) return;
    int e = tid;
    int k = e / nr, ii = e - k * nr;
    const int dk = nthr / nr, dii = nthr - dk * nr;
    for (; e < tot; e += nthr) {
        const int i = i0 + ii, x = x0 + k, off = x - i;
        if (i < n && x < n && off >= -t && off <= c + t) stg(Wg + (ku + i) + (int64_t)x * ldw1, s[k * ls + ii]);
        ii += dii;
        k += dk;
        if (ii >= nr) {
            ii -= nr;
            ++k;
        }
    }
}

// Apply the G reflectors (v_g = vs + g*VP, tau_g = v_g[MT]) to one register
// vector: element k of the vector is base[k*es] (k < G - 1 + MT); reflector g
// acts on elements [g, g + MT) and is skipped (tau := 0) when g < gfirst
// (the vector lies outside that reflector's application range, Q10/Q12).
// Chunks of U reflectors: load MT + U - 1 elements, apply U reflectors with
// static register indices, store them back.
template <class C, int MT, int U>
__device__ __forceinline__ void v5_apply(C *base, int es, int G, int gfirst, const C *__restrict__ vs, int VP)
{
#pragma unroll 1
    for (int g0 = 0; g0 < G; g0 += U) {
        C r[MT + U - 1];
#pragma unroll
        for (int k = 0; k < MT + U - 1; ++k) r[k] = base[(g0 + k) * es];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            // keep one reflector's v in registers at a time (register pressure)
            asm volatile("" ::: "memory");
            const int g = g0 + u;
            const C *v = vs + g * VP;
            const C tau = (g >= gfirst) ? v[MT] : C(0);
            C s4[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < MT; ++k) s4[k & 3] = fma(r[u + k], v[k], s4[k & 3]);
            const C w = tau * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
#pragma unroll
            for (int k = 0; k < MT; ++k) r[u + k] = fma(-w, v[k], r[u + k]);
        }
#pragma unroll
        for (int k = 0; k < MT + U - 1; ++k) base[(g0 + k) * es] = r[k];
    }
}

// Scaled slow path of a panel link (sum of squares outside the safe range),
// executed by one lane: writes v (v[0] = 1, v[k] = (x_k 2^-e) rd) and tau
// to v[0..MT], returns beta (readings Q7/Q8).  Out of line: it
// is rare and its scalbn code would bloat the hot loop.
template <class C>
__device__ __noinline__ C v5_slow_link(const C *src, int ks, int m, C *v)
{
    C tau, beta, rd;
    int e;
    v5_scalars_scaled<C>(src, ks, m, tau, beta, e, rd);
    v[0] = C(1);
    for (int k = 1; k < m; ++k) v[k] = scalbn(src[k * ks], -e) * rd;
    v[m] = tau;
    return beta;
}

// Reflector scalars for the panel, from alpha = x_0 and q = sum_{k>=1} x_k^2
// (dlarfg convention, readings Q7/Q8: beta = -sign(alpha) ||x||, sign(0) = +1,
// tau = (beta - alpha)/beta = 1 + |alpha|/||x||, rho = 1/(alpha - beta) =
// sign(alpha)/(|alpha| + ||x||)).  rsqrt / rcp by hardware approximation +
// Newton steps; the sign and the safe-range test are off the dependent chain
// (the range test compares the bit pattern of the non-negative sum as an
// integer: a dependent fp64 compare costs ~30 cycles on B200, integer ~5).
// Returns false when alpha^2 + q is outside [lo, hi] (caller: slow path).
template <class C> struct V5Bits;
template <> struct V5Bits<double> {
    static __device__ __forceinline__ bool in_range(double v)
    {
        const long long b = __double_as_longlong(v);
        return b >= 0x05CD0B15A491EB84ll /* 1e-280 */ && b <= 0x7A16A2EF4A3F5A34ll /* ~1e280 */;
    }
};
template <> struct V5Bits<float> {
    static __device__ __forceinline__ bool in_range(float v)
    {
        const int b = __float_as_int(v);
        return b >= 0x15F08FD5 /* ~1e-25 */ && b <= 0x6A0FBB2E /* ~1e25 */;
    }
};
template <class C>
__device__ __forceinline__ bool v5_scalars(C alpha, C q, C &tau, C &rho, C &beta)
{
    const C tot = fma(alpha, alpha, q);
    if (!V5Bits<C>::in_range(tot)) return false;
    const C rn = V4Math<C>::rsq(tot);
    const C nrm = tot * rn;
    const C aa = fabs(alpha);
    tau = fma(aa, rn, C(1));
    const C r = V4Math<C>::rcp(aa + nrm);
    const bool pos = alpha >= C(0);
    rho = pos ? r : -r;
    beta = pos ? -nrm : nrm;
    return true;
}

// Panel chain of one half, executed by warp 0 (a runtime loop: the code stays
// small for the instruction cache).  Element e of member l (row l of the A
// panel / column l of the B panel) lives at pan[e*ks + l*ls]:
//   A: member l = row q0 + l,  element e = col p + e:  Win[e*LA + l]          (ks = LA, ls = 1)
//   B: member l = col p + l,  element e = row p + e:  Win[l*LA + dq + e]     (ks = 1,  ls = LA)
// Link g: source x = member g's elements [g, g + MT) (after reflectors
// 0..g-1).  Every lane loads x (broadcast) and computes the dlarfg scalars
// redundantly in the same order (readings Q7/Q8); lanes l in (g, G) take
// their dot product against x (overlapping the norm), w = tau (a_0 + rho s),
// a -= w v; lane k writes v_g[k] = rho x_k (its own lane-indexed load, no
// dynamic register index), beta and exact zeros into the source.
// Latencies measured on B200 (tools/ubench/lat5.cu): DFMA 8.7 cycles, LDS
// 44, a dependent fp64 compare 30 -- so "x[1:] == 0" is decided from the sum
// of squares (an explicit test only when that sum is 0) and the safe-range
// test is integer (v5_scalars).  ~880 cycles per link (tools/ubench/panel5.cu).
// own[k*ks] = a[k] - wr * x[k*ks], k = 1 .. MT-1 (own and x are different
// members of the panel: __restrict__ lets every load issue ahead of the
// stores instead of one load-use-store round trip per element)
template <class C, int MT>
__device__ __forceinline__ void v5_axpy(C *__restrict__ own, const C *__restrict__ x, int ks, C wr, const C (&a)[MT])
{
    C xv[MT];
#pragma unroll
    for (int k = 1; k < MT; ++k) xv[k] = x[k * ks];
#pragma unroll
    for (int k = 1; k < MT; ++k) own[k * ks] = fma(-wr, xv[k], a[k]);
}

template <class C, int MT, int GT>
__device__ __forceinline__ void v5_panel(C *pan, int ks, int ls, C *vs, int VP, C * /*xb*/, int lane)
{
    // Only the member's own vector a[] lives in registers; the source x is
    // read from shared memory (broadcast) for the sums and again for the
    // update -- keeping x in registers as well (2 x MT doubles) spilled the
    // fp64 kernel to local memory inside this chain (ncu: ~95 LDL/STL per link).
    const bool member = lane < GT;
#pragma unroll 1
    for (int g = 0; g < GT; ++g) {
        C *src = pan + g * ks + g * ls; // element (g) of member g
        C *own = pan + g * ks + lane * ls;    // element (g) of member lane
        const bool upd = member && lane > g;
        // fp32: x is also kept in registers (no register pressure: faster);
        // fp64: re-read for the update (x + a in registers spilled)
        constexpr bool XREG = sizeof(C) == 4;
        C a[MT], xr[XREG ? MT : 1];
#pragma unroll
        for (int k = 0; k < MT; ++k) a[k] = upd ? own[k * ks] : C(0);
        C q4[4] = {0, 0, 0, 0}, s4[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 1; k < MT; ++k) {
            const C xk = src[k * ks];
            if constexpr (XREG) xr[k] = xk;
            q4[k & 3] = fma(xk, xk, q4[k & 3]);
            s4[k & 3] = fma(a[k], xk, s4[k & 3]);
        }
        const C alpha = src[0];
        const C xl = (lane < MT) ? src[lane * ks] : C(0);
        const C x32 = (MT > 32) ? src[(MT > 32 ? 32 : 0) * ks] : C(0);
        const C ss = (q4[0] + q4[1]) + (q4[2] + q4[3]);
        C tau = 0, rho = 0, beta = alpha;
        bool nz = ss > C(0);
        if (!nz) { // rare: all squares underflowed or x[1:] == 0
            for (int k = 1; k < MT; ++k) nz |= (src[k * ks] != C(0));
        }
        C *v = vs + g * VP;
        bool slow = nz && !v5_scalars<C>(alpha, ss, tau, rho, beta);
        __syncwarp(); // every lane has read the source
        if (slow) {
            if (lane == 0) beta = v5_slow_link<C>(src, ks, MT, v);
            __syncwarp();
            beta = __shfl_sync(0xffffffffu, beta, 0);
            tau = v[MT];
            rho = C(1);
            s4[0] = s4[1] = s4[2] = s4[3] = C(0);
            for (int k = 1; k < MT; ++k) s4[k & 3] = fma(a[k], v[k], s4[k & 3]);
        }
        if (upd && nz) {
            const C w = tau * fma(rho, (s4[0] + s4[1]) + (s4[2] + s4[3]), a[0]);
            const C wr = w * rho;
            own[0] = a[0] - w;
            if (!slow) {
                if constexpr (XREG) {
#pragma unroll
                    for (int k = 1; k < MT; ++k) own[k * ks] = fma(-wr, xr[k], a[k]);
                } else {
                    v5_axpy<C, MT>(own, src, ks, wr, a);
                }
            } else {
                v5_axpy<C, MT>(own, v, 1, wr, a);
            }
        }
        if (!slow) {
            if (lane < MT) v[lane] = (lane == 0) ? C(1) : (nz ? rho * xl : C(0));
            if (MT > 32 && lane == 0) v[32] = nz ? rho * x32 : C(0);
            if (lane == 0) v[MT] = tau;
        }
        __syncwarp(); // every lane has finished reading the source (update)
        if (lane < MT) src[lane * ks] = (lane == 0) ? beta : C(0);
        if (MT > 32 && lane == 0) src[32 * ks] = C(0);
        __syncwarp();
    }
}

#define TRACE5T(slot)                                                                                      \
    do {                                                                                                   \
        if (a.trace && tid == 32 && mat == 0 && k < a.trace_groups && j < a.trace_units)                  \
            a.trace[((int64_t)k * a.trace_units + j) * 16 + (slot)] = gtimer();                            \
    } while (0)
#define TRACE5C(slot)                                                                                      \
    do {                                                                                                   \
        if (a.trace && tid == 32 && mat == 0 && k < a.trace_groups && j < a.trace_units)                  \
            a.trace[((int64_t)k * a.trace_units + j) * 16 + (slot)] = clock64();                           \
    } while (0)
#define TRACE5(slot)                                                                                       \
    do {                                                                                                   \
        if (a.trace && tid == 0 && mat == 0 && k < a.trace_groups && j < a.trace_units)                   \
            a.trace[((int64_t)k * a.trace_units + j) * 16 + (slot)] = gtimer();                            \
    } while (0)

template <class S, int MT, int U, int GT>
__global__ void __launch_bounds__(256, 1) pass_v5_kernel(PassArgsV5 a)
{
    using C = typename ComputeOf<S>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_task;
    const int n = a.n, c = a.c, t = a.t;
    constexpr int G = GT;
    const int W = t + G;
    const int LA = a.LA, LB = a.LB;
    constexpr int VP = (MT + 2) & ~1; // v_g[0..MT-1], tau at [MT]
    C *Win = reinterpret_cast<C *>(smem_raw);
    C *Hr = Win + (size_t)W * LA;
    C *vA = Hr + (size_t)c * LB;
    vA += ((uintptr_t)vA & 15) ? (16 - ((uintptr_t)vA & 15)) / sizeof(C) : 0;
    C *vB = vA + (size_t)G * VP;
    C *xbuf = vB + (size_t)G * VP; // 2 x (MT + 1): panel source broadcast
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int ku = a.ku;
    const int64_t ldw1 = (int64_t)a.ldw - 1;
    const int total = a.batch * a.ngroups;

    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(a.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int k = task / a.batch;
        const int r0 = k * G;
        const int J = sweep_len(n, c, t, r0);
        S *Wg = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;
        const int *pprev = k > 0 ? a.progress + ((int64_t)mat * a.ngroups + (k - 1)) * a.fstride : nullptr;
        int *pme = a.progress + ((int64_t)mat * a.ngroups + k) * a.fstride;
        const int Jp = k > 0 ? sweep_len(n, c, t, r0 - G) : 0;

        for (int j = 0; j < J; ++j) {
            const int p = r0 + (c - t) + j * c;
            const int q0 = j ? p - c : r0;
            const int dq = p - q0;
            // ------------------------------------------------ A half
            TRACE5(0);
            if (tid == 0 && pprev) wait_geq(pprev, min(2 * j + a.a0, 2 * Jp));
            __syncthreads();
            TRACE5(1);
            {
                const int lo = j ? q0 + W : q0;
                v5_load<S, C>(Wg, ku, ldw1, n, c, t, lo, p + W - lo, p, W, Win + (lo - q0), LA, tid, nthr);
                v5_load_wait();
            }
            __syncthreads();
            TRACE5(2);
            if (tid < 32) v5_panel<C, MT, GT>(Win, LA, 1, vA, VP, xbuf, lane);
            __syncthreads();
            TRACE5(3);
            // A bulk, split so that the B panel overlaps the rest of the A half:
            // warps 1.. apply the G row reflectors to the rows of the B panel
            // (rows [p, p+W): the B panel needs nothing else -- its cells came with
            // the V load, and no other group touches them before our write-back)
            // first and release warp 0 at named barrier 1; warp 0 then runs the B
            // panel while warps 1.. finish the other bulk rows, write back the A
            // region, publish 2j+1, take the B wait and load H.
            // Bulk rows: q0+G .. p+W-1 (reflector g applies iff i <= p + g + t).
            if (tid >= 32) {
                const int nw = nthr - 32, tt = tid - 32;
                const int nrows = dq + t; // b in [0, dq + t): row q0 + G + b
                bool arrived = false;
                for (int bp = tt; bp < nrows; bp += nw) {
                    if (!arrived && bp >= W) {
                        nbar_arrive(1, nthr);
                        arrived = true;
                    }
                    const int b = bp < W ? dq - G + bp : bp - W; // B-panel rows first
                    const int ii = G + b, i = q0 + ii;
                    v5_apply<C, MT, U>(Win + ii, LA, G, i - p - t, vA, VP);
                }
                if (!arrived) nbar_arrive(1, nthr);
                nbar_sync(2, nw); // every A row done
                TRACE5T(4);
                TRACE5C(11);
                v5_store<S, C>(Wg, ku, ldw1, n, c, t, q0, dq, p, W, Win, LA, tt, nw);
                TRACE5C(12);
                nbar_sync(2, nw);
                if (tt == 0) {
                    TRACE5C(13);
                    fence_acq_rel();
                    TRACE5C(14);
                    st_release(pme, 2 * j + 1);
                    TRACE5C(15);
                    TRACE5T(5);
                    // ------------------------------------------------ B half
                    if (pprev) wait_geq(pprev, min(2 * j + (j + 2 < Jp ? a.b0 : a.b0t), 2 * Jp));
                    TRACE5T(6);
                }
                nbar_sync(2, nw);
                v5_load<S, C>(Wg, ku, ldw1, n, c, t, p, W, p + W, c, Hr, LB, tt, nw);
                v5_load_wait();
                TRACE5T(7);
            } else {
                nbar_sync(1, nthr); // rows [p, p+W) of the A bulk done
                v5_panel<C, MT, GT>(Win + dq, 1, LA, vB, VP, xbuf, lane);
            }
            __syncthreads(); // B panel, H load and the whole A half complete
            TRACE5(8);
            // bulk columns p+G .. p+G+c+t-1: reflector g applies iff x <= p + g + t + c
            for (int b = tid; b < c + t; b += nthr) {
                const int x = p + G + b;
                C *base = (x < p + W) ? Win + (x - p) * LA + dq : Hr + (x - p - W) * LB;
                v5_apply<C, MT, U>(base, 1, G, x - p - t - c, vB, VP);
            }
            __syncthreads();
            TRACE5(9);
            {
                const bool last = (j + 1 == J);
                v5_store<S, C>(Wg, ku, ldw1, n, c, t, p, W, p, W, Win + dq, LA, tid, nthr);
                v5_store<S, C>(Wg, ku, ldw1, n, c, t, p, W, p + W, last ? c : c - W, Hr, LB, tid, nthr);
            }
            __syncthreads();
            if (tid == 0) {
                fence_acq_rel();
                st_release(pme, 2 * j + 2);
            }
            TRACE5(10);
            // carry: H cols [p+c, p+c+W) rows [p, p+W) -> next unit's V rows [q0', q0'+W)
            if (j + 1 < J) {
                for (int e = tid; e < W * W; e += nthr) {
                    const int xx = e / W, ii = e - xx * W;
                    Win[xx * LA + ii] = Hr[(c - W + xx) * LB + ii];
                }
            }
        }
    }
}

} // namespace bb
