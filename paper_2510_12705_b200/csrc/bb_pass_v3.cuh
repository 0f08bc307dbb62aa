// bb_pass_v3.cuh -- multi-sweep persistent pass kernel with a shared-memory
// window cache (sm_100a).
//
// WHY.  A pass is a chain of ~n dependent sweep-to-sweep hand-offs (sweep r+1
// may do step j only after sweep r did (part of) step j+1; Alg. 1, P:119,
// P:145).  On B200 a hand-off through L2 costs ~1-2 us (gpu-scope release
// fence, polling, then an L2 round trip to reload the window), more than the
// step arithmetic.  Consecutive sweeps touch almost the same windows (step j
// of sweep r+1 is step j of sweep r shifted by one row and one column), so
// this kernel runs G CONSECUTIVE sweeps in one CTA -- one warp-group (WG) per
// sweep, concurrently -- and keeps their windows in shared memory:
//   * hand-off WG g -> WG g+1 is a shared-memory progress counter (CTA-scope
//     release/acquire) and the data is already in shared memory;
//   * only WG 0 reads the band from L2 (once per step, for the whole group),
//     and only every G-th hand-off crosses CTAs (global flags, RELEASE warp).
// This is the paper's "software-level loop unrolling: a single block is
// assigned multiple tasks", with the tasks overlapped.
//
// SLOTS.  Step j of the group lives in slot s(j) = j mod NS.  With
// p0 = r0 + (c - t) + j*c and q0 = (j ? p0 - c : r0) (sweep r0's geometry),
// WT = t + G, every cell has exactly ONE home:
//   slot(j).T : rows [trow0(j), trow0(j) + LDT) x cols [p0, p0 + WT)
//               trow0(0) = r0, trow0(j>0) = q0 + WT   (column-major, ld LDT)
//   slot(j).W : rows [p0, p0 + WT) x cols [p0 + WT, p0 + c + WT) (ld LDW)
// The top rows [q0, q0 + WT) of columns [p0, p0 + WT) belong to slot(j-1).W.
// Step (r0+g, j) touches only slots j-1 and j; the step windows of the G
// sweeps at step j all fit (this needs c >= t + G + 2, checked on the host).
// WG 0 fills slot(j) from L2 when it reaches step j (after waiting for the
// previous group), except the right-end columns >= p0 + c - 1, which it loads
// after waiting for A(r0 - 1, j + 1).  Everything a WG modifies is written
// through to the working band (coalesced), so L2 is always current for the
// next group and the next pass.  Slot(j) is recycled after WG G-1 finished
// A(j+1) (the last reader of its W part).
//
// Progress encoding and wait rule are those of bb_pass_v2.cuh (2j+1 after the
// A half, 2j+2 after the step; A waits for 2j+2, B for 2j+3 of sweep r-1).
#pragma once

#include "bb_pass_v2.cuh"

#include <cuda.h> // CUtensorMap

namespace bb {

struct PassArgsV3 {
    void *W;
    int64_t mat_stride;
    int ldw, ku, n;
    int c, t;
    int a0, b0;
    int batch, nsweeps;
    int ngroups;       // ceil(nsweeps / G) groups per matrix
    int *progress;     // [batch][n] global progress (last sweep of each group)
    int *counter;      // group claim counter
    int ntg;           // threads per WG (multiple of 32)
    int LDT, LDW;      // slot leading dimensions (odd)
    int NS;            // slots in the ring
    int dbg;           // debug bits (bit 0: generic warp reflector)
    int nWe;           // early W columns (c - 1 - WT); the last WT + 1 are the right end
    int WeOff, WreOff; // element offsets of the W parts inside a slot (128-byte aligned)
    int slot_elems;    // elements per slot (128-byte multiple)
    int use_tma;       // fill slots with TMA (S == C only)
    unsigned long long *trace;
    int trace_sweeps, trace_steps;
};

__device__ __forceinline__ int ld_acquire_cta_s(const int *p)
{
    int v;
    asm volatile("ld.acquire.cta.shared.b32 %0, [%1];"
                 : "=r"(v)
                 : "r"((unsigned)__cvta_generic_to_shared(p))
                 : "memory");
    return v;
}
__device__ __forceinline__ int ld_volatile_s(const int *p)
{
    int v;
    asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_s(int *p, int v)
{
    asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
                 : "memory");
}
#ifndef BB_SPIN_NS
#define BB_SPIN_NS 64
#endif
__device__ __forceinline__ void spin_geq_s(const int *p, int need)
{
    if (ld_volatile_s(p) < need)
        while (ld_volatile_s(p) < need) {
            if (BB_SPIN_NS) __nanosleep(BB_SPIN_NS);
        }
    (void)ld_acquire_cta_s(p);
}

#define TRACE3(slot)                                                                              \
    do {                                                                                          \
        if (a.trace && mat == 0 && r < a.trace_sweeps && j < a.trace_steps)                       \
            a.trace[((int64_t)r * a.trace_steps + j) * 16 + (slot)] = gtimer();                   \
    } while (0)

// HH(X) by one warp, m <= 64 (dlarfg convention, identity iff x[1:] == 0
// exactly).  One reciprocal square root and one reciprocal:
//   nrm = ssq * rsqrt(ssq), beta = -sign(alpha) nrm,
//   tau = (beta - alpha) / beta = 1 + |alpha| / nrm,  v = x / (alpha - beta).
// The max-scaled norm is used only when the plain sum of squares is outside
// the safe range (no under/overflow).
template <class C>
__device__ __forceinline__ void house_warp_fast(const C *x, int stride, int m, C *v, C &tau, C &beta)
{
    const int lane = threadIdx.x & 31;
    const C x0 = lane < m ? x[lane * stride] : C(0);
    const C x1 = lane + 32 < m ? x[(lane + 32) * stride] : C(0);
    const C alpha = __shfl_sync(0xffffffffu, x0, 0);
    const bool nz = __any_sync(0xffffffffu, (lane > 0 && x0 != C(0)) || x1 != C(0));
    if (!nz) {
        tau = 0;
        beta = alpha;
        if (lane < m) v[lane] = (lane == 0) ? C(1) : C(0);
        if (lane + 32 < m) v[lane + 32] = C(0);
        return;
    }
    const C ssq = warp_sum(fma(x1, x1, x0 * x0));
    C nrm, rn;
    if (ssq >= NormRange<C>::lo() && ssq <= NormRange<C>::hi()) {
        rn = rsqrt(ssq);
        nrm = ssq * rn;
    } else {
        const C amax = warp_max(fmax(fabs(x0), fabs(x1)));
        const C y0 = x0 / amax, y1 = x1 / amax;
        nrm = amax * sqrt(warp_sum(fma(y1, y1, y0 * y0)));
        rn = C(1) / nrm;
    }
    beta = (alpha >= C(0)) ? -nrm : nrm;
    tau = fma(fabs(alpha), rn, C(1));
    const C den = alpha - beta;
    if (fabs(den) >= SafeRcp<C>::lo()) {
        const C rd = C(1) / den;
        if (lane < m) v[lane] = (lane == 0) ? C(1) : x0 * rd;
        if (lane + 32 < m) v[lane + 32] = x1 * rd;
    } else {
        if (lane < m) v[lane] = (lane == 0) ? C(1) : x0 / den;
        if (lane + 32 < m) v[lane + 32] = x1 / den;
    }
}

template <class C> struct Slot {
    C *T;   // [LDT * WT]       rows trow0.. of columns p0 .. p0+WT-1
    C *We;  // [LDW * nWe]      rows p0.. of columns p0+WT .. p0+c-2
    C *Wre; // [LDW * (WT+1)]   rows p0.. of columns p0+c-1 .. p0+c+WT-1 (right end)
};

// ---- TMA / mbarrier helpers ------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
    asm volatile("{\n\t.reg .pred P1;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar)
{
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                 "[%5];" ::"r"(smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void mbar_add_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), 16-byte aligned, size multiple of 16
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Fill `ncol` column segments into shared memory with 1-D bulk copies issued
// by one warp.  Column k starts (in elements) at g0 + k*gstride in global
// memory; every start has the same alignment, so each copy starts delta =
// misalignment elements early and the shared column k begins at
// s0 + k*spitch (16-byte aligned); the caller addresses it from s0 + delta.
template <class C>
__device__ __forceinline__ void bulk_fill_cols(C *s0, int spitch, const C *g0, int64_t gstride, int rows, int ncol,
                                               int delta, uint64_t *bar, int lane)
{
    const int q = 16 / (int)sizeof(C);
    const unsigned bytes = (unsigned)(((rows + delta + q - 1) / q) * q * sizeof(C));
    unsigned mine = 0;
    for (int k = lane; k < ncol; k += 32) mine += bytes;
    if (mine) mbar_add_tx(bar, mine);
    __syncwarp();
    for (int k = lane; k < ncol; k += 32) bulk_g2s(s0 + (size_t)k * spitch, g0 + k * gstride - delta, bytes, bar);
}

// Geometry of one step (r0+g, j) (q0 of slot j == p0 of slot j-1).
struct StepGeo {
    int p0, q0, trow0, p, q, hi, ce, m, off, rowsT, ncols;
    int dT, dW; // bulk-copy misalignment (elements) of the slot's T / W column starts
};

__device__ __forceinline__ StepGeo step_geo(int n, int c, int t, int G, int r0, int g, int j)
{
    StepGeo s;
    s.p0 = r0 + (c - t) + j * c;
    s.q0 = j ? s.p0 - c : r0;
    s.trow0 = j ? s.q0 + t + G : r0;
    s.p = s.p0 + g;
    s.q = s.q0 + g;
    s.hi = min(s.p + t, n - 1);
    s.ce = min(s.hi + c, n - 1);
    s.m = s.hi - s.p + 1;
    s.off = s.p - s.q;
    s.rowsT = s.hi - s.q + 1;
    s.ncols = s.ce - s.p + 1;
    return s;
}

// shared-memory address of cell (i, jc) of a step in slot j (prev = slot j-1)
// (the top rows of columns p0..p0+WT-1 live in slot(j-1)'s right-end part)
template <class C>
__device__ __forceinline__ C *cell(const StepGeo &s, const Slot<C> &cur, const Slot<C> &prev, int i, int jc, int WT,
                                   int LDT, int LDW, bool has_prev, int nWe)
{
    if (jc < s.p0 + WT) {
        if (has_prev && i < s.trow0) return prev.Wre + (i - s.q0) + (jc - s.q0 - WT - nWe) * LDW;
        return cur.T + (i - s.trow0) + (jc - s.p0) * LDT;
    }
    const int k = jc - s.p0 - WT;
    return (k < nWe ? cur.We + k * LDW : cur.Wre + (k - nWe) * LDW) + (i - s.p0);
}

template <class S, int MT>
__device__ __forceinline__ void step_v3(const PassArgsV3 &a, S *Wg, int mat, int r0, int g, int G, int j, int Jp,
                                        const int *gprev, int *prog_s, const Slot<typename ComputeOf<S>::type> &cur,
                                        const Slot<typename ComputeOf<S>::type> &prv,
                                        typename ComputeOf<S>::type *v1, typename ComputeOf<S>::type *v2,
                                        typename ComputeOf<S>::type *scal, int tid, int ntg, int bar, bool wt_in,
                                        uint64_t *fbar, unsigned &fphase)
{
    using C = typename ComputeOf<S>::type;
    const int n = a.n, c = a.c, t = a.t, ku = a.ku;
    const int LDT = a.LDT, LDW = a.LDW, WT = t + G;
    const int64_t ldw = a.ldw;
    const int lane = tid & 31, wwarp = tid >> 5;
    const int r = r0 + g;
    StepGeo s = step_geo(n, c, t, G, r0, g, j);
    {
        // global column starts: W + ku + row0 + jc*(ldw-1) + mat*mat_stride, with
        // (ldw-1) and mat_stride multiples of 16 bytes -> same misalignment per slot
        const int q = 16 / (int)sizeof(C);
        s.dT = a.use_tma ? (ku + s.trow0) % q : 0;
        s.dW = a.use_tma ? (ku + s.p0) % q : 0;
    }
    // logical slot views (column starts shifted by the bulk-copy misalignment)
    const int dWp = (a.use_tma && j > 0) ? (ku + s.q0) % (16 / (int)sizeof(C)) : 0; // slot j-1's W shift
    const Slot<C> cu = {cur.T + s.dT, cur.We + s.dW, cur.Wre + s.dW};
    const Slot<C> pv = {prv.T, prv.We, prv.Wre + dWp};
    const int m = s.m;
    const bool FULL = (m == MT); // full-length reflector: unrolled register loops
    const bool has_prev = j > 0;
    auto gaddr = [&](int i, int jc) -> S * { return Wg + (ku + i - jc) + (int64_t)jc * ldw; };
    const bool wt = (a.dbg & 2) ? false : wt_in; // debug bit 2: partial write-through only (timing)

    // ------------------------------------------------ A wait (+ slot reuse for WG 0)
    if (tid == 0) {
        TRACE3(0);
        if (r > 0) {
            const int need = min(2 * j + a.a0, 2 * Jp);
            if (g > 0) spin_geq_s(prog_s + g - 1, need);
            else wait_geq(gprev, need);
        }
        // slot reuse: every WG finished A(j - NS + 1) (or its sweep)
        if (g == 0 && j >= a.NS) {
            for (int k = 0; k < G; ++k) {
                const int Jk = (r0 + k < a.nsweeps) ? sweep_len(n, c, t, r0 + k) : 0;
                if (Jk > 0) spin_geq_s(prog_s + k, min(2 * (j - a.NS + 1) + 1, 2 * Jk));
            }
        }
        TRACE3(1);
    }
    nbar_sync(bar, ntg);

    // ------------------------------------------------ WG 0: fill slot(j) from L2
    // T part: LDT rows x WT columns; W part: WT rows x (late0 - p0 - WT) columns.
    // Element e -> (column k, row ii) is stepped incrementally (no division per
    // element); every column segment is contiguous in the band, so each warp
    // instruction covers whole segments.
    if (sizeof(S) == sizeof(C) && a.use_tma) {
    if (g == 0) {
        // bulk copies (TMA engine, no registers, one round trip): T part columns
        // p0 .. p0+WT-1 (rows trow0 ..) and the early W columns (rows p0 ..)
        if (wwarp == 0) {
            if (lane == 0) fence_proxy_async(); // generic-proxy accesses before the async copies
            __syncwarp();
            const int q = 16 / (int)sizeof(C);
            const int ncT = min(WT, n - s.p0), ncW = max(0, min(a.nWe, n - s.p0 - WT));
            bulk_fill_cols<C>(cur.T, LDT, reinterpret_cast<const C *>(gaddr(s.trow0, s.p0)), ldw - 1,
                              LDT - q, ncT, s.dT, fbar, lane);
            bulk_fill_cols<C>(cur.We, LDW, reinterpret_cast<const C *>(gaddr(s.p0, s.p0 + WT)), ldw - 1, WT,
                              ncW, s.dW, fbar, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(fbar);
        }
        mbar_wait(fbar, fphase & 1);
        ++fphase;
    }
    } else {
    if (g == 0) {
        const int late0 = (a.b0 > a.a0) ? s.p0 + c - 1 : s.p0 + c + WT;
        const int nWc = max(0, min(late0, s.p0 + c + WT) - (s.p0 + WT));
        const bool interior = (s.p0 + c + WT <= n) && (s.trow0 + LDT <= n);
        for (int part = 0; part < 2; ++part) {
            const int rows = part == 0 ? LDT : WT;
            const int ncol = part == 0 ? WT : nWc;
            const int i0 = part == 0 ? s.trow0 : s.p0;
            const int j0 = part == 0 ? s.p0 : s.p0 + WT;
            C *dst0 = part == 0 ? cur.T : cur.We;
            const int ld = part == 0 ? LDT : LDW;
            const int tot = rows * ncol;
            int e = tid, k = e / rows, ii = e - k * rows;
            const int dk = ntg / rows, dii = ntg - dk * rows;
            while (e < tot) {
                C v[16];
                int o[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    o[u] = -1;
                    if (e < tot) {
                        const int i = i0 + ii, jc = j0 + k;
                        const int rho = ku + i - jc;
                        const bool ok = interior ? (rho >= 0 && rho < ldw) : (i < n && jc < n && rho >= 0 && rho < ldw);
                        v[u] = ok ? ldg_cg(gaddr(i, jc)) : C(0);
                        o[u] = ii + k * ld;
                    }
                    e += ntg; ii += dii; k += dk;
                    if (ii >= rows) { ii -= rows; ++k; }
                }
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (o[u] >= 0) dst0[o[u]] = v[u];
            }
        }
        nbar_sync(bar, ntg);
    }
    }
    if (tid == 0) TRACE3(2);

    // ------------------------------------------------ row reflector (warp 0) from A[q, p..hi]
    // row q lies in slot(j-1).W (j > 0) or slot(0).T
    C *x0 = cell<C>(s, cu, pv, s.q, s.p, WT, LDT, LDW, has_prev, a.nWe);
    const int xs = (has_prev && s.q < s.trow0) ? LDW : LDT;
    if (wwarp == 0) {
        C tau, beta;
        if ((a.dbg & 1) || sizeof(C) == 4) house_warp<C>(x0, xs, m, v1, tau, beta);
        else house_warp_fast<C>(x0, xs, m, v1, tau, beta);
        if (lane == 0) scal[0] = tau;
        __syncwarp();
        for (int k = lane; k < m; k += 32) {
            const C val = (k == 0) ? beta : C(0);
            x0[k * xs] = val;
            stg(gaddr(s.q, s.p + k), val);
        }
    }
    nbar_sync(bar, ntg);
    if (tid == 0) TRACE3(6);

    // ------------------------------------------------ right application to rows q+1..hi
    const C tau1 = scal[0];
    for (int ii = 1 + tid; ii < s.rowsT; ii += ntg) {
        const int i = s.q + ii;
        C *rb = cell<C>(s, cu, pv, i, s.p, WT, LDT, LDW, has_prev, a.nWe);
        const int rs = (has_prev && i < s.trow0) ? LDW : LDT;
        S *gb = gaddr(i, s.p);
        const int64_t gs = ldw - 1;
        if (tau1 != C(0)) {
            if (FULL) {
                // dot product, then a second pass that reloads the row: a small
                // register footprint (no spills with G warp-groups per SM)
                C s4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int k = 0; k < MT; ++k) s4[k & 3] = fma(rb[k * rs], v1[k], s4[k & 3]);
                const C wv = tau1 * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
#pragma unroll
                for (int k = 0; k < MT; ++k) {
                    const C y = fma(-wv, v1[k], rb[k * rs]);
                    rb[k * rs] = y;
                    if ((wt || k == 0) && ii < s.off) stg(gb + k * gs, y);
                }
            } else {
                C sacc = 0;
                for (int k = 0; k < m; ++k) sacc = fma(rb[k * rs], v1[k], sacc);
                const C wv = tau1 * sacc;
                for (int k = 0; k < m; ++k) {
                    const C y = fma(-wv, v1[k], rb[k * rs]);
                    rb[k * rs] = y;
                    if ((wt || k == 0) && ii < s.off) stg(gb + k * gs, y);
                }
            }
        } else if (ii < s.off) {
            for (int k = 0; k < (wt ? m : 1); ++k) stg(gb + k * gs, rb[k * rs]);
        }
    }
    nbar_sync(bar, ntg);
    if (tid == 0) {
        TRACE3(7);
        st_release_cta_s(prog_s + g, 2 * j + 1); // A half done
        TRACE3(3);
    }

    // ------------------------------------------------ column reflector (warp 0) from A[p..hi, p]
    C *cp = cell<C>(s, cu, pv, s.p, s.p, WT, LDT, LDW, has_prev, a.nWe); // contiguous over rows p..hi
    if (wwarp == 0) {
        C tau, beta;
        if ((a.dbg & 1) || sizeof(C) == 4) house_warp<C>(cp, 1, m, v2, tau, beta);
        else house_warp_fast<C>(cp, 1, m, v2, tau, beta);
        if (lane == 0) scal[2] = tau;
        __syncwarp();
        for (int kk = lane; kk < m; kk += 32) cp[kk] = (kk == 0) ? beta : C(0);
        if (lane == 0) TRACE3(8);
    }

    // ------------------------------------------------ B wait (+ WG 0: right-end columns from L2)
    if (tid == 0 && r > 0 && a.b0 > a.a0) {
        const int need = min(2 * j + a.b0, 2 * Jp);
        if (g > 0) spin_geq_s(prog_s + g - 1, need);
        else wait_geq(gprev, need);
    }
    nbar_sync(bar, ntg);
    if (sizeof(S) == sizeof(C) && a.use_tma) {
    if (g == 0 && a.b0 > a.a0) {
        if (wwarp == 0) {
            if (lane == 0) fence_proxy_async();
            __syncwarp();
            const int jlo = s.p0 + c - 1;
            const int ncR = max(0, min(WT + 1, n - jlo));
            bulk_fill_cols<C>(cur.Wre, LDW, reinterpret_cast<const C *>(gaddr(s.p0, jlo)), ldw - 1, WT, ncR,
                              s.dW, fbar, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(fbar);
        }
        mbar_wait(fbar, fphase & 1);
        ++fphase;
    }
    } else {
    if (g == 0 && a.b0 > a.a0) {
        const int jlo = s.p0 + c - 1, jhi = min(s.p0 + c + WT - 1, n - 1);
        const int ncl = jhi - jlo + 1;
        for (int e = tid; e < ncl * WT; e += ntg) {
            const int k = e / WT, ii = e - k * WT;
            const int i = s.p0 + ii, jc = jlo + k;
            const int rho = ku + i - jc;
            cur.Wre[ii + k * LDW] = (i < n && rho >= 0 && rho < ldw) ? ldg_cg(gaddr(i, jc)) : C(0);
        }
        nbar_sync(bar, ntg);
    }
    }
    if (tid == 0) TRACE3(4);

    // ------------------------------------------------ left application to columns p+1..ce
    const C tau2 = scal[2];
    if (tau2 != C(0)) {
        for (int sl = 1 + tid; sl < s.ncols; sl += ntg) {
            C *col = cell<C>(s, cu, pv, s.p, s.p + sl, WT, LDT, LDW, has_prev, a.nWe);
            if (FULL) {
                C s4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) s4[kk & 3] = fma(v2[kk], col[kk], s4[kk & 3]);
                const C wv = tau2 * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) col[kk] = fma(-wv, v2[kk], col[kk]);
            } else {
                C sacc = 0;
                for (int kk = 0; kk < m; ++kk) sacc = fma(v2[kk], col[kk], sacc);
                const C wv = tau2 * sacc;
                for (int kk = 0; kk < m; ++kk) col[kk] = fma(-wv, v2[kk], col[kk]);
            }
        }
    }
    nbar_sync(bar, ntg);
    if (tid == 0) TRACE3(9);
    // ------------------------------------------------ write rows p..hi of columns p..ce through
    // wt (last modifier of the whole window): every cell, one warp per column
    // (coalesced).  Otherwise only the cells no later sweep of the group
    // touches: column p and row p (tools/v3_cover.py).
    if (wt) {
        const int nw = ntg >> 5;
        for (int sl = wwarp; sl < s.ncols; sl += nw) {
            const int jc = s.p + sl;
            const C *src = cell<C>(s, cu, pv, s.p, jc, WT, LDT, LDW, has_prev, a.nWe);
            S *dstg = gaddr(s.p, jc);
            for (int kk = lane; kk < m; kk += 32) stg(dstg + kk, src[kk]);
        }
    } else {
        if (wwarp == 0) {
            const C *src = cell<C>(s, cu, pv, s.p, s.p, WT, LDT, LDW, has_prev, a.nWe);
            for (int kk = lane; kk < m; kk += 32) stg(gaddr(s.p + kk, s.p) , src[kk]);
        }
        for (int sl = 1 + tid; sl < s.ncols; sl += ntg)
            stg(gaddr(s.p, s.p + sl), *cell<C>(s, cu, pv, s.p, s.p + sl, WT, LDT, LDW, has_prev, a.nWe));
    }
    nbar_sync(bar, ntg);
    if (tid == 0) {
        st_release_cta_s(prog_s + g, 2 * j + 2); // step complete (written through)
        TRACE3(5);
    }
}

// G warp-groups of ntg threads + one RELEASE warp; NS slots in shared memory.
template <class S, int MT, int G, int NTMAX>
__global__ void __launch_bounds__(NTMAX, 1)
    pass_v3_kernel(PassArgsV3 a)
{
    using C = typename ComputeOf<S>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_task;
    __shared__ int prog_s[G + 1];
    __shared__ __align__(8) uint64_t fill_bar;
    unsigned fphase = 0;
    if (threadIdx.x == 0) {
        mbar_init(&fill_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    const int ntg = a.ntg;
    const int tid_all = threadIdx.x;
    const int g = tid_all / ntg;   // WG index; g == G -> release warp
    const int tid = tid_all - g * ntg;
    const int WT = a.t + G;
    const size_t slot_elems = (size_t)a.slot_elems;
    // TMA destinations must be 128-byte aligned (the host adds 128 bytes of slack)
    C *base = reinterpret_cast<C *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    C *vbase = base + slot_elems * a.NS;           // per-WG v1, v2, scal
    C *v1 = vbase + (size_t)(g < G ? g : 0) * (2 * MT + 4);
    C *v2 = v1 + MT;
    C *scal = v2 + MT;

    const int n = a.n, c = a.c, t = a.t;
    const int total = a.batch * a.ngroups;
    for (;;) {
        __syncthreads();
        if (tid_all == 0) s_task = atomicAdd(a.counter, 1);
        if (tid_all <= G) prog_s[tid_all] = 0;
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int r0 = (task / a.batch) * G;
        int *gprog = a.progress + (int64_t)mat * n;
        S *Wg = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;
        const int glast = min(G, a.nsweeps - r0) - 1;

        if (g < G) {
            const int r = r0 + g;
            if (g <= glast) {
                const int J = sweep_len(n, c, t, r);
                const int Jp = r > 0 ? sweep_len(n, c, t, r - 1) : 0;
                const int *gprev = (g == 0 && r > 0) ? gprog + (r - 1) : nullptr;
                // write-through: the last WG always; an earlier WG once the next
                // sweep of the group has no later step (matrix end, tools/v3_cover.py)
                const int Jnext = (g < glast) ? sweep_len(n, c, t, r + 1) : 0;
                for (int j = 0; j < J; ++j) {
                    const bool wt = (g == glast) || (j >= Jnext - 1);
                    Slot<C> cur, prv;
                    cur.T = base + slot_elems * (j % a.NS);
                    cur.We = cur.T + a.WeOff;
                    cur.Wre = cur.T + a.WreOff;
                    prv.T = base + slot_elems * ((j + a.NS - 1) % a.NS);
                    prv.We = prv.T + a.WeOff;
                    prv.Wre = prv.T + a.WreOff;
                    step_v3<S, MT>(a, Wg, mat, r0, g, G, j, Jp, gprev, prog_s, cur, prv, v1, v2, scal, tid, ntg, 1 + g,
                                   wt, &fill_bar, fphase);
                }
            }
        } else if ((tid_all & 31) == 0) {
            // RELEASE warp: republish the last WG's progress at gpu scope.  Every
            // cell is written through by its last modifier in the group before
            // that WG's release, and the last WG's progress v transitively orders
            // all of them (bb_pass_v3.cuh header), so one fence per value suffices.
            const int rl = r0 + glast;
            const int target = 2 * sweep_len(n, c, t, rl);
            int published = 0;
            while (published < target) {
                const int v = ld_volatile_s(prog_s + glast);
                if (v > published) {
                    (void)ld_acquire_cta_s(prog_s + glast);
                    if (!(a.dbg & 4)) fence_acq_rel(); // debug bit 4: no fence (timing experiments only)
                    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(gprog + rl), "r"(v) : "memory");
                    published = v;
                } else if (BB_SPIN_NS) {
                    __nanosleep(BB_SPIN_NS);
                }
            }
        }
    }
}

} // namespace bb
