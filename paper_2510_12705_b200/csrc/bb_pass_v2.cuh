// bb_pass_v2.cuh -- latency-optimised persistent pass kernel (sm_100a).
//
// Same step as bb_kernels.cuh::bulge_step (Alg. 2), re-mapped for
// the critical path of the sweep wavefront:
//
//  * rows of the step's tall part (rows q..hi x cols p..hi) live in REGISTERS,
//    one row per compute thread (the paper's "each thread loads a row of width
//    TW+1 into register memory"), loaded straight from L2 with m
//    independent loads per thread; the right application happens in registers
//    and rows q+1..p-1 are written back immediately;
//  * the corner rows p..hi go through a small shared-memory block so the
//    column reflector (one warp, shuffle reduction) and the left application
//    (one thread per column) can read them column-wise;
//  * the wide part (rows p..hi x cols hi+1..ce) is staged in shared memory,
//    loaded EARLY except its right-end columns >= p+c-1;
//  * two signalling warps decouple the flags from the math: a POLL warp
//    acquires the predecessor sweep's progress, a RELEASE warp fences and
//    publishes this sweep's progress, synchronised with the compute warps by
//    named barriers (bar.arrive / bar.sync), so no compute warp ever waits on
//    a fence.
//
// Progress of sweep r counts completed half-steps: 2j+1 after the A part of
// step j (row reflector + right application, rows < p written back), 2j+2
// after the whole step.  Waits (tools/depcheck.py verifies that every pair of
// conflicting half-steps is ordered, so the result is bitwise the sequential
// one):
//     A(r, j) (and the early loads) wait  progress[r-1] >= min(2j + a0, 2J)
//     B(r, j) (late loads, left apply) wait progress[r-1] >= min(2j + b0, 2J)
//   target bandwidth c-t >= 4: a0 = 2, b0 = 3   (B waits only for A(r-1, j+1))
//   c-t in {2, 3}:             a0 = b0 = 4      (whole-step distance s = 2)
//   c-t == 1:                  a0 = b0 = 6      (whole-step distance s = 3)
#pragma once

#include "bb_kernels.cuh"

namespace bb {

struct PassArgsV2 {
    void *W;
    int64_t mat_stride;
    int ldw, ku, n;
    int c, t;
    int a0, b0;          // wait offsets (see header)
    int batch, nsweeps;
    int *progress;       // [batch][n]
    int *counter;
    int ntc;             // compute threads (multiple of 32)
    int LW;              // wide-part shared leading dimension (odd)
    unsigned long long *trace;
    int trace_sweeps, trace_steps;
};

// named barriers, non-.aligned forms: a warp may reach them diverged (e.g.
// after a tid == 0 branch) -- bar.sync (= barrier.sync.aligned) requires a
// converged warp (compute-sanitizer synccheck: "Divergent thread(s)")
__device__ __forceinline__ void nbar_sync(int id, int count)
{
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count)
{
    asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

enum { BAR_START = 1, BAR_C = 2, BAR_A = 3, BAR_W1 = 4, BAR_B = 5 };

template <class C> struct SafeRcp;
template <> struct SafeRcp<double> {
    static __device__ __forceinline__ double lo() { return 1e-290; }
};
template <> struct SafeRcp<float> {
    static __device__ __forceinline__ float lo() { return 1e-30f; }
};

// HH(X) computed by ONE thread from a register row x[0..m-1] (m <= MT;
// FULL: m == MT known at compile time).  Writes v (v[0] = 1) to shared
// memory; returns tau and beta (dlarfg convention, identity iff x[1:] == 0
// exactly; the max-scaled norm is only evaluated when the plain sum of
// squares is out of the safe range).
template <class C, int MT, bool FULL>
__device__ __forceinline__ void house_thread(const C (&x)[MT], int m, C *v, C &tau, C &beta)
{
    const C alpha = x[0];
    bool nz = false;
    C s4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < MT; ++k) {
        if (FULL || k < m) {
            if (k > 0) nz |= (x[k] != C(0));
            s4[k & 3] = fma(x[k], x[k], s4[k & 3]);
        }
    }
    if (!nz) {
        tau = 0;
        beta = alpha;
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) v[k] = (k == 0) ? C(1) : C(0);
        return;
    }
    const C ssq = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    C nrm;
    if (ssq >= NormRange<C>::lo() && ssq <= NormRange<C>::hi()) {
        nrm = sqrt(ssq);
    } else {
        C amax = 0;
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (k < m) amax = fmax(amax, fabs(x[k]));
        C s2 = 0;
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (k < m) {
                C y = x[k] / amax;
                s2 = fma(y, y, s2);
            }
        nrm = amax * sqrt(s2);
    }
    beta = (alpha >= C(0)) ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    const C den = alpha - beta;
    v[0] = C(1);
    if (fabs(den) >= SafeRcp<C>::lo()) {
        const C rcp = C(1) / den;
#pragma unroll
        for (int k = 1; k < MT; ++k)
            if (FULL || k < m) v[k] = x[k] * rcp;
    } else {
#pragma unroll
        for (int k = 1; k < MT; ++k)
            if (k < m) v[k] = x[k] / den;
    }
}

// tree-shaped dot product of x[0..m-1] and y[0..m-1] (4 partial sums)
template <class C, int MT, bool FULL>
__device__ __forceinline__ C dot4(const C (&x)[MT], const C (&y)[MT], int m)
{
    C s4[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < MT; ++k)
        if (FULL || k < m) s4[k & 3] = fma(x[k], y[k], s4[k & 3]);
    return (s4[0] + s4[1]) + (s4[2] + s4[3]);
}

// shared memory layout (compute type C):
//   v1[MT], v2[MT], scal[4], bcols[LW * (c + t + 1)]

// gather/scatter of `ncols` column segments of `rows` elements (column s at
// g + s*gstride) by threads [0, nthr): consecutive threads take consecutive
// elements, so each warp instruction covers whole segments (coalesced).
template <class S, class C, int U>
__device__ __forceinline__ void gather_cols_n(const S *__restrict__ g, int64_t gstride, int rows, int ncols,
                                              C *__restrict__ s, int sstride, int tid, int nthr)
{
    const int total = rows * ncols;
    if (total <= 0) return;
    int e = tid;
    int k = e / rows, ii = e - k * rows;
    const int dk = nthr / rows, dii = nthr - dk * rows;
    while (e < total) {
        C buf[U];
        int so[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            so[u] = -1;
            if (e < total) {
                buf[u] = ldg_cg(g + k * gstride + ii);
                so[u] = ii + k * sstride;
            }
            e += nthr;
            ii += dii;
            k += dk;
            if (ii >= rows) { ii -= rows; ++k; }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (so[u] >= 0) s[so[u]] = buf[u];
    }
}

template <class S, class C>
__device__ __forceinline__ void scatter_cols_n(S *__restrict__ g, int64_t gstride, int rows, int ncols,
                                               const C *__restrict__ s, int sstride, int tid, int nthr)
{
    const int total = rows * ncols;
    if (total <= 0) return;
    int e = tid;
    int k = e / rows, ii = e - k * rows;
    const int dk = nthr / rows, dii = nthr - dk * rows;
    for (; e < total; e += nthr) {
        stg(g + k * gstride + ii, s[ii + k * sstride]);
        ii += dii;
        k += dk;
        if (ii >= rows) { ii -= rows; ++k; }
    }
}

#define TRACE2(slot)                                                                              \
    do {                                                                                          \
        if (a.trace && mat == 0 && r < a.trace_sweeps && j < a.trace_steps)                       \
            a.trace[((int64_t)r * a.trace_steps + j) * 16 + (slot)] = gtimer();                   \
    } while (0)


// One step (r, j) executed by the compute warps (threads [0, ntc)).  FULL:
// the reflector length m equals MT (every step except the clipped ones at
// the matrix end), so all per-element predicates fold away.
template <class S, int MT, bool FULL>
__device__ __forceinline__ void compute_step(const PassArgsV2 &a, S *W, int mat, int r, int j,
                                             typename ComputeOf<S>::type *v1, typename ComputeOf<S>::type *v2,
                                             typename ComputeOf<S>::type *scal,
                                             typename ComputeOf<S>::type *bcols, int NALL)
{
    using C = typename ComputeOf<S>::type;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ntc = a.ntc, n = a.n, c = a.c, t = a.t, ku = a.ku, LW = a.LW;
    const int ldw1 = a.ldw - 1;
    const int p = r + (c - t) + j * c;
    const int q = (j == 0) ? r : p - c;
    const int hi = min(p + t, n - 1);
    const int ce = min(hi + c, n - 1);
    const int m = FULL ? MT : hi - p + 1;
    const int off = p - q;        // rows q..p-1 above the corner
    const int ncols = ce - p + 1; // B columns p..ce (slot s = column - p)
    // columns with slot >= s_late are loaded after the B wait
    const int s_late = (a.b0 > a.a0) ? min(max(c - 1, m), ncols) : ncols;
    // column p+s, rows p..p+m-1 sit at bbase + s*(ldw-1) + kk
    S *bbase = W + ku + (int64_t)p * a.ldw;

    nbar_sync(BAR_START, NALL); // predecessor ready for A (and early loads)
    if (tid == 0) TRACE2(8);

    // row ownership: corner rows p..hi -> threads 0..m-1; rows q..p-1 -> m..m+off-1
    int ii = -1;
    if (tid < m) ii = off + tid;
    else if (tid - m < off) ii = tid - m;
    C row[MT];
    S *rbase = W + (ku + q - p) + (int64_t)p * a.ldw; // (q+ii, p+k) at rbase + ii + k(ldw-1)
    S *rp = rbase + ii;
    if (ii >= 0) {
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) row[k] = ldg_cg(rp + k * ldw1);
    }
    // early B columns (slots m .. s_late-1), coalesced, into shared memory
    gather_cols_n<S, C, 8>(bbase + m * ldw1, ldw1, m, s_late - m, bcols + m * LW, LW, tid, ntc);
    if (tid == 0) TRACE2(9);

    // row reflector (Alg. 2 lines 3-6) by the owner of row q
    if (ii == 0) {
        C tau, beta;
        house_thread<C, MT, FULL>(row, m, v1, tau, beta);
        scal[0] = tau;
        row[0] = beta;
#pragma unroll
        for (int k = 1; k < MT; ++k)
            if (FULL || k < m) row[k] = C(0);
    }
    nbar_sync(BAR_C, ntc);
    if (tid == 0) TRACE2(10);

    // right application to rows q+1..hi (Alg. 2 lines 8-13), in registers
    const C tau1 = scal[0];
    if (ii >= 1 && tau1 != C(0)) {
        C vr[MT];
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) vr[k] = v1[k];
        const C w = tau1 * dot4<C, MT, FULL>(row, vr, m);
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) row[k] = fma(-w, vr[k], row[k]);
    }
    if (ii >= 0 && ii < off) {
        // rows q..p-1 are final for this step: write back now (coalesced over rows)
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) stg(rp + k * ldw1, row[k]);
    }
    if (tid < m) {
        // corner row p+tid -> B-column slots 0..m-1
#pragma unroll
        for (int k = 0; k < MT; ++k)
            if (FULL || k < m) bcols[tid + k * LW] = row[k];
    }
    nbar_arrive(BAR_A, ntc + 32);  // A stores issued -> release warp publishes 2j+1
    if (tid == 0) TRACE2(11);
    nbar_sync(BAR_C, ntc);

    // column reflector from A[p..hi, p] (Alg. 2 line 15), warp 0
    if (warp == 0) {
        C tau, beta;
        house_warp<C>(bcols, 1, m, v2, tau, beta);
        if (lane == 0) scal[2] = tau;
        __syncwarp();
        for (int kk = lane; kk < m; kk += 32) bcols[kk] = (kk == 0) ? beta : C(0);
    }
    if (tid == 0) TRACE2(12);
    nbar_sync(BAR_W1, ntc + 32);    // v2 ready and predecessor ready for B
    if (tid == 0) TRACE2(13);
    // late B columns (right-end block, written by A of sweep r-1, step j+1)
    if (s_late < ncols) {
        gather_cols_n<S, C, 4>(bbase + s_late * ldw1, ldw1, m, ncols - s_late, bcols + s_late * LW, LW, tid, ntc);
        nbar_sync(BAR_C, ntc);
    }
    const C tau2 = scal[2];

    // left application to columns p+1..ce, one thread per column, in place in smem
    if (tau2 != C(0)) {
        C vv[MT];
#pragma unroll
        for (int kk = 0; kk < MT; ++kk)
            if (FULL || kk < m) vv[kk] = v2[kk];
        for (int sl = 1 + tid; sl < ncols; sl += ntc) {
            C x[MT];
            C *col = bcols + sl * LW;
#pragma unroll
            for (int kk = 0; kk < MT; ++kk)
                if (FULL || kk < m) x[kk] = col[kk];
            const C w = tau2 * dot4<C, MT, FULL>(vv, x, m);
#pragma unroll
            for (int kk = 0; kk < MT; ++kk)
                if (FULL || kk < m) col[kk] = fma(-w, vv[kk], x[kk]);
        }
    }
    nbar_sync(BAR_C, ntc);
    // write rows p..hi of columns p..ce back, coalesced
    scatter_cols_n<S, C>(bbase, ldw1, m, ncols, bcols, LW, tid, ntc);
    if (tid == 0) TRACE2(14);
    nbar_arrive(BAR_B, ntc + 32);   // B stores issued -> release warp publishes 2j+2
}

template <class S, int MT, int NTMAX>
__global__ void __launch_bounds__(NTMAX) pass_v2_kernel(PassArgsV2 a)
{
    using C = typename ComputeOf<S>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *v1 = reinterpret_cast<C *>(smem_raw);
    C *v2 = v1 + MT;
    C *scal = v2 + MT;
    C *bcols = scal + 4;             // [LW * (c + t + 1)]: rows p..hi of columns p..ce
    __shared__ int s_task;

    const int tid = threadIdx.x;
    const int ntc = a.ntc;
    const int NALL = ntc + 64;
    const int warp = tid >> 5, lane = tid & 31;
    const bool is_poll = (warp == (ntc >> 5));
    const bool is_rel = (warp == (ntc >> 5) + 1);
    const int n = a.n, c = a.c, t = a.t;
    const int total = a.batch * a.nsweeps;

    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(a.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int r = task / a.batch;
        const int J = sweep_len(n, c, t, r);
        const int Jp = r > 0 ? sweep_len(n, c, t, r - 1) : 0;
        int *prog = a.progress + (int64_t)mat * n;
        S *W = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;

        if (is_poll) {
            // ---------------- POLL warp: acquire the predecessor's progress
            for (int j = 0; j < J; ++j) {
                if (lane == 0 && r > 0) {
                    TRACE2(0);
                    wait_geq(prog + r - 1, min(2 * j + a.a0, 2 * Jp));
                    TRACE2(1);
                }
                __syncwarp();
                nbar_arrive(BAR_START, NALL);
                if (lane == 0 && r > 0 && a.b0 > a.a0) {
                    TRACE2(2);
                    wait_geq(prog + r - 1, min(2 * j + a.b0, 2 * Jp));
                    TRACE2(3);
                }
                __syncwarp();
                nbar_sync(BAR_W1, ntc + 32);
            }
        } else if (is_rel) {
            // ---------------- RELEASE warp: fence + publish this sweep's progress
            for (int j = 0; j < J; ++j) {
                nbar_arrive(BAR_START, NALL);
                nbar_sync(BAR_A, ntc + 32);
                if (lane == 0) {
                    TRACE2(4);
                    st_release(prog + r, 2 * j + 1);
                    TRACE2(5);
                }
                __syncwarp();
                nbar_sync(BAR_B, ntc + 32);
                if (lane == 0) {
                    TRACE2(6);
                    st_release(prog + r, 2 * j + 2);
                    TRACE2(7);
                }
                __syncwarp();
            }
        } else {
            // ---------------- COMPUTE warps
            for (int j = 0; j < J; ++j) {
                const int p = r + (c - t) + j * c;
                const int hi = min(p + t, n - 1);
                if (hi - p + 1 == MT)
                    compute_step<S, MT, true>(a, W, mat, r, j, v1, v2, scal, bcols, NALL);
                else
                    compute_step<S, MT, false>(a, W, mat, r, j, v1, v2, scal, bcols, NALL);
            }
        }
    }
}

} // namespace bb
