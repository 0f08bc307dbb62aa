// bb_kernels.cuh -- sm_100a device code of the band -> bidiagonal reduction.
//
// Row-bulge step = Alg. 2 of arXiv 2510.12705 (text P:189):
//   stage the step's two-sided window in shared memory, build the row
//   reflector from A[q, p..hi] (warp-shuffle norm), apply it from the right to
//   rows q+1..hi, build the column reflector from A[p..hi, p], apply it from
//   the left to columns p+1..ce, write the window back (exact zeros in the
//   annihilated slots).  Geometry (readings Q1-Q3, Q10, Q12 of DESIGN.md):
//     p = r + (c - t) + j*c,  q = (j == 0 ? r : p - c),
//     hi = min(p + t, n - 1), ce = min(hi + c, n - 1), m = hi - p + 1.
//
// Working band: LAPACK general-band storage
// with KL = tw, KU = b + tw, column-major, leading dimension ldw:
//     A(i, j) = W[(ku + i - j) + j * ldw].
// Every window column is one contiguous run of that storage.
//
// Shared-memory window of one step (compute type C):
//   tall  T[ii + k*LT]  rows q..hi   (ii = i - q)  of columns p..hi (k = j - p)
//   wide  R[kk + k'*LW] rows p..hi   (kk = i - p)  of columns hi+1..ce (k' = j - hi - 1)
//   LT, LW odd, so thread-per-column accesses are bank-conflict free.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bb {

template <class S> struct ComputeOf { using type = S; };
template <> struct ComputeOf<__half> { using type = float; };

// ---- global loads that bypass L1 (data produced by other SMs) -------------
__device__ __forceinline__ float ldg_cg(const float *p) { return __ldcg(p); }
__device__ __forceinline__ double ldg_cg(const double *p) { return __ldcg(p); }
__device__ __forceinline__ float ldg_cg(const __half *p)
{
    unsigned short u = __ldcg(reinterpret_cast<const unsigned short *>(p));
    return __half2float(__ushort_as_half(u));
}
__device__ __forceinline__ void stg(float *p, float v) { *p = v; }
__device__ __forceinline__ void stg(double *p, double v) { *p = v; }
__device__ __forceinline__ void stg(__half *p, float v) { *p = __float2half_rn(v); }
__device__ __forceinline__ float absval(float x) { return fabsf(x); }
__device__ __forceinline__ double absval(double x) { return fabs(x); }
__device__ __forceinline__ __half absval(__half x) { return __habs(x); }

// ---- flags: acquire / release at gpu scope --------------------------------
__device__ __forceinline__ int ld_acquire(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed(const int *p)
{
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// poll interval for a progress flag: short when the awaited value is close,
// long when the producer is far behind -- a CTA whose predecessor has not
// started yet must not hammer the flag's L2 line (hundreds of such pollers
// slowed the active groups' L2 traffic, measured)
__device__ __forceinline__ unsigned poll_ns(int have, int need, int near)
{
    return (need - have > near) ? 1024u : 32u;
}
// spin until *p >= need: relaxed polling, one acquire fence on success
__device__ __forceinline__ void wait_geq(const int *p, int need, int near = 2)
{
    int v = ld_relaxed(p);
    if (v < need) {
        do {
            __nanosleep(poll_ns(v, need, near));
            v = ld_relaxed(p);
        } while (v < need);
    }
    fence_acq_rel();
}
__device__ __forceinline__ void st_release(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- warp reductions --------------------------------------------------------
template <class C> __device__ __forceinline__ C warp_sum(C x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
template <class C> __device__ __forceinline__ C warp_max(C x)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

template <class C> struct NormRange;
template <> struct NormRange<double> {
    static __device__ __forceinline__ double lo() { return 1e-280; }
    static __device__ __forceinline__ double hi() { return 1e280; }
};
template <> struct NormRange<float> {
    static __device__ __forceinline__ float lo() { return 1e-25f; }
    static __device__ __forceinline__ float hi() { return 1e25f; }
};

// HH(X) of Alg. 2 line 5, executed by ONE warp.
// x[k*stride], k < m.  Writes v[0..m-1] (v[0] = 1) and returns tau, beta
// (LAPACK dlarfg convention, reading Q7; identity iff x[1:] == 0 exactly,
// reading Q8).  The norm is the plain sum of squares when that is safely in
// range and a max-scaled sum otherwise (no under/overflow).
template <class C>
__device__ __forceinline__ void house_warp(const C *x, int stride, int m, C *v, C &tau, C &beta)
{
    const int lane = threadIdx.x & 31;
    const C alpha = x[0];
    bool nz = false;
    C ssq = 0, amax = 0;
    for (int k = lane; k < m; k += 32) {
        C xv = x[k * stride];
        nz |= (k > 0) && (xv != C(0));
        ssq += xv * xv;
        amax = fmax(amax, fabs(xv));
    }
    nz = __any_sync(0xffffffffu, nz);
    if (!nz) {
        for (int k = lane; k < m; k += 32) v[k] = (k == 0) ? C(1) : C(0);
        tau = 0;
        beta = alpha;
        return;
    }
    ssq = warp_sum(ssq);
    C nrm;
    if (ssq >= NormRange<C>::lo() && ssq <= NormRange<C>::hi()) {
        nrm = sqrt(ssq);
    } else {
        amax = warp_max(amax);
        C s2 = 0;
        for (int k = lane; k < m; k += 32) {
            C y = x[k * stride] / amax;
            s2 += y * y;
        }
        s2 = warp_sum(s2);
        nrm = amax * sqrt(s2);
    }
    beta = (alpha >= C(0)) ? -nrm : nrm;
    tau = (beta - alpha) / beta;
    // v = x / (alpha - beta): a true division -- the reciprocal of a
    // denormal-scale (alpha - beta) overflows (seen in fp32 at n = 1024)
    const C den = alpha - beta;
    for (int k = lane; k < m; k += 32) v[k] = (k == 0) ? C(1) : x[k * stride] / den;
}

// Copy `ncols` columns of `rows` elements from global (column k at g + k*gstride)
// into shared memory (column k at s + k*sstride) with every thread of the CTA.
// U loads per thread are issued back to back before their shared-memory
// stores, so a step's window arrives in ~1 L2 round trip, not one per column.
template <class S, class C, int U>
__device__ __forceinline__ void gather_cols(const S *__restrict__ g, int64_t gstride, int rows, int ncols,
                                            C *__restrict__ s, int sstride)
{
    const int total = rows * ncols;
    if (total <= 0) return;
    const int nthr = blockDim.x;
    int e = threadIdx.x;
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
__device__ __forceinline__ void scatter_cols(S *__restrict__ g, int64_t gstride, int rows, int ncols,
                                             const C *__restrict__ s, int sstride)
{
    const int total = rows * ncols;
    if (total <= 0) return;
    const int nthr = blockDim.x;
    int e = threadIdx.x;
    int k = e / rows, ii = e - k * rows;
    const int dk = nthr / rows, dii = nthr - dk * rows;
    for (; e < total; e += nthr) {
        stg(g + k * gstride + ii, s[ii + k * sstride]);
        ii += dii;
        k += dk;
        if (ii >= rows) { ii -= rows; ++k; }
    }
}

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct PassArgs {
    void *W;            // working bands (batch of them)
    int64_t mat_stride; // elements between matrices
    int ldw, ku, n;
    int c, t, s;        // pass: current bandwidth, tilewidth, dependency distance
    int batch;
    int nsweeps;        // non-empty sweeps per matrix: r in [0, nsweeps)
    int *progress;      // [batch][n] steps completed per sweep (this pass)
    int *counter;       // next task to claim (this pass)
    int LT, LW;         // shared-memory leading dimensions (odd)
    int cycle_T;        // BB_SCHED_CYCLE: the cycle this launch runs
    unsigned long long *trace; // debug: per-step timestamps (nullptr = off)
    int trace_sweeps, trace_steps;
};

// debug tracing: timestamps [wait start, wait end, window staged, stored+released]
#define TRACE_MARK(slot)                                                                         \
    do {                                                                                         \
        if (a.trace && threadIdx.x == 0 && mat == 0 && r < a.trace_sweeps && j < a.trace_steps) \
            a.trace[((int64_t)r * a.trace_steps + j) * 4 + (slot)] = gtimer();                  \
    } while (0)

__device__ __forceinline__ int sweep_len(int n, int c, int t, int r)
{
    int first = r + c - t;
    return first > n - 2 ? 0 : (n - 2 - first) / c + 1;
}

// One row-bulge step (Alg. 2) on matrix `mat`, sweep r, step j.
// Caller guarantees the dependency rule; all threads of the CTA call it.
template <class S>
__device__ void bulge_step(const PassArgs &a, int mat, int r, int j, typename ComputeOf<S>::type *sm)
{
    using C = typename ComputeOf<S>::type;
    const int n = a.n, c = a.c, t = a.t;
    const int p = r + (c - t) + j * c;
    const int q = (j == 0) ? r : p - c;
    const int hi = min(p + t, n - 1);
    const int ce = min(hi + c, n - 1);
    const int m = hi - p + 1;      // reflector length (<= t + 1)
    const int rowsT = hi - q + 1;  // rows of the tall part
    const int nW = ce - hi;        // columns of the wide part
    const int LT = a.LT, LW = a.LW;
    C *T = sm;                     // [LT * (t+1)]
    C *R = T + (size_t)LT * (t + 1); // [LW * c]
    C *v = R + (size_t)LW * c;       // [t+1]
    C *scal = v + (t + 1);           // tau, beta (x2)

    S *W = reinterpret_cast<S *>(a.W) + (int64_t)mat * a.mat_stride;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ku = a.ku;
    const int64_t ldw = a.ldw;

    // ---- stage the window: tall columns p..hi (rows q..hi), wide hi+1..ce (rows p..hi)
    // Column k of either part starts (ldw - 1) elements after column k-1.
    gather_cols<S, C, 8>(W + (ku + q - p) + (int64_t)p * ldw, ldw - 1, rowsT, m, T, LT);
    gather_cols<S, C, 8>(W + (ku + p - (hi + 1)) + (int64_t)(hi + 1) * ldw, ldw - 1, m, nW, R, LW);
    __syncthreads();
    TRACE_MARK(2);

    // ---- row reflector from A[q, p..hi] (Alg. 2 lines 3-6)
    if (warp == 0) {
        C tau, beta;
        house_warp<C>(T, LT, m, v, tau, beta);
        if (lane == 0) { scal[0] = tau; scal[1] = beta; }
        __syncwarp();
        for (int k = lane; k < m; k += 32) T[k * LT] = (k == 0) ? beta : C(0);
    }
    __syncthreads();

    // ---- right application to rows q+1..hi (Alg. 2 lines 8-13)
    {
        const C tau = scal[0];
        if (tau != C(0)) {
            for (int ii = 1 + threadIdx.x; ii < rowsT; ii += blockDim.x) {
                C w = 0;
                for (int k = 0; k < m; ++k) w += T[ii + k * LT] * v[k];
                w *= tau;
                for (int k = 0; k < m; ++k) T[ii + k * LT] -= w * v[k];
            }
        }
    }
    __syncthreads();

    // ---- column reflector from A[p..hi, p] (Alg. 2 line 15)
    const int off = p - q;
    if (warp == 0) {
        C tau, beta;
        house_warp<C>(T + off, 1, m, v, tau, beta);
        if (lane == 0) { scal[2] = tau; scal[3] = beta; }
        __syncwarp();
        for (int k = lane; k < m; k += 32) T[off + k] = (k == 0) ? beta : C(0);
    }
    __syncthreads();

    // ---- left application to columns p+1..ce
    {
        const C tau = scal[2];
        if (tau != C(0)) {
            for (int jj = 1 + threadIdx.x; jj <= ce - p; jj += blockDim.x) {
                C *col = (jj < m) ? (T + off + jj * LT) : (R + (jj - m) * LW);
                C w = 0;
                for (int k = 0; k < m; ++k) w += v[k] * col[k];
                w *= tau;
                for (int k = 0; k < m; ++k) col[k] -= w * v[k];
            }
        }
    }
    __syncthreads();

    // ---- write the window back
    scatter_cols<S, C>(W + (ku + q - p) + (int64_t)p * ldw, ldw - 1, rowsT, m, T, LT);
    scatter_cols<S, C>(W + (ku + p - (hi + 1)) + (int64_t)(hi + 1) * ldw, ldw - 1, m, nW, R, LW);
}

// ---- BB_SCHED_FLAGS: one persistent launch per pass ----------------------
// CTAs claim tasks (matrix-interleaved sweeps) in order with atomicAdd; a
// claimed sweep's predecessor is always held by a running CTA, so the wait
// below always terminates (no co-residency assumption).  Dependency rule
// ("3(R-1) < j", reading Q4): step (r, j) waits until
// progress[r-1] >= min(j + s, J_{r-1}).
template <class S>
__global__ void __launch_bounds__(512) pass_flags_kernel(PassArgs a)
{
    using C = typename ComputeOf<S>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = reinterpret_cast<C *>(smem_raw);
    __shared__ int s_task;
    const int total = a.batch * a.nsweeps;
    for (;;) {
        __syncthreads();
        if (threadIdx.x == 0) s_task = atomicAdd(a.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= total) return;
        const int mat = task % a.batch;
        const int r = task / a.batch;
        const int J = sweep_len(a.n, a.c, a.t, r);
        const int Jp = r > 0 ? sweep_len(a.n, a.c, a.t, r - 1) : 0;
        int *prog = a.progress + (int64_t)mat * a.n;
        for (int j = 0; j < J; ++j) {
            TRACE_MARK(0);
            if (r > 0) {
                if (threadIdx.x == 0) {
                    const int need = min(j + a.s, Jp);
                    while (ld_acquire(prog + r - 1) < need) {
                    }
                }
                __syncthreads();
            }
            TRACE_MARK(1);
            bulge_step<S>(a, mat, r, j, sm);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                st_release(prog + r, j + 1);
            }
            TRACE_MARK(3);
        }
    }
}

// ---- BB_SCHED_CYCLE: the paper's one-launch-per-cycle form --------
// Block (x = sweep r, y = matrix) runs step j = T - s*r if it exists.
template <class S>
__global__ void __launch_bounds__(512) pass_cycle_kernel(PassArgs a)
{
    using C = typename ComputeOf<S>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = reinterpret_cast<C *>(smem_raw);
    const int r = blockIdx.x;
    const int mat = blockIdx.y;
    const int j = a.cycle_T - a.s * r;
    if (r >= a.nsweeps || j < 0 || j >= sweep_len(a.n, a.c, a.t, r)) return;
    bulge_step<S>(a, mat, r, j, sm);
}

// ---- a1: ingest + pack into the working band (zero headroom) --------------
template <class S>
__global__ void pack_kernel(const S *__restrict__ band, int64_t ldband, int64_t stride_band, int b_in,
                            int b_eff, S *__restrict__ W, int64_t mat_stride, int ldw, int ku, int n,
                            int batch)
{
    const int64_t per = (int64_t)n * ldw;
    const int64_t total = per * batch;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mat = idx / per;
        const int64_t rem = idx - mat * per;
        const int jcol = (int)(rem / ldw);
        const int rho = (int)(rem - (int64_t)jcol * ldw);
        const int i = jcol + rho - ku;            // matrix row of this slot
        S val = S(0.0f);
        if (i >= 0 && i <= jcol && jcol - i <= b_eff)
            val = band[mat * stride_band + (b_in + i - jcol) + (int64_t)jcol * ldband];
        W[mat * mat_stride + rem] = val;
    }
}

// ---- a9: extract d, e ------------------------------------------------------
template <class S>
__global__ void extract_kernel(const S *__restrict__ W, int64_t mat_stride, int ldw, int ku, int n, int batch,
                               S *__restrict__ d, int64_t stride_d, S *__restrict__ e, int64_t stride_e,
                               int nonneg)
{
    const int64_t total = (int64_t)n * batch;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mat = idx / n;
        const int i = (int)(idx - mat * n);
        const S *Wm = W + mat * mat_stride;
        S dv = Wm[ku + (int64_t)i * ldw];
        if (nonneg) dv = absval(dv);
        d[mat * stride_d + i] = dv;
        if (i + 1 < n) {
            S ev = Wm[(ku - 1) + (int64_t)(i + 1) * ldw];
            if (nonneg) ev = absval(ev);
            e[mat * stride_e + i] = ev;
        }
    }
}

// ---- BB_FLAG_CHECK_ZEROS (debug) --------------------------------------------
// Count the working-band cells outside the diagonal and the superdiagonal that
// are not exactly zero after the reduction (the structural zeros of P:308 /
// BASELINE north_star; reading Q11): every cell of the n x ldw storage of each
// matrix, A(i, j) = W[(ku + i - j) + j*ldw], except offsets j - i in {0, 1}
// (padding cells, rows outside [0, n), are zero from the pack kernel on).
__device__ __forceinline__ bool cell_nonzero(float v) { return v != 0.f; }
__device__ __forceinline__ bool cell_nonzero(double v) { return v != 0.0; }
__device__ __forceinline__ bool cell_nonzero(__half v) { return __half2float(v) != 0.f; }
template <class S>
__global__ void check_zeros_kernel(const S *__restrict__ W, int64_t mat_stride, int ldw, int ku, int n, int batch,
                                   int *__restrict__ count)
{
    const int64_t per = (int64_t)n * ldw;
    const int64_t total = per * batch;
    int local = 0;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mat = idx / per;
        const int64_t rem = idx - mat * per;
        const int r = (int)(rem % ldw);
        const int off = ku - r; // j - i
        if (off == 0 || off == 1) continue;
        local += cell_nonzero(W[mat * mat_stride + rem]) ? 1 : 0;
    }
    if (local) atomicAdd(count, local);
}

} // namespace bb
