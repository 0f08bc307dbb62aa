// bb_svals.cu -- SVD stage 3 on the device: the singular
// values of the upper bidiagonal B = bidiag(d, e) that stage 2 returns.
//
// The paper hands (d, e) to LAPACK's BDSDC for this stage.  On
// B200 every singular value is computed independently by bisection on the
// Golub-Kahan form: the 2n x 2n symmetric tridiagonal T with zero diagonal and
// off-diagonal (d_0, e_0, d_1, e_1, ..., d_{n-1}) has eigenvalues +-sigma_i,
// so for x > 0
//     #{ sigma_i < x } = #{ negative pivots of T - x I } - n,
// the pivots being the Sturm recurrence q_0 = -x, q_k = -x - b_k^2 / q_{k-1}
// (a zero pivot is replaced by -pivmin, pivmin = tiny * max(1, max b_k^2), as
// in LAPACK dstebz).  The count is monotone in x, so sigma_i (i-th smallest)
// is the point where the count passes i; one thread owns one i and narrows
// [0, Gershgorin bound] by QUADRISECTION (three independent recurrences per
// sweep of b -- instruction-level parallelism for the division chains -- and
// two bits per sweep) until the interval is below 2 ulp of its upper end or
// of the tiny absolute floor eps * bound (normwise accuracy, reading Q15).
// Arithmetic: fp64 for every input dtype; output descending, fp64.
#include "bandbidiag.h"

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace {

template <class S> __device__ __forceinline__ double to_f64(S v) { return (double)v; }
template <> __device__ __forceinline__ double to_f64<__half>(__half v) { return (double)__half2float(v); }

// b2[k] = b_k^2 of the Golub-Kahan tridiagonal, k = 0 .. 2n-2 (b_{2i} = d_i,
// b_{2i+1} = e_i); bound[0] = Gershgorin bound of T, bound[1] = max b^2
template <class S>
__global__ void gk_prep_kernel(const S *__restrict__ d, int64_t sd, const S *__restrict__ e, int64_t se, int n,
                               int batch, double *__restrict__ b2, double *__restrict__ bound)
{
    const int mat = blockIdx.y;
    if (mat >= batch) return;
    const S *dm = d + mat * sd;
    const S *em = e + mat * se;
    double *bm = b2 + (int64_t)mat * (2 * n);
    double gmax = 0, bmax = 0;
    for (int k = threadIdx.x + blockIdx.x * blockDim.x; k < 2 * n - 1; k += blockDim.x * gridDim.x) {
        const double v = (k & 1) ? to_f64(em[k >> 1]) : to_f64(dm[k >> 1]);
        bm[k] = v * v;
        const double vn = (k + 1 < 2 * n - 1) ? fabs((k & 1) ? to_f64(dm[(k + 1) >> 1]) : to_f64(em[(k + 1) >> 1])) : 0.0;
        gmax = fmax(gmax, fabs(v) + vn);
        bmax = fmax(bmax, v * v);
    }
    // block reduction, then one atomic per block (values are >= 0: bit order)
    __shared__ double sg[32], sb[32];
    for (int o = 16; o > 0; o >>= 1) {
        gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, o));
        bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        sg[threadIdx.x >> 5] = gmax;
        sb[threadIdx.x >> 5] = bmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            gmax = fmax(gmax, sg[w]);
            bmax = fmax(bmax, sb[w]);
        }
        atomicMax(reinterpret_cast<unsigned long long *>(bound + 2 * mat), (unsigned long long)__double_as_longlong(gmax));
        atomicMax(reinterpret_cast<unsigned long long *>(bound + 2 * mat + 1),
                  (unsigned long long)__double_as_longlong(bmax));
    }
}

// 1/q by the hardware approximation + two Newton steps (within ~1 ulp; the
// count only needs the sign of each pivot): a quarter of an IEEE division's
// dependent chain
__device__ __forceinline__ double fast_rcp(double q)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    double e = fma(-q, r, 1.0);
    r = fma(r, e, r);
    e = fma(-q, r, 1.0);
    return fma(r, e, r);
}

// one thread per singular value index i (ascending): quadrisection on the
// Sturm count of T - x I
__global__ void __launch_bounds__(128) gk_bisect_kernel(const double *__restrict__ b2, const double *__restrict__ bound,
                                                        int n, int batch, double *__restrict__ sigma, int64_t ss)
{
    const int mat = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (mat >= batch || i >= n) return;
    const double *bm = b2 + (int64_t)mat * (2 * n);
    const double U = bound[2 * mat] * (1.0 + 4e-16) + 1e-300;
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, bound[2 * mat + 1]);
    const double floor_abs = 2.220446049250313e-16 * U;
    double lo = 0.0, hi = U;
    const int need = i + 1; // sigma_i is the smallest x with count(x) >= i + 1 (x just above sigma_i)
    for (int it = 0; it < 40; ++it) {
        const double w = hi - lo;
        if (w <= fmax(2.0 * 2.220446049250313e-16 * hi, floor_abs)) break;
        const double x1 = lo + 0.25 * w, x2 = lo + 0.5 * w, x3 = lo + 0.75 * w;
        double q1 = -x1, q2 = -x2, q3 = -x3;
        int c1 = q1 < 0, c2 = q2 < 0, c3 = q3 < 0;
        for (int k = 0; k < 2 * n - 1; ++k) {
            const double bb = __ldg(bm + k);
            if (fabs(q1) < pivmin) q1 = -pivmin;
            if (fabs(q2) < pivmin) q2 = -pivmin;
            if (fabs(q3) < pivmin) q3 = -pivmin;
            q1 = fma(-bb, fast_rcp(q1), -x1);
            q2 = fma(-bb, fast_rcp(q2), -x2);
            q3 = fma(-bb, fast_rcp(q3), -x3);
            c1 += q1 < 0;
            c2 += q2 < 0;
            c3 += q3 < 0;
        }
        c1 -= n;
        c2 -= n;
        c3 -= n;
        if (c1 >= need) hi = x1;
        else if (c2 >= need) {
            lo = x1;
            hi = x2;
        } else if (c3 >= need) {
            lo = x2;
            hi = x3;
        } else
            lo = x3;
    }
    sigma[mat * ss + (n - 1 - i)] = 0.5 * (lo + hi);
}

template <class S>
bb_status launch_svals(int64_t n, int64_t batch, const void *d, int64_t sd, const void *e, int64_t se, double *sigma,
                       int64_t ss, void *ws, cudaStream_t st)
{
    double *b2 = reinterpret_cast<double *>(ws);
    double *bound = b2 + batch * 2 * n;
    if (cudaMemsetAsync(bound, 0, sizeof(double) * 2 * batch, st) != cudaSuccess) return BB_ERR_CUDA;
    const int thr = 256;
    dim3 g1((unsigned)std::min<int64_t>((2 * n + thr - 1) / thr, 64), (unsigned)batch);
    gk_prep_kernel<S><<<g1, thr, 0, st>>>(reinterpret_cast<const S *>(d), sd, reinterpret_cast<const S *>(e), se,
                                          (int)n, (int)batch, b2, bound);
    dim3 g2((unsigned)((n + 127) / 128), (unsigned)batch);
    gk_bisect_kernel<<<g2, 128, 0, st>>>(b2, bound, (int)n, (int)batch, sigma, ss);
    return cudaGetLastError() == cudaSuccess ? BB_SUCCESS : BB_ERR_CUDA;
}

} // namespace

extern "C" {

bb_status bb_bidiag_svals_workspace_size(int64_t n, int64_t batch, size_t *bytes)
{
    if (!bytes || n < 0 || batch < 0) return BB_ERR_INVALID_VALUE;
    *bytes = sizeof(double) * (size_t)(batch * 2 * n + 2 * batch);
    return BB_SUCCESS;
}

bb_status bb_bidiag_svals_batched(int64_t n, bb_dtype dtype, int64_t batch, const void *d, int64_t stride_d,
                                  const void *e, int64_t stride_e, double *sigma, int64_t stride_sigma,
                                  void *workspace, size_t workspace_bytes, void *stream)
{
    if (n < 0 || batch < 0) return BB_ERR_INVALID_VALUE;
    if (dtype != BB_F16 && dtype != BB_F32 && dtype != BB_F64) return BB_ERR_NOT_SUPPORTED;
    if (n == 0 || batch == 0) return BB_SUCCESS;
    if (!d || !sigma || (n > 1 && !e)) return BB_ERR_INVALID_VALUE;
    if (batch > 1 && (stride_d < n || stride_e < n - 1 || stride_sigma < n)) return BB_ERR_INVALID_VALUE;
    if (n > (1 << 28) || batch > 65535) return BB_ERR_NOT_SUPPORTED;
    size_t need = 0;
    bb_bidiag_svals_workspace_size(n, batch, &need);
    if (!workspace || workspace_bytes < need) return BB_ERR_INVALID_VALUE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    switch (dtype) {
    case BB_F16: return launch_svals<__half>(n, batch, d, stride_d, e, stride_e, sigma, stride_sigma, workspace, st);
    case BB_F32: return launch_svals<float>(n, batch, d, stride_d, e, stride_e, sigma, stride_sigma, workspace, st);
    case BB_F64: return launch_svals<double>(n, batch, d, stride_d, e, stride_e, sigma, stride_sigma, workspace, st);
    }
    return BB_ERR_NOT_SUPPORTED;
}

bb_status bb_bidiag_svals(int64_t n, bb_dtype dtype, const void *d, const void *e, double *sigma, void *workspace,
                          size_t workspace_bytes, void *stream)
{
    return bb_bidiag_svals_batched(n, dtype, 1, d, n, e, n - 1, sigma, n, workspace, workspace_bytes, stream);
}

} // extern "C"
