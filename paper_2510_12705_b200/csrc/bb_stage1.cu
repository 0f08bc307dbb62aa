// bb_stage1.cu -- SVD stage 1 on the device: dense n x n
// -> upper band with b superdiagonals by block Householder reflections, the
// "classical block Householder" first stage the paper pairs with its bulge
// chasing.  It produces the banded inputs of the paper's
// known-spectrum accuracy protocol at full scale.
//
// For every block column k = 0, b, 2b, ... (nb = min(b, n - k)):
//   1. QR of the column panel A[k:n, k:k+nb] (Householder, dlarfg
//      convention): a one-CTA panel kernel, the reflectors' dot products
//      taken by the whole CTA at once for every remaining panel column;
//   2. T factor of the block reflector (LAPACK dlarft, forward/columnwise):
//      S = V^T V by GEMM, T built column by column in one CTA;
//   3. trailing update from the left, C <- (I - V T^T V^T) C, as three GEMMs
//      (cuBLAS: the plain library GEMMs of this stage);
//   4. LQ of the row panel A[k:k+nb, k+nb:n] through the QR of its transpose
//      (the same panel kernel on a transposed copy), L written back, zeros
//      to its right; trailing update from the right, C <- C (I - V T V^T).
// After the last block column A is upper banded (offsets 0 .. b); the band is
// written in the LAPACK upper-band layout of the stage-2 input.
// Arithmetic in the storage type (fp64 or fp32).
#include "bandbidiag.h"

#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <vector>

namespace {

template <class T> struct Blas;
template <> struct Blas<double> {
    static cublasStatus_t gemm(cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k,
                               const double *al, const double *A, int lda, const double *B, int ldb, const double *be,
                               double *C, int ldc)
    {
        return cublasDgemm(h, ta, tb, m, n, k, al, A, lda, B, ldb, be, C, ldc);
    }
};
template <> struct Blas<float> {
    static cublasStatus_t gemm(cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k,
                               const float *al, const float *A, int lda, const float *B, int ldb, const float *be,
                               float *C, int ldc)
    {
        return cublasSgemm(h, ta, tb, m, n, k, al, A, lda, B, ldb, be, C, ldc);
    }
};

constexpr int PQR_THREADS = 1024;

template <class T> __device__ __forceinline__ T block_sum(T v, T *red)
{
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    T s = 0;
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : T(0);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// Householder QR of the m x nb panel P (column-major, ldp), one CTA.
// On exit: R in the upper triangle, V (unit diagonal implicit) below it, tau.
// Reflector j (dlarfg, reading Q7): beta = -sign(alpha) ||x||, tau =
// (beta - alpha) / beta, v = [1, x_{1:} / (alpha - beta)]; identity when
// x_{1:} == 0 (tau = 0).  Scaled norm when the plain sum of squares is out of
// range (no under/overflow, reading Q8).
template <class T>
__global__ void __launch_bounds__(PQR_THREADS) panel_qr_kernel(T *P, int ldp, int m, int nb, T *tau)
{
    __shared__ T red[33];
    __shared__ T wsh[512];
    for (int j = 0; j < nb && j < m; ++j) {
        T *x = P + (int64_t)j * ldp + j;
        const int len = m - j;
        T ss = 0, amax = 0;
        for (int i = 1 + threadIdx.x; i < len; i += blockDim.x) {
            ss += x[i] * x[i];
            amax = fmax(amax, fabs(x[i]));
        }
        ss = block_sum(ss, red);
        // max for the scaled path (rare): reuse the sum reduction on a flag
        const T alpha = x[0];
        T tj = 0, beta = alpha, scale = 1;
        bool nz = ss > T(0);
        if (!nz) {
            int any = 0;
            for (int i = 1 + threadIdx.x; i < len; i += blockDim.x) any |= (x[i] != T(0));
            nz = __syncthreads_or(any);
        }
        if (nz) {
            T tot = alpha * alpha + ss;
            const T lo = sizeof(T) == 8 ? T(1e-280) : T(1e-25), hi = sizeof(T) == 8 ? T(1e280) : T(1e25);
            if (!(tot >= lo && tot <= hi)) {
                // scaled: amax over the block, then sum of (x / amax)^2
                for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
                __syncthreads();
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
                __syncthreads();
                T am = fabs(alpha);
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) am = fmax(am, red[w]);
                __syncthreads();
                T s2 = 0;
                for (int i = 1 + threadIdx.x; i < len; i += blockDim.x) {
                    const T y = x[i] / am;
                    s2 += y * y;
                }
                s2 = block_sum(s2, red);
                const T ay = alpha / am;
                tot = am * am * (ay * ay + s2); // only its square root is used below
                const T nrm = am * sqrt(ay * ay + s2);
                beta = alpha >= T(0) ? -nrm : nrm;
            } else {
                const T nrm = sqrt(tot);
                beta = alpha >= T(0) ? -nrm : nrm;
            }
            tj = (beta - alpha) / beta;
            scale = T(1) / (alpha - beta);
        }
        __syncthreads();
        for (int i = 1 + threadIdx.x; i < len; i += blockDim.x) x[i] *= scale; // v (v_0 = 1 implicit)
        __syncthreads();
        // apply H_j = I - tau v v^T to panel columns j+1 .. nb-1: w_c = v . P[j:, c]
        const int nc = nb - j - 1;
        if (nz && nc > 0) {
            for (int c0 = 0; c0 < nc; c0 += 512) {
                const int cn = min(512, nc - c0);
                // one warp per column (strided over columns), lanes over rows
                const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
                for (int c = warp; c < cn; c += nw) {
                    const T *col = P + (int64_t)(j + 1 + c0 + c) * ldp + j;
                    T s = lane == 0 ? col[0] : T(0);
                    for (int i = 1 + lane; i < len; i += 32) s += x[i] * col[i];
                    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                    if (lane == 0) wsh[c] = tj * s;
                }
                __syncthreads();
                for (int c = warp; c < cn; c += nw) {
                    T *col = P + (int64_t)(j + 1 + c0 + c) * ldp + j;
                    const T w = wsh[c];
                    if (lane == 0) col[0] -= w;
                    for (int i = 1 + lane; i < len; i += 32) col[i] -= w * x[i];
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0) {
            x[0] = beta;
            tau[j] = tj;
        }
        __syncthreads();
    }
}

// V (explicit, m x nb, unit diagonal, zeros above) from the factored panel
template <class T>
__global__ void extract_v_kernel(const T *P, int ldp, int m, int nb, T *V, int ldv)
{
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)m * nb;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx / m), i = (int)(idx - (int64_t)c * m);
        V[(int64_t)c * ldv + i] = i < c ? T(0) : (i == c ? T(1) : P[(int64_t)c * ldp + i]);
    }
}

// T factor (dlarft, forward, columnwise) from S = V^T V (nb x nb) and tau:
// T[j][j] = tau_j, T[0:j, j] = -tau_j * T[0:j, 0:j] * S[0:j, j]; one CTA
template <class T>
__global__ void larft_kernel(const T *S, int lds, const T *tau, int nb, T *Tm, int ldt)
{
    for (int idx = threadIdx.x; idx < nb * nb; idx += blockDim.x) Tm[(idx / nb) * ldt + idx % nb] = 0;
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        // y = S[0:j, j]; T[0:j, j] = -tau_j * T[0:j,0:j] y (upper triangular T)
        for (int i = threadIdx.x; i < j; i += blockDim.x) {
            T s = 0;
            for (int l = i; l < j; ++l) s += Tm[l * ldt + i] * S[j * lds + l];
            Tm[j * ldt + i] = -tau[j] * s;
        }
        if (threadIdx.x == 0) Tm[j * ldt + j] = tau[j];
        __syncthreads();
    }
}

// out = transpose of in (rows x cols, column-major) -> (cols x rows)
template <class T>
__global__ void transpose_kernel(const T *in, int ldi, int rows, int cols, T *out, int ldo)
{
    __shared__ T tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = by + y, r = bx + threadIdx.x;
        if (r < rows && c < cols) tile[y][threadIdx.x] = in[(int64_t)c * ldi + r];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = bx + y, c = by + threadIdx.x;
        if (r < rows && c < cols) out[(int64_t)r * ldo + c] = tile[threadIdx.x][y];
    }
}

// row panel A[k:k+nb, k+nb:] <- (R^T, 0): R = upper triangle of the QR of its transpose
template <class T>
__global__ void lq_writeback_kernel(const T *Pt, int ldp, int mt, int nb, T *A, int64_t lda)
{
    // A row panel: element (r, c), r < nb, c < mt; value = R[c][r] if c <= r (lower), else 0
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)nb * mt;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx / nb), r = (int)(idx - (int64_t)c * nb);
        A[(int64_t)c * lda + r] = (c <= r) ? Pt[(int64_t)r * ldp + c] : T(0);
    }
}

// column panel below its R: zero (V lives in the panel buffer copy)
template <class T>
__global__ void zero_below_kernel(T *A, int64_t lda, int m, int nb)
{
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)m * nb;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(idx / m), i = (int)(idx - (int64_t)c * m);
        if (i > c) A[(int64_t)c * lda + i] = T(0);
    }
}

// LAPACK upper band (n, ldband): band[(b + i - j) + j*ldband] = A(i, j), 0 <= j - i <= b
template <class T>
__global__ void dense_to_lapack_band_kernel(const T *A, int64_t lda, int n, int b, T *band, int64_t ldband)
{
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * ldband;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(idx / ldband), r = (int)(idx - (int64_t)j * ldband);
        const int i = j - b + r;
        band[idx] = (r <= b && i >= 0) ? A[(int64_t)j * lda + i] : T(0);
    }
}

cublasHandle_t blas_handle()
{
    static std::mutex mu;
    static std::vector<cublasHandle_t> hs;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)hs.size() <= dev) hs.resize(dev + 1, nullptr);
    if (!hs[dev] && cublasCreate(&hs[dev]) != CUBLAS_STATUS_SUCCESS) hs[dev] = nullptr;
    return hs[dev];
}

size_t stage1_ws_elems(int64_t n, int64_t b)
{
    const int64_t nb = std::min<int64_t>(b, std::max<int64_t>(n, 1));
    // panel copy (n x nb), V (n x nb), W (nb x n), S (nb x nb), T (nb x nb), tau (nb), CV (n x nb)
    return (size_t)(n * nb * 3 + nb * n + 2 * nb * nb + nb + 64);
}

template <class T>
bb_status run_stage1(int64_t n64, int64_t b64, T *A, int64_t lda, T *band, int64_t ldband, int b_out, T *ws,
                     cudaStream_t st)
{
    const int n = (int)n64, b = (int)b64; // b: block size = band width produced (<= n - 1)
    cublasHandle_t h = blas_handle();
    if (!h) return BB_ERR_CUDA;
    std::lock_guard<std::mutex> lk(*[] {
        static std::mutex m;
        return &m;
    }()); // one handle per device: calls serialise on its stream binding
    if (cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return BB_ERR_CUDA;
    cublasSetPointerMode(h, CUBLAS_POINTER_MODE_HOST);
    const int NB = std::min(b, n);
    T *Pp = ws;                       // panel / transposed panel, ld = n
    T *V = Pp + (int64_t)n * NB;      // explicit V, ld = n
    T *W = V + (int64_t)n * NB;       // nb x n work, ld = NB
    T *CV = W + (int64_t)NB * n;      // n x nb work (C V), ld = n
    T *S = CV + (int64_t)n * NB;      // nb x nb
    T *Tm = S + (int64_t)NB * NB;     // nb x nb
    T *tau = Tm + (int64_t)NB * NB;   // nb
    const T one = 1, zero = 0, mone = -1;
    const int thr = 256;
    auto grid = [&](int64_t cnt) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((cnt + thr - 1) / thr, 4096)); };
    for (int k = 0; k < n; k += b) {
        const int nb = std::min(b, n - k);
        const int m = n - k; // rows of the column panel
        // ---- 1-3: QR of A[k:n, k:k+nb], left update of A[k:n, k+nb:n]
        if (m > 1) {
            cudaMemcpy2DAsync(Pp, (size_t)n * sizeof(T), A + (int64_t)k * lda + k, (size_t)lda * sizeof(T),
                              (size_t)m * sizeof(T), nb, cudaMemcpyDeviceToDevice, st);
            panel_qr_kernel<T><<<1, PQR_THREADS, 0, st>>>(Pp, n, m, nb, tau);
            // R back into A, zeros below it
            cudaMemcpy2DAsync(A + (int64_t)k * lda + k, (size_t)lda * sizeof(T), Pp, (size_t)n * sizeof(T),
                              (size_t)m * sizeof(T), nb, cudaMemcpyDeviceToDevice, st);
            zero_below_kernel<T><<<grid((int64_t)m * nb), thr, 0, st>>>(A + (int64_t)k * lda + k, lda, m, nb);
            const int ncol = n - k - nb;
            if (ncol > 0) {
                extract_v_kernel<T><<<grid((int64_t)m * nb), thr, 0, st>>>(Pp, n, m, nb, V, n);
                Blas<T>::gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nb, nb, m, &one, V, n, V, n, &zero, S, NB);
                larft_kernel<T><<<1, 256, 0, st>>>(S, NB, tau, nb, Tm, NB);
                T *C = A + (int64_t)(k + nb) * lda + k;
                // W = V^T C; W = T^T W; C -= V W
                Blas<T>::gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nb, ncol, m, &one, V, n, C, (int)lda, &zero, W, NB);
                Blas<T>::gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nb, ncol, nb, &one, Tm, NB, W, NB, &zero, CV, NB);
                Blas<T>::gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, ncol, nb, &mone, V, n, CV, NB, &one, C, (int)lda);
            }
        }
        // ---- 4: LQ of the row panel A[k:k+nb, k+nb:n] (QR of its transpose)
        const int mt = n - k - nb; // columns right of the band block
        if (mt > 1) {
            T *R = A + (int64_t)(k + nb) * lda + k;
            dim3 tg((unsigned)((nb + 31) / 32), (unsigned)((mt + 31) / 32));
            transpose_kernel<T><<<tg, dim3(32, 8), 0, st>>>(R, (int)lda, nb, mt, Pp, n); // Pp: mt x nb
            const int nq = std::min(nb, mt);
            panel_qr_kernel<T><<<1, PQR_THREADS, 0, st>>>(Pp, n, mt, nb, tau); // min(mt, nb) reflectors, applied to all nb columns
            lq_writeback_kernel<T><<<grid((int64_t)nb * mt), thr, 0, st>>>(Pp, n, mt, nb, R, lda);
            const int nrow = n - k - nb; // trailing rows below the row panel
            if (nrow > 0) {
                extract_v_kernel<T><<<grid((int64_t)mt * nq), thr, 0, st>>>(Pp, n, mt, nq, V, n);
                Blas<T>::gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nq, nq, mt, &one, V, n, V, n, &zero, S, NB);
                larft_kernel<T><<<1, 256, 0, st>>>(S, NB, tau, nq, Tm, NB);
                T *C = A + (int64_t)(k + nb) * lda + (k + nb); // nrow x mt
                // C <- C (I - V T V^T): CV = C V; W = CV T; C -= W V^T
                Blas<T>::gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, nrow, nq, mt, &one, C, (int)lda, V, n, &zero, CV, n);
                Blas<T>::gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, nrow, nq, nq, &one, CV, n, Tm, NB, &zero, W, n);
                Blas<T>::gemm(h, CUBLAS_OP_N, CUBLAS_OP_T, nrow, mt, nq, &mone, W, n, V, n, &one, C, (int)lda);
            }
        } else if (mt == 1) {
            // a single column right of the block: nothing to annihilate (already banded)
        }
    }
    dense_to_lapack_band_kernel<T><<<grid((int64_t)n * ldband), thr, 0, st>>>(A, lda, n, b_out, band, ldband);
    return cudaGetLastError() == cudaSuccess ? BB_SUCCESS : BB_ERR_CUDA;
}

} // namespace

extern "C" {

bb_status bb_dense_to_band_workspace_size(int64_t n, int64_t b, bb_dtype dtype, size_t *bytes)
{
    if (!bytes || n < 0 || b < 1) return BB_ERR_INVALID_VALUE;
    if (dtype != BB_F32 && dtype != BB_F64) return BB_ERR_NOT_SUPPORTED;
    *bytes = stage1_ws_elems(n, b) * (dtype == BB_F64 ? 8 : 4);
    return BB_SUCCESS;
}

bb_status bb_dense_to_band(int64_t n, int64_t b, bb_dtype dtype, void *A, int64_t lda, void *band, int64_t ldband,
                           void *workspace, size_t workspace_bytes, void *stream)
{
    if (n < 0 || b < 1 || lda < n || ldband < b + 1) return BB_ERR_INVALID_VALUE;
    if (dtype != BB_F32 && dtype != BB_F64) return BB_ERR_NOT_SUPPORTED;
    if (n == 0) return BB_SUCCESS;
    if (!A || !band) return BB_ERR_INVALID_VALUE;
    if (n > (1 << 30) / 4) return BB_ERR_NOT_SUPPORTED;
    size_t need = 0;
    bb_dense_to_band_workspace_size(n, b, dtype, &need);
    if (!workspace || workspace_bytes < need) return BB_ERR_INVALID_VALUE;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (dtype == BB_F64)
        return run_stage1<double>(n, std::min<int64_t>(b, std::max<int64_t>(n - 1, 1)), (double *)A, lda,
                                  (double *)band, ldband, (int)b, (double *)workspace, st);
    return run_stage1<float>(n, std::min<int64_t>(b, std::max<int64_t>(n - 1, 1)), (float *)A, lda, (float *)band,
                             ldband, (int)b, (float *)workspace, st);
}

} // extern "C"
