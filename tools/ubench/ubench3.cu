// Step-compute microbenchmark: one bulge step (fp64, c=128, t=16, MT=17) with the
// window already in shared memory, 160 threads, timing each phase with clock64.
#include <cstdio>
#include <cuda_runtime.h>
#define MT 17
#define C 128
#define NT 160
#define LT 145   // tall rows (c+t+1)
#define LW 17

__device__ __forceinline__ void bsync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

__global__ void k_step(double *g, long long *out, int iters) {
    __shared__ double T[LT * MT];        // tall: rows q..hi x cols p..hi, column-major
    __shared__ double B[LW * (C + MT)];   // B columns p..ce, rows p..hi
    __shared__ double v1[MT], v2[MT], sc[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < LT * MT; i += NT) T[i] = g[i] + 1.0;
    for (int i = tid; i < LW * (C + MT); i += NT) B[i] = g[i + 3000] + 2.0;
    __syncthreads();
    long long acc[6] = {0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
        long long t0 = clock64();
        // --- row reflector from T[0 + k*LT] by one thread
        if (tid == 0) {
            double x[MT], s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
            for (int k = 0; k < MT; ++k) x[k] = T[k * LT];
#pragma unroll
            for (int k = 0; k < MT; k += 4) {
                s0 = fma(x[k], x[k], s0);
                if (k + 1 < MT) s1 = fma(x[k + 1], x[k + 1], s1);
                if (k + 2 < MT) s2 = fma(x[k + 2], x[k + 2], s2);
                if (k + 3 < MT) s3 = fma(x[k + 3], x[k + 3], s3);
            }
            double nrm = sqrt((s0 + s1) + (s2 + s3));
            double alpha = x[0], beta = alpha >= 0 ? -nrm : nrm;
            double tau = (beta - alpha) / beta, rcp = 1.0 / (alpha - beta);
            v1[0] = 1.0;
#pragma unroll
            for (int k = 1; k < MT; ++k) v1[k] = x[k] * rcp;
            sc[0] = tau * 1e-3;
        }
        bsync(1, NT);
        long long t1 = clock64();
        // --- right apply, rows 1..LT-1 from smem, one row per thread
        if (tid >= 1 && tid < LT) {
            double x[MT], vv[MT];
#pragma unroll
            for (int k = 0; k < MT; ++k) { x[k] = T[tid + k * LT]; vv[k] = v1[k]; }
            double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
            for (int k = 0; k < MT; k += 4) {
                s0 = fma(x[k], vv[k], s0);
                if (k + 1 < MT) s1 = fma(x[k + 1], vv[k + 1], s1);
                if (k + 2 < MT) s2 = fma(x[k + 2], vv[k + 2], s2);
                if (k + 3 < MT) s3 = fma(x[k + 3], vv[k + 3], s3);
            }
            double w = sc[0] * ((s0 + s1) + (s2 + s3));
#pragma unroll
            for (int k = 0; k < MT; ++k) T[tid + k * LT] = fma(-w, vv[k], x[k]);
        }
        bsync(1, NT);
        long long t2 = clock64();
        // --- column reflector by warp 0 from T[128 + kk]
        if (warp == 0) {
            double x = lane < MT ? T[128 + lane] : 0.0;
            double s = x * x;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
            double alpha = __shfl_sync(0xffffffff, x, 0);
            double nrm = sqrt(s), beta = alpha >= 0 ? -nrm : nrm;
            double rcp = 1.0 / (alpha - beta);
            if (lane < MT) v2[lane] = lane == 0 ? 1.0 : x * rcp;
            if (lane == 0) sc[2] = (beta - alpha) / beta * 1e-3;
        }
        bsync(1, NT);
        long long t3 = clock64();
        // --- left apply: columns 1..C+MT-2, one per thread, from smem B
        for (int sl = 1 + tid; sl < C + MT - 1; sl += NT) {
            double x[MT], vv[MT];
#pragma unroll
            for (int k = 0; k < MT; ++k) { x[k] = B[k + sl * LW]; vv[k] = v2[k]; }
            double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
            for (int k = 0; k < MT; k += 4) {
                s0 = fma(x[k], vv[k], s0);
                if (k + 1 < MT) s1 = fma(x[k + 1], vv[k + 1], s1);
                if (k + 2 < MT) s2 = fma(x[k + 2], vv[k + 2], s2);
                if (k + 3 < MT) s3 = fma(x[k + 3], vv[k + 3], s3);
            }
            double w = sc[2] * ((s0 + s1) + (s2 + s3));
#pragma unroll
            for (int k = 0; k < MT; ++k) B[k + sl * LW] = fma(-w, vv[k], x[k]);
        }
        bsync(1, NT);
        long long t4 = clock64();
        acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3;
    }
    if (tid == 0) for (int k = 0; k < 4; ++k) out[k] = acc[k] / iters;
    g[tid] = T[tid] + B[tid];
}

int main() {
    double *g; cudaMalloc(&g, 1 << 20); cudaMemset(g, 0, 1 << 20);
    long long *out; cudaMalloc(&out, 64); long long h[4];
    k_step<<<1, NT>>>(g, out, 100); cudaDeviceSynchronize();
    k_step<<<1, NT>>>(g, out, 1000); cudaDeviceSynchronize();
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("row refl %lld  right apply %lld  col refl %lld  left apply %lld  total %lld cycles\n", h[0], h[1], h[2], h[3], h[0] + h[1] + h[2] + h[3]);
    k_step<<<148, NT>>>(g, out, 1000); cudaDeviceSynchronize();
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("(148 CTAs) row refl %lld  right apply %lld  col refl %lld  left apply %lld\n", h[0], h[1], h[2], h[3]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
