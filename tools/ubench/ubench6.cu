// Is reading data just written by another SM slower than reading static L2 data?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *buf, int *flag, long long *out, int mode, int iters) {
    const int tid = threadIdx.x;
    const int N = 5000;   // ~40 KB
    for (int it = 0; it < iters; ++it) {
        double *region = buf + (size_t)(it % 16) * 8192;
        if (blockIdx.x == 0) {
            if (mode == 1) {
                for (int e = tid; e < N; e += blockDim.x) region[e] = e + it;
            }
            __syncthreads();
            if (tid == 0) { __threadfence(); atomicAdd(flag, 1); }
        } else {
            if (tid == 0) { while (atomicAdd(flag, 0) < it + 1) {} __threadfence(); }
            __syncthreads();
            long long c0 = clock64();
            double v[16]; double acc = 0;
            int e0 = tid;
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = (e0 + u * 160 < N) ? __ldcg(region + e0 + u * 160) : 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) acc += v[u];
#pragma unroll
            for (int u = 0; u < 16; ++u) v[u] = (e0 + (u + 16) * 160 < N) ? __ldcg(region + e0 + (u + 16) * 160) : 0;
#pragma unroll
            for (int u = 0; u < 16; ++u) acc += v[u];
            __syncthreads();
            long long c1 = clock64();
            if (tid == 0) out[it] = c1 - c0;
            if (acc == -1.0) out[0] = 0;
        }
    }
}
int main() {
    double *buf; cudaMalloc(&buf, 16 * 8192 * 8 * 2); cudaMemset(buf, 0, 16 * 8192 * 8 * 2);
    int *flag; cudaMalloc(&flag, 4);
    long long *out; cudaMalloc(&out, 1000 * 8); long long h[1000];
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(flag, 0, 4);
        k<<<2, 160>>>(buf, flag, out, mode, 200); cudaDeviceSynchronize();
        cudaMemcpy(h, out, 200 * 8, cudaMemcpyDeviceToHost);
        long long s = 0; for (int i = 50; i < 200; ++i) s += h[i];
        printf("mode %d (%s): reader 40KB load = %lld cycles avg\n", mode, mode ? "just written by other SM" : "static", s / 150);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
