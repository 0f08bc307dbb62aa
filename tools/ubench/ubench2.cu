// Load-phase microbenchmark: the exact loads of one bulge step (fp64, c=128, t=16):
// 145 tall rows x 17 (stride ldw-1) into registers + 110 wide columns x 17 gathered
// into shared memory; 224 threads; windows of different CTAs at different places.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <int U>
__global__ void k_step_loads(const double *W, int ldw, long long *out, double *sink, int spacing, int reps) {
    __shared__ double sm[17 * 130];
    const int tid = threadIdx.x, ntc = 160;
    const int ldw1 = ldw - 1;
    long long best = 1LL << 60;
    double acc = 0;
    for (int rep = 0; rep < reps; ++rep) {
        const int p = 200 + blockIdx.x * spacing + rep * 7;
        const double *base = W + (long long)p * ldw;
        __syncthreads();
        long long c0 = clock64();
        if (tid < ntc) {
            double row[17];
            if (tid < 145) {
#pragma unroll
                for (int k = 0; k < 17; ++k) row[k] = __ldcg(base + tid + k * ldw1);
            }
            // gather 110 columns x 17 rows
            const int rows = 17, total = rows * 110;
            int e = tid, kc = e / rows, ii = e - kc * rows;
            const int dk = ntc / rows, dii = ntc - dk * rows;
            const double *g = base + 17 * ldw1 + 100;
            while (e < total) {
                double buf[U]; int so[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    so[u] = -1;
                    if (e < total) { buf[u] = __ldcg(g + kc * ldw1 + ii); so[u] = ii + kc * 17; }
                    e += ntc; ii += dii; kc += dk; if (ii >= rows) { ii -= rows; ++kc; }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) if (so[u] >= 0) sm[so[u]] = buf[u];
            }
            if (tid < 145) {
#pragma unroll
                for (int k = 0; k < 17; ++k) acc += row[k];
            }
        }
        __syncthreads();
        long long c1 = clock64();
        if (c1 - c0 < best) best = c1 - c0;
        acc += sm[tid % 1000];
    }
    if (tid == 0) out[blockIdx.x] = best;
    sink[blockIdx.x * blockDim.x + tid] = acc;
}

int main() {
    int n = 32768, ldw = 161;
    double *W; cudaMalloc(&W, (size_t)n * ldw * 8 + (1 << 20)); cudaMemset(W, 0, (size_t)n * ldw * 8);
    double *sink; cudaMalloc(&sink, 1 << 24);
    long long *out; cudaMalloc(&out, 4096 * 8);
    long long h[4096];
    for (int grid : {1, 148}) {
        for (int pass = 0; pass < 2; ++pass) {
            k_step_loads<8><<<grid, 224>>>(W, ldw, out, sink, 200, 20);
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, mn = 1LL << 60; double avg = 0;
        for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; avg += h[i]; }
        printf("U=8 grid=%d: step loads min %lld avg %.0f max %lld cycles\n", grid, mn, avg / grid, mx);
        k_step_loads<16><<<grid, 224>>>(W, ldw, out, sink, 200, 20); cudaDeviceSynchronize();
        cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
        avg = 0; for (int i = 0; i < grid; ++i) avg += h[i];
        printf("U=16 grid=%d: avg %.0f cycles\n", grid, avg / grid);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
