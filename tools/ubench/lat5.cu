// Scratch microbenchmark (not product): fp64 latencies on B200 for the panel design.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n)
{
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    double x = a, y = b;
    long long t0, t1;
    // dependent DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
    // dependent DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;
    t1 = clock64();
    if (threadIdx.x == 0) cyc[1] = (t1 - t0);
    // dependent LDS chain (pointer chasing through smem index)
    int idx = threadIdx.x & 7;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v) & 7; x += v; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[2] = (t1 - t0);
    // rsqrt.approx.f64 chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[3] = (t1 - t0);
    // dependent DSETP-or chain
    bool p = false;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { p |= (x != (double)i); x = p ? x : y; }
    t1 = clock64();
    if (threadIdx.x == 0) cyc[4] = (t1 - t0);
    // shfl double
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[5] = (t1 - t0);
    // DFMA throughput: 8 independent chains, 1 warp
    double z[8];
    for (int j = 0; j < 8; ++j) z[j] = a + j;
    t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) z[j] = fma(z[j], y, 1e-300);
    t1 = clock64();
    if (threadIdx.x == 0) cyc[6] = (t1 - t0);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += z[j];
    out[threadIdx.x] = x + s + (p ? 1 : 0);
}
int main()
{
    double *out; long long *cyc;
    cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64 * 8);
    const int n = 4096;
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(out, cyc, 0.5, 0.999, n); cudaDeviceSynchronize();
    const char *names[] = {"DFMA dep", "DADD dep", "LDS dep(+DADD)", "RSQ64 dep(+DADD)", "DSETP-or dep", "SHFL f64 dep", "DFMA 8 chains (per iter)"};
    for (int i = 0; i < 7; ++i) printf("%-26s %.1f cycles/iter\n", names[i], (double)cyc[i] / n);
    // 4 warps and 8 warps throughput of the 8-chain DFMA
    for (int w : {4, 8, 16}) {
        k<<<1, 32 * w>>>(out, cyc, 0.5, 0.999, n); cudaDeviceSynchronize();
        printf("warps=%d: DFMA 8-chain %.1f cycles/iter (warp 0)\n", w, (double)cyc[6] / n);
    }
    return 0;
}
