// Scratch microbenchmark: the unit kernel's panel chain in isolation.
#include "../../paper_2510_12705_b200/csrc/bb_pass_v5.cuh"
#include <cstdio>
using namespace bb;
template <class C, int MT, int GT>
__global__ void kpanel(C *out, long long *cyc, int LA, int reps)
{
    extern __shared__ __align__(16) unsigned char sm[];
    C *Win = reinterpret_cast<C *>(sm);
    C *vs = Win + 64 * LA;
    for (int i = threadIdx.x; i < 64 * LA; i += blockDim.x) Win[i] = C(1) / (1 + (i * 7919) % 101) - C(0.3);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x < 32) v5_panel<C, MT, GT>(Win, LA, 1, vs, (MT + 2) & ~1, nullptr, threadIdx.x & 31); // A-style
        __syncthreads();
        if (threadIdx.x < 32) v5_panel<C, MT, GT>(Win + 40, 1, LA, vs, (MT + 2) & ~1, nullptr, threadIdx.x & 31); // B-style
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps / 2;
    out[threadIdx.x] = Win[threadIdx.x];
}
template <class C, int MT, int GT> void run(const char *name, int nthr)
{
    C *out; long long *cyc;
    cudaMalloc(&out, 4096 * sizeof(C)); cudaMallocManaged(&cyc, 64);
    int LA = 177;
    size_t smem = (64 * LA + 64 * 40) * sizeof(C);
    cudaFuncSetAttribute(kpanel<C, MT, GT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kpanel<C, MT, GT><<<1, nthr, smem>>>(out, cyc, LA, 20); cudaDeviceSynchronize();
    kpanel<C, MT, GT><<<1, nthr, smem>>>(out, cyc, LA, 20); cudaDeviceSynchronize();
    printf("%-16s threads=%3d: %lld cycles per panel, %.0f per link\n", name, nthr, cyc[0], (double)cyc[0] / GT);
}
int main()
{
    run<double, 33, 16>("f64 MT33 G16", 32);
    run<double, 33, 16>("f64 MT33 G16", 160);
    run<double, 17, 16>("f64 MT17 G16", 32);
    run<float, 33, 16>("f32 MT33 G16", 32);
    run<double, 33, 32>("f64 MT33 G32", 32);
    return 0;
}
