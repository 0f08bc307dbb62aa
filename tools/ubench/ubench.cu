// Microbenchmarks of the latencies that bound one bulge-chasing step on B200.
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void k_clock(long long *out) {
    long long c0 = clock64(); unsigned long long g0 = gt();
    while (gt() - g0 < 100000) {}
    long long c1 = clock64(); unsigned long long g1 = gt();
    out[0] = c1 - c0; out[1] = (long long)(g1 - g0);
}

__global__ void k_chase(const int *next, int steps, long long *out) {
    int i = 0;
    long long c0 = clock64();
    for (int s = 0; s < steps; ++s) i = __ldcg(next + i);
    long long c1 = clock64();
    out[0] = (c1 - c0) / steps; out[1] = i;
}

__global__ void k_dfma(double *io, int steps, long long *out) {
    double x = io[threadIdx.x], y = 1.0000001;
    long long c0 = clock64();
    for (int s = 0; s < steps; ++s) x = fma(x, y, 0.5);
    long long c1 = clock64();
    io[threadIdx.x] = x; if (threadIdx.x == 0) out[0] = (c1 - c0) / steps;
}

// 160 threads each load 17 doubles at stride 160 elements (like a tall part), time to all landed
__global__ void k_rows(const double *W, int stride, long long *out, double *sink) {
    __syncthreads();
    long long c0 = clock64();
    double v[17];
#pragma unroll
    for (int k = 0; k < 17; ++k) v[k] = __ldcg(W + threadIdx.x + k * stride);
    double s = 0;
#pragma unroll
    for (int k = 0; k < 17; ++k) s += v[k];
    __syncthreads();
    long long c1 = clock64();
    if (threadIdx.x == 0) out[0] = c1 - c0;
    sink[threadIdx.x] = s;
}

__global__ void k_sync(long long *out) {
    long long c0 = clock64();
    for (int s = 0; s < 100; ++s) __syncthreads();
    long long c1 = clock64();
    if (threadIdx.x == 0) out[0] = (c1 - c0) / 100;
}

__global__ void k_fence(double *W, int *flag, long long *out) {
    // every thread stores 30 doubles, barrier, thread 0 fence.acq_rel + store
    for (int k = 0; k < 30; ++k) W[threadIdx.x + k * blockDim.x] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long c0 = clock64();
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        long long c1 = clock64();
        asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(1) : "memory");
        long long c2 = clock64();
        __threadfence();
        long long c3 = clock64();
        out[0] = c1 - c0; out[1] = c2 - c1; out[2] = c3 - c2;
    }
}

// ping-pong between two CTAs through a flag in global memory: round-trip latency
__global__ void k_pingpong(int *flags, int iters, long long *out) {
    if (threadIdx.x != 0) return;
    volatile int *f = flags;
    long long c0 = clock64();
    unsigned long long g0 = gt();
    for (int i = 0; i < iters; ++i) {
        if (blockIdx.x == 0) {
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags), "r"(2 * i + 1) : "memory");
            int v; do { asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + 32) : "memory"); } while (v < 2 * i + 1);
        } else {
            int v; do { asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags) : "memory"); } while (v < 2 * i + 1);
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + 32), "r"(2 * i + 1) : "memory");
        }
    }
    if (blockIdx.x == 0) { out[0] = (clock64() - c0) / iters; out[1] = (long long)(gt() - g0) / iters; }
}

int main() {
    long long *d_out; cudaMalloc(&d_out, 64 * sizeof(long long));
    std::vector<long long> h(8);
    auto get = [&]() { cudaDeviceSynchronize(); cudaMemcpy(h.data(), d_out, 8 * sizeof(long long), cudaMemcpyDeviceToHost); };
    k_clock<<<1, 1>>>(d_out); get();
    printf("clock: %lld cycles in %lld ns -> %.0f MHz\n", h[0], h[1], 1e3 * h[0] / (double)h[1]);
    // pointer chase over 8 MB (L2-resident) with random stride
    int N = 2 << 20; std::vector<int> nx(N); for (int i = 0; i < N; ++i) nx[i] = (int)((i * 2654435761u + 12345) % N);
    int *d_nx; cudaMalloc(&d_nx, N * 4); cudaMemcpy(d_nx, nx.data(), N * 4, cudaMemcpyHostToDevice);
    k_chase<<<1, 1>>>(d_nx, 1000, d_out); get(); k_chase<<<1, 1>>>(d_nx, 2000, d_out); get();
    printf("L2 pointer-chase latency (ld.cg): %lld cycles\n", h[0]);
    double *d_io; cudaMalloc(&d_io, 1 << 26); cudaMemset(d_io, 0, 1 << 26);
    k_dfma<<<1, 32>>>(d_io, 1000, d_out); get(); printf("dependent DFMA latency: %lld cycles\n", h[0]);
    k_rows<<<1, 160>>>(d_io, 161, d_out, d_io + (1 << 22)); get(); k_rows<<<1, 160>>>(d_io, 161, d_out, d_io + (1 << 22)); get();
    printf("160 thr x 17 strided doubles (L2 hit): %lld cycles to all landed + sync\n", h[0]);
    k_rows<<<148, 160>>>(d_io, 161, d_out, d_io + (1 << 22)); get();
    printf("  same, 148 CTAs: %lld cycles\n", h[0]);
    k_sync<<<1, 160>>>(d_out); get(); printf("__syncthreads (160 thr): %lld cycles\n", h[0]);
    int *d_flag; cudaMalloc(&d_flag, 4096); cudaMemset(d_flag, 0, 4096);
    k_fence<<<1, 160>>>(d_io, d_flag, d_out); get(); k_fence<<<1, 160>>>(d_io, d_flag, d_out); get();
    printf("fence.acq_rel after 4800 stores: %lld cycles; st.relaxed %lld; threadfence after %lld\n", h[0], h[1], h[2]);
    cudaMemset(d_flag, 0, 4096);
    k_pingpong<<<2, 32>>>(d_flag, 1000, d_out); get();
    printf("flag ping-pong round trip between 2 SMs: %lld cycles = %lld ns\n", h[0], h[1]);
    return 0;
}
