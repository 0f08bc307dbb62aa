// Does a barrier / CTA-scope release wait for outstanding global stores?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *g, long long *out, int mode) {
    __shared__ int flag;
    const int tid = threadIdx.x;
    long long t0 = 0, t1 = 0, t2 = 0;
    for (int it = 0; it < 20; ++it) {
        __syncthreads();
        t0 = clock64();
        // burst: each thread 17 stores at stride 160 (coalesced per k)
#pragma unroll
        for (int k = 0; k < 17; ++k) g[(size_t)blockIdx.x * 8192 + tid + k * 160 + it * 3000] = k + it;
        t1 = clock64();
        if (mode == 1) asm volatile("bar.sync 1, 160;" ::: "memory");
        if (mode == 2) { if (tid == 0) asm volatile("st.release.cta.shared.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&flag)), "r"(it) : "memory"); }
        if (mode == 3) { asm volatile("bar.sync 1, 160;" ::: "memory"); if (tid == 0) asm volatile("st.release.cta.shared.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&flag)), "r"(it) : "memory"); }
        if (mode == 4) { if (tid == 0) asm volatile("st.volatile.shared.b32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&flag)), "r"(it) : "memory"); }
        if (mode == 5) { if (tid == 0) asm volatile("fence.acq_rel.cta;" ::: "memory"); }
        t2 = clock64();
    }
    if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t1; }
}
int main() {
    double *g; cudaMalloc(&g, 1 << 28); long long *o; cudaMalloc(&o, 64); long long h[2];
    const char *nm[] = {"nothing", "bar.sync", "st.release.cta.shared", "bar.sync+st.release.cta", "st.volatile.shared", "fence.acq_rel.cta"};
    for (int mode = 0; mode < 6; ++mode) {
        k<<<148, 160>>>(g, o, mode); cudaDeviceSynchronize();
        k<<<148, 160>>>(g, o, mode); cudaDeviceSynchronize();
        cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
        printf("%-26s issue %5lld  after-op %6lld cycles (thread 0)\n", nm[mode], h[0], h[1]);
    }
}
