// Store / bulk-copy pattern costs of the multi-sweep kernel, in isolation.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(double *W, int ldw, long long *out, int mode) {
    extern __shared__ __align__(128) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar))); }
    for (int i = tid; i < 8192; i += blockDim.x) sm[i] = i;
    __syncthreads();
    unsigned phase = 0;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 20; ++rep) {
        const long long base = 2000 + (long long)blockIdx.x * 190 + rep * 17;
        __syncthreads();
        long long c0 = clock64();
        if (mode == 0) { // scatter: warp per column, 17 doubles each, 145 columns
            for (int sl = warp; sl < 145; sl += 5) {
                double *dst = W + 144 + base + (long long)(base + sl) * (ldw - 1);
                if (lane < 17) dst[lane] = sm[sl * 17 + lane];
            }
        } else if (mode == 1) { // scatter with 32-lane aligned chunks (coalesced by element index)
            for (int e = tid; e < 145 * 17; e += 160) {
                int sl = e / 17, kk = e - sl * 17;
                double *dst = W + 144 + base + (long long)(base + sl) * (ldw - 1);
                dst[kk] = sm[e];
            }
        } else if (mode == 2) { // 127 bulk copies of ~1 KB/176 B by warp 0
            if (warp == 0) {
                unsigned mine = 0;
                for (int kc = lane; kc < 127; kc += 32) mine += (kc < 19 ? 1088u : 176u);
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(mine));
                __syncwarp();
                for (int kc = lane; kc < 127; kc += 32) {
                    const double *src = W + ((base + kc) * (ldw - 1) + 160) / 2 * 2;
                    double *dst = sm + kc * 136;
                    unsigned bytes = kc < 19 ? 1088u : 176u;
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)), "l"(src), "r"(bytes), "r"(su(&bar)) : "memory");
                }
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&bar)) : "memory");
            }
            asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n}" ::"r"(su(&bar)), "r"(phase & 1) : "memory");
            ++phase;
        }
        __syncthreads();
        if (mode < 2) { if (tid == 0) __threadfence(); __syncthreads(); }
        long long c1 = clock64();
        if (c1 - c0 < best) best = c1 - c0;
    }
    if (tid == 0) out[blockIdx.x] = best;
}
int main() {
    int n = 32768, ldw = 161;
    double *W; cudaMalloc(&W, (size_t)n * ldw * 8 + (1 << 22)); cudaMemset(W, 0, (size_t)n * ldw * 8);
    long long *o; cudaMalloc(&o, 4096 * 8); long long h[148];
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char *nm[] = {"scatter warp/col (incl fence)", "scatter elementwise (incl fence)", "127 bulk copies"};
    for (int mode = 0; mode < 3; ++mode) for (int grid : {1, 148}) {
        k<<<grid, 160, 200 * 1024>>>(W, ldw, o, mode); cudaDeviceSynchronize();
        cudaMemcpy(h, o, grid * 8, cudaMemcpyDeviceToHost);
        double a = 0; for (int i = 0; i < grid; ++i) a += h[i];
        printf("%-34s grid %3d: %.0f cycles\n", nm[mode], grid, a / grid);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
