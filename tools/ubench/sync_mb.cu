// Scratch: does compute-sanitizer synccheck accept the kernels' mbarrier idiom
// (init by a block-stride loop, fence + __syncthreads, arrive by one warp,
// try_wait.parity with a suspend hint by another)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void k(int *out, int rounds)
{
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ volatile int cnt;
    for (int i = threadIdx.x; i < 64; i += blockDim.x) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    for (int r = 0; r < rounds; ++r) {
        uint64_t *b = bars + (r % 16);
        const unsigned par = (r / 16) & 1;
        if (warp == 0) {
            if (threadIdx.x == 0) {
                cnt = r + 1;
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
            }
        } else if (warp == 1) {
            while (cnt < r + 1) {
                unsigned ok;
                asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                             : "=r"(ok) : "r"(su32(b)), "r"(par), "r"(20000u) : "memory");
                if (ok) break;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = cnt;
}
int main()
{
    int *o;
    cudaMalloc(&o, 4 * 4);
    k<<<4, 96>>>(o, 40);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
