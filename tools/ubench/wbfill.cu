// Write-back / fill microbenchmark for the v4 slot layout (fp64, c=128, t=16,
// G=3): 147 column segments of 19 rows between shared memory and a banded
// global array, as (0) warp per column STG, (1) flattened STG all lanes,
// (2) warp per column cp.async (LDGSTS), (3) flattened LDG.cg batched + STS,
// with a large or small dynamic shared-memory allocation (L1 carveout).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o wbfill wbfill.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void k(double *W, int ldw, long long *out, int reps)
{
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5, nt = blockDim.x;
    const int NC = 147, NR = 19, TP = 25;
    for (int i = tid; i < NC * TP; i += nt) sm[i] = i;
    __syncthreads();
    double *Wb = W + (size_t)blockIdx.x * 400 * ldw;
    long long best = 1LL << 60;
    for (int rep = 0; rep < reps; ++rep) {
        __syncthreads();
        const unsigned long long t0 = gt();
        const int p0 = 10 + (rep & 7);
        if (MODE == 0) {
            for (int k = warp; k < NC; k += nw) {
                double *g = Wb + (long)(p0 + k) * (ldw - 1) + p0;
                if (lane < NR) g[lane] = sm[k * TP + lane];
            }
        } else if (MODE == 1) {
            for (int e = tid; e < NC * NR; e += nt) {
                const int k = e / NR, i = e - k * NR;
                Wb[(long)(p0 + k) * (ldw - 1) + p0 + i] = sm[k * TP + i];
            }
        } else if (MODE == 2) {
            for (int k = warp; k < NC; k += nw) {
                const double *g = Wb + (long)(p0 + k) * (ldw - 1) + p0;
                if (lane < NR)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                     (unsigned)__cvta_generic_to_shared(sm + k * TP + lane)),
                                 "l"(g + lane)
                                 : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else {
            for (int e0 = tid; e0 < NC * NR; e0 += 16 * nt) {
                double v[16];
                int so[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) {
                    const int e = e0 + u * nt;
                    so[u] = -1;
                    if (e < NC * NR) {
                        const int k = e / NR, i = e - k * NR;
                        v[u] = __ldcg(Wb + (long)(p0 + k) * (ldw - 1) + p0 + i);
                        so[u] = k * TP + i;
                    }
                }
#pragma unroll
                for (int u = 0; u < 16; ++u)
                    if (so[u] >= 0) sm[so[u]] = v[u];
            }
        }
        __syncthreads();
        const unsigned long long t1 = gt();
        if (rep > 2 && (long long)(t1 - t0) < best) best = t1 - t0;
    }
    if (tid == 0) out[blockIdx.x] = best;
}

template <int MODE> void run(int smem_kb, int nthreads, int blocks)
{
    const int ldw = 161;
    double *W;
    long long *o;
    cudaMalloc(&W, (size_t)blocks * 400 * ldw * 8 + 4096 * 8);
    cudaMemset(W, 0, (size_t)blocks * 400 * ldw * 8);
    cudaMalloc(&o, blocks * 8);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
    k<MODE><<<blocks, nthreads, smem_kb * 1024>>>(W, ldw, o, 20);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, o, blocks * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < blocks; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("mode %d smem %3d KB threads %d blocks %3d: %s  best %lld ns (block 0), max over blocks %lld ns\n", MODE,
           smem_kb, nthreads, blocks, cudaGetErrorString(e), h[0], mx);
    cudaFree(W);
    cudaFree(o);
}

int main()
{
    for (int sk : {40, 210}) {
        for (int b : {1, 148}) {
            run<0>(sk, 160, b);
            run<1>(sk, 160, b);
            run<2>(sk, 64, b);
            run<3>(sk, 64, b);
            run<3>(sk, 128, b);
        }
    }
    return 0;
}
