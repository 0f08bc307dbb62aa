// Slot-fill microbenchmark: the exact fill loop of bb_pass_v3.cuh vs a warp-per-column loop.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }

template <int U>
__global__ void k_fill(const double *W, int ldw, int ku, int n, long long *out, int mode) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, ntg = 160;
    const int c = 128, t = 16, G = 3, WT = t + G, LDT = 131, LDW = 19;
    double *T = sm, *Wr = sm + LDT * WT;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 10; ++rep) {
        const int p0 = 1000 + blockIdx.x * 200 + rep * 128, q0 = p0 - c, trow0 = q0 + WT;
        __syncthreads();
        long long c0 = clock64();
        if (mode == 0) {
            const int late0 = p0 + c - 1;
            const int nWc = late0 - (p0 + WT);
            for (int part = 0; part < 2; ++part) {
                const int rows = part == 0 ? LDT : WT;
                const int ncol = part == 0 ? WT : nWc;
                const int i0 = part == 0 ? trow0 : p0;
                const int j0 = part == 0 ? p0 : p0 + WT;
                double *dst0 = part == 0 ? T : Wr;
                const int ld = part == 0 ? LDT : LDW;
                const int tot = rows * ncol;
                int e = tid, k = e / rows, ii = e - k * rows;
                const int dk = ntg / rows, dii = ntg - dk * rows;
                while (e < tot) {
                    double v[U]; int o[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        o[u] = -1;
                        if (e < tot) {
                            const int i = i0 + ii, jc = j0 + k;
                            const int rho = ku + i - jc;
                            const bool ok = (rho >= 0 && rho < ldw);
                            v[u] = ok ? ldcg(W + rho + (long long)jc * ldw) : 0.0;
                            o[u] = ii + k * ld;
                        }
                        e += ntg; ii += dii; k += dk;
                        if (ii >= rows) { ii -= rows; ++k; }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) if (o[u] >= 0) dst0[o[u]] = v[u];
                }
            }
        } else {
            // warp per column: T columns (131 rows), then W columns (19 rows)
            const int warp = tid >> 5, lane = tid & 31;
            double v[8];
            // T: 19 columns over 5 warps, 131 rows = 5 lane-iterations
            for (int kb = warp; kb < WT; kb += 5) {
                const double *src = W + (ku + trow0 - (p0 + kb)) + (long long)(p0 + kb) * ldw;
#pragma unroll
                for (int u = 0; u < 5; ++u) v[u] = (lane + 32 * u < LDT) ? ldcg(src + lane + 32 * u) : 0.0;
#pragma unroll
                for (int u = 0; u < 5; ++u) if (lane + 32 * u < LDT) T[lane + 32 * u + kb * LDT] = v[u];
            }
            for (int kb = warp; kb < c - 1 - WT; kb += 5) {
                const int jc = p0 + WT + kb;
                const double *src = W + (ku + p0 - jc) + (long long)jc * ldw;
                if (lane < WT) Wr[lane + kb * LDW] = ldcg(src + lane);
            }
        }
        __syncthreads();
        long long c1 = clock64();
        if (c1 - c0 < best) best = c1 - c0;
    }
    if (tid == 0) out[blockIdx.x] = best;
}

int main() {
    int n = 32768, ldw = 161, ku = 144;
    double *W; cudaMalloc(&W, (size_t)n * ldw * 8); cudaMemset(W, 0, (size_t)n * ldw * 8);
    long long *out; cudaMalloc(&out, 4096 * 8); long long h[148];
    int smem = (131 * 19 + 19 * 128) * 8;
    cudaFuncSetAttribute(k_fill<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_fill<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode) for (int grid : {1, 148}) {
        k_fill<16><<<grid, 160, smem>>>(W, ldw, ku, n, out, mode); cudaDeviceSynchronize();
        k_fill<16><<<grid, 160, smem>>>(W, ldw, ku, n, out, mode); cudaDeviceSynchronize();
        cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < grid; ++i) avg += h[i];
        printf("mode %d (%s) grid %d: %.0f cycles\n", mode, mode ? "warp/column" : "kernel loop U=16", grid, avg / grid);
    }
    k_fill<4><<<1, 160, smem>>>(W, ldw, ku, n, out, 0); cudaDeviceSynchronize();
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost); printf("U=4: %lld\n", h[0]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
