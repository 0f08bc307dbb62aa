// Step-latency microbenchmark for the v4 step design (fp64/fp32, c=128, t=16):
// window in shared memory, each thread owns one row (right application) then
// one column (left application); reflector scalars computed redundantly by
// every thread (no broadcast barrier), dot products taken against x / y
// directly so they overlap the norm.  G warp-groups run independent windows
// concurrently in one CTA (the multi-sweep CTA's SM sharing).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o step4 step4.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#ifndef MT
#define MT 17
#endif
#define CB 128

__device__ __forceinline__ void bsync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

template <class C> struct RS;
template <> struct RS<double> { static __device__ __forceinline__ double rsq(double x) { return rsqrt(x); } };
template <> struct RS<float> { static __device__ __forceinline__ float rsq(float x) { return rsqrtf(x); } };

// scalars of the reflector of x (x0 = alpha, ssq = sum_{k>=1} x_k^2):
// tau, rho = 1/(alpha - beta), beta
template <class C>
__device__ __forceinline__ void refl(C alpha, C ssq, C &tau, C &rho, C &beta)
{
    if (ssq == C(0)) { tau = 0; rho = 0; beta = alpha; return; }
    const C tot = fma(alpha, alpha, ssq);
    const C rn = RS<C>::rsq(tot);
    const C nrm = tot * rn;
    beta = alpha >= C(0) ? -nrm : nrm;
    tau = fma(fabs(alpha), rn, C(1));
    rho = C(1) / (alpha - beta);
}

template <class C, int MODE>
__global__ void k_step(C *gout, long long *out, int iters, int G, int NT, int LDT, int LDW)
{
    extern __shared__ __align__(16) unsigned char sm_raw[];
    C *sm = reinterpret_cast<C *>(sm_raw);
    const int g = threadIdx.x / NT, tid = threadIdx.x - g * NT;
    const int c = CB, t = MT - 1;
    const int nR = c + t, nL = c + t, off = c;   // j > 0: q = p - c
    C *T = sm + (size_t)g * (LDT * MT + LDW * (c + 1) + 64);
    C *W = T + LDT * MT;
    C *scal = W + LDW * (c + 1);
    for (int e = tid; e < LDT * MT + LDW * (c + 1); e += NT) T[e] = C(1) / C(1 + (e * 7919) % 97);
    bsync(1 + g, NT);
    long long t0 = clock64(), tR = 0, tL = 0;
    for (int it = 0; it < iters; ++it) {
        long long a0 = clock64();
        // ---- right application: row q (x) at T[0 + k*LDT], rows q+1.. at T[1+i + k*LDT]
        if (MODE == 0) {
            if (tid < nR) {
                C x[MT], a[MT];
#pragma unroll
                for (int k = 0; k < MT; ++k) x[k] = T[k * LDT];
                C *rp = T + 1 + tid;
#pragma unroll
                for (int k = 0; k < MT; ++k) a[k] = rp[k * LDT];
                C s4[4] = {0, 0, 0, 0}, q4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int k = 1; k < MT; ++k) {
                    s4[k & 3] = fma(a[k], x[k], s4[k & 3]);
                    q4[k & 3] = fma(x[k], x[k], q4[k & 3]);
                }
                C tau, rho, beta;
                refl<C>(x[0], (q4[0] + q4[1]) + (q4[2] + q4[3]), tau, rho, beta);
                const C w = tau * fma(rho, (s4[0] + s4[1]) + (s4[2] + s4[3]), a[0]);
                const C wr = w * rho;
                rp[0] = a[0] - w;
#pragma unroll
                for (int k = 1; k < MT; ++k) rp[k * LDT] = fma(-wr, x[k], a[k]);
            }
        } else {
            // one warp computes the scalars, broadcast through shared memory
            C a[MT];
            C *rp = T + 1 + tid;
            if (tid < nR) {
#pragma unroll
                for (int k = 0; k < MT; ++k) a[k] = rp[k * LDT];
            }
            if (tid < 32) {
                const C xv = tid < MT ? T[tid * LDT] : C(0);
                C q = (tid > 0) ? xv * xv : C(0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
                const C alpha = __shfl_sync(0xffffffffu, xv, 0);
                C tau, rho, beta;
                refl<C>(alpha, q, tau, rho, beta);
                if (tid < MT) scal[8 + tid] = tid == 0 ? C(1) : xv * rho;
                if (tid == 0) scal[0] = tau;
            }
            bsync(1 + g, NT);
            if (tid < nR) {
                const C tau = scal[0];
                C s4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int k = 0; k < MT; ++k) s4[k & 3] = fma(a[k], scal[8 + k], s4[k & 3]);
                const C w = tau * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
#pragma unroll
                for (int k = 0; k < MT; ++k) rp[k * LDT] = fma(-w, scal[8 + k], a[k]);
            }
        }
        bsync(1 + g, NT);
        long long a1 = clock64();
        // ---- left application: column p (y) at T[off + kk], columns p+1..p+t in T, rest in W
        if (MODE == 0) {
            if (tid < nL) {
                C y[MT], b[MT];
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) y[kk] = T[off + kk];
                C *cp = tid < t ? T + off + (1 + tid) * LDT : W + (tid - t) * LDW;
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) b[kk] = cp[kk];
                C s4[4] = {0, 0, 0, 0}, q4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int kk = 1; kk < MT; ++kk) {
                    s4[kk & 3] = fma(b[kk], y[kk], s4[kk & 3]);
                    q4[kk & 3] = fma(y[kk], y[kk], q4[kk & 3]);
                }
                C tau, rho, beta;
                refl<C>(y[0], (q4[0] + q4[1]) + (q4[2] + q4[3]), tau, rho, beta);
                const C w = tau * fma(rho, (s4[0] + s4[1]) + (s4[2] + s4[3]), b[0]);
                const C wr = w * rho;
                cp[0] = b[0] - w;
#pragma unroll
                for (int kk = 1; kk < MT; ++kk) cp[kk] = fma(-wr, y[kk], b[kk]);
            }
        } else {
            C b[MT];
            C *cp = tid < t ? T + off + (1 + tid) * LDT : W + (tid - t) * LDW;
            if (tid < nL) {
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) b[kk] = cp[kk];
            }
            if (tid < 32) {
                const C yv = tid < MT ? T[off + tid] : C(0);
                C q = (tid > 0) ? yv * yv : C(0);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
                const C alpha = __shfl_sync(0xffffffffu, yv, 0);
                C tau, rho, beta;
                refl<C>(alpha, q, tau, rho, beta);
                if (tid < MT) scal[40 + tid] = tid == 0 ? C(1) : yv * rho;
                if (tid == 0) scal[1] = tau;
            }
            bsync(1 + g, NT);
            if (tid < nL) {
                const C tau = scal[1];
                C s4[4] = {0, 0, 0, 0};
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) s4[kk & 3] = fma(b[kk], scal[40 + kk], s4[kk & 3]);
                const C w = tau * ((s4[0] + s4[1]) + (s4[2] + s4[3]));
#pragma unroll
                for (int kk = 0; kk < MT; ++kk) cp[kk] = fma(-w, scal[40 + kk], b[kk]);
            }
        }
        bsync(1 + g, NT);
        long long a2 = clock64();
        tR += a1 - a0;
        tL += a2 - a1;
    }
    long long t1 = clock64();
    if (tid == 0) {
        out[g * 4 + 0] = (t1 - t0) / iters;
        out[g * 4 + 1] = tR / iters;
        out[g * 4 + 2] = tL / iters;
    }
    if (tid == 0) gout[g] = T[5];
}

template <class C>
void run(const char *name, int mode, int G)
{
    const int NT = 160, LDT = 145 + (sizeof(C) == 8 ? 0 : 0), LDW = MT;
    size_t per = (size_t)LDT * MT + (size_t)LDW * (CB + 1) + 64;
    size_t smem = per * G * sizeof(C);
    C *g;
    long long *o;
    cudaMalloc(&g, 64 * sizeof(C));
    cudaMalloc(&o, 64 * sizeof(long long));
    auto kern = mode == 0 ? k_step<C, 0> : k_step<C, 1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, NT * G, smem>>>(g, o, 200, G, NT, LDT, LDW);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s mode=%d G=%d: %s step %lld cyc (R %lld, L %lld)\n", name, mode, G, cudaGetErrorString(e), h[0], h[1],
           h[2]);
    cudaFree(g);
    cudaFree(o);
}

int main()
{
    for (int G : {1, 2, 3, 4}) {
        run<double>("f64", 0, G);
        run<double>("f64", 1, G);
    }
    for (int G : {1, 3, 6}) {
        run<float>("f32", 0, G);
        run<float>("f32", 1, G);
    }
    return 0;
}
