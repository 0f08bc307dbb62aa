// Scratch: clock64 probes inside one panel link (copy of v5_panel with probes).
#include "../../paper_2510_12705_b200/csrc/bb_pass_v5.cuh"
#include <cstdio>
using namespace bb;
#define PROBE(i) do { if (lane == 0 && g == 5) tp[i] = clock64(); } while (0)
template <class C, int MT, int GT>
__device__ void panel_probe(C *pan, int ks, int ls, C *vs, int VP, int lane, long long *tp)
{
    const bool member = lane < GT;
    C *mine = pan + lane * ls;
    C q_spec = 0, a_spec = 0;
    if (member) {
        C q4[4] = {0, 0, 0, 0};
        for (int k = 1; k < MT; ++k) { const C v = mine[k * ks]; q4[k & 3] = fma(v, v, q4[k & 3]); }
        q_spec = (q4[0] + q4[1]) + (q4[2] + q4[3]);
        a_spec = mine[0];
    }
#pragma unroll 1
    for (int g = 0; g < GT; ++g) {
        PROBE(0);
        C *src = pan + g * ks + g * ls;
        C *own = mine + g * ks;
        const bool upd = member && lane > g;
        C x[MT], a[MT];
#pragma unroll
        for (int k = 1; k < MT; ++k) x[k] = src[k * ks];
        if (upd) {
#pragma unroll
            for (int k = 0; k < MT; ++k) a[k] = own[k * ks];
        }
        const C xl = (lane < MT) ? src[lane * ks] : C(0);
        const C enext = (upd) ? own[MT * ks] : C(0);
        const C q = __shfl_sync(0xffffffffu, q_spec, g);
        const C alpha = __shfl_sync(0xffffffffu, a_spec, g);
        PROBE(1);
        C tau = 0, rho = 0, beta = alpha;
        bool nz = q > C(0);
        C *v = vs + g * VP;
        bool slow = nz && !v5_scalars<C>(alpha, q, tau, rho, beta);
        PROBE(2);
        __syncwarp();
        PROBE(3);
        if (upd) {
            C s4[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 1; k < MT; ++k) s4[k & 3] = fma(a[k], x[k], s4[k & 3]);
            if (nz) {
                const C w = tau * fma(rho, (s4[0] + s4[1]) + (s4[2] + s4[3]), a[0]);
                const C wr = w * rho;
                a[0] -= w;
#pragma unroll
                for (int k = 1; k < MT; ++k) a[k] = fma(-wr, x[k], a[k]);
            }
            C q4[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 2; k < MT; ++k) q4[k & 3] = fma(a[k], a[k], q4[k & 3]);
            q4[0] = fma(enext, enext, q4[0]);
            q_spec = (q4[0] + q4[1]) + (q4[2] + q4[3]);
            a_spec = a[1];
            PROBE(4);
#pragma unroll
            for (int k = 0; k < MT; ++k) own[k * ks] = a[k];
        }
        PROBE(5);
        if (!slow) {
            if (lane < MT) v[lane] = (lane == 0) ? C(1) : (nz ? rho * xl : C(0));
            if (MT > 32 && lane == 0) v[32] = nz ? rho * x[MT > 32 ? 32 : 1] : C(0);
            if (lane == 0) v[MT] = tau;
        }
        if (lane < MT) src[lane * ks] = (lane == 0) ? beta : C(0);
        if (MT > 32 && lane == 0) src[32 * ks] = C(0);
        __syncwarp();
        PROBE(6);
    }
}
template <class C, int MT, int GT>
__global__ void kp(C *out, long long *tp, int LA)
{
    extern __shared__ __align__(16) unsigned char sm[];
    C *Win = reinterpret_cast<C *>(sm);
    C *vs = Win + 64 * LA;
    for (int i = threadIdx.x; i < 64 * LA; i += blockDim.x) Win[i] = C(1) / (1 + (i * 7919) % 101) - C(0.3);
    __syncthreads();
    if (threadIdx.x < 32) panel_probe<C, MT, GT>(Win, LA, 1, vs, (MT + 2) & ~1, threadIdx.x, tp);
    out[threadIdx.x] = Win[threadIdx.x];
}
int main()
{
    double *out; long long *tp;
    cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&tp, 64 * 8);
    int LA = 177; size_t smem = (64 * LA + 64 * 40) * 8;
    cudaFuncSetAttribute(kp<double, 33, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int r = 0; r < 3; ++r) { kp<double, 33, 16><<<1, 32, smem>>>(out, tp, LA); cudaDeviceSynchronize(); }
    const char *nm[] = {"loads+shfl", "scalars", "syncwarp", "dot+update+next q", "store own", "v/src+sync"};
    for (int i = 0; i < 6; ++i) printf("%-20s %lld\n", nm[i], tp[i + 1] - tp[i]);
    printf("total %lld\n", tp[6] - tp[0]);
}
