// Scratch: v5_panel (shared memory) vs v5_panel_reg (registers) on the same random panel.
#include "../../paper_2510_12705_b200/csrc/bb_pass_v5.cuh"
#include <cstdio>
#include <cstdlib>
#include <vector>
using namespace bb;
template <int MT, int GT, bool REG>
__global__ void k(float *gp, float *gv, int ks, int ls, int size, int VP)
{
    extern __shared__ float sm[];
    float *pan = sm, *vs = sm + size, *xb = vs + GT * VP;
    for (int i = threadIdx.x; i < size; i += 32) pan[i] = gp[i];
    __syncwarp();
    if (REG) v5_panel_reg<float, MT, GT>(pan, ks, ls, vs, VP, xb, threadIdx.x);
    else v5_panel<float, MT, GT>(pan, ks, ls, vs, VP, xb, threadIdx.x);
    __syncwarp();
    for (int i = threadIdx.x; i < size; i += 32) gp[i] = pan[i];
    for (int i = threadIdx.x; i < GT * VP; i += 32) gv[i] = vs[i];
}
template <int MT, int GT>
void run(int ksmode)
{
    const int L = MT + GT - 1, LA = 101;
    const int ks = ksmode ? LA : 1, ls = ksmode ? 1 : LA;
    const int size = LA * L + 64, VP = (MT + 2) & ~1;
    std::vector<float> h(size);
    srand(1);
    for (auto &x : h) x = (rand() / (float)RAND_MAX) * 2 - 1;
    float *p1, *p2, *v1, *v2;
    cudaMalloc(&p1, size * 4); cudaMalloc(&p2, size * 4); cudaMalloc(&v1, GT * VP * 4); cudaMalloc(&v2, GT * VP * 4);
    cudaMemcpy(p1, h.data(), size * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(p2, h.data(), size * 4, cudaMemcpyHostToDevice);
    int smem = (size + GT * VP + 64) * 4;
    cudaFuncSetAttribute(k<MT, GT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<MT, GT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<MT, GT, false><<<1, 32, smem>>>(p1, v1, ks, ls, size, VP);
    k<MT, GT, true><<<1, 32, smem>>>(p2, v2, ks, ls, size, VP);
    std::vector<float> a(size), b(size), va(GT * VP), vb(GT * VP);
    cudaMemcpy(a.data(), p1, size * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), p2, size * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(va.data(), v1, GT * VP * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(vb.data(), v2, GT * VP * 4, cudaMemcpyDeviceToHost);
    int dp = 0, dv = 0, first = -1;
    for (int i = 0; i < size; ++i) if (a[i] != b[i]) { ++dp; if (first < 0) first = i; }
    for (int i = 0; i < GT * VP; ++i) if (va[i] != vb[i]) ++dv;
    printf("MT=%d GT=%d ksmode=%d: panel diffs %d (first %d: %g vs %g), v diffs %d  err=%s\n", MT, GT, ksmode, dp, first,
           first >= 0 ? a[first] : 0.f, first >= 0 ? b[first] : 0.f, dv, cudaGetErrorString(cudaGetLastError()));
}
int main()
{
    run<17, 32>(1); run<17, 32>(0); run<33, 32>(1); run<33, 32>(0); run<17, 16>(1); run<17, 8>(0); run<33, 16>(1);
    return 0;
}
