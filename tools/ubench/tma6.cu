// Scratch: one TMA box load (the segment-ring kernel's chunk load) in isolation.
// ./tma6 MODE: 0 3-D param map (.tile), 1 3-D param map, 2 2-D param map,
// 3 3-D map in global memory, 4 2-D map, 16-byte-aligned box start row
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void k(const __grid_constant__ CUtensorMap tmap, const CUtensorMap *gmap, double *out, int c0, int c1,
                  int rows, int cols)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double *buf = reinterpret_cast<double *>(sm + 128);
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(rows * cols * 8) : "memory");
        if (MODE == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(0), "r"(su32(&bar)) : "memory");
        else if (MODE == 1)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(0), "r"(su32(&bar)) : "memory");
        else if (MODE == 2 || MODE == 4)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(c0), "r"(c1), "r"(su32(&bar)) : "memory");
        else {
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gmap) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su32(buf)), "l"(reinterpret_cast<uint64_t>(gmap)), "r"(c0), "r"(c1), "r"(0), "r"(su32(&bar)) : "memory");
        }
    }
    unsigned ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(ok) : "r"(su32(&bar)) : "memory");
    for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv)
{
    const int mode = atoi(argv[1]);
    const int ldw = 130, n = 300, rows = 96, cols = 32;
    const int c0 = mode == 4 ? 32 : 33;
    std::vector<double> h((size_t)ldw * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, rows * cols * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    alignas(64) CUtensorMap map;
    const int rank = (mode == 2 || mode == 4) ? 2 : 3;
    cuuint64_t dims[3] = {(cuuint64_t)ldw, (cuuint64_t)n, 1};
    cuuint64_t strides[2] = {(cuuint64_t)ldw * 8, (cuuint64_t)ldw * n * 8};
    cuuint32_t box[3] = {(cuuint32_t)rows, (cuuint32_t)cols, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
    printf("mode %d encode %d query %d sizeof %zu\n", mode, (int)r, (int)q, sizeof(CUtensorMap));
    int smem = rows * cols * 8 + 256;
    void (*kern)(const CUtensorMap, const CUtensorMap *, double *, int, int, int, int) =
        mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : k<4>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<1, 128, smem>>>(map, gm, o, c0, 280, rows, cols);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> ho(rows * cols);
    cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int cc = 0; cc < cols; ++cc)
        for (int rr = 0; rr < rows; ++rr) {
            double want = (280 + cc < n) ? (double)((280 + cc) * ldw + c0 + rr) : 0.0;
            if (ho[cc * rows + rr] != want) ++bad;
        }
    printf("mode %d: %s bad %d\n", mode, cudaGetErrorString(e), bad);
    return e != cudaSuccess;
}
