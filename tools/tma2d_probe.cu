// tma2d_probe.cu -- isolates the raw-input A load: a 2-D tiled TMA box {136 px, 16 planes} of an
// fp32 [planes][HW] tensor into shared memory, copied back and checked on the host.
// nvcc -gencode arch=compute_100a,code=sm_100a -Ipaper_1704_04428_b200/csrc tools/tma2d_probe.cu -o tools/tma2d_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace clb;

// 2-D tiled load (CTA-local): coords (c0 innermost, c1)
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* m, uint64_t* bar, void* smem, int32_t c0, int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap m, float* out, int p0, int plane0, int bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, (uint32_t)bytes);
        tma_load_2d(&m, &bar, sm, p0, plane0);
    }
    mbar_wait(&bar, 0);
    const float* f = reinterpret_cast<const float*>(sm);
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = f[i];
}

int main(int argc, char** argv) {
    const int HW = argc > 1 ? atoi(argv[1]) : 3136, P = argc > 2 ? atoi(argv[2]) : 128, BOX = 136;
    std::vector<float> h((size_t)HW * P);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float* d = nullptr;
    float* o = nullptr;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 16 * BOX * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)HW, (cuuint64_t)P};
    cuuint64_t strides[1] = {(cuuint64_t)HW * 4};
    cuuint32_t box[2] = {(cuuint32_t)BOX, 16};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    const int bytes = 16 * BOX * 4;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int p0 : {0, 4, 8, HW - 60, -4, 2}) {
        probe<<<1, 128, bytes + 1024>>>(map, o, p0, 16, bytes);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> g(16 * BOX);
        cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int c = 0; c < 16; ++c)
            for (int x = 0; x < BOX; ++x) {
                const float want = (p0 + x < HW && p0 + x >= 0) ? h[(size_t)(16 + c) * HW + p0 + x] : 0.0f;
                bad += g[c * BOX + x] != want;
            }
        printf("p0=%d err=%s bad=%d\n", p0, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
