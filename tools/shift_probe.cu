// shift_probe.cu -- can a tcgen05 (SWIZZLE_128B, K-major) smem descriptor start at an
// arbitrary 128-byte row inside a 1024-byte swizzle atom?  One CTA: TMA-load 136 rows of A,
// B = "identity on the first 8 K-columns", MMA with A starting at row j (j = 0..7) and
// descriptor base_offset either 0 or ((addr >> 7) & 7); read D back: it must equal A rows
// [j, j + 128) x K-columns 0..7.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace clb;

__global__ void probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int j,
                      int use_base_offset, float* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;                 // 136 rows x 128 B
    uint8_t* sb = smem + 136 * 128 + 1024 - (136 * 128) % 1024;   // 16 rows x 128 B, 1024-aligned
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, 136 * 128 + 16 * 128);
        tma_load_3d(&ma, &bar, sa, 0, 0, 0);
        tma_load_3d(&mb, &bar, sb, 0, 0, 0);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a_addr = smem_u32(sa) + (uint32_t)j * 128u;
        uint64_t da = umma_desc_kmajor(a_addr, 128);
        if (use_base_offset) da |= (uint64_t)((a_addr >> 7) & 7u) << 49;
        const uint64_t db = umma_desc_kmajor(smem_u32(sb), 128);
        mma_tf32_ss(tmem, da, db, idesc_tf32(128, 16), 0u);
        mma_commit(&mbar);
    }
    mbar_wait(&mbar, 0);
    tc_fence_after();
    uint32_t r[16];
    tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16), r);
    tmem_ld_wait();
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < 16; ++c) out[row * 16 + c] = __uint_as_float(r[c]);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 32);
}

using EncT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    EncT enc = (EncT)f;
    const int rows = 256;
    std::vector<float> ha(rows * 32), hb(16 * 32, 0.0f);
    for (int r = 0; r < rows; ++r)
        for (int k = 0; k < 32; ++k) ha[r * 32 + k] = (float)((r * 7 + k * 3) % 61) - 30.0f;   // tf32-exact
    for (int n = 0; n < 8; ++n) hb[n * 32 + n] = 1.0f;                                          // identity on k 0..7
    float *da, *db, *dout;
    cudaMalloc(&da, ha.size() * 4);
    cudaMalloc(&db, hb.size() * 4);
    cudaMalloc(&dout, 128 * 16 * 4);
    cudaMemcpy(da, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMap ma, mb;
    cuuint64_t dimsa[3] = {32, (cuuint64_t)rows, 1}, stra[2] = {128, 128ull * rows};
    cuuint32_t boxa[3] = {32, 136, 1}, es[3] = {1, 1, 1};
    cuuint64_t dimsb[3] = {32, 16, 1}, strb[2] = {128, 128 * 16};
    cuuint32_t boxb[3] = {32, 16, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, da, dimsa, stra, boxa, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, db, dimsb, strb, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    std::vector<float> ho(128 * 16);
    for (int bo = 0; bo < 2; ++bo) {
        for (int j = 0; j < 8; ++j) {
            probe<<<1, 128, 48 * 1024>>>(ma, mb, j, bo, dout);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(ho.data(), dout, ho.size() * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < 8; ++n)
                    if (ho[m * 16 + n] != ha[(m + j) * 32 + n]) ++bad;
            printf("base_offset=%s j=%d: %s, mismatches %d/1024\n", bo ? "(addr>>7)&7" : "0", j,
                   cudaGetErrorString(e), bad);
        }
    }
    return 0;
}
