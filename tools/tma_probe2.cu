// tma_probe2.cu -- is TMA time per instruction, per row, or per byte?  Batches of S loads
// issued back to back (no per-load coordinate math), then one wait for the batch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace clb;

__global__ void probe(const __grid_constant__ CUtensorMap map, int mode, int box_bytes, int batch, int rounds,
                      int nrows_total, int box_rows, int issuers, unsigned long long* cycles, int W) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + batch * box_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < issuers; ++i) mbar_init(&bar[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int w = threadIdx.x / 32;
    if (w >= issuers || (threadIdx.x & 31)) return;
    tma_prefetch_desc(&map);
    const long long t0 = clock64();
    const int per = batch / issuers;
    int row = (blockIdx.x * 977 + w * 131) * box_rows % nrows_total;
    for (int r = 0; r < rounds; ++r) {
        mbar_arrive_expect_tx(&bar[w], per * box_bytes);
        for (int b = 0; b < per; ++b) {
            uint8_t* dst = smem + (w * per + b) * box_bytes;
            if (mode == 1) tma_load_im2col_4d(&map, &bar[w], dst, 0, row % W - 1, (row / W) % W - 1, row / (W * W), 1, 1);
            else tma_load_3d(&map, &bar[w], dst, 0, row, 0);
            row += box_rows;
            if (row + box_rows > nrows_total) row = 0;
        }
        mbar_wait(&bar[w], r & 1);
    }
    if (w == 0) cycles[blockIdx.x] = clock64() - t0;
}

using EncT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncI = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void *f1 = nullptr, *f2 = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q);
    EncT enc_t = (EncT)f1;
    EncI enc_i = (EncI)f2;
    const int rows = 32 * 56 * 56;
    float* buf;
    cudaMalloc(&buf, (size_t)rows * 128);   // 32 fp32 channels per pixel, contiguous pixels
    cudaMemset(buf, 0, (size_t)rows * 128);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    struct Case { int mode, box_rows, row_bytes, batch, issuers, ctas, W; };
    Case cases[] = {
        {0, 128, 128, 8, 1, 148, 56}, {0, 128, 128, 8, 4, 148, 56},
        {1, 128, 128, 8, 1, 148, 224}, {1, 128, 128, 8, 1, 148, 56}, {1, 128, 128, 8, 1, 148, 28},
        {1, 128, 128, 8, 1, 148, 14}, {1, 128, 128, 8, 1, 148, 13}, {1, 128, 128, 8, 1, 148, 7},
        {1, 128, 128, 8, 4, 148, 56}, {1, 128, 128, 8, 4, 148, 13}, {1, 128, 128, 8, 4, 148, 7},
    };
    printf("%-6s %5s %5s %5s %4s %4s %9s %9s %9s %9s\n", "mode", "rows", "rowB", "batch", "iss", "ctas", "ms",
           "TB/s", "B/clk/SM", "clk/load");
    for (const Case& cs : cases) {
        CUtensorMap map;
        const CUtensorMapSwizzle sw = cs.row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
        CUresult r;
        const int W = cs.W, H = cs.W, N = rows / (W * H);
        if (cs.mode == 1) {
            cuuint64_t dims[4] = {32, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t str[3] = {128, 128ull * W, 128ull * W * H};
            int lo[2] = {-1, -1}, up[2] = {-1, -1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            r = enc_i(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, str, lo, up, cs.row_bytes / 4, cs.box_rows,
                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[3] = {32, (cuuint64_t)rows, 1};
            cuuint64_t str[2] = {128, 128ull * rows};
            cuuint32_t box[3] = {(cuuint32_t)cs.row_bytes / 4, (cuuint32_t)cs.box_rows, 1};
            cuuint32_t es[3] = {1, 1, 1};
            r = enc_t(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int box_bytes = cs.box_rows * cs.row_bytes;
        const int rounds = 400;
        const int smem = 1024 + cs.batch * box_bytes + 256;
        probe<<<cs.ctas, 128, smem>>>(map, cs.mode, box_bytes, cs.batch, rounds, N * H * W, cs.box_rows, cs.issuers, cyc, W);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<cs.ctas, 128, smem>>>(map, cs.mode, box_bytes, cs.batch, rounds, N * H * W, cs.box_rows, cs.issuers, cyc, W);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> h(cs.ctas);
        cudaMemcpy(h.data(), cyc, cs.ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (auto v : h) avg += v;
        avg /= cs.ctas;
        const double loads = (double)rounds * cs.batch;
        printf("W=%3d %-6s %5d %5d %5d %4d %4d %9.3f %9.2f %9.1f %9.1f %s\n", cs.W, cs.mode ? "im2col" : "tiled", cs.box_rows,
               cs.row_bytes, cs.batch, cs.issuers, cs.ctas, ms, cs.ctas * loads * box_bytes / ms / 1e9,
               loads * box_bytes / avg, avg / loads, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
