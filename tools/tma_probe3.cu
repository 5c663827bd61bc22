// TMA delivery in the kernel's own pattern: a ring of `stages` smem stages with full/empty
// mbarriers; a producer refills a stage as soon as the consumer frees it (no compute: the
// consumer releases each stage the moment it lands).  Each stage = one A box of 128 rows
// (im2col over 13x13 NHWC images, or tiled) + one tiled B box of 96 rows, 128 B per row (28 KB),
// as in AlexNet conv3 (CTA pair, N = 192).  Issuers: 1 = one thread issues both loads;
// 2 = two warps (A / B), each arriving on the full barrier with its own expect_tx;
// 3 = A split into two 64-row boxes from two warps, B from a third.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1704_04428_b200/csrc
//        tools/tma_probe3.cu -o tools/tma_probe3 -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace clb;

constexpr int kA = 128 * 128, kB = 96 * 128, kStage = kA + kB;

__global__ void ring(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                     const __grid_constant__ CUtensorMap ma64, int a_im2col,
                     int stages, int issuers, int iters, int npix, int W, int nb_rows, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], issuers);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 0 || (issuers >= 2 && warp == 2) || (issuers == 3 && warp == 3)) {
        if (lane == 0) {
            const bool do_a = warp == 0 || warp == 3, do_b = issuers == 1 || warp == 2;
            const int half = issuers == 3 ? (warp == 3 ? 1 : 0) : -1;   // -1: whole 128-row A box
            int stage = 0;
            uint32_t phase = 0;
            int pix = (blockIdx.x * 977) % npix, brow = (blockIdx.x * 131) % nb_rows;
            for (int it = 0; it < iters; ++it) {
                mbar_wait(&empty[stage], phase ^ 1u);
                uint8_t* st = smem + stage * kStage;
                mbar_arrive_expect_tx(&full[stage], (do_a ? (half < 0 ? kA : kA / 2) : 0) + (do_b ? kB : 0));
                if (do_a) {
                    if (a_im2col && half >= 0) {
                        const int q = pix + 64 * half;
                        const int x = q % W, y = (q / W) % W, n = q / (W * W);
                        tma_load_im2col_4d(&ma64, &full[stage], st + half * (kA / 2), 0, x - 1, y - 1, n, 1, 1);
                    } else if (a_im2col) {
                        const int x = pix % W, y = (pix / W) % W, n = pix / (W * W);
                        tma_load_im2col_4d(&ma, &full[stage], st, 0, x - 1, y - 1, n, 1, 1);
                    } else {
                        tma_load_3d(&ma, &full[stage], st, 0, pix, 0);
                    }
                    pix += 128;
                    if (pix + 128 > npix) pix = 0;
                }
                if (do_b) {
                    tma_load_3d(&mb, &full[stage], st + kA, 0, brow, 0);
                    brow += 96;
                    if (brow + 96 > nb_rows) brow = 0;
                }
                if (++stage == stages) { stage = 0; phase ^= 1u; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
            mbar_wait(&full[stage], phase);
            mbar_arrive(&empty[stage]);
            if (++stage == stages) { stage = 0; phase ^= 1u; }
        }
        out[blockIdx.x] = clock64() - t0;
    }
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
    // A: 128 images of 13x13 pixels x 128 B (one 16-channel unit of the conv3 split input: 22 MB
    // over 16 units -> use 16 x 128 images to span the same 44 MB footprint)
    const int W = 13, N = 128 * 16, npix = N * W * W;
    const int nb_rows = 9 * 384 * 16;   // B: weights rows x units (7 MB)
    float *abuf, *bbuf;
    cudaMalloc(&abuf, (size_t)npix * 128);
    cudaMalloc(&bbuf, (size_t)nb_rows * 128);
    cudaMemset(abuf, 0, (size_t)npix * 128);
    cudaMemset(bbuf, 0, (size_t)nb_rows * 128);
    CUtensorMap ma_i, ma_t, mb, ma_i64;
    for (int bx : {128, 64}) {
        cuuint64_t dims[4] = {32, (cuuint64_t)W, (cuuint64_t)W, (cuuint64_t)N};
        cuuint64_t str[3] = {128, 128ull * W, 128ull * W * W};
        int lo[2] = {-1, -1}, up[2] = {-1, -1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc_i(bx == 128 ? &ma_i : &ma_i64, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, abuf, dims, str, lo, up, 32, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode im2col failed\n"); return 1; }
    }
    auto tiled = [&](CUtensorMap* m, float* buf, int rows, int box) {
        cuuint64_t dims[3] = {32, (cuuint64_t)rows, 1};
        cuuint64_t str[2] = {128, 128ull * rows};
        cuuint32_t bx[3] = {32, (cuuint32_t)box, 1};
        cuuint32_t es[3] = {1, 1, 1};
        return enc_t(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    if (tiled(&ma_t, abuf, npix, 128) != CUDA_SUCCESS || tiled(&mb, bbuf, nb_rows, 96) != CUDA_SUCCESS) {
        printf("encode tiled failed\n");
        return 1;
    }
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    printf("%-7s %6s %4s %9s %9s %10s\n", "A mode", "stages", "iss", "TB/s", "B/clk/SM", "clk/stage");
    struct Case { int im2col, stages, issuers; };
    const Case cases[] = {{1, 7, 1}, {1, 7, 2}, {1, 7, 3}, {1, 4, 3}, {0, 7, 1}, {0, 7, 2}};
    for (const Case& c : cases) {
        const int iters = 2000;
        const int smem = 1024 + c.stages * kStage + 256;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            ring<<<148, 128, smem>>>(c.im2col ? ma_i : ma_t, mb, ma_i64, c.im2col, c.stages, c.issuers, iters, npix, W, nb_rows,
                                     cyc);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto v : h) avg += v;
            avg /= 148;
            if (rep == 1)
                printf("%-7s %6d %4d %9.2f %9.1f %10.1f %s\n", c.im2col ? "im2col" : "tiled", c.stages, c.issuers,
                       148.0 * iters * kStage / ms / 1e9, iters * (double)kStage / avg, avg / iters,
                       err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
    }
    return 0;
}
