// tma_probe.cu -- microbenchmark of TMA load throughput (tiled vs im2col, row size, pixel
// stride) on one B200; no MMA.  148 persistent CTAs, one producer thread each, S-stage ring.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1704_04428_b200/csrc
//        tma_probe.cu -o tma_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace clb;

struct Cfg {
    int mode;        // 0 tiled, 1 im2col
    int row_bytes;   // 64 or 128
    int box_rows;    // pixels per box
    int stages;
    int loads_per_cta;
    int P, Q, N, k, pad;
    int tiled_rows;
    int prefetch, spin;
};

__global__ void probe(const __grid_constant__ CUtensorMap map, Cfg c, unsigned long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int box_bytes = c.box_rows * c.row_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + c.stages * box_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < c.stages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (c.prefetch) tma_prefetch_desc(&map);
    const long long t0 = clock64();
    const int PQ = c.P * c.Q;
    const int total_pix = c.N * PQ;
    uint32_t phase = 0;
    for (int i = 0; i < c.loads_per_cta + c.stages; ++i) {
        const int s = i % c.stages;
        if (i >= c.stages) {
            if (c.spin) {
                uint32_t ok = 0;
                while (!ok) {
                    asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.u32 %0,1,0,P;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(phase) : "memory");
                }
            } else {
                mbar_wait(&full[s], phase);
            }
            if (s == c.stages - 1) phase ^= 1;
        }
        if (i < c.loads_per_cta) {
            mbar_arrive_expect_tx(&full[s], box_bytes);
            const int t = (blockIdx.x * 7919 + i * 131) % 1000003;
            if (c.mode == 1) {
                const int row0 = (t % (total_pix / c.box_rows)) * c.box_rows;
                const int n = row0 / PQ, rem = row0 % PQ, p = rem / c.Q, q = rem % c.Q;
                const int tap = i % (c.k * c.k);
                tma_load_im2col_4d(&map, &full[s], smem + s * box_bytes, 0, q - c.pad, p - c.pad, n,
                                   (uint16_t)(tap % c.k), (uint16_t)(tap / c.k));
            } else {
                const int row0 = (t % (c.tiled_rows / c.box_rows)) * c.box_rows;
                tma_load_3d(&map, &full[s], smem + s * box_bytes, 0, row0, 0);
            }
        }
    }
    cycles[blockIdx.x] = clock64() - t0;
}

using EncT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using EncI = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* f1 = nullptr; void* f2 = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q);
    EncT enc_t = (EncT)f1;
    EncI enc_i = (EncI)f2;
    const int N = 32, H = 56, W = 56;
    float* buf;
    const size_t bytes = (size_t)N * H * W * 512;   // up to 128 fp32 channels per pixel
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * sizeof(unsigned long long));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    struct Case { const char* name; int mode, row_bytes, pixel_bytes, box_rows, stages, ctas, prefetch, spin; };
    Case cases[] = {
        {"tiled 128Bx128 st1 cta1", 0, 128, 512, 128, 1, 1, 1, 0},
        {"tiled 128Bx128 st4 cta1", 0, 128, 512, 128, 4, 1, 1, 0},
        {"tiled 128Bx128 st8 cta1", 0, 128, 512, 128, 8, 1, 1, 0},
        {"tiled 128Bx128 st8 cta148", 0, 128, 512, 128, 8, 148, 1, 0},
        {"tiled 128Bx128 st8 cta148 spin", 0, 128, 512, 128, 8, 148, 1, 1},
        {"tiled 128Bx128 st8 cta148 noprefetch", 0, 128, 512, 128, 8, 148, 0, 0},
        {"im2col 128Bx128 st1 cta1", 1, 128, 512, 128, 1, 1, 1, 0},
        {"im2col 128Bx128 st8 cta1", 1, 128, 512, 128, 8, 1, 1, 0},
        {"im2col 128Bx128 st8 cta148", 1, 128, 512, 128, 8, 148, 1, 0},
        {"im2col 128Bx128 st8 cta148 spin", 1, 128, 512, 128, 8, 148, 1, 1},
        {"im2col 64Bx128 st8 cta148 spin", 1, 64, 512, 128, 8, 148, 1, 1},
        {"tiled 128Bx256 st6 cta148 spin", 0, 128, 128, 256, 6, 148, 1, 1},
        {"im2col 128Bx256 st6 cta148 spin", 1, 128, 128, 256, 6, 148, 1, 1},
    };
    Case unused[] = {
        {"im2col 64B rows, pixel stride 512B (current)", 1, 64, 512, 128, 8},
        {"im2col 128B rows, pixel stride 512B", 1, 128, 512, 128, 8},
        {"im2col 128B rows, pixel stride 256B", 1, 128, 256, 128, 8},
        {"im2col 128B rows, contiguous pixels", 1, 128, 128, 128, 8},
        {"im2col 64B rows, contiguous pixels", 1, 64, 64, 128, 8},
        {"im2col 128B rows, contiguous, 256-pixel box", 1, 128, 128, 256, 6},
        {"im2col 128B rows, stride 512B, 16 stages", 1, 128, 512, 128, 12},
        {"tiled 64B rows, row stride 512B", 0, 64, 512, 128, 8},
        {"tiled 128B rows, row stride 512B", 0, 128, 512, 128, 8},
        {"tiled 128B rows, contiguous", 0, 128, 128, 128, 8},
        {"tiled 128B rows, contiguous, 256 rows", 0, 128, 128, 256, 6},
    };
    for (const Case& cs : cases) {
        CUtensorMap map;
        const cuuint64_t ch = cs.pixel_bytes / 4;
        const CUtensorMapSwizzle sw = cs.row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
        CUresult r;
        Cfg c{};
        c.mode = cs.mode; c.row_bytes = cs.row_bytes; c.box_rows = cs.box_rows; c.stages = cs.stages;
        c.loads_per_cta = 2000; c.prefetch = cs.prefetch; c.spin = cs.spin; c.P = H; c.Q = W; c.N = N; c.k = 3; c.pad = 1;
        if (cs.mode == 1) {
            cuuint64_t dims[4] = {ch, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t str[3] = {ch * 4, ch * 4 * W, ch * 4 * W * H};
            int lo[2] = {-1, -1}, up[2] = {-1, -1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            r = enc_i(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, buf, dims, str, lo, up, cs.row_bytes / 4, cs.box_rows,
                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            const cuuint64_t rows = (cuuint64_t)N * H * W;
            c.tiled_rows = (int)rows;
            cuuint64_t dims[3] = {ch, rows, 1};
            cuuint64_t str[2] = {ch * 4, ch * 4 * rows};
            cuuint32_t box[3] = {(cuuint32_t)cs.row_bytes / 4, (cuuint32_t)cs.box_rows, 1};
            cuuint32_t es[3] = {1, 1, 1};
            r = enc_t(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        if (r != CUDA_SUCCESS) { printf("%-40s encode failed %d\n", cs.name, (int)r); continue; }
        const int smem = 1024 + cs.stages * cs.box_rows * cs.row_bytes + 256;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        probe<<<cs.ctas, 32, smem>>>(map, c, cyc);   // warm
        cudaEventRecord(e0);
        probe<<<cs.ctas, 32, smem>>>(map, c, cyc);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> h(cs.ctas);
        cudaMemcpy(h.data(), cyc, cs.ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (auto v : h) avg += v;
        avg /= cs.ctas;
        const double tot = (double)cs.ctas * c.loads_per_cta * cs.box_rows * cs.row_bytes;
        printf("%-40s %s  %.3f ms  %.2f TB/s  %.1f B/clk/SM  %.2f clk/row\n", cs.name, cudaGetErrorString(err), ms,
               tot / ms / 1e9, (double)c.loads_per_cta * cs.box_rows * cs.row_bytes / avg,
               avg / ((double)c.loads_per_cta * cs.box_rows));
    }
    return 0;
}
