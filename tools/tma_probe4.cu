// TMA delivery vs operand layout (the padded-row kernel's pattern): a ring of 4 stages of
// A (tiled box of 130 rows x one 128 B unit) + B (tiled box of 96 rows x one unit), A issued by
// warp 0 and B by warp 2, a consumer warp releasing each stage as it lands (no compute).
// Layout cases for an input of U 16-channel units per pixel:
//   "nhwc"   : pixel rows of U units (row pitch U x 128 B); a box reads one unit per row
//              (what the kernel does today: 128 B segments strided by the pitch)
//   "planar" : unit-major planes [unit][pixel][128 B]; a box is one contiguous 16 KB run
// and two footprints: "hbm" (a 1 GB input streamed once, L2 misses) and "l2" (a 32 MB input).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_1704_04428_b200/csrc
//        tools/tma_probe4.cu -o tools/tma_probe4 -lcuda
#include <cstdio>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace clb;

constexpr int kARows = 130, kBRows = 96;
constexpr int kA = 136 * 128, kB = kBRows * 128, kStage = kA + kB;   // A region 1024-aligned (136 rows)
constexpr int kStages = 4;

// map: 3-D {32 words, rows, units}; the unit coordinate selects the 128 B column block
__global__ void ring(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int units,
                     long long a_rows, int b_rows, int iters, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage);
    uint64_t* empty = full + kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 2);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if ((warp == 0 || warp == 2) && lane == 0) {
        const bool do_a = warp == 0;
        int stage = 0;
        uint32_t phase = 0;
        // each CTA walks its own contiguous slice of pixel rows, unit-inner like the kernel's K loop
        const long long slice = a_rows / gridDim.x;
        long long row = blockIdx.x * slice;
        int u = 0, brow = (blockIdx.x * 96) % (b_rows - kBRows);
        for (int it = 0; it < iters; ++it) {
            mbar_wait(&empty[stage], phase ^ 1u);
            uint8_t* st = smem + stage * kStage;
            mbar_arrive_expect_tx(&full[stage], do_a ? kARows * 128 : kB);
            if (do_a) {
                tma_load_3d(&ma, &full[stage], st, 0, (int)row, u);
                if (++u == units) {
                    u = 0;
                    row += 128;
                    if (row + kARows > (blockIdx.x + 1) * slice) row = blockIdx.x * slice;
                }
            } else {
                tma_load_3d(&mb, &full[stage], st + kA, 0, brow, u);
                if (++u == units) u = 0;
            }
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    } else if (warp == 1 && lane == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
            mbar_wait(&full[stage], phase);
            mbar_arrive(&empty[stage]);
            if (++stage == kStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

using EncT = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* f1 = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q);
    EncT enc = (EncT)f1;
    const size_t big = 1ull << 30;
    void *abuf, *bbuf;
    cudaMalloc(&abuf, big);
    cudaMalloc(&bbuf, 64ull << 20);
    cudaMemset(abuf, 0, big);
    cudaMemset(bbuf, 0, 64ull << 20);
    // planar: dims {32, rows, units} strides {128, rows*128}; nhwc: strides {units*128, 128}
    auto map = [&](CUtensorMap* m, void* buf, long long rows, int units, bool planar, int box) {
        cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)units};
        cuuint64_t str[2] = {planar ? 128ull : 128ull * units, planar ? 128ull * rows : 128ull};
        cuuint32_t bx[3] = {32, (cuuint32_t)box, 1};
        cuuint32_t es[3] = {1, 1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    const int smem = 1024 + kStages * kStage + 256;
    printf("%-7s %-4s %5s %9s %9s %10s\n", "layout", "src", "units", "TB/s", "B/clk/SM", "clk/stage");
    for (int planar = 0; planar < 2; ++planar)
        for (int hbm = 1; hbm >= 0; --hbm)
            for (int units : {1, 2, 4, 8}) {
                const size_t bytes = hbm ? big : (32ull << 20);
                const long long a_rows = (long long)(bytes / (128ull * units));
                const int b_rows = 9 * 64 * 3;   // conv1_2-sized weights per unit
                CUtensorMap ma, mb;
                if (map(&ma, abuf, a_rows, units, planar, kARows) != CUDA_SUCCESS ||
                    map(&mb, bbuf, b_rows, units, planar, kBRows) != CUDA_SUCCESS) {
                    printf("encode failed\n");
                    return 1;
                }
                // hbm: ~one pass over the input per launch; l2: many passes over 32 MB
                const int iters = hbm ? (int)(a_rows / 148 / 128 * units) : 4000;
                for (int rep = 0; rep < 2; ++rep) {
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0);
                    ring<<<148, 128, smem>>>(ma, mb, units, a_rows, b_rows, iters, cyc);
                    cudaEventRecord(e1);
                    cudaError_t err = cudaDeviceSynchronize();
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    std::vector<unsigned long long> h(148);
                    cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
                    double avg = 0;
                    for (auto v : h) avg += v;
                    avg /= 148;
                    const double stage_bytes = kARows * 128.0 + kB;
                    if (rep == 1)
                        printf("%-7s %-4s %5d %9.2f %9.1f %10.1f %s\n", planar ? "planar" : "nhwc", hbm ? "hbm" : "l2",
                               units, 148.0 * iters * stage_bytes / ms / 1e9, iters * stage_bytes / avg, avg / iters,
                               err == cudaSuccess ? "" : cudaGetErrorString(err));
                }
            }
    return 0;
}
