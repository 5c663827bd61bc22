// mma_probe2.cu -- tcgen05 MMA issue rate with operands resident in smem, for the shapes the
// conv kernel issues: cta_group::1 vs ::2 (CTA pair, M = 256) and the fp32-faithful patterns
// (classic 3xTF32: 6 tf32 K=8 MMAs per 16 channels; mixed: 2 tf32 + 2 bf16 K=16).  Reports
// cycles per 16-channel unit and per MMA instruction.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace clb;

template <int CG>
__global__ void __cluster_dims__(CG, 1, 1) probe(int n, int iters, int mixed, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        if constexpr (CG == 2) tmem_alloc_2sm(&tslot, 256);
        else tmem_alloc(&tslot, 256);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const bool leader = CG == 1 || cluster_ctarank() == 0;
    if (warp == 1 && leader) {
        const uint64_t da = umma_desc_kmajor(smem_u32(smem), 128);
        const uint64_t db = umma_desc_kmajor(smem_u32(smem + 128 * 128), 128);
        const uint32_t it32 = idesc_tf32(128 * CG, (uint32_t)n), it16 = idesc_bf16(128 * CG, (uint32_t)n);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
                for (int s = 0; s < 16; ++s) {   // 16 units of 16 channels per commit
                    const uint32_t acc = (it | s) ? 1u : 0u;
                    if (mixed) {
                        if constexpr (CG == 2) {
                            mma_bf16_ss_2sm(tmem, da + 6, db + 4, it16, acc);
                            mma_bf16_ss_2sm(tmem, da + 4, db + 6, it16, 1u);
                            mma_tf32_ss_2sm(tmem, da, db, it32, 1u);
                            mma_tf32_ss_2sm(tmem, da + 2, db + 2, it32, 1u);
                        } else {
                            mma_bf16_ss(tmem, da + 6, db + 4, it16, acc);
                            mma_bf16_ss(tmem, da + 4, db + 6, it16, 1u);
                            mma_tf32_ss(tmem, da, db, it32, 1u);
                            mma_tf32_ss(tmem, da + 2, db + 2, it32, 1u);
                        }
                    } else {
                        for (int q = 0; q < 6; ++q) {
                            if constexpr (CG == 2) mma_tf32_ss_2sm(tmem, da + 2 * (q % 4), db + 2 * ((q + 1) % 4), it32, acc | q);
                            else mma_tf32_ss(tmem, da + 2 * (q % 4), db + 2 * ((q + 1) % 4), it32, acc | q);
                        }
                    }
                }
                if constexpr (CG == 2) mma_commit_2sm_mc(&bar, (uint16_t)0x3);
                else mma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, ph);
            ph ^= 1u;
        }
        if (lane_id() == 0) cyc[blockIdx.x] = clock64() - t0;
    } else if (warp == 1 && CG == 2) {
        uint32_t ph = 0;   // the peer waits on its copy of the multicast commit
        for (int it = 0; it < iters; ++it) {
            mbar_wait(&bar, ph);
            ph ^= 1u;
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();
    if (warp == 0) {
        if constexpr (CG == 2) tmem_dealloc_2sm(tmem, 256);
        else tmem_dealloc(tmem, 256);
    }
}

int main() {
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int n : {64, 128, 192, 256}) {
        for (int cg : {1, 2}) {
            for (int mixed : {0, 1}) {
                const int iters = 500;
                cudaMemset(cyc, 0, 148 * 8);
                if (cg == 2) probe<2><<<148, 128, 64 * 1024>>>(n, iters, mixed, cyc);
                else probe<1><<<148, 128, 64 * 1024>>>(n, iters, mixed, cyc);
                cudaError_t e = cudaDeviceSynchronize();
                std::vector<unsigned long long> h(148);
                cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
                double avg = 0;
                int cnt = 0;
                for (auto v : h)
                    if (v) avg += v, ++cnt;
                avg /= cnt > 0 ? cnt : 1;
                const int per_unit = mixed ? 4 : 6;
                const double unit = avg / (iters * 16.0);
                // ideal per 16-channel unit: (per_unit MMA slots) x N/2 cycles (each slot = one M=128 tf32 K=8)
                const double ideal = per_unit * n / 2.0;
                printf("N=%3d cta_group::%d %-7s: %s  %.1f cycles per 16-ch unit (%.1f per MMA, ideal %.0f) -> %.0f%%\n", n, cg,
                       mixed ? "mixed" : "3xtf32", cudaGetErrorString(e), unit, unit / per_unit, ideal / per_unit,
                       100.0 * ideal / unit);
            }
        }
    }
    return 0;
}
