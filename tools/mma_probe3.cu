// mma_probe3.cu -- kind::f16 MMA issue rate at small N with operands resident in smem: does the
// rate depend on (a) consecutive MMAs accumulating into the same D (a dependency chain), or
// (b) the single issuing thread?  Variants per N (cta_group::1, M = 128, K = 16):
//   same   : 16 MMAs per commit, all into one accumulator
//   alt2   : 16 MMAs per commit alternating between two accumulators
//   alt4   : ... between four accumulators
//   2warps : two issuing warps, each with its own accumulator (8 MMAs each per round)
// Reports cycles per MMA (ideal N/4 cycles for f16: 128 x N x 16 x 2 flop at 8192 flop/clk/SM).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace clb;

__global__ void probe(int n, int iters, int mode, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const int issuers = mode == 3 ? 2 : 1;
    if (warp >= 1 && warp <= issuers) {
        const int w = warp - 1;
        const uint64_t da = umma_desc_kmajor(smem_u32(smem), 128);
        const uint64_t db = umma_desc_kmajor(smem_u32(smem + 128 * 128), 128);
        const uint32_t idesc = idesc_f16(128, (uint32_t)n);
        const int per = mode == 3 ? 8 : 16;
        const int nacc = mode == 1 ? 2 : (mode == 2 ? 4 : 1);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
                for (int s = 0; s < per; ++s) {
                    const uint32_t d = tmem + (uint32_t)(((mode == 3 ? w : s % nacc)) * 128);
                    mma_bf16_ss(d, da + 2 * (s % 4), db + 2 * ((s + 1) % 4), idesc, (it | (s >= nacc)) ? 1u : 0u);
                }
                mma_commit(&bar[w]);
            }
            __syncwarp();
            mbar_wait(&bar[w], ph);
            ph ^= 1u;
        }
        if (lane_id() == 0 && w == 0) cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char* names[] = {"same", "alt2", "alt4", "2warps"};
    for (int n : {64, 128, 256}) {
        for (int mode = 0; mode < 4; ++mode) {
            const int iters = 1000;
            cudaMemset(cyc, 0, 148 * 8);
            probe<<<148, 128, 64 * 1024>>>(n, iters, mode, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            int cnt = 0;
            for (auto v : h)
                if (v) avg += v, ++cnt;
            avg /= cnt > 0 ? cnt : 1;
            const double per_mma = avg / (iters * 16.0);
            printf("N=%3d %-7s: %s  %.1f cycles per MMA (ideal %.0f) -> %.0f%%\n", n, names[mode], cudaGetErrorString(e),
                   per_mma, n / 4.0, 100.0 * (n / 4.0) / per_mma);
        }
    }
    return 0;
}
