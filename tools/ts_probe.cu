// ts_probe.cu -- tcgen05.mma kind::tf32 with the A operand staged in TMEM by tcgen05.cp
// (".ts" form) vs the same MMAs with A from shared memory: results must be bit-identical,
// including A views that start k rows into the tile (the tap shift of the tap-shared mode).
// Then the same 3xTF32 pattern is timed both ways at N = 64 / 128 (148 CTAs, operands
// resident, 16 row-shifted A views per commit).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace clb;

constexpr int kARows = 136, kN = 64;

__global__ void check(const float* a, const float* b, int shift, float* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;                    // kARows rows x 128 B, SW128 K-major (swizzle applied by hand)
    uint8_t* sb = smem + 18 * 1024;        // kN rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    // software SW128: 16-byte chunk c of row r lands at chunk c ^ (r & 7)
    for (int i = threadIdx.x; i < kARows * 32; i += blockDim.x) {
        const int r = i / 32, w = i % 32;
        const int ch = (w / 4) ^ (r & 7);
        reinterpret_cast<float*>(sa + r * 128 + ch * 16)[w % 4] = a[i];
    }
    for (int i = threadIdx.x; i < kN * 32; i += blockDim.x) {
        const int r = i / 32, w = i % 32;
        const int ch = (w / 4) ^ (r & 7);
        reinterpret_cast<float*>(sb + r * 128 + ch * 16)[w % 4] = b[i];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint64_t da = umma_desc_kmajor(smem_u32(sa) + (uint32_t)shift * 128u, 128);
        const uint64_t db = umma_desc_kmajor(smem_u32(sb), 128);
        const uint32_t idesc = idesc_tf32(128, kN);
        // SS reference into columns [0, 64)
        mma_tf32_ss(tmem, da + 4, db, idesc, 0u);
        mma_tf32_ss(tmem, da, db + 4, idesc, 1u);
        mma_tf32_ss(tmem, da, db, idesc, 1u);
        mma_tf32_ss(tmem, da + 6, db + 2, idesc, 1u);
        mma_tf32_ss(tmem, da + 2, db + 6, idesc, 1u);
        mma_tf32_ss(tmem, da + 2, db + 2, idesc, 1u);
        // TS: copy the 4 slabs (hi k0-7, hi k8-15, lo k0-7, lo k8-15) to columns [256, 288)
        const uint32_t ta = tmem + 256;
        for (int s = 0; s < 4; ++s) tmem_cp_128x256b(ta + 8 * s, da + 2 * s);
        const uint32_t d2 = tmem + 64;
        mma_tf32_ts(d2, ta + 16, db, idesc, 0u);
        mma_tf32_ts(d2, ta, db + 4, idesc, 1u);
        mma_tf32_ts(d2, ta, db, idesc, 1u);
        mma_tf32_ts(d2, ta + 24, db + 2, idesc, 1u);
        mma_tf32_ts(d2, ta + 8, db + 6, idesc, 1u);
        mma_tf32_ts(d2, ta + 8, db + 2, idesc, 1u);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c0 = 0; c0 < 2 * kN; c0 += 16) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, r);
        tmem_ld_wait();
        for (int c = 0; c < 16; ++c) out[row * 2 * kN + c0 + c] = __uint_as_float(r[c]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// timing: 148 CTAs, `taps` row-shifted views of A per stage, 3xTF32 pattern, one commit per
// 16 stages; ts = 1 copies each view to TMEM first (4 x tcgen05.cp) and runs the .ts MMAs;
// ts = 2 runs the same .ts MMAs with A already resident in TMEM (no copies: the MMA rate alone)
__global__ void timing(int n, int iters, int ts, unsigned long long* cyc) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (kARows + 256) * 32; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (warp == 1) {
        const uint64_t da0 = umma_desc_kmajor(smem_u32(smem), 128);
        const uint64_t db = umma_desc_kmajor(smem_u32(smem + 18 * 1024), 128);
        const uint32_t idesc = idesc_tf32(128, (uint32_t)n);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (elect_one()) {
                for (int s = 0; s < 16; ++s) {
                    const int t = s % 3;
                    const uint64_t da = da0 + (uint64_t)(t * 8);
                    if (ts) {
                        const uint32_t ta = tmem + 256 + (uint32_t)((s & 1) * 32);
                        if (ts == 1)
                            for (int q = 0; q < 4; ++q) tmem_cp_128x256b(ta + 8 * q, da + 2 * q);
                        mma_tf32_ts(tmem, ta + 16, db, idesc, (it | s) ? 1u : 0u);
                        mma_tf32_ts(tmem, ta, db + 4, idesc, 1u);
                        mma_tf32_ts(tmem, ta, db, idesc, 1u);
                        mma_tf32_ts(tmem, ta + 24, db + 2, idesc, 1u);
                        mma_tf32_ts(tmem, ta + 8, db + 6, idesc, 1u);
                        mma_tf32_ts(tmem, ta + 8, db + 2, idesc, 1u);
                    } else {
                        mma_tf32_ss(tmem, da + 4, db, idesc, (it | s) ? 1u : 0u);
                        mma_tf32_ss(tmem, da, db + 4, idesc, 1u);
                        mma_tf32_ss(tmem, da, db, idesc, 1u);
                        mma_tf32_ss(tmem, da + 6, db + 2, idesc, 1u);
                        mma_tf32_ss(tmem, da + 2, db + 6, idesc, 1u);
                        mma_tf32_ss(tmem, da + 2, db + 2, idesc, 1u);
                    }
                }
                mma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, ph);
            ph ^= 1u;
        }
        if (lane_id() == 0) cyc[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    std::vector<float> ha(kARows * 32), hb(kN * 32);
    srand(7);
    for (auto& v : ha) v = (float)rand() / RAND_MAX * 2.0f - 1.0f;
    for (auto& v : hb) v = (float)rand() / RAND_MAX * 2.0f - 1.0f;
    float *da, *db, *dout;
    cudaMalloc(&da, ha.size() * 4);
    cudaMalloc(&db, hb.size() * 4);
    cudaMalloc(&dout, 128 * 2 * kN * 4);
    cudaMemcpy(da, ha.data(), ha.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    std::vector<float> ho(128 * 2 * kN);
    for (int shift = 0; shift < 8; ++shift) {
        check<<<1, 128, 40 * 1024>>>(da, db, shift, dout);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(ho.data(), dout, ho.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxv = 0;
        for (int r = 0; r < 128; ++r)
            for (int c = 0; c < kN; ++c) {
                const float s = ho[r * 2 * kN + c], t = ho[r * 2 * kN + kN + c];
                if (__builtin_memcmp(&s, &t, 4) != 0) ++bad;
                maxv = std::max(maxv, (double)std::abs(s));
            }
        printf("shift %d: %s, TS vs SS bit mismatches %d/%d (max|D| %.3f)\n", shift, cudaGetErrorString(e), bad,
               128 * kN, maxv);
    }
    unsigned long long* cyc;
    cudaMalloc(&cyc, 148 * 8);
    cudaFuncSetAttribute(timing, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int n : {64, 128}) {
        for (int ts = 0; ts < 3; ++ts) {
            const int iters = 1000;
            timing<<<148, 128, 64 * 1024>>>(n, iters, ts, cyc);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<unsigned long long> h(148);
            cudaMemcpy(h.data(), cyc, 148 * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto v : h) avg += v;
            avg /= 148;
            const double per = avg / (iters * 16.0 * 6.0);
            printf("N=%3d %s: %s  %.1f cycles/MMA (ideal %d) -> %.0f%%\n", n, ts == 2 ? "A resident in TMEM (.ts)" : ts ? "A from TMEM (cp + .ts) " : "A from smem (.ss)       ",
                   cudaGetErrorString(e), per, n / 2, 100.0 * (n / 2) / per);
        }
    }
    return 0;
}
