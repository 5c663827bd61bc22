// direct.cu -- CUDA-core direct convolution for tiny-C first layers.
//
// VGG conv1_1 (C = 3) wastes 13/16 of every tensor-core K block and is HBM-bound anyway
// (AI 12.9 flop/B): 27 MACs per output.  This is the fp32 loop nest of
// conv_mcmk_loopnest (conv_direct.cpp:104-143) restated for the GPU: one CTA = 4 output rows
// x 128 output columns of one image for 16 output channels; the input halo (C x (4+k-1) x
// (128+k-1)) and the 16-channel weight slice are staged in shared memory; each thread keeps
// 4 adjacent pixels x 16 channels of fp32 accumulators (FMA) and writes float4 rows.
#include "internal.hpp"

namespace clb {

namespace {

constexpr int kTq = 128;   // output columns per CTA (32 threads x 4)
constexpr int kTp = 4;     // output rows per CTA (4 warps)
constexpr int kMb = 16;    // output channels per CTA
constexpr int kPx = 4;     // adjacent pixels per thread
constexpr int kMaxK = 11;

// KT > 0: kernel size fixed at compile time (the tap window lives in registers);
// KT == 0: any k <= kMaxK (same code with runtime taps, slower).
template <int KT>
__global__ void __launch_bounds__(128) direct_conv_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                          float* __restrict__ y, int C, int H, int W, int M, int k_rt,
                                                          int pad, int P, int Q, int m_blocks) {
    const int k = KT > 0 ? KT : k_rt;
    constexpr int KW = KT > 0 ? KT : kMaxK;   // register window width bound
    extern __shared__ float sm[];
    const int ih = kTp + k - 1, iw = kTq + k - 1;
    float* s_in = sm;                          // [C][ih][iw]
    float* s_w = sm + C * ih * iw;             // [kMb][C*k*k]
    const int n = blockIdx.z / m_blocks;
    const int m0 = (blockIdx.z - n * m_blocks) * kMb;
    const int p0 = blockIdx.y * kTp, q0 = blockIdx.x * kTq;
    const int tid = threadIdx.x;
    const int ckk = C * k * k;
    // stage the input halo (zero outside the image: the implicit padding)
    const float* xn = x + (long long)n * C * H * W;
    for (int e = tid; e < C * ih * iw; e += 128) {
        const int c = e / (ih * iw), r = e - c * ih * iw;
        const int yy = r / iw, xx = r - yy * iw;
        const int sh = p0 - pad + yy, sw = q0 - pad + xx;
        s_in[e] = (sh >= 0 && sh < H && sw >= 0 && sw < W) ? __ldg(xn + ((long long)c * H + sh) * W + sw) : 0.0f;
    }
    // weights MKKC [m][i][j][c] -> s_w[mm][(c*k + i)*k + j]
    for (int e = tid; e < kMb * ckk; e += 128) {
        const int mm = e / ckk, r = e - mm * ckk;
        const int c = r / (k * k), ij = r - c * k * k;
        const int m = m0 + mm;
        s_w[e] = m < M ? __ldg(w + ((long long)m * k * k + ij) * C + c) : 0.0f;
    }
    __syncthreads();
    const int lane = tid & 31, row = tid >> 5;
    const int qx = lane * kPx;
    float acc[kMb][kPx];
#pragma unroll
    for (int mm = 0; mm < kMb; ++mm)
#pragma unroll
        for (int t = 0; t < kPx; ++t) acc[mm][t] = 0.0f;
    for (int c = 0; c < C; ++c) {
        for (int i = 0; i < k; ++i) {
            const float* src = s_in + (c * ih + row + i) * iw + qx;
            float v[kPx + KW - 1];
#pragma unroll
            for (int t = 0; t < kPx + KW - 1; ++t)
                if (t < kPx + k - 1) v[t] = src[t];
            const float* wr = s_w + (c * k + i) * k;
#pragma unroll
            for (int j = 0; j < KW; ++j) {
                if (j >= k) break;
#pragma unroll
                for (int mm = 0; mm < kMb; ++mm) {
                    const float ww = wr[mm * ckk + j];
#pragma unroll
                    for (int t = 0; t < kPx; ++t) acc[mm][t] = fmaf(ww, v[t + j], acc[mm][t]);
                }
            }
        }
    }
    const int p = p0 + row;
    if (p >= P) return;
    const int q = q0 + qx;
    for (int mm = 0; mm < kMb; ++mm) {
        const int m = m0 + mm;
        if (m >= M) break;
        float* dst = y + (((long long)n * M + m) * P + p) * Q + q;
        if (q + kPx <= Q && (((uintptr_t)dst) & 15) == 0) {
            *reinterpret_cast<float4*>(dst) = make_float4(acc[mm][0], acc[mm][1], acc[mm][2], acc[mm][3]);
        } else {
#pragma unroll
            for (int t = 0; t < kPx; ++t)
                if (q + t < Q) dst[t] = acc[mm][t];
        }
    }
}

}  // namespace

size_t direct_smem_bytes(int C, int k) {
    return (size_t)(C * (kTp + k - 1) * (kTq + k - 1) + kMb * C * k * k) * sizeof(float);
}

void launch_direct_conv(const float* x, const float* w, float* y, int N, int C, int H, int W, int M, int k, int pad,
                        int P, int Q, cudaStream_t s) {
    if (k > kMaxK) throw Error(2, "direct-gpu supports k <= 11");
    const size_t smem = direct_smem_bytes(C, k);
    if (smem > 200 * 1024) throw Error(2, "direct-gpu: channel count too large for the shared-memory halo");
    static bool configured = false;
    if (!configured) {
        CLB_CUDA(cudaFuncSetAttribute(direct_conv_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CLB_CUDA(cudaFuncSetAttribute(direct_conv_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CLB_CUDA(cudaFuncSetAttribute(direct_conv_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CLB_CUDA(cudaFuncSetAttribute(direct_conv_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    const int m_blocks = (M + kMb - 1) / kMb;
    dim3 grid((Q + kTq - 1) / kTq, (P + kTp - 1) / kTp, N * m_blocks);
    switch (k) {
        case 1: direct_conv_kernel<1><<<grid, 128, smem, s>>>(x, w, y, C, H, W, M, k, pad, P, Q, m_blocks); break;
        case 3: direct_conv_kernel<3><<<grid, 128, smem, s>>>(x, w, y, C, H, W, M, k, pad, P, Q, m_blocks); break;
        case 5: direct_conv_kernel<5><<<grid, 128, smem, s>>>(x, w, y, C, H, W, M, k, pad, P, Q, m_blocks); break;
        default: direct_conv_kernel<0><<<grid, 128, smem, s>>>(x, w, y, C, H, W, M, k, pad, P, Q, m_blocks);
    }
    CLB_CUDA(cudaGetLastError());
}

}  // namespace clb
