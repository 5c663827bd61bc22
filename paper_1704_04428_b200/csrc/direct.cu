// direct.cu -- CUDA-core direct convolution for tiny-C first layers.
//
// VGG conv1_1 (C = 3) wastes 13/16 of every tensor-core K block and is bound by its output
// write (AI 12.9 flop/B) and the fp32 FMA rate: 27 MACs per output.  This
// is the fp32 loop nest of conv_mcmk_loopnest (conv_direct.cpp:104-143) restated for the GPU.
//
// direct_persistent_kernel (the fast path, all weights fit in shared memory):
//   * persistent grid (SMs x resident CTAs); a unit = 256 consecutive 4-pixel groups of one
//     image (row-major, Q % 4 == 0) for ALL M output channels -- no idle lanes at ragged tile
//     edges; the CTA loops over units with a stride of the grid;
//   * the weights (C*k*k*M fp32) are staged ONCE per CTA in [c][i][j][m] order, so the 16
//     weights a thread needs per tap are 4 warp-uniform LDS.128 broadcasts;
//   * the input halo (the rows the unit touches + k-1, full width) of the NEXT unit is fetched
//     with cp.async
//     (src-size 0 = zero fill = the implicit padding) into the other half of a double buffer
//     while the current tile computes, so no CTA ever waits on a cold global load;
//   * thread t owns group t of the unit (4 adjacent pixels) and loops over the output channels
//     16 at a time (64 fp32 accumulators), streaming float4s out (a warp = 512 contiguous B).
// direct_conv_kernel (fallback when the weights do not fit): the same arithmetic with the
// halo and a 16-channel weight slice staged per CTA.
#include <cstring>
#include <mutex>

#include "internal.hpp"

namespace clb {

namespace {

constexpr int kTq = 128;   // output columns per tile (32 lanes x 4)
constexpr int kTp = 4;     // output rows per CTA (fallback kernel: 4 warps)
constexpr int kMb = 16;    // output channels per accumulator pass
constexpr int kPx = 4;     // adjacent pixels per thread
constexpr int kMaxK = 11;

constexpr int kPThreads = 256;             // persistent kernel: 8 warps
constexpr size_t kPersistentSmem = 200 * 1024;


__device__ __forceinline__ void cp_async_f32(float* dst, const float* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void st_stream_f4(float* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Work unit = kUnit consecutive 4-pixel groups of one image in row-major order (Q % 4 == 0), so
// no lane idles at a ragged tile edge (224 x 224 = 49 units exactly); its halo is the input
// rows those groups touch plus k - 1, at full width.
constexpr int kUnit = kPThreads;

struct UnitGeom {
    int groups_row, groups_img, units_img, halo_rows, pitch;
};

__host__ __device__ inline UnitGeom unit_geom(int P, int Q, int k) {
    UnitGeom g;
    g.groups_row = Q / 4;
    g.groups_img = P * g.groups_row;
    g.units_img = (g.groups_img + kUnit - 1) / kUnit;
    g.halo_rows = (kUnit + g.groups_row - 1) / g.groups_row + 1 + k - 1;
    g.pitch = (Q + k - 1 + 3) & ~3;   // 16 B aligned rows
    return g;
}

// cp.async the halo of one unit: rows (c, yy) over the warps, columns over the lanes
// (coalesced); out-of-image elements are zero-filled (the implicit padding).
__device__ __forceinline__ void load_halo(float* s_in, const float* __restrict__ x, int unit, const UnitGeom& g, int C,
                                          int H, int W, int k, int pad) {
    const int n = unit / g.units_img;
    const int g0 = (unit - n * g.units_img) * kUnit;
    const int r_lo = g0 / g.groups_row;
    const int r_hi = min(g.groups_img - 1, g0 + kUnit - 1) / g.groups_row;
    const int nrows = r_hi - r_lo + k;
    const int iw = g.groups_row * 4 + k - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* xn = x + (long long)n * C * H * W;
    for (int row = warp; row < C * nrows; row += kPThreads / 32) {
        const int c = row / nrows, yy = row - c * nrows;
        const int sh = r_lo - pad + yy;
        const bool hv = sh >= 0 && sh < H;
        const float* src_row = xn + ((long long)c * H + (hv ? sh : 0)) * W;
        float* dst_row = s_in + (c * g.halo_rows + yy) * g.pitch;
        for (int xx = lane; xx < iw; xx += 32) {
            const int sw = xx - pad;
            const bool v = hv && sw >= 0 && sw < W;
            cp_async_f32(dst_row + xx, v ? src_row + sw : xn, v);
        }
    }
}

// KT / CT > 0 fix k / C at compile time (the whole tap loop unrolls); 0 = runtime value.
template <int KT, int CT>
__global__ void __launch_bounds__(kPThreads, 2)
    direct_persistent_kernel(const float* __restrict__ x, const float* __restrict__ w, float* __restrict__ y, int C_rt,
                             int H, int W, int M, int k_rt, int pad, int P, int Q, int num_units) {
    const int k = KT > 0 ? KT : k_rt;
    const int C = CT > 0 ? CT : C_rt;
    constexpr int KW = KT > 0 ? KT : kMaxK;
    extern __shared__ __align__(16) float sm[];
    const int ckk = C * k * k;
    const int Mp = (M + kMb - 1) / kMb * kMb;
    const UnitGeom g = unit_geom(P, Q, k);
    const int halo = C * g.halo_rows * g.pitch;
    float* s_w = sm;                                  // [c][i][j][Mp]
    float* s_in0 = sm + ((ckk * Mp + 3) & ~3);
    float* s_in1 = s_in0 + halo;
    const int tid = threadIdx.x;

    int unit = blockIdx.x;
    if (unit < num_units) load_halo(s_in0, x, unit, g, C, H, W, k, pad);
    cp_async_commit();
    // weights MKKC [m][i][j][c] -> s_w[((c*k + i)*k + j)*Mp + m] (zero for m >= M)
    for (int e = tid; e < ckk * Mp; e += kPThreads) {
        const int tap = e / Mp, m = e - tap * Mp;
        const int c = tap / (k * k), ij = tap - c * k * k;
        s_w[e] = m < M ? __ldg(w + ((long long)m * k * k + ij) * C + c) : 0.0f;
    }
    const bool y_aligned = (reinterpret_cast<uintptr_t>(y) & 15) == 0;
    const long long plane = (long long)P * Q;
    int buf = 0;
    for (; unit < num_units; unit += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();   // halo[buf] visible to all; everyone is done reading halo[buf ^ 1]
        const int next = unit + gridDim.x;
        if (next < num_units) load_halo(buf ? s_in0 : s_in1, x, next, g, C, H, W, k, pad);
        cp_async_commit();
        const float* s_in = buf ? s_in1 : s_in0;

        const int n = unit / g.units_img;
        const int g0 = (unit - n * g.units_img) * kUnit;
        const int gi = g0 + tid;
        if (gi < g.groups_img) {
            const int r_lo = g0 / g.groups_row;
            const int row = gi / g.groups_row;
            const int col = (gi - row * g.groups_row) * 4;
            const float* s_px = s_in + (row - r_lo) * g.pitch + col;
            float* y_px = y + (long long)n * M * plane + (long long)gi * 4;
            for (int m0 = 0; m0 < M; m0 += kMb) {
                float acc[kMb][kPx];
#pragma unroll
                for (int mm = 0; mm < kMb; ++mm)
#pragma unroll
                    for (int t = 0; t < kPx; ++t) acc[mm][t] = 0.0f;
#pragma unroll(CT > 0 ? CT : 1)
                for (int c = 0; c < C; ++c) {
#pragma unroll
                    for (int i = 0; i < KW; ++i) {
                        if (i >= k) break;
                        const float* src = s_px + (c * g.halo_rows + i) * g.pitch;
                        float v[kPx + KW - 1];
                        const float4 v4 = *reinterpret_cast<const float4*>(src);
                        v[0] = v4.x, v[1] = v4.y, v[2] = v4.z, v[3] = v4.w;
#pragma unroll
                        for (int t = kPx; t < kPx + KW - 1; ++t)
                            if (t < kPx + k - 1) v[t] = src[t];
                        const float* wt = s_w + ((c * k + i) * k) * Mp + m0;
#pragma unroll
                        for (int j = 0; j < KW; ++j) {
                            if (j >= k) break;
                            float wv[kMb];
#pragma unroll
                            for (int u = 0; u < kMb / 4; ++u) {
                                const float4 w4 = *reinterpret_cast<const float4*>(wt + j * Mp + 4 * u);
                                wv[4 * u] = w4.x, wv[4 * u + 1] = w4.y, wv[4 * u + 2] = w4.z, wv[4 * u + 3] = w4.w;
                            }
#pragma unroll
                            for (int mm = 0; mm < kMb; ++mm)
#pragma unroll
                                for (int t = 0; t < kPx; ++t) acc[mm][t] = fmaf(wv[mm], v[t + j], acc[mm][t]);
                        }
                    }
                }
#pragma unroll
                for (int mm = 0; mm < kMb; ++mm) {
                    if (m0 + mm < M) {
                        float* dst = y_px + (long long)(m0 + mm) * plane;
                        if (y_aligned) {
                            st_stream_f4(dst, acc[mm][0], acc[mm][1], acc[mm][2], acc[mm][3]);
                        } else {
#pragma unroll
                            for (int t = 0; t < kPx; ++t) dst[t] = acc[mm][t];
                        }
                    }
                }
            }
        }
        buf ^= 1;
    }
    cp_async_wait_all();
}

// 3-channel, 3x3 first layers (VGG conv1_1) with M output channels known at compile time:
// the same persistent unit / halo pipeline as direct_persistent_kernel, but the C*k*k*M
// weights travel as a __grid_constant__ kernel parameter ([c][i][j][m] order), so with every
// index a compile-time constant each FFMA takes its weight straight from the constant bank --
// no shared-memory weight loads (the smem kernel issues one LDS.128 per 16 FFMAs and measured
// issue-bound, profiles/r01_ncu_vgg16_conv1_1_direct_full.json).
template <int NW>
struct ParamWeights {
    float w[NW];
};

template <int MT>
__global__ void __launch_bounds__(kPThreads, 2)
    direct_param_kernel(const float* __restrict__ x, float* __restrict__ y, int H, int W, int pad, int P, int Q,
                        int num_units, const __grid_constant__ ParamWeights<27 * MT> wts) {
    constexpr int C = 3, k = 3;
    extern __shared__ __align__(16) float sm[];
    const UnitGeom g = unit_geom(P, Q, k);
    const int halo = C * g.halo_rows * g.pitch;
    float* s_in0 = sm;
    float* s_in1 = s_in0 + halo;
    const int tid = threadIdx.x;
    int unit = blockIdx.x;
    if (unit < num_units) load_halo(s_in0, x, unit, g, C, H, W, k, pad);
    cp_async_commit();
    const bool y_aligned = (reinterpret_cast<uintptr_t>(y) & 15) == 0;
    const long long plane = (long long)P * Q;
    int buf = 0;
    for (; unit < num_units; unit += gridDim.x) {
        cp_async_wait_all();
        __syncthreads();
        const int next = unit + gridDim.x;
        if (next < num_units) load_halo(buf ? s_in0 : s_in1, x, next, g, C, H, W, k, pad);
        cp_async_commit();
        const float* s_in = buf ? s_in1 : s_in0;
        const int n = unit / g.units_img;
        const int g0 = (unit - n * g.units_img) * kUnit;
        const int gi = g0 + tid;
        if (gi < g.groups_img) {
            const int r_lo = g0 / g.groups_row;
            const int row = gi / g.groups_row;
            const int col = (gi - row * g.groups_row) * 4;
            const float* s_px = s_in + (row - r_lo) * g.pitch + col;
            float* y_px = y + (long long)n * MT * plane + (long long)gi * 4;
            // the 27 taps' input rows are loaded once per pixel group and reused for every m
            float v[C][k][kPx + k - 1];
#pragma unroll
            for (int c = 0; c < C; ++c)
#pragma unroll
                for (int i = 0; i < k; ++i) {
                    const float* src = s_px + (c * g.halo_rows + i) * g.pitch;
                    const float4 v4 = *reinterpret_cast<const float4*>(src);
                    v[c][i][0] = v4.x, v[c][i][1] = v4.y, v[c][i][2] = v4.z, v[c][i][3] = v4.w;
                    v[c][i][4] = src[4];
                    v[c][i][5] = src[5];
                }
            // rolled over the 16-channel passes: a fully unrolled M = 64 body (~18k instructions)
            // measured 30 % slower (instruction-cache bound)
#pragma unroll 1
            for (int m0 = 0; m0 < MT; m0 += kMb) {
                float acc[kMb][kPx];
#pragma unroll
                for (int mm = 0; mm < kMb; ++mm)
#pragma unroll
                    for (int t = 0; t < kPx; ++t) acc[mm][t] = 0.0f;
#pragma unroll
                for (int c = 0; c < C; ++c)
#pragma unroll
                    for (int i = 0; i < k; ++i)
#pragma unroll
                        for (int j = 0; j < k; ++j)
#pragma unroll
                            for (int mm = 0; mm < kMb; ++mm) {
                                const float wv = wts.w[((c * k + i) * k + j) * MT + m0 + mm];
#pragma unroll
                                for (int t = 0; t < kPx; ++t) acc[mm][t] = fmaf(wv, v[c][i][t + j], acc[mm][t]);
                            }
#pragma unroll
                for (int mm = 0; mm < kMb; ++mm) {
                    float* dst = y_px + (long long)(m0 + mm) * plane;
                    if (y_aligned) {
                        st_stream_f4(dst, acc[mm][0], acc[mm][1], acc[mm][2], acc[mm][3]);
                    } else {
#pragma unroll
                        for (int t = 0; t < kPx; ++t) dst[t] = acc[mm][t];
                    }
                }
            }
        }
        buf ^= 1;
    }
    cp_async_wait_all();
}

// Fallback: KT > 0 fixes the kernel size at compile time; KT == 0 takes any k <= kMaxK.
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

// Generic loop nest (any C, k, pad, stride): conv_mcmk_loopnest (conv_direct.cpp:104-143)
// generalised to (pad, stride), one thread per output pixel x 8 output channels, taps read
// through L1 (the 8 weights of a tap are warp-uniform broadcasts).  It makes direct-gpu
// total -- every layer has a CUDA-core fp32 result, which `verify` uses as its comparator
// the way the reference's verify uses its own direct method -- not a fast path.
constexpr int kLnM = 8;

__global__ void __launch_bounds__(128) direct_loopnest_kernel(const float* __restrict__ x, const float* __restrict__ w,
                                                              float* __restrict__ y, int C, int H, int W, int M, int k,
                                                              int pad, int stride, int P, int Q) {
    const int pq = blockIdx.x * 128 + threadIdx.x;
    const int m0 = blockIdx.y * kLnM;
    const int n = blockIdx.z;
    if (pq >= P * Q) return;
    const int p = pq / Q, q = pq - p * Q;
    const int h0 = p * stride - pad, w0 = q * stride - pad;
    const float* xn = x + (long long)n * C * H * W;
    float acc[kLnM];
#pragma unroll
    for (int t = 0; t < kLnM; ++t) acc[t] = 0.0f;
    for (int c = 0; c < C; ++c) {
        const float* xc = xn + (long long)c * H * W;
        for (int i = 0; i < k; ++i) {
            const int hh = h0 + i;
            if (hh < 0 || hh >= H) continue;
            for (int j = 0; j < k; ++j) {
                const int ww = w0 + j;
                if (ww < 0 || ww >= W) continue;
                const float v = __ldg(xc + (long long)hh * W + ww);
                const long long wo = ((long long)i * k + j) * C + c;   // MKKC [m][i][j][c]
#pragma unroll
                for (int t = 0; t < kLnM; ++t)
                    if (m0 + t < M) acc[t] = fmaf(__ldg(w + (long long)(m0 + t) * k * k * C + wo), v, acc[t]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < kLnM; ++t)
        if (m0 + t < M) y[((long long)n * M + m0 + t) * P * Q + pq] = acc[t];
}

size_t persistent_smem_bytes(int C, int k, int M, int P, int Q) {
    const int Mp = (M + kMb - 1) / kMb * kMb;
    const UnitGeom g = unit_geom(P, Q, k);
    return ((size_t)((C * k * k * Mp + 3) & ~3) + 2 * (size_t)C * g.halo_rows * g.pitch) * sizeof(float);
}

template <typename K>
void set_smem(K kernel, size_t bytes) {
    CLB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

size_t direct_smem_bytes(int C, int k) {
    return (size_t)(C * (kTp + k - 1) * (kTq + k - 1) + kMb * C * k * k) * sizeof(float);
}

bool direct_fast_path(int C, int k, int stride) {
    return stride == 1 && k <= kMaxK && direct_smem_bytes(C, k) <= 200 * 1024;
}

bool direct_param_shape(int C, int k, int M, int stride, int Q) {
    return C == 3 && k == 3 && stride == 1 && Q % 4 == 0 && (M == 16 || M == 32 || M == 64);
}

void launch_direct_conv(const float* x, const float* w, float* y, int N, int C, int H, int W, int M, int k, int pad,
                        int stride, int P, int Q, cudaStream_t s, const float* w_param) {
    if (!direct_fast_path(C, k, stride)) {
        dim3 grid((P * Q + 127) / 128, (M + kLnM - 1) / kLnM, N);
        direct_loopnest_kernel<<<grid, 128, 0, s>>>(x, w, y, C, H, W, M, k, pad, stride, P, Q);
        CLB_CUDA(cudaGetLastError());
        return;
    }
    // the >48 KB smem opt-ins are per-device function attributes: configured once per device,
    // under a lock (a plan may live on any device of the process)
    static std::mutex mu;
    static bool configured[64] = {};
    static int sms_of[64] = {};
    int cur = 0;
    CLB_CUDA(cudaGetDevice(&cur));
    if (cur < 0 || cur >= 64) throw Error(1, "device index out of range");
    std::lock_guard<std::mutex> guard(mu);
    const int& sms = sms_of[cur];
    if (!configured[cur]) {
        set_smem(direct_conv_kernel<0>, 200 * 1024);
        set_smem(direct_conv_kernel<1>, 200 * 1024);
        set_smem(direct_conv_kernel<3>, 200 * 1024);
        set_smem(direct_conv_kernel<5>, 200 * 1024);
        set_smem(direct_persistent_kernel<0, 0>, kPersistentSmem);
        set_smem(direct_persistent_kernel<1, 0>, kPersistentSmem);
        set_smem(direct_persistent_kernel<3, 0>, kPersistentSmem);
        set_smem(direct_persistent_kernel<5, 0>, kPersistentSmem);
        set_smem(direct_persistent_kernel<3, 3>, kPersistentSmem);
        set_smem(direct_param_kernel<16>, kPersistentSmem / 2);
        set_smem(direct_param_kernel<32>, kPersistentSmem / 2);
        set_smem(direct_param_kernel<64>, kPersistentSmem / 2);
        CLB_CUDA(cudaDeviceGetAttribute(&sms_of[cur], cudaDevAttrMultiProcessorCount, cur));
        configured[cur] = true;
    }
    static const bool param_on = !(getenv("CLB_DIRECT_PARAM") && atoi(getenv("CLB_DIRECT_PARAM")) == 0);
    if (w_param && param_on && direct_param_shape(C, k, M, stride, Q)) {
        // weights as a kernel parameter (host copy packed [c][i][j][m] by the plan)
        const UnitGeom g = unit_geom(P, Q, k);
        const int num_units = N * g.units_img;
        const size_t psmem = 2 * (size_t)C * g.halo_rows * g.pitch * sizeof(float);
        if (psmem <= kPersistentSmem / 2 - 1024) {
            const int grid = std::min(num_units, sms * 2);
            auto go = [&](auto kernel, auto pw) {
                decltype(pw) wts;
                std::memcpy(wts.w, w_param, sizeof(wts.w));
                kernel<<<grid, kPThreads, psmem, s>>>(x, y, H, W, pad, P, Q, num_units, wts);
            };
            if (M == 64) go(direct_param_kernel<64>, ParamWeights<27 * 64>{});
            else if (M == 32) go(direct_param_kernel<32>, ParamWeights<27 * 32>{});
            else go(direct_param_kernel<16>, ParamWeights<27 * 16>{});
            CLB_CUDA(cudaGetLastError());
            return;
        }
    }
    const bool unit_ok = Q % 4 == 0 && C <= 4;   // groups of 4 never straddle a row
    const size_t psmem = unit_ok ? persistent_smem_bytes(C, k, M, P, Q) : 0;
    if (unit_ok && psmem <= kPersistentSmem) {
        const UnitGeom g = unit_geom(P, Q, k);
        const int num_units = N * g.units_img;
        const int per_sm = psmem <= kPersistentSmem / 2 - 1024 ? 2 : 1;
        const int grid = std::min(num_units, sms * per_sm);
        auto go = [&](auto kernel) {
            kernel<<<grid, kPThreads, psmem, s>>>(x, w, y, C, H, W, M, k, pad, P, Q, num_units);
        };
        if (k == 3 && C == 3) go(direct_persistent_kernel<3, 3>);
        else if (k == 1) go(direct_persistent_kernel<1, 0>);
        else if (k == 3) go(direct_persistent_kernel<3, 0>);
        else if (k == 5) go(direct_persistent_kernel<5, 0>);
        else go(direct_persistent_kernel<0, 0>);
        CLB_CUDA(cudaGetLastError());
        return;
    }
    const size_t smem = direct_smem_bytes(C, k);
    if (smem > 200 * 1024) throw Error(2, "direct-gpu: channel count too large for the shared-memory halo");
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
