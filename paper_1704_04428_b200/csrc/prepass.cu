// prepass.cu -- HBM-bound layout / split kernels around the tcgen05 engine, and the
// standalone shift-add kernels of the explicit kn2row / kn2col variants.
//
// All are coalesced on both sides (32x32 shared-memory transposes where the layout
// changes) and grid-stride free: one CTA per 32x32 tile.  None of them does arithmetic
// beyond the TF32 hi/lo split (hi = cvt.rna.tf32(x), lo = x - hi, exact in fp32).
#include <algorithm>
#include <cuda_bf16.h>

#include "internal.hpp"

namespace clb {

// Row layout (see internal.hpp): the fp32-faithful split formats pack one 128 B unit per
// 16-channel block ([hi fp32 | bf16 hi | bf16 lo] mixed, [hi | lo] fp32 for 3xTF32) so each
// 128-byte TMA row carries both halves of 16 channels; TF32 rows hold hi only.
// `base` = first element of the row (fp32 words, or bf16 elements for the BF16 mode).
__device__ __forceinline__ void store_split(void* dstv, long long base, int c, int kp, int planes, float v,
                                            Pow2 scale = Pow2{1.0f, 1.0f}) {
    (void)kp;
    if (planes == kPlanesBf16) {
        reinterpret_cast<__nv_bfloat16*>(dstv)[base + c] = __float2bfloat16_rn(v);
        return;
    }
    if (planes == kPlanesF16) {
        // unit = [hi fp16 32 | lo fp16 32] of the scaled value (32 words per 32 channels)
        const float xs = apply_pow2(v, scale);
        const __half hi = __float2half_rn(xs);
        __half* h = reinterpret_cast<__half*>(static_cast<float*>(dstv) + base + ((c >> 5) << 5));
        h[c & 31] = hi;
        h[32 + (c & 31)] = __float2half_rn(xs - __half2float(hi));
        return;
    }
    float* dst = static_cast<float*>(dstv);
    const float hi = tf32_rna(v);
    if (planes == 2) {
        const int u = (c >> 4) << 5, w = c & 15;
        dst[base + u + w] = hi;
        dst[base + u + 16 + w] = v - hi;
    } else if (planes == kPlanesMixed) {
        // unit = [hi 16 fp32 | bf16(hi) 16 | bf16(lo) 16]
        const int u = (c >> 4) << 5, w = c & 15;
        dst[base + u + w] = hi;
        __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(dst + base + u);
        h[32 + w] = __float2bfloat16_rn(hi);
        h[48 + w] = __float2bfloat16_rn(v - hi);
    } else {
        dst[base + c] = hi;
    }
}

__device__ __forceinline__ long long rowel(int planes, long long kp) { return is_split(planes) ? 2 * kp : kp; }

// ------------------------------------------------------------------ NCHW -> NHWC split ----
// Tile = 32 channels x 128 pixels of one image, 256 threads.  Loads: warp w reads channel
// rows w, w+8, w+16, w+24 in four 128-byte pieces each -- 16 independent loads in flight per
// thread (the kernel is HBM-bound; memory-level parallelism is what it needs).  Stores: per
// pixel the tile's output is one contiguous run of 64 words (two 16-channel units for the split formats, 32
// hi words for TF32), written by a warp as full 128-byte lines (lane = word).
// grid (ceil(HW/128), ceil(Cp/32), N)
// (tile body, FastDiv: split_tile.cuh)
// fp16 split: a 1-D grid walked in REVERSE (tile t = total - 1 - blockIdx.x, channel blocks of a
// pixel block adjacent): the absmax pass just streamed x front to back, so the last images are
// the ones still in L2 -- converting them first turns the second read of x into L2 hits for
// inputs up to about the L2 size.
template <int PLANES>
__global__ void __launch_bounds__(256) nchw_to_nhwc_split_kernel(const float* __restrict__ x, void* __restrict__ xsv,
                                                                 int N, int C, int HW, int Cp, int H, int W, int Wp,
                                                                 int pad, FastDiv hwd, FastDiv wpd, const int* sexp) {
    // launched as a programmatic dependent of the previous kernel in the stream (typically the
    // previous layer's contraction, whose output x is): nothing is touched before it completes
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ SplitSmem<PLANES> sm;
    int bx = (int)blockIdx.x, by = (int)blockIdx.y;
    Pow2 scale{1.0f, 1.0f};
    if constexpr (PLANES == kPlanesF16) {
        const int nty = (Cp + 31) / 32;
        const int t = (int)gridDim.x - 1 - (int)blockIdx.x;
        bx = t / nty;
        by = t - bx * nty;
        scale = pow2_factors(__ldg(sexp + 1));
    }
    split_tile<PLANES>(x, xsv, N, C, HW, Cp, H, W, Wp, pad, hwd, wpd, bx, by, (int)threadIdx.x, sm, scale);
    // let a programmatically dependent consumer (the tcgen05 kernel) start its prologue;
    // its griddepcontrol.wait still waits for this grid's completion and memory flush
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... Args>
static void launch_split_kernel(int planes, dim3 grid, cudaStream_t s, Args... args) {
    if (planes == kPlanesF16) grid = dim3(grid.x * grid.y, 1, 1);   // reversed linear tile order
    // Programmatic dependent launch: the prepass's launch and CTA ramp overlap the tail of the
    // previous kernel in the stream (the previous layer's contraction); its griddepcontrol.wait
    // keeps every memory access after that kernel's completion.  CLB_PDL_PREPASS=0 disables.
    static const bool pdl = !(getenv("CLB_PDL_PREPASS") && atoi(getenv("CLB_PDL_PREPASS")) == 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    switch (planes) {
        case 1: CLB_CUDA(cudaLaunchKernelEx(&cfg, nchw_to_nhwc_split_kernel<1>, args...)); break;
        case 2: CLB_CUDA(cudaLaunchKernelEx(&cfg, nchw_to_nhwc_split_kernel<2>, args...)); break;
        case kPlanesBf16: CLB_CUDA(cudaLaunchKernelEx(&cfg, nchw_to_nhwc_split_kernel<kPlanesBf16>, args...)); break;
        case kPlanesF16: CLB_CUDA(cudaLaunchKernelEx(&cfg, nchw_to_nhwc_split_kernel<kPlanesF16>, args...)); break;
        default: CLB_CUDA(cudaLaunchKernelEx(&cfg, nchw_to_nhwc_split_kernel<kPlanesMixed>, args...));
    }
}

void launch_nchw_to_nhwc_split(const float* x, void* xs, int N, int C, int HW, int Cp, int planes,
                               cudaStream_t s, const int* sexp) {
    if (planes == kPlanesF16 && !sexp) throw Error(6, "fp16 split prepass without its exponent slots");
    dim3 grid((unsigned)(((long long)N * HW + kSplitPx - 1) / kSplitPx), (Cp + 31) / 32, 1);
    launch_split_kernel(planes, grid, s, x, xs, N, C, HW, Cp, 1, HW, HW, 0, make_fastdiv((uint32_t)HW),
                        make_fastdiv((uint32_t)HW), sexp);
    CLB_CUDA(cudaGetLastError());
}

// The same conversion as a job over its tile grid (chained mode): the tail kernel takes tiles
// from the job's counter (left off by the previous contraction's converter warps) until all are
// done; persistent CTAs, one tile at a time through the smem staging of split_tile.
SplitJob make_split_job(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp) {
    SplitJob j{};
    const int Hp = pad > 0 ? H + pad : H, Wp = pad > 0 ? W + pad : W;
    j.x = x;
    j.xs = xs;
    j.n = N;
    j.c = C;
    j.hw = Hp * Wp;
    j.cp = Cp;
    j.h = pad > 0 ? H : 1;
    j.w = pad > 0 ? W : H * W;
    j.wp = pad > 0 ? Wp : H * W;
    j.pad = pad;
    j.hwd = make_fastdiv((uint32_t)j.hw);
    j.wpd = make_fastdiv((uint32_t)j.wp);
    j.ntx = (int)(((long long)N * j.hw + kSplitPx - 1) / kSplitPx);
    j.nty = (Cp + 31) / 32;
    return j;
}

template <int PLANES>
__global__ void __launch_bounds__(256) split_tail_kernel(const SplitJob j) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ SplitSmem<PLANES> sm;
    __shared__ int tile;
    const int total = j.ntx * j.nty;
    for (;;) {
        if (threadIdx.x == 0) tile = (int)atomicAdd(j.counter, 1u);
        __syncthreads();
        const int t = tile;
        if (t >= total) break;
        split_tile<PLANES>(j.x, j.xs, j.n, j.c, j.hw, j.cp, j.h, j.w, j.wp, j.pad, j.hwd, j.wpd, t / j.nty, t % j.nty,
                           (int)threadIdx.x, sm);
        __syncthreads();   // the staging is reused by the next tile
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

void launch_split_tail(const SplitJob& j, int planes, cudaStream_t s) {
    int dev = 0, sms = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    CLB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long total = (long long)j.ntx * j.nty;
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(total, 6LL * sms));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (planes == 2) CLB_CUDA(cudaLaunchKernelEx(&cfg, split_tail_kernel<2>, j));
    else if (planes == kPlanesMixed) CLB_CUDA(cudaLaunchKernelEx(&cfg, split_tail_kernel<kPlanesMixed>, j));
    else throw Error(6, "chained prepass: split formats only");
    // reset the counter for the job's next use (stream-ordered, graph-capturable)
    CLB_CUDA(cudaMemsetAsync(j.counter, 0, sizeof(unsigned), s));
}

void launch_nchw_to_padded_split(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp, int planes,
                                 cudaStream_t s, const int* sexp, int wp) {
    if (planes == kPlanesF16 && !sexp) throw Error(6, "fp16 split prepass without its exponent slots");
    const int Hp = H + pad, Wp = wp > 0 ? wp : W + pad;
    dim3 grid((unsigned)(((long long)N * Hp * Wp + kSplitPx - 1) / kSplitPx), (Cp + 31) / 32, 1);
    launch_split_kernel(planes, grid, s, x, xs, N, C, Hp * Wp, Cp, H, W, Wp, pad, make_fastdiv((uint32_t)(Hp * Wp)),
                        make_fastdiv((uint32_t)Wp), sexp);
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- NHWC -> split rows ----
// Channels-last input (the reference's HWC Tensor3 layout, tensor.hpp:86-90, stacked):
// the split is elementwise along each pixel row, so no transpose: thread = (output row,
// 4 channels), float4 in, hi / lo float4 out.  The output rows are either the image pixels
// or (pad > 0) the zero-padded pixel grid of the tap-shared mode.  (row, quad) comes from a
// multiply-shift divide (n < 2^31): a runtime 32/64-bit division per element costs more
// issue slots than the bytes it moves.
__global__ void __launch_bounds__(256) nhwc_split_kernel(const float* __restrict__ x, void* __restrict__ xs,
                                                         uint32_t total, FastDiv q4d, FastDiv pixd, FastDiv wpd, int C,
                                                         int Cp, int planes, int H, int W, int pad, const int* sexp) {
    const uint32_t i = blockIdx.x * 256u + threadIdx.x;
    if (i >= total) return;
    const uint32_t r = fdiv(i, q4d);                 // output row
    const int c = (int)(i - r * q4d.d) * 4;          // first of 4 channels
    long long src = r;
    if (pad > 0) {                                   // padded grid: row = (n, yp, xp)
        const uint32_t n = fdiv(r, pixd);
        const uint32_t rem = r - n * pixd.d;
        const uint32_t yp = fdiv(rem, wpd);
        const int y = (int)yp, xq = (int)(rem - yp * wpd.d);
        src = (y < H && xq < W) ? ((long long)n * H + y) * W + xq : -1;
    }
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (src >= 0) {
        const float* px = x + src * C + c;
        if ((C & 3) == 0 && c + 3 < C) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(px));
            v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (c + e < C) v[e] = __ldg(px + e);
        }
    }
    if (planes == kPlanesBf16) {
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(xs) + (long long)r * Cp + c;
        __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
        uint2 packed;
        packed.x = *reinterpret_cast<uint32_t*>(&a);
        packed.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(dst) = packed;
        return;
    }
    if (planes == kPlanesF16) {                       // [hi fp16 32 | lo fp16 32] per 32 channels
        const Pow2 sc = pow2_factors(__ldg(sexp + 1));
        uint32_t h01, l01, h23, l23;
        f16_split2(apply_pow2(v[0], sc), apply_pow2(v[1], sc), h01, l01);
        f16_split2(apply_pow2(v[2], sc), apply_pow2(v[3], sc), h23, l23);
        uint32_t* dst = reinterpret_cast<uint32_t*>(static_cast<float*>(xs) + (long long)r * Cp + ((c >> 5) << 5));
        const int w = (c & 31) >> 1;                  // word of the channel pair within each half
        *reinterpret_cast<uint2*>(dst + w) = make_uint2(h01, h23);
        *reinterpret_cast<uint2*>(dst + 16 + w) = make_uint2(l01, l23);
        return;
    }
    float hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        hi[e] = tf32_rna(v[e]);
        lo[e] = v[e] - hi[e];
    }
    float* dst = static_cast<float*>(xs) + (long long)r * rowel(planes, Cp);
    if (planes == 2) {
        const int u = (c >> 4) << 5, w = c & 15;      // 128 B unit [hi 16 | lo 16]
        *reinterpret_cast<float4*>(dst + u + w) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<float4*>(dst + u + 16 + w) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    } else if (planes == kPlanesMixed) {
        const int u = (c >> 4) << 5, w = c & 15;      // [hi 16 fp32 | bf16(hi) 16 | bf16(lo) 16]
        *reinterpret_cast<float4*>(dst + u + w) = make_float4(hi[0], hi[1], hi[2], hi[3]);
        uint32_t* bw = reinterpret_cast<uint32_t*>(dst + u);
        *reinterpret_cast<uint2*>(bw + 16 + (w >> 1)) = make_uint2(bf16x2_bits(hi[0], hi[1]), bf16x2_bits(hi[2], hi[3]));
        *reinterpret_cast<uint2*>(bw + 24 + (w >> 1)) = make_uint2(bf16x2_bits(lo[0], lo[1]), bf16x2_bits(lo[2], lo[3]));
    } else {
        *reinterpret_cast<float4*>(dst + c) = make_float4(hi[0], hi[1], hi[2], hi[3]);
    }
}

void launch_nhwc_split(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp, int planes,
                       cudaStream_t s, const int* sexp, int wp) {
    if (planes == kPlanesF16 && !sexp) throw Error(6, "fp16 split prepass without its exponent slots");
    const int Hp = H + pad, Wp = pad > 0 && wp > 0 ? wp : W + pad;   // pad > 0: shared-padding grid (see above)
    const long long rows = (long long)N * Hp * Wp;
    const int q4 = Cp / 4;
    const long long total = rows * q4;
    if (total >= (1ll << 31)) throw Error(2, "NHWC prepass: more than 2^31 channel quads (split the batch)");
    const FastDiv q4d = make_fastdiv((uint32_t)q4), pixd = make_fastdiv((uint32_t)(Hp * Wp)),
                  wpd = make_fastdiv((uint32_t)Wp);
    nhwc_split_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(x, xs, (uint32_t)total, q4d, pixd, wpd, C, Cp,
                                                                      planes, H, W, pad, sexp);
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- fp16 split exponent ----
// max|x| over the tensor -> the power-of-2 shift of the fp16 split.  Each block reduces a
// grid-stride share (float4 loads when aligned) to one partial; the last block to finish (a
// completion counter) reduces the partials, writes the exponent and resets the counter, so the
// slots need no memset between calls.  |x| as unsigned bits orders like the float (NaN above inf).
__global__ void __launch_bounds__(256) absmax_exp_kernel(const float* __restrict__ x, long long n, int* slots,
                                                         int* out_exp) {
    asm volatile("griddepcontrol.wait;" ::: "memory");   // x may be the previous kernel's output
    unsigned* part = reinterpret_cast<unsigned*>(slots + kScaleSlots);
    unsigned* counter = reinterpret_cast<unsigned*>(slots + 2);
    unsigned m = 0;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
    auto fold4 = [&](const float4& v) {
        m = max(max(m, __float_as_uint(v.x) & 0x7fffffffu), __float_as_uint(v.y) & 0x7fffffffu);
        m = max(max(m, __float_as_uint(v.z) & 0x7fffffffu), __float_as_uint(v.w) & 0x7fffffffu);
    };
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
        // 8 independent 16-byte loads in flight per thread: HBM needs several MB in flight
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const long long n4 = n >> 2;
        long long i = tid;
        for (; i + 7 * nth < n4; i += 8 * nth) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(x4 + i + u * nth);
#pragma unroll
            for (int u = 0; u < 8; ++u) fold4(v[u]);
        }
        for (; i < n4; i += nth) fold4(__ldg(x4 + i));
        for (long long j = (n4 << 2) + tid; j < n; j += nth) m = max(m, __float_as_uint(__ldg(x + j)) & 0x7fffffffu);
    } else {
        for (long long i = tid; i < n; i += nth) m = max(m, __float_as_uint(__ldg(x + i)) & 0x7fffffffu);
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ unsigned wm[8];
    __shared__ bool last;
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = max(m, wm[w]);
        part[blockIdx.x] = m;
        __threadfence();
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
        __threadfence();
        m = 0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 256) m = max(m, __ldcg(part + b));
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; ++w) m = max(m, wm[w]);
            *out_exp = f16_split_exponent(m);
            *counter = 0u;
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

void launch_absmax_exp(const float* x, long long n, int* slots, int* out_exp, cudaStream_t s) {
    int dev = 0, sms = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    CLB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const long long want = (n / 4 + 2047) / 2048;   // >= 8 float4 per thread
    const unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(want, std::min(kAbsmaxBlocks, 4 * sms)));
    static const bool pdl = !(getenv("CLB_PDL_PREPASS") && atoi(getenv("CLB_PDL_PREPASS")) == 0);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    CLB_CUDA(cudaLaunchKernelEx(&cfg, absmax_exp_kernel, x, n, slots, out_exp));
}

// ------------------------------------------------ fp16 split, speculative single pass ----
// Slots: [1] ex (exact exponent of this input, read by the contraction), [3] e_spec / [4] valid
// (the exponent of the plan's previous forward), [5] unused, [6] e_use (the exponent this
// forward's split was written with); group maxima after the absmax partials (kSpecGroups: every
// block folds its max into group blockIdx % kSpecGroups with one fire-and-forget atomicMax, so no
// address sees more than ~1/64 of the atomics).  The fixup kernel (launched right behind, PDL)
// folds the groups, publishes ex / e_spec and re-converts the input when e_use != ex; the
// contraction behind it zeroes the groups for the next forward (TcParams::reset_slots) -- every
// kernel touching them is then complete.
struct SpecHook {
    unsigned* gmax;
    uint32_t* wmax;   // shared [8]
    int g;
    __device__ __forceinline__ void after_load(uint32_t m) {
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = m;
    }
    __device__ __forceinline__ void after_sync() {   // after the mid-tile barrier: wmax is complete
        if (threadIdx.x == 0) {
            uint32_t m = wmax[0];
#pragma unroll
            for (int w = 1; w < 8; ++w) m = max(m, wmax[w]);
            atomicMax(gmax + g * kSpecStride, m);   // result unused: a RED, no wait
        }
    }
};

__global__ void __launch_bounds__(256) split_spec_kernel(const float* __restrict__ x, void* __restrict__ xsv, int N,
                                                          int C, int HW, int Cp, int H, int W, int Wp, int pad,
                                                          FastDiv hwd, FastDiv wpd, int* slots) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ SplitSmem<kPlanesF16> sm;
    __shared__ uint32_t wmax[8];
    const int nty = (Cp + 31) / 32;
    const int t = (int)gridDim.x - 1 - (int)blockIdx.x;     // reversed tile order (see the kernel above)
    const int bx = t / nty, by = t - bx * nty;
    const int e_use = slots[4] ? slots[3] : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) slots[6] = e_use;
    SpecHook hook{reinterpret_cast<unsigned*>(slots + kScaleSlots + kAbsmaxBlocks), wmax,
                  (int)(blockIdx.x % kSpecGroups)};
    split_tile<kPlanesF16>(x, xsv, N, C, HW, Cp, H, W, Wp, pad, hwd, wpd, bx, by, (int)threadIdx.x, sm,
                           pow2_factors(e_use), &hook);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Folds the group maxima into the exact exponent ex (every block computes the same value and
// publishes it), and re-converts the whole input with ex when the speculative pass used another
// exponent; otherwise returns at once.  Persistent grid; it always waits for the prepass first,
// so a contraction launched behind it (PDL) is ordered after both.
__global__ void __launch_bounds__(256) split_fixup_kernel(const float* __restrict__ x, void* __restrict__ xsv, int N,
                                                           int C, int HW, int Cp, int H, int W, int Wp, int pad,
                                                           FastDiv hwd, FastDiv wpd, int* slots, int total) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ int e_sh;
    const int e_use = __ldcg(slots + 6);   // issued with the group loads (one round trip)
    if (threadIdx.x < 32) {
        const unsigned* gmax = reinterpret_cast<const unsigned*>(slots + kScaleSlots + kAbsmaxBlocks);
        uint32_t a = 0;
        for (int g = (int)threadIdx.x; g < kSpecGroups; g += 32) a = max(a, __ldcg(gmax + g * kSpecStride));
        for (int o = 16; o > 0; o >>= 1) a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
        if (threadIdx.x == 0) {
            const int e = f16_split_exponent(a);
            e_sh = e;
            slots[1] = e;      // identical in every block
            slots[3] = e;      // the next forward's speculation
            slots[4] = 1;
        }
    }
    __syncthreads();
    const int e = e_sh;
    if (e != e_use) {
        __shared__ SplitSmem<kPlanesF16> sm;
        const int nty = (Cp + 31) / 32;
        const Pow2 sc = pow2_factors(e);
        for (int t = (int)blockIdx.x; t < total; t += (int)gridDim.x) {
            const int bx = t / nty, by = t - bx * nty;
            split_tile<kPlanesF16>(x, xsv, N, C, HW, Cp, H, W, Wp, pad, hwd, wpd, bx, by, (int)threadIdx.x, sm, sc);
            __syncthreads();   // the staging is reused by the next tile
        }
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

void launch_nchw_split_speculative(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp, int* slots,
                                   cudaStream_t s, int wp) {
    // pad > 0: the zero-padded grid of the tap-shared mode (row width wp, default W + pad);
    // pad == 0: the image pixels
    const int Hp = pad > 0 ? H + pad : H, Wp = pad > 0 ? (wp > 0 ? wp : W + pad) : W;
    const int HW = Hp * Wp;
    const long long ntx = ((long long)N * HW + kSplitPx - 1) / kSplitPx, nty = (Cp + 31) / 32;
    if (ntx * nty >= (1LL << 31)) throw Error(2, "prepass: too many tiles (split the batch)");
    const int total = (int)(ntx * nty);
    const FastDiv hwd = make_fastdiv((uint32_t)HW), wpd = make_fastdiv((uint32_t)Wp);
    const int h = pad > 0 ? H : 1, w = pad > 0 ? W : HW;   // the unpadded path reads rows of HW pixels
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)total);
    CLB_CUDA(cudaLaunchKernelEx(&cfg, split_spec_kernel, x, xs, N, C, HW, Cp, h, w, Wp, pad, hwd, wpd, slots));
    int dev = 0, sms = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    CLB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cfg.gridDim = dim3((unsigned)std::max(1, std::min(total, sms)));   // one block per SM: a hit reads 64 slots and exits
    CLB_CUDA(cudaLaunchKernelEx(&cfg, split_fixup_kernel, x, xs, N, C, HW, Cp, h, w, Wp, pad, hwd, wpd, slots, total));
}

// -------------------------------------------------------------------- row-wise split ----
// grid (ceil(Kp/128), rows), block 128
__global__ void rows_split_kernel(const float* __restrict__ a, void* __restrict__ as, int K, int Kp,
                                  int planes, const int* sexp) {
    const long long r = blockIdx.y;
    const int c = blockIdx.x * 128 + threadIdx.x;
    if (c >= Kp) return;
    const float v = c < K ? __ldg(a + r * K + c) : 0.0f;
    store_split(as, r * rowel(planes, Kp), c, Kp, planes, v, sexp ? pow2_factors(sexp[0]) : Pow2{1.0f, 1.0f});
}

void launch_rows_split(const float* a, void* as, long long rows, int K, int Kp, int planes, cudaStream_t s,
                       const int* sexp) {
    if (rows <= 0) return;
    if (planes == kPlanesF16 && !sexp) throw Error(6, "fp16 split rows without their exponent slot");
    for (long long r0 = 0; r0 < rows; r0 += 65535) {
        const long long nr = rows - r0 < 65535 ? rows - r0 : 65535;
        dim3 grid((Kp + 127) / 128, (unsigned)nr);
        rows_split_kernel<<<grid, 128, 0, s>>>(a + r0 * K, static_cast<char*>(as) + r0 * row_bytes(planes, Kp), K,
                                               Kp, planes, planes == kPlanesF16 ? sexp : nullptr);
    }
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------- transpose + split (B^T) ----
// b[K][cols] -> bs[cols][planes][Kp]; grid (ceil(cols/32), ceil(Kp/32)), block (32, 8)
__global__ void transpose_split_kernel(const float* __restrict__ b, void* __restrict__ bs, int K, int cols,
                                       int Kp, int planes) {
    __shared__ float tile[32][33];
    const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    for (int kk = threadIdx.y; kk < 32; kk += 8) {
        const int kx = k0 + kk, n = n0 + threadIdx.x;
        tile[kk][threadIdx.x] = (kx < K && n < cols) ? __ldg(b + (long long)kx * cols + n) : 0.0f;
    }
    __syncthreads();
    for (int nn = threadIdx.y; nn < 32; nn += 8) {
        const int n = n0 + nn, kx = k0 + threadIdx.x;
        if (n < cols && kx < Kp) store_split(bs, (long long)n * rowel(planes, Kp), kx, Kp, planes, tile[threadIdx.x][nn]);
    }
}

void launch_transpose_split(const float* b, void* bs, int K, int cols, int Kp, int planes, cudaStream_t s) {
    dim3 grid((cols + 31) / 32, (Kp + 31) / 32), block(32, 8);
    transpose_split_kernel<<<grid, block, 0, s>>>(b, bs, K, cols, Kp, planes);
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------ weight pre-pack ----
// kn2row_reorder_kernel (conv_kn2.cpp:28-39) fused with the split:
//   wp[(i*k+j)][m][plane][c] = split(K[m][i][j][c])
__global__ void pack_weights_kernel(const float* __restrict__ w, void* __restrict__ wp, int M, int k, int C,
                                    int Cp, int planes, int stacked, const int* sexp) {
    const long long total = (long long)k * k * M * Cp;
    const Pow2 scale = sexp ? pow2_factors(sexp[0]) : Pow2{1.0f, 1.0f};   // fp16 split: 2^ew
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e % Cp);
        const long long tm = e / Cp;
        const int m = (int)(tm % M);
        const int t = (int)(tm / M);
        const float v = c < C ? w[((long long)m * k * k + t) * C + c] : 0.0f;
        // tap-major [t][m] rows, or tap-stacked [i][m][j] (the k taps of kernel row i as
        // adjacent columns of one output channel, tc_conv.cuh stack_k)
        const long long row = stacked ? ((long long)(t / k) * M + m) * k + (t % k) : tm;
        store_split(wp, row * rowel(planes, Cp), c, Cp, planes, v, scale);
    }
}

void launch_pack_weights(const float* w, void* wp, int M, int k, int C, int Cp, int planes, cudaStream_t s,
                         bool stacked, const int* sexp) {
    if (planes == kPlanesF16 && !sexp) throw Error(6, "fp16 split weights without their exponent slot");
    const long long total = (long long)k * k * M * Cp;
    const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    pack_weights_kernel<<<blocks, 256, 0, s>>>(w, wp, M, k, C, Cp, planes, stacked ? 1 : 0,
                                               planes == kPlanesF16 ? sexp : nullptr);
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------- im2col ----
// Patch matrix in the K-major orientation the engine consumes (the im2row shape of
// conv_im2.cpp:56-85 with im2col's K order (i*k+j)*C+c of conv_im2.cpp:19-54):
//   pm[pix = (n,p,q)][plane][kk = (i*k+j)*C + c] = x[n][c][p*s-pad+i][q*s-pad+j]  (0 if OOB)
// grid (ceil(NPQ/32), ceil(Kp/32)), block (32, 8): gather coalesced along pixels, write along K.
__global__ void im2col_split_kernel(const float* __restrict__ x, void* __restrict__ pm, int C, int H, int W,
                                    int k, int pad, int stride, int P, int Q, long long npq, int Kp, int planes) {
    __shared__ float tile[32][33];
    const long long pix0 = (long long)blockIdx.x * 32;
    const int k0 = blockIdx.y * 32;
    const int KC = k * k * C;
    // this thread's pixel for the gather phase
    const long long pix = pix0 + threadIdx.x;
    int n = 0, p = 0, q = 0;
    if (pix < npq) {
        n = (int)(pix / ((long long)P * Q));
        const int rem = (int)(pix - (long long)n * P * Q);
        p = rem / Q;
        q = rem - p * Q;
    }
    for (int kk = threadIdx.y; kk < 32; kk += 8) {
        const int kx = k0 + kk;
        float v = 0.0f;
        if (pix < npq && kx < KC) {
            const int c = kx % C, t = kx / C;
            const int i = t / k, j = t - (t / k) * k;
            const int sh = p * stride - pad + i, sw = q * stride - pad + j;
            if (sh >= 0 && sh < H && sw >= 0 && sw < W)
                v = __ldg(x + (((long long)n * C + c) * H + sh) * W + sw);
        }
        tile[kk][threadIdx.x] = v;
    }
    __syncthreads();
    for (int pp = threadIdx.y; pp < 32; pp += 8) {
        const long long pr = pix0 + pp;
        const int kx = k0 + threadIdx.x;
        if (pr < npq && kx < Kp) store_split(pm, pr * rowel(planes, Kp), kx, Kp, planes, tile[threadIdx.x][pp]);
    }
}

void launch_im2col_split(const float* x, void* pm, int N, int C, int H, int W, int k, int pad, int stride,
                         int P, int Q, int Kp, int planes, cudaStream_t s) {
    const long long npq = (long long)N * P * Q;
    dim3 grid((unsigned)((npq + 31) / 32), (Kp + 31) / 32), block(32, 8);
    im2col_split_kernel<<<grid, block, 0, s>>>(x, pm, C, H, W, k, pad, stride, P, Q, npq, Kp, planes);
    CLB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------- shift-add ----
// Row orientation (conv_kn2.cpp:94-118), batched: inter[(t*M+m)][n*H*W + h*W + w].
// out[n][m][p][q] = sum_{i<k} sum_{j<k} inter[(i*k+j)*M+m][n, p-pad+i, q-pad+j], OOB skipped,
// i outer / j inner (the reference's accumulation order).  One thread per output element,
// q fastest -> coalesced loads of each tap row and coalesced stores.
__global__ void shift_add_row_kernel(const float* __restrict__ inter, float* __restrict__ y, int N, int M,
                                     int H, int W, int k, int pad, int P, int Q) {
    const long long total = (long long)N * M * P * Q;
    const long long ld = (long long)N * H * W;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(e % Q);
        long long r = e / Q;
        const int p = (int)(r % P);
        r /= P;
        const int m = (int)(r % M);
        const int n = (int)(r / M);
        float acc = 0.0f;
        for (int i = 0; i < k; ++i) {
            const int sh = p - pad + i;
            if (sh < 0 || sh >= H) continue;
            for (int j = 0; j < k; ++j) {
                const int sw = q - pad + j;
                if (sw < 0 || sw >= W) continue;
                acc += __ldg(inter + ((long long)(i * k + j) * M + m) * ld + ((long long)n * H + sh) * W + sw);
            }
        }
        y[e] = acc;
    }
}

void launch_shift_add_row(const float* inter, float* y, int N, int M, int H, int W, int k, int pad, int P,
                          int Q, cudaStream_t s) {
    const long long total = (long long)N * M * P * Q;
    const int blocks = (int)((total + 255) / 256 < 148 * 64 ? (total + 255) / 256 : 148 * 64);
    shift_add_row_kernel<<<blocks, 256, 0, s>>>(inter, y, N, M, H, W, k, pad, P, Q);
    CLB_CUDA(cudaGetLastError());
}

// Column orientation (conv_kn2.cpp:120-142), batched: inter[n*H*W + h*W + w][t*M + m].
// A 32-pixel x 32-channel output tile: gather coalesced along m, transpose through shared
// memory, store coalesced along pixels into NCHW.  grid (ceil(NPQ/32), ceil(M/32)), block (32,8)
__global__ void shift_add_col_kernel(const float* __restrict__ inter, float* __restrict__ y, int N, int M,
                                     int H, int W, int k, int pad, int P, int Q) {
    __shared__ float tile[32][33];
    const long long npq = (long long)N * P * Q;
    const long long pix0 = (long long)blockIdx.x * 32;
    const int m0 = blockIdx.y * 32;
    const long long ld = (long long)k * k * M;
    const int m = m0 + threadIdx.x;
    for (int pp = threadIdx.y; pp < 32; pp += 8) {
        const long long pix = pix0 + pp;
        float acc = 0.0f;
        if (pix < npq && m < M) {
            const int n = (int)(pix / ((long long)P * Q));
            const int rem = (int)(pix - (long long)n * P * Q);
            const int p = rem / Q, q = rem - (rem / Q) * Q;
            for (int i = 0; i < k; ++i) {
                const int sh = p - pad + i;
                if (sh < 0 || sh >= H) continue;
                for (int j = 0; j < k; ++j) {
                    const int sw = q - pad + j;
                    if (sw < 0 || sw >= W) continue;
                    acc += __ldg(inter + (((long long)n * H + sh) * W + sw) * ld + (long long)(i * k + j) * M + m);
                }
            }
        }
        tile[pp][threadIdx.x] = acc;
    }
    __syncthreads();
    for (int mm = threadIdx.y; mm < 32; mm += 8) {
        const long long pix = pix0 + threadIdx.x;
        const int mo = m0 + mm;
        if (pix < npq && mo < M) {
            const int n = (int)(pix / ((long long)P * Q));
            const int rem = (int)(pix - (long long)n * P * Q);
            y[((long long)n * M + mo) * P * Q + rem] = tile[threadIdx.x][mm];
        }
    }
}

void launch_shift_add_col(const float* inter, float* y, int N, int M, int H, int W, int k, int pad, int P,
                          int Q, cudaStream_t s) {
    const long long npq = (long long)N * P * Q;
    dim3 grid((unsigned)((npq + 31) / 32), (M + 31) / 32), block(32, 8);
    shift_add_col_kernel<<<grid, block, 0, s>>>(inter, y, N, M, H, W, k, pad, P, Q);
    CLB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------- generator ----
// rng::unit_value (tensor.cpp:117-123): top 24 bits of splitmix64(seed + (i+1) gamma),
// scaled by 2^-23 and shifted -- exact in fp32, so bit-identical to the host generator.
__global__ void fill_uniform_kernel(float* __restrict__ d, unsigned long long n, unsigned long long seed,
                                    unsigned long long first) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        unsigned long long z = seed + (first + i + 1ull) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const unsigned top = (unsigned)(z >> 40);
        d[i] = __fsub_rn(__fmul_rn((float)top, 0x1p-23f), 1.0f);
    }
}

void launch_fill_uniform(float* d, unsigned long long n, unsigned long long seed, unsigned long long first,
                         cudaStream_t s) {
    if (n == 0) return;
    const unsigned long long want = (n + 255) / 256;
    const int blocks = (int)(want < 148ull * 32 ? want : 148ull * 32);
    fill_uniform_kernel<<<blocks, 256, 0, s>>>(d, n, seed, first);
    CLB_CUDA(cudaGetLastError());
}

}  // namespace clb
