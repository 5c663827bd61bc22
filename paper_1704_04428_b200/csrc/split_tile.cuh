// split_tile.cuh -- one tile of the NCHW fp32 -> split-operand prepass (128 pixels x 32
// channels) of the prepass kernel (prepass.cu): hi = rna_tf32(x), lo = x - hi (exact in fp32),
// written as the 128-byte row units the engine's TMA boxes read.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

namespace clb {

constexpr int kPlanesBf16 = 3;    // precision codes, see internal.hpp
constexpr int kPlanesMixed = 4;
constexpr int kPlanesF16 = 5;     // fp32-faithful fp16 split of the power-of-2 scaled operand

// 2^e as a float, e in [-126, 127] (exact; the fp16 split's scale and descale factors)
__host__ __device__ __forceinline__ float exp2i(int e) {
    union { uint32_t u; float f; } v;
    v.u = (uint32_t)(127 + e) << 23;
    return v.f;
}

// x * 2^e for any e in [-252, 254] as two exact power-of-2 factors (a single float factor stops
// at 2^127: subnormal inputs need shifts up to 2^164)
struct Pow2 {
    float a, b;
};
__host__ __device__ __forceinline__ Pow2 pow2_factors(int e) {
    const int e1 = e < -126 ? -126 : (e > 127 ? 127 : e);
    return Pow2{exp2i(e1), exp2i(e - e1)};
}
__device__ __forceinline__ float apply_pow2(float v, const Pow2& f) { return (v * f.a) * f.b; }

// The fp16 split's exponent shift for a tensor whose max |x| has the (ordered) bits m: max 2^e in
// [2^14, 2^15), e in [-113, 163] for every finite nonzero max; 0 for zero / non-finite tensors.
__device__ __forceinline__ int f16_split_exponent(uint32_t m) {
    if (m == 0 || m >= 0x7f800000u) return 0;
    int ex;
    frexpf(__uint_as_float(m), &ex);   // max = f 2^ex, f in [0.5, 1)
    return 15 - ex;
}

// fp16 split of one scaled value pair: hi = fp16(x), lo = fp16(x - hi) (x - hi is exact in fp32),
// packed as the two halves of a 32-bit word each (channel c in the low half, c + 1 in the high)
__device__ __forceinline__ void f16_split2(float a, float b, uint32_t& hi, uint32_t& lo) {
    const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
    const __half la = __float2half_rn(a - __half2float(ha)), lb = __float2half_rn(b - __half2float(hb));
    hi = (uint32_t)__half_as_ushort(ha) | ((uint32_t)__half_as_ushort(hb) << 16);
    lo = (uint32_t)__half_as_ushort(la) | ((uint32_t)__half_as_ushort(lb) << 16);
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// The same rounding in two integer instructions (half an ulp of the 10-bit mantissa added to
// the magnitude, low 13 bits cleared: ties away from zero; carries into the exponent are the
// correct rounding up), bit-identical to cvt.rna.tf32.f32 for every finite input -- for the
// compute-bound in-kernel conversion (cvt.rna.tf32 is several instructions on sm_100).
__device__ __forceinline__ uint32_t tf32_rna_bits(float x) {
    return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
}

__device__ __forceinline__ uint32_t bf16x2_bits(float a, float b) {
    __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&t);
}

constexpr int kSplitPx = 128;

// Output pixel space: HW = Hp*Wp pixels per image; with pad > 0 this is the zero-padded
// grid (Hp = H + pad, Wp = W + pad, data at (y, x), zeros after each row and image) the
// tap-shared (padded-row) kernel mode reads.
struct FastDiv {
    uint32_t d, m, s;
};

inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{d, 0, 0};
    while ((1ull << f.s) < d) ++f.s;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << f.s) - d)) / d) + 1);
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (__umulhi(n, f.m) + n) >> f.s;
}

// One NCHW -> split-rows conversion (a layer's prepass) as a job over its 128-pixel x
// 32-channel tile grid, tile t = (bx = t / nty, by = t % nty).  Chained mode (cl_conv_forward_chain):
// the converter warps of the previous layer's contraction take tiles from `counter` while that
// contraction runs; a tail launch of the prepass kernel finishes the tiles left.
struct SplitJob {
    const float* x;
    void* xs;
    int n, c, hw, cp, h, w, wp, pad;   // hw = pixels per image of the output grid (Hp*Wp or H*W)
    FastDiv hwd, wpd;
    int ntx, nty;
    int planes;        // operand format (the converting kernel must share it)
    unsigned* counter;
};

// tile staging: hi (or raw for bf16 rows), 3xTF32 lo, mixed-format bf16(hi) / bf16(lo) pairs,
// fp16-split hi / lo pairs
template <int PLANES>
struct SplitSmem {
    float hi[PLANES == kPlanesF16 ? 1 : kSplitPx][33];
    float lo[PLANES == 2 ? kSplitPx : 1][33];
    uint32_t bh[(PLANES == kPlanesMixed || PLANES == kPlanesF16) ? kSplitPx : 1][17];
    uint32_t bl[(PLANES == kPlanesMixed || PLANES == kPlanesF16) ? kSplitPx : 1][17];
};

// Templated on the operand format so every element is converted exactly once (in the load
// phase, into shared tiles) and the write phase is plain 32-bit copies: converting per output
// word made the mixed format's prepass issue-bound (IPC 3.2, DRAM 21 %, ncu on GoogLeNet 1x1).
// Tile (bx, by) = pixels [128 bx, 128 bx + 128) flattened over (image, pixel) x channels
// [32 by, 32 by + 32); tid in [0, 256).  `scale` (fp16 split only) = 2^ex, the input's exponent
// shift (exact, two factors).
// Optional per-tile hook (the fp16 split's speculative prepass): after_load(max |x| of this
// thread's values, ordered bits) runs in every thread right after the load phase, after_sync()
// right after the load / write phase barrier -- so the hook's global atomics overlap the write phase.
struct NoSplitHook {
    __device__ __forceinline__ void after_load(uint32_t) {}
    __device__ __forceinline__ void after_sync() {}
};

template <int PLANES, class Hook = NoSplitHook>
__device__ __forceinline__ void split_tile(const float* __restrict__ x, void* __restrict__ xsv, int N, int C, int HW,
                                           int Cp, int H, int W, int Wp, int pad, const FastDiv& hwd,
                                           const FastDiv& wpd, int bx, int by, int tid, SplitSmem<PLANES>& sm,
                                           Pow2 scale = Pow2{1.0f, 1.0f}, Hook* hook = nullptr) {
    constexpr bool kSplit = PLANES == 2 || PLANES == kPlanesMixed;
    // pixels are flattened over (image, pixel): a tile may straddle two images, so small maps
    // (13 x 13 = 169 pixels) do not leave most of a second 128-pixel tile idle
    const long long NP = (long long)N * HW;
    const long long g0 = (long long)bx * kSplitPx;
    const int c0 = by * 32;
    const int lane = tid & 31, warp = tid >> 5;
    const long long plane = (long long)H * W;
    long long src[4];                       // element offset of channel 0 of this pixel, or -1
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const long long gp = g0 + lane + 32 * h;
        src[h] = -1;
        if (gp < NP) {
            // multiply-shift divisions (host-computed magics); 64-bit divide only past 2^31 pixels
            const int n = NP <= 0x7fffffffLL ? (int)fdiv((uint32_t)gp, hwd) : (int)(gp / HW);
            const int pix = (int)(gp - (long long)n * HW);
            int sp = pix;
            if (pad != 0) {
                const int yy = (int)fdiv((uint32_t)pix, wpd), xx = pix - yy * Wp;
                sp = (yy < H && xx < W) ? yy * W + xx : -1;
            }
            if (sp >= 0) src[h] = (long long)n * C * plane + sp;
        }
    }
    // thread (warp, lane) loads channels {2w, 2w+1, 2w+16, 2w+17} of pixels lane + 32 h: each
    // warp load is 32 consecutive pixels of one channel plane (128 B), and the thread owns
    // adjacent channel pairs, so the mixed format's bf16 halves go to smem as one 32-bit word
    float v[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int c = c0 + 2 * warp + (r & 1) + 16 * (r >> 1);
#pragma unroll
        for (int h = 0; h < 4; ++h) v[r][h] = (c < C && src[h] >= 0) ? __ldg(x + src[h] + (long long)c * plane) : 0.0f;
    }
    if constexpr (!std::is_same<Hook, NoSplitHook>::value) {
        uint32_t amax = 0;                  // this thread's max |x| (as ordered bits)
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int h = 0; h < 4; ++h) amax = max(amax, __float_as_uint(v[r][h]) & 0x7fffffffu);
        hook->after_load(amax);
    }
#pragma unroll
    for (int r = 0; r < 4; r += 2) {
        const int cc = 2 * warp + 16 * (r >> 1);      // even channel within the tile; pair (cc, cc+1)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int px = lane + 32 * h;
            if (PLANES == kPlanesBf16) {
                sm.hi[px][cc] = v[r][h];
                sm.hi[px][cc + 1] = v[r + 1][h];
            } else if (PLANES == kPlanesF16) {
                f16_split2(apply_pow2(v[r][h], scale), apply_pow2(v[r + 1][h], scale), sm.bh[px][cc >> 1],
                           sm.bl[px][cc >> 1]);
            } else {
                const float h0 = tf32_rna(v[r][h]), h1 = tf32_rna(v[r + 1][h]);
                sm.hi[px][cc] = h0;
                sm.hi[px][cc + 1] = h1;
                if (PLANES == 2) {
                    sm.lo[px][cc] = v[r][h] - h0;
                    sm.lo[px][cc + 1] = v[r + 1][h] - h1;
                }
                if (PLANES == kPlanesMixed) {
                    sm.bh[px][cc >> 1] = bf16x2_bits(h0, h1);
                    sm.bl[px][cc >> 1] = bf16x2_bits(v[r][h] - h0, v[r + 1][h] - h1);
                }
            }
        }
    }
    __syncthreads();
    if constexpr (!std::is_same<Hook, NoSplitHook>::value) hook->after_sync();
    const long long row_words = kSplit ? 2LL * Cp : (long long)Cp;
    const int nch = Cp - c0 < 32 ? Cp - c0 : 32;        // channels of this tile inside the padded row
    if (PLANES == kPlanesBf16) {                        // bf16 rows: lane = channel
        __nv_bfloat16* xb = static_cast<__nv_bfloat16*>(xsv);
        for (int pp = warp; pp < kSplitPx; pp += 8) {
            const long long gp = g0 + pp;
            if (gp >= NP) break;
            if (lane < nch) xb[gp * row_words + c0 + lane] = __float2bfloat16_rn(sm.hi[pp][lane]);
        }
        return;
    }
    const int out_words = kSplit ? 2 * nch : nch;
    uint32_t* xs = static_cast<uint32_t*>(xsv);
    // write phase: every lane stores 4 consecutive words of one pixel row (16 B), so a warp
    // instruction covers 2 pixel rows (split formats, 64 words each) or 4 (TF32, 32 words)
    constexpr int kLanesPx = (kSplit ? 64 : 32) / 4;
    constexpr int kPxPerIter = 32 / kLanesPx;
    const int sub = lane / kLanesPx, o = (lane % kLanesPx) * 4;
    for (int pp0 = warp * kPxPerIter; pp0 < kSplitPx; pp0 += 8 * kPxPerIter) {
        const int pp = pp0 + sub;
        const long long gp = g0 + pp;
        if (gp >= NP || o >= out_words) continue;
        uint32_t* dst = xs + gp * row_words + (long long)(kSplit ? 2 : 1) * c0 + o;
        const int u = o >> 5, w = o & 31;
        const uint32_t* srow;
        if (PLANES == 2) {                               // unit u = [hi 16 | lo 16]
            srow = w < 16 ? reinterpret_cast<const uint32_t*>(&sm.hi[pp][u * 16 + w])
                          : reinterpret_cast<const uint32_t*>(&sm.lo[pp][u * 16 + w - 16]);
        } else if (PLANES == kPlanesMixed) {             // unit u = [hi 16 fp32 | bf16 hi 16 | bf16 lo 16]
            srow = w < 16 ? reinterpret_cast<const uint32_t*>(&sm.hi[pp][u * 16 + w])
                          : (w < 24 ? &sm.bh[pp][u * 8 + (w - 16)] : &sm.bl[pp][u * 8 + (w - 24)]);
        } else if (PLANES == kPlanesF16) {               // the tile's unit = [hi fp16 32 | lo fp16 32]
            srow = o < 16 ? &sm.bh[pp][o] : &sm.bl[pp][o - 16];
        } else {
            srow = reinterpret_cast<const uint32_t*>(&sm.hi[pp][o]);
        }
        *reinterpret_cast<uint4*>(dst) = make_uint4(srow[0], srow[1], srow[2], srow[3]);
    }
}

}  // namespace clb
