// tc_conv.cuh -- the one tcgen05 contraction engine behind every GPU method.
//
//   D[rows x cols] = sum_{tap, cblock}  A_tap[rows x 16ch] . B_tap[cols x 16ch]^T
//
// A supplies the 128 D rows of an MMA tile (UMMA M = 128), B the BN columns (UMMA N = BN,
// a runtime multiple of 16 <= 256).  Both operands are K-major fp32 words holding TF32
// values, split hi/lo for the fp32-faithful modes (D += Alo.Bhi + Ahi.Blo + Ahi.Bhi; default:
// Ahi.Bhi in tf32, the two cross terms in bf16 -- see internal.hpp planes 4).
// Each operand is fetched by TMA either as a plain 3-D tile (k, row, tap) or -- the
// implicit kn2row path -- as a 4-D im2col box over the NHWC input whose per-tap offsets
// (j, i) shift the 128 output pixels onto their input taps; taps falling outside the image
// are zero-filled by the TMA unit, which is exactly the reference's "OOB reads discarded"
// shift-add law (conv_kn2.hpp:50-56, conv_kn2.cpp:94-118).  All k^2 taps accumulate into the
// same TMEM accumulator, so no k^2-fold intermediate and no patch matrix ever reach HBM.
//
// Work split (hybrid data-parallel + stream-K): whole tiles round-robin for all but the last
// 1-2 waves, whose (tile, K-chunk) space is cut into gridDim.x contiguous ranges, so every
// SM gets the same MMA work regardless of the tile count.  A tile
// whose chunks straddle CTAs is finished by the CTA holding its FIRST chunk (it processes
// that piece last); the CTAs holding the later pieces publish fp32 partials + a flag first.
// Summation order is fixed by the static split -> bitwise run-to-run determinism.
// Warp roles (384 threads, persistent, one CTA per SM, cooperative launch):
//   warp 0      : TMA producer (one elected lane)
//   warp 1      : MMA issuer   (one lane issues tcgen05.mma + tcgen05.commit)
//   warp 2      : TMEM allocator
//   warps 4..11 : epilogue (TMEM -> fp32 registers -> global); lane quadrant = warp % 4,
//                 column half = (warp - 4) / 4
// Pipelines: smem stages full/empty (TMA <-> MMA); two TMEM chunk accumulators full/empty
// (MMA <-> epilogue).  The epilogue folds each K chunk into registers (fp32, RNE) while
// the MMA fills the other buffer, and stores a tile after its last chunk, so stores
// overlap the next tile's main loop.
#pragma once

#include <climits>
#include <cstdint>
#include <type_traits>
#include <cuda.h>

#include "ptx.cuh"
#include "split_tile.cuh"

namespace clb {

enum : int { LOAD_TILED = 0, LOAD_IM2COL = 1 };
enum : int { EPI_NCHW = 0, EPI_ROWMAJOR = 1, EPI_NCHW_PADDED = 2, EPI_NHWC_PADDED = 3 };

constexpr int kTileM = 128;          // UMMA M (D rows per tile)
// Operand rows are 128-byte units (SWIZZLE_128B, one TMA box per operand per stage):
//   split formats: 16 channels per 128 B unit   (kBlockK = 16 channels per stage)
//     mixed (4): [hi 0..15 fp32 | bf16 hi 0..15 | bf16 lo 0..15];  3xTF32 (2): [hi 0..15 | lo 0..15]
//   TF32  : 32 channels of hi                      (32 channels per stage)
constexpr int kBlockK = 16;          // channel granularity of the split formats
constexpr int kRowWords = 32;
constexpr int kRowBytes = kRowWords * 4;
constexpr int kThreads = 512;             // 4 control warps + 8 epilogue warps + 4 converter warps
constexpr int kEpiThreads = 256;
constexpr int kConvWarps = 4;             // converter warpgroup (warps 12..15): the chained prepass
// registers per thread after setmaxnreg: 4 x 32 x 64 + 8 x 32 x 200 + 4 x 32 x 48 = 65536
constexpr int kRegsControl = 64, kRegsEpi = 200, kRegsConv = 48;
constexpr int kSmemBudget = 200 * 1024;
constexpr int kChunkK = 192;          // fp32-faithful splits: K-elements per TMEM accumulation chunk
constexpr int kChunkKF16 = 384;       // ... the fp16 split, one tap per k-iteration
constexpr int kChunkKF16Padded = 576; // ... the fp16 split, tap-shared padded rows
constexpr int kBarrierBytes = 512;
constexpr int kMaxPeers = 8;     // ranks of a fused output all-gather (one node)
constexpr int kMaxUnits = 160;   // scheduling units per launch (>= SM count; = kMaxGrid)
constexpr int kSpecGroupSlots = 64;   // = kSpecGroups (internal.hpp): maxima of the speculative fp16 prepass
constexpr int kSpecGroupStride = 16;  // ... one per 64 B (spread over L2 slices: every fixup block reads all)
// TMEM loads (16 columns each) in flight per chunk fold (2 keeps the epilogue inside its
// 200-register budget next to its 128 running sums).
constexpr int kFoldLoads = 2;
constexpr int kFastChunkIters = 16;   // TF32 / BF16 fast modes: k-iterations per chunk

struct TcParams {
    // problem
    int rows, cols;            // valid D rows / cols
    int bn;                    // tile N (multiple of 16, <= 256)
    int n_col_tiles, num_tiles;
    int taps, tap_begin, ksize;  // K loop: taps [tap_begin, tap_begin+taps), tap t -> (t/ksize, t%ksize)
    int kblocks;               // 16-channel blocks per tap
    int planes;                // 4 = mixed split (default fp32), 2 = 3xTF32, 1 = TF32 (hi), 3 = BF16
    int row_elems;             // elements per 128-byte row unit (32 fp32 or 64 bf16)
    int stages;
    int chunk_iters;           // k-iterations per TMEM accumulation chunk
    int a_mode, b_mode;        // LOAD_TILED / LOAD_IM2COL
    int a_tap3, b_tap3;        // tiled: pass the tap as 3rd coordinate (weights [tap][M][K])
    // im2col geometry of the row operand (output pixels)
    int P, Q, pad;
    // epilogue
    int epi;                   // EPI_NCHW (rows = pixels n*P*Q, cols = channels) / EPI_ROWMAJOR /
                               // EPI_NCHW_PADDED (rows = padded pixels n*Hp*Wp + y*Wp + x)
    // tap-shared A (padded-row mode): one stage = `tps` taps (a row of the kernel) x one
    // channel block; A is ONE TMA box of 128 + tps - 1 rows of the zero-padded NHWC input and
    // tap j reads it through a descriptor shifted by j rows; tap rows step by a_row_shift (Wp).
    // The padded grid is (H + pad) x (W + pad) per image, zeros AFTER each row and image: the
    // trailing zeros of one row / image are the leading padding of the next (the first image's
    // leading rows are TMA out-of-bounds zero fill), so output (y, x) sits at row y*Wp + x and
    // tap (i, j) reads row y*Wp + x + (i - pad)*Wp + (j - pad).
    int tps;                   // taps per stage (1 = one tap per stage)
    int split_issue;           // A and B TMA loads issued by two warps (0 and 3), 2 arrivals per stage
    int a_issuers;             // 2: A loads of alternate stages from warps 0 and 2 (needs split_issue)
    int fixup_smem;            // stream-K finisher stages partner partials in smem (bulk copy)
    int bps;                   // k-iterations ("sub-stages") per pipeline stage: one barrier
                               // round trip per bps TMA box pairs (chunk_iters % bps == 0)
    int a_row_shift;           // A row offset per tap group (padded row width Wp)
    int a_row_base;            // padded-row mode: A row of output row 0 (-pad*Wp - pad; TMA zero-fills < 0)
    int epi_hp, epi_wp, epi_n; // EPI_NCHW_PADDED geometry
    // tap-stacked mode (stack_k = k > 1): the k taps j of a kernel row are k column blocks of
    // ONE MMA (D column = m * k + j, weights packed [i][m][j]) over an unshifted A operand, and
    // the kn2row shift-add out[r][m] = sum_j D[r + j][m * k + j] runs in the epilogue as warp
    // shuffles.  A is ONE 3-D TMA box {unit, 32 rows, 4 quadrants} over an overlapping view of
    // the padded input (quadrant stride 33 - k rows), so each TMEM lane quadrant holds its own
    // k - 1 halo rows: 33 - k outputs per quadrant, row_step = 4 (33 - k) per CTA.  For small
    // M (N = M would be a slow, small MMA).
    int stack_k;               // 1 = off
    // two-sub-tile mode (msub = 2, padded-row mode, one tap group per stage): each CTA computes
    // TWO 128-row sub-tiles against every B stage -- sub-tile u is the CTA's rows of the u-th
    // half of the tile, its own A box in the stage, its own D columns [u * bn / 2, (u + 1) * bn / 2)
    // (the MMA's N is bn / 2).  The weights a stage carries feed twice the MMA work, so the
    // operand bytes per MMA drop by a fifth at N = 64 (VGG conv1_2); the epilogue's column
    // halves ARE the sub-tiles.
    int msub;                  // 1 = off
    int row_step;              // output rows per CTA tile (128, or 4 (33 - k) when stacked)
    int accumulate;            // out += D (accumulating shifted-GEMM variant)
    const int* sexp;           // fp16 split: the operands' exponent shifts [ew, ex] (device); the
                               // epilogue multiplies D by 2^-(ew + ex).  Null for the other formats.
    unsigned* reset_slots;     // fp16 split, speculative prepass: its group maxima, zeroed by block 0
                               // once the prepass and its fixup are complete (kSpecGroupSlots words,
                               // kSpecGroupStride apart)
    float* out;
    long long ld;              // EPI_ROWMAJOR leading dimension
    int out_channels;          // EPI_NCHW: channel count of the output tensor
    int pq_out;                // EPI_NCHW: P*Q
    // stream-K work split (chunk granularity) and its deterministic fixup
    int chunks_per_tile;       // ceil(k_iters / chunk_iters)
    int dp_tiles;              // tiles [0, dp_tiles) scheduled whole, round-robin over CTAs
    int sk_chunks;             // chunks of tiles [dp_tiles, num_tiles), split contiguously (stream-K)
    int sk_units;              // scheduling units sharing the stream-K chunks (<= grid units; the
                               // rest only run data-parallel tiles): chosen so no tile splits 3 ways
    int sk_start[kMaxUnits + 1];   // chunk_start(b, sk_chunks, sk_units), b = 0..sk_units (host-computed:
                                   // a 64-bit division in the kernel is a subroutine call, and the
                                   // registers saved around it spilled into the MMA issue loop)
    // chained prepass (nx_on): while this contraction runs, its converter warps (12-15) convert
    // tiles of the NEXT layer's input (nx) -- memory-bound work on SMs whose tensor pipe is busy
    // and whose DRAM traffic is 6-30 % of peak -- until this CTA's epilogue is done
    SplitJob nx;
    int nx_on;
    // fused output-channel all-gather (dist.MShardPlan fused mode): the NCHW epilogue stores this
    // plan's output channels [peer_m0, peer_m0 + M_plan) straight into each rank's full
    // [N][peer_M][P][Q] output (P2P stores over NVLink / NVSwitch through CUDA-IPC-mapped
    // pointers; one of them is this rank's own), so the gather overlaps the contraction tile by
    // tile instead of following it as a collective.  n_peers = 0: the plan's own output.
    float* peers[kMaxPeers];
    int n_peers, peer_m0, peer_M;
    int max_sms;               // cap on the SMs the grid may occupy (0 = every co-resident unit):
                               // lets independent launches share the GPU (concurrent small layers)
    float* partials;           // [gridDim.x][128][bn] tile-tail partial sums
    unsigned* flags;           // [gridDim.x], 0 at launch; 1 = partial ready (the finisher resets it)
    int flags_zeroed;          // flags are known to be 0 (self-resetting plan buffer): no memset
    int pdl;                   // launched as a programmatic dependent: wait before touching inputs
    unsigned long long* trace; // diagnostics (CLB_TRACE=1): per-CTA role wait cycles, else null
};

// Contiguous chunk range of CTA b: [chunk_start(b), chunk_start(b+1)).
__host__ __device__ inline int chunk_start(int b, int total, int grid) {
    return (int)(((long long)b * total) / grid);
}

// A rows of one stage (box) and their smem footprint (1024-aligned for the swizzle atom);
// B rows = tps taps x (bn / cta group).
__host__ __device__ inline int tc_a_box_rows(int tps) { return kTileM + tps - 1; }
__host__ __device__ inline int tc_a_bytes(int tps) { return (tc_a_box_rows(tps) * kRowBytes + 1023) & ~1023; }
__host__ __device__ inline int tc_stage_bytes(int b_rows, int tps, int msub = 1) {
    return msub * tc_a_bytes(tps) + tps * b_rows * kRowBytes;
}

__host__ inline int tc_num_stages(int b_rows, int tps, int bps = 1, int budget = kSmemBudget, int msub = 1) {
    int s = (budget - 1024 - kBarrierBytes) / (bps * tc_stage_bytes(b_rows, tps, msub));
    return s > 8 ? 8 : s;
}

__host__ inline int tc_smem_bytes(int b_rows, int tps, int stages, int bps = 1, int msub = 1) {
    return 1024 /*align slack*/ + stages * bps * tc_stage_bytes(b_rows, tps, msub) + kBarrierBytes;
}

// TMEM accumulator buffers: 4 when they fit (BN <= 128), else ping-pong.  Extra buffers let
// the MMA run ahead while the epilogue is busy storing a finished tile (small-BN tiles finish
// every few microseconds, so the store burst used to stall the MMA warp on TMEM).
__host__ __device__ inline int tmem_bufs_for(int bn) { return 4 * bn <= 512 ? 4 : 2; }

__host__ __device__ inline uint32_t tmem_cols_for(int bn) {
    uint32_t need = (uint32_t)tmem_bufs_for(bn) * (uint32_t)bn, c = 32;
    while (c < need) c <<= 1;
    return c;
}

constexpr int kTraceSlots = 24;   // CLB_TRACE per-CTA record (see launch_tc)

#ifdef CLB_DEFINE_TC_KERNEL
// Per-tile operand coordinates, computed once per tile so that the K loop of the single
// producer thread does no integer division (a runtime divide is ~100 cycles of dependent
// ALU latency; 8 per stage throttled the whole pipeline to ~1400 cycles per stage).
struct OperandCoord {
    int mode, tap3, c1, c2, c3;    // tiled: (k, c1=row0, tap|0); im2col: (k, c1=w0, c2=h0, c3=n0)
};

__device__ __forceinline__ OperandCoord operand_coord(int mode, int tap3, int row0, int P, int Q, int pad) {
    OperandCoord c{mode, tap3, row0, 0, 0};
    if (mode == LOAD_IM2COL) {
        const int PQ = P * Q;
        const int n = row0 / PQ;
        const int rem = row0 - n * PQ;
        const int p = rem / Q;
        c.c1 = rem - p * Q - pad;   // w of the first traversed pixel (bounding-box coordinates)
        c.c2 = p - pad;             // h
        c.c3 = n;
    }
    return c;
}

__device__ __forceinline__ void load_operand(const CUtensorMap* map, const OperandCoord& c, uint64_t* bar,
                                             uint8_t* dst, int kcoord, int tap, int ti, int tj) {
    if (c.mode == LOAD_IM2COL)
        tma_load_im2col_4d(map, bar, dst, kcoord, c.c1, c.c2, c.c3, (uint16_t)tj, (uint16_t)ti);
    else
        tma_load_3d(map, bar, dst, kcoord, c.c1, c.tap3 ? tap : 0);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void epi_bar_sync() {   // the 8 epilogue warps only
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
}

// A piece = the part of one tile's chunk range [c_lo, c_hi) that falls in this CTA's range.
struct Piece {
    int tile, c_lo, c_hi;
};

// Hybrid data-parallel + stream-K schedule of one CTA: first its share of the whole tiles
// [0, dp_tiles) round-robin (tile = b, b + grid, ...: neighbouring CTAs work on neighbouring
// tiles, which keeps the live input window compact in L2), then its contiguous range of the
// stream-K chunk space covering the remaining 1-2 waves of tiles.
struct Sched {
    int b, grid, cpt, dp_tiles, i, n_dp, g, g_end;
    __device__ Sched(const TcParams& p, int b_, int grid_)
        : b(b_), grid(grid_), cpt(p.chunks_per_tile), dp_tiles(p.dp_tiles), i(0) {
        n_dp = dp_tiles > b ? (dp_tiles - b + grid - 1) / grid : 0;
        g = b < p.sk_units ? p.sk_start[b] : 0;
        g_end = b < p.sk_units ? p.sk_start[b + 1] : 0;
    }
    __device__ bool next(Piece& pc) {
        if (i < n_dp) {
            pc.tile = b + i * grid;
            pc.c_lo = 0;
            pc.c_hi = cpt;
            ++i;
            return true;
        }
        if (g >= g_end) return false;
        const int t = g / cpt;
        pc.tile = dp_tiles + t;
        pc.c_lo = g - t * cpt;
        const int left = g_end - g;
        pc.c_hi = (cpt - pc.c_lo) < left ? cpt : pc.c_lo + left;
        g += pc.c_hi - pc.c_lo;
        return true;
    }
};

// One 128-pixel x 32-channel tile of a SplitJob by one warp, in registers (no shared memory:
// the contraction owns it): lane = pixel row (4 passes), 16 channels per unit loaded coalesced
// across the warp (consecutive pixels of one plane), the 128-byte split unit of each row written
// by its lane.  Same bytes as split_tile (tf32_rna_bits == cvt.rna.tf32 for finite values).
template <int PL>
__device__ __forceinline__ void split_tile_warp(const SplitJob& j, int bx, int by, int lane) {
    const long long NP = (long long)j.n * j.hw;
    const long long plane = (long long)j.h * j.w;
    uint32_t* xs = static_cast<uint32_t*>(j.xs);
    const long long row_words = 2LL * j.cp;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const long long gp = (long long)bx * kSplitPx + 32 * pass + lane;
        if (gp >= NP) break;
        const int n = NP <= 0x7fffffffLL ? (int)fdiv((uint32_t)gp, j.hwd) : (int)(gp / j.hw);
        const int pix = (int)(gp - (long long)n * j.hw);
        int sp = pix;
        if (j.pad != 0) {
            const int yy = (int)fdiv((uint32_t)pix, j.wpd), xx = pix - yy * j.wp;
            sp = (yy < j.h && xx < j.w) ? yy * j.w + xx : -1;
        }
        const float* src = j.x + (long long)n * j.c * plane + (sp < 0 ? 0 : sp);
#pragma unroll 1
        for (int cb = 0; cb < 2; ++cb) {
            const int c0 = by * 32 + 16 * cb;
            if (c0 >= j.cp) break;
            float v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c)
                v[c] = (sp >= 0 && c0 + c < j.c) ? __ldg(src + (long long)(c0 + c) * plane) : 0.0f;
            uint4* dst = reinterpret_cast<uint4*>(xs + gp * row_words + 2LL * c0);
            uint32_t hb[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) hb[c] = tf32_rna_bits(v[c]);
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = make_uint4(hb[4 * q], hb[4 * q + 1], hb[4 * q + 2], hb[4 * q + 3]);
            if constexpr (PL == 4) {
                uint32_t w8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    w8[k] = bf16x2_bits(__uint_as_float(hb[2 * k]), __uint_as_float(hb[2 * k + 1]));
                dst[4] = make_uint4(w8[0], w8[1], w8[2], w8[3]);
                dst[5] = make_uint4(w8[4], w8[5], w8[6], w8[7]);
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    w8[k] = bf16x2_bits(v[2 * k] - __uint_as_float(hb[2 * k]), v[2 * k + 1] - __uint_as_float(hb[2 * k + 1]));
                dst[6] = make_uint4(w8[0], w8[1], w8[2], w8[3]);
                dst[7] = make_uint4(w8[4], w8[5], w8[6], w8[7]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    dst[4 + q] = make_uint4(__float_as_uint(v[4 * q] - __uint_as_float(hb[4 * q])),
                                            __float_as_uint(v[4 * q + 1] - __uint_as_float(hb[4 * q + 1])),
                                            __float_as_uint(v[4 * q + 2] - __uint_as_float(hb[4 * q + 2])),
                                            __float_as_uint(v[4 * q + 3] - __uint_as_float(hb[4 * q + 3])));
            }
        }
    }
}

// One D row's columns into NCHW planes: column j lands at o + j * plane.  The accumulate
// branch is hoisted and the address walks by one plane per column, so each element costs a
// predicated store and a pointer add (a warp's 32 rows make each store one 128 B line).
// W = columns this thread can hold for the tile (a narrow tile takes the short loop instead of
// issuing the predicated-off stores and pointer steps of 128 columns)
template <int W>
__device__ __forceinline__ void store_nchw_w(float* o, long long plane, int nvalid, int accumulate, const float* sum) {
    if (accumulate) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if (j < nvalid) *o += sum[j];
            o += plane;
        }
    } else {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if (j < nvalid) *o = sum[j];
            o += plane;
        }
    }
}
__device__ __forceinline__ void store_nchw(float* o, long long plane, int nvalid, int accumulate, const float* sum) {
    if (nvalid <= 32) store_nchw_w<32>(o, plane, nvalid, accumulate, sum);        // warp-uniform
    else if (nvalid <= 64) store_nchw_w<64>(o, plane, nvalid, accumulate, sum);
    else if (nvalid <= 96) store_nchw_w<96>(o, plane, nvalid, accumulate, sum);
    else store_nchw_w<128>(o, plane, nvalid, accumulate, sum);
}

// One D row's columns into a row-major (channels-last) output row: float4 where aligned.
__device__ __forceinline__ void store_rowmajor(float* dst, long long ld, int col0, int hcols, int cols, int accumulate,
                                               const float* sum) {
    const bool vec = (ld % 4 == 0) && !accumulate && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
#pragma unroll
    for (int j = 0; j < 128; j += 4) {
        if (j < hcols) {
            if (vec && col0 + j + 3 < cols) {
                *reinterpret_cast<float4*>(dst + j) = make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (col0 + j + e < cols) {
                        if (accumulate) dst[j + e] += sum[j + e];
                        else dst[j + e] = sum[j + e];
                    }
            }
        }
    }
}

// Tap-stacked shift-add (conv_kn2.cpp:94-118 restated on the accumulator): this thread holds
// D row r = lane of its quadrant, columns c = m * KS + j of its half; afterwards sum[m] =
// sum_j D[r + j][m * KS + j], row r + j being lane + j of the same warp.  Lanes >= 33 - KS
// have no complete tap set (their rows are the next quadrant's halo) and are not stored.
template <int KS>
__device__ __forceinline__ void shift_add_taps(float* sum, int hcols) {
#pragma unroll
    for (int m = 0; m < 128 / KS; ++m) {
        if (m * KS < hcols) {
            float v = sum[m * KS];
#pragma unroll
            for (int j = 1; j < KS; ++j) v += __shfl_down_sync(0xffffffffu, sum[m * KS + j], j);
            sum[m] = v;
        }
    }
}

// CG = 1: one CTA per 128-row tile (tcgen05 cta_group::1).
// CG = 2: a CTA pair (cluster of 2) per 256-row tile (cta_group::2): each CTA TMA-loads its
//         128 A rows and HALF of the BN B rows into its own smem, all completion bytes land
//         on the leader's barrier, the leader issues M=256 MMAs reading both CTAs' smem and
//         multicasts its commits; each CTA's TMEM holds its 128 D rows.  Per-SM operand
//         bytes per MMA drop by BN/2 rows (-33% at BN = 256).
template <int CG, bool TRACE>
__global__ void __launch_bounds__(kThreads, 1)
tc_conv_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const long long t_entry = TRACE ? clock64() : 0;
    if (TRACE && threadIdx.x == 0) p.trace[blockIdx.x * kTraceSlots + 9] = globaltimer_ns();

    const int bn = p.bn;
    const int planes = p.planes;
    const int stages = p.stages;
    const int msub = p.msub;                      // 128-row sub-tiles per CTA sharing each B stage
    const int mma_n = bn / msub;                  // N of one MMA (bn = D columns of the tile)
    const int tile_m = kTileM * CG;               // D rows per MMA (the pair's rows for CG = 2)
    const int sub_rows = p.row_step * CG;         // output rows per sub-tile (< tile_m when tap-stacked)
    const int tile_rows = sub_rows * msub;        // output rows per tile
    const int b_rows = mma_n / CG;                // B rows this CTA loads
    const int tps = p.tps;
    const int a_bytes = tc_a_bytes(tps);          // one A box of a stage (128 + tps - 1 rows)
    const int b_bytes = tps * b_rows * kRowBytes; // B rows of one k-iteration (tps taps)
    const int stage_bytes = msub * a_bytes + b_bytes;   // one sub-stage (one k-iteration)
    const int bps = p.bps;
    const int group_bytes = bps * stage_bytes;    // one pipeline stage
    const uint32_t stage_tx = (uint32_t)(msub * tc_a_box_rows(tps) * kRowBytes + b_bytes);
    const int k_iters = (p.taps / tps) * p.kblocks;   // k-iterations per tile
    const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;       // scheduling unit
    const int nunits = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + stages * group_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + stages;
    uint64_t* tfull = bars + 2 * stages;        // [nbuf]
    uint64_t* tempty = bars + 2 * stages + 4;   // [nbuf]
    uint64_t* fix_bar = bars + 2 * stages + 8;     // stream-K partial staged in smem (finisher)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 9);
    volatile int* epi_done = reinterpret_cast<volatile int*>(tmem_slot + 1);   // chained prepass: stop

    const int warp = threadIdx.x >> 5;
    const uint32_t ncols = tmem_cols_for(bn);
    const int nbuf = tmem_bufs_for(bn);
    const uint32_t nb_shift = nbuf == 4 ? 2u : 1u;
    const uint32_t buf_cols = ncols / (uint32_t)nbuf;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], p.split_issue ? 2 : 1);   // the A and B TMA warps' expect_tx arrivals
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < nbuf; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], CG * (kEpiThreads / 32));
        }
        mbar_init(fix_bar, 1);
        *epi_done = 0;
        fence_barrier_init();
    }
    if (warp == 0 && lane_id() == 0) {
        tma_prefetch_desc(&map_a);
        tma_prefetch_desc(&map_b);
    }
    if (warp == 2) {
        if constexpr (CG == 2) {
            tmem_alloc_2sm(tmem_slot, ncols);
            tmem_relinquish_2sm();
        } else {
            tmem_alloc(tmem_slot, ncols);
            tmem_relinquish();
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();   // peer barriers initialised before any remote use
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int cpt = p.chunks_per_tile;
    const int ci = p.chunk_iters;

    // Programmatic dependent launch: everything above (barrier init, TMEM alloc, descriptor
    // prefetch) overlapped the previous kernel's tail; inputs (the split operand, output
    // buffers) are only touched after this point.
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.reset_slots && blockIdx.x == 0 && threadIdx.x < kSpecGroupSlots) p.reset_slots[threadIdx.x * kSpecGroupStride] = 0u;

    // Register split per warpgroup (setmaxnreg is warpgroup-aligned, and each role branch below
    // sits under its own setmaxnreg so ptxas allocates it with that budget).
    if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsControl));
    if (warp == 0 || (warp == 3 && p.split_issue) || (warp == 2 && p.a_issuers == 2)) {
        // ------------------------------------------------------------ TMA producer ----
        // whole warp runs the (uniform) loop; one elected lane issues the TMA.  With split_issue
        // warp 0 loads A and warp 3 loads B (TMA im2col boxes are slow to deliver from a single
        // issuing thread: tools/tma_probe3.cu 37 -> 43 B/clk per SM with two issuers).
        {
            const bool do_a = warp == 0 || warp == 2, do_b = warp == 3 || !p.split_issue;
            // two A issuers: warp 0 takes the even stages of the sequence, warp 2 the odd ones
            // (each stage still gets exactly one A arrival); the B warp takes every stage
            const uint32_t a_par = warp == 2 ? 1u : 0u;
            const bool a_alt = do_a && p.a_issuers == 2;
            uint32_t gs = 0;   // stage sequence number
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t a_tx = (uint32_t)(msub * tc_a_box_rows(tps) * kRowBytes);
            const uint32_t tx = (uint32_t)CG * ((do_a ? a_tx : 0u) + (do_b ? stage_tx - a_tx : 0u));   // both CTAs' bytes land on the leader
            long long w_empty = 0;
            const long long t_start = clock64();
            if (TRACE && lane_id() == 0 && warp == 0) p.trace[blockIdx.x * kTraceSlots + 8] = (unsigned long long)(t_start - t_entry);
            Sched sch(p, unit, nunits);
            Piece pc;
            while (sch.next(pc)) {
                const int mt = pc.tile / p.n_col_tiles;
                const int nt = pc.tile - mt * p.n_col_tiles;
                const OperandCoord ca =
                    operand_coord(p.a_mode, p.a_tap3, mt * tile_rows + (int)rank * p.row_step, p.P, p.Q, p.pad);
                const OperandCoord cb = operand_coord(p.b_mode, p.b_tap3, nt * bn + (int)rank * b_rows, p.P, p.Q, p.pad);
                const int it0 = pc.c_lo * ci;
                const int it1 = pc.c_hi * ci < k_iters ? pc.c_hi * ci : k_iters;
                // (tap group, channel block) of it0; then walk with counters, no division in the loop
                int grp = p.tap_begin / tps + it0 / p.kblocks;
                int kb = it0 - (it0 / p.kblocks) * p.kblocks;
                int tap = grp * tps;
                int ti = tap / p.ksize, tj = tap - (tap / p.ksize) * p.ksize;
                int sub = 0;
                for (int it = it0; it < it1; ++it) {
                    const int kc = kb * p.row_elems;
                    // padded-row mode: tap (i, j) -> +i Wp + j (j = 0 at a group start when tps = k)
                    const int arow = p.a_row_shift ? ca.c1 + p.a_row_base + ti * p.a_row_shift + tj : ca.c1;
                    const bool mine = !a_alt || (gs & 1u) == a_par;
                    if (sub == 0 && mine) {
                        const long long t0 = TRACE ? clock64() : 0;
                        mbar_wait(&empty[stage], phase ^ 1u);
                        if (TRACE) w_empty += clock64() - t0;
                    }
                    // a stage holds min(bps, iterations left in the piece) sub-stages
                    const uint32_t txs = tx * (uint32_t)(it1 - it < bps ? it1 - it : bps);
                    uint8_t* a_st = smem + stage * group_bytes + sub * stage_bytes;
                    if (mine && elect_one()) {
                    if constexpr (CG == 2) {
                        const uint32_t lbar = mapa_shared(smem_u32(&full[stage]), 0);
                        if (leader && sub == 0) mbar_arrive_expect_tx(&full[stage], txs);
                        if (do_a) {
                            if (ca.mode == LOAD_IM2COL)
                                tma_load_im2col_4d_2sm(&map_a, lbar, a_st, kc, ca.c1, ca.c2, ca.c3, (uint16_t)tj,
                                                       (uint16_t)ti);
                            else
                                for (int u = 0; u < msub; ++u)
                                    tma_load_3d_2sm(&map_a, lbar, a_st + u * a_bytes, kc, arow + u * sub_rows,
                                                    ca.tap3 ? tap : 0);
                        }
                        if (do_b) {
                            if (cb.mode == LOAD_IM2COL)
                                tma_load_im2col_4d_2sm(&map_b, lbar, a_st + msub * a_bytes, kc, cb.c1, cb.c2, cb.c3, (uint16_t)tj,
                                                       (uint16_t)ti);
                            else
                                tma_load_3d_2sm(&map_b, lbar, a_st + msub * a_bytes, kc, cb.c1, cb.tap3 ? tap : 0);
                        }
                    } else {
                        if (sub == 0) mbar_arrive_expect_tx(&full[stage], txs);
                        if (do_a) {
                            if (ca.mode == LOAD_IM2COL)
                                load_operand(&map_a, ca, &full[stage], a_st, kc, tap, ti, tj);
                            else
                                for (int u = 0; u < msub; ++u)
                                    tma_load_3d(&map_a, &full[stage], a_st + u * a_bytes, kc, arow + u * sub_rows,
                                                ca.tap3 ? tap : 0);
                        }
                        if (do_b) load_operand(&map_b, cb, &full[stage], a_st + msub * a_bytes, kc, tap, ti, tj);
                    }
                    }
                    __syncwarp();
                    if (++sub == bps || it + 1 == it1) {
                        sub = 0;
                        ++gs;
                        if (++stage == stages) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    if (++kb == p.kblocks) {
                        kb = 0;
                        ++grp;
                        tap += tps;
                        tj += tps;
                        while (tj >= p.ksize) {
                            tj -= p.ksize;
                            ++ti;
                        }
                    }
                }
            }
            if (TRACE && lane_id() == 0 && warp == 0) {
                p.trace[blockIdx.x * kTraceSlots + 0] = (unsigned long long)(clock64() - t_start);
                p.trace[blockIdx.x * kTraceSlots + 1] = (unsigned long long)w_empty;
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer ----
        // The K loop of a tile is cut into chunks of ci k-iterations; each chunk accumulates
        // into the next of 2-4 TMEM buffers (round robin) that the epilogue folds into fp32 registers.
        // Tensor-core accumulation rounds every update of the running fp32 accumulator
        // (error grows ~linearly in the chunk length), so bounding the chunk to kChunkK = 192
        // K-elements keeps the split-product result fp32-faithful for any K (saturates at
        // rel-L2 ~1.1e-6 against the 1e-5 bound).
        // The whole warp runs the loop (loop state is warp-uniform, so it lives in uniform
        // registers); one elected lane issues the MMAs and the commits that track them.
        if (leader) {
            // one live instruction descriptor (fp16 A/B); each MMA flavour ORs in its format code
            const uint32_t idesc0 = idesc_f16((uint32_t)tile_m, (uint32_t)mma_n);
            constexpr uint32_t kFmtTf32 = (2u << 7) | (2u << 10), kFmtBf16 = (1u << 7) | (1u << 10);
            auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {     // kind::tf32
                if constexpr (CG == 2) mma_tf32_ss_2sm(d, a, b, idesc0 | kFmtTf32, acc);
                else mma_tf32_ss(d, a, b, idesc0 | kFmtTf32, acc);
            };
            auto mma16 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {   // kind::f16, bf16 operands
                if constexpr (CG == 2) mma_bf16_ss_2sm(d, a, b, idesc0 | kFmtBf16, acc);
                else mma_bf16_ss(d, a, b, idesc0 | kFmtBf16, acc);
            };
            auto mmah = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {    // kind::f16, fp16 operands
                if constexpr (CG == 2) mma_bf16_ss_2sm(d, a, b, idesc0, acc);
                else mma_bf16_ss(d, a, b, idesc0, acc);
            };
            auto commit = [&](uint64_t* bar) {
                if constexpr (CG == 2) mma_commit_2sm_mc(bar, (uint16_t)0x3);
                else mma_commit(bar);
            };
            // Descriptors are built once: the start-address field is the low 14 bits (addr >> 4),
            // so stage / k-step / hi-lo offsets are plain adds on the 64-bit descriptor.  (Building
            // 4 descriptors per MMA made the single issuing thread slower than an N=192 MMA.)
            const uint64_t desc0 = umma_desc_kmajor(smem_u32(smem), kRowBytes);
            const uint64_t st_step = (uint64_t)(group_bytes >> 4);
            const uint64_t sub_step = (uint64_t)(stage_bytes >> 4);
            const uint64_t b_off = (uint64_t)((msub * a_bytes) >> 4);
            const uint64_t a_sub = (uint64_t)(a_bytes >> 4);                // next sub-tile's A box
            const uint32_t d_sub = (uint32_t)mma_n;                         // next sub-tile's D columns
            const uint64_t tap_b = (uint64_t)(b_rows * 8);
            long long w_full = 0, w_tempty = 0;
            const long long t_start = clock64();
            // The issue loop is specialised on the split format and on one tap per k-iteration
            // (compile-time), and one elected block issues a whole stage: at N = 192 the MMAs of a
            // k-iteration take ~384 tensor cycles, and a generic loop (format dispatch, tap loop,
            // one elect + reconvergence per k-iteration: ~100 instructions) could not keep up.
            auto run = [&](auto pl_c, auto t1_c, auto ms_c) {
                constexpr int PL = decltype(pl_c)::value;
                constexpr bool T1 = decltype(t1_c)::value;
                constexpr int MS = decltype(ms_c)::value;   // == msub
                // one k-iteration: the taps of the group x the format's MMAs; acc0 = 0 only for the
                // chunk's first k-iteration (its first MMA starts the accumulator)
                auto issue = [&](uint32_t d_tmem0, uint64_t da00, uint64_t db0, uint32_t acc0) {
                    const int ntaps = T1 ? 1 : tps;
#pragma unroll
                    for (int u = 0; u < MS; ++u)
                    for (int t = 0; t < ntaps; ++t) {
                        const uint32_t d_tmem = d_tmem0 + (uint32_t)u * d_sub;
                        const uint64_t da0 = da00 + (uint64_t)u * a_sub;
                        // tap t of the group: A shifted by t rows (8 desc units of 16 B per
                        // 128 B row), B = the t-th tap's weight tile
                        const uint64_t da = da0 + (uint64_t)(t * 8);
                        const uint64_t db = db0 + (uint64_t)t * tap_b;
                        const uint32_t first = (acc0 | (uint32_t)t) ? 1u : 0u;
                        if constexpr (PL == 2) {
                            // row = [hi 16 | lo 16]: k-step s (8 tf32 = 32 B = 2 desc units) of
                            // hi at +2 s, of lo at +4 + 2 s; small cross terms first
                            mma(d_tmem, da + 4, db, first);
                            mma(d_tmem, da, db + 4, 1u);
                            mma(d_tmem, da, db, 1u);
                            mma(d_tmem, da + 6, db + 2, 1u);
                            mma(d_tmem, da + 2, db + 6, 1u);
                            mma(d_tmem, da + 2, db + 2, 1u);
                        } else if constexpr (PL == 4) {
                            // row = [hi 16 fp32 | bf16(hi) 16 | bf16(lo) 16]: the cross terms
                            // lo*Hi and hi*Lo as one bf16 K=16 MMA each (bytes 96 / 64 of A
                            // with 64 / 96 of B), then hi*Hi as two exact tf32 K=8 MMAs
                            mma16(d_tmem, da + 6, db + 4, first);
                            mma16(d_tmem, da + 4, db + 6, 1u);
                            mma(d_tmem, da, db, 1u);
                            mma(d_tmem, da + 2, db + 2, 1u);
                        } else if constexpr (PL == 5) {
                            // row = [hi 32 fp16 | lo 32 fp16] of the scaled input: k-step s (16
                            // fp16 = 32 B = 2 desc units) of hi at +2 s, of lo at +4 + 2 s; the
                            // cross terms first, then hi*Hi (all products exact in fp32)
                            mmah(d_tmem, da + 4, db, first);
                            mmah(d_tmem, da, db + 4, 1u);
                            mmah(d_tmem, da, db, 1u);
                            mmah(d_tmem, da + 6, db + 2, 1u);
                            mmah(d_tmem, da + 2, db + 6, 1u);
                            mmah(d_tmem, da + 2, db + 2, 1u);
                        } else if constexpr (PL == 3) {
                            // 64 bf16 per row: 4 k-steps of 16 elements (32 B = 2 desc units)
                            mma16(d_tmem, da, db, first);
                            mma16(d_tmem, da + 2, db + 2, 1u);
                            mma16(d_tmem, da + 4, db + 4, 1u);
                            mma16(d_tmem, da + 6, db + 6, 1u);
                        } else {
                            mma(d_tmem, da, db, first);
                            mma(d_tmem, da + 2, db + 2, 1u);
                            mma(d_tmem, da + 4, db + 4, 1u);
                            mma(d_tmem, da + 6, db + 6, 1u);
                        }
                    }
                };
                int stage = 0;
                uint32_t phase = 0;
                uint64_t dstage = desc0;   // descriptor of the current stage's first sub-stage
                uint32_t lg = 0;
                Sched sch(p, unit, nunits);
                Piece pc;
                while (sch.next(pc))
                for (int c = pc.c_lo; c < pc.c_hi; ++c, ++lg) {
                    const int c0 = c * ci;
                    const int c1 = c0 + ci < k_iters ? c0 + ci : k_iters;
                    const uint32_t buf = lg & (uint32_t)(nbuf - 1);
                    const uint32_t tph = (lg >> nb_shift) & 1u;
                    if (TRACE) {
                        const long long t0 = clock64();
                        mbar_wait(&tempty[buf], tph ^ 1u);
                        w_tempty += clock64() - t0;
                    } else {
                        mbar_wait(&tempty[buf], tph ^ 1u);
                    }
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + buf * buf_cols;
                    // stages of bps k-iterations (chunk starts are stage starts: ci % bps == 0)
                    for (int it = c0; it < c1; it += bps) {
                        const int nsub = c1 - it < bps ? c1 - it : bps;
                        const long long t0 = TRACE ? clock64() : 0;
                        mbar_wait(&full[stage], phase);
                        if (TRACE) w_full += clock64() - t0;
                        tc_fence_after();
                        if (elect_one()) {
                            auto dbs = [&](int sb) { return dstage + (uint64_t)sb * sub_step + b_off; };   // B of sub-stage sb
                            issue(d_tmem, dstage, dbs(0), it > c0 ? 1u : 0u);
                            if (nsub > 1) issue(d_tmem, dstage + sub_step, dbs(1), 1u);
#pragma unroll 1
                            for (int sb = 2; sb < nsub; ++sb) issue(d_tmem, dstage + (uint64_t)sb * sub_step, dbs(sb), 1u);
                            commit(&empty[stage]);   // frees the smem stage once its MMAs retire
                        }
                        __syncwarp();
                        if (++stage == stages) {
                            stage = 0;
                            phase ^= 1u;
                            dstage = desc0;
                        } else {
                            dstage += st_step;
                        }
                    }
                    if (elect_one()) commit(&tfull[buf]);   // chunk complete -> epilogue(s)
                    __syncwarp();
                }
            };
            using I1 = std::integral_constant<int, 1>;
            using I2 = std::integral_constant<int, 2>;
            using I3 = std::integral_constant<int, 3>;
            using I4 = std::integral_constant<int, 4>;
            using I5 = std::integral_constant<int, 5>;
            using BT = std::true_type;
            using BF = std::false_type;
            // (two-sub-tile mode: mixed split, tap-shared stages only -- launch_tc enforces it)
            if (planes == 4) {
                if (tps == 1) run(I4{}, BT{}, I1{});
                else if (msub == 2) run(I4{}, BF{}, I2{});
                else run(I4{}, BF{}, I1{});
            } else if (planes == kPlanesF16) {
                if (tps == 1) run(I5{}, BT{}, I1{});
                else if (msub == 2) run(I5{}, BF{}, I2{});
                else run(I5{}, BF{}, I1{});
            } else if (planes == 2) {
                if (tps == 1) run(I2{}, BT{}, I1{}); else run(I2{}, BF{}, I1{});
            } else if (planes == 3) {
                if (tps == 1) run(I3{}, BT{}, I1{}); else run(I3{}, BF{}, I1{});
            } else {
                if (tps == 1) run(I1{}, BT{}, I1{}); else run(I1{}, BF{}, I1{});
            }
            if (TRACE && lane_id() == 0) {
                p.trace[blockIdx.x * kTraceSlots + 2] = (unsigned long long)(clock64() - t_start);
                p.trace[blockIdx.x * kTraceSlots + 3] = (unsigned long long)w_full;
                p.trace[blockIdx.x * kTraceSlots + 4] = (unsigned long long)w_tempty;
                p.trace[blockIdx.x * kTraceSlots + 12] = globaltimer_ns();
            }
        }
    }
    } else if (warp >= 12) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsConv));
        // -------------------------------------- converter warpgroup (warps 12-15) ----
        if (p.nx_on) {
            // chained prepass: tiles of the next layer's input, taken from the job's counter until
            // the job is done or this CTA's epilogue has finished (a tail launch does the rest)
            const int lane = (int)lane_id();
            const int total = p.nx.ntx * p.nx.nty;
            int tiles = 0;
            while (!*epi_done) {
                int t = 0;
                if (lane == 0) t = (int)atomicAdd(p.nx.counter, 1u);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t >= total) break;
                if (planes == 4) split_tile_warp<4>(p.nx, t / p.nx.nty, t % p.nx.nty, lane);
                else split_tile_warp<2>(p.nx, t / p.nx.nty, t % p.nx.nty, lane);
                ++tiles;
            }
            if (TRACE && lane == 0) atomicAdd(&p.trace[blockIdx.x * kTraceSlots + 23], (unsigned long long)tiles);
        }
    } else {
        // --------------------------------------------------------------- epilogue ----
        // 8 warps: lane quadrant = warp % 4 (TMEM access rule), column half = (warp-4)/4.
        // Each thread owns one D row and up to 128 columns of running fp32 sums.
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsEpi));
        const int quad = warp & 3;
        const int half = (warp - 4) >> 2;
        const int lane = (int)lane_id();
        const int hcols = bn >> 1;                   // multiple of 8 (bn % 16 == 0)
        const int cbase = half * hcols;
        const int trow = quad * 32 + lane;           // row within this CTA's 128 rows
        // fp16 split: D carries the operands' power-of-2 scales; 2^-(ew + ex) as two exact factors
        // (each a normal float; below 2^-252 every product underflows fp32 anyway), applied once
        // per finished tile (published partials stay scaled)
        Pow2 ds{1.0f, 1.0f};
        if (p.sexp) {
            const int d = -(p.sexp[0] + p.sexp[1]);
            ds = pow2_factors(d < -252 ? -252 : d);
        }
        uint32_t lg = 0;
        long long w_tfull = 0, w_store = 0, w_fix = 0;
        unsigned long long n_parts = 0, t_folded = 0, t_pub = 0, t_acq = 0, t_added = 0, t_stored = 0;
        const long long t_start = clock64();
        Sched sch(p, unit, nunits);
        Piece pc;
        while (sch.next(pc)) {
            const int mt = pc.tile / p.n_col_tiles;
            const int nt = pc.tile - mt * p.n_col_tiles;
            // two-sub-tile mode: column half = sub-tile (rows of the tile's half-th sub_rows)
            const int row = mt * tile_rows + (msub > 1 ? half * sub_rows : 0) + (int)rank * p.row_step +
                            (p.stack_k > 1 ? quad * (33 - p.stack_k) + lane : trow);
            int col0 = msub > 1 ? nt * mma_n : nt * bn + cbase;
            float sum[128];
#pragma unroll
            for (int j = 0; j < 128; ++j) sum[j] = 0.0f;
            // finisher of a split tile (its first chunks, always this CTA's last piece): the
            // later pieces' partials are acquired while its own last chunk is still in the MMA
            const bool finisher = pc.c_lo == 0 && pc.c_hi < cpt;
            int u_end = unit + 1;
            if (finisher) {
                const int last = (pc.tile - p.dp_tiles) * cpt + cpt - 1;   // in stream-K chunk space
                while (u_end < p.sk_units && p.sk_start[u_end] <= last) ++u_end;
            }
            for (int c = pc.c_lo; c < pc.c_hi; ++c, ++lg) {
                const uint32_t buf = lg & (uint32_t)(nbuf - 1);
                const uint32_t tph = (lg >> nb_shift) & 1u;
                if (finisher && c == pc.c_hi - 1) {
                    const uint64_t t0 = globaltimer_ns();
                    const long long c0 = TRACE ? clock64() : 0;
                    for (int u2 = unit + 1; u2 < u_end; ++u2) {
                        while (ld_acquire_u32(&p.flags[u2 * CG + (int)rank]) == 0u) {
                            if (globaltimer_ns() - t0 > 4000000000ull) __trap();
                        }
                    }
                    if (TRACE) {
                        w_fix += clock64() - c0;
                        n_parts += (unsigned long long)(u_end - unit - 1);
                        t_acq = globaltimer_ns();
                    }
                }
                if (TRACE) {
                    const long long t0 = clock64();
                    mbar_wait(&tfull[buf], tph);
                    w_tfull += clock64() - t0;
                } else {
                    mbar_wait(&tfull[buf], tph);
                }
                tc_fence_after();
                const uint32_t t_addr =
                    tmem_base + ((uint32_t)(quad * 32) << 16) + buf * buf_cols + (uint32_t)cbase;
#pragma unroll
                for (int grp = 0; grp < 8; grp += kFoldLoads) {   // kFoldLoads x 16 columns in flight
                    uint32_t r[kFoldLoads][16];
#pragma unroll
                    for (int q = 0; q < kFoldLoads; ++q)
                        if ((grp + q) * 16 < hcols) tmem_ld_32x32b_x16(t_addr + (uint32_t)((grp + q) * 16), r[q]);
                    tmem_ld_wait();
#pragma unroll
                    for (int q = 0; q < kFoldLoads; ++q)
                        if ((grp + q) * 16 < hcols)
#pragma unroll
                            for (int j = 0; j < 16; ++j) sum[(grp + q) * 16 + j] += __uint_as_float(r[q][j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {   // one arrive per epilogue warp (count = CG x 8)
                    if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[buf]), 0));
                    else mbar_arrive(&tempty[buf]);
                }
            }
            if (TRACE) t_folded = globaltimer_ns();
            if (pc.c_lo > 0) {
                // ---- tile tail handled by this CTA: publish the partial for the finisher ----
                // lane-contiguous float4 layout [slot][col/4][row]: a warp's store is 512
                // contiguous bytes (the row-per-thread layout scattered every lane 4 BN bytes
                // apart and made publish + fixup ~10x slower than the loads themselves)
                float4* dst = reinterpret_cast<float4*>(p.partials) +
                              ((long long)blockIdx.x * (bn >> 2) + (cbase >> 2)) * kTileM + trow;
#pragma unroll
                for (int j = 0; j < 128; j += 4)
                    if (j < hcols) __stcg(dst + (j >> 2) * kTileM, make_float4(sum[j], sum[j + 1], sum[j + 2], sum[j + 3]));
                // the barrier orders every epilogue thread's stores before the single gpu-scope
                // release (release is cumulative over what the releasing thread has observed)
                epi_bar_sync();
                if (threadIdx.x == 4 * 32) st_release_u32(&p.flags[blockIdx.x], 1u);
                if (TRACE) t_pub = globaltimer_ns();
                continue;
            }
            if (finisher) {
                // ---- finisher of a split tile: add the later pieces' partials in unit order ----
                // This is the CTA's last piece and all its MMAs have completed, so the pipeline
                // smem is idle: each partner's partial (one contiguous [col/4][row] float4 block)
                // is staged there by ONE bulk copy and added from smem.  Per-thread global loads
                // of the same block were latency-bound (~5 us per 128 KB partial at the tail of
                // every split layer, CLB_TRACE_DUMP); CLB_FIXUP_SMEM=0 in the launcher keeps them.
                const uint32_t pbytes = (uint32_t)(kTileM * bn * 4);
                const bool staged = p.fixup_smem && pbytes <= (uint32_t)(stages * group_bytes);
                uint32_t fph = 0;
                for (int u2 = unit + 1; u2 < u_end; ++u2) {
                    const float4* slot = reinterpret_cast<const float4*>(p.partials) +
                                         (long long)(u2 * CG + (int)rank) * (bn >> 2) * kTileM;
                    const float4* src = slot + (long long)(cbase >> 2) * kTileM + trow;
                    if (staged) {
                        epi_bar_sync();   // every epilogue thread is done with the previous partner's copy
                        if (threadIdx.x == 4 * 32) {
                            fence_proxy_async();   // acquired partial (generic) -> bulk read (async proxy)
                            mbar_arrive_expect_tx(fix_bar, pbytes);
                            bulk_copy_g2s(smem, slot, pbytes, fix_bar);
                        }
                        mbar_wait(fix_bar, fph);
                        fph ^= 1u;
                        src = reinterpret_cast<const float4*>(smem) + (cbase >> 2) * kTileM + trow;
                    }
#pragma unroll
                    for (int j = 0; j < 128; j += 4)
                        if (j < hcols) {
                            const float4 v = staged ? src[(j >> 2) * kTileM] : __ldcg(src + (j >> 2) * kTileM);
                            sum[j] += v.x;
                            sum[j + 1] += v.y;
                            sum[j + 2] += v.z;
                            sum[j + 3] += v.w;
                        }
                }
                if (TRACE) t_added = globaltimer_ns();
                // every published partial has exactly one finisher: reset its flags so the
                // buffer is clean for the next launch (no memset launch needed)
                epi_bar_sync();
                if (threadIdx.x == 4 * 32)
                    for (int u2 = unit + 1; u2 < u_end; ++u2) p.flags[u2 * CG + (int)rank] = 0u;
            }
            // ---- tap-stacked: shift-add the k column blocks across rows ----
            int ncol = min(hcols, p.cols - col0);   // valid output columns of this half
            bool row_ok = true;
            if (p.stack_k > 1) {
                if (p.stack_k == 3) shift_add_taps<3>(sum, hcols);
                else if (p.stack_k == 5) shift_add_taps<5>(sum, hcols);
                const int g = hcols / p.stack_k;    // output channels per half
                col0 = nt * (bn / p.stack_k) + half * g;
                ncol = min(g, p.out_channels - col0);
                row_ok = lane < 33 - p.stack_k;
            }
            if (p.sexp) {
                if (hcols <= 32) {   // warp-uniform: a narrow tile scales only the columns it has
#pragma unroll
                    for (int j = 0; j < 32; ++j) sum[j] = apply_pow2(sum[j], ds);
                } else if (hcols <= 64) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) sum[j] = apply_pow2(sum[j], ds);
                } else {
#pragma unroll
                    for (int j = 0; j < 128; ++j) sum[j] = apply_pow2(sum[j], ds);
                }
            }
            // ---- store the finished tile ----
            const long long t_st = TRACE ? clock64() : 0;
            if (!row_ok || ncol <= 0) {
                // dropped row (tap-stacked tile tail) or a column half past the last channel
            } else if (row < p.rows && p.epi == EPI_NCHW_PADDED) {
                // padded output space: row = n*Hp*Wp + y*Wp + x; only y < P, x < Q are outputs
                const int hw = p.epi_hp * p.epi_wp;
                const int n = row / hw;
                const int rem = row - n * hw;
                const int y = rem / p.epi_wp;
                const int xq = rem - y * p.epi_wp;
                if (n < p.epi_n && y < p.P && xq < p.Q) {
                    const long long pix = (long long)y * p.Q + xq;
                    if (p.n_peers == 0)
                        store_nchw(p.out + ((long long)n * p.out_channels + col0) * p.pq_out + pix, p.pq_out, ncol,
                                   p.accumulate, sum);
                    for (int r = 0; r < p.n_peers; ++r)
                        store_nchw(p.peers[r] + ((long long)n * p.peer_M + p.peer_m0 + col0) * p.pq_out + pix, p.pq_out,
                                   ncol, p.accumulate, sum);
                }
            } else if (row < p.rows) {
                if (p.epi == EPI_NCHW) {
                    const int n = row / p.pq_out;
                    const int pq = row - n * p.pq_out;
                    if (p.n_peers == 0)
                        store_nchw(p.out + ((long long)n * p.out_channels + col0) * p.pq_out + pq, p.pq_out,
                                   ncol, p.accumulate, sum);
                    for (int r = 0; r < p.n_peers; ++r)
                        store_nchw(p.peers[r] + ((long long)n * p.peer_M + p.peer_m0 + col0) * p.pq_out + pq,
                                   p.pq_out, ncol, p.accumulate, sum);
                } else if (p.epi == EPI_NHWC_PADDED) {
                    // padded pixel space -> channels-last output row (n*P + y)*Q + x
                    const int hw = p.epi_hp * p.epi_wp;
                    const int n = row / hw;
                    const int rem = row - n * hw;
                    const int y = rem / p.epi_wp;
                    const int xq = rem - y * p.epi_wp;
                    if (n < p.epi_n && y < p.P && xq < p.Q)
                        store_rowmajor(p.out + (((long long)n * p.P + y) * p.Q + xq) * p.ld + col0, p.ld, col0, ncol,
                                       col0 + ncol, p.accumulate, sum);
                } else {
                    store_rowmajor(p.out + (long long)row * p.ld + col0, p.ld, col0, ncol, col0 + ncol, p.accumulate, sum);
                }
            }
            if (TRACE) {
                w_store += clock64() - t_st;
                t_stored = globaltimer_ns();
            }
        }
        if (threadIdx.x == 4 * 32) *epi_done = 1;   // the chained prepass stops taking tiles
        if (TRACE && threadIdx.x == 4 * 32) {
            p.trace[blockIdx.x * kTraceSlots + 5] = (unsigned long long)(clock64() - t_start);
            p.trace[blockIdx.x * kTraceSlots + 6] = (unsigned long long)w_tfull;
            p.trace[blockIdx.x * kTraceSlots + 7] = (unsigned long long)w_store;
            p.trace[blockIdx.x * kTraceSlots + 11] = (unsigned long long)w_fix;
            p.trace[blockIdx.x * kTraceSlots + 13] = t_folded;
            p.trace[blockIdx.x * kTraceSlots + 14] = n_parts;
            p.trace[blockIdx.x * kTraceSlots + 15] = t_pub;
            p.trace[blockIdx.x * kTraceSlots + 16] = t_acq;
            p.trace[blockIdx.x * kTraceSlots + 17] = t_added;
            p.trace[blockIdx.x * kTraceSlots + 18] = t_stored;
        }
    }

    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync();   // the peer must be done with TMEM and barriers
    if (warp == 2) {
        tc_fence_after();
        if constexpr (CG == 2) tmem_dealloc_2sm(tmem_base, ncols);
        else tmem_dealloc(tmem_base, ncols);
    }
    if (TRACE && threadIdx.x == 0) {
        p.trace[blockIdx.x * kTraceSlots + 10] = globaltimer_ns();
        p.trace[blockIdx.x * kTraceSlots + 19] = (unsigned long long)(clock64() - t_entry);   // SM cycles in the CTA
    }
}

#endif  // CLB_DEFINE_TC_KERNEL

}  // namespace clb
