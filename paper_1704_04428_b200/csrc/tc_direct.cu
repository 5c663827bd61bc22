// tc_direct.cu -- tiny-C first layers (VGG conv1_1: C = 3, k = 3) on the tensor cores.
//
// conv_mcmk_loopnest (conv_direct.cpp:104-143) for layers whose whole patch fits one K block
// (C * k * k <= 32): every output pixel's im2col row -- its C k^2 input taps -- is gathered by
// the converter warps from a TMA-loaded input halo in shared memory (the load's out-of-bounds zero
// fill is the row padding) into one 128-byte fp16-split operand row ([hi fp16 32 | lo fp16 32]
// of the power-of-2 scaled values, SWIZZLE_128B), so the patch matrix never exists in HBM; one
// elected thread issues the 6 kind::f16 MMAs of a 128-pixel tile (lo*Hi, hi*Lo, hi*Hi per
// 16-element K step) into one of four TMEM accumulators; the epilogue warps descale, stage the
// tile channel-major in shared memory and one thread writes it with a single TMA tensor store
// (box {128 pixels, M planes} of the output viewed as [N*M planes][P*Q]: whole 128-byte lines,
// asynchronous).  The layer is bound by that 4 B per output element write (AI 12.9 flop/B); the
// CUDA-core kernel (direct.cu) was issue-bound at ~0.4 of it.
//
// Roles (576 threads, one CTA per SM, persistent over 128-pixel tiles t = blockIdx.x + i grid):
//   warps 0-11  converters: three groups of 4 warps (thread = tile row); group g converts the CTA's
//               tiles i = g mod 3 (one group alone is issue-bound)
//                                                 <- halo ring (hfull / hempty), -> A ring (full / empty)
//   warps 12-15 epilogue: TMEM lane quadrant = warp % 4
//   warp  16    TMEM allocator, B loader (TMA), MMA issuer   -> tfull / tempty (4 accumulators)
//   warp  17    halo producer: one 4-D TMA box per tile (rows y0 - pad .., all columns, C planes)
#include <algorithm>
#include <mutex>

#include "internal.hpp"

namespace clb {

namespace {

constexpr int kDGroups = 3;                   // converter warp groups
constexpr int kDEpiWarps = 4;                 // one per TMEM lane quadrant
constexpr int kDEpiWarp = 4 * kDGroups;       // first epilogue warp (a multiple of 4)
constexpr int kDMmaWarp = kDEpiWarp + kDEpiWarps;
constexpr int kDHaloWarp = kDMmaWarp + 1;
constexpr int kDThreads = 32 * (kDHaloWarp + 1);
constexpr int kDStages = 5;                   // A ring
constexpr int kDAStage = kTileM * kRowBytes;  // 16 KB: 128 rows x 128 B
constexpr int kDHalo = 4;                     // halo ring
constexpr int kDHaloMax = 11264;              // bytes per halo slot (VGG conv1_1: 224 x 4 x 3 x 4 B)
constexpr int kDMaxM = 64;                    // staging 2 x 64 x 128 x 4 B = 64 KB
constexpr int kDBufs = 4;                     // TMEM accumulators

struct TcDirectParams {
    int N, H, W, M, pad, P, Q;
    int tiles, tiles_per_img;
    int hb_w, hb_h;        // halo box: columns (= W, a multiple of 4), rows
    const int* sexp;       // [ew, ex]
};

// halo rows a 128-pixel tile needs: the output rows it spans + k - 1
__host__ __device__ inline int d_halo_rows(int Q, int k) { return (kTileM + Q - 1) / Q + 1 + k - 1; }
// the halo box spans the image width (a TMA box wider than the tensor is not allowed; the column
// padding is applied by the converters, the row padding is the box's out-of-bounds zero fill)
__host__ __device__ inline int d_halo_cols(int W, int pad) { return (void)pad, W; }

__host__ __device__ inline int d_halo_offset() { return kDStages * kDAStage; }
__host__ __device__ inline int d_b_offset() { return d_halo_offset() + kDHalo * kDHaloMax; }
__host__ __device__ inline int d_stg_offset(int M) { return d_b_offset() + ((M * kRowBytes + 1023) & ~1023); }
__host__ __device__ inline int d_bar_offset(int M) { return d_stg_offset(M) + 2 * M * kTileM * 4; }
__host__ inline int d_smem_bytes(int M) { return 1024 + d_bar_offset(M) + 256; }

template <int C, int K>
__global__ void __launch_bounds__(kDThreads, 1)
    tc_direct_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                     const __grid_constant__ CUtensorMap map_y, const TcDirectParams p) {
    constexpr int KK = C * K * K;
    static_assert(KK <= 32, "one K block");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int M = p.M;
    uint8_t* sA = smem;
    float* sH = reinterpret_cast<float*>(smem + d_halo_offset());
    uint8_t* sB = smem + d_b_offset();
    float* stg = reinterpret_cast<float*>(smem + d_stg_offset(M));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + d_bar_offset(M));
    uint64_t* full = bars;
    uint64_t* empty = full + kDStages;
    uint64_t* tfull = empty + kDStages;
    uint64_t* tempty = tfull + kDBufs;
    uint64_t* hfull = tempty + kDBufs;
    uint64_t* hempty = hfull + kDHalo;
    uint64_t* bbar = hempty + kDHalo;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bbar + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;
    while (ncols < (uint32_t)(kDBufs * M)) ncols <<= 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kDStages; ++s) {
            mbar_init(&full[s], kTileM);   // every converter thread of the group arrives
            mbar_init(&empty[s], 1);       // the MMA commit
        }
        for (int b = 0; b < kDBufs; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kDEpiWarps);   // one arrive per epilogue warp
        }
        for (int h = 0; h < kDHalo; ++h) {
            mbar_init(&hfull[h], 1);
            mbar_init(&hempty[h], kTileM);
        }
        mbar_init(bbar, 1);
        fence_barrier_init();
    }
    if (warp == kDMmaWarp) {
        tmem_alloc(tmem_slot, ncols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // x and the exponent slots come from the kernels before this one (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp < kDEpiWarp) {
        // ---------------------------------------------------------------- converters ----
        const int grp = warp >> 2;
        const int row = threadIdx.x & (kTileM - 1);   // tile row = TMEM lane = output pixel
        const Pow2 sc = pow2_factors(p.sexp[1]);
        uint8_t* const rbase = sA + row * kRowBytes;
        const int sw = row & 7;                        // SWIZZLE_128B: 16 B chunk c at (c ^ (row & 7))
        int roff[C * K];                               // halo offset of (channel c, tap row i), hoisted
#pragma unroll
        for (int ci = 0; ci < C * K; ++ci) roff[ci] = ((ci % C) * p.hb_h + ci / C) * p.hb_w;
        int i = grp;
        for (int t = blockIdx.x + grp * gridDim.x; t < p.tiles; t += kDGroups * gridDim.x, i += kDGroups) {
            const int s = i % kDStages, h = i % kDHalo;
            const int n = t / p.tiles_per_img;
            const int pq0 = (t - n * p.tiles_per_img) * kTileM;
            const int pq = pq0 + row;
            const int y = pq / p.Q, xq = pq - y * p.Q;
            const int base = (y - pq0 / p.Q) * p.hb_w + xq - p.pad;   // halo row of tap row 0, column of tap 0
            bool colok[K];                             // left / right padding: explicit zeros
#pragma unroll
            for (int j = 0; j < K; ++j) colok[j] = (unsigned)(xq + j - p.pad) < (unsigned)p.W;
            mbar_wait(&hfull[h], (uint32_t)(i / kDHalo) & 1u);
            const float* hb = sH + h * (kDHaloMax / 4) + base;
            float v[KK];
#pragma unroll
            for (int kx = 0; kx < KK; ++kx) {          // K index (i k + j) C + c: MKKC order
                const int tap = kx / C, c = kx % C, ti = tap / K, tj = tap % K;
                v[kx] = colok[tj] ? hb[roff[ti * C + c] + tj] : 0.0f;
            }
            mbar_arrive(&hempty[h]);
            uint32_t hw[16], lw[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const float a = 2 * q < KK ? apply_pow2(v[2 * q < KK ? 2 * q : 0], sc) : 0.0f;
                const float b = 2 * q + 1 < KK ? apply_pow2(v[2 * q + 1 < KK ? 2 * q + 1 : 0], sc) : 0.0f;
                const __half2 hh = __floats2half2_rn(a, b);          // one cvt for the pair
                const float2 hf = __half22float2(hh);
                const __half2 ll = __floats2half2_rn(a - hf.x, b - hf.y);
                hw[q] = *reinterpret_cast<const uint32_t*>(&hh);
                lw[q] = *reinterpret_cast<const uint32_t*>(&ll);
            }
            mbar_wait(&empty[s], ((uint32_t)(i / kDStages) & 1u) ^ 1u);
            uint8_t* rb = rbase + s * kDAStage;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                *reinterpret_cast<uint4*>(rb + ((c ^ sw) << 4)) =
                    make_uint4(hw[4 * c], hw[4 * c + 1], hw[4 * c + 2], hw[4 * c + 3]);
                *reinterpret_cast<uint4*>(rb + (((c + 4) ^ sw) << 4)) =
                    make_uint4(lw[4 * c], lw[4 * c + 1], lw[4 * c + 2], lw[4 * c + 3]);
            }
            fence_proxy_async_smem();   // the generic-proxy writes, before the MMA (async proxy) reads
            mbar_arrive(&full[s]);
        }
    } else if (warp == kDHaloWarp) {
        // ----------------------------------------------------------------- halo loads ----
        const uint32_t bytes = (uint32_t)(p.hb_w * p.hb_h * C) * 4u;
        int i = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++i) {
            const int h = i % kDHalo;
            mbar_wait(&hempty[h], ((uint32_t)(i / kDHalo) & 1u) ^ 1u);
            if (elect_one()) {
                const int n = t / p.tiles_per_img;
                const int y0 = (t - n * p.tiles_per_img) * kTileM / p.Q;
                mbar_arrive_expect_tx(&hfull[h], bytes);
                tma_load_4d(&map_x, &hfull[h], sH + h * (kDHaloMax / 4), 0, y0 - p.pad, 0, n);
            }
            __syncwarp();
        }
    } else if (warp == kDMmaWarp) {
        // ------------------------------------------------------------ B loader + MMA ----
        if (elect_one()) {
            tma_prefetch_desc(&map_w);
            mbar_arrive_expect_tx(bbar, (uint32_t)(M * kRowBytes));
            tma_load_3d(&map_w, bbar, sB, 0, 0, 0);
        }
        __syncwarp();
        mbar_wait(bbar, 0);
        const uint32_t idesc = idesc_f16((uint32_t)kTileM, (uint32_t)M);
        const uint64_t da0 = umma_desc_kmajor(smem_u32(sA), kRowBytes);
        const uint64_t db = umma_desc_kmajor(smem_u32(sB), kRowBytes);
        int i = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++i) {
            const int s = i % kDStages;
            const int b = i % kDBufs;
            mbar_wait(&tempty[b], ((uint32_t)(i / kDBufs) & 1u) ^ 1u);
            mbar_wait(&full[s], (uint32_t)(i / kDStages) & 1u);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t d = tmem_base + (uint32_t)(b * M);
                const uint64_t da = da0 + (uint64_t)((s * kDAStage) >> 4);
                // row = [hi 32 | lo 32] fp16: k-step s of hi at +2 s, of lo at +4 + 2 s (16 B units)
                mma_bf16_ss(d, da + 4, db, idesc, 0u);
                mma_bf16_ss(d, da, db + 4, idesc, 1u);
                mma_bf16_ss(d, da, db, idesc, 1u);
                mma_bf16_ss(d, da + 6, db + 2, idesc, 1u);
                mma_bf16_ss(d, da + 2, db + 6, idesc, 1u);
                mma_bf16_ss(d, da + 2, db + 2, idesc, 1u);
                mma_commit(&empty[s]);
                mma_commit(&tfull[b]);
            }
            __syncwarp();
        }
    } else {
        // ---------------------------------------------------------------- epilogue ----
        const int q = warp & 3;                       // TMEM lane quadrant
        const int row = q * 32 + lane;
        const bool issuer = warp == kDEpiWarp && lane == 0;
        const int dexp = -(p.sexp[0] + p.sexp[1]);
        const Pow2 ds = pow2_factors(dexp < -252 ? -252 : dexp);
        int i = 0;
        for (int t = blockIdx.x; t < p.tiles; t += gridDim.x, ++i) {
            const int b = i % kDBufs;
            mbar_wait(&tfull[b], (uint32_t)(i / kDBufs) & 1u);
            tc_fence_after();
            uint32_t r[kDMaxM / 16][16];
            const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * M);
#pragma unroll
            for (int g = 0; g < kDMaxM / 16; ++g)
                if (g * 16 < M) tmem_ld_32x32b_x16(ta + (uint32_t)(g * 16), r[g]);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
            // staging buffer i & 1: the store that last read it (tile i - 2) must be done reading
            float* st = stg + (i & 1) * (M * kTileM);
            if (issuer) bulk_wait_group_read<1>();
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kDEpiWarps) : "memory");
#pragma unroll
            for (int g = 0; g < kDMaxM / 16; ++g)
                if (g * 16 < M)
#pragma unroll
                    for (int j = 0; j < 16; ++j) st[(g * 16 + j) * kTileM + row] = apply_pow2(__uint_as_float(r[g][j]), ds);
            fence_proxy_async_smem();
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kDEpiWarps) : "memory");
            if (issuer) {
                const int n = t / p.tiles_per_img;
                tma_store_2d(&map_y, st, (t - n * p.tiles_per_img) * kTileM, n * M);
                bulk_commit_group();
            }
        }
        if (issuer) bulk_wait_group0();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kDMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, ncols);
    }
}

template <int C, int K>
void launch_tc_direct_t(const CUtensorMap& mw, const CUtensorMap& mx, const CUtensorMap& my, const TcDirectParams& prm,
                        int grid, int smem, cudaStream_t s) {
    static std::mutex mu;
    static bool configured[64] = {};
    int dev = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> g(mu);
        if (dev >= 0 && dev < 64 && !configured[dev]) {
            CLB_CUDA(cudaFuncSetAttribute(tc_direct_kernel<C, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            configured[dev] = true;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kDThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CLB_CUDA(cudaLaunchKernelEx(&cfg, tc_direct_kernel<C, K>, mw, mx, my, prm));
}

}  // namespace

bool tc_direct_shape(int C, int k, int M, int stride, int pad, int P, int Q) {
    const bool ck = (C == 3 && k == 3) || (C == 2 && k == 3) || (C == 1 && k == 3) || (C == 1 && k == 5);
    if (!ck || stride != 1 || pad != k / 2 || P < 1 || Q < 1) return false;
    // same padding (P = H, Q = W): the output tile store needs whole 128-pixel tiles per image, the
    // input halo box 16 B rows (W % 4 == 0) of at most 256 columns and kDHaloMax bytes
    const int hb_w = d_halo_cols(Q, pad), hb_h = d_halo_rows(Q, k);
    return (M == 32 || M == 64) && ((long long)P * Q) % kTileM == 0 && Q % 4 == 0 && hb_w <= 256 && hb_h <= 256 &&
           (long long)hb_w * hb_h * C * 4 <= kDHaloMax;
}

void launch_tc_direct(const float* x, const void* wpack, float* y, int N, int C, int H, int W, int M, int k, int pad,
                      int P, int Q, const int* sexp, cudaStream_t s, int max_sms) {
    if (!tc_direct_shape(C, k, M, 1, pad, P, Q) || P != H || Q != W)
        throw Error(6, "tensor-core direct kernel: unsupported shape");
    TcDirectParams prm{};
    prm.N = N;
    prm.H = H;
    prm.W = W;
    prm.M = M;
    prm.pad = pad;
    prm.P = P;
    prm.Q = Q;
    prm.tiles_per_img = P * Q / kTileM;
    prm.tiles = N * prm.tiles_per_img;
    prm.hb_w = d_halo_cols(W, pad);
    prm.hb_h = d_halo_rows(Q, k);
    prm.sexp = sexp;
    CUtensorMap mw, mx, my;
    Operand b;
    b.mode = LOAD_TILED;
    b.ptr = wpack;
    b.rows = M;
    b.taps = 1;
    b.kw = 32;   // one 128 B unit: [hi fp16 32 | lo fp16 32]
    b.planes = kPlanesF16;
    encode_operand_map(&mw, b, M, 1);
    {   // input NCHW as {W, H, C, N}; box {halo columns, halo rows, C, 1}
        cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
        cuuint64_t strides[3] = {(cuuint64_t)W * 4, (cuuint64_t)H * W * 4, (cuuint64_t)C * H * W * 4};
        cuuint32_t box[4] = {(cuuint32_t)prm.hb_w, (cuuint32_t)prm.hb_h, (cuuint32_t)C, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        encode_tiled_map(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides, box, estr);
    }
    {   // output as [N*M planes][P*Q pixels]; box {128 pixels, M planes}
        cuuint64_t dims[2] = {(cuuint64_t)P * Q, (cuuint64_t)N * M};
        cuuint64_t strides[1] = {(cuuint64_t)P * Q * 4};
        cuuint32_t box[2] = {(cuuint32_t)kTileM, (cuuint32_t)M};
        cuuint32_t estr[2] = {1, 1};
        encode_tiled_map(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, estr);
    }
    const int sms = num_sms();
    const int grid = std::min(prm.tiles, max_sms > 0 && max_sms < sms ? max_sms : sms);   // one CTA per SM
    const int smem = d_smem_bytes(M);
    if (C == 3) launch_tc_direct_t<3, 3>(mw, mx, my, prm, grid, smem, s);
    else if (C == 2) launch_tc_direct_t<2, 3>(mw, mx, my, prm, grid, smem, s);
    else if (k == 3) launch_tc_direct_t<1, 3>(mw, mx, my, prm, grid, smem, s);
    else launch_tc_direct_t<1, 5>(mw, mx, my, prm, grid, smem, s);
}

}  // namespace clb
