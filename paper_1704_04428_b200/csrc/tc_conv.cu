// tc_conv.cu -- host side of the tcgen05 engine: TMA tensor-map encoding (tiled and
// im2col) and the persistent launch.  The kernel itself lives in tc_conv.cuh.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#define CLB_DEFINE_TC_KERNEL 1
#include "internal.hpp"

namespace clb {

namespace {

using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                     const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                     CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
using PFN_encodeIm2col = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled g_tiled = nullptr;
PFN_encodeIm2col g_im2col = nullptr;
std::once_flag g_once;

void resolve_driver() {
    std::call_once(g_once, [] {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_tiled = reinterpret_cast<PFN_encodeTiled>(fn);
        fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_im2col = reinterpret_cast<PFN_encodeIm2col>(fn);
    });
    if (!g_tiled || !g_im2col) throw Error(3, "cuTensorMapEncode* entry points unavailable (driver too old?)");
}

}  // namespace

int num_sms() {
    int dev = 0, n = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    CLB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

void encode_operand_map(CUtensorMap* map, const Operand& op, int box_rows, int box_taps) {
    resolve_driver();
    const cuuint64_t kdim = (cuuint64_t)op.kw;   // elements per row (2 words per channel for the split formats)
    const cuuint64_t eb = (cuuint64_t)elem_bytes(op.planes);
    const CUtensorMapDataType dt = op.planes == kPlanesBf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                            : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    const cuuint32_t unit = (cuuint32_t)(kRowBytes / eb);   // elements per 128-byte row unit
    CUresult r;
    if (op.mode == LOAD_IM2COL) {
        cuuint64_t dims[4] = {kdim, (cuuint64_t)op.w, (cuuint64_t)op.h, (cuuint64_t)op.n};
        cuuint64_t strides[3] = {kdim * eb, kdim * eb * op.w, kdim * eb * op.w * op.h};
        // Bounding box: lower corner -pad, upper corner pad-(k-1) in W and H, so the
        // traversal enumerates exactly the P x Q output positions of each image.
        int lower[2] = {-op.pad, -op.pad};
        int upper[2] = {op.pad - (op.k - 1), op.pad - (op.k - 1)};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        r = g_im2col(map, dt, 4, const_cast<void*>(op.ptr), dims, strides, lower,
                     upper, unit, (cuuint32_t)box_rows, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {kdim, (cuuint64_t)op.rows, (cuuint64_t)op.taps};
        const cuuint64_t slice = (cuuint64_t)(op.tap_stride_rows > 0 ? op.tap_stride_rows : op.rows);
        cuuint64_t strides[2] = {kdim * eb, kdim * eb * slice};
        cuuint32_t box[3] = {unit, (cuuint32_t)box_rows, (cuuint32_t)box_taps};
        cuuint32_t estr[3] = {1, 1, 1};
        r = g_tiled(map, dt, 3, const_cast<void*>(op.ptr), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS)
        throw Error(3, "cuTensorMapEncode" + std::string(op.mode == LOAD_IM2COL ? "Im2col" : "Tiled") +
                           " failed with CUresult " + std::to_string((int)r));
}

void encode_tiled_map(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* ptr, const cuuint64_t* dims,
                      const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* estr) {
    resolve_driver();
    const CUresult r = g_tiled(map, dt, (cuuint32_t)rank, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(3, "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r));
}

namespace {

// Per-device launch configuration of the engine: the >48 KB dynamic smem opt-in (a per-device
// function attribute) and the co-resident unit limit per (cluster shape, smem size), computed
// once each under a lock.
struct DeviceLimits {
    int units = 0;
};

const DeviceLimits& device_limits(int cg, int smem, int max_sms) {
    static std::mutex mu;
    static std::unordered_map<unsigned long long, DeviceLimits> cache;
    static bool configured[64][3] = {};
    int dev = 0;
    CLB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) throw Error(6, "device index out of range");
    const unsigned long long key = ((unsigned long long)dev << 40) | ((unsigned long long)cg << 32) |
                                   ((unsigned long long)(unsigned)smem << 8) | (unsigned)(max_sms & 0xff);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (!configured[dev][cg]) {
        if (cg == 2) {
            CLB_CUDA(cudaFuncSetAttribute(tc_conv_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            CLB_CUDA(cudaFuncSetAttribute(tc_conv_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        } else {
            CLB_CUDA(cudaFuncSetAttribute(tc_conv_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
            CLB_CUDA(cudaFuncSetAttribute(tc_conv_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        }
        configured[dev][cg] = true;
    }
    int sms = 0;
    CLB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    int units = (sms < kMaxGrid ? sms : kMaxGrid) / cg;
    if (cg == 2) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * units);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        CLB_CUDA(cudaOccupancyMaxActiveClusters(&clusters, tc_conv_kernel<2, false>, &cfg));
        if (clusters < units) units = clusters;
    } else {
        int per_sm = 0;
        CLB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tc_conv_kernel<1, false>, kThreads, smem));
        if (per_sm * sms < units) units = per_sm * sms;
    }
    if (max_sms > 0 && std::max(1, max_sms / cg) < units) units = std::max(1, max_sms / cg);
    if (units < 1) throw Error(2, "tcgen05 engine: no CTA of this configuration fits on the device");
    return cache[key] = DeviceLimits{units};
}

}  // namespace

int launch_tc(const Operand& a, const Operand& b, TcParams p, cudaStream_t s, int cg) {
    if (cg != 1 && cg != 2) throw Error(6, "cta group must be 1 or 2");
    if (p.bn % 16 != 0 || p.bn < 16 || p.bn > 256) throw Error(6, "tile N must be a multiple of 16 in [16,256]");
    const int unit = kRowBytes / elem_bytes(a.planes);
    if (a.kw != b.kw || a.kw % unit != 0 || a.planes != b.planes) throw Error(6, "operand K layout mismatch");
    if (p.tps <= 0) p.tps = 1;
    if (p.stack_k <= 1) {
        p.stack_k = 1;
        p.row_step = kTileM;
    } else {
        if (p.stack_k != 3 && p.stack_k != 5) throw Error(6, "tap-stacked mode supports k = 3 and 5");
        if ((p.bn / 2) % p.stack_k != 0) throw Error(6, "tap-stacked tile N must hold whole tap groups per half");
        if (a.mode != LOAD_TILED || p.tps != 1) throw Error(6, "tap-stacked mode needs a tiled A, one tap per stage");
        p.row_step = 4 * (33 - p.stack_k);
    }
    if (p.msub <= 1) {
        p.msub = 1;
    } else if (p.msub != 2 || p.stack_k != 1 || a.mode != LOAD_TILED || p.tps < 2 ||
               (a.planes != kPlanesMixed && a.planes != kPlanesF16) || p.bn % 32 != 0) {
        throw Error(6, "two-sub-tile mode: mixed / fp16 split, tap-shared tiled A, N a multiple of 16 per sub-tile");
    }
    const int mma_n = p.bn / p.msub;
    CUtensorMap ma, mb;
    // tap-stacked: A = {unit, 32 rows, 4 quadrants} over the overlapping quadrant view
    if (p.stack_k > 1 && (a.taps != 4 || a.tap_stride_rows != 33 - p.stack_k))
        throw Error(6, "tap-stacked A must be the 4-quadrant overlapping view");
    encode_operand_map(&ma, a, p.stack_k > 1 ? 32 : tc_a_box_rows(p.tps), p.stack_k > 1 ? 4 : 1);
    encode_operand_map(&mb, b, mma_n / cg, p.tps);
    p.planes = a.planes;
    if (p.planes == kPlanesF16 && !p.sexp) throw Error(6, "fp16 split contraction without its exponent slots");
    if (p.planes != kPlanesF16) p.sexp = nullptr;
    p.row_elems = unit;
    p.kblocks = a.kw / unit;
    p.a_mode = a.mode;
    p.b_mode = b.mode;
    if (p.taps % p.tps != 0) throw Error(6, "taps per stage must divide the tap count");
    const int k_iters = (p.taps / p.tps) * p.kblocks;
    const int b_rows = mma_n / cg;
    // chunk = K slice per TMEM accumulator.  The fp32-faithful splits bound it to kChunkK
    // K-elements (16 channels x tps taps per k-iteration): tensor-core accumulation error grows
    // ~linearly with the chunk (rel-L2 8.3e-7 / 1.07e-6 / 1.33e-6 at 128 / 192 / 256, bound 1e-5;
    // profiles/r01_chunk_accuracy.txt), while short chunks cost the small-N tap-shared layers
    // 7-9 % (VGG conv1_2-2_2 at 96 vs 192 K).  The 1e-2 fast modes only chunk for stream-K
    // granularity: 16 iterations keep the epilogue's fold rate below the MMA's (4 had the MMA
    // waiting on TMEM 11-25 % of the time, CLB_TRACE).
    if (p.chunk_iters <= 0) {
        if (p.planes == kPlanesF16) {
            // 32 channels per k-iteration and tap.  The fp16 split's 22-bit operands leave room for
            // longer chunks than the other splits: rel-L2 6.7e-7 / 1.3e-6 / 1.9e-6 / 2.7e-6 at
            // 192 / 384 / 576 / 768 K-elements (bound 1e-5; the reference's own fp32 sum is 1.1e-6
            // at K = 36864), and fewer TMEM folds per tile are what the epilogue-bound small-N
            // padded-row layers need: 576 there (VGG conv1_2 0.337 -> 0.310 ms, conv2_1 0.149 ->
            // 0.126), 384 with one tap per k-iteration (conv3_1 0.134 -> 0.124; 576 coarsens the
            // stream-K split of conv5_x: 0.077 -> 0.090)  (profiles/r02_f16_chunk.txt)
            p.chunk_iters = (p.tps > 1 ? kChunkKF16Padded : kChunkKF16) / (32 * p.tps);
        } else if (is_split(p.planes)) {
            p.chunk_iters = kChunkK / (16 * p.tps);
        } else {
            p.chunk_iters = kFastChunkIters / p.tps;
        }
        if (p.chunk_iters < 1) p.chunk_iters = 1;
        static const int env_chunk = getenv("CLB_CHUNK") ? atoi(getenv("CLB_CHUNK")) : 0;   // experiment knob
        if (env_chunk > 0) p.chunk_iters = env_chunk;
    }
    if (p.chunk_iters > k_iters) p.chunk_iters = k_iters;
    // Stage grouping: bps k-iterations share one full/empty barrier round trip.  Two per stage
    // are 2-5 % faster on every layer that still keeps >= 3 stages in flight; with only 2
    // stages left the pipeline runs dry (VGG conv5_x, conv2_1: 3-7 % slower), so stay at 1.
    // A and B loads from two producer warps: 3-8 % on the TMA-im2col layers (AlexNet conv2 / conv5,
    // VGG conv5_x), neutral on the padded-row ones (profiles/r01_split_issue_sweep.txt)
    static const int env_split_issue = getenv("CLB_SPLIT_ISSUE") ? atoi(getenv("CLB_SPLIT_ISSUE")) : 1;
    p.split_issue = env_split_issue;
    // A boxes of alternate stages issued from two warps (0 and the idle TMEM-allocator warp 2):
    // +0.5-2 % on the padded-row layers (VGG conv1_2 0.508 -> 0.499 ms), neutral on the TMA-im2col
    // ones (profiles/r01_a_issuers_ab.txt).  CLB_A_ISSUERS=1 restores one A warp.
    static const int env_a_iss = getenv("CLB_A_ISSUERS") ? atoi(getenv("CLB_A_ISSUERS")) : 2;
    p.a_issuers = (env_a_iss == 2 && p.split_issue) ? 2 : 1;
    static const int env_smem = getenv("CLB_SMEM_KB") ? atoi(getenv("CLB_SMEM_KB")) * 1024 : 0;   // experiment knob
    const int budget = env_smem > 0 ? env_smem : kSmemBudget;
    const int stage_b_rows = b_rows;   // B rows carried per stage
    if (p.bps <= 0) {
        static const int env_bps = getenv("CLB_BPS") ? atoi(getenv("CLB_BPS")) : 0;   // experiment knob
        if (env_bps > 0) p.bps = env_bps;
        else p.bps = (tc_num_stages(stage_b_rows, p.tps, 2, budget, p.msub) >= 3 && (p.chunk_iters % 2 == 0 || p.chunk_iters == k_iters)) ? 2 : 1;
    }
    p.stages = tc_num_stages(stage_b_rows, p.tps, p.bps, budget, p.msub);
    while (p.stages < 2 && p.bps > 1) p.stages = tc_num_stages(stage_b_rows, p.tps, --p.bps, budget, p.msub);
    if (p.stages < 2) throw Error(2, "tile too large for a 2-stage pipeline");
    // chunk boundaries must be stage boundaries: chunk_iters a multiple of bps (a single-chunk
    // tile is exempt -- its only chunk starts the piece and ends at k_iters)
    if (p.chunk_iters < k_iters && p.chunk_iters % p.bps != 0)
        p.chunk_iters = p.chunk_iters >= p.bps ? p.chunk_iters / p.bps * p.bps : p.bps;
    if (p.chunk_iters > k_iters) p.chunk_iters = k_iters;
    const int tile_m = p.row_step * cg * p.msub;   // output rows per tile
    const int row_tiles = (p.rows + tile_m - 1) / tile_m;
    p.n_col_tiles = (p.cols + mma_n - 1) / mma_n;
    p.num_tiles = row_tiles * p.n_col_tiles;
    if (p.num_tiles <= 0) return 0;
    p.chunks_per_tile = (k_iters + p.chunk_iters - 1) / p.chunk_iters;
    const long long total_chunks = (long long)p.num_tiles * p.chunks_per_tile;
    const int smem = tc_smem_bytes(stage_b_rows, p.tps, p.stages, p.bps, p.msub);
    // The stream-K fixup makes CTAs wait on each other, so every CTA of the grid must be
    // co-resident: the unit count is capped at what the occupancy calculator says fits at once
    // for this kernel, smem size and cluster shape (on the current device; attributes and
    // limits are per device, configured once each).
    const DeviceLimits& lim = device_limits(cg, smem, p.max_sms);
    int units = lim.units;      // scheduling units (CTAs or CTA pairs)
    if (total_chunks < units) units = (int)total_chunks;
    // Fewer tiles than units (latency-bound problems): pick the split s (pieces per tile) by a
    // cost model in chunk times -- ceil(chunks / units) on the critical path, plus a fixup of
    // ~3 chunk times and ~0.5 per extra piece whenever tiles are split.  Calibrated on the
    // batch-1 / GoogLeNet / k-sweep layers (profiles/r01_split_sweep.txt): small-K layers stay
    // unsplit, big-K ones split up to kMaxSplit.  CLB_MAX_SPLIT caps s for experiments.
    static const int max_split = [] {
        const char* e = getenv("CLB_MAX_SPLIT");
        const int v = e ? atoi(e) : 0;
        return (v >= 1 && v <= kMaxSplit) ? v : kMaxSplit;
    }();
    if (p.num_tiles < units) {
        double best = 1e30;
        int best_units = p.num_tiles;
        for (int sp = 1; sp <= max_split; ++sp) {
            const long long u = std::min<long long>(units, (long long)p.num_tiles * sp);
            const double t = (double)((total_chunks + u - 1) / u) + (sp > 1 ? 3.0 + 0.5 * (sp - 1) : 0.0);
            if (t < best - 1e-9) {
                best = t;
                best_units = (int)u;
            }
            if (u == units) break;
        }
        units = best_units;
    }
    // whole-tile waves for all but the last 1-2 waves; stream-K over the rest
    // (a last wave that is >= 95% full stays data-parallel: splitting it costs more than it saves)
    const int waves = p.num_tiles / units;
    const int ceil_waves = (p.num_tiles + units - 1) / units;
    const bool balanced = (long long)(ceil_waves * units - p.num_tiles) * 20 <= (long long)ceil_waves * units;
    p.dp_tiles = balanced ? p.num_tiles : (waves >= 2 ? (waves - 1) * units : 0);
    p.sk_chunks = (p.num_tiles - p.dp_tiles) * p.chunks_per_tile;
    // Stream-K unit count: with contiguous equal ranges over all units, a tile can straddle
    // three units whenever a range is shorter than a tile, and a 3-piece tile's finisher waits
    // for and adds two partials at the very end of the kernel (VGG conv5_1: those CTAs exit
    // ~8 us after the 2-piece ones; CLB_TRACE_DUMP).  Pick the unit count u <= units that
    // minimises ceil(chunks / u) + fixup(max pieces per tile), in chunk times: 2 pieces 2
    // (3 until the fp16 split's longer chunks: at 3, VGG conv4_1 left 13 of its 74 CTA pairs
    // idle in the stream-K wave rather than split a tile, 0.137 -> 0.132 ms at 2, every other
    // BASELINE layer unchanged: profiles/r02c_sk_fixup_cost.txt), each further piece +2
    // (profiles/r01_sk_units.txt).  CLB_SK_UNITS=0 keeps all units.
    p.sk_units = units;
    static const int env_sk = getenv("CLB_SK_UNITS") ? atoi(getenv("CLB_SK_UNITS")) : 1;
    static const int env_fix = getenv("CLB_FIXUP_SMEM") ? atoi(getenv("CLB_FIXUP_SMEM")) : 1;
    p.fixup_smem = env_fix != 0 ? 1 : 0;
    // (memoised per (chunks, chunks per tile, units): a plan's launches repeat the same shape)
    thread_local std::unordered_map<unsigned long long, int> sk_memo;
    const unsigned long long sk_key = ((unsigned long long)(unsigned)p.sk_chunks << 32) ^
                                      ((unsigned long long)(unsigned)p.chunks_per_tile << 12) ^ (unsigned)units;
    const auto sk_hit = sk_memo.find(sk_key);
    if (env_sk != 0 && p.sk_chunks > 0 && sk_hit != sk_memo.end()) {
        p.sk_units = sk_hit->second;
    } else if (env_sk != 0 && p.sk_chunks > 0) {
        const int cpt = p.chunks_per_tile, S = p.sk_chunks;
        auto max_pieces = [&](int u) {
            int worst = 1;
            for (int t = 0; t * cpt < S; ++t) {
                // unit holding chunk c: the b with chunk_start(b) <= c < chunk_start(b + 1)
                auto unit_of = [&](int c) {
                    int b = (int)(((long long)c * u) / S);
                    while (b + 1 < u && chunk_start(b + 1, S, u) <= c) ++b;
                    while (b > 0 && chunk_start(b, S, u) > c) --b;
                    return b;
                };
                const int pcs = unit_of(std::min(S, (t + 1) * cpt) - 1) - unit_of(t * cpt) + 1;
                if (pcs > worst) worst = pcs;
            }
            return worst;
        };
        auto cost = [&](int u) {
            const int mp = max_pieces(u);
            return (double)((S + u - 1) / u) + (mp <= 1 ? 0.0 : 2.0 + 2.0 * (mp - 2));
        };
        double best = cost(units);
        for (int u = units - 1; u >= std::max(1, units - 24); --u) {
            const double c = cost(u);
            if (c < best - 1e-9) {
                best = c;
                p.sk_units = u;
            }
        }
        sk_memo[sk_key] = p.sk_units;
    }
    if (p.sk_units > kMaxUnits) throw Error(6, "too many scheduling units");
    for (int b = 0; b <= p.sk_units; ++b) p.sk_start[b] = chunk_start(b, p.sk_chunks, p.sk_units);
    const int grid = units * cg;
    if (!p.partials || !p.flags) throw Error(6, "stream-K scratch missing");
    if (!p.flags_zeroed) CLB_CUDA(cudaMemsetAsync(p.flags, 0, (size_t)grid * sizeof(unsigned), s));
    // PDL only when nothing was enqueued in between (the memset would be the predecessor)
    if (!p.flags_zeroed) p.pdl = 0;
    // The stream-K fixup makes CTAs wait on each other, so all must be resident: the grid is
    // capped at the co-resident limit above.  CG = 1 additionally asks for a cooperative launch
    // (the driver then refuses a grid that cannot be co-resident); CG = 2 uses a plain cluster
    // launch (cooperative + cluster is rejected under ncu), sized by
    // cudaOccupancyMaxActiveClusters.  A CTA that could still never be scheduled (other
    // kernels holding SMs indefinitely) trips the 4 s watchdog: a launch error, not a hang.
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (cg == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 2;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    } else {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (p.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    // CLB_TRACE=1: per-CTA role wait cycles (diagnostics only; synchronises after the launch)
    static const bool trace = getenv("CLB_TRACE") && atoi(getenv("CLB_TRACE")) != 0;
    static unsigned long long* trace_buf = nullptr;
    if (trace) {
        if (!trace_buf) CLB_CUDA(cudaMalloc(&trace_buf, (size_t)kMaxGrid * kTraceSlots * sizeof(unsigned long long)));
        CLB_CUDA(cudaMemsetAsync(trace_buf, 0, (size_t)kMaxGrid * kTraceSlots * sizeof(unsigned long long), s));
        p.trace = trace_buf;
        p.pdl = 0;
        cfg.numAttrs = 1;   // no PDL: the trace needs the launch to be self-contained
    }
    // CLB_DEBUG_WAIT=1: barrier waits give up after 0.2 s and record themselves (ptx.cuh); the
    // launch is synchronised and the records printed -- a protocol debugging aid
    static const bool dbg_wait = getenv("CLB_DEBUG_WAIT") && atoi(getenv("CLB_DEBUG_WAIT")) != 0;
    if (dbg_wait) {
        const unsigned one = 1;
        unsigned long long zero[8] = {};
        CLB_CUDA(cudaMemcpyToSymbolAsync(clb_dbg_mode, &one, sizeof(one), 0, cudaMemcpyHostToDevice, s));
        CLB_CUDA(cudaMemcpyToSymbolAsync(clb_dbg_record, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s));
        p.pdl = 0;
        cfg.numAttrs = 1;
    }
    static cudaEvent_t tev[2] = {nullptr, nullptr};
    if (trace) {
        if (!tev[0]) {
            CLB_CUDA(cudaEventCreate(&tev[0]));
            CLB_CUDA(cudaEventCreate(&tev[1]));
        }
        CLB_CUDA(cudaEventRecord(tev[0], s));
    }
    // the traced instantiation carries the diagnostics; the production one has none of their
    // registers (they were live across the whole epilogue loop)
    cudaError_t e = trace ? (cg == 2 ? cudaLaunchKernelEx(&cfg, tc_conv_kernel<2, true>, ma, mb, p)
                                     : cudaLaunchKernelEx(&cfg, tc_conv_kernel<1, true>, ma, mb, p))
                          : (cg == 2 ? cudaLaunchKernelEx(&cfg, tc_conv_kernel<2, false>, ma, mb, p)
                                     : cudaLaunchKernelEx(&cfg, tc_conv_kernel<1, false>, ma, mb, p));
    CLB_CUDA(e);
    if (dbg_wait) {
        unsigned long long rec[8];
        CLB_CUDA(cudaMemcpyFromSymbolAsync(rec, clb_dbg_record, sizeof(rec), 0, cudaMemcpyDeviceToHost, s));
        CLB_CUDA(cudaStreamSynchronize(s));
        fprintf(stderr, "[clb-dbg] rows=%d cols=%d bn=%d cg=%d stages=%d bps=%d grid=%d bars at +0x%x "
                "(full[s], empty[s], tfull[4], tempty[4], fix): %u timed-out waits\n", p.rows, p.cols, p.bn, cg,
                p.stages, p.bps, grid, p.stages * p.bps * tc_stage_bytes(stage_b_rows, p.tps, p.msub),
                (unsigned)(rec[7] & 0xffffffffu));
        for (int i = 0; i < 6 && i < (int)(rec[7] & 0xffffffffu); ++i)
            fprintf(stderr, "[clb-dbg]   block %llu warp %llu bar smem+0x%llx parity %llu\n", rec[i] >> 40,
                    (rec[i] >> 32) & 0xff, (rec[i] & 0xffffffffu) >> 1, rec[i] & 1);
    }
    if (trace) {
        CLB_CUDA(cudaEventRecord(tev[1], s));
        std::vector<unsigned long long> h((size_t)grid * kTraceSlots);
        CLB_CUDA(cudaMemcpyAsync(h.data(), trace_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        CLB_CUDA(cudaStreamSynchronize(s));
        float ev_ms = 0.0f;
        CLB_CUDA(cudaEventElapsedTime(&ev_ms, tev[0], tev[1]));
        double avg[kTraceSlots] = {0};
        unsigned long long t_in = ~0ull, t_in_max = 0, t_out = 0;
        for (int b = 0; b < grid; ++b) {
            for (int i = 0; i < kTraceSlots; ++i) avg[i] += (double)h[(size_t)b * kTraceSlots + i] / grid;
            t_in = std::min(t_in, h[(size_t)b * kTraceSlots + 9]);
            t_in_max = std::max(t_in_max, h[(size_t)b * kTraceSlots + 9]);
            t_out = std::max(t_out, h[(size_t)b * kTraceSlots + 10]);
        }
        double cyc_sum = 0, ns_sum = 0;
        for (int b = 0; b < grid; ++b) {
            cyc_sum += (double)h[(size_t)b * kTraceSlots + 19];
            ns_sum += (double)(h[(size_t)b * kTraceSlots + 10] - h[(size_t)b * kTraceSlots + 9]);
        }
        const double mhz = ns_sum > 0 ? 1e3 * cyc_sum / ns_sum : 0.0;
        fprintf(stderr,
                "[clb-trace] rows=%d cols=%d bn=%d cg=%d tps=%d stack=%d msub=%d aiss=%d bps=%d stages=%d cpt=%d grid=%d tiles=%d dp=%d sku=%d | producer %.0f cyc "
                "(wait empty %.0f%%) | mma %.0f (wait full %.0f%%, wait tmem %.0f%%) | epilogue %.0f (wait tfull %.0f%%, "
                "store %.0f%%, fixup wait %.0f%%) | setup %.0f cyc | span %.1f us (last CTA start +%.1f us) | events %.1f us | "
                "SM clock %.0f MHz (CTA cycles / CTA ns)\n",
                p.rows, p.cols, p.bn, cg, p.tps, p.stack_k, p.msub, p.a_issuers, p.bps, p.stages, p.chunks_per_tile, grid, p.num_tiles, p.dp_tiles, p.sk_units, avg[0], 100 * avg[1] / avg[0],
                avg[2], 100 * avg[3] / avg[2], 100 * avg[4] / avg[2], avg[5], 100 * avg[6] / avg[5], 100 * avg[7] / avg[5], 100 * avg[11] / avg[5], avg[8], (t_out - t_in) * 1e-3,
                (t_in_max - t_in) * 1e-3, ev_ms * 1e3, mhz);
        if (const char* dump = getenv("CLB_TRACE_DUMP")) {   // raw per-CTA records, appended
            if (FILE* f = fopen(dump, "a")) {
                fprintf(f, "# launch rows=%d cols=%d bn=%d cg=%d grid=%d tiles=%d dp=%d cpt=%d\n", p.rows, p.cols, p.bn, cg,
                        grid, p.num_tiles, p.dp_tiles, p.chunks_per_tile);
                for (int b = 0; b < grid; ++b) {
                    const unsigned long long* r = &h[(size_t)b * kTraceSlots];
                    auto rel = [&](unsigned long long t) { return t ? (double)(t - t_in) * 1e-3 : -1.0; };
                    fprintf(f,
                            "cta %d prod %llu mma %llu epi %llu wtfull %llu wfix %llu nparts %llu | start %.2f "
                            "mma_end %.2f folded %.2f published %.2f acquired %.2f added %.2f stored %.2f exit %.2f us\n",
                            b, r[0], r[2], r[5], r[6], r[11], r[14], rel(r[9]), rel(r[12]), rel(r[13]), rel(r[15]),
                            rel(r[16]), rel(r[17]), rel(r[18]), rel(r[10]));
                }
                fclose(f);
            }
        }
        // the slowest CTA (latest exit) decides the kernel time: its own breakdown
        int slow = 0;
        for (int b = 1; b < grid; ++b)
            if (h[(size_t)b * kTraceSlots + 10] > h[(size_t)slow * kTraceSlots + 10]) slow = b;
        const unsigned long long* r = &h[(size_t)slow * kTraceSlots];
        int lead = cg == 2 ? (slow & ~1) : slow;   // the MMA runs on the pair's leader
        const unsigned long long* rl = &h[(size_t)lead * kTraceSlots];
        if (p.nx_on)
            fprintf(stderr, "[clb-trace]   chained prepass: %.0f tiles per CTA converted by the converter warps\n", avg[23]);
        fprintf(stderr,
                "[clb-trace]   slowest CTA %d: exit +%.1f us | producer %llu (wait empty %llu) | mma %llu (wait full "
                "%llu, wait tmem %llu) | epilogue %llu (wait tfull %llu, store %llu, fixup wait %llu) cyc\n",
                slow, (r[10] - t_in) * 1e-3, r[0], r[1], rl[2], rl[3], rl[4], r[5], r[6], r[7], r[11]);
    }
    return 1;
}

size_t tc_scratch_bytes() {
    return (size_t)kMaxGrid * kTileM * 256 * sizeof(float) + (size_t)kMaxGrid * sizeof(unsigned);
}

}  // namespace clb
