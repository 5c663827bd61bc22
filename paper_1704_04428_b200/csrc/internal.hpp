// internal.hpp -- declarations shared by the CUDA translation units (not part of the ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "tc_conv.cuh"

namespace clb {

// status-carrying exception used inside the library; converted to cl_status at the ABI.
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define CLB_CUDA(expr)                                                                              \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            throw ::clb::Error(3, std::string(#expr) + ": " + cudaGetErrorString(_e));              \
    } while (0)

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
// Precision modes ("planes" code carried through the engine):
//   2 = fp32-faithful 3xTF32 (rows interleave [hi16|lo16] fp32 words per 16 channels)
//   1 = TF32 fast mode (rows of hi fp32 words)
//   3 = BF16 fast mode (rows of bf16 elements, kind::f16 MMA)
//   4 = fp32-faithful "2xTF32 + 2xBF16": per 16 channels [hi 16 fp32 | hi 16 bf16 | lo 16 bf16]
//       -- hi*Hi in two tf32 MMAs (exact products), the cross terms hi*Lo and lo*Hi in one
//       bf16 MMA each (K = 16 per MMA: 4 MMA slots per 16 channels instead of 6)
//   5 = fp32-faithful fp16 split (implicit kn2row family): the operand is scaled by an exact power
//       of two 2^e (input: from max|x| per forward; weights: from max|w| at set_weights) so its
//       largest magnitude lies in [2^14, 2^15), then x = hi + lo with hi = fp16(x), lo = fp16(x - hi)
//       (22 significant bits); per 32 channels one 128 B unit [hi fp16 32 | lo fp16 32].  D +=
//       lo*Hi + hi*Lo + hi*Hi as kind::f16 K=16 MMAs (exact products): 3 MMA slots per 16 channels
//       instead of 4, half the operand bytes; the epilogue multiplies by 2^-(ex + ew).
// kPlanesBf16 = 3, kPlanesMixed = 4, kPlanesF16 = 5: split_tile.cuh (included through tc_conv.cuh)
// hi|lo split formats with one 128-byte row unit per 16 channels (two words per channel)
__host__ __device__ inline bool is_split(int planes) { return planes == 2 || planes == kPlanesMixed; }
// fp32-faithful formats (chunked accumulation, rel-L2 <= 1e-5)
__host__ __device__ inline bool is_faithful(int planes) { return is_split(planes) || planes == kPlanesF16; }
// channel padding granularity of the split layout (one 128-byte row unit)
inline int k_granule(int planes) { return is_split(planes) ? 16 : (planes == kPlanesBf16 ? 64 : 32); }
inline int elem_bytes(int planes) { return planes == kPlanesBf16 ? 2 : 4; }
// elements (4-byte words for the split formats) per operand row of k_pad channels
inline long long row_elems(int planes, long long kp) { return is_split(planes) ? 2 * kp : kp; }
inline long long row_bytes(int planes, long long kp) { return row_elems(planes, kp) * elem_bytes(planes); }

// ---- pre-pass / post-pass kernels (prepass.cu) -------------------------------------------
// Split layout of every operand row (k_pad channels): per 16-channel block one 128 B unit
// ([hi 16 fp32 | bf16 hi 16 | bf16 lo 16] mixed, [hi 16 | lo 16] 3xTF32; row = 2*k_pad words);
// TF32 -> hi only (row = k_pad words, k_pad % 32 == 0); BF16 -> bf16 (k_pad % 64 == 0).
// x NCHW fp32 -> xs[n][h][w][row] (hi = rna_tf32(x), lo = x - hi; zero for c >= C)
// sexp (fp16 split only): the plan's exponent slots [ew, ex]; the split reads ex (written by
// launch_absmax_exp over the same input just before)
void launch_nchw_to_nhwc_split(const float* x, void* xs, int N, int C, int HW, int Cp, int planes,
                               cudaStream_t s, const int* sexp = nullptr);
// same, into the zero-padded image [n][H+2pad][W+2pad][row] (tap-shared kernel mode)
// NHWC input (channels last) -> split rows; pad > 0 writes the zero-padded grid (tap-shared mode)
// (padded grids: wp = the padded row width, 0 = W + pad; the trailing wp - W zeros of a row are the
// next row's leading padding)
void launch_nhwc_split(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp, int planes,
                       cudaStream_t s, const int* sexp = nullptr, int wp = 0);
void launch_nchw_to_padded_split(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp, int planes,
                                 cudaStream_t s, const int* sexp = nullptr, int wp = 0);
// fp16 split scale: exponent e with max|x| * 2^e in [2^14, 2^15) (0 for an all-zero or non-finite
// tensor; in [-113, 163] otherwise) written to *out_exp.  `slots` = the plan's scale buffer (partials +
// completion counter, self-resetting).  Stream-ordered, graph-capturable.
constexpr int kScaleSlots = 8;          // [0] ew, [1] ex, [2] counter, [3] e_spec, [4] e_spec valid, [6] e_use
constexpr int kAbsmaxBlocks = 1024;     // absmax partial maxima [8, 8 + 1024)
constexpr int kSpecGroups = kSpecGroupSlots;   // speculative prepass: group maxima (zeroed by the contraction)
constexpr int kSpecStride = kSpecGroupStride;   // ints between group slots (own 64 B sector each)
constexpr int kScaleBufInts = kScaleSlots + kAbsmaxBlocks + kSpecGroups * kSpecStride;
void launch_absmax_exp(const float* x, long long n, int* slots, int* out_exp, cudaStream_t s);
// fp16 split, single pass over x (NCHW input): the prepass converts with the exponent of the
// plan's previous forward (speculation) while reducing max|x|; its last block writes the exact
// maxima, and the fixup kernel launched behind it publishes the exact exponent ex and re-converts
// the whole input with it only when the speculation missed (the first forward, or a changed
// range), so the operand is always the one the two-pass form writes (bitwise).  The contraction
// must then zero the group maxima: spec_reset_slots().
void launch_nchw_split_speculative(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp,
                                   int* slots, cudaStream_t s, int wp = 0);
inline unsigned* spec_reset_slots(int* slots) { return reinterpret_cast<unsigned*>(slots + kScaleSlots + kAbsmaxBlocks); }
// the same conversion as a tile job (chained mode) and the tail launch that finishes its tiles
// left by the previous contraction's converter warps (then resets the job's counter)
SplitJob make_split_job(const float* x, void* xs, int N, int C, int H, int W, int pad, int Cp);
void launch_split_tail(const SplitJob& j, int planes, cudaStream_t s);
// a[rows][K] -> as[rows][planes][Kp]
void launch_rows_split(const float* a, void* as, long long rows, int K, int Kp, int planes, cudaStream_t s,
                       const int* sexp = nullptr);
// b[K][cols] -> bs[cols][planes][Kp]
void launch_transpose_split(const float* b, void* bs, int K, int cols, int Kp, int planes, cudaStream_t s);
// w MKKC -> wp[tap][M][planes][Cp], or (stacked) wp[i][M][j][planes][Cp]
void launch_pack_weights(const float* w, void* wp, int M, int k, int C, int Cp, int planes, cudaStream_t s,
                         bool stacked = false, const int* sexp = nullptr);
// x NCHW -> patches[n p q][planes][Kp], K index (i*k+j)*C + c  (conv_im2.cpp:19-54 order)
void launch_im2col_split(const float* x, void* pm, int N, int C, int H, int W, int k, int pad, int stride,
                         int P, int Q, int Kp, int planes, cudaStream_t s);
// inter[(t*M+m)][N*H*W] -> y NCHW (P x Q)
void launch_shift_add_row(const float* inter, float* y, int N, int M, int H, int W, int k, int pad, int P,
                          int Q, cudaStream_t s);
// inter[N*H*W][k*k*M] -> y NCHW
void launch_shift_add_col(const float* inter, float* y, int N, int M, int H, int W, int k, int pad, int P,
                          int Q, cudaStream_t s);

// direct fp32 convolution for tiny-C layers (direct.cu); weights MKKC, stride 1
// w_param (optional): host copy of the weights packed [c][i][j][m] for the parameter-weight
// kernel (direct_param_shape: C = 3, k = 3, M in {16, 32, 64}, Q % 4 == 0)
void launch_direct_conv(const float* x, const float* w, float* y, int N, int C, int H, int W, int M, int k, int pad,
                        int stride, int P, int Q, cudaStream_t s, const float* w_param = nullptr);
bool direct_param_shape(int C, int k, int M, int stride, int Q);
size_t direct_smem_bytes(int C, int k);
bool direct_fast_path(int C, int k, int stride);   // else the generic loop nest

void launch_fill_uniform(float* d, unsigned long long n, unsigned long long seed,
                         unsigned long long first, cudaStream_t s);

// ---- tcgen05 engine (tc_conv.cu) ---------------------------------------------------------
struct Operand {
    int mode = LOAD_TILED;   // LOAD_TILED: 3-D map (K=planes*Kp, rows, taps); LOAD_IM2COL: NHWC 4-D
    const void* ptr = nullptr;
    long long rows = 0;      // tiled: rows of the map
    int taps = 1;            // tiled: 3rd dim
    long long tap_stride_rows = 0;   // tiled: rows between 3rd-dim slices (0 = rows; < rows = overlapping view)
    int kw = 0;              // elements per row: 2*Cp (split formats) or Cp (TF32, BF16)
    int planes = 2;          // precision mode (see k_granule)
    // im2col only
    int n = 0, h = 0, w = 0, k = 1, pad = 0;
};

void encode_operand_map(CUtensorMap* map, const Operand& op, int box_rows, int box_taps = 1);
// a plain (unswizzled) tiled map: the TMA-store output of the tensor-core direct kernel
void encode_tiled_map(CUtensorMap* map, CUtensorMapDataType dt, int rank, void* ptr, const cuuint64_t* dims,
                      const cuuint64_t* strides, const cuuint32_t* box, const cuuint32_t* estr);

// ---- tensor-core direct kernel for tiny-C layers (tc_direct.cu) ----------------------------
// C k^2 <= 32 (C = 1..3 at k = 3, C = 1 at k = 5), stride 1, same padding, M in {16..64} % 16,
// P Q % 128 == 0.  wpack: [M][32 words] fp16-split rows of the MKKC weights (K index (i k + j) C + c,
// zero-padded to 32) scaled by 2^ew; sexp = the plan's exponent slots [ew, ex].
bool tc_direct_shape(int C, int k, int M, int stride, int pad, int P, int Q);
// max_sms > 0 caps the grid (cl_conv_set_max_sms: concurrent layers)
void launch_tc_direct(const float* x, const void* wpack, float* y, int N, int C, int H, int W, int M, int k, int pad,
                      int P, int Q, const int* sexp, cudaStream_t s, int max_sms = 0);
// p.partials / p.flags must point at tc_scratch_bytes() of device scratch (stream-K fixup).
// returns the kernels launched: 1, or 2 when a requested fused prepass ran standalone instead
int launch_tc(const Operand& a, const Operand& b, TcParams p, cudaStream_t s, int cta_group = 1);
constexpr int kMaxGrid = kMaxUnits;   // >= SM count (148 on B200)
constexpr int kMaxSplit = 10;   // max stream-K pieces per tile (latency-bound problems)
size_t tc_scratch_bytes();
// carve the stream-K scratch out of a workspace pointer
inline void set_scratch(TcParams& t, void* scratch) {
    t.partials = static_cast<float*>(scratch);
    t.flags = reinterpret_cast<unsigned*>(static_cast<char*>(scratch) + (size_t)kMaxGrid * kTileM * 256 * sizeof(float));
}
int num_sms();

}  // namespace clb
