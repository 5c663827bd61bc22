/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference ("convlab", /root/reference/proj) algorithms on the
 * kn2row / im2col hot path.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker: the product path
 * (paper_1704_04428_b200/, libconvlab_b200.so) never links or calls it.
 *
 * Parity is PINNED two ways (tests/test_oracle.py):
 *   - against the reference's own golden vectors (tensor_test.cpp:131-139 seed-0 bits,
 *     conv_kn2_test.cpp:126-132 shift-add counts, conv_direct_test.cpp:42-49 SCSK grid,
 *     conv_im2_test.cpp:31-47 patch columns, tests/data/golden_bench_columns.csv);
 *   - bitwise against the reference library itself compiled from /root/reference into
 *     oracle/_ref/libconvlab_ref.so (oracle/Makefile), plus fixtures in tests/golden/.
 *
 * Every function keeps the reference's per-element accumulation order so that the
 * restated oracle is bit-identical to the reference when compiled with
 * -ffp-contract=off (the reference's own flag, core/CMakeLists.txt:19-21).
 * Layouts: CHW images (c*H+h)*W+w (tensor.hpp:86-90), MKKC kernels
 * ((m*k+i)*k+j)*C+c (tensor.hpp:120-125), row-major matrices (tensor.hpp:33-40).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ---- counter-based generator: tensor.cpp:104-131 ------------------------------- */

static const uint64_t kGamma = 0x9E3779B97F4A7C15ull;      /* tensor.cpp:105 */
static const uint64_t kSplitGamma = 0xD1B54A32D192ED03ull; /* tensor.cpp:106 */

ORC_API uint64_t orc_mix64(uint64_t z) { /* tensor.cpp:111-115 (splitmix64 finaliser) */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

ORC_API float orc_unit_value(uint64_t seed, uint64_t index) { /* tensor.cpp:117-123 */
    const uint64_t bits = orc_mix64(seed + (index + 1) * kGamma);
    const uint32_t top = (uint32_t)(bits >> 40);
    return (float)top * 0x1p-23f - 1.0f;
}

ORC_API uint64_t orc_split(uint64_t seed, uint64_t lane) { /* tensor.cpp:125-127 */
    return orc_mix64(seed + (lane + 1) * kSplitGamma);
}

/* fill_deterministic (tensor.cpp:131-134), with an index offset so a batch buffer can be
 * filled in independent slices that are bit-identical to one whole-buffer fill. */
ORC_API void orc_fill(float* out, uint64_t n, uint64_t seed, uint64_t first_index) {
#pragma omp parallel for schedule(static) if (n > (1u << 20))
    for (int64_t i = 0; i < (int64_t)n; ++i) out[i] = orc_unit_value(seed, first_index + (uint64_t)i);
}

/* fnv1a over float bit patterns, byte order low..high: bench.cpp:25-36 */
ORC_API uint64_t orc_fnv1a(const float* data, uint64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t bits;
        memcpy(&bits, &data[i], 4);
        for (int s = 0; s < 32; s += 8) {
            h ^= (bits >> s) & 0xffu;
            h *= 0x100000001b3ull;
        }
    }
    return h;
}

/* ---- direct methods: conv_direct.cpp ------------------------------------------- */

/* conv2d_scsk (conv_direct.cpp:23-55): single plane, same padding, no flip; i outer,
 * j inner, OOB taps skipped. */
static void scsk(const float* img, int H, int W, const float* ker, int k, float* out) {
    const int half = k / 2;
    for (int x = 0; x < H; ++x) {
        for (int y = 0; y < W; ++y) {
            float acc = 0.0f;
            for (int i = 0; i < k; ++i) {
                const int sx = x - half + i;
                if (sx < 0 || sx >= H) continue;
                for (int j = 0; j < k; ++j) {
                    const int sy = y - half + j;
                    if (sy < 0 || sy >= W) continue;
                    acc += img[sx * W + sy] * ker[i * k + j];
                }
            }
            out[x * W + y] = acc;
        }
    }
}

ORC_API void orc_conv2d_scsk(const float* img, int H, int W, const float* ker, int k, float* out) {
    scsk(img, H, W, ker, k, out);
}

/* conv_mcmk_sum (conv_direct.cpp:93-102) -> conv_mcsk (57-91) -> conv2d_scsk (23-55).
 * Output channel m: out = 0; for c ascending: out += scsk(plane c, kernel (m,c)).
 * THE ORACLE. Parallel over m only, which leaves every element's arithmetic intact. */
ORC_API void orc_conv_mcmk_sum(const float* x, const float* w_mkkc, float* y, int C, int H, int W,
                               int M, int k) {
    const size_t plane = (size_t)H * W;
#pragma omp parallel for schedule(dynamic) if ((size_t)M * C * plane * k * k > (1u << 22))
    for (int m = 0; m < M; ++m) {
        float* out = y + (size_t)m * plane;
        float* chan = (float*)malloc(plane * sizeof(float));
        float ker[121 * 1];
        float* kbuf = (k * k <= 121) ? ker : (float*)malloc((size_t)k * k * sizeof(float));
        for (size_t e = 0; e < plane; ++e) out[e] = 0.0f;
        for (int c = 0; c < C; ++c) {
            for (int i = 0; i < k; ++i)
                for (int j = 0; j < k; ++j)
                    kbuf[i * k + j] = w_mkkc[(((size_t)m * k + i) * k + j) * C + c];
            scsk(x + (size_t)c * plane, H, W, kbuf, k, chan);
            for (size_t e = 0; e < plane; ++e) out[e] += chan[e];
        }
        if (kbuf != ker) free(kbuf);
        free(chan);
    }
}

/* conv_mcmk_loopnest (conv_direct.cpp:104-143) generalised to explicit pad and stride
 * (the reference fixes pad = k/2, stride = 1; SURVEY.md 8c "coverage gaps").  Output size
 * P = (H + 2 pad - k)/stride + 1.  At pad = k/2, stride 1 this is the reference loop nest
 * verbatim (h, w, o, x, y, i order).  Batched over n. */
ORC_API void orc_conv_loopnest(const float* x, const float* w_mkkc, float* y, int N, int C, int H,
                               int W, int M, int k, int pad, int stride) {
    const int P = (H + 2 * pad - k) / stride + 1;
    const int Q = (W + 2 * pad - k) / stride + 1;
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int n = 0; n < N; ++n) {
        for (int h = 0; h < P; ++h) {
            const float* xn = x + (size_t)n * C * H * W;
            float* yn = y + (size_t)n * M * P * Q;
            for (int w = 0; w < Q; ++w) {
                for (int o = 0; o < M; ++o) {
                    float sum = 0.0f;
                    for (int a = 0; a < k; ++a) {
                        const int sh = h * stride - pad + a;
                        if (sh < 0 || sh >= H) continue;
                        for (int b = 0; b < k; ++b) {
                            const int sw = w * stride - pad + b;
                            if (sw < 0 || sw >= W) continue;
                            for (int i = 0; i < C; ++i)
                                sum += xn[((size_t)i * H + sh) * W + sw] *
                                       w_mkkc[(((size_t)o * k + a) * k + b) * C + i];
                        }
                    }
                    yn[((size_t)o * P + h) * Q + w] = sum;
                }
            }
        }
    }
}

/* ---- GEMM: gemm.cpp ----------------------------------------------------------- */

/* gemm_reference (gemm.cpp:82-94): c(r,col) = sum_t a(r,t) b(t,col), t ascending. */
ORC_API void orc_gemm_ref(const float* a, const float* b, float* c, int m, int p, int n) {
#pragma omp parallel for schedule(static) if ((size_t)m * n * p > (1u << 22))
    for (int r = 0; r < m; ++r)
        for (int col = 0; col < n; ++col) {
            float acc = 0.0f;
            for (int t = 0; t < p; ++t) acc += a[(size_t)r * p + t] * b[(size_t)t * n + col];
            c[(size_t)r * n + col] = acc;
        }
}

/* ---- kn2 methods: conv_kn2.cpp ------------------------------------------------- */

/* kn2row_reorder_kernel (conv_kn2.cpp:28-39): R[(i*k+j)*M+m][c] = K[m,i,j,c]. */
ORC_API void orc_kn2row_reorder(const float* w_mkkc, float* r, int M, int k, int C) {
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
            for (int m = 0; m < M; ++m)
                for (int c = 0; c < C; ++c)
                    r[((size_t)(i * k + j) * M + m) * C + c] =
                        w_mkkc[(((size_t)m * k + i) * k + j) * C + c];
}

/* shift_add, row orientation (conv_kn2.cpp:78-118): intermediate (k^2 M) x (H W) ->
 * out M x (H W); gather, i outer / j inner, OOB skipped; k == 1 is the identity. */
ORC_API void orc_shift_add_row(const float* src, float* out, int k, int M, int H, int W) {
    const size_t pixels = (size_t)H * W;
    const int half = k / 2;
    if (k == 1) {
        memcpy(out, src, (size_t)M * pixels * sizeof(float));
        return;
    }
    for (int m = 0; m < M; ++m)
        for (int x = 0; x < H; ++x)
            for (int y = 0; y < W; ++y) {
                float acc = 0.0f;
                for (int i = 0; i < k; ++i) {
                    const int sx = x + i - half;
                    if (sx < 0 || sx >= H) continue;
                    for (int j = 0; j < k; ++j) {
                        const int sy = y + j - half;
                        if (sy < 0 || sy >= W) continue;
                        acc += src[((size_t)(i * k + j) * M + m) * pixels + (size_t)sx * W + sy];
                    }
                }
                out[(size_t)m * pixels + (size_t)x * W + y] = acc;
            }
}

/* shift_add, col orientation (conv_kn2.cpp:120-142): (H W) x (k^2 M) -> (H W) x M. */
ORC_API void orc_shift_add_col(const float* src, float* out, int k, int M, int H, int W) {
    const size_t ld = (size_t)k * k * M;
    const int half = k / 2;
    if (k == 1) {
        memcpy(out, src, (size_t)M * H * W * sizeof(float));
        return;
    }
    for (int x = 0; x < H; ++x)
        for (int y = 0; y < W; ++y)
            for (int m = 0; m < M; ++m) {
                float acc = 0.0f;
                for (int i = 0; i < k; ++i) {
                    const int sx = x + i - half;
                    if (sx < 0 || sx >= H) continue;
                    for (int j = 0; j < k; ++j) {
                        const int sy = y + j - half;
                        if (sy < 0 || sy >= W) continue;
                        acc += src[((size_t)sx * W + sy) * ld + (size_t)(i * k + j) * M + m];
                    }
                }
                out[((size_t)x * W + y) * M + m] = acc;
            }
}

/* conv_kn2row (conv_kn2.cpp:145-162): reorder -> one GEMM -> shift_add (row).  For k == 1
 * this is conv_1x1 (conv_kn2.cpp:54-76; dispatch methods.cpp:75-77).  Uses the
 * t-ascending GEMM, which is bitwise equal to the reference's blocked GEMM (gemm.hpp:34-47). */
ORC_API void orc_conv_kn2row(const float* x, const float* w_mkkc, float* y, int C, int H, int W,
                             int M, int k) {
    const size_t pixels = (size_t)H * W;
    if (k == 1) {
        orc_gemm_ref(w_mkkc, x, y, M, C, (int)pixels);
        return;
    }
    float* r = (float*)malloc((size_t)k * k * M * C * sizeof(float));
    float* inter = (float*)malloc((size_t)k * k * M * pixels * sizeof(float));
    orc_kn2row_reorder(w_mkkc, r, M, k, C);
    orc_gemm_ref(r, x, inter, k * k * M, C, (int)pixels);
    orc_shift_add_row(inter, y, k, M, H, W);
    free(inter);
    free(r);
}

/* ---- im2col: conv_im2.cpp ------------------------------------------------------ */

/* im2col_patch_matrix (conv_im2.cpp:19-54): P[(i*k+j)*C+c][x*W+y] = X[c][x-h+i][y-h+j],
 * zero when OOB. */
ORC_API void orc_im2col_patch(const float* x, float* pm, int C, int H, int W, int k) {
    const int half = k / 2;
    const size_t pixels = (size_t)H * W;
    memset(pm, 0, (size_t)k * k * C * pixels * sizeof(float));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
            for (int c = 0; c < C; ++c) {
                float* row = pm + ((size_t)(i * k + j) * C + c) * pixels;
                const float* plane = x + (size_t)c * pixels;
                for (int a = 0; a < H; ++a) {
                    const int sx = a - half + i;
                    if (sx < 0 || sx >= H) continue;
                    for (int b = 0; b < W; ++b) {
                        const int sy = b - half + j;
                        if (sy < 0 || sy >= W) continue;
                        row[(size_t)a * W + b] = plane[(size_t)sx * W + sy];
                    }
                }
            }
}

/* conv_im2col (conv_im2.cpp:108-132): MKKC kernels are the M x (k^2 C) matrix (121-123). */
ORC_API void orc_conv_im2col(const float* x, const float* w_mkkc, float* y, int C, int H, int W,
                             int M, int k) {
    const size_t pixels = (size_t)H * W;
    float* pm = (float*)malloc((size_t)k * k * C * pixels * sizeof(float));
    orc_im2col_patch(x, pm, C, H, W, k);
    orc_gemm_ref(w_mkkc, pm, y, M, k * k * C, (int)pixels);
    free(pm);
}

/* ---- tolerance law: tensor.cpp:158-163, 211-213 -------------------------------- */

ORC_API float orc_max_abs(const float* a, uint64_t n) {
    float worst = 0.0f;
    for (uint64_t i = 0; i < n; ++i) worst = fmaxf(worst, fabsf(a[i]));
    return worst;
}

/* allclose(a, b=oracle, scaled_tolerance({rel, abs}, max|oracle|)) as in verify
 * (bench.cpp:191-205).  Returns 1 when every |a-b| <= abs' + rel |b|. */
ORC_API int orc_allclose_scaled(const float* a, const float* b, uint64_t n, float rel, float abs_) {
    const float mag = orc_max_abs(b, n);
    const float abs_scaled = abs_ + rel * (mag > 0.0f ? mag : 0.0f);
    for (uint64_t i = 0; i < n; ++i)
        if (!(fabsf(a[i] - b[i]) <= abs_scaled + rel * fabsf(b[i]))) return 0;
    return 1;
}
