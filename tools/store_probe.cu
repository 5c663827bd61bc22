// store_probe.cu -- NCHW epilogue store patterns at the engine's shape: 148 persistent CTAs, 8
// storing warps, each thread owning one pixel row x COLS channels of a 128-pixel tile.
//   mode 0: the engine's pattern -- per channel one 4-byte store per thread (a warp writes 128 B
//           of one channel plane per instruction)
//   mode 1: 4x4 lane transposes (shuffles) then 16-byte stores -- lane l writes pixels 4(l/4)..+3
//           of channel 4jj + l%4 (a warp writes 4 x 128 B per instruction, 4x fewer instructions)
//   mode 2: mode 0 with streaming stores (st.global.cs)
// Reports GB/s of output written and B/clk/SM.   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 store_probe.cu -o store_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

template <int COLS, int MODE>
__global__ void __launch_bounds__(256, 1) probe(float* __restrict__ out, int n_img, int M, long long PQ, int tiles_per_img) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int quad = warp & 3, half = warp >> 2;          // 4 lane quadrants x 2 column halves
    const int total = n_img * tiles_per_img;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int n = t / tiles_per_img;
        const long long pix = (long long)(t - n * tiles_per_img) * 128 + quad * 32 + lane;
        float v[COLS];
#pragma unroll
        for (int j = 0; j < COLS; ++j) v[j] = (float)(t + j) * 0.5f + lane;
        float* o = out + ((long long)n * M + half * COLS) * PQ;
        if (MODE == 0 || MODE == 2) {
#pragma unroll
            for (int j = 0; j < COLS; ++j) {
                if (MODE == 0) o[(long long)j * PQ + pix] = v[j];
                else __stcs(o + (long long)j * PQ + pix, v[j]);
            }
        } else {
            const long long pix4 = (long long)(t - n * tiles_per_img) * 128 + quad * 32 + (lane >> 2) * 4;
#pragma unroll
            for (int j = 0; j < COLS; j += 4) {
                float a0 = v[j], a1 = v[j + 1], a2 = v[j + 2], a3 = v[j + 3];
                // 4x4 transpose across lanes l^1, l^2: afterwards lane i (= l%4) holds channel j+i of pixels 0..3
                float x0 = (lane & 1) ? a0 : a1, x1 = (lane & 1) ? a2 : a3;
                x0 = __shfl_xor_sync(0xffffffffu, x0, 1); x1 = __shfl_xor_sync(0xffffffffu, x1, 1);
                if (lane & 1) { a0 = x0; a2 = x1; } else { a1 = x0; a3 = x1; }
                x0 = (lane & 2) ? a0 : a2; x1 = (lane & 2) ? a1 : a3;
                x0 = __shfl_xor_sync(0xffffffffu, x0, 2); x1 = __shfl_xor_sync(0xffffffffu, x1, 2);
                if (lane & 2) { a0 = x0; a1 = x1; } else { a2 = x0; a3 = x1; }
                *reinterpret_cast<float4*>(o + (long long)(j + (lane & 3)) * PQ + pix4) = make_float4(a0, a1, a2, a3);
            }
        }
    }
}

template <int COLS, int MODE>
void run(const char* name, float* out, int n_img, int M, int H) {
    const long long PQ = (long long)H * H;
    const int tiles = (int)(PQ / 128);
    cudaEvent_t b, e; cudaEventCreate(&b); cudaEventCreate(&e);
    probe<COLS, MODE><<<148, 256>>>(out, n_img, M, PQ, tiles);
    cudaEventRecord(b);
    for (int i = 0; i < 5; ++i) probe<COLS, MODE><<<148, 256>>>(out, n_img, M, PQ, tiles);
    cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, b, e); ms /= 5;
    const double bytes = (double)n_img * tiles * 128 * 2 * COLS * 4;
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-28s H=%3d M=%3d cols/thread=%3d: %s  %.3f ms  %.0f GB/s  %.2f B/clk/SM (at %d MHz)\n", name, H, M, COLS,
           cudaGetErrorString(cudaGetLastError()), ms, bytes / ms / 1e6, bytes / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
}

int main() {
    float* out; cudaMalloc(&out, (size_t)32 * 64 * 224 * 224 * 4 + (1 << 20));
    run<32, 0>("st.32 per channel", out, 32, 64, 224);
    run<32, 1>("shuffle + st.128", out, 32, 64, 224);
    run<32, 2>("st.32.cs per channel", out, 32, 64, 224);
    run<64, 0>("st.32 per channel", out, 32, 128, 112);
    run<64, 1>("shuffle + st.128", out, 32, 128, 112);
    run<128, 0>("st.32 per channel", out, 32, 256, 56);
    run<128, 1>("shuffle + st.128", out, 32, 256, 56);
    run<128, 0>("st.32 per channel", out, 64, 256, 16);   // small planes (L2-resident output)
    run<128, 1>("shuffle + st.128", out, 64, 256, 16);
    return 0;
}
