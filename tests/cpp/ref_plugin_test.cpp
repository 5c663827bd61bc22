// ref_plugin_test.cpp -- TEST: the drop-in at the reference's own plugin point.
//
// Registers the B200 GEMM as an external backend of the UNMODIFIED reference library
// (register_gemm_backend, gemm.hpp:52-58; compiled into oracle/_ref) and runs the
// reference's own conv_kn2row / conv_im2col / conv_kn2col (conv_kn2.cpp:145-183,
// conv_im2.cpp:108-132) with it, against the reference oracle conv_mcmk_sum.  The adapter
// below is exactly the binding shown in INTEGRATION.md.  Second part: the reference-signature
// overload convlab_b200::run_method(convlab::ConvMethod, const convlab::ConvProblem&,
// const convlab::GemmBackend&) of include/convlab_b200_ref.hpp (CHW and HWC inputs, MKKC and
// MCKK kernels, the k == 1 routing and the conv1x1 contract).
#include <cstdio>
#include <stdexcept>
#include <cuda_runtime.h>

#include "convlab/conv_direct.hpp"
#include "convlab/conv_im2.hpp"
#include "convlab/conv_kn2.hpp"
#include "convlab/gemm.hpp"
#include "convlab/methods.hpp"
#include "convlab_b200.h"
#include "convlab_b200_ref.hpp"

namespace {

convlab::Matrix b200_gemm(convlab::MatrixView a, convlab::MatrixView b) {
    const std::size_t m = a.rows, k = a.cols, n = b.cols;
    float *da = nullptr, *db = nullptr, *dc = nullptr;
    if (cudaMalloc(&da, m * k * 4) || cudaMalloc(&db, k * n * 4) || cudaMalloc(&dc, m * n * 4))
        throw std::runtime_error("b200 gemm: device allocation failed");
    cudaMemcpy(da, a.data, m * k * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data, k * n * 4, cudaMemcpyHostToDevice);
    const cl_status s = cl_gemm_f32((int)m, (int)n, (int)k, da, db, dc, CL_PREC_FP32, nullptr, 0, nullptr);
    convlab::Matrix c(m, n);
    if (s == CL_OK) cudaMemcpy(c.data().data(), dc, m * n * 4, cudaMemcpyDeviceToHost);
    cudaFree(da);
    cudaFree(db);
    cudaFree(dc);
    if (s != CL_OK) throw std::runtime_error(cl_last_error());
    return c;
}

}  // namespace

int main() {
    convlab::register_gemm_backend("b200", b200_gemm);
    auto backend = convlab::make_backend("b200");
    if (!backend) return 2;
    int fails = 0;
    const struct { std::size_t c, h, w, m, k; } shapes[] = {{3, 6, 5, 4, 3}, {16, 13, 13, 8, 3}, {64, 28, 28, 32, 3},
                                                            {8, 9, 9, 16, 5}, {32, 7, 7, 64, 1}};
    for (const auto& s : shapes) {
        convlab::ConvProblem p(convlab::random_tensor3(s.c, s.h, s.w, convlab::Layout::CHW, convlab::rng::split(5, 0)),
                               convlab::random_kernels(s.m, s.k, s.c, convlab::KernelLayout::MKKC,
                                                       convlab::rng::split(5, 1)));
        const convlab::Tensor3 oracle = convlab::conv_mcmk_sum(p);
        const auto tol = convlab::scaled_tolerance({1e-5f, 1e-6f}, convlab::max_abs(oracle));
        for (auto m : {convlab::ConvMethod::Kn2row, convlab::ConvMethod::Kn2col, convlab::ConvMethod::Im2col,
                       convlab::ConvMethod::Im2row}) {
            const convlab::Tensor3 out = convlab::run_method(m, p, *backend);
            const bool ok = convlab::allclose(out, oracle, tol);
            std::printf("  ref %-8s via b200 GEMM  C=%zu %zux%zu M=%zu k=%zu  max|err|=%.3e  %s\n",
                        std::string(convlab::to_string(m)).c_str(), s.c, s.h, s.w, s.m, s.k,
                        convlab::max_abs_diff(out, oracle), ok ? "ok" : "FAIL");
            fails += !ok;
        }
    }
    // ---- the reference signature, served by the B200 path ----
    for (const auto& s : shapes) {
        for (int variant = 0; variant < 2; ++variant) {
            const auto lay = variant ? convlab::Layout::HWC : convlab::Layout::CHW;
            const auto klay = variant ? convlab::KernelLayout::MCKK : convlab::KernelLayout::MKKC;
            convlab::ConvProblem p(convlab::random_tensor3(s.c, s.h, s.w, lay, convlab::rng::split(6, 0)),
                                   convlab::random_kernels(s.m, s.k, s.c, klay, convlab::rng::split(6, 1)));
            const convlab::Tensor3 oracle = convlab::conv_mcmk_sum(p);
            const auto tol = convlab::scaled_tolerance({1e-5f, 1e-6f}, convlab::max_abs(oracle));
            for (auto m : convlab::default_methods()) {
                const convlab::Tensor3 out = convlab_b200::run_method(m, p, *backend);
                const bool ok = out.layout() == convlab::Layout::CHW && convlab::allclose(out, oracle, tol);
                std::printf("  b200 run_method(%-15s %s/%s) C=%zu %zux%zu M=%zu k=%zu  max|err|=%.3e  %s\n",
                            std::string(convlab::to_string(m)).c_str(), variant ? "HWC" : "CHW",
                            variant ? "MCKK" : "MKKC", s.c, s.h, s.w, s.m, s.k, convlab::max_abs_diff(out, oracle),
                            ok ? "ok" : "FAIL");
                fails += !ok;
            }
            bool threw = false;
            try {
                (void)convlab_b200::run_method(convlab::ConvMethod::Conv1x1, p, *backend);
            } catch (const std::invalid_argument&) {
                threw = true;
            }
            if ((s.k != 1) != threw) {
                std::printf("  conv1x1 contract violated for k=%zu\n", s.k);
                ++fails;
            }
        }
    }
    std::printf(fails ? "FAILED (%d)\n" : "PASSED\n", fails);
    return fails ? 1 : 0;
}
