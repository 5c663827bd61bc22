// convlab_b200_ref.hpp -- OPTIONAL: the B200 path at the reference's own operator signature.
//
//   reference:  convlab::Tensor3 convlab::run_method(ConvMethod, const ConvProblem&, const GemmBackend&)
//               (include/convlab/methods.hpp:40, src/methods.cpp:65-88)
//   here:       convlab::Tensor3 convlab_b200::run_method(convlab::ConvMethod, const convlab::ConvProblem&,
//                                                         const convlab::GemmBackend&)
//
// Include it where the reference headers (convlab/methods.hpp) are on the include path; a
// reference caller then switches by namespace only -- same arguments, same result type,
// same k == 1 routing and the same std::invalid_argument for conv1x1 on k != 1 problems:
//
//     convlab::Tensor3 y = convlab_b200::run_method(convlab::ConvMethod::Kn2row, problem, backend);
//
// Each reference method runs as the GPU method computing the same convolution:
//   Kn2row -> kn2row-gpu (implicit; shift-add folded into the tcgen05 accumulator)
//   Kn2col -> kn2col-gpu, Im2col -> im2col-gpu, Im2row -> im2row-gpu, Conv1x1 -> conv1x1-gpu
//   DirectSum / DirectLoopnest -> direct-gpu (fp32 CUDA-core loop nest)
// The GemmBackend argument is accepted for signature compatibility: the contraction always
// runs on the B200 engine (its fp32-faithful split is held to the reference's allclose, as the
// reference holds external backends, gemm.hpp:13-16).  Input may be CHW or HWC (converted to
// CHW first, as conv_kn2row does, conv_kn2.cpp:147-151); kernels MKKC or MCKK; the result is a
// CHW Tensor3 like every reference method's.  A convlab_b200::ConvMethod overload takes the GPU
// methods (and `Auto`) directly.
#pragma once

#include <string>
#include <vector>

#include "convlab/methods.hpp"
#include "convlab/tensor.hpp"
#include "convlab_b200.hpp"

namespace convlab_b200 {

inline ConvMethod gpu_method_for(convlab::ConvMethod m) {
    switch (m) {
        case convlab::ConvMethod::DirectSum:
        case convlab::ConvMethod::DirectLoopnest: return ConvMethod::DirectGpu;
        case convlab::ConvMethod::Im2col: return ConvMethod::Im2colGpu;
        case convlab::ConvMethod::Im2row: return ConvMethod::Im2rowGpu;
        case convlab::ConvMethod::Kn2row: return ConvMethod::Kn2rowGpu;
        case convlab::ConvMethod::Kn2col: return ConvMethod::Kn2colGpu;
        case convlab::ConvMethod::Conv1x1: return ConvMethod::Conv1x1Gpu;
    }
    throw std::logic_error("unreachable method");
}

inline convlab::Tensor3 run_method(ConvMethod method, const convlab::ConvProblem& p,
                                   const convlab::GemmBackend& /*backend*/ = convlab::GemmBackend::blocked(),
                                   Precision precision = Precision::Fp32) {
    const std::size_t C = p.channels(), H = p.height(), W = p.width(), M = p.kernel_count(), k = p.kernel_size();
    // input as one CHW image (the reference's HWC inputs are converted first)
    std::vector<float> x(C * H * W);
    const convlab::Tensor3& in = p.input();
    if (in.layout() == convlab::Layout::CHW) {
        const auto d = in.data();
        x.assign(d.begin(), d.end());
    } else {
        for (std::size_t c = 0; c < C; ++c)
            for (std::size_t h = 0; h < H; ++h)
                for (std::size_t w = 0; w < W; ++w) x[(c * H + h) * W + w] = in.at(c, h, w);
    }
    // kernels as MKKC (the MCKK storage is permuted; MKKC is used as is)
    std::vector<float> wk(M * k * k * C);
    const convlab::KernelSet& ks = p.kernels();
    if (ks.layout() == convlab::KernelLayout::MKKC) {
        const auto d = ks.data();
        wk.assign(d.begin(), d.end());
    } else {
        for (std::size_t m = 0; m < M; ++m)
            for (std::size_t i = 0; i < k; ++i)
                for (std::size_t j = 0; j < k; ++j)
                    for (std::size_t c = 0; c < C; ++c) wk[((m * k + i) * k + j) * C + c] = ks.at(m, i, j, c);
    }
    LayerConfig layer{"run_method", C, H, W, M, k};
    // convlab_b200::run_method applies the reference's k == 1 routing and conv1x1 contract
    std::vector<float> y = run_method(method, layer, x.data(), wk.data(), precision);
    return convlab::Tensor3(M, H, W, convlab::Layout::CHW, std::move(y));
}

inline convlab::Tensor3 run_method(convlab::ConvMethod method, const convlab::ConvProblem& p,
                                   const convlab::GemmBackend& backend = convlab::GemmBackend::blocked(),
                                   Precision precision = Precision::Fp32) {
    return run_method(gpu_method_for(method), p, backend, precision);
}

}  // namespace convlab_b200
