// convlab_b200.hpp -- C++ host facade over the C ABI (convlab_b200.h), mirroring the
// reference's conv-method API so that callers of convlab::run_method switch by name:
//
//   reference (/root/reference/proj/core/include/convlab)    this facade
//   ConvMethod            methods.hpp:15-23                   convlab_b200::ConvMethod (+ GPU enumerators)
//   to_string / method_from_name / parse_method_list          same names, same error text
//                         methods.cpp:11-61
//   method_requires_1x1   methods.cpp:63                      same
//   LayerConfig           layers.hpp:12-22                    same fields + pad, batch
//   run_method            methods.cpp:65-88                   run_method(method, layer, x, w, precision)
//   footprint / FootprintBytes  bench.cpp:58-85               same closed forms
//
// Errors: contract violations throw std::invalid_argument (as the reference does),
// everything else std::runtime_error.  The reference's CPU methods are recognised by name
// but not executed here (the product path is GPU only): run_method throws for them.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

#include "convlab_b200.h"

namespace convlab_b200 {

enum class ConvMethod {
    // reference enumerators, in reference order (methods.hpp:15-23)
    DirectSum,
    DirectLoopnest,
    Im2col,
    Im2row,
    Kn2row,
    Kn2col,
    Conv1x1,
    // B200 methods
    Kn2rowGpu,          // implicit kn2row (north-star kernel)
    Kn2rowExplicitGpu,  // one GEMM + shift-add, paper-faithful
    Kn2colGpu,
    Kn2rowAccGpu,       // k^2 accumulating shifted GEMMs
    Im2colGpu,
    Conv1x1Gpu,
    Auto,
    DirectGpu,          // fp32 CUDA-core direct loop nest (tiny-C first layers)
    Im2rowGpu,          // reference im2row; same K-major patch GEMM as Im2colGpu on the GPU
};

enum class Precision { Fp32, Tf32, Bf16 };

struct LayerConfig {
    std::string name;
    std::size_t channels = 0;      // C
    std::size_t height = 0;        // H
    std::size_t width = 0;         // W
    std::size_t kernel_count = 0;  // M
    std::size_t kernel_size = 0;   // k, odd
    std::size_t stride = 1;
    int pad = -1;                  // -1 = k/2 (the reference's implicit same padding)
    std::size_t batch = 1;         // N

    bool operator==(const LayerConfig&) const = default;
};

struct FootprintBytes {
    std::uint64_t input_bytes = 0;
    std::uint64_t kernel_bytes = 0;
    std::uint64_t intermediate_bytes = 0;
    std::uint64_t output_bytes = 0;
    bool operator==(const FootprintBytes&) const = default;
};

std::string_view to_string(ConvMethod method);
std::optional<ConvMethod> method_from_name(std::string_view name);
std::vector<ConvMethod> parse_method_list(std::string_view csv);
bool method_requires_1x1(ConvMethod method);
bool is_gpu_method(ConvMethod method);
const std::vector<ConvMethod>& default_gpu_methods();

FootprintBytes footprint(const LayerConfig& layer, ConvMethod method);

// One planned layer (owns a cl_plan).  Move-only.
class Plan {
public:
    Plan(const LayerConfig& layer, ConvMethod method, Precision precision = Precision::Fp32, int device = 0);
    ~Plan();
    Plan(Plan&&) noexcept;
    Plan& operator=(Plan&&) noexcept;
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    ConvMethod resolved_method() const;
    std::size_t out_height() const { return out_h_; }
    std::size_t out_width() const { return out_w_; }
    std::size_t workspace_bytes() const;

    void set_weights_device(const float* d_w_mkkc, void* stream = nullptr);
    void set_weights_host(const float* h_w_mkkc, void* stream = nullptr);
    void forward_device(const float* d_x, float* d_y, void* d_ws = nullptr, void* stream = nullptr);
    // channels-last device tensors: x [N][H][W][C], y [N][P][Q][M] (implicit kn2row / conv1x1)
    void forward_device_nhwc(const float* d_x, float* d_y, void* d_ws = nullptr, void* stream = nullptr);
    // host NCHW in / host NCHW out (H2D + forward + D2H)
    std::vector<float> forward_host(const float* h_x, void* stream = nullptr);
    // same, into a caller buffer, returning after enqueueing (synchronise `stream` before use)
    void forward_host_async(const float* h_x, float* h_y, void* stream);

private:
    cl_plan* plan_ = nullptr;
    LayerConfig layer_;
    std::size_t out_h_ = 0, out_w_ = 0;
};

// run_method (methods.cpp:65-88) on host data: x = batch NCHW, w = MKKC.  Applies the
// reference's k == 1 routing (kn2row/kn2col -> conv1x1) and rejects conv1x1 with k != 1.
std::vector<float> run_method(ConvMethod method, const LayerConfig& layer, const float* x_host,
                              const float* w_host, Precision precision = Precision::Fp32);

}  // namespace convlab_b200
