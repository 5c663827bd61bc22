// facade.cpp -- C++ host code over the C ABI (see include/convlab_b200.hpp).  Pure host
// logic: name mapping, descriptor translation, ownership, error mapping.  All device work
// goes through cl_* entry points.
#include "convlab_b200.hpp"

#include <stdexcept>
#include <utility>

#define CLB_EXPORT __attribute__((visibility("default")))

namespace convlab_b200 {

namespace {

struct NameEntry {
    ConvMethod method;
    const char* name;
};

constexpr NameEntry kNames[] = {
    {ConvMethod::DirectSum, "direct-sum"},
    {ConvMethod::DirectLoopnest, "direct-loopnest"},
    {ConvMethod::Im2col, "im2col"},
    {ConvMethod::Im2row, "im2row"},
    {ConvMethod::Kn2row, "kn2row"},
    {ConvMethod::Kn2col, "kn2col"},
    {ConvMethod::Conv1x1, "conv1x1"},
    {ConvMethod::Kn2rowGpu, "kn2row-gpu"},
    {ConvMethod::Kn2rowExplicitGpu, "kn2row-explicit-gpu"},
    {ConvMethod::Kn2colGpu, "kn2col-gpu"},
    {ConvMethod::Kn2rowAccGpu, "kn2row-acc-gpu"},
    {ConvMethod::Im2colGpu, "im2col-gpu"},
    {ConvMethod::Conv1x1Gpu, "conv1x1-gpu"},
    {ConvMethod::Auto, "auto"},
    {ConvMethod::DirectGpu, "direct-gpu"},
    {ConvMethod::Im2rowGpu, "im2row-gpu"},
};

void check(cl_status s) {
    if (s == CL_OK) return;
    const std::string msg = cl_last_error();
    if (s == CL_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("[cl_status " + std::to_string(static_cast<int>(s)) + "] " + msg);
}

cl_method to_cl(ConvMethod m) {
    switch (m) {
        case ConvMethod::Kn2rowGpu: return CL_METHOD_KN2ROW;
        case ConvMethod::Kn2rowExplicitGpu: return CL_METHOD_KN2ROW_EXPLICIT;
        case ConvMethod::Kn2colGpu: return CL_METHOD_KN2COL;
        case ConvMethod::Kn2rowAccGpu: return CL_METHOD_KN2ROW_ACC;
        case ConvMethod::Im2colGpu: return CL_METHOD_IM2COL;
        case ConvMethod::Conv1x1Gpu: return CL_METHOD_CONV1X1;
        case ConvMethod::Auto: return CL_METHOD_AUTO;
        case ConvMethod::DirectGpu: return CL_METHOD_DIRECT;
        case ConvMethod::Im2rowGpu: return CL_METHOD_IM2ROW;
        default:
            throw std::invalid_argument("method '" + std::string(to_string(m)) +
                                        "' is a reference CPU method; the B200 path runs GPU methods only");
    }
}

ConvMethod from_cl(cl_method m) {
    switch (m) {
        case CL_METHOD_KN2ROW: return ConvMethod::Kn2rowGpu;
        case CL_METHOD_KN2ROW_EXPLICIT: return ConvMethod::Kn2rowExplicitGpu;
        case CL_METHOD_KN2COL: return ConvMethod::Kn2colGpu;
        case CL_METHOD_KN2ROW_ACC: return ConvMethod::Kn2rowAccGpu;
        case CL_METHOD_IM2COL: return ConvMethod::Im2colGpu;
        case CL_METHOD_CONV1X1: return ConvMethod::Conv1x1Gpu;
        case CL_METHOD_DIRECT: return ConvMethod::DirectGpu;
        case CL_METHOD_IM2ROW: return ConvMethod::Im2rowGpu;
        default: return ConvMethod::Auto;
    }
}

cl_conv_desc to_desc(const LayerConfig& l) {
    cl_conv_desc d{};
    d.n = static_cast<int32_t>(l.batch);
    d.c = static_cast<int32_t>(l.channels);
    d.h = static_cast<int32_t>(l.height);
    d.w = static_cast<int32_t>(l.width);
    d.m = static_cast<int32_t>(l.kernel_count);
    d.k = static_cast<int32_t>(l.kernel_size);
    d.pad = l.pad;
    d.stride = static_cast<int32_t>(l.stride);
    return d;
}

}  // namespace

CLB_EXPORT std::string_view to_string(ConvMethod method) {
    for (const auto& e : kNames)
        if (e.method == method) return e.name;
    return "unknown";
}

CLB_EXPORT std::optional<ConvMethod> method_from_name(std::string_view name) {
    for (const auto& e : kNames)
        if (name == e.name) return e.method;
    return std::nullopt;
}

// methods.cpp:43-61 (same grammar and error texts)
CLB_EXPORT std::vector<ConvMethod> parse_method_list(std::string_view csv) {
    std::vector<ConvMethod> out;
    std::size_t pos = 0;
    while (pos <= csv.size()) {
        const std::size_t comma = csv.find(',', pos);
        const std::string_view item =
            csv.substr(pos, comma == std::string_view::npos ? csv.size() - pos : comma - pos);
        if (!item.empty()) {
            const auto m = method_from_name(item);
            if (!m) throw std::invalid_argument("unknown method '" + std::string(item) + "'");
            out.push_back(*m);
        }
        if (comma == std::string_view::npos) break;
        pos = comma + 1;
    }
    if (out.empty()) throw std::invalid_argument("empty method list");
    return out;
}

CLB_EXPORT bool method_requires_1x1(ConvMethod m) { return m == ConvMethod::Conv1x1 || m == ConvMethod::Conv1x1Gpu; }

CLB_EXPORT bool is_gpu_method(ConvMethod m) { return static_cast<int>(m) >= static_cast<int>(ConvMethod::Kn2rowGpu); }  // incl. Auto, DirectGpu

CLB_EXPORT const std::vector<ConvMethod>& default_gpu_methods() {
    static const std::vector<ConvMethod> all = {ConvMethod::Kn2rowGpu, ConvMethod::Kn2rowExplicitGpu,
                                                ConvMethod::Kn2colGpu, ConvMethod::Kn2rowAccGpu,
                                                ConvMethod::Im2colGpu, ConvMethod::Im2rowGpu,
                                                ConvMethod::DirectGpu};
    return all;
}

// bench.cpp:58-85 closed forms, per image.  The implicit / accumulating GPU kernels
// materialise no intermediate.
CLB_EXPORT FootprintBytes footprint(const LayerConfig& l, ConvMethod m) {
    const std::uint64_t c = l.channels, h = l.height, w = l.width, mm = l.kernel_count, k = l.kernel_size;
    FootprintBytes fp;
    fp.input_bytes = 4 * c * h * w;
    fp.kernel_bytes = 4 * mm * k * k * c;
    fp.output_bytes = 4 * mm * h * w;
    switch (m) {
        case ConvMethod::Im2col:
        case ConvMethod::Im2row:
        case ConvMethod::Im2colGpu:
        case ConvMethod::Im2rowGpu:
            fp.intermediate_bytes = 4 * k * k * c * h * w;
            break;
        case ConvMethod::Kn2row:
        case ConvMethod::Kn2col:
        case ConvMethod::Kn2rowExplicitGpu:
        case ConvMethod::Kn2colGpu:
            fp.intermediate_bytes = 4 * k * k * mm * h * w;
            break;
        default:
            fp.intermediate_bytes = 0;
    }
    return fp;
}

CLB_EXPORT Plan::Plan(const LayerConfig& layer, ConvMethod method, Precision precision, int device)
    : layer_(layer) {
    const cl_conv_desc d = to_desc(layer);
    check(cl_conv_plan(&d, to_cl(method),
                       precision == Precision::Fp32 ? CL_PREC_FP32 : (precision == Precision::Bf16 ? CL_PREC_BF16 : CL_PREC_TF32), device,
                       &plan_));
    int32_t p = 0, q = 0;
    check(cl_conv_output_dims(plan_, &p, &q));
    out_h_ = static_cast<std::size_t>(p);
    out_w_ = static_cast<std::size_t>(q);
}

CLB_EXPORT Plan::~Plan() { cl_conv_destroy(plan_); }

CLB_EXPORT Plan::Plan(Plan&& o) noexcept
    : plan_(std::exchange(o.plan_, nullptr)), layer_(std::move(o.layer_)), out_h_(o.out_h_), out_w_(o.out_w_) {}

CLB_EXPORT Plan& Plan::operator=(Plan&& o) noexcept {
    if (this != &o) {
        cl_conv_destroy(plan_);
        plan_ = std::exchange(o.plan_, nullptr);
        layer_ = std::move(o.layer_);
        out_h_ = o.out_h_;
        out_w_ = o.out_w_;
    }
    return *this;
}

CLB_EXPORT ConvMethod Plan::resolved_method() const { return from_cl(cl_conv_resolved_method(plan_)); }

CLB_EXPORT std::size_t Plan::workspace_bytes() const { return cl_conv_workspace_bytes(plan_); }

CLB_EXPORT void Plan::set_weights_device(const float* d_w, void* stream) { check(cl_conv_set_weights(plan_, d_w, stream)); }

CLB_EXPORT void Plan::set_weights_host(const float* h_w, void* stream) {
    check(cl_conv_set_weights_host(plan_, h_w, stream));
}

CLB_EXPORT void Plan::forward_device(const float* d_x, float* d_y, void* d_ws, void* stream) {
    check(cl_conv_forward(plan_, d_x, d_y, d_ws, stream));
}

CLB_EXPORT void Plan::forward_device_nhwc(const float* d_x, float* d_y, void* d_ws, void* stream) {
    check(cl_conv_forward_nhwc(plan_, d_x, d_y, d_ws, stream));
}

CLB_EXPORT void Plan::forward_host_async(const float* h_x, float* h_y, void* stream) {
    check(cl_conv_forward_host_async(plan_, h_x, h_y, stream));
}

CLB_EXPORT std::vector<float> Plan::forward_host(const float* h_x, void* stream) {
    std::vector<float> y(layer_.batch * layer_.kernel_count * out_h_ * out_w_);
    check(cl_conv_forward_host(plan_, h_x, y.data(), stream));
    return y;
}

// methods.cpp:65-88, GPU edition.
CLB_EXPORT std::vector<float> run_method(ConvMethod method, const LayerConfig& layer, const float* x_host,
                                         const float* w_host, Precision precision) {
    if (method_requires_1x1(method) && layer.kernel_size != 1)
        throw std::invalid_argument("conv1x1 requires a 1x1 kernel, got k = " + std::to_string(layer.kernel_size));
    ConvMethod m = method;
    if (layer.kernel_size == 1 && (m == ConvMethod::Kn2rowGpu || m == ConvMethod::Kn2colGpu ||
                                   m == ConvMethod::Kn2rowExplicitGpu))
        m = ConvMethod::Conv1x1Gpu;
    Plan plan(layer, m, precision);
    plan.set_weights_host(w_host);
    return plan.forward_host(x_host);
}

}  // namespace convlab_b200
