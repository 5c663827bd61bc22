// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" binding over the UNMODIFIED reference library (convlab core, compiled
// from its sources where they lie under /root/reference/proj/core by oracle/Makefile into
// oracle/_ref/libconvlab_ref.so).  Used (a) by tests/ to pin the oracle restatement
// (oracle/oracle.c) bitwise against the reference itself, and (b) by bench.py
// `--impl reference` / `cpu_baseline` to time the reference's own CPU kn2row / im2col
// path through its public API (convlab::benchmark, bench.cpp:87-151; run_method,
// methods.cpp:65-88).  Nothing on the product path links this.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "convlab/bench.hpp"
#include "convlab/conv_direct.hpp"
#include "convlab/conv_im2.hpp"
#include "convlab/conv_kn2.hpp"
#include "convlab/gemm.hpp"
#include "convlab/methods.hpp"
#include "convlab/tensor.hpp"

namespace {

thread_local std::string g_err;

convlab::GemmBackend backend_for(int threads) {
    if (threads <= 0) return convlab::GemmBackend::blocked();
    return convlab::GemmBackend::parallel(static_cast<std::size_t>(threads));
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) const char* ref_last_error() { return g_err.c_str(); }

__attribute__((visibility("default"))) float ref_unit_value(std::uint64_t seed, std::uint64_t i) {
    return convlab::rng::unit_value(seed, i);
}

__attribute__((visibility("default"))) std::uint64_t ref_split(std::uint64_t seed, std::uint64_t lane) {
    return convlab::rng::split(seed, lane);
}

// run_method(method, ConvProblem(CHW input, MKKC kernels), backend) -> CHW output.
// threads <= 0 selects GemmBackend::blocked() (1 core), else parallel(threads).
__attribute__((visibility("default"))) int ref_run_method(const char* method, int threads,
                                                          const float* x, const float* w, float* y,
                                                          int C, int H, int W, int M, int k) {
    try {
        auto m = convlab::method_from_name(method);
        if (!m) throw std::invalid_argument(std::string("unknown method ") + method);
        const std::size_t in_n = std::size_t(C) * H * W;
        const std::size_t w_n = std::size_t(M) * k * k * C;
        convlab::Tensor3 input(C, H, W, convlab::Layout::CHW, std::vector<float>(x, x + in_n));
        convlab::KernelSet ks(M, k, C, convlab::KernelLayout::MKKC, std::vector<float>(w, w + w_n));
        convlab::ConvProblem p(std::move(input), std::move(ks));
        convlab::Tensor3 out = convlab::run_method(*m, p, backend_for(threads));
        std::memcpy(y, out.data().data(), out.size() * sizeof(float));
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

// shift_add on a row-oriented intermediate (conv_kn2.cpp:78-118).
__attribute__((visibility("default"))) int ref_shift_add_row(const float* inter, float* out, int k,
                                                             int M, int H, int W) {
    try {
        const std::size_t rows = std::size_t(k) * k * M, cols = std::size_t(H) * W;
        convlab::Matrix mat(rows, cols, std::vector<float>(inter, inter + rows * cols));
        convlab::Kn2Intermediate it{std::move(mat), convlab::Kn2Orientation::Row,
                                    std::size_t(k), std::size_t(M), std::size_t(H), std::size_t(W)};
        convlab::Matrix r = convlab::shift_add(it);
        std::memcpy(out, r.data().data(), r.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// footprint(layer, method) (bench.cpp:58-85) -> out[4] = {input, kernel, intermediate, output}.
__attribute__((visibility("default"))) int ref_footprint(const char* method, int C, int H, int W,
                                                         int M, int k, std::uint64_t* out) {
    auto m = convlab::method_from_name(method);
    if (!m) return 1;
    convlab::LayerConfig l{"l", std::size_t(C), std::size_t(H), std::size_t(W), std::size_t(M),
                           std::size_t(k), 1};
    auto fp = convlab::footprint(l, *m);
    out[0] = fp.input_bytes;
    out[1] = fp.kernel_bytes;
    out[2] = fp.intermediate_bytes;
    out[3] = fp.output_bytes;
    return 0;
}

// convlab::benchmark (bench.cpp:87-151): 1 warm-up + `runs` timed end-to-end runs of the
// method on one seeded image.  stats[3] = {mean_s, min_s, stddev_s}; *checksum = fnv1a.
__attribute__((visibility("default"))) int ref_benchmark(const char* method, int threads, int C,
                                                         int H, int W, int M, int k, int runs,
                                                         std::uint64_t seed, double* stats,
                                                         std::uint64_t* checksum) {
    try {
        auto m = convlab::method_from_name(method);
        if (!m) throw std::invalid_argument(std::string("unknown method ") + method);
        convlab::LayerConfig l{"l", std::size_t(C), std::size_t(H), std::size_t(W), std::size_t(M),
                               std::size_t(k), 1};
        auto r = convlab::benchmark(l, *m, std::uint32_t(runs), backend_for(threads), seed);
        stats[0] = r.mean_s;
        stats[1] = r.min_s;
        stats[2] = r.stddev_s;
        *checksum = r.output_checksum;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

__attribute__((visibility("default"))) int ref_hardware_threads() {
    return int(std::thread::hardware_concurrency());
}

}  // extern "C"
