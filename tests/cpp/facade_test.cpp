// facade_test.cpp -- TEST: the C++ facade (include/convlab_b200.hpp) read like the
// reference's methods_test.cpp / conv_kn2_test.cpp, with the GPU methods swapped in.
//   facade_test cpu : host logic only (names, parsing, footprint, error contracts)
//   facade_test gpu : run_method parity against the oracle (links oracle/liboracle.so)
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "convlab_b200.hpp"

extern "C" {
void orc_fill(float* out, uint64_t n, uint64_t seed, uint64_t first_index);
uint64_t orc_split(uint64_t seed, uint64_t lane);
void orc_conv_mcmk_sum(const float* x, const float* w, float* y, int C, int H, int W, int M, int k);
}

using namespace convlab_b200;

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
            ++g_fail;                                                            \
        }                                                                        \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void cpu_tests() {
    // name round trip (methods_test.cpp pattern)
    for (auto m : {ConvMethod::DirectSum, ConvMethod::Kn2row, ConvMethod::Kn2rowGpu, ConvMethod::Im2colGpu,
                   ConvMethod::Im2rowGpu, ConvMethod::Kn2rowAccGpu, ConvMethod::Auto, ConvMethod::DirectGpu}) {
        auto back = method_from_name(to_string(m));
        CHECK(back.has_value() && *back == m);
    }
    CHECK(!method_from_name("nope").has_value());
    auto list = parse_method_list("kn2row-gpu,,im2col-gpu");
    CHECK(list.size() == 2 && list[0] == ConvMethod::Kn2rowGpu && list[1] == ConvMethod::Im2colGpu);
    CHECK(throws<std::invalid_argument>([] { parse_method_list("kn2row-gpu,bogus"); }));
    CHECK(throws<std::invalid_argument>([] { parse_method_list(","); }));
    CHECK(method_requires_1x1(ConvMethod::Conv1x1Gpu) && !method_requires_1x1(ConvMethod::Kn2rowGpu));
    CHECK(is_gpu_method(ConvMethod::Kn2rowGpu) && !is_gpu_method(ConvMethod::Kn2row));
    // footprint closed forms (bench.cpp:58-85): pinned3.net l1 = 3x8x8, M=4, k=3
    LayerConfig l1{"l1", 3, 8, 8, 4, 3};
    auto fp = footprint(l1, ConvMethod::Kn2row);
    CHECK(fp.input_bytes == 768 && fp.kernel_bytes == 432 && fp.intermediate_bytes == 9216 && fp.output_bytes == 1024);
    CHECK(footprint(l1, ConvMethod::Im2colGpu).intermediate_bytes == 6912);
    CHECK(footprint(l1, ConvMethod::Kn2rowGpu).intermediate_bytes == 0);
    // contract violations surface as std::invalid_argument before any device work
    CHECK(throws<std::invalid_argument>([] { Plan p(LayerConfig{"even", 3, 8, 8, 4, 2}, ConvMethod::Kn2rowGpu); }));
    CHECK(throws<std::invalid_argument>([] { Plan p(LayerConfig{"big", 3, 2, 2, 4, 7}, ConvMethod::Kn2rowGpu); }));
    CHECK(throws<std::invalid_argument>([] { Plan p(LayerConfig{"c1", 3, 8, 8, 4, 3}, ConvMethod::Conv1x1Gpu); }));
    CHECK(throws<std::invalid_argument>([] { Plan p(LayerConfig{"cpu", 3, 8, 8, 4, 3}, ConvMethod::Kn2row); }));
    std::vector<float> dummy(4 * 9 * 3, 0.f), x(3 * 64, 0.f);
    CHECK(throws<std::invalid_argument>(
        [&] { run_method(ConvMethod::Conv1x1Gpu, LayerConfig{"c1", 3, 8, 8, 4, 3}, x.data(), dummy.data()); }));
}

static void gpu_tests() {
    struct Case {
        ConvMethod m;
        LayerConfig l;
    } cases[] = {
        {ConvMethod::Kn2rowGpu, {"a", 16, 13, 13, 32, 3, 1, -1, 2}},
        {ConvMethod::Kn2rowGpu, {"k1", 24, 7, 9, 40, 1, 1, -1, 3}},   // k=1 -> conv1x1 routing
        {ConvMethod::Kn2rowExplicitGpu, {"e", 8, 6, 5, 4, 5, 1, -1, 1}},
        {ConvMethod::Kn2colGpu, {"c", 8, 6, 5, 4, 3, 1, -1, 2}},
        {ConvMethod::Kn2rowAccGpu, {"acc", 8, 9, 9, 12, 3, 1, -1, 1}},
        {ConvMethod::Im2colGpu, {"i", 3, 10, 10, 8, 3, 1, -1, 2}},
        {ConvMethod::Im2rowGpu, {"r", 5, 9, 7, 6, 3, 1, -1, 2}},
        {ConvMethod::Auto, {"auto", 3, 12, 12, 16, 3, 1, -1, 1}},
    };
    for (const auto& c : cases) {
        const auto& l = c.l;
        const size_t xn = l.batch * l.channels * l.height * l.width;
        const size_t wn = l.kernel_count * l.kernel_size * l.kernel_size * l.channels;
        std::vector<float> x(xn), w(wn);
        orc_fill(x.data(), xn, orc_split(3, 0), 0);
        orc_fill(w.data(), wn, orc_split(3, 1), 0);
        std::vector<float> y = run_method(c.m, l, x.data(), w.data());
        const size_t plane = l.kernel_count * l.height * l.width;
        double num = 0, den = 0;
        std::vector<float> ref(plane);
        for (size_t n = 0; n < l.batch; ++n) {
            orc_conv_mcmk_sum(x.data() + n * l.channels * l.height * l.width, w.data(), ref.data(), (int)l.channels,
                              (int)l.height, (int)l.width, (int)l.kernel_count, (int)l.kernel_size);
            for (size_t e = 0; e < plane; ++e) {
                const double d = (double)y[n * plane + e] - ref[e];
                num += d * d;
                den += (double)ref[e] * ref[e];
            }
        }
        const double rel = std::sqrt(num / (den > 0 ? den : 1));
        std::printf("  %-22s %-5s rel_l2=%.3e\n", std::string(to_string(c.m)).c_str(), l.name.c_str(), rel);
        CHECK(rel <= 1e-5);
    }
    // Plan: asynchronous host call, completed by a following synchronous call on the same
    // stream (calls on one plan run in order); both outputs must be bitwise equal
    {
        LayerConfig l{"async", 16, 13, 13, 32, 3, 1, -1, 2};
        const size_t xn = l.batch * l.channels * l.height * l.width;
        const size_t wn = l.kernel_count * l.kernel_size * l.kernel_size * l.channels;
        std::vector<float> x(xn), w(wn);
        orc_fill(x.data(), xn, orc_split(5, 0), 0);
        orc_fill(w.data(), wn, orc_split(5, 1), 0);
        Plan plan(l, ConvMethod::Kn2rowGpu);
        plan.set_weights_host(w.data());
        std::vector<float> ya(l.batch * l.kernel_count * plan.out_height() * plan.out_width(), -1.0f);
        plan.forward_host_async(x.data(), ya.data(), nullptr);
        const std::vector<float> ys = plan.forward_host(x.data());
        CHECK(ya == ys);
        std::printf("  Plan::forward_host_async == forward_host: %s\n", ya == ys ? "yes" : "NO");
    }
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cpu";
    try {
        cpu_tests();
        if (mode == "gpu") gpu_tests();
    } catch (const std::exception& e) {
        std::printf("FAIL: uncaught %s\n", e.what());
        ++g_fail;
    }
    std::printf(g_fail ? "FAILED (%d)\n" : "PASSED\n", g_fail);
    return g_fail ? 1 : 0;
}
