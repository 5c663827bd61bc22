// api.cu -- the extern "C" boundary (include/convlab_b200.h): plans, method dispatch,
// workspace management, error mapping.  No CPU fallback anywhere: every entry point
// either enqueues sm_100a kernels or returns an error.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/convlab_b200.h"
#include "internal.hpp"

using namespace clb;

namespace {

thread_local std::string g_err;

// im2col and im2row differ on the CPU only in the patch matrix orientation; on the GPU both
// contract K-major patch rows ([N*P*Q][k^2 C], the im2row layout, with the shared (i*k+j)*C+c
// K order) against the M x k^2 C weights, so they share one engine path.
inline bool is_patch_method(cl_method m) { return m == CL_METHOD_IM2COL || m == CL_METHOD_IM2ROW; }

// Operand format of a precision.  fp32-faithful: the mixed 2xTF32 + 2xBF16 split (4 MMA slots
// per 16 channels) unless CLB_SPLIT=3xtf32 selects the classic 3xTF32 split (6 slots).
int planes_for(cl_precision precision) {
    static const bool classic = [] {
        const char* e = std::getenv("CLB_SPLIT");
        return e && std::strcmp(e, "3xtf32") == 0;
    }();
    if (precision == CL_PREC_BF16) return kPlanesBf16;
    if (precision == CL_PREC_TF32) return 1;
    return classic ? 2 : kPlanesMixed;
}

// Operand format of a convolution plan.  fp32: the fp16 split (3 MMA slots per 16 channels, half
// the operand bytes of the mixed split) for the implicit kn2row family wherever
// it issues fewer MMAs than the mixed split (6 ceil(C/32) < 4 ceil(C/16): not for C = 8, 16, 48)
// and the layer is large enough (>= 1.2 GFLOP) to amortise the split's extra launch (the fixup
// behind the speculative single-pass prepass, ~2 us): whole forwards, fp16 vs mixed split
// (profiles/r02c_f16_small_layers.txt): GoogLeNet 3a/1x1 (1.23 GFLOP) 54 -> 50 us, 3a/3x3 60 ->
// 54, 4a/1x1 44 -> 42, 5b/1x1 41 -> 38.5, C5 k5 56 -> 54, k7 70 -> 65 (half the operand bytes on
// HBM-bound 1x1 layers, 3 MMA slots instead of 4); C1, C5 k1 / k3 and the AlexNet b1 layers
// (<= 0.9 GFLOP) lose 3-7 us and keep the mixed split.  (The bound was 12 GFLOP while the fp16
// split still needed a max|x| pass ahead of it, profiles/r02_f16_mode_sweep.txt.)
// Otherwise the mixed split.  CLB_SPLIT=3xtf32 / mixed / 3xf16 forces a split (3xf16: where the
// method supports it).
int conv_planes_for(cl_precision precision, cl_method m, int C, double flops) {
    static const int forced = [] {
        const char* e = std::getenv("CLB_SPLIT");
        if (!e) return 0;
        if (std::strcmp(e, "3xtf32") == 0) return 2;
        if (std::strcmp(e, "mixed") == 0) return kPlanesMixed;
        if (std::strcmp(e, "3xf16") == 0) return kPlanesF16;
        return 0;
    }();
    if (precision != CL_PREC_FP32) return planes_for(precision);
    if (forced == 2 || forced == kPlanesMixed) return forced;
    const bool implicit = m == CL_METHOD_KN2ROW || m == CL_METHOD_CONV1X1 || m == CL_METHOD_KN2ROW_ACC;
    if (!implicit) return kPlanesMixed;
    if (forced == kPlanesF16) return kPlanesF16;
    return (6 * ((C + 31) / 32) < 4 * ((C + 15) / 16) && flops >= 1.2e9) ? kPlanesF16 : kPlanesMixed;
}

cl_status fail(cl_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

template <class F>
cl_status guarded(F&& f) {
    try {
        f();
        return CL_OK;
    } catch (const Error& e) {
        return fail((cl_status)e.status, e.what());
    } catch (const std::bad_alloc&) {
        return fail(CL_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(CL_EINTERNAL, e.what());
    }
}

void require(bool ok, const std::string& what) {
    if (!ok) throw Error(CL_EINVAL, what);
}

// CTA group of the tcgen05 engine: 2 (CTA pair, M = 256) unless CLB_CTA_GROUP=1 (A/B switch
// for measurements) or the problem has fewer than 256 rows.
int cta_group_for(long long rows, int cols, int bn) {
    static int forced = [] {
        const char* e = std::getenv("CLB_CTA_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    // pairs need at least one wave of 256-row tiles to pay off; small problems want more,
    // smaller (128-row) tiles instead
    const long long pair_tiles = (rows + 255) / 256 * ((cols + bn - 1) / bn);
    return (rows >= 256 && pair_tiles >= num_sms() / 2) ? 2 : 1;
}

int bn_for(int cols) {
    const int tiles = (cols + 255) / 256;
    const int per = (cols + tiles - 1) / tiles;
    int bn = round_up(per, 16);
    if (bn < 16) bn = 16;
    return bn > 256 ? 256 : bn;
}

}  // namespace

struct cl_plan {
    cl_conv_desc d{};
    int P = 0, Q = 0;
    cl_method requested = CL_METHOD_AUTO, method = CL_METHOD_AUTO;
    cl_precision prec = CL_PREC_FP32;
    int planes = 2;
    int device = 0;
    int Cp = 0;            // channels padded to the 16-wide K block (kn2 methods)
    int Kp = 0;            // k*k*C padded (im2col)
    int bn = 0;
    float* wpack = nullptr;
    size_t wpack_bytes = 0;
    // fp16 split: exponent slots [ew, ex], the absmax pass's counter and partials (device)
    int* scale = nullptr;
    bool tc_direct = false;    // direct-gpu on the tensor cores (tc_direct.cu; tiny-C layers, fp32)
    float* wraw = nullptr;     // direct-gpu: MKKC fp32 weights as given
    // direct-gpu, 3 -> 16/32/64 channels 3x3: host weights [c][i][j][m] passed as a kernel
    // parameter (constant-bank FFMA operands).  Only filled by cl_conv_set_weights_host (the host
    // data is at hand; a device-pointer upload never blocks on a D2H copy) and only used by eager
    // launches: a CUDA graph captures kernel parameters by value, so a captured launch reads the
    // device weights instead and picks up later set_weights calls like every other method.
    std::vector<float> wparam;
    int max_sms = 0;           // engine grid cap in SMs (cl_conv_set_max_sms; 0 = all co-resident units)
    std::vector<float*> peers; // fused output all-gather targets (cl_conv_set_peer_outputs)
    int peer_m0 = 0, peer_M = 0;
    unsigned* flags = nullptr; // stream-K fixup flags, zeroed once, self-resetting
    bool padded_rows = false;  // implicit kn2row in tap-shared (zero-padded row) mode
    int wp = 0;                // padded-row mode: padded row width (W + pad; tap-stacked: see tma_store)
    int stack_k = 1;           // > 1: padded-row mode with the k taps of a kernel row stacked on N
    int bn_stack = 0;          // its tile N (k x channels per column tile)
    int msub = 1;              // 2: padded-row mode with two 128-row sub-tiles per B stage (TcParams::msub)
    bool weights_set = false;
    void* own_ws = nullptr;
    size_t own_ws_bytes = 0;
    float* host_x = nullptr;   // device staging for cl_conv_forward_host
    float* host_y = nullptr;
    int launches = 0;
    cudaEvent_t ev_begin = nullptr, ev_end = nullptr;  // optional instrumentation
    // chunked host pipeline (cl_conv_forward_host): copy-in / copy-out streams + per-chunk events
    cudaStream_t s_in = nullptr, s_out = nullptr;
    bool shared_streams = false;   // s_in / s_out are the device's shared copy streams (not owned)
    static constexpr int kMaxChunks = 16;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_comp[kMaxChunks] = {}, ev_start = nullptr, ev_done = nullptr;
    // Sharing: a plan's flags, own workspace and staging buffers are per-plan state, so calls
    // on one plan are serialised -- host side by `mu`, device side by chaining each call after
    // the previous call's completion event when it arrives on a different stream.
    std::mutex mu;
    cudaEvent_t ev_last = nullptr;
    cudaStream_t last_stream = nullptr;
    bool has_last = false;
};

namespace {

cl_method resolve(const cl_conv_desc& d, cl_method m) {
    if (m != CL_METHOD_AUTO) return m;
    // Per-layer selector.  The implicit kernel is the default; tiny-C first layers (VGG
    // conv1_1, C = 3) waste 13/16 of every 16-channel K block per tap and are HBM-bound, so
    // they take the direct CUDA-core kernel (PAPER.md:484 found direct best on that layer
    // too); im2col remains for small C the direct kernel cannot stage.
    if (d.c <= 4 && direct_fast_path(d.c, d.k, d.stride)) return CL_METHOD_DIRECT;
    if (d.k > 1 && d.c * 4 <= 16) return CL_METHOD_IM2COL;
    return CL_METHOD_KN2ROW;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// Method buffers first, then the stream-K scratch of the tcgen05 engine.
size_t method_ws_bytes(const cl_plan* p);
size_t ws_bytes(const cl_plan* p) { return align256(method_ws_bytes(p)) + tc_scratch_bytes(); }
void* scratch_of(const cl_plan* p, void* ws) { return static_cast<char*>(ws) + align256(method_ws_bytes(p)); }

// Tap-stacked mode reads A through an overlapping view whose bounds check covers only the
// row dimension: zeroed rows before (the first image's leading padding, made real) and after
// the padded grid keep every read in bounds and every out-of-image tap zero.
int stack_lead_rows(const cl_plan* p) { return p->stack_k > 1 ? p->d.pad * p->wp + p->d.pad : 0; }
int stack_trail_rows(const cl_plan* p) { return p->stack_k > 1 ? 4 * 32 : 0; }
size_t stack_slack_rows(const cl_plan* p) { return (size_t)stack_lead_rows(p) + stack_trail_rows(p); }

size_t method_ws_bytes(const cl_plan* p) {
    const cl_conv_desc& d = p->d;
    const size_t nhw = (size_t)d.n * d.h * d.w;
    const size_t npq = (size_t)d.n * p->P * p->Q;
    const size_t xs = nhw * row_bytes(p->planes, p->Cp);
    const size_t kk = (size_t)d.k * d.k;
    switch (p->method) {
        case CL_METHOD_KN2ROW:
        case CL_METHOD_CONV1X1:
        case CL_METHOD_KN2ROW_ACC:
            if (p->padded_rows)
                return ((size_t)d.n * (d.h + d.pad) * p->wp + stack_slack_rows(p)) * row_bytes(p->planes, p->Cp);
            return xs;
        case CL_METHOD_KN2ROW_EXPLICIT:
        case CL_METHOD_KN2COL:
            return xs + kk * d.m * nhw * 4;
        case CL_METHOD_IM2COL:
        case CL_METHOD_IM2ROW:
            return npq * row_bytes(p->planes, p->Kp);
        case CL_METHOD_DIRECT:
            return 0;
        default:
            return 0;
    }
}

void check_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw Error(CL_ENODEVICE, "no CUDA device visible (the B200 path has no CPU fallback)");
    }
    if (device < 0 || device >= count) throw Error(CL_EINVAL, "device index out of range");
    int major = 0;
    CLB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
    if (major != 10) throw Error(CL_ENODEVICE, "device is not sm_100 (compute capability 10.x required)");
}

Operand implicit_a(const cl_plan* p, const void* xs) {
    Operand a;
    a.mode = LOAD_IM2COL;
    a.ptr = xs;
    a.kw = (int)row_elems(p->planes, p->Cp);
    a.planes = p->planes;
    a.n = p->d.n;
    a.h = p->d.h;
    a.w = p->d.w;
    a.k = p->d.k;
    a.pad = p->d.pad;
    return a;
}

Operand tiled(const void* ptr, long long rows, int taps, int kp, int planes) {
    Operand o;
    o.mode = LOAD_TILED;
    o.ptr = ptr;
    o.rows = rows;
    o.taps = taps;
    o.kw = (int)row_elems(planes, kp);
    o.planes = planes;
    return o;
}

TcParams base_params(const cl_plan* p) {
    TcParams t{};
    t.sexp = p->planes == kPlanesF16 ? p->scale : nullptr;
    t.ksize = p->d.k;
    t.P = p->P;
    t.Q = p->Q;
    t.pad = p->d.pad;
    return t;
}

// Device-side ordering of calls on a shared plan (caller holds p->mu).
// (A stream being captured into a CUDA graph is left alone: the graph's own edges order it.)
bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    CLB_CUDA(cudaStreamIsCapturing(s, &st));
    return st != cudaStreamCaptureStatusNone;
}

void order_after_previous(cl_plan* p, cudaStream_t s) {
    if (p->has_last && p->last_stream != s && !capturing(s)) CLB_CUDA(cudaStreamWaitEvent(s, p->ev_last, 0));
}

void mark_done(cl_plan* p, cudaStream_t s) {
    if (capturing(s)) {
        p->has_last = false;
        return;
    }
    if (!p->ev_last) CLB_CUDA(cudaEventCreateWithFlags(&p->ev_last, cudaEventDisableTiming));
    CLB_CUDA(cudaEventRecord(p->ev_last, s));
    p->last_stream = s;
    p->has_last = true;
}

// n_images < 0: the plan's batch; otherwise a sub-batch (chunked host pipeline).
// nhwc: channels-last input and output (implicit kn2row / conv1x1 / accumulating only).
// ev_first / ev_last_chunk: record the plan's profile events (begin / end) in this call (a
// chunked forward brackets all of its chunks with one pair).
// The caller's workspace, or the plan's own (allocated on first use).
void* resolve_ws(cl_plan* p, void* ws) {
    const size_t need = ws_bytes(p);
    if (ws || !need) return ws;
    if (p->own_ws_bytes < need) {
        if (p->own_ws) cudaFree(p->own_ws);
        p->own_ws = nullptr;
        p->own_ws_bytes = 0;
        if (cudaMalloc(&p->own_ws, need) != cudaSuccess) {
            cudaGetLastError();
            throw Error(CL_ENOMEM, "workspace allocation failed: requires " + std::to_string(need) + " bytes");
        }
        p->own_ws_bytes = need;
    }
    return p->own_ws;
}

// Chained prepass (cl_conv_forward_chain): the plan's NCHW -> split prepass as a tile job, when
// its forward runs the standard prepass (implicit / conv1x1 / accumulating kn2row, fp32-faithful
// split formats).  The job's counter lives in the plan's flag buffer.
bool chain_job(cl_plan* p, const float* x, void* ws, SplitJob* out) {
    const bool implicit = p->method == CL_METHOD_KN2ROW || p->method == CL_METHOD_CONV1X1 ||
                          p->method == CL_METHOD_KN2ROW_ACC;
    if (!implicit || !is_split(p->planes) || (p->padded_rows && p->wp != p->d.w + p->d.pad)) return false;
    const cl_conv_desc& d = p->d;
    void* xs = ws;
    int pad = 0;
    if (p->padded_rows) {
        xs = static_cast<char*>(ws) + (size_t)stack_lead_rows(p) * row_bytes(p->planes, p->Cp);
        pad = d.pad;
    }
    *out = make_split_job(x, xs, d.n, d.c, d.h, d.w, pad, p->Cp);
    out->planes = p->planes;
    out->counter = p->flags + kMaxGrid + 2;
    return true;
}

void forward_impl(cl_plan* p, const float* x, float* y, void* ws, cudaStream_t s, int n_images, bool nhwc,
                  bool ev_first, bool ev_last_chunk, const SplitJob* next_job, bool prepass_partial);

// A forward that fails after the fp16 split's speculative prepass was enqueued leaves its group
// maxima un-zeroed (the contraction zeroes them): zero them here so the next forward's exponent
// is this input's alone.
void forward(cl_plan* p, const float* x, float* y, void* ws, cudaStream_t s, int n_images = -1, bool nhwc = false,
             bool ev_first = true, bool ev_last_chunk = true, const SplitJob* next_job = nullptr,
             bool prepass_partial = false) {
    try {
        forward_impl(p, x, y, ws, s, n_images, nhwc, ev_first, ev_last_chunk, next_job, prepass_partial);
    } catch (...) {
        if (p->scale)
            cudaMemsetAsync(spec_reset_slots(p->scale), 0, (size_t)kSpecGroups * kSpecStride * sizeof(unsigned), s);
        throw;
    }
}

void forward_impl(cl_plan* p, const float* x, float* y, void* ws, cudaStream_t s, int n_images, bool nhwc,
                  bool ev_first, bool ev_last_chunk, const SplitJob* next_job, bool prepass_partial) {
    cl_conv_desc d = p->d;
    if (n_images >= 0) d.n = n_images;
    require(p->weights_set, "cl_conv_forward: weights not set (cl_conv_set_weights)");
    require(x && y, "cl_conv_forward: null tensor");
    CLB_CUDA(cudaSetDevice(p->device));
    ws = resolve_ws(p, ws);
    // chained: this plan's prepass was started by the previous contraction's converter warps
    SplitJob own_job{};
    if (prepass_partial && !(n_images < 0 && !nhwc && chain_job(p, x, ws, &own_job)))
        throw Error(CL_EINTERNAL, "chained prepass on a plan without a chainable prepass");
    const int taps = d.k * d.k;
    const long long nhw = (long long)d.n * d.h * d.w;
    const long long npq = (long long)d.n * p->P * p->Q;
    float* wsf = static_cast<float*>(ws);
    p->launches = 0;
    bool began = false;
    void* scratch = scratch_of(p, ws);
    auto tc = [&](const Operand& a, const Operand& b, TcParams t) {
        // PDL right after the prepass kernel (its launch_dependents trigger lets this
        // kernel's prologue overlap the prepass tail); an interposed profile event only
        // removes the overlap, never the ordering
        t.pdl = !began ? 1 : 0;
        if (p->ev_begin && !began && ev_first) CLB_CUDA(cudaEventRecord(p->ev_begin, s));
        began = true;
        set_scratch(t, scratch);
        t.flags = p->flags;
        t.flags_zeroed = 1;
        t.max_sms = p->max_sms;
        if (!p->peers.empty()) {
            if (t.epi != EPI_NCHW && t.epi != EPI_NCHW_PADDED)
                throw Error(CL_EUNSUPPORTED, "peer outputs: implicit kn2row / conv1x1 / im2col plans, NCHW only");
            t.n_peers = (int)p->peers.size();
            for (int r = 0; r < t.n_peers; ++r) t.peers[r] = p->peers[r];
            t.peer_m0 = p->peer_m0;
            t.peer_M = p->peer_M;
        }
        if (next_job && is_split(p->planes) && (p->planes == next_job->planes)) {
            t.nx = *next_job;
            t.nx_on = 1;
        }
        static const int forced_bn = [] {   // experiments: CLB_BN=<multiple of 16 <= 256>
            const char* e = std::getenv("CLB_BN");
            const int v = e ? std::atoi(e) : 0;
            return (v >= 16 && v <= 256 && v % 16 == 0) ? v : 0;
        }();
        // tap-stacked: N is k x channels; two-sub-tile: N is 2 x the sub-tile's -- not free choices
        const bool fixed_bn = t.stack_k > 1 || t.msub > 1;
        if (forced_bn && !fixed_bn) t.bn = forced_bn;
        const int ms = t.msub > 1 ? t.msub : 1;
        int cg = cta_group_for(t.rows / ms, t.cols, t.bn / ms);
        if (ms > 1 && tc_num_stages(t.bn / ms / cg, t.tps, 1, kSmemBudget, ms) < 3) {   // too few stages: one sub-tile
            t.msub = 1;
            t.bn /= ms;
        }
        // few tiles even at 128 rows: halve the tile N to create more of them (B operand rows
        // are tiny anyway at these sizes)
        if (!forced_bn && !fixed_bn && cg == 1 && t.bn >= 64 &&
            (long long)(t.rows + 127) / 128 * ((t.cols + t.bn - 1) / t.bn) < num_sms() / 2)
            t.bn = round_up(t.bn / 2, 16);
        // a k-tap stage must fit twice: a sub-batch (host-buffer chunks) can drop a padded-row
        // launch to a single CTA, which holds all of B -- take a pair, or halve the tile N
        const int tps = t.tps > 0 ? t.tps : 1;
        while (tc_num_stages(t.bn / cg, tps) < 2 && t.bn > 16) {
            if (cg == 1 && t.rows >= 256 && t.bn % 32 == 0) cg = 2;
            else if (fixed_bn) break;
            else t.bn = round_up(t.bn / 2, 16);
        }
        p->launches += launch_tc(a, b, t, s, cg);
    };
    auto tc_done = [&] {
        if (p->ev_end && ev_last_chunk) CLB_CUDA(cudaEventRecord(p->ev_end, s));
    };

    switch (p->method) {
        case CL_METHOD_KN2ROW:
        case CL_METHOD_CONV1X1:
        case CL_METHOD_KN2ROW_ACC: {
            void* xs = wsf;
            // fp16 split: the input's exponent shift.  NCHW input: one speculative pass (the split
            // reduces max|x| while converting with the previous forward's exponent) + a fixup launch
            // that re-converts only on a miss; channels-last input (or CLB_F16_SPEC=0): a max|x|
            // pass ahead of the split
            static const bool spec_env = !(std::getenv("CLB_F16_SPEC") && std::atoi(std::getenv("CLB_F16_SPEC")) == 0);
            const bool spec = p->planes == kPlanesF16 && !nhwc && !prepass_partial && spec_env;
            unsigned* t_reset = nullptr;   // the contraction zeroes the speculative pass's group maxima
            if (p->planes == kPlanesF16 && !spec) {
                launch_absmax_exp(x, (long long)d.n * d.c * d.h * d.w, p->scale, p->scale + 1, s);
                ++p->launches;
            }
            if (p->padded_rows) {
                // tap-shared mode: zero-padded NHWC rows; each stage loads ONE A box of 128+k-1
                // rows per kernel row i and feeds its k taps through row-shifted descriptors
                const int Hp = d.h + d.pad, Wp = p->wp;   // shared padding (tc_conv.cuh)
                const size_t rb = (size_t)row_bytes(p->planes, p->Cp);
                const long long grid_rows = (long long)d.n * Hp * Wp;
                const int lead = stack_lead_rows(p), trail = stack_trail_rows(p);
                if (lead + trail > 0) {   // tap-stacked slack rows (zero), before the prepass (PDL pairs it with the contraction)
                    CLB_CUDA(cudaMemsetAsync(xs, 0, (size_t)lead * rb, s));
                    CLB_CUDA(cudaMemsetAsync(static_cast<char*>(xs) + ((size_t)lead + grid_rows) * rb, 0, (size_t)trail * rb, s));
                }
                void* grid = static_cast<char*>(xs) + (size_t)lead * rb;
                if (prepass_partial) {
                    launch_split_tail(own_job, p->planes, s);   // the tiles the previous contraction left
                    ++p->launches;
                } else if (spec) {
                    launch_nchw_split_speculative(x, grid, d.n, d.c, d.h, d.w, d.pad, p->Cp, p->scale, s, Wp);
                    p->launches += 2;
                    t_reset = spec_reset_slots(p->scale);
                } else {
                    if (nhwc) launch_nhwc_split(x, grid, d.n, d.c, d.h, d.w, d.pad, p->Cp, p->planes, s, p->scale, Wp);
                    else launch_nchw_to_padded_split(x, grid, d.n, d.c, d.h, d.w, d.pad, p->Cp, p->planes, s, p->scale, Wp);
                    ++p->launches;
                }
                Operand a = tiled(xs, grid_rows, 1, p->Cp, p->planes);
                Operand b = tiled(p->wpack, d.m, taps, p->Cp, p->planes);
                TcParams t = base_params(p);
                t.reset_slots = t_reset;
                t.rows = d.n * Hp * Wp;
                t.cols = d.m;
                t.bn = p->bn;
                t.b_tap3 = 1;
                t.tps = d.k;
                t.taps = taps;
                if (p->msub > 1) {
                    t.msub = p->msub;
                    t.bn = p->bn * p->msub;
                }
                if (p->stack_k > 1) {
                    // tap-stacked: one k-iteration = kernel row i x one channel block; B rows
                    // (m, j) of row i, D column m*k + j; A unshifted (the shift-add is in the epilogue)
                    b = tiled(p->wpack, (long long)d.m * d.k, d.k, p->Cp, p->planes);
                    a = tiled(xs, lead + grid_rows + trail - 3 * (33 - d.k), 4, p->Cp, p->planes);
                    a.tap_stride_rows = 33 - d.k;   // quadrant q of a box starts 33 - k rows after q - 1
                    t.cols = d.m * d.k;
                    t.bn = p->bn_stack;
                    t.tps = 1;
                    t.ksize = 1;      // tap index = kernel row i (ti = i, tj = 0)
                    t.taps = d.k;
                    t.stack_k = d.k;
                }
                t.a_row_shift = Wp;
                t.a_row_base = lead - d.pad * Wp - d.pad;   // >= 0 in tap-stacked mode
                t.epi = nhwc ? EPI_NHWC_PADDED : EPI_NCHW_PADDED;
                t.ld = d.m;
                t.epi_hp = Hp;
                t.epi_wp = Wp;
                t.epi_n = d.n;
                t.out = y;
                t.out_channels = d.m;
                t.pq_out = p->P * p->Q;
                tc(a, b, t);
                tc_done();
                break;
            }
            if (prepass_partial) launch_split_tail(own_job, p->planes, s);
            else if (spec) {
                launch_nchw_split_speculative(x, xs, d.n, d.c, d.h, d.w, 0, p->Cp, p->scale, s);
                ++p->launches;
                t_reset = spec_reset_slots(p->scale);
            } else if (nhwc) launch_nhwc_split(x, xs, d.n, d.c, d.h, d.w, 0, p->Cp, p->planes, s, p->scale);
            else launch_nchw_to_nhwc_split(x, xs, d.n, d.c, d.h * d.w, p->Cp, p->planes, s, p->scale);
            ++p->launches;
            Operand a = implicit_a(p, xs);
            a.n = d.n;
            Operand b = tiled(p->wpack, d.m, taps, p->Cp, p->planes);
            TcParams t = base_params(p);
            t.reset_slots = t_reset;
            t.rows = (int)npq;
            t.cols = d.m;
            t.bn = p->bn;
            t.b_tap3 = 1;
            t.epi = nhwc ? EPI_ROWMAJOR : EPI_NCHW;
            t.ld = d.m;                       // channels-last: D[n*P*Q + pq][m] is the output
            t.out = y;
            t.out_channels = d.m;
            t.pq_out = p->P * p->Q;
            if (p->method == CL_METHOD_KN2ROW_ACC) {
                // k^2 shifted GEMMs, each accumulating into the output (tap 0 overwrites).
                for (int tap = 0; tap < taps; ++tap) {
                    t.taps = 1;
                    t.tap_begin = tap;
                    t.accumulate = tap > 0;
                    tc(a, b, t);
                }
            } else {
                t.taps = taps;
                t.tap_begin = 0;
                tc(a, b, t);
            }
            tc_done();
            break;
        }
        case CL_METHOD_KN2ROW_EXPLICIT:
        case CL_METHOD_KN2COL: {
            if (nhwc) throw Error(CL_EUNSUPPORTED, "channels-last forward: implicit kn2row / conv1x1 / kn2row-acc only");
            void* xs = wsf;
            float* inter = reinterpret_cast<float*>(reinterpret_cast<char*>(wsf) + nhw * row_bytes(p->planes, p->Cp));
            launch_nchw_to_nhwc_split(x, xs, d.n, d.c, d.h * d.w, p->Cp, p->planes, s);
            ++p->launches;
            Operand wts = tiled(p->wpack, (long long)taps * d.m, 1, p->Cp, p->planes);
            Operand pix = tiled(xs, nhw, 1, p->Cp, p->planes);
            TcParams t = base_params(p);
            t.taps = 1;
            t.epi = EPI_ROWMAJOR;
            t.out = inter;
            if (p->method == CL_METHOD_KN2ROW_EXPLICIT) {
                // (k^2 M x C) . (C x NHW): the paper's single kn2row GEMM (conv_kn2.cpp:145-162)
                t.rows = taps * d.m;
                t.cols = (int)nhw;
                t.ld = nhw;
                t.bn = 256;
                tc(wts, pix, t);
                tc_done();
                launch_shift_add_row(inter, y, d.n, d.m, d.h, d.w, d.k, d.pad, p->P, p->Q, s);
            } else {
                // (NHW x C) . (C x k^2 M): the kn2col GEMM (conv_kn2.cpp:164-183)
                t.rows = (int)nhw;
                t.cols = taps * d.m;
                t.ld = (long long)taps * d.m;
                t.bn = bn_for(taps * d.m);
                tc(pix, wts, t);
                tc_done();
                launch_shift_add_col(inter, y, d.n, d.m, d.h, d.w, d.k, d.pad, p->P, p->Q, s);
            }
            ++p->launches;
            break;
        }
        case CL_METHOD_IM2COL:
        case CL_METHOD_IM2ROW: {
            if (nhwc) throw Error(CL_EUNSUPPORTED, "channels-last forward: implicit kn2row / conv1x1 / kn2row-acc only");
            void* pm = wsf;
            launch_im2col_split(x, pm, d.n, d.c, d.h, d.w, d.k, d.pad, d.stride, p->P, p->Q, p->Kp, p->planes, s);
            ++p->launches;
            Operand a = tiled(pm, npq, 1, p->Kp, p->planes);
            Operand b = tiled(p->wpack, d.m, 1, p->Kp, p->planes);
            TcParams t = base_params(p);
            t.rows = (int)npq;
            t.cols = d.m;
            t.bn = p->bn;
            t.taps = 1;
            t.epi = EPI_NCHW;
            t.out = y;
            t.out_channels = d.m;
            t.pq_out = p->P * p->Q;
            tc(a, b, t);
            tc_done();
            break;
        }
        case CL_METHOD_DIRECT: {
            if (nhwc) throw Error(CL_EUNSUPPORTED, "channels-last forward: implicit kn2row / conv1x1 / kn2row-acc only");
            const bool aligned16 = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
            if (p->tc_direct && aligned16) {
                // tensor cores: the input's exponent (max|x|, a small tensor), then the fused
                // gather + split + MMA + TMA-store kernel
                launch_absmax_exp(x, (long long)d.n * d.c * d.h * d.w, p->scale, p->scale + 1, s);
                if (p->ev_begin && ev_first) CLB_CUDA(cudaEventRecord(p->ev_begin, s));
                launch_tc_direct(x, p->wpack, y, d.n, d.c, d.h, d.w, d.m, d.k, d.pad, p->P, p->Q, p->scale, s,
                                 p->max_sms);
                p->launches += 2;
                tc_done();
                break;
            }
            // the dominant (and only) kernel of this method: bracket it for the profile events
            if (p->ev_begin && ev_first) CLB_CUDA(cudaEventRecord(p->ev_begin, s));
            const bool param = !p->wparam.empty() && !capturing(s);
            launch_direct_conv(x, p->wraw, y, d.n, d.c, d.h, d.w, d.m, d.k, d.pad, d.stride, p->P, p->Q, s,
                               param ? p->wparam.data() : nullptr);
            ++p->launches;
            tc_done();
            break;
        }
        default:
            throw Error(CL_EINTERNAL, "unresolved method");
    }
}

// direct-gpu parameter-weight kernel: MKKC host weights -> [c][i][j][m]
void pack_param_weights(cl_plan* p, const float* h_w_mkkc) {
    const cl_conv_desc& d = p->d;
    p->wparam.assign((size_t)d.c * d.k * d.k * d.m, 0.0f);
    for (int m = 0; m < d.m; ++m)
        for (int i = 0; i < d.k; ++i)
            for (int j = 0; j < d.k; ++j)
                for (int c = 0; c < d.c; ++c)
                    p->wparam[(((size_t)c * d.k + i) * d.k + j) * d.m + m] =
                        h_w_mkkc[(((size_t)m * d.k + i) * d.k + j) * d.c + c];
}

}  // namespace

// ---- evidence-based selection: a one-shot timing cache keyed by the descriptor ----------
// The method table over every BASELINE layer (tools/method_table.py, profiles/r02_method_table.*)
// shows the implicit kernel fastest at every benchmarked batch -- 1.3-15x over explicit kn2row,
// kn2col, im2col and the accumulating variant -- but the paper's own explicit kn2row (one
// (k^2 M) x C GEMM + shift-add) winning by 10-20 % on batch-1 3x3 layers with small maps and
// wide channels (AlexNet conv4/conv5 b1, the C5 k3 sweep layer): there the implicit kernel has a
// handful of output tiles and leans on stream-K, while the explicit GEMM's k^2 M rows make k^2
// times more tiles.  The rule below keeps the implicit kernel except in that regime, where the two
// are timed once per descriptor (device, shape, precision) on scratch buffers and the faster is
// cached for the process (the explicit one only when >= 5 % faster).  CLB_AUTOTUNE=0: the rule alone.
extern "C" cl_status cl_conv_plan(const cl_conv_desc*, cl_method, cl_precision, int, cl_plan**);

namespace {

bool tune_candidate(const cl_conv_desc& d, int P, int Q) {
    if (d.k == 1 || d.stride != 1 || d.pad != d.k / 2 || P != d.h || Q != d.w) return false;
    const int bn = bn_for(d.m);
    const long long tiles = ((long long)d.n * P * Q + 127) / 128 * ((d.m + bn - 1) / bn);
    const double inter = (double)d.k * d.k * d.m * d.n * d.h * d.w * 4.0;
    return tiles <= num_sms() && inter <= 256.0 * (1 << 20);
}

double time_forward(const cl_conv_desc& d, cl_method m, cl_precision prec, int device) {
    cl_plan* p = nullptr;
    if (cl_conv_plan(&d, m, prec, device, &p) != CL_OK) return 1e30;
    float *x = nullptr, *y = nullptr;
    void* ws = nullptr;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double best = 1e30;
    const size_t xb = (size_t)d.n * d.c * d.h * d.w * 4, yb = (size_t)d.n * d.m * p->P * p->Q * 4;
    if (cudaMalloc(&x, xb) == cudaSuccess && cudaMalloc(&y, yb) == cudaSuccess &&
        cudaMalloc(&ws, std::max<size_t>(ws_bytes(p), 256)) == cudaSuccess &&
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess && cudaEventCreate(&e0) == cudaSuccess &&
        cudaEventCreate(&e1) == cudaSuccess && cudaMemsetAsync(x, 0, xb, s) == cudaSuccess &&
        cudaMemsetAsync(p->wpack, 0, p->wpack_bytes, s) == cudaSuccess) {
        p->weights_set = true;   // timing only: the packed weights are zeros
        // a device-side lead (a 16 MB memset) before each timed forward lets the host enqueue the
        // whole forward before the GPU reaches it, so the events measure device time, as a
        // captured graph or a busy stream would see it (not the host launch latency)
        void* lead = nullptr;
        const size_t lead_bytes = 16u << 20;
        if (cudaMalloc(&lead, lead_bytes) != cudaSuccess) lead = nullptr;
        for (int r = 0; r < 6; ++r) {
            if (lead) cudaMemsetAsync(lead, r, lead_bytes, s);
            cudaEventRecord(e0, s);
            if (cl_conv_forward(p, x, y, ws, s) != CL_OK) break;
            cudaEventRecord(e1, s);
            float ms = 0.0f;
            if (cudaEventSynchronize(e1) != cudaSuccess || cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) break;
            if (r >= 2) best = std::min(best, (double)ms);   // two warm-ups
        }
        cudaFree(lead);
    }
    cudaGetLastError();
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
    cudaFree(x);
    cudaFree(y);
    cudaFree(ws);
    cl_conv_destroy(p);
    return best;
}

cl_method tuned_method(const cl_conv_desc& d, int P, int Q, cl_precision prec, int device) {
    static const bool enabled = !(std::getenv("CLB_AUTOTUNE") && std::atoi(std::getenv("CLB_AUTOTUNE")) == 0);
    if (!enabled || !tune_candidate(d, P, Q)) return CL_METHOD_KN2ROW;
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int, int, int, int, int, int>, cl_method> cache;
    const auto key = std::make_tuple(device, (int)prec, d.n, d.c, d.h, d.w, d.m, d.k, d.pad, d.stride);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const double t_impl = time_forward(d, CL_METHOD_KN2ROW, prec, device);
    const double t_expl = time_forward(d, CL_METHOD_KN2ROW_EXPLICIT, prec, device);
    const cl_method pick = t_expl < 0.95 * t_impl ? CL_METHOD_KN2ROW_EXPLICIT : CL_METHOD_KN2ROW;
    std::lock_guard<std::mutex> g(mu);
    return cache.emplace(key, pick).first->second;
}

}  // namespace

extern "C" {

cl_status cl_conv_plan(const cl_conv_desc* desc, cl_method method, cl_precision precision, int device,
                       cl_plan** out_plan) {
    return guarded([&] {
        require(desc && out_plan, "cl_conv_plan: null argument");
        *out_plan = nullptr;
        cl_conv_desc d = *desc;
        require(d.n > 0 && d.c > 0 && d.h > 0 && d.w > 0 && d.m > 0 && d.k > 0,
                "cl_conv_plan: dimensions must be positive");
        require(d.k % 2 == 1, "kernel size must be odd, got " + std::to_string(d.k));   // tensor.cpp:64,71
        if (d.pad < 0) d.pad = d.k / 2;
        if (d.stride <= 0) d.stride = 1;
        // ConvProblem's bound k <= min(H,W) + k/2 (conv_direct.cpp:15-20) at the default pad
        const int bound = (d.h < d.w ? d.h : d.w) + d.k / 2;
        require(d.pad != d.k / 2 || d.k <= bound,
                "ConvProblem: kernel size " + std::to_string(d.k) + " exceeds padded image bound " +
                    std::to_string(bound));
        require(precision == CL_PREC_FP32 || precision == CL_PREC_TF32 || precision == CL_PREC_BF16, "unknown precision");
        require(method >= CL_METHOD_AUTO && method <= CL_METHOD_IM2ROW, "unknown method " + std::to_string((int)method));
        if (method == CL_METHOD_CONV1X1)
            require(d.k == 1, "conv1x1 requires a 1x1 kernel, got k = " + std::to_string(d.k));
        const int P = (d.h + 2 * d.pad - d.k) / d.stride + 1;
        const int Q = (d.w + 2 * d.pad - d.k) / d.stride + 1;
        require(P > 0 && Q > 0, "cl_conv_plan: empty output");
        // 32-bit engine coordinates (TMA box coordinates, tile rows): one plan covers fewer than
        // 2^31 pixel rows in every layout it may use (padded grid + tap-stacked slack included);
        // larger batches are split by the caller (or by torch.distributed batch sharding)
        {
            const long long rows = std::max({(long long)d.n * (d.h + d.pad + 1) * (d.w + d.pad + 1) + 8192,
                                             (long long)d.n * P * Q, (long long)d.n * d.h * d.w,
                                             (long long)d.k * d.k * d.m});
            if (rows >= 0x7fffffffLL)
                throw Error(CL_EUNSUPPORTED, "layer too large for one plan (" + std::to_string(rows) +
                                                 " pixel rows >= 2^31): split the batch");
        }
        cl_method m = resolve(d, method);
        if (method == CL_METHOD_AUTO && m == CL_METHOD_KN2ROW) {
            check_device(device);   // (the timing cache runs on the device)
            CLB_CUDA(cudaSetDevice(device));
            m = tuned_method(d, P, Q, precision, device);
        }
        if (d.k == 1 && (m == CL_METHOD_KN2ROW_EXPLICIT || m == CL_METHOD_KN2COL)) m = CL_METHOD_CONV1X1;
        if (m == CL_METHOD_DIRECT) {
            // any shape: the shared-memory kernels where they fit, else the generic loop nest
        } else if (!is_patch_method(m)) {
            if (d.stride != 1) throw Error(CL_EUNSUPPORTED, "kn2 methods support stride 1 only (im2col supports stride)");
            if (d.pad > 127 || d.k - 1 - d.pad > 128)
                throw Error(CL_EUNSUPPORTED, "padding outside the TMA im2col bounding-box range");
            if ((m == CL_METHOD_KN2ROW_EXPLICIT || m == CL_METHOD_KN2COL) && (P != d.h || Q != d.w))
                throw Error(CL_EUNSUPPORTED, "explicit kn2row/kn2col need same padding (pad = k/2)");
        }
        check_device(device);
        CLB_CUDA(cudaSetDevice(device));
        auto* p = new cl_plan;
        p->d = d;
        p->P = P;
        p->Q = Q;
        p->requested = method;
        p->method = m;
        p->prec = precision;
        p->planes = conv_planes_for(precision, m, d.c, 2.0 * d.n * d.m * d.c * d.k * d.k * (double)P * Q);
        {
            // direct-gpu on the tensor cores where its one-K-block kernel applies (fp32-faithful fp16
            // split; CLB_DIRECT_TC=0 keeps the CUDA-core kernel): VGG conv1_1 0.154 -> see DESIGN 4.1c
            static const bool direct_tc = !(std::getenv("CLB_DIRECT_TC") && std::atoi(std::getenv("CLB_DIRECT_TC")) == 0);
            // (a forced mixed / 3xTF32 split keeps the CUDA-core kernel: the tensor-core one is fp16-split only)
            const bool f16_allowed = conv_planes_for(precision, CL_METHOD_KN2ROW, 64, 1e30) == kPlanesF16;
            if (m == CL_METHOD_DIRECT && precision == CL_PREC_FP32 && direct_tc && f16_allowed &&
                tc_direct_shape(d.c, d.k, d.m, d.stride, d.pad, P, Q)) {
                p->tc_direct = true;
                p->planes = kPlanesF16;
            }
        }
        p->device = device;
        p->Cp = round_up(d.c, k_granule(p->planes));
        p->Kp = round_up(d.k * d.k * d.c, k_granule(p->planes));
        p->bn = bn_for(d.m);
        if (is_patch_method(m)) p->wpack_bytes = (size_t)d.m * row_bytes(p->planes, p->Kp);
        else if (m == CL_METHOD_DIRECT && p->tc_direct) p->wpack_bytes = (size_t)d.m * kRowBytes;   // [M][32 words]
        else if (m == CL_METHOD_DIRECT) p->wpack_bytes = (size_t)d.m * d.k * d.k * d.c * 4;
        else p->wpack_bytes = (size_t)d.k * d.k * d.m * row_bytes(p->planes, p->Cp);
        if (cudaMalloc(&p->wpack, p->wpack_bytes) != cudaSuccess) {
            cudaGetLastError();
            delete p;
            throw Error(CL_ENOMEM, "packed-weight allocation failed");
        }
        if (m == CL_METHOD_DIRECT && !p->tc_direct) p->wraw = p->wpack;
        if (p->tc_direct && cudaMalloc(&p->wraw, (size_t)d.m * d.k * d.k * d.c * 4) != cudaSuccess) {
            // the raw MKKC weights too: the CUDA-core kernel serves inputs / outputs the tensor
            // core kernel's TMA maps cannot address (not 16 B aligned)
            cudaGetLastError();
            cudaFree(p->wpack);
            delete p;
            throw Error(CL_ENOMEM, "weight allocation failed");
        }
        if (p->planes == kPlanesF16) {
            const size_t sb = (size_t)kScaleBufInts * sizeof(int);
            if (cudaMalloc(&p->scale, sb) != cudaSuccess || cudaMemset(p->scale, 0, sb) != cudaSuccess) {
                cudaGetLastError();
                cudaFree(p->wpack);
                if (p->tc_direct) cudaFree(p->wraw);
                cudaFree(p->scale);
                delete p;
                throw Error(CL_ENOMEM, "scale slot allocation failed");
            }
        }
        {
            // tap-shared (padded-row) mode for the implicit kernel: one A box per kernel row feeds
            // its k taps through row-shifted descriptors (k x fewer A TMA bytes per MMA).  Small-BN
            // tiles are bound by shared-memory operand traffic (tools/mma_probe.cu: N = 64 tops out
            // at 63% even with operands resident), so cutting the A writes pays there -- VGG
            // conv1_2 1.06 -> 0.65 ms, conv2_x 0.71/0.77 -> 1.02/1.06 of peak.  The padded
            // positions are computed, then dropped.  CLB_PADDED_ROWS=0/1 forces it.
            static const int forced_padded = [] {
                const char* e = std::getenv("CLB_PADDED_ROWS");
                return e ? std::atoi(e) : -1;
            }();
            const double waste = (double)(d.h + d.pad) * (d.w + d.pad) / ((double)P * Q) - 1.0;
            // the CTA group the launch will pick for the padded geometry (a pair holds half of B)
            const int pcg = cta_group_for((long long)d.n * (d.h + d.pad) * (d.w + d.pad), d.m, p->bn);
            const bool fits = tc_num_stages(p->bn / pcg, d.k) >= 2;
            // pad <= k - 1: the P x Q outputs fit the shared-padding grid (H + pad) x (W + pad)
            const bool eligible = m == CL_METHOD_KN2ROW && d.k >= 3 && d.k <= 7 && d.stride == 1 && d.pad <= d.k - 1 && fits;
            // With the shared-padding grid ((H + pad) x (W + pad): 16 % waste at 13x13, 7 % at 28x28)
            // the tiled A boxes beat the TMA im2col loads (tools/tma_probe3.cu: im2col A + tiled B
            // deliver 37 B/clk per SM, tiled A + B 59) almost everywhere: AlexNet conv3/4 -12/-14 %,
            // VGG conv3_x/4_x -5..-9 %, GoogLeNet 7x7 layers -27 % even at 31-65 % waste.  It loses
            // only where BN = 256 meets >= 15 % waste (AlexNet conv2 / conv5: +2-3 %)
            // (profiles/r01_padded_shared_sweep.txt).
            // With the fp16 split (half the A bytes of the mixed split per MMA) the TMA im2col A loads
            // keep up at BN > 128, and the padded rows' dropped positions then cost more than they
            // save: VGG conv3_x / conv4_x -3..-5 %, AlexNet conv3 / conv4 -8 % in im2col mode
            // (profiles/r02_f16_mode_sweep.txt); at BN <= 128 padded rows still win (conv1_2 1.9x).
            const double max_waste = p->planes == kPlanesF16 ? (p->bn <= 128 ? 0.70 : -1.0)
                                                             : (p->bn <= 192 ? 0.70 : 0.10);
            p->padded_rows = eligible && (forced_padded == 1 || (forced_padded != 0 && waste <= max_waste));
            // Tap-stacked: with few output channels the MMA's N = M is small and pays a fixed
            // cost per instruction (N = 64: 51 cycles vs 32 ideal, tools/mma_probe.cu); stacking
            // the k taps of a kernel row on N (N = k x M, one A box per row, no tap shifts) and
            // doing the shift-add in the epilogue issues k x fewer, k x wider MMAs.  Single
            // column tile only (M <= 80 for k = 3, <= 48 for k = 5).  Measured: the MMA work per
            // tile halves, but these layers then wait on A delivery (latency-bound TMA loads,
            // tools/tma_probe4.cu), so k = 3 layers gain nothing (VGG conv1_2 -3 %) while the
            // 5x5 ones gain up to 9 % (GoogLeNet 4a_5x5): auto for k = 5 only.  CLB_STACKED=0/1 forces.
            static const int forced_stacked = [] {
                const char* e = std::getenv("CLB_STACKED");
                return e ? std::atoi(e) : -1;
            }();
            const int mt = round_up(d.m, 16);
            if (p->padded_rows && (d.k == 3 || d.k == 5) && mt * d.k <= 256 && forced_stacked != 0 &&
                (forced_stacked == 1 || (d.k == 5 && p->bn <= 128))) {
                p->stack_k = d.k;
                p->bn_stack = mt * d.k;
            }
            p->wp = d.w + d.pad;   // padded row width (see TcParams::tma_store for the tap-stacked one)
            // Two sub-tiles per B stage (TcParams::msub): each weight stage feeds two 128-row A
            // boxes, so the operand bytes per MMA drop by 20 % (N = 64) / 14 % (N = 128) at the
            // cost of a stage (4 instead of 6 at N = 64) and tiles twice as large.  Measured (ms,
            // tools/gpu_msub.sh): VGG conv1_2 0.556 -> 0.433, conv2_1 0.181 -> 0.166, conv2_2
            // 0.323 -> 0.305; slower where the bigger tiles leave < 2 waves (GoogLeNet 3a_3x3 0.045
            // -> 0.052, C1 0.018 -> 0.023), so auto asks for >= 4 waves.  Mixed split only (the
            // kernel instantiates it there); CLB_MSUB=1/2 forces.
            static const int forced_msub = [] {
                const char* e = std::getenv("CLB_MSUB");
                return e ? std::atoi(e) : -1;
            }();
            const long long grid_rows = (long long)d.n * (d.h + d.pad) * (d.w + d.pad);
            const bool many_tiles = grid_rows / (2LL * kTileM * pcg) >= 4LL * (num_sms() / pcg);
            if (p->padded_rows && p->stack_k == 1 && (p->planes == kPlanesMixed || p->planes == kPlanesF16) &&
                p->bn <= 128 && forced_msub != 1 &&
                (forced_msub == 2 || many_tiles))
                p->msub = 2;
        }
        // stream-K flags [kMaxGrid], self-resetting (zeroed once here)
        if (cudaMalloc(&p->flags, (kMaxGrid + 8) * sizeof(unsigned)) != cudaSuccess ||
            cudaMemset(p->flags, 0, (kMaxGrid + 8) * sizeof(unsigned)) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(p->wpack);
            if (p->tc_direct) cudaFree(p->wraw);
            cudaFree(p->scale);
            delete p;
            throw Error(CL_ENOMEM, "flag allocation failed");
        }
        *out_plan = p;
    });
}

cl_status cl_conv_set_weights(cl_plan* p, const float* d_w, void* stream) {
    return guarded([&] {
        require(p && d_w, "cl_conv_set_weights: null argument");
        CLB_CUDA(cudaSetDevice(p->device));
        auto s = static_cast<cudaStream_t>(stream);
        std::lock_guard<std::mutex> lock(p->mu);
        order_after_previous(p, s);
        const cl_conv_desc& d = p->d;
        if (is_patch_method(p->method))
            launch_rows_split(d_w, p->wpack, d.m, d.k * d.k * d.c, p->Kp, p->planes, s);   // MKKC == M x k^2C
        else if (p->tc_direct) {   // [M][k^2 C] MKKC rows -> fp16-split rows of 32, scaled by 2^ew
            launch_absmax_exp(d_w, (long long)d.m * d.k * d.k * d.c, p->scale, p->scale, s);
            launch_rows_split(d_w, p->wpack, d.m, d.k * d.k * d.c, 32, p->planes, s, p->scale);
            CLB_CUDA(cudaMemcpyAsync(p->wraw, d_w, (size_t)d.m * d.k * d.k * d.c * 4, cudaMemcpyDeviceToDevice, s));
        } else if (p->method == CL_METHOD_DIRECT) {
            CLB_CUDA(cudaMemcpyAsync(p->wpack, d_w, p->wpack_bytes, cudaMemcpyDeviceToDevice, s));
            p->wparam.clear();   // device weights: the kernels read p->wraw (stream-ordered, no host copy)
        } else {
            if (p->planes == kPlanesF16) launch_absmax_exp(d_w, (long long)d.m * d.k * d.k * d.c, p->scale, p->scale, s);
            launch_pack_weights(d_w, p->wpack, d.m, d.k, d.c, p->Cp, p->planes, s, p->stack_k > 1, p->scale);
        }
        p->weights_set = true;
        mark_done(p, s);
    });
}

cl_status cl_conv_set_weights_host(cl_plan* p, const float* h_w, void* stream) {
    return guarded([&] {
        require(p && h_w, "cl_conv_set_weights_host: null argument");
        CLB_CUDA(cudaSetDevice(p->device));
        auto s = static_cast<cudaStream_t>(stream);
        std::lock_guard<std::mutex> lock(p->mu);
        order_after_previous(p, s);
        const size_t bytes = (size_t)p->d.m * p->d.k * p->d.k * p->d.c * 4;
        void* dw = nullptr;
        CLB_CUDA(cudaMallocAsync(&dw, bytes, s));
        CLB_CUDA(cudaMemcpyAsync(dw, h_w, bytes, cudaMemcpyHostToDevice, s));
        const cl_conv_desc& d = p->d;
        if (is_patch_method(p->method))
            launch_rows_split(static_cast<float*>(dw), p->wpack, d.m, d.k * d.k * d.c, p->Kp, p->planes, s);
        else if (p->tc_direct) {
            launch_absmax_exp(static_cast<float*>(dw), (long long)d.m * d.k * d.k * d.c, p->scale, p->scale, s);
            launch_rows_split(static_cast<float*>(dw), p->wpack, d.m, d.k * d.k * d.c, 32, p->planes, s, p->scale);
            CLB_CUDA(cudaMemcpyAsync(p->wraw, dw, bytes, cudaMemcpyDeviceToDevice, s));
        } else if (p->method == CL_METHOD_DIRECT) {
            CLB_CUDA(cudaMemcpyAsync(p->wpack, dw, p->wpack_bytes, cudaMemcpyDeviceToDevice, s));
            p->wparam.clear();
            if (direct_param_shape(d.c, d.k, d.m, d.stride, p->Q)) pack_param_weights(p, h_w);
        }
        else {
            if (p->planes == kPlanesF16)
                launch_absmax_exp(static_cast<float*>(dw), (long long)d.m * d.k * d.k * d.c, p->scale, p->scale, s);
            launch_pack_weights(static_cast<float*>(dw), p->wpack, d.m, d.k, d.c, p->Cp, p->planes, s, p->stack_k > 1,
                                p->scale);
        }
        CLB_CUDA(cudaFreeAsync(dw, s));
        CLB_CUDA(cudaStreamSynchronize(s));
        p->weights_set = true;
        mark_done(p, s);
    });
}

cl_status cl_conv_output_dims(const cl_plan* p, int32_t* P, int32_t* Q) {
    if (!p || !P || !Q) return fail(CL_EINVAL, "cl_conv_output_dims: null argument");
    *P = p->P;
    *Q = p->Q;
    return CL_OK;
}

size_t cl_conv_workspace_bytes(const cl_plan* p) { return p ? ws_bytes(p) : 0; }

cl_method cl_conv_resolved_method(const cl_plan* p) { return p ? p->method : CL_METHOD_AUTO; }

const char* cl_conv_operand_split(const cl_plan* p) {
    if (!p) return "";
    if (p->method == CL_METHOD_DIRECT && !p->tc_direct) return "fp32-fma";
    switch (p->planes) {
        case 1: return "tf32";
        case 2: return "3xtf32";
        case kPlanesBf16: return "bf16";
        case kPlanesMixed: return "mixed";
        case kPlanesF16: return "3xf16";
    }
    return "";
}

cl_status cl_conv_forward(cl_plan* p, const float* d_x, float* d_y, void* d_ws, void* stream) {
    return guarded([&] {
        require(p, "cl_conv_forward: null plan");
        auto s = static_cast<cudaStream_t>(stream);
        std::lock_guard<std::mutex> lock(p->mu);
        CLB_CUDA(cudaSetDevice(p->device));
        order_after_previous(p, s);
        forward(p, d_x, d_y, d_ws, s, -1, false);
        mark_done(p, s);
    });
}

cl_status cl_conv_forward_chain(cl_plan* const* plans, const float* const* xs, float* const* ys, void* const* wss,
                                int count, void* stream) {
    return guarded([&] {
        require(plans && xs && ys && count > 0, "cl_conv_forward_chain: null argument");
        auto s = static_cast<cudaStream_t>(stream);
        for (int i = 0; i < count; ++i) {
            require(plans[i] != nullptr, "cl_conv_forward_chain: null plan");
            for (int j = 0; j < i; ++j) require(plans[j] != plans[i], "cl_conv_forward_chain: a plan appears twice");
            require(plans[i]->device == plans[0]->device, "cl_conv_forward_chain: plans on different devices");
        }
        // every plan's lock, taken in address order (two chains over the same plans never deadlock)
        std::vector<cl_plan*> order(plans, plans + count);
        std::sort(order.begin(), order.end());
        std::vector<std::unique_lock<std::mutex>> locks;
        for (cl_plan* q : order) locks.emplace_back(q->mu);
        CLB_CUDA(cudaSetDevice(plans[0]->device));
        std::vector<SplitJob> jobs(count);
        std::vector<char> chainable(count, 0);
        std::vector<void*> ws(count);
        for (int i = 0; i < count; ++i) {
            order_after_previous(plans[i], s);
            require(plans[i]->weights_set, "cl_conv_forward_chain: weights not set (cl_conv_set_weights)");
            ws[i] = resolve_ws(plans[i], wss ? wss[i] : nullptr);
            chainable[i] = chain_job(plans[i], xs[i], ws[i], &jobs[i]) ? 1 : 0;
        }
        // layer i+1's prepass rides on layer i's contraction when both use the split operand
        // format the converters write, layer i's launches are tcgen05 contractions, and layer i's
        // contraction is long enough to hide anything (estimated >= 50 us at ~400 TF: shorter ones
        // only add the tail launch -- GoogLeNet b64 6 % slower with every prepass hosted).  Hosting
        // slows the host contraction by 3-12 % (its converter warps' global traffic shares the
        // SM's load/store path with the operand stream) and hides most of the next prepass: VGG-16
        // b32 3.92 -> 3.85 ms per step (profiles/r02_chain_prepass.txt).  CLB_CHAIN_FORCE=1 hosts
        // every eligible prepass (tests); CLB_CHAIN_MIN_US sets the host threshold.
        static const double min_us = std::getenv("CLB_CHAIN_MIN_US") ? std::atof(std::getenv("CLB_CHAIN_MIN_US")) : 50.0;
        static const bool force = std::getenv("CLB_CHAIN_FORCE") && std::atoi(std::getenv("CLB_CHAIN_FORCE")) != 0;
        auto hosts = [&](int i) {
            if (!(i + 1 < count && chainable[i + 1] && plans[i]->method != CL_METHOD_DIRECT &&
                  is_split(plans[i]->planes) && plans[i]->planes == plans[i + 1]->planes))
                return false;
            if (force) return true;
            const cl_conv_desc& a = plans[i]->d;
            const double t_host_us = 2.0 * a.n * a.m * a.c * a.k * a.k * (double)plans[i]->P * plans[i]->Q / 4.0e8;
            return t_host_us >= min_us;
        };
        int i = 0;
        try {
            for (; i < count; ++i) {
                const bool partial = i > 0 && hosts(i - 1);
                forward(plans[i], xs[i], ys[i], ws[i], s, -1, false, true, true, hosts(i) ? &jobs[i + 1] : nullptr,
                        partial);
                mark_done(plans[i], s);
            }
        } catch (...) {
            // a failed layer may leave a hosted job's tile counter part-way (its tail never ran):
            // reset every counter of this chain so the next call starts clean, then report
            for (int j = 0; j < count; ++j)
                if (chainable[j]) cudaMemsetAsync(jobs[j].counter, 0, sizeof(unsigned), s);
            throw;
        }
    });
}

cl_status cl_conv_forward_nhwc(cl_plan* p, const float* d_x, float* d_y, void* d_ws, void* stream) {
    return guarded([&] {
        require(p, "cl_conv_forward_nhwc: null plan");
        auto s = static_cast<cudaStream_t>(stream);
        std::lock_guard<std::mutex> lock(p->mu);
        CLB_CUDA(cudaSetDevice(p->device));
        order_after_previous(p, s);
        forward(p, d_x, d_y, d_ws, s, -1, true);
        mark_done(p, s);
    });
}

namespace {

// Host-buffer forward, pipelined over batch chunks on three streams: H2D of chunk i+1
// (copy-in stream), the convolution of chunk i (caller's stream) and the D2H of chunk i-1
// (copy-out stream) overlap, so a call costs ~max(H2D, compute, D2H) instead of their sum
// (PCIe is full duplex).  The copy-in waits for prior work on the caller's stream in both
// modes (a previous call's host output may be this call's input: layer l's D2H into h_y must
// land before layer l+1's H2D reads it as h_x), and, through the plan's ordering, for this
// plan's previous call (its staging buffers).  sync: wait for completion on return (like
// run_method).  async: return after enqueueing; the caller's stream receives the completion,
// so independent layers issued on their own streams overlap their transfers.
cl_status host_forward(cl_plan* p, const float* h_x, float* h_y, void* stream, bool sync) {
    return guarded([&] {
        require(p && h_x && h_y, "cl_conv_forward_host: null argument");
        CLB_CUDA(cudaSetDevice(p->device));
        std::lock_guard<std::mutex> lock(p->mu);
        order_after_previous(p, static_cast<cudaStream_t>(stream));
        const cl_conv_desc& d = p->d;
        const size_t img_in = (size_t)d.c * d.h * d.w, img_out = (size_t)d.m * p->P * p->Q;
        const size_t xb = (size_t)d.n * img_in * 4;
        const size_t yb = (size_t)d.n * img_out * 4;
        if (!p->host_x) {
            if (cudaMalloc(&p->host_x, xb) != cudaSuccess || cudaMalloc(&p->host_y, yb) != cudaSuccess) {
                cudaGetLastError();
                throw Error(CL_ENOMEM, "staging allocation failed");
            }
        }
        if (!p->s_in) {
            // CLB_HOST_SHARED_STREAMS=1: copy streams shared by every plan of the device, so a
            // multi-layer step's copies run in call order (layer 1's input first) instead of all
            // layers' inputs sharing the H2D engine at once.  Measured mixed, so off by default:
            // VGG16 e2e 25.9 -> 27.5 TFLOP/s, AlexNet 60.0 -> 59.1 (profiles/r01_e2e_shared_streams.txt).
            static const bool shared = std::getenv("CLB_HOST_SHARED_STREAMS") &&
                                       std::atoi(std::getenv("CLB_HOST_SHARED_STREAMS")) == 1;
            if (shared) {
                static std::mutex smu;
                static cudaStream_t dev_in[64] = {}, dev_out[64] = {};
                std::lock_guard<std::mutex> g(smu);
                if (p->device < 0 || p->device >= 64) throw Error(CL_EINVAL, "device index out of range");
                if (!dev_in[p->device]) {
                    CLB_CUDA(cudaStreamCreateWithFlags(&dev_in[p->device], cudaStreamNonBlocking));
                    CLB_CUDA(cudaStreamCreateWithFlags(&dev_out[p->device], cudaStreamNonBlocking));
                }
                p->s_in = dev_in[p->device];
                p->s_out = dev_out[p->device];
                p->shared_streams = true;
            } else {
                CLB_CUDA(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
                CLB_CUDA(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
            }
            for (int i = 0; i < cl_plan::kMaxChunks; ++i) {
                CLB_CUDA(cudaEventCreateWithFlags(&p->ev_in[i], cudaEventDisableTiming));
                CLB_CUDA(cudaEventCreateWithFlags(&p->ev_comp[i], cudaEventDisableTiming));
            }
            CLB_CUDA(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
            CLB_CUDA(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
        }
        auto s = static_cast<cudaStream_t>(stream);
        // chunk count: 8 (measured on B200 + PCIe5: AlexNet b128 e2e 37 -> 45 -> 49 -> 51 TFLOP/s
        // for 1/2/4/8 chunks), 1 for small transfers where launch overheads dominate
        // (override: CLB_HOST_CHUNKS)
        static const int forced_chunks = [] {
            const char* e = std::getenv("CLB_HOST_CHUNKS");
            return e ? std::atoi(e) : 0;
        }();
        int chunks = forced_chunks > 0 ? forced_chunks : ((xb + yb) >= (8u << 20) ? 8 : 1);
        if (chunks > cl_plan::kMaxChunks) chunks = cl_plan::kMaxChunks;
        if (chunks > d.n) chunks = d.n;
        if (chunks < 1) chunks = 1;
        // CLB_HOST_TRACE=1: per-chunk timeline (timing events on each stream, printed per call)
        static const bool htrace = std::getenv("CLB_HOST_TRACE") && std::atoi(std::getenv("CLB_HOST_TRACE")) != 0;
        static cudaEvent_t tev[3 * cl_plan::kMaxChunks + 1] = {};
        if (htrace && !tev[0])
            for (auto& e : tev) CLB_CUDA(cudaEventCreate(&e));
        // the copy streams must not run ahead of prior work on the caller's stream (which, after
        // order_after_previous, includes this plan's previous call)
        CLB_CUDA(cudaEventRecord(p->ev_start, s));
        CLB_CUDA(cudaStreamWaitEvent(p->s_in, p->ev_start, 0));
        CLB_CUDA(cudaStreamWaitEvent(p->s_out, p->ev_start, 0));
        if (htrace) CLB_CUDA(cudaEventRecord(tev[0], s));
        // all copy-ins are enqueued first, so the H2D engine streams back to back and never
        // waits for the host to enqueue a chunk's kernels (that interleaving cost ~25% of the
        // duplex PCIe rate, measured with CLB_HOST_TRACE)
        for (int c = 0; c < chunks; ++c) {
            const int n0 = d.n * c / chunks, nc = d.n * (c + 1) / chunks - n0;
            if (nc == 0) continue;
            CLB_CUDA(cudaMemcpyAsync(p->host_x + n0 * img_in, h_x + n0 * img_in, nc * img_in * 4,
                                     cudaMemcpyHostToDevice, p->s_in));
            CLB_CUDA(cudaEventRecord(p->ev_in[c], p->s_in));
            if (htrace) CLB_CUDA(cudaEventRecord(tev[1 + 3 * c], p->s_in));
        }
        for (int c = 0; c < chunks; ++c) {
            const int n0 = d.n * c / chunks, nc = d.n * (c + 1) / chunks - n0;
            if (nc == 0) continue;
            CLB_CUDA(cudaStreamWaitEvent(s, p->ev_in[c], 0));
            forward(p, p->host_x + n0 * img_in, p->host_y + n0 * img_out, nullptr, s, nc);
            CLB_CUDA(cudaEventRecord(p->ev_comp[c], s));
            if (htrace) CLB_CUDA(cudaEventRecord(tev[2 + 3 * c], s));
            CLB_CUDA(cudaStreamWaitEvent(p->s_out, p->ev_comp[c], 0));
            CLB_CUDA(cudaMemcpyAsync(h_y + n0 * img_out, p->host_y + n0 * img_out, nc * img_out * 4,
                                     cudaMemcpyDeviceToHost, p->s_out));
            if (htrace) CLB_CUDA(cudaEventRecord(tev[3 + 3 * c], p->s_out));
        }
        CLB_CUDA(cudaEventRecord(p->ev_done, p->s_out));
        CLB_CUDA(cudaStreamWaitEvent(s, p->ev_done, 0));   // the caller's stream sees the outputs
        mark_done(p, s);
        if (sync || htrace) CLB_CUDA(cudaStreamSynchronize(s));
        if (htrace) {
            fprintf(stderr, "[clb-host] n=%d c=%d m=%d hw=%dx%d chunks=%d in %.1f MB out %.1f MB |", d.n, d.c, d.m, d.h,
                    d.w, chunks, xb / 1e6, yb / 1e6);
            float last_out = 0.0f;
            for (int c = 0; c < chunks; ++c) {
                float ti = 0, tc = 0, to = 0;
                CLB_CUDA(cudaEventElapsedTime(&ti, tev[0], tev[1 + 3 * c]));
                CLB_CUDA(cudaEventElapsedTime(&tc, tev[0], tev[2 + 3 * c]));
                CLB_CUDA(cudaEventElapsedTime(&to, tev[0], tev[3 + 3 * c]));
                fprintf(stderr, " [%d: in %.2f comp %.2f out %.2f]", c, ti, tc, to);
                last_out = to;
            }
            fprintf(stderr, " | total %.2f ms (H2D-only %.2f, D2H-only %.2f ms at 56 GB/s)\n", last_out, xb / 56e6,
                    yb / 56e6);
        }
    });
}

}  // namespace

cl_status cl_conv_forward_host(cl_plan* p, const float* h_x, float* h_y, void* stream) {
    return host_forward(p, h_x, h_y, stream, true);
}

cl_status cl_conv_forward_host_async(cl_plan* p, const float* h_x, float* h_y, void* stream) {
    return host_forward(p, h_x, h_y, stream, false);
}

int cl_conv_last_launch_count(const cl_plan* p) { return p ? p->launches : 0; }

void cl_conv_destroy(cl_plan* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    if (p->wpack) cudaFree(p->wpack);
    if (p->tc_direct && p->wraw) cudaFree(p->wraw);
    if (p->scale) cudaFree(p->scale);
    if (p->flags) cudaFree(p->flags);
    if (p->own_ws) cudaFree(p->own_ws);
    if (p->host_x) cudaFree(p->host_x);
    if (p->ev_last) cudaEventDestroy(p->ev_last);
    if (p->host_y) cudaFree(p->host_y);
    if (p->s_in) {
        if (!p->shared_streams) {   // the device's shared copy streams outlive every plan
            cudaStreamDestroy(p->s_in);
            cudaStreamDestroy(p->s_out);
        }
        for (int i = 0; i < cl_plan::kMaxChunks; ++i) {
            cudaEventDestroy(p->ev_in[i]);
            cudaEventDestroy(p->ev_comp[i]);
        }
        cudaEventDestroy(p->ev_start);
        cudaEventDestroy(p->ev_done);
    }
    delete p;
}

size_t cl_gemm_workspace_bytes(int m, int n, int k, cl_precision precision) {
    const int planes = planes_for(precision);
    const size_t kp = (size_t)round_up(k > 0 ? k : 1, k_granule(planes));
    return align256(((size_t)(m > 0 ? m : 0) + (size_t)(n > 0 ? n : 0)) * row_bytes(planes, kp)) + tc_scratch_bytes();
}

cl_status cl_gemm_f32(int m, int n, int k, const float* a, const float* b, float* c, cl_precision precision,
                      void* ws, size_t ws_bytes_, void* stream) {
    return guarded([&] {
        require(m > 0 && n > 0 && k > 0, "gemm: dimensions must be positive");
        require(a && b && c, "gemm: null operand");
        require(precision == CL_PREC_FP32 || precision == CL_PREC_TF32 || precision == CL_PREC_BF16, "unknown precision");
        int dev = 0;
        CLB_CUDA(cudaGetDevice(&dev));
        check_device(dev);
        auto s = static_cast<cudaStream_t>(stream);
        const int planes = planes_for(precision);
        const int kp = round_up(k, k_granule(planes));
        const size_t need = cl_gemm_workspace_bytes(m, n, k, precision);
        void* own = nullptr;
        if (!ws) {
            CLB_CUDA(cudaMallocAsync(&own, need, s));
            ws = own;
        } else {
            require(ws_bytes_ >= need, "gemm: workspace too small");
        }
        char* as = static_cast<char*>(ws);
        char* bs = as + (size_t)m * row_bytes(planes, kp);
        launch_rows_split(a, as, m, k, kp, planes, s);
        launch_transpose_split(b, bs, k, n, kp, planes, s);
        TcParams t{};
        t.rows = m;
        t.cols = n;
        t.bn = bn_for(n);
        t.taps = 1;
        t.ksize = 1;
        t.epi = EPI_ROWMAJOR;
        t.out = c;
        t.ld = n;
        set_scratch(t, static_cast<char*>(ws) + align256((size_t)(m + n) * row_bytes(planes, kp)));
        launch_tc(tiled(as, m, 1, kp, planes), tiled(bs, n, 1, kp, planes), t, s, cta_group_for(m, n, t.bn));
        if (own) CLB_CUDA(cudaFreeAsync(own, s));
    });
}

cl_status cl_shift_add_row(const float* inter, float* y, int n, int m, int h, int w, int k, int pad, void* stream) {
    return guarded([&] {
        require(inter && y && n > 0 && m > 0 && h > 0 && w > 0 && k > 0 && k % 2 == 1, "shift_add: bad arguments");
        if (pad < 0) pad = k / 2;
        const int P = h + 2 * pad - k + 1, Q = w + 2 * pad - k + 1;
        require(P > 0 && Q > 0, "shift_add: empty output");
        launch_shift_add_row(inter, y, n, m, h, w, k, pad, P, Q, static_cast<cudaStream_t>(stream));
    });
}

cl_status cl_fill_uniform(float* d, uint64_t n, uint64_t seed, uint64_t first_index, void* stream) {
    return guarded([&] {
        require(d || n == 0, "cl_fill_uniform: null pointer");
        launch_fill_uniform(d, n, seed, first_index, static_cast<cudaStream_t>(stream));
    });
}

cl_status cl_conv_set_peer_outputs(cl_plan* p, float* const* d_peer_y, int n_peers, int m_offset, int m_total) {
    return guarded([&] {
        require(p, "cl_conv_set_peer_outputs: null plan");
        require(n_peers >= 0 && n_peers <= kMaxPeers, "cl_conv_set_peer_outputs: 0..8 peers");
        require(n_peers == 0 || d_peer_y, "cl_conv_set_peer_outputs: null peer list");
        require(n_peers == 0 || (m_offset >= 0 && m_offset + p->d.m <= m_total),
                "cl_conv_set_peer_outputs: channel slice outside the full output");
        const bool ok_method = p->method == CL_METHOD_KN2ROW || p->method == CL_METHOD_CONV1X1 ||
                               p->method == CL_METHOD_IM2COL || p->method == CL_METHOD_IM2ROW;
        require(n_peers == 0 || (ok_method && p->stack_k == 1),
                "cl_conv_set_peer_outputs: implicit kn2row / conv1x1 / im2col plans only");
        std::lock_guard<std::mutex> lock(p->mu);
        p->peers.assign(d_peer_y, d_peer_y + n_peers);
        for (float* q : p->peers) require(q != nullptr, "cl_conv_set_peer_outputs: null peer pointer");
        p->peer_m0 = m_offset;
        p->peer_M = m_total;
    });
}

cl_status cl_ipc_get_mem_handle(const void* d_ptr, void* handle64, uint64_t* offset) {
    return guarded([&] {
        require(d_ptr && handle64 && offset, "cl_ipc_get_mem_handle: null argument");
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
        cudaIpcMemHandle_t h;
        CLB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
        std::memcpy(handle64, &h, 64);
        // the handle names the whole allocation (a caching allocator hands out pieces of one):
        // report where d_ptr sits in it, the opener adds it to the mapped base
        using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static PFN_range range = [] {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q{};
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<PFN_range>(fn);
        }();
        if (!range) throw Error(CL_ECUDA, "cuMemGetAddressRange unavailable");
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS)
            throw Error(CL_ECUDA, "cuMemGetAddressRange failed");
        *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    });
}

cl_status cl_ipc_open_mem_handle(const void* handle64, void** d_base) {
    return guarded([&] {
        require(handle64 && d_base, "cl_ipc_open_mem_handle: null argument");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, 64);
        CLB_CUDA(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

cl_status cl_ipc_close_mem_handle(void* d_base) {
    return guarded([&] { CLB_CUDA(cudaIpcCloseMemHandle(d_base)); });
}

cl_status cl_conv_set_max_sms(cl_plan* p, int max_sms) {
    if (!p) return fail(CL_EINVAL, "cl_conv_set_max_sms: null plan");
    if (max_sms < 0 || max_sms > 255) return fail(CL_EINVAL, "cl_conv_set_max_sms: cap must be in [0, 255]");
    std::lock_guard<std::mutex> lock(p->mu);
    p->max_sms = max_sms;
    return CL_OK;
}

cl_status cl_conv_set_profile_events(cl_plan* p, void* ev_begin, void* ev_end) {
    if (!p) return fail(CL_EINVAL, "cl_conv_set_profile_events: null plan");
    p->ev_begin = static_cast<cudaEvent_t>(ev_begin);
    p->ev_end = static_cast<cudaEvent_t>(ev_end);
    return CL_OK;
}

uint64_t cl_checksum_fnv1a(const float* h, uint64_t n) {
    uint64_t x = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t bits;
        std::memcpy(&bits, &h[i], 4);
        for (int sh = 0; sh < 32; sh += 8) {
            x ^= (bits >> sh) & 0xffu;
            x *= 0x100000001b3ull;
        }
    }
    return x;
}

const char* cl_last_error(void) { return g_err.c_str(); }

const char* cl_method_name(cl_method m) {
    switch (m) {
        case CL_METHOD_AUTO: return "auto";
        case CL_METHOD_KN2ROW: return "kn2row-gpu";
        case CL_METHOD_KN2ROW_EXPLICIT: return "kn2row-explicit-gpu";
        case CL_METHOD_KN2COL: return "kn2col-gpu";
        case CL_METHOD_KN2ROW_ACC: return "kn2row-acc-gpu";
        case CL_METHOD_IM2COL: return "im2col-gpu";
        case CL_METHOD_IM2ROW: return "im2row-gpu";
        case CL_METHOD_CONV1X1: return "conv1x1-gpu";
        case CL_METHOD_DIRECT: return "direct-gpu";
    }
    return "unknown";
}

int cl_method_from_name(const char* name, cl_method* out) {
    if (!name || !out) return 0;
    for (int m = CL_METHOD_AUTO; m <= CL_METHOD_IM2ROW; ++m) {
        if (std::strcmp(name, cl_method_name((cl_method)m)) == 0) {
            *out = (cl_method)m;
            return 1;
        }
    }
    return 0;
}

int cl_abi_version(void) { return CL_ABI_VERSION; }

int cl_device_count(void) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int usable = 0;
    for (int i = 0; i < count; ++i) {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, i) == cudaSuccess && major == 10)
            ++usable;
    }
    return usable;
}

}  // extern "C"
