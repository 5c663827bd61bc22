/* convlab_b200.h -- the drop-in C ABI of the B200-native kn2row / im2col hot path.
 *
 * Plain pointers and sizes only (no torch, no C++ types).  All tensors are fp32.
 * Device entry points take DEVICE pointers and a cudaStream_t passed as void*.
 * Layouts are the reference's: input NCHW (N stacked CHW images, tensor.hpp:86-90),
 * kernels MKKC ((m*k+i)*k+j)*C+c (tensor.hpp:120-125), output NCHW.
 *
 * Reference interfaces each entry point replaces (paths under /root/reference/proj/core):
 *   cl_conv_desc        <- LayerConfig{C,H,W,M,k,stride} (include/convlab/layers.hpp:12-22)
 *                          + the implicit pad = k/2 of ConvProblem (conv_direct.hpp:7-10)
 *                          + a batch dimension N (the reference has none)
 *   cl_method           <- ConvMethod (include/convlab/methods.hpp:15-23)
 *   cl_conv_plan        <- ConvProblem validation (src/conv_direct.cpp:8-21) + the
 *                          kn2row_reorder_kernel pre-pack (src/conv_kn2.cpp:28-39), done once
 *   cl_conv_forward     <- run_method(method, ConvProblem, GemmBackend) (src/methods.cpp:65-88)
 *   cl_conv_forward_host<- the same call with host buffers (run_method returns a host Tensor3)
 *   cl_gemm_f32         <- the external-GEMM plugin signature Matrix(MatrixView, MatrixView)
 *                          registered via register_gemm_backend (include/convlab/gemm.hpp:52-58)
 *   cl_shift_add_row    <- shift_add, row orientation (src/conv_kn2.cpp:78-118)
 *   cl_last_error       <- the what() text of the exceptions the reference throws
 *
 * Error behaviour mirrors the reference: contract violations (the reference's
 * std::invalid_argument) return CL_EINVAL; unsupported shapes CL_EUNSUPPORTED; CUDA
 * failures CL_ECUDA.  cl_last_error() returns the thread-local message of the last failure.
 *
 * Threading / streams (reference SPEC.md:149): entry points are reentrant.  A
 * plan may be shared by several host threads and streams: calls on one plan are serialised
 * on the host and execute on the device in call order (a call on a different stream than the
 * previous one waits for it), because the plan owns per-call state (stream-K fixup flags, its
 * default workspace, host staging).  For concurrent execution use one plan per stream.
 * Streams being captured into a CUDA graph are not chained (the graph orders them).
 * No entry point falls back to the CPU: without a usable sm_100 device they fail.
 */
#ifndef CONVLAB_B200_H
#define CONVLAB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CL_ABI_VERSION 1

#if defined(__GNUC__)
#define CL_API __attribute__((visibility("default")))
#else
#define CL_API
#endif

typedef enum cl_status {
    CL_OK = 0,
    CL_EINVAL = 1,        /* contract violation (reference: std::invalid_argument)        */
    CL_EUNSUPPORTED = 2,  /* valid but not implemented on this path                        */
    CL_ECUDA = 3,         /* CUDA runtime / driver failure                                 */
    CL_ENOMEM = 4,        /* device allocation failed (reference: bench.cpp:44-54 message) */
    CL_ENODEVICE = 5,     /* no sm_100 device visible                                      */
    CL_EINTERNAL = 6
} cl_status;

/* GPU conv methods.  The names mirror ConvMethod (methods.cpp:11-33) with a -gpu suffix. */
typedef enum cl_method {
    CL_METHOD_AUTO = 0,          /* per-layer selector ("auto")                                      */
    CL_METHOD_KN2ROW = 1,        /* implicit kn2row: k^2 shifted 1x1 GEMMs fused in one TMEM accumulator */
    CL_METHOD_KN2ROW_EXPLICIT = 2,/* paper-faithful: one (k^2 M x C).(C x NHW) GEMM + shift-add kernel */
    CL_METHOD_KN2COL = 3,        /* transposed: one (NHW x C).(C x k^2 M) GEMM + column shift-add      */
    CL_METHOD_KN2ROW_ACC = 4,    /* accumulating: k^2 shifted GEMM launches summing into the output    */
    CL_METHOD_IM2COL = 5,        /* baseline: patch matrix (NHW x k^2 C) + one GEMM                     */
    CL_METHOD_CONV1X1 = 6,       /* k == 1 only (CL_EINVAL otherwise, methods.cpp:81-85)                */
    CL_METHOD_DIRECT = 7,        /* fp32 CUDA-core direct loop nest for tiny-C layers (conv_direct.cpp:104-143) */
    CL_METHOD_IM2ROW = 8         /* reference im2row (conv_im2.cpp:56-85, 134-142): on the GPU the same K-major */
                                 /* patch-rows x weights GEMM as IM2COL (the orientations coincide there)       */
} cl_method;

typedef enum cl_precision {
    CL_PREC_FP32 = 0,  /* fp32-faithful split products (rel-L2 <= 1e-5 vs the fp32 oracle): hi*Hi tf32 + cross terms bf16; CLB_SPLIT=3xtf32: classic 3xTF32 */
    CL_PREC_TF32 = 1,  /* single TF32 pass (fast mode, 1e-2 tolerance)              */
    CL_PREC_BF16 = 2   /* BF16 operands, fp32 accumulate (fast mode, 1e-2 tolerance) */
} cl_precision;

typedef struct cl_conv_desc {
    int32_t n;       /* batch (images)                              */
    int32_t c;       /* input channels  C                           */
    int32_t h;       /* input height    H                           */
    int32_t w;       /* input width     W                           */
    int32_t m;       /* kernels         M (output channels)         */
    int32_t k;       /* kernel size (odd, as KernelSet enforces)    */
    int32_t pad;     /* zero padding; -1 = reference default k/2   */
    int32_t stride;  /* 1 (the reference rejects others: bench.cpp:90-92) */
} cl_conv_desc;

typedef struct cl_plan cl_plan;

/* Validates the descriptor, selects method/tile shape, allocates the packed-weight
 * storage on `device`.  *out_plan is owned by the caller (cl_conv_destroy). */
CL_API cl_status cl_conv_plan(const cl_conv_desc* desc, cl_method method, cl_precision precision, int device,
                       cl_plan** out_plan);

/* Uploads MKKC weights from a DEVICE pointer: one-time reorder + TF32 hi/lo split. */
CL_API cl_status cl_conv_set_weights(cl_plan* plan, const float* d_w_mkkc, void* stream);

/* Same, from a HOST pointer (H2D inside; synchronous on `stream`). */
CL_API cl_status cl_conv_set_weights_host(cl_plan* plan, const float* h_w_mkkc, void* stream);

/* Output spatial size chosen by the plan: P = (H + 2 pad - k)/stride + 1, Q likewise. */
CL_API cl_status cl_conv_output_dims(const cl_plan* plan, int32_t* p, int32_t* q);

/* Bytes of device scratch cl_conv_forward needs (split input, intermediates, patches). */
CL_API size_t cl_conv_workspace_bytes(const cl_plan* plan);

/* The method the plan resolved to (auto -> concrete). */
CL_API cl_method cl_conv_resolved_method(const cl_plan* plan);

/* The tensor-core operand format the plan computes with (no reference counterpart: the
 * reference is plain fp32):  "3xf16" (fp32-faithful fp16 split of the power-of-2 scaled
 * operands, default of the implicit kn2row family), "mixed" (fp32-faithful tf32 hi*Hi + bf16
 * cross terms), "3xtf32" (classic split), "tf32" / "bf16" (1e-2 fast modes), "fp32-fma" (the
 * direct CUDA-core kernel).  Static storage. */
CL_API const char* cl_conv_operand_split(const cl_plan* plan);

/* y[N][M][P][Q] = conv(x[N][C][H][W], w).  d_ws may be NULL: the plan then owns a lazily
 * allocated workspace.  Asynchronous on `stream`; returns after enqueueing. */
CL_API cl_status cl_conv_forward(cl_plan* plan, const float* d_x, float* d_y, void* d_ws, void* stream);

/* Channels-last variant: x is [N][H][W][C] and y is [N][P][Q][M] (the reference's HWC
 * Tensor3 layout, tensor.hpp:86-90, stacked; conv_kn2row accepts HWC input,
 * conv_kn2.cpp:147-151).  The prepass is an elementwise split (no transpose) and the output
 * rows are written contiguously.  Implicit kn2row / conv1x1 / kn2row-acc plans only
 * (CL_EUNSUPPORTED otherwise).  Asynchronous on `stream`. */
CL_API cl_status cl_conv_forward_nhwc(cl_plan* plan, const float* d_x, float* d_y, void* d_ws, void* stream);

/* A step of `count` layers on one stream, in order: y_i = conv_i(x_i) for every plan (NCHW device
 * tensors, workspaces may be NULL).  Where layer i+1 runs the standard NCHW -> split prepass and
 * layer i is a tcgen05 contraction in the same operand format, layer i's idle converter warps
 * convert tiles of x_{i+1} while its tensor pipe runs (the prepass is HBM-bound, the contraction
 * tensor-bound), and a tail launch finishes the tiles left before layer i+1's contraction.
 * Same results as `count` cl_conv_forward calls (bit-identical operand bytes).  No reference
 * counterpart (the reference runs one layer per call on the CPU). */
CL_API cl_status cl_conv_forward_chain(cl_plan* const* plans, const float* const* d_xs, float* const* d_ys,
                                       void* const* d_wss, int count, void* stream);

/* Fused output-channel all-gather (multi-GPU output-channel sharding): with
 * n_peers > 0 the plan's NCHW epilogue stores its M output channels into EACH of the n_peers
 * full [N][m_total][P][Q] tensors at channel offset m_offset -- P2P stores over NVLink /
 * NVSwitch when the pointers are CUDA-IPC mappings of the other ranks' buffers (one of them the
 * caller's own) -- instead of into the y argument of cl_conv_forward.  The gather thus overlaps
 * the contraction tile by tile; the caller synchronises the ranks (stream sync + a barrier)
 * before reading.  Implicit kn2row / conv1x1 / im2col plans; n_peers = 0 restores the default. */
CL_API cl_status cl_conv_set_peer_outputs(cl_plan* plan, float* const* d_peer_y, int n_peers, int m_offset,
                                          int m_total);

/* CUDA IPC helpers for the fused all-gather (64-byte cudaIpcMemHandle_t as opaque bytes).  The
 * handle names the whole allocation containing d_ptr; *offset is d_ptr's byte offset in it (a
 * caching allocator's tensor is a piece of a larger block): the peer opens the handle
 * (*d_base) and uses d_base + offset, and closes d_base. */
CL_API cl_status cl_ipc_get_mem_handle(const void* d_ptr, void* handle64, uint64_t* offset);
CL_API cl_status cl_ipc_open_mem_handle(const void* handle64, void** d_base);
CL_API cl_status cl_ipc_close_mem_handle(void* d_base);

/* Host-buffer end-to-end call (the run_method surface): H2D of x, forward, D2H of y,
 * synchronous.  Host buffers should be pinned for full PCIe bandwidth. */
CL_API cl_status cl_conv_forward_host(cl_plan* plan, const float* h_x, float* h_y, void* stream);

/* Asynchronous variant: returns after enqueueing (pinned host buffers recommended); `stream`
 * receives the completion (synchronise it before reading h_y).  The copy-in is ordered after
 * prior work on `stream` (so a chain of layers through host buffers on one stream is safe:
 * layer l's D2H into h_y completes before layer l+1's H2D reads it) and after this plan's
 * previous call.  Independent layers overlap their PCIe transfers when issued on their own
 * streams. */
CL_API cl_status cl_conv_forward_host_async(cl_plan* plan, const float* h_x, float* h_y, void* stream);

/* Number of GPU kernel launches the last cl_conv_forward enqueued. */
CL_API int cl_conv_last_launch_count(const cl_plan* plan);

CL_API void cl_conv_destroy(cl_plan* plan);

/* C[m x n] = A[m x k] . B[k x n], all row-major fp32 DEVICE pointers (the reference's
 * gemm() contract, gemm.hpp:34-50).  d_ws may be NULL (internal scratch is allocated). */
CL_API cl_status cl_gemm_f32(int m, int n, int k, const float* d_a, const float* d_b, float* d_c,
                      cl_precision precision, void* d_ws, size_t ws_bytes, void* stream);
CL_API size_t cl_gemm_workspace_bytes(int m, int n, int k, cl_precision precision);

/* shift_add (row orientation) on the device: inter[(k^2 M) x (N H W)] -> y NCHW with
 * output P x Q (pad = k/2 keeps P = H).  Exposed for the decomposition tests. */
CL_API cl_status cl_shift_add_row(const float* d_inter, float* d_y, int n, int m, int h, int w, int k, int pad,
                           void* stream);

/* Fills d[0..n) with the reference's counter-based generator on the device, bit-identical to
 * fill_deterministic (tensor.cpp:104-134): d[i] = unit_value(seed, first_index + i) in [-1,1).
 * Replaces random_tensor3 / random_kernels for device-resident synthetic inputs. */
CL_API cl_status cl_fill_uniform(float* d, uint64_t n, uint64_t seed, uint64_t first_index, void* stream);

/* Instrumentation: when set, cl_conv_forward records ev_begin (a cudaEvent_t) on the stream
 * right before its first tcgen05 contraction launch and ev_end right after its last, so the
 * caller can time the dominant kernel alone with CUDA events.  NULLs disable. */
CL_API cl_status cl_conv_set_profile_events(cl_plan* plan, void* ev_begin, void* ev_end);

/* Caps the SMs the plan's tcgen05 launches may occupy (0 = all co-resident units, the
 * default).  Independent layers on concurrent streams (e.g. GoogLeNet inception branches,
 * batch-1 stacks) then share the GPU instead of each filling it with a persistent grid whose
 * fixed costs (prologue, pipeline fill, stream-K tail) serialise.  Keep the caps of kernels
 * that may run at the same time within the SM count: every CTA of a launch must be
 * co-resident (its stream-K pieces wait on each other).  No reference counterpart (the
 * reference runs one layer at a time on the CPU). */
CL_API cl_status cl_conv_set_max_sms(cl_plan* plan, int max_sms);

/* fnv1a over the fp32 bit patterns of a HOST array, bytes low..high (bench.cpp:25-36): the
 * reference harness's output checksum. */
CL_API uint64_t cl_checksum_fnv1a(const float* h, uint64_t n);

CL_API const char* cl_last_error(void);
CL_API const char* cl_method_name(cl_method method);
CL_API int cl_method_from_name(const char* name, cl_method* out);
CL_API int cl_abi_version(void);

/* Number of sm_100 devices usable by this library (0 on a CPU-only host). */
CL_API int cl_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* CONVLAB_B200_H */
