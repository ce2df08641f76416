// host.cu — the C ABI (include/co.h): handle lifetime, validation, the host
// clock, kernel dispatch, forward_steps folding,
// canonical state transfer, the layer-stack driver (row a7) and the host-
// buffer entry point.  No CPU compute path exists: every value is produced by
// a CUDA kernel; if no kernel fits, the call fails with CO_ERR_UNSUPPORTED.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/co.h"
#include "common.cuh"
#include "dense_tc.cuh"
#include "stem_raw.cuh"
#include "depthwise.cuh"

using co::Geom;
using co::StepArgs;

// ----------------------------------------------------------------- errors

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CO_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return fail(e_ == cudaErrorMemoryAllocation ? CO_ERR_OOM : CO_ERR_CUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

extern "C" const char* co_last_error(void) { return g_err.c_str(); }
extern "C" int co_abi_version(void) { return CO_ABI_VERSION; }

// ----------------------------------------------------------------- options (options.cu)
int co_set_option_impl(const char* name, int64_t value, std::string& err);
int co_get_option_impl(const char* name, int64_t* value, std::string& err);
int co_option_count_impl();
const char* co_option_name_impl(int i);

extern "C" int co_set_option(const char* name, int64_t value) {
  std::string err;
  const int rc = co_set_option_impl(name, value, err);
  return rc == CO_OK ? CO_OK : fail(rc, "%s", err.c_str());
}
extern "C" int co_get_option(const char* name, int64_t* value) {
  std::string err;
  const int rc = co_get_option_impl(name, value, err);
  return rc == CO_OK ? CO_OK : fail(rc, "%s", err.c_str());
}
extern "C" const char* co_option_name(int index) { return co_option_name_impl(index); }

// ----------------------------------------------------------------- integer helpers

static inline int64_t floor_div(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}
static inline int64_t floor_mod(int64_t a, int64_t b) { return a - floor_div(a, b) * b; }
static inline int64_t ceil_div(int64_t a, int64_t b) { return -floor_div(-a, b); }
static inline size_t dsize(int dt) { return dt == co::F32 ? 4 : 2; }

// ----------------------------------------------------------------- handle

// Double-buffered H2D -> step -> D2H pipeline for the *_steps_host entry points:
// frame t+1 is copied in and output t-1 copied out while step t computes.
struct HostPipe {
  void* x[2] = {nullptr, nullptr};
  void* y[2] = {nullptr, nullptr};
  size_t xb = 0, yb = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t in_done[2] = {}, comp_done[2] = {}, out_done[2] = {};
  bool ok = false;
};

static void pipe_free(HostPipe& P) {
  for (int i = 0; i < 2; ++i) {
    cudaFree(P.x[i]); cudaFree(P.y[i]);
    if (P.in_done[i]) cudaEventDestroy(P.in_done[i]);
    if (P.comp_done[i]) cudaEventDestroy(P.comp_done[i]);
    if (P.out_done[i]) cudaEventDestroy(P.out_done[i]);
  }
  if (P.s_in) cudaStreamDestroy(P.s_in);
  if (P.s_out) cudaStreamDestroy(P.s_out);
  P = HostPipe{};
}

static cudaError_t pipe_init(HostPipe& P, size_t xb, size_t yb) {
  if (P.ok && P.xb == xb && P.yb == yb) return cudaSuccess;
  pipe_free(P);
  cudaError_t e;
  for (int i = 0; i < 2; ++i) {
    if ((e = cudaMalloc(&P.x[i], xb)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&P.y[i], yb)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&P.in_done[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&P.comp_done[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&P.out_done[i], cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  if ((e = cudaStreamCreateWithFlags(&P.s_in, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&P.s_out, cudaStreamNonBlocking)) != cudaSuccess) return e;
  P.xb = xb; P.yb = yb; P.ok = true;
  return cudaSuccess;
}

struct co_conv {
  co_conv_desc desc;
  Geom g;
  int kernel_used = CO_KERNEL_DIRECT;
  std::string kname;
  float* w_direct = nullptr;   // [kt][kh][kw][Cin/g][Cout] fp32
  float* bias = nullptr;       // (Cout) fp32, zeros when absent
  float* state = nullptr;      // R * slot_elems fp32
  int64_t n = 0;               // host clock: stateful steps since clean
  co::DenseTC* tc = nullptr;   // dense tcgen05 resources (packed weights)
  co::Depthwise* dw = nullptr; // depthwise resources
  void* hx = nullptr;          // staging for *_host
  void* hy = nullptr;
  HostPipe pipe;               // staging for co_forward_steps_host
  // per-stream clocks: stream b joined at tick join[b] (empty =
  // all joined at 0); the last step on the handle's clock: its n and readiness
  std::vector<int64_t> join;
  int64_t last_n = -1;
  int last_ready = 0;
};

struct co_stack {
  std::vector<co_conv*> layers;
  std::vector<std::vector<uint8_t>> pending;   // per layer: streams whose clean waits for their first valid input
  int last_ready = 0;
  std::vector<void*> act;      // inter-layer activations (one per layer but the last)
  void* hx = nullptr;          // staging for co_stack_step_host
  void* hy = nullptr;
  HostPipe pipe;               // staging for co_stack_steps_host
};

static int make_geom(const co_conv_desc* d, Geom& g) {
  if (!d) return fail(CO_ERR_ARG, "null descriptor");
  if (d->spatial_rank < 0 || d->spatial_rank > 2) return fail(CO_ERR_ARG, "spatial_rank must be 0, 1 or 2");
  int k[3], s[3], p[3], dl[3], in[2];
  for (int a = 0; a < 3; ++a) {
    const bool present = (a == 0) || (a <= d->spatial_rank);
    k[a] = present ? d->kernel[a] : 1;
    s[a] = present ? d->stride[a] : 1;
    p[a] = present ? d->padding[a] : 0;
    dl[a] = present ? d->dilation[a] : 1;
    if (k[a] < 1 || s[a] < 1 || dl[a] < 1 || p[a] < 0)
      return fail(CO_ERR_ARG, "axis %d: kernel/stride/dilation must be >= 1 and padding >= 0", a);
  }
  for (int a = 0; a < 2; ++a) {
    in[a] = (a < d->spatial_rank) ? d->in_spatial[a] : 1;
    if (in[a] < 1) return fail(CO_ERR_ARG, "in_spatial[%d] must be >= 1", a);
  }
  if (d->in_channels < 1 || d->out_channels < 1 || d->groups < 1)
    return fail(CO_ERR_ARG, "channels and groups must be >= 1");
  if (d->op == CO_OP_CONV && (d->in_channels % d->groups || d->out_channels % d->groups))
    return fail(CO_ERR_ARG, "groups (%d) must divide in_channels (%d) and out_channels (%d)", d->groups,
                d->in_channels, d->out_channels);
  if (d->n_streams < 1) return fail(CO_ERR_ARG, "n_streams must be >= 1");
  if (d->op == CO_OP_CONV && k[0] > CO_MAX_KT) return fail(CO_ERR_UNSUPPORTED, "temporal kernel %d > CO_MAX_KT", k[0]);
  if (int64_t(dl[0]) * (k[0] - 1) + 1 > (1 << 20)) return fail(CO_ERR_UNSUPPORTED, "receptive field > 2^20 frames");
  for (int t : {d->in_dtype, d->w_dtype, d->out_dtype})
    if (t != CO_F32 && t != CO_BF16) return fail(CO_ERR_ARG, "dtype must be CO_F32 or CO_BF16");
  if (d->w_dtype != d->in_dtype) return fail(CO_ERR_ARG, "w_dtype must equal in_dtype");
  if (d->activation != CO_ACT_NONE && d->activation != CO_ACT_RELU) return fail(CO_ERR_ARG, "bad activation");
  if (d->state_layout != CO_STATE_PSUM && d->state_layout != CO_STATE_RAW && d->state_layout != CO_STATE_AUTO)
    return fail(CO_ERR_ARG, "bad state_layout");
  if (d->op != CO_OP_CONV && d->op != CO_OP_MAX_POOL && d->op != CO_OP_AVG_POOL && d->op != CO_OP_DELAY)
    return fail(CO_ERR_ARG, "bad op");
  const bool pool = d->op != CO_OP_CONV;
  if (pool && d->in_channels != d->out_channels)
    return fail(CO_ERR_ARG, "pooling: in_channels (%d) != out_channels (%d)", d->in_channels, d->out_channels);
  g = Geom{};
  g.rank = d->spatial_rank;
  g.Cin = d->in_channels; g.Cout = d->out_channels; g.groups = pool ? d->in_channels : d->groups;
  g.cig = g.Cin / g.groups; g.cog = g.Cout / g.groups;
  g.kt = k[0]; g.kh = k[1]; g.kw = k[2];
  g.st = s[0]; g.sh = s[1]; g.sw = s[2];
  g.pt = p[0]; g.ph = p[1]; g.pw = p[2];
  g.dt = dl[0]; g.dh = dl[1]; g.dw = dl[2];
  g.H = in[0]; g.W = in[1];
  const int64_t ho = (int64_t(g.H) + 2 * g.ph - int64_t(g.dh) * (g.kh - 1) - 1);
  const int64_t wo = (int64_t(g.W) + 2 * g.pw - int64_t(g.dw) * (g.kw - 1) - 1);
  if (ho < 0 || wo < 0) return fail(CO_ERR_ARG, "spatial kernel larger than padded input");
  g.Ho = int(ho / g.sh + 1); g.Wo = int(wo / g.sw + 1);
  g.B = d->n_streams;
  g.in_dtype = d->in_dtype; g.out_dtype = d->out_dtype; g.act = d->activation;
  g.f = g.dt * (g.kt - 1) + 1;
  if (g.pt > g.f - 1) return fail(CO_ERR_ARG, "temporal padding %d > f-1 = %d (S:51)", g.pt, g.f - 1);
  g.delay = g.f - g.pt - 1;
  g.R = int(ceil_div(g.f - 1, g.st));
  g.Cq = (g.Cout + 3) / 4;
  g.HWo = int64_t(g.Ho) * g.Wo;
  g.splane = g.B * g.HWo;
  g.slot_elems = int64_t(g.Cq) * 4 * g.splane;
  g.op = d->op;
  g.raw = pool || d->state_layout == CO_STATE_RAW;   // pooling / delay always keep a frame ring
  if (!pool && d->state_layout == CO_STATE_AUTO) {
    // The planner's choice, by the bytes each layout moves per
    // stream-step -- RAW: the frame store + the window's kt frames; PSUM: the
    // 2 (kt-1) fp32 partial-sum accesses -- where the RAW tensor-core kernel is
    // the 1x1 (FLAT) one, which reaches its roofline (C5: 2.2x the PSUM
    // layout's throughput measured); spatial RAW windows stay PSUM (their K
    // pipeline is shared-memory bound at small N).
    const double raw_b = double(g.kt + 1) * double(g.H) * g.W * g.Cin * 2;
    const double psum_b = 2.0 * (g.kt - 1) * double(g.HWo) * g.Cout * 4;
    const bool flat = g.kh == 1 && g.kw == 1 && g.sh == 1 && g.sw == 1 && g.ph == 0 && g.pw == 0;
    g.raw = d->in_dtype == CO_BF16 && d->groups == 1 && flat && g.kt > 1 && 2.0 * raw_b <= psum_b &&
            g.Cin % 16 == 0 && g.Cout % 16 == 0;
    // small-Cin stems (RGB input, e.g. C4 layer 1): the RAW ring of raw frames is
    // an order of magnitude smaller than the partial sums (C4: 0.45 MB against
    // 6.4 MB per stream-step) and k_stem_raw.cu contracts the window on the
    // tensor cores with its weights resident
    co::StemRawPlan sp;
    if (!g.raw && g.kt > 1 && 2.0 * raw_b <= psum_b && co::stem_raw_plan(g, sp)) g.raw = 1;
    // temporal-only depthwise layers (C3-b): one streaming pass over the window's
    // frames with the frame store fused (k_step_dw_traw), (kt + 2) bf16 frame
    // accesses against 2 + 4 (kt - 1) for the partial sums
    if (!g.raw && d->in_dtype == CO_BF16 && flat && g.kt > 1 && 2.0 * raw_b <= psum_b && d->groups == g.Cin &&
        g.Cin == g.Cout && g.Cin % 8 == 0)
      g.raw = 1;
    // "same"-padded stride-1 depthwise stencils (C3-a): rolling row sets over the
    // window's frames (k_step_dw_rowraw), when the depthwise planner has a plan for it
    if (!g.raw && d->in_dtype == CO_BF16 && g.kt > 1 && 2.0 * raw_b <= psum_b && d->groups == g.Cin &&
        g.Cin == g.Cout && g.Cin % 8 == 0 && g.sh == 1 && g.sw == 1 && g.dh == 1 && g.dw == 1 && g.Ho == g.H &&
        g.Wo == g.W && g.kh * g.kw > 1) {
      Geom gr = g;
      gr.raw = 1;
      if (co::depthwise_raw_pipeline(gr)) g.raw = 1;
    }
  }
  if (g.op == CO_OP_DELAY) {
    if (g.kh != 1 || g.kw != 1 || g.sh != 1 || g.sw != 1 || g.ph || g.pw || g.dh != 1 || g.dw != 1 || g.pt ||
        g.st != 1 || g.dt != 1)
      return fail(CO_ERR_ARG, "delay: kernel (d+1, 1, 1), stride 1, dilation 1, padding 0");
    if (d->out_dtype != d->in_dtype) return fail(CO_ERR_ARG, "delay: out_dtype must equal in_dtype");
  }
  g.frame_elems = int64_t(g.H) * g.W * g.Cin;
  return CO_OK;
}

// Device bytes of a handle's state: the fp32 partial-sum ring (PSUM), or the
// ring of f + 1 input frames (RAW: f data slots + a scratch slot).
// Pooling handles keep f + 1 spatially reduced frames (k_pool.cu).
static size_t ring_slot_bytes(const Geom& g) {
  if (g.op != CO_OP_CONV) return size_t(co::pool_slot_elems(g)) * co::pool_ring_esz(g);
  return size_t(g.B) * g.frame_elems * dsize(g.in_dtype);
}
static size_t state_alloc_bytes(const Geom& g) {
  if (g.op != CO_OP_CONV) return size_t(co::pool_state_slots(g)) * ring_slot_bytes(g);
  if (g.raw) return size_t(g.f + 1) * ring_slot_bytes(g);
  return sizeof(float) * g.slot_elems * g.R;
}
// Canonical state bytes (co_state_bytes): PSUM (R, B, S', Cout) fp32; RAW
// (f-1, B, S, Cin) in_dtype; pooling (f-1, B, S', C) in the ring dtype.
static size_t state_canon_bytes(const Geom& g) {
  if (g.raw) return size_t(g.f - 1) * ring_slot_bytes(g);
  return sizeof(float) * size_t(g.R) * g.B * g.HWo * g.Cout;
}

// The host clock (a1 / a5): which ring slot each temporal slice of the frame at
// padded index m = n + p feeds.  Slice k of frame m contributes to output i
// with i s + k dil = m (A20); only outputs i >= 0 are ever emitted.
static int clock_args(const Geom& g, int64_t n, StepArgs& a) {
  const int64_t m = n + g.pt;
  const int ready = (n >= g.delay) && floor_mod(n - g.delay, g.st) == 0;
  for (int k = 0; k < co::kMaxKt; ++k) a.slot[k] = -1;
  for (int k = 0; k < g.kt; ++k) {
    const int64_t q = m - int64_t(k) * g.dt;
    if (floor_mod(q, g.st) != 0) continue;
    const int64_t i = floor_div(q, g.st);
    if (i < 0 || g.R == 0) continue;
    a.slot[k] = int(floor_mod(i, g.R));
  }
  a.emit = ready;
  return ready;
}

static int head_of(const Geom& g, int64_t n) {
  if (g.R == 0) return 0;
  return int(floor_mod(ceil_div(n - g.delay, g.st), g.R));
}

static bool dense_tc_fits(const Geom& g) { return co::dense_tc_supported(g); }
static bool depthwise_fits(const Geom& g) { return co::depthwise_supported(g); }

// Pooling handle (§8f f3): no weights, the RAW ring initialised to the padding
// value (0 AVG, -inf MAX), kernel CO_KERNEL_POOL.
static int create_pool(const co_conv_desc* desc, const Geom& g, const void* weights, const float* bias,
                       co_conv** out) {
  if (weights || bias) return fail(CO_ERR_ARG, "pooling takes no weights or bias");
  const int kern = g.op == CO_OP_DELAY ? CO_KERNEL_COPY : CO_KERNEL_POOL;
  if (desc->kernel_choice != CO_KERNEL_AUTO && desc->kernel_choice != kern)
    return fail(CO_ERR_UNSUPPORTED, g.op == CO_OP_DELAY ? "delay runs only on CO_KERNEL_COPY"
                                                        : "pooling runs only on CO_KERNEL_POOL");
  co_conv* h = new (std::nothrow) co_conv();
  if (!h) return fail(CO_ERR_OOM, "host allocation");
  h->desc = *desc;
  h->g = g;
  if (g.op != CO_OP_DELAY) {
    h->g.pool_G = co::pool_split_lanes(g);
    h->g.pool_vh = co::pool_block_decomposition(g);
  }
  h->kernel_used = kern;
  h->kname = g.op == CO_OP_DELAY ? std::string("ring_copy") : co::pool_kernel_name(h->g);
  const size_t sb = state_alloc_bytes(h->g);
  cudaError_t e;
  if ((e = cudaMalloc(&h->state, sb)) != cudaSuccess) {
    co_conv_destroy(h);
    return fail(CO_ERR_OOM, "state (%lld bytes): %s", (long long)sb, cudaGetErrorString(e));
  }
  if ((e = co::launch_fill_pad(h->g, h->state, int64_t(sb / co::pool_ring_esz(g)), 0)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess) {
    co_conv_destroy(h);
    return fail(CO_ERR_CUDA, "pool state init: %s", cudaGetErrorString(e));
  }
  *out = h;
  return CO_OK;
}

extern "C" int co_conv_create(const co_conv_desc* desc, const void* weights, const float* bias,
                              int weights_on_device, co_conv** out) {
  if (!out) return fail(CO_ERR_ARG, "null out");
  *out = nullptr;
  Geom g;
  if (int r = make_geom(desc, g)) return r;
  if (g.op != CO_OP_CONV) return create_pool(desc, g, weights, bias, out);
  if (!weights) return fail(CO_ERR_ARG, "null weights");
  // Dispatch rule: fp32 -> CUDA cores (TF32 would break 1e-4);
  // bf16 dense contractions -> tcgen05; bf16 depthwise -> CUDA-core stencil.
  int kern = desc->kernel_choice;
  if (kern == CO_KERNEL_AUTO) {
    if (g.in_dtype == co::BF16 && depthwise_fits(g)) kern = CO_KERNEL_DEPTHWISE;
    else if (g.in_dtype == co::BF16 && dense_tc_fits(g)) kern = CO_KERNEL_DENSE_TC;
    else kern = CO_KERNEL_DIRECT;
  }
  if (kern == CO_KERNEL_DENSE_TC && !dense_tc_fits(g))
    return fail(CO_ERR_UNSUPPORTED, "dense tcgen05 kernel does not support this layer shape/dtype");
  if (kern == CO_KERNEL_DEPTHWISE && !depthwise_fits(g))
    return fail(CO_ERR_UNSUPPORTED, "depthwise kernel does not support this layer shape/dtype");
  if (kern != CO_KERNEL_DIRECT && kern != CO_KERNEL_DENSE_TC && kern != CO_KERNEL_DEPTHWISE)
    return fail(CO_ERR_ARG, "bad kernel_choice");

  // the depthwise kernels stream a channels-last state ring, the dense tensor-core
  // kernel a tile-padded quad-major one (common.cuh)
  g.state_cl = (kern == CO_KERNEL_DEPTHWISE) ? 1 : 0;
  if (kern == CO_KERNEL_DENSE_TC) {
    co::dense_tc_state_layout(g);
    g.slot_elems = int64_t(g.Cq) * 4 * g.splane;
  }
  co_conv* h = new (std::nothrow) co_conv();
  if (!h) return fail(CO_ERR_OOM, "host allocation");
  h->desc = *desc;
  h->g = g;
  h->kernel_used = kern;
  auto cleanup = [&](int code) { co_conv_destroy(h); return code; };

  const int64_t wn = int64_t(g.Cout) * g.cig * g.kt * g.kh * g.kw;
  const size_t wbytes = size_t(wn) * dsize(g.in_dtype);
  void* wdev = nullptr;
  cudaError_t e;
  if (!weights_on_device) {
    if ((e = cudaMalloc(&wdev, wbytes)) != cudaSuccess) return cleanup(fail(CO_ERR_OOM, "weights: %s", cudaGetErrorString(e)));
    if ((e = cudaMemcpy(wdev, weights, wbytes, cudaMemcpyHostToDevice)) != cudaSuccess)
      return cleanup(fail(CO_ERR_CUDA, "weights copy: %s", cudaGetErrorString(e)));
  }
  const void* wsrc = weights_on_device ? weights : wdev;
  auto freew = [&]() { if (wdev) cudaFree(wdev); wdev = nullptr; };
  if ((e = cudaMalloc(&h->w_direct, sizeof(float) * wn)) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_OOM, "%s", cudaGetErrorString(e))); }
  if ((e = co::launch_pack_direct_weights(g, wsrc, h->w_direct, 0)) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_CUDA, "pack: %s", cudaGetErrorString(e))); }
  if ((e = cudaMalloc(&h->bias, sizeof(float) * g.Cout)) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_OOM, "%s", cudaGetErrorString(e))); }
  if (bias) {
    e = cudaMemcpy(h->bias, bias, sizeof(float) * g.Cout, weights_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  } else {
    e = cudaMemset(h->bias, 0, sizeof(float) * g.Cout);
  }
  if (e != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_CUDA, "bias: %s", cudaGetErrorString(e))); }
  if (state_alloc_bytes(g) > 0) {
    const size_t sb = state_alloc_bytes(g);
    if ((e = cudaMalloc(&h->state, sb)) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_OOM, "state (%lld bytes): %s", (long long)sb, cudaGetErrorString(e))); }
    if ((e = cudaMemset(h->state, 0, sb)) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_CUDA, "%s", cudaGetErrorString(e))); }
  }
  h->kname = "k_step_direct";
  if (kern == CO_KERNEL_DENSE_TC) {
    std::string err;
    h->tc = co::dense_tc_create(g, wsrc, err);
    if (!h->tc) { freew(); return cleanup(fail(CO_ERR_CUDA, "dense_tc_create: %s", err.c_str())); }
    h->kname = co::dense_tc_name(h->tc);
  } else if (kern == CO_KERNEL_DEPTHWISE) {
    std::string err;
    h->dw = co::depthwise_create(g, wsrc, err);
    if (!h->dw) { freew(); return cleanup(fail(CO_ERR_CUDA, "depthwise_create: %s", err.c_str())); }
    h->kname = co::depthwise_name(h->dw);
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) { freew(); return cleanup(fail(CO_ERR_CUDA, "create: %s", cudaGetErrorString(e))); }
  freew();
  *out = h;
  return CO_OK;
}

extern "C" int co_conv_destroy(co_conv* h) {
  if (!h) return CO_OK;
  if (h->tc) co::dense_tc_destroy(h->tc);
  if (h->dw) co::depthwise_destroy(h->dw);
  cudaFree(h->w_direct);
  cudaFree(h->bias);
  cudaFree(h->state);
  cudaFree(h->hx);
  cudaFree(h->hy);
  pipe_free(h->pipe);
  delete h;
  return CO_OK;
}

extern "C" int co_conv_info(const co_conv* h, co_info* info) {
  if (!h || !info) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  info->n = h->n;
  info->head = head_of(g, h->n);
  info->ring_slots = g.R;
  info->delay = g.delay;
  info->receptive_field = g.f;
  info->stride_t = g.st;
  info->padding_t = g.pt;
  info->out_spatial[0] = g.Ho;
  info->out_spatial[1] = g.Wo;
  info->kernel_used = h->kernel_used;
  info->state_layout = g.raw ? CO_STATE_RAW : CO_STATE_PSUM;
  if (g.raw) info->ring_slots = g.f - 1;
  return CO_OK;
}

extern "C" int co_delay(const co_conv* h, int64_t* delay) {
  if (!h || !delay) return fail(CO_ERR_ARG, "null argument");
  *delay = h->g.delay;
  return CO_OK;
}

extern "C" const char* co_kernel_name(const co_conv* h) { return h ? h->kname.c_str() : ""; }

// ----------------------------------------------------------------- step

static int launch_step(co_conv* h, const StepArgs& a, cudaStream_t s) {
  cudaError_t e;
  if (h->g.raw) {
    switch (h->kernel_used) {
      case CO_KERNEL_POOL: e = co::launch_step_pool(h->g, a, s); break;
      case CO_KERNEL_DENSE_TC: e = co::dense_tc_step(h->tc, h->g, a, h->bias, s); break;
      case CO_KERNEL_DEPTHWISE: e = co::depthwise_step(h->dw, h->g, a, h->bias, s); break;
      default: e = co::launch_step_direct_raw(h->g, a, h->w_direct, h->bias, s); break;
    }
    if (e != cudaSuccess) return fail(CO_ERR_CUDA, "raw step kernel %s: %s", h->kname.c_str(), cudaGetErrorString(e));
    return CO_OK;
  }
  switch (h->kernel_used) {
    case CO_KERNEL_DENSE_TC: e = co::dense_tc_step(h->tc, h->g, a, h->bias, s); break;
    case CO_KERNEL_DEPTHWISE: e = co::depthwise_step(h->dw, h->g, a, h->bias, s); break;
    default: e = co::launch_step_direct(h->g, a, h->w_direct, h->bias, s); break;
  }
  if (e != cudaSuccess) return fail(CO_ERR_CUDA, "step kernel %s: %s", h->kname.c_str(), cudaGetErrorString(e));
  return CO_OK;
}

// One clock tick on `state` (the handle's ring or a scratch copy).
// RAW layout tick: store the frame in its ring slot (or the scratch slot when
// the state must not change), then on a Ready tick contract the window's kt
// ring slots; a non-Ready tick moves one frame and launches nothing.
static int step_raw(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                    int64_t y_bstride, int update_state, int* ready, cudaStream_t s) {
  const Geom& g = h->g;
  const int64_t m = n + g.pt;
  const int r = (n >= g.delay) && floor_mod(n - g.delay, g.st) == 0;
  const int cur = update_state ? int(floor_mod(m, g.f)) : g.f;
  const size_t fb = size_t(g.frame_elems) * dsize(g.in_dtype);
  char* slot = reinterpret_cast<char*>(state) + size_t(cur) * g.B * fb;
  // a Ready step of the flat tensor-core kernel reads x itself and stores it into the
  // ring from shared memory (no separate copy of the frame); otherwise copy it here
  const bool fused = r && x && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                     ((h->kernel_used == CO_KERNEL_DENSE_TC && co::dense_tc_fuses_raw_store(h->tc, g, x_bstride)) ||
                      (h->kernel_used == CO_KERNEL_DEPTHWISE && co::depthwise_fuses_raw_store(h->dw, g, x_bstride) &&
                       (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (size_t(y_bstride) * dsize(g.out_dtype)) % 16 == 0));
  if (fused) {
  } else if (x) {
    CO_CUDA(cudaMemcpy2DAsync(slot, fb, x, size_t(x_bstride) * dsize(g.in_dtype), fb, g.B, cudaMemcpyDeviceToDevice, s));
  } else {
    CO_CUDA(cudaMemsetAsync(slot, 0, g.B * fb, s));
  }
  if (r) {
    StepArgs a;
    for (int k = 0; k < co::kMaxKt; ++k) a.slot[k] = -1;
    for (int k = 0; k + 1 < g.kt; ++k) a.slot[k] = int(floor_mod(m - int64_t(g.kt - 1 - k) * g.dt, g.f));
    a.slot[g.kt - 1] = cur;
    a.x = fused ? x : nullptr; a.x_bstride = fused ? x_bstride : g.frame_elems;
    a.raw_store = fused ? cur : -1;
    a.y = y; a.y_bstride = y_bstride;
    a.state = state;
    a.emit = 1;
    a.update = 0;
    if (int rc = launch_step(h, a, s)) return rc;
  }
  if (update_state) ++n;
  if (ready) *ready = r;
  return CO_OK;
}

// Pooling tick: one fused launch reduces the frame spatially into ring slot
// m mod f (update_state) and, when Ready, folds the window (k_pool.cu).
static int step_pool(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                     int64_t y_bstride, int update_state, int* ready, cudaStream_t s) {
  const Geom& g = h->g;
  const int64_t m = n + g.pt;
  const int r = (n >= g.delay) && floor_mod(n - g.delay, g.st) == 0;
  if (r || update_state) {
    StepArgs a;
    for (int k = 0; k < co::kMaxKt; ++k) a.slot[k] = -1;
    a.slot[0] = update_state ? int(floor_mod(m, g.f)) : -1;
    a.x = x; a.x_bstride = x_bstride;
    a.y = y; a.y_bstride = y_bstride;
    a.state = state;
    a.emit = r;
    a.update = update_state ? 1 : 0;
    a.m = m;
    if (int rc = launch_step(h, a, s)) return rc;
  }
  if (update_state) ++n;
  if (ready) *ready = r;
  return CO_OK;
}

// Delay tick (co.Delay): store the frame in ring slot n mod f
// (the scratch slot f when the state must not change), and once n >= d copy
// the frame of d ticks ago out.  Copies only: no arithmetic exists to fuse.
static int step_delay(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                      int64_t y_bstride, int update_state, int* ready, cudaStream_t s) {
  const Geom& g = h->g;
  const int r = n >= g.delay;
  const size_t es = dsize(g.in_dtype), fb = size_t(g.frame_elems) * es;
  char* ring = reinterpret_cast<char*>(state);
  const int cur = update_state ? int(floor_mod(n, g.f)) : g.f;
  char* slot = ring + size_t(cur) * g.B * fb;
  if (x) CO_CUDA(cudaMemcpy2DAsync(slot, fb, x, size_t(x_bstride) * es, fb, g.B, cudaMemcpyDeviceToDevice, s));
  else CO_CUDA(cudaMemsetAsync(slot, 0, g.B * fb, s));
  if (r) {
    const int src = g.delay == 0 ? cur : int(floor_mod(n - g.delay, g.f));
    CO_CUDA(cudaMemcpy2DAsync(y, size_t(y_bstride) * es, ring + size_t(src) * g.B * fb, fb, fb, g.B,
                              cudaMemcpyDeviceToDevice, s));
  }
  if (update_state) ++n;
  if (ready) *ready = r;
  return CO_OK;
}

static int step_dispatch(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                         int64_t y_bstride, int update_state, int* ready, cudaStream_t s);

// Every tick goes through here; ticks on the handle's own clock record n and
// readiness for the per-stream flags (co_stream_ready).
static int step_impl(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                     int64_t y_bstride, int update_state, int* ready, cudaStream_t s) {
  const int64_t n0 = n;
  int r = 0;
  if (int rc = step_dispatch(h, n, state, x, x_bstride, y, y_bstride, update_state, &r, s)) return rc;
  if (&n == &h->n) { h->last_n = n0; h->last_ready = r; }
  if (ready) *ready = r;
  return CO_OK;
}

static int step_dispatch(co_conv* h, int64_t& n, float* state, const void* x, int64_t x_bstride, void* y,
                         int64_t y_bstride, int update_state, int* ready, cudaStream_t s) {
  if (h->g.op == CO_OP_DELAY) return step_delay(h, n, state, x, x_bstride, y, y_bstride, update_state, ready, s);
  if (h->g.op != CO_OP_CONV) return step_pool(h, n, state, x, x_bstride, y, y_bstride, update_state, ready, s);
  if (h->g.raw) return step_raw(h, n, state, x, x_bstride, y, y_bstride, update_state, ready, s);
  StepArgs a;
  const int r = clock_args(h->g, n, a);
  a.x = x; a.x_bstride = x_bstride;
  a.y = y; a.y_bstride = y_bstride;
  a.state = state;
  a.update = update_state ? 1 : 0;
  if (r || update_state) {   // nothing to do on an Empty tick that does not update
    if (int rc = launch_step(h, a, s)) return rc;
  }
  if (update_state) ++n;
  if (ready) *ready = r;
  return CO_OK;
}

extern "C" int co_forward_step(co_conv* h, const void* x, void* y, int update_state, int* ready,
                               co_stream stream) {
  if (!h) return fail(CO_ERR_ARG, "null handle");
  if (!y) return fail(CO_ERR_ARG, "null y");
  const Geom& g = h->g;
  return step_impl(h, h->n, h->state, x, int64_t(g.H) * g.W * g.Cin, y, g.HWo * g.Cout, update_state, ready,
                   (cudaStream_t)stream);
}

extern "C" int co_forward_step_host(co_conv* h, const void* x_host, void* y_host, int update_state, int* ready,
                                    co_stream stream) {
  if (!h || !y_host) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  const size_t xb = size_t(g.B) * g.H * g.W * g.Cin * dsize(g.in_dtype);
  const size_t yb = size_t(g.B) * g.HWo * g.Cout * dsize(g.out_dtype);
  if (!h->hx) CO_CUDA(cudaMalloc(&h->hx, xb));
  if (!h->hy) CO_CUDA(cudaMalloc(&h->hy, yb));
  cudaStream_t s = (cudaStream_t)stream;
  if (x_host) CO_CUDA(cudaMemcpyAsync(h->hx, x_host, xb, cudaMemcpyHostToDevice, s));
  int r = 0;
  if (int rc = step_impl(h, h->n, h->state, x_host ? h->hx : nullptr, int64_t(g.H) * g.W * g.Cin, h->hy,
                         g.HWo * g.Cout, update_state, &r, s))
    return rc;
  if (r) CO_CUDA(cudaMemcpyAsync(y_host, h->hy, yb, cudaMemcpyDeviceToHost, s));
  CO_CUDA(cudaStreamSynchronize(s));
  if (ready) *ready = r;
  return CO_OK;
}

// The pipelined host loop shared by co_forward_steps_host / co_stack_steps_host.
// `tick(x_dev, y_dev, &ready, stream)` runs one step; frames are time-major on
// the host.  Output r (the r-th Ready tick) lands at y_host + r * yb.
template <typename Tick>
static int run_steps_host(HostPipe& P, const void* x_host, int64_t T, void* y_host, size_t xb, size_t yb,
                          uint8_t* ready_mask, int64_t* n_ready, cudaStream_t s, Tick tick) {
  if (cudaError_t e = pipe_init(P, xb, yb)) return fail(e == cudaErrorMemoryAllocation ? CO_ERR_OOM : CO_ERR_CUDA,
                                                         "host pipeline: %s", cudaGetErrorString(e));
  int64_t r = 0;
  for (int64_t t = 0; t < T; ++t) {
    const int b = int(t & 1);
    // x[b] may be overwritten once step t-2 has consumed it
    if (t >= 2) CO_CUDA(cudaStreamWaitEvent(P.s_in, P.comp_done[b], 0));
    CO_CUDA(cudaMemcpyAsync(P.x[b], static_cast<const char*>(x_host) + size_t(t) * xb, xb, cudaMemcpyHostToDevice,
                            P.s_in));
    CO_CUDA(cudaEventRecord(P.in_done[b], P.s_in));
    CO_CUDA(cudaStreamWaitEvent(s, P.in_done[b], 0));
    if (t >= 2) CO_CUDA(cudaStreamWaitEvent(s, P.out_done[b], 0));   // y[b] copied out
    int rd = 0;
    if (int rc = tick(P.x[b], P.y[b], &rd, s)) return rc;
    CO_CUDA(cudaEventRecord(P.comp_done[b], s));
    if (rd) {
      CO_CUDA(cudaStreamWaitEvent(P.s_out, P.comp_done[b], 0));
      CO_CUDA(cudaMemcpyAsync(static_cast<char*>(y_host) + size_t(r) * yb, P.y[b], yb, cudaMemcpyDeviceToHost,
                              P.s_out));
      ++r;
    }
    CO_CUDA(cudaEventRecord(P.out_done[b], P.s_out));
    if (ready_mask) ready_mask[t] = uint8_t(rd);
  }
  CO_CUDA(cudaStreamSynchronize(P.s_out));
  CO_CUDA(cudaStreamSynchronize(s));
  if (n_ready) *n_ready = r;
  return CO_OK;
}

extern "C" int co_forward_steps_host(co_conv* h, const void* x_host, int64_t T, void* y_host, uint8_t* ready_mask,
                                     int64_t* n_ready, co_stream stream) {
  if (!h || (!x_host && T > 0) || T < 0) return fail(CO_ERR_ARG, "bad argument");
  const Geom& g = h->g;
  int64_t cap = 0;
  co_steps_ready_count(h, T, 0, &cap);
  if (cap > 0 && !y_host) return fail(CO_ERR_ARG, "null y_host");
  const size_t xb = size_t(g.B) * g.H * g.W * g.Cin * dsize(g.in_dtype);
  const size_t yb = size_t(g.B) * g.HWo * g.Cout * dsize(g.out_dtype);
  return run_steps_host(h->pipe, x_host, T, y_host, xb, yb, ready_mask, n_ready, (cudaStream_t)stream,
                        [&](const void* x, void* y, int* rd, cudaStream_t s) {
                          return step_impl(h, h->n, h->state, x, int64_t(g.H) * g.W * g.Cin, y, g.HWo * g.Cout, 1,
                                           rd, s);
                        });
}

extern "C" int co_steps_ready_count(const co_conv* h, int64_t T, int pad_end, int64_t* n_ready) {
  if (!h || !n_ready || T < 0) return fail(CO_ERR_ARG, "bad argument");
  const Geom& g = h->g;
  const int64_t total = T + (pad_end ? g.pt : 0);
  int64_t c = 0;
  for (int64_t t = 0; t < total; ++t) {
    const int64_t n = h->n + t;
    c += (n >= g.delay) && floor_mod(n - g.delay, g.st) == 0;
  }
  *n_ready = c;
  return CO_OK;
}

extern "C" int co_forward_steps(co_conv* h, const void* x, int64_t T, void* y, uint8_t* ready_mask,
                                int64_t* n_ready, int pad_end, int update_state, co_stream stream) {
  if (!h || (!x && T > 0) || T < 0) return fail(CO_ERR_ARG, "bad argument");
  const Geom& g = h->g;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t cap = 0;
  co_steps_ready_count(h, T, pad_end, &cap);
  if (cap > 0 && !y) return fail(CO_ERR_ARG, "null y");
  const int64_t frame = int64_t(g.H) * g.W * g.Cin;
  const int64_t oframe = g.HWo * g.Cout;
  const size_t isz = dsize(g.in_dtype), osz = dsize(g.out_dtype);
  // update_state = 0: run the fold on a scratch copy of the ring and clock.
  float* state = h->state;
  int64_t n = h->n;
  float* scratch = nullptr;
  if (!update_state && state_alloc_bytes(g) > 0) {
    CO_CUDA(cudaMallocAsync((void**)&scratch, state_alloc_bytes(g), s));
    CO_CUDA(cudaMemcpyAsync(scratch, h->state, state_alloc_bytes(g), cudaMemcpyDeviceToDevice, s));
    state = scratch;
  }
  int64_t& clock = update_state ? h->n : n;
  const int64_t total = T + (pad_end ? g.pt : 0);
  int64_t r_count = 0;
  int rc = CO_OK;
  if (total == T && T > 1 && h->kernel_used == CO_KERNEL_DENSE_TC && co::dense_tc_chunkable(h->tc, g)) {
    // chunked tensor-core steps: chunks of Tc frames, one launch each, item-batch-
    // major so each tile's state stays L2-resident across its frames (§8f f2);
    // FLAT stages a chunk time-major, so Tc bounds that copy to ~1 GB
    const int64_t frame_bytes = g.B * g.frame_elems * int64_t(dsize(g.in_dtype));
    int64_t Tc = std::max<int64_t>(1, std::min<int64_t>({T, 256, (int64_t(1) << 30) / std::max<int64_t>(frame_bytes, 1)}));
    if (const int64_t e = co::option(co::OPT_CHUNK_T)) Tc = std::max<int64_t>(1, std::min<int64_t>(Tc, e));   // option "chunk_t"
    constexpr int kTick = 2 + co::kMaxKt;
    std::vector<int> ticks(size_t(Tc) * kTick);
    int* dticks = nullptr;
    if (cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&dticks), ticks.size() * sizeof(int), s)) {
      if (scratch) cudaFreeAsync(scratch, s);
      return fail(CO_ERR_OOM, "tick table: %s", cudaGetErrorString(e));
    }
    int last = 0;
    for (int64_t t0 = 0; t0 < T && rc == CO_OK; t0 += Tc) {
      const int64_t tn = std::min(Tc, T - t0);
      const int64_t oi0 = r_count;
      for (int64_t t = 0; t < tn; ++t) {
        StepArgs a;
        const int r = clock_args(g, clock + t, a);
        int* tk = ticks.data() + t * kTick;
        tk[0] = r;
        tk[1] = int(r_count - oi0);
        for (int k = 0; k < co::kMaxKt; ++k) tk[2 + k] = a.slot[k];
        if (ready_mask) ready_mask[t0 + t] = uint8_t(r);
        r_count += r;
        last = r;
      }
      cudaError_t e = cudaMemcpyAsync(dticks, ticks.data(), size_t(tn) * kTick * sizeof(int), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess)
        e = co::dense_tc_steps(h->tc, g, static_cast<const char*>(x) + size_t(t0) * frame * isz, tn, T, dticks,
                               static_cast<char*>(y) + size_t(oi0) * oframe * osz, cap * oframe, state, h->bias, s);
      if (e != cudaSuccess) rc = fail(CO_ERR_CUDA, "chunked dense steps: %s", cudaGetErrorString(e));
      clock += tn;
    }
    cudaFreeAsync(dticks, s);
    if (scratch) cudaFreeAsync(scratch, s);
    if (rc) return rc;
    if (update_state) { h->last_n = clock - 1; h->last_ready = last; }
    if (n_ready) *n_ready = r_count;
    return CO_OK;
  }
  if (total > 0 && h->kernel_used == CO_KERNEL_DEPTHWISE && co::depthwise_chunkable(h->dw, g)) {
    // chunked: the whole fold in one launch, state in registers
    cudaError_t e = co::depthwise_steps(h->dw, g, x, T, total, clock, y, cap * oframe, state, h->bias, s);
    if (scratch) cudaFreeAsync(scratch, s);
    if (e != cudaSuccess) return fail(CO_ERR_CUDA, "chunked steps: %s", cudaGetErrorString(e));
    int last = 0;
    for (int64_t t = 0; t < total; ++t) {
      last = (clock + t) >= g.delay;
      if (ready_mask) ready_mask[t] = uint8_t(last);
      r_count += last;
    }
    if (update_state) { h->last_n = clock + total - 1; h->last_ready = last; }
    clock += total;
    if (n_ready) *n_ready = r_count;
    return CO_OK;
  }
  for (int64_t t = 0; t < total && rc == CO_OK; ++t) {
    const void* xt = (t < T) ? static_cast<const char*>(x) + size_t(t) * frame * isz : nullptr;
    void* yt = static_cast<char*>(y) + size_t(r_count) * oframe * osz;
    int r = 0;
    rc = step_impl(h, clock, state, xt, T * frame, r_count < cap ? yt : nullptr, cap * oframe, 1, &r, s);
    if (ready_mask) ready_mask[t] = uint8_t(r);
    r_count += r;
  }
  if (scratch) cudaFreeAsync(scratch, s);
  if (rc) return rc;
  if (n_ready) *n_ready = r_count;
  return CO_OK;
}

extern "C" int co_forward_out_len(const co_conv* h, int64_t T, int64_t* T_out) {
  if (!h || !T_out) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  *T_out = g.op == CO_OP_DELAY ? T : floor_div(T + 2 * g.pt - g.f, g.st) + 1;   // batch Delay: identity
  return CO_OK;
}

extern "C" int co_forward(co_conv* h, const void* x, int64_t T, void* y, int64_t* T_out, co_stream stream) {
  if (!h || !x || !y) return fail(CO_ERR_ARG, "null argument");
  int64_t Tp = 0;
  co_forward_out_len(h, T, &Tp);
  if (Tp < 1) return fail(CO_ERR_LENGTH, "T' = %lld < 1 (T = %lld too short, S:63-65)", (long long)Tp, (long long)T);
  cudaError_t e = h->kernel_used == CO_KERNEL_COPY
                      ? cudaMemcpyAsync(y, x, size_t(h->g.B) * T * h->g.frame_elems * dsize(h->g.in_dtype),
                                        cudaMemcpyDeviceToDevice, (cudaStream_t)stream)
                  : h->kernel_used == CO_KERNEL_POOL
                      ? co::launch_forward_pool(h->g, x, T, y, Tp, (cudaStream_t)stream)
                      : co::launch_forward_direct(h->g, x, T, y, Tp, h->w_direct, h->bias, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(CO_ERR_CUDA, "forward kernel: %s", cudaGetErrorString(e));
  if (T_out) *T_out = Tp;
  return CO_OK;
}

// ----------------------------------------------------------------- state

extern "C" int co_state_bytes(const co_conv* h, size_t* bytes) {
  if (!h || !bytes) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  *bytes = state_canon_bytes(g);
  return CO_OK;
}

extern "C" int co_state_get(co_conv* h, void* dst, size_t bytes, co_info* meta, co_stream stream) {
  if (!h) return fail(CO_ERR_ARG, "null handle");
  size_t need = 0;
  co_state_bytes(h, &need);
  if (bytes != need) return fail(CO_ERR_SHAPE, "state bytes %zu != %zu", bytes, need);
  const Geom& g = h->g;
  if (need && g.raw) {   // canonical slot j = padded frame m-(f-1)+j, m = n + p
    if (!dst) return fail(CO_ERR_ARG, "null dst");
    const size_t sb = ring_slot_bytes(g);
    for (int j = 0; j < g.f - 1; ++j) {
      const int src = int(floor_mod(h->n + g.pt - (g.f - 1) + j, g.f));
      CO_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + j * sb, reinterpret_cast<char*>(h->state) + src * sb, sb,
                              cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    }
  } else if (need) {
    if (!dst) return fail(CO_ERR_ARG, "null dst");
    const int64_t i_next = ceil_div(h->n - g.delay, g.st);
    cudaError_t e = co::launch_state_get(g, h->state, (float*)dst, head_of(g, h->n), i_next, h->n + g.pt,
                                         (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(CO_ERR_CUDA, "state_get: %s", cudaGetErrorString(e));
  }
  if (meta) co_conv_info(h, meta);
  return CO_OK;
}

extern "C" int co_state_set(co_conv* h, const void* src, size_t bytes, const co_info* meta, co_stream stream) {
  if (!h || !meta) return fail(CO_ERR_ARG, "null argument");
  size_t need = 0;
  co_state_bytes(h, &need);
  if (bytes != need) return fail(CO_ERR_SHAPE, "state bytes %zu != %zu", bytes, need);
  const Geom& g = h->g;
  if (meta->ring_slots != (g.raw ? g.f - 1 : g.R) || meta->delay != g.delay || meta->stride_t != g.st ||
      meta->receptive_field != g.f || meta->out_spatial[0] != g.Ho || meta->out_spatial[1] != g.Wo || meta->n < 0)
    return fail(CO_ERR_SHAPE, "state meta does not match this layer");
  if (need && g.raw) {
    if (!src) return fail(CO_ERR_ARG, "null src");
    const size_t sb = ring_slot_bytes(g);
    for (int j = 0; j < g.f - 1; ++j) {
      const int dstslot = int(floor_mod(meta->n + g.pt - (g.f - 1) + j, g.f));
      CO_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(h->state) + dstslot * sb, static_cast<const char*>(src) + j * sb,
                              sb, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    }
    if (g.op != CO_OP_CONV)   // derived block-decomposition state (k_pool.cu)
      CO_CUDA(co::launch_pool_rebuild(g, h->state, meta->n + g.pt, (cudaStream_t)stream));
  } else if (need) {
    if (!src) return fail(CO_ERR_ARG, "null src");
    cudaError_t e = co::launch_state_set(g, h->state, (const float*)src, head_of(g, meta->n), (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(CO_ERR_CUDA, "state_set: %s", cudaGetErrorString(e));
  }
  h->n = meta->n;
  h->join.clear();          // per-stream join ticks are not part of the canonical state
  h->last_n = -1;
  h->last_ready = 0;
  return CO_OK;
}

extern "C" int co_state_clean(co_conv* h, co_stream stream) {
  if (!h) return fail(CO_ERR_ARG, "null handle");
  const Geom& g = h->g;
  if (g.op != CO_OP_CONV)
    CO_CUDA(co::launch_fill_pad(g, h->state, int64_t(state_alloc_bytes(g) / co::pool_ring_esz(g)), (cudaStream_t)stream));
  else if (state_alloc_bytes(g) > 0)
    CO_CUDA(cudaMemsetAsync(h->state, 0, state_alloc_bytes(g), (cudaStream_t)stream));
  h->n = 0;
  h->join.clear();
  h->last_n = -1;
  h->last_ready = 0;
  return CO_OK;
}

// ----------------------------------------------------------------- stack

extern "C" int co_stack_create(co_conv* const* layers, int n_layers, co_stack** out) {
  if (!layers || n_layers < 1 || !out) return fail(CO_ERR_ARG, "bad argument");
  *out = nullptr;
  for (int l = 0; l < n_layers; ++l)
    if (!layers[l]) return fail(CO_ERR_ARG, "null layer %d", l);
  for (int l = 0; l + 1 < n_layers; ++l) {
    const Geom& a = layers[l]->g;
    const Geom& b = layers[l + 1]->g;
    if (a.B != b.B || a.Cout != b.Cin || a.Ho != b.H || a.Wo != b.W || a.out_dtype != b.in_dtype)
      return fail(CO_ERR_SHAPE, "layer %d output (B=%lld C=%d %dx%d dt=%d) != layer %d input (B=%lld C=%d %dx%d dt=%d)",
                  l, (long long)a.B, a.Cout, a.Ho, a.Wo, a.out_dtype, l + 1, (long long)b.B, b.Cin, b.H, b.W, b.in_dtype);
  }
  co_stack* st = new (std::nothrow) co_stack();
  if (!st) return fail(CO_ERR_OOM, "host allocation");
  st->layers.assign(layers, layers + n_layers);
  for (int l = 0; l + 1 < n_layers; ++l) {
    const Geom& a = layers[l]->g;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, size_t(a.B) * a.HWo * a.Cout * dsize(a.out_dtype));
    if (e != cudaSuccess) { co_stack_destroy(st); return fail(CO_ERR_OOM, "stack activation: %s", cudaGetErrorString(e)); }
    st->act.push_back(p);
  }
  *out = st;
  return CO_OK;
}

extern "C" int co_stack_destroy(co_stack* st) {
  if (!st) return CO_OK;
  for (void* p : st->act) cudaFree(p);
  cudaFree(st->hx);
  pipe_free(st->pipe);
  cudaFree(st->hy);
  delete st;
  return CO_OK;
}

extern "C" int co_stack_step(co_stack* st, const void* x, void* y, int update_state, int* ready, co_stream stream) {
  if (!st || !y) return fail(CO_ERR_ARG, "null argument");
  const void* cur = x;
  const int L = int(st->layers.size());
  st->last_ready = 0;
  for (int l = 0; l < L; ++l) {
    void* out = (l + 1 < L) ? st->act[l] : y;
    if (l > 0 && update_state && !st->pending.empty() && !st->pending[l].empty()) {
      // a joined stream reaches layer l with its first valid input: clean it here now
      std::vector<uint8_t>& pend = st->pending[l];
      std::vector<uint8_t> prev(pend.size()), mask(pend.size(), 0);
      co_stream_ready(st->layers[l - 1], prev.data());
      if (st->pending[l - 1].size() == prev.size())   // still waiting below: not a valid input yet
        for (size_t b = 0; b < prev.size(); ++b) prev[b] &= st->pending[l - 1][b] ? 0 : 1;
      bool any = false, left = false;
      for (size_t b = 0; b < pend.size(); ++b) {
        if (pend[b] && prev[b]) { mask[b] = 1; pend[b] = 0; any = true; }
        left |= pend[b] != 0;
      }
      if (any)
        if (int rc = co_state_clean_streams(st->layers[l], mask.data(), stream)) return rc;
      if (!left) pend.clear();
    }
    int r = 0;
    if (int rc = co_forward_step(st->layers[l], cur, out, update_state, &r, stream)) return rc;
    if (!r) {   // Empty ends the tick; downstream layers are not advanced
      if (ready) *ready = 0;
      return CO_OK;
    }
    cur = out;
  }
  st->last_ready = 1;
  if (ready) *ready = 1;
  return CO_OK;
}

extern "C" int co_stack_step_host(co_stack* st, const void* x_host, void* y_host, int update_state, int* ready,
                                  co_stream stream) {
  if (!st || !x_host || !y_host) return fail(CO_ERR_ARG, "null argument");
  const Geom& g0 = st->layers.front()->g;
  const Geom& gl = st->layers.back()->g;
  const size_t xb = size_t(g0.B) * g0.H * g0.W * g0.Cin * dsize(g0.in_dtype);
  const size_t yb = size_t(gl.B) * gl.HWo * gl.Cout * dsize(gl.out_dtype);
  if (!st->hx) CO_CUDA(cudaMalloc(&st->hx, xb));
  if (!st->hy) CO_CUDA(cudaMalloc(&st->hy, yb));
  cudaStream_t s = (cudaStream_t)stream;
  CO_CUDA(cudaMemcpyAsync(st->hx, x_host, xb, cudaMemcpyHostToDevice, s));
  int r = 0;
  if (int rc = co_stack_step(st, st->hx, st->hy, update_state, &r, stream)) return rc;
  if (r) CO_CUDA(cudaMemcpyAsync(y_host, st->hy, yb, cudaMemcpyDeviceToHost, s));
  CO_CUDA(cudaStreamSynchronize(s));
  if (ready) *ready = r;
  return CO_OK;
}

extern "C" int co_stack_steps_host(co_stack* st, const void* x_host, int64_t T, void* y_host, uint8_t* ready_mask,
                                   int64_t* n_ready, co_stream stream) {
  if (!st || (!x_host && T > 0) || T < 0 || !y_host) return fail(CO_ERR_ARG, "bad argument");
  const Geom& g0 = st->layers.front()->g;
  const Geom& gl = st->layers.back()->g;
  const size_t xb = size_t(g0.B) * g0.H * g0.W * g0.Cin * dsize(g0.in_dtype);
  const size_t yb = size_t(gl.B) * gl.HWo * gl.Cout * dsize(gl.out_dtype);
  return run_steps_host(st->pipe, x_host, T, y_host, xb, yb, ready_mask, n_ready, (cudaStream_t)stream,
                        [&](const void* x, void* y, int* rd, cudaStream_t s) {
                          return co_stack_step(st, x, y, 1, rd, (co_stream)s);
                        });
}

extern "C" int co_stack_delay(const co_stack* st, int64_t* d_nn) {
  if (!st || !d_nn) return fail(CO_ERR_ARG, "null argument");
  // Principle 6 in the worked-example reading (A3).
  int64_t s_acc = 0, p_acc = 0, f_acc = 0;
  for (size_t l = 0; l < st->layers.size(); ++l) {
    const Geom& g = st->layers[l]->g;
    if (l == 0) { s_acc = g.st; p_acc = g.pt; f_acc = g.f; }
    else { p_acc += int64_t(g.pt) * s_acc; f_acc += int64_t(g.f - 1) * s_acc; s_acc *= g.st; }
  }
  *d_nn = f_acc - p_acc - 1;
  return CO_OK;
}

extern "C" int co_stack_clean(co_stack* st, co_stream stream) {
  if (!st) return fail(CO_ERR_ARG, "null stack");
  st->pending.clear();
  st->last_ready = 0;
  for (co_conv* h : st->layers)
    if (int rc = co_state_clean(h, stream)) return rc;
  return CO_OK;
}

// ----------------------------------------------------------------- residual
// Residual(body) with Sum (Listing 3; SPEC
// S:452-458).  The body runs as a co_stack; the identity branch is a ring of
// d_skip + 1 input frames (+ one scratch slot for update_state = 0), and the
// merge is one streaming add kernel over the body's output (k_compose.cu).

struct co_residual {
  co_stack* stack = nullptr;
  std::vector<co_conv*> body;
  int shrink = 0, act = 0;
  int64_t f_acc = 0, d_body = 0, d_skip = 0, p_acc = 0;
  int64_t n = 0;
  void* ring = nullptr;
  int in_dtype = 0, out_dtype = 0;
  int64_t B = 0, frame_elems = 0;     // input frame (H, W, C) elements per stream; the output has the same
};

extern "C" int co_residual_create(co_conv* const* body, int n_layers, int shrink, int activation,
                                  co_residual** out) {
  if (!out || !body || n_layers < 1) return fail(CO_ERR_ARG, "bad argument");
  *out = nullptr;
  if (activation != CO_ACT_NONE && activation != CO_ACT_RELU) return fail(CO_ERR_ARG, "bad activation");
  co_stack* st = nullptr;
  if (int rc = co_stack_create(body, n_layers, &st)) return rc;
  auto bail = [&](int code) { co_stack_destroy(st); return code; };
  // Principle 6 (A3): accumulated stride, padding and receptive field of the body
  int64_t s_acc = 1, p_acc = 0, f_acc = 1;
  for (int l = 0; l < n_layers; ++l) {
    const Geom& g = body[l]->g;
    p_acc += int64_t(g.pt) * s_acc;
    f_acc += int64_t(g.f - 1) * s_acc;
    s_acc *= g.st;
  }
  if (s_acc != 1) return bail(fail(CO_ERR_SHAPE, "residual body must keep the frame rate (s_acc = %lld)", (long long)s_acc));
  const Geom& a = body[0]->g;
  const Geom& z = body[n_layers - 1]->g;
  if (a.Cin != z.Cout || a.H != z.Ho || a.W != z.Wo)
    return bail(fail(CO_ERR_SHAPE, "residual body must keep channels and spatial shape (%d %dx%d -> %d %dx%d)", a.Cin,
                     a.H, a.W, z.Cout, z.Ho, z.Wo));
  const int64_t d_body = f_acc - p_acc - 1;
  int64_t d_skip;
  if (shrink) {
    if (f_acc % 2 == 0) return bail(fail(CO_ERR_SHAPE, "centered residual needs an odd receptive field (f = %lld)", (long long)f_acc));
    d_skip = (f_acc - 1) / 2;
    if (d_skip > d_body) return bail(fail(CO_ERR_SHAPE, "centered residual: body padding exceeds (f-1)/2"));
  } else {
    if (2 * p_acc != f_acc - 1)
      return bail(fail(CO_ERR_SHAPE, "residual without shrink needs equal padding (2 p_acc = %lld != f_acc - 1 = %lld)",
                       (long long)(2 * p_acc), (long long)(f_acc - 1)));
    d_skip = d_body;
  }
  co_residual* r = new (std::nothrow) co_residual();
  if (!r) return bail(fail(CO_ERR_OOM, "host allocation"));
  r->stack = st;
  r->body.assign(body, body + n_layers);
  r->shrink = shrink ? 1 : 0;
  r->act = activation;
  r->f_acc = f_acc; r->d_body = d_body; r->d_skip = d_skip; r->p_acc = p_acc;
  r->in_dtype = a.in_dtype; r->out_dtype = z.out_dtype;
  r->B = a.B; r->frame_elems = a.frame_elems;
  {
    const size_t bytes = size_t(d_skip + 2) * r->B * r->frame_elems * dsize(r->in_dtype);
    cudaError_t e = cudaMalloc(&r->ring, bytes);
    if (e == cudaSuccess) e = cudaMemset(r->ring, 0, bytes);
    if (e != cudaSuccess) { co_residual_destroy(r); return fail(CO_ERR_OOM, "residual ring: %s", cudaGetErrorString(e)); }
  }
  *out = r;
  return CO_OK;
}

extern "C" int co_residual_destroy(co_residual* r) {
  if (!r) return CO_OK;
  co_stack_destroy(r->stack);
  cudaFree(r->ring);
  delete r;
  return CO_OK;
}

extern "C" int co_residual_step(co_residual* r, const void* x, void* y, int update_state, int* ready,
                                co_stream stream) {
  if (!r || !y) return fail(CO_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t fb = size_t(r->B) * r->frame_elems * dsize(r->in_dtype);
  // the identity branch: frame n goes to ring slot n mod (d_skip + 1) (the
  // scratch slot d_skip + 1 when the state must not change; a padding step,
  // x == NULL, stores zeros), the merge reads frame n - d_skip
  char* ring = static_cast<char*>(r->ring);
  const int64_t R = r->d_skip + 1;
  char* cur = ring + size_t(update_state ? floor_mod(r->n, R) : R) * fb;
  if (x) CO_CUDA(cudaMemcpyAsync(cur, x, fb, cudaMemcpyDeviceToDevice, s));
  else CO_CUDA(cudaMemsetAsync(cur, 0, fb, s));
  const void* skip = r->d_skip == 0 ? cur : ring + size_t(floor_mod(r->n - r->d_skip, R)) * fb;
  int rb = 0;
  if (int rc = co_stack_step(r->stack, x, y, update_state, &rb, stream)) return rc;
  if (rb)
    CO_CUDA(co::launch_residual_add(r->out_dtype, y, r->frame_elems, r->in_dtype, skip, r->frame_elems, r->B,
                                    r->frame_elems, r->act, s));
  if (update_state) ++r->n;
  if (ready) *ready = rb;
  return CO_OK;
}

// Batch forward of a layer sequence (stream-ordered temporaries between layers).
static int layers_forward(const std::vector<co_conv*>& layers, const void* x, int64_t T, void* y, int64_t* T_out,
                          co_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const void* cur = x;
  int64_t Tc = T;
  void* tmp_prev = nullptr;
  const int L = int(layers.size());
  for (int l = 0; l < L; ++l) {
    co_conv* h = layers[l];
    int64_t Tn = 0;
    co_forward_out_len(h, Tc, &Tn);
    if (Tn < 1) { if (tmp_prev) cudaFreeAsync(tmp_prev, s); return fail(CO_ERR_LENGTH, "residual: T' < 1 at layer %d", l); }
    void* dst = y;
    if (l + 1 < L) {
      const size_t bytes = size_t(h->g.B) * Tn * h->g.HWo * h->g.Cout * dsize(h->g.out_dtype);
      cudaError_t e = cudaMallocAsync(&dst, bytes, s);
      if (e != cudaSuccess) { if (tmp_prev) cudaFreeAsync(tmp_prev, s); return fail(CO_ERR_OOM, "%s", cudaGetErrorString(e)); }
    }
    int64_t Tgot = 0;
    int rc = co_forward(h, cur, Tc, dst, &Tgot, stream);
    if (tmp_prev) cudaFreeAsync(tmp_prev, s);
    tmp_prev = (l + 1 < L) ? dst : nullptr;
    if (rc) { if (tmp_prev) cudaFreeAsync(tmp_prev, s); return rc; }
    cur = dst;
    Tc = Tgot;
  }
  if (T_out) *T_out = Tc;
  return CO_OK;
}

// Output length of a layer sequence's batch forward.
static int64_t layers_out_len(const std::vector<co_conv*>& layers, int64_t T) {
  for (co_conv* h : layers) {
    int64_t t = 0;
    co_forward_out_len(h, T, &t);
    T = t;
  }
  return T;
}

extern "C" int co_residual_forward(co_residual* r, const void* x, int64_t T, void* y, int64_t* T_out,
                                   co_stream stream) {
  if (!r || !x || !y) return fail(CO_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t Tc = 0;
  if (int rc = layers_forward(r->body, x, T, y, &Tc, stream)) return rc;
  // identity branch: the input clip aligned with each output's receptive-field
  // center: column i covers padded frames i .. i + f_acc - 1, center
  // = real frame i + (f_acc-1)/2 - p_acc, so the crop is d_skip - p_acc (0 for
  // equal padding); create guarantees 0 <= c and c + Tc <= T (p_acc <= d_skip)
  const int64_t c = r->shrink ? r->d_skip - r->p_acc : 0;
  const int64_t fe = r->frame_elems;
  const char* xs = static_cast<const char*>(x) + size_t(c) * fe * dsize(r->in_dtype);
  CO_CUDA(co::launch_residual_add(r->out_dtype, y, Tc * fe, r->in_dtype, xs, T * fe, r->B, Tc * fe, r->act, s));
  if (T_out) *T_out = Tc;
  return CO_OK;
}

extern "C" int co_residual_clean(co_residual* r, co_stream stream) {
  if (!r) return fail(CO_ERR_ARG, "null residual");
  if (int rc = co_stack_clean(r->stack, stream)) return rc;
  if (r->ring)
    CO_CUDA(cudaMemsetAsync(r->ring, 0, size_t(r->d_skip + 2) * r->B * r->frame_elems * dsize(r->in_dtype),
                            (cudaStream_t)stream));
  r->n = 0;
  return CO_OK;
}

extern "C" int co_residual_delay(const co_residual* r, int64_t* delay, int64_t* skip_delay) {
  if (!r) return fail(CO_ERR_ARG, "null residual");
  if (delay) *delay = r->d_body;
  if (skip_delay) *skip_delay = r->d_skip;
  return CO_OK;
}

// ----------------------------------------------------------------- per-stream clocks
// streams join (and leave) independently.  A handle keeps one
// clock (A19); stream b's own step count is n_b = n - join[b].  Cleaning
// a stream resets its state slice to the clean state and sets join[b] = n; its
// outputs are valid (co_stream_ready) on the handle's Ready ticks with
// n_b >= d.  Under temporal stride s the join must fall on n = 0 mod s, so the
// stream's Ready phase and the emitted outputs' ring slots (A20) are the
// handle's.

extern "C" int co_state_clean_streams(co_conv* h, const uint8_t* mask, co_stream stream) {
  if (!h || !mask) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  if (floor_mod(h->n, g.st) != 0)
    return fail(CO_ERR_ARG, "per-stream clean at tick n = %lld: needs n = 0 mod s = %d", (long long)h->n, g.st);
  std::vector<int64_t> ids;
  for (int64_t b = 0; b < g.B; ++b)
    if (mask[b]) ids.push_back(b);
  if (ids.empty()) return CO_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* dids = nullptr;
  CO_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dids), ids.size() * sizeof(int64_t), s));
  cudaError_t e = cudaMemcpyAsync(dids, ids.data(), ids.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) {
    cudaFreeAsync(dids, s);
    return fail(CO_ERR_CUDA, "clean streams: %s", cudaGetErrorString(e));
  }
  const int nm = int(ids.size());
  if (!g.raw && g.op == CO_OP_CONV) {
    if (g.R > 0) e = co::launch_clean_streams_psum(g, h->state, dids, nm, s);
  } else {
    const size_t sb = ring_slot_bytes(g);
    const int esz = g.op == CO_OP_CONV ? int(dsize(g.in_dtype)) : co::pool_ring_esz(g);
    const int64_t slots = g.op == CO_OP_CONV ? g.f + 1 : co::pool_state_slots(g);
    const int64_t per = int64_t(sb / esz) / g.B;
    uint32_t value = 0;
    if (g.op == CO_OP_MAX_POOL) value = esz == 2 ? 0xFF80u : 0xFF800000u;   // -inf: MAX's padding (A22)
    e = co::launch_fill_streams(h->state, esz, slots, g.B, per, dids, nm, value, s);
  }
  cudaFreeAsync(dids, s);
  if (e != cudaSuccess) return fail(CO_ERR_CUDA, "clean streams: %s", cudaGetErrorString(e));
  if (h->join.empty()) h->join.assign(size_t(g.B), 0);
  for (int64_t b : ids) h->join[size_t(b)] = h->n;
  return CO_OK;
}

extern "C" int co_stream_ready(const co_conv* h, uint8_t* ready) {
  if (!h || !ready) return fail(CO_ERR_ARG, "null argument");
  const Geom& g = h->g;
  for (int64_t b = 0; b < g.B; ++b) {
    const int64_t jb = h->join.empty() ? 0 : h->join[size_t(b)];
    ready[b] = uint8_t(h->last_ready && h->last_n >= 0 && h->last_n - jb >= g.delay);
  }
  return CO_OK;
}

extern "C" int co_stack_clean_streams(co_stack* st, const uint8_t* mask, co_stream stream) {
  if (!st || !mask) return fail(CO_ERR_ARG, "null argument");
  const int L = int(st->layers.size());
  for (int l = 1; l < L; ++l)
    if (st->layers[l]->g.st != 1)
      return fail(CO_ERR_UNSUPPORTED, "per-stream clean in a stack needs temporal stride 1 after layer 0 (layer %d)", l);
  if (int rc = co_state_clean_streams(st->layers[0], mask, stream)) return rc;
  const size_t B = size_t(st->layers[0]->g.B);
  if (st->pending.size() != size_t(L)) st->pending.assign(size_t(L), {});
  for (int l = 1; l < L; ++l) {
    std::vector<uint8_t>& p = st->pending[l];
    if (p.empty()) p.assign(B, 0);
    for (size_t b = 0; b < B; ++b) p[b] |= mask[b] ? 1 : 0;
  }
  return CO_OK;
}

extern "C" int co_stack_stream_ready(const co_stack* st, uint8_t* ready) {
  if (!st || !ready) return fail(CO_ERR_ARG, "null argument");
  const co_conv* last = st->layers.back();
  if (!st->last_ready) {
    for (int64_t b = 0; b < last->g.B; ++b) ready[b] = 0;
    return CO_OK;
  }
  if (int rc = co_stream_ready(last, ready)) return rc;
  for (const std::vector<uint8_t>& p : st->pending)      // a clean still pending in some layer
    if (p.size() == size_t(last->g.B))
      for (size_t b = 0; b < p.size(); ++b) ready[b] &= p[b] ? 0 : 1;
  return CO_OK;
}

// ----------------------------------------------------------------- continual MHA
// co.MultiheadAttention "single-output" (k_mha.cu): two kt = 1
// layers (the input projection E -> 3E and the output projection E -> E, RAW
// layout so the tensor-core K loop runs over 128 flattened stream rows) around
// the attention kernel, and a (k, v) ring of `window` slots.

struct co_mha {
  co_mha_desc d{};
  co_conv* in_proj = nullptr;
  co_conv* out_proj = nullptr;
  void* qkv = nullptr;       // (B, 3E) bf16
  void* att = nullptr;       // (B, E) bf16
  void* kring = nullptr;     // [n][B][E] bf16
  void* vring = nullptr;
  int64_t n = 0;
};

static co_conv_desc linear_desc(int64_t B, int cin, int cout, int out_dtype) {
  co_conv_desc c{};
  c.spatial_rank = 0;
  c.in_channels = cin; c.out_channels = cout; c.groups = 1;
  for (int a = 0; a < 3; ++a) { c.kernel[a] = 1; c.stride[a] = 1; c.padding[a] = 0; c.dilation[a] = 1; }
  c.in_spatial[0] = c.in_spatial[1] = 1;
  c.n_streams = B;
  c.in_dtype = c.w_dtype = CO_BF16;
  c.out_dtype = out_dtype;
  c.activation = CO_ACT_NONE;
  c.kernel_choice = CO_KERNEL_AUTO;
  c.state_layout = CO_STATE_RAW;
  c.op = CO_OP_CONV;
  return c;
}

extern "C" int co_mha_create(const co_mha_desc* d, const void* w_qkv, const float* b_qkv, const void* w_o,
                             const float* b_o, int weights_on_device, co_mha** out) {
  if (!d || !w_qkv || !w_o || !out) return fail(CO_ERR_ARG, "null argument");
  *out = nullptr;
  if (d->embed_dim < 1 || d->window < 1 || d->n_streams < 1) return fail(CO_ERR_ARG, "bad mha descriptor");
  if (!co::mha_supported(d->embed_dim, d->num_heads))
    return fail(CO_ERR_UNSUPPORTED, "mha: head dim E/heads must be 32, 64 or 128");
  if (d->out_dtype != CO_BF16 && d->out_dtype != CO_F32) return fail(CO_ERR_ARG, "bad out_dtype");
  co_mha* m = new (std::nothrow) co_mha();
  if (!m) return fail(CO_ERR_OOM, "host allocation");
  m->d = *d;
  const int64_t B = d->n_streams, E = d->embed_dim;
  co_conv_desc ci = linear_desc(B, int(E), int(3 * E), CO_BF16), co_ = linear_desc(B, int(E), int(E), d->out_dtype);
  if (int rc = co_conv_create(&ci, w_qkv, b_qkv, weights_on_device, &m->in_proj)) { co_mha_destroy(m); return rc; }
  if (int rc = co_conv_create(&co_, w_o, b_o, weights_on_device, &m->out_proj)) { co_mha_destroy(m); return rc; }
  const size_t fb = size_t(B) * E * 2;
  cudaError_t e = cudaMalloc(&m->qkv, 3 * fb);
  if (e == cudaSuccess) e = cudaMalloc(&m->att, fb);
  if (e == cudaSuccess) e = cudaMalloc(&m->kring, size_t(d->window) * fb);
  if (e == cudaSuccess) e = cudaMalloc(&m->vring, size_t(d->window) * fb);
  if (e == cudaSuccess) e = cudaMemset(m->kring, 0, size_t(d->window) * fb);
  if (e == cudaSuccess) e = cudaMemset(m->vring, 0, size_t(d->window) * fb);
  if (e != cudaSuccess) { co_mha_destroy(m); return fail(CO_ERR_OOM, "mha buffers: %s", cudaGetErrorString(e)); }
  *out = m;
  return CO_OK;
}

extern "C" int co_mha_destroy(co_mha* m) {
  if (!m) return CO_OK;
  co_conv_destroy(m->in_proj);
  co_conv_destroy(m->out_proj);
  cudaFree(m->qkv); cudaFree(m->att); cudaFree(m->kring); cudaFree(m->vring);
  delete m;
  return CO_OK;
}

static co::MhaArgs mha_args(const co_mha* m) {
  co::MhaArgs a{};
  a.E = m->d.embed_dim; a.heads = m->d.num_heads; a.n = m->d.window;
  a.B = m->d.n_streams; a.T = 1;
  a.scale_log2e = 1.4426950408889634f / sqrtf(float(a.E / a.heads));
  return a;
}

extern "C" int co_mha_step(co_mha* m, const void* x, void* y, int update_state, int* ready, co_stream stream) {
  if (!m || !x || !y) return fail(CO_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = m->d.n_streams, E = m->d.embed_dim;
  int r0 = 0;
  if (int rc = co_forward_step(m->in_proj, x, m->qkv, 1, &r0, stream)) return rc;   // kt = 1: always Ready
  const int r = m->n >= m->d.window - 1;
  if (r) {
    co::MhaArgs a = mha_args(m);
    a.qkv = static_cast<const __nv_bfloat16*>(m->qkv);
    a.kring = static_cast<__nv_bfloat16*>(m->kring);
    a.vring = static_cast<__nv_bfloat16*>(m->vring);
    a.out = static_cast<__nv_bfloat16*>(m->att);
    a.m = m->n; a.store = update_state ? 1 : 0;
    CO_CUDA(co::launch_mha_attend(a, s));
    int r1 = 0;
    if (int rc = co_forward_step(m->out_proj, m->att, y, 1, &r1, stream)) return rc;
  } else if (update_state) {   // not Ready: only the ring update (strided copies of k and v)
    const size_t slot = size_t(m->n % m->d.window);
    const size_t row = size_t(E) * 2, pitch = row * m->d.window;   // ring [B][n][E]
    char* qkv = static_cast<char*>(m->qkv);
    CO_CUDA(cudaMemcpy2DAsync(static_cast<char*>(m->kring) + slot * row, pitch, qkv + row, 3 * row, row, B,
                              cudaMemcpyDeviceToDevice, s));
    CO_CUDA(cudaMemcpy2DAsync(static_cast<char*>(m->vring) + slot * row, pitch, qkv + 2 * row, 3 * row, row, B,
                              cudaMemcpyDeviceToDevice, s));
  }
  if (update_state) ++m->n;
  if (ready) *ready = r;
  return CO_OK;
}

extern "C" int co_mha_forward(co_mha* m, const void* x, int64_t T, void* y, co_stream stream) {
  if (!m || !x || !y || T < 1) return fail(CO_ERR_ARG, "bad argument");
  // batch mode is the fixed-window form (T == window); only then is
  // every column the step output of its window (mode equivalence, Definition 1)
  if (T != m->d.window) return fail(CO_ERR_LENGTH, "mha batch mode needs T == window (%lld != %d)", (long long)T, m->d.window);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t B = m->d.n_streams, E = m->d.embed_dim;
  void *qkv = nullptr, *att = nullptr;
  CO_CUDA(cudaMallocAsync(&qkv, size_t(B) * T * 3 * E * 2, s));
  cudaError_t e = cudaMallocAsync(&att, size_t(B) * T * E * 2, s);
  int64_t To = 0;
  int rc = CO_OK;
  if (e != cudaSuccess) rc = fail(CO_ERR_OOM, "%s", cudaGetErrorString(e));
  if (!rc) rc = co_forward(m->in_proj, x, T, qkv, &To, stream);
  if (!rc) {
    co::MhaArgs a = mha_args(m);
    a.qkv = static_cast<const __nv_bfloat16*>(qkv);
    a.out = static_cast<__nv_bfloat16*>(att);
    a.T = T; a.batch = 1;
    e = co::launch_mha_attend(a, s);
    if (e != cudaSuccess) rc = fail(CO_ERR_CUDA, "mha attend: %s", cudaGetErrorString(e));
  }
  if (!rc) rc = co_forward(m->out_proj, att, T, y, &To, stream);
  cudaFreeAsync(qkv, s);
  if (att) cudaFreeAsync(att, s);
  return rc;
}

extern "C" int co_mha_clean(co_mha* m, co_stream stream) {
  if (!m) return fail(CO_ERR_ARG, "null mha");
  const size_t fb = size_t(m->d.n_streams) * m->d.embed_dim * 2 * m->d.window;
  CO_CUDA(cudaMemsetAsync(m->kring, 0, fb, (cudaStream_t)stream));
  CO_CUDA(cudaMemsetAsync(m->vring, 0, fb, (cudaStream_t)stream));
  m->n = 0;
  return CO_OK;
}

extern "C" int co_mha_delay(const co_mha* m, int64_t* delay) {
  if (!m || !delay) return fail(CO_ERR_ARG, "null argument");
  *delay = m->d.window - 1;
  return CO_OK;
}

extern "C" int co_mha_state_bytes(const co_mha* m, size_t* bytes) {
  if (!m || !bytes) return fail(CO_ERR_ARG, "null argument");
  *bytes = size_t(m->d.window - 1) * 2 * m->d.n_streams * m->d.embed_dim * 2;
  return CO_OK;
}

// canonical slot j (oldest first) = step n - (n-1) + j, i.e. ring slot (n - (n_win-1) + j) mod n_win
extern "C" int co_mha_state_get(co_mha* m, void* dst, size_t bytes, int64_t* n, co_stream stream) {
  size_t need = 0;
  if (int rc = co_mha_state_bytes(m, &need)) return rc;
  if (bytes != need) return fail(CO_ERR_SHAPE, "state bytes %zu != %zu", bytes, need);
  const int W = m->d.window;
  const size_t row = size_t(m->d.embed_dim) * 2, fb = size_t(m->d.n_streams) * row, pitch = row * W;
  for (int j = 0; j < W - 1; ++j) {   // ring [B][n][E] -> canonical (n-1, 2, B, E)
    const size_t slot = size_t(floor_mod(m->n - (W - 1) + j, W));
    char* o = static_cast<char*>(dst) + size_t(j) * 2 * fb;
    CO_CUDA(cudaMemcpy2DAsync(o, row, static_cast<char*>(m->kring) + slot * row, pitch, row, m->d.n_streams,
                              cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    CO_CUDA(cudaMemcpy2DAsync(o + fb, row, static_cast<char*>(m->vring) + slot * row, pitch, row, m->d.n_streams,
                              cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  if (n) *n = m->n;
  return CO_OK;
}

extern "C" int co_mha_state_set(co_mha* m, const void* src, size_t bytes, int64_t n, co_stream stream) {
  size_t need = 0;
  if (int rc = co_mha_state_bytes(m, &need)) return rc;
  if (bytes != need || n < 0) return fail(CO_ERR_SHAPE, "state bytes %zu != %zu", bytes, need);
  const int W = m->d.window;
  const size_t row = size_t(m->d.embed_dim) * 2, fb = size_t(m->d.n_streams) * row, pitch = row * W;
  for (int j = 0; j < W - 1; ++j) {
    const size_t slot = size_t(floor_mod(n - (W - 1) + j, W));
    const char* i = static_cast<const char*>(src) + size_t(j) * 2 * fb;
    CO_CUDA(cudaMemcpy2DAsync(static_cast<char*>(m->kring) + slot * row, pitch, i, row, row, m->d.n_streams,
                              cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    CO_CUDA(cudaMemcpy2DAsync(static_cast<char*>(m->vring) + slot * row, pitch, i + fb, row, row, m->d.n_streams,
                              cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  }
  m->n = n;
  return CO_OK;
}

// ----------------------------------------------------------------- broadcast-reduce
// BroadcastReduce (include/co.h): branches are stacks (or the
// identity); a branch with delay d_i < d_max keeps a ring of its last
// k_i + 1 = d_max - d_i + 1 Ready outputs (+ a scratch slot) and contributes the
// one of k_i Ready outputs ago; the merge adds (k_compose.cu) or copies channel
// slices.

struct co_parallel {
  std::vector<co_stack*> br;         // nullptr = identity
  int reduce = CO_REDUCE_SUM;
  std::vector<int64_t> d, k, count, C;
  std::vector<int> dt;               // per-branch output dtype (SUM may mix: the identity's is the input's)
  int64_t d_max = 0, n = 0;
  std::vector<void*> out, ring;      // per branch: step output buffer, alignment ring
  int64_t B = 0, HWo = 0, Ctot = 0, in_frame = 0;
  int dtype = 0;
};

extern "C" int co_parallel_create(co_stack* const* branches, int n_branches, int reduce, co_parallel** out) {
  if (!branches || n_branches < 1 || !out) return fail(CO_ERR_ARG, "bad argument");
  if (reduce != CO_REDUCE_SUM && reduce != CO_REDUCE_CONCAT) return fail(CO_ERR_ARG, "bad reduce");
  *out = nullptr;
  // the common input: any stack branch's first layer (an all-identity composite has no geometry source)
  const Geom* in = nullptr;
  for (int i = 0; i < n_branches; ++i)
    if (branches[i]) { in = &branches[i]->layers.front()->g; break; }
  if (!in) return fail(CO_ERR_ARG, "at least one branch must be a stack");
  co_parallel* p = new (std::nothrow) co_parallel();
  if (!p) return fail(CO_ERR_OOM, "host allocation");
  auto bail = [&](int code) { co_parallel_destroy(p); return code; };
  p->reduce = reduce;
  p->B = in->B;
  p->in_frame = in->frame_elems;
  int64_t Ho = -1, Wo = -1;
  int odt = -1;
  for (int i = 0; i < n_branches; ++i) {
    co_stack* st = branches[i];
    int64_t di = 0, ci, ho, wo;
    int dt;
    if (st) {
      const Geom& a = st->layers.front()->g;
      const Geom& z = st->layers.back()->g;
      if (a.B != in->B || a.H != in->H || a.W != in->W || a.Cin != in->Cin || a.in_dtype != in->in_dtype)
        return bail(fail(CO_ERR_SHAPE, "branch %d: input differs from branch inputs", i));
      int64_t s_acc = 1;
      for (co_conv* h : st->layers) s_acc *= h->g.st;
      if (s_acc != 1) return bail(fail(CO_ERR_SHAPE, "branch %d: accumulated temporal stride %lld != 1", i, (long long)s_acc));
      co_stack_delay(st, &di);
      ci = z.Cout; ho = z.Ho; wo = z.Wo; dt = z.out_dtype;
    } else {
      ci = in->Cin; ho = in->H; wo = in->W; dt = in->in_dtype;
    }
    if (Ho < 0) { Ho = ho; Wo = wo; }
    if (st && odt < 0) odt = dt;       // the composite's output dtype: the (first) stack branch's
    if (ho != Ho || wo != Wo) return bail(fail(CO_ERR_SHAPE, "branch %d: output shape differs", i));
    if (st && dt != odt) return bail(fail(CO_ERR_SHAPE, "branch %d: output dtype differs", i));
    if (!st && reduce == CO_REDUCE_CONCAT && dt != in->in_dtype)
      return bail(fail(CO_ERR_SHAPE, "branch %d: dtype differs", i));
    p->dt.push_back(dt);
    if (reduce == CO_REDUCE_SUM && !p->C.empty() && ci != p->C[0])
      return bail(fail(CO_ERR_SHAPE, "branch %d: sum needs equal channel counts", i));
    p->br.push_back(st); p->d.push_back(di); p->C.push_back(ci);
    p->d_max = std::max(p->d_max, di);
  }
  p->HWo = Ho * Wo;
  p->dtype = odt;
  p->Ctot = reduce == CO_REDUCE_SUM ? p->C[0] : 0;
  if (reduce == CO_REDUCE_CONCAT)
    for (int64_t c : p->C) p->Ctot += c;
  if (reduce == CO_REDUCE_CONCAT)
    for (int i = 0; i < n_branches; ++i)
      if (p->dt[i] != odt) return bail(fail(CO_ERR_SHAPE, "concat: branch %d dtype differs", i));
  for (int i = 0; i < n_branches; ++i) {
    p->k.push_back(p->d_max - p->d[i]);
    p->count.push_back(0);
    const size_t fb = size_t(p->B) * p->HWo * p->C[i] * dsize(p->dt[i]);
    void* o = nullptr;
    void* r = nullptr;
    cudaError_t e = cudaSuccess;
    if (p->br[i]) e = cudaMalloc(&o, fb);
    if (e == cudaSuccess && p->k[i] > 0) e = cudaMalloc(&r, fb * size_t(p->k[i] + 2));
    p->out.push_back(o); p->ring.push_back(r);
    if (e != cudaSuccess) return bail(fail(CO_ERR_OOM, "branch buffers: %s", cudaGetErrorString(e)));
  }
  *out = p;
  return CO_OK;
}

extern "C" int co_parallel_destroy(co_parallel* p) {
  if (!p) return CO_OK;
  for (void* o : p->out) cudaFree(o);
  for (void* r : p->ring) cudaFree(r);
  delete p;
  return CO_OK;
}

// Merge branch frames src[i] (each B * HWo * C_i, stream stride sstride[i]) into y.
static int merge_into(co_parallel* p, const std::vector<const void*>& src, const std::vector<int64_t>& sstride,
                      void* y, int64_t ystride, int64_t cols, cudaStream_t s) {
  const size_t esz = dsize(p->dtype);
  const int nb = int(src.size());
  if (p->reduce == CO_REDUCE_SUM) {
    // start from the first branch in the output dtype, add the others (converted)
    int first = 0;
    while (p->dt[first] != p->dtype) ++first;
    const size_t row = size_t(cols) * p->HWo * p->Ctot * esz;
    CO_CUDA(cudaMemcpy2DAsync(y, size_t(ystride) * esz, src[first], size_t(sstride[first]) * esz, row, p->B,
                              cudaMemcpyDeviceToDevice, s));
    for (int i = 0; i < nb; ++i)
      if (i != first)
        CO_CUDA(co::launch_residual_add(p->dtype, y, ystride, p->dt[i], src[i], sstride[i], p->B,
                                        cols * p->HWo * p->Ctot, CO_ACT_NONE, s));
    return CO_OK;
  }
  int64_t off = 0;   // concat: channel slice per branch, pixel rows of every stream
  for (int i = 0; i < nb; ++i) {
    for (int64_t b = 0; b < p->B; ++b)
      CO_CUDA(cudaMemcpy2DAsync(static_cast<char*>(y) + (size_t(b) * ystride + off) * esz, size_t(p->Ctot) * esz,
                                static_cast<const char*>(src[i]) + size_t(b) * sstride[i] * esz, size_t(p->C[i]) * esz,
                                size_t(p->C[i]) * esz, size_t(cols) * p->HWo, cudaMemcpyDeviceToDevice, s));
    off += p->C[i];
  }
  return CO_OK;
}

extern "C" int co_parallel_step(co_parallel* p, const void* x, void* y, int update_state, int* ready,
                                co_stream stream) {
  if (!p || !x || !y) return fail(CO_ERR_ARG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = int(p->br.size());
  std::vector<const void*> aligned(nb, nullptr);
  std::vector<int64_t> stride(nb);
  bool all = p->n >= p->d_max;
  for (int i = 0; i < nb; ++i) {
    const size_t fb = size_t(p->B) * p->HWo * p->C[i] * dsize(p->dt[i]);
    int r = 1;
    const void* fresh = x;
    if (p->br[i]) {
      if (int rc = co_stack_step(p->br[i], x, p->out[i], update_state, &r, stream)) return rc;
      fresh = p->out[i];
    }
    stride[i] = p->HWo * p->C[i];
    const int64_t k = p->k[i];
    if (k == 0) {
      aligned[i] = r ? fresh : nullptr;
    } else {
      char* ring = static_cast<char*>(p->ring[i]);
      const int64_t R = k + 1;
      if (r) {
        char* slot = ring + size_t(update_state ? floor_mod(p->count[i], R) : R) * fb;   // scratch when probing
        CO_CUDA(cudaMemcpyAsync(slot, fresh, fb, cudaMemcpyDeviceToDevice, s));
      }
      const int64_t idx = p->count[i] + (r ? 1 : 0) - 1 - k;     // the output k Ready outputs ago
      aligned[i] = (r && idx >= 0) ? ring + size_t(floor_mod(idx, R)) * fb : nullptr;
      if (r && update_state) ++p->count[i];
    }
    all = all && aligned[i];
  }
  if (all)
    if (int rc = merge_into(p, aligned, stride, y, p->HWo * p->Ctot, 1, s)) return rc;
  if (update_state) ++p->n;
  if (ready) *ready = all ? 1 : 0;
  return CO_OK;
}

extern "C" int co_parallel_forward(co_parallel* p, const void* x, int64_t T, void* y, int64_t* T_out,
                                   co_stream stream) {
  if (!p || !x || !y || T < 1) return fail(CO_ERR_ARG, "bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = int(p->br.size());
  std::vector<int64_t> Ti(nb);
  int64_t T_min = T;
  for (int i = 0; i < nb; ++i) {
    Ti[i] = p->br[i] ? layers_out_len(p->br[i]->layers, T) : T;
    T_min = std::min(T_min, Ti[i]);
  }
  if (T_min < 1) return fail(CO_ERR_LENGTH, "broadcast-reduce: T' < 1");
  std::vector<void*> tmp(nb, nullptr);
  std::vector<const void*> src(nb);
  std::vector<int64_t> sstride(nb);
  int rc = CO_OK;
  for (int i = 0; i < nb && !rc; ++i) {
    sstride[i] = Ti[i] * p->HWo * p->C[i];
    if (!p->br[i]) { src[i] = x; continue; }
    cudaError_t e = cudaMallocAsync(&tmp[i], size_t(p->B) * sstride[i] * dsize(p->dt[i]), s);
    if (e != cudaSuccess) { rc = fail(CO_ERR_OOM, "%s", cudaGetErrorString(e)); break; }
    int64_t t = 0;
    rc = layers_forward(p->br[i]->layers, x, T, tmp[i], &t, stream);
    src[i] = tmp[i];
  }
  if (!rc) rc = merge_into(p, src, sstride, y, T_min * p->HWo * p->Ctot, T_min, s);
  for (void* t : tmp)
    if (t) cudaFreeAsync(t, s);
  if (!rc && T_out) *T_out = T_min;
  return rc;
}

extern "C" int co_parallel_clean(co_parallel* p, co_stream stream) {
  if (!p) return fail(CO_ERR_ARG, "null composite");
  for (co_stack* st : p->br)
    if (st)
      if (int rc = co_stack_clean(st, stream)) return rc;
  for (size_t i = 0; i < p->count.size(); ++i) p->count[i] = 0;
  p->n = 0;
  return CO_OK;
}

extern "C" int co_parallel_delay(const co_parallel* p, int64_t* delay) {
  if (!p || !delay) return fail(CO_ERR_ARG, "null argument");
  *delay = p->d_max;
  return CO_OK;
}

extern "C" int co_parallel_out_channels(const co_parallel* p, int32_t* channels) {
  if (!p || !channels) return fail(CO_ERR_ARG, "null argument");
  *channels = int32_t(p->Ctot);
  return CO_OK;
}

// ----------------------------------------------------------------- CUDA-graph step loops

// A stack's tick sequence depends only on the host clocks (a1: readiness, ring
// slots and the clock-derived kernel arguments are integer functions of each
// layer's n), so n_ticks consecutive ticks can be captured
// once and replayed: the replay is valid whenever every layer's clock is where
// the captured schedule starts -- the same n, or, once past the transients,
// the same phase modulo a period of all those functions.
struct co_graph {
  co_stack* st = nullptr;
  int64_t n_ticks = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<int64_t> n_cap, gen_cap, period, steady;
  int pdl = 1;
};

static int64_t gcd64(int64_t a, int64_t b) { while (b) { const int64_t t = a % b; a = b; b = t; } return a; }
static int64_t lcm64(int64_t a, int64_t b) { return a / gcd64(a, b) * b; }

// A period (in the layer's own steps) of every clock-derived argument of its
// step launches: partial-sum ring slots floor((m - k dil)/s) mod R and the
// stride phase (n - d) mod s repeat every s R steps; the RAW / Delay frame
// rings every f (slot m mod f); pooling adds the block decomposition's
// (m div dil) mod kt.
static int64_t clock_period(const Geom& g) {
  const int64_t s = std::max(1, g.st), f = std::max(1, g.f);
  if (g.op == CO_OP_DELAY) return f;
  if (g.op != CO_OP_CONV) return lcm64(lcm64(f, s), int64_t(std::max(1, g.dt)) * std::max(1, g.kt));
  if (g.raw) return lcm64(f, s);
  return s * std::max(1, g.R);
}
// From this clock on the schedule is periodic (no output index < 0, past the delay).
static int64_t clock_steady(const Geom& g) { return int64_t(g.f) + g.pt + g.delay + 2 * g.st; }

static int64_t layer_gen(const co_conv* h) { return h->tc ? co::dense_tc_buffer_gen(h->tc) : 0; }

// Advance the host side of one stack tick without launching anything: the
// clocks and last-step readiness exactly as co_stack_step leaves them.
static int dry_tick(co_stack* st) {
  st->last_ready = 0;
  for (co_conv* h : st->layers) {
    const Geom& g = h->g;
    const int r = (g.op == CO_OP_DELAY) ? (h->n >= g.delay)
                                         : ((h->n >= g.delay) && floor_mod(h->n - g.delay, g.st) == 0);
    h->last_n = h->n;
    h->last_ready = r;
    ++h->n;
    if (!r) return 0;
  }
  st->last_ready = 1;
  return 1;
}

extern "C" int co_stack_graph_create(co_stack* st, int64_t n_ticks, const void* const* x, void* const* y,
                                     co_graph** out) {
  if (!st || n_ticks < 1 || !x || !y || !out) return fail(CO_ERR_ARG, "bad argument");
  *out = nullptr;
  for (int64_t t = 0; t < n_ticks; ++t)
    if (!x[t] || !y[t]) return fail(CO_ERR_ARG, "null frame / output pointer at tick %lld", (long long)t);
  for (const auto& p : st->pending)
    if (!p.empty()) return fail(CO_ERR_UNSUPPORTED, "a per-stream clean is pending: step eagerly until it lands");
  const size_t L = st->layers.size();
  std::vector<int64_t> n0(L), ln(L);
  std::vector<int> lr(L);
  for (size_t l = 0; l < L; ++l) { n0[l] = st->layers[l]->n; ln[l] = st->layers[l]->last_n; lr[l] = st->layers[l]->last_ready; }
  const int sr = st->last_ready;
  auto restore = [&]() {
    for (size_t l = 0; l < L; ++l) { st->layers[l]->n = n0[l]; st->layers[l]->last_n = ln[l]; st->layers[l]->last_ready = lr[l]; }
    st->last_ready = sr;
  };
  cudaStream_t cs = nullptr;
  CO_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  co_graph* G = new (std::nothrow) co_graph();
  if (!G) { cudaStreamDestroy(cs); return fail(CO_ERR_OOM, "host allocation"); }
  int rc = CO_OK;
  // first with programmatic dependent launch (captured as programmatic edges),
  // then, if this driver cannot instantiate those, with plain launches
  for (int pdl = 1; pdl >= 0; --pdl) {
    co::set_thread_no_pdl(pdl ? 0 : 1);
    rc = CO_OK;
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) { rc = fail(CO_ERR_CUDA, "begin capture: %s", cudaGetErrorString(e)); break; }
    for (int64_t t = 0; t < n_ticks && !rc; ++t) {
      int r = 0;
      rc = co_stack_step(st, x[t], y[t], 1, &r, cs);
    }
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cs, &graph);
    restore();
    if (rc) { if (graph) cudaGraphDestroy(graph); break; }
    if (e != cudaSuccess) { cudaGetLastError(); rc = fail(CO_ERR_CUDA, "end capture: %s", cudaGetErrorString(e)); continue; }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) {
      cudaGetLastError();
      cudaGraphDestroy(graph);
      rc = fail(CO_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
      continue;
    }
    G->graph = graph; G->exec = exec; G->pdl = pdl;
    break;
  }
  co::set_thread_no_pdl(0);
  cudaStreamDestroy(cs);
  if (rc || !G->exec) { delete G; return rc ? rc : fail(CO_ERR_CUDA, "graph capture failed"); }
  G->st = st;
  G->n_ticks = n_ticks;
  for (co_conv* h : st->layers) {
    G->n_cap.push_back(h->n);
    G->gen_cap.push_back(layer_gen(h));
    G->period.push_back(clock_period(h->g));
    G->steady.push_back(clock_steady(h->g));
  }
  *out = G;
  return CO_OK;
}

extern "C" int co_stack_graph_period(const co_stack* st, int64_t* period) {
  if (!st || !period) return fail(CO_ERR_ARG, "null argument");
  // layer l steps once per s_acc(l) ticks (the product of the strides below it)
  int64_t P = 1, s_acc = 1;
  for (const co_conv* h : st->layers) {
    P = lcm64(P, clock_period(h->g) * s_acc);
    s_acc *= std::max(1, h->g.st);
  }
  *period = P;
  return CO_OK;
}

extern "C" int co_graph_upload(co_graph* G, co_stream stream) {
  if (!G) return fail(CO_ERR_ARG, "null graph");
  CO_CUDA(cudaGraphUpload(G->exec, (cudaStream_t)stream));
  return CO_OK;
}

extern "C" int co_graph_launch(co_graph* G, int64_t* n_ready, co_stream stream) {
  if (!G) return fail(CO_ERR_ARG, "null graph");
  co_stack* st = G->st;
  for (const auto& p : st->pending)
    if (!p.empty()) return fail(CO_ERR_UNSUPPORTED, "a per-stream clean is pending");
  for (size_t l = 0; l < st->layers.size(); ++l) {
    const co_conv* h = st->layers[l];
    if (layer_gen(h) != G->gen_cap[l])
      return fail(CO_ERR_ARG, "layer %zu's staging buffers moved since capture: capture again", l);
    const int64_t n = h->n, c = G->n_cap[l];
    const bool same = n == c ||
                      (n >= G->steady[l] && c >= G->steady[l] && floor_mod(n - c, G->period[l]) == 0);
    if (!same)
      return fail(CO_ERR_ARG, "layer %zu clock %lld is not at the captured phase (%lld mod %lld)", l, (long long)n,
                  (long long)c, (long long)G->period[l]);
  }
  CO_CUDA(cudaGraphLaunch(G->exec, (cudaStream_t)stream));
  int64_t nr = 0;
  for (int64_t t = 0; t < G->n_ticks; ++t) nr += dry_tick(st);
  if (n_ready) *n_ready = nr;
  return CO_OK;
}

extern "C" int co_graph_destroy(co_graph* G) {
  if (!G) return CO_OK;
  if (G->exec) cudaGraphExecDestroy(G->exec);
  if (G->graph) cudaGraphDestroy(G->graph);
  delete G;
  return CO_OK;
}

extern "C" int co_graph_info(const co_graph* G, int64_t* n_ticks, int* pdl) {
  if (!G) return fail(CO_ERR_ARG, "null graph");
  if (n_ticks) *n_ticks = G->n_ticks;
  if (pdl) *pdl = G->pdl;
  return CO_OK;
}
