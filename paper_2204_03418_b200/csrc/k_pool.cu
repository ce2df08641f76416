// k_pool.cu — continual max / average pooling (PAPER.md
// P:380-394 "Pooling: co.AvgPool1d, co.MaxPool1d, etc.").
//
// Pooling keeps the RAW frame ring (co_state_layout RAW, §8f f1): a step
// stores its frame in ring slot m mod f (host.cu step_raw) and a Ready step
// reduces the window's kt frames x spatial window.  Temporal padding lives in
// the ring as the operator's identity-under-padding value -- 0 for AVG (counted
// in the divisor, count_include_pad, A21) and -inf for MAX (ignored,
// PyTorch's implicit MAX padding, A22) -- so start padding (clean state),
// pad_end steps (x == NULL) and saved / restored state need no flags, and the
// kernel is a plain max / sum over the window.  Spatial out-of-frame taps are
// skipped (MAX) or contribute 0 (AVG).
//
// CUDA cores: pooling is pure data movement + compare/add (no contraction), so
// the bound is HBM: one Ready step reads kt frames (B H W C elements each) and
// writes one output frame.  Thread = (stream, output pixel, vector of V
// channels); consecutive threads take consecutive channel vectors, so every
// frame read and output write is a coalesced 16-byte access, and the spatial
// window's overlapping reads hit L1.
#include "common.cuh"

namespace co {

namespace {

template <typename T, int V>
struct alignas(sizeof(T) * V) Vec {
  T v[V];
};

template <typename T> __device__ __forceinline__ T pad_value(int op);
template <> __device__ __forceinline__ float pad_value<float>(int op) { return op == 1 ? -INFINITY : 0.f; }
template <> __device__ __forceinline__ __nv_bfloat16 pad_value<__nv_bfloat16>(int op) {
  return op == 1 ? __ushort_as_bfloat16(0xFF80) : __ushort_as_bfloat16(0);
}

// Reduce one temporal frame's spatial window into acc[V].
template <typename Tin, int V, bool MAX>
__device__ __forceinline__ void reduce_frame(const Geom& g, const Tin* __restrict__ fb, int ho, int wo, int c0,
                                             float (&acc)[V]) {
  for (int u = 0; u < g.kh; ++u) {
    const int hi = ho * g.sh + u * g.dh - g.ph;
    if (hi < 0 || hi >= g.H) continue;
    for (int v = 0; v < g.kw; ++v) {
      const int wi = wo * g.sw + v * g.dw - g.pw;
      if (wi < 0 || wi >= g.W) continue;
      const Vec<Tin, V> x = *reinterpret_cast<const Vec<Tin, V>*>(fb + (int64_t(hi) * g.W + wi) * g.Cin + c0);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float f = to_f(x.v[j]);
        acc[j] = MAX ? fmaxf(acc[j], f) : acc[j] + f;
      }
    }
  }
}

template <typename Tout, int V, bool MAX>
__device__ __forceinline__ void store_out(const Geom& g, Tout* __restrict__ yp, const float (&acc)[V]) {
  const float inv = 1.f / float(g.kt * g.kh * g.kw);
  Vec<Tout, V> o;
#pragma unroll
  for (int j = 0; j < V; ++j) o.v[j] = from_f<Tout>(activate(MAX ? acc[j] : acc[j] * inv, g.act));
  *reinterpret_cast<Vec<Tout, V>*>(yp) = o;
}

// Step: a.slot[k] = ring slot of temporal tap k (host clock); ring layout
// [slot][B][H][W][C].  Only launched on Ready ticks.
template <typename Tin, typename Tout, int V, bool MAX>
__global__ void __launch_bounds__(256) k_step_pool(Geom g, StepArgs a) {
  const int CV = g.Cin / V;
  const int64_t total = g.B * g.HWo * CV;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const Tin* ring = reinterpret_cast<const Tin*>(a.state);
  const int64_t slot_elems = g.B * g.frame_elems;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c0 = int(idx % CV) * V;
    const int64_t r = idx / CV;
    const int p = int(r % g.HWo);
    const int64_t b = r / g.HWo;
    const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = MAX ? -INFINITY : 0.f;
    for (int k = 0; k < g.kt; ++k)
      reduce_frame<Tin, V, MAX>(g, ring + int64_t(a.slot[k]) * slot_elems + b * g.frame_elems, ho, wo, c0, acc);
    store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + int64_t(p) * g.Cout + c0, acc);
  }
}

// Batch mode: y[b, t'] = pool over frames t' s + k dil - p_t, frames
// outside [0, T) are padding (0 for AVG, ignored by MAX).  Reads no state.
template <typename Tin, typename Tout, int V, bool MAX>
__global__ void __launch_bounds__(256) k_forward_pool(Geom g, const Tin* __restrict__ x, int64_t T,
                                                       Tout* __restrict__ y, int64_t Tp) {
  const int CV = g.Cin / V;
  const int64_t total = g.B * Tp * g.HWo * CV;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c0 = int(idx % CV) * V;
    int64_t r = idx / CV;
    const int p = int(r % g.HWo);
    r /= g.HWo;
    const int64_t tp = r % Tp;
    const int64_t b = r / Tp;
    const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = MAX ? -INFINITY : 0.f;
    for (int k = 0; k < g.kt; ++k) {
      const int64_t t = tp * g.st + int64_t(k) * g.dt - g.pt;
      if (t < 0 || t >= T) continue;
      reduce_frame<Tin, V, MAX>(g, x + (b * T + t) * g.frame_elems, ho, wo, c0, acc);
    }
    store_out<Tout, V, MAX>(g, y + ((b * Tp + tp) * g.HWo + p) * g.Cout + c0, acc);
  }
}

template <typename T>
__global__ void k_fill(T* __restrict__ p, int64_t n, int op) {
  const T v = pad_value<T>(op);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

int vec_width(const Geom& g) {
  const int v = g.in_dtype == BF16 ? 8 : 4;   // 16-byte input vectors
  if (g.Cin % v == 0) return v;
  if (g.Cin % 2 == 0) return 2;
  return 1;
}

int grid_for(int64_t total) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (total + 255) / 256;
  const int64_t cap = int64_t(sms) * 8;          // 8 x 256 threads resident per SM
  return int(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

template <typename Tin, typename Tout, bool MAX>
cudaError_t step_t(const Geom& g, const StepArgs& a, cudaStream_t s) {
  const int V = vec_width(g);
  const int64_t total = g.B * g.HWo * (g.Cin / V);
  const int grid = grid_for(total);
  switch (V) {
    case 8: k_step_pool<Tin, Tout, 8, MAX><<<grid, 256, 0, s>>>(g, a); break;
    case 4: k_step_pool<Tin, Tout, 4, MAX><<<grid, 256, 0, s>>>(g, a); break;
    case 2: k_step_pool<Tin, Tout, 2, MAX><<<grid, 256, 0, s>>>(g, a); break;
    default: k_step_pool<Tin, Tout, 1, MAX><<<grid, 256, 0, s>>>(g, a); break;
  }
  return cudaGetLastError();
}

template <typename Tin, typename Tout, bool MAX>
cudaError_t forward_t(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp, cudaStream_t s) {
  const int V = vec_width(g);
  const int64_t total = g.B * Tp * g.HWo * (g.Cin / V);
  const int grid = grid_for(total);
  const Tin* xp = static_cast<const Tin*>(x);
  Tout* yp = static_cast<Tout*>(y);
  switch (V) {
    case 8: k_forward_pool<Tin, Tout, 8, MAX><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
    case 4: k_forward_pool<Tin, Tout, 4, MAX><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
    case 2: k_forward_pool<Tin, Tout, 2, MAX><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
    default: k_forward_pool<Tin, Tout, 1, MAX><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
  }
  return cudaGetLastError();
}

template <bool MAX>
cudaError_t step_dispatch(const Geom& g, const StepArgs& a, cudaStream_t s) {
  if (g.in_dtype == BF16)
    return g.out_dtype == BF16 ? step_t<__nv_bfloat16, __nv_bfloat16, MAX>(g, a, s)
                               : step_t<__nv_bfloat16, float, MAX>(g, a, s);
  return g.out_dtype == BF16 ? step_t<float, __nv_bfloat16, MAX>(g, a, s) : step_t<float, float, MAX>(g, a, s);
}

template <bool MAX>
cudaError_t forward_dispatch(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp, cudaStream_t s) {
  if (g.in_dtype == BF16)
    return g.out_dtype == BF16 ? forward_t<__nv_bfloat16, __nv_bfloat16, MAX>(g, x, T, y, Tp, s)
                               : forward_t<__nv_bfloat16, float, MAX>(g, x, T, y, Tp, s);
  return g.out_dtype == BF16 ? forward_t<float, __nv_bfloat16, MAX>(g, x, T, y, Tp, s)
                             : forward_t<float, float, MAX>(g, x, T, y, Tp, s);
}

}  // namespace

cudaError_t launch_step_pool(const Geom& g, const StepArgs& a, cudaStream_t s) {
  return g.op == OP_MAX_POOL ? step_dispatch<true>(g, a, s) : step_dispatch<false>(g, a, s);
}

cudaError_t launch_forward_pool(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp, cudaStream_t s) {
  if (g.B * Tp * g.HWo == 0) return cudaSuccess;
  return g.op == OP_MAX_POOL ? forward_dispatch<true>(g, x, T, y, Tp, s) : forward_dispatch<false>(g, x, T, y, Tp, s);
}

cudaError_t launch_fill_pad(const Geom& g, void* p, int64_t n_elems, cudaStream_t s) {
  if (n_elems <= 0) return cudaSuccess;
  if (g.op != OP_MAX_POOL) return cudaMemsetAsync(p, 0, size_t(n_elems) * (g.in_dtype == BF16 ? 2 : 4), s);
  const int grid = grid_for(n_elems);
  if (g.in_dtype == BF16) k_fill<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(p), n_elems, g.op);
  else k_fill<float><<<grid, 256, 0, s>>>(static_cast<float*>(p), n_elems, g.op);
  return cudaGetLastError();
}

const char* pool_kernel_name(const Geom& g) {
  static const char* names[2][4] = {{"k_step_pool<avg,V1>", "k_step_pool<avg,V2>", "k_step_pool<avg,V4>",
                                     "k_step_pool<avg,V8>"},
                                    {"k_step_pool<max,V1>", "k_step_pool<max,V2>", "k_step_pool<max,V4>",
                                     "k_step_pool<max,V8>"}};
  const int v = vec_width(g);
  return names[g.op == OP_MAX_POOL][v == 8 ? 3 : v == 4 ? 2 : v == 2 ? 1 : 0];
}

}  // namespace co
