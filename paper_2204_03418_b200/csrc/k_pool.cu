// k_pool.cu — continual max / average pooling (PAPER.md
// P:380-394 "Pooling: co.AvgPool1d, co.MaxPool1d, etc.").
//
// Pooling is separable: a window's max / sum over (t, h, w) is the max / sum
// over its kt temporal taps of each frame's spatial-window reduction.  So the
// handle keeps a ring of f + 1 SPATIALLY REDUCED frames (B, Ho, Wo, C) -- the
// input dtype for MAX (a max of representable values is exact), fp32 spatial
// sums for AVG -- and one fused kernel per step reduces the new frame once,
// stores it in slot m mod f, and on a Ready tick folds the window's kt-1 older
// slots with it.  Each input frame is read from HBM once (the spatial window's
// overlapping reads hit L1), however long the temporal window: the paper's
// expanded 64-step global average pooling reads 64 reduced 1x1 frames,
// not 64 full ones.  Temporal padding lives in the ring as the reduction's
// identity -- 0 for AVG (counted in the divisor kt kh kw, count_include_pad,
// DESIGN.md A21), -inf for MAX (ignored, PyTorch's implicit MAX padding, A22)
// -- so clean state, pad_end steps (x == NULL) and saved state need no flags.
// Spatial out-of-frame taps are skipped (the identity).  Ring slots are
// computed on the device from m, so kt is not bounded by CO_MAX_KT.
//
// CUDA cores: no contraction, the bound is HBM.  Thread = (stream, output
// pixel, vector of V channels); consecutive threads take consecutive channel
// vectors, so frame reads, ring accesses and output writes are coalesced
// 16-byte accesses.
#include <type_traits>

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

// Spatial window reduction of one frame into s[V] (the identity for an
// all-outside window).  Shared by the step and batch kernels, so both reduce in
// the same order and agree bitwise.
template <typename Tin, int V, bool MAX>
__device__ __forceinline__ void spatial_reduce(const Geom& g, const Tin* __restrict__ fb, int ho, int wo, int c0,
                                               float (&s)[V]) {
#pragma unroll
  for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
  for (int u = 0; u < g.kh; ++u) {
    const int hi = ho * g.sh + u * g.dh - g.ph;
    if (hi < 0 || hi >= g.H) continue;
    for (int v = 0; v < g.kw; ++v) {
      const int wi = wo * g.sw + v * g.dw - g.pw;
      if (wi < 0 || wi >= g.W) continue;
      const Vec<Tin, V> x = *reinterpret_cast<const Vec<Tin, V>*>(fb + (int64_t(hi) * g.W + wi) * g.Cin + c0);
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(x.v[j])) : s[j] + to_f(x.v[j]);
    }
  }
}

template <int V, bool MAX>
__device__ __forceinline__ void combine(float (&acc)[V], const float (&s)[V]) {
#pragma unroll
  for (int j = 0; j < V; ++j) acc[j] = MAX ? fmaxf(acc[j], s[j]) : acc[j] + s[j];
}

template <typename Tout, int V, bool MAX>
__device__ __forceinline__ void store_out(const Geom& g, Tout* __restrict__ yp, const float (&acc)[V]) {
  const float inv = 1.f / float(g.kt * g.kh * g.kw);
  Vec<Tout, V> o;
#pragma unroll
  for (int j = 0; j < V; ++j) o.v[j] = from_f<Tout>(activate(MAX ? acc[j] : acc[j] * inv, g.act));
  *reinterpret_cast<Vec<Tout, V>*>(yp) = o;
}

__device__ __forceinline__ int64_t fmod_pos(int64_t a, int64_t b) {
  const int64_t r = a % b;
  return r < 0 ? r + b : r;
}

// Step: reduce the new frame spatially (x == NULL: a padding frame), store it
// in ring slot a.slot[0] (-1: update_state = 0, nothing stored), and on a Ready
// tick fold the window's kt-1 older slots (m - j dil) mod f with it.
// Ring layout [slot][B][Ho][Wo][C] in Tr (input dtype for MAX, fp32 for AVG).
template <typename Tin, typename Tout, typename Tr, int V, bool MAX>
__global__ void __launch_bounds__(256) k_step_pool(Geom g, StepArgs a) {
  const int CV = g.Cin / V;
  const int64_t total = g.B * g.HWo * CV;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  Tr* ring = reinterpret_cast<Tr*>(a.state);
  const int64_t slot_elems = g.B * g.HWo * g.Cin;
  const Tin* x = static_cast<const Tin*>(a.x);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c0 = int(idx % CV) * V;
    const int64_t r = idx / CV;                 // b * HWo + p
    const int p = int(r % g.HWo);
    const int64_t b = r / g.HWo;
    const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
    float s[V];
    if (x) {
      spatial_reduce<Tin, V, MAX>(g, x + b * a.x_bstride, ho, wo, c0, s);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
    }
    const int64_t off = r * g.Cin + c0;
    if (a.slot[0] >= 0) {
      Vec<Tr, V> w;
#pragma unroll
      for (int j = 0; j < V; ++j) w.v[j] = from_f<Tr>(s[j]);
      *reinterpret_cast<Vec<Tr, V>*>(ring + int64_t(a.slot[0]) * slot_elems + off) = w;
    }
    if (!a.emit) continue;
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = MAX ? -INFINITY : 0.f;
    for (int k = 0; k + 1 < g.kt; ++k) {
      const int64_t slot = fmod_pos(a.m - int64_t(g.kt - 1 - k) * g.dt, g.f);
      const Vec<Tr, V> q = *reinterpret_cast<const Vec<Tr, V>*>(ring + slot * slot_elems + off);
      float t[V];
#pragma unroll
      for (int j = 0; j < V; ++j) t[j] = to_f(q.v[j]);
      combine<V, MAX>(acc, t);
    }
    combine<V, MAX>(acc, s);
    store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + int64_t(p) * g.Cout + c0, acc);
  }
}

// Batch mode: y[b, t'] = fold over taps k of the spatial reduction of
// frame t' s + k dil - p_t (padding outside [0, T): the identity).  Same
// reduction order as the step kernel.  Reads no state.
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
      if (t < 0 || t >= T) continue;            // padding: the identity
      float s[V];
      spatial_reduce<Tin, V, MAX>(g, x + (b * T + t) * g.frame_elems, ho, wo, c0, s);
      combine<V, MAX>(acc, s);
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
  using Tr = typename std::conditional<MAX, Tin, float>::type;
  const int V = vec_width(g);
  const int64_t total = g.B * g.HWo * (g.Cin / V);
  const int grid = grid_for(total);
  switch (V) {
    case 8: k_step_pool<Tin, Tout, Tr, 8, MAX><<<grid, 256, 0, s>>>(g, a); break;
    case 4: k_step_pool<Tin, Tout, Tr, 4, MAX><<<grid, 256, 0, s>>>(g, a); break;
    case 2: k_step_pool<Tin, Tout, Tr, 2, MAX><<<grid, 256, 0, s>>>(g, a); break;
    default: k_step_pool<Tin, Tout, Tr, 1, MAX><<<grid, 256, 0, s>>>(g, a); break;
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
  if (g.op != OP_MAX_POOL) return cudaMemsetAsync(p, 0, size_t(n_elems) * pool_ring_esz(g), s);
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
