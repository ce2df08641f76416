// k_direct.cu — generic CUDA-core kernels (sm_100a) for the continual
// convolution step: K1 `k_step_direct` (any groups / dilation / spatial and
// temporal stride, fp32 or bf16 in, fp32 accumulate + fp32 state), K5
// `k_forward_direct` (batch mode, verification), weight packing and the
// canonical state get / set gathers.
//
// K1 is the path for fp32 layers (config C1: TF32 tensor cores would break the
// 1e-4 tolerance, SURVEY §8a dispatch rule) and for shapes the specialised
// kernels do not cover.  One thread owns one (stream, output pixel, output
// channel) element; consecutive threads are consecutive output channels, so
// the packed weights [kt][kh][kw][Cin/g][Cout] are read coalesced and the
// channels-last input pixel is a warp broadcast.
//
// Per step (BASELINE.json north_star): for every temporal
// slice k the partial P_k = W[:,:,k] (*) x_t is formed and routed to the ring
// slot the host clock assigned: k = kt-1 completes an output (y = S + P + b,
// emitted if ready), 0 < k < kt-1 accumulate (S += P), k = 0 starts a new
// output (S = P) after the emit has read the slot.
#include "common.cuh"

namespace co {

template <typename Tin>
__device__ __forceinline__ float slice_partial(const Geom& g, const Tin* __restrict__ xb,
                                               const float* __restrict__ w, int k, int ho, int wo, int o,
                                               int grp) {
  float acc = 0.f;
  for (int u = 0; u < g.kh; ++u) {
    const int hi = ho * g.sh + u * g.dh - g.ph;
    if (hi < 0 || hi >= g.H) continue;
    for (int v = 0; v < g.kw; ++v) {
      const int wi = wo * g.sw + v * g.dw - g.pw;
      if (wi < 0 || wi >= g.W) continue;
      const Tin* xp = xb + (int64_t(hi) * g.W + wi) * g.Cin + grp * g.cig;
      const float* wp = w + ((int64_t(k * g.kh + u) * g.kw + v) * g.cig) * g.Cout + o;
      for (int c = 0; c < g.cig; ++c) acc = fmaf(wp[int64_t(c) * g.Cout], to_f(xp[c]), acc);
    }
  }
  return acc;
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) k_step_direct(Geom g, StepArgs a, const float* __restrict__ w,
                                                     const float* __restrict__ bias) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = g.B * g.HWo * g.Cout;
  if (idx >= total) return;
  const int o = int(idx % g.Cout);
  const int64_t pix = idx / g.Cout;          // b * HWo + p
  const int64_t b = pix / g.HWo;
  const int p = int(pix - b * g.HWo);
  const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
  const int grp = o / g.cog;
  const Tin* xb = a.x ? static_cast<const Tin*>(a.x) + b * a.x_bstride : nullptr;
  auto P = [&](int k) -> float { return xb ? slice_partial<Tin>(g, xb, w, k, ho, wo, o, grp) : 0.f; };

  // (1) complete + emit: read the slot before any overwrite of it.
  if (a.emit) {
    const int k = g.kt - 1;
    float v = P(k) + (bias ? bias[o] : 0.f);
    if (g.kt > 1) v += a.state[state_index(g, a.slot[k], pix, o)];
    v = activate(v, g.act);
    static_cast<Tout*>(a.y)[b * a.y_bstride + int64_t(p) * g.Cout + o] = from_f<Tout>(v);
  }
  if (!a.update || g.kt == 1) return;
  // (2) accumulate into the pending outputs.
  for (int k = g.kt - 2; k >= 1; --k) {
    if (a.slot[k] < 0) continue;
    const int64_t si = state_index(g, a.slot[k], pix, o);
    a.state[si] += P(k);
  }
  // (3) start the newest output (overwrites the slot the emit just read).
  if (a.slot[0] >= 0) a.state[state_index(g, a.slot[0], pix, o)] = P(0);
}

// RAW layout: the whole window column from the ring of input
// frames -- y = b + sum_k W[:,:,k] (*) frame(slot[k]) -- with no state written
// (the host stored the frame in its ring slot before the launch).
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) k_step_direct_raw(Geom g, StepArgs a, const float* __restrict__ w,
                                                         const float* __restrict__ bias) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = g.B * g.HWo * g.Cout;
  if (idx >= total) return;
  const int o = int(idx % g.Cout);
  const int64_t pix = idx / g.Cout;
  const int64_t b = pix / g.HWo;
  const int p = int(pix - b * g.HWo);
  const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
  const int grp = o / g.cog;
  const Tin* ring = static_cast<const Tin*>(static_cast<const void*>(a.state));
  float acc = bias ? bias[o] : 0.f;
  for (int k = 0; k < g.kt; ++k)
    acc += slice_partial<Tin>(g, ring + (int64_t(a.slot[k]) * g.B + b) * g.frame_elems, w, k, ho, wo, o, grp);
  static_cast<Tout*>(a.y)[b * a.y_bstride + int64_t(p) * g.Cout + o] = from_f<Tout>(activate(acc, g.act));
}

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) k_forward_direct(Geom g, const Tin* __restrict__ x, int64_t T,
                                                        Tout* __restrict__ y, int64_t Tp,
                                                        const float* __restrict__ w,
                                                        const float* __restrict__ bias) {
  // Batch mode: y[b, t', p, o] = b[o] + sum_k W_k (*) x[b, t' s + k dil - p_t]
  // with zero frames outside [0, T).  Reads no state.
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = g.B * Tp * g.HWo * g.Cout;
  if (idx >= total) return;
  const int o = int(idx % g.Cout);
  int64_t r = idx / g.Cout;
  const int p = int(r % g.HWo);
  r /= g.HWo;
  const int64_t tp = r % Tp;
  const int64_t b = r / Tp;
  const int ho = p / g.Wo, wo = p % g.Wo;
  const int grp = o / g.cog;
  const int64_t frame = int64_t(g.H) * g.W * g.Cin;
  float acc = bias ? bias[o] : 0.f;
  for (int k = 0; k < g.kt; ++k) {
    const int64_t t = tp * g.st + int64_t(k) * g.dt - g.pt;
    if (t < 0 || t >= T) continue;
    acc += slice_partial<Tin>(g, x + (b * T + t) * frame, w, k, ho, wo, o, grp);
  }
  acc = activate(acc, g.act);
  y[((b * Tp + tp) * g.HWo + p) * g.Cout + o] = from_f<Tout>(acc);
}

template <typename Tw>
__global__ void k_pack_direct(Geom g, const Tw* __restrict__ w, float* __restrict__ out) {
  // (Cout, Cin/g, kt, kh, kw) -> [kt][kh][kw][Cin/g][Cout] fp32 (exact for bf16).
  const int64_t n = int64_t(g.Cout) * g.cig * g.kt * g.kh * g.kw;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t r = i;
  const int v = int(r % g.kw); r /= g.kw;
  const int u = int(r % g.kh); r /= g.kh;
  const int k = int(r % g.kt); r /= g.kt;
  const int c = int(r % g.cig); r /= g.cig;
  const int o = int(r);
  out[(((int64_t(k) * g.kh + u) * g.kw + v) * g.cig + c) * g.Cout + o] = to_f(w[i]);
}

// Canonical state (R, B, Ho, Wo, Cout): slot j <-> output i = i_next + j, held
// physically in ring slot (head + j) mod R.  Outputs never emitted (i < 0) or
// not started yet (i s >= m_next, possible only for s > 1) read as 0.
__global__ void k_state_get(Geom g, const float* __restrict__ state, float* __restrict__ dst, int head,
                            int64_t i_next, int64_t m_next) {
  const int64_t per_slot = g.B * g.HWo * g.Cout;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= per_slot * g.R) return;
  const int j = int(idx / per_slot);
  const int64_t r = idx - int64_t(j) * per_slot;
  const int o = int(r % g.Cout);
  const int64_t pix = r / g.Cout;
  const int64_t i = i_next + j;
  float v = 0.f;
  if (i >= 0 && i * g.st < m_next) v = state[state_index(g, (head + j) % g.R, pix, o)];
  dst[idx] = v;
}

__global__ void k_state_set(Geom g, float* __restrict__ state, const float* __restrict__ src, int head) {
  const int64_t per_slot = g.B * g.HWo * g.Cout;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= per_slot * g.R) return;
  const int j = int(idx / per_slot);
  const int64_t r = idx - int64_t(j) * per_slot;
  const int o = int(r % g.Cout);
  const int64_t pix = r / g.Cout;
  state[state_index(g, (head + j) % g.R, pix, o)] = src[idx];
}

static inline unsigned blocks_for(int64_t n, int t) { return unsigned((n + t - 1) / t); }

cudaError_t launch_step_direct(const Geom& g, const StepArgs& a, const float* w, const float* bias,
                               cudaStream_t s) {
  const int64_t n = g.B * g.HWo * g.Cout;
  if (n == 0) return cudaSuccess;
  const unsigned nb = blocks_for(n, 256);
  if (g.in_dtype == F32 && g.out_dtype == F32)
    k_step_direct<float, float><<<nb, 256, 0, s>>>(g, a, w, bias);
  else if (g.in_dtype == F32 && g.out_dtype == BF16)
    k_step_direct<float, __nv_bfloat16><<<nb, 256, 0, s>>>(g, a, w, bias);
  else if (g.in_dtype == BF16 && g.out_dtype == F32)
    k_step_direct<__nv_bfloat16, float><<<nb, 256, 0, s>>>(g, a, w, bias);
  else
    k_step_direct<__nv_bfloat16, __nv_bfloat16><<<nb, 256, 0, s>>>(g, a, w, bias);
  return cudaGetLastError();
}

cudaError_t launch_step_direct_raw(const Geom& g, const StepArgs& a, const float* w, const float* bias,
                                   cudaStream_t s) {
  const int64_t n = g.B * g.HWo * g.Cout;
  if (n == 0) return cudaSuccess;
  const unsigned nb = blocks_for(n, 256);
  if (g.in_dtype == F32 && g.out_dtype == F32)
    k_step_direct_raw<float, float><<<nb, 256, 0, s>>>(g, a, w, bias);
  else if (g.in_dtype == F32 && g.out_dtype == BF16)
    k_step_direct_raw<float, __nv_bfloat16><<<nb, 256, 0, s>>>(g, a, w, bias);
  else if (g.in_dtype == BF16 && g.out_dtype == F32)
    k_step_direct_raw<__nv_bfloat16, float><<<nb, 256, 0, s>>>(g, a, w, bias);
  else
    k_step_direct_raw<__nv_bfloat16, __nv_bfloat16><<<nb, 256, 0, s>>>(g, a, w, bias);
  return cudaGetLastError();
}

cudaError_t launch_forward_direct(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp,
                                  const float* w, const float* bias, cudaStream_t s) {
  const int64_t n = g.B * Tp * g.HWo * g.Cout;
  if (n == 0) return cudaSuccess;
  const unsigned nb = blocks_for(n, 256);
  if (g.in_dtype == F32 && g.out_dtype == F32)
    k_forward_direct<float, float><<<nb, 256, 0, s>>>(g, (const float*)x, T, (float*)y, Tp, w, bias);
  else if (g.in_dtype == F32 && g.out_dtype == BF16)
    k_forward_direct<float, __nv_bfloat16><<<nb, 256, 0, s>>>(g, (const float*)x, T, (__nv_bfloat16*)y, Tp, w, bias);
  else if (g.in_dtype == BF16 && g.out_dtype == F32)
    k_forward_direct<__nv_bfloat16, float><<<nb, 256, 0, s>>>(g, (const __nv_bfloat16*)x, T, (float*)y, Tp, w, bias);
  else
    k_forward_direct<__nv_bfloat16, __nv_bfloat16><<<nb, 256, 0, s>>>(g, (const __nv_bfloat16*)x, T,
                                                                      (__nv_bfloat16*)y, Tp, w, bias);
  return cudaGetLastError();
}

cudaError_t launch_pack_direct_weights(const Geom& g, const void* w, float* out, cudaStream_t s) {
  const int64_t n = int64_t(g.Cout) * g.cig * g.kt * g.kh * g.kw;
  if (g.in_dtype == F32)
    k_pack_direct<float><<<blocks_for(n, 256), 256, 0, s>>>(g, (const float*)w, out);
  else
    k_pack_direct<__nv_bfloat16><<<blocks_for(n, 256), 256, 0, s>>>(g, (const __nv_bfloat16*)w, out);
  return cudaGetLastError();
}

cudaError_t launch_state_get(const Geom& g, const float* state, float* dst, int head, int64_t i_next,
                             int64_t m_next, cudaStream_t s) {
  const int64_t n = g.B * g.HWo * g.Cout * g.R;
  if (n == 0) return cudaSuccess;
  k_state_get<<<blocks_for(n, 256), 256, 0, s>>>(g, state, dst, head, i_next, m_next);
  return cudaGetLastError();
}

cudaError_t launch_state_set(const Geom& g, float* state, const float* src, int head, cudaStream_t s) {
  const int64_t n = g.B * g.HWo * g.Cout * g.R;
  if (n == 0) return cudaSuccess;
  k_state_set<<<blocks_for(n, 256), 256, 0, s>>>(g, state, src, head);
  return cudaGetLastError();
}

}  // namespace co

// ---- per-stream clean --------------------------------------
namespace co {

// PSUM layouts: zero every state element (slot, pixel, channel) of the listed
// streams, through state_index so every physical layout (quad-major,
// tile-blocked, channels-last) is covered.
__global__ void k_clean_streams_psum(Geom g, float* __restrict__ state, const int64_t* __restrict__ ids, int nm) {
  const int64_t per = g.HWo * g.Cout;
  const int64_t total = int64_t(g.R) * nm * per;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int o = int(i % g.Cout);
    int64_t r = i / g.Cout;
    const int64_t p = r % g.HWo;
    r /= g.HWo;
    const int j = int(r % nm);
    const int slot = int(r / nm);
    state[state_index(g, slot, ids[j] * g.HWo + p, o)] = 0.f;
  }
}

// Ring layouts ([slot][B][per-stream elements]): set the listed streams'
// elements of every slot to `value` (a 2- or 4-byte bit pattern).
template <typename T>
__global__ void k_fill_streams(T* __restrict__ ring, int64_t slots, int64_t B, int64_t per, const int64_t* __restrict__ ids,
                               int nm, T value) {
  const int64_t total = slots * nm * per;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = i % per;
    const int64_t r = i / per;
    const int j = int(r % nm);
    const int64_t slot = r / nm;
    ring[(slot * B + ids[j]) * per + e] = value;
  }
}

static int clean_grid(int64_t total) {
  const int64_t b = (total + 255) / 256;
  return int(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

cudaError_t launch_clean_streams_psum(const Geom& g, float* state, const int64_t* ids, int nm, cudaStream_t s) {
  const int64_t total = int64_t(g.R) * nm * g.HWo * g.Cout;
  if (total == 0) return cudaSuccess;
  k_clean_streams_psum<<<clean_grid(total), 256, 0, s>>>(g, state, ids, nm);
  return cudaGetLastError();
}

cudaError_t launch_fill_streams(void* ring, int esz, int64_t slots, int64_t B, int64_t per, const int64_t* ids, int nm,
                                uint32_t value, cudaStream_t s) {
  const int64_t total = slots * nm * per;
  if (total == 0) return cudaSuccess;
  if (esz == 2)
    k_fill_streams<uint16_t><<<clean_grid(total), 256, 0, s>>>(static_cast<uint16_t*>(ring), slots, B, per, ids, nm,
                                                               uint16_t(value));
  else
    k_fill_streams<uint32_t><<<clean_grid(total), 256, 0, s>>>(static_cast<uint32_t*>(ring), slots, B, per, ids, nm,
                                                               value);
  return cudaGetLastError();
}

}  // namespace co
