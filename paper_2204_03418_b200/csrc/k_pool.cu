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
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace co {

namespace {

// Temporal windows of at least this many taps use the block decomposition
// (temporal_step VH) instead of the direct fold of kt-1 ring slots.
constexpr int kVhMinKt = 6;
}  // namespace
bool pool_band_enabled();
namespace {

// Loads in flight per thread in the window loops (4 x 16 B: enough with >= 32
// resident warps per SM; deeper chunks cost registers and occupancy).
constexpr int kChunk = 4;

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
// all-outside window): taps j = j0, j0 + jstep, ... of the kh x kw window in
// row-major order, loaded kChunk at a time so their latencies overlap.  The step and
// batch kernels use the same order (jstep = 1), so they agree bitwise.
template <typename Tin, int V, bool MAX, int CH = kChunk>
__device__ __forceinline__ void spatial_reduce(const Geom& g, const Tin* __restrict__ fb, int ho, int wo, int c0,
                                               float (&s)[V], int j0 = 0, int jstep = 1) {
#pragma unroll
  for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
  const int nt = g.kh * g.kw;
  const int h0 = ho * g.sh - g.ph, w0 = wo * g.sw - g.pw;
  if constexpr (CH == 1) {       // one load in flight: plain nested loops (no per-tap divide)
    if (jstep == 1) {
      for (int u = 0; u < g.kh; ++u) {
        const int hi = h0 + u * g.dh;
        if (hi < 0 || hi >= g.H) continue;
        for (int v = 0; v < g.kw; ++v) {
          const int wi = w0 + v * g.dw;
          if (wi < 0 || wi >= g.W) continue;
          const Vec<Tin, V> x = *reinterpret_cast<const Vec<Tin, V>*>(fb + (int64_t(hi) * g.W + wi) * g.Cin + c0);
#pragma unroll
          for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(x.v[j])) : s[j] + to_f(x.v[j]);
        }
      }
      return;
    }
  }
  for (int jb = j0; jb < nt; jb += CH * jstep) {
    Vec<Tin, V> x[CH];
    bool ok[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int j = jb + i * jstep;
      const int u = j / g.kw, v = j - (j / g.kw) * g.kw;
      const int hi = h0 + u * g.dh, wi = w0 + v * g.dw;
      ok[i] = j < nt && hi >= 0 && hi < g.H && wi >= 0 && wi < g.W;
      if (ok[i]) x[i] = *reinterpret_cast<const Vec<Tin, V>*>(fb + (int64_t(hi) * g.W + wi) * g.Cin + c0);
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (!ok[i]) continue;
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(x[i].v[j])) : s[j] + to_f(x[i].v[j]);
    }
  }
}

// Compile-time KH x KW window (dilation 1): every tap's load is issued before
// any is combined (predicated, no per-tap branch), so a thread has KH*KW
// 16-byte loads in flight -- the runtime-bounds loop above issues them one at a
// time.  Same tap order, so the same results bit for bit.
template <typename Tin, int V, bool MAX, int KH, int KW>
__device__ __forceinline__ void spatial_reduce_fixed(const Geom& g, const Tin* __restrict__ fb, int ho, int wo,
                                                     int c0, float (&s)[V]) {
  const int h0 = ho * g.sh - g.ph, w0 = wo * g.sw - g.pw;
  Vec<Tin, V> x[KH * KW];
  bool ok[KH * KW];
#pragma unroll
  for (int u = 0; u < KH; ++u)
#pragma unroll
    for (int v = 0; v < KW; ++v) {
      const int hi = h0 + u, wi = w0 + v;
      ok[u * KW + v] = hi >= 0 && hi < g.H && wi >= 0 && wi < g.W;
      if (ok[u * KW + v]) x[u * KW + v] = *reinterpret_cast<const Vec<Tin, V>*>(fb + (int64_t(hi) * g.W + wi) * g.Cin + c0);
    }
#pragma unroll
  for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
#pragma unroll
  for (int t = 0; t < KH * KW; ++t) {
    if (!ok[t]) continue;
#pragma unroll
    for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(x[t].v[j])) : s[j] + to_f(x[t].v[j]);
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

// (mm - d) mod f for 0 <= mm < f, 0 <= d < f
__device__ __forceinline__ int wrap_sub(int mm, int d, int f) {
  const int r = mm - d;
  return r < 0 ? r + f : r;
}

// Fold the window's older ring slots k = k0, k0 + kstep, ... < kt-1 (slot of
// tap k: (m - (kt-1-k) dil) mod f, from mm = m mod f) into acc, in k order,
// kChunk loads in flight.
template <typename Tr, int V, bool MAX, int CH = kChunk>
__device__ __forceinline__ void ring_fold(const Geom& g, const Tr* __restrict__ ring, int64_t slot_elems,
                                          int64_t off, int mm, float (&acc)[V], int k0 = 0, int kstep = 1) {
  for (int kb = k0; kb + 1 < g.kt; kb += CH * kstep) {
    Vec<Tr, V> q[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int k = kb + i * kstep;
      if (k + 1 < g.kt) {
        const int slot = wrap_sub(mm, (g.kt - 1 - k) * g.dt, g.f);
        q[i] = *reinterpret_cast<const Vec<Tr, V>*>(ring + slot * slot_elems + off);
      }
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (kb + i * kstep + 1 >= g.kt) continue;
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = MAX ? fmaxf(acc[j], to_f(q[i].v[j])) : acc[j] + to_f(q[i].v[j]);
    }
  }
}

// Temporal part of a step, given the new frame's spatial reduction s: store s
// in ring slot a.slot[0] (-1: update_state = 0, nothing stored) and, when
// Ready, produce the window's reduction win.
//  !VH: direct fold of the window's kt-1 older ring slots, then s (the batch
//       kernel's order: bitwise equal to it).
//   VH: van Herk / Gil-Werman block decomposition per temporal phase q =
//       m mod dil (phase index i = m div dil, blocks of kt phase frames): P[q]
//       is the running reduction of the current block up to i, and at a block
//       end one suffix pass writes S[q][j mod kt] = reduction of frames j..end
//       of that block.  A window [i-kt+1, i] is P[q] when i ends a block, else
//       S[q][(i-kt+1) mod kt] (+) P[q].  O(1) per step (plus one kt-long pass
//       per kt steps) -- the role of SPEC's running-sum average and monotonic
//       deque, but exact for MAX, drift-free for AVG (a fixed two-term
//       sum, no subtraction) and free of data-dependent control flow.
//  State after the ring: P (dil slots), then S (dil * kt slots), each slot
//  laid out like a ring slot.
template <typename Tr, int V, bool MAX, bool VH, int CH>
__device__ __forceinline__ void temporal_step(const Geom& g, const StepArgs& a, Tr* __restrict__ st, int64_t SE,
                                              int64_t off, const float (&s)[V], float (&win)[V]) {
  if (a.slot[0] >= 0) {
    Vec<Tr, V> w;
#pragma unroll
    for (int j = 0; j < V; ++j) w.v[j] = from_f<Tr>(s[j]);
    *reinterpret_cast<Vec<Tr, V>*>(st + int64_t(a.slot[0]) * SE + off) = w;
  }
  if constexpr (!VH) {
    if (a.emit) {
#pragma unroll
      for (int j = 0; j < V; ++j) win[j] = MAX ? -INFINITY : 0.f;
      ring_fold<Tr, V, MAX, CH>(g, st, SE, off, a.pm_f, win);
      combine<V, MAX>(win, s);
    }
  } else {
    const int q = a.pm_q, pos = a.pm_pos;
    Tr* P = st + (int64_t(g.f + 1) + q) * SE + off;
    Tr* S = st + (int64_t(g.f + 1) + g.dt + q * g.kt) * SE + off;
    float pn[V];
#pragma unroll
    for (int j = 0; j < V; ++j) pn[j] = MAX ? -INFINITY : 0.f;
    if (pos > 0) {
      const Vec<Tr, V> pv = *reinterpret_cast<const Vec<Tr, V>*>(P);
#pragma unroll
      for (int j = 0; j < V; ++j) pn[j] = to_f(pv.v[j]);
    }
    combine<V, MAX>(pn, s);
    if (a.emit) {
      if (pos == g.kt - 1) {
#pragma unroll
        for (int j = 0; j < V; ++j) win[j] = pn[j];
      } else {
        const Vec<Tr, V> sv = *reinterpret_cast<const Vec<Tr, V>*>(S + a.pm_js * SE);
#pragma unroll
        for (int j = 0; j < V; ++j) win[j] = to_f(sv.v[j]);
        combine<V, MAX>(win, pn);
      }
    }
    if (a.update) {
      Vec<Tr, V> w;
#pragma unroll
      for (int j = 0; j < V; ++j) w.v[j] = from_f<Tr>(pn[j]);
      *reinterpret_cast<Vec<Tr, V>*>(P) = w;
      if (pos == g.kt - 1) {           // block end: suffix pass over its kt phase frames
        // (64-bit index arithmetic kept here: the 32-bit wrap_sub form of this
        // rare branch measured 8 us slower per step on the expanded 64-step pool)
        const int64_t i = a.m / g.dt;
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = s[j];
        Vec<Tr, V> o;
#pragma unroll
        for (int j = 0; j < V; ++j) o.v[j] = from_f<Tr>(acc[j]);
        *reinterpret_cast<Vec<Tr, V>*>(S + fmod_pos(i, g.kt) * SE) = o;
        for (int t = 1; t < g.kt; ++t) {
          const Vec<Tr, V> r =
              *reinterpret_cast<const Vec<Tr, V>*>(st + fmod_pos(a.m - int64_t(t) * g.dt, g.f) * SE + off);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            acc[j] = MAX ? fmaxf(to_f(r.v[j]), acc[j]) : to_f(r.v[j]) + acc[j];
            o.v[j] = from_f<Tr>(acc[j]);
          }
          *reinterpret_cast<Vec<Tr, V>*>(S + fmod_pos(i - t, g.kt) * SE) = o;
        }
      }
    }
  }
}

// Rebuild P and S of the block decomposition from the ring (after
// co_state_set): for phase q, with m' the last stepped frame of the phase,
// P[q] = the reduction of m''s block up to m' in step order, and S = the suffix
// pass of the last completed block, restricted to the window starts that
// future steps read (all inside the f-1 frames the ring holds).  Same
// operations in the same order as the steps, so the values are bitwise those
// an uninterrupted run would hold.
template <typename Tr, int V, bool MAX>
__global__ void k_pool_rebuild(Geom g, Tr* __restrict__ st, int64_t m_next) {
  const int CV = g.Cin / V;
  const int64_t SE = g.B * g.HWo * g.Cin;
  const int64_t total = g.B * g.HWo * CV;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t off = (idx / CV) * g.Cin + (idx % CV) * V;
    auto ring = [&](int64_t m) { return *reinterpret_cast<const Vec<Tr, V>*>(st + fmod_pos(m, g.f) * SE + off); };
    for (int q = 0; q < g.dt; ++q) {
      Tr* P = st + (int64_t(g.f + 1) + q) * SE + off;
      Tr* S = st + (int64_t(g.f + 1) + g.dt + int64_t(q) * g.kt) * SE + off;
      const int64_t mp = (m_next - 1) - fmod_pos(m_next - 1 - q, g.dt);   // last stepped frame of phase q
      Vec<Tr, V> o;
      float acc[V];
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = MAX ? -INFINITY : 0.f;
      if (mp < 0) {                    // nothing stepped in this phase: identity
#pragma unroll
        for (int j = 0; j < V; ++j) o.v[j] = from_f<Tr>(acc[j]);
        *reinterpret_cast<Vec<Tr, V>*>(P) = o;
        for (int k = 0; k < g.kt; ++k) *reinterpret_cast<Vec<Tr, V>*>(S + k * SE) = o;
        continue;
      }
      const int64_t ip = (mp - q) / g.dt;
      const int pos = int(ip % g.kt);
      for (int t = pos; t >= 0; --t) {
        const Vec<Tr, V> r = ring(mp - int64_t(t) * g.dt);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = MAX ? fmaxf(acc[j], to_f(r.v[j])) : acc[j] + to_f(r.v[j]);
      }
#pragma unroll
      for (int j = 0; j < V; ++j) o.v[j] = from_f<Tr>(acc[j]);
      *reinterpret_cast<Vec<Tr, V>*>(P) = o;
      const int64_t e = (pos == g.kt - 1) ? ip : ip - pos - 1;        // last completed block's end
      if (e < 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) o.v[j] = from_f<Tr>(MAX ? -INFINITY : 0.f);
        for (int k = 0; k < g.kt; ++k) *reinterpret_cast<Vec<Tr, V>*>(S + k * SE) = o;
        continue;
      }
      const int64_t jmin = (ip - g.kt + 2 > e - g.kt + 1) ? ip - g.kt + 2 : e - g.kt + 1;
      {
        const Vec<Tr, V> r = ring(e * g.dt + q);
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = to_f(r.v[j]);
        *reinterpret_cast<Vec<Tr, V>*>(S + fmod_pos(e, g.kt) * SE) = r;
      }
      for (int64_t jj = e - 1; jj >= jmin; --jj) {
        const Vec<Tr, V> r = ring(jj * g.dt + q);
#pragma unroll
        for (int j = 0; j < V; ++j) {
          acc[j] = MAX ? fmaxf(to_f(r.v[j]), acc[j]) : to_f(r.v[j]) + acc[j];
          o.v[j] = from_f<Tr>(acc[j]);
        }
        *reinterpret_cast<Vec<Tr, V>*>(S + fmod_pos(jj, g.kt) * SE) = o;
      }
    }
  }
}

// Step: reduce the new frame spatially (x == NULL: a padding frame), then the
// temporal part (temporal_step).  Ring layout [slot][B][Ho][Wo][C] in Tr (input
// dtype for MAX, fp32 for AVG).
template <typename Tin, typename Tout, typename Tr, int V, bool MAX, int CH, bool VH, int KHW = 0>
__global__ void __launch_bounds__(256, (CH == 1 && KHW == 0) ? 4 : 2) k_step_pool(Geom g, StepArgs a) {
  const int CV = g.Cin / V;
  const int64_t total = g.B * g.HWo * CV;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  Tr* st = reinterpret_cast<Tr*>(a.state);
  const int64_t SE = g.B * g.HWo * g.Cin;
  const Tin* x = static_cast<const Tin*>(a.x);
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += stride) {
    const int c0 = int(idx % CV) * V;
    const int64_t r = idx / CV;                 // b * HWo + p
    const int p = int(r % g.HWo);
    const int64_t b = r / g.HWo;
    const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
    float s[V], win[V];
    if (x) {
      if constexpr (KHW > 0)
        spatial_reduce_fixed<Tin, V, MAX, KHW / 10, KHW % 10>(g, x + b * a.x_bstride, ho, wo, c0, s);
      else
        spatial_reduce<Tin, V, MAX, CH>(g, x + b * a.x_bstride, ho, wo, c0, s);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
    }
    temporal_step<Tr, V, MAX, VH, CH>(g, a, st, SE, r * g.Cin + c0, s, win);
    if (a.emit)
      store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + int64_t(p) * g.Cout + c0, win);
  }
}

// Row-band kernel for spatial windows (e.g. the I3D-style 3x3 s2 max pool): a
// CTA takes a band of TH output rows of one stream, stages the input rows the
// band's windows touch into shared memory with 16-byte cp.async (each input
// row read from HBM once, however many windows overlap it -- the plain kernel
// relies on L1 for that and measured 23% L1 hits on the stride-2 windows), then
// thread = (output pixel of the band, channel vector) reduces its window from
// shared memory in spatial_reduce's tap order (so the two kernels agree bit
// for bit) and runs the temporal part.  Out-of-frame taps are skipped, so
// MAX's -inf padding needs no fill.
template <typename Tin, typename Tout, typename Tr, int V, bool MAX, bool VH, int KHW = 0>
__global__ void __launch_bounds__(1024) k_step_pool_band(Geom g, StepArgs a, int TH, int rows) {
  // KHW > 0: compile-time KH x KW window (dilation 1), taps unrolled
  constexpr int CKH = KHW / 10, CKW = KHW % 10;
  extern __shared__ __align__(16) uint8_t pool_smem[];
  Tin* xs = reinterpret_cast<Tin*>(pool_smem);                  // [rows][W][C]
  const int CV = g.Cin / V;
  const int bands = (g.Ho + TH - 1) / TH;
  const int64_t SE = g.B * g.HWo * g.Cin;
  Tr* st = reinterpret_cast<Tr*>(a.state);
  const Tin* x = static_cast<const Tin*>(a.x);
  const int row_chunks = int(int64_t(g.W) * g.Cin * sizeof(Tin) / 16);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // see k_step_pool_split
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int64_t band = blockIdx.x; band < g.B * bands; band += gridDim.x) {
    const int64_t b = band / bands;
    const int ho0 = int(band % bands) * TH;
    const int hi0 = ho0 * g.sh - g.ph;                             // first input row the band touches
    __syncthreads();                                                // previous band finished reading xs
    if (x) {
      const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
      for (int rr = 0; rr < rows; ++rr) {
        const int hi = hi0 + rr;
        if (hi < 0 || hi >= g.H) continue;
        const char* src = reinterpret_cast<const char*>(x + b * a.x_bstride + int64_t(hi) * g.W * g.Cin);
        for (int i = threadIdx.x; i < row_chunks; i += blockDim.x)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + uint32_t((rr * row_chunks + i) * 16)),
                       "l"(src + int64_t(i) * 16)
                       : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    const int th = min(TH, g.Ho - ho0);
    for (int idx = threadIdx.x; idx < th * g.Wo * CV; idx += blockDim.x) {
      const int c0 = (idx % CV) * V;
      const int pl = idx / CV;                                      // pixel within the band
      const int ho = ho0 + pl / g.Wo, wo = pl % g.Wo;
      float s[V];
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
      if (x && KHW > 0) {
        const int h0 = ho * g.sh - g.ph, w0 = wo * g.sw - g.pw;
        const Tin* xb = xs + ((h0 - hi0) * g.W + w0) * g.Cin + c0;
#pragma unroll
        for (int u = 0; u < CKH; ++u) {
          if (h0 + u < 0 || h0 + u >= g.H) continue;
#pragma unroll
          for (int v = 0; v < CKW; ++v) {
            if (w0 + v < 0 || w0 + v >= g.W) continue;
            const Vec<Tin, V> xv = *reinterpret_cast<const Vec<Tin, V>*>(xb + (u * g.W + v) * g.Cin);
#pragma unroll
            for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(xv.v[j])) : s[j] + to_f(xv.v[j]);
          }
        }
      } else if (x) {
        for (int u = 0; u < g.kh; ++u) {
          const int hi = ho * g.sh - g.ph + u * g.dh;
          if (hi < 0 || hi >= g.H) continue;
          for (int v = 0; v < g.kw; ++v) {
            const int wi = wo * g.sw - g.pw + v * g.dw;
            if (wi < 0 || wi >= g.W) continue;
            const Vec<Tin, V> xv = *reinterpret_cast<const Vec<Tin, V>*>(xs + ((hi - hi0) * g.W + wi) * g.Cin + c0);
#pragma unroll
            for (int j = 0; j < V; ++j) s[j] = MAX ? fmaxf(s[j], to_f(xv.v[j])) : s[j] + to_f(xv.v[j]);
          }
        }
      }
      const int64_t r = b * g.HWo + int64_t(ho) * g.Wo + wo;
      float win[V];
      temporal_step<Tr, V, MAX, VH, 1>(g, a, st, SE, r * g.Cin + c0, s, win);
      if (a.emit)
        store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + (r - b * g.HWo) * g.Cout + c0, win);
    }
  }
}

// Band plan: TH output rows whose input rows fit in ~96 KB of shared memory and
// whose (pixel, vector) threads fit a 1024-thread CTA; 0 = no band kernel.
int band_rows(const Geom& g, int V, int& rows, size_t& smem) {
  if (g.kh * g.kw < 2 || (int64_t(g.W) * g.Cin * (g.in_dtype == BF16 ? 2 : 4)) % 16) return 0;
  const size_t row_bytes = size_t(g.W) * g.Cin * (g.in_dtype == BF16 ? 2 : 4);
  const int CV = g.Cin / V;
  // one output row per CTA (measured best on max3: 74.7 us vs 84.6 us at 2 rows and
  // 98.7 us at 4 -- small CTAs, many per SM, overlap one another's staging), or
  // just enough rows for 128 threads
  int th_max = std::min(g.Ho, std::min(1024 / std::max(1, g.Wo * CV), (128 + g.Wo * CV - 1) / std::max(1, g.Wo * CV)));
  th_max = std::max(th_max, 1);
  if (const int e = CO_EXP("CO_POOL_BAND_TH", 0)) th_max = std::min(th_max, std::max(1, e));   // A/B experiments
  for (int TH = th_max; TH >= 1; --TH) {
    rows = (TH - 1) * g.sh + (g.kh - 1) * g.dh + 1;
    smem = size_t(rows) * row_bytes;
    if (smem <= 96 * 1024) return TH;
  }
  return 0;
}

// Few output rows (e.g. the expanded global pool: one 1x1 row per stream) give
// the one-thread-per-vector kernel too few threads to cover HBM latency, so
// this variant gives each output row (b, pixel) a block of G x CV threads:
// lane g reduces spatial taps g, g+G, ... and ring slots g, g+G, ..., and the G
// partials are combined in g order through shared memory.  Same results as
// k_step_pool up to the AVG summation order (MAX: bitwise).
template <typename Tin, typename Tout, typename Tr, int V, bool MAX, bool VH>
__global__ void __launch_bounds__(512) k_step_pool_split(Geom g, StepArgs a) {
  extern __shared__ float sm_part[];                 // [2][G][CV][V]
  const int CV = g.Cin / V, G = blockDim.y;
  const int cv = threadIdx.x, gi = threadIdx.y;
  float* sp = sm_part;
  float* tp = sm_part + G * CV * V;
  Tr* ring = reinterpret_cast<Tr*>(a.state);
  const int64_t slot_elems = g.B * g.HWo * g.Cin;
  const Tin* x = static_cast<const Tin*>(a.x);
  const int c0 = cv * V;
  // programmatic dependent launch (launch_step_pool): let the next step's
  // blocks be scheduled, and wait for the previous grid's frame / ring writes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int64_t r = blockIdx.x; r < g.B * g.HWo; r += gridDim.x) {
    const int p = int(r % g.HWo);
    const int64_t b = r / g.HWo;
    const int ho = p / g.Wo, wo = p - (p / g.Wo) * g.Wo;
    const int64_t off = r * g.Cin + c0;
    float s[V], t[V];
    if (x) {
      spatial_reduce<Tin, V, MAX>(g, x + b * a.x_bstride, ho, wo, c0, s, gi, G);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) s[j] = MAX ? -INFINITY : 0.f;
    }
#pragma unroll
    for (int j = 0; j < V; ++j) t[j] = MAX ? -INFINITY : 0.f;
    if (!VH && a.emit) ring_fold<Tr, V, MAX>(g, ring, slot_elems, off, a.pm_f, t, gi, G);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      sp[(gi * CV + cv) * V + j] = s[j];
      tp[(gi * CV + cv) * V + j] = t[j];
    }
    __syncthreads();
    if (gi == 0) {
      for (int q = 1; q < G; ++q) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const float sv = sp[(q * CV + cv) * V + j], tv = tp[(q * CV + cv) * V + j];
          s[j] = MAX ? fmaxf(s[j], sv) : s[j] + sv;
          t[j] = MAX ? fmaxf(t[j], tv) : t[j] + tv;
        }
      }
      if constexpr (VH) {
        temporal_step<Tr, V, MAX, true, kChunk>(g, a, ring, slot_elems, off, s, t);
      } else {
        if (a.slot[0] >= 0) {
          Vec<Tr, V> w;
#pragma unroll
          for (int j = 0; j < V; ++j) w.v[j] = from_f<Tr>(s[j]);
          *reinterpret_cast<Vec<Tr, V>*>(ring + int64_t(a.slot[0]) * slot_elems + off) = w;
        }
        if (a.emit) combine<V, MAX>(t, s);
      }
      if (a.emit)
        store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + int64_t(p) * g.Cout + c0, t);
    }
    __syncthreads();
  }
}

// Batch mode: y[b, t'] = fold over taps k of the spatial reduction of
// frame t' s + k dil - p_t (padding outside [0, T): the identity).  Same
// reduction order as the step kernel.  Reads no state.
template <typename Tin, typename Tout, int V, bool MAX, int CH>
__global__ void __launch_bounds__(256, CH == 1 ? 4 : 2) k_forward_pool(Geom g, const Tin* __restrict__ x, int64_t T,
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
      spatial_reduce<Tin, V, MAX, CH>(g, x + (b * T + t) * g.frame_elems, ho, wo, c0, s);
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

int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Lanes per output vector of the split step kernel (1: the plain kernel).  The
// plain kernel needs about 2 x 148 x 1024 threads to keep HBM busy.
int split_lanes(const Geom& g) {
  const int CV = g.Cin / vec_width(g);
  const int64_t threads = g.B * g.HWo * CV;
  const int64_t target = int64_t(num_sms()) * 2048;
  if (threads >= target || CV > 256) return 1;
  // the fewest lanes that reach an eighth of the target (measured: x3d64's 27.6K
  // vectors run best at G = 2; more lanes add shared-memory reduction latency)
  int G = int((target / 8 + threads - 1) / threads);
  G = G < 2 ? 2 : (G > 8 ? 8 : G);
  while (G > 1 && G * CV > 512) --G;
  const int work = (g.kh * g.kw > g.kt - 1) ? g.kh * g.kw : g.kt - 1;
  if (G > work) G = work;
  return G < 2 ? 1 : G;
}

// Per-thread load depth of the plain kernels: with enough threads to fill the
// GPU several times over, occupancy hides latency best (1 load in flight, 6
// blocks / SM); few threads or long windows take kChunk loads in flight.
bool deep_chunks(const Geom& g, int64_t threads) {
  return threads < int64_t(num_sms()) * 2048 * 4 || g.kh * g.kw > 16;
}

bool pool_pdl() { return option(OPT_PDL) != 0; }   // option "pdl" = 0: plain stream serialization

int grid_for(int64_t total) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (total + 255) / 256;
  const int64_t cap = int64_t(sms) * 8;          // 8 x 256 threads resident per SM
  return int(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

template <typename Tin, typename Tout, typename Tr, int V, bool MAX, bool VH>
cudaError_t step_split(const Geom& g, const StepArgs& a, int G, cudaStream_t s) {
  const int CV = g.Cin / V;
  const size_t smem = size_t(2) * G * CV * V * sizeof(float);
  const int64_t rows = g.B * g.HWo;
  const int per_sm = 2048 / (G * CV) > 0 ? 2048 / (G * CV) : 1;   // resident blocks per SM
  const int64_t cap = int64_t(num_sms()) * per_sm;
  const int grid = int(rows < cap ? rows : cap);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_step_pool_split<Tin, Tout, Tr, V, MAX, VH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
  // launched with programmatic stream serialization: consecutive steps (a few
  // microseconds each for the expanded global pool) overlap launch and drain
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(unsigned(CV), unsigned(G));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pool_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_step_pool_split<Tin, Tout, Tr, V, MAX, VH>, g, a);
}

// ------------------------------------------------------------------ row pipeline (k_step_pool_seg)
// The band kernel's work with its memory traffic decoupled from the arithmetic
// (the K2s recipe, k_depthwise.cu): the band kernel stages a row's input rows
// with cp.async, waits for them, reduces, then reads its ring slots -- one
// dependent chain per block, ~0.5 of HBM on the I3D-style 3x3x3 max pool.  Here
// a block walks a contiguous range of units (stream, output row); a producer
// thread streams each unit's input rows (one contiguous run, clipped to the
// frame) and, on Ready steps, the kt - 1 older ring-slot rows into a ring of
// shared-memory stages by bulk copies; every consumer warp consumes every stage
// (thread = (output pixel, V-channel vector)), reducing the window from shared
// memory in the plain kernel's tap order and folding the ring rows in its slot
// order -- the same operations in the same order, so results are bitwise those
// of k_step_pool / k_step_pool_band.  Direct-fold windows only (kt < 6).
struct PoolSegPlan {
  int nst, stage_bytes;       // stage ring
  int x_rows, xrow_b;         // staged input rows per unit, bytes per input row
  int rrow_b, r_off;          // bytes per ring-slot row, offset of the ring rows in a stage
  int cwarps;                 // consumer warps
  int per_sm;
};

template <typename Tin, typename Tout, typename Tr, int V, bool MAX, int KHW = 0>
__global__ void __launch_bounds__(1024) k_step_pool_seg(Geom g, StepArgs a, PoolSegPlan pl) {
  // KHW > 0: compile-time KH x KW window (dilation 1), taps unrolled
  constexpr int CKH = KHW / 10, CKW = KHW % 10;
  extern __shared__ __align__(128) uint8_t seg_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(seg_smem + size_t(pl.nst) * pl.stage_bytes);
  uint64_t* empty = full + pl.nst;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < pl.nst; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], pl.cwarps);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // see k_step_pool_split
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t units = g.B * g.Ho;
  const int64_t lo = units * blockIdx.x / gridDim.x, hi = units * (blockIdx.x + 1) / gridDim.x;
  const int64_t SE = g.B * g.HWo * g.Cin;
  Tr* ring = reinterpret_cast<Tr*>(a.state);
  const Tin* x = static_cast<const Tin*>(a.x);
  const int nring = a.emit ? g.kt - 1 : 0;
  if (warp == pl.cwarps) {                          // ---- producer thread
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;                                // fill k of a stage waits for empty phase k - 1: parity ph ^ 1
    bool refill = false;
    int64_t b = lo / g.Ho;
    int ho = int(lo - b * g.Ho);
    for (int64_t u = lo; u < hi; ++u) {
      if (refill) ptx::mbar_wait(&empty[s], ph ^ 1u);
      uint8_t* st = seg_smem + size_t(s) * pl.stage_bytes;
      const int hi0 = ho * g.sh - g.ph;
      const int r_lo = max(hi0, 0), r_hi = min(hi0 + pl.x_rows - 1, g.H - 1);
      const uint32_t xb = (x && r_hi >= r_lo) ? uint32_t(r_hi - r_lo + 1) * uint32_t(pl.xrow_b) : 0u;
      const uint32_t tx = xb + uint32_t(nring) * uint32_t(pl.rrow_b);
      if (tx == 0) {
        ptx::mbar_arrive(&full[s]);
      } else {
        ptx::mbar_arrive_expect_tx(&full[s], tx);
        if (xb) ptx::bulk_g2s(st + (r_lo - hi0) * pl.xrow_b, x + b * a.x_bstride + int64_t(r_lo) * g.W * g.Cin, xb, &full[s]);
        for (int k = 0; k < nring; ++k) {
          const int slot = wrap_sub(a.pm_f, (g.kt - 1 - k) * g.dt, g.f);
          ptx::bulk_g2s(st + pl.r_off + k * pl.rrow_b,
                        ring + int64_t(slot) * SE + (b * g.HWo + int64_t(ho) * g.Wo) * g.Cin, uint32_t(pl.rrow_b),
                        &full[s]);
        }
      }
      if (++s == pl.nst) { s = 0; ph ^= 1u; refill = true; }
      if (++ho == g.Ho) { ho = 0; ++b; }
    }
    return;
  }
  // ---- consumers: thread = (output pixel wo, channel vector) of the unit's row
  const int CV = g.Cin / V;
  const bool active = tid < g.Wo * CV;
  const int wo = tid / CV, c0 = (tid - wo * CV) * V;
  const int w0 = wo * g.sw - g.pw;
  int s = 0;
  uint32_t ph = 0;
  int64_t b = lo / g.Ho;
  int ho = int(lo - b * g.Ho);
  for (int64_t u = lo; u < hi; ++u) {
    ptx::mbar_wait(&full[s], ph);
    if (active) {
      const uint8_t* st = seg_smem + size_t(s) * pl.stage_bytes;
      const Tin* xs = reinterpret_cast<const Tin*>(st);
      float sv[V];
#pragma unroll
      for (int j = 0; j < V; ++j) sv[j] = MAX ? -INFINITY : 0.f;
      if (x && KHW > 0) {
        const int hi0 = ho * g.sh - g.ph;
        const Tin* xb = xs + w0 * g.Cin + c0;
#pragma unroll
        for (int uu = 0; uu < CKH; ++uu) {
          if (hi0 + uu < 0 || hi0 + uu >= g.H) continue;
#pragma unroll
          for (int v = 0; v < CKW; ++v) {
            if (w0 + v < 0 || w0 + v >= g.W) continue;
            const Vec<Tin, V> xv = *reinterpret_cast<const Vec<Tin, V>*>(xb + (uu * g.W + v) * g.Cin);
#pragma unroll
            for (int j = 0; j < V; ++j) sv[j] = MAX ? fmaxf(sv[j], to_f(xv.v[j])) : sv[j] + to_f(xv.v[j]);
          }
        }
      } else if (x) {
        const int hi0 = ho * g.sh - g.ph;
        for (int uu = 0; uu < g.kh; ++uu) {
          const int hr = hi0 + uu * g.dh;
          if (hr < 0 || hr >= g.H) continue;
          for (int v = 0; v < g.kw; ++v) {
            const int wi = w0 + v * g.dw;
            if (wi < 0 || wi >= g.W) continue;
            const Vec<Tin, V> xv = *reinterpret_cast<const Vec<Tin, V>*>(xs + ((uu * g.dh) * g.W + wi) * g.Cin + c0);
#pragma unroll
            for (int j = 0; j < V; ++j) sv[j] = MAX ? fmaxf(sv[j], to_f(xv.v[j])) : sv[j] + to_f(xv.v[j]);
          }
        }
      }
      const int64_t r = b * g.HWo + int64_t(ho) * g.Wo + wo;
      if (a.slot[0] >= 0) {
        Vec<Tr, V> w;
#pragma unroll
        for (int j = 0; j < V; ++j) w.v[j] = from_f<Tr>(sv[j]);
        *reinterpret_cast<Vec<Tr, V>*>(ring + int64_t(a.slot[0]) * SE + r * g.Cin + c0) = w;
      }
      if (a.emit) {
        float win[V];
#pragma unroll
        for (int j = 0; j < V; ++j) win[j] = MAX ? -INFINITY : 0.f;
        const Tr* rs = reinterpret_cast<const Tr*>(st + pl.r_off) + wo * g.Cin + c0;
        for (int k = 0; k + 1 < g.kt; ++k) {
          const Vec<Tr, V> q = *reinterpret_cast<const Vec<Tr, V>*>(reinterpret_cast<const uint8_t*>(rs) + k * pl.rrow_b);
#pragma unroll
          for (int j = 0; j < V; ++j) win[j] = MAX ? fmaxf(win[j], to_f(q.v[j])) : win[j] + to_f(q.v[j]);
        }
        combine<V, MAX>(win, sv);
        store_out<Tout, V, MAX>(g, reinterpret_cast<Tout*>(a.y) + b * a.y_bstride + (r - b * g.HWo) * g.Cout + c0, win);
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_relaxed(&empty[s]);   // the stage's reads are consumed
    if (++s == pl.nst) { s = 0; ph ^= 1u; }
    if (++ho == g.Ho) { ho = 0; ++b; }
  }
}

// Plan of the row pipeline; false: the shape keeps the band / plain kernels.
bool pool_seg_plan(const Geom& g, int V, PoolSegPlan& pl) {
  if (option(OPT_POOL_SEG) == 0 || g.pool_vh || g.pool_G > 1 || g.kh * g.kw < 2 || g.in_dtype != BF16) return false;
  const int esz = 2, resz = pool_ring_esz(g);
  const int CV = g.Cin / V;
  const int items = g.Wo * CV;
  if (items > 992 || g.Cin % V) return false;
  pl.cwarps = (items + 31) / 32;
  pl.x_rows = (g.kh - 1) * g.dh + 1;
  pl.xrow_b = g.W * g.Cin * esz;
  pl.rrow_b = g.Wo * g.Cin * resz;
  if (pl.xrow_b % 16 || pl.rrow_b % 16) return false;
  pl.r_off = (pl.x_rows * pl.xrow_b + 127) / 128 * 128;
  pl.stage_bytes = (pl.r_off + (g.kt - 1) * pl.rrow_b + 127) / 128 * 128;
  // two blocks per SM with 3-4 stages each when they fit, else one block with up to 6
  const int threads = pl.cwarps * 32 + 32;
  if (4 * pl.stage_bytes <= 100 * 1024 && threads <= 512) { pl.nst = 4; pl.per_sm = 2; }
  else if (3 * pl.stage_bytes <= 100 * 1024 && threads <= 512) { pl.nst = 3; pl.per_sm = 2; }
  else {
    pl.nst = std::min(6, int((200 * 1024) / pl.stage_bytes));
    pl.per_sm = 1;
    if (pl.nst < 3) return false;
  }
  return true;
}

template <typename Tin, typename Tout, typename Tr, int V, bool MAX, int KHW = 0>
cudaError_t step_seg(const Geom& g, const StepArgs& a, const PoolSegPlan& pl, cudaStream_t s) {
  const size_t smem = size_t(pl.nst) * pl.stage_bytes + 2 * size_t(pl.nst) * sizeof(uint64_t);
  static size_t set_smem = 0;                      // (per instantiation)
  if (smem > set_smem) {
    cudaError_t e = cudaFuncSetAttribute(k_step_pool_seg<Tin, Tout, Tr, V, MAX, KHW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    set_smem = smem;
  }
  const int64_t units = g.B * g.Ho;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(std::max<int64_t>(1, std::min<int64_t>(units, int64_t(num_sms()) * pl.per_sm))));
  cfg.blockDim = dim3(unsigned(pl.cwarps * 32 + 32));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pool_pdl() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_step_pool_seg<Tin, Tout, Tr, V, MAX, KHW>, g, a, pl);
}

template <typename Tin, typename Tout, typename Tr, int V, bool MAX>
cudaError_t step_v(const Geom& g, const StepArgs& a, cudaStream_t s) {
  if (g.pool_G > 1)
    return g.pool_vh ? step_split<Tin, Tout, Tr, V, MAX, true>(g, a, g.pool_G, s)
                     : step_split<Tin, Tout, Tr, V, MAX, false>(g, a, g.pool_G, s);
  if constexpr (std::is_same<Tin, __nv_bfloat16>::value) {
    PoolSegPlan spl;
    if (pool_seg_plan(g, V, spl) && (!a.x || (reinterpret_cast<uintptr_t>(a.x) % 16 == 0 && (a.x_bstride * 2) % 16 == 0)))
      return (g.kh == 3 && g.kw == 3 && g.dh == 1 && g.dw == 1) ? step_seg<Tin, Tout, Tr, V, MAX, 33>(g, a, spl, s)
                                                                 : step_seg<Tin, Tout, Tr, V, MAX>(g, a, spl, s);
  }
  const int64_t total = g.B * g.HWo * (g.Cin / V);
  const int grid = grid_for(total);
  const int khw = (g.dh == 1 && g.dw == 1 && g.kh <= 3 && g.kw <= 3 && g.kh == g.kw) ? g.kh * 10 + g.kw : 0;
  int rows = 0;
  size_t smem = 0;
  const int TH = pool_band_enabled() ? band_rows(g, V, rows, smem) : 0;
  if (TH > 0) {   // spatial window: stage the band's input rows once (k_step_pool_band)
    const int threads = std::min(1024, (TH * g.Wo * (g.Cin / V) + 31) / 32 * 32);
    const int64_t nb = g.B * ((g.Ho + TH - 1) / TH);
    const void* fn = g.pool_vh ? (const void*)k_step_pool_band<Tin, Tout, Tr, V, MAX, true>
                     : khw == 33 ? (const void*)k_step_pool_band<Tin, Tout, Tr, V, MAX, false, 33>
                                 : (const void*)k_step_pool_band<Tin, Tout, Tr, V, MAX, false>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    const int bgrid = int(std::min<int64_t>(nb, int64_t(num_sms()) * std::max(per_sm, 1)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(bgrid));
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pool_pdl() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (g.pool_vh) return cudaLaunchKernelEx(&cfg, k_step_pool_band<Tin, Tout, Tr, V, MAX, true>, g, a, TH, rows);
    if (khw == 33) return cudaLaunchKernelEx(&cfg, k_step_pool_band<Tin, Tout, Tr, V, MAX, false, 33>, g, a, TH, rows);
    return cudaLaunchKernelEx(&cfg, k_step_pool_band<Tin, Tout, Tr, V, MAX, false>, g, a, TH, rows);
  }
  if (g.pool_vh) k_step_pool<Tin, Tout, Tr, V, MAX, kChunk, true><<<grid, 256, 0, s>>>(g, a);
  else if (khw == 33) k_step_pool<Tin, Tout, Tr, V, MAX, 1, false, 33><<<grid, 256, 0, s>>>(g, a);
  else if (khw == 22) k_step_pool<Tin, Tout, Tr, V, MAX, 1, false, 22><<<grid, 256, 0, s>>>(g, a);
  else if (khw == 11) k_step_pool<Tin, Tout, Tr, V, MAX, 1, false, 11><<<grid, 256, 0, s>>>(g, a);
  else if (deep_chunks(g, total)) k_step_pool<Tin, Tout, Tr, V, MAX, kChunk, false><<<grid, 256, 0, s>>>(g, a);
  else k_step_pool<Tin, Tout, Tr, V, MAX, 1, false><<<grid, 256, 0, s>>>(g, a);
  return cudaGetLastError();
}

template <typename Tin, typename Tout, bool MAX>
cudaError_t step_t(const Geom& g, const StepArgs& a, cudaStream_t s) {
  using Tr = typename std::conditional<MAX, Tin, float>::type;
  switch (vec_width(g)) {
    case 8: return step_v<Tin, Tout, Tr, 8, MAX>(g, a, s);
    case 4: return step_v<Tin, Tout, Tr, 4, MAX>(g, a, s);
    case 2: return step_v<Tin, Tout, Tr, 2, MAX>(g, a, s);
    default: return step_v<Tin, Tout, Tr, 1, MAX>(g, a, s);
  }
}

template <typename Tr, bool MAX>
cudaError_t rebuild_t(const Geom& g, void* state, int64_t m_next, cudaStream_t s) {
  const int V = vec_width(g);
  const int grid = grid_for(g.B * g.HWo * (g.Cin / V));
  Tr* st = static_cast<Tr*>(state);
  switch (V) {
    case 8: k_pool_rebuild<Tr, 8, MAX><<<grid, 256, 0, s>>>(g, st, m_next); break;
    case 4: k_pool_rebuild<Tr, 4, MAX><<<grid, 256, 0, s>>>(g, st, m_next); break;
    case 2: k_pool_rebuild<Tr, 2, MAX><<<grid, 256, 0, s>>>(g, st, m_next); break;
    default: k_pool_rebuild<Tr, 1, MAX><<<grid, 256, 0, s>>>(g, st, m_next); break;
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
  if (deep_chunks(g, total)) {
    switch (V) {
      case 8: k_forward_pool<Tin, Tout, 8, MAX, kChunk><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      case 4: k_forward_pool<Tin, Tout, 4, MAX, kChunk><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      case 2: k_forward_pool<Tin, Tout, 2, MAX, kChunk><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      default: k_forward_pool<Tin, Tout, 1, MAX, kChunk><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
    }
  } else {
    switch (V) {
      case 8: k_forward_pool<Tin, Tout, 8, MAX, 1><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      case 4: k_forward_pool<Tin, Tout, 4, MAX, 1><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      case 2: k_forward_pool<Tin, Tout, 2, MAX, 1><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
      default: k_forward_pool<Tin, Tout, 1, MAX, 1><<<grid, 256, 0, s>>>(g, xp, T, yp, Tp); break;
    }
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

cudaError_t launch_step_pool(const Geom& g, const StepArgs& a0, cudaStream_t s) {
  StepArgs a = a0;
  const int64_t i = a.m / g.dt;
  a.pm_f = int(((a.m % g.f) + g.f) % g.f);
  a.pm_q = int(a.m % g.dt);
  a.pm_pos = int(i % g.kt);
  a.pm_js = int((((i - g.kt + 1) % g.kt) + g.kt) % g.kt);
  return g.op == OP_MAX_POOL ? step_dispatch<true>(g, a, s) : step_dispatch<false>(g, a, s);
}

cudaError_t launch_forward_pool(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp, cudaStream_t s) {
  if (g.B * Tp * g.HWo == 0) return cudaSuccess;
  return g.op == OP_MAX_POOL ? forward_dispatch<true>(g, x, T, y, Tp, s) : forward_dispatch<false>(g, x, T, y, Tp, s);
}

cudaError_t launch_pool_rebuild(const Geom& g, void* state, int64_t m_next, cudaStream_t s) {
  if (!g.pool_vh) return cudaSuccess;
  if (g.op == OP_AVG_POOL) return rebuild_t<float, false>(g, state, m_next, s);
  return g.in_dtype == BF16 ? rebuild_t<__nv_bfloat16, true>(g, state, m_next, s)
                            : rebuild_t<float, true>(g, state, m_next, s);
}

bool pool_band_enabled() { return option(OPT_POOL_BAND) != 0; }   // option "pool_band" (default on)

int pool_block_decomposition(const Geom& g) {
  const int64_t v = option(OPT_POOL_VH);             // option "pool_vh": -1 auto, 0 / 1 pinned
  if (v >= 0) return int(v);
  return g.kt >= kVhMinKt ? 1 : 0;
}

cudaError_t launch_fill_pad(const Geom& g, void* p, int64_t n_elems, cudaStream_t s) {
  if (n_elems <= 0) return cudaSuccess;
  if (g.op != OP_MAX_POOL) return cudaMemsetAsync(p, 0, size_t(n_elems) * pool_ring_esz(g), s);
  const int grid = grid_for(n_elems);
  if (g.in_dtype == BF16) k_fill<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(p), n_elems, g.op);
  else k_fill<float><<<grid, 256, 0, s>>>(static_cast<float*>(p), n_elems, g.op);
  return cudaGetLastError();
}

int pool_split_lanes(const Geom& g) {
  if (const int e = int(option(OPT_POOL_G))) {   // option "pool_g": pinned lanes per vector
    const int CV = g.Cin / vec_width(g);
    int G = e;
    G = G < 1 ? 1 : (G > 32 ? 32 : G);
    while (G > 1 && G * CV > 512) --G;
    return G;
  }
  return split_lanes(g);
}

std::string pool_kernel_name(const Geom& g) {
  char out[64];
  const int G = g.pool_G;
  const char* kind = g.op == OP_MAX_POOL ? "max" : "avg";
  const char* vh = g.pool_vh ? ",vh" : "";
  int rows;
  size_t smem;
  PoolSegPlan spl;
  if (G > 1) snprintf(out, 64, "k_step_pool_split<%s,V%d,G%d%s>", kind, vec_width(g), G, vh);
  else if (pool_seg_plan(g, vec_width(g), spl)) snprintf(out, 64, "k_step_pool_seg<%s,V%d>", kind, vec_width(g));
  else if (pool_band_enabled() && band_rows(g, vec_width(g), rows, smem) > 0)
    snprintf(out, 64, "k_step_pool_band<%s,V%d%s>", kind, vec_width(g), vh);
  else snprintf(out, 64, "k_step_pool<%s,V%d%s>", kind, vec_width(g), vh);
  return out;
}

}  // namespace co
