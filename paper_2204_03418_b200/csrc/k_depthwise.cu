// k_depthwise.cu — K2 / K3: depthwise (groups == Cin == Cout) continual-
// convolution step kernels on CUDA cores (BASELINE.json north_star
// "Depthwise/grouped step kernel: runs on CUDA cores with vectorised 128-bit
// coalesced loads, shared-memory staging of the spatial halo").
//
// A depthwise layer has (kt kh kw) MACs per output element (C3-a: 27, C3-b: 5)
// against 2 (kt-1) fp32 state accesses, so it is HBM-bound by two orders of
// magnitude (AI 2.7 and 0.3 FLOP/B); tensor cores have nothing to
// contract.  Both kernels therefore aim at streaming the fp32 state ring at HBM
// bandwidth:
//  * state layout channels-last, S[slot][B*Ho*Wo][C] (common.cuh state_cl = 1):
//    a thread owns one (output pixel, channel quad); consecutive threads take
//    consecutive quads of the same pixel, so every state / frame / output
//    access of a warp is one contiguous run (512 B of state per float4 access);
//  * each thread first issues the state loads of a batch of NB items (emit slot
//    + the kt-2 accumulating slots), then computes, so NB x (kt-1) x 16 B per
//    thread are in flight;
//  * K2 (spatial kh x kw stencil): persistent CTAs keep the packed fp32 weights
//    [kt][kh][kw][C] in shared memory; per tile (stream, band of TH output
//    rows) the input halo (TH+kh-1) x (W+2pw) x C is staged in shared memory by
//    cp.async (16 B, zero-fill = spatial padding), then each strip issues its
//    state loads before its taps; the 3x3 taps are read from shared memory
//    (8 B per tap per thread, conflict-free: consecutive threads, consecutive
//    8-byte words);
//  * K3 (temporal-only, 1x1 spatial): a pure streaming kernel, no halo.
//
// Per item (BASELINE.json north_star):
//   y = S[slot_{kt-1}] + P_{kt-1} + b  (emitted when ready, activation, RNE)
//   S[slot_k] += P_k  for 0 < k < kt-1;   S[slot_0] = P_0 (after the emit read)
// with P_k = W[:, k] (*) x_t per channel.  The slots come from the host clock.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "depthwise.cuh"
#include "tc_ptx.cuh"

namespace co {

namespace {

constexpr int kDwThreads = 256;
#ifndef CO_DW_NB
#define CO_DW_NB 2
#endif
constexpr int kNB = CO_DW_NB;           // K3 items per thread per batch (state loads in flight)
#ifndef CO_DW_HALO_KB
#define CO_DW_HALO_KB 72                // K2 staged-halo bytes per CTA (experiments: -DCO_DW_HALO_KB=n)
#endif
constexpr size_t kHaloBudget = size_t(CO_DW_HALO_KB) * 1024;

struct DwParams {
  const __nv_bfloat16* x;               // frame of stream 0 (nullptr = zero frame)
  int64_t x_bstride;                    // elements between streams
  void* y;
  int64_t y_bstride;
  float* state;                         // S[slot][plane][C]
  const float* w;                       // [kt][kh][kw][C] fp32
  const float* bias;                    // [C]
  int slot[kMaxKt];
  int emit, update, act, out_f32;
  int C, Cq, H, W, Ho, Wo, ph, pw;
  int64_t HWo, plane;
  int TH, bands;                        // K2 tiling: TH output rows per tile
  int64_t n_tiles;
  int WC, HR;                           // halo width (W + 2 pw) and rows (TH + kh - 1)
  int64_t frame;                        // RAW layout: elements of one stream's frame (H*W*C)
  int raw_store;                        // RAW temporal kernel: ring slot this step's frame (read from x) is stored into
  // K2s segment pipeline (k_step_dw_seg): units = (stream, output row, segment of WS pixels)
  int64_t n_units;
  int nseg, WS, WX, nst, spu, gthreads; // WX = WS + kw - 1 staged input columns; spu strips per unit
  int ngroups;                          // consumer groups (alternate units)
  const void* zeros;                    // >= WX * C * 2 zero bytes: the bulk-copy source of padding columns
  int stage_bytes, x_off, stage_off, bar_off;   // shared-memory layout (bytes)
};

__device__ __forceinline__ float4 ld_bf16x4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  return make_float4(fa.x, fa.y, fb.x, fb.y);
}

__device__ __forceinline__ void st_out4(const DwParams& p, int64_t b, int64_t pin, int q, float4 v) {
  const int64_t off = b * p.y_bstride + pin * p.C + 4 * q;
  if (p.out_f32) {
    *reinterpret_cast<float4*>(static_cast<float*>(p.y) + off) = v;
  } else {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.y) + off) = u;
  }
}

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// Packed fp32 FMA (sm_100 FFMA2): two IEEE fmas (round to nearest) per
// instruction, so results equal fmaf lane by lane -- half the FMA issue slots
// of the stencil, which is issue-bound at ~60% busy with scalar FFMA.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const unsigned long long*>(&a)), "l"(*reinterpret_cast<const unsigned long long*>(&b)),
        "l"(*reinterpret_cast<const unsigned long long*>(&c)));
  return *reinterpret_cast<const float2*>(&d);
}
__device__ __forceinline__ float4 f4_fma(float4 w, float4 x, float4 acc) {
  const float2 lo = ffma2(make_float2(w.x, w.y), make_float2(x.x, x.y), make_float2(acc.x, acc.y));
  const float2 hi = ffma2(make_float2(w.z, w.w), make_float2(x.z, x.w), make_float2(acc.z, acc.w));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}
__device__ __forceinline__ float4 f4_act(float4 v, int act) {
  if (act == 1) {
    v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
  }
  return v;
}
__device__ __forceinline__ float4* srow(const DwParams& p, int slot, int64_t pix, int q) {
  return reinterpret_cast<float4*>(p.state + (int64_t(slot) * p.plane + pix) * p.C) + q;
}

// Prefetched state of one item: [0] = emit slot (k = kt-1), [k] = slot k (0 < k < kt-1).
template <int KT>
struct Pre {
  float4 s[KT > 1 ? KT - 1 : 1];
};

template <int KT>
__device__ __forceinline__ void prefetch(const DwParams& p, int64_t pix, int q, Pre<KT>& pr) {
  if (KT > 1) {
    if (p.emit) pr.s[0] = __ldcs(srow(p, p.slot[KT - 1], pix, q));
    if (p.update) {
#pragma unroll
      for (int k = 1; k < KT - 1; ++k)
        if (p.slot[k] >= 0) pr.s[k] = __ldcs(srow(p, p.slot[k], pix, q));
    }
  }
}

// Apply the step to one item given its per-slice partials P(k).
template <int KT, typename PF>
__device__ __forceinline__ void apply(const DwParams& p, int64_t b, int64_t pin, int64_t pix, int q,
                                      const Pre<KT>& pr, const float4 bias4, PF P) {
  if (p.emit) {
    float4 v = f4_add(P(KT - 1), bias4);
    if (KT > 1) v = f4_add(pr.s[0], v);
    st_out4(p, b, pin, q, f4_act(v, p.act));
  }
  if (KT > 1 && p.update) {
#pragma unroll
    for (int k = KT - 2; k >= 1; --k)
      if (p.slot[k] >= 0) __stcs(srow(p, p.slot[k], pix, q), f4_add(pr.s[k], P(k)));
    if (p.slot[0] >= 0) __stcs(srow(p, p.slot[0], pix, q), P(0));
  }
}

// ------------------------------------------------------------------ K2: spatial stencil
// Thread = (channel quad q, fixed for the thread's life) x strips of PX output
// pixels of one row.  Per strip: the state of its PX pixels is loaded first,
// then for each tap row u the PX+KW-1 input columns are read from the staged
// halo once and every (v, k) weight float4 once, so shared-memory traffic per
// pixel is (KT*KH*KW*16 + KH*(PX+KW-1)*8) / PX bytes -- PX times less than a
// thread-per-pixel stencil, which made the first K2 shared-memory bound.
// The per-slice FMA order (u-major, then v) is k_step_direct's, so the two
// kernels agree bitwise.
template <int KT, int KH, int KW, int PX>
#ifndef CO_DW_ST_MINB
#define CO_DW_ST_MINB 2
#endif
__global__ void __launch_bounds__(256, CO_DW_ST_MINB) k_step_dw_st(const DwParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  float* ws = reinterpret_cast<float*>(smem);                       // [KT][KH][KW][C]
  float* bs = ws + KT * KH * KW * p.C;                              // [C]
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(bs + p.C);   // [HR][WC][C]
  const int tid = threadIdx.x;
  const int nthr = blockDim.x;                                      // = Cq * n_srow
  for (int i = tid; i < KT * KH * KW * p.C; i += nthr) ws[i] = p.w[i];
  for (int i = tid; i < p.C; i += nthr) bs[i] = p.bias[i];
  const int q = tid % p.Cq;                                         // this thread's channel quad
  const int srow = tid / p.Cq;
  const int n_srow = nthr / p.Cq;
  const int spr = (p.Wo + PX - 1) / PX;                             // strips per output row
  const int c8 = p.C / 8;
  const int row_chunks = p.WC * c8;
  const uint32_t xs_u32 = static_cast<uint32_t>(__cvta_generic_to_shared(xs));
  const float4* ws4 = reinterpret_cast<const float4*>(ws) + q;     // + ((k*KH + u)*KW + v) * Cq
  const float4 bias4 = reinterpret_cast<const float4*>(bs)[q];
  (void)bias4;
  // programmatic dependent launch: weights staged above overlap the previous
  // kernel's drain; frames / state only after it completed
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int64_t b = tile / p.bands;
    const int ho0 = int(tile % p.bands) * p.TH;
    const int th = min(p.TH, p.Ho - ho0);
    __syncthreads();   // previous tile finished reading xs (and ws/bs are visible)
    // input halo -> shared memory (cp.async 16 B, zero fill outside the frame)
    const __nv_bfloat16* xb = p.x ? p.x + b * p.x_bstride : nullptr;
    for (int r = 0; r < p.HR; ++r) {
      const int hi = ho0 - p.ph + r;
      const bool row_in = xb && hi >= 0 && hi < p.H;
      for (int i = tid; i < row_chunks; i += nthr) {
        const int c = i / c8, ch = i - (i / c8) * c8;
        const int wi = c - p.pw;
        const bool in = row_in && wi >= 0 && wi < p.W;
        // src-size 0 zero-fills; the (unread) address stays a valid one
        const void* src = in ? static_cast<const void*>(xb + (int64_t(hi) * p.W + wi) * p.C + ch * 8)
                             : static_cast<const void*>(p.w);
        const uint32_t dst = xs_u32 + uint32_t(r * row_chunks + i) * 16u;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0)
                     : "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    for (int sidx = srow; sidx < th * spr; sidx += n_srow) {
      const int r = sidx / spr;
      const int wo0 = (sidx - r * spr) * PX;
      const int64_t pin0 = int64_t(ho0 + r) * p.Wo + wo0;           // pixel index inside the stream
      const int64_t pix0 = b * p.HWo + pin0;
      // (1) the strip's state goes out first
      Pre<KT> pre[PX];
#pragma unroll
      for (int j = 0; j < PX; ++j)
        if (wo0 + j < p.Wo) prefetch<KT>(p, pix0 + j, q, pre[j]);
      // (2) all kt partials of the PX pixels, one pass over the taps
      float4 acc[KT][PX];
#pragma unroll
      for (int k = 0; k < KT; ++k)
#pragma unroll
        for (int j = 0; j < PX; ++j) acc[k][j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < KH; ++u) {
        float4 xv[PX + KW - 1];
        const __nv_bfloat16* xr = xs + (int64_t(r + u) * p.WC + wo0) * p.C + 4 * q;
#pragma unroll
        for (int t = 0; t < PX + KW - 1; ++t) xv[t] = ld_bf16x4(xr + int64_t(t) * p.C);
#pragma unroll
        for (int v = 0; v < KW; ++v)
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const float4 w = ws4[((k * KH + u) * KW + v) * p.Cq];
#pragma unroll
            for (int j = 0; j < PX; ++j) acc[k][j] = f4_fma(w, xv[j + v], acc[k][j]);
          }
      }
      // (3) emit / accumulate / start
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        if (wo0 + j >= p.Wo) continue;
        auto P = [&](int k) -> float4 { return acc[k][j]; };
        apply<KT>(p, b, pin0 + j, pix0 + j, q, pre[j], reinterpret_cast<const float4*>(bs)[q], P);
      }
    }
  }
}

// ------------------------------------------------------------------ K2s: segment pipeline
// The stencil with its memory traffic decoupled from the arithmetic.  K2's
// per-thread state loads are issued one strip ahead of their use and its halo
// is loaded and waited for per tile, so its bytes in flight per SM (~30 KB)
// sit below what HBM latency x bandwidth asks for (ncu: 0.69 of HBM, long-
// scoreboard and barrier stalls).  Here one producer thread streams, per unit
// (stream b, output row ho, segment of WS output pixels), the unit's state rows
// (emit slot + accumulating slots: each one contiguous run of WS x C fp32 in
// the channels-last layout) and its kh input-row pieces (WS + kw - 1 columns,
// clipped to the frame) into a ring of `nst` shared-memory stages with bulk
// copies (cp.async.bulk, mbarrier complete_tx), so nst - 2 units of loads are
// in flight while the consumer groups compute alternate units: a thread =
// (channel quad q, strip of PX pixels), taps read unpredicated from the stage
// (padding columns / rows are bulk copies from a zero buffer), the thread's
// weights at immediate offsets ([Cq][taps] layout), the per-slice FMA order
// of K1 / K2 (bitwise equal), y and the written state slots stored straight
// from registers.  A CTA walks a contiguous unit range, so the input
// rows it re-reads for the next output row come from L2.
#ifndef CO_DW_SEG_THREADS
#define CO_DW_SEG_THREADS 384           // <= 12 warps (3 per SM sub-partition): up to 168 registers per thread
#endif
constexpr int kSegMaxThreads = CO_DW_SEG_THREADS;
constexpr int kSegGroupMax = (kSegMaxThreads - 32) / 2;   // >= 2 consumer groups

template <int KT, int KH, int KW, int PX>
__global__ void __launch_bounds__(kSegMaxThreads, 1) k_step_dw_seg(const DwParams p) {
  constexpr int NT = KT * KH * KW;                                  // taps per channel
  extern __shared__ __align__(128) uint8_t smem[];
  float4* wt = reinterpret_cast<float4*>(smem);                     // [Cq][NT] float4: a thread's taps at
  float* bs = reinterpret_cast<float*>(wt + NT * p.Cq);             // immediate offsets (NT odd: conflict-free)
  uint8_t* stages = smem + p.stage_off;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.nst;
  const int tid = threadIdx.x;
  for (int i = tid; i < NT * p.Cq; i += blockDim.x) {
    const int qq = i / NT, tap = i - qq * NT;
    wt[i] = *reinterpret_cast<const float4*>(p.w + int64_t(tap) * p.C + 4 * qq);
  }
  for (int i = tid; i < p.C; i += blockDim.x) bs[i] = p.bias[i];
  if (tid == 0) {
    for (int s = 0; s < p.nst; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], p.gthreads / 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: wait for the previous grid, but never trigger
  // early -- dependents launch as these CTAs exit.  An early trigger lets a
  // grid-stride successor (K3 in the C3 chain, several CTAs per SM) place its
  // CTAs on whichever SMs this persistent grid frees first, unevenly: C3 tick
  // 0.72 -> 0.62 M stream-steps/s measured with the trigger at entry.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t lo = p.n_units * blockIdx.x / gridDim.x;
  const int64_t hi = p.n_units * (blockIdx.x + 1) / gridDim.x;
  const int64_t rows_u = int64_t(p.Ho) * p.nseg;                   // units per stream
  const int warp = tid / 32, lane = tid % 32;
  const int64_t row_e = int64_t(p.WS) * p.C;                       // state elements per staged slot row
  const int xrow_b = p.WX * p.C * 2;                                // bytes of one staged input row
  if (warp == p.ngroups * p.gthreads / 32) {                        // ---- producer thread
    if (lane != 0) return;
    int64_t b = lo / rows_u;                                        // unit lo's (stream, row, segment),
    int ho = int(lo - b * rows_u) / p.nseg;                         // then stepped incrementally
    int sg = int(lo - b * rows_u) - ho * p.nseg;
    const uint8_t* zsrc = static_cast<const uint8_t*>(p.zeros);
    for (int64_t j = lo; j < hi; ++j) {
      const int64_t i = j - lo;
      const int s = int(i % p.nst);
      if (i >= p.nst) ptx::mbar_wait(&empty[s], (uint32_t(i / p.nst) & 1u) ^ 1u);
      const int wo0 = sg * p.WS;
      const int wsz = min(p.WS, p.Wo - wo0);
      uint8_t* st = stages + int64_t(s) * p.stage_bytes;
      const int64_t pix0 = b * p.HWo + int64_t(ho) * p.Wo + wo0;
      const uint32_t sbytes = uint32_t(wsz) * p.C * 4;
      // staged column c holds input column wlo + c (c < ncol are read for real
      // pixels); [a, e] is the part inside the frame, the rest is padding: zero
      // bytes bulk-copied like the data, so the consumers read every tap
      // unpredicated and no generic-proxy write ever touches a stage
      const int wlo = wo0 - p.pw, ncol = wsz + KW - 1;
      const int a = max(wlo, 0), e = min(wlo + ncol - 1, p.W - 1);
      const uint32_t pxb = uint32_t(p.C) * 2;
      uint32_t tx = 0;
      if (KT > 1 && p.emit) tx += sbytes;
      if (KT > 2 && p.update)
        for (int k = 1; k < KT - 1; ++k) tx += (p.slot[k] >= 0) ? sbytes : 0u;
      tx += uint32_t(KH * ncol) * pxb;                              // every staged column: data or zeros
      ptx::mbar_arrive_expect_tx(&full[s], tx);
      if (KT > 1 && p.emit)
        ptx::bulk_g2s(st, p.state + (int64_t(p.slot[KT - 1]) * p.plane + pix0) * p.C, sbytes, &full[s]);
      if (KT > 2 && p.update)
        for (int k = 1; k < KT - 1; ++k)
          if (p.slot[k] >= 0)
            ptx::bulk_g2s(st + int64_t(k) * row_e * 4, p.state + (int64_t(p.slot[k]) * p.plane + pix0) * p.C,
                          sbytes, &full[s]);
      for (int u = 0; u < KH; ++u) {
        const int hr = ho - p.ph + u;
        uint8_t* row = st + p.x_off + u * xrow_b;
        if (!p.x || hr < 0 || hr >= p.H || a > e) {
          ptx::bulk_g2s(row, zsrc, uint32_t(ncol) * pxb, &full[s]);
          continue;
        }
        if (a > wlo) ptx::bulk_g2s(row, zsrc, uint32_t(a - wlo) * pxb, &full[s]);
        ptx::bulk_g2s(row + (a - wlo) * pxb, p.x + b * p.x_bstride + (int64_t(hr) * p.W + a) * p.C,
                      uint32_t(e - a + 1) * pxb, &full[s]);
        if (e - wlo + 1 < ncol)
          ptx::bulk_g2s(row + (e - wlo + 1) * pxb, zsrc, uint32_t(ncol - (e - wlo + 1)) * pxb, &full[s]);
      }
      if (++sg == p.nseg) {
        sg = 0;
        if (++ho == p.Ho) { ho = 0; ++b; }
      }
    }
    return;
  }
  // ---- consumers: group g takes units lo + g, lo + g + ngroups, ...  A parity
  // wait must never run more than one phase ahead of its barrier: after unit i
  // a group waits on unit i + ngroups, whose stage was last filled by unit
  // i + ngroups - nst -- another group's (nst is not a multiple of ngroups),
  // issued before unit i, but bulk copies complete in any order.  Had that fill
  // not landed, the wait on full[] would pass on the phase before (seen at the
  // full C3-a size as one corrupted unit in ~10^5).  So a consumer first waits
  // for the stage's previous fill to have been *consumed* (the phase of empty[]
  // the producer itself waits on before refilling: at most one behind, and its
  // completion implies that fill landed), then for its own fill.  (Measured
  // alternatives, both correct: every warp waiting on and releasing every stage
  // in order, 0.272 ms on C3-a; the producer holding unit i back until unit
  // i - 2 has landed, 0.284 ms.)
  const int g = tid / p.gthreads, tg = tid - g * p.gthreads;
  const bool active = tg < p.Cq * p.spu;
  const int q = tg % p.Cq, sp = tg / p.Cq;                          // channel quad, strip of the unit
  const int cstep = p.C;                                            // elements between pixels (x, y, state)
  for (int64_t j = lo + g; j < hi; j += p.ngroups) {
    const int64_t i = j - lo;
    const int s_cur = int(i % p.nst);
    const uint32_t fill = uint32_t(i / p.nst);
    if (fill > 0) ptx::mbar_wait(&empty[s_cur], (fill & 1u) ^ 1u);
    ptx::mbar_wait(&full[s_cur], fill & 1u);
    const uint32_t ju = uint32_t(j);                                // n_units < 2^31 (plan)
    const int64_t b = ju / uint32_t(rows_u);
    const int r = int(ju - uint32_t(b) * uint32_t(rows_u));
    const int ho = r / p.nseg, wo0 = (r - ho * p.nseg) * p.WS;
    const int wsz = min(p.WS, p.Wo - wo0);
    const int c0 = sp * PX;                                         // first staged column / pixel of the strip
    const int nv = wsz - c0;                                        // real pixels of the strip (compared with
    if (active && nv > 0) {                                         // the unrolled index: no per-pixel constants)
      const uint8_t* st = stages + int64_t(s_cur) * p.stage_bytes;
      float4 acc[KT][PX];
#pragma unroll
      for (int k = 0; k < KT; ++k)
#pragma unroll
        for (int jj = 0; jj < PX; ++jj) acc[k][jj] = make_float4(0.f, 0.f, 0.f, 0.f);
      const __nv_bfloat16* xr = reinterpret_cast<const __nv_bfloat16*>(st + p.x_off) + int64_t(c0) * cstep + 4 * q;
      const float4* wq = wt + q * NT;
#pragma unroll 1                                                    // rolled: fewer live registers (no spills)
      for (int u = 0; u < KH; ++u, wq += KW) {
        float4 xv[PX + KW - 1];
#pragma unroll
        for (int t = 0; t < PX + KW - 1; ++t) xv[t] = ld_bf16x4(xr + t * cstep);
        xr += p.WX * cstep;
#pragma unroll
        for (int v = 0; v < KW; ++v)
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const float4 w = wq[k * KH * KW + v];
#pragma unroll
            for (int jj = 0; jj < PX; ++jj) acc[k][jj] = f4_fma(w, xv[jj + v], acc[k][jj]);
          }
      }
      // emit / accumulate / start (apply()'s arithmetic); the read slots come
      // from the stage only now, so no registers hold them across the taps
      const float4* ss4 = reinterpret_cast<const float4*>(st) + int64_t(c0) * p.Cq + q;   // [KT-1][WS][Cq]
      const float4 bias4 = reinterpret_cast<const float4*>(bs)[q];  // re-read per unit: 4 registers fewer
      const int64_t pin0 = int64_t(ho) * p.Wo + wo0 + c0;
      const int64_t yoff = b * p.y_bstride + pin0 * cstep + 4 * q;
      float* sp_k[KT > 1 ? KT - 1 : 1];                             // written slot rows of pixel 0 of the strip
#pragma unroll
      for (int k = 0; k < KT - 1; ++k)
        sp_k[k] = p.state + (int64_t(p.slot[k]) * p.plane + b * p.HWo + pin0) * cstep + 4 * q;
#pragma unroll
      for (int jj = 0; jj < PX; ++jj) {
        if (jj >= nv) continue;
        if (p.emit) {
          float4 v = f4_add(acc[KT - 1][jj], bias4);
          if (KT > 1) v = f4_add(ss4[jj * p.Cq], v);
          v = f4_act(v, p.act);
          if (p.out_f32) {
            *reinterpret_cast<float4*>(static_cast<float*>(p.y) + yoff + jj * cstep) = v;
          } else {
            __nv_bfloat162 lo2 = __floats2bfloat162_rn(v.x, v.y), hi2 = __floats2bfloat162_rn(v.z, v.w);
            uint2 uu;
            uu.x = *reinterpret_cast<uint32_t*>(&lo2);
            uu.y = *reinterpret_cast<uint32_t*>(&hi2);
            *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.y) + yoff + jj * cstep) = uu;
          }
        }
        if (KT > 1 && p.update) {
#pragma unroll
          for (int k = KT - 2; k >= 1; --k)
            if (p.slot[k] >= 0)
              __stcs(reinterpret_cast<float4*>(sp_k[k] + jj * cstep),
                     f4_add(ss4[(k * p.WS + jj) * p.Cq], acc[k][jj]));
          if (p.slot[0] >= 0) __stcs(reinterpret_cast<float4*>(sp_k[0] + jj * cstep), acc[0][jj]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_relaxed(&empty[s_cur]);   // the stage's reads are consumed (see dense epilogue)
  }
}

// ------------------------------------------------------------------ K3: temporal only
#ifndef CO_DW_T_MINB
#define CO_DW_T_MINB 3                  // K3 measured best at 2 items x 3 CTAs per SM; experiments: resident CTAs per SM the registers must allow
#endif
template <int KT>
__global__ void __launch_bounds__(kDwThreads, CO_DW_T_MINB) k_step_dw_t(const DwParams p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");   // see k_step_dw_st
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t n_items = p.plane * p.Cq;
  const int64_t stride = int64_t(gridDim.x) * kDwThreads;
  for (int64_t base = int64_t(blockIdx.x) * kDwThreads + threadIdx.x; base < n_items; base += kNB * stride) {
    Pre<KT> pre[kNB];
    float4 xv[kNB];
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      const int64_t it = base + j * stride;
      if (it < n_items) {
        const int q = int(it % p.Cq);
        const int64_t pix = it / p.Cq;
        prefetch<KT>(p, pix, q, pre[j]);
        const int64_t b = pix / p.HWo;
        xv[j] = p.x ? ld_bf16x4(p.x + b * p.x_bstride + (pix - b * p.HWo) * p.C + 4 * q)
                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      const int64_t it = base + j * stride;
      if (it >= n_items) continue;
      const int q = int(it % p.Cq);
      const int64_t pix = it / p.Cq;
      const int64_t b = pix / p.HWo;
      auto P = [&](int k) -> float4 {
        return f4_fma(__ldg(reinterpret_cast<const float4*>(p.w + k * p.C) + q), xv[j], make_float4(0.f, 0.f, 0.f, 0.f));
      };
      apply<KT>(p, b, pix - b * p.HWo, pix, q, pre[j], __ldg(reinterpret_cast<const float4*>(p.bias) + q), P);
    }
  }
}

// ------------------------------------------------------------------ K3c: chunked steps
// SURVEY §8f f2 "chunked co_forward_steps that keeps state tiles on-chip across
// T frames": a thread owns one (pixel, channel quad) for a whole clip and keeps
// its kt-1 pending outputs in registers as a shift register, Q[j] = the output
// completing j ticks ahead; per frame
//   y = Q[0] + (P_{kt-1} + b),  Q[j-1] = Q[j] + P_{kt-1-j} (j = 1..kt-2),  Q[kt-2] = P_0
// -- k_step_dw_t's operations in its order, so chunked and per-step folds agree
// bitwise -- and the fp32 ring is read once before the clip and written once
// after it (outputs i < 0, never emitted, are neither read nor written, as in
// the per-step kernel).  HBM per stream-step: x + y (+ 2 (kt-1) state / T):
// the state round trip that dominates the per-step kernel
// leaves the hot loop.  Temporal stride 1, dilation 1 (R = kt - 1).
struct ChunkArgs {
  const __nv_bfloat16* x;               // clip of stream 0, (T, H*W*C); stream stride x_bstride
  int64_t x_bstride, T, total;          // frames present, ticks to run (T + pad_end padding)
  int64_t m0;                           // padded index n0 + p of the first tick
  int64_t oi0;                          // output index of tick t: n0 + t - oi0 (when Ready)
  int64_t y_bstride;
  int d;                                // delay: tick t is Ready when n0 + t >= d
  int64_t n0;
};

template <int KT>
__global__ void __launch_bounds__(kDwThreads, 2) k_steps_dw_t(const DwParams p, const ChunkArgs c) {
  constexpr int NQ = KT > 1 ? KT - 1 : 1;
  const int64_t n_items = p.plane * p.Cq;
  const int R = KT - 1;
  for (int64_t it = int64_t(blockIdx.x) * kDwThreads + threadIdx.x; it < n_items;
       it += int64_t(gridDim.x) * kDwThreads) {
    const int q = int(it % p.Cq);
    const int64_t pix = it / p.Cq;
    const int64_t b = pix / p.HWo;
    const int64_t pin = pix - b * p.HWo;
    float4 w[KT];
#pragma unroll
    for (int k = 0; k < KT; ++k) w[k] = __ldg(reinterpret_cast<const float4*>(p.w + k * p.C) + q);
    const float4 bias4 = __ldg(reinterpret_cast<const float4*>(p.bias) + q);
    float4 Q[NQ];
    const int64_t i0 = c.m0 - (KT - 1);            // output completing at the first tick
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      Q[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (KT > 1 && i0 + j >= 0) Q[j] = __ldcs(srow(p, int((i0 + j) % R), pix, q));
    }
    const __nv_bfloat16* xs = c.x + b * c.x_bstride + pin * p.C + 4 * q;
    const int64_t fstride = int64_t(p.HWo) * p.C;
    constexpr int U = 4;                           // frames in flight per thread
    for (int64_t t0 = 0; t0 < c.total; t0 += U) {
      float4 xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        xv[u] = (t0 + u < c.T) ? ld_bf16x4(xs + (t0 + u) * fstride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t t = t0 + u;
        if (t >= c.total) break;
        auto P = [&](int k) { return f4_fma(w[k], xv[u], make_float4(0.f, 0.f, 0.f, 0.f)); };
        if (c.n0 + t >= c.d) {
          float4 v = f4_add(P(KT - 1), bias4);
          if (KT > 1) v = f4_add(Q[0], v);
          st_out4(p, b, (c.n0 + t - c.oi0) * p.HWo + pin, q, f4_act(v, p.act));
        }
        if (KT > 1) {
#pragma unroll
          for (int j = 1; j < KT - 1; ++j) Q[j - 1] = f4_add(Q[j], P(KT - 1 - j));
          Q[NQ - 1] = P(0);
        }
      }
    }
    const int64_t i1 = c.m0 + c.total - (KT - 1);  // output completing at the next tick
#pragma unroll
    for (int j = 0; j < NQ; ++j)
      if (KT > 1 && i1 + j >= 0) __stcs(srow(p, int((i1 + j) % R), pix, q), Q[j]);
  }
}

// ------------------------------------------------------------------ K2c: chunked spatial steps
// The K2 stencil folded over a clip: a CTA owns one tile
// (stream b, TH output rows) for all T frames; thread = (channel quad q, strip
// of PX output pixels), fixed for the clip, with its strip's kt-1 pending
// outputs in registers (Q[j][px], the K3c shift register).  Per frame the
// tile's input halo is staged by cp.async into one of two buffers (frame t+1
// lands while frame t is folded); the taps are folded in K2's order (u, v, k),
// so the result equals the per-step kernel bit for bit.  The fp32 ring is read
// before and written after the clip only.
template <int KT, int KH, int KW, int PX>
__global__ void __launch_bounds__(1024, 1) k_steps_dw_st(const DwParams p, const ChunkArgs c) {
  constexpr int NQ = KT > 1 ? KT - 1 : 1;
  extern __shared__ __align__(16) uint8_t smem[];
  float* ws = reinterpret_cast<float*>(smem);                       // [KT][KH][KW][C]
  float* bs = ws + KT * KH * KW * p.C;                              // [C]
  __nv_bfloat16* xs0 = reinterpret_cast<__nv_bfloat16*>(bs + p.C);  // 2 x [HR][WC][C]
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int i = tid; i < KT * KH * KW * p.C; i += nthr) ws[i] = p.w[i];
  for (int i = tid; i < p.C; i += nthr) bs[i] = p.bias[i];
  const int q = tid % p.Cq;
  const int sidx = tid / p.Cq;                                      // this thread's strip in the tile
  const int spr = (p.Wo + PX - 1) / PX;
  const int c8 = p.C / 8;
  const int row_chunks = p.WC * c8;
  const size_t buf_elems = size_t(p.HR) * p.WC * p.C;
  const float4* ws4 = reinterpret_cast<const float4*>(ws) + q;
  const int R = KT - 1;
  for (int64_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
    const int64_t b = tile / p.bands;
    const int ho0 = int(tile % p.bands) * p.TH;
    const int th = min(p.TH, p.Ho - ho0);
    const int r = sidx / spr;
    const int wo0 = (sidx - r * spr) * PX;
    const bool active = sidx < th * spr;
    const int64_t pin0 = int64_t(ho0 + r) * p.Wo + wo0;
    const int64_t pix0 = b * p.HWo + pin0;
    __syncthreads();   // the previous tile finished reading both halo buffers (and ws / bs are visible)
    auto stage = [&](int t, int buf) {   // frame t's halo -> buffer buf (zero fill outside the frame / clip)
      const __nv_bfloat16* xb = (t < c.T) ? c.x + b * c.x_bstride + int64_t(t) * p.H * p.W * p.C : nullptr;
      const uint32_t dst0 = static_cast<uint32_t>(__cvta_generic_to_shared(xs0 + buf * buf_elems));
      for (int rr = 0; rr < p.HR; ++rr) {
        const int hi = ho0 - p.ph + rr;
        const bool row_in = xb && hi >= 0 && hi < p.H;
        for (int i = tid; i < row_chunks; i += nthr) {
          const int cc = i / c8, ch = i - (i / c8) * c8;
          const int wi = cc - p.pw;
          const bool in = row_in && wi >= 0 && wi < p.W;
          const void* src = in ? static_cast<const void*>(xb + (int64_t(hi) * p.W + wi) * p.C + ch * 8)
                               : static_cast<const void*>(p.w);
          const uint32_t dst = dst0 + uint32_t(rr * row_chunks + i) * 16u;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(in ? 16 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // the strip's pending outputs: Q[j] = output i0 + j (i0 completes at the first tick)
    float4 Q[NQ][PX];
    const int64_t i0 = c.m0 - (KT - 1);
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
      for (int x = 0; x < PX; ++x) {
        Q[j][x] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (KT > 1 && active && wo0 + x < p.Wo && i0 + j >= 0)
          Q[j][x] = __ldcs(reinterpret_cast<const float4*>(p.state + ((int64_t((i0 + j) % R) * p.plane) + pix0 + x) * p.C) + q);
      }
    const float4 bias4 = reinterpret_cast<const float4*>(bs)[q];
    stage(0, 0);
    for (int64_t t = 0; t < c.total; ++t) {
      const int buf = int(t & 1);
      if (t + 1 < c.total) {
        __syncthreads();                                  // buffer buf ^ 1 is no longer read (frame t-1)
        stage(int(t + 1), buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();                                    // frame t's halo visible to every thread
      if (!active) continue;
      const __nv_bfloat16* xs = xs0 + buf * buf_elems;
      float4 acc[KT][PX];
#pragma unroll
      for (int k = 0; k < KT; ++k)
#pragma unroll
        for (int x = 0; x < PX; ++x) acc[k][x] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < KH; ++u) {
        float4 xv[PX + KW - 1];
        const __nv_bfloat16* xr = xs + (int64_t(r + u) * p.WC + wo0) * p.C + 4 * q;
#pragma unroll
        for (int tt = 0; tt < PX + KW - 1; ++tt) xv[tt] = ld_bf16x4(xr + int64_t(tt) * p.C);
#pragma unroll
        for (int v = 0; v < KW; ++v)
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            const float4 w = ws4[((k * KH + u) * KW + v) * p.Cq];
#pragma unroll
            for (int x = 0; x < PX; ++x) acc[k][x] = f4_fma(w, xv[x + v], acc[k][x]);
          }
      }
      const bool emit = c.n0 + t >= c.d;
#pragma unroll
      for (int x = 0; x < PX; ++x) {
        if (wo0 + x >= p.Wo) continue;
        if (emit) {
          float4 v = f4_add(acc[KT - 1][x], bias4);
          if (KT > 1) v = f4_add(Q[0][x], v);
          st_out4(p, b, (c.n0 + t - c.oi0) * p.HWo + pin0 + x, q, f4_act(v, p.act));
        }
        if (KT > 1) {
#pragma unroll
          for (int j = 1; j < KT - 1; ++j) Q[j - 1][x] = f4_add(Q[j][x], acc[KT - 1 - j][x]);
          Q[NQ - 1][x] = acc[0][x];
        }
      }
    }
    const int64_t i1 = c.m0 + c.total - (KT - 1);
#pragma unroll
    for (int j = 0; j < NQ; ++j)
#pragma unroll
      for (int x = 0; x < PX; ++x)
        if (KT > 1 && active && wo0 + x < p.Wo && i1 + j >= 0)
          __stcs(reinterpret_cast<float4*>(p.state + ((int64_t((i1 + j) % R) * p.plane) + pix0 + x) * p.C) + q, Q[j][x]);
  }
}

// ------------------------------------------------------------------ RAW layout, spatial stencil: rolling rows
// A Ready step of a "same"-padded stride-1 stencil over the RAW frame ring
// with every input row of every window frame copied exactly once:
// a block owns a contiguous range of global output rows (stream b, row ho); a
// producer thread streams the global input rows that range touches, in order,
// as row sets -- row hr of each of the kt frames (the new frame from x, the older
// ones from the ring), kt bulk copies of W C bf16 -- into a ring of nst row-set
// stages whose kw - 1 side columns stay zero (the padding); all consumer warps
// walk the output rows together: wait (once, in order) for the row sets up to the
// window's last row, compute the kt kh kw taps of the row's pixels (thread =
// (channel quad, strip of PX pixels); rows outside the frame read a zero stage),
// write y, store the new frame's row into its ring slot, and release the row
// sets the next output row no longer needs.  (The per-unit pipeline of K2s needs
// kt kh row pieces per unit and is bound by the producer's issue rate: 0.73 ms.)
template <int KT, int KH, int KW, int PX>
__global__ void __launch_bounds__(kSegMaxThreads, 1) k_step_dw_rowraw(const DwParams p) {
  constexpr int NT = KT * KH * KW;
  extern __shared__ __align__(128) uint8_t smem[];
  float4* wt = reinterpret_cast<float4*>(smem);                     // [Cq][NT] float4
  float* bs = reinterpret_cast<float*>(wt + NT * p.Cq);
  uint8_t* stages = smem + p.stage_off;                             // [nst + 1][KT][WX][C] bf16 (the last: zeros)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* empty = full + p.nst;
  const int tid = threadIdx.x;
  for (int i = tid; i < NT * p.Cq; i += blockDim.x) {
    const int qq = i / NT, tap = i - qq * NT;
    wt[i] = *reinterpret_cast<const float4*>(p.w + int64_t(tap) * p.C + 4 * qq);
  }
  for (int i = tid; i < p.C; i += blockDim.x) bs[i] = p.bias[i];
  for (int i = tid; i < (p.nst + 1) * p.stage_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(stages)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (tid == 0) {
    for (int s = 0; s < p.nst; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], p.gthreads / 32);
    }
    ptx::fence_mbar_init();
  }
  ptx::fence_proxy_async();                                          // the zeroed stages before any bulk copy into them
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");                // (no early trigger: see k_step_dw_seg)
  const int64_t lo = p.n_units * blockIdx.x / gridDim.x;            // global output rows g = b H + ho
  const int64_t hi = p.n_units * (blockIdx.x + 1) / gridDim.x;
  if (lo >= hi) return;
  const int warp = tid / 32, lane = tid % 32;
  const int rowp_b = p.WX * p.C * 2;                                // bytes of one staged (padded) row
  const int64_t B = p.plane / p.HWo;
  const int64_t n_rows = B * p.H;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(p.state);
  // global input rows this range touches (windows never cross a stream: rows outside it are zeros)
  const int64_t g0 = max(lo - p.ph, (lo / p.H) * p.H);
  const int64_t g1 = min(min(hi - 1 - p.ph + KH, ((hi - 1) / p.H + 1) * p.H), n_rows);   // exclusive
  if (warp == p.gthreads / 32) {                                    // ---- producer thread
    if (lane != 0) return;
    const uint32_t rb = uint32_t(p.W) * p.C * 2;
    for (int64_t gi = g0; gi < g1; ++gi) {
      const int64_t i = gi - g0;
      const int s = int(i % p.nst);
      if (i >= p.nst) ptx::mbar_wait(&empty[s], (uint32_t(i / p.nst) & 1u) ^ 1u);
      const int64_t b = gi / p.H;
      const int hr = int(gi - b * p.H);
      uint8_t* st = stages + int64_t(s) * p.stage_bytes + p.pw * p.C * 2;
      ptx::mbar_arrive_expect_tx(&full[s], uint32_t(KT) * rb);
#pragma unroll 1
      for (int k = 0; k < KT; ++k) {
        const __nv_bfloat16* fr = (k == KT - 1) ? p.x + b * p.x_bstride : ring + (int64_t(p.slot[k]) * B + b) * p.frame;
        ptx::bulk_g2s(st + k * rowp_b, fr + int64_t(hr) * p.W * p.C, rb, &full[s]);
      }
    }
    return;
  }
  // ---- consumers: every warp waits on every row set once, in order (no waiter runs ahead of a barrier)
  const bool active = tid < p.Cq * p.spu;
  const int q = tid % p.Cq, sp = tid / p.Cq;
  const int cstep = p.C;
  const int c0 = sp * PX;
  const int nv = p.Wo - c0;                                         // real pixels of the strip (<= 0: none)
  const uint32_t stages_a = ptx::smem_u32(stages), zst_a = stages_a + uint32_t(p.nst) * uint32_t(p.stage_bytes);
  const uint32_t col_a = uint32_t(c0 * cstep + 4 * q) * 2u;         // this thread's first staged column / quad (bytes)
  uint32_t coff[PX + KW - 1];
#pragma unroll
  for (int t = 0; t < PX + KW - 1; ++t) coff[t] = uint32_t(t * cstep) * 2u;
  // 32-bit counters relative to g0, stages / parities stepped incrementally (64-bit
  // divisions per row made the first version instruction-bound)
  const int n_out = int(hi - lo), n_in = int(g1 - g0);
  int waited = 0, ws = 0, released = 0, rs_i = 0;                   // row sets waited for / released, and their stages
  uint32_t wph = 0;
  int64_t b = lo / p.H;
  int ho = int(lo - b * p.H);
  int gi = int(lo - g0);                                            // this output row's own input row set, relative to g0
  int cs = gi % p.nst;                                              // ... and its stage
  for (int r = 0; r < n_out; ++r) {
    const int last = min(gi - p.ph + KH - 1, gi + (p.H - 1 - ho));   // the window's last row inside the stream
    for (; waited <= last; ++waited) {
      ptx::mbar_wait(&full[ws], wph);
      if (++ws == p.nst) { ws = 0; wph ^= 1u; }
    }
    if (active && nv > 0) {
      float4 acc[PX];
#pragma unroll
      for (int jj = 0; jj < PX; ++jj) acc[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* wq = wt + q * NT;
#pragma unroll
      for (int u = 0; u < KH; ++u) {
        const int hr = ho - p.ph + u;
        int su = cs - p.ph + u;                                     // stage of row set gi - ph + u
        su += su < 0 ? p.nst : 0;
        su -= su >= p.nst ? p.nst : 0;
        // 32-bit shared addresses: row set + this thread's first column, then one add per load
        uint32_t xa = ((hr < 0 || hr >= p.H) ? zst_a : stages_a + uint32_t(su) * uint32_t(p.stage_bytes)) + col_a;
#pragma unroll
        for (int k = 0; k < KT; ++k, xa += uint32_t(rowp_b)) {
          float4 xv[PX + KW - 1];
#pragma unroll
          for (int t = 0; t < PX + KW - 1; ++t) {
            const uint2 raw = ptx::lds64(xa + coff[t]);
            xv[t] = make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xffff0000u),
                                __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xffff0000u));
          }
#pragma unroll
          for (int v = 0; v < KW; ++v) {
            const float4 w = wq[(k * KH + u) * KW + v];
#pragma unroll
            for (int jj = 0; jj < PX; ++jj) acc[jj] = f4_fma(w, xv[jj + v], acc[jj]);
          }
        }
      }
      const float4 bias4 = reinterpret_cast<const float4*>(bs)[q];
      const int64_t pin0 = int64_t(ho) * p.Wo + c0;
      const int64_t yoff = b * p.y_bstride + pin0 * cstep + 4 * q;
      // the new frame's pixels of this strip: row set g, frame kt-1, columns c0 + pw ...
      const uint8_t* crow = stages + cs * p.stage_bytes + (KT - 1) * rowp_b;
      const uint2* xc = reinterpret_cast<const uint2*>(crow) + (int64_t(c0 + p.pw) * cstep + 4 * q) / 4;
      __nv_bfloat16* rs = p.raw_store >= 0 ? ring + (int64_t(p.raw_store) * B + b) * p.frame + pin0 * cstep + 4 * q : nullptr;
#pragma unroll
      for (int jj = 0; jj < PX; ++jj) {
        if (jj >= nv) continue;
        const float4 v = f4_act(f4_add(acc[jj], bias4), p.act);
        if (p.out_f32) {
          *reinterpret_cast<float4*>(static_cast<float*>(p.y) + yoff + jj * cstep) = v;
        } else {
          __nv_bfloat162 lo2 = __floats2bfloat162_rn(v.x, v.y), hi2 = __floats2bfloat162_rn(v.z, v.w);
          uint2 uu;
          uu.x = *reinterpret_cast<uint32_t*>(&lo2);
          uu.y = *reinterpret_cast<uint32_t*>(&hi2);
          *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.y) + yoff + jj * cstep) = uu;
        }
        if (rs) __stcs(reinterpret_cast<uint2*>(rs + jj * cstep), xc[jj * cstep / 4]);
      }
    }
    // release the row sets the next output row does not read (its window starts at its
    // own stream's first row at the earliest)
    const bool wrap = ho + 1 == p.H;
    const int first_next = r + 1 < n_out ? (wrap ? gi + 1 : max(gi + 1 - p.ph, gi - ho)) : n_in;
    __syncwarp();
    for (; released < first_next; ++released) {
      if (lane == 0) ptx::mbar_arrive_relaxed(&empty[rs_i]);
      if (++rs_i == p.nst) rs_i = 0;
    }
    ++gi;
    if (++cs == p.nst) cs = 0;
    if (wrap) { ho = 0; ++b; } else ++ho;
  }
}

// ------------------------------------------------------------------ RAW layout, temporal only, fused store
// A Ready step of a temporal-only depthwise layer over the RAW frame ring
// as one streaming pass: thread item = (pixel, 8 channels), 16-byte
// accesses; the new frame is read straight from x and stored into its ring slot
// here (no separate frame copy), the window's kt - 1 older frames come from the
// ring, y is written once: (kt + 2) frame-sized accesses per step against
// 2 + 4 (kt - 1) for the fp32 partial sums (C3-b, kt = 5: 2.1 MB against 5.4 MB
// per stream-step).  Two items per thread, all 2 kt loads issued before the
// FMAs; per channel the same operations in the same order as k_step_dw_raw.
template <int KT>
__global__ void __launch_bounds__(kDwThreads, KT <= 3 ? 3 : 2) k_step_dw_traw(const DwParams p) {   // (no spills: 2 x KT x 4 load registers)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(p.state);
  const int64_t B = p.plane / p.HWo;
  const int Co = p.C / 8;
  const int64_t n_items = p.plane * Co;
  const int64_t stride = int64_t(gridDim.x) * kDwThreads;
  for (int64_t base = int64_t(blockIdx.x) * kDwThreads + threadIdx.x; base < n_items; base += 2 * stride) {
    uint4 xv[2][KT];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t it = base + j * stride;
      if (it >= n_items) continue;
      const int o = int(it % Co);
      const int64_t pix = it / Co;
      const int64_t b = pix / p.HWo;
#pragma unroll
      for (int k = 0; k < KT - 1; ++k)
        xv[j][k] = *reinterpret_cast<const uint4*>(ring + (int64_t(p.slot[k]) * B) * p.frame + pix * p.C + 8 * o);
      xv[j][KT - 1] = *reinterpret_cast<const uint4*>(p.x + b * p.x_bstride + (pix - b * p.HWo) * p.C + 8 * o);
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int64_t it = base + j * stride;
      if (it >= n_items) continue;
      const int o = int(it % Co);
      const int64_t pix = it / Co;
      const int64_t b = pix / p.HWo;
      if (p.raw_store >= 0)
        __stcs(reinterpret_cast<uint4*>(ring + (int64_t(p.raw_store) * B) * p.frame + pix * p.C + 8 * o), xv[j][KT - 1]);
      float4 acc[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc[h] = __ldg(reinterpret_cast<const float4*>(p.bias) + 2 * o + h);
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          const uint32_t w0 = h ? xv[j][k].z : xv[j][k].x, w1 = h ? xv[j][k].w : xv[j][k].y;
          const float4 xf = make_float4(__uint_as_float(w0 << 16), __uint_as_float(w0 & 0xffff0000u),
                                        __uint_as_float(w1 << 16), __uint_as_float(w1 & 0xffff0000u));
          acc[h] = f4_add(acc[h], f4_fma(__ldg(reinterpret_cast<const float4*>(p.w + k * p.C) + 2 * o + h), xf,
                                         make_float4(0.f, 0.f, 0.f, 0.f)));
        }
        acc[h] = f4_act(acc[h], p.act);
      }
      const int64_t off = b * p.y_bstride + (pix - b * p.HWo) * p.C + 8 * o;
      if (p.out_f32) {
        float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + off);
        __stcs(yp, acc[0]);
        __stcs(yp + 1, acc[1]);
      } else {
        uint4 u;
        __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
        hp[0] = __floats2bfloat162_rn(acc[0].x, acc[0].y);
        hp[1] = __floats2bfloat162_rn(acc[0].z, acc[0].w);
        hp[2] = __floats2bfloat162_rn(acc[1].x, acc[1].y);
        hp[3] = __floats2bfloat162_rn(acc[1].z, acc[1].w);
        *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + off) = u;
      }
    }
  }
}

// ------------------------------------------------------------------ RAW layout
// (SURVEY §8f f1): a Ready step reads the window's kt frames from the frame
// ring (slot[k]) and writes y; no state traffic beyond those reads.  Thread =
// (output pixel, channel quad), NB items per thread with all their loads
// issued before the FMAs; taps read straight from global memory (the 3x3
// neighbours of consecutive pixels are L1 hits).
template <int KT, int KH, int KW>
__global__ void __launch_bounds__(kDwThreads, (KH * KW == 1) ? 3 : 2) k_step_dw_raw(const DwParams p) {
  const __nv_bfloat16* ring = reinterpret_cast<const __nv_bfloat16*>(p.state);
  const int64_t B = p.plane / p.HWo;
  if constexpr (KH * KW == 1) {
    // temporal only: 2 items per thread, all 2 x KT frame reads issued first
    const int64_t n_items = p.plane * p.Cq;
    const int64_t stride = int64_t(gridDim.x) * kDwThreads;
    for (int64_t base = int64_t(blockIdx.x) * kDwThreads + threadIdx.x; base < n_items; base += 2 * stride) {
      float4 xv[2][KT];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t it = base + j * stride;
        if (it >= n_items) continue;
        const int q = int(it % p.Cq);
        const int64_t pix = it / p.Cq;
#pragma unroll
        for (int k = 0; k < KT; ++k)
          xv[j][k] = ld_bf16x4(ring + (int64_t(p.slot[k]) * B) * p.frame + pix * p.C + 4 * q);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t it = base + j * stride;
        if (it >= n_items) continue;
        const int q = int(it % p.Cq);
        const int64_t pix = it / p.Cq;
        const int64_t b = pix / p.HWo;
        float4 acc = __ldg(reinterpret_cast<const float4*>(p.bias) + q);
#pragma unroll
        for (int k = 0; k < KT; ++k)
          acc = f4_add(acc, f4_fma(__ldg(reinterpret_cast<const float4*>(p.w + k * p.C) + q), xv[j][k],
                                   make_float4(0.f, 0.f, 0.f, 0.f)));
        st_out4(p, b, pix - b * p.HWo, q, f4_act(acc, p.act));
      }
    }
  } else {
    // spatial stencil: thread = fixed channel quad x strips of 2 output pixels;
    // per (k, u) the strip's KW+1 input columns are read once (L1 serves the
    // neighbouring strips' overlap), each weight float4 once per strip
    constexpr int PX = 2;
    const int nthr = blockDim.x;
    const int q = int((int64_t(blockIdx.x) * nthr + threadIdx.x) % p.Cq);
    const int64_t sgrp = (int64_t(blockIdx.x) * nthr + threadIdx.x) / p.Cq;
    const int64_t n_sgrp = (int64_t(gridDim.x) * nthr) / p.Cq;
    const int spr = (p.Wo + PX - 1) / PX;
    const int64_t n_strips = B * p.Ho * spr;
    const float4 bias4 = __ldg(reinterpret_cast<const float4*>(p.bias) + q);
    for (int64_t sidx = sgrp; sidx < n_strips && sgrp < n_sgrp; sidx += n_sgrp) {
      const int64_t b = sidx / (int64_t(p.Ho) * spr);
      const int rr = int(sidx - b * p.Ho * spr);
      const int ho = rr / spr, wo0 = (rr - (rr / spr) * spr) * PX;
      float4 acc[PX];
#pragma unroll
      for (int j = 0; j < PX; ++j) acc[j] = bias4;
#pragma unroll
      for (int k = 0; k < KT; ++k) {
        const __nv_bfloat16* fr = ring + (int64_t(p.slot[k]) * B + b) * p.frame + 4 * q;
        float4 part[PX];
#pragma unroll
        for (int j = 0; j < PX; ++j) part[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < KH; ++u) {
          const int hi = ho + u - p.ph;
          if (hi < 0 || hi >= p.H) continue;
          float4 xv[PX + KW - 1];
#pragma unroll
          for (int t = 0; t < PX + KW - 1; ++t) {
            const int wi = wo0 + t - p.pw;
            xv[t] = (wi >= 0 && wi < p.W) ? ld_bf16x4(fr + (int64_t(hi) * p.W + wi) * p.C)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int v = 0; v < KW; ++v) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(p.w + ((k * KH + u) * KW + v) * p.C) + q);
#pragma unroll
            for (int j = 0; j < PX; ++j) part[j] = f4_fma(w, xv[j + v], part[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < PX; ++j) acc[j] = f4_add(acc[j], part[j]);
      }
#pragma unroll
      for (int j = 0; j < PX; ++j)
        if (wo0 + j < p.Wo) st_out4(p, b, int64_t(ho) * p.Wo + wo0 + j, q, f4_act(acc[j], p.act));
    }
  }
}

// (C, 1, kt, kh, kw) bf16 -> [kt][kh][kw][C] fp32 (exact)
__global__ void k_pack_dw(const __nv_bfloat16* __restrict__ w, float* __restrict__ out, int C, int kt, int kh,
                          int kw) {
  const int n = C * kt * kh * kw;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int r = i;
  const int v = r % kw; r /= kw;
  const int u = r % kh; r /= kh;
  const int k = r % kt; r /= kt;
  const int c = r;
  out[((k * kh + u) * kw + v) * C + c] = __bfloat162float(w[i]);
}

typedef void (*DwFn)(const DwParams);
typedef void (*DwChunkFn)(const DwParams, const ChunkArgs);
struct DwVariant {
  int KT, KH, KW;
  DwFn fn;
  int PX = 1;                           // K2: output pixels per thread strip
  DwFn raw = nullptr;                   // RAW-layout kernel for this shape
  DwChunkFn chunk = nullptr;            // chunked-steps kernel (temporal only)
  DwFn seg = nullptr;                   // K2s segment-pipeline kernel (spatial stencils)
  int SPX = 4;                          // K2s: output pixels per thread strip
  DwFn traw = nullptr;                  // RAW layout, temporal only: fused frame store (k_step_dw_traw)
  DwFn rowraw = nullptr;                // RAW layout, "same"-padded stencils: rolling row sets, frame store fused
};
#ifndef CO_DW_PX
#define CO_DW_PX 2                      // output pixels per thread strip (experiments: -DCO_DW_PX=n)
#endif
// K2s strip: 7 pixels (WS = 14: C3-a's 28-pixel rows in two units of 96
// threads; weights read from shared memory once per 7 pixels), 4 for the
// register-heavier 5x5 / kt = 5 stencils
#define CO_DW_SEG_PX(kt, kh, kw) ((kt) <= 3 && (kh) * (kw) <= 9 ? 7 : 4)
#ifndef CO_DW_ROWRAW_PX
#define CO_DW_ROWRAW_PX 4                // rolling-row RAW stencil: output pixels per thread strip (C3-a: 4 -> 0.228 ms on
                                        // 11 consumer warps, 7 -> 0.252 ms on 6)
#endif
#define CO_DW_ST(kt, kh, kw) {kt, kh, kw, (DwFn)k_step_dw_st<kt, kh, kw, (kt <= 3 ? CO_DW_PX : 2)>, \
                              (kt <= 3 ? CO_DW_PX : 2), (DwFn)k_step_dw_raw<kt, kh, kw>, \
                              (DwChunkFn)k_steps_dw_st<kt, kh, kw, (kt <= 3 ? CO_DW_PX : 2)>, \
                              (DwFn)k_step_dw_seg<kt, kh, kw, CO_DW_SEG_PX(kt, kh, kw)>, CO_DW_SEG_PX(kt, kh, kw), nullptr, \
                              (DwFn)k_step_dw_rowraw<kt, kh, kw, CO_DW_ROWRAW_PX>}
#define CO_DW_T(kt) {kt, 1, 1, (DwFn)k_step_dw_t<kt>, 1, (DwFn)k_step_dw_raw<kt, 1, 1>, (DwChunkFn)k_steps_dw_t<kt>, \
                     nullptr, 4, (DwFn)k_step_dw_traw<kt>}
const DwVariant kDwVariants[] = {
    CO_DW_ST(1, 3, 3), CO_DW_ST(2, 3, 3), CO_DW_ST(3, 3, 3), CO_DW_ST(5, 3, 3), CO_DW_ST(3, 5, 5),
    CO_DW_T(2), CO_DW_T(3), CO_DW_T(4), CO_DW_T(5), CO_DW_T(7), CO_DW_T(9),
};

struct DwPlan {
  const DwVariant* var = nullptr;
  bool temporal = false;
  int threads = kDwThreads;             // K2: Cq * (rows of strips) <= 256
  int TH = 0, bands = 0, HR = 0, WC = 0;
  int64_t n_tiles = 0;
  size_t smem = 0;
  // K2s segment pipeline (option "dw_seg")
  bool seg = false;
  int nseg = 0, WS = 0, WX = 0, nst = 0, spu = 0, gthreads = 0, ngroups = 0;
  int stage_bytes = 0, x_off = 0, stage_off = 0, bar_off = 0;
  int64_t n_units = 0;
  size_t seg_smem = 0;
};

#ifndef CO_DW_SEG_SMEM_KB
#define CO_DW_SEG_SMEM_KB 220           // K2s shared-memory budget per CTA (one CTA per SM)
#endif

// K2s plan: the fewest segments per output row whose strips fit one consumer
// group (<= kSegGroupMax threads) and whose nst stages (ngroups + 2, else + 1)
// fit the budget; up to three consumer groups (C3-a: 3 x 96 threads, 5 stages;
// measured 0.37 ms with 2 groups / 4 stages, 0.30 with 3 / 5; experiments:
// CO_DW_SEG_NG / _NST).
bool make_seg_plan(const Geom& g, const DwVariant& v, DwPlan& pl) {
  if (!v.seg || g.Cout / 4 > kSegGroupMax) return false;
  const int PX = v.SPX, Cq = g.Cout / 4;
  const size_t base = (size_t(g.kt * g.kh * g.kw + 1) * g.Cin * 4 + 127) / 128 * 128;
  for (int nseg = 1; nseg <= g.Wo; ++nseg) {
    const int WS = ((g.Wo + nseg - 1) / nseg + PX - 1) / PX * PX;
    if (int64_t(nseg - 1) * WS >= g.Wo) continue;                  // would leave an empty segment
    const int spu = WS / PX;
    const int gth = (Cq * spu + 31) / 32 * 32;
    if (gth > kSegGroupMax) continue;
    const int ng = std::max(2, std::min(CO_EXP("CO_DW_SEG_NG", 3), (kSegMaxThreads - 32) / gth));
    const int WX = WS + g.kw - 1;
    const size_t x_off = size_t(std::max(g.kt - 1, 0)) * WS * g.Cout * 4;
    const size_t sb = (x_off + size_t(g.kh) * WX * g.Cin * 2 + 127) / 128 * 128;
    for (int nst = std::max(CO_EXP("CO_DW_SEG_NST", ng + 2), ng + 1); nst >= ng + 1; --nst) {
      const size_t smem = base + nst * sb + 2 * size_t(nst) * 8;
      if (smem > size_t(CO_DW_SEG_SMEM_KB) * 1024) continue;
      pl.seg = true;
      pl.nseg = nseg; pl.WS = WS; pl.WX = WX; pl.nst = nst; pl.spu = spu; pl.gthreads = gth; pl.ngroups = ng;
      pl.stage_bytes = int(sb); pl.x_off = int(x_off); pl.stage_off = int(base);
      pl.bar_off = int(base + nst * sb);
      pl.n_units = g.B * g.Ho * nseg;
      if (pl.n_units >= (int64_t(1) << 31)) return false;
      pl.seg_smem = smem;
      return true;
    }
  }
  return false;
}

// Rolling-row plan of the RAW stencil (k_step_dw_rowraw): all consumer threads on one
// output row (channel quads x strips of 4 pixels), kh + 2 row-set stages (kh + 1
// if shared memory is short) + the zero stage.
bool make_rowraw_plan(const Geom& g, const DwVariant& v, DwPlan& pl) {
  if (!v.rowraw) return false;
  const int PX = CO_DW_ROWRAW_PX, Cq = g.Cout / 4;
  const int spu = (g.Wo + PX - 1) / PX;
  const int gth = (Cq * spu + 31) / 32 * 32;
  if (gth + 32 > kSegMaxThreads) return false;
  const int WX = std::max(g.W + g.kw - 1, spu * PX + g.kw - 1);
  const size_t sb = (size_t(g.kt) * WX * g.Cin * 2 + 127) / 128 * 128;
  const size_t base = (size_t(g.kt * g.kh * g.kw + 1) * g.Cin * 4 + 127) / 128 * 128;
  for (int nst = g.kh + 2; nst >= g.kh + 1; --nst) {
    const size_t smem = base + size_t(nst + 1) * sb + 2 * size_t(nst) * 8;
    if (smem > size_t(227) * 1024) continue;
    pl.seg = true;
    pl.nseg = 1; pl.WS = g.Wo; pl.WX = WX; pl.nst = nst; pl.spu = spu; pl.gthreads = gth; pl.ngroups = 1;
    pl.stage_bytes = int(sb); pl.x_off = 0; pl.stage_off = int(base);
    pl.bar_off = int(base + size_t(nst + 1) * sb);
    pl.n_units = g.B * g.Ho;
    pl.seg_smem = smem;
    return true;
  }
  return false;
}

bool make_dw_plan(const Geom& g, DwPlan& pl) {
  if (g.in_dtype != BF16 || g.groups != g.Cin || g.Cin != g.Cout || g.Cin % 8 != 0) return false;
  if (g.sh != 1 || g.sw != 1 || g.dh != 1 || g.dw != 1) return false;
  const bool temporal = (g.kh == 1 && g.kw == 1 && g.ph == 0 && g.pw == 0);
  for (const DwVariant& v : kDwVariants) {
    if (v.KT != g.kt) continue;
    if (temporal ? (v.KH != 1) : (v.KH != g.kh || v.KW != g.kw)) continue;
    pl.var = &v;
  }
  if (!pl.var) return false;
  pl.temporal = temporal;
  if (g.raw && !temporal && option(OPT_DW_SEG) && g.Ho == g.H && g.Wo == g.W)
    make_rowraw_plan(g, *pl.var, pl);   // RAW stencil, "same" padding: a row's threads store their own input pixels
  if (temporal || g.raw) return true;   // no staged halo (RAW reads the ring directly)
  // staged halo width: every strip reads PX + kw - 1 columns (zero beyond the frame)
  const int px = pl.var->PX;
  pl.WC = std::max(g.W + 2 * g.pw, (g.Wo + px - 1) / px * px + g.kw - 1);
  const size_t row_bytes = size_t(pl.WC) * g.Cin * 2;
  int TH = int(kHaloBudget / row_bytes) - (g.kh - 1);
  if (TH < 1) {
    if (size_t(g.kh) * row_bytes > 160 * 1024) return false;
    TH = 1;
  }
  TH = std::min(TH, g.Ho);
  pl.TH = TH;
  pl.HR = TH + g.kh - 1;
  pl.bands = (g.Ho + TH - 1) / TH;
  pl.n_tiles = g.B * pl.bands;
  pl.smem = size_t(g.kt * g.kh * g.kw + 1) * g.Cin * 4 + size_t(pl.HR) * row_bytes;
  const int Cq = g.Cin / 4;
  if (Cq > 256) return false;
  pl.threads = Cq * (256 / Cq);
  if (option(OPT_DW_SEG)) make_seg_plan(g, *pl.var, pl);
  return pl.seg || pl.smem <= 227 * 1024;
}

}  // namespace

struct Depthwise {
  DwPlan pl;
  float* w = nullptr;
  void* zeros = nullptr;                // K2s: padding source (WX * C * 2 zero bytes)
  int grid = 0;
  int grid_traw = 0;                    // RAW temporal kernel with the fused frame store (16-byte items)
  int grid_rowraw = 0;                  // RAW stencil over rolling row sets with the fused frame store
  std::string name;
};

bool depthwise_supported(const Geom& g) {
  DwPlan pl;
  return make_dw_plan(g, pl);
}

Depthwise* depthwise_create(const Geom& g, const void* w_dev, std::string& err) {
  DwPlan pl;
  if (!make_dw_plan(g, pl)) { err = "unsupported shape"; return nullptr; }
  Depthwise* t = new Depthwise();
  t->pl = pl;
  const int n = g.Cin * g.kt * g.kh * g.kw;
  cudaError_t e = cudaMalloc(&t->w, size_t(n) * 4);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); delete t; return nullptr; }
  k_pack_dw<<<(n + 255) / 256, 256>>>(static_cast<const __nv_bfloat16*>(w_dev), t->w, g.Cin, g.kt, g.kh, g.kw);
  if ((e = cudaGetLastError()) != cudaSuccess) { err = cudaGetErrorString(e); depthwise_destroy(t); return nullptr; }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g.raw) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.var->raw, kDwThreads, 0);
    per_sm = std::max(per_sm, 1);
    const int64_t items = g.B * g.HWo * (g.Cout / 4);
    t->grid = int(std::max<int64_t>(1, std::min<int64_t>((items + kDwThreads - 1) / kDwThreads, int64_t(sms) * per_sm)));
    if (!pl.temporal) {   // the stencil maps threads to (quad, strip group): whole quad sets per grid
      const int64_t cq = g.Cout / 4;
      const int64_t thr = int64_t(t->grid) * kDwThreads;
      if (thr < cq) t->grid = int((cq + kDwThreads - 1) / kDwThreads);
    }
    char buf[96];
    snprintf(buf, sizeof(buf), "k_step_dw_raw<%d,%d,%d>", pl.var->KT, pl.var->KH, pl.var->KW);
    if (pl.temporal && pl.var->traw) {
      int per = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pl.var->traw, kDwThreads, 0);
      const int64_t it8 = g.B * g.HWo * (g.Cout / 8);
      t->grid_traw = int(std::max<int64_t>(1, std::min<int64_t>((it8 + 2 * kDwThreads - 1) / (2 * kDwThreads),
                                                                int64_t(sms) * std::max(per, 1))));
      snprintf(buf, sizeof(buf), "k_step_dw_traw<%d>", pl.var->KT);
    }
    if (pl.seg) {   // RAW stencil over rolling row sets for Ready steps that read x (k_step_dw_rowraw)
      if ((e = cudaFuncSetAttribute(pl.var->rowraw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.seg_smem))) != cudaSuccess) {
        err = cudaGetErrorString(e); depthwise_destroy(t); return nullptr;
      }
      t->grid_rowraw = int(std::max<int64_t>(1, std::min<int64_t>(pl.n_units, int64_t(sms))));
      snprintf(buf, sizeof(buf), "k_step_dw_rowraw<%d,%d,%d>", pl.var->KT, pl.var->KH, pl.var->KW);
    }
    t->name = buf;
    return t;
  }
  if (pl.seg) {
    const size_t zb = size_t(pl.WX) * g.Cin * 2;
    if ((e = cudaMalloc(&t->zeros, zb)) != cudaSuccess || (e = cudaMemset(t->zeros, 0, zb)) != cudaSuccess) {
      err = cudaGetErrorString(e); depthwise_destroy(t); return nullptr;
    }
    e = cudaFuncSetAttribute(pl.var->seg, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.seg_smem));
    if (e != cudaSuccess) { err = cudaGetErrorString(e); depthwise_destroy(t); return nullptr; }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.var->seg, pl.ngroups * pl.gthreads + 32, pl.seg_smem);
    per_sm = std::max(per_sm, 1);
    t->grid = int(std::max<int64_t>(1, std::min<int64_t>(pl.n_units, int64_t(sms) * per_sm)));
    char buf[96];
    snprintf(buf, sizeof(buf), "k_step_dw_seg<%d,%d,%d>", pl.var->KT, pl.var->KH, pl.var->KW);
    t->name = buf;
    return t;
  }
  if (!pl.temporal) {
    e = cudaFuncSetAttribute(pl.var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
    if (e != cudaSuccess) { err = cudaGetErrorString(e); depthwise_destroy(t); return nullptr; }
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pl.var->fn, pl.temporal ? kDwThreads : pl.threads,
                                                pl.temporal ? 0 : pl.smem);
  per_sm = std::max(per_sm, 1);
  if (pl.temporal) {
    const int64_t items = g.B * g.HWo * (g.Cout / 4);
    const int64_t need = (items + int64_t(kNB) * kDwThreads - 1) / (int64_t(kNB) * kDwThreads);
    t->grid = int(std::max<int64_t>(1, std::min<int64_t>(need, int64_t(sms) * per_sm)));
  } else {
    t->grid = int(std::max<int64_t>(1, std::min<int64_t>(pl.n_tiles, int64_t(sms) * per_sm)));
  }
  char buf[96];
  if (pl.temporal)
    snprintf(buf, sizeof(buf), "k_step_dw_t<%d>", pl.var->KT);
  else
    snprintf(buf, sizeof(buf), "k_step_dw_st<%d,%d,%d>", pl.var->KT, pl.var->KH, pl.var->KW);
  t->name = buf;
  return t;
}

// Chunked K2 tile plan: TH output rows per CTA with one thread per (quad, strip),
// two halo buffers; 0 rows = not chunkable.
static int st_chunk_rows(const Depthwise* t, const Geom& g, int& WC, size_t& smem) {
  const int px = t->pl.var->PX;
  const int spr = (g.Wo + px - 1) / px;
  const int Cq = g.Cout / 4;
  if (Cq * spr > 1024) return 0;
  WC = std::max(g.W + 2 * g.pw, spr * px + g.kw - 1);
  int TH = std::min(g.Ho, 1024 / (Cq * spr));
  for (; TH >= 1; --TH) {
    smem = size_t(g.kt * g.kh * g.kw + 1) * g.Cin * 4 + 2 * size_t(TH + g.kh - 1) * WC * g.Cin * 2;
    if (smem <= 200 * 1024) return TH;
  }
  return 0;
}

bool depthwise_chunkable(const Depthwise* t, const Geom& g) {
  if (!option(OPT_CHUNK)) return false;          // option "chunk" = 0: always fold per step
  if (!t || !t->pl.var->chunk || g.raw || g.st != 1 || g.dt != 1 || g.kt < 2) return false;
  if (t->pl.temporal) return true;
  // chunked K2 (k_steps_dw_st) is correct but slower than the per-step K2 on C3-a
  // (1.12 M vs 1.48 M stream-steps/s: shared-memory / latency bound at one
  // 672-thread CTA per SM), so the stencil folds per step unless option "chunk_st" = 1
  if (!option(OPT_CHUNK_ST)) return false;
  int WC;
  size_t smem;
  return st_chunk_rows(t, g, WC, smem) > 0;
}

cudaError_t depthwise_steps(Depthwise* t, const Geom& g, const void* x, int64_t T, int64_t total, int64_t n0, void* y,
                            int64_t y_bstride, float* state, const float* bias, cudaStream_t s) {
  DwParams p{};
  p.y = y;
  p.y_bstride = y_bstride;
  p.state = state;
  p.w = t->w;
  p.bias = bias;
  p.act = g.act; p.out_f32 = (g.out_dtype == F32);
  p.C = g.Cout; p.Cq = g.Cout / 4; p.H = g.H; p.W = g.W; p.Ho = g.Ho; p.Wo = g.Wo;
  p.HWo = g.HWo; p.plane = g.B * g.HWo;
  ChunkArgs c{};
  c.x = static_cast<const __nv_bfloat16*>(x);
  c.x_bstride = T * g.frame_elems;
  c.T = T; c.total = total;
  c.n0 = n0; c.m0 = n0 + g.pt; c.d = g.delay;
  c.oi0 = n0 > g.delay ? n0 : g.delay;
  c.y_bstride = y_bstride;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* args[] = {&p, &c};
  if (!t->pl.temporal) {   // K2c: one CTA per (stream, TH-row band), Cq x strips threads
    int WC;
    size_t smem;
    const int TH = st_chunk_rows(t, g, WC, smem);
    if (TH < 1) return cudaErrorInvalidValue;
    p.H = g.H; p.W = g.W; p.ph = g.ph; p.pw = g.pw;
    p.TH = TH; p.HR = TH + g.kh - 1; p.WC = WC;
    p.bands = (g.Ho + TH - 1) / TH;
    p.n_tiles = g.B * p.bands;
    const int spr = (g.Wo + t->pl.var->PX - 1) / t->pl.var->PX;
    const int threads = p.Cq * TH * spr;
    cudaFuncSetAttribute(t->pl.var->chunk, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, t->pl.var->chunk, threads, smem);
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(p.n_tiles, int64_t(sms) * std::max(per_sm, 1))));
    return cudaLaunchKernel(reinterpret_cast<const void*>(t->pl.var->chunk), dim3(unsigned(grid)), dim3(threads),
                            args, smem, s);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, t->pl.var->chunk, kDwThreads, 0);
  const int64_t items = p.plane * p.Cq;
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((items + kDwThreads - 1) / kDwThreads,
                                                              int64_t(sms) * std::max(per_sm, 1))));
  return cudaLaunchKernel(reinterpret_cast<const void*>(t->pl.var->chunk), dim3(unsigned(grid)), dim3(kDwThreads),
                          args, 0, s);
}

void depthwise_destroy(Depthwise* t) {
  if (!t) return;
  cudaFree(t->w);
  cudaFree(t->zeros);
  delete t;
}

const char* depthwise_name(const Depthwise* t) { return t->name.c_str(); }

bool depthwise_fuses_raw_store(const Depthwise* t, const Geom& g, int64_t x_bstride) {
  if (!t || !g.raw || g.Cout % 8 != 0 || (x_bstride * 2) % 16 != 0) return false;
  return t->pl.temporal ? t->grid_traw > 0 : t->grid_rowraw > 0;
}

bool depthwise_raw_pipeline(const Geom& g) {
  DwPlan pl;
  return g.raw && make_dw_plan(g, pl) && !pl.temporal && pl.seg;
}

cudaError_t depthwise_step(Depthwise* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s) {
  const DwPlan& pl = t->pl;
  DwParams p{};
  p.x = static_cast<const __nv_bfloat16*>(a.x);
  p.x_bstride = a.x_bstride;
  p.y = a.y;
  p.y_bstride = a.y_bstride;
  p.state = a.state;
  p.w = t->w;
  p.bias = bias;
  for (int k = 0; k < kMaxKt; ++k) p.slot[k] = a.slot[k];
  p.emit = a.emit; p.update = a.update; p.act = g.act; p.out_f32 = (g.out_dtype == F32);
  p.frame = g.frame_elems;
  p.C = g.Cout; p.Cq = g.Cout / 4; p.H = g.H; p.W = g.W; p.Ho = g.Ho; p.Wo = g.Wo; p.ph = g.ph; p.pw = g.pw;
  p.HWo = g.HWo; p.plane = g.B * g.HWo;
  p.TH = pl.TH; p.bands = pl.bands; p.n_tiles = pl.n_tiles; p.WC = pl.WC; p.HR = pl.HR;
  void* args[] = {&p};
  if (g.raw && a.x && a.emit && depthwise_fuses_raw_store(t, g, a.x_bstride)) {
    // Ready step reading the new frame from x (host.cu step_raw): one streaming pass, frame stored here
    p.raw_store = a.raw_store;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(t->grid_traw));
    cfg.blockDim = dim3(kDwThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = option(OPT_PDL) != 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!pl.temporal) {   // the stencil over rolling row sets
      p.n_units = pl.n_units; p.nseg = pl.nseg; p.WS = pl.WS; p.WX = pl.WX; p.nst = pl.nst; p.spu = pl.spu;
      p.gthreads = pl.gthreads; p.stage_bytes = pl.stage_bytes; p.x_off = pl.x_off; p.stage_off = pl.stage_off;
      p.bar_off = pl.bar_off; p.ngroups = pl.ngroups;
      cfg.gridDim = dim3(unsigned(t->grid_rowraw));
      cfg.blockDim = dim3(unsigned(pl.gthreads + 32));
      cfg.dynamicSmemBytes = pl.seg_smem;
      return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(pl.var->rowraw), args);
    }
    return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(pl.var->traw), args);
  }
  if (g.raw)
    return cudaLaunchKernel(reinterpret_cast<const void*>(pl.var->raw), dim3(unsigned(t->grid)), dim3(kDwThreads),
                            args, 0, s);
  if (pl.seg) {
    p.n_units = pl.n_units; p.nseg = pl.nseg; p.WS = pl.WS; p.WX = pl.WX; p.nst = pl.nst; p.spu = pl.spu;
    p.gthreads = pl.gthreads; p.stage_bytes = pl.stage_bytes; p.x_off = pl.x_off; p.stage_off = pl.stage_off;
    p.bar_off = pl.bar_off; p.ngroups = pl.ngroups; p.zeros = t->zeros;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(t->grid));
  cfg.blockDim = dim3(pl.seg ? pl.ngroups * pl.gthreads + 32 : pl.temporal ? kDwThreads : pl.threads);
  cfg.dynamicSmemBytes = pl.seg ? pl.seg_smem : pl.temporal ? 0 : pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // option "pdl" = 0: off
  attr[0].val.programmaticStreamSerializationAllowed = option(OPT_PDL) != 0 ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(pl.seg ? pl.var->seg : pl.var->fn), args);
}

}  // namespace co
