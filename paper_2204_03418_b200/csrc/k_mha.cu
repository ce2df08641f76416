// k_mha.cu — continual single-output multi-head attention (
// PAPER.md P:430-432 co.MultiheadAttention "single-output").
//
// A step is three launches on B lockstep streams:
//   1. qkv = x W_qkv^T + b_qkv   -- a kt = 1 continual layer (co_conv, tcgen05)
//   2. k_mha_attend: store (k_t, v_t) in ring slot m mod n, then per (stream,
//      head) the attention of q_t against the window's n keys / values (the
//      newest from qkv, the n-1 older from the ring)
//   3. y = a W_o^T + b_o         -- a kt = 1 continual layer (co_conv, tcgen05)
// Step 2 is the decode-attention shape: one query against an n-entry KV ring,
// 2 n E bf16 read per stream-step -- HBM-bound (SURVEY §8d style:
// arithmetic intensity ~ 1 FLOP/B).  Warp per (row, head), dh = 64: 8 lanes
// cover one 128-byte key row with 16-byte loads, so a warp reads 4 keys per
// iteration (512 contiguous bytes per request); each 8-lane key group keeps an
// online softmax (running max m, sum l, accumulator o[8]) over its keys, and the
// 4 groups are merged at the end (max-rescaled sums) -- all scores stay in
// registers, any window length.  Ring layout [B][n][E]: a stream's window is
// one contiguous n E run (a [n][B][E] layout spread each warp's keys over n
// regions 2 MB apart and ran at a third of HBM bandwidth).  Batch mode (co_mha_forward) runs the same
// kernel with keys / values read from the projected clip (all T columns).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace co {


namespace {

// ring-pipeline attention (k_mha_attend_ring): one consumer warp per head + a producer warp
constexpr int kMhaRingMaxHeads = 16;
constexpr int kMhaRingMaxThreads = (kMhaRingMaxHeads + 1) * 32;
struct MhaRingPlan {
  int kc, nchunks;          // keys per stage, stages per stream
  int nst, stage_bytes;     // ring depth; K chunk + V chunk
};

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 v = __bfloat1622float2(h[i]);
    f[2 * i] = v.x;
    f[2 * i + 1] = v.y;
  }
}

// DH = head dim; LPK = lanes per key row (DH / 8); KPI = keys per iteration.
template <int DH, int KU = 1>
__global__ void __launch_bounds__(256, KU == 1 ? 4 : 3) k_mha_attend(const MhaArgs a) {
  constexpr int LPK = DH / 8, KPI = 32 / LPK;
  const int lane = threadIdx.x & 31;
  const int g = lane % LPK;           // 8-dim chunk of the head this lane owns
  const int ks = lane / LPK;          // key subgroup
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t rows = a.B * a.T;
  // programmatic dependent launch: scheduled while the QKV projection drains,
  // reads its output only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int64_t w = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < rows * a.heads; w += warps) {
    const int h = int(w % a.heads);
    const int64_t r = w / a.heads;                 // row = (b, t)
    const int64_t b = a.T == 1 ? r : r / a.T;
    const int hc = h * DH + g * 8;                 // this lane's 8 channels
    const __nv_bfloat16* qrow = a.qkv + r * 3 * a.E;
    float q[8];
    ld8(qrow + hc, q);

    const int nk = a.batch ? int(a.T) : a.n;
    float mx = -INFINITY, l = 0.f, o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = 0.f;
    // software pipeline: the next key group's K / V rows (raw bf16, 4 + 4
    // registers) are in flight while the current one is folded into the
    // online softmax
    // key j: batch -> column j of the clip; step -> j steps ago, j = 0 from qkv,
    // else ring slot (m - j) mod n = s0 - j (+ n) (32-bit: no 64-bit modulo
    // in the loop -- it made the first version instruction-bound)
    const int s0 = a.batch ? 0 : int(a.m % a.n);
    const __nv_bfloat16* kbase = a.batch ? a.qkv + (b * a.T) * 3 * a.E + a.E + hc : a.kring + b * a.n * a.E + hc;
    const __nv_bfloat16* vbase = a.batch ? kbase + a.E : a.vring + b * a.n * a.E + hc;
    const int kstride = a.batch ? 3 * a.E : a.E;
    if (!a.batch && a.store && ks == 0) {          // ring update: this step's key / value
      *reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(kbase) + s0 * a.E) =
          *reinterpret_cast<const uint4*>(qrow + a.E + hc);
      *reinterpret_cast<uint4*>(const_cast<__nv_bfloat16*>(vbase) + s0 * a.E) =
          *reinterpret_cast<const uint4*>(qrow + 2 * a.E + hc);
    }
    auto load = [&](int j, uint4& kr, uint4& vr) {
      const __nv_bfloat16 *kp, *vp;
      if (!a.batch && j == 0) {
        kp = qrow + a.E + hc;
        vp = qrow + 2 * a.E + hc;
      } else {
        int idx = j;
        if (!a.batch) {
          idx = s0 - j;
          idx += idx < 0 ? a.n : 0;
        }
        kp = kbase + idx * kstride;
        vp = vbase + idx * kstride;
      }
      kr = *reinterpret_cast<const uint4*>(kp);
      vr = *reinterpret_cast<const uint4*>(vp);
    };
    // KU keys per lane per iteration (key j0 + u KPI + ks): KU x (K, V) rows in
    // flight for the current group and KU for the next one
    constexpr int KSTEP = KPI * KU;
    uint4 kc[KU], vc[KU], kn[KU], vn[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      kc[u] = vc[u] = kn[u] = vn[u] = make_uint4(0, 0, 0, 0);
      if (u * KPI + ks < nk) load(u * KPI + ks, kc[u], vc[u]);
    }
    for (int j0 = 0; j0 < nk; j0 += KSTEP) {
#pragma unroll
      for (int u = 0; u < KU; ++u)
        if (j0 + KSTEP + u * KPI + ks < nk) load(j0 + KSTEP + u * KPI + ks, kn[u], vn[u]);
      float sc[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        float s = 0.f;
        const __nv_bfloat162* kh2 = reinterpret_cast<const __nv_bfloat162*>(&kc[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 kf = __bfloat1622float2(kh2[i]);
          s = fmaf(q[2 * i], kf.x, s);
          s = fmaf(q[2 * i + 1], kf.y, s);
        }
        sc[u] = s;
      }
#pragma unroll
      for (int off = LPK / 2; off > 0; off >>= 1)
#pragma unroll
        for (int u = 0; u < KU; ++u) sc[u] += __shfl_xor_sync(0xffffffffu, sc[u], off);   // within the key row
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        if (j0 + u * KPI + ks >= nk) continue;      // (keys in index order per lane: same fold as KU = 1)
        const float s = sc[u] * a.scale_log2e;     // base-2 logits
        const float mn = fmaxf(mx, s);
        const float c = exp2f(mx - mn), e = exp2f(s - mn);
        l = l * c + e;
        const __nv_bfloat162* vh2 = reinterpret_cast<const __nv_bfloat162*>(&vc[u]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 vf = __bfloat1622float2(vh2[i]);
          o[2 * i] = fmaf(e, vf.x, o[2 * i] * c);
          o[2 * i + 1] = fmaf(e, vf.y, o[2 * i + 1] * c);
        }
        mx = mn;
      }
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        kc[u] = kn[u];
        vc[u] = vn[u];
      }
    }
    // merge the KPI key subgroups (lanes g, g + LPK, ...)
#pragma unroll
    for (int off = LPK; off < 32; off <<= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, mx, off);
      const float lo = __shfl_xor_sync(0xffffffffu, l, off);
      const float mn = fmaxf(mx, mo);
      const float c1 = (mx == -INFINITY) ? 0.f : exp2f(mx - mn), c2 = (mo == -INFINITY) ? 0.f : exp2f(mo - mn);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float oo = __shfl_xor_sync(0xffffffffu, o[i], off);
        o[i] = o[i] * c1 + oo * c2;
      }
      l = l * c1 + lo * c2;
      mx = mn;
    }
    if (ks == 0) {
      const float inv = 1.f / l;
      uint4 u;
      __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int i = 0; i < 4; ++i) hp[i] = __floats2bfloat162_rn(o[2 * i] * inv, o[2 * i + 1] * inv);
      *reinterpret_cast<uint4*>(a.out + r * a.E + hc) = u;
    }
  }
}

// ------------------------------------------------------------------ ring pipeline (step mode)
// The step-mode attention with its memory traffic decoupled from the
// arithmetic (the K2s recipe, k_depthwise.cu).  k_mha_attend keeps 2-4 K / V
// rows per lane in flight and measured latency-bound at 0.62 of HBM (ncu: issue
// 47%, DRAM 49%).  Here a CTA owns a contiguous range of streams; one producer
// thread streams each stream's K ring and V ring -- contiguous [n][E] runs --
// in chunks of `kc` keys (kc E bf16 of K + the same of V per stage) into a
// ring of `nst` shared-memory stages with bulk copies (cp.async.bulk,
// mbarrier complete_tx), so nst - 1 stages (~128 KB per SM) are in flight while
// one warp per head folds the staged keys into its online softmax (the same
// lane = (8-channel chunk, key subgroup) arrangement and merge as
// k_mha_attend; keys are taken in ring-slot order, the slot of this step --
// m mod n, holding the key that left the window -- is replaced by (k_t, v_t)
// from the projection's output, and written back once its chunk has landed).
template <int DH>
__global__ void __launch_bounds__(kMhaRingMaxThreads, 1) k_mha_attend_ring(const MhaArgs a, const MhaRingPlan pl) {
  constexpr int LPK = DH / 8, KPI = 32 / LPK;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + size_t(pl.nst) * pl.stage_bytes);
  uint64_t* empty = full + pl.nst;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < pl.nst; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], a.heads);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // programmatic dependent launch: the ring (previous attention launch) and
  // qkv (the projection before this one) are read only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t lo = a.B * blockIdx.x / gridDim.x, hi = a.B * (blockIdx.x + 1) / gridDim.x;
  const int half = pl.stage_bytes / 2;              // K chunk at 0, V chunk at `half`
  const int row_b = a.E * 2;
  if (warp == a.heads) {                            // ---- producer thread
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;                                // fill k of a stage waits for empty phase k - 1: parity ph ^ 1
    bool refill = false;
    for (int64_t b = lo; b < hi; ++b)
      for (int c = 0; c < pl.nchunks; ++c) {
        if (refill) ptx::mbar_wait(&empty[s], ph ^ 1u);
        const int rows = min(pl.kc, a.n - c * pl.kc);
        const uint32_t bytes = uint32_t(rows) * row_b;
        uint8_t* st = stages + size_t(s) * pl.stage_bytes;
        const int64_t off = (b * a.n + int64_t(c) * pl.kc) * a.E;
        ptx::mbar_arrive_expect_tx(&full[s], 2 * bytes);
        ptx::bulk_g2s(st, a.kring + off, bytes, &full[s]);
        ptx::bulk_g2s(st + half, a.vring + off, bytes, &full[s]);
        if (++s == pl.nst) { s = 0; ph ^= 1u; refill = true; }
      }
    return;
  }
  // ---- consumers: warp = head.  Branch-free inner loop (the first version ran
  // 137 instructions per 4-key iteration, issue-bound at 65%): a lane folds two
  // keys per iteration with one rescale (o = o cf + e0 v0 + e1 v1, 3 exp2 per
  // 2 keys); masked keys (past the window, or this step's slot) score -inf and
  // read a clamped row (ring rows are finite, so their zero weights stay zeros);
  // the running max starts at -1e30 instead of -inf, so no inf - inf arises;
  // this step's (k_t, v_t) is folded first, by key subgroup 0.
  constexpr float kNegBig = -1e30f;
  const int g = lane % LPK, ks = lane / LPK;
  const int hc = warp * DH + g * 8;                 // this lane's 8 channels
  const int n = a.n, kc = pl.kc, nchunks = pl.nchunks, nst = pl.nst, E = a.E;
  const int s0 = int(a.m % n), c0 = s0 / kc;        // this step's ring slot and its chunk
  const float scale = a.scale_log2e;
  const uint32_t stage0 = ptx::smem_u32(stages) + uint32_t(hc) * 2u;
  const uint32_t stage_b = uint32_t(pl.stage_bytes), half_b = uint32_t(half), row_u = uint32_t(row_b);
  const bool store = a.store != 0 && ks == 0;
  int st = 0;
  uint32_t ph = 0;
  auto dot8 = [&](const float (&q)[8], const uint4& kr) {
    const uint32_t w[4] = {kr.x, kr.y, kr.z, kr.w};
    float s0a = 0.f, s1a = 0.f;                      // two chains (even / odd channels)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      s0a = fmaf(q[2 * t], __uint_as_float(w[t] << 16), s0a);
      s1a = fmaf(q[2 * t + 1], __uint_as_float(w[t] & 0xffff0000u), s1a);
    }
    float sc = s0a + s1a;
#pragma unroll
    for (int off = LPK / 2; off > 0; off >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, off);
    return sc;
  };
  // the next stream's (q, k_t, v_t) chunks are loaded a stream ahead (their L2
  // latency, ~1 us, otherwise idles every warp at each stream's start)
  uint4 qn = make_uint4(0, 0, 0, 0), kn = qn, vn = qn;
  auto load_row = [&](int64_t b) {
    const __nv_bfloat16* qrow = a.qkv + b * 3 * E + hc;
    qn = *reinterpret_cast<const uint4*>(qrow);
    kn = *reinterpret_cast<const uint4*>(qrow + E);
    vn = *reinterpret_cast<const uint4*>(qrow + 2 * E);
  };
  if (lo < hi) load_row(lo);
  for (int64_t b = lo; b < hi; ++b) {
    float q[8];
    {
      const uint32_t w[4] = {qn.x, qn.y, qn.z, qn.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        q[2 * t] = __uint_as_float(w[t] << 16);
        q[2 * t + 1] = __uint_as_float(w[t] & 0xffff0000u);
      }
    }
    const uint4 kq = kn, vq = vn;
    if (b + 1 < hi) load_row(b + 1);
    float mx = kNegBig, l = 0.f, o[8];
    {                                               // this step's key, folded by subgroup 0
      const float sq = dot8(q, kq) * scale;          // (all lanes: the shuffles are warp-wide)
      const float sc = ks == 0 ? sq : -INFINITY;
      const float mn = fmaxf(mx, sc);
      const float e = exp2f(sc - mn);
      l = e;
      const uint32_t w[4] = {vq.x, vq.y, vq.z, vq.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        o[2 * t] = e * __uint_as_float(w[t] << 16);
        o[2 * t + 1] = e * __uint_as_float(w[t] & 0xffff0000u);
      }
      mx = mn;
    }
    int snew = s0;                                  // this step's slot relative to the current chunk
    for (int c = 0; c < nchunks; ++c, snew -= kc) {
      ptx::mbar_wait(&full[st], ph);
      const int kcnt = min(kc, n - c * kc);
      const uint32_t kst = stage0 + uint32_t(st) * stage_b;
      if (c == c0 && store) {                       // ring update: the chunk's copy has landed
        const int64_t off = (b * n + s0) * E + hc;
        *reinterpret_cast<uint4*>(a.kring + off) = kq;
        *reinterpret_cast<uint4*>(a.vring + off) = vq;
      }
      for (int k0 = ks; k0 < kcnt + ks; k0 += 2 * KPI) {   // (uniform trip count: k0 - ks < kcnt)
        const int ka = k0, kb = k0 + KPI;
        const bool va = ka < kcnt && ka != snew, vb = kb < kcnt && kb != snew;
        const uint32_t ra = kst + uint32_t(min(ka, kcnt - 1)) * row_u, rb = kst + uint32_t(min(kb, kcnt - 1)) * row_u;
        const uint4 kra = ptx::lds128(ra), krb = ptx::lds128(rb);
        const uint4 vra = ptx::lds128(ra + half_b), vrb = ptx::lds128(rb + half_b);
        float sa = dot8(q, kra) * scale, sb = dot8(q, krb) * scale;   // base-2 logits
        sa = va ? sa : -INFINITY;
        sb = vb ? sb : -INFINITY;
        const float mn = fmaxf(mx, fmaxf(sa, sb));
        const float cf = exp2f(mx - mn), ea = exp2f(sa - mn), eb = exp2f(sb - mn);
        l = fmaf(l, cf, ea + eb);
        const uint32_t wa[4] = {vra.x, vra.y, vra.z, vra.w}, wb[4] = {vrb.x, vrb.y, vrb.z, vrb.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          o[2 * t] = fmaf(eb, __uint_as_float(wb[t] << 16), fmaf(ea, __uint_as_float(wa[t] << 16), o[2 * t] * cf));
          o[2 * t + 1] = fmaf(eb, __uint_as_float(wb[t] & 0xffff0000u),
                              fmaf(ea, __uint_as_float(wa[t] & 0xffff0000u), o[2 * t + 1] * cf));
        }
        mx = mn;
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_relaxed(&empty[st]);   // the stage's reads are consumed
      if (++st == nst) { st = 0; ph ^= 1u; }
    }
    // merge the KPI key subgroups (lanes g, g + LPK, ...)
#pragma unroll
    for (int off = LPK; off < 32; off <<= 1) {
      const float mo = __shfl_xor_sync(0xffffffffu, mx, off);
      const float lo2 = __shfl_xor_sync(0xffffffffu, l, off);
      const float mn = fmaxf(mx, mo);
      const float c1 = exp2f(mx - mn), c2 = exp2f(mo - mn);   // both finite (>= -1e30): no inf - inf
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float oo = __shfl_xor_sync(0xffffffffu, o[t], off);
        o[t] = o[t] * c1 + oo * c2;
      }
      l = l * c1 + lo2 * c2;
      mx = mn;
    }
    if (ks == 0) {
      const float inv = 1.f / l;
      uint4 u;
      __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int t = 0; t < 4; ++t) hp[t] = __floats2bfloat162_rn(o[2 * t] * inv, o[2 * t + 1] * inv);
      *reinterpret_cast<uint4*>(a.out + b * E + hc) = u;
    }
  }
}

}  // namespace

bool mha_supported(int E, int heads) {
  if (heads < 1 || E % heads) return false;
  const int dh = E / heads;
  return dh == 32 || dh == 64 || dh == 128;
}

// keys per lane per iteration for dh = 64: 2 (default) keeps twice the K / V
// rows in flight per warp at 3 blocks per SM -- MHA step 106 -> 97 us; 4
// measured the same; CO_MHA_KU=1 restores one key (A/B, experiment builds).
// Each lane still folds its keys in index order, so all variants give identical results.
int ku() { return CO_EXP("CO_MHA_KU", 2); }

cudaError_t launch_mha_attend(const MhaArgs& a, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t warps = a.B * a.T * a.heads;
  const int64_t blocks = (warps + 7) / 8;
  // one wave of resident blocks looping over (row, head) warps: no partial tail wave
  auto grid_of = [&](const void* fn) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
    const int64_t cap = int64_t(sms) * (per_sm > 0 ? per_sm : 1);
    return int(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
  };
  auto launch = [&](auto fn) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(grid_of((const void*)fn)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = option(OPT_PDL) != 0 ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, a);
  };
  // step mode: the bulk-copy ring pipeline (option "mha_ring"), one consumer warp per head
  if (!a.batch && a.T == 1 && option(OPT_MHA_RING) != 0 && a.heads <= kMhaRingMaxHeads && a.B > 0) {
    MhaRingPlan pl{};
    const int row_b = a.E * 2;
    pl.kc = std::max(1, std::min(a.n, 16384 / row_b));           // <= 16 KB of K (and of V) per stage
    pl.nchunks = (a.n + pl.kc - 1) / pl.kc;
    pl.stage_bytes = 2 * pl.kc * row_b;
    pl.nst = 5;
    const size_t smem = size_t(pl.nst) * pl.stage_bytes + 2 * pl.nst * sizeof(uint64_t);
    auto launch_ring = [&](auto fn) {
      static size_t set_smem_dh[3] = {0, 0, 0};                    // per kernel instantiation (DH = 32, 64, 128)
      size_t& set_smem = set_smem_dh[a.E / a.heads / 64];
      if (smem > set_smem) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        set_smem = smem;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(unsigned(std::min<int64_t>(a.B, sms)));
      cfg.blockDim = dim3(unsigned(a.heads + 1) * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = option(OPT_PDL) != 0 ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      return cudaLaunchKernelEx(&cfg, fn, a, pl);
    };
    switch (a.E / a.heads) {
      case 32: return launch_ring(k_mha_attend_ring<32>);
      case 64: return launch_ring(k_mha_attend_ring<64>);
      case 128: return launch_ring(k_mha_attend_ring<128>);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.E / a.heads) {
    case 32: return launch(k_mha_attend<32>);
    case 64: return ku() == 1 ? launch(k_mha_attend<64>) : launch(k_mha_attend<64, 2>);
    case 128: return launch(k_mha_attend<128>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace co
