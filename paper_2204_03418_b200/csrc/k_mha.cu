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
#include <cstdio>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace co {


namespace {

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
  switch (a.E / a.heads) {
    case 32: return launch(k_mha_attend<32>);
    case 64: return ku() == 1 ? launch(k_mha_attend<64>) : launch(k_mha_attend<64, 2>);
    case 128: return launch(k_mha_attend<128>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace co
