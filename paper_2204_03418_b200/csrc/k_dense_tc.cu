// k_dense_tc.cu — K4: dense continual-convolution step on the 5th-generation
// tensor cores (sm_100a: tcgen05.mma + TMEM accumulators, operands staged by
// TMA), with the state read-accumulate-write, the emit and the ring rotation
// fused into the epilogue (BASELINE.json north_star "Dense step kernel").
//
// The step as an implicit GEMM:
//   M = output pixels of a tile (128 rows), N = kt * Cc (every temporal slice
//   of Cc output channels), K = kh * kw * Cin (spatial taps x input channels).
//   Column block k of the accumulator is the partial P_k = W[:,:,k] (*) x_t.
// Epilogue (row a4): y = S[slot(kt-1)] + P_{kt-1} + b (emitted when ready),
//   S[slot(k)] += P_k for 0 < k < kt-1, S[slot(0)] = P_0 (after the emit read).
//
// Design (B200-first):
//  * Persistent CTAs, one per SM.  Work item = (pixel tile, channel part);
//    the grid is a multiple of the number of parts, so a CTA always serves the
//    same part and keeps that part's packed weights resident in shared memory
//    for the whole launch (one bulk copy at start).
//  * A operand = the input halo of the tile, loaded by ONE TMA box per item
//    (zero fill at the image border = the spatial padding).  Shared memory holds
//    it as K-major "interleaved" core matrices ([channel group of 8][halo
//    pixel][16 B]); the operand of spatial tap (u, v) is the same buffer with
//    its start address shifted by (u * Wp + v) pixels (implicit im2col: no data
//    is duplicated).  Output rows are enumerated in the halo's padded width Wp,
//    the Wp - Wo junk columns are computed and discarded.
//  * Warp roles: warps 0 .. 4 EG-1 = EG epilogue warpgroups (warp w reads TMEM
//    lane quadrant w % 4), warp 4 EG = TMA producer, warp 4 EG + 1 = MMA issuer
//    (one thread) and TMEM owner.  The EG groups take items round-robin, each
//    with its own TMEM accumulator buffer, so the MMAs of later items overlap
//    the state traffic of earlier ones, and EG items' state loads are in
//    flight at once (the step is HBM-bound: the state RMW is ~80% of its bytes).
//    Epilogue threads issue the state loads of their item BEFORE waiting for
//    the accumulator.
//  * State layout S[slot][Cout/4][B*Ho*Wo][4] fp32: thread = output pixel, a
//    warp moves 512 contiguous bytes per float4 instruction.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dense_tc.cuh"
#include "tc_ptx.cuh"

namespace co {

namespace {

constexpr int kMaxStages = 4;   // A-operand pipeline depth: as many as fit in shared memory
__host__ __device__ constexpr int tc_threads(int eg) { return 32 * (4 * eg + 2); }
constexpr int kApad = 512;        // slack after each A stage (junk rows may read past the box)

struct TcParams {
  int B, H, W, Cin, Cout, Ho, Wo;
  int64_t HWo, plane;             // plane = B * HWo
  int kh, kw, ph, pw;
  int flat;                       // 1: 1x1 spatial, rows = (stream, pixel) flattened
  int MT, Wp, tiles_per_stream;   // halo mode geometry
  int64_t n_tiles, n_items;
  int n_split;
  int a_bytes, a_stride;          // A box bytes, A stage stride in smem
  int stages;                     // A pipeline depth (<= kMaxStages)
  int chunk_stride;               // bytes between 8-channel groups inside an A stage
  int w_bytes;                    // packed weights of one part
  int w_off;                      // A stages start here (1 KB aligned)
  int slot[kMaxKt];
  int emit, update, act, out_f32;
  int Cq;
  float* state;
  void* y;
  int64_t y_bstride;
  const __nv_bfloat16* wpack;     // [n_split][K/8][N][8]
  const float* bias;
};

__device__ __forceinline__ void bar_sync_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int KT, int CC, int EG>
__global__ void __launch_bounds__(tc_threads(EG), 1)
    k_step_dense_tc(const __grid_constant__ CUtensorMap tmap, const TcParams p) {
  constexpr int N = KT * CC;
  constexpr int BUF = (N <= 128) ? 128 : 256;
  static_assert(EG * BUF <= 512, "accumulator buffers exceed TMEM");
  constexpr int TMEM_COLS = 512;
  constexpr int kProducer = 4 * EG, kMma = 4 * EG + 1;
  static_assert(N % 16 == 0 && N <= 256, "invalid UMMA N");
  static_assert(CC % 16 == 0, "CC must be a multiple of 16");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* w_s = smem;                                  // [K/8][N][16 B]
  uint8_t* a_s = smem + p.w_off;                        // stages x a_stride
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_s + p.stages * p.a_stride);
  uint64_t* full = bars;                                // [kMaxStages]
  uint64_t* empty = bars + kMaxStages;                  // [kMaxStages]
  uint64_t* acc_full = bars + 2 * kMaxStages;           // [EG]
  uint64_t* acc_empty = bars + 2 * kMaxStages + EG;     // [EG]
  uint64_t* w_full = bars + 2 * kMaxStages + 2 * EG;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 2 * EG + 1);
  float* bias_s = reinterpret_cast<float*>(bars + 2 * kMaxStages + 2 * EG + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grid = gridDim.x;
  const int part = blockIdx.x % p.n_split;
  const int c0 = part * CC;                             // first output channel of this part

  if (warp == kProducer && lane == 0) {
    for (int s = 0; s < p.stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
    for (int e = 0; e < EG; ++e) { ptx::mbar_init(&acc_full[e], 1); ptx::mbar_init(&acc_empty[e], 128); }
    ptx::mbar_init(w_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == kMma) ptx::tmem_alloc(tmem_holder, TMEM_COLS);
  if (threadIdx.x < CC) bias_s[threadIdx.x] = p.bias[c0 + threadIdx.x];
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == kProducer) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::prefetch_tmap(&tmap);
      ptx::mbar_arrive_expect_tx(w_full, p.w_bytes);
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wpack) + size_t(part) * p.w_bytes;
      for (int off = 0; off < p.w_bytes; off += 32768) {
        const int n = min(32768, p.w_bytes - off);
        ptx::bulk_g2s(w_s + off, wsrc + off, n, w_full);
      }
      int s = 0;
      uint32_t ph = 0;
      for (int64_t item = blockIdx.x; item < p.n_items; item += grid) {
        ptx::mbar_wait(&empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], p.a_bytes);
        const int64_t tile = item / p.n_split;
        uint8_t* dst = a_s + s * p.a_stride;
        if (p.flat) {
          ptx::tma_load_3d(dst, &tmap, &full[s], 0, int(tile * 128), 0);
        } else {
          const int b = int(tile / p.tiles_per_stream);
          const int ho0 = int(tile % p.tiles_per_stream) * p.MT;
          ptx::tma_load_5d(dst, &tmap, &full[s], 0, -p.pw, ho0 - p.ph, 0, b);
        }
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  if (warp == kMma) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(128, N);
      ptx::mbar_wait(w_full, 0);
      const uint32_t a_base = ptx::smem_u32(a_s);
      // Descriptors are advanced by adding (byte offset >> 4) to their 14-bit
      // start-address field (shared memory < 256 KB, so it never carries out).
      const uint64_t b_desc0 = ptx::smem_desc(ptx::smem_u32(w_s), N * 16, 128);
      const int kc2 = p.Cin / 16;                       // MMAs (K = 16) per spatial tap
      const uint32_t chunk16 = uint32_t(p.chunk_stride) >> 3;   // 2 channel groups, in 16 B units
      int s = 0;
      uint32_t ph = 0;
      int e = 0;
      uint32_t eph = 0;
      for (int64_t item = blockIdx.x; item < p.n_items; item += grid) {
        ptx::mbar_wait(&acc_empty[e], eph ^ 1);
        ptx::tc_fence_after();
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(e * BUF);
        const uint64_t a_desc0 = ptx::smem_desc(a_base + uint32_t(s * p.a_stride), p.chunk_stride, 128);
        uint64_t bd = b_desc0;
        uint32_t acc = 0;
        for (int u = 0; u < p.kh; ++u) {
          for (int v = 0; v < p.kw; ++v) {
            uint64_t ad = a_desc0 + uint64_t(u * p.Wp + v);   // tap (u, v): shift by u Wp + v rows
            for (int kc = 0; kc < kc2; ++kc) {
              ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, acc);
              acc = 1;
              ad += chunk16;
              bd += uint64_t(2 * N);                         // 2 groups of N rows x 16 B
            }
          }
        }
        ptx::tc_commit(&empty[s]);      // A stage free once these MMAs retire
        ptx::tc_commit(&acc_full[e]);   // accumulator e ready for the epilogue
        if (++s == p.stages) { s = 0; ph ^= 1; }
        if (++e == EG) { e = 0; eph ^= 1; }
      }
    }
    __syncwarp();
    bar_sync_named(1, 32 + 128 * EG);
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, TMEM_COLS);
    return;
  }

  // ===================== epilogue warpgroups (warps 0 .. 4 EG - 1) =====================
  const int e = warp >> 2;                             // group = accumulator buffer
  const int q = warp & 3;                              // TMEM lane quadrant of this warp
  const int m = q * 32 + lane;                         // accumulator row = tile pixel
  const int64_t plane = p.plane;
  constexpr int NQ = CC / 4;                           // channel quads per thread
  constexpr int NS = (KT > 1) ? KT - 1 : 1;
  int li = e;
  for (int64_t item = blockIdx.x + int64_t(e) * grid; item < p.n_items; item += EG * int64_t(grid), li += EG) {
    const int j = li / EG;
    const int64_t tile = item / p.n_split;
    // ---- this row's output pixel
    bool valid;
    int64_t pix, b;
    if (p.flat) {
      pix = tile * 128 + m;
      valid = pix < plane;
      b = valid ? pix / p.HWo : 0;
    } else {
      b = tile / p.tiles_per_stream;
      const int ho = int(tile % p.tiles_per_stream) * p.MT + m / p.Wp;
      const int wo = m % p.Wp;
      valid = (m < p.MT * p.Wp) && (wo < p.Wo) && (ho < p.Ho);
      pix = b * p.HWo + int64_t(ho) * p.Wo + wo;
    }
    // ---- prefetch the state this pixel needs (before the accumulator is ready)
    float4 sv[NS][NQ];
    if (KT > 1 && valid) {
      if (p.emit) {
        const float4* src = reinterpret_cast<const float4*>(p.state) +
                            (int64_t(p.slot[KT - 1]) * p.Cq + c0 / 4) * plane + pix;
#pragma unroll
        for (int i = 0; i < NQ; ++i) sv[0][i] = __ldcs(src + int64_t(i) * plane);
      }
      if (p.update) {
#pragma unroll
        for (int k = 1; k < KT - 1; ++k) {
          if (p.slot[k] < 0) continue;
          const float4* src = reinterpret_cast<const float4*>(p.state) +
                              (int64_t(p.slot[k]) * p.Cq + c0 / 4) * plane + pix;
#pragma unroll
          for (int i = 0; i < NQ; ++i) sv[k][i] = __ldcs(src + int64_t(i) * plane);
        }
      }
    }
    ptx::mbar_wait(&acc_full[e], j & 1);
    ptx::tc_fence_after();
    const uint32_t t_row = tmem + (uint32_t(q * 32) << 16) + uint32_t(e * BUF);
    float v[16];
    // ---- (1) complete + emit
    if (p.emit) {
#pragma unroll
      for (int c = 0; c < CC; c += 16) {
        ptx::tmem_ld16(t_row + uint32_t((KT - 1) * CC + c), v);
        ptx::tc_wait_ld();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float s = 0.f;
            if (KT > 1) {
              const float4 t4 = sv[0][(c + i) >> 2];
              s = ((i & 3) == 0) ? t4.x : ((i & 3) == 1) ? t4.y : ((i & 3) == 2) ? t4.z : t4.w;
            }
            float r = v[i] + s + bias_s[c + i];
            v[i] = (p.act == 1 && r < 0.f) ? 0.f : r;
          }
          const int64_t yoff = b * p.y_bstride + (pix - b * p.HWo) * p.Cout + c0 + c;
          if (p.out_f32) {
            float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + yoff);
#pragma unroll
            for (int i = 0; i < 4; ++i) yp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
            uint4* yp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.y) + yoff);
#pragma unroll
            for (int i = 0; i < 2; ++i)
              yp[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                 pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
          }
        }
      }
    }
    if (p.update && KT > 1) {
      // ---- (2) accumulate into pending outputs
#pragma unroll
      for (int k = KT - 2; k >= 1; --k) {
        if (p.slot[k] < 0) continue;
        float4* dst = reinterpret_cast<float4*>(p.state) + (int64_t(p.slot[k]) * p.Cq + c0 / 4) * plane + pix;
#pragma unroll
        for (int c = 0; c < CC; c += 16) {
          ptx::tmem_ld16(t_row + uint32_t(k * CC + c), v);
          ptx::tc_wait_ld();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float4 t4 = sv[k][c / 4 + i];
              t4.x += v[4 * i]; t4.y += v[4 * i + 1]; t4.z += v[4 * i + 2]; t4.w += v[4 * i + 3];
              __stcs(dst + int64_t(c / 4 + i) * plane, t4);
            }
          }
        }
      }
      // ---- (3) start the newest output (overwrites the emitted slot)
      if (p.slot[0] >= 0) {
        float4* dst = reinterpret_cast<float4*>(p.state) + (int64_t(p.slot[0]) * p.Cq + c0 / 4) * plane + pix;
#pragma unroll
        for (int c = 0; c < CC; c += 16) {
          ptx::tmem_ld16(t_row + uint32_t(c), v);
          ptx::tc_wait_ld();
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              __stcs(dst + int64_t(c / 4 + i) * plane, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          }
        }
      }
    }
    ptx::tc_fence_before();
    ptx::mbar_arrive(&acc_empty[e]);
  }
  bar_sync_named(1, 32 + 128 * EG);
}

// ------------------------------------------------------------------ host side

__global__ void k_pack_tc_weights(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int Cout,
                                  int Cin, int kt, int kh, int kw, int CC, int n_split) {
  // (Cout, Cin, kt, kh, kw) -> [part][K/8][N][8], N = kt*CC rows (n = k*CC + c),
  // K index = (u*kw + v)*Cin + ci.
  const int64_t total = int64_t(Cout) * Cin * kt * kh * kw;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int64_t r = i;
  const int v = int(r % kw); r /= kw;
  const int u = int(r % kh); r /= kh;
  const int k = int(r % kt); r /= kt;
  const int ci = int(r % Cin); r /= Cin;
  const int o = int(r);
  const int part = o / CC, c = o % CC;
  const int N = kt * CC;
  const int64_t K = int64_t(Cin) * kh * kw;
  const int64_t kidx = int64_t(u * kw + v) * Cin + ci;
  const int n = k * CC + c;
  out[int64_t(part) * K * N + ((kidx / 8) * N + n) * 8 + (kidx % 8)] = w[i];
}

typedef void (*KernFn)(const CUtensorMap, const TcParams);

struct Variant {
  int KT, CC, EG;
  KernFn fn;
};

#define CO_TC_VARIANT(kt, cc, eg) {kt, cc, eg, (KernFn)k_step_dense_tc<kt, cc, eg>}
const Variant kVariants[] = {
    CO_TC_VARIANT(1, 32, 4), CO_TC_VARIANT(1, 64, 4), CO_TC_VARIANT(2, 32, 4), CO_TC_VARIANT(3, 16, 4),
    CO_TC_VARIANT(3, 32, 2), CO_TC_VARIANT(3, 32, 3), CO_TC_VARIANT(3, 32, 4), CO_TC_VARIANT(5, 16, 4),
    CO_TC_VARIANT(5, 32, 2), CO_TC_VARIANT(9, 16, 2),
};

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

struct Plan {
  bool ok = false;
  const Variant* var = nullptr;
  int n_split = 0, flat = 0, MT = 0, Wp = 0, tiles_per_stream = 0;
  int a_bytes = 0, a_stride = 0, chunk_stride = 0, w_bytes = 0, stages = 2;
  int64_t n_tiles = 0;
  size_t smem = 0;
};

constexpr size_t kSmemLimit = 227 * 1024;

Plan make_plan(const Geom& g) {
  Plan pl;
  if (g.in_dtype != BF16 || g.groups != 1 || g.Cin % 16 != 0 || g.Cin / 8 > 256) return pl;
  if (g.sh != 1 || g.sw != 1 || g.dh != 1 || g.dw != 1) return pl;
  if (g.Cout % 4 != 0) return pl;
  const bool flat = (g.kh == 1 && g.kw == 1 && g.ph == 0 && g.pw == 0);
  int Wp = 1, MT = 1, halo_rows = 1, a_rows = 128;
  if (!flat) {
    Wp = g.Wo + g.kw - 1;
    if (Wp > 128 || Wp > 256) return pl;
    MT = std::min(128 / Wp, g.Ho);
    halo_rows = MT + g.kh - 1;
    if (halo_rows > 256) return pl;
    a_rows = Wp * halo_rows;
  }
  const int a_bytes = (g.Cin / 8) * a_rows * 16;
  const int a_stride = ((a_bytes + kApad + 1023) / 1024) * 1024;
  const int64_t K = int64_t(g.Cin) * g.kh * g.kw;
  // largest CC (fewest parts) whose weights + A stages fit in shared memory;
  // among equal CC the most epilogue groups (CO_TC_EG=<n> pins it, for A/B runs)
  const char* eg_env = getenv("CO_TC_EG");
  const int eg_pin = eg_env ? atoi(eg_env) : 0;
  for (const Variant& v : kVariants) {
    if (v.KT != g.kt || g.Cout % v.CC != 0) continue;
    if (eg_pin && v.EG != eg_pin) continue;
    const int N = v.KT * v.CC;
    const int64_t w_bytes = int64_t(N) * K * 2;
    const size_t fixed = 1024 + size_t((w_bytes + 1023) / 1024 * 1024) + 256 + v.CC * 4;
    if (fixed + 2 * size_t(a_stride) > kSmemLimit) continue;
    const int stages = int(std::min<size_t>(kMaxStages, (kSmemLimit - fixed) / size_t(a_stride)));
    if (!pl.ok || v.CC > pl.var->CC || (v.CC == pl.var->CC && v.EG > pl.var->EG)) {
      pl.ok = true;
      pl.var = &v;
      pl.w_bytes = int(w_bytes);
      pl.stages = stages;
      pl.smem = fixed + size_t(stages) * a_stride;
    }
  }
  if (!pl.ok) return pl;
  pl.n_split = g.Cout / pl.var->CC;
  pl.flat = flat;
  pl.MT = MT;
  pl.Wp = Wp;
  pl.a_bytes = a_bytes;
  pl.a_stride = a_stride;
  pl.chunk_stride = a_rows * 16;
  if (flat) {
    pl.n_tiles = (g.B * g.HWo + 127) / 128;
  } else {
    pl.tiles_per_stream = (g.Ho + MT - 1) / MT;
    pl.n_tiles = g.B * pl.tiles_per_stream;
  }
  return pl;
}

}  // namespace

struct DenseTC {
  Plan pl;
  __nv_bfloat16* wpack = nullptr;
  float* xstage = nullptr;   // contiguous staging for strided clips in flat mode
  size_t xstage_bytes = 0;
  int num_sms = 148;
  std::string name;
};

bool dense_tc_supported(const Geom& g) { return make_plan(g).ok && get_encode() != nullptr; }

DenseTC* dense_tc_create(const Geom& g, const void* w_dev, std::string& err) {
  Plan pl = make_plan(g);
  if (!pl.ok) { err = "unsupported shape"; return nullptr; }
  if (!get_encode()) { err = "cuTensorMapEncodeTiled unavailable"; return nullptr; }
  DenseTC* t = new DenseTC();
  t->pl = pl;
  const int64_t total = int64_t(g.Cout) * g.Cin * g.kt * g.kh * g.kw;
  cudaError_t e = cudaMalloc(&t->wpack, size_t(total) * 2);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); delete t; return nullptr; }
  k_pack_tc_weights<<<unsigned((total + 255) / 256), 256>>>(static_cast<const __nv_bfloat16*>(w_dev), t->wpack,
                                                           g.Cout, g.Cin, g.kt, g.kh, g.kw, pl.var->CC, pl.n_split);
  if ((e = cudaGetLastError()) != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
  e = cudaFuncSetAttribute(pl.var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pl.smem));
  if (e != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, dev);
  char buf[96];
  snprintf(buf, sizeof(buf), "k_step_dense_tc<%d,%d,%d>", pl.var->KT, pl.var->CC, pl.var->EG);
  if (getenv("CO_LOG")) fprintf(stderr, "[co] %s: %d parts, %lld tiles, A stages %d x %d B, smem %zu B\n", buf,
                                pl.n_split, (long long)pl.n_tiles, pl.stages, pl.a_stride, pl.smem);
  t->name = buf;
  return t;
}

void dense_tc_destroy(DenseTC* t) {
  if (!t) return;
  cudaFree(t->wpack);
  cudaFree(t->xstage);
  delete t;
}

const char* dense_tc_name(const DenseTC* t) { return t->name.c_str(); }

cudaError_t dense_tc_step(DenseTC* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s) {
  const Plan& pl = t->pl;
  const void* x = a.x;
  int64_t x_bstride = a.x_bstride;
  const int64_t frame = int64_t(g.H) * g.W * g.Cin;
  if (!x || (pl.flat && x_bstride != frame)) {
    // zero frame (pad_end) or a strided clip column in flat mode: stage it densely
    const size_t need = size_t(g.B) * frame * 2;
    if (t->xstage_bytes < need) {
      cudaFree(t->xstage);
      cudaError_t e = cudaMalloc(&t->xstage, need);
      if (e != cudaSuccess) return e;
      t->xstage_bytes = need;
    }
    cudaError_t e = x ? cudaMemcpy2DAsync(t->xstage, frame * 2, x, x_bstride * 2, frame * 2, g.B,
                                          cudaMemcpyDeviceToDevice, s)
                      : cudaMemsetAsync(t->xstage, 0, need, s);
    if (e != cudaSuccess) return e;
    x = t->xstage;
    x_bstride = frame;
  }
  CUtensorMap map;
  CUresult r;
  auto encode = get_encode();
  if (pl.flat) {
    cuuint64_t dims[3] = {8, cuuint64_t(g.B * g.HWo), cuuint64_t(g.Cin / 8)};
    cuuint64_t strides[2] = {cuuint64_t(g.Cin) * 2, 16};
    cuuint32_t box[3] = {8, 128, cuuint32_t(g.Cin / 8)};
    cuuint32_t es[3] = {1, 1, 1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[5] = {8, cuuint64_t(g.W), cuuint64_t(g.H), cuuint64_t(g.Cin / 8), cuuint64_t(g.B)};
    cuuint64_t strides[4] = {cuuint64_t(g.Cin) * 2, cuuint64_t(g.W) * g.Cin * 2, 16, cuuint64_t(x_bstride) * 2};
    cuuint32_t box[5] = {8, cuuint32_t(pl.Wp), cuuint32_t(pl.MT + g.kh - 1), cuuint32_t(g.Cin / 8), 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;

  TcParams p{};
  p.B = int(g.B); p.H = g.H; p.W = g.W; p.Cin = g.Cin; p.Cout = g.Cout; p.Ho = g.Ho; p.Wo = g.Wo;
  p.HWo = g.HWo; p.plane = g.B * g.HWo;
  p.kh = g.kh; p.kw = g.kw; p.ph = g.ph; p.pw = g.pw;
  p.flat = pl.flat; p.MT = pl.MT; p.Wp = pl.Wp; p.tiles_per_stream = pl.tiles_per_stream;
  p.n_tiles = pl.n_tiles; p.n_split = pl.n_split; p.n_items = pl.n_tiles * pl.n_split;
  p.a_bytes = pl.a_bytes; p.a_stride = pl.a_stride; p.stages = pl.stages; p.chunk_stride = pl.chunk_stride; p.w_bytes = pl.w_bytes;
  p.w_off = (pl.w_bytes + 1023) / 1024 * 1024;
  for (int k = 0; k < kMaxKt; ++k) p.slot[k] = a.slot[k];
  p.emit = a.emit; p.update = a.update; p.act = g.act; p.out_f32 = (g.out_dtype == F32);
  p.Cq = g.Cq;
  p.state = a.state;
  p.y = a.y;
  p.y_bstride = a.y_bstride;
  p.wpack = t->wpack;
  p.bias = bias;
  const int per = t->num_sms / pl.n_split;
  const int64_t grid = std::min<int64_t>(per, pl.n_tiles) * pl.n_split;
  void* args[] = {&map, &p};
  return cudaLaunchKernel(reinterpret_cast<const void*>(pl.var->fn), dim3(unsigned(grid)),
                          dim3(tc_threads(pl.var->EG)), args, pl.smem, s);
}

}  // namespace co
