// k_stem_raw.cu — RAW-ring step of a small-Cin stem on the 5th-generation
// tensor cores (sm_100a: tcgen05.mma, TMEM accumulators, bulk copies).
//
// What it computes (SPEC S:227, S:239 raw-input ring; PAPER P:56 continual
// conv, Eq. 1 over the kt frames of the window): on a Ready step
//   y[b, ho, wo, o] = bias[o] + sum_{k, u, v, c} W[o, c, k, u, v]
//                     * frame_k[b, ho sh + u - ph, wo sw + v - pw, c]
// where frame_k is ring slot slot[k] (the frame i s + k dil of output i; the
// newest frame, k = kt - 1, was stored by the host) -- the full window
// contraction of the layer, with no partial-sum state.  For an RGB stem the
// RAW ring moves ~8x fewer bytes than the fp32 partial-sum ring (C4 layer 1:
// 0.85 MB against 6.9 MB per stream-step) at the same tensor-core work.
//
// Design (B200-first):
//  * Implicit GEMM per 128-row tile (TH output rows x Wp row slots of one
//    stream): M = 128, N = Cout (the whole layer), K = kt * kh * Kp.
//  * Channel-padded rows ARE the A operand.  A raw row is kept in shared memory
//    with every pixel padded to CP = 8 / sw channels (16 / sw bytes), so output
//    pixel wo's window (pixels wo sw - pw .. + kw - 1) starts exactly 16 B
//    after wo - 1's: the row read as a K-major no-swizzle matrix with row
//    stride 16 B, K-group stride (LBO) 16 B and 8-row stride (SBO) 128 B is the
//    im2col of one row tap -- K index v CP + c, Kp = kw CP rounded up to 16,
//    weights zero for v >= kw or c >= Cin.  Rows are stored by row phase (q mod
//    sh) with pitch Wp * 16 B (Wp >= Wo row slots: wide enough for the last
//    window and the data), so the TH output rows of a tile continue the same
//    descriptor, and row tap u is ONE shifted descriptor (phase u mod sh, first
//    row u div sh).  Nothing is duplicated: a frame row costs 16/sw B per pixel.
//  * The B operand (all packed weights, [K/8][N][16 B]) stays resident in
//    shared memory for the launch: the K loop streams only raw input rows.
//  * Per (tile, temporal tap k) the producer bulk-copies the (TH-1) sh + kh raw
//    rows of ring slot slot[k] the tile needs (C4: 9 rows of 672 B, ONE copy:
//    they are contiguous in the frame) and an expander group pads them (3 -> 4
//    channels, zero halo / padding) into an image of the ring; the MMA warp
//    issues kh * Kp / 16 MMAs per image from a descriptor table built once.
//  * CTA pairs (cta_group::2): each CTA builds the images of its own 128-row
//    tile and holds half of the weight rows; the leader issues M = 256 MMAs
//    over both -- at N = 64 an MMA instruction, not its MACs, sets the pace
//    (scripts/mma_probe.cu: ~44 cycles for 256 rows on a pair, ~49 for 128 on
//    one CTA).  The peer's images reach the leader through ONE cluster-scope
//    release per tile (a relay in the peer's idle MMA warp; a cluster-scope
//    release costs a GPU-wide membar), the image ring holding two tiles.
//  * Warp roles (26 warps): 0-7 epilogue (two groups taking alternate tiles:
//    y = acc + bias, ReLU, bf16 / fp32 stores), 8-23 expanders (four groups,
//    images round-robin), 24 producer, 25 MMA issuer (leader) / relay (peer) /
//    TMEM owner.  Images, raw-row buffers and TMEM accumulators are rings with
//    full / empty mbarriers.
#include <algorithm>
#include <cstdio>

#include "stem_raw.cuh"
#include "tc_ptx.cuh"

namespace co {
namespace {

constexpr int kNI = 10;          // image ring: two tiles of kt <= 5 images in flight (the pair relays per tile)
constexpr int kNR = 4;           // raw-row ring
constexpr int kEpiWarps = 8;     // two epilogue groups of 4 warps (alternate tiles)
constexpr int kExpGroups = 4;    // expander groups of 4 warps (images round-robin)
constexpr int kExpWarps = 4 * kExpGroups;
constexpr int kThreads = 32 * (kEpiWarps + kExpWarps + 2);
constexpr int kProducer = kEpiWarps + kExpWarps, kMma = kProducer + 1;
constexpr size_t kSmemLimit = 227 * 1024;

struct SrParams {
  const __nv_bfloat16* ring;     // [f+1][B][H][W][Cin]
  int64_t slot_elems, frame_elems;
  int slot[kMaxKt];
  int kt, kh, sh, ph, pw, Cin, H, W, Ho, Wo, Cout;
  int Kp;
  int TH, tiles_h, Wp;
  int64_t n_tiles;
  int nraw, rpitch, pad, img_rows;
  int base0, base1;              // first 16-B row of each row phase in an image
  int w_bytes, img_off, img_bytes, raw_off, raw_bytes, bias_off, bar_off, tab_off;
  void* y;
  int64_t y_bstride;
  int out_f32, act;
  const __nv_bfloat16* wpack;    // [PAIR][K/8][N/PAIR][8]: CTA rank r's half of the weight rows
  const float* bias;
  int dbg;                       // experiment builds only: 1 no expansion, 2 no MMAs, 4 no raw loads, 8 no work,
                                 // 64 no y stores, 128 no epilogue TMEM reads, 512 print per-role wait cycles
};
#ifdef CO_EXPERIMENTS
#define SDBG(bits) (p.dbg & (bits))
#define TWAIT(bar, par, acc)                      \
  {                                               \
    const long long t0_ = clock64();              \
    ptx::mbar_wait(bar, par);                     \
    acc += clock64() - t0_;                       \
  }
#else
#define SDBG(bits) (0)
#define TWAIT(bar, par, acc) ptx::mbar_wait(bar, par)
#endif

// position in a ring of n buffers: index and phase parity, advanced without division
struct Ring {
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int n) {
    if (++i == n) { i = 0; ph ^= 1u; }
  }
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// PER > 0: compile-time MMAs per image (kh Kp / 16; C4's stem: 7 x 2), the
// image's A descriptors held in registers and the issue loop unrolled.
// PAIR = 2: a CTA pair (cluster of 2, cta_group::2) -- each CTA builds the image
// of its own 128-row tile and holds half of the weight rows; the leader issues
// M = 256 MMAs over both.  At N = 64 an MMA instruction costs ~44 cycles for 256
// rows on a pair against ~49 for 128 rows on one CTA (scripts/mma_probe.cu): a
// small-N contraction is bound by MMA instructions, not by MACs.
template <int N, int SW, int PER, int PAIR>
__global__ void __launch_bounds__(kThreads, 1) k_step_stem_raw(const __grid_constant__ SrParams p) {
  constexpr int NBUF = 4;                              // TMEM accumulators: 2 per epilogue group
  constexpr int CP = 8 / SW;                            // padded channels per pixel (16 / SW bytes)
  constexpr int NB = N / PAIR;                          // weight rows held by this CTA
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* w_s = smem;
  uint8_t* img = smem + p.img_off;
  uint8_t* raw = smem + p.raw_off;
  float* bias_s = reinterpret_cast<float*>(smem + p.bias_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bar_off);
  uint64_t* w_full = bars;
  uint64_t* w_peer = bars + 1;                          // PAIR: the peer's weight half landed (leader)
  uint64_t* raw_full = bars + 2;
  uint64_t* raw_empty = raw_full + kNR;
  uint64_t* img_full = raw_empty + kNR;                 // PAIR: the leader's copy collects both CTAs
  uint64_t* img_empty = img_full + kNI;
  uint64_t* acc_full = img_empty + kNI;
  uint64_t* acc_empty = acc_full + NBUF;                // PAIR: the leader's copy collects both CTAs
  uint64_t* peer_tile = acc_empty + NBUF;               // PAIR leader: [2] the peer's images of tile T built
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(peer_tile + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR == 2 ? ptx::cluster_ctarank() : 0u;   // (before the barrier init: it uses rank)
  const bool leader = rank == 0;
  // arrive on the leader CTA's copy of a barrier (the pair's MMA issuer waits there)
  auto arrive_leader = [&](uint64_t* bar) {
    if constexpr (PAIR == 2) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(bar), 0));
    else ptx::mbar_arrive(bar);
  };
  if (warp == kProducer && lane == 0) {
    ptx::mbar_init(w_full, 1);
    ptx::mbar_init(w_peer, 1);
    for (int r = 0; r < kNR; ++r) { ptx::mbar_init(&raw_full[r], 1); ptx::mbar_init(&raw_empty[r], 4); }
    // img_full: the CTA's 4 expander warps of the image (CTA-scope arrivals);
    // peer_tile: on a pair leader, the peer's relay -- one cluster-scope arrival
    // per tile once all of the peer's images of the tile are built
    for (int i = 0; i < kNI; ++i) { ptx::mbar_init(&img_full[i], 4); ptx::mbar_init(&img_empty[i], 1); }
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&peer_tile[i], 1);
    for (int e = 0; e < NBUF; ++e) { ptx::mbar_init(&acc_full[e], 1); ptx::mbar_init(&acc_empty[e], 4 * PAIR); }
    ptx::fence_mbar_init();
  }
  if (warp == kMma) {
    if constexpr (PAIR == 2) ptx::tmem_alloc_pair(tmem_holder, 512);
    else ptx::tmem_alloc(tmem_holder, 512);
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) bias_s[i] = p.bias[i];
  // zero the images once: their slack past the last row is read (times zero
  // weights, or by junk rows) and must hold finite values
  for (int i = threadIdx.x; i < kNI * p.img_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(img)[i] = make_uint4(0u, 0u, 0u, 0u);
  // and the raw buffers: the bulk copies write only the rows' data bytes, the
  // zeros around them are the horizontal padding
  for (int i = threadIdx.x; i < kNR * p.raw_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(raw)[i] = make_uint4(0u, 0u, 0u, 0u);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  if constexpr (PAIR == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // work units: a CTA (PAIR 1) or a pair; unit u's T-th tile pair is u + T n_units,
  // and CTA `rank` of the unit takes tile (u + T n_units) PAIR + rank (the peer of
  // an odd last tile runs a dummy: no rows, no stores, same barriers)
  const int n_units = gridDim.x / PAIR, unit = blockIdx.x / PAIR;
  const int n_tiles = SDBG(8) ? 0 : int(p.n_tiles);     // < 2^31 (stem_raw_plan)
  const int n_groups = (n_tiles + PAIR - 1) / PAIR;     // tile pairs
  auto tile_of = [&](int T) { return (unit + T * n_units) * PAIR + int(rank); };
  auto has = [&](int T) { return unit + T * n_units < n_groups; };
  long long tw0 = 0, tw1 = 0;                             // experiment builds: cycles spent waiting
  const long long tstart = clock64();
  (void)tstart; (void)tw0; (void)tw1;

  if (warp == kProducer) {
    // ===================== producer: resident weights, then raw rows per (tile, k) =====================
    if (lane == 0) {
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wpack) + size_t(rank) * p.w_bytes;
      ptx::mbar_arrive_expect_tx(w_full, uint32_t(p.w_bytes));
      for (int off = 0; off < p.w_bytes; off += 32768)
        ptx::bulk_g2s(w_s + off, wsrc + off, uint32_t(std::min(32768, p.w_bytes - off)), w_full);
      if (PAIR == 2 && !leader) {                        // tell the leader this half landed
        ptx::mbar_wait(w_full, 0);
        arrive_leader(w_peer);
      }
      const int rowbytes = p.W * p.Cin * 2;
      Ring rr;
      for (int T = 0; has(T); ++T) {
        const int tile = tile_of(T);
        const int b = tile / p.tiles_h;
        const int r0 = (tile - b * p.tiles_h) * p.TH * p.sh - p.ph;
        const int lo = max(0, -r0), hi = tile < n_tiles ? min(p.nraw, p.H - r0) : 0;
        const __nv_bfloat16* fb = p.ring + int64_t(b) * p.frame_elems + int64_t(r0) * p.W * p.Cin;
        for (int k = 0; k < p.kt; ++k, rr.next(kNR)) {
          const int rb = rr.i;
          TWAIT(&raw_empty[rb], rr.ph ^ 1u, tw0);
          if (hi <= lo || SDBG(4)) { ptx::mbar_arrive(&raw_full[rb]); continue; }
          // the tile's in-frame rows are contiguous in the frame: one bulk copy
          ptx::mbar_arrive_expect_tx(&raw_full[rb], uint32_t((hi - lo) * rowbytes));
          const __nv_bfloat16* src = fb + int64_t(p.slot[k]) * p.slot_elems + int64_t(lo) * p.W * p.Cin;
          ptx::bulk_g2s(raw + rb * p.raw_bytes + p.pad * 2 + lo * rowbytes, src, uint32_t((hi - lo) * rowbytes),
                        &raw_full[rb]);
        }
      }
    }
  } else if (warp >= kEpiWarps && warp < kEpiWarps + kExpWarps) {
    // ===================== expanders: raw rows -> channel-padded phase rows =====================
    // 16-B chunk t of image row q holds the SW pixels x = t SW + i - pw, CP channels
    // each.  Raw rows sit back to back in shared memory (one bulk copy) after pad
    // zero elements; a pixel outside the frame row is zeroed by a per-thread mask
    // (a thread keeps its column slot t).  Thread = (column slot t, row group):
    // the rows of a thread's column are independent (unrolled).  Group g (4 warps)
    // builds images j = g, g + kExpGroups, ...
    const int g = (warp - kEpiWarps) >> 2;
    const int ct = threadIdx.x - 32 * kEpiWarps - 128 * g;
    const int cols = p.Wp <= 64 ? 64 : 128, ngroups = 128 / cols;
    const int t = ct % cols, qg = ct / cols;
    const bool fast3 = SW == 2 && p.Cin == 3;              // RGB at stride 2: word loads + byte permutes
    // element of the first pixel of chunk t in a padded raw row, and its word / parity
    const int e0 = p.pad + (t * SW - p.pw) * p.Cin;
    const int rowel = p.W * p.Cin;                          // elements per raw row
    bool pin[SW];                                           // pixel i of this column inside the frame row
#pragma unroll
    for (int i = 0; i < SW; ++i) pin[i] = t * SW + i - p.pw >= 0 && t * SW + i - p.pw < p.W;
    Ring ri, rr;                                         // image / raw-buffer position of image j
    int j = 0;                                           // image index of (tile, k) in this CTA
    for (int T = 0; has(T); ++T) {
      const int tile = tile_of(T);
      const int r0 = (tile % p.tiles_h) * p.TH * p.sh - p.ph;
      const bool real = tile < n_tiles;
      for (int k = 0; k < p.kt; ++k, ++j, ri.next(kNI), rr.next(kNR)) {
        if (j % kExpGroups != g) continue;
        const int ib = ri.i, rb = rr.i;
        TWAIT(&img_empty[ib], ri.ph ^ 1u, tw0);          // the MMAs of image j - kNI are done
        TWAIT(&raw_full[rb], rr.ph, tw1);                // image j's raw rows landed
        uint4* im = reinterpret_cast<uint4*>(img + ib * p.img_bytes);
        const uint8_t* rw0 = raw + rb * p.raw_bytes;
        if (t < p.Wp && !SDBG(1)) {
#pragma unroll 3
          for (int q = qg; q < p.nraw; q += ngroups) {
            const bool odd = p.sh == 2 && (q & 1);
            const int row = (odd ? p.base1 : p.base0) + (p.sh == 2 ? (q >> 1) : q) * p.Wp + t;
            uint4 o = make_uint4(0u, 0u, 0u, 0u);
            if (real && r0 + q >= 0 && r0 + q < p.H) {
              if (fast3) {
                // pixels a, b = 6 elements from e0: 4 words from the even boundary, then
                // (a0 a1) (a2 0) (b0 b1) (b2 0)
                const uint32_t* rw = reinterpret_cast<const uint32_t*>(rw0) + ((e0 + q * rowel) >> 1);
                uint32_t v0 = rw[0], v1 = rw[1], v2 = rw[2];
                if (e0 & 1) {
                  const uint32_t v3 = rw[3];
                  v0 = __byte_perm(v0, v1, 0x5432); v1 = __byte_perm(v1, v2, 0x5432); v2 = __byte_perm(v2, v3, 0x5432);
                }
                o = make_uint4(pin[0] ? v0 : 0u, pin[0] ? (v1 & 0xFFFFu) : 0u,
                               pin[SW - 1] ? __byte_perm(v1, v2, 0x5432) : 0u, pin[SW - 1] ? (v2 >> 16) : 0u);
              } else {
                const uint16_t* rr16 = reinterpret_cast<const uint16_t*>(rw0) + e0 + q * rowel;
                uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int i = 0; i < SW; ++i)
#pragma unroll
                  for (int c = 0; c < CP; ++c)
                    if (c < p.Cin && pin[i]) {
                      const uint32_t h = rr16[i * p.Cin + c];
                      const int e = i * CP + c;                 // element of the 16-B chunk
                      w[e >> 1] |= (e & 1) ? (h << 16) : h;
                    }
                o = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
            im[row] = o;
          }
        }
        ptx::fence_proxy_async();                         // generic image writes -> tensor-core reads
        __syncwarp();                                     // the warp's writes and fences, then one arrival
        if (lane == 0) {
          ptx::mbar_arrive(&raw_empty[rb]);
          ptx::mbar_arrive(&img_full[ib]);              // CTA scope (a cluster-scope release costs a GPU membar)
        }
      }
    }
  } else if (warp == kMma) {
    // ===================== MMA issuer (the leader CTA of a pair) =====================
    // The A descriptors of every (image buffer, row tap, K16 step) are built once
    // into a shared table (runtime-divisor math in the issue loop would make the
    // single issuing thread, not the tensor core, the bottleneck); B advances by
    // one K16 step (2 K groups x NB rows x 16 B) per MMA.  A: row stride 16 B,
    // LBO 16 B (the next K group is the next 8 channels of the same row), SBO 128 B.
    // A pair MMA reads the same shared offsets in both CTAs: each its own image
    // (its 128 rows) and its half of the weight rows.
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128 * PAIR, N);
    const int nk = p.Kp / 16;                             // MMAs (K = 16) per row tap
    const int per_img = p.kh * nk;
    uint64_t* atab = reinterpret_cast<uint64_t*>(smem + p.tab_off);
    {
      const uint32_t img_base = ptx::smem_u32(img);
      for (int i = lane; i < kNI * per_img; i += 32) {
        const int ib = i / per_img, u = (i % per_img) / nk, jj = i % nk;
        const uint32_t row0 = uint32_t(((u % p.sh) ? p.base1 : p.base0) + (u / p.sh) * p.Wp);
        atab[i] = ptx::smem_desc(img_base + uint32_t(ib * p.img_bytes) + row0 * 16u + uint32_t(jj) * 32u, 16u, 128u);
      }
    }
    __syncwarp();
    uint64_t a0[PER > 0 ? PER : 1];
    if constexpr (PER > 0) {
#pragma unroll
      for (int i = 0; i < PER; ++i) a0[i] = atab[i];      // image buffer 0
    }
    (void)a0;
    if (PAIR == 2 && !leader) {
      // relay: once all of this CTA's images of tile T are built (its expanders'
      // CTA-scope releases, acquired here), ONE cluster-scope release on the
      // leader's peer_tile[T mod 2] carries them (cumulativity) to the leader's
      // MMAs, which read them -- a cluster-scope release costs a GPU-wide membar,
      // so once per tile, not per image (the image ring holds two tiles)
      Ring ri;
      for (int T = 0; has(T); ++T) {
        for (int k = 0; k < p.kt; ++k, ri.next(kNI)) ptx::mbar_wait(&img_full[ri.i], ri.ph);
        if (lane == 0) arrive_leader(&peer_tile[T & 1]);
        __syncwarp();
      }
    }
    if (leader) {
      ptx::mbar_wait(w_full, 0);
      if constexpr (PAIR == 2) ptx::mbar_wait_cluster(w_peer, 0);
      ptx::tc_fence_after();
      const uint64_t bd0 = ptx::smem_desc(ptx::smem_u32(w_s), uint32_t(NB * 16), 128);
      const uint64_t bstep = uint64_t(2 * NB);            // one K16 step, 16-B units
      auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc) {
        if constexpr (PAIR == 2) ptx::mma_bf16_ss_pair(d, ad, bd, idesc, acc);
        else ptx::mma_bf16_ss(d, ad, bd, idesc, acc);
      };
      auto commit = [&](uint64_t* bar) {
        if constexpr (PAIR == 2) ptx::tc_commit_pair(bar, 0x3);   // both CTAs' copies
        else ptx::tc_commit(bar);
      };
      Ring re, ri;
      for (int T = 0; has(T); ++T) {
        const int e = re.i;
        if constexpr (PAIR == 2) ptx::mbar_wait_cluster(&acc_empty[e], re.ph ^ 1u);
        else TWAIT(&acc_empty[e], re.ph ^ 1u, tw0);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(e * N);
        if constexpr (PAIR == 2) ptx::mbar_wait_cluster(&peer_tile[T & 1], uint32_t(T >> 1) & 1u);   // peer's images
        uint64_t bd = bd0;
        for (int k = 0; k < p.kt; ++k, ri.next(kNI)) {
          const int ib = ri.i;
          TWAIT(&img_full[ib], ri.ph, tw1);               // this CTA's image
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if constexpr (PER > 0) {
              const uint64_t off = uint64_t(ib) * uint64_t(p.img_bytes >> 4);   // start-address field only
#pragma unroll
              for (int i = 0; i < PER; ++i)
                if (!SDBG(2)) mma(d_tmem, a0[i] + off, bd + uint64_t(i) * bstep, (k | i) ? 1u : 0u);
            } else {
              const uint64_t* at = atab + ib * per_img;
#pragma unroll 2
              for (int i = 0; i < per_img; ++i)
                if (!SDBG(2)) mma(d_tmem, at[i], bd + uint64_t(i) * bstep, (k | i) ? 1u : 0u);
            }
            commit(&img_empty[ib]);                       // image free once these MMAs completed
          }
          __syncwarp();
          bd += uint64_t(per_img) * bstep;
        }
        if (ptx::elect_one()) commit(&acc_full[e]);
        __syncwarp();
        re.next(NBUF);
      }
    }
  } else if (warp < kEpiWarps) {
    // ===================== epilogue: y = acc + bias (ReLU), bf16 / fp32 =====================
    // group eg (4 warps) takes the CTA's tiles T = eg, eg + 2, ...: accumulators eg, eg + 2
    const int eg = warp >> 2;
    const int m = (warp & 3) * 32 + lane;                 // accumulator row = tile row slot
    const int r = m / p.Wp, wo = m - (m / p.Wp) * p.Wp;
    Ring re;                                             // over this group's 2 accumulators
    for (int T = eg; has(T); T += 2) {
      const int tile = tile_of(T);
      const int b = tile / p.tiles_h;
      const int ho = (tile - b * p.tiles_h) * p.TH + r;
      const bool valid = tile < n_tiles && r < p.TH && wo < p.Wo && ho < p.Ho;
      const int e = eg + 2 * re.i;
      TWAIT(&acc_full[e], re.ph, tw0);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(e * N);
      const int64_t yoff = int64_t(b) * p.y_bstride + (int64_t(ho) * p.Wo + wo) * p.Cout;
#pragma unroll 1
      for (int c = 0; c < N; c += 16) {
        float v[16] = {};
        if (!SDBG(128)) ptx::tmem_ld16(t_row + uint32_t(c), v);
        ptx::tc_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          v[i] += bias_s[c + i];
          if (p.act == 1) v[i] = fmaxf(v[i], 0.f);
        }
        if (p.out_f32) {
          float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + yoff + c);
          if (valid && !SDBG(64)) {
#pragma unroll
            for (int i = 0; i < 4; ++i) yp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          }
        } else {
          uint4 h[2];
#pragma unroll
          for (int i = 0; i < 2; ++i)
            h[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                              pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
          // lanes 2k / 2k+1 swap halves so each store instruction writes whole 32-B sectors
          __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(p.y);
          const bool odd = lane & 1;
          const uint4 give = odd ? h[0] : h[1];
          uint4 got;
          got.x = __shfl_xor_sync(0xffffffffu, give.x, 1);
          got.y = __shfl_xor_sync(0xffffffffu, give.y, 1);
          got.z = __shfl_xor_sync(0xffffffffu, give.z, 1);
          got.w = __shfl_xor_sync(0xffffffffu, give.w, 1);
          const int64_t poff = __shfl_xor_sync(0xffffffffu, (long long)(yoff + c), 1);
          const bool pvalid = __shfl_xor_sync(0xffffffffu, int(valid), 1) != 0;
          if (SDBG(64)) continue;
          if (odd ? pvalid : valid) *reinterpret_cast<uint4*>(yb + (odd ? poff + 8 : yoff + c)) = odd ? got : h[0];
          if (odd ? valid : pvalid) *reinterpret_cast<uint4*>(yb + (odd ? yoff + c + 8 : poff)) = odd ? h[1] : got;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // every tcgen05.ld above was waited on: a relaxed arrive suffices (the y
        // stores need no ordering with the MMA warp)
        if constexpr (PAIR == 2) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&acc_empty[e]), 0));
        else ptx::mbar_arrive_relaxed(&acc_empty[e]);
      }
      re.next(2);
    }
  }
#ifdef CO_EXPERIMENTS
  if (SDBG(512) && blockIdx.x < 2 && lane == 0 && (warp == 0 || warp == kEpiWarps || warp == kProducer || warp == kMma))
    printf("cta %d warp %2d total %lld wait0 %lld wait1 %lld\n", blockIdx.x, warp, clock64() - tstart, tw0, tw1);
#endif
  ptx::tc_fence_before();
  if constexpr (PAIR == 2) ptx::cluster_sync(); else __syncthreads();   // no CTA leaves while its peer may signal it
  if (warp == kMma) {
    ptx::tc_fence_after();
    if constexpr (PAIR == 2) ptx::tmem_dealloc_pair(tmem, 512);
    else ptx::tmem_dealloc(tmem, 512);
  }
}

// (Cout, Cin, kt, kh, kw) bf16 -> [PAIR][K/8][N/PAIR][8], K index (k kh + u) Kp +
// v CP + c (zero for v >= kw or c >= Cin); output channel o lives in half o / (N / PAIR)
__global__ void k_pack_stem_raw(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int N, int Cin,
                                int kt, int kh, int kw, int Kp, int CP, int pair) {
  const int64_t K = int64_t(kt) * kh * Kp;
  const int64_t total = K * N;
  const int NB = N / pair;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kidx = i / N;
    const int o = int(i % N);
    const int j = int(kidx % Kp);
    const int u = int((kidx / Kp) % kh), k = int(kidx / (int64_t(Kp) * kh));
    const int v = j / CP, c = j % CP;
    __nv_bfloat16 val = __float2bfloat16_rn(0.f);
    if (v < kw && c < Cin) val = w[(((int64_t(o) * Cin + c) * kt + k) * kh + u) * kw + v];
    const int half = o / NB, oo = o % NB;
    out[((int64_t(half) * (K / 8) + kidx / 8) * NB + oo) * 8 + (kidx % 8)] = val;
  }
}

using SrFn = void (*)(SrParams);
constexpr int kPair = 2;         // every stem runs on CTA pairs (the kernel also compiles for PAIR = 1)
SrFn sr_kernel(int N, int sw, int per) {
  if (sw == 2 && N == 64 && per == 14) return k_step_stem_raw<64, 2, 14, 2>;   // C4's RGB 5x7x7 stem
  if (sw == 2) {
    if (N == 32) return k_step_stem_raw<32, 2, 0, 2>;
    if (N == 64) return k_step_stem_raw<64, 2, 0, 2>;
  } else if (sw == 1) {
    if (N == 32) return k_step_stem_raw<32, 1, 0, 2>;
    if (N == 64) return k_step_stem_raw<64, 1, 0, 2>;
  }
  return nullptr;
}
constexpr int kPerVariants[] = {0, 14};

}  // namespace

bool stem_raw_plan(const Geom& g, StemRawPlan& sp) {
  sp = StemRawPlan{};
  if (g.op != OP_CONV || g.in_dtype != BF16 || g.groups != 1) return false;
  // (the image ring holds two tiles' kt images: kt <= kNI / 2)
  if (g.sw < 1 || g.sw > 2 || g.sh < 1 || g.sh > 2 || g.dh != 1 || g.dw != 1 || 2 * g.kt > kNI) return false;
  const int CP = 8 / g.sw;
  if (g.Cin > CP || !sr_kernel(g.Cout, g.sw, 0) || (int64_t(g.W) * g.Cin * 2) % 16 != 0) return false;
  sp.N = g.Cout;
  sp.pair = kPair;
  sp.CP = CP;
  sp.Kp = (g.kw * CP + 15) / 16 * 16;
  // row slots: every valid window (pixels up to (Wo-1) sw + kw - 1 after pw zeros) and the data fit
  const int px = std::max(g.pw + g.W, (g.Wo - 1) * g.sw + g.kw);
  sp.Wp = (px + g.sw - 1) / g.sw;
  if (sp.Wp > 128) return false;
  sp.TH = 128 / sp.Wp;
  sp.tiles_h = (g.Ho + sp.TH - 1) / sp.TH;
  sp.n_tiles = g.B * sp.tiles_h;
  if (sp.n_tiles >= (int64_t(1) << 31)) return false;
  const int sh = g.sh;
  sp.nraw = (sp.TH - 1) * sh + g.kh;
  int rows = 0;
  for (int ph = 0; ph < sh; ++ph) {
    sp.base[ph] = rows;
    rows += ((sp.nraw - ph + sh - 1) / sh) * sp.Wp;
  }
  // the MMA of tap u reads 128 rows from its first row, plus Kp / 8 - 1 trailing 16-B groups
  int top = rows;
  for (int u = 0; u < g.kh; ++u) top = std::max(top, sp.base[u % sh] + (u / sh) * sp.Wp + 128 + sp.Kp / 8);
  sp.img_rows = top;
  // raw rows back to back (pitch = the frame row), after pad zero elements (>= pw
  // Cin, 16-B aligned data); reads past the last row (masked pixels, + 3 words)
  // stay inside the buffer
  sp.pad = (g.pw * g.Cin + 7) / 8 * 8;
  sp.rpitch = g.W * g.Cin * 2;
  const int over = std::max(0, (sp.Wp * g.sw - g.pw - g.W + 1) * g.Cin) + CP + 8;   // elements past the last row
  sp.w_bytes = g.kt * g.kh * sp.Kp * sp.N * 2 / sp.pair;   // this CTA's weight rows (half on a pair)
  sp.img_off = (sp.w_bytes + 1023) / 1024 * 1024;
  sp.img_bytes = (sp.img_rows * 16 + 127) / 128 * 128;
  sp.raw_off = sp.img_off + kNI * sp.img_bytes;
  sp.raw_bytes = (sp.pad * 2 + sp.nraw * sp.rpitch + over * 2 + 127) / 128 * 128;
  sp.bias_off = (sp.raw_off + kNR * sp.raw_bytes + 15) / 16 * 16;
  sp.bar_off = (sp.bias_off + sp.N * 4 + 63) / 64 * 64;
  sp.tab_off = sp.bar_off + 512;                           // after the barriers + TMEM holder
  const int n_desc = kNI * g.kh * (sp.Kp / 16);            // the MMA warp's A descriptor table
  sp.smem = size_t(sp.tab_off) + size_t(n_desc) * 8 + 1024;   // + 1 KB alignment slack
  if (sp.smem > kSmemLimit) return false;
  sp.ok = true;
  return true;
}

size_t stem_raw_wpack_elems(const StemRawPlan& sp, const Geom& g) { return size_t(g.kt) * g.kh * sp.Kp * sp.N; }

cudaError_t stem_raw_pack(const Geom& g, const StemRawPlan& sp, const void* w_dev, void* wpack) {
  k_pack_stem_raw<<<256, 256>>>(static_cast<const __nv_bfloat16*>(w_dev), static_cast<__nv_bfloat16*>(wpack), sp.N,
                               g.Cin, g.kt, g.kh, g.kw, sp.Kp, sp.CP, sp.pair);
  return cudaGetLastError();
}

cudaError_t stem_raw_prepare() {
  for (int sw : {1, 2})
    for (int n : {32, 64})
      for (int per : kPerVariants)
        if (SrFn fn = sr_kernel(n, sw, per))
          if (cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemLimit)))
            return e;
  return cudaSuccess;
}

cudaError_t stem_raw_step(const Geom& g, const StemRawPlan& sp, const StepArgs& a, const void* wpack,
                          const float* bias, int num_sms, cudaStream_t s) {
  SrParams p{};
  p.ring = static_cast<const __nv_bfloat16*>(static_cast<const void*>(a.state));
  p.frame_elems = int64_t(g.H) * g.W * g.Cin;
  p.slot_elems = g.B * p.frame_elems;
  for (int k = 0; k < kMaxKt; ++k) p.slot[k] = a.slot[k];
  p.kt = g.kt; p.kh = g.kh; p.sh = g.sh; p.ph = g.ph; p.pw = g.pw;
  p.Cin = g.Cin; p.H = g.H; p.W = g.W; p.Ho = g.Ho; p.Wo = g.Wo; p.Cout = g.Cout;
  p.Kp = sp.Kp;
  p.TH = sp.TH; p.tiles_h = sp.tiles_h; p.Wp = sp.Wp; p.n_tiles = sp.n_tiles;
  p.nraw = sp.nraw; p.rpitch = sp.rpitch; p.pad = sp.pad; p.img_rows = sp.img_rows;
  p.base0 = sp.base[0]; p.base1 = sp.base[1];
  p.w_bytes = sp.w_bytes; p.img_off = sp.img_off; p.img_bytes = sp.img_bytes;
  p.raw_off = sp.raw_off; p.raw_bytes = sp.raw_bytes; p.bias_off = sp.bias_off; p.bar_off = sp.bar_off;
  p.tab_off = sp.tab_off;
  p.y = a.y; p.y_bstride = a.y_bstride;
  p.out_f32 = g.out_dtype == F32; p.act = g.act;
  p.wpack = static_cast<const __nv_bfloat16*>(wpack);
  p.bias = bias;
  p.dbg = CO_EXP("CO_SR_DEBUG", 0);
  // a CTA (pair) per SM (pair of SMs); units only as many as there are tile groups
  const int64_t units = std::min<int64_t>(num_sms / sp.pair, (sp.n_tiles + sp.pair - 1) / sp.pair);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(units * sp.pair));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sp.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(sp.pair);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sr_kernel(sp.N, g.sw, g.kh * sp.Kp / 16), p);
}

const char* stem_raw_name(const StemRawPlan& sp) {
  static char buf[2][48];
  const int i = sp.N == 32 ? 0 : 1;
  snprintf(buf[i], sizeof(buf[i]), "k_step_stem_raw<%d%s>", sp.N, sp.pair == 2 ? ",pair" : "");
  return buf[i];
}

}  // namespace co
