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
//
// Three operand modes share the warp roles and the fused epilogue:
//  * HALO (spatial stride 1, weights fit in shared memory): the above;
//  * FLAT (1x1 spatial): rows = (stream, pixel) flattened, one 128-row box;
//  * KLOOP (spatial stride > 1, or weights too large to stay resident): a
//    classic K pipeline.  Per (tap (u,v), block of kb input channels) one stage
//    holds the A chunk -- 128 output pixels x kb channels, gathered by ONE TMA
//    box whose traversal strides (elementStrides) equal the spatial conv
//    stride, so strided im2col costs nothing -- and the B chunk (kb x N packed
//    weights, one bulk copy).  Small-Cin stems (Cin < 16, TMA needs 16-byte
//    rows) are first packed "W-im2col": xp[b,h,wo,(v,c)] = x[b,h,wo*sw+v-pw,c]
//    padded to a multiple of 16 channels, which turns the layer into a
//    (kt, kh, 1) convolution over xp with K = kh * roundup(kw*Cin, 16).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "dense_tc.cuh"
#include "stem_raw.cuh"
#include "tc_ptx.cuh"

namespace co {

namespace {

constexpr int kMaxStages = 8;   // operand pipeline depth (barrier slots): as many as fit in shared memory
constexpr int kMaxStagesStd = 6;   // HALO / FLAT / KLOOP: 7-8 measured no better (C4 K-loop layers)
// EG epilogue groups of 4*CS warps (CS warps share a TMEM lane quadrant and split
// its columns), then the producer and MMA warps
__host__ __device__ constexpr int tc_threads(int eg, int cs = 1) { return 32 * (4 * eg * cs + 2); }
constexpr int kApad = 512;        // slack after each A stage (junk rows may read past the box)
constexpr int kTickInts = 2 + kMaxKt;   // chunked steps: [emit, output index, slot[kMaxKt]] per tick
constexpr int kMaxAStages = 4;  // KHALO: input-halo ring depth
// KHALO: HALO's implicit im2col (one input-halo box per 64-channel block, the
// spatial taps as shifted descriptors) with the weights streamed per (tap,
// channel block) through the stage ring like KLOOP -- for layers whose weights
// do not fit in shared memory (C4 layers 3-5).  Spatial stride s splits the
// input into s x s phase sub-images (residues of the row / column mod s): tap
// (u, v) reads phase ((u-ph) mod s, (v-pw) mod s) at a whole-row shift, and
// each phase halo is one TMA box with elementStrides = s, so a stride-2 layer
// stages ~4 (MT+1) x (Wo+1) rows per channel block instead of 9 x 128.
// STEM (small-Cin stems such as C4's RGB 5x7x7 s(1,2,2) layer): the W-im2col
// is built in shared memory, not in HBM.  Per tile the producer bulk-copies the
// few raw input rows it needs (Cin = 3 channels: 672-B rows), and one epilogue
// warpgroup expands them -- overlapped with its own state loads -- into an
// im2col image [K group][row][16 B] whose row (pixel wo of raw row q) holds the
// window x[q, wo sw + v - pw, c] at K index v Cin + c.  Rows are stored by row
// phase (q mod sh), so spatial tap u of a tile's TH output rows is ONE shifted
// descriptor (phase u mod sh, first row u div sh), and both channel parts of the
// tile run consecutively on the same image (weights streamed per tap).
enum { MODE_HALO = 0, MODE_FLAT = 1, MODE_KLOOP = 2, MODE_KHALO = 3, MODE_STEM = 4 };

struct TcParams {
  int B, H, W, Cin, Cout, Ho, Wo;
  int64_t HWo, plane;             // plane = B * HWo
  int64_t splane;                 // state tiles * 128 (tile-blocked rows S[slot][tile][Cq][128][4])
  int kh, kw, ph, pw;
  int sh, sw, dh, dw;
  int mode;
  int MT, Wp, tiles_per_stream;   // halo mode geometry
  int TH, TW, tiles_h, tiles_w;   // kloop output tile (TH x TW <= 128 pixels)
  int kb, n_cb;                   // kloop: input channels per K chunk, chunks per tap
  int ka_stages, ka_stride;       // KHALO: input-halo ring (at the start of shared memory)
  int mc;                         // KLOOP, PAIR == 1: cluster of mc CTAs on consecutive row tiles of one
                                  // part; each loads 1/mc of every weight chunk, multicast to all
  int ka_phase, dmin_h, dmin_w;   // KHALO: bytes per phase halo; first sub-row / column offset floor(-p / s)
  int b_bytes, b_off;             // kloop: B chunk bytes, B offset inside a stage
  int64_t n_tiles, n_items;
  int n_split;
  int a_bytes, a_stride;          // A box bytes, stage stride in smem
  int stages;                     // pipeline depth (<= kMaxStages)
  int chunk_stride;               // bytes between 8-channel groups inside an A stage
  int w_bytes;                    // packed weights of one part
  int w_off;                      // stages start here (1 KB aligned)
  int slot[kMaxKt];
  int emit, update, act, out_f32;
  int raw_kh, raw_B;
  int raw_xslot, raw_xk;          // RAW flat: tap raw_xk reads the frame from xmap, stored into ring slot raw_xslot (-1: no)
  int kflat;                      // KLOOP over 128 flattened (stream, pixel) rows (RAW, 1x1 spatial)              // RAW layout: real spatial kh (the K loop walks kt*kh rows), streams per ring slot
  int ring_slot[kMaxKt];          // RAW layout: ring slot of temporal tap k
  int swa, a_rows;                // A staged swizzled: 0 none, 1 128-B rows ([Cin/64][rows][128 B]),
                                  // 2 64-B rows (KLOOP with kb = 32); rows per 64-channel block
  int ystage, y_off;              // HALO bf16: y transposed through a per-warp shared-memory buffer at y_off
  int l2last;                     // HALO / FLAT: frame tiles loaded with an L2 evict_last policy
  int pdl;                        // launched with programmatic stream serialization (see pdl_wait)
  int fparts;                     // KHALO: channel parts float over items (item i -> part i mod n_split), so
                                  // the grid need not be a multiple of the parts (weights stream per item)
  int l2pf;                       // L2 bulk prefetch of the state one item ahead (epilogue)
  int dbg;                        // CO_TC_DEBUG bits (experiments only): 1 no state/y traffic, 2 no MMA,
                                  // 4 no A loads, 8 no TMEM reads, 16 (with 2) no accumulator handshakes
  int Cq;
  // MODE_STEM: raw rows -> shared-memory W-im2col image (see above)
  const __nv_bfloat16* x;         // the step's frame (stream 0); nullptr = zero frame
  int64_t x_bstride;              // elements between streams
  int st_Hin, st_Win, st_cin;     // raw frame geometry
  int st_sw, st_pw, st_kwc;       // horizontal stride / padding, real K of a tap (kw Cin)
  int st_nraw;                    // raw rows per tile: (TH-1) sh + kh
  int st_rpitch, st_pad;          // bytes per padded raw row in shared memory, zero elements before the data
  int st_raw_off;                 // shared offset of the 2 raw-row buffers
  int st_img_rows, st_img_bytes;  // rows / bytes of one image buffer (2 buffers at offset 0)
  int st_groups, st_data_groups;  // 8-element K groups of the image, groups holding data
  int st_phase_base[2];           // first image row of each row phase (sh <= 2)
  // chunked co_forward_steps (HALO / FLAT): T frames per item,
  // processed item-batch-major so a tile's state stays L2-resident between its
  // frames; ticks = T rows of kTickInts: [emit, output index, ring slot of tap k...]
  int T;
  int x_tmul;                     // HALO chunks: frame (b, t) is clip "stream" b x_tmul + t (x_tmul = clip length)
  const int* ticks;
  int64_t y_tstride;              // elements between a stream's consecutive Ready outputs in y
  int64_t a_trows;                // FLAT: rows between frames of the time-major staged clip
  float* state;
  void* y;
  int64_t y_bstride;
  const __nv_bfloat16* wpack;     // [n_split][K/8][N][8]
  const float* bias;
};

// Programmatic dependent launch (p.pdl): the next launch in the stream may start
// its prologue (barriers, TMEM, resident weights) while this one drains; every
// access to data an earlier kernel wrote (frames, state, y) waits on
// griddepcontrol.wait, which returns once the prerequisite grid completed and
// its writes are visible (a no-op for a normal launch).
// CO_TC_DEBUG bits (p.dbg): experiment builds only; the release kernels
// compile every DBG() test to 0, so no work can be skipped in a shipped build.
#ifdef CO_EXPERIMENTS
#define DBG(bits) (p.dbg & (bits))
#else
#define DBG(bits) (0)
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void bar_sync_named(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// state load without an L1 allocation (CO_TC_DEBUG bit 32: experiment)
__device__ __forceinline__ float4 ld_state_na(const float4* p) {
  float4 v;
  asm volatile("ld.global.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

// state store: st.global.cs (streaming); experiment builds can A/B other flavours
// (CO_TC_DEBUG 2048: plain st.global, 4096: L1::no_allocate, 8192: .wt)
template <typename P>
__device__ __forceinline__ void st_state(const P& p, float4* dst, float4 v) {
#ifdef CO_EXPERIMENTS
  if (p.dbg & 2048) { *dst = v; return; }
  if (p.dbg & 4096) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w) : "memory");
    return;
  }
  if (p.dbg & 8192) { __stwt(dst, v); return; }
#endif
  (void)p;
  __stcs(dst, v);
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// CE: output channels per epilogue pass (bounds the prefetched-state registers
// at (kt-1) * CE / 4 float4 per thread); KH, KW, KC (= Cin / 16) > 0: compile-
// time tap / K loops of the HALO / FLAT modes, fully unrolled, so the issuing
// warp spends ~3 uniform instructions per tcgen05.mma.
template <int KT, int CC, int EG, int CE, int KH = 0, int KW = 0, int KC = 0, int CS = 1, int PAIR = 1,
          bool STM = false>
__global__ void __launch_bounds__(tc_threads(EG, CS), 1)
    k_step_dense_tc(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap wmap,
                    const __grid_constant__ CUtensorMap xmap, const TcParams p) {
  // wmap: the packed weights as a tensor, used by KLOOP CTA pairs (each CTA
  // streams its N/2 half of every B chunk with a pair TMA load)
  constexpr int N = KT * CC;
  // TMEM accumulator ring: as many N-column buffers as 512 columns hold, at
  // least one per epilogue group, so the MMA can run ahead of the state traffic.
  constexpr int BUF = (N + 31) / 32 * 32;
  constexpr int NBUF = (512 / BUF) < 8 ? (512 / BUF) : 8;
  static_assert(NBUF >= EG, "accumulator buffers exceed TMEM");
  constexpr int TMEM_COLS = 512;
  constexpr int kProducer = 4 * EG * CS, kMma = 4 * EG * CS + 1;
  static_assert(CC % (CS * CE) == 0, "channel split must tile CC");
  static_assert(N % 16 == 0 && N <= 256, "invalid UMMA N");
  static_assert(CC % CE == 0 && CE % 16 == 0, "CE must divide CC, multiple of 16");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment by pointer arithmetic on the __shared__ array (an integer
  // round trip would turn every derived access into a generic one)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* w_s = smem;                                  // [K/8][N][16 B] (HALO / FLAT)
  uint8_t* a_s = smem + p.w_off;                        // stages x a_stride
  uint64_t* bars = reinterpret_cast<uint64_t*>(a_s + p.stages * p.a_stride);
  uint64_t* full = bars;                                // [kMaxStages]
  uint64_t* empty = bars + kMaxStages;                  // [kMaxStages]
  uint64_t* acc_full = bars + 2 * kMaxStages;           // [NBUF]
  uint64_t* acc_empty = bars + 2 * kMaxStages + NBUF;   // [NBUF]
  uint64_t* w_full = bars + 2 * kMaxStages + 2 * NBUF;
  uint64_t* w_peer = w_full + 1;                        // PAIR: the peer's weight half landed
  uint64_t* a_full = w_full + 2;                        // [kMaxAStages] KHALO halo ring
  uint64_t* a_empty = a_full + kMaxAStages;             // [kMaxAStages]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(a_empty + kMaxAStages);
  // 16-byte aligned: the epilogue reads the bias as float4
  float* bias_s = reinterpret_cast<float*>(bars + ((2 * kMaxStages + 2 * NBUF + 2 + 2 * kMaxAStages + 1 + 1) & ~1));

  constexpr int NS = (KT > 1) ? KT - 1 : 1;            // state slots an item reads
  constexpr int NQ = CE / 4;                           // channel quads per thread and pass
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grid = gridDim.x;
  // CTA pairs (cta_group::2, PAIR == 2): the cluster's two CTAs share one M = 256
  // MMA issued by the leader; each holds the A rows of its own 128-row tile and
  // half (N/2 rows) of the part's weights, so per-CTA weight shared memory halves.
  const int CLU = (PAIR == 2) ? 2 : p.mc;              // CTAs per cluster (pair / weight multicast group)
  const uint32_t rank = (CLU > 1) ? ptx::cluster_ctarank() : 0u;
  const bool leader = (PAIR == 1) || (rank == 0);
  const uint16_t mc_mask = uint16_t((1u << CLU) - 1u);
  const int unit = blockIdx.x / CLU;                    // work unit: a CTA, a CTA pair or a multicast cluster
  const int n_units = grid / CLU;
  const int part = unit % p.n_split;
  const int c0 = part * CC;                             // first output channel of this part
  const bool kloop = (p.mode == MODE_KLOOP);
  const bool khalo = (p.mode == MODE_KHALO);
  constexpr int NB = N / PAIR;                          // weight rows held by this CTA
  auto tile_of = [&](int64_t item) -> int64_t { return (item / p.n_split) * CLU + rank; };

  if (warp == kProducer && lane == 0) {
    // multicast clusters: a stage is free once every CTA of the cluster consumed it
    for (int s = 0; s < p.stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], PAIR == 1 ? CLU : 1); }
    for (int e = 0; e < NBUF; ++e) { ptx::mbar_init(&acc_full[e], 1); ptx::mbar_init(&acc_empty[e], 128 * CS * PAIR); }
    ptx::mbar_init(w_full, 1);
    ptx::mbar_init(w_peer, 1);
    for (int s = 0; s < kMaxAStages; ++s) { ptx::mbar_init(&a_full[s], 1); ptx::mbar_init(&a_empty[s], 1); }
    if (p.mode == MODE_STEM) {
      // images: full when the converting group's 128 CS threads arrived, empty on the
      // MMA's commit; raw rows: full on the bulk copies' bytes, empty when converted
      for (int b = 0; b < 2; ++b) { ptx::mbar_init(&a_full[b], 128 * CS); ptx::mbar_init(&a_empty[2 + b], 128 * CS); }
    }
    ptx::fence_mbar_init();
  }
  if (warp == kMma) {
    if constexpr (PAIR == 2) ptx::tmem_alloc_pair(tmem_holder, TMEM_COLS);
    else ptx::tmem_alloc(tmem_holder, TMEM_COLS);
  }
  // MODE_STEM only in the STM instantiations (the shared-memory W-im2col code
  // stays out of every other variant's registers)
  constexpr bool kStem = STM && PAIR == 1 && CS == 1;
  const bool stem = kStem && (p.mode == MODE_STEM);
  // STEM CTAs serve every channel part (all Cout biases); other modes one part
  if (stem) {
    for (int i = threadIdx.x; i < p.Cout; i += blockDim.x) bias_s[i] = p.bias[i];
    // zero the image K groups that never hold data and the raw rows' padding, once
    // (the converter writes only data groups, the bulk copies only row interiors)
    for (int b = 0; b < 2; ++b)
      for (int gq = p.st_data_groups; gq < p.st_groups; ++gq) {
        uint4* z = reinterpret_cast<uint4*>(smem + b * p.st_img_bytes + gq * p.st_img_rows * 16);
        for (int i = threadIdx.x; i < p.st_img_rows; i += blockDim.x) z[i] = make_uint4(0u, 0u, 0u, 0u);
      }
    uint4* zr = reinterpret_cast<uint4*>(smem + p.st_raw_off);
    for (int i = threadIdx.x; i < 2 * p.st_nraw * p.st_rpitch / 16; i += blockDim.x) zr[i] = make_uint4(0u, 0u, 0u, 0u);
    ptx::fence_proxy_async();                           // generic zeros, read by the tensor cores
  } else {
    // floating parts (KHALO): every part's biases; otherwise this CTA's part
    for (int i = threadIdx.x; i < (p.fparts ? p.Cout : CC); i += blockDim.x) bias_s[i] = p.bias[(p.fparts ? 0 : c0) + i];
  }
  ptx::tc_fence_before();
  if (CLU > 1) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (p.pdl) pdl_trigger();                             // the next step may be scheduled as SMs free up

  if (warp == kProducer) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      ptx::prefetch_tmap(&tmap);
      const uint64_t l2pol = p.l2last ? ptx::l2_policy_evict_last() : 0;
      const uint8_t* wsrc =
          reinterpret_cast<const uint8_t*>(p.wpack) + size_t(part * PAIR + (PAIR == 2 ? rank : 0u)) * p.w_bytes;
      int s = 0;
      uint32_t ph = 0;
      if (stem) {
        if (p.pdl) pdl_wait();
        const int rowbytes = p.st_Win * p.st_cin * 2;
        // raw rows of CTA-local tile T into raw buffer T & 1 (one tile ahead of the weights)
        auto load_raw = [&](int64_t T) {
          const int64_t tile = int64_t(blockIdx.x) + T * grid;
          if (tile >= p.n_tiles) return;
          const int rb = int(T & 1);
          ptx::mbar_wait(&a_empty[2 + rb], (uint32_t(T >> 1) & 1u) ^ 1u);
          const int bs = int(tile / p.tiles_h);
          const int r0 = int(tile % p.tiles_h) * p.TH * p.sh - p.ph;
          int nv = 0;
          for (int q = 0; q < p.st_nraw; ++q) nv += (p.x && r0 + q >= 0 && r0 + q < p.st_Hin) ? 1 : 0;
          if (!nv) { ptx::mbar_arrive(&a_full[2 + rb]); return; }
          ptx::mbar_arrive_expect_tx(&a_full[2 + rb], uint32_t(nv * rowbytes));
          uint8_t* dst = smem + p.st_raw_off + rb * p.st_nraw * p.st_rpitch + p.st_pad * 2;
          const __nv_bfloat16* src = p.x + int64_t(bs) * p.x_bstride;
          for (int q = 0; q < p.st_nraw; ++q)
            if (r0 + q >= 0 && r0 + q < p.st_Hin)
              ptx::bulk_g2s(dst + q * p.st_rpitch, src + int64_t(r0 + q) * p.st_Win * p.st_cin, rowbytes, &a_full[2 + rb]);
        };
        load_raw(0);
        for (int64_t T = 0; int64_t(blockIdx.x) + T * grid < p.n_tiles; ++T) {
          load_raw(T + 1);
          for (int pt = 0; pt < p.n_split; ++pt) {
            const uint8_t* bsrc = reinterpret_cast<const uint8_t*>(p.wpack) + size_t(pt) * p.w_bytes;
            for (int u = 0; u < p.kh; ++u) {
              ptx::mbar_wait(&empty[s], ph ^ 1);
              ptx::mbar_arrive_expect_tx(&full[s], p.b_bytes);
              ptx::bulk_g2s(a_s + s * p.a_stride, bsrc + size_t(u) * p.b_bytes, p.b_bytes, &full[s]);
              if (++s == p.stages) { s = 0; ph ^= 1; }
            }
          }
        }
      } else if (khalo) {
        if (p.pdl) pdl_wait();
        int as = 0;
        uint32_t aph = 0;
        for (int64_t item = unit; item < p.n_items; item += n_units) {
          const int64_t tile = tile_of(item);
          const int b = int(tile / p.tiles_per_stream);
          const int ho0 = int(tile % p.tiles_per_stream) * p.MT;
          const int ipart = p.fparts ? int(item % p.n_split) : part;   // this item's channel part
          const uint8_t* wsrc_i =
              reinterpret_cast<const uint8_t*>(p.wpack) + size_t(ipart * PAIR + (PAIR == 2 ? rank : 0u)) * p.w_bytes;
          for (int cb = 0; cb < p.n_cb; ++cb) {
            // the 64-channel block's input halo, then its (tap) weight chunks
            ptx::mbar_wait(&a_empty[as], aph ^ 1);
            uint8_t* adst = smem + as * p.ka_stride;
            const int n_ph = p.sh * p.sw;
            if (DBG(4)) {                               // experiment: no halo loads
              if (!(PAIR == 2 && !leader)) ptx::mbar_arrive(&a_full[as]);
            } else if (!(PAIR == 2 && !leader)) ptx::mbar_arrive_expect_tx(&a_full[as], p.a_bytes * n_ph * PAIR);
            for (int rr = 0; rr < p.sh && !DBG(4); ++rr)
              for (int rc = 0; rc < p.sw; ++rc) {
                // phase (rr, rc): original rows s (ho0 + dmin_h + i) + rr, columns s (dmin_w + j) + rc
                uint8_t* pd = adst + (rr * p.sw + rc) * p.ka_phase;
                const int r0 = p.sh * (ho0 + p.dmin_h) + rr, c0w = p.sw * p.dmin_w + rc;
                if constexpr (PAIR == 2) ptx::tma_load_5d_pair(pd, &tmap, &a_full[as], 0, c0w, r0, cb, b);
                else ptx::tma_load_5d(pd, &tmap, &a_full[as], 0, c0w, r0, cb, b);
              }
            if (++as == p.ka_stages) { as = 0; aph ^= 1; }
            for (int tap = 0; tap < p.kh * p.kw; ++tap) {
              const int kblk = tap * p.n_cb + cb;       // packed K index (u kw + v) Cin + ci, in 64-blocks
              ptx::mbar_wait(&empty[s], ph ^ 1);
              uint8_t* dst = a_s + s * p.a_stride;
              if (DBG(1024)) {                          // experiment: no weight loads
                if (leader) ptx::mbar_arrive(&full[s]);
              } else if constexpr (PAIR == 2) {
                if (leader) ptx::mbar_arrive_expect_tx(&full[s], p.b_bytes * PAIR);
                ptx::tma_load_4d_pair(dst, &wmap, &full[s], 0, 0, kblk, ipart * PAIR + int(rank));
              } else {
                ptx::mbar_arrive_expect_tx(&full[s], p.b_bytes);
                ptx::bulk_g2s(dst, wsrc_i + size_t(kblk) * p.b_bytes, p.b_bytes, &full[s]);
              }
              if (++s == p.stages) { s = 0; ph ^= 1; }
            }
          }
        }
      } else if (!kloop) {
        ptx::mbar_arrive_expect_tx(w_full, p.w_bytes);
        for (int off = 0; off < p.w_bytes; off += 32768) {
          const int n = min(32768, p.w_bytes - off);
          ptx::bulk_g2s(w_s + off, wsrc + off, n, w_full);
        }
        if constexpr (PAIR == 2) {
          if (!leader) {   // tell the leader's MMA warp that this half of the weights landed
            ptx::mbar_wait(w_full, 0);
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(w_peer), 0));
          }
        }
        if (p.pdl) pdl_wait();                          // the resident weights are never written by a kernel
        // works in item-batch-major order (T == 1: one work per item, as before)
        for (int64_t bi = unit; bi < p.n_items; bi += int64_t(EG) * n_units) {
          const int64_t left = (p.n_items - bi + n_units - 1) / n_units;
          const int nb = left < EG ? int(left) : EG;
          for (int t = 0; t < p.T; ++t)
            for (int e = 0; e < nb; ++e) {
              const int64_t item = bi + int64_t(e) * n_units;
              ptx::mbar_wait(&empty[s], ph ^ 1);
              if DBG(4) {
                if (leader) ptx::mbar_arrive(&full[s]);
                if (++s == p.stages) { s = 0; ph ^= 1; }
                continue;
              }
              // the leader's barrier counts both CTAs' A bytes (pair-TMA completes on it)
              if (leader) ptx::mbar_arrive_expect_tx(&full[s], p.a_bytes * PAIR);
              const int64_t tile = tile_of(item);
              uint8_t* dst = a_s + s * p.a_stride;
              // p.l2last: the frame tile every channel part re-reads is kept in L2
              // (evict_last) while the state streams through (evict_first)
              if (p.mode == MODE_FLAT) {
                const int row = int(tile * 128 + t * p.a_trows);     // staged clip: frame t's rows
                if (p.l2last) {
                  if constexpr (PAIR == 2) ptx::tma_load_3d_pair_hint(dst, &tmap, &full[s], 0, row, 0, l2pol);
                  else ptx::tma_load_3d_hint(dst, &tmap, &full[s], 0, row, 0, l2pol);
                } else {
                  if constexpr (PAIR == 2) ptx::tma_load_3d_pair(dst, &tmap, &full[s], 0, row, 0);
                  else ptx::tma_load_3d(dst, &tmap, &full[s], 0, row, 0);
                }
              } else {
                const int b = int(tile / p.tiles_per_stream) * p.x_tmul + t;   // clip: (stream, frame) -> b T + t
                const int ho0 = int(tile % p.tiles_per_stream) * p.MT;
                if (p.l2last) {
                  if constexpr (PAIR == 2) ptx::tma_load_5d_pair_hint(dst, &tmap, &full[s], 0, -p.pw, ho0 - p.ph, 0, b, l2pol);
                  else ptx::tma_load_5d_hint(dst, &tmap, &full[s], 0, -p.pw, ho0 - p.ph, 0, b, l2pol);
                } else {
                  if constexpr (PAIR == 2) ptx::tma_load_5d_pair(dst, &tmap, &full[s], 0, -p.pw, ho0 - p.ph, 0, b);
                  else ptx::tma_load_5d(dst, &tmap, &full[s], 0, -p.pw, ho0 - p.ph, 0, b);
                }
              }
              if (++s == p.stages) { s = 0; ph ^= 1; }
            }
        }
      } else {
        if (p.pdl) pdl_wait();
        const int per_stream = p.tiles_h * p.tiles_w;
        // RAW flat fused ring store: stages holding chunks of the new frame, stored into
        // the ring from shared memory once the MMA released them (tile * 16 + cc, -1 none)
        int pend[kMaxStages];
        for (int i = 0; i < kMaxStages; ++i) pend[i] = -1;
        const bool xstore = p.kflat && p.raw_xslot >= 0 && part == 0;
        auto flush = [&](int st) {
          if (pend[st] < 0) return;
          ptx::tma_store_4d(&tmap, a_s + st * p.a_stride, 0, (pend[st] >> 5) * 128, pend[st] & 31, p.raw_xslot);
          ptx::bulk_commit();
          ptx::bulk_wait_read0();                         // the stage may be refilled now
          pend[st] = -1;
        };
        for (int64_t item = unit; item < p.n_items; item += n_units) {
          const int64_t tile = tile_of(item);
          const int b = p.kflat ? 0 : int(tile / per_stream);
          const int r = p.kflat ? 0 : int(tile % per_stream);
          const int ho0 = (r / p.tiles_w) * p.TH, wo0 = (r % p.tiles_w) * p.TW;
          const uint8_t* bsrc = wsrc;
          int kg = 0;                                   // K-group (8 channels) index of the chunk
          for (int uu = 0; uu < p.kh; ++uu) {
            // RAW layout: row uu = (temporal tap k, spatial row u), frame from ring slot k
            const int kk = p.raw_kh ? uu / p.raw_kh : 0;
            const int u = p.raw_kh ? uu - kk * p.raw_kh : uu;
            const int bb = p.raw_kh ? b + p.ring_slot[kk] * p.raw_B : b;
            for (int v = 0; v < p.kw; ++v)
              for (int cb = 0; cb < p.n_cb; ++cb) {
                ptx::mbar_wait(&empty[s], ph ^ 1);
                if (xstore) flush(s);
                uint8_t* dst = a_s + s * p.a_stride;
                const int cw = wo0 * p.sw + v * p.dw - p.pw, ch = ho0 * p.sh + u * p.dh - p.ph;
                const int cc = p.swa ? cb : cb * (p.kb / 8);   // swizzled: kb-channel blocks
                // weight chunk: whole (one CTA), or this CTA's 1/mc byte range multicast to the cluster
                auto load_b = [&]() {
                  if (CLU > 1) {
                    const uint32_t piece = uint32_t(p.b_bytes / CLU);
                    ptx::bulk_g2s_mc(dst + p.b_off + rank * piece, bsrc + rank * piece, piece, &full[s], mc_mask);
                  } else {
                    ptx::bulk_g2s(dst + p.b_off, bsrc, p.b_bytes, &full[s]);
                  }
                };
                if (p.kflat) {    // rows tile*128 .. of ring slot k, viewed as a (B*HW, Cin) matrix
                  // the new frame (tap raw_xk) straight from x when the kernel stores it into the ring
                  const bool fromx = p.raw_xslot >= 0 && kk == p.raw_xk;
                  const CUtensorMap* am = fromx ? &xmap : &tmap;
                  const int aslot = fromx ? 0 : p.ring_slot[kk];
                  if constexpr (PAIR == 2) {
                    // CTA pair: each CTA its own 128 rows and its N/2 half of the weight
                    // chunk, both completing on the leader's barrier
                    if (leader) ptx::mbar_arrive_expect_tx(&full[s], (p.a_bytes + p.b_bytes) * PAIR);
                    ptx::tma_load_4d_pair(dst, am, &full[s], 0, int(tile * 128), cc, aslot);
                    ptx::tma_load_4d_pair(dst + p.b_off, &wmap, &full[s], 0, 0, kg / (p.kb / 8), part * PAIR + int(rank));
                  } else {
                    ptx::mbar_arrive_expect_tx(&full[s], p.a_bytes + p.b_bytes);
                    ptx::tma_load_4d(dst, am, &full[s], 0, int(tile * 128), cc, aslot);
                    load_b();
                  }
                  if (xstore && fromx) pend[s] = int(tile) * 32 + cc;
                } else if constexpr (PAIR == 2) {
                  if (leader) ptx::mbar_arrive_expect_tx(&full[s], (p.a_bytes + p.b_bytes) * PAIR);
                  ptx::tma_load_5d_pair(dst, &tmap, &full[s], 0, cw, ch, cc, bb);
                  ptx::tma_load_4d_pair(dst + p.b_off, &wmap, &full[s], 0, 0, kg / (p.kb / 8), part * PAIR + int(rank));
                } else {
                  ptx::mbar_arrive_expect_tx(&full[s], p.a_bytes + p.b_bytes);
                  ptx::tma_load_5d(dst, &tmap, &full[s], 0, cw, ch, cc, bb);
                  load_b();
                }
                bsrc += p.b_bytes;
                kg += p.kb / 8;
                if (++s == p.stages) { s = 0; ph ^= 1; }
              }
          }
        }
        if (xstore) {
          // the last stages' new-frame chunks: store each once the MMA released it
          for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_wait(&empty[s], ph ^ 1);
            flush(s);
            if (++s == p.stages) { s = 0; ph ^= 1; }
          }
          ptx::bulk_wait0();
        }
      }
    }
  } else if (warp == kMma) {
    // ===================== MMA issuer =====================
    // The whole warp runs the loop (warp-uniform descriptors live in uniform
    // registers); one elected lane issues each tcgen05.mma / commit.
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(128 * PAIR, N);
    const uint32_t a_base = ptx::smem_u32(a_s);
    // Descriptors are advanced by adding (byte offset >> 4) to their 14-bit
    // start-address field (shared memory < 256 KB, so it never carries out).
    const uint32_t chunk16 = uint32_t(p.chunk_stride) >> 3;   // 2 channel groups, in 16 B units
    int s = 0;
    uint32_t ph = 0;
    int e = 0;
    uint32_t eph = 0;
    auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t acc) {
      if constexpr (PAIR == 2) ptx::mma_bf16_ss_pair(d, ad, bd, idesc, acc);
      else ptx::mma_bf16_ss(d, ad, bd, idesc, acc);
    };
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR == 2) ptx::tc_commit_pair(bar, 0x3);   // both CTAs' copies of the barrier
      else ptx::tc_commit(bar);
    };
    if (PAIR == 2 && !leader) {
      // the peer's tensor-core work is issued by the leader
    } else if (stem) {
      const uint32_t lbo = uint32_t(p.st_img_rows) * 16u;       // bytes between the image's K groups
      const int nk = p.kb / 16;                                  // MMAs (K = 16) per tap
      int64_t li = 0;
      for (int64_t T = 0; int64_t(blockIdx.x) + T * grid < p.n_tiles; ++T) {
        const int b = int(T & 1);
        ptx::mbar_wait(&a_full[b], uint32_t(T >> 1) & 1u);      // the tile's image was built
        ptx::tc_fence_after();
        const uint64_t a0 = ptx::smem_desc(ptx::smem_u32(smem + b * p.st_img_bytes), lbo, 128);
        for (int pt = 0; pt < p.n_split; ++pt, ++li) {
          ptx::mbar_wait(&acc_empty[e], eph ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem + uint32_t(e * BUF);
          for (int u = 0; u < p.kh; ++u) {
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            const uint64_t bd = ptx::smem_desc(a_base + uint32_t(s * p.a_stride), NB * 16, 128);
            // tap u: phase u mod sh, first row u div sh (16-B units per row)
            const uint64_t ad = a0 + uint64_t(p.st_phase_base[u % p.sh] + (u / p.sh) * p.Wo);
            if (ptx::elect_one()) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                if (j < nk) mma(d_tmem, ad + uint64_t(j) * (2u * lbo >> 4), bd + uint64_t(j) * uint64_t(2 * NB),
                                (u | j) ? 1u : 0u);
              commit(&empty[s]);
            }
            __syncwarp();
            if (++s == p.stages) { s = 0; ph ^= 1; }
          }
          if (ptx::elect_one()) {
            commit(&acc_full[e]);
            if (pt == p.n_split - 1) commit(&a_empty[b]);          // image free after the tile's last part
          }
          __syncwarp();
          if (++e == NBUF) { e = 0; eph ^= 1; }
        }
      }
      (void)li;
    } else if (khalo) {
      const int taps = p.kh * p.kw;
      const uint32_t ka_base = ptx::smem_u32(smem);
      // per-tap descriptor offset (16-B units): phase block + row shift, computed
      // once (runtime-divisor divisions would otherwise sit in the issue loop)
      uint32_t* tap_tab = reinterpret_cast<uint32_t*>(bias_s + (p.fparts ? p.Cout : CC));
      for (int tap = lane; tap < taps; tap += 32) {
        const int u = tap / p.kw, v = tap - (tap / p.kw) * p.kw;
        // input row s ho + u - ph = s (ho + floor((u-ph)/s)) + (u-ph) mod s
        const int eu = u - p.ph + p.sh * 8, ev = v - p.pw + p.sw * 8;   // shifted nonnegative
        const int rr = eu % p.sh, rc = ev % p.sw;
        const int du = eu / p.sh - 8 - p.dmin_h, dv = ev / p.sw - 8 - p.dmin_w;
        tap_tab[tap] = uint32_t((rr * p.sw + rc) * p.ka_phase) / 16u + uint32_t(du * p.Wp + dv) * 8u;
      }
      __syncwarp();
      int as = 0;
      uint32_t aph = 0;
      if constexpr (KH > 0 && KC == 0 && PAIR == 2) {
        // compile-time taps (the C4 layers' 3 x 3): tap offsets in registers, each
        // chunk's 4 MMAs + commit in one branch-free elected issue
        uint32_t toff[KH * KW];
#pragma unroll
        for (int t = 0; t < KH * KW; ++t) toff[t] = tap_tab[t];
        for (int64_t item = unit; item < p.n_items; item += n_units) {
          ptx::mbar_wait(&acc_empty[e], eph ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem + uint32_t(e * BUF);
          for (int cb = 0; cb < p.n_cb; ++cb) {
            ptx::mbar_wait(&a_full[as], aph);
            ptx::tc_fence_after();
            const uint64_t a0 = ptx::smem_desc_sw128(ka_base + uint32_t(as * p.ka_stride));
#pragma unroll
            for (int tap = 0; tap < KH * KW; ++tap) {
              ptx::mbar_wait(&full[s], ph);
              ptx::tc_fence_after();
              const uint64_t bd = ptx::smem_desc_sw128(a_base + uint32_t(s * p.a_stride));
              ptx::mma4_commit_pair(d_tmem, a0 + toff[tap], 2u, bd, 2u, idesc, (cb | tap) ? 1u : 0u, &empty[s], 0x3);
              if (++s == p.stages) { s = 0; ph ^= 1; }
            }
            if (ptx::elect_one()) commit(&a_empty[as]);   // halo free after its last tap
            __syncwarp();
            if (++as == p.ka_stages) { as = 0; aph ^= 1; }
          }
          if (ptx::elect_one()) commit(&acc_full[e]);
          __syncwarp();
          if (++e == NBUF) { e = 0; eph ^= 1; }
        }
      } else
      for (int64_t item = unit; item < p.n_items; item += n_units) {
        ptx::mbar_wait(&acc_empty[e], eph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(e * BUF);
        for (int cb = 0; cb < p.n_cb; ++cb) {
          ptx::mbar_wait(&a_full[as], aph);
          ptx::tc_fence_after();
          const uint64_t a0 = ptx::smem_desc_sw128(ka_base + uint32_t(as * p.ka_stride));
          for (int tap = 0; tap < taps; ++tap) {
            ptx::mbar_wait(&full[s], ph);
            ptx::tc_fence_after();
            const uint32_t st = a_base + uint32_t(s * p.a_stride);
            const uint64_t bd = (PAIR == 1) ? ptx::smem_desc(st, NB * 16, 128) : ptx::smem_desc_sw128(st);
            const uint64_t bstep = (PAIR == 1) ? uint64_t(2 * NB) : 2u;
            const uint64_t ad = a0 + tap_tab[tap];     // phase block, then a du Wp + dv row shift
            if (ptx::elect_one()) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                mma(d_tmem, ad + uint64_t(j) * 2u, bd + uint64_t(j) * bstep, (cb | tap | j) ? 1u : 0u);
              commit(&empty[s]);      // weight stage free once these MMAs retire
            }
            __syncwarp();
            if (++s == p.stages) { s = 0; ph ^= 1; }
          }
          if (ptx::elect_one()) commit(&a_empty[as]);   // halo free after its last tap
          __syncwarp();
          if (++as == p.ka_stages) { as = 0; aph ^= 1; }
        }
        if (ptx::elect_one()) commit(&acc_full[e]);
        __syncwarp();
        if (++e == NBUF) { e = 0; eph ^= 1; }
      }
    } else if (!kloop) {
      ptx::mbar_wait(w_full, 0);
      if constexpr (PAIR == 2) ptx::mbar_wait(w_peer, 0);
      const uint64_t b_desc0 = ptx::smem_desc(ptx::smem_u32(w_s), NB * 16, 128);
      const int kc2 = p.Cin / 16;                       // MMAs (K = 16) per spatial tap
      int64_t n_works = 0;                              // this unit's works: items x T frames
      for (int64_t item = unit; item < p.n_items; item += n_units) n_works += p.T;
      for (int64_t w = 0; w < n_works; ++w) {
        if (!DBG(16)) ptx::mbar_wait(&acc_empty[e], eph ^ 1);
        ptx::tc_fence_after();
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(e * BUF);
        const uint64_t a_desc0 = p.swa ? ptx::smem_desc_sw128(a_base + uint32_t(s * p.a_stride))
                                       : ptx::smem_desc(a_base + uint32_t(s * p.a_stride), p.chunk_stride, 128);
        // K16 step kc of a tap: 32 B along the swizzled 128-B row (next 64-channel
        // block every 4 steps), or two 8-channel core-matrix groups unswizzled
        auto kc_off = [&](int kc) -> uint64_t {
          return p.swa ? uint64_t((kc >> 2) * p.a_rows * 8 + (kc & 3) * 2) : uint64_t(kc) * chunk16;
        };
        const uint32_t row16 = p.swa ? 8u : 1u;        // one halo row in 16-B units
        if constexpr (KH > 0) {
          if (!DBG(2) && ptx::elect_one()) {
#pragma unroll
            for (int u = 0; u < KH; ++u)
#pragma unroll
              for (int v = 0; v < KW; ++v) {
                const uint64_t ad = a_desc0 + uint64_t(u * p.Wp + v) * row16;
#pragma unroll
                for (int kc = 0; kc < KC; ++kc)
                  mma(d_tmem, ad + kc_off(kc), b_desc0 + uint64_t(((u * KW + v) * KC + kc) * 2 * NB),
                      (u | v | kc) ? 1u : 0u);
              }
          }
          __syncwarp();
        } else {
          uint64_t bd = b_desc0;
          uint32_t acc = 0;
          for (int u = 0; u < p.kh; ++u) {
            for (int v = 0; v < p.kw; ++v) {
              const uint64_t ad = a_desc0 + uint64_t(u * p.Wp + v) * row16;   // tap (u, v): shift by u Wp + v rows
              for (int kc = 0; kc < kc2; ++kc) {
                if (ptx::elect_one()) mma(d_tmem, ad + kc_off(kc), bd, acc);
                __syncwarp();
                acc = 1;
                bd += uint64_t(2 * NB);                        // 2 groups of NB rows x 16 B
              }
            }
          }
        }
        if (ptx::elect_one()) {
          commit(&empty[s]);      // A stage free once these MMAs retire
          commit(&acc_full[e]);   // accumulator e ready for the epilogue
        }
        __syncwarp();
        if (++s == p.stages) { s = 0; ph ^= 1; }
        if (++e == NBUF) { e = 0; eph ^= 1; }
      }
    } else {
      const int n_chunks = p.kh * p.kw * p.n_cb;
      const int nk = p.kb / 16;                         // MMAs per chunk (<= 4)
      for (int64_t item = unit; item < p.n_items; item += n_units) {
        ptx::mbar_wait(&acc_empty[e], eph ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + uint32_t(e * BUF);
        for (int ch = 0; ch < n_chunks; ++ch) {
          ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
          const uint32_t st = a_base + uint32_t(s * p.a_stride);
          const uint64_t ad = p.swa == 1 ? ptx::smem_desc_sw128(st)
                              : p.swa == 2 ? ptx::smem_desc_sw64(st) : ptx::smem_desc(st, p.chunk_stride, 128);
          // B: core-matrix layout, or (pairs) swizzled kb-element rows like A
          const uint64_t bd = (PAIR == 1) ? ptx::smem_desc(st + uint32_t(p.b_off), NB * 16, 128)
                              : p.kb == 64 ? ptx::smem_desc_sw128(st + uint32_t(p.b_off))
                                           : ptx::smem_desc_sw64(st + uint32_t(p.b_off));
          const uint64_t bstep = (PAIR == 1) ? uint64_t(2 * NB) : 2u;
          const uint64_t astep = p.swa ? 2u : chunk16;     // one K16 step: 32 B of a swizzled row
          if (ptx::elect_one()) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nk) mma(d_tmem, ad + uint64_t(j) * astep, bd + uint64_t(j) * bstep, (ch | j) ? 1u : 0u);
            // stage free once these MMAs retire (multicast: in every CTA of the cluster)
            if (PAIR == 1 && CLU > 1) ptx::tc_commit_mc(&empty[s], mc_mask);
            else commit(&empty[s]);
          }
          __syncwarp();
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
        if (ptx::elect_one()) commit(&acc_full[e]);
        __syncwarp();
        if (++e == NBUF) { e = 0; eph ^= 1; }
      }
    }
    __syncwarp();
  } else {
  // ===================== epilogue warpgroups (warps 0 .. 4 EG - 1) =====================
  if (p.pdl) pdl_wait();                               // state / y of the previous step
  const int e = warp / (4 * CS);                       // group
  const int q = warp & 3;                              // TMEM lane quadrant of this warp
  const int cs = (warp >> 2) % CS;                     // column share of this warp
  constexpr int CPW = CC / CS;                         // output channels per warp
  const int m = q * 32 + lane;                         // accumulator row = tile pixel
  const int64_t plane = p.plane;
  const int64_t stiles = p.splane >> 7;                // state tiles per slot (S[slot][tile][Cq][128][4])
  // y staging (p.ystage): this warp's 32 rows x CE bf16 channels, 16-B units
  // swizzled so both the row-wise writes and the column-wise reads are
  // conflict-free per quarter warp
  constexpr int YU = CE / 8;                           // 16-B units per row
  uint4* ybuf = reinterpret_cast<uint4*>(smem + p.y_off) + warp * 32 * YU;
  auto yswz = [](int row) { return (row / (8 / YU)) & (YU - 1); };
  // One work (an item at one tick) of this group: buf / bph pick the accumulator,
  // tk the chunk's tick row (nullptr: the launch's single tick from p).  Called
  // from two loops so the one-step path keeps its own (lower) register use.
  // STEM: build CTA-local tile T's W-im2col image from its raw rows (this
  // group's 128 CS threads), then release the raw buffer and publish the image
  const int gtid = threadIdx.x - e * 128 * CS;          // thread index inside the group
  auto convert = [&](int64_t T) {
    if constexpr (!kStem) return;
    const int64_t tile = int64_t(blockIdx.x) + T * grid;
    if (tile >= p.n_tiles) return;
    const int b = int(T & 1);
    const uint32_t tph = uint32_t(T >> 1) & 1u;
    ptx::mbar_wait(&a_empty[b], tph ^ 1u);               // the MMA is done with tile T-2's image
    ptx::mbar_wait(&a_full[2 + b], tph);                 // tile T's raw rows landed
    const int r0 = int(tile % p.tiles_h) * p.TH * p.sh - p.ph;
    uint8_t* img = smem + b * p.st_img_bytes;
    const uint8_t* raw = smem + p.st_raw_off + b * p.st_nraw * p.st_rpitch;
    const int Wo = p.Wo, nt = p.st_nraw * Wo, gstride = p.st_img_rows * 16;
    for (int task = gtid; task < nt; task += 128 * CS) {
      const int q = task / Wo, wo = task - q * Wo;
      const int row = p.st_phase_base[q % p.sh] + (q / p.sh) * Wo + wo;
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) w[k] = 0u;
      if (p.x && r0 + q >= 0 && r0 + q < p.st_Hin) {
        // the window x[q, wo sw - pw + v, c] = padded-row elements e0 .. e0 + kwc - 1
        const int e0 = p.st_pad + (wo * p.st_sw - p.st_pw) * p.st_cin;
        const uint32_t* rw = reinterpret_cast<const uint32_t*>(raw + q * p.st_rpitch) + (e0 >> 1);
        const int nw = p.st_data_groups * 4;             // 32-bit words of the data groups
        if (e0 & 1) {                                    // window starts mid-word: funnel pairs
          uint32_t prev = rw[0];
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (k < nw) { const uint32_t nx = rw[k + 1]; w[k] = __byte_perm(prev, nx, 0x5432); prev = nx; }
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (k < nw) w[k] = rw[k];
        }
        // K index >= kw Cin: zero (the packed weights are zero there too)
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (2 * k >= p.st_kwc) w[k] = 0u;
          else if (2 * k + 1 >= p.st_kwc) w[k] &= 0xFFFFu;
        }
      }
#pragma unroll
      for (int gq = 0; gq < 4; ++gq)
        if (gq < p.st_data_groups)
          *reinterpret_cast<uint4*>(img + gq * gstride + row * 16) =
              make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
    }
    ptx::fence_proxy_async();                             // generic image writes -> tensor-core reads
    ptx::mbar_arrive(&a_empty[2 + b]);                    // raw rows consumed
    ptx::mbar_arrive(&a_full[b]);                         // image ready
  };
  // L2 prefetch of an item's state rows (every slot the step reads: the emit
  // slot and the accumulated ones), issued by one thread of the group one item
  // ahead: a (slot, tile, part) block is CC/4 channel quads x 128 rows x 16 B,
  // contiguous, so it is one bulk prefetch -- DRAM -> L2 runs ahead of the
  // epilogue's register loads, which then see L2 latency.
  auto prefetch_state = [&](const int64_t tile, const int c0v) {
    if (KT < 2 || gtid != 0 || !p.l2pf) return;
    const int64_t stiles = p.splane >> 7;
    auto one = [&](int sl) {
      const float4* src = reinterpret_cast<const float4*>(p.state) + ((int64_t(sl) * stiles + tile) * p.Cq + c0v / 4) * 128;
      ptx::bulk_prefetch_l2(src, uint32_t(CC) * 512u);
    };
    if (p.emit) one(p.slot[KT - 1]);
    if (p.update)
      for (int k = 1; k < KT - 1; ++k)
        if (p.slot[k] >= 0) one(p.slot[k]);
  };
  auto work = [&](const int64_t tile, const int c0v, const int64_t li, const int* tk) {
    const int buf = int(li % NBUF);                    // accumulator buffer of this work
    const uint32_t bph = uint32_t(li / NBUF) & 1u;
    const int emit = tk ? tk[0] : p.emit;
    const int64_t yt = tk ? int64_t(tk[1]) * p.y_tstride : 0;
    auto slot = [&](int k) -> int { return tk ? tk[2 + k] : p.slot[k]; };
    const int bias0 = (stem || p.fparts) ? c0v : 0;    // bias_s holds all Cout (STEM, floating parts) or this part's CC
    // ---- this row's output pixel
    bool valid;
    int64_t pix, b;
    if (p.mode == MODE_FLAT || p.kflat) {
      pix = tile * 128 + m;
      valid = pix < plane;
      b = valid ? pix / p.HWo : 0;
    } else if (p.mode == MODE_HALO || p.mode == MODE_KHALO) {
      b = tile / p.tiles_per_stream;
      const int ho = int(tile % p.tiles_per_stream) * p.MT + m / p.Wp;
      const int wo = m % p.Wp;
      valid = (m < p.MT * p.Wp) && (wo < p.Wo) && (ho < p.Ho) && (tile < p.n_tiles);
      pix = b * p.HWo + int64_t(ho) * p.Wo + wo;
    } else {
      const int per_stream = p.tiles_h * p.tiles_w;
      b = tile / per_stream;
      const int r = int(tile % per_stream);
      const int ho = (r / p.tiles_w) * p.TH + m / p.TW;
      const int wo = (r % p.tiles_w) * p.TW + m % p.TW;
      valid = (m < p.TH * p.TW) && (wo < p.Wo) && (ho < p.Ho) && (tile < p.n_tiles);
      pix = b * p.HWo + int64_t(ho) * p.Wo + wo;
    }
    // state row: the TMEM lane inside the tile (tile-padded layout, common.cuh)
    const int64_t stile = tile;                        // state block of this item (row m of the tile)
    const uint32_t t_row = tmem + (uint32_t(q * 32) << 16) + uint32_t(buf * BUF);
#pragma unroll 1
    for (int cb = cs * CPW; cb < (cs + 1) * CPW; cb += CE) {
      // ---- prefetch the state this pass needs (pass 0: before the accumulator is ready)
      float4 sv[NS][NQ];
      if DBG(64) {
#pragma unroll
        for (int k = 0; k < NS; ++k)
#pragma unroll
          for (int i = 0; i < NQ; ++i) sv[k][i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (KT > 1 && valid && !DBG(65)) {
        if (emit) {
          const float4* src = reinterpret_cast<const float4*>(p.state) +
                              ((int64_t(slot(KT - 1)) * stiles + stile) * p.Cq + (c0v + cb) / 4) * 128 + m;
#pragma unroll
          for (int i = 0; i < NQ; ++i) sv[0][i] = DBG(32) ? ld_state_na(src + i * 128) : __ldcs(src + i * 128);
        }
        if (p.update) {
#pragma unroll
          for (int k = 1; k < KT - 1; ++k) {
            if (slot(k) < 0) continue;
            const float4* src = reinterpret_cast<const float4*>(p.state) +
                                ((int64_t(slot(k)) * stiles + stile) * p.Cq + (c0v + cb) / 4) * 128 + m;
#pragma unroll
            for (int i = 0; i < NQ; ++i) sv[k][i] = DBG(32) ? ld_state_na(src + i * 128) : __ldcs(src + i * 128);
          }
        }
      }
      // STEM: the first part of tile T converts tile T+1 while this item's state loads fly
      if (stem && cb == cs * CPW && li % p.n_split == 0) convert(li / p.n_split + 1);
      if (cb == cs * CPW && !DBG(16)) {
        ptx::mbar_wait(&acc_full[buf], bph);
        ptx::tc_fence_after();
      }
      float v[16];
      // ---- (1) complete + emit
      if (emit) {
#pragma unroll
        for (int c = 0; c < CE; c += 16) {
          if (!DBG(8)) ptx::tmem_ld16(t_row + uint32_t((KT - 1) * CC + cb + c), v);
          ptx::tc_wait_ld();
          if (!DBG(257)) {
            // y = (P + S) + b, the activation only behind a uniform branch
            // (computed on every lane: the bf16 stores below pair lanes up)
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const float4 bb = *reinterpret_cast<const float4*>(bias_s + bias0 + cb + c + i);
              if (KT > 1) {
                const float4 t4 = sv[0][(c + i) >> 2];
                v[i] += t4.x; v[i + 1] += t4.y; v[i + 2] += t4.z; v[i + 3] += t4.w;
              }
              v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
            }
            if (p.act == 1) {
#pragma unroll
              for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            const int64_t yoff = b * p.y_bstride + yt + (pix - b * p.HWo) * p.Cout + c0v + cb + c;
            if (p.out_f32) {
              float4* yp = reinterpret_cast<float4*>(static_cast<float*>(p.y) + yoff);
              if (valid) {
#pragma unroll
                for (int i = 0; i < 4; ++i) yp[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              }
            } else {
              uint4 h[2];
#pragma unroll
              for (int i = 0; i < 2; ++i)
                h[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
              __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(p.y);
              if (p.ystage) {                   // row = lane, written out after the pass
                ybuf[lane * YU + (((c >> 3) + 0) ^ yswz(lane))] = h[0];
                ybuf[lane * YU + (((c >> 3) + 1) ^ yswz(lane))] = h[1];
              } else if DBG(512) {
                if (valid) {
                  reinterpret_cast<uint4*>(yb + yoff)[0] = h[0];
                  reinterpret_cast<uint4*>(yb + yoff)[1] = h[1];
                }
              } else {
                // A thread's 16 channels are one 32-B sector, written as two 16-B
                // halves.  Lanes 2k / 2k+1 swap halves so that each store
                // instruction writes whole sectors (even: its own first half and the
                // partner's first half; odd: the partner's second half and its own),
                // not 32 half sectors the L2 has to merge.
                const bool odd = lane & 1;
                const uint4 give = odd ? h[0] : h[1];
                uint4 got;
                got.x = __shfl_xor_sync(0xffffffffu, give.x, 1);
                got.y = __shfl_xor_sync(0xffffffffu, give.y, 1);
                got.z = __shfl_xor_sync(0xffffffffu, give.z, 1);
                got.w = __shfl_xor_sync(0xffffffffu, give.w, 1);
                const int64_t poff = __shfl_xor_sync(0xffffffffu, (long long)yoff, 1);
                const bool pvalid = __shfl_xor_sync(0xffffffffu, int(valid), 1) != 0;
                // store 1: the even lane's pixel (first half by even, second by odd)
                if (odd ? pvalid : valid)
                  *reinterpret_cast<uint4*>(yb + (odd ? poff + 8 : yoff)) = odd ? got : h[0];
                // store 2: the odd lane's pixel
                if (odd ? valid : pvalid)
                  *reinterpret_cast<uint4*>(yb + (odd ? yoff + 8 : poff)) = odd ? h[1] : got;
              }
            }
          }
        }
        if (p.ystage && !DBG(257)) {
          // the warp's 32 rows go out row-contiguously: 32 / YU rows of CE
          // channels per store instruction (whole 2 CE-byte runs, not 16-B pieces)
          __syncwarp();
          const int64_t ybase = b * p.y_bstride + yt + (pix - b * p.HWo) * p.Cout + c0v + cb;
          __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(p.y);
#pragma unroll
          for (int j = 0; j < YU; ++j) {
            const int q = j * (32 / YU) + lane / YU, k = lane % YU;
            const uint4 val = ybuf[q * YU + (k ^ yswz(q))];
            const int64_t qoff = __shfl_sync(0xffffffffu, (long long)ybase, q);
            const bool qv = __shfl_sync(0xffffffffu, int(valid), q) != 0;
            if (qv) *reinterpret_cast<uint4*>(yb + qoff + 8 * k) = val;
          }
          __syncwarp();
        }
      }
      if (p.update && KT > 1) {
        // ---- (2) accumulate into pending outputs
#pragma unroll
        for (int k = KT - 2; k >= 1; --k) {
          if (slot(k) < 0) continue;
          float4* dst = reinterpret_cast<float4*>(p.state) +
                        ((int64_t(slot(k)) * stiles + stile) * p.Cq + (c0v + cb) / 4) * 128 + m;
#pragma unroll
          for (int c = 0; c < CE; c += 16) {
            if (!DBG(8)) ptx::tmem_ld16(t_row + uint32_t(k * CC + cb + c), v);
            ptx::tc_wait_ld();
            if (valid && !DBG(1)) {
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                float4 t4 = sv[k][c / 4 + i];
                t4.x += v[4 * i]; t4.y += v[4 * i + 1]; t4.z += v[4 * i + 2]; t4.w += v[4 * i + 3];
                if (!DBG(128)) st_state(p, dst + (c / 4 + i) * 128, t4);
              }
            }
          }
        }
        // ---- (3) start the newest output (overwrites the emitted slot)
        if (slot(0) >= 0) {
          float4* dst = reinterpret_cast<float4*>(p.state) +
                        ((int64_t(slot(0)) * stiles + stile) * p.Cq + (c0v + cb) / 4) * 128 + m;
#pragma unroll
          for (int c = 0; c < CE; c += 16) {
            if (!DBG(8)) ptx::tmem_ld16(t_row + uint32_t(cb + c), v);
            ptx::tc_wait_ld();
            if (valid && !DBG(1)) {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (!DBG(128)) st_state(p, dst + (c / 4 + i) * 128, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
            }
          }
        }
      }
    }
    // accumulator consumed: every tcgen05.ld above was waited on (wait::ld), so a
    // relaxed arrive suffices -- the state / y stores need no ordering with the
    // MMA warp, and a release arrive would stall on them (ptx::mbar_arrive_relaxed)
    ptx::tc_fence_before();
    if constexpr (PAIR == 2) ptx::mbar_arrive_cluster_relaxed(ptx::mapa(ptx::smem_u32(&acc_empty[buf]), 0));
    else ptx::mbar_arrive_relaxed(&acc_empty[buf]);
  };
  if (stem) {
    // CTA-local works li = (tile T, part li mod n_split); group e takes every EG-th
    const int64_t n_t = p.n_tiles > blockIdx.x ? (p.n_tiles - blockIdx.x + grid - 1) / grid : 0;
    auto tile_li = [&](int64_t li) { return int64_t(blockIdx.x) + (li / p.n_split) * grid; };
    if (e == 0) convert(0);
    if (e < n_t * p.n_split) prefetch_state(tile_li(e), int(e % p.n_split) * CC);
    for (int64_t li = e; li < n_t * p.n_split; li += EG) {
      if (li + EG < n_t * p.n_split) prefetch_state(tile_li(li + EG), int((li + EG) % p.n_split) * CC);
      work(tile_li(li), int(li % p.n_split) * CC, li, nullptr);
    }
  } else if (!p.ticks) {
    int64_t li = e;
    const int64_t step = EG * int64_t(n_units);
    auto c0_of = [&](int64_t item) { return p.fparts ? int(item % p.n_split) * CC : c0; };
    if (unit + int64_t(e) * n_units < p.n_items)
      prefetch_state(tile_of(unit + int64_t(e) * n_units), c0_of(unit + int64_t(e) * n_units));
    for (int64_t item = unit + int64_t(e) * n_units; item < p.n_items; item += step, li += EG) {
      if (item + step < p.n_items) prefetch_state(tile_of(item + step), c0_of(item + step));
      work(tile_of(item), c0_of(item), li, nullptr);
    }
  } else {
    // chunked: item bi + e n_units of every batch, all T frames in order; the work
    // index over the unit's sequence (batch-major, then frame, then item) picks the buffer
    int64_t wbase = 0;
    for (int64_t bi = unit; bi < p.n_items; bi += int64_t(EG) * n_units) {
      const int64_t left = (p.n_items - bi + n_units - 1) / n_units;
      const int nb = left < EG ? int(left) : EG;
      for (int t = 0; e < nb && t < p.T; ++t)
        work(tile_of(bi + int64_t(e) * n_units), c0, wbase + int64_t(t) * nb + e, p.ticks + t * kTickInts);
      wbase += int64_t(nb) * p.T;
    }
  }
  }
  // ===================== teardown (all threads) =====================
  ptx::tc_fence_before();
  if (CLU > 1) ptx::cluster_sync(); else __syncthreads();   // no CTA leaves while peers may still signal it
  if (warp == kMma) {
    ptx::tc_fence_after();
    if constexpr (PAIR == 2) ptx::tmem_dealloc_pair(tmem, TMEM_COLS);
    else ptx::tmem_dealloc(tmem, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host side

__global__ void k_pack_tc_weights(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int Cout,
                                  int Cin, int kt, int kh, int kw, int CC, int n_split, int pair, int kblk) {
  // kblk > 0 (KLOOP CTA pairs): [part][half][K/kblk][N/pair][kblk] instead --
  // kblk-element (128-B / 64-B) rows a swizzled TMA box loads in one request
  // (Cout, Cin, kt, kh, kw) -> [part][half][K/8][N/pair][8], N = kt*CC rows
  // (n = k*CC + c; a CTA pair splits them into halves n < N/2 and n >= N/2),
  // K index = (u*kw + v)*Cin + ci.  Each K chunk of a tap is one contiguous block.
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
  const int NB = N / pair, half = n / NB, nn = n - half * NB;
  if (kblk)
    out[int64_t(part * pair + half) * K * NB + ((kidx / kblk) * NB + nn) * kblk + (kidx % kblk)] = w[i];
  else
    out[int64_t(part * pair + half) * K * NB + ((kidx / 8) * NB + nn) * 8 + (kidx % 8)] = w[i];
}

// W-im2col of the weights for a small-Cin stem: (Cout, Cin, kt, kh, kw) ->
// (Cout, Kp, kt, kh, 1) with channel j = v*Cin + c (zero for j >= kw*Cin).
__global__ void k_wcols_weights(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ out, int Cout,
                                int Cin, int kt, int kh, int kw, int Kp) {
  const int64_t total = int64_t(Cout) * Kp * kt * kh;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= total) return;
  int64_t r = i;
  const int u = int(r % kh); r /= kh;
  const int k = int(r % kt); r /= kt;
  const int j = int(r % Kp); r /= Kp;
  const int o = int(r);
  __nv_bfloat16 val = __float2bfloat16_rn(0.f);
  if (j < kw * Cin) {
    const int v = j / Cin, c = j % Cin;
    val = w[(((int64_t(o) * Cin + c) * kt + k) * kh + u) * kw + v];
  }
  out[i] = val;
}

// W-im2col of one step's frame: xp[b][h][wo][j] = x[b][h][wo*sw + v*dw - pw][c],
// j = v*Cin + c, zero outside the frame and for j >= kw*Cin.  One thread per
// output pixel builds its KP channels in registers (unrolled, compile-time j)
// and writes them as KP/8 16-byte stores (consecutive threads, consecutive
// 2*KP-byte rows); the inputs it reads overlap its neighbours' (L1 hits).
template <int KP, int CIN = 0>
__global__ void __launch_bounds__(256) k_wcols_frame(const __nv_bfloat16* __restrict__ x, int64_t x_bstride,
                                                     __nv_bfloat16* __restrict__ xp, int64_t B, int H, int W,
                                                     int Cin_rt, int Wo, int kw, int sw, int dw, int pw) {
  // CIN > 0: the channel count at compile time (RGB stems), so the unrolled
  // j -> (v, c) split is free instead of a runtime division per channel
  const int Cin = CIN > 0 ? CIN : Cin_rt;
  const int64_t total = B * H * Wo;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // the warp's 32 pixels are one contiguous run of xp: staged in shared memory
  // and stored linearly, 512 contiguous bytes per store instruction
  __shared__ __align__(16) uint4 stage[256 * (KP / 8)];
  const bool live = i < total;                                  // (all lanes stay for the warp's stores)
  const int64_t ic = live ? i : total - 1;
  const int wo = int(ic % Wo);
  const int64_t r = ic / Wo;
  const int h = int(r % H);
  const int64_t b = r / H;
  const __nv_bfloat16* xr = x ? x + b * x_bstride + int64_t(h) * W * Cin : nullptr;
  __align__(16) __nv_bfloat16 vals[KP];
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
#pragma unroll
  for (int j = 0; j < KP; ++j) {
    __nv_bfloat16 val = zero;
    const int v = j / Cin, c = j - (j / Cin) * Cin;
    const int wi = wo * sw + v * dw - pw;
    if (xr && v < kw && wi >= 0 && wi < W) val = xr[int64_t(wi) * Cin + c];
    vals[j] = val;
  }
  constexpr int U = KP / 8;                                     // 16-B units per pixel
  const int lane = threadIdx.x & 31;
  uint4* ws = stage + (threadIdx.x & ~31) * U;
  const int64_t wbase = i - lane;
  const int nw = (total - wbase) < 32 ? int(total - wbase) : 32;
#pragma unroll
  for (int t = 0; t < U; ++t) ws[lane * U + ((t + lane) % U)] = reinterpret_cast<const uint4*>(vals)[t];
  __syncwarp();
  uint4* dst = reinterpret_cast<uint4*>(xp + wbase * KP);
#pragma unroll
  for (int t = 0; t < U; ++t) {
    const int k = t * 32 + lane, px = k / U, u = k % U;
    if (px < nw) dst[k] = ws[px * U + ((u + px) % U)];
  }
}

typedef void (*KernFn)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const TcParams);

struct Variant {
  int KT, CC, EG, CE;
  KernFn fn;
  int KH = 0, KW = 0, KC = 0;     // > 0: specialised (unrolled) HALO/FLAT variant for this kernel / Cin
  int CS = 1;                     // epilogue warps per TMEM lane quadrant (column split)
  int PAIR = 1;                   // 2: CTA pairs (cta_group::2, M = 256), HALO / FLAT only
  int STEM = 0;                   // 1: the MODE_STEM instantiation (shared-memory W-im2col)
};

#define CO_TC_VARIANT(kt, cc, eg, ce) {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce>}
#define CO_TC_SPEC(kt, cc, eg, ce, kh, kw, kc) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, kh, kw, kc>, kh, kw, kc}
#define CO_TC_SPLIT(kt, cc, eg, ce, kh, kw, kc, cs) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, kh, kw, kc, cs>, kh, kw, kc, cs}
#define CO_TC_PAIRG(kt, cc, eg, ce) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, 0, 0, 0, 1, 2>, 0, 0, 0, 1, 2}
#define CO_TC_PAIR(kt, cc, eg, ce, kh, kw, kc) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, kh, kw, kc, 1, 2>, kh, kw, kc, 1, 2}
// CTA pairs whose one epilogue group splits every item's channels over 2 x 4 warps
// (CS = 2): an item's state traffic is drained by 8 warps at once instead of 4
#define CO_TC_PAIRGS(kt, cc, eg, ce, cs) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, 0, 0, 0, cs, 2>, 0, 0, 0, cs, 2}
// KHALO pairs with compile-time 3 x 3 taps (the C4 layers): KH = KW = 3, KC = 0
#define CO_TC_KH3(kt, cc, eg, ce) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, 3, 3, 0, 1, 2>, 3, 3, 0, 1, 2}
#define CO_TC_STEMV(kt, cc, eg, ce) \
  {kt, cc, eg, ce, (KernFn)k_step_dense_tc<kt, cc, eg, ce, 0, 0, 0, 1, 1, true>, 0, 0, 0, 1, 1, 1}
const Variant kVariants[] = {
    CO_TC_PAIR(3, 32, 2, 32, 3, 3, 4), CO_TC_PAIR(3, 32, 3, 32, 3, 3, 4), CO_TC_PAIR(9, 16, 2, 16, 1, 1, 16),
    CO_TC_PAIR(1, 128, 2, 32, 3, 3, 4), CO_TC_SPEC(1, 128, 2, 32, 3, 3, 4), CO_TC_PAIR(3, 64, 2, 32, 3, 3, 4),
    CO_TC_PAIRG(3, 64, 2, 32), CO_TC_PAIRG(5, 32, 2, 16), CO_TC_PAIRG(1, 256, 2, 32), CO_TC_KH3(3, 64, 2, 32),
#ifdef CO_EXPERIMENTS
    CO_TC_PAIRGS(3, 64, 1, 32, 2), CO_TC_PAIRG(3, 32, 3, 32),   // measured slower on C4 L3 / L4 / L5
#endif
    CO_TC_SPLIT(3, 32, 2, 16, 3, 3, 4, 2), CO_TC_SPLIT(3, 32, 3, 16, 3, 3, 4, 2),
    CO_TC_SPEC(3, 32, 2, 32, 3, 3, 4), CO_TC_SPEC(3, 32, 3, 32, 3, 3, 4), CO_TC_SPEC(9, 16, 2, 16, 1, 1, 16),
    CO_TC_VARIANT(1, 32, 4, 32), CO_TC_VARIANT(1, 64, 4, 32), CO_TC_VARIANT(1, 128, 2, 32),
    CO_TC_VARIANT(1, 256, 2, 32),
    CO_TC_VARIANT(2, 32, 4, 32), CO_TC_VARIANT(2, 64, 2, 32), CO_TC_VARIANT(3, 16, 4, 16),
    CO_TC_VARIANT(3, 32, 2, 32), CO_TC_VARIANT(3, 32, 3, 32), CO_TC_VARIANT(3, 32, 4, 32),
    CO_TC_VARIANT(3, 64, 2, 32), CO_TC_VARIANT(5, 16, 4, 16), CO_TC_VARIANT(5, 32, 2, 16),
    CO_TC_VARIANT(5, 32, 3, 16),
    CO_TC_VARIANT(9, 16, 2, 16),
    // STEM twins of the K-pipeline variants small-Cin stems plan to (plan_stem)
    CO_TC_STEMV(1, 64, 4, 32), CO_TC_STEMV(2, 32, 4, 32), CO_TC_STEMV(3, 32, 3, 32), CO_TC_STEMV(5, 32, 3, 16),
    CO_TC_STEMV(9, 16, 2, 16),
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
  Geom gk;                        // geometry the kernel sees (the W-im2col'd one for a stem)
  int wcols = 0, Kp = 0;          // small-Cin stem packed W-im2col
  int swa = 0;                    // HALO: 128-B swizzled A (Cin % 64 == 0)
  int kflat = 0;                  // RAW 1x1: KLOOP over flattened 128-row tiles
  int mode = MODE_HALO;
  int n_split = 0, MT = 0, Wp = 0, tiles_per_stream = 0;
  int TH = 0, TW = 0, tiles_h = 0, tiles_w = 0, kb = 0, n_cb = 0, b_bytes = 0, b_off = 0;
  int a_bytes = 0, a_stride = 0, chunk_stride = 0, w_bytes = 0, w_off = 0, stages = 2;
  int ystage = 0, y_off = 0;      // HALO bf16: y stores transposed through shared memory
  int ka_stages = 0, ka_stride = 0, ka_phase = 0, dmin_h = 0, dmin_w = 0;   // KHALO input-halo ring
  // STEM (fused W-im2col): raw rows per tile, padded raw-row pitch / left pad, image rows / bytes
  int st_nraw = 0, st_rpitch = 0, st_pad = 0, st_img_rows = 0, st_img_bytes = 0, st_raw_off = 0;
  int st_groups = 0, st_data_groups = 0, st_phase_base[2] = {0, 0};
  int fparts = 0;                 // KHALO: channel parts float over items (all SMs busy)
  int64_t n_tiles = 0;
  size_t smem = 0;
};

constexpr size_t kSmemLimit = 227 * 1024;
// Shared memory the planner fills before it takes more stages: beyond ~190 KB
// the L1 left over (< ~38 KB) can no longer land the epilogue's in-flight
// state loads and HBM throughput drops ~20% (measured: scripts/bw_probe.cu,
// full bandwidth at 190 KB of shared memory, -18% at 200 KB).
constexpr size_t kSmemBudget = 190 * 1024;
// HALO (weights resident): a lower budget.  Its epilogue warps carry the whole
// state RMW, so L1 room for in-flight loads beats deeper A pipelines:
// C2 measured 1.19 M (one CTA, 173 KB) / 1.19 M (pair, 4 stages, 177 KB) /
// 1.24 M (pair, 3 stages, 147 KB) / 1.20 M (pair, 2 stages, 117 KB); C4 layer 2
// (pair) 0.438 ms at 164 KB, 0.391 ms at 134 KB.
constexpr size_t kHaloBudget = 150 * 1024;

// 128-B swizzled A operand (TMA boxes with 128-B rows instead of 16-B ones):
// default on, CO_TC_SWA=0 restores the interleaved layout (A/B runs).
bool swa_enabled() { return CO_EXP("CO_TC_SWA", 1) != 0; }

// KLOOP CTA pairs (each CTA streams half of every weight chunk through a
// swizzled 128-B-row TMA box): default for 64-channel K chunks (C4 L3 / L5
// measured ~8% faster, L4 equal); 32-channel chunks (the stem) stay single.
// option "kpair" (co_set_option) = 1 | 2 pins it.
int kloop_pair(int kb) {
  const int v = int(option(OPT_KPAIR));
  return v ? v : (kb == 64 ? 2 : 1);
}

int pinned_cs() { return CO_EXP("CO_TC_CS", 1); }           // A/B experiments only
int pinned_eg() { return int(option(OPT_EG)); }              // option "eg": 0 = planner's choice
int pinned_cc() { return CO_EXP("CO_TC_CC", 0); }           // A/B experiments only
int pinned_ce() { return CO_EXP("CO_TC_CE", 0); }           // A/B experiments only

// y stores transposed through shared memory (HALO, bf16 y; CO_TC_YSTAGE in experiment builds)
int ystage_mode() { return CO_EXP("CO_TC_YSTAGE", 1); }

// KHALO for stride-1 K-pipeline layers (option "khalo" = 0 keeps KLOOP)
bool khalo_enabled() { return option(OPT_KHALO) != 0; }

int pinned_stages() {                                         // A/B experiments: cap the A pipeline depth
  return std::max(2, CO_EXP("CO_TC_STAGES", kMaxStagesStd));
}

// HALO / FLAT: weights resident.  Largest CC whose weights + 2 A stages fit.
bool plan_resident(const Geom& g, Plan& pl) {
  if (g.sh != 1 || g.sw != 1 || g.dh != 1 || g.dw != 1 || g.Cin % 16 != 0 || g.Cin / 8 > 256) return false;
  const bool flat = (g.kh == 1 && g.kw == 1 && g.ph == 0 && g.pw == 0);
  int Wp = 1, MT = 1, a_rows = 128;
  if (!flat) {
    Wp = g.Wo + g.kw - 1;
    if (Wp > 128) return false;
    MT = std::min(128 / Wp, g.Ho);
    const int halo_rows = MT + g.kh - 1;
    if (halo_rows > 256) return false;
    a_rows = Wp * halo_rows;
  }
  const int a_bytes = (g.Cin / 8) * a_rows * 16;
  const int a_stride = ((a_bytes + kApad + 1023) / 1024) * 1024;
  // The MMA of tap (u, v) reads 128 rows from row u Wp + v of every channel
  // block: up to (kh-1) Wp + kw - 1 + 128 rows, past the box into the next
  // stage (junk rows, discarded) -- and past the LAST stage into whatever
  // follows, so the allocation keeps that over-read inside shared memory.
  const int max_row = flat ? 128 : (g.kh - 1) * Wp + (g.kw - 1) + 128;
  const int over = std::max(0, (max_row - a_rows) * (g.Cin % 64 == 0 && swa_enabled() ? 128 : 16));
  const size_t tail = size_t(std::max(0, over - (a_stride - a_bytes)));
  const int64_t K = int64_t(g.Cin) * g.kh * g.kw;
  // FLAT (C5's 64 KB A stages) keeps the general budget: its pair fits only there
  const size_t budget = flat ? kSmemBudget : kHaloBudget;
  const int eg_pin = pinned_eg();
  const int pair_pin = int(option(OPT_PAIR));     // option "pair": 0 auto, 1 / 2 pinned
  const Variant* best = nullptr;
  int64_t best_rank = -1;
  for (const Variant& v : kVariants) {
    if (v.KT != g.kt || g.Cout % v.CC != 0 || v.STEM) continue;
    if (v.KH && (v.KH != g.kh || v.KW != g.kw || v.KC * 16 != g.Cin)) continue;
    if ((eg_pin && v.EG != eg_pin) || (pinned_cc() && v.CC != pinned_cc()) || (pinned_ce() && v.CE != pinned_ce()))
      continue;
    if (v.CS != pinned_cs() || (pair_pin && v.PAIR != pair_pin)) continue;
    const int64_t w_bytes = int64_t(v.KT * v.CC) * K * 2 / v.PAIR;   // per CTA
    const size_t fixed = 1024 + size_t((w_bytes + 1023) / 1024 * 1024) + 512 + v.CC * 4 + tail;
    if (fixed + 2 * size_t(a_stride) > kSmemLimit) continue;
    const bool fits = fixed + 2 * size_t(a_stride) <= budget;
    // prefer: staying under the L1 budget (a CTA pair halves the resident
    // weights), a specialised (unrolled) variant, one CTA over a pair when both
    // fit (the pair's 64-channel epilogue costs more than its MMA saves), more
    // channels per part, more epilogue groups
    const int64_t rank = (fits ? 100000000 : 0) + (v.KH ? 10000000 : 0) + (v.PAIR == 1 ? 1000000 : 0) + v.CC * 1000 + v.EG;
    if (rank > best_rank) {
      best = &v;
      best_rank = rank;
      pl.w_bytes = int(w_bytes);
      const size_t cap = fits ? budget : kSmemLimit;
      pl.stages = int(std::min<size_t>(pinned_stages(), (cap - fixed) / size_t(a_stride)));
      pl.smem = fixed + size_t(pl.stages) * a_stride;
    }
  }
  if (!best) return false;
  if (!flat && ystage_mode() && best->CS == 1) {
    // per epilogue warp 32 rows x CE bf16 channels, after the stages, the
    // barriers / bias and the over-read tail
    const size_t ybytes = size_t(best->EG) * 4 * 32 * best->CE * 2;
    const size_t w_al = (size_t(pl.w_bytes) + 1023) / 1024 * 1024;
    const size_t rest = 512 + best->CC * 4 + tail;
    for (int st = pl.stages; st >= 2; --st) {
      const size_t y_off = (w_al + size_t(st) * a_stride + rest + 1023) / 1024 * 1024;
      if (1024 + y_off + ybytes <= kSmemLimit) {
        pl.ystage = 1;
        pl.y_off = int(y_off);
        pl.stages = st;
        pl.smem = 1024 + y_off + ybytes;
        break;
      }
    }
  }
  pl.var = best;
  pl.mode = flat ? MODE_FLAT : MODE_HALO;
  pl.MT = MT;
  pl.Wp = Wp;
  pl.a_bytes = a_bytes;
  pl.a_stride = a_stride;
  pl.chunk_stride = a_rows * 16;
  pl.w_off = (pl.w_bytes + 1023) / 1024 * 1024;
  if (flat) {
    pl.n_tiles = (g.B * g.HWo + 127) / 128;
  } else {
    pl.tiles_per_stream = (g.Ho + MT - 1) / MT;
    pl.n_tiles = g.B * pl.tiles_per_stream;
  }
  return true;
}

// KLOOP: K streamed through a stage ring; any spatial stride/dilation <= 8.
int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

bool plan_kloop(const Geom& g, Plan& pl, bool flat = false) {
  if (g.Cin % 16 != 0 || g.Cin / 8 > 256 || g.sh > 8 || g.sw > 8) return false;
  // flat: rows are 128 consecutive (stream, pixel) pairs (RAW 1x1 layers)
  const int TW = flat ? 128 : std::min(g.Wo, 128);
  const int TH = flat ? 1 : std::max(1, std::min(128 / TW, g.Ho));
  if (TW * g.sw > 256 || TH * g.sh > 256) return false;
  const int kb = (g.Cin % 64 == 0) ? 64 : (g.Cin % 32 == 0) ? 32 : 16;
  const int rows = TH * TW;
  const int a_bytes = (kb / 8) * rows * 16;
  const int eg_pin = pinned_eg();
  const Variant* best = nullptr;
  const int want = kloop_pair(kb);
  for (int pair : {want, 3 - want}) {           // the preferred pairing, else the other
    if (option(OPT_KPAIR) && pair != want) break;
    for (const Variant& v : kVariants) {
      // K-pipeline pairs may split an item's channels over 2 x 4 epilogue warps (CS = 2)
      // KC == 0 KH / KW variants: compile-time taps of the K pipeline (KHALO), this kernel size only
      if (v.KT != g.kt || g.Cout % v.CC != 0 || v.PAIR != pair || v.STEM) continue;
      if (v.KH && (v.KC != 0 || v.KH != g.kh || v.KW != g.kw || !CO_EXP("CO_TC_KH3", 1))) continue;
      if (v.PAIR == 2 && v.KT == 1 && !flat) continue;        // kt = 1 pairs: the RAW flat window contractions
      if (v.CS != 1 && !(pair == 2 && v.CS == 2 && CO_EXP("CO_TC_KCS", 0))) continue;
      if ((eg_pin && v.EG != eg_pin) || (pinned_cc() && v.CC != pinned_cc())) continue;
      // prefer a width whose items fill at least half the SMs, then the widest
      // N (fewest A re-reads), then more groups (MHA: the 1024 x 1024 output
      // projection is 32 items at N = 256, 128 at N = 64)
      const int64_t tiles = flat ? (g.B * g.HWo + 127) / 128 : g.B * ((g.Ho + TH - 1) / TH) * ((g.Wo + TW - 1) / TW);
      auto rank = [&](const Variant* x) {
        const int64_t items = (tiles + x->PAIR - 1) / x->PAIR * (g.Cout / x->CC) * x->PAIR;
        const bool fills = !CO_EXP("CO_TC_FILL", 1) ? true : items * 2 >= sm_count();
        return (fills ? 1000000 : 0) + x->CC * 1000 + (x->CS == 2 ? 500 : 0) + (x->KH ? 100 : 0) + x->EG;
      };
      if (!best || rank(&v) > rank(best)) best = &v;
    }
    if (best) break;
  }
  if (!best) return false;
  const int N = best->KT * best->CC;
  const int b_bytes = (kb / 8) * (N / best->PAIR) * 16;      // this CTA's share of a B chunk
  // A chunk, slack for the junk rows the 128-row MMA reads past it, then B
  // swizzled A (kb == 64): 128-B rows; the 128-row MMA reads up to 16 KB
  const int swa = !swa_enabled() ? 0 : kb == 64 ? 1 : kb == 32 ? 2 : 0;
  int b_off = swa ? std::max(a_bytes, 128 * kb * 2) : (a_bytes + (128 - rows) * 16 + 127) / 128 * 128;
  if (best->PAIR == 2) b_off = (b_off + 1023) / 1024 * 1024;   // swizzled B rows: 1 KB-aligned atoms
  const int stage = (b_off + b_bytes + 1023) / 1024 * 1024;
  const size_t fixed = 1024 + 512 + best->CC * 4 + 64 * 4;   // + the KHALO tap table
  const size_t cap = (fixed + 2 * size_t(stage) <= kSmemBudget) ? kSmemBudget : kSmemLimit;
  const int ks = CO_EXP("CO_TC_KSTAGES", 0);     // A/B experiments only: cap the K pipeline depth
  const int stages = int(std::min<size_t>(ks ? std::max(2, ks) : kMaxStagesStd, (cap - fixed) / size_t(stage)));
  if (stages < 2) return false;
  pl.var = best;
  pl.mode = MODE_KLOOP;
  pl.TH = TH; pl.TW = TW;
  pl.tiles_h = (g.Ho + TH - 1) / TH;
  pl.tiles_w = (g.Wo + TW - 1) / TW;
  pl.kb = kb; pl.n_cb = g.Cin / kb;
  pl.a_bytes = a_bytes; pl.b_bytes = b_bytes; pl.b_off = b_off;
  pl.a_stride = stage;
  pl.stages = stages;
  pl.chunk_stride = rows * 16;
  pl.swa = swa;
  pl.w_bytes = int(int64_t(N / best->PAIR) * g.Cin * g.kh * g.kw * 2);
  pl.w_off = 0;
  pl.smem = fixed + size_t(stages) * stage;
  pl.n_tiles = g.B * pl.tiles_h * pl.tiles_w;
  pl.kflat = flat;
  if (flat) { pl.tiles_h = 1; pl.tiles_w = 1; pl.n_tiles = (g.B * g.HWo + 127) / 128; }
  // KHALO: stride s <= 2 (s x s phase halos), dilation 1, 64-channel blocks,
  // phase boxes of <= 256 elements per dimension
  auto fdiv = [](int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); };
  const int sh = g.sh, sw = g.sw;
  const int dmin_h = fdiv(-g.ph, sh), dmin_w = fdiv(-g.pw, sw);
  const int Wq = g.Wo + fdiv(g.kw - 1 - g.pw, sw) - dmin_w;     // phase-halo row width
  const int MT = Wq <= 128 ? std::min(128 / Wq, g.Ho) : 0;
  const int prow = MT + fdiv(g.kh - 1 - g.ph, sh) - dmin_h;      // phase-halo rows
  if (khalo_enabled() && !flat && !g.raw && swa == 1 && sh == sw && sh <= 2 && g.dh == 1 && g.dw == 1 && MT > 0 &&
      g.kh * g.kw <= 64 &&
      prow * sh <= 256 && Wq * sw <= 256) {
    const int a_rows = Wq * prow;
    const int ka_phase = (a_rows * 128 + 1023) / 1024 * 1024;
    const int ka_stride = ka_phase * sh * sw;
    const int b_stride = (b_bytes + 1023) / 1024 * 1024;
    const int ka_stages = 2;
    // the last phase's taps read up to (prow - MT) Wq + (Wq - Wo) rows past its
    // start + 128: inside the next phase / stage / the weight ring (junk rows)
    // floating channel parts (weights stream per item anyway): a CTA may take any
    // part's item, so the grid fills every SM (C4 L3-L5: 144 -> 148); its bias
    // table then holds all Cout
    const int fparts = (g.Cout / best->CC > 1 && CO_EXP("CO_TC_FPARTS", 1)) ? 1 : 0;
    const size_t fixed2 = fixed + size_t(ka_stages) * ka_stride + (fparts ? size_t(g.Cout - best->CC) * 4 : 0);
    // the K-pipelined layers are tensor-bound and their epilogues wait on the
    // MMA, so the weight ring takes all of shared memory (C4: L3 1.73 -> 1.42 ms,
    // L5 1.53 -> 1.39 ms against the 190 KB budget); CO_TC_KHALO_SMEM (KB, experiment builds) caps it
    const int kf = CO_EXP("CO_TC_KHALO_SMEM", 0);
    const size_t cap2 = kf ? std::min(kSmemLimit, size_t(kf) * 1024) : kSmemLimit;
    const int bst = fixed2 + 2 * size_t(b_stride) <= cap2
                        ? int(std::min<size_t>(ks ? std::max(2, ks) : kMaxStages, (cap2 - fixed2) / size_t(b_stride)))
                        : 0;
    const size_t over = size_t((prow - MT) * Wq + (Wq - g.Wo) + 128) * 128;
    if (bst >= 2 && over <= size_t(ka_phase) + size_t(bst) * b_stride) {
      pl.mode = MODE_KHALO;
      pl.MT = MT; pl.Wp = Wq;
      pl.tiles_per_stream = (g.Ho + MT - 1) / MT;
      pl.n_tiles = g.B * pl.tiles_per_stream;
      pl.TH = pl.TW = pl.tiles_h = pl.tiles_w = 0;
      pl.a_bytes = a_rows * 128;                 // per phase box
      pl.ka_stages = ka_stages; pl.ka_stride = ka_stride; pl.ka_phase = ka_phase;
      pl.dmin_h = dmin_h; pl.dmin_w = dmin_w;
      pl.a_stride = b_stride; pl.b_off = 0;
      pl.stages = bst;
      pl.w_off = ka_stages * ka_stride;
      pl.chunk_stride = a_rows * 16;
      pl.smem = fixed2 + size_t(bst) * b_stride;
      pl.fparts = fparts;
    }
  }
  return true;
}

// STEM: the W-im2col of a small-Cin stem built in shared memory from raw rows
// (MODE_STEM above) instead of an HBM pass.  Takes the K-pipeline plan of the
// W-im2col'd layer (variant, weight chunks) and replaces its A operand.
bool plan_stem(const Geom& g, Plan& pl) {
  const Geom& k = pl.gk;
  if (!option(OPT_STEM) || pl.mode != MODE_KLOOP || pl.var->PAIR != 1 || pl.var->CS != 1) return false;
  // an STM instantiation for this kt: the widest channel part, then more epilogue groups
  const Variant* twin = nullptr;
  for (const Variant& v : kVariants)
    if (v.STEM && v.KT == g.kt && g.Cout % v.CC == 0 &&
        (!twin || v.CC * 100 + v.EG > twin->CC * 100 + twin->EG))
      twin = &v;
  if (!twin) return false;
  if (pl.tiles_w != 1 || pl.TW != g.Wo || k.sh > 2 || g.dh != 1 || g.dw != 1 || (k.Cin != 16 && k.Cin != 32)) return false;
  if ((int64_t(g.W) * g.Cin * 2) % 16 != 0 || pl.kb != k.Cin) return false;
  const int sh = k.sh, TH = pl.TH, Wo = g.Wo;
  const int nraw = (TH - 1) * sh + k.kh;
  int base[2] = {0, 0}, rows = 0;
  for (int ph = 0; ph < sh; ++ph) {
    base[ph] = rows;
    rows += ((nraw - ph + sh - 1) / sh) * Wo;
  }
  const int img_rows = rows + 128;                        // + the 128-row MMA's over-read past the last phase
  const int groups = k.Cin / 8, data_groups = (g.kw * g.Cin + 7) / 8;
  const int img_bytes = (groups * img_rows * 16 + 1023) / 1024 * 1024;
  // padded raw row: zeros before (>= pw Cin + 1 for the mid-word funnel) and after the data
  const int pad = ((g.pw * g.Cin + 1 + 7) / 8) * 8;
  const int max_e = pad + ((Wo - 1) * g.sw - g.pw) * g.Cin + data_groups * 8 + 1;
  const int rpitch = ((std::max(pad + g.W * g.Cin, max_e + 1) * 2 + 15) / 16) * 16;
  const int raw_off = 2 * img_bytes;
  const int w_off = ((raw_off + 2 * nraw * rpitch) + 1023) / 1024 * 1024;
  const int N = twin->KT * twin->CC;
  const int b_bytes = (pl.kb / 8) * N * 16;               // one tap's weight chunk of one part
  const int b_stride = (b_bytes + 1023) / 1024 * 1024;
  const size_t fixed = 1024 + 512 + size_t(g.Cout) * 4 + 64 * 4 + size_t(w_off);
  const int stages = int(std::min<size_t>(kMaxStagesStd, (kSmemBudget > fixed ? kSmemBudget - fixed : 0) / b_stride));
  if (stages < 2 || fixed + size_t(stages) * b_stride > kSmemLimit) return false;
  pl.mode = MODE_STEM;
  pl.var = twin;
  pl.st_nraw = nraw; pl.st_rpitch = rpitch; pl.st_pad = pad; pl.st_img_rows = img_rows; pl.st_img_bytes = img_bytes;
  pl.st_raw_off = raw_off; pl.st_groups = groups; pl.st_data_groups = data_groups;
  pl.st_phase_base[0] = base[0]; pl.st_phase_base[1] = base[1];
  pl.w_off = w_off;
  pl.b_bytes = b_bytes;
  pl.w_bytes = N * k.Cin * k.kh * k.kw * 2;
  pl.a_stride = b_stride; pl.b_off = 0; pl.a_bytes = 0;
  pl.stages = stages;
  pl.swa = 0;
  pl.smem = fixed + size_t(stages) * b_stride;
  return true;
}

Plan make_plan(const Geom& g) {
  Plan pl;
  if (g.in_dtype != BF16 || g.groups != 1 || g.Cout % 4 != 0) return pl;
  pl.gk = g;
  if (g.raw) {
    // RAW layout: one window contraction per Ready step, the kt temporal taps
    // folded into K (weights viewed as (Cout, Cin, 1, kt*kh, kw), the same
    // memory); always the K pipeline, one accumulator (no slices, no state)
    if (g.Cin % 16 != 0) return pl;
    Geom& k = pl.gk;
    k.kh = g.kt * g.kh; k.kt = 1;
    const bool flat = g.kh == 1 && g.kw == 1 && g.ph == 0 && g.pw == 0 && g.sh == 1 && g.sw == 1;
    pl.ok = plan_kloop(k, pl, flat);
    if (pl.ok) pl.n_split = g.Cout / pl.var->CC;
    return pl;
  }
  if (g.Cin < 16 && g.Cin * g.kw <= 64) {
    // small-Cin stem: W-im2col'd frame, kernel (kt, kh, 1), stride (st, sh, 1)
    pl.wcols = 1;
    pl.Kp = (g.Cin * g.kw + 15) / 16 * 16;
    Geom& k = pl.gk;
    k.Cin = pl.Kp; k.cig = pl.Kp;
    k.W = g.Wo; k.kw = 1; k.sw = 1; k.pw = 0; k.dw = 1;
  } else if (g.Cin % 16 != 0) {
    return pl;
  }
  const bool force_kloop = option(OPT_TC_MODE) == 1;   // option "tc_mode" = 1 forces the K pipeline
  pl.ok = (!force_kloop && plan_resident(pl.gk, pl)) || plan_kloop(pl.gk, pl);
  if (pl.ok && pl.wcols) plan_stem(g, pl);
  if (pl.ok && pl.mode != MODE_KLOOP && pl.mode != MODE_STEM && pl.gk.Cin % 64 == 0 && swa_enabled()) pl.swa = 1;
  if (pl.ok) pl.n_split = g.Cout / pl.var->CC;
  return pl;
}

}  // namespace

struct DenseTC {
  Plan pl;
  __nv_bfloat16* wpack = nullptr;
  __nv_bfloat16* xstage = nullptr;   // dense staging (strided clips in flat mode, zero frames, W-im2col)
  size_t xstage_bytes = 0;
  int64_t gen = 0;                   // bumped whenever xstage moves (captured graphs hold its address)
  int num_sms = 148;
  std::string name;
  // RAW-ring small-Cin stem (k_stem_raw.cu): its own plan and kernel
  bool stemraw = false;
  StemRawPlan sp;
};

bool dense_tc_supported(const Geom& g) {
  StemRawPlan sp;
  if (g.raw && !make_plan(g).ok) return stem_raw_plan(g, sp);
  return make_plan(g).ok && get_encode() != nullptr;
}

void dense_tc_state_layout(Geom& g) {
  const Plan pl = make_plan(g);
  g.spad = 0;
  g.sflat = 0;
  g.splane = g.B * g.HWo;
  if (!pl.ok || g.raw) return;                // RAW: the state is the frame ring
  g.spad = 1;
  if (pl.mode == MODE_FLAT) {          // tiles are 128 consecutive pixels: row = pixel
    g.sflat = 1;
    g.splane = (g.B * g.HWo + 127) / 128 * 128;
    return;
  }
  if (pl.mode == MODE_HALO || pl.mode == MODE_KHALO) {
    g.sTH = pl.MT; g.sTW = g.Wo; g.sRS = pl.Wp; g.stiles_h = pl.tiles_per_stream; g.stiles_w = 1;
  } else {
    g.sTH = pl.TH; g.sTW = pl.TW; g.sRS = pl.TW; g.stiles_h = pl.tiles_h; g.stiles_w = pl.tiles_w;
  }
  g.splane = pl.n_tiles * 128;
}

DenseTC* dense_tc_create(const Geom& g, const void* w_dev, std::string& err) {
  Plan pl = make_plan(g);
  if (g.raw && !pl.ok) {
    // a small-Cin stem over the RAW ring: the resident-weight W-im2col kernel
    DenseTC* t = new DenseTC();
    if (!stem_raw_plan(g, t->sp)) { err = "unsupported shape"; delete t; return nullptr; }
    t->stemraw = true;
    cudaError_t e = cudaMalloc(&t->wpack, stem_raw_wpack_elems(t->sp, g) * 2);
    if (e == cudaSuccess) e = stem_raw_pack(g, t->sp, w_dev, t->wpack);
    if (e == cudaSuccess) e = stem_raw_prepare();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, dev);
    t->name = stem_raw_name(t->sp);
    return t;
  }
  if (!pl.ok) { err = "unsupported shape"; return nullptr; }
  if (!get_encode()) { err = "cuTensorMapEncodeTiled unavailable"; return nullptr; }
  DenseTC* t = new DenseTC();
  t->pl = pl;
  const Geom& k = pl.gk;
  const int64_t total = int64_t(k.Cout) * k.Cin * k.kt * k.kh * k.kw;
  cudaError_t e = cudaMalloc(&t->wpack, size_t(total) * 2);
  if (e != cudaSuccess) { err = cudaGetErrorString(e); delete t; return nullptr; }
  const __nv_bfloat16* wsrc = static_cast<const __nv_bfloat16*>(w_dev);
  __nv_bfloat16* wtmp = nullptr;
  if (pl.wcols) {
    if ((e = cudaMalloc(&wtmp, size_t(total) * 2)) != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
    k_wcols_weights<<<unsigned((total + 255) / 256), 256>>>(wsrc, wtmp, g.Cout, g.Cin, g.kt, g.kh, g.kw, pl.Kp);
    wsrc = wtmp;
  }
  k_pack_tc_weights<<<unsigned((total + 255) / 256), 256>>>(wsrc, t->wpack, k.Cout, k.Cin, k.kt, k.kh, k.kw,
                                                           pl.var->CC, pl.n_split, pl.var->PAIR,
                                                           ((pl.mode == MODE_KLOOP || pl.mode == MODE_KHALO) && pl.var->PAIR == 2) ? pl.kb : 0);
  e = cudaGetLastError();
  if (wtmp) { cudaDeviceSynchronize(); cudaFree(wtmp); }
  if (e != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
  // one kernel variant may serve several layers with different footprints: allow the maximum
  e = cudaFuncSetAttribute(pl.var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemLimit));
  if (e != cudaSuccess) { err = cudaGetErrorString(e); dense_tc_destroy(t); return nullptr; }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, dev);
  char buf[128];
  const char* mname = pl.mode == MODE_KLOOP ? (pl.wcols ? ",kloop+wcols" : ",kloop")
                      : pl.mode == MODE_KHALO ? ",khalo" : pl.mode == MODE_STEM ? ",stem" : "";
  if (pl.var->KH && pl.var->KC == 0)          // compile-time taps of the K pipeline
    snprintf(buf, sizeof(buf), "k_step_dense_tc<%d,%d,%d,%dx%d%s%s>", pl.var->KT, pl.var->CC, pl.var->EG,
             pl.var->KH, pl.var->KW, pl.var->PAIR > 1 ? ",pair" : "", mname);
  else if (pl.var->KH)
    snprintf(buf, sizeof(buf), "k_step_dense_tc<%d,%d,%d,%dx%dx%d%s%s%s>", pl.var->KT, pl.var->CC, pl.var->EG,
             pl.var->KH, pl.var->KW, pl.var->KC * 16, pl.var->CS > 1 ? ",split" : "",
             pl.var->PAIR > 1 ? ",pair" : "", mname);
  else
    snprintf(buf, sizeof(buf), "k_step_dense_tc<%d,%d,%d%s%s>", pl.var->KT, pl.var->CC, pl.var->EG,
             pl.var->PAIR > 1 ? ",pair" : "", mname);
  if (option(OPT_LOG))
    fprintf(stderr, "[co] %s: %d parts, %lld tiles, %d stages x %d B, smem %zu B%s\n", buf, pl.n_split,
            (long long)pl.n_tiles, pl.stages, pl.a_stride, pl.smem, pl.ystage ? ", y staged" : "");
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
int64_t dense_tc_buffer_gen(const DenseTC* t) { return t ? t->gen : 0; }
bool dense_tc_fuses_raw_store(const DenseTC* t, const Geom& g, int64_t x_bstride) {
  return t && g.raw && !t->stemraw && t->pl.kflat && g.kt > 1 && x_bstride == g.frame_elems && CO_EXP("CO_TC_RAWSTORE", 1);
}

static cudaError_t ensure_stage(DenseTC* t, size_t need) {
  if (t->xstage_bytes >= need) return cudaSuccess;
  cudaFree(t->xstage);
  t->xstage = nullptr;
  t->xstage_bytes = 0;
  ++t->gen;
  cudaError_t e = cudaMalloc(&t->xstage, need);
  if (e == cudaSuccess) t->xstage_bytes = need;
  return e;
}

// One launch: a step (T == 1), or a chunk of T frames of a clip x (B, T, H, W,
// Cin) with the tick table `ticks` on the device (HALO / FLAT only).
static cudaError_t tc_launch(DenseTC* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s,
                             int T, const int* ticks, int64_t y_tstride) {
  const Plan& pl = t->pl;
  const Geom& k = pl.gk;
  const void* x = a.x;
  int64_t x_bstride = a.x_bstride;
  const int64_t frame = int64_t(g.H) * g.W * g.Cin;
  int64_t n_batch = k.B;                        // the tensor map's outermost extent
  int64_t flat_rows = k.B * k.HWo;              // FLAT: rows of the tensor map
  const int64_t clip_T = T > 1 ? a.x_bstride / frame : 1;   // frames per stream of the clip x points into
  if (T > 1) {
    if (pl.mode == MODE_FLAT) {
      // FLAT tiles are 128 consecutive (stream, pixel) rows of one frame: stage the
      // chunk time-major, (T, B*HW, Cin), so frame t's rows are contiguous
      if (cudaError_t e = ensure_stage(t, size_t(T) * g.B * frame * 2)) return e;
      for (int tt = 0; tt < T; ++tt)
        if (cudaError_t e = cudaMemcpy2DAsync(t->xstage + size_t(tt) * g.B * frame, frame * 2,
                                              static_cast<const __nv_bfloat16*>(x) + size_t(tt) * frame,
                                              size_t(a.x_bstride) * 2, frame * 2, g.B, cudaMemcpyDeviceToDevice, s))
          return e;
      x = t->xstage;
      flat_rows = int64_t(T) * k.B * k.HWo;
    } else {
      n_batch = k.B * clip_T;                   // HALO: frame (b, t) is "stream" b T + t of the clip
      x_bstride = frame;
    }
  } else if (g.raw) {                           // the frame ring: (f + 1) slots of B streams
    x = a.state;
    x_bstride = frame;
    n_batch = k.B * (g.f + 1);
  } else if (pl.mode == MODE_STEM) {
    // the kernel bulk-copies raw rows itself: they must be 16-B aligned
    if (x && ((reinterpret_cast<uintptr_t>(x) & 15) || (x_bstride * 2) % 16)) {
      if (cudaError_t e = ensure_stage(t, size_t(g.B) * frame * 2)) return e;
      if (cudaError_t e = cudaMemcpy2DAsync(t->xstage, frame * 2, x, x_bstride * 2, frame * 2, g.B,
                                            cudaMemcpyDeviceToDevice, s))
        return e;
      x = t->xstage;
      x_bstride = frame;
    }
  } else if (pl.wcols) {
    // small-Cin stem: W-im2col the frame (a zero frame stays zero)
    const int64_t kframe = int64_t(k.H) * k.W * k.Cin;
    if (cudaError_t e = ensure_stage(t, size_t(g.B) * kframe * 2)) return e;
    const int64_t n = g.B * k.H * k.W;
    const unsigned nb = unsigned((n + 255) / 256);
    const __nv_bfloat16* xs = static_cast<const __nv_bfloat16*>(x);
    switch (pl.Kp) {
      case 16: k_wcols_frame<16><<<nb, 256, 0, s>>>(xs, x_bstride, t->xstage, g.B, g.H, g.W, g.Cin, g.Wo, g.kw, g.sw, g.dw, g.pw); break;
      case 32:
        if (g.Cin == 3) k_wcols_frame<32, 3><<<nb, 256, 0, s>>>(xs, x_bstride, t->xstage, g.B, g.H, g.W, g.Cin, g.Wo, g.kw, g.sw, g.dw, g.pw);
        else k_wcols_frame<32><<<nb, 256, 0, s>>>(xs, x_bstride, t->xstage, g.B, g.H, g.W, g.Cin, g.Wo, g.kw, g.sw, g.dw, g.pw);
        break;
      case 48: k_wcols_frame<48><<<nb, 256, 0, s>>>(xs, x_bstride, t->xstage, g.B, g.H, g.W, g.Cin, g.Wo, g.kw, g.sw, g.dw, g.pw); break;
      default: k_wcols_frame<64><<<nb, 256, 0, s>>>(xs, x_bstride, t->xstage, g.B, g.H, g.W, g.Cin, g.Wo, g.kw, g.sw, g.dw, g.pw); break;
    }
    if (cudaError_t e = cudaGetLastError()) return e;
    x = t->xstage;
    x_bstride = kframe;
  } else if (T == 1 && (!x || (pl.mode == MODE_FLAT && x_bstride != frame))) {
    // zero frame (pad_end) or a strided clip column in flat mode: stage it densely
    if (cudaError_t e = ensure_stage(t, size_t(g.B) * frame * 2)) return e;
    cudaError_t e = x ? cudaMemcpy2DAsync(t->xstage, frame * 2, x, x_bstride * 2, frame * 2, g.B,
                                          cudaMemcpyDeviceToDevice, s)
                      : cudaMemsetAsync(t->xstage, 0, size_t(g.B) * frame * 2, s);
    if (e != cudaSuccess) return e;
    x = t->xstage;
    x_bstride = frame;
  }
  CUtensorMap map;
  CUresult r = CUDA_SUCCESS;
  auto encode = get_encode();
  if (pl.mode == MODE_STEM) {
    memset(&map, 0, sizeof(map));                     // STEM reads raw rows by bulk copy: no A tensor map
  } else if (pl.mode == MODE_FLAT) {
    const cuuint32_t cw = pl.swa ? 64 : 8;    // channels per row of the box (128-B swizzled or 16-B)
    cuuint64_t dims[3] = {cw, cuuint64_t(flat_rows), cuuint64_t(k.Cin / cw)};
    cuuint64_t strides[2] = {cuuint64_t(k.Cin) * 2, cw * 2};
    cuuint32_t box[3] = {cw, 128, cuuint32_t(k.Cin / cw)};
    cuuint32_t es[3] = {1, 1, 1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, pl.swa ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (pl.kflat) {
    // ring slots as (B*HW rows, Cin) matrices: {cw, rows, Cin/cw, f+1 slots}
    const cuuint32_t cw = pl.swa ? cuuint32_t(pl.kb) : 8;
    cuuint64_t dims[4] = {cw, cuuint64_t(g.B * g.HWo), cuuint64_t(k.Cin / cw), cuuint64_t(g.f + 1)};
    cuuint64_t strides[3] = {cuuint64_t(k.Cin) * 2, cuuint64_t(cw) * 2, cuuint64_t(g.B) * frame * 2};
    cuuint32_t box[4] = {cw, 128, pl.swa ? 1u : cuuint32_t(pl.kb / 8), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE,
               pl.swa == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : pl.swa == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[5] = {8, cuuint64_t(k.W), cuuint64_t(k.H), cuuint64_t(k.Cin / 8), cuuint64_t(n_batch)};
    cuuint64_t strides[4] = {cuuint64_t(k.Cin) * 2, cuuint64_t(k.W) * k.Cin * 2, 16, cuuint64_t(x_bstride) * 2};
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
    if ((pl.mode == MODE_HALO && pl.swa) || pl.mode == MODE_KHALO) {
      // 64-channel (128-B) rows, swizzled: smem [Cin/64][halo rows][128 B] (KHALO: one block per box)
      dims[0] = 64; dims[3] = cuuint64_t(k.Cin / 64); strides[2] = 128;
      box[0] = 64; box[1] = cuuint32_t(pl.Wp); box[2] = cuuint32_t(pl.MT + k.kh - 1);
      box[3] = pl.mode == MODE_KHALO ? 1u : cuuint32_t(k.Cin / 64);
      if (pl.mode == MODE_KHALO) {     // one phase sub-image: every s-th column / row
        box[1] = cuuint32_t(pl.Wp * k.sw); box[2] = cuuint32_t((pl.a_bytes / 128 / pl.Wp) * k.sh);
        es[1] = cuuint32_t(k.sw); es[2] = cuuint32_t(k.sh);
      }
      box[4] = 1;
      sw = CU_TENSOR_MAP_SWIZZLE_128B;
    } else if (pl.mode == MODE_HALO) {
      box[0] = 8; box[1] = cuuint32_t(pl.Wp); box[2] = cuuint32_t(pl.MT + k.kh - 1); box[3] = cuuint32_t(k.Cin / 8);
      box[4] = 1;
    } else {
      // strided gather: TMA loads ceil(box / elementStride) elements per dimension
      box[0] = 8; box[1] = cuuint32_t(pl.TW * k.sw); box[2] = cuuint32_t(pl.TH * k.sh); box[3] = cuuint32_t(pl.kb / 8);
      box[4] = 1;
      es[1] = cuuint32_t(k.sw); es[2] = cuuint32_t(k.sh);
      if (pl.swa) {   // one swizzled kb-channel row (128 B or 64 B) per output pixel
        dims[0] = cuuint64_t(pl.kb); dims[3] = cuuint64_t(k.Cin / pl.kb); strides[2] = cuuint64_t(pl.kb) * 2;
        box[0] = cuuint32_t(pl.kb); box[3] = 1;
        sw = pl.swa == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
      }
    }
    r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;

  TcParams p{};
  p.B = int(g.B); p.H = k.H; p.W = k.W; p.Cin = k.Cin; p.Cout = g.Cout; p.Ho = g.Ho; p.Wo = g.Wo;
  p.HWo = g.HWo; p.plane = g.B * g.HWo; p.splane = g.splane;
  p.kh = k.kh; p.kw = k.kw; p.ph = k.ph; p.pw = k.pw;
  p.sh = k.sh; p.sw = k.sw; p.dh = k.dh; p.dw = k.dw;
  p.mode = pl.mode;
  p.MT = pl.MT; p.Wp = pl.Wp; p.tiles_per_stream = pl.tiles_per_stream;
  p.TH = pl.TH; p.TW = pl.TW; p.tiles_h = pl.tiles_h; p.tiles_w = pl.tiles_w;
  p.kb = pl.kb; p.n_cb = pl.n_cb; p.b_bytes = pl.b_bytes; p.b_off = pl.b_off;
  p.ka_stages = pl.ka_stages; p.ka_stride = pl.ka_stride; p.ka_phase = pl.ka_phase;
  p.dmin_h = pl.dmin_h; p.dmin_w = pl.dmin_w;
  const int pair = pl.var->PAIR;
  // weight-multicast clusters for one-CTA K-pipeline layers (CO_TC_MC = cluster size, A/B runs)
  int mc = 1;
  if (pl.mode == MODE_KLOOP && pair == 1 && T == 1) {
    mc = int(option(OPT_MC));                        // option "mc" (weight multicast cluster size)
    while (mc > 1 && ((pl.b_bytes / 16) % mc != 0 || pl.n_tiles < mc)) mc /= 2;
  }
  const int clu = pair > 1 ? pair : mc;                  // CTAs per cluster
  const int64_t units_tiles = (pl.n_tiles + clu - 1) / clu;       // tiles per unit position (clusters take clu)
  p.n_tiles = pl.n_tiles; p.n_split = pl.n_split; p.n_items = units_tiles * pl.n_split;
  p.a_bytes = pl.a_bytes; p.a_stride = pl.a_stride; p.stages = pl.stages; p.chunk_stride = pl.chunk_stride;
  p.w_bytes = pl.w_bytes; p.w_off = pl.w_off;
  for (int i = 0; i < kMaxKt; ++i) p.slot[i] = a.slot[i];
  p.emit = a.emit; p.update = a.update; p.act = g.act; p.out_f32 = (g.out_dtype == F32);
  p.dbg = CO_EXP("CO_TC_DEBUG", 0);              // experiment builds only (work-skipping A/B bits)
  // measured (same box, interleaved A/B): C2 (HALO) 0.205 -> 0.200 ms, C5 (FLAT) 1.53 -> 1.40 ms;
  // the C4 KHALO layers unchanged, the stem (4 slots read per item) 1.49 -> 1.62 ms
  p.l2pf = CO_EXP("CO_TC_L2PF", (pl.mode == MODE_HALO || pl.mode == MODE_FLAT) ? 1 : 0);
  p.ystage = (pl.ystage && g.out_dtype == BF16) ? 1 : 0;
  {
    // programmatic dependent launch for single steps (CO_PDL=0 turns it off):
    // C5 +1.7%, C4 +0.5%, C2 unchanged (its launches were already back to back)
    p.pdl = (T == 1 && option(OPT_PDL) != 0) ? 1 : 0;
  }
  {
    p.l2last = (pl.mode == MODE_HALO || pl.mode == MODE_FLAT) && CO_EXP("CO_TC_L2LAST", 0) != 0;   // A/B
  }
  p.y_off = pl.y_off;
  p.raw_kh = g.raw ? g.kh : 0;
  p.kflat = pl.kflat;
  p.raw_B = int(g.B);
  for (int i = 0; i < kMaxKt; ++i) p.ring_slot[i] = g.raw ? a.slot[i] : -1;
  p.swa = pl.swa;
  p.a_rows = pl.chunk_stride / 16;
  p.Cq = g.Cq;
  if (pl.mode == MODE_STEM) {
    p.x = static_cast<const __nv_bfloat16*>(x);
    p.x_bstride = x_bstride;
    p.st_Hin = g.H; p.st_Win = g.W; p.st_cin = g.Cin;
    p.st_sw = g.sw; p.st_pw = g.pw; p.st_kwc = g.kw * g.Cin;
    p.st_nraw = pl.st_nraw; p.st_rpitch = pl.st_rpitch; p.st_pad = pl.st_pad; p.st_raw_off = pl.st_raw_off;
    p.st_img_rows = pl.st_img_rows; p.st_img_bytes = pl.st_img_bytes;
    p.st_groups = pl.st_groups; p.st_data_groups = pl.st_data_groups;
    p.st_phase_base[0] = pl.st_phase_base[0]; p.st_phase_base[1] = pl.st_phase_base[1];
  }
  p.T = T;
  p.x_tmul = int(clip_T);
  p.ticks = ticks;
  p.y_tstride = y_tstride;
  p.a_trows = k.B * k.HWo;
  p.state = a.state;
  p.y = a.y;
  p.y_bstride = a.y_bstride;
  p.wpack = t->wpack;
  p.bias = bias;
  p.mc = mc;
  const int per = std::max(1, t->num_sms / clu / pl.n_split);
  // STEM: a CTA serves every part of its tiles (one image per tile), one CTA per SM;
  // floating parts (KHALO, single steps): every SM, whatever the part count
  p.fparts = (pl.fparts && T == 1) ? 1 : 0;
  const int64_t grid = pl.mode == MODE_STEM ? std::min<int64_t>(t->num_sms, pl.n_tiles)
                       : p.fparts           ? std::min<int64_t>(t->num_sms / clu, units_tiles * pl.n_split) * clu
                                            : std::min<int64_t>(per, units_tiles) * pl.n_split * clu;
  // KLOOP pairs stream their weight halves through a tensor map over the packed
  // weights [part*2 + half][K/8][N/2][8]: box = one chunk (kb/8 K-groups)
  CUtensorMap wmap = map;
  if ((pl.mode == MODE_KLOOP || pl.mode == MODE_KHALO) && pl.var->PAIR == 2) {
    const int NBh = pl.var->KT * pl.var->CC / 2;
    const int64_t nblk = int64_t(k.Cin) * k.kh * k.kw / pl.kb;        // kb-element K blocks
    cuuint64_t dims[4] = {cuuint64_t(pl.kb), cuuint64_t(NBh), cuuint64_t(nblk), cuuint64_t(pl.n_split * 2)};
    cuuint64_t strides[3] = {cuuint64_t(pl.kb) * 2, cuuint64_t(NBh) * pl.kb * 2, cuuint64_t(nblk) * NBh * pl.kb * 2};
    cuuint32_t box[4] = {cuuint32_t(pl.kb), cuuint32_t(NBh), 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&wmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, t->wpack, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, pl.kb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  // RAW flat: the Ready step reads the new frame from x (a map like the ring's,
  // one slot) and stores it into its ring slot from shared memory
  CUtensorMap xmap = map;
  p.raw_xslot = -1;
  p.raw_xk = -1;
  if (pl.kflat && a.raw_store >= 0 && a.x) {
    const cuuint32_t cw = pl.swa ? cuuint32_t(pl.kb) : 8;
    cuuint64_t dims[4] = {cw, cuuint64_t(g.B * g.HWo), cuuint64_t(k.Cin / cw), 1};
    cuuint64_t strides[3] = {cuuint64_t(k.Cin) * 2, cuuint64_t(cw) * 2, cuuint64_t(g.B) * frame * 2};
    cuuint32_t box[4] = {cw, 128, pl.swa ? 1u : cuuint32_t(pl.kb / 8), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.x), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE,
               pl.swa == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : pl.swa == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    p.raw_xslot = a.raw_store;
    p.raw_xk = g.kt - 1;
  }
  void* args[] = {&map, &wmap, &xmap, &p};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(tc_threads(pl.var->EG, pl.var->CS));
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (clu > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = unsigned(clu);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (p.pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = na ? attr : nullptr;
  cfg.numAttrs = na;
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(pl.var->fn), args);
}

cudaError_t dense_tc_step(DenseTC* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s) {
  if (t->stemraw) return stem_raw_step(g, t->sp, a, t->wpack, bias, t->num_sms, s);
  return tc_launch(t, g, a, bias, s, 1, nullptr, 0);
}

bool dense_tc_chunkable(const DenseTC* t, const Geom& g) {
  if (!option(OPT_CHUNK)) return false;          // option "chunk" = 0: always fold per step
  // HALO only: FLAT chunks must first be staged time-major (a 128-row tile spans
  // streams), which costs more than the L2 reuse saves (measured on C5: 9.5 M
  // chunked vs 9.7 M per-step stream-steps/s); option "chunk_flat" = 1 enables it
  const bool flat_ok = option(OPT_CHUNK_FLAT) != 0;
  return t && !g.raw && !t->pl.wcols && (t->pl.mode == MODE_HALO || (flat_ok && t->pl.mode == MODE_FLAT)) &&
         g.st == 1;
}

cudaError_t dense_tc_steps(DenseTC* t, const Geom& g, const void* x, int64_t T, int64_t clip_T, const int* ticks_dev,
                           void* y, int64_t y_bstride, float* state, const float* bias, cudaStream_t s) {
  StepArgs a{};
  a.x = x;
  a.x_bstride = clip_T * int64_t(g.H) * g.W * g.Cin;
  a.y = y;
  a.y_bstride = y_bstride;
  a.state = state;
  a.update = 1;
  return tc_launch(t, g, a, bias, s, int(T), ticks_dev, g.HWo * g.Cout);
}

}  // namespace co
