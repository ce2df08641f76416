// common.cuh — definitions shared by the sm_100a kernels and the host library
// of the continual-convolution step (arXiv 2204.03418).  Product code: shares
// nothing with oracle/.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <string>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace co {

constexpr int kMaxKt = 32;   // == CO_MAX_KT

// Documented planner / launch options (include/co.h co_set_option; options.cu).
enum Opt : int {
  OPT_TC_MODE, OPT_KHALO, OPT_PAIR, OPT_KPAIR, OPT_EG, OPT_MC, OPT_PDL, OPT_CHUNK, OPT_CHUNK_FLAT, OPT_CHUNK_ST,
  OPT_CHUNK_T, OPT_POOL_BAND, OPT_POOL_VH, OPT_POOL_G, OPT_LOG, OPT_STEM, OPT_DW_SEG, OPT_MHA_RING, OPT_POOL_SEG, OPT_COUNT
};
int64_t option(Opt o);
void set_thread_no_pdl(int v);   // graph capture fallback: plain launches on this thread

// A/B experiment knobs: read from the environment only in -DCO_EXPERIMENTS
// builds; the release library compiles them to their defaults (no getenv, no
// variable names in the binary).
#ifdef CO_EXPERIMENTS
int experiment_knob(const char* name, int dflt);
#define CO_EXP(name, dflt) ::co::experiment_knob(name, dflt)
#define CO_EXP_SET(name) (std::getenv(name) != nullptr)
#else
#define CO_EXP(name, dflt) (dflt)
#define CO_EXP_SET(name) false
#endif

enum Dtype : int { F32 = 0, BF16 = 1 };
enum Op : int { OP_CONV = 0, OP_MAX_POOL = 1, OP_AVG_POOL = 2, OP_DELAY = 3 };   // == co_op

// Normalised layer geometry (absent spatial axes are extent 1, kernel 1).
struct Geom {
  int rank;
  int Cin, Cout, groups, cig, cog;
  int kt, kh, kw;
  int st, sh, sw;        // strides (t, h, w)
  int pt, ph, pw;        // paddings
  int dt, dh, dw;        // dilations
  int H, W, Ho, Wo;
  int64_t B;
  int in_dtype, out_dtype, act;
  int f, delay, R;       // receptive field, d = f - p - 1, ring slots R = ceil((f-1)/s)
  int Cq;                // ceil(Cout / 4): channel quads of the state layout
  int64_t HWo;           // Ho * Wo
  int64_t slot_elems;    // Cq * 4 * splane
  int state_cl;          // physical state layout: 0 = quad-major, 1 = channels-last (see state_index)
  // tile-padded quad-major rows (dense tensor-core handles): state row of
  // output pixel (b, ho, wo) = tile * 128 + m, m = its TMEM lane in that tile
  int spad, sflat, sTH, sTW, sRS, stiles_h, stiles_w;
  // RAW state layout (co_state_layout RAW): ring of f + 1 input
  // frames [slot][B][H][W][Cin] in in_dtype (f data slots + one scratch slot
  // for update_state = 0); a Ready step reads the window's kt slots
  int raw;
  int64_t frame_elems;   // H * W * Cin
  int64_t splane;        // state rows per slot and channel quad: B*HWo, or n_tiles*128 when tile-blocked
  int op;                // Op: continual conv, or max / avg pooling over the RAW ring (§8f f3)
  int pool_G;            // pooling: lanes per output vector of the step kernel (1 = plain, k_pool.cu)
  int pool_vh;           // pooling: block-decomposition state (P, S after the ring) for long windows
};

// Physical state layouts (internal; co_state_get converts to the canonical one):
//  quad-major (state_cl = 0, dense / direct kernels):
//   direct kernel: S[slot][Cout/4][B*HWo][4] fp32, row = b*HWo + pixel;
//   dense tensor-core kernel (spad = 1, tile-blocked):
//   S[slot][tile][Cout/4][128][4] -- the 128 rows of a tile are its TMEM lanes,
//   so each warp of an epilogue moves exactly one aligned 512-byte run per
//   access (its halo tiles hold e.g. 2 output rows of 56 in 58 lanes, which
//   unpadded would straddle 128-byte lines: -21% HBM bandwidth in
//   scripts/bw_probe.cu), and a thread's channel quads sit 2 KB apart, so
//   every state access is an immediate offset from one base per slot;
//  channels-last (state_cl = 1, depthwise kernels, Cout % 4 == 0):
//   S[slot][B * Ho * Wo][Cout] fp32 -- a thread owns one (pixel, channel quad)
//   and consecutive threads take consecutive quads, so the state, the
//   channels-last frame and the output are all read/written contiguously.
__host__ __device__ inline int64_t state_row(const Geom& g, int64_t pix) {
  if (!g.spad || g.sflat) return pix;   // FLAT tiles are 128 consecutive pixels
  const int64_t b = pix / g.HWo;
  const int r = int(pix - b * g.HWo);
  const int ho = r / g.Wo, wo = r - (r / g.Wo) * g.Wo;
  const int th = ho / g.sTH, tw = wo / g.sTW;
  const int64_t tile = (b * g.stiles_h + th) * g.stiles_w + tw;
  return tile * 128 + (ho - th * g.sTH) * g.sRS + (wo - tw * g.sTW);
}
__host__ __device__ inline int64_t state_index(const Geom& g, int slot, int64_t pix, int o) {
  if (g.state_cl) return (int64_t(slot) * (g.B * g.HWo) + pix) * g.Cout + o;
  if (g.spad) {
    const int64_t row = state_row(g, pix);
    return (((int64_t(slot) * (g.splane >> 7) + (row >> 7)) * g.Cq + (o >> 2)) * 128 + (row & 127)) * 4 + (o & 3);
  }
  return ((int64_t(slot) * g.Cq + (o >> 2)) * g.splane + pix) * 4 + (o & 3);
}

// One step's clock decisions, computed on the host:
// slot[k] is the ring slot of the output that temporal slice k of this frame
// contributes to (-1: no contribution, i.e. an output that is never emitted or
// a stride-skipped phase).  k = kt-1 completes (emit), k = 0 starts
// (overwrite), 0 < k < kt-1 accumulate.
struct StepArgs {
  const void* x;         // frame of stream 0, channels-last (H, W, Cin); nullptr = zero frame
  int64_t x_bstride;     // elements between consecutive streams
  void* y;               // output of stream 0, channels-last (Ho, Wo, Cout)
  int64_t y_bstride;
  float* state;
  int slot[kMaxKt];
  int emit;              // ready: produce y from slice kt-1
  int update;            // update_state: write the ring
  int64_t m;             // padded index n + p of this frame (pooling: ring slots computed on the device)
  // pooling, derived from m once per launch (launch_step_pool): m mod f, and for
  // the block decomposition the phase q = m mod dil, i = m div dil, i mod kt and
  // (i - kt + 1) mod kt -- 32-bit, so no kernel divides 64-bit values per item
  int pm_f, pm_q, pm_pos, pm_js;
  // RAW layout, dense 1x1 kernel: the Ready step reads the new frame straight
  // from x and stores it into ring slot raw_store itself (-1: the host copied it)
  int raw_store = -1;
};

// Pooling ring (§8f f3): slot = one spatially reduced frame (B, Ho, Wo, C); MAX
// keeps the input dtype (a max is exact), AVG fp32 spatial sums.
inline int pool_ring_esz(const Geom& g) { return g.op == OP_AVG_POOL ? 4 : (g.in_dtype == BF16 ? 2 : 4); }
inline int64_t pool_slot_elems(const Geom& g) { return g.B * g.HWo * g.Cin; }
// Slots of a pooling handle's state: the ring (f + 1), plus P (dil) and S
// (dil * kt) of the block decomposition.
inline int64_t pool_state_slots(const Geom& g) { return g.f + 1 + (g.pool_vh ? int64_t(g.dt) * (g.kt + 1) : 0); }

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float activate(float v, int act) { return (act == 1 && v < 0.f) ? 0.f : v; }

// RAW layout step (StepArgs.state = ring, slot[k] = ring slot of temporal tap k)
cudaError_t launch_step_direct_raw(const Geom& g, const StepArgs& a, const float* w_direct, const float* bias,
                                   cudaStream_t s);

// Continual pooling (k_pool.cu): Ready-step reduction over the
// RAW ring, batch forward, and the ring's padding fill (0 AVG, -inf MAX).
cudaError_t launch_step_pool(const Geom& g, const StepArgs& a, cudaStream_t s);
cudaError_t launch_forward_pool(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp, cudaStream_t s);
cudaError_t launch_fill_pad(const Geom& g, void* p, int64_t n_elems, cudaStream_t s);
std::string pool_kernel_name(const Geom& g);
int pool_split_lanes(const Geom& g);   // choice of pool_G (option "pool_g" overrides)
int pool_block_decomposition(const Geom& g);   // choice of pool_vh (option "pool_vh" overrides)
cudaError_t launch_pool_rebuild(const Geom& g, void* state, int64_t m_next, cudaStream_t s);

// Per-stream clean (k_direct.cu): zero the listed streams'
// partial-sum state (any PSUM layout), or fill their slices of a ring layout.
cudaError_t launch_clean_streams_psum(const Geom& g, float* state, const int64_t* ids, int nm, cudaStream_t s);
cudaError_t launch_fill_streams(void* ring, int esz, int64_t slots, int64_t B, int64_t per, const int64_t* ids, int nm,
                                uint32_t value, cudaStream_t s);

// Continual single-output MHA (k_mha.cu)
struct MhaArgs {
  const __nv_bfloat16* qkv;   // step: (B, 3E); batch: (B, T, 3E)
  __nv_bfloat16* kring;       // [B][n][E] (step mode)
  __nv_bfloat16* vring;
  __nv_bfloat16* out;         // step: (B, E); batch: (B, T, E)
  int64_t B, T;               // T: batch columns (batch mode), 1 in step mode
  int E, heads, n;            // n = window
  int64_t m;                  // step: index of this step (ring slot m mod n)
  int store;                  // step: write (k_t, v_t) into the ring
  int batch;                  // 1: keys / values from qkv over all T columns
  float scale_log2e;          // log2(e) / sqrt(dh)
};
bool mha_supported(int E, int heads);
cudaError_t launch_mha_attend(const MhaArgs& a, cudaStream_t s);

// Residual composite merge (k_compose.cu): y[r, :n] <- act(y[r, :n] + x[r, :n]) over rows.
cudaError_t launch_residual_add(int y_dtype, void* y, int64_t y_rstride, int x_dtype, const void* x,
                                int64_t x_rstride, int64_t rows, int64_t n, int act, cudaStream_t s);

// ---- launchers implemented in the .cu files (host side) --------------------
cudaError_t launch_step_direct(const Geom& g, const StepArgs& a, const float* w_direct, const float* bias,
                               cudaStream_t s);
cudaError_t launch_forward_direct(const Geom& g, const void* x, int64_t T, void* y, int64_t Tp,
                                  const float* w_direct, const float* bias, cudaStream_t s);
cudaError_t launch_state_get(const Geom& g, const float* state, float* dst, int head, int64_t i_next,
                             int64_t m_next, cudaStream_t s);
cudaError_t launch_state_set(const Geom& g, float* state, const float* src, int head, cudaStream_t s);
cudaError_t launch_pack_direct_weights(const Geom& g, const void* w, float* w_direct, cudaStream_t s);

}  // namespace co
