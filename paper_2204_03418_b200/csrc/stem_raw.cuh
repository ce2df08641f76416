// stem_raw.cuh — interface of the RAW-ring tensor-core step of small-Cin stems
// (`k_step_stem_raw`, k_stem_raw.cu): the window contraction of SPEC's raw
// input ring for layers whose Cin is too small
// for a TMA box (C4 layer 1: RGB, 5x7x7, stride (1,2,2)).  Reached through the
// dense tensor-core handle (dense_tc_create / dense_tc_step) when the layer's
// state layout is RAW.
#pragma once
#include <cstddef>
#include "common.cuh"

namespace co {

struct StemRawPlan {
  bool ok = false;
  int N = 0;                       // output channels (the whole layer: one part)
  int CP = 0, Kp = 0;              // channels per padded pixel (8 / sw), K per (temporal, row) tap
  int pair = 2;                    // CTAs per MMA (cta_group::2 pairs; w_bytes is one CTA's half)
  int TH = 0, tiles_h = 0, Wp = 0; // output rows per 128-row tile, tiles per stream, row slots per output row
  int64_t n_tiles = 0;
  int nraw = 0, rpitch = 0, pad = 0;     // raw rows per image, their shared pitch, zero elements before the data
  int img_rows = 0, base[2] = {0, 0};    // 16-B rows of an image (incl. the MMA over-read), first row of each phase
  int w_bytes = 0, img_off = 0, img_bytes = 0, raw_off = 0, raw_bytes = 0, bias_off = 0, bar_off = 0;
  int tab_off = 0;                 // the MMA warp's A descriptor table
  size_t smem = 0;
};

// Shape check + shared-memory plan (bf16, groups 1, Cin <= 8 / sw, dilation 1
// in space, spatial strides <= 2, <= 128 row slots, Cout in {32, 64}, 16-B raw rows).
bool stem_raw_plan(const Geom& g, StemRawPlan& sp);
// Packed weights [K/8][N][8] bf16, K index = (k kh + u) Kp + v CP + c (zero for
// v >= kw or c >= Cin): the B operand, resident in shared memory.
size_t stem_raw_wpack_elems(const StemRawPlan& sp, const Geom& g);
cudaError_t stem_raw_pack(const Geom& g, const StemRawPlan& sp, const void* w_dev, void* wpack);
cudaError_t stem_raw_prepare();   // kernel attributes (max dynamic shared memory)
// One Ready step: a.state = the ring [f+1][B][H][W][Cin], a.slot[k] = ring slot of
// temporal tap k (the new frame already stored in its slot), y (B, Ho, Wo, Cout).
cudaError_t stem_raw_step(const Geom& g, const StemRawPlan& sp, const StepArgs& a, const void* wpack,
                          const float* bias, int num_sms, cudaStream_t s);
const char* stem_raw_name(const StemRawPlan& sp);

}  // namespace co
