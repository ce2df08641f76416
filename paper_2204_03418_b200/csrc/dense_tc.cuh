// dense_tc.cuh — interface of the dense tcgen05 / TMEM / TMA continual-conv
// step kernel (K4, `k_step_dense_tc`).  Implementation: k_dense_tc.cu.
#pragma once
#include <string>
#include "common.cuh"

namespace co {
struct DenseTC;
bool dense_tc_supported(const Geom& g);
// Fill g's tile-padded state-row fields (spad, sTH, sTW, sRS, stiles_*, splane)
// for the tiles the kernel's plan uses.
void dense_tc_state_layout(Geom& g);
DenseTC* dense_tc_create(const Geom& g, const void* w_dev, std::string& err);
void dense_tc_destroy(DenseTC* t);
const char* dense_tc_name(const DenseTC* t);
int64_t dense_tc_buffer_gen(const DenseTC* t);
// RAW layout: can the Ready-step kernel read frame x directly and store it into its ring slot?
bool dense_tc_fuses_raw_store(const DenseTC* t, const Geom& g, int64_t x_bstride);   // changes whenever a step's staging buffer moves
cudaError_t dense_tc_step(DenseTC* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s);
// Chunked steps: T consecutive ticks of a clip in one launch --
// x points at the chunk's first frame of a clip (B, clip_T, H, W, Cin) -- item-batch-major so each tile's state stays L2-resident
// across its frames; ticks_dev = T rows of (2 + kMaxKt) ints [emit, output
// index, ring slot of tap k]; y (B, n_ready, Ho, Wo, Cout), stream stride
// y_bstride.  HALO / FLAT partial-sum layers with temporal stride 1.
bool dense_tc_chunkable(const DenseTC* t, const Geom& g);
cudaError_t dense_tc_steps(DenseTC* t, const Geom& g, const void* x, int64_t T, int64_t clip_T, const int* ticks_dev,
                           void* y, int64_t y_bstride, float* state, const float* bias, cudaStream_t s);
}  // namespace co
