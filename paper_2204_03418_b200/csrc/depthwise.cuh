// depthwise.cuh — interface of the CUDA-core depthwise continual-conv step
// kernels (K2 spatio-temporal stencil, K3 temporal-only).  Implementation:
// k_depthwise.cu.
#pragma once
#include <string>
#include "common.cuh"

namespace co {
struct Depthwise;
bool depthwise_supported(const Geom& g);
Depthwise* depthwise_create(const Geom& g, const void* w_dev, std::string& err);
void depthwise_destroy(Depthwise* t);
const char* depthwise_name(const Depthwise* t);
cudaError_t depthwise_step(Depthwise* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s);
// RAW layout, temporal-only layers: a Ready step can read the new frame from x and
// store it into its ring slot itself (StepArgs.x / raw_store), no separate frame copy.
bool depthwise_fuses_raw_store(const Depthwise* t, const Geom& g, int64_t x_bstride);
// True when a RAW-layout stencil of this geometry has a rolling-row plan (the planner's test).
bool depthwise_raw_pipeline(const Geom& g);
// Chunked steps: the fold of `total` ticks starting at clock n0
// over a clip x (B, T, H, W, C) (ticks >= T are padding frames) in one launch,
// state kept in registers; y (B, n_ready, Ho, Wo, C) with stream stride y_bstride.
bool depthwise_chunkable(const Depthwise* t, const Geom& g);
cudaError_t depthwise_steps(Depthwise* t, const Geom& g, const void* x, int64_t T, int64_t total, int64_t n0, void* y,
                            int64_t y_bstride, float* state, const float* bias, cudaStream_t s);
}  // namespace co
