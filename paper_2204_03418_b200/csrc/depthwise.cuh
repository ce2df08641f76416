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
}  // namespace co
