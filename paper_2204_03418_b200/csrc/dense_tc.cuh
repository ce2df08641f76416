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
cudaError_t dense_tc_step(DenseTC* t, const Geom& g, const StepArgs& a, const float* bias, cudaStream_t s);
}  // namespace co
