// k_dense_tc.cu — placeholder until the tcgen05 kernel lands.
#include "dense_tc.cuh"
namespace co {
struct DenseTC { int dummy; };
bool dense_tc_supported(const Geom&) { return false; }
DenseTC* dense_tc_create(const Geom&, const void*, std::string& err) { err = "not built"; return nullptr; }
void dense_tc_destroy(DenseTC* t) { delete t; }
const char* dense_tc_name(const DenseTC*) { return "k_step_dense_tc"; }
cudaError_t dense_tc_step(DenseTC*, const Geom&, const StepArgs&, const float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace co
