// k_depthwise.cu — placeholder until the depthwise kernels land.
#include "depthwise.cuh"
namespace co {
struct Depthwise { int dummy; };
bool depthwise_supported(const Geom&) { return false; }
Depthwise* depthwise_create(const Geom&, const void*, std::string& err) { err = "not built"; return nullptr; }
void depthwise_destroy(Depthwise* t) { delete t; }
const char* depthwise_name(const Depthwise*) { return "k_step_depthwise"; }
cudaError_t depthwise_step(Depthwise*, const Geom&, const StepArgs&, const float*, cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace co
