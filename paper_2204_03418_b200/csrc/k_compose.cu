// k_compose.cu — the merge of the Residual composite (PAPER.md
// P:301-326, Listing 3): y <- act(y + skip), where y
// already holds the body's output and skip is the identity branch's frame
// (delayed in the composite's ring, or a temporally cropped clip column in
// batch mode).  Pure streaming: one read of y and skip, one write of y, 16-byte
// vectors, grid-stride over rows (streams or clip rows) of n elements each.
#include "common.cuh"

namespace co {

namespace {

template <typename T, int V>
struct alignas(sizeof(T) * V) VecC {
  T v[V];
};

template <typename Ty, typename Tx, int V>
__global__ void __launch_bounds__(256) k_residual_add(Ty* __restrict__ y, int64_t y_rstride, const Tx* __restrict__ x,
                                                      int64_t x_rstride, int64_t rows, int64_t n, int act) {
  const int64_t nv = n / V;
  const int64_t total = rows * nv;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / nv, c = (i - r * nv) * V;
    VecC<Ty, V>* yp = reinterpret_cast<VecC<Ty, V>*>(y + r * y_rstride + c);
    const VecC<Tx, V> xv = *reinterpret_cast<const VecC<Tx, V>*>(x + r * x_rstride + c);
    VecC<Ty, V> yv = *yp;
#pragma unroll
    for (int j = 0; j < V; ++j) yv.v[j] = from_f<Ty>(activate(to_f(yv.v[j]) + to_f(xv.v[j]), act));
    *yp = yv;
  }
}

template <typename Ty, typename Tx>
cudaError_t add_t(void* y, int64_t ys, const void* x, int64_t xs, int64_t rows, int64_t n, int act, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  auto aligned = [&](int V) {
    const int64_t ay = int64_t(sizeof(Ty)) * V, ax = int64_t(sizeof(Tx)) * V;
    return n % V == 0 && ys % V == 0 && xs % V == 0 && reinterpret_cast<uintptr_t>(y) % ay == 0 &&
           reinterpret_cast<uintptr_t>(x) % ax == 0;
  };
  const int V = aligned(8) ? 8 : aligned(4) ? 4 : 1;
  const int64_t items = rows * (n / V);
  const int64_t blocks = (items + 255) / 256, cap = int64_t(sms) * 8;
  const int grid = int(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
  Ty* yp = static_cast<Ty*>(y);
  const Tx* xp = static_cast<const Tx*>(x);
  if (V == 8) k_residual_add<Ty, Tx, 8><<<grid, 256, 0, s>>>(yp, ys, xp, xs, rows, n, act);
  else if (V == 4) k_residual_add<Ty, Tx, 4><<<grid, 256, 0, s>>>(yp, ys, xp, xs, rows, n, act);
  else k_residual_add<Ty, Tx, 1><<<grid, 256, 0, s>>>(yp, ys, xp, xs, rows, n, act);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_residual_add(int y_dtype, void* y, int64_t y_rstride, int x_dtype, const void* x,
                                int64_t x_rstride, int64_t rows, int64_t n, int act, cudaStream_t s) {
  if (rows * n == 0) return cudaSuccess;
  if (y_dtype == BF16)
    return x_dtype == BF16 ? add_t<__nv_bfloat16, __nv_bfloat16>(y, y_rstride, x, x_rstride, rows, n, act, s)
                           : add_t<__nv_bfloat16, float>(y, y_rstride, x, x_rstride, rows, n, act, s);
  return x_dtype == BF16 ? add_t<float, __nv_bfloat16>(y, y_rstride, x, x_rstride, rows, n, act, s)
                         : add_t<float, float>(y, y_rstride, x, x_rstride, rows, n, act, s);
}

}  // namespace co
