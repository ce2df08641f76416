// mma_probe.cu — tcgen05.mma issue-rate microbenchmark (experiment tool, not
// product code): cycles per back-to-back SS-mode kind::f16 MMA (K = 16) into
// one TMEM accumulator, for M = 128 (cta_group::1) and M = 256 (cta_group::2,
// a CTA pair), across N.  Operands are zero shared memory (no-swizzle K-major
// descriptors); timing is clock64 around ITERS MMAs + commit + wait on the
// issuing CTA; "walk" gives every MMA fresh operand addresses (A +4 KB, B the
// next K16 step), as a real K loop does.  Questions it answers: is the ~70-cycle
// cost of an N = 64 MMA (k_step_stem_raw) per instruction or per CTA, and does
// the operand fetch alone keep up at larger N?  Measured (B200, 148 CTAs):
// M = 128: 40.8 / 48.9 / 56.9 / 64.9 / 80.9 / 96.9 / 128.9 cycles at N = 32 / 64 /
// 96 / 128 / 160 / 192 / 256; pairs (M = 256): 40.0 / 44.0 / 50.4 / 65.1 / 81.1 /
// 97.1 / 129.1; identical with fresh operands -- an instruction floor of ~40
// cycles below N = 128, the 128 N / 256 floor above.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2204_03418_b200/csrc \
//        scripts/mma_probe.cu -o scripts/mma_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace co;

constexpr int ITERS = 256;

template <int PAIR>
__global__ void __launch_bounds__(128, 1) k_probe(int N, int lbo_bytes, long long* out, int walk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
  uint32_t* holder = reinterpret_cast<uint32_t*>(bar + 2);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { ptx::mbar_init(bar, 1); ptx::fence_mbar_init(); }
  ptx::fence_proxy_async();
  if (warp == 0) {
    if constexpr (PAIR == 2) ptx::tmem_alloc_pair(holder, 512);
    else ptx::tmem_alloc(holder, 512);
  }
  ptx::tc_fence_before();
  if (PAIR == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *holder;
  const bool leader = PAIR == 1 || ptx::cluster_ctarank() == 0;
  if (warp == 0 && leader) {
    const uint32_t idesc = ptx::idesc_bf16_f32(128 * PAIR, N);
    const uint64_t ad = ptx::smem_desc(ptx::smem_u32(smem), uint32_t(lbo_bytes), 128);
    const uint64_t bd = ptx::smem_desc(ptx::smem_u32(smem + 32 * 1024), uint32_t((N / PAIR) * 16), 128);
    long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int i = 0; i < ITERS; ++i) {
        // walk: each MMA reads fresh operands (A: the next 4 KB of a 32 KB region,
        // B: the next K group pair of the weights), as a real K loop does
        const uint64_t da = walk ? uint64_t((i & 7) * 256) : 0;            // 4 KB steps (16-B units)
        const uint64_t db = walk ? uint64_t((i & 3) * 2 * (N / PAIR)) : 0;  // next K16 of B
        if constexpr (PAIR == 2) ptx::mma_bf16_ss_pair(tmem, ad + da, bd + db, idesc, i ? 1u : 0u);
        else ptx::mma_bf16_ss(tmem, ad + da, bd + db, idesc, i ? 1u : 0u);
      }
      if constexpr (PAIR == 2) ptx::tc_commit_pair(bar, 0x1);
      else ptx::tc_commit(bar);
    }
    __syncwarp();
    ptx::mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  }
  ptx::tc_fence_before();
  if (PAIR == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    if constexpr (PAIR == 2) ptx::tmem_dealloc_pair(tmem, 512);
    else ptx::tmem_dealloc(tmem, 512);
  }
}

template <int PAIR>
long long run(int N, int lbo, int grid, int walk = 0) {
  long long* d;
  cudaMalloc(&d, sizeof(long long));
  const size_t smem = 64 * 1024 + 64;
  cudaFuncSetAttribute(k_probe<PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k_probe<PAIR>, N, lbo, d, walk);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = -1;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return -1; }
  return h;
}

int main() {
  printf("cycles per MMA (K = 16, %d back-to-back, one accumulator)\n", ITERS);
  for (int walk : {0, 1}) {
    printf(walk ? "fresh operands per MMA (A +4 KB, B +1 K16 step)\n" : "the same operands every MMA\n");
    for (int N : {32, 64, 96, 128, 160, 192, 256}) {
      const long long a = run<1>(N, 16, 148, walk), b = run<1>(N, 128 * 16, 148, walk), c = run<2>(N, 16, 148, walk);
      printf("  N %3d: M=128 lbo16 %.1f  M=128 lbo2K %.1f  M=256 pair %.1f  (floor %d / %d)\n", N,
             double(a) / ITERS, double(b) / ITERS, double(c) / ITERS, 128 * N / 256, 256 * N / 512);
    }
  }
  return 0;
}
