// bw_probe.cu — HBM streaming microbenchmark for the state read-modify-write
// pattern of the dense step epilogue (experiment tool, not product code).
//
// State C2-shaped: 256 streams x 3136 px x 64 ch fp32, R = 2 slots (411 MB).
// One "item" = 128 pixel rows x 32 channels; per item a thread (= row) reads
// 2 slots x 8 quads (float4) and writes 2 slots x 8 quads + 64 B of bf16 y.
//   mode 0: quad-major layout  S[slot][Cq][plane][4]     (current kernel)
//   mode 1: channels-last      S[slot][plane][C], thread = (pixel, quad)
//   mode 2: plain float4 copy of the same byte volume (reference)
// usage: bw_probe <mode> <threads per block> <blocks per SM> <items in flight per thread>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

constexpr long long B = 256, HW = 3136, C = 64, R = 2;
constexpr long long PLANE = B * HW;                 // pixels
constexpr int CQ = C / 4;

template <int F>
__device__ __forceinline__ float4 ld_flavor(const float4* p) {
  float4 v;
  if constexpr (F == 0) return __ldcs(p);
  if constexpr (F == 1) return __ldcg(p);
  if constexpr (F == 2) {
    asm volatile("ld.global.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
  }
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

template <int NI, bool HALO, bool PAD = false, int F = 0>
__global__ void k_quadmajor(float4* __restrict__ st, __nv_bfloat16* __restrict__ y, long long n_items, int work) {
  extern __shared__ float4 dummy_smem[];        // optional: shrink L1 like the dense kernel's 200 KB carve-out
  work &= 0xffff;
  if (work == 0xfff) dummy_smem[threadIdx.x] = make_float4(0, 0, 0, 0);
  // item = (tile of 128 pixels, channel half); thread = pixel row of the tile.
  // HALO: the dense kernel's C2 tile shape -- 2 output rows of 56 in a 58-wide
  // padded halo, rows m -> pixel (m/58)*56 + m%58, 112 valid of 128 lanes.
  const int m = threadIdx.x & 127;
  const int row = HALO ? (m / 58) * 56 + m % 58 : m;
  const bool lane_ok = HALO ? (m % 58 < 56 && m < 116) : true;
  const int TP = HALO ? 112 : 128;
  const int sub = threadIdx.x >> 7;                 // several items per block
  const int per_block = blockDim.x >> 7;
  for (long long it0 = (long long)blockIdx.x * per_block + sub; it0 < n_items; it0 += (long long)gridDim.x * per_block * NI) {
    float4 a[NI][2][8];
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const long long it = it0 + (long long)j * gridDim.x * per_block;
      if (it >= n_items) continue;
      const long long pix = (it >> 1) * TP + row;
      const int q0 = (int)(it & 1) * 8;
      if (pix >= PLANE || !lane_ok) continue;
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[j][s][q] = ld_flavor<F>(st + ((long long)s * CQ + q0 + q) * PLANE + (PAD ? (it >> 1) * 128 + m : pix));
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const long long it = it0 + (long long)j * gridDim.x * per_block;
      if (it >= n_items) continue;
      const long long pix = (it >> 1) * TP + row;
      const int q0 = (int)(it & 1) * 8;
      if (pix >= PLANE || !lane_ok) continue;
      uint4 yv[4];
      // synthetic per-item ALU work (dependent chain), folded into the stored values
      float z = a[j][0][0].x;
      for (int w = 0; w < work; ++w) z = fmaf(z, 0.999f, 1e-7f);
      a[j][0][0].x = z;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 v0 = a[j][0][q], v1 = a[j][1][q];
        v0.x += 1.f; v1.y += 1.f;
        const long long sp = PAD ? (it >> 1) * 128 + m : pix;
        __stcs(st + ((long long)0 * CQ + q0 + q) * PLANE + sp, v1);
        __stcs(st + ((long long)1 * CQ + q0 + q) * PLANE + sp, v0);
        reinterpret_cast<float*>(yv)[q] = v0.x + v1.x;
      }
      *reinterpret_cast<uint4*>(y + pix * C + q0 * 4) = yv[0];
      *reinterpret_cast<uint4*>(y + pix * C + q0 * 4 + 8) = yv[1];
      *reinterpret_cast<uint4*>(y + pix * C + q0 * 4 + 16) = yv[2];
      *reinterpret_cast<uint4*>(y + pix * C + q0 * 4 + 24) = yv[3];
    }
  }
}

template <int NI>
__global__ void k_chlast(float4* __restrict__ st, uint2* __restrict__ y, long long n) {
  // thread = (pixel, quad); state S[slot][plane][C]
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * NI) {
    float4 a[NI][2];
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const long long i = i0 + j * stride;
      if (i < n) { a[j][0] = __ldcs(st + i); a[j][1] = __ldcs(st + n + i); }
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const long long i = i0 + j * stride;
      if (i >= n) continue;
      float4 v0 = a[j][0], v1 = a[j][1];
      v0.x += 1.f; v1.y += 1.f;
      __stcs(st + i, v1);
      __stcs(st + n + i, v0);
      y[i] = make_uint2(__float_as_uint(v0.x), __float_as_uint(v1.x));
    }
  }
}

template <int NI>
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += stride * NI) {
    float4 v[NI];
#pragma unroll
    for (int j = 0; j < NI; ++j) if (i0 + j * stride < n) v[j] = __ldcs(a + i0 + j * stride);
#pragma unroll
    for (int j = 0; j < NI; ++j) if (i0 + j * stride < n) __stcs(b + i0 + j * stride, v[j]);
  }
}

int main(int argc, char** argv) {
  const int mode = atoi(argv[1]), threads = atoi(argv[2]), bps = atoi(argv[3]), ni = atoi(argv[4]);
  const int work = argc > 5 ? atoi(argv[5]) : 0;             // low 16 bits: ALU work; bits 16+: load flavour
  const int smem_bytes = argc > 6 ? atoi(argv[6]) : 0;       // unused dynamic shared memory (L1 carve-out)
  cudaFuncSetAttribute(k_quadmajor<1, true, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_quadmajor<1, true, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_quadmajor<1, true, true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(k_quadmajor<1, true, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long st_elems = R * C * PLANE;         // floats
  float4* st;
  void* y;
  cudaMalloc(&st, st_elems * 4);
  cudaMalloc(&y, PLANE * C * 2 + 4096);
  cudaMemset(st, 0, st_elems * 4);
  float4* other = nullptr;
  const long long bytes_rw = st_elems * 4 * 2 + PLANE * C * 2;   // state read+write + y write
  if (mode == 2) cudaMalloc(&other, bytes_rw / 2 + 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = sms * bps;
  auto launch = [&]() {
    if (mode == 0) {
      const long long n_items = (PLANE + 127) / 128 * 2;
      if (ni == 1) k_quadmajor<1, false><<<grid, threads>>>(st, (__nv_bfloat16*)y, n_items, work);
      else k_quadmajor<2, false><<<grid, threads>>>(st, (__nv_bfloat16*)y, n_items, work);
    } else if (mode == 4) {
      const long long n_items = (PLANE + 111) / 112 * 2 * 112 / 128 - 2;   // padded rows stay inside the buffer
      const int f = work >> 16;
      if (f == 0) k_quadmajor<1, true, true, 0><<<grid, threads, smem_bytes>>>(st, (__nv_bfloat16*)y, n_items, work);
      if (f == 1) k_quadmajor<1, true, true, 1><<<grid, threads, smem_bytes>>>(st, (__nv_bfloat16*)y, n_items, work);
      if (f == 2) k_quadmajor<1, true, true, 2><<<grid, threads, smem_bytes>>>(st, (__nv_bfloat16*)y, n_items, work);
      if (f == 3) k_quadmajor<1, true, true, 3><<<grid, threads, smem_bytes>>>(st, (__nv_bfloat16*)y, n_items, work);
    } else if (mode == 3) {
      const long long n_items = (PLANE + 111) / 112 * 2;
      if (ni == 1) k_quadmajor<1, true><<<grid, threads>>>(st, (__nv_bfloat16*)y, n_items, work);
      else k_quadmajor<2, true><<<grid, threads>>>(st, (__nv_bfloat16*)y, n_items, work);
    } else if (mode == 1) {
      const long long n = PLANE * CQ;
      if (ni == 1) k_chlast<1><<<grid, threads>>>(st, (uint2*)y, n);
      else if (ni == 2) k_chlast<2><<<grid, threads>>>(st, (uint2*)y, n);
      else k_chlast<4><<<grid, threads>>>(st, (uint2*)y, n);
    } else {
      const long long n = bytes_rw / 2 / 16;
      if (ni == 1) k_copy<1><<<grid, threads>>>(st, other, n);
      else if (ni == 2) k_copy<2><<<grid, threads>>>(st, other, n);
      else k_copy<4><<<grid, threads>>>(st, other, n);
    }
  };
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  printf("mode %d threads %d blocks/SM %d NI %d work %d smem %d: %.1f us/launch, %.1f GB/s %s\n", mode, threads, bps, ni, work, smem_bytes,
         ms * 1e3 / reps, bytes_rw / (ms / reps * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  return 0;
}
