// Input generation and precision conversion on the device.
//
// The generator is the reference's counter-based splitmix64 stream
// (/root/reference/proj/include/poas/rng.hpp:17-25): draw i of Rng(seed) is
// mix(seed + (i+1)*0x9e3779b97f4a7c15), so any element can be produced
// independently, in place, bit-identical to the host. Value = 2u - 1 with
// u = (draw >> 11) * 2^-53 (rng.hpp:23), rounded RNE to the storage type.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace poas_b200 {
namespace {

__device__ __forceinline__ double uniform_pm1(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  return 2.0 * u - 1.0;
}

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }

template <typename T>
__global__ void fill_kernel(T* dst, int64_t ld, int64_t rows, int64_t cols, int64_t row0,
                            int64_t col0, int64_t total_cols, uint64_t seed) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int64_t c = i - r * cols;
    const uint64_t idx = static_cast<uint64_t>((row0 + r) * total_cols + col0 + c);
    // fp32 first (the canonical input), then RNE to the storage type.
    const float v = __double2float_rn(uniform_pm1(seed, idx));
    dst[r * ld + c] = from_f32<T>(v);
  }
}

template <typename T>
__global__ void convert_kernel(const float* src, int64_t ld_src, T* dst, int64_t ld_dst,
                               int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols;
    const int64_t c = i - r * cols;
    dst[r * ld_dst + c] = from_f32<T>(src[r * ld_src + c]);
  }
}

// Vectorised contiguous path: 4 fp32 -> 4 x 16-bit per thread.
template <typename T>
__global__ void convert_contig_kernel(const float4* src, T* dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    T o[4] = {from_f32<T>(v.x), from_f32<T>(v.y), from_f32<T>(v.z), from_f32<T>(v.w)};
    *reinterpret_cast<uint2*>(dst + 4 * i) = *reinterpret_cast<uint2*>(o);
  }
}

// Streaming read of n4 float4s by `gridDim.x` CTAs: what a unit on that SM
// budget can pull from HBM. The checksum store is never taken in practice
// (it defeats dead-code elimination).
__global__ void __launch_bounds__(512) stream_read_kernel(const float4* __restrict__ p, int64_t n4,
                                                          float* sink) {
  float acc = 0.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldcs(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345678e-30f) sink[0] = acc;
}

// Start gate of one executor repeat: holds the stream until the host sets
// *flag (mapped pinned memory), so the events recorded after it mark when
// the whole repeat is queued. Gives up after `timeout_ns` (a host that died
// mid-enqueue must not leave the GPU spinning).
__global__ void gate_kernel(const volatile int* flag, unsigned long long timeout_ns) {
  unsigned long long start, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (*flag == 0) {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > timeout_ns) break;
  }
}

int grid_for(int64_t n) {
  const int64_t blocks = (n + 255) / 256;
  const int64_t cap = static_cast<int64_t>(device_sm_count()) * 16;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace

cudaError_t gate_wait(const int* flag, cudaStream_t stream) {
  gate_kernel<<<1, 1, 0, stream>>>(flag, 10ull * 1000000000ull);
  return cudaGetLastError();
}

cudaError_t stream_read(const void* src, size_t bytes, int num_ctas, float* sink,
                        cudaStream_t stream) {
  if (bytes < 16) return cudaSuccess;
  const int grid = num_ctas > 0 ? num_ctas : device_sm_count();
  stream_read_kernel<<<grid, 512, 0, stream>>>(static_cast<const float4*>(src),
                                               static_cast<int64_t>(bytes / 16), sink);
  return cudaGetLastError();
}

cudaError_t fill_uniform(AbType t, void* dst, int64_t ld, int64_t rows, int64_t cols,
                         int64_t row0, int64_t col0, int64_t total_cols, uint64_t seed,
                         cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int g = grid_for(rows * cols);
  switch (t) {
    case AbType::f32:
      fill_kernel<float><<<g, 256, 0, stream>>>(static_cast<float*>(dst), ld, rows, cols, row0,
                                                col0, total_cols, seed);
      break;
    case AbType::bf16:
      fill_kernel<__nv_bfloat16><<<g, 256, 0, stream>>>(static_cast<__nv_bfloat16*>(dst), ld,
                                                        rows, cols, row0, col0, total_cols, seed);
      break;
    case AbType::f16:
      fill_kernel<__half><<<g, 256, 0, stream>>>(static_cast<__half*>(dst), ld, rows, cols, row0,
                                                 col0, total_cols, seed);
      break;
  }
  return cudaGetLastError();
}

cudaError_t convert_f32(AbType t, const float* src, int64_t ld_src, void* dst, int64_t ld_dst,
                        int64_t rows, int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (t == AbType::f32) return cudaErrorInvalidValue;
  const bool contig = ld_src == cols && ld_dst == cols && (rows * cols) % 4 == 0 &&
                      ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(dst) & 7) == 0);
  if (contig) {
    const int64_t n4 = rows * cols / 4;
    const int g = grid_for(n4);
    if (t == AbType::bf16)
      convert_contig_kernel<__nv_bfloat16><<<g, 256, 0, stream>>>(
          reinterpret_cast<const float4*>(src), static_cast<__nv_bfloat16*>(dst), n4);
    else
      convert_contig_kernel<__half><<<g, 256, 0, stream>>>(reinterpret_cast<const float4*>(src),
                                                           static_cast<__half*>(dst), n4);
    return cudaGetLastError();
  }
  const int g = grid_for(rows * cols);
  if (t == AbType::bf16)
    convert_kernel<__nv_bfloat16><<<g, 256, 0, stream>>>(src, ld_src,
                                                         static_cast<__nv_bfloat16*>(dst), ld_dst,
                                                         rows, cols);
  else
    convert_kernel<__half><<<g, 256, 0, stream>>>(src, ld_src, static_cast<__half*>(dst), ld_dst,
                                                  rows, cols);
  return cudaGetLastError();
}

}  // namespace poas_b200
