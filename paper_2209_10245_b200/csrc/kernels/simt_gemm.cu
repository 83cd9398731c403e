// CUDA-core unit of one B200: fp32 SIMT GEMM (FFMA pipe).
//
//   C[M x N] (=|+=) A[M x K] . B[K x N]     all fp32, row-major
//
// Replaces the GPU-kind synthetic law of the reference (SyntheticBackend::
// time_gemm, /root/reference/proj/src/simulator.cpp:30-34).
//
// Default kernel: simt_gemm2_kernel<.., 32, 256, 4, true> (FFMA2, 128 x 256
// x 32 tiles, fragments double buffered in registers, B-pair-major FFMA2
// order, grouped raster; below). simt_gemm_kernel: the earlier plain-FFMA kernel, 128 x 128
// (or 128 x 256) x 16 CTA tiles, 256 threads, 8 x 8 (8 x 16) register
// micro-tile per thread (4-column quadrants 64 apart so the float4
// shared-memory reads stay conflict-free), 128-bit coalesced global loads
// prefetched into registers one K-step ahead, shared memory double buffered
// (one barrier per K-step). Persistent over tiles: grid = the SM budget.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kernels.hpp"

namespace poas_b200 {
namespace {

constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kBK = 16;
constexpr int kThreads = 256;
constexpr int kPad = 4;  // As row padding keeps the transposed stores spread over banks
constexpr int kSmemFloats = 2 * kBK * (kBM + kPad) + 2 * kBK * kBN;

struct SimtArgs {
  int M, N, K;
  const float* A;
  long long lda;
  const float* B;
  long long ldb;
  float* C;
  long long ldc;
  int accumulate;
  int tiles_m, tiles_n;
};

// kWN = 2: 128 x 128 CTA tile, 8 x 8 per thread; kWN = 4: 128 x 256, 8 x 16
// per thread (four 4-column quadrants 64 apart: fewer shared-memory reads
// per FMA).
template <bool kVec, int kWN, int kMinBlocks = 1>
__global__ void __launch_bounds__(kThreads, kMinBlocks) simt_gemm_kernel(const SimtArgs p) {
  constexpr int kTN = 64 * kWN;  // CTA tile width
  constexpr int kCols = 4 * kWN;  // per-thread columns
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float* As = smem;                          // [2][kBK][kBM + kPad]  (A transposed)
  float* Bs = smem + 2 * kBK * (kBM + kPad);  // [2][kBK][kTN]

  const int tid = threadIdx.x;
  const int tx = tid & 15;  // column group
  const int ty = tid >> 4;  // row group

  // Global-load assignment: A tile 128 x 16 -> two float4 per thread along K;
  // B tile 16 x kTN -> kWN float4 per thread, 64 columns apart.
  const int a_row = tid >> 1;          // 0..127
  const int a_k = (tid & 1) * 8;       // 0 or 8 (two float4: +0, +4)
  const int b_k = tid >> 4;            // 0..15
  const int b_col = (tid & 15) * 4;    // + 64 h

  const int tiles_n = (p.N + kTN - 1) / kTN;
  const int total = p.tiles_m * tiles_n;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int mb = t / tiles_n;
    const int nb = t % tiles_n;
    const int m0 = mb * kBM;
    const int n0 = nb * kTN;

    float acc[8][kCols];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < kCols; ++j) acc[i][j] = 0.f;

    float ra[8], rb[4 * kWN];
    auto load_global = [&](int k0) {
      const int gr = m0 + a_row;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gk = k0 + a_k + h * 4;
        if (kVec && gr < p.M && gk + 3 < p.K) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(p.A + (long long)gr * p.lda + gk));
          ra[4 * h] = v.x; ra[4 * h + 1] = v.y; ra[4 * h + 2] = v.z; ra[4 * h + 3] = v.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            ra[4 * h + e] = (gr < p.M && gk + e < p.K) ? p.A[(long long)gr * p.lda + gk + e] : 0.f;
        }
      }
      const int gk = k0 + b_k;
#pragma unroll
      for (int h = 0; h < kWN; ++h) {
        const int gc = n0 + b_col + h * 64;
        if (kVec && gk < p.K && gc + 3 < p.N) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(p.B + (long long)gk * p.ldb + gc));
          rb[4 * h] = v.x; rb[4 * h + 1] = v.y; rb[4 * h + 2] = v.z; rb[4 * h + 3] = v.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            rb[4 * h + e] = (gk < p.K && gc + e < p.N) ? p.B[(long long)gk * p.ldb + gc + e] : 0.f;
        }
      }
    };
    auto store_shared = [&](int buf) {
      float* as = As + buf * kBK * (kBM + kPad);
#pragma unroll
      for (int e = 0; e < 8; ++e) as[(a_k + e) * (kBM + kPad) + a_row] = ra[e];
      float* bs = Bs + buf * kBK * kTN + b_k * kTN + b_col;
#pragma unroll
      for (int h = 0; h < kWN; ++h)
        *reinterpret_cast<float4*>(bs + 64 * h) =
            make_float4(rb[4 * h], rb[4 * h + 1], rb[4 * h + 2], rb[4 * h + 3]);
    };

    const int k_steps = (p.K + kBK - 1) / kBK;
    load_global(0);
    __syncthreads();  // previous tile's readers are done with both buffers
    store_shared(0);
    __syncthreads();

    for (int ks = 0; ks < k_steps; ++ks) {
      const int buf = ks & 1;
      if (ks + 1 < k_steps) load_global((ks + 1) * kBK);
      const float* as = As + buf * kBK * (kBM + kPad);
      const float* bs = Bs + buf * kBK * kTN;
#pragma unroll
      for (int k = 0; k < kBK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * (kBM + kPad) + ty * 4);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * (kBM + kPad) + 64 + ty * 4);
        float b[kCols];
#pragma unroll
        for (int h = 0; h < kWN; ++h) {
          const float4 v = *reinterpret_cast<const float4*>(bs + k * kTN + 64 * h + tx * 4);
          b[4 * h] = v.x; b[4 * h + 1] = v.y; b[4 * h + 2] = v.z; b[4 * h + 3] = v.w;
        }
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < kCols; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      if (ks + 1 < k_steps) store_shared(buf ^ 1);
      __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      if (r >= p.M) continue;
      float* crow = p.C + (long long)r * p.ldc;
#pragma unroll
      for (int h = 0; h < kWN; ++h) {
        const int c = n0 + h * 64 + tx * 4;
        if (kVec && c + 3 < p.N) {
          float4 o = make_float4(acc[i][4 * h], acc[i][4 * h + 1], acc[i][4 * h + 2],
                                 acc[i][4 * h + 3]);
          if (p.accumulate) {
            const float4 q = *reinterpret_cast<const float4*>(crow + c);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4*>(crow + c) = o;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c + e < p.N) {
              float o = acc[i][4 * h + e];
              if (p.accumulate) o += crow[c + e];
              crow[c + e] = o;
            }
          }
        }
      }
    }
  }
}

// FFMA2 kernel (default for M >= 128). Blackwell's fp32 pipe takes packed
// pairs: fma.rn.f32x2 (SASS FFMA2) does two FMAs per lane per issue, with a
// scalar operand broadcast to both halves -- exactly the outer-product step
// acc[i][j..j+1] += a[i] * b[j..j+1]. With plain FFMA every FMA costs an
// issue slot and the loop sat at ~65% of the FMA pipe (shared-memory loads,
// address arithmetic and barriers compete for the same slots); with FFMA2
// the 128 FMAs of a thread's k-step are 64 issues.
//   CTA tile 128 x 256 x 16, 256 threads, 8 x 16 accumulators per thread
//   (acc2[8][8] float2 pairs: four 4-column quadrants 64 apart, so the
//   float4 shared-memory reads stay conflict-free), A transposed into shared
//   memory, 128-bit global loads one K-step ahead in registers, two shared
//   buffers (one barrier per K-step), persistent over tiles in a grouped
//   raster (8 M-tiles per group: the ~148 tiles in flight share their A and
//   B panels through L2 instead of streaming all of B per M-row of tiles).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int kN>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(kN) : "memory");
}

constexpr int kGroupM2 = 8;

// FFMA2 kernel family. A CTA of kThr threads computes a 128 x kTN tile;
// each thread owns 8 rows (two 4-row groups 64 apart) x 4*kNQ columns
// (kNQ 4-column quadrants kTN/kNQ apart) as float2 accumulators, and the
// float4 shared-memory reads stay conflict-free. Variants (POAS_SIMT_TILE):
//   ffma2    kThr 256, kNQ 4: 128 x 256, one CTA per SM (8 x 16 per thread)
//   ffma2x2  kThr 128, kNQ 4: 128 x 128, two CTAs per SM (8 x 16 per thread)
//   ffma2w16 kThr 256, kNQ 2: 128 x 128, two CTAs per SM (8 x 8 per thread,
//            16 warps per SM: twice the warps to hide shared-memory and
//            fixed-latency waits, 1/3 more shared-memory reads per FMA)
template <bool kVec, int kBK2 = 16, int kThr = kThreads, int kNQ = 4, bool kJOuter = false>
__global__ void __launch_bounds__(kThr, (kThr * kNQ) == 1024 ? 1 : 2) simt_gemm2_kernel(const SimtArgs p) {
  constexpr int kTX = kThr / 16;      // threads across a row of the tile (16 down)
  constexpr int kQ = kTX * 4;         // column distance of a thread's quadrants
  constexpr int kTN = kQ * kNQ;       // CTA tile width (columns)
  constexpr int kBK = kBK2;           // K depth of a step (16 or 32)
  constexpr int kAV = kBM * kBK / (4 * kThr);  // A float4 loads per thread per step
  constexpr int kBP = kBK / 16;       // B passes per step (16 rows, kNQ float4 per thread each)
  static_assert(kAV >= 1 && kBM * kBK == 4 * kThr * kAV, "A tile split");
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float* As = smem;                          // [2][kBK][kBM + kPad]  (A transposed)
  float* Bs = smem + 2 * kBK * (kBM + kPad);  // [2][kBK][kTN]

  const int tid = threadIdx.x;
  const int tx = tid % kTX;
  const int ty = tid / kTX;
  // a warp loads 32 consecutive rows of A at one k offset: its transposed
  // shared stores hit 32 distinct banks
  const int a_row = tid & 127;
  const int a_k = (tid >> 7) * (kAV * 4);
  const int b_k = tid / kTX;
  const int b_col = tx * 4;

  const int tiles_n = (p.N + kTN - 1) / kTN;
  const int total = p.tiles_m * tiles_n;
  const int per_group = kGroupM2 * tiles_n;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int group = t / per_group;
    const int first_m = group * kGroupM2;
    const int gm = min(p.tiles_m - first_m, kGroupM2);
    const int in_group = t - group * per_group;
    const int mb = first_m + in_group % gm;
    const int nb = in_group / gm;
    const int m0 = mb * kBM;
    const int n0 = nb * kTN;

    float2 acc[8][2 * kNQ];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 2 * kNQ; ++j) acc[i][j] = make_float2(0.f, 0.f);

    // A: 128-bit loads into registers one K-step ahead (unconditional for
    // interior tiles), stored transposed at the end of the step. B: cp.async
    // straight into the other shared buffer (no registers, no transpose;
    // out-of-range bytes zero-filled) for 16-byte aligned operands.
    const bool full_m = kVec && m0 + kBM <= p.M;
    float4 ra[kAV], rb[kNQ * kBP];
    auto load_a = [&](int k0) {
      const int gr = m0 + a_row;
      if (full_m && k0 + kBK <= p.K) {
        const float4* src = reinterpret_cast<const float4*>(p.A + (long long)gr * p.lda + k0 + a_k);
#pragma unroll
        for (int h = 0; h < kAV; ++h) ra[h] = __ldg(src + h);
        return;
      }
#pragma unroll
      for (int h = 0; h < kAV; ++h) {
        const int gk = k0 + a_k + h * 4;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = (gr < p.M && gk + e < p.K) ? p.A[(long long)gr * p.lda + gk + e] : 0.f;
        ra[h] = make_float4(v[0], v[1], v[2], v[3]);
      }
    };
    auto load_b = [&](int k0, int buf) {
#pragma unroll
      for (int q = 0; q < kBP; ++q) {
        const int gk = k0 + b_k + 16 * q;
        if constexpr (kVec) {
          float* bs = Bs + buf * kBK * kTN + (b_k + 16 * q) * kTN + b_col;
#pragma unroll
          for (int h = 0; h < kNQ; ++h) {
            const int gc = n0 + b_col + h * kQ;
            const int bytes = gk < p.K ? max(0, min(16, (p.N - gc) * 4)) : 0;
            cp_async16(bs + kQ * h, bytes ? p.B + (long long)gk * p.ldb + gc : p.B, bytes);
          }
        } else {
#pragma unroll
          for (int h = 0; h < kNQ; ++h) {
            const int gc = n0 + b_col + h * kQ;
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              v[e] = (gk < p.K && gc + e < p.N) ? p.B[(long long)gk * p.ldb + gc + e] : 0.f;
            rb[kNQ * q + h] = make_float4(v[0], v[1], v[2], v[3]);
          }
        }
      }
      if constexpr (kVec) cp_async_commit();
    };
    auto store_shared = [&](int buf) {
      float* as = As + buf * kBK * (kBM + kPad) + a_row;
#pragma unroll
      for (int h = 0; h < kAV; ++h) {
        as[(a_k + 4 * h) * (kBM + kPad)] = ra[h].x;
        as[(a_k + 4 * h + 1) * (kBM + kPad)] = ra[h].y;
        as[(a_k + 4 * h + 2) * (kBM + kPad)] = ra[h].z;
        as[(a_k + 4 * h + 3) * (kBM + kPad)] = ra[h].w;
      }
      if constexpr (kVec) {
        cp_async_wait<0>();  // this thread's B copies for the step have landed
      } else {
#pragma unroll
        for (int q = 0; q < kBP; ++q) {
          float4* bs = reinterpret_cast<float4*>(Bs + buf * kBK * kTN + (b_k + 16 * q) * kTN + b_col);
#pragma unroll
          for (int h = 0; h < kNQ; ++h) bs[(kQ / 4) * h] = rb[kNQ * q + h];
        }
      }
    };

    const int k_steps = (p.K + kBK - 1) / kBK;
    __syncthreads();  // previous tile's readers are done with both buffers
    load_a(0);
    load_b(0, 0);
    store_shared(0);
    __syncthreads();

    // Fragments (one k's 8 A values and 4*kNQ B values) are double
    // buffered in registers: the next k's are read while this k's FFMA2s
    // issue, and the step's barrier sits before its LAST k, so the next
    // step's first fragment is read (after the barrier) while that k's
    // FFMA2s still have work -- no warp waits on shared memory right after
    // the barrier.
    float4 fa[2][2], fb[2][kNQ];
    auto load_frag = [&](int buf, int k, int slot) {
      const float* as = As + buf * kBK * (kBM + kPad) + ty * 4 + k * (kBM + kPad);
      const float4* bs = reinterpret_cast<const float4*>(Bs + buf * kBK * kTN) + tx + k * (kTN / 4);
      fa[slot][0] = *reinterpret_cast<const float4*>(as);
      fa[slot][1] = *reinterpret_cast<const float4*>(as + 64);
#pragma unroll
      for (int h = 0; h < kNQ; ++h) fb[slot][h] = bs[(kQ / 4) * h];
    };
    load_frag(0, 0, 0);
    for (int ks = 0; ks < k_steps; ++ks) {
      const int buf = ks & 1;
      const bool more = ks + 1 < k_steps;
      if (more) {
        load_a((ks + 1) * kBK);
        load_b((ks + 1) * kBK, buf ^ 1);
      }
#pragma unroll
      for (int k = 0; k < kBK; ++k) {
        const int cur = k & 1;
        if (k + 1 < kBK) {
          load_frag(buf, k + 1, cur ^ 1);
        } else {
          if (more) store_shared(buf ^ 1);
          __syncthreads();
          if (more) load_frag(buf ^ 1, 0, cur ^ 1);
        }
        const float4 a0 = fa[cur][0], a1 = fa[cur][1];
        float2 b[2 * kNQ];
#pragma unroll
        for (int h = 0; h < kNQ; ++h) {
          const float4 v = fb[cur][h];
          b[2 * h] = make_float2(v.x, v.y);
          b[2 * h + 1] = make_float2(v.z, v.w);
        }
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        if constexpr (kJOuter) {  // consecutive FFMA2s share the B pair
#pragma unroll
          for (int j = 0; j < 2 * kNQ; ++j)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][j] = __ffma2_rn(make_float2(a[i], a[i]), b[j], acc[i][j]);
        } else {  // consecutive FFMA2s share the A scalar
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float2 ai = make_float2(a[i], a[i]);
#pragma unroll
            for (int j = 0; j < 2 * kNQ; ++j) acc[i][j] = __ffma2_rn(ai, b[j], acc[i][j]);
          }
        }
      }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      if (r >= p.M) continue;
      float* crow = p.C + (long long)r * p.ldc;
#pragma unroll
      for (int h = 0; h < kNQ; ++h) {
        const int c = n0 + h * kQ + tx * 4;
        const float2 lo = acc[i][2 * h], hi = acc[i][2 * h + 1];
        if (kVec && c + 3 < p.N) {
          float4 o = make_float4(lo.x, lo.y, hi.x, hi.y);
          if (p.accumulate) {
            const float4 q = *reinterpret_cast<const float4*>(crow + c);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4*>(crow + c) = o;
        } else {
          const float v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c + e < p.N) {
              float o = v[e];
              if (p.accumulate) o += crow[c + e];
              crow[c + e] = o;
            }
          }
        }
      }
    }
  }
}

// FFMA2 with 16 warps per SM: the same 128 x 256 x 16 CTA tile over 512
// threads, 8 x 8 accumulators each (two 4-row groups 64 apart x two
// 4-column quadrants 128 apart). With 8 warps (two per scheduler) a
// warp's shared-memory latency and fixed-latency waits leave the FP32 pipe
// idle ~25% of the time (ncu: stall "wait" 1.2 + short scoreboard 0.35 per
// issue); four warps per scheduler cover them, at 1/3 more shared-memory
// loads per FMA (still ~60% of the smem wavefront budget).
constexpr int kThreads3 = 512;

template <bool kVec>
__global__ void __launch_bounds__(kThreads3, 1) simt_gemm3_kernel(const SimtArgs p) {
  constexpr int kTN = 256;
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  float* As = smem;                          // [2][kBK][kBM + kPad]  (A transposed)
  float* Bs = smem + 2 * kBK * (kBM + kPad);  // [2][kBK][kTN]

  const int tid = threadIdx.x;
  const int tx = tid & 31;  // columns tx*4 + {0..3} and 128 + tx*4 + {0..3}
  const int ty = tid >> 5;  // rows ty*4 + {0..3} and 64 + ty*4 + {0..3}
  // global loads: A 128 x 16 (one float4 per thread: a warp = 32 rows, so
  // the transposed shared stores hit 32 distinct banks); B 16 x 256 (two)
  const int a_row = tid & 127;
  const int a_k = (tid >> 7) * 4;
  const int b_k = tid >> 5;
  const int b_col = tx * 4;

  const int tiles_n = (p.N + kTN - 1) / kTN;
  const int total = p.tiles_m * tiles_n;
  const int per_group = kGroupM2 * tiles_n;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int group = t / per_group;
    const int first_m = group * kGroupM2;
    const int gm = min(p.tiles_m - first_m, kGroupM2);
    const int in_group = t - group * per_group;
    const int m0 = (first_m + in_group % gm) * kBM;
    const int n0 = (in_group / gm) * kTN;

    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);

    float4 ra, rb[2];
    auto load_global = [&](int k0) {
      const int gr = m0 + a_row;
      const int gk = k0 + a_k;
      if (kVec && gr < p.M && gk + 3 < p.K) {
        ra = __ldg(reinterpret_cast<const float4*>(p.A + (long long)gr * p.lda + gk));
      } else {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          v[e] = (gr < p.M && gk + e < p.K) ? p.A[(long long)gr * p.lda + gk + e] : 0.f;
        ra = make_float4(v[0], v[1], v[2], v[3]);
      }
      const int bk = k0 + b_k;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gc = n0 + b_col + h * 128;
        if (kVec && bk < p.K && gc + 3 < p.N) {
          rb[h] = __ldg(reinterpret_cast<const float4*>(p.B + (long long)bk * p.ldb + gc));
        } else {
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[e] = (bk < p.K && gc + e < p.N) ? p.B[(long long)bk * p.ldb + gc + e] : 0.f;
          rb[h] = make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    };
    auto store_shared = [&](int buf) {
      float* as = As + buf * kBK * (kBM + kPad) + a_k * (kBM + kPad) + a_row;
      as[0] = ra.x;
      as[kBM + kPad] = ra.y;
      as[2 * (kBM + kPad)] = ra.z;
      as[3 * (kBM + kPad)] = ra.w;
      float4* bs = reinterpret_cast<float4*>(Bs + buf * kBK * kTN + b_k * kTN + b_col);
      bs[0] = rb[0];
      bs[32] = rb[1];
    };

    const int k_steps = (p.K + kBK - 1) / kBK;
    load_global(0);
    __syncthreads();  // previous tile's readers are done with both buffers
    store_shared(0);
    __syncthreads();

    for (int ks = 0; ks < k_steps; ++ks) {
      const int buf = ks & 1;
      if (ks + 1 < k_steps) load_global((ks + 1) * kBK);
      const float* as = As + buf * kBK * (kBM + kPad) + ty * 4;
      const float4* bs = reinterpret_cast<const float4*>(Bs + buf * kBK * kTN) + tx;
#pragma unroll
      for (int k = 0; k < kBK; ++k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * (kBM + kPad));
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * (kBM + kPad) + 64);
        const float4 v0 = bs[k * (kTN / 4)];
        const float4 v1 = bs[k * (kTN / 4) + 32];
        const float2 b[4] = {make_float2(v0.x, v0.y), make_float2(v0.z, v0.w), make_float2(v1.x, v1.y),
                             make_float2(v1.z, v1.w)};
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 ai = make_float2(a[i], a[i]);
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __ffma2_rn(ai, b[j], acc[i][j]);
        }
      }
      if (ks + 1 < k_steps) store_shared(buf ^ 1);
      __syncthreads();
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      if (r >= p.M) continue;
      float* crow = p.C + (long long)r * p.ldc;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + h * 128 + tx * 4;
        const float2 lo = acc[i][2 * h], hi = acc[i][2 * h + 1];
        if (kVec && c + 3 < p.N) {
          float4 o = make_float4(lo.x, lo.y, hi.x, hi.y);
          if (p.accumulate) {
            const float4 q = *reinterpret_cast<const float4*>(crow + c);
            o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
          }
          *reinterpret_cast<float4*>(crow + c) = o;
        } else {
          const float v[4] = {lo.x, lo.y, hi.x, hi.y};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (c + e < p.N) {
              float o = v[e];
              if (p.accumulate) o += crow[c + e];
              crow[c + e] = o;
            }
          }
        }
      }
    }
  }
}

// Skinny-M path (M < 128: a co-executed CUDA-core share is often a handful
// of rows). A 16 x 1024 output block per CTA: each thread keeps all 16 rows
// x 4 columns in registers, streams its B columns straight from global
// memory (one coalesced 128-bit load per k, 8 k-steps in flight), and reads
// the 16 x kSkBK A panel from shared memory as warp-broadcast float4s.
constexpr int kSkCols = 1024;
constexpr int kSkBK = 32;

template <bool kVec, int kSkRows>
__global__ void __launch_bounds__(kThreads, 1) simt_skinny_kernel(const SimtArgs p) {
  __shared__ __align__(16) float As[kSkBK][kSkRows];  // A panel, transposed
  const int tid = threadIdx.x;
  const int row_groups = (p.M + kSkRows - 1) / kSkRows;
  const int col_blocks = (p.N + kSkCols - 1) / kSkCols;
  const int total = row_groups * col_blocks;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int r0 = (t % row_groups) * kSkRows;
    const int c = (t / row_groups) * kSkCols + tid * 4;
    float acc[kSkRows][4];
#pragma unroll
    for (int i = 0; i < kSkRows; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    const bool col_vec = kVec && c + 3 < p.N;
    for (int k0 = 0; k0 < p.K; k0 += kSkBK) {
      __syncthreads();
      // 256 threads stage 16 x 32 A values (2 each), transposed.
      for (int e = tid; e < kSkRows * kSkBK; e += kThreads) {
        const int rr = e / kSkBK, kk = e % kSkBK;
        const int gr = r0 + rr, gk = k0 + kk;
        As[kk][rr] = (gr < p.M && gk < p.K) ? p.A[(long long)gr * p.lda + gk] : 0.f;
      }
      __syncthreads();
      const int kn = min(kSkBK, p.K - k0);
#pragma unroll 8
      for (int kk = 0; kk < kSkBK; ++kk) {
        if (kk >= kn) break;
        const float* brow = p.B + (long long)(k0 + kk) * p.ldb;
        float4 b;
        if (col_vec) {
          b = __ldg(reinterpret_cast<const float4*>(brow + c));
        } else {
          b.x = c < p.N ? brow[c] : 0.f;
          b.y = c + 1 < p.N ? brow[c + 1] : 0.f;
          b.z = c + 2 < p.N ? brow[c + 2] : 0.f;
          b.w = c + 3 < p.N ? brow[c + 3] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < kSkRows / 4; ++q) {
          const float4 a = *reinterpret_cast<const float4*>(&As[kk][4 * q]);
          const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            acc[4 * q + i][0] = fmaf(av[i], b.x, acc[4 * q + i][0]);
            acc[4 * q + i][1] = fmaf(av[i], b.y, acc[4 * q + i][1]);
            acc[4 * q + i][2] = fmaf(av[i], b.z, acc[4 * q + i][2]);
            acc[4 * q + i][3] = fmaf(av[i], b.w, acc[4 * q + i][3]);
          }
        }
      }
    }
    if (c >= p.N) continue;
#pragma unroll
    for (int i = 0; i < kSkRows; ++i) {
      const int r = r0 + i;
      if (r >= p.M) break;
      float* crow = p.C + (long long)r * p.ldc;
      if (col_vec) {
        float4 o = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (p.accumulate) {
          const float4 q = *reinterpret_cast<const float4*>(crow + c);
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        *reinterpret_cast<float4*>(crow + c) = o;
      } else {
        for (int e = 0; e < 4 && c + e < p.N; ++e) {
          float o = acc[i][e];
          if (p.accumulate) o += crow[c + e];
          crow[c + e] = o;
        }
      }
    }
  }
}

// Pipelined skinny path for 16-byte aligned operands. A skinny share is
// bound by streaming B (each B element feeds only `kRows` FMAs), so the
// kernel is built around bytes in flight: every thread cp.async's its own
// 4 columns of `kPipeK` consecutive B rows per stage into a `stages`-deep
// shared-memory ring (up to ~190 KB in flight per SM on an exclusive SM).
// A thread only ever reads the smem it filled itself, so the ring needs no
// block barrier -- only per-thread cp.async group waits. A values come
// through L1 as warp-uniform 128-bit loads.
constexpr int kPipeK = 8;  // B rows per stage: 8 x 1024 x 4 B = 32 KB per stage

template <int kRows>
__global__ void __launch_bounds__(kThreads, 1) simt_skinny_pipe_kernel(const SimtArgs p,
                                                                         int stages) {
  // Ring slot = B part [kPipeK][kThreads] float4 (thread-private columns)
  //           + A part [kRows][kPipeK] floats (shared, filled by 2*kRows threads).
  constexpr int kSlotB = kPipeK * kThreads;            // float4s
  constexpr int kSlotA = kRows * kPipeK / 4;           // float4s
  constexpr int kSlot = kSlotB + kSlotA;
  extern __shared__ float4 ring[];
  const int tid = threadIdx.x;
  const int row_groups = (p.M + kRows - 1) / kRows;
  const int col_blocks = (p.N + kSkCols - 1) / kSkCols;
  const int total = row_groups * col_blocks;
  const int steps = (p.K + kPipeK - 1) / kPipeK;
  constexpr int kAhead = 5;  // wait depth below is compile-time: stages must be kAhead + 1

  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int r0 = (t % row_groups) * kRows;
    const int c = (t / row_groups) * kSkCols + tid * 4;
    const int col_bytes = c < p.N ? min(16, (p.N - c) * 4) : 0;
    const float* bcol = p.B + (c < p.N ? c : 0);
    // A staging role: threads [0, 2*kRows) copy 4 floats each per stage.
    const int a_row = tid >> 1, a_half = tid & 1;
    const bool a_loader = tid < 2 * kRows;
    const bool a_row_ok = a_loader && r0 + a_row < p.M;
    const float* arow = p.A + (long long)(a_row_ok ? r0 + a_row : 0) * p.lda;

    auto issue = [&](int step) {
      if (step < steps) {
        float4* slot = ring + (step % stages) * kSlot;
        const int k0 = step * kPipeK;
#pragma unroll
        for (int kk = 0; kk < kPipeK; ++kk) {
          const bool in = k0 + kk < p.K;
          cp_async16(slot + kk * kThreads + tid, in ? bcol + (long long)(k0 + kk) * p.ldb : bcol,
                     in ? col_bytes : 0);
        }
        if (a_loader) {
          const int ka = k0 + a_half * 4;
          const int bytes = a_row_ok ? max(0, min(16, (p.K - ka) * 4)) : 0;
          cp_async16(slot + kSlotB + a_row * (kPipeK / 4) + a_half, bytes ? arow + ka : arow, bytes);
        }
      }
      cp_async_commit();  // empty groups keep the wait arithmetic uniform
    };

    float acc[kRows][4];
#pragma unroll
    for (int i = 0; i < kRows; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;

    __syncthreads();  // the previous tile's readers are done with every slot
    for (int s = 0; s < kAhead; ++s) issue(s);
    for (int step = 0; step < steps; ++step) {
      cp_async_wait<kAhead - 1>();  // this thread's copies for `step` have landed
      __syncthreads();               // ... and every thread's (the shared A part)
      issue(step + kAhead);          // refills the slot everyone finished last step
      const float4* slot = ring + (step % stages) * kSlot;
      const float* As = reinterpret_cast<const float*>(slot + kSlotB);
#pragma unroll
      for (int kk = 0; kk < kPipeK; ++kk) {
        const float4 b = slot[kk * kThreads + tid];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
          const float a = As[i * kPipeK + kk];  // warp-uniform: broadcast
          acc[i][0] = fmaf(a, b.x, acc[i][0]);
          acc[i][1] = fmaf(a, b.y, acc[i][1]);
          acc[i][2] = fmaf(a, b.z, acc[i][2]);
          acc[i][3] = fmaf(a, b.w, acc[i][3]);
        }
      }
    }
    cp_async_wait<0>();
    if (c >= p.N) continue;
#pragma unroll
    for (int i = 0; i < kRows; ++i) {
      const int r = r0 + i;
      if (r >= p.M) break;
      float* crow = p.C + (long long)r * p.ldc;
      if (c + 3 < p.N) {
        float4 o = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (p.accumulate) {
          const float4 q = *reinterpret_cast<const float4*>(crow + c);
          o.x += q.x; o.y += q.y; o.z += q.z; o.w += q.w;
        }
        *reinterpret_cast<float4*>(crow + c) = o;
      } else {
        for (int e = 0; e < 4 && c + e < p.N; ++e) {
          float o = acc[i][e];
          if (p.accumulate) o += crow[c + e];
          crow[c + e] = o;
        }
      }
    }
  }
}

template <int kRows>
cudaError_t launch_pipe_t(int grid, cudaStream_t stream, const SimtArgs& p) {
  constexpr int stages = 6;  // kAhead + 1
  const size_t smem =
      static_cast<size_t>(stages) * (kPipeK * kThreads + kRows * kPipeK / 4) * sizeof(float4);
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [smem] {
    err = cudaFuncSetAttribute(simt_skinny_pipe_kernel<kRows>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  });
  if (err != cudaSuccess) return err;
  simt_skinny_pipe_kernel<kRows><<<grid, kThreads, smem, stream>>>(p, stages);
  return cudaGetLastError();
}

template <bool kVec, int kRows>
cudaError_t launch_skinny_t(int grid, size_t dyn, cudaStream_t stream, const SimtArgs& p) {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    err = cudaFuncSetAttribute(simt_skinny_kernel<kVec, kRows>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  });
  if (err != cudaSuccess) return err;
  simt_skinny_kernel<kVec, kRows><<<grid, kThreads, dyn, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_skinny(bool vec, int rows, int grid, size_t dyn, cudaStream_t s,
                          const SimtArgs& p) {
  if (vec) {
    if (rows == 4) return launch_skinny_t<true, 4>(grid, dyn, s, p);
    if (rows == 8) return launch_skinny_t<true, 8>(grid, dyn, s, p);
    return launch_skinny_t<true, 16>(grid, dyn, s, p);
  }
  if (rows == 4) return launch_skinny_t<false, 4>(grid, dyn, s, p);
  if (rows == 8) return launch_skinny_t<false, 8>(grid, dyn, s, p);
  return launch_skinny_t<false, 16>(grid, dyn, s, p);
}

}  // namespace

cudaError_t simt_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                      int num_ctas, bool exclusive_sm, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return cudaErrorInvalidValue;
  if (K <= 0) {
    if (accumulate) return cudaSuccess;
    return cudaMemset2DAsync(C, static_cast<size_t>(ldc) * 4, 0, static_cast<size_t>(N) * 4,
                             static_cast<size_t>(M), stream);
  }
  SimtArgs p;
  p.M = static_cast<int>(M);
  p.N = static_cast<int>(N);
  p.K = static_cast<int>(K);
  p.A = A;
  p.lda = lda;
  p.B = B;
  p.ldb = ldb;
  p.C = C;
  p.ldc = ldc;
  p.accumulate = accumulate ? 1 : 0;
  p.tiles_m = static_cast<int>((M + kBM - 1) / kBM);
  p.tiles_n = static_cast<int>((N + kBN - 1) / kBN);
  const bool vec = lda % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                     reinterpret_cast<uintptr_t>(C)) & 15) == 0;
  // An "exclusive" CTA requests enough shared memory that nothing else (in
  // particular a tensor-core CTA) can share its SM: the unit owns whole SMs.
  const size_t smem = exclusive_sm ? 120 * 1024 : kSmemFloats * sizeof(float);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    for (const void* f : {reinterpret_cast<const void*>(simt_gemm_kernel<true, 2>),
                          reinterpret_cast<const void*>(simt_gemm_kernel<false, 2>),
                          reinterpret_cast<const void*>(simt_gemm_kernel<true, 4>),
                          reinterpret_cast<const void*>(simt_gemm_kernel<false, 4>),
                          reinterpret_cast<const void*>(simt_gemm_kernel<true, 2, 2>),
                          reinterpret_cast<const void*>(simt_gemm_kernel<false, 2, 2>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true, 32>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false, 32>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true, 16, 128>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false, 16, 128>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true, 16, 256, 2>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true, 32, 256, 4, true>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false, 32, 256, 4, true>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<true, 16, 256, 4, true>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false, 16, 256, 4, true>),
                          reinterpret_cast<const void*>(simt_gemm2_kernel<false, 16, 256, 2>),
                          reinterpret_cast<const void*>(simt_gemm3_kernel<true>),
                          reinterpret_cast<const void*>(simt_gemm3_kernel<false>)})
      if (attr_err == cudaSuccess)
        attr_err = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
  });
  if (attr_err != cudaSuccess) return attr_err;
  int grid = num_ctas > 0 ? num_ctas : device_sm_count();
  if (M < kBM) {
    // Row-group height: smallest of 4/8/16 covering M (no padded FMAs for
    // the common 4- or 8-row shares).
    const int rg = M <= 4 ? 4 : (M <= 8 ? 8 : 16);
    const int tiles = static_cast<int>(((M + rg - 1) / rg) * ((N + kSkCols - 1) / kSkCols));
    if (grid > tiles) grid = tiles;
    if (vec && exclusive_sm) {  // the unit owns its SMs: spend their smem on bytes in flight
      if (rg == 4) return launch_pipe_t<4>(grid, stream, p);
      if (rg == 8) return launch_pipe_t<8>(grid, stream, p);
      return launch_pipe_t<16>(grid, stream, p);
    }
    // Exclusive units pad dynamic shared memory so no tensor CTA shares the SM.
    const size_t dyn = exclusive_sm ? 100 * 1024 : 0;
    return launch_skinny(vec, rg, grid, dyn, stream, p);
  }
  // Default: the FFMA2 kernel (128 x 256 tiles, grouped raster). Earlier
  // FFMA kernels for A/B comparisons: POAS_SIMT_TILE=256: 128 x 256 (8 x 16
  // per thread, one CTA per SM); =128: 128 x 128 (8 x 8); =128x2: 128 x 128
  // with registers capped so two CTAs share an SM. Exclusive units pad
  // shared memory so that no tensor-core CTA (210 KB) fits beside them.
  const char* tw = std::getenv("POAS_SIMT_TILE");
  const std::string tile = tw ? tw : "ffma2";
  if (tile == "ffma2x512") {
    const int tiles3 = p.tiles_m * static_cast<int>((N + 255) / 256);
    if (grid > tiles3) grid = tiles3;
    const size_t smem3 = exclusive_sm ? 120 * 1024 : (2 * kBK * (kBM + kPad) + 2 * kBK * 256) * sizeof(float);
    if (vec)
      simt_gemm3_kernel<true><<<grid, kThreads3, smem3, stream>>>(p);
    else
      simt_gemm3_kernel<false><<<grid, kThreads3, smem3, stream>>>(p);
    return cudaGetLastError();
  }
  if (tile == "ffma2x2" || tile == "ffma2w16") {  // 128 x 128 tiles, two CTAs per SM
    const int tiles2 = p.tiles_m * static_cast<int>((N + 127) / 128);
    grid *= 2;
    if (grid > tiles2) grid = tiles2;
    const size_t need = (2 * kBK * (kBM + kPad) + 2 * kBK * 128) * sizeof(float);
    // exclusive: two of these fit an SM (2 x 100 KB), a tensor CTA does not
    const size_t smem2 = exclusive_sm ? std::max<size_t>(100 * 1024, need) : need;
    if (tile == "ffma2w16") {
      if (vec)
        simt_gemm2_kernel<true, 16, 256, 2><<<grid, 256, smem2, stream>>>(p);
      else
        simt_gemm2_kernel<false, 16, 256, 2><<<grid, 256, smem2, stream>>>(p);
    } else if (vec) {
      simt_gemm2_kernel<true, 16, 128><<<grid, 128, smem2, stream>>>(p);
    } else {
      simt_gemm2_kernel<false, 16, 128><<<grid, 128, smem2, stream>>>(p);
    }
    return cudaGetLastError();
  }
  // The FFMA2 128 x 256 kernel: default K depth 32 with B-pair-major FFMA2
  // order (8192^3: 58.4 TFLOP/s, 0.91x cuBLAS SGEMM; A-scalar-major order
  // 56.3, K depth 16 56.0 -- profiles/r02_simt). "ffma2k16" / "ffma2k16j" /
  // "ffma2k32": the other (depth, order) pairs.
  if (tile == "ffma2" || tile == "ffma2k32j" || tile == "ffma2k32" || tile == "ffma2k16" ||
      tile == "ffma2k16j") {
    const int tiles2 = p.tiles_m * static_cast<int>((N + 255) / 256);
    if (grid > tiles2) grid = tiles2;
    const int bk = (tile == "ffma2k16" || tile == "ffma2k16j") ? 16 : 32;
    const bool jouter = tile == "ffma2" || tile == "ffma2k32j" || tile == "ffma2k16j";
    const size_t need = (2 * bk * (kBM + kPad) + 2 * bk * 256) * sizeof(float);
    const size_t smem2 = exclusive_sm ? std::max<size_t>(120 * 1024, need) : need;
#define POAS_SIMT2(BK, J)                                                           \
  (vec ? (simt_gemm2_kernel<true, BK, 256, 4, J><<<grid, kThreads, smem2, stream>>>(p), 0) \
       : (simt_gemm2_kernel<false, BK, 256, 4, J><<<grid, kThreads, smem2, stream>>>(p), 0))
    if (bk == 32)
      jouter ? POAS_SIMT2(32, true) : POAS_SIMT2(32, false);
    else
      jouter ? POAS_SIMT2(16, true) : POAS_SIMT2(16, false);
#undef POAS_SIMT2
    return cudaGetLastError();
  }
  const bool wide = tile != "128" && tile != "128x2";
  const bool two = tile == "128x2";
  const int tn = wide ? 256 : 128;
  const int per_sm = two ? 2 : 1;
  const int tiles = p.tiles_m * static_cast<int>((N + tn - 1) / tn);
  grid *= per_sm;
  if (grid > tiles) grid = tiles;
  const size_t smem_w = exclusive_sm ? (two ? 100 * 1024 : 120 * 1024)
                                     : (2 * kBK * (kBM + kPad) + 2 * kBK * tn) * sizeof(float);
  if (wide) {
    if (vec)
      simt_gemm_kernel<true, 4><<<grid, kThreads, smem_w, stream>>>(p);
    else
      simt_gemm_kernel<false, 4><<<grid, kThreads, smem_w, stream>>>(p);
  } else if (two) {
    if (vec)
      simt_gemm_kernel<true, 2, 2><<<grid, kThreads, smem_w, stream>>>(p);
    else
      simt_gemm_kernel<false, 2, 2><<<grid, kThreads, smem_w, stream>>>(p);
  } else if (vec) {
    simt_gemm_kernel<true, 2><<<grid, kThreads, smem_w, stream>>>(p);
  } else {
    simt_gemm_kernel<false, 2><<<grid, kThreads, smem_w, stream>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace poas_b200
