// Tensor-core unit of one B200: persistent tcgen05 GEMM.
//
//   C[M x N] (=|+=) A[M x K] . B[K x N]     A, B row-major bf16/fp16, C fp32
//
// Replaces the XPU-kind synthetic law of the reference (SyntheticBackend::
// time_gemm, /root/reference/proj/src/simulator.cpp:30-34) with real work.
//
// Kernels (all persistent over output tiles, one CTA per SM):
//   tc_gemm_2cta_kernel<W, PAIRS>  CTA pairs (cta_group::2), 256 x W tiles:
//     W = 512 (default from K >= 6144; 4 x 48 KB stages, the accumulator
//     fills TMEM and its halves are released separately, 8 epilogue warps),
//     W = 256 (6 x 32 KB stages, double-buffered accumulator, 4 epilogue
//     warps); PAIRS = 2 puts two pairs in a cluster sharing B by multicast.
//     Opt-in (POAS_TC_SPLIT=1): a last wave of at most half a wave of tiles
//     runs as two K-halves (store, then add-reduce after a ready flag).
//   tc_gemm_kernel<BN, STAGES>     one SM, 128 x BN tiles (small GEMMs).
// Roles: warp 0 lane 0 TMA producer (A K-major, B N-major, 128B-swizzled
// ring), warp 1 lane 0 MMA issuer (tcgen05.mma .kind::f16, fp32 accumulator
// in TMEM), the remaining warps the epilogue (tcgen05.ld -> registers ->
// swizzled smem box -> TMA store / reduce-add). M/N/K tails come from TMA
// out-of-bounds zero fill and clipped stores. See DESIGN.md section 2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "sm100_ptx.cuh"

namespace poas_b200 {
namespace {

using namespace ptx;

constexpr int kBM = 128;
constexpr int kBN = 256;  // pair tile width; the single-SM kernel's is a template argument
constexpr int kBK = 64;  // one 128-byte swizzle row of 16-bit elements
constexpr int kUmmaK = 16;
constexpr int kABytes = kBM * kBK * 2;       // 16 KiB
constexpr int kBChunkBytes = 64 * kBK * 2;   // one 64-column N chunk: 8 KiB
constexpr int kThreads = 192;
constexpr int kTmemCols = 512;  // pair kernel: two 256-column fp32 accumulators
constexpr int kGroupM = 16;     // tile raster: 16 M-tiles per group for L2 reuse

struct TcArgs {
  int M, N, K;
  int tiles_m, tiles_n;
  float* C;
  long long ldc;
  int accumulate;
  uint32_t idesc;
  int group;  // raster: M-tiles per group (a wave covers group x (grid/group) tiles)
  int raster_n;        // 1: groups run along N instead of M (experiments)
  int kserp;           // 1: tiles of odd waves (t / workers) sweep K last-to-first (L2 tail reuse)
  uint64_t hint_a, hint_b;  // TMA L2 cache-policy hints per operand
  uint64_t hint_c;          // TMA-store epilogue: L2 policy of the C writes
  int* tile_counter;     // {next, done}, zero at launch: dynamic tile scheduler (or null)
  int wave_sync;         // 1: static order + per-wave barrier on tile_counter[0]
  int tma_store;         // pair kernel: 1 = epilogue through smem + TMA store (map_c)
  unsigned long long* trace;  // dev: per-CTA %globaltimer stamps (POAS_TC_TRACE), or null
  int epi_skip;               // dev (POAS_TC_EPI_SKIP): TMA-store epilogue stages boxes, stores nothing
  // Panel-major B (pair kernel): `panels` column panels of tiles_n_panel
  // N-tiles each, B loaded through a 3-D map {column, k, panel}; tiles are
  // ordered panel by panel. With panel_flags, a producer starts on panel p
  // once panel_flags[p] >= panel_epoch (set in panel order by whoever
  // delivers B, e.g. after each panel's broadcast).
  int panels;
  int tiles_n_panel;
  int panel_order;  // 1: tiles panel by panel (else the grouped raster over all panels)
  const int* panel_flags;
  int panel_epoch;
  // Streamed operands (pair kernel; see tc_gemm_stream): tiles ordered by a
  // block table {mb0 | tiles_m << 16, nb0 | tiles_n << 16, first tile,
  // item_a | item_b << 16}; a producer starts a tile once both link items
  // of its block are flagged (item_flags[i] >= stream_epoch); the epilogue
  // counts finished tiles per block (8 warps per pair tile) and raises the
  // block's flag once its C is in global memory.
  const int4* sblocks;
  int nsblocks;
  const int* item_flags;
  int* block_count;
  int* block_flags;
  int stream_epoch;
  // Last-wave K split (pair kernel, dynamic scheduler): tiles [split_base,
  // tiles) run as two K-halves, work units split_base + 2j + part; part 0
  // sweeps k-blocks [0, split_kb) and stores, part 1 sweeps the rest and
  // add-reduces once part 0's boxes are in global memory. split_cnt: per
  // split tile {part-0 warps done, ready flag, part-1 warps released, -},
  // all zero again when the launch ends (so graph replays need no reset).
  int split_base;
  int split_kb;
  int* split_cnt;
};

// Work unit u -> tile, k-block range [kb0, kb1) and split part (-1: whole tile).
__device__ __forceinline__ int unit_tile(const TcArgs& a, int u, int k_blocks, int& kb0, int& kb1,
                                         int& part) {
  if (!a.split_cnt || u < a.split_base) {
    kb0 = 0;
    kb1 = k_blocks;
    part = -1;
    return u;
  }
  const int v = u - a.split_base;
  part = v & 1;
  kb0 = part ? a.split_kb : 0;
  kb1 = part ? k_blocks : a.split_kb;
  return a.split_base + (v >> 1);
}

// Spin (acquire, with backoff) until *flag >= epoch; traps after 10 s so a
// missing signal fails the launch instead of hanging the GPU.
__device__ __forceinline__ void wait_panel_flag(const int* flag, int epoch) {
  unsigned long long start, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (true) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= epoch) break;
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > 10000000000ull) __trap();
  }
  fence_proxy_async_global();  // B's bytes (another kernel's writes) before our TMA reads
}

// Dev instrumentation (POAS_TC_TRACE=1): per CTA, 16 %globaltimer slots.
//   0 entry  1 prologue done  2 first TMA issued  3 first stage full (MMA)
//   4 last MMA commit  5 epilogue sees its first accumulator  6 last box
//   issued  7 exit  8 producer: first tile published  9 producer: first
//   empty-slot wait passed
// Write-only (no global read on the traced thread's path); callers stamp
// each event once.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Slots 10..13 accumulate durations (ns) over the CTA's tiles: 10 MMA
// blocked on the accumulator (half 0), 11 MMA blocked on half 1 (wide
// tiles), 12 epilogue from accumulator-full to the release of its first
// half, 13 ... to the release of its last half.
__device__ __forceinline__ void trace_add(const TcArgs& a, int idx, unsigned long long d) {
  if (a.trace) a.trace[blockIdx.x * 16 + idx] += d;
}
__device__ __forceinline__ void trace_stamp(const TcArgs& a, int idx) {
  if (!a.trace) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  a.trace[blockIdx.x * 16 + idx] = t;
}

// ---------------------------------------------------------- tile scheduler
// The producer thread (of the CTA, or of the pair's leader) owns the tile
// sequence and hands each tile id to the other roles through a small smem
// ring (tile_full / tile_empty mbarriers; -1 ends the sequence).
//
// Dynamic mode: a worker's first tile is its own index (no claim on the
// critical path of the first loads); later tiles are claimed with one global
// atomicAdd per tile (counter + number of workers), so the
// tiles in flight are always a contiguous window of the raster order however
// far individual CTAs drift (launch stagger, far-die L2 latency, co-running
// kernels taking SMs). With a static round-robin a lagging CTA works on a
// tile of an older wave whose A/B panels have already left L2. The counter
// resets itself: the last worker to finish zeroes it for the next launch.
constexpr int kTileSlots = 4;

__device__ __forceinline__ int claim_tile(const TcArgs& a, int& next_static, int step) {
  if (a.tile_counter && !a.wave_sync) return atomicAdd(a.tile_counter, 1) + step;
  const int t = next_static;
  next_static += step;
  return t;
}

__device__ __forceinline__ void release_counter(const TcArgs& a, int workers) {
  if (!a.tile_counter) return;
  __threadfence();  // this worker's claims precede its "done"
  if (atomicAdd(a.tile_counter + 1, 1) == workers - 1) {
    atomicExch(a.tile_counter, 0);
    atomicExch(a.tile_counter + 1, 0);
  }
}

// Wave mode (large problems, see tc_gemm): static round-robin order, and
// before its i-th tile (i >= 1) a worker waits until every worker that has an
// i-th tile has reached it, so the tiles of a wave sweep K in step and share
// A/B panels through L2. `target` accumulates the arrivals expected by wave
// i. The wait gives up after 200 us (a worker that is not resident -- SMs
// held by another kernel -- must not stall the grid); the caller then stops
// synchronising, and the others time out once and follow: plain static order.
__device__ __forceinline__ bool wave_barrier(const TcArgs& a, int i, int workers, int total,
                                             int& target) {
  target += min(workers, total - i * workers);
  atomicAdd(a.tile_counter, 1);
  unsigned long long start, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(start));
  while (true) {
    int seen;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(a.tile_counter) : "memory");
    if (seen >= target) return true;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now - start > 200000ull) return false;  // 200 us: a worker is not resident
  }
}

// Grouped raster: consecutive tile ids walk `group` M-tiles down a column of
// N-tiles, so one wave of the persistent grid shares A row panels and B
// column panels through L2.
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group, int& mb,
                                            int& nb, int raster_n = 0) {
  if (raster_n) {  // transpose the raster: groups of N-tiles walk down M
    const int per_group_n = group * tiles_m;
    const int gn_idx = t / per_group_n;
    const int first_n = gn_idx * group;
    const int gn = min(tiles_n - first_n, group);
    const int rn = t - gn_idx * per_group_n;
    nb = first_n + rn % gn;
    mb = rn / gn;
    return;
  }
  const int per_group = group * tiles_n;
  const int g = t / per_group;
  const int first_m = g * group;
  const int gm = min(tiles_m - first_m, group);
  const int r = t - g * per_group;
  mb = first_m + r % gm;
  nb = r / gm;
}

// Tile t of a streamed problem: its block (binary search over first tiles)
// and the grouped raster inside the block.
__device__ __forceinline__ int4 tile_coords_stream(const TcArgs& a, int t, int& mb, int& nb,
                                                   int& blk) {
  int lo = 0, hi = a.nsblocks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.sblocks[mid].z <= t) lo = mid; else hi = mid - 1;
  }
  const int4 d = a.sblocks[lo];
  blk = lo;
  int lm, ln;
  tile_coords(t - d.z, d.x >> 16, d.y >> 16, a.group, lm, ln);
  mb = (d.x & 0xffff) + lm;
  nb = (d.y & 0xffff) + ln;
  return d;
}

// Tile t of a (possibly panel-major) problem: M-tile mb, global N-tile nb,
// its panel p and N-tile inside the panel nbl. Default: the grouped raster
// over the whole grid (the panels are only where B's columns live), so the
// tiles in flight share A row panels through L2; with panel_order the tiles
// go panel by panel (each panel consumed as soon as it lands, at the price
// of re-reading every A row panel once per B panel: C4 per GPU at 8 GPUs,
// 16 panels, 1381 vs 1551 TFLOP/s row-major, profiles/r02_panels).
__device__ __forceinline__ void tile_coords_panel(const TcArgs& a, int t, int& mb, int& nb, int& p,
                                                  int& nbl) {
  if (a.panels > 1 && a.panel_order) {
    const int per = a.tiles_m * a.tiles_n_panel;
    p = t / per;
    tile_coords(t - p * per, a.tiles_m, a.tiles_n_panel, a.group, mb, nbl, a.raster_n);
    nb = p * a.tiles_n_panel + nbl;
    return;
  }
  if (a.panels > 1) {
    tile_coords(t, a.tiles_m, a.tiles_n, a.group, mb, nb, a.raster_n);
    p = nb / a.tiles_n_panel;
    nbl = nb - p * a.tiles_n_panel;
    return;
  }
  p = 0;
  tile_coords(t, a.tiles_m, a.tiles_n, a.group, mb, nb, a.raster_n);
  nbl = nb;
}

// Single-SM kernel, templated on its tile width: 128 x 256 (4 stages; the
// POAS_TC_KERNEL=1cta variant) and 128 x 128 (6 stages; small GEMMs whose
// 256 x 256 pair tiles cannot fill the SMs).
template <int BN, int STAGES>
struct Tile1 {
  static constexpr int kB = BN * kBK * 2;       // B bytes per stage
  static constexpr int kStage = kABytes + kB;
  static constexpr int kTmem = 2 * BN;          // two accumulators
  static constexpr size_t kSmem = 1024 + STAGES * kStage + 256;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, const TcArgs args) {
  using T1 = Tile1<BN, STAGES>;
  constexpr int kBN = BN;
  constexpr int kStages = STAGES;
  constexpr int kBBytes = T1::kB;
  constexpr int kStageBytes = T1::kStage;
  constexpr uint32_t kTmemCols = T1::kTmem;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* s_a = smem;
  uint8_t* s_b = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* tile_full = acc_empty + 2;
  uint64_t* tile_empty = tile_full + kTileSlots;
  int* tile_ring = reinterpret_cast<int*>(tile_empty + kTileSlots);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kTileSlots);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    for (int s = 0; s < kTileSlots; ++s) {
      mbar_init(&tile_full[s], 1);
      mbar_init(&tile_empty[s], 5);  // MMA thread + 4 epilogue warps
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic launch: the prologue above overlapped the previous kernel
  // of the stream; global memory only from here on
  griddep_launch();
  griddep_wait();

  const int total = args.tiles_m * args.tiles_n;
  const int k_blocks = (args.K + kBK - 1) / kBK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int next_static = blockIdx.x;
      int slot = 0;
      uint32_t tphase = 0;
      int wave = 0, wave_target = 0;
      bool wave_on = args.wave_sync != 0;
      // first tile = blockIdx.x without a claim; claims continue after the grid
      int t = next_static;
      next_static += gridDim.x;
      while (true) {
        const int tt = t < total ? t : -1;
        mbar_wait(&tile_empty[slot], tphase ^ 1);
        tile_ring[slot] = tt;
        mbar_arrive(&tile_full[slot]);
        if (++slot == kTileSlots) {
          slot = 0;
          tphase ^= 1;
        }
        if (tt < 0) break;
        if (wave_on && wave > 0) wave_on = wave_barrier(args, wave, gridDim.x, total, wave_target);
        ++wave;
        const int t_next = claim_tile(args, next_static, gridDim.x);  // latency hidden by the loads
        int mb, nb;
        tile_coords(t, args.tiles_m, args.tiles_n, args.group, mb, nb, args.raster_n);
        const bool rev = args.kserp && ((t / static_cast<int>(gridDim.x)) & 1);
        for (int kb = 0; kb < k_blocks; ++kb) {
          const int kc = (rev ? k_blocks - 1 - kb : kb) * kBK;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d(s_a + stage * kABytes, &map_a, &full[stage], kc, mb * kBM, args.hint_a);
#pragma unroll
          for (int j = 0; j < kBN / 64; ++j)
            tma_load_2d(s_b + stage * kBBytes + j * kBChunkBytes, &map_b, &full[stage],
                        nb * kBN + j * 64, kc, args.hint_b);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        t = t_next;
      }
      release_counter(args, gridDim.x);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int slot = 0;
      uint32_t tphase = 0;
      while (true) {
        mbar_wait(&tile_full[slot], tphase);
        const int t = tile_ring[slot];
        mbar_arrive(&tile_empty[slot]);
        if (++slot == kTileSlots) {
          slot = 0;
          tphase ^= 1;
        }
        if (t < 0) break;
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * kBN);
        for (int kb = 0; kb < k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = smem_addr(s_a + stage * kABytes);
          const uint32_t b0 = smem_addr(s_b + stage * kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / kUmmaK; ++k) {
            // A (K-major): advance 16 elements = 32 bytes inside the swizzle row.
            const uint64_t ad = sdesc_sw128(a0 + k * kUmmaK * 2, 16, 1024);
            // B (N-major): 16 K-rows = two 8-row (1024 B) swizzle atoms;
            // 64-column N chunks sit kBChunkBytes apart.
            const uint64_t bd = sdesc_sw128(b0 + k * 2 * 1024, kBChunkBytes, 1024);
            umma_f16(d_tmem, ad, bd, args.idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // Epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32).
    const int quad = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec = (args.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    int slot = 0;
    uint32_t tphase = 0;
    while (true) {
      mbar_wait(&tile_full[slot], tphase);
      const int t = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[slot]);
      if (++slot == kTileSlots) {
        slot = 0;
        tphase ^= 1;
      }
      if (t < 0) break;
      int mb, nb;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group, mb, nb, args.raster_n);
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      const int row = mb * kBM + quad * 32 + lane;
      float* crow = args.C + static_cast<long long>(row) * args.ldc;
#pragma unroll 1
      for (int c = 0; c < kBN / 32; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                               static_cast<uint32_t>(acc * kBN + c * 32),
                           v);
        tmem_wait_ld();
        if (row < args.M) {
          const int col0 = nb * kBN + c * 32;
          if (vec && col0 + 32 <= args.N) {
            float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 o = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                     __uint_as_float(v[4 * j + 2]),
                                     __uint_as_float(v[4 * j + 3]));
              if (args.accumulate) {
                const float4 p = dst[j];
                o.x += p.x;
                o.y += p.y;
                o.z += p.z;
                o.w += p.w;
              }
              dst[j] = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < args.N) {
                float o = __uint_as_float(v[j]);
                if (args.accumulate) o += crow[col];
                crow[col] = o;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ------------------------------------------------- 2-SM (cta_group::2) kernel
// A CTA pair (cluster of 2 on one TPC) owns a 256 x W output tile. Each CTA
// stages 128 rows of A and W/2 columns of B per 64-deep K block; the
// leader's single thread issues tcgen05.mma.cta_group::2 (M=256, N=256,
// K=16) once per 256-column half of the tile, which reads both CTAs' shared
// memory and writes both CTAs' TMEM (each holds its 128 rows x W fp32
// columns).
//
//   W = 256: 6 stages of 32 KB per CTA; two 256-column accumulators, double
//            buffered (the epilogue of tile i overlaps the MMAs of tile i+1).
//            Versus two independent 128 x 256 CTAs: 1/3 fewer operand bytes
//            from L2 into shared memory per MAC.
//   W = 512: 4 stages of 48 KB; the accumulator fills all 512 TMEM columns.
//            Another 1/4 fewer operand bytes from L2 per MAC than W = 256
//            (16384^3: 68.7 -> 51.5 GB through the L2 -> SM crossbar), which
//            under the power cap is energy and therefore clock. The epilogue
//            releases each 256-column half as soon as it is in registers; the
//            next tile's MMAs start on half 0 and catch half 1 up (its
//            k-blocks stay staged, at most a ring's worth) once it is free.
constexpr int k2ABytes = 128 * kBK * 2;  // this CTA's 128 rows of A: 16 KB
constexpr int kGroupM2 = 8;  // default raster group: 8 x 256 rows
// Epilogue staging (TMA-store path), per epilogue warp: W = 256 two 32-row x
// 16-column fp32 boxes with 64-byte swizzled rows (2 x 2 KB); W = 512 one
// 32-row x 32-column box with 128-byte swizzled rows (4 KB).

template <int W, int EPI = 0>
struct Pair {
  static_assert(W == 256 || W == 512, "pair tile width");
  static constexpr int kHalves = W / 256;
  static constexpr int kStages = W == 256 ? 6 : 4;
  static constexpr int kBBytes = (W / 2) * kBK * 2;  // this CTA's W/2 columns of B
  static constexpr int kStageBytes = k2ABytes + kBBytes;
  // epilogue warps: 8 (two per TMEM lane quarter, alternate 32-column
  // chunks: twice the warps read TMEM and issue stores) where the drain is
  // exposed -- every 256 x 512 tile, and 256 x 256 tiles when the GEMM is one
  // wave of them (2048^3: drain 4.4 -> 3.45 us, +2%); 4 (one per quarter)
  // for 256 x 256 tiles whose drain hides behind the other accumulator
  // (there 8 cost 0.6-1%: 4096^3 1318 -> 1305 TFLOP/s, profiles/r02_epi256)
  static constexpr int kEpiWarps = EPI ? EPI : (W == 512 ? 8 : 4);
  static constexpr int kThreads = 64 + 32 * kEpiWarps;
  static constexpr int kStagingBytes = kEpiWarps * 4096;
  static constexpr size_t kSmem = 1024 + kStages * kStageBytes + kStagingBytes + 256;
  static_assert(kSmem <= 232448, "shared memory per CTA");
};

// PAIRS = 2 (W = 512 only): a cluster of two CTA pairs stacked in M (a
// 512 x 512 cluster tile) shares B: each CTA loads the 256-column half of its
// B slice that matches its pair index and multicasts it to the same-rank CTA
// of the other pair, so B crosses the L2 -> SM crossbar once per cluster
// (1/3 fewer operand bytes per MAC than PAIRS = 1). A stage of a CTA is then
// written by both pairs' producers: it is free once BOTH pairs' MMAs have
// consumed it (every MMA commit is multicast to the four CTAs). The cluster
// leader (rank 0) claims the tiles for all four CTAs. The cluster shape is
// compiled in (__cluster_dims__): launching the same kernel with a runtime
// cluster-dimension attribute instead ran the 256 x 256 tiles 10-15% slower
// (profiles/r02_sizes).
template <int W, int PAIRS, int EPI = 0>
__global__ void __cluster_dims__(2 * PAIRS, 1, 1) __launch_bounds__(Pair<W, EPI>::kThreads, 1)
    tc_gemm_2cta_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b,
                        const __grid_constant__ CUtensorMap map_c, const TcArgs args) {
  using P = Pair<W, EPI>;
  constexpr int k2StagingBytes = P::kStagingBytes;
  constexpr int k2Stages = P::kStages;
  constexpr int k2BBytes = P::kBBytes;
  constexpr int k2StageBytes = P::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* s_a = smem;
  uint8_t* s_b = smem + k2Stages * k2ABytes;
  uint8_t* s_c = smem + k2Stages * k2StageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(s_c + k2StagingBytes);
  uint64_t* empty = full + k2Stages;
  uint64_t* acc_full = empty + k2Stages;
  uint64_t* acc_empty = acc_full + 2;  // W = 256: per accumulator; W = 512: per half
  uint64_t* tile_full = acc_empty + 2;
  uint64_t* tile_empty = tile_full + kTileSlots;
  int* tile_ring = reinterpret_cast<int*>(tile_empty + kTileSlots);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kTileSlots);

  static_assert(PAIRS == 1 || PAIRS == 2, "one or two CTA pairs per cluster");
  constexpr int kCtas = 2 * PAIRS;
  constexpr int kRowsT = 256 * PAIRS;  // rows of a (cluster) tile
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t prank = rank & 1;        // rank inside the pair
  const int pair = static_cast<int>(rank >> 1);
  const uint32_t pair_leader = rank & ~1u;
  const bool leader = prank == 0;         // issues the pair's MMAs
  const bool cleader = rank == 0;         // claims and publishes the tiles
  // a stage is free once every pair has consumed it: each MMA commit that
  // releases stages arrives in all CTAs of the cluster
  constexpr uint16_t kFreeMask = static_cast<uint16_t>((1u << kCtas) - 1u);
  if (threadIdx.x == 0) trace_stamp(args, 0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_b);
    if (args.tma_store) tma_prefetch_desc(&map_c);
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], 1);   // pair leader: its expect_tx arrive + both CTAs' bytes
      mbar_init(&empty[s], PAIRS);  // every pair leader's MMA commit, multicast to all CTAs
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * P::kEpiWarps);  // pair leader: the epilogue warps of both CTAs
    }
    for (int s = 0; s < kTileSlots; ++s) {
      mbar_init(&tile_full[s], 1);  // the cluster leader's producer (local or remote arrive)
      // cluster leader: the pairs' MMA threads + the other producers + the
      // epilogue warps of every CTA
      mbar_init(&tile_empty[s], PAIRS + (kCtas - 1) + P::kEpiWarps * kCtas);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic launch: the prologue above overlapped the previous kernel
  // of the stream; global memory only from here on
  griddep_launch();
  griddep_wait();
  if (threadIdx.x == 0) trace_stamp(args, 1);

  // work units: one per tile, two per last-wave split tile (unit_tile)
  const int total = args.tiles_m * args.tiles_n +
                    (args.split_cnt ? args.tiles_m * args.tiles_n - args.split_base : 0);
  const int k_blocks = (args.K + kBK - 1) / kBK;
  const int first = static_cast<int>(cluster_id_x());
  const int step = static_cast<int>(num_clusters_x());

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int next_static = first;
      int slot = 0;
      uint32_t tphase = 0;
      // The leader claims tiles and publishes them to both CTAs' rings; the
      // peer's producer follows its own ring.
      int wave = 0, wave_target = 0;
      bool wave_on = args.wave_sync != 0;
      // The first tile of every worker is its cluster id: every role starts
      // on it without a claim or a ring round trip. The ring carries the
      // later tiles; dynamic claims continue after the first wave.
      int t = first < total ? first : -1;
      next_static = first + step;
      uint64_t panels_seen = 0;  // B panels seen ready (P <= 64; more: checked per tile)
      uint64_t seen_lo = 0, seen_hi = 0;  // streamed link items seen ready
      while (t >= 0) {
        if (cleader && wave_on && wave > 0) wave_on = wave_barrier(args, wave, step, total, wave_target);
        ++wave;
        int t_next = 0;  // claimed once this tile's first loads are out
        int mb, nb, pnl, nbl;
        int kb0 = 0, kb1 = k_blocks, part = -1;
        if (args.sblocks) {
          int blk;
          const int4 d = tile_coords_stream(args, t, mb, nb, blk);
          pnl = 0;
          nbl = nb;
          for (int h = 0; h < 2; ++h) {  // the block's A part, then its B panel
            const int item = h ? (d.w >> 16) : (d.w & 0xffff);
            uint64_t& mask = item < 64 ? seen_lo : seen_hi;
            const uint64_t bit = 1ull << (item & 63);
            if (!(mask & bit)) {
              wait_panel_flag(args.item_flags + item, args.stream_epoch);
              mask |= bit;
            }
          }
        } else {
          tile_coords_panel(args, unit_tile(args, t, k_blocks, kb0, kb1, part), mb, nb, pnl, nbl);
        }
        if (args.panel_flags && (pnl >= 64 || !(panels_seen & (1ull << pnl)))) {
          wait_panel_flag(args.panel_flags + pnl, args.panel_epoch);
          if (pnl < 64) panels_seen |= 1ull << pnl;
        }
        const int row0 = mb * kRowsT + pair * 256 + static_cast<int>(prank) * 128;
        // this CTA's columns of each 256-column half: [h*256 + prank*128, +128)
        const int col0 = nbl * W + static_cast<int>(prank) * 128;  // inside the panel
        // K serpentine: the tiles of a wave that follows one sweeping K
        // forwards start where it ended, on the K-slices still in L2
        const bool rev = args.kserp && part < 0 && ((t / step) & 1);
        for (int kb = 0; kb < kb1 - kb0; ++kb) {
          const int kc = (rev ? k_blocks - 1 - kb : kb0 + kb) * kBK;
          mbar_wait(&empty[stage], phase ^ 1);
          if (wave == 1 && kb == 0) trace_stamp(args, 9);
          if (leader) mbar_arrive_expect_tx(&full[stage], 2 * k2StageBytes);
          tma_load_2d_pair(s_a + stage * k2ABytes, &map_a, &full[stage], kc, row0,
                           args.hint_a);
          uint8_t* sb = s_b + stage * k2BBytes;
#pragma unroll
          for (int j = 0; j < W / 128; ++j) {  // 64-column chunks: half j/2, chunk j%2
            const int cj = col0 + (j >> 1) * 256 + (j & 1) * 64;
            if constexpr (PAIRS == 2) {  // my pair's share of the chunks, to me and my twin
              if (j / (W / 256) != pair) continue;
              const uint16_t mask = static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 2u)));
              if (args.panels > 1)
                tma_load_3d_pair_mc(sb + j * kBChunkBytes, &map_b, &full[stage], cj, kc, pnl, mask,
                                    args.hint_b);
              else
                tma_load_2d_pair_mc(sb + j * kBChunkBytes, &map_b, &full[stage], cj, kc, mask,
                                    args.hint_b);
            } else if (args.panels > 1) {
              tma_load_3d_pair(sb + j * kBChunkBytes, &map_b, &full[stage], cj, kc, pnl,
                               args.hint_b);
            } else {
              tma_load_2d_pair(sb + j * kBChunkBytes, &map_b, &full[stage], cj, kc, args.hint_b);
            }
          }
          if (wave == 1 && kb == 0) trace_stamp(args, 2);
          if (kb == 0 && cleader) t_next = claim_tile(args, next_static, step);  // behind the first loads
          if (++stage == k2Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        // hand the next tile to every CTA's roles (the cluster leader publishes)
        if (cleader) {
          t = t_next < total ? t_next : -1;
          mbar_wait_cluster(&tile_empty[slot], tphase ^ 1);
          tile_ring[slot] = t;
#pragma unroll
          for (uint32_t r = 1; r < kCtas; ++r) st_shared_cluster(&tile_ring[slot], r, t);
          mbar_arrive(&tile_full[slot]);
#pragma unroll
          for (uint32_t r = 1; r < kCtas; ++r) mbar_arrive_cluster(&tile_full[slot], r);
        } else {
          mbar_wait_cluster(&tile_full[slot], tphase);
          t = tile_ring[slot];
          mbar_arrive_cluster(&tile_empty[slot], 0);
        }
        if (wave == 1) trace_stamp(args, 8);
        if (++slot == kTileSlots) {
          slot = 0;
          tphase ^= 1;
        }
      }
      if (cleader) release_counter(args, step);
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int slot = 0;
      uint32_t tphase = 0;
      bool traced = false;
      // one 256-column half of the tile for the k-block staged in `st`
      auto issue = [&](uint32_t d_tmem, int st, int kb, int h) {
        const uint32_t a0 = smem_addr(s_a + st * k2ABytes);
        const uint32_t b0 = smem_addr(s_b + st * k2BBytes) + static_cast<uint32_t>(h * 2 * kBChunkBytes);
#pragma unroll
        for (int k = 0; k < kBK / kUmmaK; ++k) {
          const uint64_t ad = sdesc_sw128(a0 + k * kUmmaK * 2, 16, 1024);
          const uint64_t bd = sdesc_sw128(b0 + k * 2 * 1024, kBChunkBytes, 1024);
          umma_f16_pair(d_tmem + static_cast<uint32_t>(h * 256), ad, bd, args.idesc,
                        (kb | k) != 0 ? 1u : 0u);
        }
      };
      for (int t = first < total ? first : -1; t >= 0;) {
        const unsigned long long tw0 = args.trace ? gtimer() : 0;
        mbar_wait(&acc_empty[acc], acc_phase ^ 1);  // W = 512: half 0
        tc_fence_after();
        if (args.trace) trace_add(args, 10, gtimer() - tw0);
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(W == 256 ? acc * 256 : 0);
        // W = 512: half 1 of the previous tile may still be draining; its
        // MMAs trail half 0's by the k-blocks held in `npend` stages (each
        // stage is released once both halves have consumed it)
        bool h1 = W == 256;
        int npend = 0, pend_kb = 0, pend_stage = 0;
        int kb0, kb1, part;
        unit_tile(args, t, k_blocks, kb0, kb1, part);
        for (int kb = 0; kb < kb1 - kb0; ++kb) {  // local k-block: the first one overwrites D
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (!traced) {
            trace_stamp(args, 3);
            traced = true;
          }
          issue(d_tmem, stage, kb, 0);
          if constexpr (W == 256) {
            umma_commit_pair(&empty[stage], kFreeMask);
          } else {
            if (npend++ == 0) {
              pend_kb = kb;
              pend_stage = stage;
            }
            if (!h1 && (npend == k2Stages || mbar_test_wait(&acc_empty[1], acc_phase ^ 1))) {
              const unsigned long long tw1 = args.trace ? gtimer() : 0;
              mbar_wait(&acc_empty[1], acc_phase ^ 1);
              tc_fence_after();
              if (args.trace) trace_add(args, 11, gtimer() - tw1);
              h1 = true;
            }
            if (h1) {
              for (int i = 0, st = pend_stage; i < npend; ++i) {
                issue(d_tmem, st, pend_kb + i, 1);
                umma_commit_pair(&empty[st], kFreeMask);
                if (++st == k2Stages) st = 0;
              }
              npend = 0;
            }
          }
          if (++stage == k2Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (W == 512) {
          if (npend) {  // a tile shorter than the drain of half 1
            mbar_wait(&acc_empty[1], acc_phase ^ 1);
            tc_fence_after();
            for (int i = 0, st = pend_stage; i < npend; ++i) {
              issue(d_tmem, st, pend_kb + i, 1);
              umma_commit_pair(&empty[st], kFreeMask);
              if (++st == k2Stages) st = 0;
            }
          }
        }
        umma_commit_pair(&acc_full[acc], static_cast<uint16_t>(0x3u << pair_leader));
        if (args.trace) {  // the last commit of this worker overwrites
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          args.trace[blockIdx.x * 16 + 4] = tt;
        }
        if (W == 512 || (acc ^= 1) == 0) acc_phase ^= 1;
        mbar_wait_cluster(&tile_full[slot], tphase);  // the next tile
        t = tile_ring[slot];
        mbar_arrive_cluster(&tile_empty[slot], 0);  // the cluster leader's barrier
        if (++slot == kTileSlots) {
          slot = 0;
          tphase ^= 1;
        }
      }
    }
  } else {
    const int quad = warp & 3;          // the TMEM lane quarter this warp may access
    const int sub = (warp - 2) >> 2;    // W = 512: which of the quarter's two warps
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool vec = (args.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    int slot = 0;
    uint32_t tphase = 0;
    bool epi_traced = false;
    auto next_tile = [&]() {
      mbar_wait_cluster(&tile_full[slot], tphase);
      const int tn = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&tile_empty[slot], 0);  // the leader's barrier
      if (++slot == kTileSlots) {
        slot = 0;
        tphase ^= 1;
      }
      return tn;
    };
    for (int t = first < total ? first : -1; t >= 0; t = next_tile()) {
      int mb, nb;
      int pnl_unused, nbl_unused, blk = 0, blk_tiles = 0;
      int kb0, kb1, part = -1;
      if (args.sblocks) {
        const int4 d = tile_coords_stream(args, t, mb, nb, blk);
        blk_tiles = (d.x >> 16) * (d.y >> 16);
      } else {
        tile_coords_panel(args, unit_tile(args, t, k_blocks, kb0, kb1, part), mb, nb, pnl_unused,
                          nbl_unused);
      }
      mbar_wait(&acc_full[acc], acc_phase);
      tc_fence_after();
      if (part == 1) {
        // the tile's other K-half stores first; this half add-reduces onto it
        // (a fixed order: C is the same for every run of this configuration)
        int* sc = args.split_cnt + 4 * (unit_tile(args, t, k_blocks, kb0, kb1, part) - args.split_base);
        if (lane == 0) {
          wait_panel_flag(sc + 1, 1);
          // the last part-1 warp past the flag clears it for the next launch
          if (atomicAdd(sc + 2, 8 / P::kEpiWarps) + 8 / P::kEpiWarps == 16) {
            atomicExch(sc + 2, 0);
            atomicExch(sc + 1, 0);
          }
        }
        __syncwarp();
      }
      const unsigned long long te0 = args.trace ? gtimer() : 0;
      if (quad == 0 && sub == 0 && lane == 0 && !epi_traced) {
        trace_stamp(args, 5);
        epi_traced = true;
      }
      const int row_base = mb * kRowsT + pair * 256 + static_cast<int>(prank) * 128 + quad * 32;
      if (args.tma_store) {
        if constexpr (W == 256) {
          // 256 x 256 tiles (the accumulator is double buffered, so the
          // drain overlaps the next tile's MMAs and only the completion of a
          // short GEMM's last tile is exposed): TMEM -> registers -> a
          // 32-row x 16-column staging box of this warp (64-byte swizzled
          // rows) -> one TMA store (or f32 add-reduction) per box. Two boxes
          // per warp, so a box's store drains while the next one fills; the
          // TMEM load of the next 32 columns is in flight while the current
          // ones are written. (With one fence per 2 KB this finishes a
          // single-tile GEMM sooner than the wide tiles' 8 KB steps, which
          // wait for the previous step's stores: 2048^3 922 vs 817 TFLOP/s,
          // profiles/r02_sizes.)
          constexpr int S = P::kEpiWarps / 4;  // warps per TMEM lane quarter
          constexpr int kChunks = 8 / S;         // this warp's 32-column chunks
          uint8_t* boxes = s_c + (warp - 2) * 4096;
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                                 static_cast<uint32_t>(acc * 256);
          auto put_box = [&](const uint32_t* w, int c) {  // 16 columns, box (c & 1)
            uint8_t* box = boxes + (c & 1) * 2048;
            if (lane == 0) bulk_wait_read<1>();  // the store two boxes back has left smem
            __syncwarp();
            uint8_t* my_row = box + lane * 64;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(my_row + ((j ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !args.epi_skip) {
              const int col0 = nb * W + c * 16;
              if (args.accumulate || part == 1)
                tma_reduce_add_2d(&map_c, box, col0, row_base);
              else if (args.hint_c != kEvictNormal)
                tma_store_2d_hint(&map_c, box, col0, row_base, args.hint_c);
              else
                tma_store_2d(&map_c, box, col0, row_base);
              bulk_commit();
            }
          };
          uint32_t va[32], vb[32];
          tmem_ld_32x32b_x32(taddr + sub * 32, va);
          tmem_wait_ld();
#pragma unroll 1
          for (int i = 0; i < kChunks; i += 2) {  // chunks sub + S * i
            const int c = sub + S * i;
            tmem_ld_32x32b_x32(taddr + (c + S) * 32, vb);
            put_box(va, 2 * c);
            put_box(va + 16, 2 * c + 1);
            tmem_wait_ld();
            if (i + 2 < kChunks) {
              tmem_ld_32x32b_x32(taddr + (c + 2 * S) * 32, va);
            } else {  // this warp's columns are in registers: free the accumulator
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&acc_empty[acc], pair_leader);
              if (args.trace && quad == 0 && sub == 0 && lane == 0)
                trace_add(args, 12, gtimer() - te0);
            }
            put_box(vb, 2 * (c + S));
            put_box(vb + 16, 2 * (c + S) + 1);
            tmem_wait_ld();
          }
        } else {
          // Two warps per TMEM lane quarter, alternate 32-column chunks:
          // TMEM -> registers (the warp's next chunk in flight while this
          // one is written) -> this warp's 32-row x 32-column staging box
          // (128-byte rows, 128-byte swizzle: conflict-free, the TMA's
          // layout) -> proxy fence -> TMA store (or f32 add-reduction). Each
          // 256-column half of the accumulator is released as soon as both
          // warps of every quarter hold their last chunks of it: the drain
          // is exposed once per wide tile, and twice the warps read TMEM and
          // issue stores concurrently.
          uint8_t* box = s_c + (warp - 2) * 4096;
          const uint32_t taddr = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
          auto put = [&](const uint32_t* w, int c) {  // columns [c*32, c*32+32)
            if (lane == 0) bulk_wait_read<0>();  // this warp's previous store has left smem
            __syncwarp();
            uint8_t* my_row = box + lane * 128;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(my_row + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && !args.epi_skip) {
              const int col0 = nb * W + c * 32;
              if (args.accumulate || part == 1)
                tma_reduce_add_2d(&map_c, box, col0, row_base);
              else if (args.hint_c != kEvictNormal)
                tma_store_2d_hint(&map_c, box, col0, row_base, args.hint_c);
              else
                tma_store_2d(&map_c, box, col0, row_base);
              bulk_commit();
            }
          };
          uint32_t va[32], vb[32];
          tmem_ld_32x32b_x32(taddr + sub * 32, va);
          tmem_wait_ld();
#pragma unroll 1
          for (int i = 0; i < 8; i += 2) {  // this warp's chunks sub + 2i (8 of 16)
            const int ca = sub + 2 * i;
            tmem_ld_32x32b_x32(taddr + (ca + 2) * 32, vb);
            put(va, ca);
            tmem_wait_ld();
            if (i == 2 || i == 6) {  // this warp's last chunk of a half is in registers
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_cluster(&acc_empty[i == 2 ? 0 : 1], pair_leader);
              if (args.trace && quad == 0 && sub == 0 && lane == 0)
                trace_add(args, i == 2 ? 12 : 13, gtimer() - te0);
            }
            if (i + 2 < 8) tmem_ld_32x32b_x32(taddr + (ca + 4) * 32, va);
            put(vb, ca + 2);
            tmem_wait_ld();
          }
        }
        if (args.trace && quad == 0 && sub == 0 && lane == 0) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          args.trace[blockIdx.x * 16 + 6] = tt;
        }
        if (args.sblocks && lane == 0) {
          // this warp's boxes of the tile are in global memory: count it;
          // the block's last warp raises the block flag (its copy-out waits
          // on it, cuStreamWaitValue32)
          bulk_wait_all();
          fence_proxy_async_global();
          __threadfence();
          const int target = args.stream_epoch * blk_tiles * 2 * P::kEpiWarps;
          if (atomicAdd(args.block_count + blk, 1) + 1 == target) {
            __threadfence();
            atomicExch(args.block_flags + blk, args.stream_epoch);
          }
        }
        if (part == 0 && lane == 0) {
          // this warp's boxes of the first K-half are in global memory: the
          // tile's last warp (16 shares per pair tile) raises its ready flag
          bulk_wait_all();
          fence_proxy_async_global();
          __threadfence();
          int* sc = args.split_cnt + 4 * (unit_tile(args, t, k_blocks, kb0, kb1, part) - args.split_base);
          if (atomicAdd(sc, 8 / P::kEpiWarps) + 8 / P::kEpiWarps == 16) {
            atomicExch(sc, 0);
            __threadfence();
            atomicExch(sc + 1, 1);
          }
        }
        if (W == 512 || (acc ^= 1) == 0) acc_phase ^= 1;
        continue;  // (the for-increment fetches the next tile)
      }
      const int row = row_base + lane;
      float* crow = args.C + static_cast<long long>(row) * args.ldc;
#pragma unroll 1
      for (int c = sub; c < W / 32; c += P::kEpiWarps / 4) {  // this warp's 32-column chunks
        uint32_t v[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                               static_cast<uint32_t>((W == 256 ? acc * 256 : 0) + c * 32),
                           v);
        tmem_wait_ld();
        if (row < args.M) {
          const int col0 = nb * W + c * 32;
          if (vec && col0 + 32 <= args.N) {
            float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4 o = make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                     __uint_as_float(v[4 * j + 2]),
                                     __uint_as_float(v[4 * j + 3]));
              if (args.accumulate) {
                const float4 p = dst[j];
                o.x += p.x;
                o.y += p.y;
                o.z += p.z;
                o.w += p.w;
              }
              dst[j] = o;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = col0 + j;
              if (col < args.N) {
                float o = __uint_as_float(v[j]);
                if (args.accumulate) o += crow[col];
                crow[col] = o;
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // the leader's barrier(s)
        mbar_arrive_cluster(&acc_empty[W == 256 ? acc : 0], pair_leader);
        if (W == 512) mbar_arrive_cluster(&acc_empty[1], pair_leader);
      }
      if (args.sblocks) {
        // direct stores (C pitch TMA cannot map): the same per-block count
        // as the TMA-store path, after this warp's st.global are visible
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          const int target = args.stream_epoch * blk_tiles * 2 * P::kEpiWarps;
          if (atomicAdd(args.block_count + blk, 1) + 1 == target) {
            __threadfence();
            atomicExch(args.block_flags + blk, args.stream_epoch);
          }
        }
      }
      if (W == 512 || (acc ^= 1) == 0) acc_phase ^= 1;
    }
    if (args.tma_store && lane == 0) bulk_wait_all();  // C written before the CTA retires
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer may still be reading TMEM / signalling the leader
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, kTmemCols);
  }
  if (threadIdx.x == 0) trace_stamp(args, 7);
}

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D map over a row-major [rows x cols] 16-bit matrix with leading dim `ld`.
bool make_map(CUtensorMap* map, AbType t, const void* base, int64_t rows, int64_t cols,
              int64_t ld, uint32_t box_cols, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r =
      fn(map, t == AbType::bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
         2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 3-D map over panel-major 16-bit B: P panels of [K x np] (row pitch ld
// elements, panel stride K * ld), boxes of 64 columns x 64 k x 1 panel.
bool make_map_panels(CUtensorMap* map, AbType t, const void* base, int64_t K, int64_t np,
                     int64_t ld, int P) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(np), static_cast<cuuint64_t>(K),
                              static_cast<cuuint64_t>(P)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2,
                                 static_cast<cuuint64_t>(K) * static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(kBK), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, t == AbType::bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
            3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D map over a row-major fp32 [rows x cols] C with leading dim `ld`
// (elements): the epilogue's staging boxes -- 32 x 32 with 128-byte swizzle
// for 256 x 512 tiles, 16 columns x 32 rows with 64-byte swizzle for 256 x 256.
bool make_map_c(CUtensorMap* map, float* base, int64_t rows, int64_t cols, int64_t ld, bool wide) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {wide ? 32u : 16u, 32};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// POAS_TC_TRACE: synchronise, read the stamps back, print per-event
// percentiles (us after the earliest entry) to stderr.
void print_trace(unsigned long long* dev, int ctas, cudaStream_t stream, int64_t M, int64_t N,
                 int64_t K) {
  std::vector<unsigned long long> h(static_cast<size_t>(ctas) * 16);
  cudaStreamSynchronize(stream);
  cudaMemcpy(h.data(), dev, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int c = 0; c < ctas; ++c)
    if (h[c * 16]) t0 = std::min(t0, h[c * 16]);
  static const char* names[14] = {"entry", "prologue", "first_tma", "first_full", "last_commit",
                                  "epi_acc", "epi_issued", "exit", "published", "empty_ok",
                                  "sum_mma_wait_h0", "sum_mma_wait_h1", "sum_epi_h0", "sum_epi_h1"};
  std::fprintf(stderr, "tc_trace M=%lld N=%lld K=%lld ctas=%d:", static_cast<long long>(M),
               static_cast<long long>(N), static_cast<long long>(K), ctas);
  for (int e = 0; e < 14; ++e) {
    std::vector<double> v;
    for (int c = 0; c < ctas; ++c)
      if (h[c * 16 + e]) v.push_back((h[c * 16 + e] - (e < 10 ? t0 : 0)) * 1e-3);
    std::sort(v.begin(), v.end());
    if (v.empty()) continue;
    std::fprintf(stderr, " %s[min %.2f med %.2f max %.2f n %zu]", names[e], v.front(),
                 v[v.size() / 2], v.back(), v.size());
  }
  std::fprintf(stderr, "\n");
}

}  // namespace

int device_sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

namespace {
// Tile-scheduler counters {next, done}, one per (device, stream). Zeroed
// once at allocation; every launch leaves its counter zero again
// (release_counter), so no per-launch memset. Launches on one stream run
// one after another, so they can share a counter; launches on different
// streams may run at the same time and never do (a shared
// per-device ring could hand two concurrent launches the same slot once one
// stream had queued more launches than the ring had slots).
// Last-wave split counters (TcArgs::split_cnt), 4 ints per split tile, one
// zeroed block per (device, stream); every launch leaves them zero.
constexpr int kSplitMax = 128;
int* split_counters(cudaStream_t stream) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> by_stream;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(dev, stream);
  if (auto it = by_stream.find(key); it != by_stream.end()) return it->second;
  int* p = nullptr;
  const size_t bytes = kSplitMax * 4 * sizeof(int);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return nullptr;
  }
  by_stream.emplace(key, p);
  return p;
}

int* next_tile_counter(cudaStream_t stream) {
  constexpr int kBlock = 64;  // counters per allocation, 128 B apart
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> by_stream;
  static int* block[64] = {};
  static int used[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  const auto key = std::make_pair(dev, stream);
  if (auto it = by_stream.find(key); it != by_stream.end()) return it->second;
  if (!block[dev] || used[dev] == kBlock) {
    int* p = nullptr;
    const size_t bytes = kBlock * 32 * sizeof(int);
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(p);
      return nullptr;
    }
    block[dev] = p;  // earlier blocks stay allocated: their counters are in use
    used[dev] = 0;
  }
  int* c = block[dev] + used[dev]++ * 32;
  by_stream.emplace(key, c);
  return c;
}
}  // namespace

namespace {
// Kernel variants: the CTA-pair kernel wherever its tiles keep the SM budget
// reasonably busy -- 256 x 512 tiles (1/4 fewer operand bytes from L2 per
// MAC than 256 x 256, whose tiles in turn move 1/3 fewer than a single SM's
// 128 x 256) once there are at least two waves of them, 256 x 256 below;
// when at most a quarter of the pairs would have a 256 x 256 tile (e.g.
// 1024^3: 16 tiles for 74 pairs) the single-SM kernel with 128 x 128 tiles
// spreads the work over 4x as many CTAs. POAS_TC_KERNEL = 2cta512 | 2cta |
// 1cta (128 x 256) | 1cta128 overrides.
enum class TcVariant { pair512x2, pair256x2, pair512, pair, single256, single128, single64 };

TcVariant choose_variant(int64_t M, int64_t N, int64_t K, int budget) {
  if (const char* v = std::getenv("POAS_TC_KERNEL")) {
    const std::string s(v);
    if (s == "1cta") return TcVariant::single256;
    if (s == "1cta128") return TcVariant::single128;
    if (s == "1cta64") return TcVariant::single64;
    if (s == "2cta") return TcVariant::pair;
    if (s == "2cta512") return TcVariant::pair512;
    if (s == "2cta512x2") return TcVariant::pair512x2;
    if (s == "2cta256x2") return TcVariant::pair256x2;
  }
  // Single-SM tiles when the grid of 128 x 128 tiles fits in one wave of the
  // budget: 128 x 64 tiles when even those would leave half the SMs idle
  // (1024^3: 242 vs 213 TFLOP/s, cuBLAS 242-247), else 128 x 128 (1536^3:
  // 497 vs 454 for pair tiles); pair tiles from there on (2048^3: 906 vs
  // 682), profiles/r02_n64.
  const int64_t t128 = ((M + 127) / 128) * ((N + 127) / 128);
  if (2 * t128 <= budget) return TcVariant::single64;
  if (t128 <= budget) return TcVariant::single128;
  // 256 x 512 tiles need two waves of them, and a long K: their
  // accumulator drain is exposed once per tile (4096^3: 1343 -> 1190
  // TFLOP/s with wide tiles; 8192^3 and up they win, profiles/r02_sizes4)
  const int64_t wide_tiles = ((M + 255) / 256) * ((N + 511) / 512);
  return wide_tiles >= 2 * (budget / 2) && K >= 6144 ? TcVariant::pair512 : TcVariant::pair;
}

const char* variant_name(TcVariant v) {
  switch (v) {
    case TcVariant::single256: return "tc_gemm_kernel";
    case TcVariant::single128: return "tc_gemm_kernel_n128";
    case TcVariant::single64: return "tc_gemm_kernel_n64";
    case TcVariant::pair512: return "tc_gemm_2cta_kernel<512>";
    case TcVariant::pair512x2: return "tc_gemm_2cta_kernel<512,2>";
    case TcVariant::pair256x2: return "tc_gemm_2cta_kernel<256,2>";
    case TcVariant::pair: break;
  }
  return "tc_gemm_2cta_kernel<256>";
}
}  // namespace

// Clusters of two CTA pairs that fit on the device at once (a cluster of 4
// must sit inside one GPC; GPCs with an SM count not divisible by 4 leave
// SMs idle). Cached per device.
int max_active_clusters_x2();

cudaError_t tc_prepare_stream(cudaStream_t stream) {
  return next_tile_counter(stream) && split_counters(stream) ? cudaSuccess : cudaErrorMemoryAllocation;
}

const char* tc_gemm_kernel_name(int64_t M, int64_t N, int64_t K) {
  return variant_name(choose_variant(M, N, K, device_sm_count()));
}

const char* tc_gemm_scheduler_name(int64_t M, int64_t N, int64_t K) {
  if (const char* v = std::getenv("POAS_TC_SCHED")) {
    const std::string s(v);
    if (s == "static" || s == "wave" || s == "dynamic") return s == "static" ? "static"
                                                               : s == "wave" ? "wave" : "dynamic";
  }
  const double macs = static_cast<double>(M) * static_cast<double>(N) * static_cast<double>(K);
  return macs >= 17592186044416.0 ? "wave" : "dynamic";
}

namespace {
cudaError_t tc_gemm_impl(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                         const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                         int num_ctas, const TcPanels* ps, const TcStream* ss, cudaStream_t stream);
}

cudaError_t tc_gemm(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                    const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                    int num_ctas, cudaStream_t stream) {
  return tc_gemm_impl(t, M, N, K, A, lda, B, ldb, C, ldc, accumulate, num_ctas, nullptr, nullptr,
                      stream);
}

cudaError_t tc_gemm_stream(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                           const void* B, int64_t ldb, float* C, int64_t ldc, int num_ctas,
                           const TcStream& s, cudaStream_t stream) {
  return tc_gemm_impl(t, M, N, K, A, lda, B, ldb, C, ldc, false, num_ctas, nullptr, &s, stream);
}

cudaError_t tc_gemm_panels(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                           const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                           int num_ctas, const TcPanels& panels, cudaStream_t stream) {
  return tc_gemm_impl(t, M, N, K, A, lda, B, ldb, C, ldc, accumulate, num_ctas, &panels, nullptr,
                      stream);
}

namespace {
// Launch with programmatic stream serialization (the kernels call
// griddepcontrol.wait before touching global memory), so a GEMM's launch
// and prologue overlap the previous kernel of its stream. POAS_TC_PDL=0
// launches plainly.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int threads, size_t smem,
                       cudaStream_t stream, int cluster, Args&&... args) {
  static const bool pdl = [] {
    const char* e = std::getenv("POAS_TC_PDL");
    return !(e && std::string(e) == "0");
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (cluster > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

cudaError_t tc_gemm_impl(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                         const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                         int num_ctas, const TcPanels* ps, const TcStream* ss, cudaStream_t stream) {
  if (t != AbType::bf16 && t != AbType::f16) return cudaErrorInvalidValue;
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int P = ps ? ps->panels : 1;
  if (P < 1 || N % P != 0) return cudaErrorInvalidValue;
  const int64_t np = N / P;  // columns per panel
  if (P > 1 && np % 256 != 0) return cudaErrorInvalidValue;  // a pair tile never straddles panels
  if (K <= 0) {
    if (accumulate) return cudaSuccess;
    return cudaMemset2DAsync(C, static_cast<size_t>(ldc) * 4, 0, static_cast<size_t>(N) * 4,
                             static_cast<size_t>(M), stream);
  }
  // TMA: 16-byte aligned base and row pitch (ldb: a panel's row pitch).
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (lda * 2) % 16 || (ldb * 2) % 16 || lda < K || ldb < np || ldc < N)
    return cudaErrorInvalidValue;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return cudaErrorInvalidValue;

  CUtensorMap ma, mb;
  if (!make_map(&ma, t, A, M, K, lda, kBK, kBM)) return cudaErrorInvalidValue;
  if (P > 1) {
    if (!make_map_panels(&mb, t, B, K, np, ldb, P)) return cudaErrorInvalidValue;
  } else if (!make_map(&mb, t, B, K, N, ldb, 64, kBK)) {
    return cudaErrorInvalidValue;
  }

  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(tc_gemm_kernel<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(Tile1<256, 4>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_kernel<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Tile1<64, 8>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_kernel<128, 6>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Tile1<128, 6>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_2cta_kernel<256, 1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Pair<256>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_2cta_kernel<256, 1, 8>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Pair<256, 8>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_2cta_kernel<512, 1>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Pair<512>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_2cta_kernel<256, 2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Pair<256>::kSmem));
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(tc_gemm_2cta_kernel<512, 2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Pair<512>::kSmem));
  });
  if (attr_err != cudaSuccess) return attr_err;
  // Kernel choice: the CTA-pair kernel (1/3 fewer operand bytes into shared
  // memory per MAC than the single-SM kernel; faster at every size measured
  // once its scheduler fits the size, profiles/r01_tile_scheduler).
  // POAS_TC_KERNEL=1cta|2cta overrides (A/B comparisons, tests).
  const int budget_all = num_ctas > 0 ? num_ctas : device_sm_count();
  TcVariant variant = choose_variant(M, N, K, budget_all);
  if (P > 1 || ss) {
    // panels / streamed operands: the pair kernel only; streamed block
    // tables are in 256 x 256 tiles, panels take 512-wide tiles when every
    // panel is a whole number of them
    const char* v = std::getenv("POAS_TC_KERNEL");
    if (v && std::string(v) != "2cta" && std::string(v) != "2cta512" && std::string(v) != "2cta512x2" &&
        std::string(v) != "2cta256x2")
      return cudaErrorNotSupported;
    const bool wide = (variant == TcVariant::pair512 || variant == TcVariant::pair512x2) && !ss &&
                      np % 512 == 0;
    if (!wide) variant = variant == TcVariant::pair256x2 && !ss ? variant : TcVariant::pair;
  }
  const bool force_1cta = variant != TcVariant::pair && variant != TcVariant::pair512 &&
                          variant != TcVariant::pair512x2 && variant != TcVariant::pair256x2;
  const char* group_env = std::getenv("POAS_TC_GROUP");  // raster experiments
  const int group_override = group_env ? std::atoi(group_env) : 0;

  const int sms = device_sm_count();
  const int budget = num_ctas > 0 ? num_ctas : sms;
  // panel flags / block tables / block flags exist only in the pair kernel:
  // a one-SM budget would run the single-SM kernel, which ignores them
  // (and a copy-out waiting on a block flag would never be released)
  if ((P > 1 || ss) && budget < 2) return cudaErrorNotSupported;
  TcArgs args;
  args.M = static_cast<int>(M);
  args.N = static_cast<int>(N);
  args.K = static_cast<int>(K);
  args.C = C;
  args.ldc = ldc;
  args.accumulate = accumulate ? 1 : 0;
  auto hint = [](const char* name) {
    const char* v = std::getenv(name);
    if (v && std::string(v) == "first") return kEvictFirst;
    if (v && std::string(v) == "last") return kEvictLast;
    return kEvictNormal;
  };
  args.hint_a = hint("POAS_TC_HINT_A");  // experiment knobs; default evict_normal
  args.hint_b = hint("POAS_TC_HINT_B");
  // C is written once and never re-read here: evict_first keeps the A/B
  // panels in L2 (16384^3: DRAM reads 10.5 -> 10.1 GB, profiles/r01_epilogue)
  const char* hc = std::getenv("POAS_TC_HINT_C");
  args.hint_c = hc && std::string(hc) == "normal" ? kEvictNormal : kEvictFirst;
  const char* raster_env = std::getenv("POAS_TC_RASTER");
  args.raster_n = raster_env && std::string(raster_env) == "n";
  // K serpentine (default on; POAS_TC_KSERP=0 = every tile sweeps K
  // forwards): DRAM reads per launch -7.5% at 8192^3 and 16384^3, -5.7% at
  // 32768^3, time neutral to +0.25% (profiles/r01_kserp)
  const char* kserp_env = std::getenv("POAS_TC_KSERP");
  args.kserp = !(kserp_env && std::string(kserp_env) == "0");
  // Tile scheduler: dynamic claiming below 2^44 MACs; wave-synchronised
  // static order from there on (a tile lasts long enough that the claim
  // order's stagger spreads A-panel sharers over more than an L2 lifetime:
  // 206 -> 69 GB DRAM and +25% sustained at 32768^3). POAS_TC_SCHED=
  // dynamic|wave|static overrides.
  const std::string sched = tc_gemm_scheduler_name(M, N, K);
  args.tile_counter = nullptr;
  args.tma_store = 0;
  args.trace = nullptr;
  args.panels = P;
  {
    const char* po = std::getenv("POAS_TC_PANEL_ORDER");  // "panel": tiles panel by panel
    args.panel_order = po && std::string(po) == "panel";
  }
  args.tiles_n_panel = static_cast<int>(
      np / (variant == TcVariant::pair512 || variant == TcVariant::pair512x2 ? 512 : 256));
  args.panel_flags = ps ? ps->flags : nullptr;
  args.panel_epoch = ps ? ps->epoch : 0;
  args.sblocks = nullptr;
  args.nsblocks = 0;
  args.item_flags = nullptr;
  args.block_count = nullptr;
  args.block_flags = nullptr;
  args.stream_epoch = 0;
  args.split_base = 0;
  args.split_kb = 0;
  args.split_cnt = nullptr;
  if (ss) {
    args.sblocks = reinterpret_cast<const int4*>(ss->blocks);
    args.nsblocks = ss->nblocks;
    args.item_flags = ss->item_flags;
    args.block_count = ss->block_count;
    args.block_flags = ss->block_flags;
    args.stream_epoch = ss->epoch;
  }
  args.epi_skip = std::getenv("POAS_TC_EPI_SKIP") != nullptr;
  args.wave_sync = sched == "wave";
  if (sched != "static") {
    args.tile_counter = next_tile_counter(stream);
    if (!args.tile_counter) return cudaErrorMemoryAllocation;
  }

  if (!force_1cta && budget >= 2) {
    // CTA pairs: 256 x 256 tiles, grid = even SM budget (one pair per TPC).
    // Epilogue through TMA stores when C allows a tensor map (16-byte
    // aligned base and row pitch); POAS_TC_EPILOGUE=direct forces the
    // register -> global path.
    // clusters of two pairs need a budget of at least one cluster
    const bool x2 = (variant == TcVariant::pair512x2 || variant == TcVariant::pair256x2) &&
                    std::min(budget / 4, max_active_clusters_x2()) >= 1;
    const bool wide = variant == TcVariant::pair512x2 || variant == TcVariant::pair512;
    const int w = wide ? 512 : 256;
    const int rows_t = x2 ? 512 : 256;
    args.tiles_m = static_cast<int>((M + rows_t - 1) / rows_t);
    args.tiles_n = static_cast<int>((N + w - 1) / w);
    CUtensorMap mc;
    const char* epi = std::getenv("POAS_TC_EPILOGUE");
    const bool direct = epi && std::string(epi) == "direct";
    args.tma_store = !direct && (reinterpret_cast<uintptr_t>(C) & 15) == 0 && ldc % 4 == 0 &&
                     make_map_c(&mc, C, M, N, ldc, wide);
    if (!args.tma_store) mc = ma;  // unused
    args.idesc = idesc_f16(t == AbType::bf16, 256, 256, false, true);  // per 256-column half
    args.group = group_override > 0 ? group_override : (x2 ? kGroupM2 / 2 : kGroupM2);
    const int tiles = args.tiles_m * args.tiles_n;
    int pairs = budget / 2;
    if (x2) {  // whole clusters of two pairs, no more than can be resident at once
      int clusters = std::min(budget / 4, max_active_clusters_x2());
      if (clusters > tiles) clusters = tiles;
      pairs = 2 * clusters;
    } else if (pairs > tiles) {
      pairs = tiles;
    }
    // 256 x 256 tiles: 8 epilogue warps when the GEMM is one wave of tiles
    // (its drain is all exposed); POAS_TC_EPI=4|8 overrides
    const char* epi_env = std::getenv("POAS_TC_EPI");
    const bool epi8 = epi_env ? std::atoi(epi_env) == 8 : tiles <= pairs;
    // Last-wave K split (opt-in, POAS_TC_SPLIT=1): when the last wave holds
    // at most half a wave of tiles, those tiles run as two K-halves on
    // twice the pairs (4096^3 with 256 x 256 tiles: 256 tiles on 74 pairs,
    // the last 34 as 68 halves). Measured, it does not pay: 4096^3-5120^3
    // within +-0.5%, 2560^3 -6% (profiles/r02_split) -- a part-filled last
    // wave already runs faster per tile than a full one. Dynamic scheduler
    // only (a half's partner is claimed no later than itself), TMA-store
    // epilogue, one pair per cluster, no panel flags / streamed blocks; never
    // in the deterministic mode (POAS_TC_KSERP=0).
    {
      const int all_pairs = budget / 2;
      const int rem = tiles % all_pairs;
      const int kbl = static_cast<int>((K + kBK - 1) / kBK);
      const char* split_env = std::getenv("POAS_TC_SPLIT");
      const bool split_on = split_env && std::string(split_env) == "1";
      if (split_on && args.kserp && !x2 && args.tma_store && !ss && !ps && P == 1 &&
          args.tile_counter && !args.wave_sync && kbl >= 8 && rem > 0 && 2 * rem <= all_pairs &&
          rem <= kSplitMax) {
        args.split_cnt = split_counters(stream);
        if (!args.split_cnt) return cudaErrorMemoryAllocation;
        args.split_base = tiles - rem;
        args.split_kb = kbl / 2;
        pairs = std::min(all_pairs, tiles + rem);
      }
    }
    static unsigned long long* trace_buf = nullptr;
    const bool trace = std::getenv("POAS_TC_TRACE") != nullptr;
    if (trace) {
      if (!trace_buf && cudaMalloc(&trace_buf, 4096 * 16 * sizeof(unsigned long long)) != cudaSuccess)
        return cudaErrorMemoryAllocation;
      cudaMemsetAsync(trace_buf, 0, 2 * pairs * 16 * sizeof(unsigned long long), stream);
      args.trace = trace_buf;
    }
    const cudaError_t e =
        x2 && wide ? launch_pdl(tc_gemm_2cta_kernel<512, 2>, 2 * pairs, Pair<512>::kThreads, Pair<512>::kSmem,
                                stream, 1, ma, mb, mc, args)
        : x2       ? launch_pdl(tc_gemm_2cta_kernel<256, 2>, 2 * pairs, Pair<256>::kThreads, Pair<256>::kSmem,
                                stream, 1, ma, mb, mc, args)
        : wide     ? launch_pdl(tc_gemm_2cta_kernel<512, 1>, 2 * pairs, Pair<512>::kThreads, Pair<512>::kSmem,
                                stream, 1, ma, mb, mc, args)
        : epi8     ? launch_pdl(tc_gemm_2cta_kernel<256, 1, 8>, 2 * pairs, Pair<256, 8>::kThreads,
                                Pair<256, 8>::kSmem, stream, 1, ma, mb, mc, args)
                   : launch_pdl(tc_gemm_2cta_kernel<256, 1>, 2 * pairs, Pair<256>::kThreads, Pair<256>::kSmem,
                                stream, 1, ma, mb, mc, args);
    if (trace) print_trace(trace_buf, 2 * pairs, stream, M, N, K);
    return e;
  }
  const int bn = variant == TcVariant::single64 ? 64 : variant == TcVariant::single128 ? 128 : 256;
  args.tiles_m = static_cast<int>((M + kBM - 1) / kBM);
  args.tiles_n = static_cast<int>((N + bn - 1) / bn);
  args.idesc = idesc_f16(t == AbType::bf16, kBM, bn, false, true);
  args.group = group_override > 0 ? group_override : kGroupM;
  int grid = budget;
  const int tiles = args.tiles_m * args.tiles_n;
  if (grid > tiles) grid = tiles;
  if (bn == 64)
    return launch_pdl(tc_gemm_kernel<64, 8>, grid, kThreads, Tile1<64, 8>::kSmem, stream, 1, ma, mb, args);
  if (bn == 128)
    return launch_pdl(tc_gemm_kernel<128, 6>, grid, kThreads, Tile1<128, 6>::kSmem, stream, 1, ma, mb, args);
  return launch_pdl(tc_gemm_kernel<256, 4>, grid, kThreads, Tile1<256, 4>::kSmem, stream, 1, ma, mb, args);
}
}  // namespace

int max_active_clusters_x2() {
  static std::mutex mu;
  static std::map<int, int> by_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (auto it = by_dev.find(dev); it != by_dev.end()) return it->second;
  int n = 0;
  if (cudaFuncSetAttribute(tc_gemm_2cta_kernel<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(Pair<512>::kSmem)) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * 64);
    cfg.blockDim = dim3(Pair<512>::kThreads);
    cfg.dynamicSmemBytes = Pair<512>::kSmem;
    cfg.numAttrs = 0;  // the cluster shape (4) is compiled into the kernel
    if (cudaOccupancyMaxActiveClusters(&n, tc_gemm_2cta_kernel<512, 2>, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  by_dev[dev] = n;
  return n;
}

cudaError_t wait_flag(const int* flag, int value, cudaStream_t stream) {
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitFn>(p);
  });
  if (!fn) return cudaErrorNotSupported;
  return fn(reinterpret_cast<CUstream>(stream),
            reinterpret_cast<CUdeviceptr>(const_cast<int*>(flag)), static_cast<cuuint32_t>(value),
            CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

// Writes `value` to a device int in `stream` order (cuStreamWriteValue32:
// no kernel, no SM).
cudaError_t signal_flag(int* flag, int value, cudaStream_t stream) {
  using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WriteFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteFn>(p);
  });
  if (!fn) return cudaErrorNotSupported;
  return fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag),
            static_cast<cuuint32_t>(value), 0) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

}  // namespace poas_b200
