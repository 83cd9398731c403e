// Host-side launch entry points for the sm_100a unit kernels. All pointers
// are device pointers; all launches are asynchronous on `stream`.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace poas_b200 {

enum class AbType : int { f32 = 0, f16 = 1, bf16 = 2 };

// Tensor-core unit: C[M x N] (=|+=) A[M x K] * B[K x N], A and B row-major
// 16-bit (bf16 or fp16), fp32 accumulate, fp32 C. `num_ctas` bounds the
// persistent grid (the unit's SM budget); 0 = every SM.
// Returns a cudaError_t (cudaSuccess = 0).
cudaError_t tc_gemm(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                    const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                    int num_ctas, cudaStream_t stream);

// Panel-major B for tc_gemm_panels: `panels` column panels, panel p =
// B[:, p*N/P : (p+1)*N/P] stored as its own row-major [K x N/P] block (row
// pitch ldb, panel stride K*ldb) -- the layout a per-panel broadcast lands.
// N/P must be a multiple of 256 (the pair tile). With `flags`, the kernel's
// producers start on panel p once flags[p] >= epoch: whoever delivers B
// writes the flags in panel order (signal_flag after each panel's copy or
// broadcast), so one launch consumes B as it arrives. A flag never written
// traps the kernel after 10 s.
struct TcPanels {
  int panels = 1;
  const int* flags = nullptr;
  int epoch = 0;
};
cudaError_t tc_gemm_panels(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                           const void* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                           int num_ctas, const TcPanels& panels, cudaStream_t stream);

// Streamed operands: one launch over an R x Q grid of output blocks whose A
// row parts and B column panels arrive over time (overlapped copies). Block
// b: `blocks[4*b .. 4*b+3]` = {first M-tile | M-tiles << 16, first N-tile |
// N-tiles << 16, first tile id, A item | B item << 16} in 256-element tile
// units (device memory; blocks in compute order, first tile ids ascending,
// together covering every tile of C once). Producers start a block's tiles
// once item_flags of both its items are >= epoch; when every tile of block
// b is in global memory the kernel sets block_flags[b] = epoch
// (block_count[b] counts 8 per tile and must be epoch-1 times that at
// launch: zero it with the flags and count epochs from 1).
struct TcStream {
  const int* blocks = nullptr;
  int nblocks = 0;
  const int* item_flags = nullptr;
  int* block_count = nullptr;
  int* block_flags = nullptr;
  int epoch = 0;
};
cudaError_t tc_gemm_stream(AbType t, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda,
                           const void* B, int64_t ldb, float* C, int64_t ldc, int num_ctas,
                           const TcStream& s, cudaStream_t stream);

// *flag = value in stream order (cuStreamWriteValue32).
cudaError_t signal_flag(int* flag, int value, cudaStream_t stream);
// Creates the per-stream state tc_gemm launches on `stream` use (its tile
// scheduler counter), so that a launch can be captured into a CUDA graph.
cudaError_t tc_prepare_stream(cudaStream_t stream);
// The stream waits until *flag >= value (cuStreamWaitValue32, GEQ).
cudaError_t wait_flag(const int* flag, int value, cudaStream_t stream);

// The kernel tc_gemm launches: "tc_gemm_2cta_kernel" (CTA pairs,
// cta_group::2); POAS_TC_KERNEL=1cta selects "tc_gemm_kernel" (single SM).
const char* tc_gemm_kernel_name(int64_t M, int64_t N, int64_t K);
// Its tile scheduler: "dynamic" (atomic claiming) below 2^44 MACs, "wave"
// (static order, per-wave barrier) from there on; POAS_TC_SCHED overrides.
const char* tc_gemm_scheduler_name(int64_t M, int64_t N, int64_t K);

// CUDA-core unit: fp32 SIMT GEMM, same conventions.
cudaError_t simt_gemm(int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                      const float* B, int64_t ldb, float* C, int64_t ldc, bool accumulate,
                      int num_ctas, bool exclusive_sm, cudaStream_t stream);

// Counter-based uniform [-1, 1) fill, bit-identical to the host generator:
// element (r, c) of a rows x cols block at (row0, col0) inside a matrix of
// `total_cols` columns takes splitmix64 draw number (row0+r)*total_cols+col0+c
// of Rng(seed). Written as fp32 or rounded (RNE) to bf16/fp16.
cudaError_t fill_uniform(AbType t, void* dst, int64_t ld, int64_t rows, int64_t cols,
                         int64_t row0, int64_t col0, int64_t total_cols, uint64_t seed,
                         cudaStream_t stream);

// fp32 -> bf16/fp16 (RNE) of a rows x cols block.
cudaError_t convert_f32(AbType t, const float* src, int64_t ld_src, void* dst, int64_t ld_dst,
                        int64_t rows, int64_t cols, cudaStream_t stream);

// One-thread kernel that holds `stream` until the host writes a non-zero
// value to *flag (mapped pinned memory); times out after 10 s.
cudaError_t gate_wait(const int* flag, cudaStream_t stream);

// Streaming read of `bytes` (multiple of 16) by `num_ctas` CTAs of 512
// threads (0 = one per SM): the HBM bandwidth a unit on that SM budget sees.
cudaError_t stream_read(const void* src, size_t bytes, int num_ctas, float* sink,
                        cudaStream_t stream);

int device_sm_count();

}  // namespace poas_b200
