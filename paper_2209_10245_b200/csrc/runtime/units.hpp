// Compute units of a B200 box and their DeviceBackend plugins.
//
// A unit is one concurrently running share of the machine:
//   cpu : the host cores                 (host_gemm, no link)
//   gpu : the CUDA cores of one B200      (simt_gemm fp32 on an SM budget)
//   xpu : the tensor cores of one B200    (tc_gemm bf16/fp16 -> fp32 on an SM budget)
// Each unit implements poas::DeviceBackend (reference
// proj/include/poas/backend.hpp:11-24) with real timed work, so the
// reference's profiler drives it unchanged.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../kernels/kernels.hpp"
#include "poas/backend.hpp"
#include "poas/device_model.hpp"

namespace poas_b200 {

// What a unit's operands cross before it computes (what time_transfer
// measures): pcie = pinned host memory over the unit's PCIe link; hbm =
// resident operands streamed into the unit's own SMs (a streaming read on
// its budget: what a few-row CUDA-core share pays to read all of B); fused
// = resident operands whose stream is part of the probed GEMM itself (a
// tensor unit's fat share reads A and B while it computes, which its
// square-GEMM probes already time: a separate copy phase would count the
// stream twice -- 2048^3: +32% predicted, profiles/r02_lent5).
enum class Link { pcie, hbm, fused };

struct UnitSpec {
  std::string id;
  poas::DeviceKind kind = poas::DeviceKind::cpu;
  int device = 0;         // CUDA ordinal (gpu/xpu)
  int sms = 0;            // SM budget = persistent grid size (0 = all SMs)
  bool exclusive = true;  // gpu: own whole SMs (no co-residency with xpu CTAs)
  AbType dtype = AbType::bf16;  // xpu operand type
  std::uint32_t elem = 4;       // bytes per element crossing the link
  int threads = 0;              // cpu: OpenMP threads (0 = all cores)
  // xpu row alignment written to the profile (the adapter floors the unit's
  // rows to it and requires k % align == 0). The tcgen05 kernel needs none:
  // M/N/K tails are TMA out-of-bounds fills and the 16-byte row-pitch rule
  // is met by padded leading dimensions, so the default is 1 -- an align of
  // 8 (the paper's tensor cores) would push shaved rows onto a 25x slower
  // unit. "align=8" reproduces the reference's setting.
  std::int64_t align = 1;
  Link link = Link::pcie;       // what time_transfer measures
  std::int64_t probe_min = 0;   // own probe side range ("probe=MIN-MAX"); 0 = config's
  std::int64_t probe_max = 0;
  double preroll_ms = 0.0;      // GPU units: back-to-back launches before each timed probe
};

// "<id>=<kind>[:key=value]*"
UnitSpec parse_unit_spec(const std::string& text);
// ';'-separated unit specs plus optional machine tokens: "bus=0|1" (shared
// link, default 1), "lend=0|1" (idle units lend their SMs to the one busy
// unit on the same GPU during execute, default 1) and "overlap=0|1" (host
// operand runs pipeline each link unit's row parts: copies overlap compute,
// see poas/overlap.hpp; default 0 = the paper's synchronous copies) and
// "pipeline=0|1" (overlapped host runs of one streamed tensor unit: repeat
// r+1's host->device copies start once repeat r's GEMM is done, beside
// repeat r's device->host tail; C double-buffered; default 0).
std::vector<UnitSpec> parse_unit_list(const std::string& text, bool* bus = nullptr,
                                      bool* lend = nullptr, bool* overlap = nullptr,
                                      bool* pipeline = nullptr);

// Device scratch that grows on demand and is reused across calls.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void* ensure(std::size_t bytes);
  void* get() const { return ptr_; }

 private:
  void* ptr_ = nullptr;
  std::size_t bytes_ = 0;
};

class PinnedBuffer {
 public:
  PinnedBuffer() = default;
  ~PinnedBuffer();
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  void* ensure(std::size_t bytes);

 private:
  void* ptr_ = nullptr;
  std::size_t bytes_ = 0;
};

class Unit : public poas::DeviceBackend {
 public:
  explicit Unit(UnitSpec spec);
  ~Unit() override;

  const UnitSpec& spec() const { return spec_; }
  bool on_gpu() const { return spec_.kind != poas::DeviceKind::cpu; }
  cudaStream_t stream() const { return stream_; }

  // Probe plugin (DeviceBackend).
  double time_gemm(std::int64_t side) override;
  double time_transfer(std::uint64_t bytes) override;
  bool has_transfers() const override { return on_gpu(); }

  // The unit's GEMM on already-placed operands (device pointers for GPU
  // units -- 16-bit for xpu -- host pointers for cpu). Asynchronous on
  // stream() for GPU units, synchronous for cpu. `extra_sms` widens a GPU
  // unit's SM budget for this call (SMs lent by idle units on its GPU).
  void gemm(std::int64_t m, std::int64_t n, std::int64_t k, const void* a, std::int64_t lda,
            const void* b, std::int64_t ldb, float* c, std::int64_t ldc, bool accumulate,
            int extra_sms = 0);

  // xpu only: all `panels` column panels of panel-major B in one launch,
  // panel p gated on flags[p] >= epoch (kernels.hpp TcPanels).
  void gemm_panels(std::int64_t m, std::int64_t n, std::int64_t k, const void* a, std::int64_t lda,
                   const void* b, std::int64_t ldb, float* c, std::int64_t ldc, int panels,
                   const int* flags, int epoch, int extra_sms = 0);

  // xpu only: the streamed launch of an overlapped grid (kernels.hpp
  // TcStream), on stream().
  void gemm_stream(std::int64_t m, std::int64_t n, std::int64_t k, const void* a, std::int64_t lda,
                   const void* b, std::int64_t ldb, float* c, std::int64_t ldc, const TcStream& s,
                   int extra_sms = 0);

  // Scratch owned by the unit (staging for link copies in execute()).
  DeviceBuffer& scratch(int slot) { return scratch_[slot]; }

 private:
  UnitSpec spec_;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
  DeviceBuffer probe_a_, probe_b_, probe_c_, probe_a32_, probe_b32_, xfer_dev_, xfer_dev2_;
  PinnedBuffer xfer_host_;
  std::vector<float> host_a_, host_b_, host_c_;
  std::int64_t probe_side_ = 0;
  double last_probe_s_ = 0.0;  // the previous probe (pre-roll sizing)
  std::size_t xfer_warm_bytes_ = 0;  // link probe buffers warmed for this size
  std::int64_t last_probe_side_ = 0;
  // 0-4 staging, 5 streamed-launch state, 6 second C (pipelined), 7-8 second
  // 16-bit A / B staging (pipelined: repeat r+1 lands while r computes)
  DeviceBuffer scratch_[9];
};

// RAII device selection.
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev);
  ~DeviceGuard();

 private:
  int prev_ = 0;
};

}  // namespace poas_b200
