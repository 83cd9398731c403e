// The multi-GPU exchange of the row-sharded GEMM: B, resident
// on rank 0, reaches every GPU of the box once per GEMM.
//
// One process per GPU. A Comm joins the ranks of one job through a POSIX
// shared-memory segment (bootstrap, host barrier, small all-gathers, and the
// cross-rank panel flags), maps the upstream rank's B buffers with CUDA IPC,
// and moves B in column panels as a pipelined CHAIN: rank r pulls panel p
// from rank r-1 with a peer copy (copy engines over NVLink -- no SMs, so a
// persistent GEMM spinning on panel flags can never starve it) once rank
// r-1's flag for (panel p, epoch) is up (cuStreamWaitValue32 on the
// host-mapped flag), then raises its own flags: the host-mapped one in the
// segment (for rank r+1) and a device int (for the local tensor GEMM's
// producers), and records a per-panel CUDA event (for a CUDA-core unit).
// Every link of the chain carries B once; with P panels and G GPUs the last
// panel lands after about (P + G - 2) panel copy times.
//
// Non-root ranks receive into two comm-owned buffers used by alternate
// epochs, so the broadcast of step e+1 overlaps the GEMM of step e; rank 0
// serves the caller's B. Optional transport "nccl": ncclBroadcast per panel
// (libnccl.so.2, loaded at run time) on the same stream, same flags -- its
// kernels need SMs beside the GEMM (leave them free in the units' budgets).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace poas_b200 {

enum class Transport { ce, nccl };
Transport parse_transport(const std::string& s);
const char* transport_name(Transport t);

class Comm {
 public:
  static constexpr int kMaxRanks = 16;
  static constexpr int kMaxPanels = 64;

  // `name`: the job's rendezvous token (same on every rank, unique per job).
  // `device` < 0: a host-only comm (barrier / all-gather; no CUDA).
  Comm(const std::string& name, int rank, int world, int device);
  ~Comm();
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;

  int rank() const { return rank_; }
  int world() const { return world_; }
  int device() const { return device_; }

  // Host barrier over the segment (all ranks; throws after `timeout_s`).
  void barrier(double timeout_s = 600.0);
  // Every rank's `mine` (<= 64 KiB), in rank order (collective).
  std::vector<std::string> allgather(const std::string& mine);
  // max over ranks (collective)
  double allreduce_max(double v);

  // NCCL communicator over the same ranks (collective). `id` = rank 0's
  // ncclUniqueId bytes, distributed by the caller (e.g. allgather).
  static std::vector<unsigned char> nccl_unique_id();
  void init_nccl(const void* id, std::size_t bytes);
  bool has_nccl() const { return nccl_ != nullptr; }

  // Collective. This rank's panel-major B ([panels][k][n/panels]) in the
  // tensor units' 16-bit type (b16) and, optionally, fp32 (b32): rank 0's
  // are served; the others receive into comm-owned buffers.
  void register_b(const void* b16, const void* b32, std::int64_t k, std::int64_t n, int panels);
  bool registered() const { return panels_ > 0; }
  bool has_b32() const { return sets_[1].active; }
  int panels() const { return panels_; }

  // One broadcast of B (the fp32 copy too when `with_b32` and registered),
  // enqueued on the comm stream after the events in `after` (this GPU).
  // Returns the epoch; the GEMMs reading b16_for(epoch) wait on dev_flags()
  // (>= epoch) or panel_events().
  int enqueue_broadcast(Transport t, bool with_b32, const std::vector<cudaEvent_t>& after);
  // The consumers of epoch `epoch`'s buffers are queued on `s`: the
  // broadcast that next reuses those buffers (epoch + 2) waits for them.
  void consumed(int epoch, cudaStream_t s);
  const void* b16_for(int epoch) const;
  const float* b32_for(int epoch) const;
  const int* dev_flags() const { return dev_flags_; }
  void* const* panel_events() const { return reinterpret_cast<void* const*>(events_.data()); }
  cudaStream_t stream() const { return stream_; }
  int epoch() const { return epoch_; }

  // The link probe (DeviceBackend::time_transfer of a GPU's level-1 link):
  // seconds to deliver `bytes` to every rank in 16 chunks by transport `t`,
  // max over ranks, mean of `reps` (collective).
  double time_broadcast(Transport t, std::uint64_t bytes, int reps = 3);

 private:
  struct Shared;
  // One broadcast buffer set (slot 0 = B bf16/fp16, 1 = B fp32, 2 = probe).
  struct BufSet {
    const void* own = nullptr;  // rank 0: the served buffer
    void* recv[2] = {nullptr, nullptr};
    const void* up[2] = {nullptr, nullptr};  // rank r-1's buffers, by parity
    void* mapped[2] = {nullptr, nullptr};    // the IPC mappings behind up[]
    int last[2] = {0, 0};  // epoch that last filled recv[parity] (0 = none)
    std::size_t bytes = 0;
    bool active = false;
  };
  void map_segment(const std::string& name);
  const int* flag_dev(int r, int p) const;  // device pointer of a host-mapped flag
  int* flag_dev_mut(int r, int p) const;
  void register_set(int slot, const void* own, std::size_t bytes, bool present);
  void release_set(int slot);
  void enqueue_sets(Transport t, int epoch, const std::vector<int>& slots, int panels);
  void* dst(int slot, int epoch) const;

  int rank_, world_, device_;
  Shared* sh_ = nullptr;
  std::size_t sh_bytes_ = 0;
  int* flags_dev_base_ = nullptr;
  bool flags_registered_ = false;
  cudaStream_t stream_ = nullptr;
  void* nccl_ = nullptr;  // ncclComm_t
  int epoch_ = 0;
  int panels_ = 0;
  std::int64_t k_ = 0, n_ = 0;
  BufSet sets_[3];
  int* dev_flags_ = nullptr;
  std::vector<cudaEvent_t> events_;
  std::vector<cudaEvent_t> consumed_[2];
};

}  // namespace poas_b200

// The C ABI's opaque handle (include/poas_b200.h poas_comm_t).
struct poas_comm_s {
  std::unique_ptr<poas_b200::Comm> comm;
};
