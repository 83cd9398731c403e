#include "comm.hpp"

#include <cuda.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>

#include "../kernels/kernels.hpp"
#include "capi_util.hpp"
#include "poas/error.hpp"
#include "units.hpp"

namespace poas_b200 {

using capi::cuda_check;

Transport parse_transport(const std::string& s) {
  if (s == "ce" || s.empty()) return Transport::ce;
  if (s == "nccl") return Transport::nccl;
  poas::fail(poas::errc::invalid_argument, "unknown B transport '" + s + "' (ce|nccl)");
}

const char* transport_name(Transport t) { return t == Transport::nccl ? "nccl" : "ce"; }

namespace {

constexpr std::uint32_t kMagic = 0x504f4153;  // "POAS"
constexpr std::size_t kText = 65536;

// ---- libnccl.so.2, resolved at run time (the process may already hold the
// copy torch ships; dlopen returns that one)
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = dlerror() ? dlerror() : "dlopen failed";
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.broadcast || !api.get_unique_id || !api.comm_init_rank)
    capi::raise(POAS_E_CUDA, "NCCL unavailable (libnccl.so.2): " + why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    capi::raise(POAS_E_CUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "error"));
}

// Base of the allocation holding `p` (IPC handles name allocations).
void* alloc_base(const void* p) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(f);
  });
  if (!fn) capi::raise(POAS_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    capi::raise(POAS_E_CUDA, "cuMemGetAddressRange failed (B must be device memory from cudaMalloc)");
  return reinterpret_cast<void*>(base);
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct Comm::Shared {
  std::uint32_t magic;
  int world;
  int bar_count;
  int bar_gen;
  struct Info {
    cudaIpcMemHandle_t h[3][2];
    std::uint64_t off[3][2];
    int has[3];
  } info[kMaxRanks];
  double value[kMaxRanks];
  int text_len[kMaxRanks];
  alignas(4096) int flags[kMaxRanks][kMaxPanels];  // host-mapped: value = epoch landed
  alignas(4096) char text[kMaxRanks][kText];
};

void Comm::map_segment(const std::string& name) {
  const std::string path = "/poas." + name;
  const int fd = shm_open(path.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) poas::fail(poas::errc::io_failure, "shm_open " + path + " failed");
  sh_bytes_ = (sizeof(Shared) + 4095) / 4096 * 4096;
  if (ftruncate(fd, static_cast<off_t>(sh_bytes_)) != 0) {
    close(fd);
    poas::fail(poas::errc::io_failure, "ftruncate " + path + " failed");
  }
  void* p = mmap(nullptr, sh_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) poas::fail(poas::errc::io_failure, "mmap " + path + " failed");
  sh_ = static_cast<Shared*>(p);
}

Comm::Comm(const std::string& name, int rank, int world, int device)
    : rank_(rank), world_(world), device_(device) {
  if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world)
    poas::fail(poas::errc::invalid_argument, "comm: bad rank/world");
  if (name.empty() || name.find('/') != std::string::npos)
    poas::fail(poas::errc::invalid_argument, "comm: name must be a non-empty token without '/'");
  map_segment(name);
  barrier();  // every rank has the segment mapped
  if (rank_ == 0) {
    shm_unlink(("/poas." + name).c_str());  // nothing left behind; the mappings persist
    __atomic_store_n(&sh_->magic, kMagic, __ATOMIC_SEQ_CST);
    __atomic_store_n(&sh_->world, world, __ATOMIC_SEQ_CST);
  }
  barrier();
  if (__atomic_load_n(&sh_->world, __ATOMIC_SEQ_CST) != world)
    poas::fail(poas::errc::invalid_argument, "comm: ranks disagree on the world size");
  if (device_ >= 0) {
    DeviceGuard g(device_);
    cuda_check(cudaHostRegister(&sh_->flags[0][0], sizeof(sh_->flags),
                                cudaHostRegisterMapped | cudaHostRegisterPortable),
               "cudaHostRegister (comm flags)");
    flags_registered_ = true;
    void* dp = nullptr;
    cuda_check(cudaHostGetDevicePointer(&dp, &sh_->flags[0][0], 0), "cudaHostGetDevicePointer");
    flags_dev_base_ = static_cast<int*>(dp);
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaMalloc(&dev_flags_, kMaxPanels * sizeof(int)), "cudaMalloc flags");
    cuda_check(cudaMemset(dev_flags_, 0, kMaxPanels * sizeof(int)), "cudaMemset flags");
    events_.assign(kMaxPanels, nullptr);
    for (auto& e : events_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  }
}

Comm::~Comm() {
  if (device_ >= 0) {
    DeviceGuard g(device_);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& list : consumed_)
      for (cudaEvent_t e : list) cudaEventDestroy(e);
    for (int s = 0; s < 3; ++s) release_set(s);
    for (cudaEvent_t e : events_) cudaEventDestroy(e);
    if (dev_flags_) cudaFree(dev_flags_);
    if (nccl_ && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(nccl_));
    if (stream_) cudaStreamDestroy(stream_);
    if (flags_registered_) cudaHostUnregister(&sh_->flags[0][0]);
  }
  if (sh_) munmap(sh_, sh_bytes_);
}

void Comm::barrier(double timeout_s) {
  const int gen = __atomic_load_n(&sh_->bar_gen, __ATOMIC_SEQ_CST);
  if (__atomic_fetch_add(&sh_->bar_count, 1, __ATOMIC_SEQ_CST) == world_ - 1) {
    __atomic_store_n(&sh_->bar_count, 0, __ATOMIC_SEQ_CST);
    __atomic_fetch_add(&sh_->bar_gen, 1, __ATOMIC_SEQ_CST);
    return;
  }
  const double t0 = now_s();
  int spins = 0;
  while (__atomic_load_n(&sh_->bar_gen, __ATOMIC_SEQ_CST) == gen) {
    if (++spins > 1000) std::this_thread::sleep_for(std::chrono::microseconds(50));
    if (now_s() - t0 > timeout_s) poas::fail(poas::errc::backend_failure, "comm barrier timed out");
  }
}

std::vector<std::string> Comm::allgather(const std::string& mine) {
  if (mine.size() > kText) poas::fail(poas::errc::invalid_argument, "comm allgather: text over 64 KiB");
  std::memcpy(sh_->text[rank_], mine.data(), mine.size());
  __atomic_store_n(&sh_->text_len[rank_], static_cast<int>(mine.size()), __ATOMIC_SEQ_CST);
  barrier();
  std::vector<std::string> out(static_cast<std::size_t>(world_));
  for (int r = 0; r < world_; ++r)
    out[static_cast<std::size_t>(r)].assign(
        sh_->text[r], static_cast<std::size_t>(__atomic_load_n(&sh_->text_len[r], __ATOMIC_SEQ_CST)));
  barrier();  // nobody overwrites a slot before everyone read it
  return out;
}

double Comm::allreduce_max(double v) {
  sh_->value[rank_] = v;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  barrier();
  double mx = v;
  for (int r = 0; r < world_; ++r) mx = std::max(mx, sh_->value[r]);
  barrier();
  return mx;
}

std::vector<unsigned char> Comm::nccl_unique_id() {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  return std::vector<unsigned char>(reinterpret_cast<unsigned char*>(&id),
                                    reinterpret_cast<unsigned char*>(&id) + sizeof id);
}

void Comm::init_nccl(const void* id, std::size_t bytes) {
  if (device_ < 0) poas::fail(poas::errc::invalid_argument, "init_nccl: host-only comm");
  if (bytes != sizeof(ncclUniqueId)) poas::fail(poas::errc::invalid_argument, "init_nccl: bad id size");
  if (nccl_) return;
  DeviceGuard g(device_);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t c = nullptr;
  nccl_check(nccl().comm_init_rank(&c, world_, uid, rank_), "ncclCommInitRank");
  nccl_ = c;
}

const int* Comm::flag_dev(int r, int p) const { return flags_dev_base_ + r * kMaxPanels + p; }
int* Comm::flag_dev_mut(int r, int p) const { return flags_dev_base_ + r * kMaxPanels + p; }

// Collective: rank 0 serves `own`; the others allocate two receive
// buffers; rank r > 0 maps rank r-1's (by parity) through CUDA IPC.
void Comm::register_set(int slot, const void* own, std::size_t bytes, bool present) {
  DeviceGuard g(device_);
  BufSet& set = sets_[slot];
  Shared::Info& me = sh_->info[rank_];
  std::memset(&me.h[slot], 0, sizeof me.h[slot]);
  me.off[slot][0] = me.off[slot][1] = 0;
  me.has[slot] = present ? 1 : 0;
  set = BufSet{};
  set.bytes = bytes;
  if (present) {
    if (rank_ == 0) {
      set.own = own;
      void* base = alloc_base(own);
      cuda_check(cudaIpcGetMemHandle(&me.h[slot][0], base), "cudaIpcGetMemHandle");
      me.h[slot][1] = me.h[slot][0];
      me.off[slot][0] = me.off[slot][1] =
          static_cast<std::uint64_t>(static_cast<const char*>(own) - static_cast<char*>(base));
    } else {
      for (int q = 0; q < 2; ++q) {
        cuda_check(cudaMalloc(&set.recv[q], bytes), "cudaMalloc broadcast receive buffer");
        cuda_check(cudaIpcGetMemHandle(&me.h[slot][q], set.recv[q]), "cudaIpcGetMemHandle");
      }
    }
  }
  barrier();
  for (int r = 0; r < world_; ++r)
    if (sh_->info[r].has[slot] != me.has[slot])
      poas::fail(poas::errc::invalid_argument, "comm: ranks disagree on a broadcast buffer");
  if (present && rank_ > 0) {
    const Shared::Info& in = sh_->info[rank_ - 1];
    for (int q = 0; q < 2; ++q) {
      if (q == 1 && rank_ - 1 == 0) {  // the root serves one buffer to both parities
        set.up[1] = set.up[0];
        break;
      }
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, in.h[slot][q], cudaIpcMemLazyEnablePeerAccess),
                 "cudaIpcOpenMemHandle");
      set.mapped[q] = p;
      set.up[q] = static_cast<char*>(p) + in.off[slot][q];
    }
  }
  set.active = present;
  cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  barrier();
}

void Comm::release_set(int slot) {
  BufSet& set = sets_[slot];
  for (void* m : set.mapped)
    if (m) cudaIpcCloseMemHandle(m);
  for (void* r : set.recv)
    if (r) cudaFree(r);
  set = BufSet{};
}

void Comm::register_b(const void* b16, const void* b32, std::int64_t k, std::int64_t n, int panels) {
  if (device_ < 0) poas::fail(poas::errc::invalid_argument, "register_b: host-only comm");
  if (panels < 1 || panels > kMaxPanels || n % panels != 0 || k < 1)
    poas::fail(poas::errc::invalid_argument, "register_b: bad panel split");
  if (!b16) poas::fail(poas::errc::invalid_argument, "register_b: b16 is required");
  if (panels_ > 0) poas::fail(poas::errc::invalid_argument, "register_b: B already registered");
  const std::size_t bytes16 = static_cast<std::size_t>(k) * static_cast<std::size_t>(n) * 2;
  register_set(0, b16, bytes16, true);
  register_set(1, b32, bytes16 * 2, b32 != nullptr);
  k_ = k;
  n_ = n;
  panels_ = panels;
}

void* Comm::dst(int slot, int epoch) const {
  const BufSet& s = sets_[slot];
  return rank_ == 0 ? const_cast<void*>(s.own) : s.recv[epoch & 1];
}

const void* Comm::b16_for(int epoch) const { return dst(0, epoch); }
const float* Comm::b32_for(int epoch) const { return static_cast<const float*>(dst(1, epoch)); }

void Comm::consumed(int epoch, cudaStream_t s) {
  DeviceGuard g(device_);
  cudaEvent_t e = nullptr;
  cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
  consumed_[epoch & 1].push_back(e);
}

void Comm::enqueue_sets(Transport t, int epoch, const std::vector<int>& slots, int panels) {
  const int q = epoch & 1;
  if (t == Transport::nccl && !nccl_) poas::fail(poas::errc::invalid_argument, "transport nccl: init_nccl first");
  // the epoch whose contents the downstream rank last pulled from these
  // receive buffers (it ran the same operation then, with the same panels)
  int prev = 0;
  for (int slot : slots) prev = std::max(prev, sets_[slot].last[q]);
  for (int slot : slots) sets_[slot].last[q] = epoch;
  for (int p = 0; p < panels; ++p) {
    if (t == Transport::nccl) {
      for (int slot : slots) {
        const std::size_t pb = sets_[slot].bytes / static_cast<std::size_t>(panels);
        char* d = static_cast<char*>(dst(slot, epoch)) + p * pb;
        nccl_check(nccl().broadcast(d, d, pb, ncclUint8, 0, static_cast<ncclComm_t>(nccl_), stream_),
                   "ncclBroadcast");
      }
    } else if (rank_ > 0) {
      cuda_check(wait_flag(flag_dev(rank_ - 1, p), epoch, stream_), "wait upstream panel");
      // the downstream rank finished pulling this buffer's previous contents
      if (rank_ + 1 < world_ && prev > 0)
        cuda_check(wait_flag(flag_dev(rank_ + 1, p), prev, stream_), "wait downstream panel");
      for (int slot : slots) {
        const std::size_t pb = sets_[slot].bytes / static_cast<std::size_t>(panels);
        cuda_check(cudaMemcpyAsync(static_cast<char*>(dst(slot, epoch)) + p * pb,
                                   static_cast<const char*>(sets_[slot].up[q]) + p * pb, pb,
                                   cudaMemcpyDeviceToDevice, stream_),
                   "peer copy of a B panel");
      }
    }
    cuda_check(signal_flag(flag_dev_mut(rank_, p), epoch, stream_), "signal panel (peers)");
    cuda_check(signal_flag(dev_flags_ + p, epoch, stream_), "signal panel (local GEMM)");
    cuda_check(cudaEventRecord(events_[static_cast<std::size_t>(p)], stream_), "cudaEventRecord");
  }
}

int Comm::enqueue_broadcast(Transport t, bool with_b32, const std::vector<cudaEvent_t>& after) {
  if (!registered()) poas::fail(poas::errc::invalid_argument, "broadcast: register_b first");
  DeviceGuard g(device_);
  const int epoch = ++epoch_;
  for (cudaEvent_t e : after) cuda_check(cudaStreamWaitEvent(stream_, e, 0), "cudaStreamWaitEvent");
  // the GEMMs that read this parity's buffers two epochs ago are done
  for (cudaEvent_t e : consumed_[epoch & 1]) {
    cuda_check(cudaStreamWaitEvent(stream_, e, 0), "cudaStreamWaitEvent");
    cudaEventDestroy(e);  // released once it has completed
  }
  consumed_[epoch & 1].clear();
  std::vector<int> slots{0};
  if (with_b32 && sets_[1].active) slots.push_back(1);
  enqueue_sets(t, epoch, slots, panels_);
  return epoch;
}

double Comm::time_broadcast(Transport t, std::uint64_t bytes, int reps) {
  if (device_ < 0) poas::fail(poas::errc::invalid_argument, "time_broadcast: host-only comm");
  if (bytes < (1ULL << 20) || reps < 1) poas::fail(poas::errc::invalid_argument, "time_broadcast: bad size");
  DeviceGuard g(device_);
  const int P = 16;
  const std::size_t b = static_cast<std::size_t>((bytes + P * 256 - 1) / (P * 256) * (P * 256));
  void* own = nullptr;
  if (rank_ == 0) {
    cuda_check(cudaMalloc(&own, b), "cudaMalloc probe");
    cuda_check(cudaMemset(own, 0, b), "cudaMemset probe");
  }
  register_set(2, own, b, true);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cuda_check(cudaEventCreate(&e0), "cudaEventCreate");
  cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
  double sum = 0.0;
  for (int r = 0; r < reps; ++r) {
    cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
    barrier();
    const int epoch = ++epoch_;
    cuda_check(cudaEventRecord(e0, stream_), "cudaEventRecord");
    enqueue_sets(t, epoch, {2}, P);
    cuda_check(cudaEventRecord(e1, stream_), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
    float ms = 0.0f;
    cuda_check(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    sum += allreduce_max(static_cast<double>(ms) * 1e-3);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  barrier();  // nobody still pulls from a probe buffer
  release_set(2);
  if (own) cudaFree(own);
  return sum / reps;
}

}  // namespace poas_b200
