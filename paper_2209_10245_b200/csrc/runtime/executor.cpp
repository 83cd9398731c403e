// The co-execution engine: runs a schedule's shares concurrently on real
// units and measures every phase (replaces the reference's discrete-event
// simulate(), proj/src/simulator.cpp:104-209, with the same result shape).
//
// Per repeat:
//   gate        the repeat is enqueued behind a one-thread kernel that waits
//               for a host flag; the flag is set once everything is queued,
//               so enqueue latency is not measured as GPU phase time
//   t0          one event per GPU after the gate (on every unit stream's
//               critical path) and a host steady_clock stamp when the gate
//               opens: the common clock origin
//   chaining    GPU-only repeats follow each other on the device (t0 of
//               repeat r waits for repeat r-1's last events), no host sync;
//               with host-CPU units every repeat is host-synchronous
//   cpu unit    a host thread runs host_gemm on its rows from t0
//   copy-in     GPU units in schedule (priority) order; on a shared bus each
//               copy-in waits for the previous unit's copy-in (link order)
//   compute     right after the unit's own copy-in, on its SM budget
//   copy-out    schedule order; the first waits for the last copy-in, each
//               later one for the previous copy-out (shared bus)
// Resident runs (operands already in HBM) skip both copy phases.
// Overlapped host runs ("overlap=1", poas/overlap.hpp): each link unit has
// its own host->device and device->host streams; its A row parts and B
// column panels go host->device interleaved, each block (part x panel) is
// computed once both landed, and its C goes device->host while later blocks
// compute. On a shared bus each direction is served in schedule order.
// Rows are contiguous in schedule order (poas::row_offsets).
#include "poas/executor.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <thread>

#include "capi_util.hpp"
#include "comm.hpp"
#include "poas/error.hpp"
#include "poas/overlap.hpp"
#include "units.hpp"

namespace poas {

using poas_b200::AbType;
using poas_b200::DeviceGuard;
using poas_b200::Unit;
using poas_b200::capi::cuda_check;

double rel_err_pct(double measured, double predicted) {
  if (measured == 0.0 && predicted == 0.0) return 0.0;
  return 100.0 * (measured - predicted) / measured;
}

namespace {

double rms(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s / static_cast<double>(v.size()));
}

std::int64_t round_up(std::int64_t x, std::int64_t a) { return (x + a - 1) / a * a; }

struct PhaseEvents {
  cudaEvent_t ci0 = nullptr, ci1 = nullptr, cp0 = nullptr, cp1 = nullptr, co0 = nullptr,
              co1 = nullptr;
  void create() {
    for (cudaEvent_t* e : {&ci0, &ci1, &cp0, &cp1, &co0, &co1})
      if (!*e) cuda_check(cudaEventCreate(e), "cudaEventCreate");
  }
  void destroy() {
    for (cudaEvent_t* e : {&ci0, &ci1, &cp0, &cp1, &co0, &co1})
      if (*e) cudaEventDestroy(*e);
  }
};

void copy2d(void* dst, std::int64_t ld_dst, const void* src, std::int64_t ld_src,
            std::int64_t rows, std::int64_t cols, std::size_t esz, cudaMemcpyKind kind,
            cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return;
  if (ld_dst == cols && ld_src == cols)
    cuda_check(cudaMemcpyAsync(dst, src, static_cast<std::size_t>(rows * cols) * esz, kind, s),
               "cudaMemcpyAsync");
  else
    cuda_check(cudaMemcpy2DAsync(dst, static_cast<std::size_t>(ld_dst) * esz, src,
                                 static_cast<std::size_t>(ld_src) * esz,
                                 static_cast<std::size_t>(cols) * esz,
                                 static_cast<std::size_t>(rows), kind, s),
               "cudaMemcpy2DAsync");
}

// Untimed events of one run(), destroyed with it.
class EventPool {
 public:
  EventPool() = default;
  ~EventPool() {
    for (auto& [dev, e] : events_) {
      DeviceGuard g(dev);
      cudaEventDestroy(e);
    }
  }
  EventPool(const EventPool&) = delete;
  EventPool& operator=(const EventPool&) = delete;
  cudaEvent_t make(int dev) {
    DeviceGuard g(dev);
    cudaEvent_t e = nullptr;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    events_.emplace_back(dev, e);
    return e;
  }

 private:
  std::vector<std::pair<int, cudaEvent_t>> events_;
};

// The start gates of one run() (see gate_wait): flag r opens repeat r.
// Every flag is opened on destruction, so an exception between a gate's
// launch and its opening cannot leave a kernel waiting.
class StartGates {
 public:
  StartGates(int repeats, Executor::GateBuffer* buf) : buf_(buf), n_(repeats) {
    if (repeats <= 0) return;
    const std::size_t need = static_cast<std::size_t>(repeats);
    if (buf->capacity < need) {
      void* p = nullptr;
      cuda_check(cudaHostAlloc(&p, need * sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable),
                 "cudaHostAlloc");
      if (buf->host) buf->retired.push_back(buf->host);  // freed with the executor
      buf->host = static_cast<int*>(p);
      buf->capacity = need;
    }
    for (int r = 0; r < repeats; ++r) __atomic_store_n(buf->host + r, 0, __ATOMIC_SEQ_CST);
    void* dp = nullptr;
    cuda_check(cudaHostGetDevicePointer(&dp, buf->host, 0), "cudaHostGetDevicePointer");
    dev_ = static_cast<const int*>(dp);
  }
  ~StartGates() {
    for (int r = 0; r < n_; ++r) open(r);
  }
  StartGates(const StartGates&) = delete;
  StartGates& operator=(const StartGates&) = delete;
  const int* device_flag(int r) const { return dev_ + r; }
  void open(int r) {
    if (r < n_) __atomic_store_n(buf_->host + r, 1, __ATOMIC_SEQ_CST);
  }

 private:
  Executor::GateBuffer* buf_;
  int n_;
  const int* dev_ = nullptr;
};

// Page-locks pageable host operand ranges for the duration of one run()
// (pinned memory -- cudaHostAlloc or registered -- is left alone). Without
// it an async copy to or from pageable memory would block the enqueueing
// thread until the copy ran, i.e. until a start gate it is queued behind
// opened -- which only that thread can do.
class HostPins {
 public:
  HostPins() = default;
  ~HostPins() {
    if (regs_.empty()) return;
    cudaDeviceSynchronize();  // nothing in flight may still read them
    for (void* p : regs_) cudaHostUnregister(p);
  }
  HostPins(const HostPins&) = delete;
  HostPins& operator=(const HostPins&) = delete;
  void ensure(const void* p, std::size_t bytes) {
    if (!p || bytes == 0) return;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      at.type = cudaMemoryTypeUnregistered;
    }
    if (at.type != cudaMemoryTypeUnregistered) return;
    void* q = const_cast<void*>(p);
    for (void* r : regs_)
      if (r == q) return;
    const cudaError_t e = cudaHostRegister(q, bytes, cudaHostRegisterPortable);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {  // shares pages with one registered above
      cudaGetLastError();
      return;
    }
    cuda_check(e, "cudaHostRegister (pageable host operand)");
    regs_.push_back(q);
  }

 private:
  std::vector<void*> regs_;
};

}  // namespace

Executor::Executor(const std::string& spec) {
  const std::vector<poas_b200::UnitSpec> specs =
      poas_b200::parse_unit_list(spec, &bus_, &lend_, &overlap_, &pipeline_);
  std::vector<DeviceIdentity> ids;
  for (const auto& s : specs) {
    if (find(s.id)) fail(errc::invalid_argument, "duplicate unit id '" + s.id + "'");
    units_.push_back(std::make_unique<Unit>(s));
    ids.push_back({s.id, s.kind, s.elem});
  }
  hash_ = machine_identity_hash(ids, bus_);
  h2d_.assign(units_.size(), nullptr);
  d2h_.assign(units_.size(), nullptr);
  if (overlap_)
    for (std::size_t i = 0; i < units_.size(); ++i) {
      if (!units_[i]->on_gpu()) continue;
      DeviceGuard g(units_[i]->spec().device);
      cudaStream_t a = nullptr, b = nullptr;
      cuda_check(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "cudaStreamCreate");
      h2d_[i] = a;
      cuda_check(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "cudaStreamCreate");
      d2h_[i] = b;
    }
}

void Executor::release_graph(RepeatGraph& g) {
  DeviceGuard dg(g.device);
  if (g.exec) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g.exec));
  if (g.graph) cudaGraphDestroy(static_cast<cudaGraph_t>(g.graph));
  for (void* e : g.events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  g = RepeatGraph{};
}

Executor::~Executor() {
  for (auto& gr : graphs_) release_graph(*gr);
  for (std::size_t i = 0; i < units_.size(); ++i)
    for (void* s : {h2d_[i], d2h_[i]})
      if (s) {
        DeviceGuard g(units_[i]->spec().device);
        cudaStreamDestroy(static_cast<cudaStream_t>(s));
      }
  if (gates_.host) cudaFreeHost(gates_.host);
  for (int* p : gates_.retired) cudaFreeHost(p);
}

Unit* Executor::find(const std::string& id) const {
  for (const auto& u : units_)
    if (u->spec().id == id) return u.get();
  return nullptr;
}

SimulationResult Executor::run(const Schedule& schedule, const GemmOperands& io, int repeats) {
  if (repeats < 1) fail(errc::invalid_argument, "repeats must be positive");
  if (schedule.devices.empty()) fail(errc::invalid_argument, "schedule has no devices");
  if (schedule.machine_hash != hash_)
    fail(errc::hash_mismatch, "schedule was planned for machine " + schedule.machine_hash +
                                  ", executor units describe " + hash_);
  const MatrixDims& d = schedule.dims;
  if (io.m != d.m || io.n != d.n || io.k != d.k)
    fail(errc::invalid_argument, "operand dims do not match the schedule dims");

  const std::size_t nd = schedule.devices.size();
  std::vector<Unit*> unit(nd);
  std::vector<cudaStream_t> h2d(nd, nullptr), d2h(nd, nullptr);  // overlapped runs
  std::int64_t covered = 0;
  for (std::size_t i = 0; i < nd; ++i) {
    unit[i] = find(schedule.devices[i].id);
    if (!unit[i]) fail(errc::missing_device, "no unit '" + schedule.devices[i].id + "'");
    covered += schedule.devices[i].rows;
    for (std::size_t j = 0; j < units_.size(); ++j)
      if (units_[j].get() == unit[i]) {
        h2d[i] = static_cast<cudaStream_t>(h2d_[j]);
        d2h[i] = static_cast<cudaStream_t>(d2h_[j]);
      }
  }
  if (covered != d.m) fail(errc::invalid_argument, "schedule rows do not cover m");
  const std::vector<std::int64_t> row0 = row_offsets(schedule);

  // Operand availability checks, up front (no partial launches).
  bool any_cpu = false;
  for (std::size_t i = 0; i < nd; ++i) {
    if (schedule.devices[i].rows == 0) continue;
    if (!unit[i]->on_gpu()) any_cpu = true;
  }
  // A tensor unit with a 2-byte link reads 16-bit host operands when given.
  const auto host16_link = [&](const Unit* u) {
    return u->spec().kind == DeviceKind::xpu && u->spec().elem == 2 && io.a16_host && io.b16_host;
  };
  if ((any_cpu || !io.resident) && !io.c_host)
    fail(errc::invalid_argument, "host operand c_host is required");
  for (std::size_t i = 0; i < nd; ++i) {
    if (schedule.devices[i].rows == 0) continue;
    const bool needs_f32_host = !unit[i]->on_gpu() || (!io.resident && !host16_link(unit[i]));
    if (needs_f32_host && (!io.a_host || !io.b_host))
      fail(errc::invalid_argument, "host operands (a_host, b_host, c_host) are required");
  }
  const int panels = io.b_panels > 1 ? io.b_panels : 1;
  poas_b200::Comm* const comm = io.comm;
  const poas_b200::Transport transport =
      io.b_transport == 1 ? poas_b200::Transport::nccl : poas_b200::Transport::ce;
  if (comm) {
    if (!io.resident) fail(errc::invalid_argument, "a comm (B broadcast) needs resident operands");
    if (!comm->registered() || comm->panels() != panels)
      fail(errc::invalid_argument, "comm: register B with the same panel count as b_panels first");
    if (io.b_flags || io.b_ready)
      fail(errc::invalid_argument, "comm: the executor signals B itself (no b_flags / b_ready)");
    for (std::size_t i = 0; i < nd; ++i)
      if (schedule.devices[i].rows > 0 && unit[i]->on_gpu() && unit[i]->spec().device != comm->device())
        fail(errc::invalid_argument, "comm: every busy GPU unit must be on the comm's GPU");
  }
  if (panels > 1) {
    if (!io.resident) fail(errc::invalid_argument, "B panels need resident operands");
    if (d.n % panels != 0 || (d.n / panels) % 8 != 0)
      fail(errc::invalid_argument, "n must split into b_panels panels of a multiple of 8 columns");
    for (std::size_t i = 0; i < nd; ++i)
      if (schedule.devices[i].rows > 0 && unit[i]->spec().kind == DeviceKind::xpu &&
          !(io.a16_dev && io.b16_dev))
        fail(errc::invalid_argument, "B panels with a tensor unit need a16/b16 operands");
  }
  if (io.resident) {
    for (std::size_t i = 0; i < nd; ++i) {
      if (schedule.devices[i].rows == 0 || !unit[i]->on_gpu()) continue;
      if (!io.c_dev) fail(errc::invalid_argument, "resident run needs c_dev");
      const bool tensor = unit[i]->spec().kind == DeviceKind::xpu;
      if (tensor && !(io.a16_dev && io.b16_dev) && !(io.a_dev && io.b_dev))
        fail(errc::invalid_argument, "resident tensor unit needs a16/b16 or a/b device operands");
      if (!tensor && !(io.a_dev && io.b_dev))
        fail(errc::invalid_argument, "resident CUDA-core unit needs a_dev/b_dev");
    }
  }

  // Overlapped host runs: every busy link unit pipelines its row parts.
  const bool overlapped = overlap_ && !io.resident;

  // SM lending: when exactly one unit of a GPU has rows in this schedule,
  // the SM budgets of its idle siblings are added to its launch (the plan
  // left them nothing to do; a static partition would leave them dark).
  // Not while B arrives through readiness events: the idle SMs are where
  // the collective's kernels run concurrently with the GEMM.
  std::vector<int> extra_sms(nd, 0);
  // (copy-engine broadcasts need no SMs; NCCL's kernels do)
  if (lend_ && !io.b_ready && !io.b_flags && !(comm && transport == poas_b200::Transport::nccl)) {
    std::map<int, std::vector<std::size_t>> by_dev;
    for (std::size_t i = 0; i < nd; ++i)
      if (unit[i]->on_gpu()) by_dev[unit[i]->spec().device].push_back(i);
    for (const auto& [dev, idx] : by_dev) {
      std::size_t busy = nd;
      int busy_count = 0, idle_sms = 0;
      bool budgets = true;
      for (std::size_t i : idx) {
        budgets = budgets && unit[i]->spec().sms > 0;
        if (schedule.devices[i].rows > 0) {
          busy = i;
          ++busy_count;
        } else {
          idle_sms += unit[i]->spec().sms;
        }
      }
      if (budgets && busy_count == 1) extra_sms[busy] = idle_sms;
    }
  }

  // Per GPU with work: its first busy unit (schedule order) hosts the start
  // gate and t0 on its own stream; other busy units of that GPU wait on t0.
  std::map<int, std::size_t> host_unit;
  for (std::size_t i = 0; i < nd; ++i)
    if (unit[i]->on_gpu() && schedule.devices[i].rows > 0 && !host_unit.count(unit[i]->spec().device))
      host_unit[unit[i]->spec().device] = i;

  // Events: per repeat, one t0 per GPU and one phase set per busy GPU unit;
  // one entry event per GPU (orders the run after work already queued on the
  // legacy default stream, e.g. the caller's input preparation).
  std::map<int, std::vector<cudaEvent_t>> t0;  // device -> [repeat]
  std::map<int, cudaEvent_t> entry;
  std::vector<std::vector<PhaseEvents>> ev(static_cast<std::size_t>(repeats),
                                           std::vector<PhaseEvents>(nd));
  struct Cleanup {
    std::map<int, std::vector<cudaEvent_t>>& t0;
    std::map<int, cudaEvent_t>& entry;
    std::vector<std::vector<PhaseEvents>>& ev;
    std::vector<Unit*>& unit;
    bool borrowed = false;  // graph replay: t0 / cp0 / cp1 belong to the cached graph
    ~Cleanup() {
      for (auto& per_rep : ev)
        for (std::size_t i = 0; i < per_rep.size(); ++i) {
          if (!unit[i]->on_gpu()) continue;
          DeviceGuard g(unit[i]->spec().device);
          if (borrowed) per_rep[i].cp0 = per_rep[i].cp1 = nullptr;
          per_rep[i].destroy();
        }
      for (auto& [dev, v] : t0) {
        DeviceGuard g(dev);
        if (!borrowed)
          for (cudaEvent_t e : v)
            if (e) cudaEventDestroy(e);
        if (entry.count(dev) && entry[dev]) cudaEventDestroy(entry[dev]);
      }
    }
  } cleanup{t0, entry, ev, unit};
  for (const auto& [dev, h] : host_unit) {
    DeviceGuard g(dev);
    std::vector<cudaEvent_t>& v = t0[dev];
    v.assign(static_cast<std::size_t>(repeats), nullptr);
    for (cudaEvent_t& e : v) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    entry[dev] = nullptr;
    cuda_check(cudaEventCreateWithFlags(&entry[dev], cudaEventDisableTiming), "cudaEventCreate");
  }
  for (std::size_t i = 0; i < nd; ++i) {
    if (!unit[i]->on_gpu() || schedule.devices[i].rows == 0) continue;
    DeviceGuard g(unit[i]->spec().device);
    for (auto& per_rep : ev) per_rep[i].create();
  }
  // Overlapped runs: each busy link unit's grid of row parts x column panels
  // (the schedule's tiles, poas::schedule_grid), its link order and block
  // order (poas/overlap.hpp), and readiness events per link item and per
  // block, reused by every repeat (repeats are serialised on the device).
  EventPool pool;
  std::vector<RowColGrid> grid(nd);
  std::vector<std::vector<OverlapItem>> link_order(nd);
  std::vector<std::vector<OverlapBlock>> block_order(nd);
  std::vector<std::vector<cudaEvent_t>> in_ev(nd), cp_ev(nd);
  if (overlapped)
    for (std::size_t i = 0; i < nd; ++i) {
      if (!unit[i]->on_gpu() || schedule.devices[i].rows == 0) continue;
      if (!h2d[i] || !d2h[i]) fail(errc::invalid_argument, "overlap: unit has no copy streams");
      grid[i] = schedule_grid(schedule.devices[i], d);
      const int R = static_cast<int>(grid[i].parts.size()), Q = static_cast<int>(grid[i].panels.size());
      link_order[i] = overlap_link_order(R, Q);
      block_order[i] = overlap_block_order(R, Q);
      for (std::size_t k = 0; k < link_order[i].size(); ++k)
        in_ev[i].push_back(pool.make(unit[i]->spec().device));
      for (std::size_t b = 0; b < block_order[i].size(); ++b)
        cp_ev[i].push_back(pool.make(unit[i]->spec().device));
    }
  // A tensor unit with a 16-bit link streams its grid through ONE launch
  // (tc_gemm_stream): the H2D stream flags each link item as it lands, the
  // persistent kernel's producers wait for their block's two items, the
  // epilogue flags each finished block and the D2H stream waits on those
  // flags (cuStreamWaitValue32) -- no per-block launches, every SM busy on
  // whatever blocks are ready. Needs the pair kernel and 256-aligned parts
  // and panels (a tile never straddles two link items).
  struct StreamState {
    int* item_flags = nullptr;
    int* block_count = nullptr;
    int* block_flags = nullptr;
    int* blocks = nullptr;
    cudaEvent_t ready = nullptr;
  };
  std::vector<StreamState> sstate(nd);
  const auto aligned256 = [](const std::vector<std::int64_t>& v) {
    for (std::size_t x = 0; x + 1 < v.size(); ++x)
      if (v[x] % 256) return false;
    return true;
  };
  if (overlapped)
    for (std::size_t i = 0; i < nd; ++i) {
      Unit* u = unit[i];
      if (!u->on_gpu() || schedule.devices[i].rows == 0) continue;
      if (u->spec().kind != DeviceKind::xpu || !host16_link(u)) continue;
      if (const char* kv = std::getenv("POAS_TC_KERNEL"))  // a forced single-SM variant
        if (std::string(kv) != "2cta") continue;
      if (!aligned256(grid[i].parts) || !aligned256(grid[i].panels)) continue;
      // the pair kernel needs >= 2 SMs (one CTA pair); a 1-SM budget runs
      // the single-SM kernel, which has no block flags
      if (u->spec().sms == 1 && extra_sms[i] == 0) continue;
      if (link_order[i].size() > 128 || block_order[i].size() > 4096) continue;
      DeviceGuard g(u->spec().device);
      const std::size_t ni = link_order[i].size(), nb = block_order[i].size();
      std::vector<int> item_a(grid[i].parts.size()), item_b(grid[i].panels.size());
      for (std::size_t k = 0; k < ni; ++k)
        (link_order[i][k].a ? item_a : item_b)[static_cast<std::size_t>(link_order[i][k].index)] =
            static_cast<int>(k);
      std::vector<std::int64_t> roff(grid[i].parts.size(), 0), coff(grid[i].panels.size(), 0);
      for (std::size_t x = 1; x < roff.size(); ++x) roff[x] = roff[x - 1] + grid[i].parts[x - 1];
      for (std::size_t x = 1; x < coff.size(); ++x) coff[x] = coff[x - 1] + grid[i].panels[x - 1];
      std::vector<int> table(4 * nb);
      int first = 0;
      for (std::size_t b = 0; b < nb; ++b) {
        const std::size_t pp = static_cast<std::size_t>(block_order[i][b].part);
        const std::size_t qq = static_cast<std::size_t>(block_order[i][b].panel);
        const int tm = static_cast<int>((grid[i].parts[pp] + 255) / 256);
        const int tn = static_cast<int>((grid[i].panels[qq] + 255) / 256);
        table[4 * b] = static_cast<int>(roff[pp] / 256) | (tm << 16);
        table[4 * b + 1] = static_cast<int>(coff[qq] / 256) | (tn << 16);
        table[4 * b + 2] = first;
        table[4 * b + 3] = item_a[pp] | (item_b[qq] << 16);
        first += tm * tn;
      }
      // block table first: the kernel reads it as int4 (16-byte aligned)
      const std::size_t ints = 4 * nb + ni + 2 * nb;
      int* base = static_cast<int*>(u->scratch(5).ensure(ints * sizeof(int)));
      StreamState& st = sstate[i];
      st.blocks = base;
      st.item_flags = base + 4 * nb;
      st.block_count = st.item_flags + ni;
      st.block_flags = st.block_count + nb;
      cudaStream_t cs = u->stream();
      cuda_check(cudaMemsetAsync(st.item_flags, 0, (ni + 2 * nb) * sizeof(int), cs), "cudaMemsetAsync");
      cuda_check(cudaMemcpyAsync(st.blocks, table.data(), table.size() * sizeof(int),
                                 cudaMemcpyHostToDevice, cs),
                 "cudaMemcpyAsync");
      st.ready = pool.make(u->spec().device);
      cuda_check(cudaEventRecord(st.ready, cs), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(h2d[i], st.ready, 0), "wait stream setup");
      cuda_check(cudaStreamWaitEvent(d2h[i], st.ready, 0), "wait stream setup");
    }
  // Pipelined repeats (units token "pipeline=1"): one busy GPU unit on the
  // streamed path, no host-CPU unit. Repeat r+1 is queued behind repeat r's
  // GEMM only (its gate sits on the compute stream after that launch), not
  // behind r's copy-out: its host->device copies run beside r's
  // device->host tail. A and B staging are free again once r's GEMM is
  // done; C is double-buffered (r+1 writes one buffer while r's copy-out
  // reads the other; r+2 waits for r's copy-out).
  std::size_t busy_gpu_units = 0, busy_unit = nd;
  for (std::size_t i = 0; i < nd; ++i)
    if (unit[i]->on_gpu() && schedule.devices[i].rows > 0) {
      ++busy_gpu_units;
      busy_unit = i;
    }
  const bool pipelined = overlapped && pipeline_ && !any_cpu && busy_gpu_units == 1 &&
                         sstate[busy_unit].item_flags != nullptr;
  // POAS_EXEC_PIPE_STAGING=1: one A / B staging set (each repeat's copy-in
  // waits for the previous repeat's start gate, i.e. its GEMM's end)
  const char* pipe_env = std::getenv("POAS_EXEC_PIPE_STAGING");
  const bool two_sets = pipelined && !(pipe_env && std::string(pipe_env) == "1");
  if (pipelined && repeats > 1) {  // the second C / A / B buffers, before any repeat is queued
    DeviceGuard g(unit[busy_unit]->spec().device);
    const std::int64_t r = schedule.devices[busy_unit].rows;
    unit[busy_unit]->scratch(6).ensure(static_cast<std::size_t>(r * d.n) * 4);
    unit[busy_unit]->scratch(7).ensure(static_cast<std::size_t>(r * round_up(d.k, 8)) * 2);
    unit[busy_unit]->scratch(8).ensure(static_cast<std::size_t>(d.k * round_up(d.n, 8)) * 2);
  }

  // One repeat of an overlapped link unit: host->device (A parts and B
  // panels interleaved in link order), one GEMM per block as soon as its A
  // part and B panel landed, each block's C device->host as soon as it is
  // computed; `prev_in`/`prev_out` are the previous busy link unit in
  // schedule order (shared-bus order).
  const auto enqueue_overlapped = [&](std::size_t i, std::size_t rr, std::size_t prev_in,
                                      std::size_t prev_out) {
    const ScheduledDevice& sd = schedule.devices[i];
    Unit* u = unit[i];
    PhaseEvents& e = ev[rr][i];
    cudaStream_t cs = u->stream(), hs = h2d[i], ds = d2h[i];
    const bool tensor = u->spec().kind == DeviceKind::xpu;
    const bool link16 = tensor && host16_link(u);
    const bool convert = tensor && !link16;
    const std::int64_t r = sd.rows, r0 = row0[i];
    const std::size_t esz = link16 ? 2 : 4;
    const std::int64_t lda_l = link16 ? round_up(d.k, 8) : d.k;
    const std::int64_t ldb_l = link16 ? round_up(d.n, 8) : d.n;
    // pipelined (16-bit link, one streamed launch per repeat): odd repeats
    // land their A / B in a second staging set, so a repeat's copy-in runs
    // while the previous repeat still computes on the first
    const bool second = two_sets && link16 && (rr & 1) && sstate[i].item_flags;
    char* a_l = static_cast<char*>(
        u->scratch(second ? 7 : (link16 ? 2 : 0)).ensure(static_cast<std::size_t>(r * lda_l) * esz));
    char* b_l = static_cast<char*>(
        u->scratch(second ? 8 : (link16 ? 3 : 1)).ensure(static_cast<std::size_t>(d.k * ldb_l) * esz));
    float* c = static_cast<float*>(u->scratch(4).ensure(static_cast<std::size_t>(r * d.n) * 4));
    const std::vector<std::int64_t>& rp = grid[i].parts;
    const std::vector<std::int64_t>& cp = grid[i].panels;
    std::vector<std::int64_t> roff(rp.size(), 0), coff(cp.size(), 0);
    for (std::size_t p = 1; p < rp.size(); ++p) roff[p] = roff[p - 1] + rp[p - 1];
    for (std::size_t q = 1; q < cp.size(); ++q) coff[q] = coff[q - 1] + cp[q - 1];

    // host -> device: after this repeat's start -- or, pipelined with two
    // staging sets, once the repeat that last used this set has computed
    // (its GEMM read it), without waiting for the previous repeat
    if (two_sets && link16 && sstate[i].item_flags && rr >= 1) {
      if (rr >= 2) cuda_check(cudaStreamWaitEvent(hs, ev[rr - 2][i].cp1, 0), "wait staging set");
    } else {
      cuda_check(cudaStreamWaitEvent(hs, t0[u->spec().device][rr], 0), "wait t0");
    }
    if (bus_ && prev_in != nd) cuda_check(cudaStreamWaitEvent(hs, ev[rr][prev_in].ci1, 0), "wait");
    cuda_check(cudaEventRecord(e.ci0, hs), "cudaEventRecord");
    for (std::size_t k = 0; k < link_order[i].size(); ++k) {
      const OverlapItem& it = link_order[i][k];
      const std::size_t x = static_cast<std::size_t>(it.index);
      if (it.a) {
        if (link16)
          copy2d(a_l + roff[x] * lda_l * 2, lda_l,
                 static_cast<const char*>(io.a16_host) + (r0 + roff[x]) * io.lda16_host * 2,
                 io.lda16_host, rp[x], d.k, 2, cudaMemcpyHostToDevice, hs);
        else
          copy2d(a_l + roff[x] * lda_l * 4, lda_l, io.a_host + (r0 + roff[x]) * io.lda_host,
                 io.lda_host, rp[x], d.k, 4, cudaMemcpyHostToDevice, hs);
      } else {
        if (link16)
          copy2d(b_l + coff[x] * 2, ldb_l, static_cast<const char*>(io.b16_host) + coff[x] * 2,
                 io.ldb16_host, d.k, cp[x], 2, cudaMemcpyHostToDevice, hs);
        else
          copy2d(b_l + coff[x] * 4, ldb_l, io.b_host + coff[x], io.ldb_host, d.k, cp[x], 4,
                 cudaMemcpyHostToDevice, hs);
      }
      cuda_check(cudaEventRecord(in_ev[i][k], hs), "cudaEventRecord");
      if (sstate[i].item_flags)
        cuda_check(poas_b200::signal_flag(sstate[i].item_flags + k, static_cast<int>(rr) + 1, hs),
                   "signal item");
    }
    cuda_check(cudaEventRecord(e.ci1, hs), "cudaEventRecord");

    if (sstate[i].item_flags) {  // one streamed launch; copy-out on block flags
      const StreamState& st = sstate[i];
      const int epoch = static_cast<int>(rr) + 1;
      float* cb = c;  // pipelined: odd repeats write the second C buffer
      if (pipelined && (rr & 1))
        cb = static_cast<float*>(u->scratch(6).ensure(static_cast<std::size_t>(r * d.n) * 4));
      if (pipelined && rr >= 2)  // that buffer's previous copy-out is done
        cuda_check(cudaStreamWaitEvent(cs, ev[rr - 2][i].co1, 0), "wait C buffer");
      cuda_check(cudaEventRecord(e.cp0, cs), "cudaEventRecord");
      poas_b200::TcStream ts;
      ts.blocks = st.blocks;
      ts.nblocks = static_cast<int>(block_order[i].size());
      ts.item_flags = st.item_flags;
      ts.block_count = st.block_count;
      ts.block_flags = st.block_flags;
      ts.epoch = epoch;
      u->gemm_stream(r, d.n, d.k, a_l, lda_l, b_l, ldb_l, cb, d.n, ts, extra_sms[i]);
      cuda_check(cudaEventRecord(e.cp1, cs), "cudaEventRecord");
      if (bus_ && prev_out != nd) cuda_check(cudaStreamWaitEvent(ds, ev[rr][prev_out].co1, 0), "wait");
      for (std::size_t bi = 0; bi < block_order[i].size(); ++bi) {
        const OverlapBlock& blk = block_order[i][bi];
        const std::size_t p = static_cast<std::size_t>(blk.part), q = static_cast<std::size_t>(blk.panel);
        cuda_check(poas_b200::wait_flag(st.block_flags + bi, epoch, ds), "wait block flag");
        if (bi == 0) cuda_check(cudaEventRecord(e.co0, ds), "cudaEventRecord");
        copy2d(io.c_host + (r0 + roff[p]) * io.ldc_host + coff[q], io.ldc_host,
               cb + roff[p] * d.n + coff[q], d.n, rp[p], cp[q], 4, cudaMemcpyDeviceToHost, ds);
      }
      cuda_check(cudaEventRecord(e.co1, ds), "cudaEventRecord");
      return;
    }

    // compute, block by block as their operands land
    const std::int64_t lda16 = round_up(d.k, 8), ldb16 = round_up(d.n, 8);
    char* a16 = convert ? static_cast<char*>(u->scratch(2).ensure(static_cast<std::size_t>(r * lda16) * 2)) : nullptr;
    char* b16 = convert ? static_cast<char*>(u->scratch(3).ensure(static_cast<std::size_t>(d.k * ldb16) * 2)) : nullptr;
    std::vector<char> a_done(rp.size(), 0), b_done(cp.size(), 0);  // converted (fp32 link)
    for (std::size_t bi = 0; bi < block_order[i].size(); ++bi) {
      const OverlapBlock& blk = block_order[i][bi];
      const std::size_t p = static_cast<std::size_t>(blk.part), q = static_cast<std::size_t>(blk.panel);
      cuda_check(cudaStreamWaitEvent(cs, in_ev[i][static_cast<std::size_t>(blk.ready_item)], 0),
                 "wait operands");
      if (bi == 0) cuda_check(cudaEventRecord(e.cp0, cs), "cudaEventRecord");
      const void* ap = a_l + roff[p] * lda_l * static_cast<std::int64_t>(esz);
      const void* bp = b_l + coff[q] * static_cast<std::int64_t>(esz);
      std::int64_t ldak = lda_l, ldbk = ldb_l;
      if (convert) {  // fp32 crossed the link: each part / panel converted once
        if (!a_done[p]) {
          cuda_check(poas_b200::convert_f32(u->spec().dtype, reinterpret_cast<const float*>(ap), lda_l,
                                            a16 + roff[p] * lda16 * 2, lda16, rp[p], d.k, cs),
                     "convert A");
          a_done[p] = 1;
        }
        if (!b_done[q]) {
          cuda_check(poas_b200::convert_f32(u->spec().dtype, reinterpret_cast<const float*>(bp), ldb_l,
                                            b16 + coff[q] * 2, ldb16, d.k, cp[q], cs),
                     "convert B");
          b_done[q] = 1;
        }
        ap = a16 + roff[p] * lda16 * 2;
        bp = b16 + coff[q] * 2;
        ldak = lda16;
        ldbk = ldb16;
      }
      u->gemm(rp[p], cp[q], d.k, ap, ldak, bp, ldbk, c + roff[p] * d.n + coff[q], d.n, false,
              extra_sms[i]);
      cuda_check(cudaEventRecord(cp_ev[i][bi], cs), "cudaEventRecord");
    }
    cuda_check(cudaEventRecord(e.cp1, cs), "cudaEventRecord");

    // device -> host, block by block as they are computed
    if (bus_ && prev_out != nd) cuda_check(cudaStreamWaitEvent(ds, ev[rr][prev_out].co1, 0), "wait");
    for (std::size_t bi = 0; bi < block_order[i].size(); ++bi) {
      const OverlapBlock& blk = block_order[i][bi];
      const std::size_t p = static_cast<std::size_t>(blk.part), q = static_cast<std::size_t>(blk.panel);
      cuda_check(cudaStreamWaitEvent(ds, cp_ev[i][bi], 0), "wait block");
      if (bi == 0) cuda_check(cudaEventRecord(e.co0, ds), "cudaEventRecord");
      copy2d(io.c_host + (r0 + roff[p]) * io.ldc_host + coff[q], io.ldc_host,
             c + roff[p] * d.n + coff[q], d.n, rp[p], cp[q], 4, cudaMemcpyDeviceToHost, ds);
    }
    cuda_check(cudaEventRecord(e.co1, ds), "cudaEventRecord");
  };

  // Resident runs have no copy phases: only compute is bracketed by events.
  const auto last_event = [&](std::size_t rep, std::size_t i) {
    return io.resident ? ev[rep][i].cp1 : ev[rep][i].co1;
  };

  // Nothing inside the enqueue loop below may block on the device while a
  // gate kernel spins on a flag the host has not opened yet:
  // (1) every scratch buffer gets its final size here -- growing one later
  //     calls cudaFree, which synchronizes the device;
  // (2) pageable host operands are page-locked for this run -- a
  //     cudaMemcpyAsync to or from pageable memory returns only after the
  //     copy, i.e. after the gate it is queued behind.
  for (std::size_t i = 0; i < nd; ++i) {
    Unit* u = unit[i];
    const std::int64_t r = schedule.devices[i].rows;
    if (!u->on_gpu() || r == 0) continue;
    DeviceGuard g(u->spec().device);
    const bool tensor = u->spec().kind == DeviceKind::xpu;
    const bool link16 = !io.resident && tensor && host16_link(u);
    const std::int64_t lda16 = round_up(d.k, 8), ldb16 = round_up(d.n, 8);
    const auto sz = [](std::int64_t a, std::int64_t b, std::size_t e) {
      return static_cast<std::size_t>(a) * static_cast<std::size_t>(b) * e;
    };
    if (!io.resident) {
      if (link16) {
        u->scratch(2).ensure(sz(r, lda16, 2));
        u->scratch(3).ensure(sz(d.k, ldb16, 2));
      } else {
        u->scratch(0).ensure(sz(r, d.k, 4));
        u->scratch(1).ensure(sz(d.k, d.n, 4));
      }
      u->scratch(4).ensure(sz(r, d.n, 4));
    }
    if (tensor && !(io.resident && io.a16_dev && io.b16_dev) && !link16) {
      u->scratch(2).ensure(sz(r, lda16, 2));
      u->scratch(3).ensure(sz(d.k, ldb16, 2));
    }
    if (pipelined && repeats > 1 && i == busy_unit) u->scratch(6).ensure(sz(r, d.n, 4));
  }
  HostPins pins;
  if (!io.resident) {
    bool gpu_copies = false;
    for (std::size_t i = 0; i < nd; ++i)
      gpu_copies = gpu_copies || (unit[i]->on_gpu() && schedule.devices[i].rows > 0);
    if (gpu_copies) {
      const auto span = [](std::int64_t rows, std::int64_t ld, std::int64_t cols, std::size_t e) {
        return rows <= 0 ? std::size_t{0}
                         : (static_cast<std::size_t>(rows - 1) * static_cast<std::size_t>(ld) +
                            static_cast<std::size_t>(cols)) * e;
      };
      pins.ensure(io.a_host, span(d.m, io.lda_host, d.k, 4));
      pins.ensure(io.b_host, span(d.k, io.ldb_host, d.n, 4));
      pins.ensure(io.c_host, span(d.m, io.ldc_host, d.n, 4));
      pins.ensure(io.a16_host, span(d.m, io.lda16_host, d.k, 2));
      pins.ensure(io.b16_host, span(d.k, io.ldb16_host, d.n, 2));
    }
  }

  // Start gates: each repeat's GPU work is enqueued behind a tiny kernel
  // that waits for a host flag (gate_wait); t0 is recorded after it, so the
  // host's enqueue latency is not charged to the measured phases.
  StartGates gates(host_unit.empty() ? 0 : repeats, &gates_);

  // Repeats with host threads (CPU units) are host-synchronous: the threads
  // start when the gate opens. GPU-only repeats are chained on the device
  // (the next gate waits for the previous repeat's last events) so the GPU
  // never idles between them.
  const bool host_sync_repeats = any_cpu;
  std::vector<std::vector<double>> cpu_start(static_cast<std::size_t>(repeats),
                                             std::vector<double>(nd, 0.0));
  std::vector<std::vector<double>> cpu_end = cpu_start;
  double sum_wall = 0.0;
  auto quiesce = [&] {
    for (std::size_t i = 0; i < nd; ++i)
      if (unit[i]->on_gpu()) {
        DeviceGuard g(unit[i]->spec().device);
        cuda_check(cudaStreamSynchronize(unit[i]->stream()), "cudaStreamSynchronize");
        for (cudaStream_t x : {h2d[i], d2h[i]})
          if (x) cuda_check(cudaStreamSynchronize(x), "cudaStreamSynchronize");
      }
  };
  std::chrono::steady_clock::time_point first_open;

  for (const auto& [dev, h] : host_unit) {
    DeviceGuard g(dev);
    cuda_check(cudaEventRecord(entry[dev], nullptr), "cudaEventRecord");
    for (std::size_t i = 0; i < nd; ++i)
      if (unit[i]->on_gpu() && schedule.devices[i].rows > 0 && unit[i]->spec().device == dev)
        cuda_check(cudaStreamWaitEvent(unit[i]->stream(), entry[dev], 0), "cudaStreamWaitEvent");
  }

  // ---- CUDA-graph replay. A resident plan with ONE busy unit (a GPU unit,
  // B in place: no delivery events, flags or broadcast) runs a fixed
  // device-side sequence per repeat: the unit's (conversion +) GEMM launch.
  // All `repeats` of them are captured once as one CUDA graph, between a
  // t0 / cp0 record before the first and a cp1 record after the last (on
  // events the graph owns), and launched at once: no start-gate kernel, no
  // per-repeat host enqueue (tensor-map encoding included) pacing a small
  // GEMM, and consecutive GEMMs are kernel-to-kernel edges (no event node
  // between them; programmatic launches overlap a GEMM's prologue with the
  // previous one's tail). Every repeat reports the mean step. The last few graphs
  // (schedule, operands, repeats) are kept for reuse. POAS_EXEC_GRAPH=0
  // turns it off.
  const char* graph_env = std::getenv("POAS_EXEC_GRAPH");
  std::size_t graph_unit = nd;
  for (std::size_t i = 0; i < nd; ++i)
    if (schedule.devices[i].rows > 0) graph_unit = graph_unit == nd ? i : nd + 1;
  int amortized = 1;  // graph replay: events span all repeats (per-repeat = mean)
  const bool graph_mode = io.resident && !any_cpu && !overlapped && !comm && !io.b_flags && !io.b_ready &&
                          panels <= 1 && graph_unit < nd && unit[graph_unit]->on_gpu() && repeats <= 256 &&
                          !(graph_env && std::string(graph_env) == "0");
  if (graph_mode) {
    const std::size_t i = graph_unit;
    Unit* u = unit[i];
    const int dev = u->spec().device;
    DeviceGuard g(dev);
    cudaStream_t s = u->stream();
    char buf[512];
    std::snprintf(buf, sizeof buf, "|%p,%lld|%p,%lld|%p,%lld|%p,%lld|%p,%lld|%d|%d",
                  static_cast<const void*>(io.a_dev), static_cast<long long>(io.lda_dev),
                  static_cast<const void*>(io.b_dev), static_cast<long long>(io.ldb_dev), io.a16_dev,
                  static_cast<long long>(io.lda16_dev), io.b16_dev, static_cast<long long>(io.ldb16_dev),
                  static_cast<const void*>(io.c_dev), static_cast<long long>(io.ldc_dev), extra_sms[i], repeats);
    const std::string key = format_schedule(schedule) + buf;
    RepeatGraph* hit = nullptr;
    for (auto& gr : graphs_)
      if (gr->key == key) hit = gr.get();
    if (!hit) {
      auto rg = std::make_unique<RepeatGraph>();
      rg->key = key;
      rg->device = dev;
      if (u->spec().kind == DeviceKind::xpu)  // per-stream state the capture must not create
        cuda_check(poas_b200::tc_prepare_stream(s), "tc_prepare_stream");
      for (int k = 0; k < 3; ++k) {
        cudaEvent_t e = nullptr;
        cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        rg->events.push_back(e);
      }
      const bool tensor = u->spec().kind == DeviceKind::xpu;
      const std::int64_t r = schedule.devices[i].rows, r0 = row0[i];
      float* c = io.c_dev + r0 * io.ldc_dev;
      const void* a = nullptr;
      const void* b = nullptr;
      std::int64_t lda = 0, ldb = 0;
      const bool sixteen = tensor && io.a16_dev && io.b16_dev;
      if (sixteen) {
        a = static_cast<const char*>(io.a16_dev) + r0 * io.lda16_dev * 2;
        b = io.b16_dev;
        lda = io.lda16_dev;
        ldb = io.ldb16_dev;
      } else {
        a = io.a_dev + r0 * io.lda_dev;
        b = io.b_dev;
        lda = io.lda_dev;
        ldb = io.ldb_dev;
      }
      const std::int64_t lda16 = round_up(d.k, 8), ldb16 = round_up(d.n, 8);
      cudaGraph_t graph = nullptr;
      cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
      try {
        for (int rep = 0; rep < repeats; ++rep) {
          const auto rec = [&](int k) {
            cuda_check(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(rg->events[k]), s,
                                                cudaEventRecordExternal), "cudaEventRecord");
          };
          if (rep == 0) {
            rec(0);
            rec(1);
          }
          if (tensor && !sixteen) {  // fp32 operands: converted inside the compute phase
            void* a16 = u->scratch(2).get();
            void* b16 = u->scratch(3).get();
            cuda_check(poas_b200::convert_f32(u->spec().dtype, static_cast<const float*>(a), lda, a16, lda16, r,
                                              d.k, s), "convert A");
            cuda_check(poas_b200::convert_f32(u->spec().dtype, static_cast<const float*>(b), ldb, b16, ldb16,
                                              d.k, d.n, s), "convert B");
            u->gemm(r, d.n, d.k, a16, lda16, b16, ldb16, c, io.ldc_dev, false, extra_sms[i]);
          } else {
            u->gemm(r, d.n, d.k, a, lda, b, ldb, c, io.ldc_dev, false, extra_sms[i]);
          }
          if (rep == repeats - 1) rec(2);
        }
      } catch (...) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        for (void* e : rg->events) cudaEventDestroy(static_cast<cudaEvent_t>(e));
        throw;
      }
      cuda_check(cudaStreamEndCapture(s, &graph), "cudaStreamEndCapture");
      rg->graph = graph;
      cudaGraphExec_t exec = nullptr;
      cuda_check(cudaGraphInstantiate(&exec, graph, 0), "cudaGraphInstantiate");
      rg->exec = exec;
      if (graphs_.size() >= 4) {
        release_graph(*graphs_.front());
        graphs_.erase(graphs_.begin());
      }
      graphs_.push_back(std::move(rg));
      hit = graphs_.back().get();
    }
    // the run's timing events are the graph's: one start and one end around
    // all repeats (no event node between two GEMMs, so each launch is staged
    // while the previous one runs); every repeat reports the mean step
    for (int rep = 0; rep < repeats; ++rep) {
      const std::size_t rr = static_cast<std::size_t>(rep);
      cudaEventDestroy(t0[dev][rr]);
      t0[dev][rr] = static_cast<cudaEvent_t>(hit->events[0]);
      PhaseEvents& pe = ev[rr][i];
      cudaEventDestroy(pe.cp0);
      cudaEventDestroy(pe.cp1);
      pe.cp0 = static_cast<cudaEvent_t>(hit->events[1]);
      pe.cp1 = static_cast<cudaEvent_t>(hit->events[2]);
    }
    amortized = repeats;
    cleanup.borrowed = true;
    first_open = std::chrono::steady_clock::now();
    cuda_check(cudaGraphLaunch(static_cast<cudaGraphExec_t>(hit->exec), s), "cudaGraphLaunch");
  }

  for (int rep = 0; rep < (graph_mode ? 0 : repeats); ++rep) {
    const std::size_t rr = static_cast<std::size_t>(rep);
    std::vector<PhaseEvents>& evr = ev[rr];
    if (host_sync_repeats) quiesce();
    for (const auto& [dev, h] : host_unit) {
      DeviceGuard g(dev);
      cudaStream_t hs = unit[h]->stream();
      if (rep > 0 && !host_sync_repeats && !pipelined)  // chain after the previous repeat
        for (std::size_t j = 0; j < nd; ++j)
          if ((j != h || overlapped) && unit[j]->on_gpu() && schedule.devices[j].rows > 0 &&
              unit[j]->spec().device == dev)
            cuda_check(cudaStreamWaitEvent(hs, last_event(rr - 1, j), 0), "cudaStreamWaitEvent");
      cuda_check(poas_b200::gate_wait(gates.device_flag(rep), hs), "gate_wait");
      cuda_check(cudaEventRecord(t0[dev][rr], hs), "cudaEventRecord");
      for (std::size_t i = 0; i < nd; ++i)
        if (i != h && unit[i]->on_gpu() && schedule.devices[i].rows > 0 &&
            unit[i]->spec().device == dev)
          cuda_check(cudaStreamWaitEvent(unit[i]->stream(), t0[dev][rr], 0), "cudaStreamWaitEvent");
    }

    // Row-sharded run: this repeat's broadcast of B over the comm (every
    // rank relays every epoch, busy or not), gated on the repeat's t0.
    int bepoch = io.b_epoch;
    const void* b16_rep = io.b16_dev;
    const float* b32_rep = io.b_dev;
    const int* bflags_rep = io.b_flags;
    void* const* bready_rep = io.b_ready;
    if (comm) {
      bool needs32 = false;  // a busy unit reading fp32 B (CUDA cores, or converting)
      for (std::size_t i = 0; i < nd; ++i)
        if (schedule.devices[i].rows > 0 && unit[i]->on_gpu() &&
            !(unit[i]->spec().kind == DeviceKind::xpu && io.a16_dev && io.b16_dev))
          needs32 = true;
      std::vector<cudaEvent_t> after;
      if (auto it = t0.find(comm->device()); it != t0.end()) after.push_back(it->second[rr]);
      if (needs32 && !comm->has_b32())
        fail(errc::invalid_argument, "comm: a busy unit reads fp32 B but only 16-bit B is registered");
      bepoch = comm->enqueue_broadcast(transport, needs32, after);
      b16_rep = comm->b16_for(bepoch);
      b32_rep = comm->b32_for(bepoch);
      bflags_rep = comm->dev_flags();
      bready_rep = comm->panel_events();
    }

    // Copy-in + compute, in schedule order.
    std::size_t prev_in = nd;  // previous busy bus unit (link order)
    for (std::size_t i = 0; i < nd; ++i) {
      const ScheduledDevice& sd = schedule.devices[i];
      Unit* u = unit[i];
      if (!u->on_gpu() || sd.rows == 0) continue;
      DeviceGuard g(u->spec().device);
      if (overlapped) {  // copy-in, compute and copy-out of this unit
        enqueue_overlapped(i, rr, prev_in, prev_in);
        prev_in = i;
        continue;
      }
      cudaStream_t s = u->stream();
      const bool tensor = u->spec().kind == DeviceKind::xpu;
      const std::int64_t r = sd.rows, r0 = row0[i];

      const void* a = nullptr;
      const void* b = nullptr;
      std::int64_t lda = 0, ldb = 0;
      float* c = nullptr;
      std::int64_t ldc = 0;

      const bool link16 = !io.resident && tensor && host16_link(u);
      if (!io.resident) {
        if (bus_ && prev_in != nd) cuda_check(cudaStreamWaitEvent(s, evr[prev_in].ci1, 0), "wait");
        cuda_check(cudaEventRecord(evr[i].ci0, s), "cudaEventRecord");
        if (link16) {
          // 16-bit operands cross the link and land in the kernel's layout
          // (row pitch a multiple of 8 elements): no conversion pass.
          const std::int64_t lda16 = round_up(d.k, 8), ldb16 = round_up(d.n, 8);
          void* a16 = u->scratch(2).ensure(static_cast<std::size_t>(r * lda16) * 2);
          void* b16 = u->scratch(3).ensure(static_cast<std::size_t>(d.k * ldb16) * 2);
          copy2d(a16, lda16, static_cast<const char*>(io.a16_host) + r0 * io.lda16_host * 2,
                 io.lda16_host, r, d.k, 2, cudaMemcpyHostToDevice, s);
          copy2d(b16, ldb16, io.b16_host, io.ldb16_host, d.k, d.n, 2, cudaMemcpyHostToDevice, s);
          a = a16;
          b = b16;
          lda = lda16;
          ldb = ldb16;
        } else {
          float* da = static_cast<float*>(u->scratch(0).ensure(static_cast<std::size_t>(r * d.k) * 4));
          float* db = static_cast<float*>(u->scratch(1).ensure(static_cast<std::size_t>(d.k * d.n) * 4));
          copy2d(da, d.k, io.a_host + r0 * io.lda_host, io.lda_host, r, d.k, 4,
                 cudaMemcpyHostToDevice, s);
          copy2d(db, d.n, io.b_host, io.ldb_host, d.k, d.n, 4, cudaMemcpyHostToDevice, s);
          a = da;
          b = db;
          lda = d.k;
          ldb = d.n;
        }
        c = static_cast<float*>(u->scratch(4).ensure(static_cast<std::size_t>(r * d.n) * 4));
        ldc = d.n;
        prev_in = i;
      } else {
        c = io.c_dev + r0 * io.ldc_dev;
        ldc = io.ldc_dev;
        if (tensor && io.a16_dev && io.b16_dev) {
          a = static_cast<const char*>(io.a16_dev) + r0 * io.lda16_dev * 2;
          b = b16_rep;
          lda = io.lda16_dev;
          ldb = io.ldb16_dev;
        } else {
          a = io.a_dev + r0 * io.lda_dev;
          b = b32_rep;
          lda = io.lda_dev;
          ldb = io.ldb_dev;
        }
      }
      if (!io.resident) cuda_check(cudaEventRecord(evr[i].ci1, s), "cudaEventRecord");

      cuda_check(cudaEventRecord(evr[i].cp0, s), "cudaEventRecord");
      const bool need_convert = tensor && !(io.resident && io.a16_dev && io.b16_dev) && !link16;
      if (need_convert) {
        const AbType t = u->spec().dtype;
        const std::int64_t lda16 = round_up(d.k, 8), ldb16 = round_up(d.n, 8);
        void* a16 = u->scratch(2).ensure(static_cast<std::size_t>(r * lda16) * 2);
        void* b16 = u->scratch(3).ensure(static_cast<std::size_t>(d.k * ldb16) * 2);
        cuda_check(poas_b200::convert_f32(t, static_cast<const float*>(a), lda, a16, lda16, r, d.k, s),
                   "convert A");
        cuda_check(poas_b200::convert_f32(t, static_cast<const float*>(b), ldb, b16, ldb16, d.k, d.n, s),
                   "convert B");
        a = a16;
        b = b16;
        lda = lda16;
        ldb = ldb16;
      }
      if (panels > 1 && bflags_rep && tensor && !need_convert && (d.n / panels) % 256 == 0) {
        // Panel-major B arriving panel by panel, consumed by ONE launch:
        // the kernel's producers start on panel p once b_flags[p] reaches
        // b_epoch (written in panel order by the deliverer), so compute on
        // early panels overlaps the transfer of later ones without per-panel
        // launches (no wave-quantisation tail per panel).
        u->gemm_panels(r, d.n, d.k, a, lda, b, d.n / panels, c, ldc, panels, bflags_rep, bepoch,
                       extra_sms[i]);
      } else if (panels > 1) {
        // Panel-major B arriving panel by panel: compute each column panel
        // as soon as it has landed (overlaps e.g. a chunked broadcast).
        const std::int64_t np = d.n / panels;
        const std::size_t esz = (tensor && !need_convert) ? 2 : 4;
        for (int p = 0; p < panels; ++p) {
          if (bready_rep && bready_rep[p])
            cuda_check(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(bready_rep[p]), 0),
                       "wait B panel");
          const void* bp = static_cast<const char*>(b) + static_cast<std::size_t>(p) * d.k * np * esz;
          u->gemm(r, np, d.k, a, lda, bp, np, c + p * np, ldc, false, extra_sms[i]);
        }
      } else {
        // One readiness event for the whole of B (e.g. a single broadcast).
        if (io.resident && bready_rep && bready_rep[0])
          cuda_check(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(bready_rep[0]), 0),
                     "wait B");
        u->gemm(r, d.n, d.k, a, lda, b, ldb, c, ldc, false, extra_sms[i]);
      }
      cuda_check(cudaEventRecord(evr[i].cp1, s), "cudaEventRecord");
      if (comm) comm->consumed(bepoch, s);  // the next writer of these B buffers waits for it
    }

    // Copy-outs, in schedule order.
    const std::size_t last_in = prev_in;
    std::size_t prev_out = nd;
    for (std::size_t i = 0; i < nd; ++i) {
      const ScheduledDevice& sd = schedule.devices[i];
      Unit* u = unit[i];
      if (!u->on_gpu() || sd.rows == 0) continue;
      DeviceGuard g(u->spec().device);
      cudaStream_t s = u->stream();
      if (!io.resident && !overlapped) {
        if (bus_) {
          if (prev_out == nd) {
            if (last_in != nd && last_in != i)
              cuda_check(cudaStreamWaitEvent(s, evr[last_in].ci1, 0), "wait");
          } else {
            cuda_check(cudaStreamWaitEvent(s, evr[prev_out].co1, 0), "wait");
          }
        }
        cuda_check(cudaEventRecord(evr[i].co0, s), "cudaEventRecord");
        copy2d(io.c_host + row0[i] * io.ldc_host, io.ldc_host, u->scratch(4).get(), d.n, sd.rows,
               d.n, 4, cudaMemcpyDeviceToHost, s);
        prev_out = i;
        cuda_check(cudaEventRecord(evr[i].co1, s), "cudaEventRecord");
      }
    }

    // Open the gate: the whole repeat is queued. Host threads start now.
    gates.open(rep);
    const auto host_t0 = std::chrono::steady_clock::now();
    if (rep == 0) first_open = host_t0;
    std::vector<std::thread> host_jobs;
    std::vector<std::exception_ptr> cpu_err(nd);
    // The first busy host unit runs on this thread (the others get their
    // own): its OpenMP team is then the one the unit's probes ran on, reused
    // across repeats, instead of a fresh team per repeat on a new OS thread
    // (C1 2048^3: thread start-up and cold caches cost ~20% of the step).
    std::size_t inline_unit = nd;
    for (std::size_t i = 0; i < nd && inline_unit == nd; ++i)
      if (!unit[i]->on_gpu() && schedule.devices[i].rows > 0) inline_unit = i;
    auto run_host = [&](std::size_t i, int rep) {
        try {
          const ScheduledDevice& s = schedule.devices[i];
          const auto a = std::chrono::steady_clock::now();
          unit[i]->gemm(s.rows, d.n, d.k, io.a_host + row0[i] * io.lda_host, io.lda_host,
                        io.b_host, io.ldb_host, io.c_host + row0[i] * io.ldc_host, io.ldc_host,
                        false);
          const auto b = std::chrono::steady_clock::now();
          cpu_start[static_cast<std::size_t>(rep)][i] = std::chrono::duration<double>(a - host_t0).count();
          cpu_end[static_cast<std::size_t>(rep)][i] = std::chrono::duration<double>(b - host_t0).count();
        } catch (...) {
          cpu_err[i] = std::current_exception();
        }
    };
    for (std::size_t i = 0; i < nd; ++i) {
      if (unit[i]->on_gpu() || schedule.devices[i].rows == 0 || i == inline_unit) continue;
      host_jobs.emplace_back([&run_host, i, rep] { run_host(i, rep); });
    }
    if (inline_unit < nd) run_host(inline_unit, rep);
    if (host_sync_repeats) {
      for (std::thread& t : host_jobs) t.join();
      quiesce();
      sum_wall += std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count();
      for (auto& e : cpu_err)
        if (e) std::rethrow_exception(e);
    }
  }
  if (!host_sync_repeats) {
    quiesce();
    sum_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - first_open).count();
  }

  // Measured timelines, relative to each repeat's t0.
  SimulationResult res;
  res.repeats = repeats;
  std::vector<double> sum_in(nd, 0.0), sum_cp(nd, 0.0), sum_out(nd, 0.0), sum_fin(nd, 0.0);
  double sum_makespan = 0.0;
  for (int rep = 0; rep < repeats; ++rep) {
    const std::size_t r = static_cast<std::size_t>(rep);
    std::vector<DeviceTimeline> tl(nd);
    double makespan = 0.0;
    for (std::size_t i = 0; i < nd; ++i) {
      const ScheduledDevice& sd = schedule.devices[i];
      DeviceTimeline& t = tl[i];
      if (sd.rows == 0) {
        t = sd.timeline;  // idle: nothing to measure, keep the plan's placement
        continue;
      }
      if (!unit[i]->on_gpu()) {
        t.copy_in = {0.0, 0.0};
        t.compute = {cpu_start[r][i], cpu_end[r][i]};
        t.copy_out = {cpu_end[r][i], cpu_end[r][i]};
        t.finish = cpu_end[r][i];
      } else {
        DeviceGuard g(unit[i]->spec().device);
        cudaEvent_t z = t0[unit[i]->spec().device][r];
        const auto at = [&](cudaEvent_t e) {
          float ms = 0.f;
          cuda_check(cudaEventElapsedTime(&ms, z, e), "cudaEventElapsedTime");
          return static_cast<double>(ms) * 1e-3 / amortized;
        };
        const PhaseEvents& e = ev[r][i];
        t.compute = {at(e.cp0), at(e.cp1)};
        if (io.resident) {
          t.copy_in = {t.compute.start, t.compute.start};
          t.copy_out = {t.compute.end, t.compute.end};
        } else {
          t.copy_in = {at(e.ci0), at(e.ci1)};
          t.copy_out = {at(e.co0), at(e.co1)};
        }
        t.finish = t.copy_out.end;
      }
      makespan = std::max(makespan, t.finish);
    }
    for (std::size_t i = 0; i < nd; ++i) {
      sum_in[i] += tl[i].copy_in.duration();
      sum_cp[i] += tl[i].compute.duration();
      sum_out[i] += tl[i].copy_out.duration();
      sum_fin[i] += tl[i].finish;
    }
    sum_makespan += makespan;
    res.repeat_timelines.push_back(std::move(tl));
  }

  const double inv = 1.0 / repeats;
  std::vector<double> e_cp, e_copy, e_fin;
  for (std::size_t i = 0; i < nd; ++i) {
    const ScheduledDevice& sd = schedule.devices[i];
    const bool link = unit[i]->on_gpu();
    DeviceOutcome o;
    o.id = sd.id;
    o.rows = sd.rows;
    o.copy_in = {sum_in[i] * inv, sd.timeline.copy_in.duration(), 0.0};
    o.compute = {sum_cp[i] * inv, sd.timeline.compute.duration(), 0.0};
    o.copy_out = {sum_out[i] * inv, sd.timeline.copy_out.duration(), 0.0};
    o.copy = {(sum_in[i] + sum_out[i]) * inv,
              sd.timeline.copy_in.duration() + sd.timeline.copy_out.duration(), 0.0};
    o.finish = {sum_fin[i] * inv, link ? sd.timeline.copy_out.end : sd.timeline.compute.end, 0.0};
    o.overlapped = overlapped && link && sd.rows > 0;
    for (PhaseError* p : {&o.copy_in, &o.compute, &o.copy_out, &o.copy, &o.finish})
      p->error_pct = rel_err_pct(p->measured, p->predicted);
    if (sd.rows > 0) {
      e_cp.push_back(o.compute.error_pct);
      e_fin.push_back(o.finish.error_pct);
      if (link && !io.resident) e_copy.push_back(o.copy.error_pct);
    }
    res.devices.push_back(std::move(o));
  }
  res.measured_makespan = sum_makespan * inv;
  res.predicted_makespan = schedule.makespan;
  res.makespan_error_pct = rel_err_pct(res.measured_makespan, res.predicted_makespan);
  res.rmse_compute = rms(e_cp);
  res.rmse_copy = rms(e_copy);
  res.rmse_finish = rms(e_fin);
  res.measured_wall = sum_wall * inv;
  return res;
}

namespace {

std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[40];
  for (int prec = 15; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

std::string phase_json(const PhaseError& p) {
  return "{\"measured\": " + num(p.measured) + ", \"predicted\": " + num(p.predicted) +
         ", \"error_pct\": " + num(p.error_pct) + "}";
}

}  // namespace

std::string format_execution_report(const Schedule& s, const SimulationResult& r) {
  std::string o = "{\n";
  o += "  \"machine_hash\": \"" + s.machine_hash + "\",\n";
  o += "  \"dims\": {\"m\": " + std::to_string(s.dims.m) + ", \"n\": " + std::to_string(s.dims.n) +
       ", \"k\": " + std::to_string(s.dims.k) + "},\n";
  o += "  \"seed\": " + std::to_string(r.seed) + ",\n";
  o += "  \"repeats\": " + std::to_string(r.repeats) + ",\n";
  o += "  \"predicted_makespan\": " + num(r.predicted_makespan) + ",\n";
  o += "  \"measured_makespan\": " + num(r.measured_makespan) + ",\n";
  o += "  \"makespan_error_pct\": " + num(r.makespan_error_pct) + ",\n";
  o += "  \"devices\": [\n";
  for (std::size_t i = 0; i < r.devices.size(); ++i) {
    const DeviceOutcome& d = r.devices[i];
    o += "    {\"id\": \"" + d.id + "\", \"rows\": " + std::to_string(d.rows) +
         ",\n     \"copy_in\": " + phase_json(d.copy_in) + ",\n     \"compute\": " +
         phase_json(d.compute) + ",\n     \"copy_out\": " + phase_json(d.copy_out) +
         ",\n     \"copy\": " + phase_json(d.copy) + ",\n     \"finish\": " +
         phase_json(d.finish) + (d.overlapped ? ",\n     \"overlapped\": true" : "") + "}";
    o += i + 1 < r.devices.size() ? ",\n" : "\n";
  }
  o += "  ],\n";
  o += "  \"rmse\": {\"finish\": " + num(r.rmse_finish) + ", \"compute\": " + num(r.rmse_compute) +
       ", \"copy\": " + num(r.rmse_copy) + "},\n";
  o += "  \"measured_wall\": " + num(r.measured_wall) + ",\n";
  o += "  \"repeat_makespans\": [";
  for (std::size_t k = 0; k < r.repeat_timelines.size(); ++k) {
    double m = 0.0;  // busy units only, as measured_makespan
    for (std::size_t i = 0; i < r.repeat_timelines[k].size() && i < s.devices.size(); ++i)
      if (s.devices[i].rows > 0) m = std::max(m, r.repeat_timelines[k][i].finish);
    o += (k ? ", " : "") + num(m);
  }
  o += "]\n}\n";
  return o;
}

}  // namespace poas
