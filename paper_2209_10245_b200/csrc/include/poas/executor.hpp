#pragma once
// Execute: the real replacement of the reference's simulate()
// (proj/include/poas/simulator.hpp:68-69, proj/src/simulator.cpp:104-209).
//
// A schedule is run on the units of this box: every unit's share
// concurrently (one CUDA stream per GPU unit, OpenMP host threads for the
// CPU unit), link copies ordered by the schedule's bus discipline, every
// phase timed on a common clock. The result has the reference's
// SimulationResult shape (simulator.hpp:34-60) with measured = real time.

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "poas/scheduler.hpp"
#include "poas/timeline.hpp"

namespace poas_b200 {
class Unit;
}

namespace poas_b200 {
class Comm;
}

namespace poas {

struct PhaseError {
  double measured = 0.0;
  double predicted = 0.0;
  double error_pct = 0.0;  // 100 (measured - predicted) / measured
};

struct DeviceOutcome {
  std::string id;
  std::int64_t rows = 0;
  PhaseError copy_in, compute, copy_out;
  PhaseError copy;
  PhaseError finish;
  bool overlapped = false;  // its copies ran pipelined with compute (overlap=1)
};

struct SimulationResult {
  std::vector<DeviceOutcome> devices;  // schedule order
  double measured_makespan = 0.0;      // mean over repeats
  double predicted_makespan = 0.0;
  double makespan_error_pct = 0.0;
  double rmse_compute = 0.0;
  double rmse_copy = 0.0;
  double rmse_finish = 0.0;
  int repeats = 0;
  std::uint64_t seed = 0;
  std::vector<std::vector<DeviceTimeline>> repeat_timelines;  // [repeat][device], measured
  double measured_wall = 0.0;  // host wall clock per repeat (mean), launch to last completion
};

// Operands of one GEMM (row-major). See poas_gemm_io in include/poas_b200.h.
struct GemmOperands {
  std::int64_t m = 0, n = 0, k = 0;
  const float* a_host = nullptr;
  std::int64_t lda_host = 0;
  const float* b_host = nullptr;
  std::int64_t ldb_host = 0;
  float* c_host = nullptr;
  std::int64_t ldc_host = 0;
  const float* a_dev = nullptr;
  std::int64_t lda_dev = 0;
  const float* b_dev = nullptr;
  std::int64_t ldb_dev = 0;
  const void* a16_dev = nullptr;
  std::int64_t lda16_dev = 0;
  const void* b16_dev = nullptr;
  std::int64_t ldb16_dev = 0;
  float* c_dev = nullptr;
  std::int64_t ldc_dev = 0;
  bool resident = false;
  // Panel-major B with per-panel readiness events (see poas_gemm_io).
  int b_panels = 0;
  void* const* b_ready = nullptr;
  const int* b_flags = nullptr;  // per-panel device flags: one fused tensor launch
  int b_epoch = 0;
  // 16-bit host operands for elem=2 tensor units (see poas_gemm_io).
  const void* a16_host = nullptr;
  std::int64_t lda16_host = 0;
  const void* b16_host = nullptr;
  std::int64_t ldb16_host = 0;
  // Row-sharded multi-GPU run (see poas_gemm_io.comm): the executor
  // broadcasts B itself, every repeat, over this communicator.
  poas_b200::Comm* comm = nullptr;
  int b_transport = 0;  // 0 copy engines (chain), 1 NCCL
};

double rel_err_pct(double measured, double predicted);

class Executor {
 public:
  // `units`: ';'-separated unit specs (runtime/units.hpp), optional "bus=0|1".
  explicit Executor(const std::string& units);
  ~Executor();
  Executor(const Executor&) = delete;
  Executor& operator=(const Executor&) = delete;

  // Identity hash over the units (id, kind, link elem_size) and the bus
  // flag; a schedule planned for this box carries the same hash.
  const std::string& machine_hash() const { return hash_; }
  bool bus() const { return bus_; }
  bool overlap() const { return overlap_; }
  poas_b200::Unit* find(const std::string& id) const;
  const std::vector<std::unique_ptr<poas_b200::Unit>>& units() const { return units_; }

  SimulationResult run(const Schedule& schedule, const GemmOperands& io, int repeats);

 private:
  std::vector<std::unique_ptr<poas_b200::Unit>> units_;
  bool bus_ = true;
  bool lend_ = true;      // idle units' SMs go to the one busy unit on their GPU
  bool overlap_ = false;  // host runs: pipeline link units' row parts (poas/overlap.hpp)
  bool pipeline_ = false;  // overlapped host runs: consecutive repeats overlap (units.hpp)
  // Per unit (units_ order; null for cpu units): the host->device and
  // device->host copy streams of overlapped runs.
  std::vector<void*> h2d_, d2h_;

 public:
  // Start-gate flags (mapped pinned ints, one per repeat; grown on demand,
  // released with the executor). Used by run().
  struct GateBuffer {
    int* host = nullptr;
    std::size_t capacity = 0;
    std::vector<int*> retired;
  };

  // The repeats of a one-unit resident plan captured as one CUDA graph (see
  // Executor::run), with the timing events its record nodes use.
  struct RepeatGraph {
    std::string key;
    void* graph = nullptr;  // cudaGraph_t
    void* exec = nullptr;   // cudaGraphExec_t
    std::vector<void*> events;  // t0, cp0 (before the first repeat), cp1 (after the last)
    int device = 0;
  };

 private:
  static void release_graph(RepeatGraph& g);
  GateBuffer gates_;
  std::string hash_;
  std::vector<std::unique_ptr<RepeatGraph>> graphs_;  // most recent last
};

// The reference's simulate report JSON (proj/tools/poas.cpp:85-114) for a
// real run, plus "measured_wall".
std::string format_execution_report(const Schedule& schedule, const SimulationResult& result);

}  // namespace poas
