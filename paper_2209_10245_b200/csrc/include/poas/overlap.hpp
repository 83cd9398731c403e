#pragma once
// Overlapped copies: the "overlap" planner policy (B200 extension, opt-in).
//
// The paper copies synchronously and notes that "this simple approach could
// be improved using CUDA streams and overlapping the computation with memory
// copies ... the performance predictor can be adapted to predict the memory
// copies with or without overlap". This is that
// adaptation. A link unit's rows are cut into row parts (the adapter's
// tiles, k' = k); the executor (units option "overlap=1") sends B and then
// the A parts host->device back to back, computes part p as soon as it has
// landed, and returns part p's C device->host while part p+1 computes. The
// link is full duplex (PCIe, NVLink): host->device and device->host are two
// queues, each served in priority order as in the paper's shared-bus scheme
// (proj/src/timeline.cpp:37-69), but a copy-out no longer waits for the last
// copy-in. C crosses the link in fp32 (what every unit produces here), so a
// 2-byte tensor unit's copy-out is charged 4 bytes per element.

#include <cstdint>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/scheduler.hpp"
#include "poas/timeline.hpp"

namespace poas {

// Per-unit phase durations, one entry per row part.
struct OverlapEntry {
  int priority = 0;
  bool uses_bus = false;
  double b_in = 0.0;               // all of B, host->device
  std::vector<double> a_in;        // A rows of each part, host->device
  std::vector<double> compute;     // each part's GEMM (one launch each)
  std::vector<double> c_out;       // C rows of each part, device->host
};

// Places every part on the clock: B then the A parts back to back on the
// host->device queue; part p computes after its A part and part p-1; its C
// leaves after its compute and the previous copy-out on the device->host
// queue. With a shared bus the queues are shared in priority order; with
// private links each unit has its own pair. The DeviceTimeline of a unit is
// the span of each phase (first start .. last end). Returns the makespan.
double evaluate_overlap_timeline(const std::vector<OverlapEntry>& entries, bool shared_bus,
                                 std::vector<DeviceTimeline>* out);

// Row parts of `rows` for `parts` parts: whole 128-row blocks (the tensor
// kernel's tile height) spread evenly, earlier parts one block larger, the
// rows % 128 tail on the last part; fewer parts when there are fewer blocks.
std::vector<std::int64_t> overlap_row_parts(std::int64_t rows, int parts);

// The row parts a schedule assigns a device: its tiles are k'-strip-major
// (q row parts per k-strip, proj/src/adapter.cpp:159-167), so the parts are
// the heights of the first q = tiles / (k / k') tiles. Falls back to one
// part when the tiles do not describe whole rows.
std::vector<std::int64_t> schedule_row_parts(const ScheduledDevice& device, const MatrixDims& dims);

// Lays a tile plan out with overlapped copies: every busy link unit is
// re-tiled into overlap_row_parts(rows, parts) full-K tiles; host-CPU
// units keep the adapter's tiles and run from t = 0.
Schedule build_overlap_schedule(const TilePlan& plan, const MachineProfile& machine, int parts);

// The policy: every non-empty subset of units planned with the reference
// pipeline (as "best-subset"), each laid out with 1, 2, 4, ... 64 parts;
// the smallest predicted makespan wins; a later candidate (a smaller
// subset, more parts) must beat the best so far by more than 0.1%.
Schedule plan_overlap(const MachineProfile& machine, const MatrixDims& dims);

}  // namespace poas
