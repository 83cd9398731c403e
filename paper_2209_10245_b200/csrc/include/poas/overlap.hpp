#pragma once
// Overlapped copies: the "overlap" planner policy (B200 extension, opt-in).
//
// The paper copies synchronously and notes that "this simple approach could
// be improved using CUDA streams and overlapping the computation with memory
// copies ... the performance predictor can be adapted to predict the memory
// copies with or without overlap". This is that
// adaptation. A link unit's share is cut into R row parts of A and Q column
// panels of B -- an R x Q grid of blocks, the adapter's tiles (k' = k). The
// executor (units option "overlap=1") sends A parts and B panels
// host->device interleaved (overlap_link_order), computes each block as soon
// as its A part and B panel have landed, and returns each block's C
// device->host while later blocks compute. Q = 1 is "B, then the A parts".
// The link is full duplex (PCIe, NVLink): host->device and device->host are
// two queues, each served in priority order as in the paper's shared-bus
// scheme (proj/src/timeline.cpp:37-69), but a copy-out no longer waits for
// the last copy-in. C crosses the link in fp32 (what every unit produces
// here), so a 2-byte tensor unit's copy-out is charged 4 bytes per element.

#include <cstdint>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/scheduler.hpp"
#include "poas/timeline.hpp"

namespace poas {

// One host->device transfer of a unit: A row part `index` or B panel `index`.
struct OverlapItem {
  bool a = true;
  int index = 0;
};

// The host->device order of R row parts and Q column panels: start with A
// part 0, then always the operand that is proportionally behind (A while
// a_done / R <= b_done / Q, else B). Q = 1: A0, B, A1, A2, ...
std::vector<OverlapItem> overlap_link_order(int parts, int panels);

// One output block (row part, column panel) and the position in the link
// order of the transfer after which both its operands are on the device.
struct OverlapBlock {
  int part = 0;
  int panel = 0;
  int ready_item = 0;
};

// Blocks in compute order: as each link item lands, the blocks it completes
// (A part i: (i, j) for every landed panel j ascending; B panel j: (i, j)
// for every landed part i ascending).
std::vector<OverlapBlock> overlap_block_order(int parts, int panels);

// Per-unit phase durations.
struct OverlapEntry {
  int priority = 0;
  bool uses_bus = false;
  std::vector<double> link_in;  // host->device items, in link order
  std::vector<int> ready;       // per block (compute order): its ready_item
  std::vector<double> compute;  // per block: its GEMM (one launch each)
  std::vector<double> c_out;    // per block: its C, device->host
};

// Places every block on the clock: link items back to back on the
// host->device queue; block b computes after its ready item and block b-1;
// its C leaves after its compute and the previous copy-out on the
// device->host queue. With a shared bus the queues are shared in priority
// order; with private links each unit has its own pair. A unit without a
// link (cpu) computes from t = 0 (compute holds its whole share). The
// DeviceTimeline of a unit is the span of each phase (first start .. last
// end). Returns the makespan.
double evaluate_overlap_timeline(const std::vector<OverlapEntry>& entries, bool shared_bus,
                                 std::vector<DeviceTimeline>* out);

// `extent` cut into at most `parts` pieces of whole `block`-sized blocks,
// spread evenly (earlier pieces one block larger), the extent % block tail
// on the last piece; fewer pieces when there are fewer blocks.
std::vector<std::int64_t> overlap_split(std::int64_t extent, int parts, std::int64_t block);
// Row parts: 256-row blocks (the pair kernel's tile height: a streamed
// launch never lets a tile straddle two parts).
std::vector<std::int64_t> overlap_row_parts(std::int64_t rows, int parts);
// Column panels: 256-column blocks (the pair kernel's tile width).
std::vector<std::int64_t> overlap_col_panels(std::int64_t n, int panels);

// A device's row parts and column panels as a schedule records them. The
// overlap policy writes the R x Q blocks part-major as tiles (m_p, k, n_q);
// reference tiles are k'-strip-major (q row parts per k-strip,
// proj/src/adapter.cpp:159-167) with n' = n. Either way: panels = the n of
// the leading tiles until they cover n (one panel for n' = n), parts = the
// m of every panels-th tile of the first strip. Falls back to one part x
// one panel when the tiles describe no such grid.
struct RowColGrid {
  std::vector<std::int64_t> parts;
  std::vector<std::int64_t> panels;
};
RowColGrid schedule_grid(const ScheduledDevice& device, const MatrixDims& dims);
// Row parts only (the grid's parts).
std::vector<std::int64_t> schedule_row_parts(const ScheduledDevice& device, const MatrixDims& dims);

// Lays a tile plan out with overlapped copies: every busy link unit is
// re-tiled into overlap_row_parts(rows, parts) x overlap_col_panels(n,
// panels) full-K blocks; host-CPU units keep the adapter's tiles and run
// from t = 0.
Schedule build_overlap_schedule(const TilePlan& plan, const MachineProfile& machine, int parts,
                                int panels = 1);

// The policy: every non-empty subset of units planned with the reference
// pipeline (as "best-subset"), each laid out with 1, 2, 4, ... 64 row parts
// and 1, 2, 4, 8, 16 column panels of at least 4096 columns (narrower C
// blocks make slow device->host DMA segments); the smallest predicted
// makespan wins; a later candidate (a smaller subset, more parts or panels)
// must beat the best so far by more than 0.1%.
Schedule plan_overlap(const MachineProfile& machine, const MatrixDims& dims);

}  // namespace poas
