#pragma once
// Two-level plan of the row-sharded multi-GPU GEMM.
//
// Level 1 splits the rows of A across the G GPUs of a box with the SAME
// planner (reference pipeline, proj/src/optimizer.cpp:238-325): every GPU is
// one xpu device whose model is its units' combined throughput -- slope =
// 1 / sum(1/slope_u) over its GPU units (throughputs add), intercept = max,
// align = lcm of its tensor units' aligns -- on a PRIVATE link (bus false:
// NVSwitch gives every GPU its own full-bandwidth port, the reference's
// private-link timeline proj/src/timeline.cpp:24-35 and LP rows
// proj/src/optimizer.cpp:108-115) whose bandwidth is that GPU's measured
// B-broadcast throughput. Heterogeneous GPUs (a throttled one, a different
// SM partition) get proportionally fewer rows; identical GPUs split evenly.
// Level 2 is each GPU's own plan of its rows over its units (any policy).
// A flat plan with every unit of the box is never made: the reference LP
// charges B per unit and the rounding residue lands on the host CPU
// (SURVEY.md 8e).
#include <optional>
#include <string>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/scheduler.hpp"

namespace poas {

struct ShardedPlan {
  MachineProfile level1;
  Schedule level1_schedule;
  std::vector<std::int64_t> rows;  // per GPU, rank order
  std::vector<std::int64_t> row0;  // first row of A per GPU
  std::vector<std::optional<Schedule>> plans;  // per GPU (none when it has no rows)
};

MachineProfile level1_profile(const std::vector<MachineProfile>& gpus, const std::vector<double>& link_bw);
ShardedPlan plan_sharded(const std::vector<MachineProfile>& gpus, const std::vector<double>& link_bw,
                         const MatrixDims& dims, const std::string& policy);

}  // namespace poas
