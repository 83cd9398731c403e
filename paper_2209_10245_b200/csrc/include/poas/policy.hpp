#pragma once
// Planner policies. "reference" (default) is the reference pipeline,
// byte-identical plans; "best-subset" is an opt-in B200 extension that also
// considers leaving units idle (see csrc/planner/policy.cpp); "overlap"
// adds overlapped copies on top of it (poas/overlap.hpp).

#include <string>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/scheduler.hpp"

namespace poas {

Schedule plan_schedule(const MachineProfile& machine, const MatrixDims& dims);
// Every non-empty subset of units planned with the reference pipeline
// (solve_split -> build_tile_plan on the sub-machine), as full-machine tile
// plans (left-out units idle): the full machine first, then by decreasing
// unit count. Subsets that cannot hold the rows are skipped.
std::vector<TilePlan> subset_tile_plans(const MachineProfile& machine, const MatrixDims& dims);
Schedule plan_best_subset(const MachineProfile& machine, const MatrixDims& dims);
Schedule plan_with_policy(const MachineProfile& machine, const MatrixDims& dims,
                          const std::string& policy);

}  // namespace poas
