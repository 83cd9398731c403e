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

// SM partition of one GPU between its tensor unit and its CUDA-core unit
// (B200 extension: the Optimize stage choosing the partition instead of
// taking it as given). The profile describes the two units at their
// measured budgets (tc_sms, simt_sms). For each candidate CUDA-core budget s
// (0 = the unit left out, its SMs lent to the tensor unit), the model scales
// each unit's compute slope inversely with its SM count (intercepts stay)
// and the CUDA-core unit's resident-operand bandwidth -- a streaming read on
// its own SMs -- with s; every candidate is planned with `policy`. The
// result is in candidate order; best = the smallest predicted makespan
// (ties: the smaller s).
struct PartitionCandidate {
  int simt_sms = 0;
  int tc_sms = 0;
  Schedule schedule;
};
struct PartitionChoice {
  std::vector<PartitionCandidate> candidates;
  std::size_t best = 0;
};
PartitionChoice plan_sm_partitions(const MachineProfile& machine, const MatrixDims& dims,
                                   const std::string& tc_id, int tc_sms, const std::string& simt_id,
                                   int simt_sms, const std::vector<int>& simt_budgets,
                                   const std::string& policy);

}  // namespace poas
