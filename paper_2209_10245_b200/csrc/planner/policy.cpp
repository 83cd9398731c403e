// Planner policies (B200 extension, opt-in; the default is the reference's
// algorithm and stays byte-identical to it).
//
// "best-subset": the reference LP charges every formulated unit the whole B
// transfer and launch overhead (proj/src/optimizer.cpp:21-32) and only
// drops units worth less than one row (:257-275). On a B200 a 2-SM CUDA-core
// unit's fixed cost -- receiving all of B -- can exceed what it contributes,
// yet it keeps a few rows and delays the tensor unit's copy-out on the
// shared link (the "subset-selection problem" the reference declares out of
// its scope, proj/tests/support.hpp:97-102). This policy plans every
// non-empty subset of units with the reference pipeline (solve_split ->
// build_tile_plan on the sub-machine) and keeps the plan whose full-machine
// schedule has the smallest predicted makespan; ties keep the larger subset
// (the full machine first, i.e. the reference plan when it is best).
#include <algorithm>
#include <cmath>
#include <limits>

#include "poas/adapter.hpp"
#include "poas/error.hpp"
#include "poas/optimizer.hpp"
#include "poas/overlap.hpp"
#include "poas/policy.hpp"
#include "poas/scheduler.hpp"

namespace poas {

Schedule plan_schedule(const MachineProfile& machine, const MatrixDims& dims) {
  const WorkloadSplit split = solve_split(machine, dims);
  return build_schedule(build_tile_plan(machine, dims, split), machine);
}

std::vector<TilePlan> subset_tile_plans(const MachineProfile& machine, const MatrixDims& dims) {
  validate_machine(machine);
  validate_dims(dims);
  const std::size_t nd = machine.devices.size();
  if (nd > 12) fail(errc::too_many_devices, "subset policies support at most 12 units");

  // Masks in decreasing popcount order (full machine first), then ascending.
  std::vector<unsigned> masks;
  for (unsigned mask = 1; mask < (1u << nd); ++mask) masks.push_back(mask);
  std::stable_sort(masks.begin(), masks.end(), [](unsigned a, unsigned b) {
    return __builtin_popcount(a) > __builtin_popcount(b);
  });

  std::vector<TilePlan> out;
  for (const unsigned mask : masks) {
    MachineProfile sub;
    sub.bus = machine.bus;
    std::vector<std::size_t> index;
    for (std::size_t i = 0; i < nd; ++i)
      if (mask & (1u << i)) {
        sub.devices.push_back(machine.devices[i]);
        index.push_back(i);
      }
    TilePlan sub_plan;
    try {
      const WorkloadSplit split = solve_split(sub, dims);
      sub_plan = build_tile_plan(sub, dims, split);
    } catch (const Error& e) {
      // A subset that cannot hold the rows (e.g. only aligned units and an
      // unaligned m) is simply not a candidate.
      if (e.code() == errc::no_feasible_tiling || e.code() == errc::unalignable_k) continue;
      throw;
    }
    TilePlan full;
    full.dims = dims;
    for (std::size_t i = 0; i < nd; ++i) {
      PlannedDevice pd;
      pd.device_id = machine.devices[i].id;
      full.devices.push_back(pd);
    }
    for (std::size_t j = 0; j < index.size(); ++j) full.devices[index[j]] = sub_plan.devices[j];
    out.push_back(std::move(full));
  }
  if (out.empty()) fail(errc::no_feasible_tiling, "no subset of units can hold the workload");
  return out;
}

Schedule plan_best_subset(const MachineProfile& machine, const MatrixDims& dims) {
  Schedule best;
  double best_makespan = std::numeric_limits<double>::infinity();
  for (const TilePlan& full : subset_tile_plans(machine, dims)) {
    Schedule s = build_schedule(full, machine);
    if (s.makespan < best_makespan) {
      best_makespan = s.makespan;
      best = std::move(s);
    }
  }
  return best;
}

Schedule plan_with_policy(const MachineProfile& machine, const MatrixDims& dims,
                          const std::string& policy) {
  if (policy.empty() || policy == "reference") return plan_schedule(machine, dims);
  if (policy == "best-subset") return plan_best_subset(machine, dims);
  if (policy == "overlap") return plan_overlap(machine, dims);
  fail(errc::invalid_argument, "unknown planner policy '" + policy + "'");
}

PartitionChoice plan_sm_partitions(const MachineProfile& machine, const MatrixDims& dims,
                                   const std::string& tc_id, int tc_sms, const std::string& simt_id,
                                   int simt_sms, const std::vector<int>& simt_budgets,
                                   const std::string& policy) {
  validate_machine(machine);
  const DeviceProfile* tc = machine.find(tc_id);
  const DeviceProfile* simt = machine.find(simt_id);
  if (!tc || !simt) fail(errc::invalid_argument, "partition: unknown unit id");
  if (tc_sms < 1 || simt_sms < 1) fail(errc::invalid_argument, "partition: SM budgets must be >= 1");
  if (simt_budgets.empty()) fail(errc::invalid_argument, "partition: no candidate budgets");
  const int total = tc_sms + simt_sms;
  PartitionChoice out;
  for (const int s : simt_budgets) {
    if (s < 0 || s >= total) fail(errc::invalid_argument, "partition: candidate budget out of range");
    MachineProfile m;
    m.bus = machine.bus;
    for (const DeviceProfile& d : machine.devices) {
      if (d.id == simt_id) {
        if (s == 0) continue;  // left out: its SMs go to the tensor unit
        DeviceProfile x = d;
        x.compute.slope *= static_cast<double>(simt_sms) / s;
        if (x.bandwidth > 0.0) x.bandwidth *= static_cast<double>(s) / simt_sms;
        m.devices.push_back(x);
      } else if (d.id == tc_id) {
        DeviceProfile x = d;
        x.compute.slope *= static_cast<double>(tc_sms) / (total - s);
        m.devices.push_back(x);
      } else {
        m.devices.push_back(d);
      }
    }
    PartitionCandidate c;
    c.simt_sms = s;
    c.tc_sms = total - s;
    c.schedule = plan_with_policy(m, dims, policy);
    const double best = out.candidates.empty() ? 0.0 : out.candidates[out.best].schedule.makespan;
    out.candidates.push_back(std::move(c));
    if (out.candidates.size() == 1 || out.candidates.back().schedule.makespan < best)
      out.best = out.candidates.size() - 1;
  }
  return out;
}

}  // namespace poas
