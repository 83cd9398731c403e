// Two-level (GPU, then unit) plan of the row-sharded GEMM; see poas/sharded.hpp.
#include "poas/sharded.hpp"

#include <numeric>

#include "poas/adapter.hpp"
#include "poas/error.hpp"
#include "poas/optimizer.hpp"
#include "poas/policy.hpp"

namespace poas {

MachineProfile level1_profile(const std::vector<MachineProfile>& gpus, const std::vector<double>& link_bw) {
  if (gpus.empty()) fail(errc::invalid_argument, "sharded plan: no GPUs");
  if (link_bw.size() != gpus.size()) fail(errc::invalid_argument, "sharded plan: one link bandwidth per GPU");
  MachineProfile m;
  m.bus = false;
  for (std::size_t g = 0; g < gpus.size(); ++g) {
    double inv = 0.0, intercept = 0.0;
    std::int64_t align = 1;
    bool any = false;
    for (const DeviceProfile& u : gpus[g].devices) {
      if (u.kind == DeviceKind::cpu) continue;  // the host is not a GPU's unit
      any = true;
      inv += 1.0 / u.compute.slope;
      intercept = std::max(intercept, u.compute.intercept);
      if (u.kind == DeviceKind::xpu) align = std::lcm(align, u.align > 0 ? u.align : 1);
    }
    if (!any) fail(errc::invalid_argument, "sharded plan: GPU " + std::to_string(g) + " has no GPU units");
    if (!(link_bw[g] > 0.0)) fail(errc::invalid_argument, "sharded plan: link bandwidth must be positive");
    DeviceProfile d;
    d.id = "gpu" + std::to_string(g);
    d.kind = DeviceKind::xpu;
    d.compute = LinearModel{1.0 / inv, intercept};
    d.bandwidth = link_bw[g];
    d.elem_size = 2;
    d.priority = static_cast<int>(g);
    d.align = align;
    // Tile window of a whole GPU's share: at least 2^40 MACs (~1 ms of a
    // B200) per tile, so the adapter's tiling search stays a few candidates
    // (ops_min = 1 would search up to `rows` tile counts, O(rows^2) work at
    // ragged shapes); smaller shares fall back to one tile (the tiling of a
    // level-1 device is informational -- its rows are what level 2 plans).
    d.ops_min = OpsCount{1} << 40;
    d.ops_max = OpsCount{1} << 62;
    m.devices.push_back(d);
  }
  validate_machine(m);
  return m;
}

ShardedPlan plan_sharded(const std::vector<MachineProfile>& gpus, const std::vector<double>& link_bw,
                         const MatrixDims& dims, const std::string& policy) {
  validate_dims(dims);
  ShardedPlan out;
  out.level1 = level1_profile(gpus, link_bw);
  const WorkloadSplit split = solve_split(out.level1, dims);
  out.level1_schedule = build_schedule(build_tile_plan(out.level1, dims, split), out.level1);
  std::int64_t at = 0;
  for (std::size_t g = 0; g < gpus.size(); ++g) {
    std::int64_t r = 0;
    for (const ScheduledDevice& d : out.level1_schedule.devices)
      if (d.id == "gpu" + std::to_string(g)) r = d.rows;
    out.rows.push_back(r);
    out.row0.push_back(at);  // rank order (= level-1 priority order)
    at += r;
    if (r > 0)
      out.plans.emplace_back(plan_with_policy(gpus[g], MatrixDims{r, dims.n, dims.k}, policy));
    else
      out.plans.emplace_back(std::nullopt);
  }
  if (at != dims.m) fail(errc::numerical_failure, "sharded plan: level-1 rows do not cover m");
  return out;
}

}  // namespace poas
