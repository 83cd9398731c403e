// Overlapped copies: timeline, row parts and the "overlap" policy
// (see poas/overlap.hpp; B200 extension of PAPER.md:486-489).
#include "poas/overlap.hpp"

#include <algorithm>
#include <limits>
#include <numeric>

#include "poas/error.hpp"
#include "poas/policy.hpp"

namespace poas {

double evaluate_overlap_timeline(const std::vector<OverlapEntry>& entries, bool shared_bus,
                                 std::vector<DeviceTimeline>* out) {
  const std::size_t n = entries.size();
  out->assign(n, DeviceTimeline{});
  std::vector<std::size_t> order(n);
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
    return entries[a].priority < entries[b].priority;
  });

  double h2d_free = 0.0, d2h_free = 0.0, makespan = 0.0;
  for (const std::size_t i : order) {
    const OverlapEntry& e = entries[i];
    DeviceTimeline& t = (*out)[i];
    const std::size_t parts = e.compute.size();
    if (!e.uses_bus) {
      double c = 0.0;
      for (double x : e.compute) c += x;
      t.copy_in = {0.0, 0.0};
      t.compute = {0.0, c};
      t.copy_out = {c, c};
      t.finish = c;
      makespan = std::max(makespan, t.finish);
      continue;
    }
    if (parts == 0) {  // idle link unit: zero-length phases where its queue stands
      const double at = shared_bus ? h2d_free : 0.0;
      t.copy_in = t.compute = t.copy_out = {at, at};
      t.finish = at;
      continue;
    }
    if (e.a_in.size() != parts || e.c_out.size() != parts)
      fail(errc::invalid_argument, "overlap entry: a_in/compute/c_out part counts differ");
    double in = shared_bus ? h2d_free : 0.0;
    double out_free = shared_bus ? d2h_free : 0.0;
    t.copy_in.start = in;
    in += e.b_in;
    double compute_end = in;
    for (std::size_t p = 0; p < parts; ++p) {
      in += e.a_in[p];
      const double cs = std::max(in, compute_end);
      compute_end = cs + e.compute[p];
      const double os = std::max(compute_end, out_free);
      out_free = os + e.c_out[p];
      if (p == 0) {
        t.compute.start = cs;
        t.copy_out.start = os;
      }
    }
    t.copy_in.end = in;
    t.compute.end = compute_end;
    t.copy_out.end = out_free;
    t.finish = out_free;
    if (shared_bus) {
      h2d_free = in;
      d2h_free = out_free;
    }
    makespan = std::max(makespan, t.finish);
  }
  return makespan;
}

std::vector<std::int64_t> overlap_row_parts(std::int64_t rows, int parts) {
  constexpr std::int64_t kBlock = 128;
  if (rows <= 0) return {};
  const std::int64_t blocks = rows / kBlock;
  const std::int64_t q = std::max<std::int64_t>(1, std::min<std::int64_t>(parts, blocks));
  if (blocks == 0) return {rows};
  std::vector<std::int64_t> out(static_cast<std::size_t>(q));
  for (std::int64_t p = 0; p < q; ++p)
    out[static_cast<std::size_t>(p)] = (blocks / q + (p < blocks % q ? 1 : 0)) * kBlock;
  out.back() += rows % kBlock;
  return out;
}

std::vector<std::int64_t> schedule_row_parts(const ScheduledDevice& device, const MatrixDims& dims) {
  if (device.rows <= 0) return {};
  const std::vector<Tile>& t = device.tiles;
  if (t.empty() || t[0].k <= 0 || dims.k % t[0].k != 0) return {device.rows};
  const std::size_t strips = static_cast<std::size_t>(dims.k / t[0].k);
  if (t.size() % strips != 0) return {device.rows};
  const std::size_t q = t.size() / strips;
  std::vector<std::int64_t> out;
  std::int64_t sum = 0;
  for (std::size_t p = 0; p < q; ++p) {
    if (t[p].m <= 0) return {device.rows};
    out.push_back(t[p].m);
    sum += t[p].m;
  }
  if (sum != device.rows) return {device.rows};
  return out;
}

Schedule build_overlap_schedule(const TilePlan& plan, const MachineProfile& machine, int parts) {
  validate_machine(machine);
  validate_dims(plan.dims);
  if (parts < 1) fail(errc::invalid_argument, "overlap needs at least one part");
  const std::size_t nd = machine.devices.size();
  if (plan.devices.size() != nd) fail(errc::invalid_argument, "plan/machine size mismatch");
  const MatrixDims& dims = plan.dims;
  std::int64_t covered = 0;
  for (std::size_t i = 0; i < nd; ++i) {
    if (plan.devices[i].device_id != machine.devices[i].id)
      fail(errc::invalid_argument, "plan/machine device order mismatch");
    covered += plan.devices[i].rows;
  }
  if (covered != dims.m) fail(errc::invalid_argument, "plan does not cover m");

  std::vector<OverlapEntry> entries(nd);
  std::vector<std::vector<Tile>> tiles(nd);
  for (std::size_t i = 0; i < nd; ++i) {
    const DeviceProfile& dev = machine.devices[i];
    const std::int64_t rows = plan.devices[i].rows;
    OverlapEntry& e = entries[i];
    e.priority = dev.priority;
    e.uses_bus = dev.uses_bus();
    tiles[i] = plan.devices[i].tiling.tiles;
    if (rows <= 0) continue;
    if (!dev.uses_bus()) {
      e.compute = {predicted_phase_durations(dev, rows, dims).compute};
      continue;
    }
    const double bw = dev.bandwidth;
    const double e_in = static_cast<double>(dev.elem_size);
    e.b_in = e_in * static_cast<double>(dims.k) * static_cast<double>(dims.n) / bw;
    tiles[i].clear();
    for (const std::int64_t r : overlap_row_parts(rows, parts)) {
      const OpsCount ops = static_cast<OpsCount>(r) * dims.row_ops();
      e.a_in.push_back(e_in * static_cast<double>(r) * static_cast<double>(dims.k) / bw);
      e.compute.push_back(predict_compute(dev, ops));
      e.c_out.push_back(4.0 * static_cast<double>(r) * static_cast<double>(dims.n) / bw);
      tiles[i].push_back({r, dims.k, dims.n});
    }
  }
  std::vector<DeviceTimeline> tl;
  const double makespan = evaluate_overlap_timeline(entries, machine.bus, &tl);

  Schedule s;
  s.machine_hash = machine_hash(machine);
  s.dims = dims;
  s.makespan = makespan;
  std::vector<std::size_t> order(nd);
  std::iota(order.begin(), order.end(), std::size_t{0});
  std::sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) {
    return machine.devices[a].priority < machine.devices[b].priority;
  });
  for (const std::size_t i : order) {
    ScheduledDevice d;
    d.id = machine.devices[i].id;
    d.priority = machine.devices[i].priority;
    d.rows = plan.devices[i].rows;
    d.tiles = std::move(tiles[i]);
    d.timeline = tl[i];
    s.devices.push_back(std::move(d));
  }
  return s;
}

Schedule plan_overlap(const MachineProfile& machine, const MatrixDims& dims) {
  Schedule best;
  double best_makespan = std::numeric_limits<double>::infinity();
  for (const TilePlan& full : subset_tile_plans(machine, dims)) {
    for (int parts = 1; parts <= 64; parts *= 2) {
      // A candidate must gain > 0.1%: per-part launch/copy latencies are
      // not modelled, so more parts (or fewer units) win only on a margin.
      Schedule s = build_overlap_schedule(full, machine, parts);
      if (s.makespan < best_makespan * (1.0 - 1e-3)) {
        best_makespan = s.makespan;
        best = std::move(s);
      }
    }
  }
  return best;
}

}  // namespace poas
