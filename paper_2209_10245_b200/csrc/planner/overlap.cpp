// Overlapped copies: link order, timeline, row parts x column panels and
// the "overlap" policy (see poas/overlap.hpp; B200 extension of
// PAPER.md:486-489).
#include "poas/overlap.hpp"

#include <algorithm>
#include <limits>
#include <numeric>

#include "poas/error.hpp"
#include "poas/policy.hpp"

namespace poas {

namespace {
constexpr std::int64_t kMinPanelCols = 4096;
// Fixed cost of one block's copy-out beyond its bytes (one stream wait + one
// 2-D copy): ~20 us measured past ~128 blocks (profiles/r01_overlap/
// grid_sweep.json: 64 x 8 blocks 37.5 ms vs 32 x 4 at 30.1 ms).
constexpr double kBlockCopyLatency = 20e-6;
}  // namespace

std::vector<OverlapItem> overlap_link_order(int parts, int panels) {
  std::vector<OverlapItem> out;
  int a = 0, b = 0;
  while (a < parts || b < panels) {
    // A while it is proportionally behind (a / parts <= b / panels)
    const bool take_a =
        b >= panels || (a < parts && static_cast<long long>(a) * panels <= static_cast<long long>(b) * parts);
    if (take_a)
      out.push_back({true, a++});
    else
      out.push_back({false, b++});
  }
  return out;
}

std::vector<OverlapBlock> overlap_block_order(int parts, int panels) {
  std::vector<OverlapBlock> out;
  int a = 0, b = 0;
  const std::vector<OverlapItem> order = overlap_link_order(parts, panels);
  for (std::size_t it = 0; it < order.size(); ++it) {
    const int item = static_cast<int>(it);
    if (order[it].a) {
      for (int j = 0; j < b; ++j) out.push_back({a, j, item});
      ++a;
    } else {
      for (int i = 0; i < a; ++i) out.push_back({i, b, item});
      ++b;
    }
  }
  return out;
}

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
  std::vector<double> landed;
  for (const std::size_t i : order) {
    const OverlapEntry& e = entries[i];
    DeviceTimeline& t = (*out)[i];
    const std::size_t blocks = e.compute.size();
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
    if (blocks == 0) {  // idle link unit: zero-length phases where its queue stands
      const double at = shared_bus ? h2d_free : 0.0;
      t.copy_in = t.compute = t.copy_out = {at, at};
      t.finish = at;
      continue;
    }
    if (e.ready.size() != blocks || e.c_out.size() != blocks)
      fail(errc::invalid_argument, "overlap entry: ready/compute/c_out block counts differ");
    double in = shared_bus ? h2d_free : 0.0;
    t.copy_in.start = in;
    landed.assign(e.link_in.size(), 0.0);
    for (std::size_t k = 0; k < e.link_in.size(); ++k) {
      in += e.link_in[k];
      landed[k] = in;
    }
    t.copy_in.end = in;
    double out_free = shared_bus ? d2h_free : 0.0;
    double compute_end = 0.0;
    for (std::size_t b = 0; b < blocks; ++b) {
      const int r = e.ready[b];
      if (r < 0 || static_cast<std::size_t>(r) >= landed.size())
        fail(errc::invalid_argument, "overlap entry: block ready item out of range");
      const double cs = std::max(landed[static_cast<std::size_t>(r)], compute_end);
      compute_end = cs + e.compute[b];
      const double os = std::max(compute_end, out_free);
      out_free = os + e.c_out[b];
      if (b == 0) {
        t.compute.start = cs;
        t.copy_out.start = os;
      }
    }
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

std::vector<std::int64_t> overlap_split(std::int64_t extent, int parts, std::int64_t block) {
  if (extent <= 0) return {};
  const std::int64_t blocks = extent / block;
  if (blocks == 0) return {extent};
  const std::int64_t q = std::max<std::int64_t>(1, std::min<std::int64_t>(parts, blocks));
  std::vector<std::int64_t> out(static_cast<std::size_t>(q));
  for (std::int64_t p = 0; p < q; ++p)
    out[static_cast<std::size_t>(p)] = (blocks / q + (p < blocks % q ? 1 : 0)) * block;
  out.back() += extent % block;
  return out;
}

std::vector<std::int64_t> overlap_row_parts(std::int64_t rows, int parts) {
  return overlap_split(rows, parts, 256);
}

std::vector<std::int64_t> overlap_col_panels(std::int64_t n, int panels) {
  return overlap_split(n, panels, 256);
}

RowColGrid schedule_grid(const ScheduledDevice& device, const MatrixDims& dims) {
  RowColGrid g;
  if (device.rows <= 0) return g;
  const RowColGrid whole{{device.rows}, {dims.n}};
  const std::vector<Tile>& t = device.tiles;
  if (t.empty() || t[0].k <= 0 || dims.k % t[0].k != 0) return whole;
  // panels: the leading tiles' widths until they cover n
  std::int64_t covered = 0;
  std::size_t q = 0;
  while (q < t.size() && covered < dims.n) {
    if (t[q].n <= 0) return whole;
    covered += t[q].n;
    ++q;
  }
  if (covered != dims.n || q == 0) return whole;
  const std::size_t strips = static_cast<std::size_t>(dims.k / t[0].k);
  if (t.size() % (strips * q) != 0) return whole;
  const std::size_t r = t.size() / (strips * q);  // row parts per strip
  for (std::size_t j = 0; j < q; ++j) g.panels.push_back(t[j].n);
  std::int64_t rows = 0;
  for (std::size_t p = 0; p < r; ++p) {
    for (std::size_t j = 0; j < q; ++j) {
      const Tile& x = t[p * q + j];
      if (x.m != t[p * q].m || x.n != g.panels[j] || x.m <= 0) return whole;
    }
    g.parts.push_back(t[p * q].m);
    rows += t[p * q].m;
  }
  if (rows != device.rows) return whole;
  return g;
}

std::vector<std::int64_t> schedule_row_parts(const ScheduledDevice& device, const MatrixDims& dims) {
  return schedule_grid(device, dims).parts;
}

Schedule build_overlap_schedule(const TilePlan& plan, const MachineProfile& machine, int parts,
                                int panels) {
  validate_machine(machine);
  validate_dims(plan.dims);
  if (parts < 1 || panels < 1) fail(errc::invalid_argument, "overlap needs at least one part and panel");
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
    const double es = static_cast<double>(dev.elem_size);
    const std::vector<std::int64_t> rp = overlap_row_parts(rows, parts);
    const std::vector<std::int64_t> cp = overlap_col_panels(dims.n, panels);
    for (const OverlapItem& it : overlap_link_order(static_cast<int>(rp.size()), static_cast<int>(cp.size())))
      e.link_in.push_back(es * static_cast<double>(dims.k) *
                          static_cast<double>(it.a ? rp[static_cast<std::size_t>(it.index)]
                                                   : cp[static_cast<std::size_t>(it.index)]) /
                          bw);
    for (const OverlapBlock& b : overlap_block_order(static_cast<int>(rp.size()), static_cast<int>(cp.size()))) {
      const double m = static_cast<double>(rp[static_cast<std::size_t>(b.part)]);
      const double w = static_cast<double>(cp[static_cast<std::size_t>(b.panel)]);
      e.ready.push_back(b.ready_item);
      e.compute.push_back(predict_compute(
          dev, static_cast<OpsCount>(rp[static_cast<std::size_t>(b.part)]) *
                   static_cast<OpsCount>(cp[static_cast<std::size_t>(b.panel)]) *
                   static_cast<OpsCount>(dims.k)));
      e.c_out.push_back(4.0 * m * w / bw + (rp.size() * cp.size() > 1 ? kBlockCopyLatency : 0.0));
    }
    tiles[i].clear();  // the R x Q grid, part-major
    for (const std::int64_t m : rp)
      for (const std::int64_t w : cp) tiles[i].push_back({m, dims.k, w});
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
    for (int panels = 1; panels <= 16; panels *= 2) {
      // Column panels no narrower than kMinPanelCols: a C block's rows are
      // separate DMA segments, and device->host copies of 4 KB segments run
      // at ~38 GB/s beside host->device traffic against ~48 GB/s for 16 KB
      // and ~50 GB/s contiguous (profiles/r01_overlap/pcie_calls.json) --
      // a per-segment cost the bandwidth model does not carry.
      if (panels > 1 && dims.n / panels < kMinPanelCols) break;
      for (int parts = 1; parts <= 64; parts *= 2) {
        // A candidate must gain > 0.1%: per-block launch/copy latencies are
        // not modelled, so more blocks (or fewer units) win only on a margin.
        Schedule s = build_overlap_schedule(full, machine, parts, panels);
        if (s.makespan < best_makespan * (1.0 - 1e-3)) {
          best_makespan = s.makespan;
          best = std::move(s);
        }
      }
    }
  }
  return best;
}

}  // namespace poas
