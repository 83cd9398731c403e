// C-ABI: plan, predict and execute entry points (include/poas_b200.h).
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "capi_util.hpp"
#include "comm.hpp"
#include "host_gemm.hpp"
#include "host_rng.hpp"
#include "poas/adapter.hpp"
#include "poas/dynamic.hpp"
#include "poas/error.hpp"
#include "poas/executor.hpp"
#include "poas/optimizer.hpp"
#include "poas/policy.hpp"
#include "poas/profiler.hpp"
#include "poas/scheduler.hpp"
#include "poas_b200.h"
#include "units.hpp"

using poas_b200::capi::dup_string;
using poas_b200::capi::guard;
using poas_b200::capi::json_escape;
using poas_b200::capi::raise;

struct poas_unit_s {
  std::unique_ptr<poas_b200::Unit> unit;
};

struct poas_executor_s {
  std::unique_ptr<poas::Executor> ex;
};

namespace {

poas::MatrixDims dims_of(int64_t m, int64_t n, int64_t k) {
  poas::MatrixDims d{m, n, k};
  poas::validate_dims(d);
  return d;
}

std::string need_str(const char* s, const char* what) {
  if (!s) raise(POAS_E_INVALID_ARGUMENT, std::string(what) + " is NULL");
  return s;
}

template <class P>
void need_ptr(P* p, const char* what) {
  if (!p) raise(POAS_E_INVALID_ARGUMENT, std::string(what) + " is NULL");
}

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string iv(const poas::Interval& i) { return "[" + g17(i.start) + ", " + g17(i.end) + "]"; }

std::string split_json(const poas::WorkloadSplit& s) {
  std::string o = "{\"makespan\": " + g17(s.makespan) + ", \"lp_objective\": " +
                  g17(s.lp_objective) + ", \"lp_iterations\": " + std::to_string(s.lp_iterations) +
                  ", \"shares\": [";
  for (std::size_t i = 0; i < s.shares.size(); ++i) {
    const poas::DeviceShare& d = s.shares[i];
    o += (i ? ", " : "");
    o += "{\"id\": \"" + d.device_id + "\", \"rows\": " + std::to_string(d.rows) +
         ", \"ops\": " + std::to_string(d.ops) + ", \"fraction\": " + g17(d.fraction) +
         ", \"copy_in\": " + iv(d.timeline.copy_in) + ", \"compute\": " + iv(d.timeline.compute) +
         ", \"copy_out\": " + iv(d.timeline.copy_out) + ", \"finish\": " + g17(d.timeline.finish) +
         "}";
  }
  return o + "]}";
}

std::string tile_plan_json(const poas::TilePlan& p) {
  std::string o = "{\"devices\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) {
    const poas::PlannedDevice& d = p.devices[i];
    o += (i ? ", " : "");
    o += "{\"id\": \"" + d.device_id + "\", \"rows\": " + std::to_string(d.rows) +
         ", \"k_prime\": " + std::to_string(d.tiling.k_prime) + ", \"sq\": " + g17(d.tiling.sq) +
         ", \"window_fallback\": " + (d.window_fallback ? "true" : "false") + ", \"tiles\": [";
    for (std::size_t t = 0; t < d.tiling.tiles.size(); ++t) {
      const poas::Tile& x = d.tiling.tiles[t];
      o += (t ? ", " : "");
      o += "[" + std::to_string(x.m) + ", " + std::to_string(x.k) + ", " + std::to_string(x.n) + "]";
    }
    o += "]}";
  }
  return o + "]}";
}


poas::GemmOperands operands_of(const poas_gemm_io& io) {
  poas::GemmOperands op;
  op.m = io.m;
  op.n = io.n;
  op.k = io.k;
  op.a_host = io.a_host;
  op.lda_host = io.lda_host;
  op.b_host = io.b_host;
  op.ldb_host = io.ldb_host;
  op.c_host = io.c_host;
  op.ldc_host = io.ldc_host;
  op.a_dev = io.a_dev;
  op.lda_dev = io.lda_dev;
  op.b_dev = io.b_dev;
  op.ldb_dev = io.ldb_dev;
  op.a16_dev = io.a16_dev;
  op.lda16_dev = io.lda16_dev;
  op.b16_dev = io.b16_dev;
  op.ldb16_dev = io.ldb16_dev;
  op.c_dev = io.c_dev;
  op.ldc_dev = io.ldc_dev;
  op.resident = io.resident != 0;
  op.b_panels = io.b_panels;
  op.b_ready = io.b_ready;
  op.b_flags = io.b_flags;
  op.b_epoch = io.b_epoch;
  op.a16_host = io.a16_host;
  op.lda16_host = io.lda16_host;
  op.b16_host = io.b16_host;
  op.ldb16_host = io.ldb16_host;
  op.comm = io.comm ? io.comm->comm.get() : nullptr;
  op.b_transport = io.b_transport;
  return op;
}

poas::ProfilingConfig parse_profiling(const char* text) {
  poas::ProfilingConfig c;
  if (!text) return c;
  std::stringstream in(text);
  std::string item;
  while (std::getline(in, item, ',')) {
    if (item.empty()) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) poas::fail(poas::errc::invalid_argument, "profiling: bad item " + item);
    const std::string k = item.substr(0, eq);
    const long long v = std::stoll(item.substr(eq + 1));
    if (k == "probes") c.probes = static_cast<int>(v);
    else if (k == "repetitions") c.repetitions = static_cast<int>(v);
    else if (k == "cpu_min_side") c.cpu_range.min_side = v;
    else if (k == "cpu_max_side") c.cpu_range.max_side = v;
    else if (k == "accel_min_side") c.accel_range.min_side = v;
    else if (k == "accel_max_side") c.accel_range.max_side = v;
    else if (k == "bandwidth_payload") c.bandwidth_payload = static_cast<std::uint64_t>(v);
    else poas::fail(poas::errc::invalid_argument, "profiling: unknown key " + k);
  }
  poas::validate_profiling_config(c);
  return c;
}

std::uint64_t llc_bytes() {
  const long v = sysconf(_SC_LEVEL3_CACHE_SIZE);
  return v > 0 ? static_cast<std::uint64_t>(v) : (32ULL << 20);
}

}  // namespace

namespace poas_b200 {

// profile_machine (reference proj/src/simulator.cpp:53-74) over real units.
poas::MachineProfile profile_units(const std::vector<std::unique_ptr<Unit>>& units,
                                   const poas::ProfilingConfig& cfg, bool bus) {
  std::vector<poas::DeviceProbeData> probes;
  std::vector<poas::SideRange> ranges;
  for (const auto& u : units) {
    poas::DeviceProbeData p;
    p.id = u->spec().id;
    p.kind = u->spec().kind;
    p.elem_size = u->spec().elem;
    poas::SideRange range = cfg.range_for(p.kind);
    if (u->spec().probe_min > 0) range = {u->spec().probe_min, u->spec().probe_max};
    ranges.push_back(range);
    p.samples = poas::run_compute_probes(*u, range, cfg.probes, cfg.repetitions);
    if (u->has_transfers())
      p.bandwidth = poas::run_bandwidth_probe(*u, cfg.bandwidth_payload, cfg.repetitions);
    if (p.kind == poas::DeviceKind::xpu) p.align = u->spec().align;
    if (p.kind == poas::DeviceKind::cpu) p.cache_bytes = llc_bytes();
    probes.push_back(std::move(p));
  }
  return poas::fit_machine_ranges(probes, bus, cfg, ranges);
}

}  // namespace poas_b200

extern "C" {

int poas_b200_plan(const char* profile_text, int64_t m, int64_t n, int64_t k,
                   char** schedule_json) {
  return guard([&] {
    need_ptr(schedule_json, "schedule_json");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::MatrixDims d = dims_of(m, n, k);
    const poas::WorkloadSplit split = poas::solve_split(machine, d);
    const poas::TilePlan plan = poas::build_tile_plan(machine, d, split);
    *schedule_json = dup_string(poas::format_schedule(poas::build_schedule(plan, machine)));
  });
}

int poas_b200_plan_policy(const char* profile_text, int64_t m, int64_t n, int64_t k,
                          const char* policy, char** schedule_json) {
  return guard([&] {
    need_ptr(schedule_json, "schedule_json");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    *schedule_json = dup_string(poas::format_schedule(
        poas::plan_with_policy(machine, dims_of(m, n, k), policy ? policy : "")));
  });
}

int poas_b200_plan_partitions(const char* profile_text, int64_t m, int64_t n, int64_t k,
                              const char* tc_id, int tc_sms, const char* simt_id, int simt_sms,
                              const int* simt_budgets, int count, const char* policy,
                              char** out_json) {
  return guard([&] {
    need_ptr(out_json, "out_json");
    if (count < 1 || !simt_budgets) raise(POAS_E_INVALID_ARGUMENT, "no candidate budgets");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    const std::vector<int> budgets(simt_budgets, simt_budgets + count);
    const poas::PartitionChoice c = poas::plan_sm_partitions(
        machine, dims_of(m, n, k), need_str(tc_id, "tc_id"), tc_sms, need_str(simt_id, "simt_id"),
        simt_sms, budgets, policy ? policy : "");
    std::string o = "{\"best\": " + std::to_string(c.best) + ", \"candidates\": [";
    for (std::size_t i = 0; i < c.candidates.size(); ++i) {
      const poas::PartitionCandidate& x = c.candidates[i];
      o += std::string(i ? ", " : "") + "{\"simt_sms\": " + std::to_string(x.simt_sms) +
           ", \"tc_sms\": " + std::to_string(x.tc_sms) + ", \"makespan\": " + g17(x.schedule.makespan) +
           ", \"rows\": {";
      for (std::size_t j = 0; j < x.schedule.devices.size(); ++j)
        o += std::string(j ? ", " : "") + "\"" + json_escape(x.schedule.devices[j].id) +
             "\": " + std::to_string(x.schedule.devices[j].rows);
      o += "}}";
    }
    o += "]}";
    *out_json = dup_string(o);
  });
}

int poas_b200_plan_standalone(const char* profile_text, const char* device_id, int64_t m,
                              int64_t n, int64_t k, char** schedule_json) {
  return guard([&] {
    need_ptr(schedule_json, "schedule_json");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    *schedule_json = dup_string(poas::format_schedule(
        poas::standalone_schedule(machine, need_str(device_id, "device_id"), dims_of(m, n, k))));
  });
}

int poas_b200_split(const char* profile_text, int64_t m, int64_t n, int64_t k, char** out) {
  return guard([&] {
    need_ptr(out, "out");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    *out = dup_string(split_json(poas::solve_split(machine, dims_of(m, n, k))));
  });
}

int poas_b200_oracle_split(const char* profile_text, int64_t m, int64_t n, int64_t k,
                           int64_t resolution, int parallel, char** out) {
  return guard([&] {
    need_ptr(out, "out");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::MatrixDims d = dims_of(m, n, k);
    *out = dup_string(split_json(parallel ? poas::oracle_grid_search(machine, d, resolution)
                                          : poas::oracle_grid_search_serial(machine, d, resolution)));
  });
}

int poas_b200_tile_plan(const char* profile_text, int64_t m, int64_t n, int64_t k,
                        const int64_t* rows, size_t count, char** out) {
  return guard([&] {
    need_ptr(out, "out");
    need_ptr(rows, "rows");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::MatrixDims d = dims_of(m, n, k);
    const std::vector<std::int64_t> r(rows, rows + count);
    const poas::WorkloadSplit split = poas::evaluate_rows(machine, d, r);
    *out = dup_string(tile_plan_json(poas::build_tile_plan(machine, d, split)));
  });
}

int poas_b200_schedule_roundtrip(const char* schedule_json, char** canonical_json) {
  return guard([&] {
    need_ptr(canonical_json, "out");
    *canonical_json = dup_string(
        poas::format_schedule(poas::parse_schedule(need_str(schedule_json, "schedule"))));
  });
}

int poas_b200_profile_roundtrip(const char* profile_text, char** canonical_text) {
  return guard([&] {
    need_ptr(canonical_text, "out");
    *canonical_text =
        dup_string(poas::format_profile(poas::parse_profile(need_str(profile_text, "profile"))));
  });
}

int poas_b200_machine_hash(const char* profile_text, char out[17]) {
  return guard([&] {
    need_ptr(out, "out");
    const std::string h = poas::machine_hash(poas::parse_profile(need_str(profile_text, "profile")));
    std::memcpy(out, h.c_str(), 17);
  });
}

int poas_b200_fit_linear(const uint64_t* ops, const double* seconds, size_t count, double* slope,
                         double* intercept) {
  return guard([&] {
    need_ptr(slope, "slope");
    need_ptr(intercept, "intercept");
    if (count && (!ops || !seconds)) raise(POAS_E_INVALID_ARGUMENT, "samples are NULL");
    std::vector<poas::ModelSample> s;
    for (size_t i = 0; i < count; ++i) s.push_back({ops[i], seconds[i]});
    const poas::LinearModel mdl = poas::fit_linear(s);
    *slope = mdl.slope;
    *intercept = mdl.intercept;
  });
}

int poas_b200_transfer_bytes(const char* profile_text, const char* device_id, uint64_t ops,
                             int64_t m, int64_t n, int64_t k, uint64_t* in_bytes,
                             uint64_t* out_bytes) {
  return guard([&] {
    need_ptr(in_bytes, "in_bytes");
    need_ptr(out_bytes, "out_bytes");
    const poas::MachineProfile machine = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::DeviceProfile* dev = machine.find(need_str(device_id, "device_id"));
    if (!dev) poas::fail(poas::errc::missing_device, "no device '" + std::string(device_id) + "'");
    const poas::TransferBytes tb = poas::transfer_bytes(*dev, ops, dims_of(m, n, k));
    *in_bytes = tb.in;
    *out_bytes = tb.out;
  });
}

int poas_b200_simplex(int num_vars, const double* objective, int n_eq, const double* eq_a,
                      const double* eq_b, int n_ge, const double* ge_a, const double* ge_b,
                      double* x_out, double* objective_out, long* iterations_out) {
  return guard([&] {
    if (num_vars < 0 || n_eq < 0 || n_ge < 0) raise(POAS_E_INVALID_ARGUMENT, "negative sizes");
    need_ptr(objective, "objective");
    need_ptr(x_out, "x_out");
    poas::SimplexProblem p;
    p.num_vars = num_vars;
    p.objective.assign(objective, objective + num_vars);
    for (int i = 0; i < n_eq; ++i) {
      p.eq_a.emplace_back(eq_a + static_cast<size_t>(i) * num_vars,
                          eq_a + static_cast<size_t>(i + 1) * num_vars);
      p.eq_b.push_back(eq_b[i]);
    }
    for (int i = 0; i < n_ge; ++i) {
      p.ge_a.emplace_back(ge_a + static_cast<size_t>(i) * num_vars,
                          ge_a + static_cast<size_t>(i + 1) * num_vars);
      p.ge_b.push_back(ge_b[i]);
    }
    const poas::SimplexSolution s = poas::solve_simplex(p);
    std::memcpy(x_out, s.x.data(), sizeof(double) * static_cast<size_t>(num_vars));
    if (objective_out) *objective_out = s.objective;
    if (iterations_out) *iterations_out = s.iterations;
  });
}

int poas_b200_unit_create(const char* spec, poas_unit_t* out) {
  return guard([&] {
    need_ptr(out, "out");
    auto h = std::make_unique<poas_unit_s>();
    h->unit = std::make_unique<poas_b200::Unit>(poas_b200::parse_unit_spec(need_str(spec, "spec")));
    *out = h.release();
  });
}

void poas_b200_unit_destroy(poas_unit_t unit) { delete unit; }

int poas_b200_time_gemm(poas_unit_t unit, int64_t side, double* seconds) {
  return guard([&] {
    need_ptr(unit, "unit");
    need_ptr(seconds, "seconds");
    *seconds = unit->unit->time_gemm(side);
  });
}

int poas_b200_time_transfer(poas_unit_t unit, uint64_t bytes, double* seconds) {
  return guard([&] {
    need_ptr(unit, "unit");
    need_ptr(seconds, "seconds");
    *seconds = unit->unit->time_transfer(bytes);
  });
}

int poas_b200_has_transfers(poas_unit_t unit) { return unit && unit->unit->has_transfers() ? 1 : 0; }

int poas_b200_profile_machine(const char* units, const char* profiling, int bus,
                              char** profile_text) {
  return guard([&] {
    need_ptr(profile_text, "profile_text");
    std::vector<std::unique_ptr<poas_b200::Unit>> us;
    for (const auto& s : poas_b200::parse_unit_list(need_str(units, "units")))
      us.push_back(std::make_unique<poas_b200::Unit>(s));
    const poas::MachineProfile m = poas_b200::profile_units(us, parse_profiling(profiling), bus != 0);
    *profile_text = dup_string(poas::format_profile(m));
  });
}

int poas_b200_profile_backends(const poas_probe_backend* backends, size_t count,
                               const char* profiling, int bus, char** profile_text) {
  // A DeviceBackend over the caller's callbacks (reference backend.hpp:11-24).
  class CallbackBackend final : public poas::DeviceBackend {
   public:
    explicit CallbackBackend(const poas_probe_backend& b) : b_(b) {}
    double time_gemm(std::int64_t side) override { return b_.time_gemm(b_.ctx, side); }
    double time_transfer(std::uint64_t bytes) override { return b_.time_transfer(b_.ctx, bytes); }
    bool has_transfers() const override { return b_.time_transfer != nullptr; }

   private:
    const poas_probe_backend& b_;
  };
  return guard([&] {
    need_ptr(profile_text, "profile_text");
    if (count == 0) raise(POAS_E_INVALID_ARGUMENT, "no backends");
    need_ptr(backends, "backends");
    const poas::ProfilingConfig cfg = parse_profiling(profiling);
    std::vector<poas::DeviceProbeData> probes;
    std::vector<poas::SideRange> ranges;
    for (size_t i = 0; i < count; ++i) {
      const poas_probe_backend& b = backends[i];
      if (!b.time_gemm) raise(POAS_E_INVALID_ARGUMENT, "backend without time_gemm");
      if (b.kind < POAS_KIND_CPU || b.kind > POAS_KIND_XPU) raise(POAS_E_INVALID_ARGUMENT, "bad kind");
      poas::DeviceProbeData p;
      p.id = need_str(b.id, "id");
      p.kind = b.kind == POAS_KIND_CPU   ? poas::DeviceKind::cpu
               : b.kind == POAS_KIND_GPU ? poas::DeviceKind::gpu
                                         : poas::DeviceKind::xpu;
      p.elem_size = b.elem_size;
      poas::SideRange range = cfg.range_for(p.kind);
      if (b.probe_min_side > 0 && b.probe_max_side > 0) range = {b.probe_min_side, b.probe_max_side};
      ranges.push_back(range);
      CallbackBackend be(b);
      p.samples = poas::run_compute_probes(be, range, cfg.probes, cfg.repetitions);
      if (be.has_transfers())
        p.bandwidth = poas::run_bandwidth_probe(be, cfg.bandwidth_payload, cfg.repetitions);
      if (p.kind == poas::DeviceKind::xpu) p.align = b.align;
      if (p.kind == poas::DeviceKind::cpu) p.cache_bytes = b.cache_bytes;
      if (b.priority >= 0) p.fixed_priority = b.priority;
      probes.push_back(std::move(p));
    }
    *profile_text = dup_string(poas::format_profile(poas::fit_machine_ranges(probes, bus != 0, cfg, ranges)));
  });
}

int poas_b200_executor_create(const char* units, poas_executor_t* out) {
  return guard([&] {
    need_ptr(out, "out");
    auto h = std::make_unique<poas_executor_s>();
    h->ex = std::make_unique<poas::Executor>(need_str(units, "units"));
    *out = h.release();
  });
}

void poas_b200_executor_destroy(poas_executor_t ex) { delete ex; }

int poas_b200_execute(poas_executor_t ex, const char* schedule_json, const poas_gemm_io* io,
                      int repeats, char** report_json) {
  return guard([&] {
    need_ptr(ex, "executor");
    need_ptr(io, "io");
    const poas::Schedule s = poas::parse_schedule(need_str(schedule_json, "schedule"));
    const poas::SimulationResult r = ex->ex->run(s, operands_of(*io), repeats);
    if (report_json) *report_json = dup_string(poas::format_execution_report(s, r));
  });
}

int poas_b200_profile_splice_unit(const char* profile_text, const char* unit_profile_text,
                                  const char* unit_id, char** out_profile) {
  return guard([&] {
    need_ptr(out_profile, "out_profile");
    poas::MachineProfile m = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::MachineProfile u = poas::parse_profile(need_str(unit_profile_text, "unit profile"));
    const std::string id = need_str(unit_id, "unit_id");
    const poas::DeviceProfile* src = u.find(id);
    poas::DeviceProfile* dst = nullptr;
    for (poas::DeviceProfile& d : m.devices)
      if (d.id == id) dst = &d;
    if (!src || !dst) raise(POAS_E_INVALID_ARGUMENT, "splice: unit '" + id + "' missing");
    if (src->kind != dst->kind) raise(POAS_E_INVALID_ARGUMENT, "splice: unit kinds differ");
    dst->compute = src->compute;
    dst->bandwidth = src->bandwidth;
    dst->ops_min = src->ops_min;
    dst->ops_max = src->ops_max;
    poas::validate_machine(m);
    *out_profile = dup_string(poas::format_profile(m));
  });
}

int poas_b200_refit_profile(const char* profile_text, const char* report_json, double alpha,
                            char** out_profile) {
  return guard([&] {
    need_ptr(out_profile, "out_profile");
    const poas::MachineProfile prior = poas::parse_profile(need_str(profile_text, "profile"));
    const poas::SimulationResult r =
        poas::parse_execution_report(need_str(report_json, "report_json"));
    poas::RefitOptions opt;
    opt.alpha = alpha;
    *out_profile = dup_string(poas::format_profile(poas::refit_profile(prior, r.devices, opt)));
  });
}

int poas_b200_run_dynamic(poas_executor_t ex, const char* profile_text, int64_t m, int64_t n,
                          int64_t k, const char* policy, const poas_gemm_io* io, int iterations,
                          int repeats, double alpha, double replan_threshold_pct,
                          char** out_json) {
  return guard([&] {
    need_ptr(ex, "executor");
    need_ptr(io, "io");
    need_ptr(out_json, "out_json");
    if (iterations < 1) raise(POAS_E_INVALID_ARGUMENT, "iterations must be >= 1");
    if (repeats < 1) raise(POAS_E_INVALID_ARGUMENT, "repeats must be >= 1");
    poas::DynamicOptions opt;
    opt.refit.alpha = alpha;
    opt.replan_threshold_pct = replan_threshold_pct;
    if (policy) opt.policy = policy;
    poas::DynamicScheduler dyn(poas::parse_profile(need_str(profile_text, "profile")),
                               dims_of(m, n, k), opt);
    const poas::GemmOperands op = operands_of(*io);
    std::string o = "{\n  \"iterations\": [\n";
    bool replanned = false;
    for (int it = 0; it < iterations; ++it) {
      const poas::SimulationResult r = ex->ex->run(dyn.schedule(), op, repeats);
      o += "    {\"iteration\": " + std::to_string(it) +
           ", \"replanned\": " + (replanned ? "true" : "false") + ", \"rows\": {";
      for (std::size_t i = 0; i < r.devices.size(); ++i)
        o += (i ? ", \"" : "\"") + json_escape(r.devices[i].id) +
             "\": " + std::to_string(r.devices[i].rows);
      o += "}, \"predicted_makespan\": " + g17(r.predicted_makespan) +
           ", \"measured_makespan\": " + g17(r.measured_makespan) +
           ", \"makespan_error_pct\": " + g17(r.makespan_error_pct) + "}";
      o += it + 1 < iterations ? ",\n" : "\n";
      replanned = dyn.observe(r);
    }
    o += "  ],\n  \"replans\": " + std::to_string(dyn.replans()) + ",\n";
    o += "  \"profile\": \"" + json_escape(poas::format_profile(dyn.profile())) + "\",\n";
    // the fastest measured plan (the last re-plan may be unmeasured, and a
    // plan from a re-fit can be slower than the one it replaced)
    o += "  \"best_iteration\": " + std::to_string(dyn.best_observation()) + ",\n";
    o += "  \"last_schedule\": " + poas::format_schedule(dyn.schedule()) + ",\n";
    o += "  \"schedule\": " + poas::format_schedule(dyn.best_schedule()) + "}\n";
    *out_json = dup_string(o);
  });
}

int poas_b200_executor_hash(poas_executor_t ex, char out[17]) {
  return guard([&] {
    need_ptr(ex, "executor");
    need_ptr(out, "out");
    std::memcpy(out, ex->ex->machine_hash().c_str(), 17);
  });
}

int poas_b200_host_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
                        const float* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                        int threads) {
  return guard([&] {
    if (m > 0 && n > 0 && k > 0 && (!a || !b || !c))
      raise(POAS_E_INVALID_ARGUMENT, "host_gemm: NULL operand");
    poas_b200::host_gemm(m, n, k, a, lda, b, ldb, c, ldc, accumulate != 0, threads);
  });
}

int poas_b200_fill_uniform_host(float* dst, int64_t ld, int64_t rows, int64_t cols, int64_t row0,
                                int64_t col0, int64_t total_cols, uint64_t seed) {
  return guard([&] {
    if (rows > 0 && cols > 0) need_ptr(dst, "dst");
    poas_b200::fill_uniform_host(dst, ld, rows, cols, row0, col0, total_cols, seed);
  });
}

uint64_t poas_b200_stream_seed(uint64_t master_seed, const char* name) {
  return poas::Rng::for_stream(master_seed, name ? name : "").state();
}

}  // extern "C"
