// Dynamic scheduling: model re-fit from measured executions and re-planning
// (see poas/dynamic.hpp).
#include "poas/dynamic.hpp"

#include <algorithm>
#include <cmath>
#include <utility>

#include "json_lite.hpp"
#include "poas/error.hpp"
#include "poas/policy.hpp"

namespace poas {
namespace {

// EWMA update of a measured/predicted ratio, clamped to one step.
bool update_factor(const PhaseError& e, const RefitOptions& o, double* g) {
  if (!(e.measured > 0.0) || !(e.predicted > 0.0) || !std::isfinite(e.measured) ||
      !std::isfinite(e.predicted))
    return false;
  const double r = e.measured / e.predicted;
  *g = std::clamp(1.0 + o.alpha * (r - 1.0), 1.0 / o.max_step, o.max_step);
  return true;
}

[[noreturn]] void bad_report(const std::string& what) {
  fail(errc::parse_failure, "execution report: " + what);
}

const json::Value& member(const json::Value& obj, const std::string& key) {
  const json::Value* v = obj.is_object() ? obj.get(key) : nullptr;
  if (!v) bad_report("missing \"" + key + "\"");
  return *v;
}

// A measured/predicted number; JSON null (a non-finite value) reads as 0,
// which the re-fit ignores.
double number(const json::Value& obj, const std::string& key) {
  const json::Value& v = member(obj, key);
  if (v.type == json::Value::Type::null) return 0.0;
  if (!v.is_number()) bad_report("\"" + key + "\" is not a number");
  return v.as_double();
}

PhaseError phase(const json::Value& dev, const std::string& key) {
  const json::Value& p = member(dev, key);
  return {number(p, "measured"), number(p, "predicted"), number(p, "error_pct")};
}

}  // namespace

SimulationResult parse_execution_report(const std::string& report_json) {
  const json::Value root = json::parse(report_json, "execution report");
  SimulationResult r;
  r.measured_makespan = number(root, "measured_makespan");
  r.predicted_makespan = number(root, "predicted_makespan");
  r.makespan_error_pct = number(root, "makespan_error_pct");
  const json::Value& devs = member(root, "devices");
  if (!devs.is_array()) bad_report("\"devices\" is not an array");
  for (const json::Value& d : devs.items) {
    DeviceOutcome o;
    const json::Value& id = member(d, "id");
    if (!id.is_string()) bad_report("device id is not a string");
    o.id = id.s;
    const json::Value& rows = member(d, "rows");
    if (!rows.is_integer()) bad_report("device rows is not an integer");
    o.rows = rows.as_int64();
    o.copy_in = phase(d, "copy_in");
    o.compute = phase(d, "compute");
    o.copy_out = phase(d, "copy_out");
    if (d.get("finish")) o.finish = phase(d, "finish");
    if (const json::Value* ov = d.get("overlapped")) {
      if (ov->type != json::Value::Type::boolean) bad_report("\"overlapped\" is not a boolean");
      o.overlapped = ov->b;
    }
    r.devices.push_back(std::move(o));
  }
  return r;
}

MachineProfile refit_profile(const MachineProfile& prior, const std::vector<DeviceOutcome>& observed,
                             const RefitOptions& options) {
  if (!(options.alpha > 0.0 && options.alpha <= 1.0))
    fail(errc::invalid_argument, "refit alpha must be in (0, 1]");
  if (!(options.max_step >= 1.0) || !std::isfinite(options.max_step))
    fail(errc::invalid_argument, "refit max_step must be a finite number >= 1");
  MachineProfile out = prior;
  for (const DeviceOutcome& o : observed) {
    DeviceProfile* d = nullptr;
    for (DeviceProfile& c : out.devices)
      if (c.id == o.id) d = &c;
    if (!d) fail(errc::missing_device, "refit: unit '" + o.id + "' is not in the profile");
    if (o.rows <= 0) continue;
    const double pred_link = o.copy_in.predicted + o.copy_out.predicted;
    const bool fused = d->uses_bus() && pred_link > 0.0 && o.copy_in.measured == 0.0 &&
                       o.copy_out.measured == 0.0;
    double g = 1.0;
    if (o.overlapped && d->uses_bus() && d->bandwidth > 0.0) {
      // Overlapped copies (poas/overlap.hpp): the phases are overlapping
      // spans, each paced by the others, and the link's two directions
      // contend while both are busy (measured: PCIe H2D 55 GB/s alone, ~45
      // GB/s beside a D2H stream). One factor moves the bound the plan
      // predicted: a link-bound unit's finish is B plus its busiest copy
      // stream, so its finish ratio rescales the link bandwidth; a
      // compute-bound unit's compute span is its back-to-back part GEMMs.
      const bool link_bound =
          std::max(o.copy_in.predicted, o.copy_out.predicted) >= o.compute.predicted;
      if (link_bound) {
        if (update_factor(o.finish, options, &g)) d->bandwidth /= g;
      } else if (update_factor(o.compute, options, &g)) {
        d->compute.slope *= g;
        d->compute.intercept *= g;
      }
      continue;
    }
    if (fused) {
      // Operands resident where the unit computes: the modelled link phases
      // happen inside the kernel (it streams its operands while computing),
      // so the measured compute phase stands for copy-in + compute +
      // copy-out. Move the compute model so the three predicted phases sum
      // to the measurement; the link model is left as profiled.
      // With the unit's finish measured (from its repeat's t0), its whole
      // predicted timeline -- compute and the modelled streaming of its
      // operands -- scales by the finish ratio: that also absorbs the
      // launch latency between t0 and the kernel's start (small GEMMs), and
      // converges for a unit whose time is mostly the operand stream (a
      // one-row CUDA-core share reads all of B; scaling compute alone would
      // need thousands of clamped steps).
      if (update_factor(o.finish, options, &g)) {
        d->compute.slope *= g;
        d->compute.intercept *= g;
        if (d->bandwidth > 0.0) d->bandwidth /= g;
        continue;
      }
      PhaseError whole;
      whole.measured = o.compute.measured;
      whole.predicted = o.compute.predicted + pred_link;
      double gw = 1.0;
      if (update_factor(whole, options, &gw) && o.compute.predicted > 0.0) {
        const double target = o.compute.predicted + (gw - 1.0) * whole.predicted;
        g = std::clamp(target / o.compute.predicted, 1.0 / options.max_step, options.max_step);
        d->compute.slope *= g;
        d->compute.intercept *= g;
      }
      continue;
    }
    if (update_factor(o.compute, options, &g)) {
      d->compute.slope *= g;
      d->compute.intercept *= g;
    }
    if (d->uses_bus() && d->bandwidth > 0.0) {
      PhaseError link;
      link.measured = o.copy_in.measured + o.copy_out.measured;
      link.predicted = o.copy_in.predicted + o.copy_out.predicted;
      if (update_factor(link, options, &g)) d->bandwidth /= g;
    }
  }
  validate_machine(out);
  return out;
}

DynamicScheduler::DynamicScheduler(MachineProfile prior, MatrixDims dims, DynamicOptions options)
    : profile_(std::move(prior)), dims_(dims), options_(std::move(options)) {
  if (!(options_.replan_threshold_pct >= 0.0))
    fail(errc::invalid_argument, "replan threshold must be >= 0");
  schedule_ = plan_with_policy(profile_, dims_, options_.policy);
}

const Schedule& DynamicScheduler::best_schedule() const {
  if (!(best_measured_ > 0.0)) return schedule_;
  bool same = best_.devices.size() == schedule_.devices.size();
  for (std::size_t i = 0; same && i < best_.devices.size(); ++i)
    same = best_.devices[i].id == schedule_.devices[i].id &&
           best_.devices[i].rows == schedule_.devices[i].rows;
  return same ? schedule_ : best_;
}

bool DynamicScheduler::observe(const SimulationResult& result) {
  const double t = result.measured_makespan;
  if (t > 0.0 && std::isfinite(t) && (best_measured_ <= 0.0 || t < best_measured_)) {
    best_ = schedule_;
    best_measured_ = t;
    best_observation_ = observations_;
  }
  profile_ = refit_profile(profile_, result.devices, options_.refit);
  ++observations_;
  if (!(std::fabs(result.makespan_error_pct) > options_.replan_threshold_pct)) return false;
  schedule_ = plan_with_policy(profile_, dims_, options_.policy);
  ++replans_;
  return true;
}

}  // namespace poas
