#pragma once
// Dynamic scheduling (paper §3.4.2): keep measuring the
// executions, adapt the performance model, re-optimize. The reference ships
// only the static scheduler; this is the rebuild's extension (SURVEY.md
// §8f-4). The re-fit works on the per-phase measured/predicted pairs the
// executor reports (SimulationResult, the shape of proj/src/simulator.cpp:
// 104-209), so any executor that fills that result drives it.
//
// Model update. A unit's measured/predicted compute ratio r scales its whole
// linear model (slope and intercept) by g = 1 + alpha (r - 1): clock and
// power-cap drift stretch every probe by the same factor, so the fitted shape
// is kept and only its scale follows the evidence (EWMA with weight alpha).
// Link bandwidth is divided by the same update of the copy-phase ratio
// (overlapped runs, poas/overlap.hpp: by the finish ratio of a link-bound
// unit, see refit_profile). A
// bus unit whose copy phases were predicted but measured as zero ran on
// resident operands: its kernel streams them while computing, so its
// measured compute stands for all three phases and only the compute model
// moves (to make the three predicted phases add up to the measurement).
// Priorities, ops windows, align and elem_size are left as profiled, so the
// machine hash (identity only) is unchanged and re-planned schedules still run
// on the same executor.

#include <string>
#include <vector>

#include "poas/device_model.hpp"
#include "poas/executor.hpp"
#include "poas/scheduler.hpp"

namespace poas {

struct RefitOptions {
  double alpha = 0.5;     // weight of the newest observation, (0, 1]
  double max_step = 4.0;  // one update scales a model by at most this factor (or its inverse)
};

// `prior` with every observed unit's model moved toward its measurement.
// Units with no rows, or phases with a zero measured/predicted time, are left
// unchanged. An id not in `prior` is errc::missing_device.
MachineProfile refit_profile(const MachineProfile& prior, const std::vector<DeviceOutcome>& observed,
                             const RefitOptions& options = {});

// Inverse of format_execution_report (poas/executor.hpp) for the fields the
// re-fit reads: devices[] {id, rows, copy_in, compute, copy_out} and the
// makespan triple. errc::parse_failure on malformed or incomplete reports.
SimulationResult parse_execution_report(const std::string& report_json);

struct DynamicOptions {
  RefitOptions refit;
  double replan_threshold_pct = 2.0;  // re-plan when |makespan error| exceeds this
  std::string policy = "reference";   // planner policy (poas/policy.hpp)
};

class DynamicScheduler {
 public:
  DynamicScheduler(MachineProfile prior, MatrixDims dims, DynamicOptions options = {});

  const Schedule& schedule() const { return schedule_; }
  const MachineProfile& profile() const { return profile_; }
  int replans() const { return replans_; }
  int observations() const { return observations_; }

  // Feed the result of running schedule(). The model is always re-fitted;
  // the schedule is re-planned when the result's |makespan_error_pct| exceeds
  // the threshold. Returns true when it re-planned (schedule() replaced).
  bool observe(const SimulationResult& result);

  // The fastest schedule measured so far (schedule() before any
  // observation). schedule() after a re-plan has not been measured yet, and
  // a plan derived from a re-fit can be worse than the one it replaces, so
  // the adapt step hands this one to the run that follows.
  // When the latest plan splits the rows exactly as the fastest one did, the
  // latest is returned: same work, prediction from the latest re-fit.
  const Schedule& best_schedule() const;
  double best_measured_makespan() const { return best_measured_; }
  int best_observation() const { return best_observation_; }

 private:
  MachineProfile profile_;
  MatrixDims dims_;
  DynamicOptions options_;
  Schedule schedule_;
  Schedule best_;
  double best_measured_ = 0.0;
  int best_observation_ = -1;
  int replans_ = 0;
  int observations_ = 0;
};

}  // namespace poas
