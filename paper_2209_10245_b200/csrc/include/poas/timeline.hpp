#pragma once
// The makespan semantics shared by planner, scheduler, exhaustive search and
// executor report (reference: proj/include/poas/timeline.hpp).
//
// Shared link, units taken by ascending priority: copy-ins back to back from
// 0; compute right after the unit's own copy-in; copy-outs back to back in
// the same order, the first one not before the last copy-in ended. Private
// links: every unit copies in from 0 and copies out right after computing.
// Units without a link (cpu) neither copy nor occupy the link.

#include <cstddef>
#include <vector>

namespace poas {

struct Interval {
  double start = 0.0;
  double end = 0.0;
  double duration() const { return end - start; }
};

struct DeviceTimeline {
  Interval copy_in;
  Interval compute;
  Interval copy_out;
  double finish = 0.0;
};

struct TimelineEntry {
  int priority = 0;
  bool uses_bus = false;
  double copy_in = 0.0;
  double compute = 0.0;
  double copy_out = 0.0;
};

// Writes `count` timelines into `out` (input order); returns the makespan.
double evaluate_timeline_into(const TimelineEntry* entries, std::size_t count, bool shared_bus,
                              DeviceTimeline* out);

struct TimelineResult {
  std::vector<DeviceTimeline> devices;
  double makespan = 0.0;
};

TimelineResult evaluate_timeline(const std::vector<TimelineEntry>& entries, bool shared_bus);

}  // namespace poas
