#pragma once
// Planner policies. "reference" (default) is the reference pipeline,
// byte-identical plans; "best-subset" is an opt-in B200 extension that also
// considers leaving units idle (see csrc/planner/policy.cpp).

#include <string>

#include "poas/device_model.hpp"
#include "poas/scheduler.hpp"

namespace poas {

Schedule plan_schedule(const MachineProfile& machine, const MatrixDims& dims);
Schedule plan_best_subset(const MachineProfile& machine, const MatrixDims& dims);
Schedule plan_with_policy(const MachineProfile& machine, const MatrixDims& dims,
                          const std::string& policy);

}  // namespace poas
