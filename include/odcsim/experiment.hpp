// odcsim/experiment.hpp — drop-in façade (B200 build). Only the plan
// serialiser of the reference's experiment module is on the hot path
// (/root/reference/proj/src/experiment.cpp:215-233): it is the fixture format
// for bit-exact load-balancer parity. The string form is byte-identical to
// nlohmann::json::dump(); the json form is provided when nlohmann is on the
// include path, as in the reference.
#ifndef ODCSIM_EXPERIMENT_HPP
#define ODCSIM_EXPERIMENT_HPP

#include <string>

#include "odcsim/partition.hpp"

#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define ODCSIM_HAVE_NLOHMANN 1
#endif

namespace odcsim {

std::string solutions_to_json_string(const PlanResult& plan_result);

#ifdef ODCSIM_HAVE_NLOHMANN
inline nlohmann::json solutions_to_json(const PlanResult& plan_result) {
    return nlohmann::json::parse(solutions_to_json_string(plan_result));
}
#endif

}  // namespace odcsim

#endif
