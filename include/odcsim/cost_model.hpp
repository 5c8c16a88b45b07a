// odcsim/cost_model.hpp — drop-in façade (B200 build) of the LB cost model
// (/root/reference/proj/include/odcsim/cost_model.hpp:10-39,
//  /root/reference/proj/src/cost_model.cpp:8-38).
// cost(s) = alpha*s*s + beta*s per layer (attention ~ L^2, dense ~ L).
#ifndef ODCSIM_COST_MODEL_HPP
#define ODCSIM_COST_MODEL_HPP

#include <span>

#include "odcsim/types.hpp"

namespace odcsim {

struct CostModel {
    double alpha = 1.0;  // quadratic (attention) coefficient
    double beta = 0.0;   // linear (dense layers) coefficient
    int layers = 1;
    void validate() const;  // ParamError unless alpha,beta >= 0, alpha+beta > 0, layers >= 1
};

struct MemoryBudget {
    Tokens max_tokens_per_microbatch = 0;  // activation-memory proxy
};

double compute_cost(const CostModel& model, Tokens s);                        // ParamError if s < 1
double microbatch_cost(const CostModel& model, std::span<const Tokens> lengths);  // sum; ParamError if empty
Tokens token_budget(Tokens max_len, double packing_ratio);                    // floor(max_len * ratio)
bool check_oom(std::span<const Tokens> lengths, const MemoryBudget& budget);  // token sum > budget

}  // namespace odcsim

#endif
