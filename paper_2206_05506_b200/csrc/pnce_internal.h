// Private interface between the library's translation units (not part of the C ABI).
#pragma once
#include <string>

#include "../../include/pnce_b200.h"

namespace pnce_internal {

struct PlanView {
    pnce_cfg_t cfg;
    int n_batches;
    const float* chips;  // device [m], +-1
};

PlanView plan_view(const pnce_plan_t* plan);
pnce_status_t set_error(pnce_status_t code, const std::string& msg);
void count_launch();

}  // namespace pnce_internal
