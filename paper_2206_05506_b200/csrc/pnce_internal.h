// Private interface between the library's translation units (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <string>

#include "../../include/pnce_b200.h"

namespace pnce_internal {

struct PlanView {
    pnce_cfg_t cfg;
    int n_batches;
    const float* chips;  // device [m], +-1
    void** synth_cache;  // per-plan state of the synthesiser (owned by pnce_synth.cu)
};

PlanView plan_view(const pnce_plan_t* plan);
void synth_cache_free(void* cache);  // called by pnce_plan_destroy
pnce_status_t set_error(pnce_status_t code, const std::string& msg);
void count_launch();
// 2-D row-major [rows][cols] 16-bit tensor map, box [box_rows][64 elements], 128B swizzle
// (the UMMA K-major operand layout the correlator uses).
pnce_status_t encode_tmap_k16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                              int bf16);

}  // namespace pnce_internal
