// ctx.h — internal accessors shared by ctx.cu and planner.cpp.
#pragma once

#include "pushplan_gpu.h"

namespace ppg {
struct SimHook {
  ppg_simulate_fn fn;
  void* user;
};
SimHook ctx_sim_hook(const ppg_ctx* ctx);
const ppg_params& ctx_params(const ppg_ctx* ctx);
int ctx_n_objects(const ppg_ctx* ctx);
int ctx_planner(const ppg_ctx* ctx);
void ctx_set_error(ppg_ctx* ctx, const char* msg);
}  // namespace ppg
