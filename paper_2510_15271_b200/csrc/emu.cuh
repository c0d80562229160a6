// emu.cuh -- point-sharded BA with R logical ranks on one device (test path).
#pragma once
#include "common.cuh"

namespace sfm {

void ba_solve_emulated(int device, int n_shards, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                       double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report);

}  // namespace sfm
