// imap.cuh -- device-resident iterative_map (mapping.py:569-624).
#pragma once
#include "common.cuh"

namespace sfm {

struct DeviceGroup;

// group: a multi-device context's devices (null or size 1: everything on
// the calling device).  With a group, the RANSAC / gating / list state stay
// on this device and every bundle adjustment runs point-sharded over the
// group (ba_solve_multi).
void iterative_map(cudaStream_t s, Profiler* prof, const sfm_map_problem& prob, const sfm_map_options& opt,
                   double* out_q, double* out_t, double* out_X, uint8_t* out_mask, int8_t* out_status,
                   int64_t* out_lm, int64_t* out_nlm, sfm_round_stat* out_stats, int32_t* out_nstats,
                   const DeviceGroup* group = nullptr);

}  // namespace sfm
