// tri.cuh -- batched triangulation and reprojection gating on device.
#pragma once
#include "common.cuh"

namespace sfm {

// ransac_triangulate (mapping.py:255-305) over every active track.
void tri_ransac(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, double thr, double min_angle,
                int method, double* out_X, uint8_t* out_mask, int8_t* out_status);
// triangulate_dlt / triangulate_midpoint (mapping.py:194-240) over all
// observations of every active track.
void tri_direct(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, double min_angle, int method,
                double* out_X, int8_t* out_status);
// remove_outliers (mapping.py:544-566).
void tri_gate(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, const double* points, double thr,
              uint8_t* mask_inout, int32_t* out_inliers, int64_t* out_removed);
// reprojection_error (mapping.py:243-252) per observation.
void tri_reproj_errors(cudaStream_t s, Profiler* prof, const sfm_tracks& tr, const double* points,
                       double* out_err);

}  // namespace sfm
