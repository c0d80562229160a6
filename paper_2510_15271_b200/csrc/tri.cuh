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

// ---- device-resident form (iterative_map loop, csrc/imap.cu) ----------------
// Every pointer is device memory.
struct TriDeviceTracks {
  int n_frames;
  const double* Rt;                  // [F*12] R row-major | t
  const int* frame_model;
  const sfm_camera_model* models;
  int64_t n_tracks, n_obs;
  const int64_t* ptr;                // [T+1]
  const int* obs_frame;              // [N]
  const double* obs_uv;              // [N*2]
  const double* ray;                 // [N*3] from tri_rays_device
  const int* ray_st;                 // [N]
};
// R|t records from quaternions + translations.
void tri_rt_device(cudaStream_t s, int F, const double* q, const double* t, double* Rt);
// unproject every observation (pose-independent camera rays).
void tri_rays_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, double* ray, int* ray_st);
// ransac_triangulate over the active tracks (outputs per track / per obs).
void tri_ransac_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, const uint8_t* active,
                       double thr, double min_angle, int method, double* X, uint8_t* mask, int8_t* status);
// remove_outliers gate over every track with points P (only set mask bits
// are tested); inliers per track, removed count accumulated into *removed.
void tri_gate_device(cudaStream_t s, Profiler* prof, const TriDeviceTracks& tr, const double* P, double thr,
                     uint8_t* mask, int* inliers, unsigned long long* removed);

}  // namespace sfm
