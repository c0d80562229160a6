// tracks.cuh -- build_tracks (mapping.py:113-161), host-native.
#pragma once
#include "common.cuh"

namespace sfm {

void build_tracks(int64_t n_pairs, const int32_t* pair_frames, const int64_t* pair_ptr, const int32_t* match_index,
                  int64_t* out_track_ptr, int32_t* out_obs_frame, int32_t* out_obs_feature, int64_t* out_n_tracks,
                  int64_t* out_n_obs);

}  // namespace sfm
