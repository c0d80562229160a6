// tracks.cu -- build_tracks (mapping.py:113-161), host-native.
//
// The reference merges match edges union-find style in a fixed order (pairs
// by (frame_a, frame_b), matches by (index_a, index_b)) and skips a merge
// that would put two features of one frame into a track: the outcome
// depends on that order, so it is a sequential greedy, not a data-parallel
// kernel.  This is its native form (no context, no device), producing the
// tracks the triangulation consumes as CSR, bit-identical to the reference:
// components ordered by their root (= smallest (frame, feature) node, since
// a merge always hangs the larger root under the smaller), nodes sorted,
// singletons dropped.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "common.cuh"

namespace sfm {

void build_tracks(int64_t n_pairs, const int32_t* pair_frames, const int64_t* pair_ptr, const int32_t* match_index,
                  int64_t* out_track_ptr, int32_t* out_obs_frame, int32_t* out_obs_feature, int64_t* out_n_tracks,
                  int64_t* out_n_obs) {
  SFM_REQUIRE(n_pairs >= 0, "negative pair count");
  const int64_t n_matches = n_pairs ? pair_ptr[n_pairs] : 0;
  SFM_REQUIRE(n_pairs == 0 || pair_ptr[0] == 0, "pair_ptr must start at 0");
  // nodes (frame, feature) in tuple order
  std::vector<uint64_t> keys;
  keys.reserve(2 * n_matches);
  auto key = [](int32_t f, int32_t i) { return ((uint64_t)(uint32_t)f << 32) | (uint32_t)i; };
  for (int64_t p = 0; p < n_pairs; ++p) {
    SFM_REQUIRE(pair_ptr[p + 1] >= pair_ptr[p], "pair_ptr must be non-decreasing");
    for (int64_t m = pair_ptr[p]; m < pair_ptr[p + 1]; ++m) {
      SFM_REQUIRE(pair_frames[2 * p] >= 0 && pair_frames[2 * p + 1] >= 0 && match_index[2 * m] >= 0 &&
                      match_index[2 * m + 1] >= 0,
                  "negative frame / feature index");
      keys.push_back(key(pair_frames[2 * p], match_index[2 * m]));
      keys.push_back(key(pair_frames[2 * p + 1], match_index[2 * m + 1]));
    }
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  const int64_t n = (int64_t)keys.size();
  auto id_of = [&](uint64_t k) { return (int64_t)(std::lower_bound(keys.begin(), keys.end(), k) - keys.begin()); };
  std::vector<int64_t> parent(n);
  std::iota(parent.begin(), parent.end(), 0);
  std::vector<std::vector<int32_t>> frames(n);  // per root, sorted; empty = {own frame}
  auto find = [&](int64_t x) {
    int64_t r = x;
    while (parent[r] != r) r = parent[r];
    while (parent[x] != r) {
      const int64_t nx = parent[x];
      parent[x] = r;
      x = nx;
    }
    return r;
  };
  auto frames_of = [&](int64_t r) -> std::vector<int32_t>& {
    if (frames[r].empty()) frames[r].push_back((int32_t)(keys[r] >> 32));
    return frames[r];
  };
  // pairs by (frame_a, frame_b); matches by (index_a, index_b) (both stable)
  std::vector<int64_t> order(n_pairs);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    return std::make_pair(pair_frames[2 * a], pair_frames[2 * a + 1]) <
           std::make_pair(pair_frames[2 * b], pair_frames[2 * b + 1]);
  });
  std::vector<int64_t> ms;
  for (int64_t p : order) {
    ms.resize(pair_ptr[p + 1] - pair_ptr[p]);
    std::iota(ms.begin(), ms.end(), pair_ptr[p]);
    std::stable_sort(ms.begin(), ms.end(), [&](int64_t a, int64_t b) {
      return std::make_pair(match_index[2 * a], match_index[2 * a + 1]) <
             std::make_pair(match_index[2 * b], match_index[2 * b + 1]);
    });
    const int32_t fa = pair_frames[2 * p], fb = pair_frames[2 * p + 1];
    for (int64_t m : ms) {
      int64_t ra = find(id_of(key(fa, match_index[2 * m])));
      int64_t rb = find(id_of(key(fb, match_index[2 * m + 1])));
      if (ra == rb) continue;
      std::vector<int32_t>& sa = frames_of(ra);
      std::vector<int32_t>& sb = frames_of(rb);
      bool clash = false;
      for (size_t i = 0, j = 0; i < sa.size() && j < sb.size();) {
        if (sa[i] == sb[j]) { clash = true; break; }
        if (sa[i] < sb[j]) ++i; else ++j;
      }
      if (clash) continue;  // conflicting join: keep both fragments
      if (rb < ra) std::swap(ra, rb);
      parent[rb] = ra;
      std::vector<int32_t> merged;
      std::merge(frames[ra].begin(), frames[ra].end(), frames[rb].begin(), frames[rb].end(),
                 std::back_inserter(merged));
      frames[ra].swap(merged);
      std::vector<int32_t>().swap(frames[rb]);
    }
  }
  // components by root, nodes ascending (node ids are in tuple order)
  std::vector<int64_t> root(n), cnt(n, 0);
  for (int64_t x = 0; x < n; ++x) ++cnt[root[x] = find(x)];
  int64_t nt = 0, no = 0;
  out_track_ptr[0] = 0;
  std::vector<int64_t> start(n, -1);
  for (int64_t r = 0; r < n; ++r)
    if (root[r] == r && cnt[r] >= 2) {
      start[r] = no;
      no += cnt[r];
      out_track_ptr[++nt] = no;
    }
  std::vector<int64_t> fill(n, 0);
  for (int64_t x = 0; x < n; ++x) {
    const int64_t r = root[x];
    if (start[r] < 0) continue;
    const int64_t o = start[r] + fill[r]++;
    out_obs_frame[o] = (int32_t)(keys[x] >> 32);
    out_obs_feature[o] = (int32_t)(keys[x] & 0xffffffffu);
  }
  *out_n_tracks = nt;
  *out_n_obs = no;
}

}  // namespace sfm
