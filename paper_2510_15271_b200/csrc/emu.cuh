// emu.cuh -- point-sharded BA driven from ONE process: R ranks as R host
// threads, each on its own device (a multi-device context, NCCL
// communicators from ncclCommInitAll) or all on one device (shard emulation,
// the test path -- NCCL rejects a device twice in a communicator).
#pragma once
#include <nccl.h>

#include <vector>

#include "common.cuh"

namespace sfm {

struct DeviceGroup {
  std::vector<int> devices;        // device of each rank
  std::vector<ncclComm_t> comms;   // one per rank (ncclCommInitAll), empty = shard emulation
  bool peer = false;               // peer access enabled between every pair of devices
  int size() const { return (int)devices.size(); }
};

// Contiguous point ranges with (near) equal observation counts (SURVEY.md
// 8(e), the same split as mapping.shard_ranges); pose terms on rank 0 only.
// obs_point may be host or device memory; the shards point into `full`'s
// arrays except for the rank-local point indices held in `local_op`.
struct ShardSet {
  std::vector<sfm_ba_problem> shards;
  std::vector<std::vector<int>> local_op;
  std::vector<int64_t> p0;
};
ShardSet shard_problem(const sfm_ba_problem& full, int world);
// The point boundaries of that split from host obs_point (world+1 entries):
// rank r owns points [b[r], b[r+1]).
std::vector<int64_t> shard_bounds(const int* obs_point, int64_t n_obs, int64_t n_points, int world);

void ba_solve_group(const DeviceGroup& g, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                    double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report);

void ba_solve_emulated(int device, int n_shards, const sfm_ba_problem* shards, const sfm_ba_options& opt,
                       double* out_q, double* out_t, double* const* out_points, sfm_ba_report* report);

// sfm_ba_solve on a multi-device context: shard, solve, write back.
void ba_solve_multi(const DeviceGroup& g, const sfm_ba_problem& full, const sfm_ba_options& opt,
                    double* out_q, double* out_t, double* out_points, sfm_ba_report* report);

}  // namespace sfm
