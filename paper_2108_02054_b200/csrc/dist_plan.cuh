// Device-built row partition of a hierarchy over W ranks (dist_plan.cu): the
// arrays of amgr_dist_level, computed from the hierarchy's device patterns and
// aggregates with the rules of paper_2108_02054_b200/partition.py.
#pragma once

#include <vector>

#include "hierarchy.cuh"

namespace amgr {

struct PlanLevel {
    int64_t n_own = 0, n_halo = 0, nnz = 0, n_cown = 0;
    DevArray<int> owned, rp, col, nnz_map, halo, agg, mptr, midx, send_idx;
    std::vector<int> send_peer, recv_peer;
    std::vector<int64_t> send_cnt, recv_off, recv_cnt;
};

struct DevicePlan {
    int top = -1;
    std::vector<PlanLevel> lv;
    std::vector<int64_t> t_counts;  // level top+1 rows per rank (contiguous ranges)
};

// last partitioned level: the coarsest with >= replicate_below rows, never the
// coarsest level (partition.py choose_top); -1: nothing to partition
int choose_top_level(const Hier& h, int64_t replicate_below);
DevicePlan build_device_plan(Hier& h, int rank, int world, int64_t replicate_below);
// compact the indices i in [0, n) with flag[i] into out; returns the count
int64_t select_flagged(Ctx& c, const char* flag, int64_t n, DevArray<int>& out);

}  // namespace amgr
