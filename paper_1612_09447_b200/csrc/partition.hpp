// Node-ownership domain decomposition of the fine dofs and of every AMG level
// (SURVEY.md §8e). Everything here is a deterministic function of the global
// problem, so every rank computes the same plan without communication, and a
// CPU recomputation (tests/test_partition.py) reproduces it bit-exactly.
#pragma once

#include <vector>

#include "eqs_internal.hpp"

namespace eqsb {

// One index space (level 0 = free dofs, level l = AMG level l) seen by one rank.
// Local numbering: [owned (ascending global id) | ghosts (by owner rank, then global id)].
struct LocalSpace {
  int n_global = 0;
  std::vector<int> owned;
  std::vector<int> ghosts;
  std::vector<int> recv_ranks;               // peers we receive ghosts from (ascending)
  std::vector<int> recv_off;                 // ghost slice per recv peer (size recv_ranks + 1)
  std::vector<int> send_ranks;               // peers we send owned entries to (ascending)
  std::vector<std::vector<int>> send_local;  // per send peer: local owned indices in the peer's ghost order
  int n_own() const { return (int)owned.size(); }
  int n_ghost() const { return (int)ghosts.size(); }
  int n_local() const { return n_own() + n_ghost(); }
};

struct PartitionPlan {
  int nranks = 1, rank = 0, axis = 2;
  int rep_level = 1;                    // levels >= rep_level are replicated whole on every rank
  std::vector<std::vector<int>> owner;  // per level: global id -> rank
  std::vector<LocalSpace> space;        // per level, this rank
  // this rank's rows with local column ids
  HostCsr mii;                          // level 0: owned rows x (own | ghost)
  HostCsr mib;                          // owned rows x fixed dofs (global fixed index)
  std::vector<HostCsr> A, P, R;         // per level (P, R absent on the coarsest)
  // stiffness operator (owner computes): local tets and their dofs in the
  // local "full" numbering [owned | ghosts | local fixed]
  std::vector<int> tets;                // global tet ids touching an owned free dof (ascending)
  std::vector<int> fixed;               // global dof ids of the fixed dofs used by local tets (ascending)
  std::vector<int> tet_dofs;            // [tets][n_local] local full numbering
};

// owner rank of every free dof: stable sort by (coordinate along the longest
// bounding-box axis, preferring z then y then x on ties; free index), then
// contiguous equal chunks
// (device >= 0: the sort runs on that GPU, k_setup.cu, same result)
std::vector<int> partition_free_dofs(const Problem& p, int nranks, int* axis_out = nullptr, int device = -1);

// full plan for `rank` (levels from the AMG hierarchy; a single level when h
// is empty). Coarse levels with at most rep_threshold rows, and always the
// dense coarsest level, are replicated: every rank holds all rows, the
// restriction into the first replicated level sums the ranks' partial
// products (allreduce), and no halo is exchanged below it.
// level_A (optional): replacement operators per level (entries with n_rows == 0 keep h's)
PartitionPlan build_plan(const Problem& p, const HostCsr& m_ii, const HostCsr& m_ib, const AmgHierarchy& h,
                         int nranks, int rank, int rep_threshold, const std::vector<HostCsr>* level_A = nullptr,
                         int max_levels = 1 << 30, int device = -1);

}  // namespace eqsb
