// Blocked deterministic scatter of the fused stiffness kernel K1 (DESIGN.md
// §3 "K(x)x"): tets are grouped into spatially compact blocks (centroid
// buckets, split to at most `block_tets`), one CTA per block computes the
// local products into shared memory and then sums them per touched dof over a
// fixed slot list. Dofs whose incident tets all lie in the block are written
// directly; the others (block-boundary dofs) write a partial sum that a
// second, small pass adds up per dof in block order. No atomics, fixed
// summation order: results are bit-reproducible run to run, and the per-tet
// local products never travel through HBM.
#pragma once

#include <cstdint>
#include <vector>

namespace eqsb {

struct KxBlocks {
  int nl = 4, n_tets = 0, n_blocks = 0, n_partials = 0, max_block_tets = 0, max_block_dofs = 0, max_block_slots = 0;
  std::vector<int> tet_perm;      // blocked order -> input tet index
  std::vector<int> blk_tet0;      // [n_blocks + 1] first tet (blocked order) of each block
  std::vector<int> blk_dof0;      // [n_blocks + 1] first block-dof entry of each block
  std::vector<int> ldof_sptr;     // [n_ldof + 1] slot range of each block-dof
  std::vector<uint16_t> slots;    // shared-memory slot i * max_block_tets + tet_in_block, ascending (tet, i)
  std::vector<int> ldof_out;      // >= 0: dof (written directly); < 0: -(partial index) - 1
  std::vector<int> ldof_dof;      // dof of every block-dof entry
  std::vector<uint16_t> tet_local;  // [n_tets][nl] blocked order: block-local dof index (into the block's dofs)
  std::vector<int> bdof, bptr, bpart;  // boundary dofs: partial indices in block order
};

// tet_dofs: [n_tets][nl] dof ids (< n_dofs); coords4: [n_dofs][4] (x, y, z, pad),
// the first 4 dofs of a tet are its vertices. Deterministic.
KxBlocks build_kx_blocks(const std::vector<int>& tet_dofs, int nl, int n_tets, const std::vector<double>& coords4,
                         int n_dofs, int block_tets);

}  // namespace eqsb
