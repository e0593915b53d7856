// CPU check of the blocked K1 scatter structure (kxblock.hpp): emulate the
// two kernel passes with random per-slot values and compare with a direct
// scatter; every slot is used exactly once, interior dofs are written by one
// block, boundary dofs receive their partials in block order. Built and run
// by tests/test_sell_format.py.
#include <cmath>
#include <cstdio>
#include <random>

#include "kxblock.hpp"

using namespace eqsb;

int main() {
  int fails = 0;
  for (int nl : {4, 10})
    for (int n : {3, 9, 17}) {
      // structured cube of n^3 cells, 6 tets per cell (node ids like mesh.cpp), P2 edges fake-numbered
      const int nn = (n + 1) * (n + 1) * (n + 1);
      auto id = [&](int i, int j, int k) { return (k * (n + 1) + j) * (n + 1) + i; };
      std::vector<double> c4(4L * (nn + 7L * n * n * n * 6), 0.0);
      for (int k = 0; k <= n; ++k)
        for (int j = 0; j <= n; ++j)
          for (int i = 0; i <= n; ++i) {
            c4[4L * id(i, j, k)] = i;
            c4[4L * id(i, j, k) + 1] = j;
            c4[4L * id(i, j, k) + 2] = k;
          }
      std::vector<int> td;
      int extra = nn;
      const int paths[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
          for (int i = 0; i < n; ++i)
            for (auto& p : paths) {
              int v[3] = {i, j, k};
              td.push_back(id(v[0], v[1], v[2]));
              for (int s = 0; s < 3; ++s) {
                ++v[p[s]];
                td.push_back(id(v[0], v[1], v[2]));
              }
              for (int e = 4; e < nl; ++e) td.push_back(extra++ % (nn + 3 * n * n * n));  // shared fake edge dofs
            }
      const int nt = (int)td.size() / nl, ndofs = nn + 3 * n * n * n;
      for (int bt : {64, 333}) {
        KxBlocks kb = build_kx_blocks(td, nl, nt, c4, ndofs, bt);
        std::mt19937 g(7);
        std::vector<double> yt((size_t)nt * nl);
        for (auto& y : yt) y = std::uniform_real_distribution<double>(-1, 1)(g);
        std::vector<double> ref(ndofs, 0.0), out(ndofs, 0.0), part(std::max(1, kb.n_partials), 0.0);
        for (int t = 0; t < nt; ++t)
          for (int i = 0; i < nl; ++i) ref[td[(size_t)nl * t + i]] += yt[(size_t)nl * t + i];
        std::vector<int> used((size_t)nt * nl, 0), written(ndofs, 0);
        for (int b = 0; b < kb.n_blocks; ++b)
          for (int e = kb.blk_dof0[b]; e < kb.blk_dof0[b + 1]; ++e) {
            double s = 0.0;
            for (int k = kb.ldof_sptr[e]; k < kb.ldof_sptr[e + 1]; ++k) {
              const int sl = kb.slots[k], tl = sl % kb.max_block_tets, i = sl / kb.max_block_tets;
              const int t = kb.tet_perm[kb.blk_tet0[b] + tl];
              ++used[(size_t)nl * t + i];
              s += yt[(size_t)nl * t + i];
            }
            if (kb.ldof_out[e] >= 0) {
              out[kb.ldof_out[e]] = s;
              ++written[kb.ldof_out[e]];
            } else {
              part[-kb.ldof_out[e] - 1] = s;
            }
          }
        for (size_t i = 0; i + 1 < kb.bptr.size(); ++i) {
          double s = 0.0;
          for (int k = kb.bptr[i]; k < kb.bptr[i + 1]; ++k) s += part[kb.bpart[k]];
          out[kb.bdof[i]] = s;
          ++written[kb.bdof[i]];
        }
        int bad = 0;
        for (int u : used) bad += u != 1;
        for (int b = 0; b < kb.n_blocks; ++b)
          for (int tl = 0; tl < kb.blk_tet0[b + 1] - kb.blk_tet0[b]; ++tl)
            for (int i = 0; i < nl; ++i) {
              const int t = kb.tet_perm[kb.blk_tet0[b] + tl];
              const int e = kb.blk_dof0[b] + kb.tet_local[(size_t)nl * (kb.blk_tet0[b] + tl) + i];
              bad += kb.ldof_dof[e] != td[(size_t)nl * t + i];
            }
        for (int d = 0; d < ndofs; ++d) {
          bool touched = false;
          (void)touched;
          if (written[d] > 1) ++bad;
          if (std::abs(out[d] - ref[d]) > 1e-12 * (1.0 + std::abs(ref[d]))) ++bad;
        }
        printf("nl %d n %d block %d: %d blocks, %d partials, max %d tets -> %s\n", nl, n, bt, kb.n_blocks,
               kb.n_partials, kb.max_block_tets, bad ? "FAIL" : "ok");
        fails += bad != 0;
      }
    }
  return fails ? 1 : 0;
}
