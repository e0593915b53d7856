// Host construction of the blocked K1 scatter (kxblock.hpp). Deterministic:
// a stable counting sort of the tets by centroid bucket, blocks of at most
// `block_tets` consecutive tets of a bucket, per-block dof lists sorted by dof
// with their slots in ascending local order, and boundary partials numbered in
// block order. Blocks are independent, so the per-block work runs in parallel.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>

#include "kxblock.hpp"

namespace eqsb {

KxBlocks build_kx_blocks(const std::vector<int>& tet_dofs, int nl, int n_tets, const std::vector<double>& coords4,
                         int n_dofs, int block_tets) {
  if (block_tets < 1 || (long)block_tets * nl > 65535) throw std::invalid_argument("kx blocks: bad block size");
  // shared-memory slot of local product i of block tet tl: i * max_block_tets + tl
  KxBlocks kb;
  kb.nl = nl;
  kb.n_tets = n_tets;
  // centroid buckets: a uniform grid with ~0.75 block_tets tets per bucket
  std::vector<double> cen(3L * std::max(1, n_tets));
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  double lo0 = INFINITY, lo1 = INFINITY, lo2 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY, hi2 = -INFINITY;
#pragma omp parallel for schedule(static) reduction(min : lo0, lo1, lo2) reduction(max : hi0, hi1, hi2)
  for (int t = 0; t < n_tets; ++t) {
    for (int d = 0; d < 3; ++d) {
      double c = 0.0;
      for (int k = 0; k < 4; ++k) c += coords4[4L * tet_dofs[(long)nl * t + k] + d];
      cen[3L * t + d] = 0.25 * c;
    }
    lo0 = std::min(lo0, cen[3L * t]);
    lo1 = std::min(lo1, cen[3L * t + 1]);
    lo2 = std::min(lo2, cen[3L * t + 2]);
    hi0 = std::max(hi0, cen[3L * t]);
    hi1 = std::max(hi1, cen[3L * t + 1]);
    hi2 = std::max(hi2, cen[3L * t + 2]);
  }
  lo[0] = lo0, lo[1] = lo1, lo[2] = lo2, hi[0] = hi0, hi[1] = hi1, hi[2] = hi2;
  int dims[3] = {1, 1, 1};
  if (n_tets > 0) {
    const double nb = std::max(1.0, n_tets / (0.75 * block_tets));
    double ext[3], vol = 1.0;
    int active = 0;
    for (int d = 0; d < 3; ++d) {
      ext[d] = hi[d] - lo[d];
      if (ext[d] > 0) {
        vol *= ext[d];
        ++active;
      }
    }
    const double h = active ? std::pow(vol / nb, 1.0 / active) : 1.0;
    for (int d = 0; d < 3; ++d) dims[d] = ext[d] > 0 ? std::max(1, (int)std::ceil(ext[d] / h)) : 1;
  }
  const long nbk = (long)dims[0] * dims[1] * dims[2];
  std::vector<long> bucket(std::max(1, n_tets));
  std::vector<long> cnt(nbk + 1, 0);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < n_tets; ++t) {
    long id = 0;
    for (int d = 2; d >= 0; --d) {
      const double ext = hi[d] - lo[d];
      int i = ext > 0 ? (int)((cen[3L * t + d] - lo[d]) / ext * dims[d]) : 0;
      i = std::min(std::max(i, 0), dims[d] - 1);
      id = id * dims[d] + i;
    }
    bucket[t] = id;
  }
  for (int t = 0; t < n_tets; ++t) ++cnt[bucket[t] + 1];
  for (long b = 0; b < nbk; ++b) cnt[b + 1] += cnt[b];
  kb.tet_perm.assign(n_tets, 0);
  {
    std::vector<long> next(cnt.begin(), cnt.end() - 1);
    for (int t = 0; t < n_tets; ++t) kb.tet_perm[next[bucket[t]]++] = t;
  }
  // blocks: consecutive runs of <= block_tets tets of one bucket
  kb.blk_tet0.push_back(0);
  for (long b = 0; b < nbk; ++b)
    for (long s = cnt[b]; s < cnt[b + 1]; s += block_tets) kb.blk_tet0.push_back((int)std::min(cnt[b + 1], s + block_tets));
  kb.n_blocks = (int)kb.blk_tet0.size() - 1;
  for (int b = 0; b < kb.n_blocks; ++b) kb.max_block_tets = std::max(kb.max_block_tets, kb.blk_tet0[b + 1] - kb.blk_tet0[b]);
  // global incidence counts
  std::vector<int> inc(std::max(1, n_dofs), 0);
  for (long k = 0; k < (long)n_tets * nl; ++k) ++inc[tet_dofs[k]];
  // per-block dof lists (two passes: sizes, then fill)
  const int B = kb.n_blocks;
  std::vector<int> nd(B + 1, 0);
  std::vector<long> ns(B + 1, 0);
  auto block_pairs = [&](int b, std::vector<std::pair<int, int>>& pr) {
    pr.clear();
    const int t0 = kb.blk_tet0[b], t1 = kb.blk_tet0[b + 1];
    for (int tl = 0; tl < t1 - t0; ++tl) {
      const int t = kb.tet_perm[t0 + tl];
      for (int i = 0; i < nl; ++i) pr.push_back({tet_dofs[(long)nl * t + i], i * kb.max_block_tets + tl});
    }
    // by dof, then ascending (tet, local index): the summation order
    std::sort(pr.begin(), pr.end(), [&](const std::pair<int, int>& a, const std::pair<int, int>& b) {
      if (a.first != b.first) return a.first < b.first;
      const int ta = a.second % kb.max_block_tets, tb = b.second % kb.max_block_tets;
      return ta != tb ? ta < tb : a.second < b.second;
    });
  };
#pragma omp parallel
  {
    std::vector<std::pair<int, int>> pr;
#pragma omp for schedule(dynamic, 64)
    for (int b = 0; b < B; ++b) {
      block_pairs(b, pr);
      int u = 0;
      for (size_t k = 0; k < pr.size(); ++k)
        if (k == 0 || pr[k].first != pr[k - 1].first) ++u;
      nd[b + 1] = u;
      ns[b + 1] = (long)pr.size();
    }
  }
  for (int b = 0; b < B; ++b) {
    nd[b + 1] += nd[b];
    ns[b + 1] += ns[b];
  }
  if (ns[B] >= (1L << 31)) throw std::invalid_argument("kx blocks: too many slots for int32 offsets");
  kb.blk_dof0.assign(nd.begin(), nd.end());
  const int nld = nd[B];
  kb.ldof_sptr.assign(nld + 1, 0);
  kb.slots.assign(std::max<long>(1, ns[B]), 0);
  kb.ldof_out.assign(std::max(1, nld), 0);
  std::vector<int>& ldof_dof = kb.ldof_dof;
  ldof_dof.assign(std::max(1, nld), 0);
  kb.tet_local.assign((size_t)std::max(1, n_tets) * nl, 0);
  std::vector<char> boundary(std::max(1, nld), 0);
#pragma omp parallel
  {
    std::vector<std::pair<int, int>> pr;
#pragma omp for schedule(dynamic, 64)
    for (int b = 0; b < B; ++b) {
      block_pairs(b, pr);
      int e = nd[b] - 1;
      long s = ns[b];
      int run = 0;
      for (size_t k = 0; k < pr.size(); ++k) {
        if (k == 0 || pr[k].first != pr[k - 1].first) {
          if (e >= nd[b]) boundary[e] = run != inc[ldof_dof[e]];
          ++e;
          ldof_dof[e] = pr[k].first;
          kb.ldof_sptr[e] = (int)s;
          run = 0;
        }
        kb.slots[s++] = (uint16_t)pr[k].second;
        {
          const int tl = pr[k].second % kb.max_block_tets, i = pr[k].second / kb.max_block_tets;
          kb.tet_local[(size_t)nl * (kb.blk_tet0[b] + tl) + i] = (uint16_t)(e - nd[b]);
        }
        ++run;
      }
      if (e >= nd[b]) boundary[e] = run != inc[ldof_dof[e]];
    }
  }
  kb.ldof_sptr[nld] = (int)ns[B];
  for (int b = 0; b < B; ++b) {
    if (nd[b + 1] - nd[b] > 65535) throw std::invalid_argument("kx blocks: too many dofs in a block");
    kb.max_block_dofs = std::max(kb.max_block_dofs, nd[b + 1] - nd[b]);
    kb.max_block_slots = std::max(kb.max_block_slots, (int)(ns[b + 1] - ns[b]));
  }
  // outputs: interior dofs directly, boundary dofs through numbered partials
  int np = 0;
  std::vector<int> pcnt(std::max(1, n_dofs) + 1, 0);
  for (int e = 0; e < nld; ++e) {
    if (boundary[e]) {
      kb.ldof_out[e] = -(np++) - 1;
      ++pcnt[ldof_dof[e] + 1];
    } else {
      kb.ldof_out[e] = ldof_dof[e];
    }
  }
  kb.n_partials = np;
  // pass-2 lists: boundary dofs ascending, their partials in block order
  for (int d = 0; d < n_dofs; ++d) pcnt[d + 1] += pcnt[d];
  kb.bpart.assign(std::max(1, np), 0);
  {
    std::vector<int> next(pcnt.begin(), pcnt.end() - 1);
    for (int e = 0; e < nld; ++e)
      if (boundary[e]) kb.bpart[next[ldof_dof[e]]++] = -kb.ldof_out[e] - 1;
  }
  kb.bptr.push_back(0);
  for (int d = 0; d < n_dofs; ++d)
    if (pcnt[d + 1] > pcnt[d]) {
      kb.bdof.push_back(d);
      kb.bptr.push_back(pcnt[d + 1]);
    }
  return kb;
}

}  // namespace eqsb
