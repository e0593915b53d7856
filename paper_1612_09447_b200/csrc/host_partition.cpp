// Deterministic node-ownership partition of the fine dofs and of the AMG
// hierarchy: owner-computes for the stiffness operator, owned
// rows + ghost columns for every CSR operator, halo lists per peer, and
// replicated (agglomerated) small coarse levels.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <numeric>

#include "partition.hpp"

namespace eqsb {

namespace {

// coordinates of every dof (vertex dofs: nodes; P2 edge dofs: midpoint of the edge)
std::vector<double> dof_coords(const Problem& p) {
  const Dofs& dm = p.dm;
  const Mesh& m = p.mesh;
  std::vector<double> c((size_t)dm.n_dofs * 3, 0.0);
  std::copy(m.nodes.begin(), m.nodes.end(), c.begin());
  if (dm.order == 2) {
    for (int t = 0; t < m.n_tets; ++t)
      for (int e = 0; e < 6; ++e) {
        const int d = dm.element_dofs[10L * t + 4 + e];
        const int a = m.tets[4L * t + kTetEdgeVertices[e][0]], b = m.tets[4L * t + kTetEdgeVertices[e][1]];
        for (int k = 0; k < 3; ++k) c[3L * d + k] = 0.5 * (m.nodes[3L * a + k] + m.nodes[3L * b + k]);
      }
  }
  return c;
}

// rows `rows` of a (all rows when rows == nullptr); columns mapped through
// g2l (identity when empty); entries whose column maps to -1 are an error
// unless drop_unmapped (then they are skipped)
HostCsr local_rows(const HostCsr& a, const std::vector<int>* rows, const std::vector<int>& g2l, int n_cols,
                   bool drop_unmapped = false) {
  HostCsr out;
  const long nr = rows ? (long)rows->size() : a.n_rows;
  auto row_of = [&](long r) { return rows ? (*rows)[r] : (int)r; };
  out.n_rows = (int)nr;
  out.n_cols = n_cols;
  out.row_ptr.assign(nr + 1, 0);
#pragma omp parallel for schedule(static)
  for (long r = 0; r < nr; ++r) {
    int cnt = 0;
    const int i = row_of(r);
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (g2l.empty() || !drop_unmapped || g2l[a.col_idx[k]] >= 0) ++cnt;
    out.row_ptr[r + 1] = cnt;
  }
  for (long r = 0; r < nr; ++r) out.row_ptr[r + 1] += out.row_ptr[r];
  out.col_idx.resize(out.row_ptr.back());
  out.values.resize(out.row_ptr.back());
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (long r = 0; r < nr; ++r) {
    int pos = out.row_ptr[r];
    const int i = row_of(r);
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int lc = g2l.empty() ? a.col_idx[k] : g2l[a.col_idx[k]];
      if (lc < 0) {
        if (!drop_unmapped) bad = 1;
        continue;
      }
      out.col_idx[pos] = lc;
      out.values[pos++] = a.values[k];
    }
  }
  if (bad) throw std::logic_error("partition: column without a local index");
  return out;
}

}  // namespace

std::vector<int> partition_free_dofs(const Problem& p, int nranks, int* axis_out, int device) {
  const Dofs& dm = p.dm;
  const int nf = dm.n_free();
  const std::vector<double> c = dof_coords(p);
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int n = 0; n < p.mesh.n_nodes; ++n)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], p.mesh.nodes[3L * n + k]);
      hi[k] = std::max(hi[k], p.mesh.nodes[3L * n + k]);
    }
  int axis = 2;
  for (int k : {1, 0})
    if (hi[k] - lo[k] > hi[axis] - lo[axis]) axis = k;
  if (axis_out) *axis_out = axis;
  std::vector<int> owner(nf, 0);
  if (nranks == 1) return owner;
  if (device >= 0) {
    std::vector<double> key(nf);
    for (int a = 0; a < nf; ++a) key[a] = c[3L * dm.free_dofs[a] + axis];
    return dev_partition_owner(key, nranks, device);
  }
  std::vector<int> order(nf);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return c[3L * dm.free_dofs[a] + axis] < c[3L * dm.free_dofs[b] + axis];
  });
  for (long k = 0; k < nf; ++k) owner[order[k]] = (int)(k * nranks / std::max(1, nf));
  return owner;
}

PartitionPlan build_plan(const Problem& p, const HostCsr& m_ii, const HostCsr& m_ib, const AmgHierarchy& h,
                         int nranks, int rank, int rep_threshold, const std::vector<HostCsr>* level_A,
                         int max_levels, int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("build_plan: bad rank/nranks");
  PartitionPlan plan;
  plan.nranks = nranks;
  plan.rank = rank;
  const int L = h.levels.empty() ? 1 : std::min((int)h.levels.size(), std::max(1, max_levels));
  auto A_of = [&](int l) -> const HostCsr& {
    if (h.levels.empty()) return m_ii;
    if (level_A && l < (int)level_A->size() && (*level_A)[l].n_rows > 0) return (*level_A)[l];
    return h.levels[l].A;
  };
  // first replicated level: small coarse levels (and always the dense coarsest)
  // are held whole on every rank; a single level (no hierarchy) stays partitioned
  int rep = L;
  if (L > 1) {
    rep = L - 1;
    for (int l = 1; l < L; ++l)
      if (A_of(l).n_rows <= rep_threshold) {
        rep = l;
        break;
      }
  }
  plan.rep_level = rep;
  // ownership per level
  plan.owner.resize(L);
  plan.owner[0] = partition_free_dofs(p, nranks, &plan.axis, device);
  for (int l = 0; l + 1 < L; ++l) {
    const std::vector<int>& agg = h.levels[l].aggregates;
    const int nc = A_of(l + 1).n_rows;
    std::vector<int> first(nc, -1);
    for (int i = 0; i < (int)agg.size(); ++i)
      if (first[agg[i]] < 0) first[agg[i]] = i;
    plan.owner[l + 1].resize(nc);
    for (int j = 0; j < nc; ++j) plan.owner[l + 1][j] = plan.owner[l][first[j]];
  }
  // rows owned by every rank, per partitioned level
  std::vector<std::vector<std::vector<int>>> rows_of(L, std::vector<std::vector<int>>(nranks));
  for (int l = 0; l < std::min(rep, L); ++l)
    for (int i = 0; i < (int)plan.owner[l].size(); ++i) rows_of[l][plan.owner[l][i]].push_back(i);
  plan.space.resize(L);
  std::vector<std::vector<int>> g2l(L);
  for (int l = 0; l < L; ++l) {
    const std::vector<int>& own = plan.owner[l];
    LocalSpace& sp = plan.space[l];
    sp.n_global = (int)own.size();
    if (l >= rep) {  // replicated: every rank holds the whole level, no halo
      sp.owned.resize(sp.n_global);
      std::iota(sp.owned.begin(), sp.owned.end(), 0);
      g2l[l] = sp.owned;
      continue;
    }
    // ghost sets of every rank: columns (level l) of A_l[own_l], R_l[own_l+1]
    // (when l+1 is partitioned), P_l-1[own_l-1]
    std::vector<std::vector<int>> ghosts(nranks);
#pragma omp parallel for schedule(dynamic, 1)
    for (int q = 0; q < nranks; ++q) {
      std::vector<int>& gs = ghosts[q];
      auto scan = [&](const HostCsr& m, const std::vector<int>& rows) {
        for (int r : rows)
          for (int k = m.row_ptr[r]; k < m.row_ptr[r + 1]; ++k)
            if (own[m.col_idx[k]] != q) gs.push_back(m.col_idx[k]);
      };
      scan(A_of(l), rows_of[l][q]);
      if (l + 1 < rep) scan(h.levels[l].R, rows_of[l + 1][q]);
      if (l >= 1) scan(h.levels[l - 1].P, rows_of[l - 1][q]);
      std::sort(gs.begin(), gs.end());
      gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
      std::stable_sort(gs.begin(), gs.end(), [&](int a, int b) { return own[a] < own[b]; });
    }
    sp.owned = rows_of[l][rank];
    sp.ghosts = ghosts[rank];
    g2l[l].assign(own.size(), -1);
    for (int i = 0; i < sp.n_own(); ++i) g2l[l][sp.owned[i]] = i;
    for (int i = 0; i < sp.n_ghost(); ++i) g2l[l][sp.ghosts[i]] = sp.n_own() + i;
    sp.recv_off.push_back(0);
    for (int i = 0; i < sp.n_ghost(); ++i) {
      const int q = own[sp.ghosts[i]];
      if (sp.recv_ranks.empty() || sp.recv_ranks.back() != q) {
        if (!sp.recv_ranks.empty()) sp.recv_off.push_back(i);
        sp.recv_ranks.push_back(q);
      }
    }
    if (!sp.recv_ranks.empty()) sp.recv_off.push_back(sp.n_ghost());
    for (int q = 0; q < nranks; ++q) {
      if (q == rank) continue;
      std::vector<int> s;
      for (int gid : ghosts[q])
        if (own[gid] == rank) s.push_back(g2l[l][gid]);
      if (!s.empty()) {
        sp.send_ranks.push_back(q);
        sp.send_local.push_back(std::move(s));
      }
    }
  }
  // local operators
  plan.A.resize(L);
  plan.P.resize(L);
  plan.R.resize(L);
  for (int l = 0; l < L; ++l) {
    const LocalSpace& sp = plan.space[l];
    const bool part = l < rep;
    plan.A[l] = part ? local_rows(A_of(l), &sp.owned, g2l[l], sp.n_local()) : local_rows(A_of(l), nullptr, {}, sp.n_global);
    if (l + 1 < L) {
      const LocalSpace& sc = plan.space[l + 1];
      plan.P[l] = part ? local_rows(h.levels[l].P, &sp.owned, g2l[l + 1], sc.n_local())
                       : local_rows(h.levels[l].P, nullptr, {}, sc.n_global);
      if (l + 1 < rep) {
        plan.R[l] = local_rows(h.levels[l].R, &sc.owned, g2l[l], sp.n_local());
      } else if (part) {
        // restriction into a replicated level: all coarse rows, owned fine
        // columns only; the ranks' partial results are summed by allreduce
        std::vector<int> own_only(sp.n_global, -1);
        for (int i = 0; i < sp.n_own(); ++i) own_only[sp.owned[i]] = i;
        plan.R[l] = local_rows(h.levels[l].R, nullptr, own_only, sp.n_local(), true);
      } else {
        plan.R[l] = local_rows(h.levels[l].R, nullptr, {}, sp.n_global);
      }
    }
  }
  plan.mii = h.levels.empty() ? plan.A[0] : local_rows(m_ii, &plan.space[0].owned, g2l[0], plan.space[0].n_local());
  plan.mib = local_rows(m_ib, &plan.space[0].owned, {}, m_ib.n_cols);
  // stiffness operator: tets touching an owned free dof, local full numbering
  const Dofs& dm = p.dm;
  const int nl = dm.n_local;
  std::vector<int> free_index(dm.n_dofs, -1);
  for (int i = 0; i < dm.n_free(); ++i) free_index[dm.free_dofs[i]] = i;
  std::vector<char> fixed_used(dm.n_dofs, 0);
  for (int t = 0; t < p.mesh.n_tets; ++t) {
    bool mine = false;
    for (int i = 0; i < nl && !mine; ++i) {
      const int fi = free_index[dm.element_dofs[(size_t)nl * t + i]];
      mine = fi >= 0 && plan.owner[0][fi] == rank;
    }
    if (!mine) continue;
    plan.tets.push_back(t);
    for (int i = 0; i < nl; ++i) {
      const int d = dm.element_dofs[(size_t)nl * t + i];
      if (free_index[d] < 0) fixed_used[d] = 1;
    }
  }
  std::vector<int> fixed_pos(dm.n_dofs, -1);
  for (int d = 0; d < dm.n_dofs; ++d)
    if (fixed_used[d]) {
      fixed_pos[d] = (int)plan.fixed.size();
      plan.fixed.push_back(d);
    }
  const int base = plan.space[0].n_local();
  plan.tet_dofs.resize(plan.tets.size() * nl);
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (long k = 0; k < (long)plan.tets.size(); ++k)
    for (int i = 0; i < nl; ++i) {
      const int d = dm.element_dofs[(size_t)nl * plan.tets[k] + i];
      const int fi = free_index[d];
      const int loc = fi >= 0 ? g2l[0][fi] : base + fixed_pos[d];
      if (loc < 0) bad = 1;
      plan.tet_dofs[k * nl + i] = loc;
    }
  if (bad) throw std::logic_error("partition: tet dof without a local index");
  return plan;
}

}  // namespace eqsb
