// One-time host setup: element colouring, mass assembly + Dirichlet split,
// smoothed-aggregation AMG hierarchy. All integer artefacts (colours,
// sparsity, aggregates) and all matrix values are bit-identical to the
// reference algorithm; the loops are restructured (flat CSR incidence, row-
// parallel SpGEMM, OpenMP) so that 10^7-10^8 dof setups finish in seconds.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>

#include "element.hpp"
#include "eqs_internal.hpp"

namespace eqsb {

namespace {

// dof -> incident tets (ascending), as CSR.
void dof_incidence(const Dofs& dm, int n_tets, std::vector<long>& ptr, std::vector<int>& tets,
                   std::vector<unsigned char>* local = nullptr) {
  const int nl = dm.n_local;
  ptr.assign((size_t)dm.n_dofs + 1, 0);
  for (size_t k = 0; k < dm.element_dofs.size(); ++k) ++ptr[dm.element_dofs[k] + 1];
  for (int d = 0; d < dm.n_dofs; ++d) ptr[d + 1] += ptr[d];
  tets.resize(ptr.back());
  if (local) local->resize(ptr.back());
  std::vector<long> next(ptr.begin(), ptr.end() - 1);
  for (int t = 0; t < n_tets; ++t)
    for (int i = 0; i < nl; ++i) {
      const long pos = next[dm.element_dofs[(size_t)nl * t + i]]++;
      tets[pos] = t;
      if (local) (*local)[pos] = (unsigned char)i;
    }
}

}  // namespace

// proj/src/matfree.cpp:11-38. Greedy smallest-free colour in ascending tet
// order over tets sharing a dof; the used-colour set is a bitset instead of a
// sorted vector (same result).
std::vector<int> color_elements(const Dofs& dm, int n_tets, int* n_colors_out) {
  std::vector<long> ptr;
  std::vector<int> inc;
  dof_incidence(dm, n_tets, ptr, inc);
  const int nl = dm.n_local;
  std::vector<int> color(n_tets, -1);
  std::vector<uint64_t> used(4, 0);
  int n_colors = 0;
  for (int t = 0; t < n_tets; ++t) {
    std::fill(used.begin(), used.end(), 0);
    for (int i = 0; i < nl; ++i) {
      const int d = dm.element_dofs[(size_t)nl * t + i];
      for (long k = ptr[d]; k < ptr[d + 1]; ++k) {
        const int c = color[inc[k]];
        if (c >= 0) {
          if ((size_t)(c >> 6) >= used.size()) used.resize((c >> 6) + 1, 0);
          used[c >> 6] |= 1ull << (c & 63);
        }
      }
    }
    int c = 0;
    for (size_t w = 0;; ++w) {
      const uint64_t free_bits = w < used.size() ? ~used[w] : ~0ull;
      if (free_bits) {
        c = (int)(w * 64 + __builtin_ctzll(free_bits));
        break;
      }
    }
    color[t] = c;
    n_colors = std::max(n_colors, c + 1);
  }
  if (n_colors_out) *n_colors_out = n_colors;
  return color;
}

// assemble_matrix with the permittivity coefficient (proj/src/assembly.cpp:130-176)
// restricted to the free rows, then split_dirichlet (:188-193) — the fixed rows
// of the full M are never used on the explicit path. Per slot, element
// contributions are summed in ascending tet order exactly like the serial
// reference loop, so every value is bit-identical.
void assemble_mass_blocks(const Problem& p, HostCsr& m_ii, HostCsr& m_ib) {
  const Dofs& dm = p.dm;
  const Mesh& mesh = p.mesh;
  const int nl = dm.n_local;
  std::vector<long> ptr;
  std::vector<int> inc;
  std::vector<unsigned char> loc;
  dof_incidence(dm, mesh.n_tets, ptr, inc, &loc);
  std::vector<int> block_col(dm.n_dofs);  // dof -> column within its block
  std::vector<char> is_free(dm.n_dofs, 0);
  for (int i = 0; i < dm.n_free(); ++i) {
    block_col[dm.free_dofs[i]] = i;
    is_free[dm.free_dofs[i]] = 1;
  }
  for (int i = 0; i < dm.n_fixed(); ++i) block_col[dm.fixed_dofs[i]] = i;
  std::vector<double> eps_of_tet(mesh.n_tets);
  for (int t = 0; t < mesh.n_tets; ++t) {
    auto it = p.materials.find(mesh.region[t]);
    if (it == p.materials.end()) throw ConfigError("no material for region " + std::to_string(mesh.region[t]));
    eps_of_tet[t] = it->second.permittivity();
  }
  // geometry check up front (tet_geometry throws on det == 0, assembly.cpp:52)
  for (int t = 0; t < mesh.n_tets; ++t) {
    double x[4][3];
    for (int v = 0; v < 4; ++v)
      for (int d = 0; d < 3; ++d) x[v][d] = mesh.nodes[3L * mesh.tets[4L * t + v] + d];
    TetGeo g;
    if (!tet_geometry(x, g)) throw GeometryError("degenerate tetrahedron in element kernel");
  }
  const int nf = dm.n_free();
  std::vector<int> len_ii(nf + 1, 0), len_ib(nf + 1, 0);
  // pass 1: row patterns (sorted unique element dofs of incident tets)
#pragma omp parallel
  {
    std::vector<int> buf;
#pragma omp for schedule(dynamic, 4096)
    for (int r = 0; r < nf; ++r) {
      const int gi = dm.free_dofs[r];
      buf.clear();
      for (long k = ptr[gi]; k < ptr[gi + 1]; ++k)
        for (int j = 0; j < nl; ++j) buf.push_back(dm.element_dofs[(size_t)nl * inc[k] + j]);
      std::sort(buf.begin(), buf.end());
      buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      int a = 0, b = 0;
      for (int c : buf) (is_free[c] ? a : b)++;
      len_ii[r + 1] = a;
      len_ib[r + 1] = b;
    }
  }
  m_ii.n_rows = m_ib.n_rows = nf;
  m_ii.n_cols = nf;
  m_ib.n_cols = dm.n_fixed();
  m_ii.row_ptr.assign(nf + 1, 0);
  m_ib.row_ptr.assign(nf + 1, 0);
  for (int r = 0; r < nf; ++r) {
    m_ii.row_ptr[r + 1] = m_ii.row_ptr[r] + len_ii[r + 1];
    m_ib.row_ptr[r + 1] = m_ib.row_ptr[r] + len_ib[r + 1];
  }
  m_ii.col_idx.resize(m_ii.row_ptr[nf]);
  m_ii.values.assign(m_ii.row_ptr[nf], 0.0);
  m_ib.col_idx.resize(m_ib.row_ptr[nf]);
  m_ib.values.assign(m_ib.row_ptr[nf], 0.0);
  // pass 2: columns + values
#pragma omp parallel
  {
    std::vector<int> buf;
    std::vector<double> acc;
#pragma omp for schedule(dynamic, 4096)
    for (int r = 0; r < nf; ++r) {
      const int gi = dm.free_dofs[r];
      buf.clear();
      for (long k = ptr[gi]; k < ptr[gi + 1]; ++k)
        for (int j = 0; j < nl; ++j) buf.push_back(dm.element_dofs[(size_t)nl * inc[k] + j]);
      std::sort(buf.begin(), buf.end());
      buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
      acc.assign(buf.size(), 0.0);
      for (long k = ptr[gi]; k < ptr[gi + 1]; ++k) {  // ascending tet order
        const int t = inc[k];
        const int li = loc[k];
        double x[4][3];
        for (int v = 0; v < 4; ++v)
          for (int d = 0; d < 3; ++d) x[v][d] = mesh.nodes[3L * mesh.tets[4L * t + v] + d];
        TetGeo g;
        tet_geometry(x, g);
        if (nl == 4) {
          double S[10];
          element_laplacian_p1(g, eps_of_tet[t], S);
          for (int j = 0; j < 4; ++j) {
            const int gj = dm.element_dofs[4L * t + j];
            const size_t pos = std::lower_bound(buf.begin(), buf.end(), gj) - buf.begin();
            acc[pos] += S[tri_index(li, j)];
          }
        } else {
          double S[55];
          const double c4[4] = {eps_of_tet[t], eps_of_tet[t], eps_of_tet[t], eps_of_tet[t]};
          element_laplacian_p2(g, c4, S);
          for (int j = 0; j < 10; ++j) {
            const int gj = dm.element_dofs[10L * t + j];
            const size_t pos = std::lower_bound(buf.begin(), buf.end(), gj) - buf.begin();
            acc[pos] += S[tri_index(li, j)];
          }
        }
      }
      int a = m_ii.row_ptr[r], b = m_ib.row_ptr[r];
      for (size_t q = 0; q < buf.size(); ++q) {
        const int c = buf[q];
        if (is_free[c]) {
          m_ii.col_idx[a] = block_col[c];
          m_ii.values[a++] = acc[q];
        } else {
          m_ib.col_idx[b] = block_col[c];
          m_ib.values[b++] = acc[q];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ AMG
namespace {

double coeff(const HostCsr& a, int i, int j) {
  const int* b = a.col_idx.data() + a.row_ptr[i];
  const int* e = a.col_idx.data() + a.row_ptr[i + 1];
  const int* it = std::lower_bound(b, e, j);
  return (it != e && *it == j) ? a.values[it - a.col_idx.data()] : 0.0;
}

std::vector<double> diagonal(const HostCsr& a) {
  std::vector<double> d(a.n_rows);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < a.n_rows; ++i) d[i] = coeff(a, i, i);
  return d;
}

// proj/src/csr.cpp:79-90
double symmetry_error(const HostCsr& a) {
  if (a.n_rows != a.n_cols) return std::numeric_limits<double>::infinity();
  double scale = 0.0;
  for (double v : a.values) scale = std::max(scale, std::abs(v));
  if (scale == 0.0) return 0.0;
  double err = 0.0;
#pragma omp parallel for schedule(static) reduction(max : err)
  for (int i = 0; i < a.n_rows; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      err = std::max(err, std::abs(a.values[k] - coeff(a, a.col_idx[k], i)));
  return err / scale;
}

// proj/src/preconditioners.cpp:7-20
void check_diagonal(const HostCsr& a) {
  for (int i = 0; i < a.n_rows; ++i) {
    int pos = -1;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.col_idx[k] == i) {
        pos = k;
        break;
      }
    if (pos < 0 || a.values[pos] == 0.0)
      throw NumericalError("matrix has a missing or zero diagonal entry at row " + std::to_string(i));
  }
}

void spmv(const HostCsr& a, const std::vector<double>& x, std::vector<double>& y) {
  y.resize(a.n_rows);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < a.n_rows; ++i) {
    double s = 0.0;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) s += a.values[k] * x[a.col_idx[k]];
    y[i] = s;
  }
}

// proj/src/csr.cpp:133-166, row-parallel: each thread owns a contiguous row
// range and its own accumulator; per-row arithmetic order is unchanged.
HostCsr multiply(const HostCsr& a, const HostCsr& b) {
  if (a.n_cols != b.n_rows) throw NumericalError("csr multiply: dimension mismatch");
  HostCsr c;
  c.n_rows = a.n_rows;
  c.n_cols = b.n_cols;
  c.row_ptr.assign(a.n_rows + 1, 0);
  const int nthreads = omp_get_max_threads();
  std::vector<std::vector<int>> tcols(nthreads);
  std::vector<std::vector<double>> tvals(nthreads);
  std::vector<int> row_len(a.n_rows);
#pragma omp parallel num_threads(nthreads)
  {
    const int tid = omp_get_thread_num();
    const int nt = omp_get_num_threads();
    const long lo = (long)a.n_rows * tid / nt, hi = (long)a.n_rows * (tid + 1) / nt;
    std::vector<double> accum(b.n_cols, 0.0);
    std::vector<int> marker(b.n_cols, -1);
    std::vector<int> cols;
    auto& oc = tcols[tid];
    auto& ov = tvals[tid];
    for (long i = lo; i < hi; ++i) {
      cols.clear();
      for (int ka = a.row_ptr[i]; ka < a.row_ptr[i + 1]; ++ka) {
        const int k = a.col_idx[ka];
        const double av = a.values[ka];
        for (int kb = b.row_ptr[k]; kb < b.row_ptr[k + 1]; ++kb) {
          const int j = b.col_idx[kb];
          if (marker[j] != i) {
            marker[j] = (int)i;
            accum[j] = 0.0;
            cols.push_back(j);
          }
          accum[j] += av * b.values[kb];
        }
      }
      std::sort(cols.begin(), cols.end());
      for (int j : cols) {
        oc.push_back(j);
        ov.push_back(accum[j]);
      }
      row_len[i] = (int)cols.size();
    }
  }
  for (int i = 0; i < a.n_rows; ++i) c.row_ptr[i + 1] = c.row_ptr[i] + row_len[i];
  c.col_idx.reserve(c.row_ptr.back());
  c.values.reserve(c.row_ptr.back());
  for (int t = 0; t < nthreads; ++t) {
    c.col_idx.insert(c.col_idx.end(), tcols[t].begin(), tcols[t].end());
    c.values.insert(c.values.end(), tvals[t].begin(), tvals[t].end());
  }
  return c;
}

// proj/src/csr.cpp:52-70. Threads own contiguous row ranges; each column's
// entries are laid out thread by thread, so the result (entries of a column in
// ascending row order) is the serial one.
HostCsr transposed(const HostCsr& a) {
  HostCsr t;
  t.n_rows = a.n_cols;
  t.n_cols = a.n_rows;
  t.row_ptr.assign(a.n_cols + 1, 0);
  t.col_idx.resize(a.col_idx.size());
  t.values.resize(a.values.size());
  const int nt = std::max(1, std::min(omp_get_max_threads(), a.n_rows / 4096 + 1));
  std::vector<std::vector<int>> cnt(nt);
#pragma omp parallel num_threads(nt)
  {
    const int tid = omp_get_thread_num();
    const long lo = (long)a.n_rows * tid / nt, hi = (long)a.n_rows * (tid + 1) / nt;
    std::vector<int>& c = cnt[tid];
    c.assign(a.n_cols, 0);
    for (long i = lo; i < hi; ++i)
      for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) ++c[a.col_idx[k]];
#pragma omp barrier
#pragma omp for schedule(static)
    for (int col = 0; col < a.n_cols; ++col) {
      int s = 0;
      for (int q = 0; q < nt; ++q) s += cnt[q][col];
      t.row_ptr[col + 1] = s;
    }
#pragma omp single
    for (int col = 0; col < a.n_cols; ++col) t.row_ptr[col + 1] += t.row_ptr[col];
#pragma omp for schedule(static)
    for (int col = 0; col < a.n_cols; ++col) {  // per-thread start of each column: row_ptr + earlier threads
      int s = t.row_ptr[col];
      for (int q = 0; q < nt; ++q) {
        const int c = cnt[q][col];
        cnt[q][col] = s;
        s += c;
      }
    }
    for (long i = lo; i < hi; ++i)
      for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
        const int pos = c[a.col_idx[k]]++;
        t.col_idx[pos] = (int)i;
        t.values[pos] = a.values[k];
      }
  }
  return t;
}

// proj/src/amg.cpp:15-26 + 49-88 with the strength graph kept as a per-entry flag.
std::vector<int> aggregate(const HostCsr& a, double theta) {
  const int n = a.n_rows;
  const std::vector<double> d = diagonal(a);
  std::vector<char> strong(a.nnz(), 0);
  std::vector<int> n_strong(n, 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j == i) continue;
      if (std::abs(a.values[k]) >= theta * std::sqrt(std::abs(d[i] * d[j]))) {
        strong[k] = 1;
        ++n_strong[i];
      }
    }
  std::vector<int> agg(n, -1);
  int n_agg = 0;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    bool clean = true;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1] && clean; ++k)
      if (strong[k] && agg[a.col_idx[k]] >= 0) clean = false;
    if (!clean || n_strong[i] == 0) continue;
    agg[i] = n_agg;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (strong[k]) agg[a.col_idx[k]] = n_agg;
    ++n_agg;
  }
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    int best = -1;
    double best_w = -1.0;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j == i || agg[j] < 0) continue;
      const double w = std::abs(a.values[k]);
      if (w > best_w) {
        best_w = w;
        best = agg[j];
      }
    }
    if (best >= 0) agg[i] = best;
  }
  for (int i = 0; i < n; ++i)
    if (agg[i] < 0) agg[i] = n_agg++;
  return agg;
}

}  // namespace

// Eigen's v.norm() = sqrt(squaredNorm()) in the summation order of Eigen 3.4's
// vectorised redux with SSE2 packets of 2 doubles (the reference's default
// x86-64 build): four interleaved accumulators (two packets) over blocks of 4,
// then the leftover packet, the horizontal add and the scalar tail. The
// coarse AMG hierarchy depends on omega = (4/3)/lambda_max through borderline
// strength decisions, so this order is what makes the hierarchy bit-exact to
// the compiled reference (tests/test_ref_pinning.py).
double seq_norm(const std::vector<double>& v) {
  const size_t n = v.size();
  if (n == 0) return 0.0;
  const size_t a2 = n / 4 * 4, a1 = n / 2 * 2;
  double r;
  if (a1 == 0) {
    r = v[0] * v[0];
  } else {
    double p00 = v[0] * v[0], p01 = v[1] * v[1];
    if (a1 > 2) {
      double p10 = v[2] * v[2], p11 = v[3] * v[3];
      for (size_t i = 4; i < a2; i += 4) {
        p00 = p00 + v[i] * v[i];
        p01 = p01 + v[i + 1] * v[i + 1];
        p10 = p10 + v[i + 2] * v[i + 2];
        p11 = p11 + v[i + 3] * v[i + 3];
      }
      p00 = p00 + p10;
      p01 = p01 + p11;
      if (a1 > a2) {
        p00 = p00 + v[a2] * v[a2];
        p01 = p01 + v[a2 + 1] * v[a2 + 1];
      }
    }
    r = p00 + p01;
    for (size_t i = a1; i < n; ++i) r = r + v[i] * v[i];
  }
  return std::sqrt(r);
}

// proj/src/amg.cpp:28-45 (seed 20240811, 10 iterations, sequential norms)
double estimate_lambda_max_scaled(const HostCsr& a, int iters, unsigned seed) {
  const std::vector<double> d = diagonal(a);
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<double> v(a.n_rows), w;
  for (int i = 0; i < a.n_rows; ++i) v[i] = uni(rng);
  const double nv = seq_norm(v);
  for (double& e : v) e /= nv;
  double lambda = 1.0;
  for (int it = 0; it < iters; ++it) {
    spmv(a, v, w);
    for (int i = 0; i < a.n_rows; ++i) w[i] /= d[i];
    lambda = seq_norm(w);
    if (lambda == 0.0) return 1.0;
    for (int i = 0; i < a.n_rows; ++i) v[i] = w[i] / lambda;
  }
  return lambda;
}

// proj/src/amg.cpp:90-143
AmgHierarchy build_amg(const HostCsr& a, const SolverParams& sp, int device) {
  if (a.n_rows != a.n_cols) throw std::invalid_argument("amg: matrix must be square");
  if (symmetry_error(a) > 1e-10) throw std::invalid_argument("amg: matrix is not symmetric");
  check_diagonal(a);
  AmgHierarchy h;
  std::unique_ptr<AmgDeviceBuilder> dev_builder;
  // EQS_HOST_AMG=1: aggregation and lambda_max on the host, products on the device (the round-1 path)
  static const bool host_amg = getenv("EQS_HOST_AMG") != nullptr && atoi(getenv("EQS_HOST_AMG")) != 0;
  h.levels.push_back({a, {}, {}, {}, 0.0});
  while ((int)h.levels.size() < sp.amg_max_levels && h.levels.back().A.n_rows > sp.amg_coarse_limit) {
    AmgHostLevel& lv = h.levels.back();
    const HostCsr& fine = lv.A;
    auto T0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      static const bool on = getenv("EQS_MEMTRACE") != nullptr;
      const auto now = std::chrono::steady_clock::now();
      if (on) fprintf(stderr, "[amg] level %zu %-12s %.2f s\n", h.levels.size() - 1, what,
                      std::chrono::duration<double>(now - T0).count());
      T0 = now;
    };
    const long long batch = getenv("EQS_SPGEMM_BATCH") ? atoll(getenv("EQS_SPGEMM_BATCH")) : (1ll << 28);
    if (device >= 0 && !host_amg) {
      // the whole level on the device (k_amgsetup.cu + k_spgemm.cu), bit-identical
      if (!dev_builder) dev_builder = std::make_unique<AmgDeviceBuilder>(device);
      HostCsr coarse;
      if (!dev_builder->next_level(fine, sp, batch, lv, coarse)) break;
      lap("device level");
      h.levels.push_back({std::move(coarse), {}, {}, {}, 0.0});
      continue;
    }
    std::vector<int> agg = aggregate(fine, sp.amg_theta);
    lap("aggregate");
    const int n_agg = *std::max_element(agg.begin(), agg.end()) + 1;
    if (n_agg >= fine.n_rows) break;
    std::vector<int> agg_size(n_agg, 0);
    for (int id : agg) ++agg_size[id];
    HostCsr p_tent;
    p_tent.n_rows = fine.n_rows;
    p_tent.n_cols = n_agg;
    p_tent.row_ptr.resize(fine.n_rows + 1);
    p_tent.col_idx.resize(fine.n_rows);
    p_tent.values.resize(fine.n_rows);
    for (int i = 0; i < fine.n_rows; ++i) {
      p_tent.row_ptr[i] = i;
      p_tent.col_idx[i] = agg[i];
      p_tent.values[i] = 1.0 / std::sqrt((double)agg_size[agg[i]]);
    }
    p_tent.row_ptr[fine.n_rows] = fine.n_rows;
    lap("p_tent");
    lv.lambda_max_scaled = estimate_lambda_max_scaled(fine, 10, 20240811u);
    lap("lambda");
    const double omega = sp.amg_omega / lv.lambda_max_scaled;
    const std::vector<double> d = diagonal(fine);
    // EQS_SPGEMM_BATCH: products per device batch (tests force many batches)
    HostCsr p;
    if (device >= 0) {
      if (!dev_builder) dev_builder = std::make_unique<AmgDeviceBuilder>(device);
      p = dev_builder->prolongator(fine, p_tent, d, omega, batch);  // (I - omega D^-1 A) P_tent on the device
    } else {
      HostCsr scaled = fine;
#pragma omp parallel for schedule(static)
      for (int i = 0; i < fine.n_rows; ++i)
        for (int k = scaled.row_ptr[i]; k < scaled.row_ptr[i + 1]; ++k) {
          scaled.values[k] = -omega * scaled.values[k] / d[i];
          if (scaled.col_idx[k] == i) scaled.values[k] += 1.0;
        }
      p = multiply(scaled, p_tent);
    }
    lap("P");
    HostCsr r = transposed(p);
    lap("R");
    HostCsr coarse = device >= 0 ? dev_builder->galerkin(r, batch) : multiply(r, multiply(fine, p));
    lap("RAP");
    lv.P = std::move(p);
    lv.R = std::move(r);
    lv.aggregates = std::move(agg);
    check_diagonal(coarse);
    h.levels.push_back({std::move(coarse), {}, {}, {}, 0.0});
  }
  // coarsest: LDLT (amg.cpp:140) then an explicit inverse for a one-kernel dense solve
  h.coarse_n = h.levels.back().A.n_rows;
  h.coarse_inverse = dense_inverse(h.levels.back().A);
  const HostCsr& c = h.levels.back().A;
  if (h.levels.size() > 1) h.levels.back().lambda_max_scaled = estimate_lambda_max_scaled(c, 10, 20240811u);
  return h;
}

std::vector<double> dense_inverse(const HostCsr& c) {
  const int n = c.n_rows;
  std::vector<double> dense((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int k = c.row_ptr[i]; k < c.row_ptr[i + 1]; ++k) dense[(size_t)i * n + c.col_idx[k]] += c.values[k];
  DenseLdlt ldlt;
  ldlt.compute(dense, n);
  if (!ldlt.ok) throw NumericalError("amg: coarsest-level factorization failed");
  std::vector<double> inv((size_t)n * n, 0.0);
#pragma omp parallel if (n > 256)
  {
    std::vector<double> e(n), col(n);
#pragma omp for schedule(static)
    for (int j = 0; j < n; ++j) {
      std::fill(e.begin(), e.end(), 0.0);
      e[j] = 1.0;
      ldlt.solve(e.data(), col.data());
      for (int i = 0; i < n; ++i) inv[(size_t)i * n + j] = col[i];
    }
  }
  return inv;
}

HostCsr filter_lumped(const HostCsr& a, double eps) {
  const std::vector<double> d = diagonal(a);
  HostCsr f;
  f.n_rows = a.n_rows;
  f.n_cols = a.n_cols;
  f.row_ptr.assign(a.n_rows + 1, 0);
  std::vector<char> keep(a.nnz(), 0);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < a.n_rows; ++i) {
    int cnt = 0;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j == i || std::abs(a.values[k]) >= eps * std::sqrt(std::abs(d[i] * d[j]))) {
        keep[k] = 1;
        ++cnt;
      }
    }
    f.row_ptr[i + 1] = cnt;
  }
  for (int i = 0; i < a.n_rows; ++i) f.row_ptr[i + 1] += f.row_ptr[i];
  f.col_idx.resize(f.row_ptr.back());
  f.values.resize(f.row_ptr.back());
#pragma omp parallel for schedule(static)
  for (int i = 0; i < a.n_rows; ++i) {
    double lumped = 0.0;
    int pos = f.row_ptr[i], diag = -1;
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      if (!keep[k]) {
        lumped += a.values[k];
        continue;
      }
      if (a.col_idx[k] == i) diag = pos;
      f.col_idx[pos] = a.col_idx[k];
      f.values[pos++] = a.values[k];
    }
    if (diag >= 0) f.values[diag] += lumped;
  }
  return f;
}

// Eigen::LDLT semantics (see oracle/solvers.cpp for the same restatement).
void DenseLdlt::compute(const std::vector<double>& a, int n_) {
  n = n_;
  lmat = a;
  perm.assign(n, 0);
  ok = true;
  std::vector<double> temp(n);
  auto M = [&](int i, int j) -> double& { return lmat[(size_t)i * n + j]; };
  for (int k = 0; k < n; ++k) {
    int idx = k;
    double biggest = std::abs(M(k, k));
    for (int i = k + 1; i < n; ++i)
      if (std::abs(M(i, i)) > biggest) {
        biggest = std::abs(M(i, i));
        idx = i;
      }
    perm[k] = idx;
    if (idx != k) {
      for (int j = 0; j < n; ++j) std::swap(M(k, j), M(idx, j));
      for (int i = 0; i < n; ++i) std::swap(M(i, k), M(i, idx));
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = M(j, j) * M(k, j);
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += M(k, j) * temp[j];
      M(k, k) -= s;
      // rows are independent: same per-row summation order at any thread count
#pragma omp parallel for schedule(static) if ((long)(n - k) * k > 200000)
      for (int i = k + 1; i < n; ++i) {
        double t = 0.0;
        for (int j = 0; j < k; ++j) t += M(i, j) * temp[j];
        M(i, k) -= t;
      }
    }
    const double akk = M(k, k);
    const bool valid = std::abs(akk) > std::numeric_limits<double>::min();
    if (k < n - 1 && valid) {
      for (int i = k + 1; i < n; ++i) M(i, k) /= akk;
    } else if (k < n - 1) {
      for (int i = k + 1; i < n; ++i)
        if (M(i, k) != 0.0) ok = false;
    }
  }
  d.resize(n);
  for (int i = 0; i < n; ++i) d[i] = M(i, i);
}

void DenseLdlt::solve(const double* b, double* x) const {
  std::vector<double> y(b, b + n);
  for (int k = 0; k < n; ++k)
    if (perm[k] != k) std::swap(y[k], y[perm[k]]);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) y[i] -= lmat[(size_t)i * n + j] * y[j];
  const double tol = std::numeric_limits<double>::min();
  for (int i = 0; i < n; ++i) y[i] = std::abs(d[i]) > tol ? y[i] / d[i] : 0.0;
  for (int i = n - 1; i >= 0; --i)
    for (int j = i + 1; j < n; ++j) y[i] -= lmat[(size_t)j * n + i] * y[j];
  for (int k = n - 1; k >= 0; --k)
    if (perm[k] != k) std::swap(y[k], y[perm[k]]);
  std::copy(y.begin(), y.end(), x);
}

// proj/src/integrators.cpp:86-133
RkcCoefficients RkcCoefficients::compute(int s) {
  if (s < 2) throw std::invalid_argument("rkc: stage count must be >= 2");
  RkcCoefficients k;
  k.s = s;
  const double eps0 = 2.0 / 13.0;
  k.w0 = 1.0 + eps0 / ((double)s * s);
  k.t_w0.assign(s + 1, 0.0);
  k.tp_w0.assign(s + 1, 0.0);
  k.tpp_w0.assign(s + 1, 0.0);
  k.t_w0[0] = 1.0;
  k.t_w0[1] = k.w0;
  k.tp_w0[1] = 1.0;
  for (int j = 2; j <= s; ++j) {
    k.t_w0[j] = 2.0 * k.w0 * k.t_w0[j - 1] - k.t_w0[j - 2];
    k.tp_w0[j] = 2.0 * k.t_w0[j - 1] + 2.0 * k.w0 * k.tp_w0[j - 1] - k.tp_w0[j - 2];
    k.tpp_w0[j] = 4.0 * k.tp_w0[j - 1] + 2.0 * k.w0 * k.tpp_w0[j - 1] - k.tpp_w0[j - 2];
  }
  k.w1 = k.tp_w0[s] / k.tpp_w0[s];
  k.b.assign(s + 1, 0.0);
  k.a.assign(s + 1, 0.0);
  k.c.assign(s + 1, 0.0);
  for (int j = 2; j <= s; ++j) k.b[j] = k.tpp_w0[j] / (k.tp_w0[j] * k.tp_w0[j]);
  k.b[0] = k.b[1] = k.b[2];
  for (int j = 0; j <= s; ++j) k.a[j] = 1.0 - k.b[j] * k.t_w0[j];
  for (int j = 2; j <= s; ++j) k.c[j] = (k.tp_w0[s] / k.tpp_w0[s]) * (k.tpp_w0[j] / k.tp_w0[j]);
  k.c[1] = k.c[2] / 4.0;
  k.mu1_tilde = k.b[1] * k.w1;
  k.mu.assign(s + 1, 0.0);
  k.nu.assign(s + 1, 0.0);
  k.mu_tilde.assign(s + 1, 0.0);
  k.gamma_tilde.assign(s + 1, 0.0);
  for (int j = 2; j <= s; ++j) {
    k.mu[j] = 2.0 * k.b[j] * k.w0 / k.b[j - 1];
    k.nu[j] = -k.b[j] / k.b[j - 2];
    k.mu_tilde[j] = 2.0 * k.b[j] * k.w1 / k.b[j - 1];
    k.gamma_tilde[j] = -k.a[j - 1] * k.mu_tilde[j];
  }
  return k;
}

HostCsr csr_multiply(const HostCsr& a, const HostCsr& b) { return multiply(a, b); }
HostCsr csr_transposed(const HostCsr& a) { return transposed(a); }

}  // namespace eqsb
