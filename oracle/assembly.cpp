// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/assembly.cpp, csr.cpp, matfree.cpp.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>

#include "oracle.hpp"

namespace ora {

namespace {
// proj/src/assembly.cpp:13-18
constexpr double kQa = 0.58541019662496845446;
constexpr double kQb = 0.13819660112501051518;
constexpr double kQuadPoints[4][4] = {
    {kQa, kQb, kQb, kQb}, {kQb, kQa, kQb, kQb}, {kQb, kQb, kQa, kQb}, {kQb, kQb, kQb, kQa}};
constexpr double kCentroid[4] = {0.25, 0.25, 0.25, 0.25};
const double* barycentric_point(int order, int q) { return order == 1 ? kCentroid : kQuadPoints[q]; }
const MaterialModel& material_for(const MaterialTable& materials, int region) {
  auto it = materials.find(region);
  if (it == materials.end()) throw ConfigError("no material for region " + std::to_string(region));
  return it->second;
}
}  // namespace

// proj/src/assembly.cpp:34-61
TetGeometry tet_geometry(const std::array<std::array<double, 3>, 4>& p) {
  double e[3][3];
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d) e[c][d] = p[c + 1][d] - p[0][d];
  double cr[3][3];
  cr[0][0] = e[1][1] * e[2][2] - e[1][2] * e[2][1];
  cr[0][1] = e[1][2] * e[2][0] - e[1][0] * e[2][2];
  cr[0][2] = e[1][0] * e[2][1] - e[1][1] * e[2][0];
  cr[1][0] = e[2][1] * e[0][2] - e[2][2] * e[0][1];
  cr[1][1] = e[2][2] * e[0][0] - e[2][0] * e[0][2];
  cr[1][2] = e[2][0] * e[0][1] - e[2][1] * e[0][0];
  cr[2][0] = e[0][1] * e[1][2] - e[0][2] * e[1][1];
  cr[2][1] = e[0][2] * e[1][0] - e[0][0] * e[1][2];
  cr[2][2] = e[0][0] * e[1][1] - e[0][1] * e[1][0];
  const double det = e[0][0] * cr[0][0] + e[0][1] * cr[0][1] + e[0][2] * cr[0][2];
  if (det == 0.0) throw GeometryError("degenerate tetrahedron in element kernel");
  TetGeometry g;
  g.volume = det / 6.0;
  for (int i = 0; i < 3; ++i)
    for (int d = 0; d < 3; ++d) g.grad_lambda[i + 1][d] = cr[i][d] / det;
  for (int d = 0; d < 3; ++d)
    g.grad_lambda[0][d] = -g.grad_lambda[1][d] - g.grad_lambda[2][d] - g.grad_lambda[3][d];
  return g;
}

int quadrature_size(int order) { return order == 1 ? 1 : 4; }
double quadrature_weight(const TetGeometry& geo, int order, int) { return order == 1 ? geo.volume : 0.25 * geo.volume; }

// proj/src/assembly.cpp:69-85
void shape_gradients(const TetGeometry& geo, int order, int q, std::array<std::array<double, 3>, 10>& grads) {
  if (order == 1) {
    for (int i = 0; i < 4; ++i) grads[i] = geo.grad_lambda[i];
    return;
  }
  const double* lam = barycentric_point(order, q);
  for (int i = 0; i < 4; ++i) {
    const double f = 4.0 * lam[i] - 1.0;
    for (int d = 0; d < 3; ++d) grads[i][d] = f * geo.grad_lambda[i][d];
  }
  for (int e = 0; e < 6; ++e) {
    const int a = kTetEdgeVertices[e][0], b = kTetEdgeVertices[e][1];
    for (int d = 0; d < 3; ++d)
      grads[4 + e][d] = 4.0 * (lam[a] * geo.grad_lambda[b][d] + lam[b] * geo.grad_lambda[a][d]);
  }
}

// proj/src/assembly.cpp:87-95
double gradient_magnitude(const TetGeometry& geo, int order, int q, const double* x_loc) {
  std::array<std::array<double, 3>, 10> grads;
  shape_gradients(geo, order, q, grads);
  const int n = order == 1 ? 4 : 10;
  double g[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) g[d] += x_loc[i] * grads[i][d];
  return std::sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
}

// proj/src/assembly.cpp:97-116
void element_laplacian(const TetGeometry& geo, int order, const double* coeff_at_qp, double S[10][10]) {
  const int n = order == 1 ? 4 : 10;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) S[i][j] = 0.0;
  std::array<std::array<double, 3>, 10> grads;
  for (int q = 0; q < quadrature_size(order); ++q) {
    shape_gradients(geo, order, q, grads);
    const double wc = quadrature_weight(geo, order, q) * coeff_at_qp[q];
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) {
        const double gij = grads[i][0] * grads[j][0] + grads[i][1] * grads[j][1] + grads[i][2] * grads[j][2];
        S[i][j] += wc * gij;
      }
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) S[i][j] = S[j][i];
}

namespace {
using CoefficientFn = std::function<double(int, int, double)>;
// proj/src/assembly.cpp:130-170
CsrMatrix assemble_matrix(const TetMesh& mesh, const DofMap& dm, const CoefficientFn& coeff, const Vec& state) {
  const int n = dm.n_local;
  const bool has_state = (int)state.size() == dm.n_dofs;
  std::vector<std::vector<int>> pattern(dm.n_dofs);
  for (int t = 0; t < mesh.n_tets(); ++t)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) pattern[dm.element_dofs[t][i]].push_back(dm.element_dofs[t][j]);
  for (auto& row : pattern) {
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
  }
  CsrMatrix a = CsrMatrix::from_pattern(std::move(pattern));
  double S[10][10], c_at_qp[4], x_loc[10];
  for (int t = 0; t < mesh.n_tets(); ++t) {
    std::array<std::array<double, 3>, 4> coords;
    for (int v = 0; v < 4; ++v) coords[v] = mesh.nodes[mesh.tets[t][v]];
    const TetGeometry geo = tet_geometry(coords);
    if (has_state)
      for (int i = 0; i < n; ++i) x_loc[i] = state[dm.element_dofs[t][i]];
    for (int q = 0; q < quadrature_size(dm.order); ++q) {
      const double e_mag = has_state ? gradient_magnitude(geo, dm.order, q, x_loc) : 0.0;
      c_at_qp[q] = coeff(t, q, e_mag);
    }
    element_laplacian(geo, dm.order, c_at_qp, S);
    for (int i = 0; i < n; ++i) {
      const int gi = dm.element_dofs[t][i];
      for (int j = 0; j < n; ++j) *a.find(gi, dm.element_dofs[t][j]) += S[i][j];
    }
  }
  return a;
}
}  // namespace

// proj/src/assembly.cpp:172-176
CsrMatrix assemble_mass(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials) {
  return assemble_matrix(
      mesh, dm, [&](int t, int, double) { return material_for(materials, mesh.region_id[t]).permittivity(); }, Vec());
}
// proj/src/assembly.cpp:178-186
CsrMatrix assemble_stiffness(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials, const Vec& x_full) {
  return assemble_matrix(
      mesh, dm, [&](int t, int, double e) { return kappa_of_e(material_for(materials, mesh.region_id[t]), e); }, x_full);
}
// proj/src/assembly.cpp:188-193
DirichletBlocks split_dirichlet(const CsrMatrix& a, const DofMap& dm) {
  DirichletBlocks b;
  b.AII = extract_block(a, dm.free_dofs, dm.free_dofs);
  b.AIB = extract_block(a, dm.free_dofs, dm.fixed_dofs);
  return b;
}

// ------------------------------------------------------------------ csr
// proj/src/csr.cpp:14-22
void CsrMatrix::apply(const Vec& x, Vec& y) const {
  if ((int)x.size() != n_cols) throw NumericalError("CsrMatrix::apply: dimension mismatch");
  y.resize(n_rows);
  for (int i = 0; i < n_rows; ++i) {
    double s = 0.0;
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += values[k] * x[col_idx[k]];
    y[i] = s;
  }
}
// proj/src/csr.cpp:30-44
double CsrMatrix::coeff(int i, int j) const {
  const int* b = col_idx.data() + row_ptr[i];
  const int* e = col_idx.data() + row_ptr[i + 1];
  const int* it = std::lower_bound(b, e, j);
  if (it != e && *it == j) return values[it - col_idx.data()];
  return 0.0;
}
double* CsrMatrix::find(int i, int j) {
  const int* b = col_idx.data() + row_ptr[i];
  const int* e = col_idx.data() + row_ptr[i + 1];
  const int* it = std::lower_bound(b, e, j);
  if (it != e && *it == j) return values.data() + (it - col_idx.data());
  return nullptr;
}
Vec CsrMatrix::diagonal() const {
  Vec d(n_rows);
  for (int i = 0; i < n_rows; ++i) d[i] = coeff(i, i);
  return d;
}
// proj/src/csr.cpp:52-70
CsrMatrix CsrMatrix::transposed() const {
  CsrMatrix t;
  t.n_rows = n_cols;
  t.n_cols = n_rows;
  t.row_ptr.assign(n_cols + 1, 0);
  for (int c : col_idx) ++t.row_ptr[c + 1];
  for (int i = 0; i < n_cols; ++i) t.row_ptr[i + 1] += t.row_ptr[i];
  t.col_idx.resize(col_idx.size());
  t.values.resize(values.size());
  std::vector<int> next(t.row_ptr.begin(), t.row_ptr.end() - 1);
  for (int i = 0; i < n_rows; ++i)
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
      int pos = next[col_idx[k]]++;
      t.col_idx[pos] = i;
      t.values[pos] = values[k];
    }
  return t;
}
// proj/src/csr.cpp:79-90
double CsrMatrix::symmetry_error() const {
  if (n_rows != n_cols) return INFINITY;
  double scale = 0.0;
  for (double v : values) scale = std::max(scale, std::abs(v));
  if (scale == 0.0) return 0.0;
  double err = 0.0;
  for (int i = 0; i < n_rows; ++i)
    for (int k = row_ptr[i]; k < row_ptr[i + 1]; ++k) err = std::max(err, std::abs(values[k] - coeff(col_idx[k], i)));
  return err / scale;
}
// proj/src/csr.cpp:92-119
CsrMatrix CsrMatrix::from_triplets(int n_rows, int n_cols, std::vector<std::array<int, 2>> pattern,
                                   const std::vector<double>& vals) {
  std::vector<int> order(pattern.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return pattern[a] < pattern[b]; });
  CsrMatrix m;
  m.n_rows = n_rows;
  m.n_cols = n_cols;
  m.row_ptr.assign(n_rows + 1, 0);
  int li = -1, lj = -1;
  for (int o : order) {
    int i = pattern[o][0], j = pattern[o][1];
    if (i == li && j == lj) {
      m.values.back() += vals[o];
      continue;
    }
    ++m.row_ptr[i + 1];
    m.col_idx.push_back(j);
    m.values.push_back(vals[o]);
    li = i;
    lj = j;
  }
  for (int i = 0; i < n_rows; ++i) m.row_ptr[i + 1] += m.row_ptr[i];
  return m;
}
// proj/src/csr.cpp:121-131
CsrMatrix CsrMatrix::from_pattern(std::vector<std::vector<int>> row_cols) {
  CsrMatrix m;
  m.n_rows = (int)row_cols.size();
  m.n_cols = m.n_rows;
  m.row_ptr.assign(m.n_rows + 1, 0);
  for (int i = 0; i < m.n_rows; ++i) m.row_ptr[i + 1] = m.row_ptr[i] + (int)row_cols[i].size();
  m.col_idx.reserve(m.row_ptr.back());
  for (auto& cols : row_cols) m.col_idx.insert(m.col_idx.end(), cols.begin(), cols.end());
  m.values.assign(m.col_idx.size(), 0.0);
  return m;
}
// proj/src/csr.cpp:133-166
CsrMatrix multiply(const CsrMatrix& a, const CsrMatrix& b) {
  if (a.n_cols != b.n_rows) throw NumericalError("csr multiply: dimension mismatch");
  CsrMatrix c;
  c.n_rows = a.n_rows;
  c.n_cols = b.n_cols;
  c.row_ptr.assign(a.n_rows + 1, 0);
  std::vector<double> accum(b.n_cols, 0.0);
  std::vector<int> marker(b.n_cols, -1);
  std::vector<int> cols;
  for (int i = 0; i < a.n_rows; ++i) {
    cols.clear();
    for (int ka = a.row_ptr[i]; ka < a.row_ptr[i + 1]; ++ka) {
      const int k = a.col_idx[ka];
      const double av = a.values[ka];
      for (int kb = b.row_ptr[k]; kb < b.row_ptr[k + 1]; ++kb) {
        const int j = b.col_idx[kb];
        if (marker[j] != i) {
          marker[j] = i;
          accum[j] = 0.0;
          cols.push_back(j);
        }
        accum[j] += av * b.values[kb];
      }
    }
    std::sort(cols.begin(), cols.end());
    for (int j : cols) {
      c.col_idx.push_back(j);
      c.values.push_back(accum[j]);
    }
    c.row_ptr[i + 1] = (int)c.col_idx.size();
  }
  return c;
}
// proj/src/csr.cpp:168-195 (pattern union, values alpha a + beta b)
CsrMatrix add(double alpha, const CsrMatrix& a, double beta, const CsrMatrix& b) {
  if (a.n_rows != b.n_rows || a.n_cols != b.n_cols) throw NumericalError("csr add: dimension mismatch");
  CsrMatrix c;
  c.n_rows = a.n_rows;
  c.n_cols = a.n_cols;
  c.row_ptr.assign(a.n_rows + 1, 0);
  for (int i = 0; i < a.n_rows; ++i) {
    int ka = a.row_ptr[i], kb = b.row_ptr[i];
    const int ea = a.row_ptr[i + 1], eb = b.row_ptr[i + 1];
    while (ka < ea || kb < eb) {
      const int ja = ka < ea ? a.col_idx[ka] : c.n_cols;
      const int jb = kb < eb ? b.col_idx[kb] : c.n_cols;
      if (ja == jb) {
        c.col_idx.push_back(ja);
        c.values.push_back(alpha * a.values[ka++] + beta * b.values[kb++]);
      } else if (ja < jb) {
        c.col_idx.push_back(ja);
        c.values.push_back(alpha * a.values[ka++]);
      } else {
        c.col_idx.push_back(jb);
        c.values.push_back(beta * b.values[kb++]);
      }
    }
    c.row_ptr[i + 1] = (int)c.col_idx.size();
  }
  return c;
}

// proj/src/csr.cpp:197-229
CsrMatrix extract_block(const CsrMatrix& a, const std::vector<int>& rows, const std::vector<int>& cols) {
  std::vector<int> col_map(a.n_cols, -1);
  for (int c = 0; c < (int)cols.size(); ++c) col_map[cols[c]] = c;
  CsrMatrix blk;
  blk.n_rows = (int)rows.size();
  blk.n_cols = (int)cols.size();
  blk.row_ptr.assign(blk.n_rows + 1, 0);
  for (int r = 0; r < blk.n_rows; ++r) {
    const int i = rows[r];
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int c = col_map[a.col_idx[k]];
      if (c >= 0) {
        blk.col_idx.push_back(c);
        blk.values.push_back(a.values[k]);
      }
    }
    blk.row_ptr[r + 1] = (int)blk.col_idx.size();
    int b = blk.row_ptr[r], e = blk.row_ptr[r + 1];
    std::vector<std::pair<int, double>> tmp;
    for (int k = b; k < e; ++k) tmp.emplace_back(blk.col_idx[k], blk.values[k]);
    std::sort(tmp.begin(), tmp.end());
    for (int k = b; k < e; ++k) {
      blk.col_idx[k] = tmp[k - b].first;
      blk.values[k] = tmp[k - b].second;
    }
  }
  return blk;
}

// ------------------------------------------------------------------ matfree
// proj/src/matfree.cpp:11-38
std::vector<std::vector<int>> color_elements(const DofMap& dm, int n_tets) {
  const int n = dm.n_local;
  std::vector<std::vector<int>> tets_of_dof(dm.n_dofs);
  for (int t = 0; t < n_tets; ++t)
    for (int i = 0; i < n; ++i) tets_of_dof[dm.element_dofs[t][i]].push_back(t);
  std::vector<int> color(n_tets, -1);
  std::vector<int> used;
  int n_colors = 0;
  for (int t = 0; t < n_tets; ++t) {
    used.clear();
    for (int i = 0; i < n; ++i)
      for (int nb : tets_of_dof[dm.element_dofs[t][i]])
        if (color[nb] >= 0) used.push_back(color[nb]);
    std::sort(used.begin(), used.end());
    int c = 0;
    for (int u : used) {
      if (u == c) ++c;
      else if (u > c) break;
    }
    color[t] = c;
    n_colors = std::max(n_colors, c + 1);
  }
  std::vector<std::vector<int>> batches(n_colors);
  for (int t = 0; t < n_tets; ++t) batches[color[t]].push_back(t);
  return batches;
}

// proj/src/matfree.cpp:40-52
MatFreeStiffness::MatFreeStiffness(const TetMesh& mesh, const DofMap& dm, const MaterialTable& materials, int workers)
    : mesh_(mesh), dm_(dm), workers_(std::max(1, workers)) {
  material_of_tet_.resize(mesh.n_tets());
  for (int t = 0; t < mesh.n_tets(); ++t) {
    auto it = materials.find(mesh.region_id[t]);
    if (it == materials.end()) throw ConfigError("no material for region " + std::to_string(mesh.region_id[t]));
    material_of_tet_[t] = &it->second;
  }
  color_batches_ = color_elements(dm, mesh.n_tets());
}

namespace {
struct ElementScratch {
  double S[10][10], kappa_at_qp[4], x_loc[10], v_loc[10], y_loc[10];
};
// proj/src/matfree.cpp:65-86
inline void fused_element_product(const TetMesh& mesh, const DofMap& dm, const MaterialModel& mat, int t,
                                  const Vec& x_state, const Vec& v, ElementScratch& s) {
  const int n = dm.n_local;
  std::array<std::array<double, 3>, 4> coords;
  for (int vtx = 0; vtx < 4; ++vtx) coords[vtx] = mesh.nodes[mesh.tets[t][vtx]];
  const TetGeometry geo = tet_geometry(coords);
  for (int i = 0; i < n; ++i) {
    s.x_loc[i] = x_state[dm.element_dofs[t][i]];
    s.v_loc[i] = v[dm.element_dofs[t][i]];
  }
  for (int q = 0; q < quadrature_size(dm.order); ++q)
    s.kappa_at_qp[q] = kappa_of_e(mat, gradient_magnitude(geo, dm.order, q, s.x_loc));
  element_laplacian(geo, dm.order, s.kappa_at_qp, s.S);
  for (int i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += s.S[i][j] * s.v_loc[j];
    s.y_loc[i] = acc;
  }
}
}  // namespace

// proj/src/matfree.cpp:90-117 (colored scatter)
void MatFreeStiffness::apply(const Vec& x_state, const Vec& v, Vec& y) const {
  if ((int)x_state.size() != dm_.n_dofs || (int)v.size() != dm_.n_dofs)
    throw std::invalid_argument("MatFreeStiffness::apply: dimension mismatch");
  ++applies_;
  const int n = dm_.n_local;
  y.assign(dm_.n_dofs, 0.0);
  for (const auto& batch : color_batches_) {
    const int m = (int)batch.size();
    // exceptions cannot cross an OpenMP region: capture the first one
    std::exception_ptr err;
#pragma omp parallel num_threads(workers_)
    {
      ElementScratch scratch;
#pragma omp for schedule(static)
      for (int k = 0; k < m; ++k) {
        const int t = batch[k];
        try {
          fused_element_product(mesh_, dm_, *material_of_tet_[t], t, x_state, v, scratch);
          for (int i = 0; i < n; ++i) y[dm_.element_dofs[t][i]] += scratch.y_loc[i];
        } catch (...) {
#pragma omp critical
          if (!err) err = std::current_exception();
        }
      }
    }
    if (err) std::rethrow_exception(err);
  }
}

// proj/src/matfree.cpp:138-143
void MatFreeStiffness::residual(const Vec& x_full, const Vec& b_mass, Vec& r) const {
  Vec y;
  apply(x_full, x_full, y);
  r.resize(dm_.n_free());
  for (int i = 0; i < dm_.n_free(); ++i) r[i] = b_mass[i] - y[dm_.free_dofs[i]];
}

}  // namespace ora
