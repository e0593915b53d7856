// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/pcg.cpp, preconditioners.cpp, amg.cpp and the Eigen::LDLT
// calls they make.
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>

#include "oracle.hpp"

namespace ora {

namespace {
double dot(const Vec& a, const Vec& b) {  // Eigen's a.dot(b) summation order
  return eigen_redux_sum(a.size(), [&](size_t i) { return a[i] * b[i]; });
}
double norm(const Vec& a) { return std::sqrt(dot(a, a)); }
}  // namespace

// proj/src/pcg.cpp:9-72
PcgResult pcg_solve(const LinearOperator& a, const LinearOperator& precond, const Vec& b, const Vec& x0,
                    double rel_tol, int max_iter) {
  const int n = a.rows();
  if ((int)b.size() != n || (!x0.empty() && (int)x0.size() != n))
    throw std::invalid_argument("pcg_solve: dimension mismatch");
  PcgResult res;
  const double bnorm = norm(b);
  if (bnorm == 0.0) {
    res.x.assign(n, 0.0);
    res.converged = true;
    return res;
  }
  res.x = (int)x0.size() == n ? x0 : Vec(n, 0.0);
  Vec r(n), q(n), z(n);
  if ((int)x0.size() == n && dot(x0, x0) != 0.0) {
    a.apply(res.x, q);
    for (int i = 0; i < n; ++i) r[i] = b[i] - q[i];
  } else {
    r = b;
  }
  double rel = norm(r) / bnorm;
  res.initial_rel_residual = rel;
  res.rel_residual = rel;
  if (!std::isfinite(rel)) throw NumericalError("pcg: non-finite initial residual");
  if (rel <= rel_tol) {
    res.converged = true;
    return res;
  }
  precond.apply(r, z);
  Vec p = z;
  double rz = dot(r, z);
  if (!std::isfinite(rz)) throw NumericalError("pcg: non-finite preconditioned residual");
  for (int k = 1; k <= max_iter; ++k) {
    a.apply(p, q);
    const double pq = dot(p, q);
    if (!(pq > 0.0) || !std::isfinite(pq)) throw NumericalError("pcg: operator not positive definite");
    const double alpha = rz / pq;
    for (int i = 0; i < n; ++i) res.x[i] += alpha * p[i];
    for (int i = 0; i < n; ++i) r[i] -= alpha * q[i];
    rel = norm(r) / bnorm;
    res.iterations = k;
    res.rel_residual = rel;
    if (!std::isfinite(rel)) throw NumericalError("pcg: non-finite residual");
    if (rel <= rel_tol) {
      res.converged = true;
      return res;
    }
    precond.apply(r, z);
    const double rz_new = dot(r, z);
    if (!std::isfinite(rz_new)) throw NumericalError("pcg: non-finite preconditioned residual");
    const double beta = rz_new / rz;
    for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  return res;
}

// proj/src/preconditioners.cpp:7-20
std::vector<int> diagonal_positions(const CsrMatrix& a) {
  std::vector<int> pos(a.n_rows, -1);
  for (int i = 0; i < a.n_rows; ++i) {
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.col_idx[k] == i) {
        pos[i] = k;
        break;
      }
    if (pos[i] < 0 || a.values[pos[i]] == 0.0)
      throw NumericalError("matrix has a missing or zero diagonal entry at row " + std::to_string(i));
  }
  return pos;
}
// proj/src/preconditioners.cpp:22-32
JacobiPreconditioner::JacobiPreconditioner(const CsrMatrix& a) {
  inv_diag_ = a.diagonal();
  for (double& d : inv_diag_) {
    if (d == 0.0) throw NumericalError("Jacobi: zero diagonal");
    d = 1.0 / d;
  }
}
void JacobiPreconditioner::apply(const Vec& r, Vec& z) const {
  z.resize(r.size());
  for (size_t i = 0; i < r.size(); ++i) z[i] = inv_diag_[i] * r[i];
}
// proj/src/preconditioners.cpp:34-60
SsorPreconditioner::SsorPreconditioner(const CsrMatrix& a) : a_(a) { diag_pos_ = diagonal_positions(a_); }
void SsorPreconditioner::apply(const Vec& r, Vec& z) const {
  const int n = a_.n_rows;
  Vec y(n);
  for (int i = 0; i < n; ++i) {
    double s = r[i];
    for (int k = a_.row_ptr[i]; k < a_.row_ptr[i + 1]; ++k) {
      const int j = a_.col_idx[k];
      if (j < i) s -= a_.values[k] * y[j];
    }
    y[i] = s / a_.values[diag_pos_[i]];
  }
  z.resize(n);
  for (int i = n - 1; i >= 0; --i) {
    double s = a_.values[diag_pos_[i]] * y[i];
    for (int k = a_.row_ptr[i]; k < a_.row_ptr[i + 1]; ++k) {
      const int j = a_.col_idx[k];
      if (j > i) s -= a_.values[k] * z[j];
    }
    z[i] = s / a_.values[diag_pos_[i]];
  }
}
// proj/src/preconditioners.cpp:62-84
void gauss_seidel_forward(const CsrMatrix& a, const std::vector<int>& dp, const Vec& b, Vec& x) {
  for (int i = 0; i < a.n_rows; ++i) {
    double s = b[i];
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j != i) s -= a.values[k] * x[j];
    }
    x[i] = s / a.values[dp[i]];
  }
}
void gauss_seidel_backward(const CsrMatrix& a, const std::vector<int>& dp, const Vec& b, Vec& x) {
  for (int i = a.n_rows - 1; i >= 0; --i) {
    double s = b[i];
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j != i) s -= a.values[k] * x[j];
    }
    x[i] = s / a.values[dp[i]];
  }
}

// Eigen::LDLT<MatrixXd> (lower, diagonal pivoting on the largest remaining
// |diagonal|), restated for the coarse solve (proj/src/amg.cpp:140) and the
// SPE reduced system (proj/src/start_vector.cpp:42-48).
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
      // symmetric swap of rows/cols k and idx (lower triangle semantics on a full copy)
      for (int j = 0; j < n; ++j) std::swap(M(k, j), M(idx, j));
      for (int i = 0; i < n; ++i) std::swap(M(i, k), M(i, idx));
    }
    const int rs = n - k - 1;
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = M(j, j) * M(k, j);
      double s = 0.0;
      for (int j = 0; j < k; ++j) s += M(k, j) * temp[j];
      M(k, k) -= s;
      for (int i = k + 1; i < n; ++i) {
        double t = 0.0;
        for (int j = 0; j < k; ++j) t += M(i, j) * temp[j];
        M(i, k) -= t;
      }
    }
    const double akk = M(k, k);
    const bool valid = std::abs(akk) > std::numeric_limits<double>::min();
    if (rs > 0 && valid) {
      for (int i = k + 1; i < n; ++i) M(i, k) /= akk;
    } else if (rs > 0) {
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

namespace {
// proj/src/amg.cpp:15-26
std::vector<std::vector<int>> strength_graph(const CsrMatrix& a, double theta) {
  const Vec d = a.diagonal();
  std::vector<std::vector<int>> strong(a.n_rows);
  for (int i = 0; i < a.n_rows; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
      const int j = a.col_idx[k];
      if (j == i) continue;
      if (std::abs(a.values[k]) >= theta * std::sqrt(std::abs(d[i] * d[j]))) strong[i].push_back(j);
    }
  return strong;
}
// proj/src/amg.cpp:28-45
double estimate_lambda_max_scaled(const CsrMatrix& a) {
  const Vec d = a.diagonal();
  std::mt19937 rng(20240811u);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  Vec v(a.n_rows);
  for (int i = 0; i < a.n_rows; ++i) v[i] = uni(rng);
  double nv = norm(v);
  for (double& e : v) e /= nv;
  double lambda = 1.0;
  Vec w;
  for (int it = 0; it < 10; ++it) {
    a.apply(v, w);
    for (int i = 0; i < a.n_rows; ++i) w[i] /= d[i];
    lambda = norm(w);
    if (lambda == 0.0) return 1.0;
    for (int i = 0; i < a.n_rows; ++i) v[i] = w[i] / lambda;
  }
  return lambda;
}
}  // namespace

// proj/src/amg.cpp:49-88
std::vector<int> aggregate(const CsrMatrix& a, double theta) {
  const auto strong = strength_graph(a, theta);
  const int n = a.n_rows;
  std::vector<int> agg(n, -1);
  int n_agg = 0;
  for (int i = 0; i < n; ++i) {
    if (agg[i] >= 0) continue;
    bool clean = true;
    for (int j : strong[i])
      if (agg[j] >= 0) {
        clean = false;
        break;
      }
    if (!clean || strong[i].empty()) continue;
    agg[i] = n_agg;
    for (int j : strong[i]) agg[j] = n_agg;
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

// proj/src/amg.cpp:90-143
AmgPreconditioner::AmgPreconditioner(const CsrMatrix& a, const AmgParams& params) : params_(params) {
  if (a.n_rows != a.n_cols) throw std::invalid_argument("amg: matrix must be square");
  if (a.symmetry_error() > 1e-10) throw std::invalid_argument("amg: matrix is not symmetric");
  levels_.push_back({a, diagonal_positions(a), {}, {}, {}});
  while ((int)levels_.size() < params_.max_levels && levels_.back().A.n_rows > params_.coarse_limit) {
    const CsrMatrix& fine = levels_.back().A;
    std::vector<int> agg = aggregate(fine, params_.strength_threshold);
    const int n_agg = *std::max_element(agg.begin(), agg.end()) + 1;
    if (n_agg >= fine.n_rows) break;
    std::vector<int> agg_size(n_agg, 0);
    for (int id : agg) ++agg_size[id];
    CsrMatrix p_tent;
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
    const double omega = params_.prolongation_omega / estimate_lambda_max_scaled(fine);
    CsrMatrix scaled = fine;
    const Vec d = fine.diagonal();
    for (int i = 0; i < fine.n_rows; ++i)
      for (int k = scaled.row_ptr[i]; k < scaled.row_ptr[i + 1]; ++k) {
        scaled.values[k] = -omega * scaled.values[k] / d[i];
        if (scaled.col_idx[k] == i) scaled.values[k] += 1.0;
      }
    CsrMatrix p = multiply(scaled, p_tent);
    CsrMatrix r = p.transposed();
    CsrMatrix coarse = multiply(r, multiply(fine, p));
    levels_.back().P = std::move(p);
    levels_.back().R = std::move(r);
    levels_.back().aggregates = std::move(agg);
    levels_.push_back({std::move(coarse), {}, {}, {}, {}});
    levels_.back().diag_pos = diagonal_positions(levels_.back().A);
  }
  const CsrMatrix& c = levels_.back().A;
  std::vector<double> dense((size_t)c.n_rows * c.n_rows, 0.0);
  for (int i = 0; i < c.n_rows; ++i)
    for (int k = c.row_ptr[i]; k < c.row_ptr[i + 1]; ++k) dense[(size_t)i * c.n_rows + c.col_idx[k]] += c.values[k];
  coarse_.compute(dense, c.n_rows);
  if (!coarse_.ok) throw NumericalError("amg: coarsest-level factorization failed");
}

// proj/src/amg.cpp:145-172
void AmgPreconditioner::vcycle(size_t l, const Vec& r, Vec& z) const {
  const AmgLevel& lev = levels_[l];
  if (l + 1 == levels_.size()) {
    z.resize(r.size());
    coarse_.solve(r.data(), z.data());
    return;
  }
  z.assign(lev.A.n_rows, 0.0);
  for (int s = 0; s < params_.smoother_sweeps; ++s) {
    gauss_seidel_forward(lev.A, lev.diag_pos, r, z);
    gauss_seidel_backward(lev.A, lev.diag_pos, r, z);
  }
  Vec az;
  lev.A.apply(z, az);
  for (size_t i = 0; i < az.size(); ++i) az[i] = r[i] - az[i];
  Vec rc;
  lev.R.apply(az, rc);
  Vec zc;
  vcycle(l + 1, rc, zc);
  Vec pz;
  lev.P.apply(zc, pz);
  for (size_t i = 0; i < z.size(); ++i) z[i] += pz[i];
  for (int s = 0; s < params_.smoother_sweeps; ++s) {
    gauss_seidel_forward(lev.A, lev.diag_pos, r, z);
    gauss_seidel_backward(lev.A, lev.diag_pos, r, z);
  }
}

}  // namespace ora
