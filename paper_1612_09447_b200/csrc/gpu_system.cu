// GpuSystem: device-resident FemSystem + integrator.
//
// Device dof numbering: free dofs first (in DofMap::free_dofs order), then the
// fixed dofs. A "full" vector therefore holds the free state in [0, n_free)
// and the Dirichlet values in the tail, so lifting a stage vector
// (DofMap::lift, proj/src/dofmap.cpp:11-15) is a write of n_fixed entries and
// restricting (restrict_free, :17-20) is free.
#include "gpu_system.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

namespace eqsb {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class T>
DevBuf<T>::~DevBuf() {
  if (p) cudaFree(p);
}
template <class T>
void DevBuf<T>::alloc(size_t count) {
  if (p) cudaFree(p);
  p = nullptr;
  n = count;
  if (count) CK(cudaMalloc(&p, count * sizeof(T)));
}
template <class T>
void DevBuf<T>::upload(const T* host, size_t count, cudaStream_t s) {
  if (count) CK(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
void DevBuf<T>::download(T* host, size_t count, cudaStream_t s) const {
  if (count) CK(cudaMemcpyAsync(host, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}
template struct DevBuf<double>;
template struct DevBuf<int>;
template struct DevBuf<long>;
template struct DevBuf<unsigned>;
template struct DevBuf<unsigned char>;

namespace {
using clk = std::chrono::steady_clock;
struct PhaseTimer {
  double& slot;
  clk::time_point t0;
  explicit PhaseTimer(double& s) : slot(s), t0(clk::now()) {}
  ~PhaseTimer() { slot += std::chrono::duration<double>(clk::now() - t0).count(); }
};

// threads per row: enough that each thread handles <= 8 entries (one batch of
// the row kernels' prefetch), capped at a warp
int choose_tpr(const HostCsr& a) {
  if (a.n_rows == 0) return 1;
  const double avg = (double)a.nnz() / a.n_rows;
  int t = 1;
  while (t < 32 && t * 8 < avg) t <<= 1;
  return t;
}

void upload_csr(const HostCsr& h, DevCsr& d, DevBuf<int>& rp, DevBuf<int>& ci, DevBuf<double>& v, cudaStream_t s) {
  d.n_rows = h.n_rows;
  d.n_cols = h.n_cols;
  d.nnz = h.nnz();
  rp.alloc(h.row_ptr.size());
  ci.alloc(std::max<size_t>(1, h.col_idx.size()));
  v.alloc(std::max<size_t>(1, h.values.size()));
  rp.upload(h.row_ptr.data(), h.row_ptr.size(), s);
  ci.upload(h.col_idx.data(), h.col_idx.size(), s);
  v.upload(h.values.data(), h.values.size(), s);
  d.row_ptr = rp.p;
  d.col_idx = ci.p;
  d.values = v.p;
  d.tpr = choose_tpr(h);
}

std::vector<double> inv_diagonal(const HostCsr& a) {
  std::vector<double> d(a.n_rows, 0.0);
  for (int i = 0; i < a.n_rows; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.col_idx[k] == i) d[i] = 1.0 / a.values[k];
  return d;
}
}  // namespace

GpuSystem::GpuSystem(Problem&& p, int device) : prob_(std::move(p)), device_(device) {
  PhaseTimer timer(stats_.t_setup);
  if (device_ >= 0) {
    CK(cudaSetDevice(device_));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    CK(cudaMallocHost(&pinned_, sizeof(double) * (S_COUNT + 8)));
  }
  const Dofs& dm = prob_.dm;
  n_dofs_ = dm.n_dofs;
  n_free_ = dm.n_free();
  n_fixed_ = dm.n_fixed();
  n_tets_ = prob_.mesh.n_tets;
  n_local_ = dm.n_local;
  order_ = dm.order;
  n_sets_ = (int)dm.set_names.size();
  if (n_sets_ > kMaxSets) throw ConfigError("too many Dirichlet sets for the GPU backend");
  if ((int)prob_.materials.size() > kMaxMaterials) throw ConfigError("too many materials for the GPU backend");
  for (int t = 0; t < n_tets_; ++t)
    if (!prob_.materials.count(prob_.mesh.region[t]))
      throw ConfigError("no material for region " + std::to_string(prob_.mesh.region[t]));
  dev2ref_.resize(n_dofs_);
  ref2dev_.resize(n_dofs_);
  for (int i = 0; i < n_free_; ++i) dev2ref_[i] = dm.free_dofs[i];
  for (int i = 0; i < n_fixed_; ++i) dev2ref_[n_free_ + i] = dm.fixed_dofs[i];
  for (int k = 0; k < n_dofs_; ++k) ref2dev_[dev2ref_[k]] = k;
  // FemSystem ctor: assemble M once (fem_system.cpp:27-36)
  assemble_mass_blocks(prob_, m_ii_, m_ib_);
  ++stats_.assemblies;
  // mass preconditioner (built once; the reference builds it lazily on first use, fem_system.cpp:48-54)
  if (prob_.solver.precond == 2) amg_ = build_amg(m_ii_, prob_.solver);
  ++stats_.precond_setups;
  if (device_ >= 0) build_device();  // device < 0: host-only setup (artefact checks without a GPU)
}

GpuSystem::~GpuSystem() {
  invalidate_graphs();
  for (auto& e : events_) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  if (pinned_) cudaFreeHost(pinned_);
  if (stream_) cudaStreamDestroy(stream_);
}

void GpuSystem::build_device() {
  const Dofs& dm = prob_.dm;
  const Mesh& mesh = prob_.mesh;
  cudaStream_t s = stream_;
  // coordinates per device dof (vertex dofs = nodes; P2 edge dofs = midpoints, unused by K1)
  {
    std::vector<double> c((size_t)n_dofs_ * 4, 0.0);
    std::vector<std::array<double, 3>> dc(n_dofs_);
    for (int n = 0; n < mesh.n_nodes; ++n) dc[n] = {mesh.nodes[3L * n], mesh.nodes[3L * n + 1], mesh.nodes[3L * n + 2]};
    for (int k = 0; k < n_dofs_; ++k) {
      const int r = dev2ref_[k];
      if (r < mesh.n_nodes)
        for (int d = 0; d < 3; ++d) c[4L * k + d] = dc[r][d];
    }
    coords_.alloc(c.size());
    coords_.upload(c.data(), c.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  // connectivity in device numbering + material index
  std::map<int, int> mat_index;
  std::vector<DevMaterial> mats;
  for (const auto& [region, m] : prob_.materials) {
    mat_index[region] = (int)mats.size();
    DevMaterial d{};
    d.kind = m.kind;
    d.kappa = m.kappa;
    if (m.kind == 1) {
      d.lo = std::log10(m.kappa_lo);
      d.hi = std::log10(m.kappa_hi);
      d.e_switch = m.e_switch;
      d.inv_width = 1.0 / m.width;
    }
    mats.push_back(d);
  }
  set_materials(mats.data(), (int)mats.size(), s);
  {
    std::vector<int> td((size_t)n_tets_ * n_local_);
    std::vector<unsigned char> tm(n_tets_);
#pragma omp parallel for schedule(static)
    for (long t = 0; t < n_tets_; ++t) {
      for (int i = 0; i < n_local_; ++i) td[t * n_local_ + i] = ref2dev_[dm.element_dofs[t * n_local_ + i]];
      tm[t] = (unsigned char)mat_index.at(mesh.region[t]);
    }
    tet_dofs_.alloc(td.size());
    tet_dofs_.upload(td.data(), td.size(), s);
    tet_mat_.alloc(tm.size());
    tet_mat_.upload(tm.data(), tm.size(), s);
    // slot lists: device dof -> (t * n_local + i), ascending t
    std::vector<long> ptr((size_t)n_dofs_ + 1, 0);
    for (size_t k = 0; k < td.size(); ++k) ++ptr[td[k] + 1];
    for (int d = 0; d < n_dofs_; ++d) ptr[d + 1] += ptr[d];
    if (ptr.back() >= (1L << 31)) throw ConfigError("mesh too large for int32 slot indices");
    std::vector<int> sl(ptr.back());
    std::vector<long> next(ptr.begin(), ptr.end() - 1);
    for (size_t k = 0; k < td.size(); ++k) sl[next[td[k]]++] = (int)k;
    slot_ptr_.alloc(ptr.size());
    slot_ptr_.upload(ptr.data(), ptr.size(), s);
    slots_.alloc(sl.size());
    slots_.upload(sl.data(), sl.size(), s);
    ytet_.alloc((size_t)n_tets_ * n_local_);
    CK(cudaStreamSynchronize(s));
  }
  err_.alloc(4);
  CK(cudaMemsetAsync(err_.p, 0, 4 * sizeof(int), s));
  // Dirichlet data: set of every fixed dof; compressed M_IB rows per set
  {
    std::vector<int> sof(std::max(1, n_fixed_));
    for (int i = 0; i < n_fixed_; ++i) sof[i] = dm.fixed_set[dm.fixed_dofs[i]];
    set_of_fixed_.alloc(sof.size());
    set_of_fixed_.upload(sof.data(), sof.size(), s);
    std::vector<int> rows;
    std::vector<double> coef;
    for (int r = 0; r < m_ib_.n_rows; ++r) {
      if (m_ib_.row_ptr[r] == m_ib_.row_ptr[r + 1]) continue;
      rows.push_back(r);
      std::vector<double> c(n_sets_, 0.0);
      for (int k = m_ib_.row_ptr[r]; k < m_ib_.row_ptr[r + 1]; ++k) c[sof[m_ib_.col_idx[k]]] += m_ib_.values[k];
      coef.insert(coef.end(), c.begin(), c.end());
    }
    n_bl_rows_ = (int)rows.size();
    bl_rows_.alloc(std::max<size_t>(1, rows.size()));
    bl_rows_.upload(rows.data(), rows.size(), s);
    bl_coef_.alloc(std::max<size_t>(1, coef.size()));
    bl_coef_.upload(coef.data(), coef.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  // M_II
  upload_csr(m_ii_, mii_, mii_rp_, mii_ci_, mii_v_, s);
  {
    const std::vector<double> invd = inv_diagonal(m_ii_);
    for (double v : invd)
      if (!std::isfinite(v)) throw NumericalError("Jacobi: zero diagonal");
    mii_invd_.alloc(std::max(1, n_free_));
    mii_invd_.upload(invd.data(), invd.size(), s);
  }
  // AMG hierarchy
  if (prob_.solver.precond == 2) {
    const int L = (int)amg_.levels.size();
    levels_.resize(L);
    auto f32 = [&](const std::vector<double>& v, DevBuf<float>& out) {
      std::vector<float> f(v.begin(), v.end());
      out.alloc(std::max<size_t>(1, f.size()));
      out.upload(f.data(), f.size(), s);
      CK(cudaStreamSynchronize(s));
    };
    const double eps = prob_.solver.amg_coarse_filter;
    for (int l = 0; l < L; ++l) {
      DevLevel& lv = levels_[l];
      const AmgHostLevel& hl = amg_.levels[l];
      // V-cycle operator: the fine level uses M_II itself; coarse levels use the
      // lumped filtered Galerkin operator
      HostCsr filtered;
      const bool filt = l > 0 && l + 1 < L && eps > 0.0;
      if (filt) filtered = filter_lumped(hl.A, eps);
      const HostCsr& av = filt ? filtered : hl.A;
      if (l == 0) {
        lv.A = mii_;  // shares indices / fp64 values with the PCG operator
      } else {
        upload_csr(av, lv.A, lv.a_rp, lv.a_ci, lv.a_v, s);
      }
      const int n = hl.A.n_rows;
      if (l + 1 < L) {
        f32(av.values, lv.a_vf);
        upload_csr(hl.P, lv.P, lv.p_rp, lv.p_ci, lv.p_v, s);
        upload_csr(hl.R, lv.R, lv.r_rp, lv.r_ci, lv.r_v, s);
        f32(hl.P.values, lv.p_vf);
        f32(hl.R.values, lv.r_vf);
        const std::vector<double> invd = inv_diagonal(av);
        lv.invd.alloc(n);
        lv.invd.upload(invd.data(), n, s);
        lv.t.alloc(n);
        lv.z2.alloc(std::max(1, n));
      }
      lv.z.alloc(std::max(1, n));
      if (l > 0) lv.b.alloc(std::max(1, n));
      CK(cudaStreamSynchronize(s));
    }
    set_vcycle_fp32(vcycle_fp32_);
    coarse_n_ = amg_.coarse_n;
    coarse_inv_.alloc(amg_.coarse_inverse.size());
    coarse_inv_.upload(amg_.coarse_inverse.data(), amg_.coarse_inverse.size(), s);
  }
  // reductions + work vectors
  red_partials_.alloc((size_t)S_COUNT * kRedGrid);
  red_scal_.alloc(S_COUNT);
  red_counters_.alloc(S_COUNT);
  CK(cudaMemsetAsync(red_counters_.p, 0, sizeof(unsigned) * S_COUNT, s));
  CK(cudaMemsetAsync(red_scal_.p, 0, sizeof(double) * S_COUNT, s));
  red_ = Reducer{red_partials_.p, red_counters_.p, red_scal_.p};
  const size_t nf = std::max(1, n_free_), nd = std::max(1, n_dofs_);
  for (auto* b : {&w_r_, &w_z_, &w_p_, &w_q_, &w_free_a_, &w_free_b_, &F0_, &F_, &Fn_, &rho_v_, &rho_w_}) b->alloc(nf);
  for (auto* b : {&w_full_a_, &w_full_b_}) b->alloc(nd);
  for (auto& b : full_) {
    b.alloc(nd);
    launch_fill((long)nd, 0.0, b.p, s);
  }
  X_ = full_[0].p;
  CK(cudaStreamSynchronize(s));
  // smoother bounds: lambda_max(D^-1 A) per level by 20 device power iterations
  if (prob_.solver.precond == 2) {
    std::mt19937 rng(12345u);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (int l = 0; l + 1 < (int)levels_.size(); ++l) {
      DevLevel& lv = levels_[l];
      const int n = lv.A.n_rows;
      std::vector<double> v(n);
      double nrm = 0.0;
      for (auto& e : v) {
        e = uni(rng);
        nrm += e * e;
      }
      nrm = std::sqrt(nrm);
      for (auto& e : v) e /= nrm;
      lv.z.upload(v.data(), n, s);
      double lam = 1.0;
      for (int it = 0; it < 20; ++it) {
        launch_scaled_spmv(lv.A, lv.invd.p, lv.z.p, lv.t.p, s);
        launch_dot(n, lv.t.p, lv.t.p, red_, S_NORM, s);
        lam = std::sqrt(read_scalar(S_NORM));
        if (lam == 0.0) {
          lam = 1.0;
          break;
        }
        launch_scale(n, 1.0 / lam, lv.t.p, lv.z.p, s);
      }
      // level 0 operator == the hierarchy's A_0: also use the setup's 10-step estimate
      lv.lambda_smoother = l == 0 ? std::max(lam, amg_.levels[l].lambda_max_scaled) : lam;
    }
    set_cheb(cheb_ratio);
  }
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
}

// Chebyshev smoother on [lmax/ratio, lmax] of D^-1 A, lmax = 1.1 x the power
// estimate. Degree 2: x += c0 D^-1 r0 + c1 D^-1 (r0 - A D^-1 r0 / theta);
// degree 1: x += D^-1 r0 / theta.
void GpuSystem::set_cheb(double ratio) {
  invalidate_graphs();  // coefficients are baked into the captured kernel parameters
  cheb_ratio = ratio;
  for (auto& lv : levels_) {
    const double lmax = 1.1 * lv.lambda_smoother, lmin = lmax / ratio;
    const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
    const double sigma = theta / delta, rho0 = 1.0 / sigma, rho1 = 1.0 / (2.0 * sigma - rho0);
    lv.cheb.c0 = (1.0 + rho1 * rho0) / theta;
    lv.cheb.c1 = 2.0 * rho1 / delta;
    lv.cheb.inv_theta = 1.0 / theta;
    lv.cheb1 = ChebCoef{0.0, 0.0, 1.0 / theta};
  }
}

void GpuSystem::invalidate_graphs() {
  if (vcycle_graph_) cudaGraphExecDestroy(vcycle_graph_);
  vcycle_graph_ = nullptr;
}

void GpuSystem::set_level_tpr(int level, int tpr) {
  if (tpr < 1 || tpr > 32 || (tpr & (tpr - 1))) throw std::invalid_argument("tpr must be a power of two <= 32");
  invalidate_graphs();
  if (level == 0) mii_.tpr = tpr;
  if (level < (int)levels_.size()) levels_[level].A.tpr = tpr;
}

void GpuSystem::set_vcycle_fp32(bool on) {
  invalidate_graphs();
  vcycle_fp32_ = on;
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    DevLevel& lv = levels_[l];
    lv.A.values_f = on ? lv.a_vf.p : nullptr;
    lv.P.values_f = on ? lv.p_vf.p : nullptr;
    lv.R.values_f = on ? lv.r_vf.p : nullptr;
  }
}

const std::vector<int>& GpuSystem::colors() {
  if (n_colors_ < 0) colors_ = color_elements(prob_.dm, n_tets_, &n_colors_);
  return colors_;
}
int GpuSystem::n_colors() {
  colors();
  return n_colors_;
}

// ------------------------------------------------------------------ helpers
void GpuSystem::sync() { CK(cudaStreamSynchronize(stream_)); }

double GpuSystem::read_scalar(int slot) {
  CK(cudaMemcpyAsync(pinned_, red_scal_.p + slot, sizeof(double), cudaMemcpyDeviceToHost, stream_));
  sync();
  return pinned_[0];
}
void GpuSystem::read_scalars(int first, int count, double* out) {
  CK(cudaMemcpyAsync(pinned_, red_scal_.p + first, sizeof(double) * count, cudaMemcpyDeviceToHost, stream_));
  sync();
  std::memcpy(out, pinned_, sizeof(double) * count);
}

void GpuSystem::check_kernel_flags() {
  int flags = 0;
  CK(cudaMemcpyAsync(&pinned_[S_COUNT], err_.p, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  sync();
  std::memcpy(&flags, &pinned_[S_COUNT], sizeof(int));
  CK(cudaGetLastError());
  if (flags) {
    CK(cudaMemsetAsync(err_.p, 0, sizeof(int), stream_));
    if (flags & 1) throw GeometryError("degenerate tetrahedron in element kernel");
    if (flags & 2) throw std::invalid_argument("kappa_of_e: negative field magnitude");
  }
}

std::vector<double> GpuSystem::set_values(double t, bool rates) const {
  std::vector<double> v(kMaxSets, 0.0);
  for (int s = 0; s < n_sets_; ++s)
    v[s] = rates ? prob_.set_waveforms[s].rate_at(t) : prob_.set_waveforms[s].value_at(t);
  return v;
}

cudaEvent_t GpuSystem::get_event() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}
void GpuSystem::tic(int cls) {
  if (!timing_on) return;
  if (open_cls_ >= 0) {  // nested region: attributed to the outer one
    ++nest_;
    return;
  }
  open_cls_ = cls;
  open_ev_ = get_event();
  CK(cudaEventRecord(open_ev_, stream_));
}
void GpuSystem::toc(int cls, double bytes) {
  if (!timing_on || open_cls_ < 0) return;
  if (nest_ > 0) {
    --nest_;
    return;
  }
  (void)cls;
  cudaEvent_t b = get_event();
  CK(cudaEventRecord(b, stream_));
  events_.push_back({open_ev_, b, cls, bytes});
  open_cls_ = -1;
  if (events_.size() > 4096) {
    double ms[TC_COUNT];
    long n[TC_COUNT];
    double by[TC_COUNT];
    timing_resolve(ms, n, by);
  }
}
void GpuSystem::timing_resolve(double ms[TC_COUNT], long launches[TC_COUNT], double bytes[TC_COUNT]) {
  sync();
  for (auto& e : events_) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e.a, e.b));
    acc_ms_[e.cls] += t;
    acc_n_[e.cls] += 1;
    acc_bytes_[e.cls] += e.bytes;
    ev_pool_.push_back(e.a);
    ev_pool_.push_back(e.b);
  }
  events_.clear();
  for (int c = 0; c < TC_COUNT; ++c) {
    ms[c] = acc_ms_[c];
    launches[c] = acc_n_[c];
    bytes[c] = acc_bytes_[c];
  }
}
void GpuSystem::timing_reset() {
  double ms[TC_COUNT];
  long n[TC_COUNT];
  double by[TC_COUNT];
  timing_resolve(ms, n, by);
  for (int c = 0; c < TC_COUNT; ++c) acc_ms_[c] = acc_bytes_[c] = 0, acc_n_[c] = 0;
}

// K(x)v P1 = 20 n_tets + 48 n_dofs (x, v gathered, coords 24 B,
// y written); P2 = 44 n_tets + 24 n_nodes + 24 n_dofs.
double GpuSystem::kx_bytes() const {
  if (order_ == 1) return 20.0 * n_tets_ + 48.0 * n_dofs_;
  return 44.0 * n_tets_ + 24.0 * prob_.mesh.n_nodes + 24.0 * n_dofs_;
}
double GpuSystem::spmv_bytes(const DevCsr& a) const {
  return 12.0 * a.nnz + 4.0 * (a.n_rows + 1) + 8.0 * a.n_cols + 8.0 * a.n_rows;
}

// ------------------------------------------------------------------ operators
void GpuSystem::lift_dev(double t, double* x_full) {
  const std::vector<double> v = set_values(t, false);
  SetVals sv;
  std::copy(v.begin(), v.end(), sv.v);
  launch_lift_fixed(n_fixed_, set_of_fixed_.p, sv, x_full + n_free_, stream_);
}

void GpuSystem::kx_tets(const double* x, const double* v) {
  launch_kx_tets(order_, n_tets_, tet_dofs_.p, tet_mat_.p, coords_.p, x, v, ytet_.p, err_.p, stream_);
  ++stats_.applies;
}

// coloured single-pass scatter (matfree.cpp:100-117): y (n_dofs) = K(x) v
static void colored_apply(GpuSystem& g, int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat,
                          const double* coords, const double* x, const double* v, double* y, int* err, int n_dofs,
                          const int* color_tets, const std::vector<long>& off, cudaStream_t s) {
  (void)g;
  (void)n_tets;
  launch_fill(n_dofs, 0.0, y, s);
  for (size_t c = 0; c + 1 < off.size(); ++c)
    launch_kx_colored(order, (int)(off[c + 1] - off[c]), color_tets + off[c], tet_dofs, tet_mat, coords, x, v, y, err,
                      s);
}

void GpuSystem::kx_apply_full_dev(const double* x_state, const double* v, double* y) {
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    if (color_off_.empty()) {
      const std::vector<int>& col = colors();
      std::vector<long> off(n_colors_ + 1, 0);
      for (int c : col) ++off[c + 1];
      for (int c = 0; c < n_colors_; ++c) off[c + 1] += off[c];
      std::vector<int> order_t(n_tets_);
      std::vector<long> nx(off.begin(), off.end() - 1);
      for (int t = 0; t < n_tets_; ++t) order_t[nx[col[t]]++] = t;
      color_tets_.alloc(order_t.size());
      color_tets_.upload(order_t.data(), order_t.size(), stream_);
      color_off_ = off;
    }
    colored_apply(*this, order_, n_tets_, tet_dofs_.p, tet_mat_.p, coords_.p, x_state, v, y, err_.p, n_dofs_,
                  color_tets_.p, color_off_, stream_);
    ++stats_.applies;
  } else {
    kx_tets(x_state, v);
    launch_kx_gather(n_dofs_, slot_ptr_.p, slots_.p, ytet_.p, nullptr, 1.0, y, stream_);
  }
  toc(TC_STIFF, kx_bytes());
}

// eval_residual core (fem_system.cpp:62-67 + matfree.cpp:138-143):
// r = -M_IB xdot_B(t) - (K(x) x)|free with x lifted at t.
void GpuSystem::residual_dev(double t, double* x_full, double* r) {
  lift_dev(t, x_full);
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    kx_apply_full_dev(x_full, x_full, w_full_a_.p);
    launch_scale(n_free_, -1.0, w_full_a_.p, r, stream_);
  } else {
    kx_tets(x_full, x_full);
    launch_kx_gather(n_free_, slot_ptr_.p, slots_.p, ytet_.p, nullptr, -1.0, r, stream_);
  }
  toc(TC_STIFF, kx_bytes() - 8.0 * n_fixed_);
  const std::vector<double> rt = set_values(t, true);
  SetVals sv;
  std::copy(rt.begin(), rt.end(), sv.v);
  launch_boundary_load(n_bl_rows_, bl_rows_.p, bl_coef_.p, n_sets_, sv, r, stream_);
  check_kernel_flags();
}

void GpuSystem::mass_apply_dev(const double* v, double* y) { launch_spmv(mii_, v, y, stream_); }

// Symmetric V-cycle (amg.cpp:145-172 structure) with Chebyshev smoothing:
// degree `cheb_degree` on the fine level, `coarse_degree` below; the same
// polynomial pre and post keeps the preconditioner symmetric for PCG.
double* GpuSystem::vcycle(int l, const double* b, bool dot_into_rz) {
  const int L = (int)levels_.size();
  DevLevel& lv = levels_[l];
  if (l == L - 1) {
    launch_dense_solve(coarse_n_, coarse_inv_.p, b, lv.z.p, stream_);
    if (dot_into_rz) launch_dot(coarse_n_, b, lv.z.p, red_, S_RZ, stream_);
    return lv.z.p;
  }
  DevLevel& nx = levels_[l + 1];
  const int deg = l == 0 ? cheb_degree : coarse_degree;
  double* z = lv.z.p;
  if (deg >= 2) {
    launch_cheb_pre(lv.A, lv.invd.p, b, z, lv.cheb, stream_);
    launch_residual(lv.A, b, z, lv.t.p, nullptr, 0, stream_);
  } else if (lv.A.tpr <= 4) {
    launch_cheb1_pre_resid(lv.A, lv.invd.p, b, z, lv.t.p, lv.cheb1, stream_);
  } else {
    // dense rows: one gathered vector per entry instead of two (b and D^-1)
    launch_diag_scale(lv.A.n_rows, lv.invd.p, b, lv.cheb1.inv_theta, z, stream_);
    launch_residual(lv.A, b, z, lv.t.p, nullptr, 0, stream_);
  }
  launch_spmv(lv.R, lv.t.p, nx.b.p, stream_);
  const double* zc = vcycle(l + 1, nx.b.p, false);
  launch_prolong_add(lv.P, zc, z, stream_);
  if (deg >= 2) {
    launch_residual(lv.A, b, z, lv.t.p, nullptr, 0, stream_);
    Reducer r = red_;
    launch_cheb_post2(lv.A, lv.invd.p, lv.t.p, z, lv.cheb, dot_into_rz ? b : nullptr, dot_into_rz ? &r : nullptr,
                      S_RZ, stream_);
    return z;
  }
  launch_cheb1_post(lv.A, lv.invd.p, b, z, lv.z2.p, lv.cheb1, stream_);
  if (dot_into_rz) launch_dot(lv.A.n_rows, b, lv.z2.p, red_, S_RZ, stream_);
  return lv.z2.p;
}

// The V-cycle is a fixed sequence of ~4 kernels per level on fixed buffers,
// so it is captured once into a CUDA graph and replayed: one launch per
// preconditioner application instead of ~30, no host gaps between the short
// coarse-level kernels.
double* GpuSystem::precondition(const double* r) {
  tic(TC_VCYCLE);
  double* z;
  if (prob_.solver.precond == 2) {
    if (use_graphs && r == w_r_.p) {
      if (!vcycle_graph_) {
        cudaGraph_t graph;
        const long before = g_launch_count;
        CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        vcycle_out_ = vcycle(0, r, true);
        CK(cudaStreamEndCapture(stream_, &graph));
        vcycle_graph_kernels_ = g_launch_count - before;
        g_launch_count = before;
        CK(cudaGraphInstantiate(&vcycle_graph_, graph, 0));
        CK(cudaGraphDestroy(graph));
      }
      CK(cudaGraphLaunch(vcycle_graph_, stream_));
      g_launch_count += vcycle_graph_kernels_;
      z = vcycle_out_;
    } else {
      z = vcycle(0, r, true);
    }
  } else {
    Reducer rr = red_;
    z = w_z_.p;
    launch_jacobi(n_free_, mii_invd_.p, r, z, &rr, S_RZ, stream_);
  }
  toc(TC_VCYCLE, 0.0);
  return z;
}

// pcg_solve (proj/src/pcg.cpp:9-72) with device vectors; host reads three
// scalars per iteration for the stopping rule and the breakdown checks.
PcgResult GpuSystem::pcg_dev(const double* b, const double* x0, double* x, double tol, int max_iter) {
  const int n = n_free_;
  PcgResult res;
  launch_dot(n, b, b, red_, S_BB, stream_);
  const double bnorm = std::sqrt(read_scalar(S_BB));
  if (bnorm == 0.0) {
    launch_fill(n, 0.0, x, stream_);
    res.converged = true;
    return res;
  }
  bool use_x0 = false;
  if (x0) {
    launch_dot(n, x0, x0, red_, S_X0X0, stream_);
    use_x0 = read_scalar(S_X0X0) != 0.0;
  }
  double* r = w_r_.p;
  double* z = nullptr;
  double* p = w_p_.p;
  double* q = w_q_.p;
  double rr;
  tic(TC_PCG);
  if (use_x0) {
    if (x0 != x) CK(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    Reducer rd = red_;
    launch_residual(mii_, b, x, r, &rd, S_RR, stream_);
    toc(TC_PCG, spmv_bytes(mii_) + 16.0 * n);
    rr = read_scalar(S_RR);
  } else {
    launch_fill(n, 0.0, x, stream_);
    CK(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    toc(TC_PCG, 24.0 * n);
    rr = bnorm * bnorm;
  }
  double rel = std::sqrt(rr) / bnorm;
  res.initial_rel_residual = rel;
  res.rel_residual = rel;
  if (!std::isfinite(rel)) throw NumericalError("pcg: non-finite initial residual");
  if (rel <= tol) {
    res.converged = true;
    return res;
  }
  z = precondition(r);
  double sc[3];
  read_scalars(S_RZ, 1, sc);
  if (!std::isfinite(sc[0])) throw NumericalError("pcg: non-finite preconditioned residual");
  CK(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));  // p = z
  for (int k = 1; k <= max_iter; ++k) {
    tic(TC_PCG);
    launch_spmv_dot(mii_, p, q, red_, S_PQ, stream_);
    launch_pcg_update(n, x, r, p, q, red_, stream_);
    toc(TC_PCG, spmv_bytes(mii_) + 8.0 * n + 48.0 * n);
    read_scalars(S_PQ, 3, sc);  // pq, rr, rz
    const double pq = sc[0];
    if (!std::isfinite(sc[2])) throw NumericalError("pcg: non-finite preconditioned residual");
    if (!(pq > 0.0) || !std::isfinite(pq))
      throw NumericalError("pcg: operator not positive definite (p'Ap = " + std::to_string(pq) + ")");
    rel = std::sqrt(sc[1]) / bnorm;
    res.iterations = k;
    res.rel_residual = rel;
    if (!std::isfinite(rel)) throw NumericalError("pcg: non-finite residual");
    if (rel <= tol) {
      res.converged = true;
      return res;
    }
    CK(cudaMemcpyAsync(red_scal_.p + S_RZ_OLD, red_scal_.p + S_RZ, sizeof(double), cudaMemcpyDeviceToDevice,
                       stream_));
    z = precondition(r);
    tic(TC_PCG);
    launch_pcg_direction(n, p, z, red_scal_.p, stream_);
    toc(TC_PCG, 24.0 * n);
  }
  read_scalars(S_RZ, 1, sc);
  if (!std::isfinite(sc[0])) throw NumericalError("pcg: non-finite preconditioned residual");
  return res;
}

// ------------------------------------------------------------------ estimator
// StartVectorEstimator::next (proj/src/start_vector.cpp:84-109); writes the
// start vector into x0 and returns true when it is non-zero-by-construction.
// SPE (proj/src/start_vector.cpp:33-62,84-109,152-164). The reference
// re-orthonormalises its whole window with MGS on every solve and applies
// M to every basis vector (2 sum_k (dot + axpy) + m SpMVs per solve). The
// Galerkin start vector x0 = V (V'MV)^-1 V'b only depends on span(V), so the
// device keeps an orthonormal basis Q of the window, W = M Q, G = Q'MQ and R
// with H = Q R across solves: the new solution is appended by two classical
// Gram-Schmidt passes with the reference's drop test (against the same span
// the reference's MGS would test it against), the oldest is removed by a
// Givens downdate of R and a rotation of Q and W. Windows containing a dropped
// or zero vector (where the reference's drop decisions can change when the
// window slides) fall back to the reference's full MGS rebuild.
double* GpuSystem::spe_q(int set, int j) { return spe_q_[set][j]->p; }
double* GpuSystem::spe_w(int set, int j) { return spe_w_[set][j]->p; }

void GpuSystem::spe_alloc(int window) {
  if ((int)spe_q_[0].size() >= window) return;
  for (int s = 0; s < 2; ++s)
    while ((int)spe_q_[s].size() < window) {
      spe_q_[s].push_back(std::make_unique<DevBuf<double>>());
      spe_q_[s].back()->alloc(std::max(1, n_free_));
      spe_w_[s].push_back(std::make_unique<DevBuf<double>>());
      spe_w_[s].back()->alloc(std::max(1, n_free_));
    }
}

// G row/column k (G_ik = q_i' W_k) for the basis vectors 0..k of the current set
void GpuSystem::spe_g_column(int k) {
  std::vector<const double*> Q(k + 1);
  for (int i = 0; i <= k; ++i) Q[i] = spe_q(spe_set_, i);
  launch_multi_dot(n_free_, k + 1, Q.data(), spe_w(spe_set_, k), red_, S_MDOT, stream_);
  double g[kMaxMulti];
  read_scalars(S_MDOT, k + 1, g);
  spe_G_.resize((size_t)kMaxMulti * kMaxMulti);
  for (int i = 0; i <= k; ++i) spe_G_[(size_t)i * kMaxMulti + k] = spe_G_[(size_t)k * kMaxMulti + i] = g[i];
}

// mgs_orthonormalize (start_vector.cpp:10-28) over the whole history, reference order
void GpuSystem::spe_rebuild() {
  const int n = n_free_;
  const double drop = prob_.solver.mgs_drop_tol;
  spe_alloc((int)history_.size());
  spe_k_ = 0;
  bool all_kept = true;
  for (double* cand : history_) {
    launch_dot(n, cand, cand, red_, S_NORM, stream_);
    const double norm0 = std::sqrt(read_scalar(S_NORM));
    if (norm0 == 0.0) {
      all_kept = false;
      continue;
    }
    const int m = spe_k_;
    double* w = spe_q(spe_set_, m);
    CK(cudaMemcpyAsync(w, cand, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    std::vector<double> rc(m + 1, 0.0);
    bool keep = true;
    for (int pass = 0; pass < 2 && keep; ++pass) {
      for (int u = 0; u < m; ++u) {  // modified Gram-Schmidt, sequential projections
        launch_dot(n, spe_q(spe_set_, u), w, red_, S_DOT, stream_);
        launch_axpy_dev(n, red_scal_.p + S_DOT, -1.0, spe_q(spe_set_, u), w, stream_);
      }
      launch_dot(n, w, w, red_, S_NORM, stream_);
      const double nrm = std::sqrt(read_scalar(S_NORM));
      if (nrm <= drop * norm0) keep = false;
      else if (pass == 1) {
        launch_scale(n, 1.0 / nrm, w, w, stream_);
        rc[m] = nrm;
      }
    }
    if (!keep) {
      all_kept = false;
      continue;
    }
    launch_spmv(mii_, w, spe_w(spe_set_, m), stream_);
    ++spe_k_;
    spe_g_column(m);
  }
  spe_clean_ = all_kept && (int)history_.size() <= kMaxWin - 1;
  if (spe_clean_) {  // R = Q' H (H = Q R exactly in this state)
    const int k = spe_k_;
    spe_R_.assign((size_t)kMaxWin * kMaxWin, 0.0);
    std::vector<const double*> Q(k);
    for (int i = 0; i < k; ++i) Q[i] = spe_q(spe_set_, i);
    int j = 0;
    for (double* h : history_) {
      launch_multi_dot(n, k, Q.data(), h, red_, S_MDOT, stream_);
      double col[kMaxMulti];
      read_scalars(S_MDOT, k, col);
      for (int i = 0; i <= j; ++i) spe_R_[(size_t)i * kMaxWin + j] = col[i];
      ++j;
    }
  }
}

// append h (newest) with two classical Gram-Schmidt passes and the MGS drop test
void GpuSystem::spe_append(const double* h) {
  const int n = n_free_;
  const double drop = prob_.solver.mgs_drop_tol;
  const int m = spe_k_;
  launch_dot(n, h, h, red_, S_NORM, stream_);
  const double norm0 = std::sqrt(read_scalar(S_NORM));
  if (norm0 == 0.0) {
    spe_clean_ = false;
    return;
  }
  double* w = spe_q(spe_set_, m);
  CK(cudaMemcpyAsync(w, h, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
  std::vector<const double*> Q(m);
  for (int i = 0; i < m; ++i) Q[i] = spe_q(spe_set_, i);
  std::vector<double> r(m + 1, 0.0);
  double nrm = norm0;
  for (int pass = 0; pass < 2; ++pass) {
    if (m > 0) {
      launch_multi_dot(n, m, Q.data(), w, red_, S_MDOT, stream_);
      double c[kMaxMulti];
      read_scalars(S_MDOT, m, c);
      CoefPack cp{};
      for (int i = 0; i < m; ++i) {
        cp.c[i] = c[i];
        r[i] += c[i];
      }
      launch_orth_update(n, m, Q.data(), cp, w, red_, S_NORM, stream_);
      nrm = std::sqrt(read_scalar(S_NORM));
    }
    if (nrm <= drop * norm0) {
      spe_clean_ = false;
      return;
    }
  }
  launch_scale(n, 1.0 / nrm, w, w, stream_);
  r[m] = nrm;
  for (int i = 0; i <= m; ++i) spe_R_[(size_t)i * kMaxWin + m] = r[i];
  launch_spmv(mii_, w, spe_w(spe_set_, m), stream_);
  spe_k_ = m + 1;
  spe_g_column(m);
}

// remove the oldest window vector: Givens downdate of R[:,1:], rotate Q and W
void GpuSystem::spe_downdate() {
  const int k = spe_k_;
  if (k <= 1) {
    spe_k_ = 0;
    return;
  }
  // Hessenberg Rh = R[:, 1:k] (k x (k-1)); J accumulates the rotations (k x k)
  double Rh[kMaxWin][kMaxWin] = {}, J[kMaxWin][kMaxWin] = {};
  for (int i = 0; i < k; ++i)
    for (int j = 0; j + 1 < k; ++j) Rh[i][j] = spe_R_[(size_t)i * kMaxWin + j + 1];
  for (int i = 0; i < k; ++i) J[i][i] = 1.0;
  for (int i = 0; i + 1 < k; ++i) {
    const double a = Rh[i][i], b = Rh[i + 1][i];
    const double rr = std::hypot(a, b);
    const double c = rr == 0.0 ? 1.0 : a / rr, s = rr == 0.0 ? 0.0 : b / rr;
    for (int j = 0; j + 1 < k; ++j) {
      const double u = Rh[i][j], v = Rh[i + 1][j];
      Rh[i][j] = c * u + s * v;
      Rh[i + 1][j] = -s * u + c * v;
    }
    for (int j = 0; j < k; ++j) {
      const double u = J[i][j], v = J[i + 1][j];
      J[i][j] = c * u + s * v;
      J[i + 1][j] = -s * u + c * v;
    }
  }
  // Q' = Q J^T (first k-1 columns); T[a][b] = J[b][a]
  RotPack T{};
  for (int a = 0; a < k; ++a)
    for (int b = 0; b + 1 < k; ++b) T.t[a][b] = J[b][a];
  std::vector<const double*> qi(k), wi(k);
  std::vector<double*> qo(k - 1), wo(k - 1);
  for (int i = 0; i < k; ++i) {
    qi[i] = spe_q(spe_set_, i);
    wi[i] = spe_w(spe_set_, i);
  }
  for (int j = 0; j + 1 < k; ++j) {
    qo[j] = spe_q(1 - spe_set_, j);
    wo[j] = spe_w(1 - spe_set_, j);
  }
  launch_lincomb_multi(n_free_, k, k - 1, qi.data(), qo.data(), T, stream_);
  launch_lincomb_multi(n_free_, k, k - 1, wi.data(), wo.data(), T, stream_);
  // G' = T' G T, R' = rows 0..k-2 of the rotated Rh
  std::vector<double> G2((size_t)kMaxMulti * kMaxMulti, 0.0);
  for (int a = 0; a + 1 < k; ++a)
    for (int b = 0; b + 1 < k; ++b) {
      double s = 0.0;
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) s += T.t[i][a] * spe_G_[(size_t)i * kMaxMulti + j] * T.t[j][b];
      G2[(size_t)a * kMaxMulti + b] = s;
    }
  spe_G_ = G2;
  spe_R_.assign((size_t)kMaxWin * kMaxWin, 0.0);
  for (int i = 0; i + 1 < k; ++i)
    for (int j = i; j + 1 < k; ++j) spe_R_[(size_t)i * kMaxWin + j] = Rh[i][j];
  spe_set_ = 1 - spe_set_;
  spe_k_ = k - 1;
}

// StartVectorEstimator::next (proj/src/start_vector.cpp:84-109); writes the
// start vector into x0 and returns true when it is non-zero-by-construction.
bool GpuSystem::estimator_next(const double* b, double* x0) {
  const int n = n_free_;
  const int mode = prob_.solver.estimator_mode;
  if (mode == 0) return false;
  if (history_.empty()) return false;
  if (mode == 1) {
    CK(cudaMemcpyAsync(x0, history_.back(), sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    return true;
  }
  tic(TC_SPE);
  if (!spe_clean_ || !spe_incremental) spe_rebuild();
  const int m = spe_k_;
  estimator_rank_ = m;
  if (m == 0) {
    toc(TC_SPE, 0.0);
    return false;
  }
  // spe_start (start_vector.cpp:33-62): x0 = V (V'MV)^-1 V' b with the pivoted LDLT of G
  std::vector<double> g((size_t)m * m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) g[(size_t)i * m + j] = spe_G_[(size_t)i * kMaxMulti + j];
  DenseLdlt ldlt;
  ldlt.compute(g, m);
  double dmax = 0.0, dmin = INFINITY;
  for (double d : ldlt.d) {
    dmax = std::max(dmax, std::abs(d));
    dmin = std::min(dmin, d);
  }
  const bool ok = ldlt.ok && dmax > 0.0 && dmin > 1e-14 * dmax;
  if (!ok) {
    ++stats_.spe_fallbacks;
    std::fprintf(stderr, "start_vector: singular reduced system, zero start used\n");
    toc(TC_SPE, 0.0);
    return false;
  }
  std::vector<double> ginv((size_t)m * m), e(m), col(m);
  for (int c = 0; c < m; ++c) {
    std::fill(e.begin(), e.end(), 0.0);
    e[c] = 1.0;
    ldlt.solve(e.data(), col.data());
    for (int r = 0; r < m; ++r) ginv[(size_t)r * m + c] = col[r];
  }
  std::vector<const double*> V(m);
  for (int c = 0; c < m; ++c) V[c] = spe_q(spe_set_, c);
  launch_multi_dot(n, m, V.data(), b, red_, S_MDOT, stream_);
  double vtb[kMaxMulti];
  read_scalars(S_MDOT, m, vtb);
  CoefPack y{};
  for (int r = 0; r < m; ++r) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) s += ginv[(size_t)r * m + c] * vtb[c];
    y.c[r] = s;
  }
  launch_lincomb(n, m, V.data(), y, x0, stream_);
  toc(TC_SPE, 0.0);
  return true;
}

// StartVectorEstimator::feedback (proj/src/start_vector.cpp:152-164)
void GpuSystem::estimator_feedback(const double* x) {
  const int mode = prob_.solver.estimator_mode;
  if (mode == 0) return;
  const size_t window = mode == 1 ? 1 : (size_t)prob_.solver.spe_window;
  double* buf;
  if (history_.size() >= window) {
    buf = history_.front();
    history_.pop_front();
    if (mode == 2 && spe_clean_ && spe_incremental) spe_downdate();
  } else {
    hist_pool_.push_back(std::make_unique<DevBuf<double>>());
    hist_pool_.back()->alloc(std::max(1, n_free_));
    buf = hist_pool_.back()->p;
  }
  CK(cudaMemcpyAsync(buf, x, sizeof(double) * n_free_, cudaMemcpyDeviceToDevice, stream_));
  history_.push_back(buf);
  if (mode == 2 && spe_clean_ && spe_incremental) {
    if (window > (size_t)(kMaxWin - 1)) {
      spe_clean_ = false;  // large windows always use the full rebuild
    } else {
      tic(TC_SPE);
      spe_alloc((int)window);
      spe_append(buf);
      toc(TC_SPE, 0.0);
    }
  }
}

// FemSystem::eval_rhs (proj/src/fem_system.cpp:69-99)
PcgResult GpuSystem::eval_rhs_dev(double t, double* x_full, double* f) {
  double* b = w_free_a_.p;
  {
    PhaseTimer pt(stats_.t_residual);
    residual_dev(t, x_full, b);
  }
  bool has_x0;
  {
    PhaseTimer pt(stats_.t_estimator);
    has_x0 = estimator_next(b, f);
  }
  PcgResult res;
  {
    PhaseTimer pt(stats_.t_solve);
    res = pcg_dev(b, has_x0 ? f : nullptr, f, prob_.solver.rel_tol, prob_.solver.max_iter);
  }
  if (!res.converged) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "mass solve failed to converge (relative residual %f)", res.rel_residual);
    throw NumericalError(buf);
  }
  {
    PhaseTimer pt(stats_.t_estimator);
    estimator_feedback(f);
  }
  ++stats_.m_solves;
  stats_.pcg_iterations += res.iterations;
  records_.push_back({t, estimator_rank_, res.iterations, res.initial_rel_residual});
  return res;
}

// FemSystem::apply_minv_stiffness (proj/src/fem_system.cpp:103-122)
void GpuSystem::apply_minv_stiffness_dev(double t, double* x_full, const double* v_free, double* y) {
  double* vfull = w_full_b_.p;
  double* kv = w_free_b_.p;
  {
    PhaseTimer pt(stats_.t_residual);
    lift_dev(t, x_full);
    CK(cudaMemcpyAsync(vfull, v_free, sizeof(double) * n_free_, cudaMemcpyDeviceToDevice, stream_));
    launch_fill(n_fixed_, 0.0, vfull + n_free_, stream_);
    tic(TC_STIFF);
    if (stiffness_mode == 1) {
      kx_apply_full_dev(x_full, vfull, w_full_a_.p);
      CK(cudaMemcpyAsync(kv, w_full_a_.p, sizeof(double) * n_free_, cudaMemcpyDeviceToDevice, stream_));
    } else {
      kx_tets(x_full, vfull);
      launch_kx_gather(n_free_, slot_ptr_.p, slots_.p, ytet_.p, nullptr, 1.0, kv, stream_);
    }
    toc(TC_STIFF, kx_bytes());
    check_kernel_flags();
  }
  PhaseTimer pt(stats_.t_solve);
  PcgResult res = pcg_dev(kv, nullptr, y, prob_.solver.rho_solve_tol, prob_.solver.max_iter);
  ++stats_.rho_solves;
  stats_.rho_pcg_iterations += res.iterations;
}

// estimate_spectral_radius (proj/src/integrators.cpp:49-75)
double GpuSystem::estimate_spectral_radius(double t, double* x_full) {
  const int n = n_free_;
  for (int restart = 0; restart < 4; ++restart) {
    std::mt19937 rng(7919u + 31u * (unsigned)restart);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::vector<double> v(n);
    for (int i = 0; i < n; ++i) v[i] = uni(rng);
    double nrm = 0.0;
    for (double e : v) nrm += e * e;
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    for (double& e : v) e /= nrm;
    rho_v_.upload(v.data(), n, stream_);
    double rho = 0.0;
    bool annihilated = false;
    for (int it = 0; it < 15; ++it) {
      apply_minv_stiffness_dev(t, x_full, rho_v_.p, rho_w_.p);
      launch_dot(n, rho_w_.p, rho_w_.p, red_, S_NORM, stream_);
      rho = std::sqrt(read_scalar(S_NORM));
      if (rho == 0.0) {
        annihilated = true;
        break;
      }
      launch_scale(n, 1.0 / rho, rho_w_.p, rho_v_.p, stream_);
    }
    if (!annihilated) return 1.2 * rho;
  }
  return 0.0;
}

// ------------------------------------------------------------------ host wrappers
void GpuSystem::kx_apply_host(const double* x_state, const double* v, double* y) {
  std::vector<double> xd(n_dofs_), vd(n_dofs_), yd(n_dofs_);
  for (int k = 0; k < n_dofs_; ++k) {
    xd[k] = x_state[dev2ref_[k]];
    vd[k] = v[dev2ref_[k]];
  }
  w_full_a_.upload(xd.data(), n_dofs_, stream_);
  w_full_b_.upload(vd.data(), n_dofs_, stream_);
  double* out = scratch_full();
  kx_apply_full_dev(w_full_a_.p, w_full_b_.p, out);
  CK(cudaMemcpyAsync(yd.data(), out, sizeof(double) * n_dofs_, cudaMemcpyDeviceToHost, stream_));
  check_kernel_flags();
  for (int k = 0; k < n_dofs_; ++k) y[dev2ref_[k]] = yd[k];
}

// MatFreeStiffness::residual (matfree.cpp:138-143)
void GpuSystem::kx_residual_host(const double* x_full, const double* b_mass, double* r) {
  std::vector<double> xd(n_dofs_), yd(n_dofs_);
  for (int k = 0; k < n_dofs_; ++k) xd[k] = x_full[dev2ref_[k]];
  w_full_a_.upload(xd.data(), n_dofs_, stream_);
  w_free_a_.upload(b_mass, n_free_, stream_);
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    kx_apply_full_dev(w_full_a_.p, w_full_a_.p, w_full_b_.p);
    launch_axpby_into(n_free_, w_free_a_.p, -1.0, w_full_b_.p, w_free_b_.p, stream_);
  } else {
    kx_tets(w_full_a_.p, w_full_a_.p);
    launch_kx_gather(n_free_, slot_ptr_.p, slots_.p, ytet_.p, w_free_a_.p, -1.0, w_free_b_.p, stream_);
  }
  toc(TC_STIFF, kx_bytes());
  w_free_b_.download(r, n_free_, stream_);
  check_kernel_flags();
}

void GpuSystem::eval_residual_host(double t, const double* x, double* r) {
  PhaseTimer pt(stats_.t_residual);
  double* xf = w_full_b_.p;
  CK(cudaMemcpyAsync(xf, x, sizeof(double) * n_free_, cudaMemcpyHostToDevice, stream_));
  residual_dev(t, xf, w_free_b_.p);
  w_free_b_.download(r, n_free_, stream_);
  sync();
}

PcgResult GpuSystem::eval_rhs_host(double t, const double* x, double* f) {
  double* xf = w_full_b_.p;
  CK(cudaMemcpyAsync(xf, x, sizeof(double) * n_free_, cudaMemcpyHostToDevice, stream_));
  PcgResult r = eval_rhs_dev(t, xf, F_.p);
  F_.download(f, n_free_, stream_);
  sync();
  return r;
}

PcgResult GpuSystem::mass_solve_host(const double* b, const double* x0, double tol, int max_iter, double* x) {
  F0_.upload(b, n_free_, stream_);
  if (x0) Fn_.upload(x0, n_free_, stream_);
  PhaseTimer pt(stats_.t_solve);
  PcgResult r = pcg_dev(F0_.p, x0 ? Fn_.p : nullptr, F_.p, tol, max_iter);
  F_.download(x, n_free_, stream_);
  sync();
  return r;
}

void GpuSystem::mass_apply_host(const double* v, double* y) {
  F0_.upload(v, n_free_, stream_);
  mass_apply_dev(F0_.p, F_.p);
  F_.download(y, n_free_, stream_);
  sync();
}

void GpuSystem::apply_minv_stiffness_host(double t, const double* x_state, const double* v, double* y) {
  double* xf = scratch_full();
  CK(cudaMemcpyAsync(xf, x_state, sizeof(double) * n_free_, cudaMemcpyHostToDevice, stream_));
  F0_.upload(v, n_free_, stream_);
  apply_minv_stiffness_dev(t, xf, F0_.p, F_.p);
  F_.download(y, n_free_, stream_);
  sync();
}

void GpuSystem::lift_full_host(double t, const double* x_free, double* x_full) {
  std::vector<double> b = set_values(t, false);
  for (int i = 0; i < n_free_; ++i) x_full[prob_.dm.free_dofs[i]] = x_free[i];
  for (int i = 0; i < n_fixed_; ++i) x_full[prob_.dm.fixed_dofs[i]] = b[prob_.dm.fixed_set[prob_.dm.fixed_dofs[i]]];
}

// ------------------------------------------------------------------ integrators
void GpuSystem::set_state(double t, const double* x_host, double dt) {
  state_t = t;
  state_dt = dt;
  CK(cudaMemcpyAsync(X_, x_host, sizeof(double) * n_free_, cudaMemcpyHostToDevice, stream_));
  sync();
  rho_valid = false;
  rho_age = 0;
}
void GpuSystem::get_state(double* x_host) {
  CK(cudaMemcpyAsync(x_host, X_, sizeof(double) * n_free_, cudaMemcpyDeviceToHost, stream_));
  sync();
}

double GpuSystem::spectral_radius_cached(int refresh_every) {  // integrators.cpp:77-84
  if (!rho_valid || rho_age >= refresh_every) {
    rho_value = estimate_spectral_radius(state_t, X_);
    rho_age = 0;
    rho_valid = true;
  }
  return rho_value;
}

namespace {
const RkcCoefficients& rkc_coefficients(int s) {  // integrators.cpp:148-153
  static std::map<int, RkcCoefficients> cache;
  auto it = cache.find(s);
  if (it == cache.end()) it = cache.emplace(s, RkcCoefficients::compute(s)).first;
  return it->second;
}
}  // namespace

// rkc_stages (proj/src/integrators.cpp:156-173). Returns the buffer holding Y_s.
static double* rkc_stages(GpuSystem& g, double t, double dt, const RkcCoefficients& k, double* X, double* bufs[3],
                          double* f0, double* f) {
  const int n = g.n_free();
  g.eval_rhs_dev(t, X, f0);
  double* jm2 = X;
  double* jm1 = bufs[0];
  g.tic(TC_RKC);
  launch_axpby_into(n, X, k.mu1_tilde * dt, f0, jm1, g.stream());
  g.toc(TC_RKC, 24.0 * n);
  for (int j = 2; j <= k.s; ++j) {
    g.eval_rhs_dev(t + k.c[j - 1] * dt, jm1, f);
    double* target = nullptr;
    for (int b = 0; b < 3; ++b)
      if (bufs[b] != jm1 && bufs[b] != jm2) {
        target = bufs[b];
        break;
      }
    g.tic(TC_RKC);
    launch_rkc_stage(n, 1.0 - k.mu[j] - k.nu[j], k.mu[j], k.nu[j], k.mu_tilde[j] * dt, k.gamma_tilde[j] * dt, X, jm1,
                     jm2, f, f0, target, g.stream());
    g.toc(TC_RKC, 48.0 * n);
    jm2 = jm1;
    jm1 = target;
  }
  return jm1;
}

// rkc_step (proj/src/integrators.cpp:177-225)
StepAttempt GpuSystem::rkc_step(const RkcOptions& o) {
  StepAttempt att;
  att.t_start = state_t;
  const double rho = spectral_radius_cached(o.rho_refresh_every);
  att.rho = rho;
  double dt = state_dt;
  int s = 2;
  if (rho > 0.0) {
    s = std::max(2, (int)std::ceil(std::sqrt(dt * rho / 0.653 + 1.0)));
    if (s > o.max_stages) {
      s = o.max_stages;
      dt = 0.95 * RkcCoefficients::stability_boundary(s) / rho;
    }
  }
  att.dt = dt;
  att.stages = s;
  try {
    const RkcCoefficients& k = rkc_coefficients(s);
    double* bufs[3];
    int bi = 0;
    for (auto& b : full_)
      if (b.p != X_) bufs[bi++] = b.p;
    double* x_new = rkc_stages(*this, state_t, dt, k, X_, bufs, F0_.p, F_.p);
    eval_rhs_dev(state_t + dt, x_new, Fn_.p);
    tic(TC_RKC);
    launch_rkc_error(n_free_, X_, x_new, F0_.p, Fn_.p, dt, o.atol, o.rtol, red_, S_ERR, stream_);
    toc(TC_RKC, 32.0 * n_free_);
    const double acc = read_scalar(S_ERR);
    att.error = n_free_ == 0 ? 0.0 : std::sqrt(acc / (double)n_free_);
    // step_controller (integrators.cpp:12-18), order 2
    const double err = att.error;
    bool accept;
    double dt_next;
    if (!std::isfinite(err)) {
      accept = false;
      dt_next = 0.1 * dt;
    } else {
      accept = err <= 1.0;
      const double factor = err == 0.0 ? 10.0 : std::clamp(0.8 * std::pow(err, -1.0 / 3.0), 0.1, 10.0);
      dt_next = dt * factor;
    }
    att.accepted = accept;  // finite err implies finite x_new
    att.dt_next = dt_next;
    st_stages += s;
    if (att.accepted) {
      X_ = x_new;
      state_t += dt;
      ++st_accepted;
      ++rho_age;
    } else {
      ++st_rejected;
      rho_valid = false;
    }
  } catch (const NumericalError&) {
    att.accepted = false;
    att.dt_next = 0.5 * dt;
    ++st_rejected;
    rho_valid = false;
  }
  state_dt = att.dt_next;
  return att;
}

// rkc_advance_fixed (proj/src/integrators.cpp:227-235)
void GpuSystem::rkc_advance_fixed(double dt, int s) {
  const RkcCoefficients& k = rkc_coefficients(s);
  double* bufs[3];
  int bi = 0;
  for (auto& b : full_)
    if (b.p != X_) bufs[bi++] = b.p;
  X_ = rkc_stages(*this, state_t, dt, k, X_, bufs, F0_.p, F_.p);
  state_t += dt;
  ++st_accepted;
  st_stages += s;
}

// euler_step (proj/src/integrators.cpp:33-47)
StepAttempt GpuSystem::euler_step(double dt) {
  StepAttempt att;
  att.t_start = state_t;
  att.dt = dt;
  eval_rhs_dev(state_t + dt, X_, F_.p);
  tic(TC_RKC);
  launch_axpy(n_free_, dt, F_.p, X_, stream_);
  toc(TC_RKC, 24.0 * n_free_);
  state_t += dt;
  ++st_accepted;
  ++st_stages;
  att.accepted = true;
  att.stages = 1;
  att.dt_next = dt;
  return att;
}

}  // namespace eqsb
