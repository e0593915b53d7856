// GpuSystem: device-resident FemSystem + integrator.
//
// Local numbering of the fine dofs on a rank: [owned free | ghost free |
// local fixed]. A "full" vector holds the owned state, room for the ghosts
// that a halo exchange fills, and the Dirichlet values of the fixed dofs used
// by the local tets, so lifting a stage vector (DofMap::lift,
// proj/src/dofmap.cpp:11-15) is a write of the fixed tail and restricting
// (restrict_free, :17-20) is free. With one rank the owned set is every free
// dof in DofMap::free_dofs order and there are no ghosts.
#include "gpu_system.hpp"
#include "amg_device.hpp"
#include "element.hpp"
#include "kxblock.hpp"
#include "sell.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <random>
#include <type_traits>

#include <malloc.h>
#include <nvtx3/nvToolsExt.h>

namespace eqsb {

thread_local std::function<void()> setup_gate_release;

struct GpuSystem::ShiftAmg {
  SpgemmDevice sd;
  std::vector<DCsr> A, P, R;
  std::vector<DevBuf<float>> vals32;  // fp32 copies of the level values (the fp32 V-cycle reads them)
  std::vector<DevLevel> levels;
  int coarse_n = 0;
  DevBuf<double> inv;
  DevBuf<float> inv32;
  int builds = 0;
  // the mass solve's operator / graph state, swapped in while a shifted
  // system is solved through pcg_dev (shift_swap)
  DevCsr op;
  cudaGraphExec_t vgraph = nullptr;
  double* vout = nullptr;
  long vkern = 0;
  double vbytes = 0.0;
  std::unordered_map<double*, cudaGraphExec_t> graphs;
  std::unordered_map<double*, long> graph_use;
  long graph_clock = 0, body_kernels = 0;
  double body_bytes = 0.0;
  void drop_graphs() {
    if (vgraph) cudaGraphExecDestroy(vgraph);
    vgraph = nullptr;
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
    graph_use.clear();
  }
  ~ShiftAmg() { drop_graphs(); }
};

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
template struct DevBuf<float>;
template struct DevBuf<int>;
template struct DevBuf<long>;
template struct DevBuf<unsigned>;
template struct DevBuf<unsigned char>;
template struct DevBuf<unsigned short>;
template struct DevBuf<unsigned long long>;

namespace {
using clk = std::chrono::steady_clock;
// Host wall time of a phase bucket (the reference's metrics.cpp phases:
// residual / estimator / solve / setup) plus an NVTX range of the same name,
// so profilers can attribute kernels to the buckets.
struct PhaseTimer {
  double& slot;
  clk::time_point t0;
  PhaseTimer(double& s, const char* name) : slot(s), t0(clk::now()) { nvtxRangePushA(name); }
  ~PhaseTimer() {
    nvtxRangePop();
    slot += std::chrono::duration<double>(clk::now() - t0).count();
  }
};

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
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
  rp.alloc(std::max<size_t>(1, h.row_ptr.size()));
  ci.alloc(std::max<size_t>(1, h.col_idx.size()));
  v.alloc(std::max<size_t>(1, h.values.size()));
  rp.upload(h.row_ptr.data(), h.row_ptr.size(), s);
  ci.upload(h.col_idx.data(), h.col_idx.size(), s);
  v.upload(h.values.data(), h.values.size(), s);
  d.row_ptr = rp.p;
  d.col_idx = ci.p;
  d.values = v.p;
  d.values_f = nullptr;
  d.tpr = choose_tpr(h);
}

void upload_sell16(const HostCsr& h, const HostSell& hs, DevCsr& d, SellBufs& b, cudaStream_t s) {
  const size_t np = std::max<long>(1, hs.padded());
  // chunk pointers and bases padded past the end: the pipelined kernels copy
  // whole tiles of metadata (10 pointers, 64 bases) with bulk copies
  std::vector<long> cp = hs.chunk_ptr;
  cp.resize(cp.size() + 16, cp.back());
  std::vector<int> bases = hs.bases;
  bases.resize(bases.size() + 64, 0);
  b.cp.alloc(cp.size());
  b.cp.upload(cp.data(), cp.size(), s);
  b.bases.alloc(bases.size());
  b.bases.upload(bases.data(), bases.size(), s);
  b.code.alloc(np);
  b.code.upload(hs.code.data(), hs.code.size(), s);
  {
    const std::vector<double> v = sell_values<double>(hs, h.values);
    b.v64.alloc(np);
    b.v64.upload(v.data(), v.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  {
    const std::vector<float> v = sell_values<float>(hs, h.values);
    b.v32.alloc(np);
    b.v32.upload(v.data(), v.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  {
    std::vector<uint16_t> v(hs.src.size());
#pragma omp parallel for schedule(static)
    for (long k = 0; k < (long)v.size(); ++k) v[k] = hs.src[k] >= 0 ? to_bf16(h.values[hs.src[k]]) : 0;
    b.v16.alloc(np);
    b.v16.upload(v.data(), v.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  d.sell.tpr = hs.tpr;
  d.sell.n_chunks = hs.n_chunks;
  d.sell.padded = hs.padded();
  d.sell.chunk_ptr = b.cp.p;
  d.sell.bases = b.bases.p;
  d.sell.code = b.code.p;
  d.sell.v64 = b.v64.p;
  d.sell.v32 = b.v32.p;
  d.sell.v16 = b.v16.p;
}

// SELL copies of h (sell.hpp): SELL-16 with fp64/fp32/bf16 values and the
// packed bf16 SELL-P; each stays absent when some chunk cannot be encoded.
// sell16_always = false (V-cycle operators): SELL-16 only when the packed
// encoding fails; the non-default fp64/fp32 V-cycles then read CSR.
void upload_sell(const HostCsr& h, DevCsr& d, SellBufs& b, cudaStream_t s, bool sell16_always = true) {
  d.sell = DevSell{};
  d.pk = DevSellP{};
  if (h.n_rows == 0) return;
  // packed bf16 copy for the V-cycle kernels (sell.hpp "SELL-P")
  HostSellP hp;
  const int tpr = choose_sellp_tpr(h);
  bool packed = build_sell_packed(h, tpr, hp);
  // EQS_SELLP_SIGMA=256: rows sorted by length within windows of sigma rows
  // (SELL-C-sigma) when that saves more entry bytes than the permutation
  // costs (4 B per row) and at least 5%. Off by default: at C3 it cuts the
  // V-cycle's bytes by 5.4% (4.76 -> 4.51 GB) without changing its time,
  // the permuted epilogue rows cost what the padding saved
  static const int sigma = getenv("EQS_SELLP_SIGMA") ? atoi(getenv("EQS_SELLP_SIGMA")) : 0;
  if (packed && sigma > 0 && hp.uniform == 0) {
    HostSellP hs;
    if (build_sell_packed(h, tpr, hs, sigma)) {
      const double before = 4.0 * hp.padded(), after = 4.0 * hs.padded() + 4.0 * h.n_rows;
      if (after <= 0.95 * before) hp = std::move(hs);
    }
  }
  if (sell16_always || !packed) {
    HostSell hs;
    if (build_sell(h, choose_sell_tpr(h), hs)) upload_sell16(h, hs, d, b, s);
  }
  if (!packed) return;
  std::vector<int> pcp = hp.chunk_ptr;
  b.pk_cp.alloc(pcp.size());
  b.pk_cp.upload(pcp.data(), pcp.size(), s);
  b.pk_bases.alloc(std::max<size_t>(1, hp.bases.size()));
  b.pk_bases.upload(hp.bases.data(), hp.bases.size(), s);
  b.pk_words.alloc(std::max<size_t>(4, hp.words.size()));
  b.pk_words.upload(hp.words.data(), hp.words.size(), s);
  CK(cudaStreamSynchronize(s));
  d.pk.tpr = hp.tpr;
  d.pk.n_chunks = hp.n_chunks;
  d.pk.shift = hp.shift;
  d.pk.windows = hp.windows;
  d.pk.uniform = hp.uniform;
  d.pk.padded = hp.padded();
  d.pk.chunk_ptr = b.pk_cp.p;
  d.pk.bases = b.pk_bases.p;
  d.pk.words = reinterpret_cast<const uint4*>(b.pk_words.p);
  d.pk.perm = nullptr;
  if (!hp.perm.empty()) {
    b.pk_perm.alloc(hp.perm.size());
    b.pk_perm.upload(hp.perm.data(), hp.perm.size(), s);
    CK(cudaStreamSynchronize(s));
    d.pk.perm = b.pk_perm.p;
  }
}

// stencil-coded bf16 copy (sell.hpp SELL-S) for the fine-level V-cycle
// operator; absent when the rows need too many patterns (unstructured meshes)
void upload_stencil(const HostCsr& h, DevCsr& d, SellBufs& b, cudaStream_t s) {
  d.st = DevSellS{};
  HostSellS hs;
  // SELL-SH (symmetric half storage) is built only on request (EQS_SELL_SH=1):
  // measured slower than the full stencil copy on B200
  const bool want_sym = getenv("EQS_SELL_SH") != nullptr && atoi(getenv("EQS_SELL_SH")) != 0;
  if (h.n_rows == 0 || !build_sell_stencil(h, hs, true, want_sym)) return;
  b.st_vals.alloc(hs.vals.size());
  b.st_vals.upload(hs.vals.data(), hs.vals.size(), s);
  b.st_pid.alloc(hs.pid.size());
  b.st_pid.upload(hs.pid.data(), hs.pid.size(), s);
  b.st_pat.alloc(hs.pat.size());
  b.st_pat.upload(hs.pat.data(), hs.pat.size(), s);
  b.st_v64.alloc(hs.vals64.size());
  b.st_v64.upload(hs.vals64.data(), hs.vals64.size(), s);
  CK(cudaStreamSynchronize(s));
  d.st.n_chunks = hs.n_chunks;
  d.st.G = hs.G;
  d.st.P = hs.P;
  d.st.common = hs.common;
  if (hs.G == 2)
    for (int j = 0; j < 16; ++j) d.st.coff[j] = hs.pat[(size_t)hs.common * 16 + j];
  // the common pattern's offsets as kernel parameters, other patterns through L1 (no
  // per-CTA staging barrier; interleaved A/B at C3: 112.4 vs 115.2 ms per step);
  // EQS_SELLS_STAGE=1 stages the table in shared memory
  static const int stage = getenv("EQS_SELLS_STAGE") ? atoi(getenv("EQS_SELLS_STAGE")) : 0;
  d.st.stage = stage;
  d.st.n_cols = h.n_cols;
  d.st.vals = reinterpret_cast<const uint4*>(b.st_vals.p);
  d.st.pid = b.st_pid.p;
  d.st.pat = b.st_pat.p;
  d.st.vals64 = hs.vals64.empty() ? nullptr : b.st_v64.p;
  if (hs.sym) {
    b.sh_u16.alloc(hs.uvals.size());
    b.sh_u16.upload(hs.uvals.data(), hs.uvals.size(), s);
    b.sh_u64.alloc(hs.uvals64.size());
    b.sh_u64.upload(hs.uvals64.data(), hs.uvals64.size(), s);
    b.sh_spid.alloc(hs.spid.size());
    b.sh_spid.upload(hs.spid.data(), hs.spid.size(), s);
    b.sh_sinfo.alloc(hs.sinfo.size());
    b.sh_sinfo.upload(hs.sinfo.data(), hs.sinfo.size(), s);
    b.sh_slow.alloc(hs.slow_code.size() + 32 * 16);  // padded lanes of the last chunk may index past the table
    if (!hs.slow_code.empty()) b.sh_slow.upload(hs.slow_code.data(), hs.slow_code.size(), s);
    b.sh_slow_base.alloc(hs.slow_base.size());
    b.sh_slow_base.upload(hs.slow_base.data(), hs.slow_base.size(), s);
    CK(cudaStreamSynchronize(s));
    d.st.u16 = b.sh_u16.p;
    d.st.u64 = b.sh_u64.p;
    d.st.spid = b.sh_spid.p;
    d.st.sinfo = b.sh_sinfo.p;
    d.st.slow_code = reinterpret_cast<const uint4*>(b.sh_slow.p);
    d.st.slow_base = b.sh_slow_base.p;
    d.st.sym = true;
  }
}

// 1/diag of the owned rows (local row i <-> local column i)
// EQS_MEMTRACE=1: host RSS / peak at setup checkpoints (stderr)
void memtrace(const char* tag) {
  static const bool on = getenv("EQS_MEMTRACE") != nullptr;
  if (!on) return;
  FILE* f = fopen("/proc/self/status", "r");
  if (!f) return;
  char line[256];
  long rss = 0, hwm = 0;
  while (fgets(line, sizeof line, f)) {
    if (!strncmp(line, "VmRSS:", 6)) rss = atol(line + 6);
    if (!strncmp(line, "VmHWM:", 6)) hwm = atol(line + 6);
  }
  fclose(f);
  static auto last = std::chrono::steady_clock::now();
  const auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[memtrace] %-28s rss %7.2f GB  peak %7.2f GB  +%.2f s\n", tag, rss / 1048576.0, hwm / 1048576.0,
          std::chrono::duration<double>(now - last).count());
  last = now;
}

std::vector<double> inv_diagonal(const HostCsr& a) {
  std::vector<double> d(a.n_rows, 0.0);
  for (int i = 0; i < a.n_rows; ++i)
    for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
      if (a.col_idx[k] == i) d[i] = 1.0 / a.values[k];
  return d;
}
}  // namespace

// V-cycle truncation of the prolongators (additive key
// solver.amg_vcycle_truncate = [theta_0, theta_1, ...], default [0.1, 0.15,
// 0.03]): P_l keeps the entries with |p_ij| >= theta_l max_j |p_ij| of its
// row, rescaled to the row's sum (so constants are still interpolated
// exactly; rows whose kept entries cannot carry the sum stay whole),
// R_l = P_l^T, and every coarser Galerkin operator A_{m+1} = R_m A_m P_m is
// recomputed from the first truncated level on (device SpGEMM). The reference hierarchy is stashed and restored once the device
// levels are built, so the hierarchy the API reports stays the reference's.
void GpuSystem::truncate_vcycle_prolongators() {
  auto& L = amg_.levels;
  const int nl = (int)L.size();
  // theta per level: solver.amg_vcycle_truncate; the coarsest level's P is
  // never truncated below a 3-level hierarchy
  std::vector<double> theta(nl, 0.0);
  for (int l = 0; l + 1 < nl && l < (int)prob_.solver.amg_vcycle_truncate.size(); ++l)
    if (nl >= 3) theta[l] = prob_.solver.amg_vcycle_truncate[l];
  for (int l = 0; l + 1 < nl; ++l) {  // EQS_VCYCLE_TRUNCATE_L<l>=theta overrides level l (experiments)
    const std::string key = "EQS_VCYCLE_TRUNCATE_L" + std::to_string(l);
    if (getenv(key.c_str())) theta[l] = atof(getenv(key.c_str()));
  }
  int l0 = -1;
  for (int l = 0; l + 1 < nl && l0 < 0; ++l)
    if (theta[l] > 0.0) l0 = l;
  if (l0 < 0) return;
  amg_stash_.assign(nl, AmgHostLevel{});
  amg_stash_coarse_inv_ = amg_.coarse_inverse;
  for (int l = l0; l + 1 < nl; ++l) {
    if (theta[l] > 0.0) {
      HostCsr& P = L[l].P;
      HostCsr q;
      q.n_rows = P.n_rows;
      q.n_cols = P.n_cols;
      q.row_ptr.assign(P.n_rows + 1, 0);
      for (int i = 0; i < P.n_rows; ++i) {
        double mx = 0.0, s0 = 0.0, s1 = 0.0;
        for (int k = P.row_ptr[i]; k < P.row_ptr[i + 1]; ++k) {
          mx = std::max(mx, std::fabs(P.values[k]));
          s0 += P.values[k];
        }
        const size_t start = q.col_idx.size();
        for (int k = P.row_ptr[i]; k < P.row_ptr[i + 1]; ++k)
          if (std::fabs(P.values[k]) >= theta[l] * mx) {
            q.col_idx.push_back(P.col_idx[k]);
            q.values.push_back(P.values[k]);
            s1 += P.values[k];
          }
        const double f = s1 != 0.0 ? s0 / s1 : 0.0;
        if (f >= 0.5 && f <= 2.0) {
          for (size_t k = start; k < q.values.size(); ++k) q.values[k] *= f;
        } else {  // the kept entries cannot carry the row sum: keep the row whole
          q.col_idx.resize(start);
          q.values.resize(start);
          for (int k = P.row_ptr[i]; k < P.row_ptr[i + 1]; ++k) {
            q.col_idx.push_back(P.col_idx[k]);
            q.values.push_back(P.values[k]);
          }
        }
        q.row_ptr[i + 1] = (int)q.col_idx.size();
      }
      amg_stash_[l].P = std::move(P);
      amg_stash_[l].R = std::move(L[l].R);
      P = std::move(q);
      L[l].R = csr_transposed(P);
    }
  }
  // Galerkin operators below the first truncated level
  std::vector<const HostCsr*> ps, rs;
  for (int l = l0; l + 1 < nl; ++l) {
    ps.push_back(&L[l].P);
    rs.push_back(&L[l].R);
  }
  std::vector<HostCsr> ac;
  if (device_ >= 0) {
    ac = galerkin_chain_device(L[l0].A, ps, rs, device_);
  } else {
    ac.reserve(ps.size());
    const HostCsr* a = &L[l0].A;
    for (size_t k = 0; k < ps.size(); ++k) {
      ac.push_back(csr_multiply(*rs[k], csr_multiply(*a, *ps[k])));
      a = &ac.back();
    }
  }
  for (int l = l0; l + 1 < nl; ++l) {
    amg_stash_[l + 1].A = std::move(L[l + 1].A);
    L[l + 1].A = std::move(ac[l - l0]);
  }
  if (amg_.coarse_n > 0) amg_.coarse_inverse = dense_inverse(L.back().A);
  memtrace("v-cycle prolongators truncated");
}

// puts the reference hierarchy back (or drops the stash when the global
// hierarchy has been released on a multi-rank context)
void GpuSystem::restore_reference_hierarchy() {
  if (amg_stash_.empty()) return;
  auto& L = amg_.levels;
  const bool released = L.size() > 1 && L[0].A.n_rows == 0 && L[1].A.n_rows == 0;
  if (!released)
    for (size_t l = 0; l < L.size() && l < amg_stash_.size(); ++l) {
      if (amg_stash_[l].P.n_rows) L[l].P = std::move(amg_stash_[l].P);
      if (amg_stash_[l].R.n_rows) L[l].R = std::move(amg_stash_[l].R);
      if (amg_stash_[l].A.n_rows) L[l].A = std::move(amg_stash_[l].A);
    }
  if (!released) amg_.coarse_inverse = std::move(amg_stash_coarse_inv_);
  std::vector<AmgHostLevel>().swap(amg_stash_);
  std::vector<double>().swap(amg_stash_coarse_inv_);
}

GpuSystem::GpuSystem(Problem&& p, int device, std::unique_ptr<Comm> comm)
    : prob_(std::move(p)), device_(device), comm_(comm ? std::move(comm) : std::make_unique<SelfComm>()) {
  PhaseTimer timer(stats_.t_setup, "setup");
  if (device_ >= 0) {
    CK(cudaSetDevice(device_));
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    CK(cudaMallocHost(&pinned_, sizeof(double) * (S_COUNT + 8)));
    CK(cudaMallocHost(&pcg_pinned_, sizeof(double) * 9));
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
  memtrace("problem");
  // FemSystem ctor: assemble M once (fem_system.cpp:27-36)
  assemble_mass_blocks(prob_, m_ii_, m_ib_);
  memtrace("mass assembled");
  ++stats_.assemblies;
  // mass preconditioner (built once; the reference builds it lazily on first use, fem_system.cpp:48-54)
  if (prob_.solver.precond == 2) amg_ = build_amg(m_ii_, prob_.solver, device_);
  ++stats_.precond_setups;
  memtrace("amg built");
  if (prob_.solver.precond == 2) truncate_vcycle_prolongators();
  // device V-cycle depth: the first coarse level with at most amg_dense_coarse
  // rows is solved directly (explicit inverse of its Galerkin operator) instead
  // of recursing through the remaining latency-bound levels
  dev_levels_ = (int)amg_.levels.size();
  if (prob_.solver.precond == 2 && prob_.solver.amg_dense_coarse > 0)
    for (int l = 1; l + 1 < (int)amg_.levels.size(); ++l)
      if (amg_.levels[l].A.n_rows <= prob_.solver.amg_dense_coarse) {
        dev_levels_ = l + 1;
        break;
      }
  if (prob_.solver.precond == 2 && dev_levels_ < (int)amg_.levels.size()) {
    dev_coarse_n_ = amg_.levels[dev_levels_ - 1].A.n_rows;
    dev_coarse_inv_ = dense_inverse(amg_.levels[dev_levels_ - 1].A);
  } else {
    dev_coarse_n_ = amg_.coarse_n;
    dev_coarse_inv_ = amg_.coarse_inverse;
  }
  memtrace("dense coarse");
  // V-cycle operators of the coarse levels: lumped filtered Galerkin matrices
  // (DESIGN.md §4); the hierarchy reported through the API stays the reference's
  {
    std::vector<HostCsr> filtered;
    if (prob_.solver.precond == 2) {
      filtered.resize(amg_.levels.size());
      const double eps = prob_.solver.amg_coarse_filter;
      for (size_t l = 1; l + 1 < amg_.levels.size(); ++l)
        if (eps > 0.0) filtered[l] = filter_lumped(amg_.levels[l].A, eps);
    }
    memtrace("coarse filter");
    plan_ = build_plan(prob_, m_ii_, m_ib_, amg_, comm_->size(), comm_->rank(), prob_.solver.amg_replicate_rows,
                       &filtered, dev_levels_, device_);
  }
  memtrace("plan");
  if (comm_->size() > 1 && device_ >= 0) {
    // the rank's plan holds its operators: the global hierarchy's matrices
    // are only needed for single-rank API queries; release them before the
    // device build, then let the next rank of the node start its host setup
    // (setup_gate: bounded concurrency of the host phase, capi.cpp)
    for (auto& lv : amg_.levels) lv.A = lv.P = lv.R = HostCsr{};
    restore_reference_hierarchy();  // drops the stash
    malloc_trim(0);
    memtrace("global hierarchy released");
  }
  if (setup_gate_release) {
    setup_gate_release();
    setup_gate_release = nullptr;
  }
  const LocalSpace& s0 = plan_.space[0];
  n_own_ = s0.n_own();
  n_ghost_ = s0.n_ghost();
  n_loc_ = s0.n_local();
  n_fixloc_ = (int)plan_.fixed.size();
  n_full_ = n_loc_ + n_fixloc_;
  n_tets_loc_ = (int)plan_.tets.size();
  loc2ref_.assign(n_full_, -1);
  for (int i = 0; i < n_loc_; ++i) loc2ref_[i] = dm.free_dofs[i < n_own_ ? s0.owned[i] : s0.ghosts[i - n_own_]];
  for (int j = 0; j < n_fixloc_; ++j) loc2ref_[n_loc_ + j] = plan_.fixed[j];
  if (device_ >= 0) {
    build_device();
    // the rank's operators now live in HBM: drop their host copies (the index
    // spaces stay for the partition queries)
    for (auto* v : {&plan_.A, &plan_.P, &plan_.R}) std::vector<HostCsr>().swap(*v);
    plan_.mii = HostCsr{};
    plan_.mib = HostCsr{};
    std::vector<int>().swap(plan_.tet_dofs);
  }
  restore_reference_hierarchy();
  memtrace("device built");
}

GpuSystem::~GpuSystem() {
  invalidate_graphs();
  for (auto& e : events_) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto e : ev_pool_) cudaEventDestroy(e);
  if (pinned_) cudaFreeHost(pinned_);
  if (pcg_pinned_) cudaFreeHost(pcg_pinned_);
  if (stream_) cudaStreamDestroy(stream_);
}

void GpuSystem::require_single(const char* what) const {
  if (comm_->size() != 1)
    throw std::invalid_argument(std::string(what) + ": host-vector API needs a single-rank context");
}

void GpuSystem::build_halo(const LocalSpace& sp, DevHalo& h) {
  h.n_own = sp.n_own();
  std::map<int, std::pair<int, int>> rel;  // peer -> (send index, recv index)
  for (size_t k = 0; k < sp.send_ranks.size(); ++k) rel[sp.send_ranks[k]].first = (int)k + 1;
  for (size_t k = 0; k < sp.recv_ranks.size(); ++k) rel[sp.recv_ranks[k]].second = (int)k + 1;
  std::vector<int> idx;
  for (auto& [peer, sr] : rel) {
    h.peers.push_back(peer);
    h.send_off.push_back((int)idx.size());
    if (sr.first) {
      const auto& l = sp.send_local[sr.first - 1];
      idx.insert(idx.end(), l.begin(), l.end());
      h.send_cnt.push_back((int)l.size());
    } else {
      h.send_cnt.push_back(0);
    }
    if (sr.second) {
      h.recv_off.push_back(sp.recv_off[sr.second - 1]);
      h.recv_cnt.push_back(sp.recv_off[sr.second] - sp.recv_off[sr.second - 1]);
    } else {
      h.recv_off.push_back(0);
      h.recv_cnt.push_back(0);
    }
  }
  h.n_send = (int)idx.size();
  h.send_idx.alloc(std::max<size_t>(1, idx.size()));
  h.send_idx.upload(idx.data(), idx.size(), stream_);
  h.send_buf.alloc(std::max<size_t>(1, idx.size()));
  h.send_buf32.alloc(std::max<size_t>(1, idx.size()));
  CK(cudaStreamSynchronize(stream_));
}

template <class T>
void GpuSystem::halo(DevHalo& h, T* vec) {
  if (comm_->size() == 1 || h.peers.empty()) return;
  T* buf;
  if constexpr (std::is_same_v<T, double>) {
    buf = h.send_buf.p;
    launch_gather(h.n_send, h.send_idx.p, vec, buf, stream_);
  } else {
    buf = h.send_buf32.p;
    launch_gather_f(h.n_send, h.send_idx.p, vec, buf, stream_);
  }
  std::vector<HaloMsg> msgs;
  for (size_t k = 0; k < h.peers.size(); ++k)
    msgs.push_back({h.peers[k], buf + h.send_off[k], h.send_cnt[k], vec + h.n_own + h.recv_off[k], h.recv_cnt[k],
                    (int)sizeof(T)});
  comm_->exchange(msgs, stream_);
}
template void GpuSystem::halo<double>(DevHalo&, double*);
template void GpuSystem::halo<float>(DevHalo&, float*);

void GpuSystem::allreduce(int slot, int count) {
  if (comm_->size() > 1) comm_->allreduce(red_scal_.p + slot, count, stream_);
}

void GpuSystem::build_device() {
  const Dofs& dm = prob_.dm;
  const Mesh& mesh = prob_.mesh;
  cudaStream_t s = stream_;
  // coordinates per local dof (vertex dofs = nodes; P2 edge dofs unused by K1)
  {
    std::vector<double> c((size_t)std::max(1, n_full_) * 4, 0.0);
    for (int k = 0; k < n_full_; ++k) {
      const int r = loc2ref_[k];
      if (r >= 0 && r < mesh.n_nodes)
        for (int d = 0; d < 3; ++d) c[4L * k + d] = mesh.nodes[3L * r + d];
    }
    coords_.alloc(c.size());
    coords_.upload(c.data(), c.size(), s);
    CK(cudaStreamSynchronize(s));
  }
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
    const std::vector<int>& td = plan_.tet_dofs;
    std::vector<unsigned char> tm(n_tets_loc_);
    for (int k = 0; k < n_tets_loc_; ++k) tm[k] = (unsigned char)mat_index.at(mesh.region[plan_.tets[k]]);
    tet_dofs_.alloc(std::max<size_t>(1, td.size()));
    tet_dofs_.upload(td.data(), td.size(), s);
    tet_mat_.alloc(std::max<size_t>(1, tm.size()));
    tet_mat_.upload(tm.data(), tm.size(), s);
    CK(cudaStreamSynchronize(s));
    // blocked deterministic scatter (kxblock.hpp)
    const int nl = order_ == 1 ? 4 : 10;
    static const int env_bt = getenv("EQS_KX_BLOCK_TETS") ? atoi(getenv("EQS_KX_BLOCK_TETS")) : 0;
    const int bt = env_bt > 0 ? env_bt : (order_ == 1 ? 1024 : 512);
    std::vector<double> c4((size_t)std::max(1, n_full_) * 4, 0.0);
    CK(cudaMemcpy(c4.data(), coords_.p, sizeof(double) * c4.size(), cudaMemcpyDeviceToHost));
    KxBlocks kb = build_kx_blocks(td, nl, n_tets_loc_, c4, n_full_, bt);
    std::vector<int> btd((size_t)std::max(1, n_tets_loc_) * nl);
    std::vector<unsigned char> btm(std::max(1, n_tets_loc_) + 4, 0);  // k_kx_block4 copies whole words
    for (int k = 0; k < n_tets_loc_; ++k) {
      const int t = kb.tet_perm[k];
      for (int i = 0; i < nl; ++i) btd[(size_t)nl * k + i] = td[(size_t)nl * t + i];
      btm[k] = tm[t];
    }
    auto up = [&](auto& buf, const auto& v) {
      buf.alloc(std::max<size_t>(1, v.size()));
      buf.upload(v.data(), v.size(), s);
    };
    if (nl == 4) {
      up(kb_tloc_, kb.tet_local);
      // coordinates per block-dof entry, streamed by k_kx_block4 instead of gathered
      const size_t nld = kb.ldof_dof.size();
      std::vector<double> bc(3 * std::max<size_t>(1, nld));
      for (size_t i = 0; i < nld; ++i) {  // [nld] {x, y} pairs, then [nld] z
        bc[2 * i] = c4[4 * (size_t)kb.ldof_dof[i]];
        bc[2 * i + 1] = c4[4 * (size_t)kb.ldof_dof[i] + 1];
        bc[2 * nld + i] = c4[4 * (size_t)kb.ldof_dof[i] + 2];
      }
      up(kb_bxyz_, bc);
    } else {
      up(kb_tets_, btd);
    }
    up(kb_ldof_, kb.ldof_dof);
    up(kb_mat_, btm);
    up(kb_tet0_, kb.blk_tet0);
    up(kb_dof0_, kb.blk_dof0);
    up(kb_sptr_, kb.ldof_sptr);
    up(kb_slots_, kb.slots);
    up(kb_lout_, kb.ldof_out);
    up(kb_bdof_, kb.bdof);
    up(kb_bptr_, kb.bptr);
    up(kb_bpart_, kb.bpart);
    kb_partials_.alloc(std::max(1, kb.n_partials));
    CK(cudaStreamSynchronize(s));
    kxd_.nl = nl;
    kxd_.n_blocks = kb.n_blocks;
    kxd_.max_block_tets = kb.max_block_tets;
    kxd_.max_block_dofs = kb.max_block_dofs;
    kxd_.max_block_slots = kb.max_block_slots;
    kxd_.n_bdof = (int)kb.bdof.size();
    kxd_.blk_tet0 = kb_tet0_.p;
    kxd_.tets = nl == 4 ? reinterpret_cast<const int*>(kb_tloc_.p) : kb_tets_.p;
    kxd_.ldof_dof = kb_ldof_.p;
    kxd_.mat = kb_mat_.p;
    kxd_.blk_dof0 = kb_dof0_.p;
    kxd_.sptr = kb_sptr_.p;
    kxd_.slots = kb_slots_.p;
    kxd_.lout = kb_lout_.p;
    kxd_.partials = kb_partials_.p;
    kxd_.bdof = kb_bdof_.p;
    kxd_.bptr = kb_bptr_.p;
    kxd_.bpart = kb_bpart_.p;
    if (nl == 4 && !getenv("EQS_KX_GENERIC")) {
      const size_t nld = kb.ldof_dof.size();
      kxd_.bxy = kb_bxyz_.p;
      // EQS_KX_GATHER_COORDS=1: gather the padded coordinate rows instead of
      // streaming the per-block-dof copy
      const bool gather = getenv("EQS_KX_GATHER_COORDS") && atoi(getenv("EQS_KX_GATHER_COORDS")) != 0;
      kxd_.bz = gather ? nullptr : kb_bxyz_.p + 2 * nld;
    }
    kx_partials_ = kb.n_partials;
    kx_ldofs_ = (long)kb.ldof_out.size();
    kx_slots_ = (long)kb.slots.size();
  }
  err_.alloc(4);
  CK(cudaMemsetAsync(err_.p, 0, 4 * sizeof(int), s));
  memtrace("dev: coords + kx blocks");
  // Dirichlet data: set of every local fixed dof; compressed M_IB rows (owned) per set
  {
    std::vector<int> sof(std::max(1, n_fixloc_));
    for (int j = 0; j < n_fixloc_; ++j) sof[j] = dm.fixed_set[plan_.fixed[j]];
    set_of_fixed_.alloc(sof.size());
    set_of_fixed_.upload(sof.data(), sof.size(), s);
    const HostCsr& mib = plan_.mib;
    std::vector<int> rows;
    std::vector<double> coef;
    for (int r = 0; r < mib.n_rows; ++r) {
      if (mib.row_ptr[r] == mib.row_ptr[r + 1]) continue;
      rows.push_back(r);
      std::vector<double> c(n_sets_, 0.0);
      for (int k = mib.row_ptr[r]; k < mib.row_ptr[r + 1]; ++k)
        c[dm.fixed_set[dm.fixed_dofs[mib.col_idx[k]]]] += mib.values[k];
      coef.insert(coef.end(), c.begin(), c.end());
    }
    n_bl_rows_ = (int)rows.size();
    bl_rows_.alloc(std::max<size_t>(1, rows.size()));
    bl_rows_.upload(rows.data(), rows.size(), s);
    bl_coef_.alloc(std::max<size_t>(1, coef.size()));
    bl_coef_.upload(coef.data(), coef.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  memtrace("dev: dirichlet");
  // M_II (owned rows, local columns) + level-0 halo
  upload_csr(plan_.mii, mii_, mii_rp_, mii_ci_, mii_v_, s);
  upload_sell(plan_.mii, mii_, mii_s_, s);
  upload_stencil(plan_.mii, mii_, mii_s_, s);
  if (mii_.st.vals) launch_sells_rowsum(mii_.n_rows, mii_.st, mii_s_.st_vals.p, stencil_rowsum, s);
  set_sell(sell_on_);
  build_halo(plan_.space[0], halo0_);
  {
    std::vector<double> invd = inv_diagonal(plan_.mii);
    for (double v : invd)
      if (!std::isfinite(v)) throw NumericalError("Jacobi: zero diagonal");
    invd.resize(std::max(1, n_loc_), 0.0);
    mii_invd_.alloc(invd.size());
    mii_invd_.upload(invd.data(), invd.size(), s);
    halo(halo0_, mii_invd_.p);
  }
  memtrace("dev: M_II sell");
  // reductions + work vectors
  red_partials_.alloc((size_t)S_COUNT * kRedGrid);
  red_scal_.alloc(S_COUNT);
  pcg_stat_.alloc(9);
  red_counters_.alloc(S_COUNT);
  CK(cudaMemsetAsync(red_counters_.p, 0, sizeof(unsigned) * S_COUNT, s));
  CK(cudaMemsetAsync(red_scal_.p, 0, sizeof(double) * S_COUNT, s));
  red_ = Reducer{red_partials_.p, red_counters_.p, red_scal_.p};
  const size_t nl = std::max(1, n_loc_), nf = std::max(1, n_full_);
  for (auto* b : {&w_r_, &w_z_, &w_p_, &w_q_, &w_free_a_, &w_free_b_, &F0_, &F_, &Fn_, &rho_v_, &rho_w_}) b->alloc(nl);
  for (auto* b : {&w_full_a_, &w_full_b_}) b->alloc(nf);
  for (auto& b : full_) {
    b.alloc(nf);
    launch_fill((long)nf, 0.0, b.p, s);
  }
  X_ = full_[0].p;
  CK(cudaStreamSynchronize(s));
  if (prob_.solver.precond == 2) build_levels();
  set_sell(sell_on_);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
}

// AMG levels on this rank: owned rows of A_l (level 0: M_II; coarse levels:
// the lumped filtered operator), P_l, R_l, fp32 copies, halos, and the
// replicated dense coarsest solve.
void GpuSystem::build_levels() {
  cudaStream_t s = stream_;
  const int L = std::min((int)amg_.levels.size(), dev_levels_);
  levels_.clear();
  levels_.resize(L);
  auto f32 = [&](const std::vector<double>& v, DevBuf<float>& out) {
    std::vector<float> f(v.begin(), v.end());
    out.alloc(std::max<size_t>(1, f.size()));
    out.upload(f.data(), f.size(), s);
    CK(cudaStreamSynchronize(s));
  };
  for (int l = 0; l < L; ++l) {
    DevLevel& lv = levels_[l];
    const LocalSpace& sp = plan_.space[l];
    lv.n_own = sp.n_own();
    lv.n_loc = sp.n_local();
    lv.n_global = sp.n_global;
    lv.replicated = l >= plan_.rep_level;
    if (l == 0) {
      lv.A = mii_;  // shares indices / fp64 values with the PCG operator
    } else {
      upload_csr(plan_.A[l], lv.A, lv.a_rp, lv.a_ci, lv.a_v, s);
      if (l + 1 < L) upload_sell(plan_.A[l], lv.A, lv.a_s, s, false);
    }
    build_halo(sp, lv.halo);
    const size_t nloc = std::max(1, lv.n_loc);
    lv.z.alloc(nloc);
    lv.b.alloc(nloc);
    lv.t.alloc(nloc);
    lv.z2.alloc(nloc);
    lv.z32.alloc(nloc);
    lv.b32.alloc(nloc);
    lv.t32.alloc(nloc);
    lv.z2_32.alloc(nloc);
    lv.db.alloc(nloc);
    lv.dt.alloc(nloc);
    lv.db32.alloc(nloc);
    lv.dt32.alloc(nloc);
    if (l + 1 < L) {
      f32(plan_.A[l].values, lv.a_vf);
      upload_csr(plan_.P[l], lv.P, lv.p_rp, lv.p_ci, lv.p_v, s);
      upload_csr(plan_.R[l], lv.R, lv.r_rp, lv.r_ci, lv.r_v, s);
      f32(plan_.P[l].values, lv.p_vf);
      f32(plan_.R[l].values, lv.r_vf);
      upload_sell(plan_.P[l], lv.P, lv.p_s, s, false);
      upload_sell(plan_.R[l], lv.R, lv.r_s, s, false);
      std::vector<double> invd = inv_diagonal(plan_.A[l]);
      invd.resize(nloc, 0.0);
      lv.invd.alloc(nloc);
      lv.invd.upload(invd.data(), invd.size(), s);
      halo(lv.halo, lv.invd.p);
      lv.invd32.alloc(nloc);
      launch_to_f32(lv.n_loc, lv.invd.p, lv.invd32.p, s);  // owned + ghosts
    } else if (!lv.replicated) {
      // partitioned coarsest (single-level hierarchy): every rank solves the
      // dense system on the full vector assembled by scatter + allreduce
      std::vector<int> glob(nloc, 0);
      for (int i = 0; i < lv.n_loc; ++i) glob[i] = i < lv.n_own ? sp.owned[i] : sp.ghosts[i - lv.n_own];
      lv.glob.alloc(glob.size());
      lv.glob.upload(glob.data(), glob.size(), s);
      lv.full_b.alloc(std::max(1, sp.n_global));
      lv.full_z.alloc(std::max(1, sp.n_global));
    }
    CK(cudaStreamSynchronize(s));
  }
  coarse_n_ = dev_coarse_n_;
  coarse_inv_.alloc(std::max<size_t>(1, dev_coarse_inv_.size()));
  coarse_inv_.upload(dev_coarse_inv_.data(), dev_coarse_inv_.size(), s);
  {
    std::vector<float> f(dev_coarse_inv_.begin(), dev_coarse_inv_.end());
    coarse_inv32_.alloc(std::max<size_t>(1, f.size()));
    coarse_inv32_.upload(f.data(), f.size(), s);
    CK(cudaStreamSynchronize(s));
  }
  std::vector<double>().swap(dev_coarse_inv_);
  set_vcycle_precision(vcycle_prec_);
  set_sell(sell_on_);
  memtrace("dev: levels uploaded");
  // smoother bounds: lambda_max(D^-1 A_l) by 20 power iterations from a
  // global random vector (same on every rank), norms reduced over ranks
  std::mt19937 rng(12345u);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  for (int l = 0; l + 1 < L; ++l) {
    DevLevel& lv = levels_[l];
    const LocalSpace& sp = plan_.space[l];
    std::vector<double> g(sp.n_global);
    double nrm = 0.0;
    for (auto& e : g) {
      e = uni(rng);
      nrm += e * e;
    }
    nrm = std::sqrt(nrm);
    std::vector<double> v(std::max(1, lv.n_loc), 0.0);
    for (int i = 0; i < lv.n_own; ++i) v[i] = g[sp.owned[i]] / nrm;
    lv.z.upload(v.data(), v.size(), s);
    double lam = 1.0;
    for (int it = 0; it < 20; ++it) {
      halo(lv.halo, lv.z.p);
      launch_scaled_spmv(lv.A, lv.invd.p, lv.z.p, lv.t.p, s);
      lam = std::sqrt(lv.replicated ? dot_local(lv.n_own, lv.t.p, lv.t.p, S_NORM)
                                    : dot_n(lv.n_own, lv.t.p, lv.t.p, S_NORM));
      if (lam == 0.0) {
        lam = 1.0;
        break;
      }
      launch_scale(lv.n_own, 1.0 / lam, lv.t.p, lv.z.p, s);
    }
    // level 0 operator == the hierarchy's A_0: also use the setup's 10-step estimate
    lv.lambda_smoother = l == 0 ? std::max(lam, amg_.levels[l].lambda_max_scaled) : lam;
  }
  set_cheb(cheb_ratio);
}

// dot over n local entries of a replicated level (no reduction), read on the host
double GpuSystem::dot_local(int n, const double* a, const double* b, int slot) {
  launch_dot(n, a, b, red_, slot, stream_);
  return read_scalar(slot);
}

// global dot over n owned entries (reduced over ranks), read on the host
double GpuSystem::dot_n(int n, const double* a, const double* b, int slot) {
  launch_dot(n, a, b, red_, slot, stream_);
  allreduce(slot);
  return read_scalar(slot);
}

// Chebyshev smoother on [lmax/ratio, lmax] of D^-1 A, lmax = 1.1 x the power
// estimate. Degree 2: x += c0 D^-1 r0 + c1 D^-1 (r0 - A D^-1 r0 / theta);
// degree 1: x += D^-1 r0 / theta.
//
// cheb_kind 1: fourth-kind Chebyshev smoother (no lower bound), same kernels:
// d1 = 4/(3 lmax) D^-1 r, d2 = d1/5 + 12/(5 lmax) D^-1 (r - A d1), z = d1 + d2;
// degree 1 is z = 4/(3 lmax) D^-1 r. cheb_scale multiplies the power estimate.
void GpuSystem::set_cheb(double ratio) {
  invalidate_graphs();  // coefficients are baked into the captured kernel parameters
  cheb_ratio = ratio;
  for (auto& lv : levels_) {
    const double lmax = cheb_scale * lv.lambda_smoother;
    if (cheb_kind >= 1) {
      // kind 2: Lottes' optimised weights z = sum_k beta_k d_k (residual
      // recurrence unweighted): degree 1 beta 1.125; degree 2 (1.0239, 1.2641)
      const double b1 = cheb_kind == 2 ? 1.02387287570313 : 1.0, b2 = cheb_kind == 2 ? 1.26408905371085 : 1.0;
      const double b11 = cheb_kind == 2 ? 1.125 : 1.0;
      lv.cheb.c0 = (b1 + b2 / 5.0) * 4.0 / (3.0 * lmax);
      lv.cheb.c1 = b2 * 12.0 / (5.0 * lmax);
      lv.cheb.inv_theta = 4.0 / (3.0 * lmax);
      lv.cheb1 = ChebCoef{0.0, 0.0, b11 * 4.0 / (3.0 * lmax)};
      continue;
    }
    cheb_first_kind(lmax, ratio, lv);
  }
}

// first-kind Chebyshev on [lmax/ratio, lmax]: degree-2 and degree-1 coefficients
void cheb_first_kind(double lmax, double ratio, DevLevel& lv) {
  const double lmin = lmax / ratio;
  const double theta = 0.5 * (lmax + lmin), delta = 0.5 * (lmax - lmin);
  const double sigma = theta / delta, rho0 = 1.0 / sigma, rho1 = 1.0 / (2.0 * sigma - rho0);
  lv.cheb.c0 = (1.0 + rho1 * rho0) / theta;
  lv.cheb.c1 = 2.0 * rho1 / delta;
  lv.cheb.inv_theta = 1.0 / theta;
  lv.cheb1 = ChebCoef{0.0, 0.0, 1.0 / theta};
}

void GpuSystem::invalidate_graphs() {
  if (vcycle_graph_) cudaGraphExecDestroy(vcycle_graph_);
  vcycle_graph_ = nullptr;
  for (auto& kv : pcg_graphs_) cudaGraphExecDestroy(kv.second);
  pcg_graphs_.clear();
  pcg_graph_use_.clear();
}

void GpuSystem::set_level_tpr(int level, int tpr) {
  if (tpr < 1 || tpr > 32 || (tpr & (tpr - 1))) throw std::invalid_argument("tpr must be a power of two <= 32");
  invalidate_graphs();
  if (level == 0) mii_.tpr = tpr;
  if (level < (int)levels_.size()) levels_[level].A.tpr = tpr;
}

// V-cycle operators only: the PCG operator M_II stays fp64. bf16 is read from
// the SELL copies; a matrix without one falls back to its fp32 CSR values.
void GpuSystem::set_vcycle_precision(int prec) {
  if (prec < 0 || prec > 2) throw std::invalid_argument("V-cycle precision must be 0 (fp64), 1 (fp32) or 2 (bf16)");
  invalidate_graphs();
  vcycle_prec_ = prec;
  for (size_t l = 0; l + 1 < levels_.size(); ++l) {
    DevLevel& lv = levels_[l];
    lv.A.values_f = lv.a_vf.p;
    lv.P.values_f = lv.p_vf.p;
    lv.R.values_f = lv.r_vf.p;
    lv.A.prec = lv.P.prec = lv.R.prec = prec;
  }
}

void GpuSystem::set_stencil(bool on) {
  invalidate_graphs();
  mii_.use_stencil = on;
  for (auto& lv : levels_) lv.A.use_stencil = on;
}

// symmetric half storage of the stencil-coded fine operator (SELL-SH) where built
void GpuSystem::set_stencil_rowsum(bool on) {
  stencil_rowsum = on;
  if (device_ >= 0 && mii_.st.vals) {
    launch_sells_rowsum(mii_.n_rows, mii_.st, mii_s_.st_vals.p, on, stream_);
    CK(cudaStreamSynchronize(stream_));
  }
}

void GpuSystem::set_stencil_sym(bool on) {
  invalidate_graphs();
  mii_.st.sym = on && mii_.st.u64 != nullptr;
  if (!levels_.empty()) levels_[0].A.st.sym = mii_.st.sym;
}

void GpuSystem::set_sell(bool on) {
  invalidate_graphs();
  sell_on_ = on;
  mii_.use_sell = on && mii_.sell.tpr > 0;
  for (size_t l = 0; l < levels_.size(); ++l) {
    DevLevel& lv = levels_[l];
    for (DevCsr* m : {&lv.A, &lv.P, &lv.R}) m->use_sell = on && (m->sell.tpr > 0 || m->pk.tpr > 0);
  }
}

const std::vector<int>& GpuSystem::colors() {
  // device waves (k_setup.cu) on a GPU context; EQS_HOST_COLOR=1 keeps the sequential host loop
  static const bool host_color = getenv("EQS_HOST_COLOR") != nullptr && atoi(getenv("EQS_HOST_COLOR")) != 0;
  if (n_colors_ < 0)
    colors_ = device_ >= 0 && !host_color ? dev_color_elements(prob_.dm, n_tets_, &n_colors_, device_)
                                          : color_elements(prob_.dm, n_tets_, &n_colors_);
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
  open_bytes_ = g_algo_bytes;
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
  if (bytes < 0.0) bytes = g_algo_bytes - open_bytes_;  // launchers' own byte counts since tic
  cudaEvent_t b = get_event();
  CK(cudaEventRecord(b, stream_));
  events_.push_back({open_ev_, b, open_cls_, bytes});
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
// y written); P2 = 44 n_tets + 24 n_nodes + 24 n_dofs (this rank's share).
double GpuSystem::kx_bytes() const {
  if (order_ == 1) return 20.0 * n_tets_loc_ + 48.0 * n_full_;
  return 44.0 * n_tets_loc_ + 24.0 * prob_.mesh.n_nodes * ((double)n_full_ / std::max(1, n_dofs_)) + 24.0 * n_full_;
}
double GpuSystem::spmv_bytes(const DevCsr& a) const { return matrix_pass_bytes(a, 1, 1); }

// ------------------------------------------------------------------ operators
void GpuSystem::lift_dev(double t, double* x_full) {
  const std::vector<double> v = set_values(t, false);
  SetVals sv;
  std::copy(v.begin(), v.end(), sv.v);
  launch_lift_fixed(n_fixloc_, set_of_fixed_.p, sv, x_full + n_loc_, stream_);
}

// two-pass gather mode (stiffness_mode 2): per-tet products through HBM, then
// one thread per dof over an ascending-tet slot list; built on first use
void GpuSystem::build_kx_gather() {
  if (slots_built_) return;
  const std::vector<int>& td = tet_dofs_host();
  std::vector<long> ptr((size_t)n_full_ + 1, 0);
  for (size_t k = 0; k < td.size(); ++k) ++ptr[td[k] + 1];
  for (int d = 0; d < n_full_; ++d) ptr[d + 1] += ptr[d];
  if (ptr.back() >= (1L << 31)) throw ConfigError("mesh too large for int32 slot indices");
  std::vector<int> sl(std::max<long>(1, ptr.back()));
  std::vector<long> next(ptr.begin(), ptr.end() - 1);
  for (size_t k = 0; k < td.size(); ++k) sl[next[td[k]]++] = (int)k;
  slot_ptr_.alloc(ptr.size());
  slot_ptr_.upload(ptr.data(), ptr.size(), stream_);
  slots_.alloc(sl.size());
  slots_.upload(sl.data(), sl.size(), stream_);
  ytet_.alloc(std::max<size_t>(1, td.size()));
  CK(cudaStreamSynchronize(stream_));
  slots_built_ = true;
}

// tet dofs in the tet_dofs_ (unblocked) order, read back from the device
const std::vector<int>& GpuSystem::tet_dofs_host() {
  if (tet_dofs_h_.empty()) {
    tet_dofs_h_.resize((size_t)std::max(1, n_tets_loc_) * (order_ == 1 ? 4 : 10));
    CK(cudaMemcpy(tet_dofs_h_.data(), tet_dofs_.p, sizeof(int) * tet_dofs_h_.size(), cudaMemcpyDeviceToHost));
    tet_dofs_h_.resize((size_t)n_tets_loc_ * (order_ == 1 ? 4 : 10));
  }
  return tet_dofs_h_;
}

// out[d] = base[d] + sign * (K(x) v)[d] for the first n_out local dofs
// (blocked scatter by default, the two-pass gather in stiffness_mode 2)
void GpuSystem::kx_into(const double* x, const double* v, const double* base, double sign, double* out, int n_out) {
  if (stiffness_mode == 2) {
    build_kx_gather();
    kx_tets(x, v);
    launch_kx_gather(n_out, slot_ptr_.p, slots_.p, ytet_.p, base, sign, out, stream_);
    return;
  }
  launch_kx_blocked(kxd_, coords_.p, x, v, base, sign, n_out, out, err_.p, stream_);
  ++stats_.applies;
}

void GpuSystem::kx_tets(const double* x, const double* v) {
  launch_kx_tets(order_, n_tets_loc_, tet_dofs_.p, tet_mat_.p, coords_.p, x, v, ytet_.p, err_.p, stream_);
  ++stats_.applies;
}

// y (all local rows) = K(x) v; x and v carry valid ghost and fixed entries
void GpuSystem::kx_apply_full_dev(const double* x_state, const double* v, double* y) {
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    if (color_off_.empty()) {  // coloured batches of the local tets (matfree.cpp:100-117)
      const std::vector<int>& col = colors();
      std::vector<long> off(n_colors_ + 1, 0);
      for (int k = 0; k < n_tets_loc_; ++k) ++off[col[plan_.tets[k]] + 1];
      for (int c = 0; c < n_colors_; ++c) off[c + 1] += off[c];
      std::vector<int> order_t(std::max(1, n_tets_loc_));
      std::vector<long> nx(off.begin(), off.end() - 1);
      for (int k = 0; k < n_tets_loc_; ++k) order_t[nx[col[plan_.tets[k]]]++] = k;
      color_tets_.alloc(order_t.size());
      color_tets_.upload(order_t.data(), order_t.size(), stream_);
      color_off_ = off;
    }
    launch_fill(n_full_, 0.0, y, stream_);
    for (size_t c = 0; c + 1 < color_off_.size(); ++c)
      launch_kx_colored(order_, (int)(color_off_[c + 1] - color_off_[c]), color_tets_.p + color_off_[c],
                        tet_dofs_.p, tet_mat_.p, coords_.p, x_state, v, y, err_.p, stream_);
    ++stats_.applies;
  } else {
    kx_into(x_state, v, nullptr, 1.0, y, n_full_);
  }
  toc(TC_STIFF, kx_bytes());
}

// eval_residual core (fem_system.cpp:62-67 + matfree.cpp:138-143):
// r = -M_IB xdot_B(t) - (K(x) x)|owned with x lifted at t and its ghosts exchanged.
void GpuSystem::residual_dev(double t, double* x_full, double* r) {
  lift_dev(t, x_full);
  halo(halo0_, x_full);
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    kx_apply_full_dev(x_full, x_full, w_full_a_.p);
    launch_scale(n_own_, -1.0, w_full_a_.p, r, stream_);
  } else {
    kx_into(x_full, x_full, nullptr, -1.0, r, n_own_);
  }
  toc(TC_STIFF, kx_bytes() - 8.0 * n_fixloc_);
  const std::vector<double> rt = set_values(t, true);
  SetVals sv;
  std::copy(rt.begin(), rt.end(), sv.v);
  launch_boundary_load(n_bl_rows_, bl_rows_.p, bl_coef_.p, n_sets_, sv, r, stream_);
  check_kernel_flags();
}

void GpuSystem::mass_apply_dev(double* v, double* y) {
  halo(halo0_, v);
  launch_spmv(mii_, v, y, stream_);
}

// level buffers of the V-cycle vector type
template <class XT>
struct VBufs;
template <>
struct VBufs<double> {
  static double* b(DevLevel& l) { return l.b.p; }
  static double* z(DevLevel& l) { return l.z.p; }
  static double* z2(DevLevel& l) { return l.z2.p; }
  static double* t(DevLevel& l) { return l.t.p; }
  static double* invd(DevLevel& l) { return l.invd.p; }
  static double* db(DevLevel& l) { return l.db.p; }
  static double* dt(DevLevel& l) { return l.dt.p; }
};
template <>
struct VBufs<float> {
  static float* b(DevLevel& l) { return l.b32.p; }
  static float* z(DevLevel& l) { return l.z32.p; }
  static float* z2(DevLevel& l) { return l.z2_32.p; }
  static float* t(DevLevel& l) { return l.t32.p; }
  static float* invd(DevLevel& l) { return l.invd32.p; }
  static float* db(DevLevel& l) { return l.db32.p; }
  static float* dt(DevLevel& l) { return l.dt32.p; }
};

// Symmetric V-cycle (amg.cpp:145-172 structure) with Chebyshev smoothing:
// degree `cheb_degree` on the fine level, `coarse_degree` below; the same
// polynomial pre and post keeps the preconditioner symmetric for PCG. Every
// gathered vector has its ghosts exchanged first (no-op on one rank). XT is
// the vector type of the levels (fp32 by default). With fp32
// vectors the fine level reads the fp32 copy of r (b) and its last kernel
// writes z in fp64 (out64, with r64 . z when dot_into_rz).
template <class XT>
XT* GpuSystem::vcycle_t(int l, const XT* b_in, bool dot_into_rz, const double* r64, double* out64, const XT* pre) {
  using V = VBufs<XT>;
  const int L = (int)levels_.size();
  DevLevel& lv = levels_[l];
  XT* b = const_cast<XT*>(b_in);
  if (l == L - 1) {
    // dense solve on the full vector (replicated level: b is already whole)
    XT* z = V::z(lv);
    if (comm_->size() == 1 || lv.replicated) {
      launch_dense_solve<XT>(coarse_n_, coarse_inv_.p, coarse_inv32_.p, b, z, stream_);
    } else {
      if constexpr (std::is_same_v<XT, double>) {
        launch_fill(coarse_n_, 0.0, lv.full_b.p, stream_);
        launch_scatter(lv.n_own, lv.glob.p, b, lv.full_b.p, stream_);
        comm_->allreduce(lv.full_b.p, coarse_n_, stream_);
        launch_dense_solve<double>(coarse_n_, coarse_inv_.p, nullptr, lv.full_b.p, lv.full_z.p, stream_);
        launch_gather(lv.n_loc, lv.glob.p, lv.full_z.p, z, stream_);  // owned + ghosts
      } else {
        throw std::logic_error("fp32 V-cycle needs a replicated coarsest level");
      }
    }
    if (dot_into_rz) {
      if constexpr (std::is_same_v<XT, double>) {
        launch_dot(lv.n_own, b, z, red_, S_RZ, stream_);
        allreduce(S_RZ);
      }
    }
    return z;
  }
  DevLevel& nx = levels_[l + 1];
  const int deg = l == 0 ? cheb_degree : coarse_degree;
  const int deg_pre = (l == 0 && fine_pre_degree > 0) ? fine_pre_degree : deg;
  XT* z = V::z(lv);
  XT* t = V::t(lv);
  XT* invd = V::invd(lv);
  // pre: D^-1 b, written by the producer of b (PCG update or the restriction),
  // gathered by the smoother instead of b and D^-1 (k_rows.cu OP 8/9)
  if (deg_pre >= 2) {
    halo(lv.halo, pre ? const_cast<XT*>(pre) : b);
    launch_cheb_pre<XT>(lv.A, invd, b, z, lv.cheb, stream_, pre);
    halo(lv.halo, z);
    launch_residual<XT>(lv.A, b, z, t, nullptr, 0, stream_);
  } else if (pre || lv.A.lanes() <= 4) {
    halo(lv.halo, pre ? const_cast<XT*>(pre) : b);
    launch_cheb1_pre_resid<XT>(lv.A, invd, b, z, t, lv.cheb1, stream_, pre);
  } else {
    // dense rows: one gathered vector per entry instead of two (b and D^-1)
    halo(lv.halo, b);
    launch_diag_scale<XT>(lv.n_loc, invd, b, lv.cheb1.inv_theta, z, stream_);
    launch_residual<XT>(lv.A, b, z, t, nullptr, 0, stream_);
  }
  halo(lv.halo, t);
  XT* bc = V::b(nx);
  // entering the replicated levels: every rank holds the partial restriction
  // of its owned rows for all coarse rows; the sum is the coarse right-hand side
  const bool to_rep = nx.replicated && !lv.replicated && comm_->size() > 1;
  XT* prec = (!to_rep && level_takes_pre(l + 1)) ? V::db(nx) : nullptr;
  if (prec)
    launch_spmv_scaled<XT>(lv.R, t, V::invd(nx), bc, prec, stream_);
  else
    launch_spmv<XT>(lv.R, t, bc, stream_);
  if (to_rep) comm_->allreduce(bc, nx.n_loc, stream_);
  XT* zc = vcycle_t<XT>(l + 1, bc, false, nullptr, nullptr, prec);
  halo(nx.halo, zc);  // no-op on replicated levels
  launch_prolong_add<XT>(lv.P, zc, z, stream_);
  halo(lv.halo, z);
  if (wcycle_from > 0 && l >= wcycle_from && l + 2 < L && comm_->size() == 1) {
    // W-cycle on the coarse levels (option 28): a second coarse-grid
    // correction from the updated residual before the post-smoother; the
    // cycle stays symmetric (same correction twice between the smoothers)
    launch_residual<XT>(lv.A, b, z, t, nullptr, 0, stream_);
    if (prec)
      launch_spmv_scaled<XT>(lv.R, t, V::invd(nx), bc, prec, stream_);
    else
      launch_spmv<XT>(lv.R, t, bc, stream_);
    zc = vcycle_t<XT>(l + 1, bc, false, nullptr, nullptr, prec);
    launch_prolong_add<XT>(lv.P, zc, z, stream_);
  }
  const bool to64 = out64 != nullptr;  // fine level of an fp32 V-cycle
  Reducer r = red_;
  if (deg >= 2) {
    XT* dtp = lv.A.packed() ? V::dt(lv) : nullptr;  // D^-1 t for the post step's gather
    if (dtp)
      launch_residual_scaled<XT>(lv.A, b, z, invd, t, dtp, stream_);
    else
      launch_residual<XT>(lv.A, b, z, t, nullptr, 0, stream_);
    halo(lv.halo, dtp ? dtp : t);
    if constexpr (std::is_same_v<XT, float>) {
      if (to64) {
        launch_cheb_post2_out64(lv.A, invd, t, z, lv.cheb, out64, r64, dot_into_rz ? &r : nullptr, S_RZ, stream_,
                                dtp);
        if (dot_into_rz) allreduce(S_RZ);
        return nullptr;
      }
    }
    launch_cheb_post2<XT>(lv.A, invd, t, z, lv.cheb, dot_into_rz ? b : nullptr, dot_into_rz ? &r : nullptr, S_RZ,
                          stream_, dtp);
    if (dot_into_rz) allreduce(S_RZ);
    return z;
  }
  XT* z2 = V::z2(lv);
  launch_cheb1_post<XT>(lv.A, invd, b, z, z2, lv.cheb1, stream_);
  if constexpr (std::is_same_v<XT, float>) {
    if (to64) {
      launch_to_f64_dot(lv.n_own, z2, out64, r64, dot_into_rz ? &r : nullptr, S_RZ, stream_);
      if (dot_into_rz) allreduce(S_RZ);
      return nullptr;
    }
  }
  if (dot_into_rz) {
    if constexpr (std::is_same_v<XT, double>) {
      launch_dot(lv.n_own, b, z2, red_, S_RZ, stream_);
      allreduce(S_RZ);
    }
  }
  return z2;
}

// level l's pre-smoother gathers D^-1 b (packed operator with a scaled-gather op)
bool GpuSystem::level_takes_pre(int l) const {
  if (l <= 0 || l + 1 >= (int)levels_.size()) return false;
  const DevLevel& lv = levels_[l];
  return lv.A.packed();
}

// fp32 V-cycle inputs of the fine level: b32 = (float) r, db32 = D^-1 b32
void GpuSystem::vcycle_prepare(const double* r) {
  if (vcycle_f32_ && levels_.size() >= 2) {
    DevLevel& f = levels_[0];
    launch_to_f32_scaled(n_own_, r, f.invd32.p, f.b32.p, f.db32.p, stream_);
  }
}

// V-cycle on the fine residual r (fp64): returns z (fp64) and r.z in S_RZ.
// The fp32 V-cycle reads b32/db32, prepared by vcycle_prepare or the PCG update.
double* GpuSystem::vcycle(const double* r) {
  if (vcycle_f32_ && levels_.size() >= 2) {
    DevLevel& f = levels_[0];
    vcycle_t<float>(0, f.b32.p, true, r, f.z.p, f.A.packed() ? f.db32.p : nullptr);
    return f.z.p;
  }
  return vcycle_t<double>(0, r, true, nullptr, nullptr, nullptr);
}

// The V-cycle is a fixed sequence of kernels (and, on several ranks, NCCL
// halo/allreduce calls) on fixed buffers, so it is captured once into a CUDA
// graph and replayed: one launch per preconditioner application.
double* GpuSystem::precondition(double* r, bool prepared) {
  tic(TC_VCYCLE);
  const double bytes0 = g_algo_bytes;
  double* z;
  if (prob_.solver.precond == 2) {
    if (!prepared) vcycle_prepare(r);
    if (use_graphs && comm_->capturable() && r == w_r_.p) {
      if (!vcycle_graph_) {
        cudaGraph_t graph;
        const long before = g_launch_count;
        const double bytes_before = g_algo_bytes;
        CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        vcycle_out_ = vcycle(r);
        CK(cudaStreamEndCapture(stream_, &graph));
        vcycle_graph_kernels_ = g_launch_count - before;
        vcycle_graph_bytes_ = g_algo_bytes - bytes_before;
        g_launch_count = before;
        g_algo_bytes = bytes_before;
        CK(cudaGraphInstantiate(&vcycle_graph_, graph, 0));
        CK(cudaGraphDestroy(graph));
      }
      CK(cudaGraphLaunch(vcycle_graph_, stream_));
      g_launch_count += vcycle_graph_kernels_;
      g_algo_bytes += vcycle_graph_bytes_;
      z = vcycle_out_;
    } else {
      z = vcycle(r);
    }
  } else {
    Reducer rr = red_;
    z = w_z_.p;
    launch_jacobi(n_own_, mii_invd_.p, r, z, &rr, S_RZ, stream_);
    allreduce(S_RZ);
    g_algo_bytes += 24.0 * n_own_;
  }
  toc(TC_VCYCLE, g_algo_bytes - bytes0);
  return z;
}

// The whole PCG iteration of pcg_dev as one CUDA graph: k_pcg_check0 tests
// the initial residual and sets the condition of a WHILE node whose body is
// one iteration (V-cycle on r with r.z, p = z (first) or z + beta p, q = A p
// with p.q, the x/r update with r.r and the next V-cycle's fp32 inputs), closed
// by k_pcg_check (the stopping rule and breakdown tests on the device).
// Kernels and arguments are those of the host loop, so every iteration
// computes the same values; the host reads the verdict once per solve.
cudaGraphExec_t GpuSystem::pcg_loop_graph(double* x, bool f32) {
  auto it = pcg_graphs_.find(x);
  if (it != pcg_graphs_.end()) {
    pcg_graph_use_[x] = ++pcg_graph_clock_;
    return it->second;
  }
  if (pcg_graphs_.size() >= 8) {  // bounded cache: evict the least recently used graph
    double* lru = nullptr;
    long oldest = -1;
    for (auto& kv : pcg_graph_use_)
      if (oldest < 0 || kv.second < oldest) {
        oldest = kv.second;
        lru = kv.first;
      }
    cudaGraphExecDestroy(pcg_graphs_[lru]);
    pcg_graphs_.erase(lru);
    pcg_graph_use_.erase(lru);
  }
  ++pcg_graph_captures;  // counted: a caller cycling through many x buffers re-captures
  pcg_graph_use_[x] = ++pcg_graph_clock_;
  const int n = n_own_;
  double* r = w_r_.p;
  double* p = w_p_.p;
  double* q = w_q_.p;
  cudaGraph_t graph;
  CK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle handle;
  CK(cudaGraphConditionalHandleCreate(&handle, graph, 0, cudaGraphCondAssignDefault));
  const long before = g_launch_count;
  const double bytes_before = g_algo_bytes;
  CK(cudaStreamBeginCaptureToGraph(stream_, graph, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  launch_pcg_check0(red_scal_.p, pcg_stat_.p, handle, stream_);
  CK(cudaStreamEndCapture(stream_, &graph));
  cudaGraphNode_t check0;
  size_t n_nodes = 1;
  CK(cudaGraphGetNodes(graph, &check0, &n_nodes));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, graph, &check0, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const long body_before = g_launch_count;
  const double body_bytes_before = g_algo_bytes;
  CK(cudaStreamBeginCaptureToGraph(stream_, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  if (!f32) vcycle_prepare(r);
  double* z = vcycle(r);  // r.z allreduced inside on several ranks
  // x += alpha p of iteration k is applied by the direction kernel of
  // iteration k+1 (which reads p anyway) or by k_pcg_xfinal after the loop
  launch_pcg_direction(n, p, z, red_scal_.p, stream_, pcg_stat_.p, x);
  halo(halo0_, p);  // no-ops on one rank; NCCL calls on a multi-rank context
  launch_spmv_dot(mii_, p, q, red_, S_PQ, stream_);
  allreduce(S_PQ);
  DevLevel& f0 = levels_.empty() ? dummy_level_ : levels_[0];
  if (f32)
    launch_pcg_update(n, nullptr, r, p, q, red_, stream_, f0.b32.p, f0.invd32.p, f0.db32.p);
  else
    launch_pcg_update(n, nullptr, r, p, q, red_, stream_);
  allreduce(S_RR);
  launch_pcg_check(red_scal_.p, pcg_stat_.p, handle, stream_);
  CK(cudaStreamEndCapture(stream_, &body));
  pcg_body_kernels_ = g_launch_count - body_before;
  pcg_body_bytes_ = g_algo_bytes - body_bytes_before;
  g_launch_count = before;
  g_algo_bytes = bytes_before;
  cudaGraphExec_t exec;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  CK(cudaGraphDestroy(graph));
  pcg_graphs_[x] = exec;
  return exec;
}

// pcg_dev with the iteration in one graph launch (pcg_loop_graph): the
// start (x = x0 and r = b - A x0, or x = 0 and r = b) is enqueued, then the
// graph; one host read of the verdict per solve.
PcgResult GpuSystem::pcg_dev_graph(const double* b, bool use_x0, const double* x0, double* x, double tol,
                                   int max_iter, double bnorm) {
  const int n = n_own_;
  PcgResult res;
  double* r = w_r_.p;
  double* p = w_p_.p;
  if (use_x0) {
    if (x0 != x) CK(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    CK(cudaMemcpyAsync(p, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    halo(halo0_, p);
    Reducer rd = red_;
    launch_residual(mii_, b, p, r, &rd, S_RR, stream_);
    allreduce(S_RR);
  } else {
    launch_fill(n, 0.0, x, stream_);
    CK(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
  }
  const bool f32 = vcycle_f32_ && levels_.size() >= 2;
  if (f32) vcycle_prepare(r);  // the first V-cycle's fp32 inputs (later ones come out of the update)
  cudaGraphExec_t loop = pcg_loop_graph(x, f32);
  double* st = pcg_pinned_;
  st[0] = 0.0;
  st[1] = 0.0;
  st[2] = 0.0;
  st[3] = 0.0;
  st[4] = bnorm;
  st[5] = tol;
  st[6] = max_iter;
  st[7] = use_x0 ? -1.0 : bnorm * bnorm;
  st[8] = 0.0;
  CK(cudaMemcpyAsync(pcg_stat_.p, st, sizeof(double) * 9, cudaMemcpyHostToDevice, stream_));
  tic(TC_PCG_GRAPH);
  CK(cudaGraphLaunch(loop, stream_));
  toc(TC_PCG_GRAPH, 0.0);
  CK(cudaMemcpyAsync(st, pcg_stat_.p, sizeof(double) * 9, cudaMemcpyDeviceToHost, stream_));
  sync();
  const int k_end = (int)st[0];
  if (timing_on && !events_.empty() && events_.back().cls == TC_PCG_GRAPH)
    events_.back().bytes = (double)k_end * pcg_body_bytes_;
  const int status = (int)st[1];
  g_launch_count += 1 + (long)k_end * pcg_body_kernels_;
  g_algo_bytes += (double)k_end * pcg_body_bytes_;
  res.iterations = k_end;
  res.initial_rel_residual = st[8];
  res.rel_residual = st[2];
  if (k_end >= 1 && (status == PCG_CONVERGED || status == PCG_MAX_ITER)) {
    launch_pcg_xfinal(n, x, p, red_scal_.p, stream_);
  }
  switch (status) {
    case PCG_CONVERGED: res.converged = true; return res;
    case PCG_BAD_INIT: throw NumericalError("pcg: non-finite initial residual");
    case PCG_BAD_RZ: throw NumericalError("pcg: non-finite preconditioned residual");
    case PCG_BAD_PQ:
      throw NumericalError("pcg: operator not positive definite (p'Ap = " + std::to_string(st[3]) + ")");
    case PCG_BAD_REL: throw NumericalError("pcg: non-finite residual");
    default: break;
  }
  // PCG_MAX_ITER: the host loop's last precondition + direction, then its check
  CK(cudaMemcpyAsync(red_scal_.p + S_RZ_OLD, red_scal_.p + S_RZ, sizeof(double), cudaMemcpyDeviceToDevice, stream_));
  double* z = precondition(r, f32);
  launch_pcg_direction(n, p, z, red_scal_.p, stream_);
  double sc[1];
  read_scalars(S_RZ, 1, sc);
  if (!std::isfinite(sc[0])) throw NumericalError("pcg: non-finite preconditioned residual");
  return res;
}

// pcg_solve (proj/src/pcg.cpp:9-72) with device vectors; host reads three
// scalars per iteration for the stopping rule and the breakdown checks.
// b, x: owned entries; x0 may be null.
PcgResult GpuSystem::pcg_dev(const double* b, const double* x0, double* x, double tol, int max_iter) {
  const int n = n_own_;
  PcgResult res;
  // The iteration runs as one CUDA graph (pcg_loop_graph) when the V-cycle
  // is capturable and no per-class timing is requested; the decisions are the
  // same tests on the same scalars, evaluated on the device.
  // multi-rank: only on capturable (NCCL) communicators, whose halo and
  // allreduce calls are captured into the loop body
  const bool graph_loop = pcg_graph_loop && use_graphs && (!timing_on || timing_graph) && prob_.solver.precond == 2 &&
                          comm_->capturable() && device_ >= 0 && max_iter >= 1 &&
                          (comm_->size() == 1 || pcg_graph_multi);
  launch_dot(n, b, b, red_, S_BB, stream_);
  allreduce(S_BB);
  if (x0) {  // S_X0X0 follows S_BB: one read for both
    launch_dot(n, x0, x0, red_, S_X0X0, stream_);
    allreduce(S_X0X0);
  }
  double bx[2] = {0.0, 0.0};
  read_scalars(S_BB, x0 ? 2 : 1, bx);
  const double bnorm = std::sqrt(bx[0]);
  if (bnorm == 0.0) {
    launch_fill(n, 0.0, x, stream_);
    res.converged = true;
    return res;
  }
  const bool use_x0 = x0 && bx[1] != 0.0;
  if (graph_loop) return pcg_dev_graph(b, use_x0, x0, x, tol, max_iter, bnorm);
  double* r = w_r_.p;
  double* z = nullptr;
  double* p = w_p_.p;
  double* q = w_q_.p;
  double rr;
  tic(TC_PCG);
  if (use_x0) {
    if (x0 != x) CK(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    // the residual gathers x: stage it in p, which has room for ghosts
    CK(cudaMemcpyAsync(p, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    halo(halo0_, p);
    Reducer rd = red_;
    launch_residual(mii_, b, p, r, &rd, S_RR, stream_);
    allreduce(S_RR);
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
    halo(halo0_, p);
    launch_spmv_dot(mii_, p, q, red_, S_PQ, stream_);
    allreduce(S_PQ);
    const bool f32 = prob_.solver.precond == 2 && vcycle_f32_ && levels_.size() >= 2;
    DevLevel& f0 = levels_.empty() ? dummy_level_ : levels_[0];
    if (f32)  // the next V-cycle's fp32 inputs come out of the update
      launch_pcg_update(n, x, r, p, q, red_, stream_, f0.b32.p, f0.invd32.p, f0.db32.p);
    else
      launch_pcg_update(n, x, r, p, q, red_, stream_);
    allreduce(S_RR);
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
    z = precondition(r, f32);
    tic(TC_PCG);
    launch_pcg_direction(n, p, z, red_scal_.p, stream_);
    toc(TC_PCG, 24.0 * n);
  }
  read_scalars(S_RZ, 1, sc);
  if (!std::isfinite(sc[0])) throw NumericalError("pcg: non-finite preconditioned residual");
  return res;
}

// ------------------------------------------------------------------ estimator
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
      spe_q_[s].back()->alloc(std::max(1, n_loc_));
      spe_w_[s].push_back(std::make_unique<DevBuf<double>>());
      spe_w_[s].back()->alloc(std::max(1, n_loc_));
    }
}

double GpuSystem::dot_own(const double* a, const double* b, int slot) { return dot_n(n_own_, a, b, slot); }

// G row/column k (G_ik = q_i' W_k) for the basis vectors 0..k of the current set
void GpuSystem::spe_g_column(int k) {
  std::vector<const double*> Q(k + 1);
  for (int i = 0; i <= k; ++i) Q[i] = spe_q(spe_set_, i);
  launch_multi_dot(n_own_, k + 1, Q.data(), spe_w(spe_set_, k), red_, S_MDOT, stream_);
  allreduce(S_MDOT, k + 1);
  double g[kMaxMulti];
  read_scalars(S_MDOT, k + 1, g);
  spe_G_.resize((size_t)kMaxMulti * kMaxMulti);
  for (int i = 0; i <= k; ++i) spe_G_[(size_t)i * kMaxMulti + k] = spe_G_[(size_t)k * kMaxMulti + i] = g[i];
}

// mgs_orthonormalize (start_vector.cpp:10-28) over the whole history, reference order
void GpuSystem::spe_rebuild() {
  const int n = n_own_;
  const double drop = prob_.solver.mgs_drop_tol;
  spe_alloc((int)history_.size());
  spe_k_ = 0;
  bool all_kept = true;
  for (double* cand : history_) {
    const double norm0 = std::sqrt(dot_own(cand, cand, S_NORM));
    if (norm0 == 0.0) {
      all_kept = false;
      continue;
    }
    const int m = spe_k_;
    double* w = spe_q(spe_set_, m);
    CK(cudaMemcpyAsync(w, cand, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    bool keep = true;
    for (int pass = 0; pass < 2 && keep; ++pass) {
      for (int u = 0; u < m; ++u) {  // modified Gram-Schmidt, sequential projections
        launch_dot(n, spe_q(spe_set_, u), w, red_, S_DOT, stream_);
        allreduce(S_DOT);
        launch_axpy_dev(n, red_scal_.p + S_DOT, -1.0, spe_q(spe_set_, u), w, stream_);
      }
      const double nrm = std::sqrt(dot_own(w, w, S_NORM));
      if (nrm <= drop * norm0) keep = false;
      else if (pass == 1) launch_scale(n, 1.0 / nrm, w, w, stream_);
    }
    if (!keep) {
      all_kept = false;
      continue;
    }
    mass_apply_dev(w, spe_w(spe_set_, m));
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
      allreduce(S_MDOT, k);
      double col[kMaxMulti];
      read_scalars(S_MDOT, k, col);
      for (int i = 0; i <= j; ++i) spe_R_[(size_t)i * kMaxWin + j] = col[i];
      ++j;
    }
  }
}

// append h (newest) with two classical Gram-Schmidt passes and the MGS drop test
// Append h to the basis: the device runs both Gram-Schmidt passes (the
// coefficients go from the multi-dot slots straight into the update), the
// normalisation, W_m = M q_m and the new G column back to back; the host reads
// all their scalars once and replays the reference's drop decisions
// (start_vector.cpp:10-28) on them. A dropped vector only leaves scratch in
// the unused slot m, so the committed state equals the step-by-step version.
void GpuSystem::spe_append(double* h) {
  const int n = n_own_;
  const double drop = prob_.solver.mgs_drop_tol;
  const int m = spe_k_;
  double* w = spe_q(spe_set_, m);
  launch_dot(n, h, h, red_, S_APP, stream_);
  allreduce(S_APP);
  CK(cudaMemcpyAsync(w, h, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
  std::vector<const double*> Q(m);
  for (int i = 0; i < m; ++i) Q[i] = spe_q(spe_set_, i);
  if (m > 0)
    for (int pass = 0; pass < 2; ++pass) {
      const int cs = S_APP_C + pass * kMaxMulti;
      launch_multi_dot(n, m, Q.data(), w, red_, cs, stream_);
      allreduce(cs, m);
      launch_orth_update_dev(n, m, Q.data(), red_scal_.p + cs, w, red_, S_APP_NRM + pass, stream_);
      allreduce(S_APP_NRM + pass);
    }
  launch_scale_rsqrt(n, red_scal_.p + (m > 0 ? S_APP_NRM + 1 : S_APP), w, w, stream_);
  double* wm = spe_w(spe_set_, m);
  mass_apply_dev(w, wm);
  Q.push_back(w);
  launch_multi_dot(n, m + 1, Q.data(), wm, red_, S_APP_G, stream_);
  allreduce(S_APP_G, m + 1);
  double sc[S_COUNT - S_APP];
  read_scalars(S_APP, S_COUNT - S_APP, sc);
  const double norm0 = std::sqrt(sc[0]);
  if (norm0 == 0.0) {
    spe_clean_ = false;
    return;
  }
  std::vector<double> r(m + 1, 0.0);
  double nrm = norm0;
  for (int pass = 0; pass < 2; ++pass) {
    if (m > 0) {
      for (int i = 0; i < m; ++i) r[i] += sc[S_APP_C - S_APP + pass * kMaxMulti + i];
      nrm = std::sqrt(sc[S_APP_NRM - S_APP + pass]);
    }
    if (nrm <= drop * norm0) {
      spe_clean_ = false;
      return;
    }
  }
  r[m] = nrm;
  for (int i = 0; i <= m; ++i) spe_R_[(size_t)i * kMaxWin + m] = r[i];
  spe_k_ = m + 1;
  spe_G_.resize((size_t)kMaxMulti * kMaxMulti);
  for (int i = 0; i <= m; ++i)
    spe_G_[(size_t)i * kMaxMulti + m] = spe_G_[(size_t)m * kMaxMulti + i] = sc[S_APP_G - S_APP + i];
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
  // W = M Q is only read for the newest column (spe_g_column right after its
  // SpMV), and G is rotated below on the host, so W is not rotated
  std::vector<const double*> qi(k);
  std::vector<double*> qo(k - 1);
  for (int i = 0; i < k; ++i) qi[i] = spe_q(spe_set_, i);
  for (int j = 0; j + 1 < k; ++j) qo[j] = spe_q(1 - spe_set_, j);
  launch_lincomb_multi(n_own_, k, k - 1, qi.data(), qo.data(), T, stream_);
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


// ------------------------------------------------------------------ POD estimators
// proj/src/start_vector.cpp:64-71 (pod_build), 111-131 (pod_start), 133-150
// (factor_reduced, rolling_threshold), 165-183 (feedback). The reference runs
// Eigen::JacobiSVD on the n x k snapshot matrix S. Here S = Q R is first
// factored on the device (classical Gram-Schmidt, two passes), then the small
// k-column R goes through a one-sided Jacobi SVD on the host: R V = U_R Sigma
// gives S V = (Q U_R) Sigma, i.e. the same rotations applied to S, so the
// singular values and left singular vectors are those of S. Only the basis
// U = Q U_R[:, :keep] (keep <= rank, sigma > 1e-12 sigma_0) is formed on the
// device, followed by W = M U and the reduced inverse (U'MU)^-1.
namespace {
// One-sided Jacobi on the columns of R (m rows, k columns, column-major):
// returns sigma (descending) and the matching normalised left singular
// vectors (m each).
void jacobi_svd_left(int m, int k, std::vector<double> R, std::vector<double>& sigma,
                     std::vector<std::vector<double>>& u) {
  auto col = [&](int j) { return R.data() + (size_t)j * m; };
  auto dotc = [&](int a, int b) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += col(a)[i] * col(b)[i];
    return s;
  };
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < k; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double al = dotc(p, p), be = dotc(q, q), ga = dotc(p, q);
        if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        double *x = col(p), *y = col(q);
        for (int i = 0; i < m; ++i) {
          const double a = x[i], b = y[i];
          x[i] = c * a - sn * b;
          y[i] = sn * a + c * b;
        }
      }
    if (!rotated) break;
  }
  std::vector<std::pair<double, int>> sv(k);
  for (int j = 0; j < k; ++j) sv[j] = {std::sqrt(dotc(j, j)), j};
  std::stable_sort(sv.begin(), sv.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
  sigma.assign(k, 0.0);
  u.assign(k, std::vector<double>(m, 0.0));
  for (int j = 0; j < k; ++j) {
    sigma[j] = sv[j].first;
    if (sv[j].first > 0.0)
      for (int i = 0; i < m; ++i) u[j][i] = col(sv[j].second)[i] / sv[j].first;
  }
}
}  // namespace

DevBuf<double>* GpuSystem::pod_buf(std::vector<std::unique_ptr<DevBuf<double>>>& v, int j) {
  while ((int)v.size() <= j) {
    v.push_back(std::make_unique<DevBuf<double>>());
    v.back()->alloc(std::max(1, n_loc_));
  }
  return v[j].get();
}

// out[k] = V_k . w for k < m (chunks of kMaxMulti), allreduced
void GpuSystem::multi_dot_chunked(int m, const double* const* V, const double* w, double* out) {
  for (int c0 = 0; c0 < m; c0 += kMaxMulti) {
    const int mc = std::min<int>(kMaxMulti, m - c0);
    launch_multi_dot(n_own_, mc, V + c0, w, red_, S_MDOT, stream_);
    allreduce(S_MDOT, mc);
    read_scalars(S_MDOT, mc, out + c0);
  }
}

// y = sum_k c[k] V_k (chunks of kMaxMulti)
void GpuSystem::lincomb_chunked(int m, const double* const* V, const double* c, double* y) {
  if (m == 0) {
    launch_fill(n_own_, 0.0, y, stream_);
    return;
  }
  for (int c0 = 0; c0 < m; c0 += kMaxMulti) {
    const int mc = std::min<int>(kMaxMulti, m - c0);
    CoefPack cp{};
    for (int i = 0; i < mc; ++i) cp.c[i] = c[c0 + i];
    if (c0 == 0) launch_lincomb(n_own_, mc, V + c0, cp, y, stream_);
    else launch_lincomb_acc(n_own_, mc, V + c0, cp, y, stream_);
  }
}

void GpuSystem::pod_build_dev() {
  const int n = n_own_;
  const int k = pod_nsnap_;
  const int rank = prob_.solver.pod_rank;
  // thin QR of S by classical Gram-Schmidt with re-orthogonalisation; R is m x k
  std::vector<double> R;  // column-major, leading dimension k (m <= k)
  R.assign((size_t)k * k, 0.0);
  int m = 0;
  std::vector<const double*> Q;
  std::vector<double> c(k), r(k);
  for (int j = 0; j < k; ++j) {
    const double* s = pod_snap_[j]->p;
    const double norm0 = std::sqrt(dot_own(s, s, S_NORM));
    if (norm0 == 0.0) continue;  // zero column: R(:, j) = 0
    double* w = pod_buf(pod_q_, m)->p;
    CK(cudaMemcpyAsync(w, s, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    std::fill(r.begin(), r.end(), 0.0);
    double nrm = norm0;
    for (int pass = 0; pass < 2 && m > 0; ++pass) {
      multi_dot_chunked(m, Q.data(), w, c.data());
      for (int c0 = 0; c0 < m; c0 += kMaxMulti) {
        const int mc = std::min<int>(kMaxMulti, m - c0);
        CoefPack cp{};
        for (int i = 0; i < mc; ++i) {
          cp.c[i] = c[c0 + i];
          r[c0 + i] += c[c0 + i];
        }
        launch_orth_update(n, mc, Q.data() + c0, cp, w, red_, S_NORM, stream_);
      }
      allreduce(S_NORM);
      nrm = std::sqrt(read_scalar(S_NORM));
    }
    for (int i = 0; i < m; ++i) R[(size_t)j * k + i] = r[i];
    // residual at the rounding level of S: a numerically dependent column
    // (its singular-value contribution is below the 1e-12 sigma_0 cut)
    if (nrm <= 1e-13 * norm0) continue;
    launch_scale(n, 1.0 / nrm, w, w, stream_);
    R[(size_t)j * k + m] = nrm;
    Q.push_back(w);
    ++m;
  }
  // small SVD of R (m x k) on the host
  std::vector<double> Rm((size_t)m * k);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < m; ++i) Rm[(size_t)j * m + i] = R[(size_t)j * k + i];
  std::vector<double> sigma;
  std::vector<std::vector<double>> ur;
  if (m > 0) jacobi_svd_left(m, k, Rm, sigma, ur);
  int keep = 0;
  if (m > 0 && sigma[0] > 0.0)
    while (keep < k && keep < rank && sigma[keep] > 1e-12 * sigma[0]) ++keep;
  for (int b = 0; b < keep; ++b) lincomb_chunked(m, Q.data(), ur[b].data(), pod_buf(pod_u_, b)->p);
  pod_rank_ = keep;
}

void GpuSystem::pod_factor() {
  const int r = pod_rank_;
  pod_ok_ = r > 0;
  if (!pod_ok_) return;  // empty-basis signal, zero start without noise
  std::vector<const double*> U(r);
  for (int a = 0; a < r; ++a) {
    U[a] = pod_u_[a]->p;
    mass_apply_dev(pod_u_[a]->p, pod_buf(pod_w_, a)->p);
  }
  std::vector<double> g((size_t)r * r), col(r);
  for (int b = 0; b < r; ++b) {
    multi_dot_chunked(r, U.data(), pod_w_[b]->p, col.data());
    for (int a = 0; a < r; ++a) g[(size_t)a * r + b] = col[a];
  }
  DenseLdlt ldlt;
  ldlt.compute(g, r);
  double dmax = 0.0, dmin = INFINITY;
  for (double d : ldlt.d) {
    dmax = std::max(dmax, std::abs(d));
    dmin = std::min(dmin, d);
  }
  pod_ok_ = ldlt.ok && dmax > 0.0 && dmin > 1e-14 * dmax;
  if (!pod_ok_) {
    ++stats_.spe_fallbacks;
    std::fprintf(stderr, "start_vector: singular reduced system, zero start used\n");
    return;
  }
  pod_ginv_.assign((size_t)r * r, 0.0);
  std::vector<double> e(r);
  for (int c = 0; c < r; ++c) {
    std::fill(e.begin(), e.end(), 0.0);
    e[c] = 1.0;
    ldlt.solve(e.data(), col.data());
    for (int a = 0; a < r; ++a) pod_ginv_[(size_t)a * r + c] = col[a];
  }
}

double GpuSystem::pod_rolling_threshold() const {
  if (prob_.solver.pod_threshold > 0.0) return prob_.solver.pod_threshold;
  if (iteration_history_.empty()) return -1.0;  // always append while empty
  std::vector<int> h = iteration_history_;
  const size_t mid = h.size() / 2;
  std::nth_element(h.begin(), h.begin() + mid, h.end());
  return 1.25 * (double)h[mid];
}

bool GpuSystem::pod_start(const double* b, double* x0) {
  const int mode = prob_.solver.estimator_mode;
  if (mode == 3 && !pod_built_ && pod_nsnap_ >= prob_.solver.pod_snapshots) {
    pod_build_dev();
    ++stats_.svd_count;
    pod_built_ = true;
    pod_factor();
  }
  if (mode == 4 && pod_stale_ && pod_nsnap_ > 0) {
    pod_build_dev();
    ++stats_.svd_count;
    pod_stale_ = false;
    pod_factor();
  }
  estimator_rank_ = pod_rank_;
  const int r = pod_rank_;
  if (r == 0 || !pod_ok_) return false;
  std::vector<const double*> U(r);
  for (int a = 0; a < r; ++a) U[a] = pod_u_[a]->p;
  std::vector<double> vtb(r), y(r, 0.0);
  multi_dot_chunked(r, U.data(), b, vtb.data());
  for (int a = 0; a < r; ++a) {
    double s = 0.0;
    for (int c = 0; c < r; ++c) s += pod_ginv_[(size_t)a * r + c] * vtb[c];
    y[a] = s;
  }
  lincomb_chunked(r, U.data(), y.data(), x0);
  return true;
}

bool GpuSystem::estimator_next_dev(const double* b, double* x0, int* rank) {
  const bool nz = estimator_next(b, x0);
  if (!nz) launch_fill(n_own_, 0.0, x0, stream_);
  if (rank) *rank = prob_.solver.estimator_mode >= 2 ? estimator_rank_ : 0;
  return nz;
}

// StartVectorEstimator::next (proj/src/start_vector.cpp:84-109); writes the
// start vector into x0 and returns true when it is non-zero-by-construction.
bool GpuSystem::estimator_next(const double* b, double* x0) {
  const int n = n_own_;
  const int mode = prob_.solver.estimator_mode;
  if (mode == 0) return false;
  if (mode >= 3) {
    tic(TC_SPE);
    const bool nz = pod_start(b, x0);
    toc(TC_SPE, -1.0);
    return nz;
  }
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
    toc(TC_SPE, -1.0);
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
    toc(TC_SPE, -1.0);
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
  allreduce(S_MDOT, m);
  double vtb[kMaxMulti];
  read_scalars(S_MDOT, m, vtb);
  CoefPack y{};
  for (int r = 0; r < m; ++r) {
    double s = 0.0;
    for (int c = 0; c < m; ++c) s += ginv[(size_t)r * m + c] * vtb[c];
    y.c[r] = s;
  }
  launch_lincomb(n, m, V.data(), y, x0, stream_);
  toc(TC_SPE, -1.0);
  return true;
}

// StartVectorEstimator::feedback (proj/src/start_vector.cpp:152-164)
void GpuSystem::estimator_feedback(const double* x, int iterations) {
  const int mode = prob_.solver.estimator_mode;
  if (mode >= 3) {
    int slot = -1;
    if (mode == 3) {
      if (!pod_built_ && pod_nsnap_ < prob_.solver.pod_snapshots) slot = pod_nsnap_++;
    } else if ((double)iterations > pod_rolling_threshold()) {
      if (pod_nsnap_ < prob_.solver.pod_capacity) {
        slot = pod_nsnap_++;
      } else {
        slot = pod_next_slot_;  // overwrite the oldest
        pod_next_slot_ = (pod_next_slot_ + 1) % prob_.solver.pod_capacity;
      }
      pod_stale_ = true;
    }
    if (slot >= 0) {
      CK(cudaMemcpyAsync(pod_buf(pod_snap_, slot)->p, x, sizeof(double) * n_own_, cudaMemcpyDeviceToDevice,
                         stream_));
      ++stats_.appends;
    }
    iteration_history_.push_back(iterations);
    return;
  }
  iteration_history_.push_back(iterations);
  if (mode == 0) return;
  if (mode == 2) ++stats_.appends;
  const size_t window = mode == 1 ? 1 : (size_t)prob_.solver.spe_window;
  double* buf;
  if (history_.size() >= window) {
    buf = history_.front();
    history_.pop_front();
    if (mode == 2 && spe_clean_ && spe_incremental) spe_downdate();
  } else {
    hist_pool_.push_back(std::make_unique<DevBuf<double>>());
    hist_pool_.back()->alloc(std::max(1, n_loc_));
    buf = hist_pool_.back()->p;
  }
  CK(cudaMemcpyAsync(buf, x, sizeof(double) * n_own_, cudaMemcpyDeviceToDevice, stream_));
  history_.push_back(buf);
  // with the incremental basis switched off the window changed without the
  // basis following it: the next next() must rebuild
  if (mode == 2 && !spe_incremental) spe_clean_ = false;
  if (mode == 2 && spe_clean_ && spe_incremental) {
    if (window > (size_t)(kMaxWin - 1)) {
      spe_clean_ = false;  // large windows always use the full rebuild
    } else {
      tic(TC_SPE);
      spe_alloc((int)window);
      spe_append(buf);
      toc(TC_SPE, -1.0);
    }
  }
}

// FemSystem::eval_rhs (proj/src/fem_system.cpp:69-99)
PcgResult GpuSystem::eval_rhs_dev(double t, double* x_full, double* f) {
  double* b = w_free_a_.p;
  {
    PhaseTimer pt(stats_.t_residual, "residual");
    residual_dev(t, x_full, b);
  }
  bool has_x0;
  {
    PhaseTimer pt(stats_.t_estimator, "estimator");
    has_x0 = estimator_next(b, f);
  }
  PcgResult res;
  {
    PhaseTimer pt(stats_.t_solve, "solve");
    res = pcg_dev(b, has_x0 ? f : nullptr, f, prob_.solver.rel_tol, prob_.solver.max_iter);
  }
  if (!res.converged) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "mass solve failed to converge (relative residual %f)", res.rel_residual);
    throw NumericalError(buf);
  }
  {
    PhaseTimer pt(stats_.t_estimator, "estimator");
    estimator_feedback(f, res.iterations);
  }
  ++stats_.m_solves;
  stats_.pcg_iterations += res.iterations;
  records_.push_back({t, estimator_rank_, res.iterations, res.initial_rel_residual});
  return res;
}

// FemSystem::apply_minv_stiffness (proj/src/fem_system.cpp:103-122)
void GpuSystem::apply_minv_stiffness_dev(double t, double* x_full, const double* v_own, double* y) {
  double* vfull = w_full_b_.p;
  double* kv = w_free_b_.p;
  {
    PhaseTimer pt(stats_.t_residual, "residual");
    lift_dev(t, x_full);
    halo(halo0_, x_full);
    CK(cudaMemcpyAsync(vfull, v_own, sizeof(double) * n_own_, cudaMemcpyDeviceToDevice, stream_));
    halo(halo0_, vfull);
    launch_fill(n_fixloc_, 0.0, vfull + n_loc_, stream_);
    tic(TC_STIFF);
    if (stiffness_mode == 1) {
      kx_apply_full_dev(x_full, vfull, w_full_a_.p);
      CK(cudaMemcpyAsync(kv, w_full_a_.p, sizeof(double) * n_own_, cudaMemcpyDeviceToDevice, stream_));
    } else {
      kx_into(x_full, vfull, nullptr, 1.0, kv, n_own_);
    }
    toc(TC_STIFF, kx_bytes());
    check_kernel_flags();
  }
  PhaseTimer pt(stats_.t_solve, "solve");
  PcgResult res = pcg_dev(kv, nullptr, y, prob_.solver.rho_solve_tol, prob_.solver.max_iter);
  ++stats_.rho_solves;
  stats_.rho_pcg_iterations += res.iterations;
}

// estimate_spectral_radius (proj/src/integrators.cpp:49-75); the start vector
// is generated in global free order, each rank keeps its owned entries
double GpuSystem::estimate_spectral_radius(double t, double* x_full) {
  const int n = n_free_;
  const std::vector<int>& own = plan_.space[0].owned;
  for (int restart = 0; restart < 4; ++restart) {
    std::mt19937 rng(7919u + 31u * (unsigned)restart);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::vector<double> v(n);
    for (int i = 0; i < n; ++i) v[i] = uni(rng);
    double nrm = 0.0;
    for (double e : v) nrm += e * e;
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) continue;
    std::vector<double> vo(std::max(1, n_own_));
    for (int i = 0; i < n_own_; ++i) vo[i] = v[own[i]] / nrm;
    rho_v_.upload(vo.data(), n_own_, stream_);
    double rho = 0.0;
    bool annihilated = false;
    for (int it = 0; it < 15; ++it) {
      apply_minv_stiffness_dev(t, x_full, rho_v_.p, rho_w_.p);
      rho = std::sqrt(dot_own(rho_w_.p, rho_w_.p, S_NORM));
      if (rho == 0.0) {
        annihilated = true;
        break;
      }
      launch_scale(n_own_, 1.0 / rho, rho_w_.p, rho_v_.p, stream_);
    }
    if (!annihilated) return 1.2 * rho;
  }
  return 0.0;
}

// ------------------------------------------------------------------ host wrappers (single rank)
void GpuSystem::kx_apply_host(const double* x_state, const double* v, double* y) {
  require_single("kx_apply");
  std::vector<double> xd(n_full_), vd(n_full_), yd(n_full_);
  for (int k = 0; k < n_full_; ++k) {
    xd[k] = x_state[loc2ref_[k]];
    vd[k] = v[loc2ref_[k]];
  }
  w_full_a_.upload(xd.data(), n_full_, stream_);
  w_full_b_.upload(vd.data(), n_full_, stream_);
  double* out = scratch_full();
  kx_apply_full_dev(w_full_a_.p, w_full_b_.p, out);
  CK(cudaMemcpyAsync(yd.data(), out, sizeof(double) * n_full_, cudaMemcpyDeviceToHost, stream_));
  check_kernel_flags();
  std::fill(y, y + n_dofs_, 0.0);  // dofs in no tet
  for (int k = 0; k < n_full_; ++k) y[loc2ref_[k]] = yd[k];
}

// MatFreeStiffness::residual (matfree.cpp:138-143)
void GpuSystem::kx_residual_host(const double* x_full, const double* b_mass, double* r) {
  require_single("kx_residual");
  std::vector<double> xd(n_full_);
  for (int k = 0; k < n_full_; ++k) xd[k] = x_full[loc2ref_[k]];
  w_full_a_.upload(xd.data(), n_full_, stream_);
  w_free_a_.upload(b_mass, n_own_, stream_);
  tic(TC_STIFF);
  if (stiffness_mode == 1) {
    kx_apply_full_dev(w_full_a_.p, w_full_a_.p, w_full_b_.p);
    launch_axpby_into(n_own_, w_free_a_.p, -1.0, w_full_b_.p, w_free_b_.p, stream_);
  } else {
    kx_into(w_full_a_.p, w_full_a_.p, w_free_a_.p, -1.0, w_free_b_.p, n_own_);
  }
  toc(TC_STIFF, kx_bytes());
  w_free_b_.download(r, n_own_, stream_);
  check_kernel_flags();
}

void GpuSystem::eval_residual_host(double t, const double* x, double* r) {
  require_single("eval_residual");
  PhaseTimer pt(stats_.t_residual, "residual");
  double* xf = w_full_b_.p;
  CK(cudaMemcpyAsync(xf, x, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  residual_dev(t, xf, w_free_b_.p);
  w_free_b_.download(r, n_own_, stream_);
  sync();
}

PcgResult GpuSystem::eval_rhs_host(double t, const double* x, double* f) {
  require_single("eval_rhs");
  double* xf = w_full_b_.p;
  CK(cudaMemcpyAsync(xf, x, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  PcgResult r = eval_rhs_dev(t, xf, F_.p);
  F_.download(f, n_own_, stream_);
  sync();
  return r;
}

PcgResult GpuSystem::mass_solve_host(const double* b, const double* x0, double tol, int max_iter, double* x) {
  require_single("mass_solve");
  F0_.upload(b, n_own_, stream_);
  if (x0) Fn_.upload(x0, n_own_, stream_);
  PhaseTimer pt(stats_.t_solve, "solve");
  PcgResult r = pcg_dev(F0_.p, x0 ? Fn_.p : nullptr, F_.p, tol, max_iter);
  F_.download(x, n_own_, stream_);
  sync();
  return r;
}

// StartVectorEstimator::next / feedback with host vectors (start_vector.hpp:52-58)
int GpuSystem::estimator_next_host(const double* b, double* x0) {
  require_single("estimator_next");
  F0_.upload(b, n_own_, stream_);
  int rank = 0;
  {
    PhaseTimer pt(stats_.t_estimator, "estimator");
    estimator_next_dev(F0_.p, F_.p, &rank);
  }
  F_.download(x0, n_own_, stream_);
  sync();
  return rank;
}
void GpuSystem::estimator_feedback_host(const double* x, int iterations) {
  require_single("estimator_feedback");
  F_.upload(x, n_own_, stream_);
  PhaseTimer pt(stats_.t_estimator, "estimator");
  estimator_feedback(F_.p, iterations);
  sync();
}

// Config-5 MRHS microbenchmark: k right-hand sides solved in
// sequence on the device with the configured start-vector estimator (the
// eval_rhs solve path without K(x)x). B and X are host [k][n_free]; X may be
// null. Returns the device time of the k solves (CUDA events, inputs resident).
double GpuSystem::mass_solve_sequence(const double* B, int k, double tol, int max_iter, double* X, int* its) {
  require_single("mass_solve_sequence");
  const size_t n = (size_t)n_own_;
  DevBuf<double> Bd, Xd;
  Bd.alloc(std::max<size_t>(1, n * k));
  Xd.alloc(std::max<size_t>(1, n * k));
  Bd.upload(B, n * k, stream_);
  sync();
  cudaEvent_t e0 = get_event(), e1 = get_event();
  CK(cudaEventRecord(e0, stream_));
  for (int j = 0; j < k; ++j) {
    const double* b = Bd.p + n * j;
    double* x = Xd.p + n * j;
    const bool has_x0 = estimator_next(b, x);
    const PcgResult r = pcg_dev(b, has_x0 ? x : nullptr, x, tol, max_iter);
    if (!r.converged) throw NumericalError("mass_solve_sequence: PCG did not converge");
    estimator_feedback(x, r.iterations);
    if (its) its[j] = r.iterations;
  }
  CK(cudaEventRecord(e1, stream_));
  sync();
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  if (X) Xd.download(X, n * k, stream_);
  sync();
  return ms;
}

void GpuSystem::reset_estimator(int mode) {
  if (mode < 0 || mode > 4)
    throw std::invalid_argument("estimator mode must be 0 (zero), 1 (previous), 2 (spe), 3 (pod_fixed) or 4 (pod_rolling)");
  prob_.solver.estimator_mode = mode;
  history_.clear();
  hist_pool_.clear();
  spe_clean_ = false;
  pod_nsnap_ = pod_next_slot_ = pod_rank_ = 0;  // POD buffers stay allocated for the next run
  pod_stale_ = pod_built_ = pod_ok_ = false;
  iteration_history_.clear();
  estimator_rank_ = 0;
}

void GpuSystem::mass_apply_host(const double* v, double* y) {
  require_single("mass_apply");
  F0_.upload(v, n_own_, stream_);
  mass_apply_dev(F0_.p, F_.p);
  F_.download(y, n_own_, stream_);
  sync();
}

void GpuSystem::apply_minv_stiffness_host(double t, const double* x_state, const double* v, double* y) {
  require_single("apply_minv_stiffness");
  double* xf = scratch_full();
  CK(cudaMemcpyAsync(xf, x_state, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  F0_.upload(v, n_own_, stream_);
  apply_minv_stiffness_dev(t, xf, F0_.p, F_.p);
  F_.download(y, n_own_, stream_);
  sync();
}

void GpuSystem::lift_full_host(double t, const double* x_free, double* x_full) {
  std::vector<double> b = set_values(t, false);
  for (int i = 0; i < n_free_; ++i) x_full[prob_.dm.free_dofs[i]] = x_free[i];
  for (int i = 0; i < n_fixed_; ++i) x_full[prob_.dm.fixed_dofs[i]] = b[prob_.dm.fixed_set[prob_.dm.fixed_dofs[i]]];
}

// ------------------------------------------------------------------ integrators
void GpuSystem::set_state(double t, const double* x_own, double dt) {
  state_t = t;
  state_dt = dt;
  CK(cudaMemcpyAsync(X_, x_own, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  sync();
  rho_valid = false;
  rho_age = 0;
}
void GpuSystem::get_state(double* x_own) {
  CK(cudaMemcpyAsync(x_own, X_, sizeof(double) * n_own_, cudaMemcpyDeviceToHost, stream_));
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

// rkc_stages (proj/src/integrators.cpp:156-173) on the owned entries. Returns the buffer holding Y_s.
static double* rkc_stages(GpuSystem& g, double t, double dt, const RkcCoefficients& k, double* X, double* bufs[3],
                          double* f0, double* f) {
  const int n = g.n_own();
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
  NvtxRange nv("rkc_step");
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
    launch_rkc_error(n_own_, X_, x_new, F0_.p, Fn_.p, dt, o.atol, o.rtol, red_, S_ERR, stream_);
    allreduce(S_ERR);
    toc(TC_RKC, 32.0 * n_own_);
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
  NvtxRange nv("rkc_step");
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
  launch_axpy(n_own_, dt, F_.p, X_, stream_);
  toc(TC_RKC, 24.0 * n_own_);
  state_t += dt;
  ++st_accepted;
  ++st_stages;
  att.accepted = true;
  att.stages = 1;
  att.dt_next = dt;
  return att;
}


// ------------------------------------------------------------------ SDIRK3(2)
// proj/src/integrators.cpp:237-343 and FemSystem::shifted_solve
// (proj/src/fem_system.cpp:124-145). The Newton matrix M_II + gamma dt K_II(z)
// is assembled on the device every Newton iteration: per-tet element matrices
// (k_kelem, the reference's element arithmetic), then one thread per M_II
// entry sums its contributions in ascending tet order (assemble_matrix order)
// and forms 1.0 m + gdt k (csr.cpp add on the common pattern). Deviation
// (DESIGN.md §4): the shifted system is preconditioned with Jacobi (diagonal
// of the matrix at the last refresh) instead of rebuilding the AMG hierarchy
// every step; the PCG stopping rule is the reference's, so each Newton update
// is the same to the solver tolerance.
double* GpuSystem::sd(int i) {
  if (!sd_buf_[i].p) sd_buf_[i].alloc(std::max(1, n_full_));
  return sd_buf_[i].p;
}

void GpuSystem::build_shift_map() {
  if (shift_built_) return;
  require_single("sdirk");
  const int nl = order_ == 1 ? 4 : 10, ntri = nl * (nl + 1) / 2;
  const std::vector<int>& td = tet_dofs_host();
  const LocalSpace& s0 = plan_.space[0];
  const HostCsr& m = m_ii_;
  auto entry = [&](int li, int lj) -> long {  // local free dofs -> M_II entry
    const int r = s0.owned[li], c = s0.owned[lj];
    const int* b = m.col_idx.data() + m.row_ptr[r];
    const int* e = m.col_idx.data() + m.row_ptr[r + 1];
    const int* f = std::lower_bound(b, e, c);
    if (f == e || *f != c) throw NumericalError("sdirk: element pair outside the M_II pattern");
    return (long)(f - m.col_idx.data());
  };
  std::vector<int> order(n_tets_loc_);
  for (int k = 0; k < n_tets_loc_; ++k) order[k] = k;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return plan_.tets[a] < plan_.tets[b]; });
  const long nnz = m.nnz();
  std::vector<long> ptr(nnz + 1, 0);
  for (int k : order)
    for (int a = 0; a < nl; ++a)
      for (int b = 0; b < nl; ++b) {
        const int ra = td[(size_t)k * nl + a], cb = td[(size_t)k * nl + b];
        if (ra < n_own_ && cb < n_own_) ++ptr[entry(ra, cb) + 1];
      }
  for (long e = 0; e < nnz; ++e) ptr[e + 1] += ptr[e];
  std::vector<long> src(ptr[nnz]), next(ptr.begin(), ptr.end() - 1);
  for (int k : order)
    for (int a = 0; a < nl; ++a)
      for (int b = 0; b < nl; ++b) {
        const int ra = td[(size_t)k * nl + a], cb = td[(size_t)k * nl + b];
        if (ra < n_own_ && cb < n_own_) src[next[entry(ra, cb)]++] = (long)k * ntri + tri_index(a, b);
      }
  sh_ptr_.alloc(nnz + 1);
  sh_ptr_.upload(ptr.data(), ptr.size(), stream_);
  sh_src_.alloc(std::max<size_t>(1, src.size()));
  sh_src_.upload(src.data(), src.size(), stream_);
  sh_S_.alloc(std::max<long>(1, (long)n_tets_loc_ * ntri));
  sh_vals_.alloc(std::max<long>(1, nnz));
  sh_diag_.alloc(std::max(1, n_own_));
  sh_err_.alloc(1);
  CK(cudaMemsetAsync(sh_err_.p, 0, sizeof(int), stream_));
  sh_csr_ = DevCsr{};
  sh_csr_.n_rows = mii_.n_rows;
  sh_csr_.n_cols = mii_.n_cols;
  sh_csr_.nnz = nnz;
  sh_csr_.row_ptr = mii_rp_.p;
  sh_csr_.col_idx = mii_ci_.p;
  sh_csr_.values = sh_vals_.p;
  sh_csr_.tpr = mii_.tpr;
  sync();
  shift_built_ = true;
}

// SA-AMG of the shifted matrix M_II + gdt K_II(z) (make_preconditioner,
// proj/src/fem_system.cpp:38-46 -> AmgPreconditioner, proj/src/amg.cpp:90-143),
// rebuilt on the device at every refresh: strength graph, greedy aggregation,
// P_tent, lambda_max, P = (I - omega/lambda D^-1 A) P_tent, R = P^T and
// R (A P) with the k_amgsetup.cu / k_spgemm.cu kernels (bit-identical to the
// host algorithm), the coarsest level (<= amg_coarse_limit rows) as an explicit
// inverse of its pivoted LDLT. Nothing leaves the device but the coarsest
// matrix. The V-cycle is vcycle_t<double> over fp64 CSR levels with the
// Chebyshev smoothers of the mass V-cycle.

void GpuSystem::build_shift_amg() {
  if (!sh_amg_) {
    sh_amg_ = std::make_unique<ShiftAmg>();
    sh_amg_->sd.init(device_);
  }
  ShiftAmg& S = *sh_amg_;
  cudaStream_t s = S.sd.stream();
  CK(cudaStreamSynchronize(stream_));  // the shifted values were written on the context stream
  static const bool trace = getenv("EQS_MEMTRACE") != nullptr;
  auto T0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[shift-amg] %-12s %.4f s\n", what, std::chrono::duration<double>(now - T0).count());
    T0 = now;
  };
  S.drop_graphs();  // the level buffers are reallocated below
  S.vals32.clear();
  S.levels.clear();
  S.A.clear();
  S.P.clear();
  S.R.clear();
  const SolverParams& sp = prob_.solver;
  const long long batch = 1ll << 28;
  {
    S.A.emplace_back();
    DCsr& a0 = S.A.back();
    a0.rows = a0.cols = sh_csr_.n_rows;
    a0.nnz = sh_csr_.nnz;
    a0.rp.alloc(a0.rows + 1);
    a0.ci.alloc(std::max<long long>(1, a0.nnz));
    a0.v.alloc(std::max<long long>(1, a0.nnz));
    CK(cudaMemcpyAsync(a0.rp.p, sh_csr_.row_ptr, sizeof(int) * (a0.rows + 1), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(a0.ci.p, sh_csr_.col_idx, sizeof(int) * a0.nnz, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(a0.v.p, sh_csr_.values, sizeof(double) * a0.nnz, cudaMemcpyDeviceToDevice, s));
  }
  dev_check_diagonal(S.A[0], s);
  lap("copy A0");
  std::vector<double> lam;
  while ((int)S.A.size() < sp.amg_max_levels && S.A.back().rows > sp.amg_coarse_limit) {
    const DCsr& a = S.A.back();
    DevBuf<double> d;
    dev_diagonal(a, d, s);
    DevBuf<int> agg;
    const int n_agg = dev_aggregate(a, d.p, sp.amg_theta, agg, s);
    lap("aggregate");
    if (n_agg >= a.rows) break;  // coarsening stalled (amg.cpp:102)
    DCsr pt, p, r, ap, c;
    dev_tentative(agg, a.rows, n_agg, pt, s);
    const double lm = dev_lambda_max(a, d.p, 10, 20240811u, s);
    lap("lambda");
    S.sd.multiply(a, pt, p, d.p, sp.amg_omega / lm, batch);
    dev_transpose(p, r, s);
    lap("P, R");
    S.sd.multiply(a, p, ap, nullptr, 0.0, batch);
    S.sd.multiply(r, ap, c, nullptr, 0.0, batch);
    dev_check_diagonal(c, s);
    lap("RAP");
    lam.push_back(lm);
    S.P.push_back(std::move(p));
    S.R.push_back(std::move(r));
    S.A.push_back(std::move(c));
  }
  // coarsest: explicit inverse of the pivoted LDLT (amg.cpp:138-141 + DESIGN.md §4.5)
  HostCsr hc;
  S.sd.download(S.A.back(), hc);
  const std::vector<double> inv = dense_inverse(hc);
  lap("coarse inv");
  S.coarse_n = hc.n_rows;
  S.inv.alloc(std::max<size_t>(1, inv.size()));
  S.inv.upload(inv.data(), inv.size(), s);
  {
    std::vector<float> f(inv.begin(), inv.end());
    S.inv32.alloc(std::max<size_t>(1, f.size()));
    S.inv32.upload(f.data(), f.size(), s);
  }
  const int L = (int)S.A.size();
  S.levels.resize(L);
  auto view = [](DCsr& m) {
    DevCsr v;
    v.n_rows = m.rows;
    v.n_cols = m.cols;
    v.nnz = m.nnz;
    v.row_ptr = m.rp.p;
    v.col_idx = m.ci.p;
    v.values = m.v.p;
    const double avg = m.rows ? (double)m.nnz / m.rows : 0.0;
    int t = 1;
    while (t < 32 && t * 8 < avg) t <<= 1;
    v.tpr = t;
    return v;
  };
  for (int l = 0; l < L; ++l) {
    DevLevel& lv = S.levels[l];
    const int n = S.A[l].rows;
    lv.n_own = lv.n_loc = lv.n_global = n;
    lv.A = view(S.A[l]);
    const size_t nb = std::max(1, n);
    lv.b.alloc(nb);
    lv.z.alloc(nb);
    lv.z2.alloc(nb);
    lv.t.alloc(nb);
    for (DevBuf<float>* v : {&lv.b32, &lv.z32, &lv.z2_32, &lv.t32, &lv.db32, &lv.dt32, &lv.invd32}) v->alloc(nb);
    auto f32 = [&](DCsr& m, DevCsr& v) {  // fp32 value copy read by the fp32 V-cycle (CSR kernels)
      S.vals32.emplace_back();
      S.vals32.back().alloc(std::max<long long>(1, m.nnz));
      launch_to_f32(m.nnz, m.v.p, S.vals32.back().p, s);
      v.values_f = S.vals32.back().p;
    };
    if (l + 1 < L) f32(S.A[l], lv.A);
    if (l + 1 < L) {
      lv.P = view(S.P[l]);
      lv.R = view(S.R[l]);
      f32(S.P[l], lv.P);
      f32(S.R[l], lv.R);
      DevBuf<double> d;
      dev_diagonal(S.A[l], d, s);
      lv.invd.alloc(nb);
      launch_recip(n, d.p, lv.invd.p, s);
      launch_to_f32(n, lv.invd.p, lv.invd32.p, s);
      CK(cudaStreamSynchronize(s));
      // smoother bound: the setup's 10-step lambda_max(D^-1 A) estimate (amg.cpp:28-45)
      lv.lambda_smoother = lam[l];
      cheb_first_kind(cheb_scale * lv.lambda_smoother, cheb_ratio, lv);
    }
  }
  CK(cudaStreamSynchronize(s));
  lap("levels");
  ++S.builds;
}

// Exchange the mass solve's operator, hierarchy and captured graphs with the
// shifted system's, so pcg_dev (graph-resident loop, fp32 V-cycle) solves
// the shifted system; called in pairs around the solve.
void GpuSystem::shift_swap() {
  ShiftAmg& S = *sh_amg_;
  std::swap(mii_, S.op);
  std::swap(levels_, S.levels);
  std::swap(coarse_n_, S.coarse_n);
  std::swap(coarse_inv_, S.inv);
  std::swap(coarse_inv32_, S.inv32);
  std::swap(vcycle_graph_, S.vgraph);
  std::swap(vcycle_out_, S.vout);
  std::swap(vcycle_graph_kernels_, S.vkern);
  std::swap(vcycle_graph_bytes_, S.vbytes);
  std::swap(pcg_graphs_, S.graphs);
  std::swap(pcg_graph_use_, S.graph_use);
  std::swap(pcg_graph_clock_, S.graph_clock);
  std::swap(pcg_body_kernels_, S.body_kernels);
  std::swap(pcg_body_bytes_, S.body_bytes);
}

// one V-cycle of the shifted hierarchy on r (fp64): z, and r.z in S_RZ
double* GpuSystem::shift_vcycle(const double* r) {
  ShiftAmg& S = *sh_amg_;
  std::swap(levels_, S.levels);
  std::swap(coarse_n_, S.coarse_n);
  std::swap(coarse_inv_, S.inv);
  std::swap(coarse_inv32_, S.inv32);
  double* z = nullptr;
  try {
    z = vcycle_t<double>(0, r, true, nullptr, nullptr, nullptr);
  } catch (...) {
    std::swap(levels_, S.levels);
    std::swap(coarse_n_, S.coarse_n);
    std::swap(coarse_inv_, S.inv);
    std::swap(coarse_inv32_, S.inv32);
    throw;
  }
  std::swap(levels_, S.levels);
  std::swap(coarse_n_, S.coarse_n);
  std::swap(coarse_inv_, S.inv);
  std::swap(coarse_inv32_, S.inv32);
  return z;
}

// the shifted operator as the PCG operator of pcg_dev (fp64 CSR on M_II's pattern)
void GpuSystem::S_op_view() {
  DevCsr& o = sh_amg_->op;
  o = sh_csr_;
  o.use_sell = false;
  o.prec = 0;
}

void GpuSystem::shifted_solve_dev(double t, double* z_full, double gdt, const double* rhs, double* delta,
                                  bool refresh) {
  build_shift_map();
  const int n = n_own_;
  {
    PhaseTimer pt(stats_.t_setup, "setup");
    lift_dev(t, z_full);
    launch_k_element(order_, n_tets_loc_, tet_dofs_.p, tet_mat_.p, coords_.p, z_full, sh_S_.p, sh_err_.p, stream_);
    ++stats_.assemblies;
    launch_shift_gather(sh_csr_.nnz, sh_ptr_.p, sh_src_.p, sh_S_.p, mii_v_.p, gdt, sh_vals_.p, stream_);
    if (refresh || !shift_precond_) {  // make_preconditioner (fem_system.cpp:38-46)
      launch_csr_diag(n, sh_csr_.row_ptr, sh_csr_.col_idx, sh_vals_.p, sh_diag_.p, stream_);
      shift_amg_on_ = shift_amg && prob_.solver.precond == 2;
      if (shift_amg_on_) build_shift_amg();
      ++stats_.precond_setups;
      shift_precond_ = true;
    }
  }
  PhaseTimer pt(stats_.t_solve, "solve");
  if (shift_amg_on_ && shift_pcg_graph) {
    // pcg_solve (proj/src/pcg.cpp:9-72) with a zero start through pcg_dev:
    // the graph-resident loop with the fp32 V-cycle of the shifted hierarchy
    S_op_view();
    shift_swap();
    PcgResult res;
    try {
      res = pcg_dev(rhs, nullptr, delta, prob_.solver.rel_tol, prob_.solver.max_iter);
    } catch (...) {
      shift_swap();
      throw;
    }
    shift_swap();
    if (!res.converged) throw NumericalError("shifted-system solve failed to converge");
    ++stats_.newton_linear_solves;
    stats_.newton_pcg_iterations += res.iterations;
    return;
  }
  // pcg_solve (proj/src/pcg.cpp:9-72) with a zero start
  double* x = delta;
  double* r = sd(12);
  double* z = sd(13);
  double* p = sd(14);
  double* q = sd(15);
  const double tol = prob_.solver.rel_tol;
  const int max_iter = prob_.solver.max_iter;
  const double bnorm = std::sqrt(dot_own(rhs, rhs, S_NORM));
  launch_fill(n, 0.0, x, stream_);
  if (bnorm == 0.0) {
    ++stats_.newton_linear_solves;
    return;
  }
  CK(cudaMemcpyAsync(r, rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
  double rel = 1.0;
  if (!std::isfinite(bnorm)) throw NumericalError("pcg: non-finite initial residual");
  if (rel <= tol) return;
  auto precond = [&]() {  // z = B r and r.z in S_RZ
    if (shift_amg_on_) {
      const double* zv = shift_vcycle(r);
      CK(cudaMemcpyAsync(z, zv, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    } else {
      launch_jacobi_div(n, sh_diag_.p, r, z, red_, S_RZ, stream_);
    }
  };
  precond();
  double rz = read_scalar(S_RZ);
  if (!std::isfinite(rz)) throw NumericalError("pcg: non-finite preconditioned residual");
  CK(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
  int k = 1;
  bool converged = false;
  for (; k <= max_iter; ++k) {
    launch_spmv(sh_csr_, p, q, stream_);
    const double pq = dot_own(p, q, S_PQ);
    if (!(pq > 0.0) || !std::isfinite(pq)) throw NumericalError("pcg: operator not positive definite");
    const double alpha = rz / pq;
    launch_axpy(n, alpha, p, x, stream_);
    launch_axpy(n, -alpha, q, r, stream_);
    rel = std::sqrt(dot_own(r, r, S_RR)) / bnorm;
    if (!std::isfinite(rel)) throw NumericalError("pcg: non-finite residual");
    if (rel <= tol) {
      converged = true;
      break;
    }
    precond();
    const double rz_new = read_scalar(S_RZ);
    if (!std::isfinite(rz_new)) throw NumericalError("pcg: non-finite preconditioned residual");
    launch_scale(n, rz_new / rz, p, p, stream_);
    launch_axpy(n, 1.0, z, p, stream_);
    rz = rz_new;
  }
  if (!converged) throw NumericalError("shifted-system solve failed to converge");
  ++stats_.newton_linear_solves;
  stats_.newton_pcg_iterations += k;
}

void GpuSystem::cell_kappa_host(double* kappa) {
  require_single("cell_kappa");
  double* xf = sd(11);
  CK(cudaMemcpyAsync(xf, X_, sizeof(double) * n_own_, cudaMemcpyDeviceToDevice, stream_));
  lift_dev(state_t, xf);
  DevBuf<double> kd;
  kd.alloc(std::max(1, n_tets_loc_));
  launch_cell_kappa(order_, n_tets_loc_, tet_dofs_.p, tet_mat_.p, coords_.p, xf, kd.p, stream_);
  std::vector<double> loc(n_tets_loc_);
  kd.download(loc.data(), loc.size(), stream_);
  sync();
  for (int k = 0; k < n_tets_loc_; ++k) kappa[plan_.tets[k]] = loc[k];
}

void GpuSystem::shifted_solve_host(double t, const double* z, double gdt, const double* rhs, double* delta,
                                   bool refresh) {
  require_single("shifted_solve");
  double* zf = sd(11);
  double* b = sd(10);
  double* d = sd(6);
  CK(cudaMemcpyAsync(zf, z, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  CK(cudaMemcpyAsync(b, rhs, sizeof(double) * n_own_, cudaMemcpyHostToDevice, stream_));
  shifted_solve_dev(t, zf, gdt, b, d, refresh);
  CK(cudaMemcpyAsync(delta, d, sizeof(double) * n_own_, cudaMemcpyDeviceToHost, stream_));
  sync();
}

namespace {
constexpr double kSdG = 0.435866521508459;
constexpr double kSdC[3] = {kSdG, (1.0 + kSdG) / 2.0, 1.0};
constexpr double kSdB1 = -1.5 * kSdG * kSdG + 4.0 * kSdG - 0.25;
constexpr double kSdB2 = 1.5 * kSdG * kSdG - 5.0 * kSdG + 1.25;
constexpr double kSdA[3][3] = {{kSdG, 0.0, 0.0}, {(1.0 - kSdG) / 2.0, kSdG, 0.0}, {kSdB1, kSdB2, kSdG}};
constexpr double kSdBh1 = kSdG / (1.0 - kSdG);
constexpr double kSdBh2 = 1.0 - kSdBh1;
}  // namespace

// sdirk_stages (integrators.cpp:256-292); the new state is left in sd(1), the
// error estimate in est (may be null)
bool GpuSystem::sdirk_stages(double dt, const SdirkOptions& o, int& newton_iters, double* est) {
  require_single("sdirk");
  const int n = n_own_;
  const double t = state_t, gdt = kSdG * dt;
  double *w = sd(0), *z = sd(1), *zw = sd(2), *r = sd(3), *mz = sd(4), *g = sd(5), *delta = sd(6);
  double* kk[3] = {sd(7), sd(8), sd(9)};
  newton_iters = 0;
  for (int stage = 0; stage < 3; ++stage) {
    CK(cudaMemcpyAsync(w, X_, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    for (int j = 0; j < stage; ++j) launch_axpy(n, dt * kSdA[stage][j], kk[j], w, stream_);
    const double ts = t + kSdC[stage] * dt;
    CK(cudaMemcpyAsync(z, w, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    double scale = -1.0;
    bool converged = false;
    for (int it = 0;; ++it) {
      {
        PhaseTimer pt(stats_.t_residual, "residual");
        residual_dev(ts, z, r);
      }
      CK(cudaMemcpyAsync(zw, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
      launch_axpy(n, -1.0, w, zw, stream_);
      mass_apply_dev(zw, mz);
      CK(cudaMemcpyAsync(g, mz, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
      launch_axpy(n, -gdt, r, g, stream_);
      const double gn = std::sqrt(dot_own(g, g, S_NORM));
      if (!std::isfinite(gn)) return false;
      if (scale < 0.0) scale = gn;
      if (gn <= o.newton_tol * scale || gn == 0.0) {
        converged = true;
        break;
      }
      if (it >= o.max_newton) break;
      launch_scale(n, -1.0, g, g, stream_);
      try {
        shifted_solve_dev(ts, z, gdt, g, delta, stage == 0 && it == 0);
      } catch (const NumericalError&) {
        return false;
      }
      launch_axpy(n, 1.0, delta, z, stream_);
      ++newton_iters;
    }
    if (!converged) return false;
    CK(cudaMemcpyAsync(kk[stage], z, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    launch_axpy(n, -1.0, w, kk[stage], stream_);
    launch_scale(n, 1.0 / gdt, kk[stage], kk[stage], stream_);
  }
  if (est) {
    CoefPack c{};
    c.c[0] = dt * (kSdA[2][0] - kSdBh1);
    c.c[1] = dt * (kSdA[2][1] - kSdBh2);
    c.c[2] = dt * kSdG;
    const double* V[3] = {kk[0], kk[1], kk[2]};
    launch_lincomb(n, 3, V, c, est, stream_);
  }
  return true;
}

// sdirk_step (integrators.cpp:297-327)
StepAttempt GpuSystem::sdirk_step(const SdirkOptions& o) {
  StepAttempt att;
  att.t_start = state_t;
  att.dt = state_dt;
  att.stages = 3;
  int newton_iters = 0;
  double* est = sd(10);
  const bool ok = sdirk_stages(state_dt, o, newton_iters, est);
  att.newton_iterations = newton_iters;
  st_newton += newton_iters;
  if (!ok) {
    att.accepted = false;
    att.dt_next = 0.5 * state_dt;
    ++st_rejected;
    state_dt = att.dt_next;
    return att;
  }
  const int n = n_own_;
  launch_weighted_sq(n, est, X_, sd(1), o.atol, o.rtol, red_, S_ERR, stream_);
  const double acc = read_scalar(S_ERR);
  att.error = n == 0 ? 0.0 : std::sqrt(acc / (double)n);
  // step_controller (integrators.cpp:12-18), order 3
  const double err = att.error;
  bool accept;
  double dt_next;
  if (!std::isfinite(err)) {
    accept = false;
    dt_next = 0.1 * state_dt;
  } else {
    accept = err <= 1.0;
    const double factor = err == 0.0 ? 10.0 : std::clamp(0.8 * std::pow(err, -1.0 / 4.0), 0.1, 10.0);
    dt_next = state_dt * factor;
  }
  att.accepted = accept;  // finite err implies finite x_new
  att.dt_next = dt_next;
  if (att.accepted) {
    CK(cudaMemcpyAsync(X_, sd(1), sizeof(double) * n, cudaMemcpyDeviceToDevice, stream_));
    state_t += state_dt;
    ++st_accepted;
  } else {
    ++st_rejected;
  }
  state_dt = dt_next;
  return att;
}

// sdirk_advance_fixed (integrators.cpp:329-341)
bool GpuSystem::sdirk_advance_fixed(double dt, const SdirkOptions& o) {
  int newton_iters = 0;
  if (!sdirk_stages(dt, o, newton_iters, nullptr)) return false;
  st_newton += newton_iters;
  CK(cudaMemcpyAsync(X_, sd(1), sizeof(double) * n_own_, cudaMemcpyDeviceToDevice, stream_));
  state_t += dt;
  ++st_accepted;
  return true;
}

}  // namespace eqsb
