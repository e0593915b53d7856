// extern "C" boundary (include/eqs_b200.h). Each entry point maps the
// reference exception taxonomy onto an int code and keeps the message for
// eqs_last_error(); the C++ shim in INTEGRATION.md rethrows the same classes.
#include <cuda_runtime.h>

#include <cstring>
#include <fcntl.h>
#include <semaphore.h>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "eqs_b200.h"
#include "gpu_system.hpp"
#include "scenario.hpp"

using namespace eqsb;

struct eqs_ctx {
  std::unique_ptr<GpuSystem> sys;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return EQS_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return EQS_ERR_CONFIG;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return EQS_ERR_NUMERICAL;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return EQS_ERR_GEOMETRY;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EQS_ERR_INVALID_ARGUMENT;
  } catch (const ParseError& e) {
    g_err = e.what();
    return EQS_ERR_PARSE;
  } catch (const CudaError& e) {
    g_err = e.what();
    return EQS_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EQS_ERR_OTHER;
  }
}

// need_device: compute entry points refuse a host-only context (device < 0)
GpuSystem& S(eqs_ctx* c, bool need_device = true) {
  if (!c || !c->sys) throw std::invalid_argument("null eqs_ctx");
  if (need_device && c->sys->host_only()) throw CudaError("context was created host-only (device < 0)");
  return *c->sys;
}
GpuSystem& H(eqs_ctx* c) { return S(c, false); }

SolverParams solver_from(const eqs_solver_params& s) {
  SolverParams p;
  p.precond = s.precond;
  p.rel_tol = s.rel_tol;
  p.max_iter = s.max_iter;
  p.rho_solve_tol = s.rho_solve_tol;
  p.amg_theta = s.amg_strength_threshold;
  p.amg_omega = s.amg_prolongation_omega;
  p.amg_sweeps = s.amg_smoother_sweeps;
  p.amg_max_levels = s.amg_max_levels;
  p.amg_coarse_limit = s.amg_coarse_limit;
  p.estimator_mode = s.estimator_mode;
  p.spe_window = s.spe_window;
  p.mgs_drop_tol = s.mgs_drop_tol;
  if (s.pod_snapshots > 0) p.pod_snapshots = s.pod_snapshots;
  if (s.pod_rank > 0) p.pod_rank = s.pod_rank;
  if (s.pod_capacity > 0) p.pod_capacity = s.pod_capacity;
  p.pod_threshold = s.pod_threshold;
  p.amg_coarse_filter = s.amg_coarse_filter;
  p.amg_dense_coarse = s.amg_dense_coarse;
  return p;
}

void fill_stats(GpuSystem& g, eqs_solve_stats* o) {
  const SolveStats& s = g.stats();
  std::memset(o, 0, sizeof(*o));
  o->m_solves = s.m_solves;
  o->pcg_iterations = s.pcg_iterations;
  o->rho_solves = s.rho_solves;
  o->rho_pcg_iterations = s.rho_pcg_iterations;
  o->precond_setups = s.precond_setups;
  o->assemblies = s.assemblies;
  o->time_residual = s.t_residual;
  o->time_solve = s.t_solve;
  o->time_setup = s.t_setup;
  o->time_estimator = s.t_estimator;
  o->applies = s.applies;
  o->spe_fallbacks = s.spe_fallbacks;
  o->svd_count = s.svd_count;
  o->estimator_appends = s.appends;
  o->newton_linear_solves = s.newton_linear_solves;
  o->newton_pcg_iterations = s.newton_pcg_iterations;
}

void fill_pcg(const PcgResult& r, eqs_pcg_result* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->rel_residual = r.rel_residual;
  o->initial_rel_residual = r.initial_rel_residual;
  o->converged = r.converged ? 1 : 0;
}
}  // namespace

extern "C" {

const char* eqs_last_error(void) { return g_err.c_str(); }

int eqs_create(const eqs_problem_desc* d, eqs_ctx** out) {
  return guard([&] {
    if (!d || !out) throw std::invalid_argument("eqs_create: null argument");
    if (d->order != 1 && d->order != 2) throw ConfigError("element order must be 1 or 2");
    Problem p;
    p.mesh.n_nodes = d->n_nodes;
    p.mesh.n_tets = d->n_tets;
    p.mesh.nodes.assign(d->nodes, d->nodes + 3L * d->n_nodes);
    p.mesh.tets.assign(d->tets, d->tets + 4L * d->n_tets);
    p.mesh.region.assign(d->region_id, d->region_id + d->n_tets);
    p.dm.order = d->order;
    p.dm.n_local = d->order == 1 ? 4 : 10;
    p.dm.n_dofs = d->n_dofs;
    p.dm.element_dofs.assign(d->element_dofs, d->element_dofs + (long)p.dm.n_local * d->n_tets);
    p.dm.free_dofs.assign(d->free_dofs, d->free_dofs + d->n_free);
    p.dm.fixed_dofs.assign(d->fixed_dofs, d->fixed_dofs + d->n_fixed);
    p.dm.fixed_set.assign(d->fixed_set, d->fixed_set + d->n_dofs);
    if ((long)d->n_free + d->n_fixed != d->n_dofs) throw std::invalid_argument("eqs_create: n_free + n_fixed != n_dofs");
    for (int s = 0; s < d->n_sets; ++s) {
      p.dm.set_names.push_back("set" + std::to_string(s));
      const eqs_waveform& w = d->set_waveforms[s];
      Waveform wf;
      wf.kind = w.kind;
      wf.amplitude = w.amplitude;
      wf.frequency = w.frequency;
      wf.phase = w.phase;
      wf.rise_time = w.rise_time;
      wf.value = w.value;
      p.set_waveforms.push_back(wf);
    }
    for (int m = 0; m < d->n_materials; ++m) {
      const eqs_material& em = d->materials[m];
      Material mm;
      mm.kind = em.kind;
      mm.eps_r = em.eps_r;
      mm.kappa = em.kappa;
      mm.kappa_lo = em.kappa_lo;
      mm.kappa_hi = em.kappa_hi;
      mm.e_switch = em.e_switch;
      mm.width = em.width;
      mm.validate();
      p.materials[em.region] = mm;
    }
    p.solver = solver_from(d->solver);
    auto ctx = std::make_unique<eqs_ctx>();
    ctx->sys = std::make_unique<GpuSystem>(std::move(p), d->device);
    *out = ctx.release();
  });
}

int eqs_create_from_config(const char* json_text, int device, eqs_ctx** out) {
  return guard([&] {
    if (!json_text || !out) throw std::invalid_argument("eqs_create_from_config: null argument");
    SimConfig c = parse_config(json_text);
    auto ctx = std::make_unique<eqs_ctx>();
    ctx->sys = std::make_unique<GpuSystem>(build_problem(c), device);
    *out = ctx.release();
  });
}

void eqs_destroy(eqs_ctx* ctx) { delete ctx; }

int eqs_nccl_unique_id(char* id128) {
  return guard([&] {
    const std::string id = nccl_unique_id();
    std::memcpy(id128, id.data(), id.size());
  });
}

// Host setup of the ranks of one node, at most EQS_SETUP_CONCURRENCY at a
// time (default: all): every rank builds the global mesh, M and AMG
// hierarchy before extracting its partition, so the node's peak host memory
// is (concurrency) x (one global build) + the others' partitions. A POSIX
// semaphore named after the job's NCCL id gates the phase from before
// build_problem to the release of the global hierarchy (GpuSystem ctor,
// setup_gate_release); the collective device build runs after it.
struct SetupGate {
  sem_t* sem = nullptr;
  bool held = false;
  char name[64] = {};
  SetupGate(const std::string& key, int nranks) {
    const char* e = getenv("EQS_SETUP_CONCURRENCY");
    const int k = e ? atoi(e) : 0;
    if (k <= 0 || k >= nranks) return;
    unsigned long h = 1469598103934665603ul;
    for (unsigned char ch : key) h = (h ^ ch) * 1099511628211ul;
    std::snprintf(name, sizeof name, "/eqs_setup_%016lx", h);
    sem = sem_open(name, O_CREAT, 0600, (unsigned)k);
    if (sem == SEM_FAILED) {
      sem = nullptr;
      return;
    }
    while (sem_wait(sem) != 0) {
    }
    held = true;
  }
  void release() {
    if (held) sem_post(sem);
    held = false;
  }
  // once any rank's context is built every rank has passed the gate (the
  // device build's collectives need all of them): the name can go
  void unlink() {
    if (sem) sem_unlink(name);
  }
  ~SetupGate() {
    release();
    if (sem) sem_close(sem);
  }
};

int eqs_create_distributed(const char* json_text, int device, int nranks, int rank, const char* id128,
                           eqs_ctx** out) {
  return guard([&] {
    if (!json_text || !out || !id128) throw std::invalid_argument("eqs_create_distributed: null argument");
    SimConfig c = parse_config(json_text);
    std::unique_ptr<Comm> comm;
    if (nranks > 1) {
      cuda_check(cudaSetDevice(device), "cudaSetDevice");
      comm = make_nccl_comm(std::string(id128, 128), nranks, rank);
    }
    SetupGate gate(std::string(id128, 128), nranks);
    setup_gate_release = [&gate] { gate.release(); };
    auto ctx = std::make_unique<eqs_ctx>();
    try {
      ctx->sys = std::make_unique<GpuSystem>(build_problem(c), device, std::move(comm));
    } catch (...) {
      setup_gate_release = nullptr;
      throw;
    }
    setup_gate_release = nullptr;
    if (rank == 0) gate.unlink();
    *out = ctx.release();
  });
}

int eqs_create_distributed_shm(const char* json_text, int device, int nranks, int rank, const char* shm_name,
                               eqs_ctx** out) {
  return guard([&] {
    if (!json_text || !out || !shm_name) throw std::invalid_argument("eqs_create_distributed_shm: null argument");
    SimConfig c = parse_config(json_text);
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    std::unique_ptr<Comm> comm = make_shm_comm(shm_name, nranks, rank);
    SetupGate gate(shm_name, nranks);
    setup_gate_release = [&gate] { gate.release(); };
    auto ctx = std::make_unique<eqs_ctx>();
    try {
      ctx->sys = std::make_unique<GpuSystem>(build_problem(c), device, std::move(comm));
    } catch (...) {
      setup_gate_release = nullptr;
      throw;
    }
    setup_gate_release = nullptr;
    if (rank == 0) gate.unlink();
    *out = ctx.release();
  });
}

struct eqs_comm {
  std::unique_ptr<Comm> comm;
};

int eqs_comm_open_shm(const char* shm_name, int nranks, int rank, eqs_comm** out) {
  return guard([&] {
    if (!shm_name || !out) throw std::invalid_argument("eqs_comm_open_shm: null argument");
    auto c = std::make_unique<eqs_comm>();
    c->comm = make_shm_comm(shm_name, nranks, rank);
    *out = c.release();
  });
}
void eqs_comm_close(eqs_comm* c) { delete c; }
int eqs_comm_barrier(eqs_comm* c) {
  return guard([&] { c->comm->barrier(); });
}
int eqs_comm_allreduce_host(eqs_comm* c, double* buf, int count) {
  return guard([&] { shm_allreduce_host(*c->comm, buf, count); });
}
int eqs_comm_exchange_host(eqs_comm* c, int n_msgs, const int* peers, const double* const* send,
                           const int* send_counts, double* const* recv, const int* recv_counts) {
  return guard([&] {
    std::vector<HaloMsg> msgs;
    for (int k = 0; k < n_msgs; ++k)
      msgs.push_back({peers[k], send[k], send_counts[k], recv[k], recv_counts[k], 8});
    shm_exchange_host(*c->comm, msgs);
  });
}

int eqs_create_virtual_group(const char* json_text, int device, int nranks, eqs_ctx** out) {
  return guard([&] {
    if (!json_text || !out || nranks < 1) throw std::invalid_argument("eqs_create_virtual_group: bad argument");
    SimConfig c = parse_config(json_text);
    auto group = make_thread_group(nranks);
    std::vector<std::unique_ptr<eqs_ctx>> ctx(nranks);
    std::vector<std::string> err(nranks);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r)
      th.emplace_back([&, r] {
        try {
          ctx[r] = std::make_unique<eqs_ctx>();
          ctx[r]->sys = std::make_unique<GpuSystem>(build_problem(c), device, make_thread_comm(group, r));
        } catch (const std::exception& e) {
          err[r] = e.what();
        }
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < nranks; ++r)
      if (!err[r].empty()) throw std::runtime_error("virtual rank " + std::to_string(r) + ": " + err[r]);
    for (int r = 0; r < nranks; ++r) out[r] = ctx[r].release();
  });
}

int eqs_create_partition_host(const char* json_text, int nranks, int rank, eqs_ctx** out) {
  return guard([&] {
    SimConfig c = parse_config(json_text);
    auto ctx = std::make_unique<eqs_ctx>();
    ctx->sys = std::make_unique<GpuSystem>(build_problem(c), -1, std::make_unique<StaticComm>(rank, nranks));
    *out = ctx.release();
  });
}

int eqs_partition_info(eqs_ctx* ctx, long* info) {
  return guard([&] {
    const PartitionPlan& p = H(ctx).plan();
    info[0] = p.rank;
    info[1] = p.nranks;
    info[2] = (long)p.space.size();
    info[3] = p.space[0].n_own();
  });
}

int eqs_partition_level(eqs_ctx* ctx, int level, long* info) {
  return guard([&] {
    const PartitionPlan& p = H(ctx).plan();
    if (level < 0 || level >= (int)p.space.size()) throw std::invalid_argument("eqs_partition_level: bad level");
    const LocalSpace& s = p.space[level];
    info[0] = s.n_global;
    info[1] = s.n_own();
    info[2] = s.n_ghost();
    info[3] = (long)s.recv_ranks.size();
    info[4] = (long)s.send_ranks.size();
    info[5] = (long)p.tets.size();
    info[6] = (long)p.fixed.size();
    info[7] = level >= p.rep_level ? 1 : 0;
  });
}

int eqs_partition_owner(eqs_ctx* ctx, int level, int* owner) {
  return guard([&] {
    const PartitionPlan& p = H(ctx).plan();
    if (level < 0 || level >= (int)p.owner.size()) throw std::invalid_argument("eqs_partition_owner: bad level");
    std::memcpy(owner, p.owner[level].data(), sizeof(int) * p.owner[level].size());
  });
}

int eqs_partition_owned(eqs_ctx* ctx, int level, int* ids) {
  return guard([&] {
    const LocalSpace& s = H(ctx).plan().space.at(level);
    std::memcpy(ids, s.owned.data(), sizeof(int) * s.owned.size());
  });
}

int eqs_partition_ghosts(eqs_ctx* ctx, int level, int* ids) {
  return guard([&] {
    const LocalSpace& s = H(ctx).plan().space.at(level);
    std::memcpy(ids, s.ghosts.data(), sizeof(int) * s.ghosts.size());
  });
}

int eqs_partition_send(eqs_ctx* ctx, int level, int peer, int* ids, int* count) {
  return guard([&] {
    const LocalSpace& s = H(ctx).plan().space.at(level);
    *count = 0;
    for (size_t k = 0; k < s.send_ranks.size(); ++k)
      if (s.send_ranks[k] == peer) {
        const auto& l = s.send_local[k];
        if (ids)
          for (size_t i = 0; i < l.size(); ++i) ids[i] = s.owned[l[i]];
        *count = (int)l.size();
      }
  });
}

int eqs_get_sizes(eqs_ctx* ctx, eqs_sizes* o) {
  return guard([&] {
    GpuSystem& g = H(ctx);
    const Problem& p = g.problem();
    o->n_nodes = p.mesh.n_nodes;
    o->n_tets = p.mesh.n_tets;
    o->n_dofs = p.dm.n_dofs;
    o->n_free = p.dm.n_free();
    o->n_fixed = p.dm.n_fixed();
    o->n_local = p.dm.n_local;
    o->order = p.dm.order;
    o->n_colors = -1;
    o->nnz_mass_free = g.mass_ii().nnz();
    o->nnz_mass_ib = g.mass_ib().nnz();
    o->amg_levels = (long)g.amg().levels.size();
  });
}

int eqs_get_colors(eqs_ctx* ctx, int* color_of_tet) {
  return guard([&] {
    const std::vector<int>& c = H(ctx).colors();
    std::memcpy(color_of_tet, c.data(), sizeof(int) * c.size());
  });
}

int eqs_get_mesh(eqs_ctx* ctx, double* nodes, int* tets, int* region_id) {
  return guard([&] {
    const Mesh& m = H(ctx).problem().mesh;
    if (nodes) std::memcpy(nodes, m.nodes.data(), sizeof(double) * m.nodes.size());
    if (tets) std::memcpy(tets, m.tets.data(), sizeof(int) * m.tets.size());
    if (region_id) std::memcpy(region_id, m.region.data(), sizeof(int) * m.region.size());
  });
}

int eqs_get_dofs(eqs_ctx* ctx, int* element_dofs, int* free_dofs, int* fixed_dofs) {
  return guard([&] {
    const Dofs& d = H(ctx).problem().dm;
    if (element_dofs) std::memcpy(element_dofs, d.element_dofs.data(), sizeof(int) * d.element_dofs.size());
    if (free_dofs) std::memcpy(free_dofs, d.free_dofs.data(), sizeof(int) * d.free_dofs.size());
    if (fixed_dofs) std::memcpy(fixed_dofs, d.fixed_dofs.data(), sizeof(int) * d.fixed_dofs.size());
  });
}

int eqs_get_mass(eqs_ctx* ctx, int which, int* row_ptr, int* col_idx, double* values) {
  return guard([&] {
    const HostCsr& m = which == 0 ? H(ctx).mass_ii() : H(ctx).mass_ib();
    std::memcpy(row_ptr, m.row_ptr.data(), sizeof(int) * m.row_ptr.size());
    std::memcpy(col_idx, m.col_idx.data(), sizeof(int) * m.col_idx.size());
    std::memcpy(values, m.values.data(), sizeof(double) * m.values.size());
  });
}

int eqs_amg_levels(eqs_ctx* ctx, int* n_levels, long* rows_nnz) {
  return guard([&] {
    const AmgHierarchy& h = H(ctx).amg();
    *n_levels = (int)h.levels.size();
    if (rows_nnz)
      for (size_t l = 0; l < h.levels.size(); ++l) {
        rows_nnz[2 * l] = h.levels[l].A.n_rows;
        rows_nnz[2 * l + 1] = h.levels[l].A.nnz();
      }
  });
}

int eqs_amg_aggregates(eqs_ctx* ctx, int level, int* agg) {
  return guard([&] {
    const AmgHierarchy& h = H(ctx).amg();
    if (level < 0 || level >= (int)h.levels.size()) throw std::invalid_argument("eqs_amg_aggregates: bad level");
    const auto& a = h.levels[level].aggregates;
    std::memcpy(agg, a.data(), sizeof(int) * a.size());
  });
}

int eqs_amg_level_csr(eqs_ctx* ctx, int level, int which, int* dims, int* row_ptr, int* col_idx, double* values) {
  return guard([&] {
    const AmgHierarchy& h = H(ctx).amg();
    if (level < 0 || level >= (int)h.levels.size() || which < 0 || which > 2)
      throw std::invalid_argument("eqs_amg_level_csr: bad level or matrix");
    const AmgHostLevel& lv = h.levels[level];
    const HostCsr& m = which == 0 ? lv.A : which == 1 ? lv.P : lv.R;
    if (m.row_ptr.empty() && !(which > 0 && level + 1 == (int)h.levels.size()))
      throw std::invalid_argument("eqs_amg_level_csr: host copy released (multi-rank context)");
    dims[0] = m.n_rows;
    dims[1] = m.n_cols;
    dims[2] = (int)m.nnz();
    if (row_ptr) {
      std::memcpy(row_ptr, m.row_ptr.data(), sizeof(int) * m.row_ptr.size());
      std::memcpy(col_idx, m.col_idx.data(), sizeof(int) * m.nnz());
      std::memcpy(values, m.values.data(), sizeof(double) * m.nnz());
    }
  });
}

int eqs_kx_apply(eqs_ctx* ctx, const double* x_state, const double* v, double* y) {
  return guard([&] { S(ctx).kx_apply_host(x_state, v, y); });
}
int eqs_kx_apply_dev(eqs_ctx* ctx, const double* x_state, const double* v, double* y) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    g.kx_apply_full_dev(x_state, v, y);
    cuda_check(cudaStreamSynchronize(g.stream()), "eqs_kx_apply_dev");
  });
}
int eqs_kx_residual(eqs_ctx* ctx, const double* x_full, const double* b_mass, double* r) {
  return guard([&] { S(ctx).kx_residual_host(x_full, b_mass, r); });
}
int eqs_kx_residual_dev(eqs_ctx* ctx, const double* x_full, const double* b_mass, double* r) {
  return guard([&] {
    (void)x_full;
    (void)b_mass;
    (void)r;
    throw std::invalid_argument("eqs_kx_residual_dev: use eqs_eval_residual on the resident state");
  });
}
int eqs_mass_apply(eqs_ctx* ctx, const double* v, double* y) {
  return guard([&] { S(ctx).mass_apply_host(v, y); });
}
int eqs_mass_solve(eqs_ctx* ctx, const double* b, const double* x0, double tol, int max_iter, double* x,
                   eqs_pcg_result* res) {
  return guard([&] { fill_pcg(S(ctx).mass_solve_host(b, x0, tol, max_iter, x), res); });
}
int eqs_mass_solve_sequence(eqs_ctx* ctx, const double* B, int k, double tol, int max_iter, double* X,
                            int* iterations, double* device_ms) {
  return guard([&] {
    if (k < 1 || !B) throw std::invalid_argument("eqs_mass_solve_sequence: need k >= 1 right-hand sides");
    const double ms = S(ctx).mass_solve_sequence(B, k, tol, max_iter, X, iterations);
    if (device_ms) *device_ms = ms;
  });
}
int eqs_estimator_next(eqs_ctx* ctx, const double* b, double* x0, int* rank) {
  return guard([&] {
    if (!b || !x0) throw std::invalid_argument("eqs_estimator_next: null vector");
    const int r = S(ctx).estimator_next_host(b, x0);
    if (rank) *rank = r;
  });
}
int eqs_estimator_feedback(eqs_ctx* ctx, const double* x, int iterations) {
  return guard([&] {
    if (!x) throw std::invalid_argument("eqs_estimator_feedback: null vector");
    S(ctx).estimator_feedback_host(x, iterations);
  });
}
int eqs_eval_residual(eqs_ctx* ctx, double t, const double* x, double* r) {
  return guard([&] { S(ctx).eval_residual_host(t, x, r); });
}
int eqs_eval_rhs(eqs_ctx* ctx, double t, const double* x, double* f, eqs_pcg_result* res) {
  return guard([&] { fill_pcg(S(ctx).eval_rhs_host(t, x, f), res); });
}
int eqs_apply_minv_stiffness(eqs_ctx* ctx, double t, const double* x_state, const double* v, double* y) {
  return guard([&] { S(ctx).apply_minv_stiffness_host(t, x_state, v, y); });
}
int eqs_lift_full(eqs_ctx* ctx, double t, const double* x_free, double* x_full) {
  return guard([&] { H(ctx).lift_full_host(t, x_free, x_full); });
}
int eqs_get_stats(eqs_ctx* ctx, eqs_solve_stats* out) {
  return guard([&] { fill_stats(H(ctx), out); });
}
int eqs_set_state(eqs_ctx* ctx, double t, const double* x, double dt) {
  return guard([&] { S(ctx).set_state(t, x, dt); });
}
int eqs_get_state(eqs_ctx* ctx, double* x, eqs_state_info* info) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    if (x) g.get_state(x);
    if (info) {
      info->t = g.state_t;
      info->dt = g.state_dt;
      info->accepted = g.st_accepted;
      info->rejected = g.st_rejected;
      info->stages = g.st_stages;
      info->rho_value = g.rho_value;
      info->rho_age = g.rho_age;
      info->rho_valid = g.rho_valid ? 1 : 0;
    }
  });
}
int eqs_spectral_radius(eqs_ctx* ctx, double* rho) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    *rho = g.estimate_spectral_radius(g.state_t, g.state_dev());
  });
}
int eqs_rkc_step(eqs_ctx* ctx, const eqs_rkc_options* o, eqs_step_attempt* att) {
  return guard([&] {
    RkcOptions ro;
    if (o) {
      ro.rtol = o->rtol;
      ro.atol = o->atol;
      ro.max_stages = o->max_stages;
      ro.rho_refresh_every = o->rho_refresh_every;
    }
    const StepAttempt a = S(ctx).rkc_step(ro);
    if (att) {
      att->t_start = a.t_start;
      att->dt = a.dt;
      att->accepted = a.accepted ? 1 : 0;
      att->stages = a.stages;
      att->newton_iterations = 0;
      att->error = a.error;
      att->rho = a.rho;
      att->dt_next = a.dt_next;
    }
  });
}
namespace {
SdirkOptions sdirk_from(const eqs_sdirk_options* o) {
  SdirkOptions so;
  if (o) {
    so.rtol = o->rtol;
    so.atol = o->atol;
    if (o->newton_tol > 0) so.newton_tol = o->newton_tol;
    if (o->max_newton > 0) so.max_newton = o->max_newton;
  }
  return so;
}
}  // namespace
int eqs_shifted_solve(eqs_ctx* ctx, double t, const double* z, double gdt, const double* rhs, double* delta,
                      int refresh_precond) {
  return guard([&] {
    if (!z || !rhs || !delta) throw std::invalid_argument("eqs_shifted_solve: null vector");
    S(ctx).shifted_solve_host(t, z, gdt, rhs, delta, refresh_precond != 0);
  });
}
int eqs_sdirk_step(eqs_ctx* ctx, const eqs_sdirk_options* o, eqs_step_attempt* att) {
  return guard([&] {
    const StepAttempt a = S(ctx).sdirk_step(sdirk_from(o));
    if (att) {
      att->t_start = a.t_start;
      att->dt = a.dt;
      att->accepted = a.accepted ? 1 : 0;
      att->stages = a.stages;
      att->newton_iterations = a.newton_iterations;
      att->error = a.error;
      att->rho = 0.0;
      att->dt_next = a.dt_next;
    }
  });
}
int eqs_sdirk_advance_fixed(eqs_ctx* ctx, double dt, int nsteps, const eqs_sdirk_options* o) {
  return guard([&] {
    if (!(dt > 0) || nsteps < 0) throw std::invalid_argument("eqs_sdirk_advance_fixed: need dt > 0, nsteps >= 0");
    const SdirkOptions so = sdirk_from(o);
    for (int i = 0; i < nsteps; ++i)
      if (!S(ctx).sdirk_advance_fixed(dt, so)) throw NumericalError("sdirk: Newton iteration failed");
  });
}
int eqs_rkc_advance_fixed(eqs_ctx* ctx, double dt, int s, int nsteps) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    if (s < 2) throw std::invalid_argument("rkc: stage count must be >= 2");
    for (int i = 0; i < nsteps; ++i) g.rkc_advance_fixed(dt, s);
    cuda_check(cudaStreamSynchronize(g.stream()), "eqs_rkc_advance_fixed");
  });
}
int eqs_euler_step(eqs_ctx* ctx, double dt, eqs_step_attempt* att) {
  return guard([&] {
    const StepAttempt a = S(ctx).euler_step(dt);
    if (att) {
      std::memset(att, 0, sizeof(*att));
      att->t_start = a.t_start;
      att->dt = a.dt;
      att->accepted = 1;
      att->stages = 1;
      att->dt_next = a.dt_next;
    }
  });
}

int eqs_run_scenario(const char* json_text, const char* out_dir, int device, eqs_run_result* res, double* x_final,
                     long x_cap) {
  return guard([&] {
    SimConfig c = parse_config(json_text);
    RunResult r = run_scenario(c, out_dir ? out_dir : "", device);
    std::memset(res, 0, sizeof(*res));
    res->exit_code = r.exit_code;
    res->accepted = r.accepted;
    res->rejected = r.rejected;
    res->stages = r.stages;
    res->final_t = r.final_t;
    res->wall_time = r.wall_time;
    res->n_free = (long)r.final_x_free.size();
    res->stats.m_solves = r.stats.m_solves;
    res->stats.pcg_iterations = r.stats.pcg_iterations;
    res->stats.rho_solves = r.stats.rho_solves;
    res->stats.rho_pcg_iterations = r.stats.rho_pcg_iterations;
    res->stats.precond_setups = r.stats.precond_setups;
    res->stats.assemblies = r.stats.assemblies;
    res->stats.time_residual = r.stats.t_residual;
    res->stats.time_solve = r.stats.t_solve;
    res->stats.time_setup = r.stats.t_setup;
    res->stats.time_estimator = r.stats.t_estimator;
    res->stats.applies = r.stats.applies;
    res->stats.spe_fallbacks = r.stats.spe_fallbacks;
    res->stats.svd_count = r.stats.svd_count;
    res->stats.estimator_appends = r.stats.appends;
    res->stats.newton_linear_solves = r.stats.newton_linear_solves;
    res->stats.newton_pcg_iterations = r.stats.newton_pcg_iterations;
    if (x_final && (long)r.final_x_free.size() <= x_cap)
      std::memcpy(x_final, r.final_x_free.data(), sizeof(double) * r.final_x_free.size());
    if (r.exit_code != 0) {
      g_err = r.error;
      if (r.exit_code == 1) throw ConfigError(r.error);
      throw NumericalError(r.error);
    }
  });
}

int eqs_timing_enable(eqs_ctx* ctx, int on) {
  return guard([&] { S(ctx).timing_on = on != 0; });
}
int eqs_timing_get(eqs_ctx* ctx, eqs_timing* out) {
  return guard([&] {
    std::memset(out, 0, sizeof(*out));
    S(ctx).timing_resolve(out->ms, out->launches, out->bytes);
  });
}
int eqs_timing_reset(eqs_ctx* ctx) {
  return guard([&] { S(ctx).timing_reset(); });
}
int eqs_set_option(eqs_ctx* ctx, int key, double value) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    switch (key) {
      case 0: g.stiffness_mode = (int)value; break;
      case 1: g.cheb_degree = (int)value; g.invalidate_graphs(); break;
      case 2: g.set_cheb(value); break;
      case 3: g.coarse_degree = (int)value; g.invalidate_graphs(); break;
      case 4: g.set_vcycle_precision((int)value); break;
      case 5: g.set_level_tpr(0, (int)value); break;
      case 6: g.set_level_tpr(1, (int)value); break;
      case 7: g.set_level_tpr(2, (int)value); break;
      case 8: g.use_graphs = value != 0.0; g.invalidate_graphs(); break;
      case 9: g.spe_incremental = value != 0.0; break;
      case 10: g.set_sell(value != 0.0); break;
      case 11: g.set_vcycle_vectors_f32(value != 0.0); break;
      case 12: g.reset_estimator((int)value); break;
      case 13: g.cheb_kind = (int)value; g.set_cheb(g.cheb_ratio); break;
      case 14: g.cheb_scale = value; g.set_cheb(g.cheb_ratio); break;
      case 15: g.set_pod_params((int)value, 0, 0, -1.0); break;
      case 16: g.set_pod_params(0, (int)value, 0, -1.0); break;
      case 17: g.set_pod_params(0, 0, (int)value, -1.0); break;
      case 18: g.set_pod_params(0, 0, 0, std::max(0.0, value)); break;
      case 19: g.set_stencil(value != 0.0); break;
      case 20: g.pcg_graph_loop = value != 0.0; g.invalidate_graphs(); break;
      case 21: g_pdl = value != 0.0; g.invalidate_graphs(); break;
      case 22: g.pcg_graph_multi = value != 0.0; g.invalidate_graphs(); break;
      case 23: g.set_stencil_sym(value != 0.0); break;
      case 24: g.timing_graph = value != 0.0; break;
      case 26: g.shift_amg = value != 0.0; break;
      case 27: g.shift_pcg_graph = value != 0.0; break;
      case 28: g.wcycle_from = (int)value; g.invalidate_graphs(); break;
      case 29: g.fine_pre_degree = (int)value; g.invalidate_graphs(); break;
      case 30: g.set_stencil_rowsum(value != 0.0); break;
      default: throw std::invalid_argument("eqs_set_option: unknown key");
    }
  });
}
int eqs_set_rho(eqs_ctx* ctx, double value, int valid, long age) {
  return guard([&] {
    GpuSystem& g = S(ctx);
    g.rho_value = value;
    g.rho_valid = valid != 0;
    g.rho_age = age;
  });
}
int eqs_get_stream(eqs_ctx* ctx, void** stream) {
  return guard([&] { *stream = (void*)S(ctx).stream(); });
}
long eqs_launch_count(void) { return g_launch_count; }
int eqs_random_vec(int n, unsigned seed, double* out) {
  return guard([&] {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (int i = 0; i < n; ++i) out[i] = uni(rng);
  });
}

}  // extern "C"
