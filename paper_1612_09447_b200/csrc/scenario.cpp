// Drop-in scenario runner: run_scenario (proj/src/scenario.cpp:217-383) on
// the GPU-resident system, with the reference's CSV schemas
// (proj/src/metrics.cpp:20-66), probes (proj/src/probes.cpp:7-43) and legacy
// VTK output (proj/src/vtk_writer.cpp:11-49).
#include "scenario.hpp"

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>

#include "element.hpp"

namespace eqsb {

namespace fs = std::filesystem;

namespace {

std::string join_path(const std::string& dir, const std::string& file) {
  if (file.empty()) return {};
  if (dir.empty() || fs::path(file).is_absolute()) return file;
  return (fs::path(dir) / file).string();
}

struct PointLocation {
  int tet = -1;
  double lambda[4] = {0, 0, 0, 0};
};

// proj/src/probes.cpp:7-27 (brute-force scan)
bool locate_point(const Mesh& mesh, const std::array<double, 3>& p, PointLocation& loc) {
  // proj/src/probes.cpp:9-25: the first tet (ascending id) whose barycentric
  // coordinates are all >= -1e-12. Scanned in parallel with a min-reduction
  // over the containing ids, so the result is the sequential one.
  int best = INT_MAX;
  bool degenerate = false;
#pragma omp parallel for schedule(static) reduction(min : best) reduction(|| : degenerate)
  for (int t = 0; t < mesh.n_tets; ++t) {
    double x[4][3];
    for (int v = 0; v < 4; ++v)
      for (int d = 0; d < 3; ++d) x[v][d] = mesh.nodes[3L * mesh.tets[4L * t + v] + d];
    TetGeo g;
    if (!tet_geometry(x, g)) {
      degenerate = true;
      continue;
    }
    double min_lambda = 1.0;
    for (int i = 0; i < 4; ++i) {
      double l = i == 0 ? 1.0 : 0.0;
      for (int d = 0; d < 3; ++d) l += g.g[i][d] * (p[d] - x[0][d]);
      min_lambda = std::min(min_lambda, l);
    }
    if (min_lambda >= -1e-12 && t < best) best = t;
  }
  if (degenerate) throw GeometryError("degenerate tetrahedron in element kernel");
  if (best == INT_MAX) return false;
  double x[4][3];
  for (int v = 0; v < 4; ++v)
    for (int d = 0; d < 3; ++d) x[v][d] = mesh.nodes[3L * mesh.tets[4L * best + v] + d];
  TetGeo g;
  tet_geometry(x, g);
  for (int i = 0; i < 4; ++i) {
    double l = i == 0 ? 1.0 : 0.0;
    for (int d = 0; d < 3; ++d) l += g.g[i][d] * (p[d] - x[0][d]);
    loc.lambda[i] = l;
  }
  loc.tet = best;
  return true;
}

// proj/src/probes.cpp:29-43 on the element's dof values
double interpolate(int order, const double* vals, const PointLocation& loc) {
  const double* lam = loc.lambda;
  double value = 0.0;
  if (order == 1) {
    for (int i = 0; i < 4; ++i) value += lam[i] * vals[i];
    return value;
  }
  for (int i = 0; i < 4; ++i) value += lam[i] * (2.0 * lam[i] - 1.0) * vals[i];
  for (int e = 0; e < 6; ++e) {
    const int a = kTetEdgeVertices[e][0], b = kTetEdgeVertices[e][1];
    value += 4.0 * lam[a] * lam[b] * vals[4 + e];
  }
  return value;
}

}  // namespace

// proj/src/vtk_writer.cpp:11-49 (VTK 2.0 unstructured grid, potential + per-cell
// kappa). kappa comes from the device (GpuSystem::cell_kappa_host). binary
// (additive key output.vtk_binary): legacy BINARY, big-endian, same arrays.
namespace {
template <class T>
void put_be(std::ostream& os, T v) {
  unsigned char b[sizeof(T)];
  std::memcpy(b, &v, sizeof(T));
  std::reverse(b, b + sizeof(T));
  os.write(reinterpret_cast<const char*>(b), sizeof(T));
}
}  // namespace

void write_vtk(const std::string& path, const Problem& p, const std::vector<double>& x_full,
               const std::vector<double>& kappa, bool binary) {
  std::ofstream os(path, std::ios::binary);
  if (!os) throw ConfigError("cannot open for writing: " + path);
  const Mesh& mesh = p.mesh;
  char buf[128];
  os << "# vtk DataFile Version 2.0\npotential\n" << (binary ? "BINARY" : "ASCII") << "\nDATASET UNSTRUCTURED_GRID\n";
  os << "POINTS " << mesh.n_nodes << " double\n";
  if (binary) {
    for (long k = 0; k < 3L * mesh.n_nodes; ++k) put_be(os, mesh.nodes[k]);
    os << "\n";
  } else {
    for (int n = 0; n < mesh.n_nodes; ++n) {
      std::snprintf(buf, sizeof buf, "%.9g %.9g %.9g\n", mesh.nodes[3L * n], mesh.nodes[3L * n + 1],
                    mesh.nodes[3L * n + 2]);
      os << buf;
    }
  }
  os << "CELLS " << mesh.n_tets << " " << 5L * mesh.n_tets << "\n";
  if (binary) {
    for (int t = 0; t < mesh.n_tets; ++t) {
      put_be<int32_t>(os, 4);
      for (int v = 0; v < 4; ++v) put_be<int32_t>(os, mesh.tets[4L * t + v]);
    }
    os << "\n";
  } else {
    for (int t = 0; t < mesh.n_tets; ++t)
      os << "4 " << mesh.tets[4L * t] << " " << mesh.tets[4L * t + 1] << " " << mesh.tets[4L * t + 2] << " "
         << mesh.tets[4L * t + 3] << "\n";
  }
  os << "CELL_TYPES " << mesh.n_tets << "\n";
  if (binary) {
    for (int t = 0; t < mesh.n_tets; ++t) put_be<int32_t>(os, 10);
    os << "\n";
  } else {
    for (int t = 0; t < mesh.n_tets; ++t) os << "10\n";
  }
  os << "POINT_DATA " << mesh.n_nodes << "\nSCALARS potential double 1\nLOOKUP_TABLE default\n";
  for (int n = 0; n < mesh.n_nodes; ++n) {  // vertex dofs lead
    if (binary) {
      put_be(os, x_full[n]);
    } else {
      std::snprintf(buf, sizeof buf, "%.9g\n", x_full[n]);
      os << buf;
    }
  }
  if (binary) os << "\n";
  os << "CELL_DATA " << mesh.n_tets << "\nSCALARS kappa double 1\nLOOKUP_TABLE default\n";
  for (int t = 0; t < mesh.n_tets; ++t) {
    if (binary) {
      put_be(os, kappa[t]);
    } else {
      std::snprintf(buf, sizeof buf, "%.9g\n", kappa[t]);
      os << buf;
    }
  }
  if (binary) os << "\n";
}

// proj/src/metrics.cpp:20-35
void write_metrics_csv(const std::string& path, const std::vector<StepMetrics>& rows) {
  std::ofstream os(path);
  if (!os) throw ConfigError("cannot open for writing: " + path);
  os << "step,t,dt,method,accepted,stages,newton_iters,m_solves,pcg_iters,rho,"
        "estimator_mode,estimator_rank,err_est,"
        "time_residual_s,time_solve_s,time_setup_s,time_estimator_s\n";
  char buf[512];
  for (const auto& r : rows) {
    std::snprintf(buf, sizeof buf, "%ld,%.17g,%.17g,%s,%d,%d,%d,%ld,%ld,%.17g,%s,%d,%.17g,%.6g,%.6g,%.6g,%.6g\n",
                  r.step, r.t, r.dt, r.method.c_str(), r.accepted ? 1 : 0, r.stages, r.newton_iters, r.m_solves, r.pcg_iters,
                  r.rho, r.estimator_mode.c_str(), r.estimator_rank, r.err_est, r.t_residual, r.t_solve, r.t_setup,
                  r.t_estimator);
    os << buf;
  }
}
// proj/src/metrics.cpp:37-48
void write_solves_csv(const std::string& path, const std::vector<SolveRecord>& rows, const std::string& mode) {
  std::ofstream os(path);
  if (!os) throw ConfigError("cannot open for writing: " + path);
  os << "solve,t,estimator_mode,estimator_rank,iterations,initial_rel_residual\n";
  char buf[256];
  long i = 0;
  for (const auto& r : rows) {
    std::snprintf(buf, sizeof buf, "%ld,%.17g,%s,%d,%d,%.17g\n", i++, r.t, mode.c_str(), r.estimator_rank,
                  r.iterations, r.initial_rel_residual);
    os << buf;
  }
}
// proj/src/metrics.cpp:50-66
void write_probe_csv(const std::string& path, const std::vector<std::string>& names,
                     const std::vector<std::pair<double, std::vector<double>>>& rows) {
  std::ofstream os(path);
  if (!os) throw ConfigError("cannot open for writing: " + path);
  os << "t";
  for (const auto& n : names) os << "," << n;
  os << "\n";
  char buf[64];
  for (const auto& [t, values] : rows) {
    std::snprintf(buf, sizeof buf, "%.17g", t);
    os << buf;
    for (double v : values) {
      std::snprintf(buf, sizeof buf, ",%.17g", v);
      os << buf;
    }
    os << "\n";
  }
}

const char* estimator_mode_name(int m) {
  switch (m) {
    case 0: return "zero";
    case 1: return "previous";
    case 2: return "spe";
    case 3: return "pod_fixed";
    case 4: return "pod_rolling";
  }
  return "?";
}

RunResult run_scenario(const SimConfig& config, const std::string& out_dir, int device) {
  RunResult res;
  const auto wall0 = std::chrono::steady_clock::now();
  std::vector<std::string> probe_names;
  for (size_t p = 0; p < config.probes.size(); ++p) probe_names.push_back("p" + std::to_string(p));
  try {
    if (!out_dir.empty()) fs::create_directories(out_dir);
    Problem prob = build_problem(config);
    std::vector<PointLocation> locs;
    for (const auto& p : config.probes) {
      PointLocation loc;
      if (!locate_point(prob.mesh, p, loc)) throw ConfigError("probe point outside the mesh");
      locs.push_back(loc);
    }
    GpuSystem sys(std::move(prob), device);
    const Problem& P = sys.problem();
    std::vector<double> zero(sys.n_free(), 0.0);
    sys.set_state(0.0, zero.data(), config.dt0);
    RkcOptions opts;
    opts.rtol = config.tolerance;
    opts.atol = config.effective_atol();
    opts.max_stages = config.max_stages;
    std::vector<double> x_host, x_full;
    auto record_probes = [&]() {
      if (config.probes.empty()) return;
      x_host.resize(sys.n_free());
      x_full.resize(P.dm.n_dofs);
      sys.get_state(x_host.data());
      sys.lift_full_host(sys.state_t, x_host.data(), x_full.data());
      std::vector<double> vals;
      for (const auto& loc : locs) {
        double ev[10];
        for (int i = 0; i < P.dm.n_local; ++i) ev[i] = x_full[P.dm.element_dofs[(size_t)P.dm.n_local * loc.tet + i]];
        vals.push_back(interpolate(P.dm.order, ev, loc));
      }
      res.probe_rows.emplace_back(sys.state_t, std::move(vals));
    };
    record_probes();
    long step_index = 0, vtk_index = 0;
    int consecutive_rejections = 0;
    const double t_final = config.t_end * (1.0 - 1e-12);
    while (sys.state_t < t_final) {
      if (step_index > 500000) throw NumericalError("step limit exceeded");
      if (config.max_steps >= 0 && step_index >= config.max_steps) break;
      const SolveStats before = sys.stats();
      StepAttempt att;
      if (config.integrator == 0) {
        const double rho = sys.spectral_radius_cached(25);
        const double dt_stab = rho > 0 ? 1.8 / rho : config.dt0;
        const double dt = std::min({config.dt0, dt_stab, config.t_end - sys.state_t});
        att = sys.euler_step(dt);
        att.rho = rho;
        ++sys.rho_age;
      } else if (config.integrator == 2) {  // scenario.cpp:299-302
        sys.state_dt = std::min(sys.state_dt, config.t_end - sys.state_t);
        SdirkOptions so;
        so.rtol = opts.rtol;
        so.atol = opts.atol;
        att = sys.sdirk_step(so);
      } else {
        sys.state_dt = std::min(sys.state_dt, config.t_end - sys.state_t);
        att = sys.rkc_step(opts);
      }
      const SolveStats& after = sys.stats();
      StepMetrics row;
      row.step = step_index++;
      row.t = att.t_start;
      row.dt = att.dt;
      row.method = config.integrator == 0 ? "euler" : config.integrator == 2 ? "sdirk32" : "rkc";
      row.newton_iters = att.newton_iterations;
      row.accepted = att.accepted;
      row.stages = att.stages;
      row.m_solves = after.m_solves - before.m_solves;
      row.pcg_iters = after.pcg_iterations - before.pcg_iterations;
      row.rho = att.rho;
      row.estimator_mode = estimator_mode_name(config.solver.estimator_mode);
      row.estimator_rank = sys.solve_records().empty() ? 0 : sys.solve_records().back().estimator_rank;
      row.err_est = att.error;
      row.t_residual = after.t_residual - before.t_residual;
      row.t_solve = after.t_solve - before.t_solve;
      row.t_setup = after.t_setup - before.t_setup;
      row.t_estimator = after.t_estimator - before.t_estimator;
      res.steps.push_back(row);
      if (att.accepted) {
        consecutive_rejections = 0;
        record_probes();
        if (config.vtk_every > 0 && !config.vtk_prefix.empty() && sys.st_accepted % config.vtk_every == 0) {
          char name[256];
          std::snprintf(name, sizeof name, "%s_%06ld.vtk", config.vtk_prefix.c_str(), vtk_index++);
          x_host.resize(sys.n_free());
          x_full.resize(P.dm.n_dofs);
          sys.get_state(x_host.data());
          sys.lift_full_host(sys.state_t, x_host.data(), x_full.data());
          std::vector<double> kappa(P.mesh.n_tets);
          sys.cell_kappa_host(kappa.data());
          write_vtk(join_path(out_dir, name), P, x_full, kappa, config.vtk_binary);
        }
      } else if (++consecutive_rejections > 40) {
        throw NumericalError("no accepted step after 40 attempts");
      }
      if (!(sys.state_dt > 0) || !std::isfinite(sys.state_dt)) throw NumericalError("step size collapsed");
    }
    res.final_x_free.resize(sys.n_free());
    sys.get_state(res.final_x_free.data());
    res.final_t = sys.state_t;
    res.accepted = sys.st_accepted;
    res.rejected = sys.st_rejected;
    res.stages = sys.st_stages;
    res.stats = sys.stats();
    res.solves = sys.solve_records();
  } catch (const ConfigError& e) {
    res.exit_code = 1;
    res.error = e.what();
  } catch (const ParseError& e) {
    res.exit_code = 1;
    res.error = e.what();
  } catch (const GeometryError& e) {
    res.exit_code = 1;
    res.error = e.what();
  } catch (const std::invalid_argument& e) {
    res.exit_code = 1;
    res.error = e.what();
  } catch (const std::exception& e) {
    res.exit_code = 2;
    res.error = e.what();
  }
  res.wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  if (res.exit_code != 1) {
    if (!out_dir.empty()) fs::create_directories(out_dir);
    if (!config.metrics_csv.empty()) write_metrics_csv(join_path(out_dir, config.metrics_csv), res.steps);
    if (!config.probe_csv.empty()) write_probe_csv(join_path(out_dir, config.probe_csv), probe_names, res.probe_rows);
    if (!config.solves_csv.empty())
      write_solves_csv(join_path(out_dir, config.solves_csv), res.solves,
                       estimator_mode_name(config.solver.estimator_mode));
  }
  return res;
}

}  // namespace eqsb
