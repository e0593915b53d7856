// Scenario config parsing (proj/src/scenario.cpp:26-211, the reference JSON
// schema, proj/README.md:77-113) and problem construction
// (proj/src/scenario.cpp:224-236). Additive keys: mesh.box.jitter /
// jitter_seed, max_steps (bounded runs).
#include <algorithm>
#include <cmath>

#include "eqs_internal.hpp"
#include "nlohmann/json.hpp"

namespace eqsb {

using nlohmann::json;

namespace {
Waveform waveform_from_json(const json& j) {  // scenario.cpp:26-35
  const std::string kind = j.at("kind").get<std::string>();
  Waveform w;
  if (kind == "sinusoid") {
    w.kind = 0;
    w.amplitude = j.at("amplitude").get<double>();
    w.frequency = j.at("frequency").get<double>();
    w.phase = j.value("phase", 0.0);
  } else if (kind == "ramp") {
    w.kind = 1;
    w.amplitude = j.at("amplitude").get<double>();
    w.rise_time = j.at("rise_time").get<double>();
  } else if (kind == "constant") {
    w.kind = 2;
    w.value = j.at("value").get<double>();
  } else {
    throw ConfigError("unknown waveform kind '" + kind + "'");
  }
  return w;
}
Material material_from_json(const json& j) {  // scenario.cpp:37-53
  Material m;
  m.eps_r = j.at("eps_r").get<double>();
  const json& c = j.at("conductivity");
  const std::string kind = c.at("kind").get<std::string>();
  if (kind == "constant") {
    m.kind = 0;
    m.kappa = c.at("kappa").get<double>();
  } else if (kind == "microvaristor") {
    m.kind = 1;
    m.kappa_lo = c.value("kappa_lo", 1e-10);
    m.kappa_hi = c.value("kappa_hi", 1e-4);
    m.e_switch = c.value("e_switch", 5e5);
    m.width = c.value("width", 5e4);
  } else {
    throw ConfigError("unknown conductivity kind '" + kind + "'");
  }
  m.validate();
  return m;
}
}  // namespace

double SimConfig::effective_atol() const {  // scenario.cpp:90-100
  if (atol > 0) return atol;
  double amp = 0.0;
  for (const auto& [name, w] : excitations) {
    if (w.kind == 0 || w.kind == 1) amp = std::max(amp, std::abs(w.amplitude));
    if (w.kind == 2) amp = std::max(amp, std::abs(w.value));
  }
  return std::max(1e-6 * amp, 1e-12);
}

SimConfig parse_config(const std::string& text) {
  json j;
  try {
    j = json::parse(text);
  } catch (const json::exception& e) {
    throw ConfigError(std::string("config is not valid JSON: ") + e.what());
  }
  try {
    SimConfig c;
    c.name = j.value("name", c.name);
    const json& mesh = j.at("mesh");
    if (mesh.contains("file")) {
      c.has_file = true;
      c.mesh_file = mesh.at("file").get<std::string>();
    } else if (mesh.contains("box")) {
      const json& b = mesh.at("box");
      c.nx = b.at("nx").get<int>();
      c.ny = b.at("ny").get<int>();
      c.nz = b.at("nz").get<int>();
      c.lx = b.at("lx").get<double>();
      c.ly = b.at("ly").get<double>();
      c.lz = b.at("lz").get<double>();
      c.layers.z_planes = b.value("z_planes", std::vector<double>{});
      c.layers.regions = b.value("regions", std::vector<int>{1});
      c.jitter = b.value("jitter", 0.0);
      c.jitter_seed = b.value("jitter_seed", 1612u);
    } else {
      throw ConfigError("mesh: need either \"file\" or \"box\"");
    }
    c.order = j.value("order", 1);
    for (const auto& [key, jm] : j.at("materials").items()) {
      int region = 0;
      try {
        region = std::stoi(key);
      } catch (const std::exception&) {
        throw ConfigError("material key must be a region id, got '" + key + "'");
      }
      c.materials[region] = material_from_json(jm);
    }
    for (const auto& [key, jw] : j.at("excitations").items()) c.excitations[key] = waveform_from_json(jw);
    if (j.contains("integrator")) {
      const json& ji = j.at("integrator");
      const std::string kind = ji.value("kind", "rkc");
      if (kind == "euler") c.integrator = 0;
      else if (kind == "rkc") c.integrator = 1;
      else if (kind == "sdirk32") c.integrator = 2;
      else throw ConfigError("unknown integrator kind '" + kind + "'");
      c.tolerance = ji.value("tolerance", c.tolerance);
      c.atol = ji.value("atol", c.atol);
      c.t_end = ji.value("t_end", c.t_end);
      c.dt0 = ji.value("dt0", c.dt0);
      c.max_stages = ji.value("max_stages", c.max_stages);
    }
    if (!(c.tolerance > 0)) throw ConfigError("integrator tolerance must be positive");
    if (!(c.t_end > 0) || !(c.dt0 > 0)) throw ConfigError("t_end and dt0 must be positive");
    if (j.contains("solver")) {
      const json& js = j.at("solver");
      const std::string p = js.value("preconditioner", "amg");
      if (p == "jacobi") c.solver.precond = 0;
      else if (p == "ssor") c.solver.precond = 1;
      else if (p == "amg") c.solver.precond = 2;
      else throw ConfigError("unknown preconditioner '" + p + "'");
      c.solver.rel_tol = js.value("rel_tol", c.solver.rel_tol);
      c.solver.max_iter = js.value("max_iter", c.solver.max_iter);
      c.solver.amg_theta = js.value("amg_strength_threshold", c.solver.amg_theta);
      c.solver.amg_coarse_limit = js.value("amg_coarse_limit", c.solver.amg_coarse_limit);
      c.solver.amg_coarse_filter = js.value("amg_coarse_filter", c.solver.amg_coarse_filter);  // additive key
      if (js.contains("amg_vcycle_truncate")) {  // additive key: per-level thresholds, or 0 = off
        const json& jt = js.at("amg_vcycle_truncate");
        if (jt.is_number()) {
          if (jt.get<double>() != 0.0) throw ConfigError("solver amg_vcycle_truncate: a list of per-level thresholds or 0");
          c.solver.amg_vcycle_truncate.clear();
        } else if (jt.is_array()) {
          c.solver.amg_vcycle_truncate = jt.get<std::vector<double>>();
        } else {
          throw ConfigError("solver amg_vcycle_truncate: a list of per-level thresholds or 0");
        }
        for (double t : c.solver.amg_vcycle_truncate)
          if (!(t >= 0.0 && t < 1.0)) throw ConfigError("solver amg_vcycle_truncate thresholds must be in [0, 1)");
      }
      c.solver.amg_replicate_rows = js.value("amg_replicate_rows", c.solver.amg_replicate_rows);  // additive key
      c.solver.amg_dense_coarse = js.value("amg_dense_coarse", c.solver.amg_dense_coarse);        // additive key
      if (!(c.solver.rel_tol > 0)) throw ConfigError("solver rel_tol must be positive");
    }
    if (j.contains("estimator")) {
      const json& je = j.at("estimator");
      const std::string mode = je.value("mode", "zero");
      if (mode == "zero") c.solver.estimator_mode = 0;
      else if (mode == "previous") c.solver.estimator_mode = 1;
      else if (mode == "spe") c.solver.estimator_mode = 2;
      else if (mode == "pod_fixed") c.solver.estimator_mode = 3;
      else if (mode == "pod_rolling") c.solver.estimator_mode = 4;
      else throw ConfigError("unknown estimator mode '" + mode + "'");
      c.solver.spe_window = je.value("window", c.solver.spe_window);
      c.solver.pod_snapshots = je.value("snapshots", c.solver.pod_snapshots);  // scenario.cpp:64-67
      c.solver.pod_rank = je.value("rank", c.solver.pod_rank);
      c.solver.pod_capacity = je.value("capacity", c.solver.pod_capacity);
      c.solver.pod_threshold = je.value("threshold", c.solver.pod_threshold);
      c.solver.mgs_drop_tol = je.value("mgs_drop_tol", c.solver.mgs_drop_tol);
      if (c.solver.spe_window < 1 || c.solver.pod_snapshots < 1 || c.solver.pod_rank < 1 ||
          c.solver.pod_capacity < 1)
        throw ConfigError("estimator window/snapshot/rank/capacity values must be >= 1");
    }
    for (const auto& jp : j.value("probes", json::array())) {
      if (!jp.is_array() || jp.size() != 3) throw ConfigError("probe must be [x, y, z]");
      c.probes.push_back({jp[0].get<double>(), jp[1].get<double>(), jp[2].get<double>()});
    }
    if (j.contains("output")) {
      const json& jo = j.at("output");
      c.metrics_csv = jo.value("metrics_csv", c.metrics_csv);
      c.probe_csv = jo.value("probe_csv", c.probe_csv);
      c.solves_csv = jo.value("solves_csv", c.solves_csv);
      c.vtk_prefix = jo.value("vtk_prefix", c.vtk_prefix);
      c.vtk_every = jo.value("vtk_every", c.vtk_every);
      c.vtk_binary = jo.value("vtk_binary", c.vtk_binary);  // additive key
    }
    c.max_steps = j.value("max_steps", -1L);
    c.workers = j.value("workers", 1);
    if (c.workers < 1) throw ConfigError("workers must be >= 1");
    return c;
  } catch (const json::exception& e) {
    throw ConfigError(std::string("config: ") + e.what());
  }
}

Problem build_problem(const SimConfig& c) {
  Problem p;
  if (c.has_file) {
    p.mesh = load_msh(c.mesh_file);
  } else {
    p.mesh = generate_box_mesh(c.nx, c.ny, c.nz, c.lx, c.ly, c.lz, c.layers);
    if (c.jitter != 0.0) jitter_box_mesh(p.mesh, c.nx, c.ny, c.nz, c.lx, c.ly, c.lz, c.jitter, c.jitter_seed);
  }
  for (int t = 0; t < p.mesh.n_tets; ++t)
    if (!c.materials.count(p.mesh.region[t]))
      throw ConfigError("no material for mesh region " + std::to_string(p.mesh.region[t]));
  std::vector<std::string> dirichlet;
  for (const auto& [set, w] : c.excitations) dirichlet.push_back(set);
  p.dm = build_dof_map(p.mesh, c.order, dirichlet);
  for (const auto& name : p.dm.set_names) p.set_waveforms.push_back(c.excitations.at(name));
  p.materials = c.materials;
  p.solver = c.solver;
  return p;
}

}  // namespace eqsb
