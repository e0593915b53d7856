// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp header).
// Restates proj/src/mesh.cpp, msh_io.cpp (load_msh), dofmap.cpp, materials.cpp,
// excitation.cpp.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <map>
#include <numbers>
#include <random>
#include <set>
#include <sstream>

#include "oracle.hpp"

namespace ora {

namespace {
// proj/src/mesh.cpp:14-24
double signed_volume(const std::array<double, 3>& a, const std::array<double, 3>& b,
                     const std::array<double, 3>& c, const std::array<double, 3>& d) {
  const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double e3[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) -
                     e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                     e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
  return det / 6.0;
}
// proj/src/mesh.cpp:26-37
double max_edge_length(const TetMesh& m, int t) {
  double h = 0.0;
  for (int i = 0; i < 4; ++i)
    for (int j = i + 1; j < 4; ++j) {
      const auto& a = m.nodes[m.tets[t][i]];
      const auto& b = m.nodes[m.tets[t][j]];
      const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
      h = std::max(h, std::sqrt(dx * dx + dy * dy + dz * dz));
    }
  return h;
}
}  // namespace

double TetMesh::tet_volume(int t) const {
  const auto& k = tets[t];
  return signed_volume(nodes[k[0]], nodes[k[1]], nodes[k[2]], nodes[k[3]]);
}

// proj/src/mesh.cpp:48-53
std::array<double, 3> TetMesh::tet_centroid(int t) const {
  std::array<double, 3> c = {0, 0, 0};
  for (int i = 0; i < 4; ++i)
    for (int d = 0; d < 3; ++d) c[d] += 0.25 * nodes[tets[t][i]][d];
  return c;
}

// proj/src/mesh.cpp:57-91
void TetMesh::finalize() {
  if (tets.empty()) throw GeometryError("mesh has no tetrahedra");
  if (region_id.size() != tets.size()) throw GeometryError("region_id size does not match tet count");
  const int nn = n_nodes();
  for (int t = 0; t < n_tets(); ++t) {
    for (int i = 0; i < 4; ++i)
      if (tets[t][i] < 0 || tets[t][i] >= nn)
        throw GeometryError("tet " + std::to_string(t) + " references node out of range");
    double v = tet_volume(t);
    if (v < 0.0) {
      std::swap(tets[t][2], tets[t][3]);
      v = -v;
    }
    const double h = max_edge_length(*this, t);
    if (!(v > 1e-14 * h * h * h)) throw GeometryError("tet " + std::to_string(t) + " is degenerate");
  }
  std::map<int, std::string> owner;
  for (auto& [name, set] : boundary_sets) {
    std::sort(set.begin(), set.end());
    set.erase(std::unique(set.begin(), set.end()), set.end());
    for (int n : set) {
      if (n < 0 || n >= nn) throw GeometryError("boundary set '" + name + "' references node out of range");
      auto [it, inserted] = owner.emplace(n, name);
      if (!inserted) throw GeometryError("boundary sets '" + it->second + "' and '" + name + "' overlap");
    }
  }
}

// proj/src/mesh.cpp:93-154
TetMesh generate_box_mesh(int nx, int ny, int nz, double lx, double ly, double lz,
                          const LayerSpec& layers) {
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("generate_box_mesh: cell counts must be >= 1");
  if (!(lx > 0.0 && ly > 0.0 && lz > 0.0)) throw std::invalid_argument("generate_box_mesh: extents must be positive");
  if (layers.regions.size() != layers.z_planes.size() + 1)
    throw std::invalid_argument("generate_box_mesh: need one region per layer");
  for (double z : layers.z_planes)
    if (!(z > 0.0 && z < lz)) throw std::invalid_argument("generate_box_mesh: layer plane outside (0, lz)");

  TetMesh m;
  const auto node_id = [&](int i, int j, int k) { return (k * (ny + 1) + j) * (nx + 1) + i; };
  m.nodes.resize((size_t)(nx + 1) * (ny + 1) * (nz + 1));
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) m.nodes[node_id(i, j, k)] = {lx * i / nx, ly * j / ny, lz * k / nz};

  static const int paths[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  m.tets.reserve((size_t)6 * nx * ny * nz);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const int base[3] = {i, j, k};
        for (const auto& p : paths) {
          std::array<int, 4> tet;
          int pos[3] = {base[0], base[1], base[2]};
          tet[0] = node_id(pos[0], pos[1], pos[2]);
          for (int s = 0; s < 3; ++s) {
            ++pos[p[s]];
            tet[s + 1] = node_id(pos[0], pos[1], pos[2]);
          }
          m.tets.push_back(tet);
        }
      }
  m.region_id.resize(m.tets.size());
  for (int t = 0; t < m.n_tets(); ++t) {
    const double zc = m.tet_centroid(t)[2];
    size_t layer = 0;
    while (layer < layers.z_planes.size() && zc >= layers.z_planes[layer]) ++layer;
    m.region_id[t] = layers.regions[layer];
  }
  const double ztol = 1e-12 * lz;
  std::vector<int> ground, hv;
  for (int n = 0; n < m.n_nodes(); ++n) {
    if (std::abs(m.nodes[n][2]) <= ztol) ground.push_back(n);
    if (std::abs(m.nodes[n][2] - lz) <= ztol) hv.push_back(n);
  }
  m.boundary_sets["ground"] = std::move(ground);
  m.boundary_sets["hv"] = std::move(hv);
  m.finalize();
  return m;
}

// Additive jitter: for every node in id order draw three
// uniform[-1,1) values from mt19937(seed); move coordinate d by
// amplitude * h_d * u_d unless the node lies on a boundary face normal to d.
// Then re-run finalize() (orientation + validation).
void jitter_box_mesh(TetMesh& m, int nx, int ny, int nz, double lx, double ly, double lz,
                     double amplitude, unsigned seed) {
  if (amplitude == 0.0) return;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  const int n[3] = {nx, ny, nz};
  const double h[3] = {lx / nx, ly / ny, lz / nz};
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const int id = (k * (ny + 1) + j) * (nx + 1) + i;
        const int idx[3] = {i, j, k};
        double u[3];
        for (int d = 0; d < 3; ++d) u[d] = uni(rng);
        for (int d = 0; d < 3; ++d)
          if (idx[d] > 0 && idx[d] < n[d]) m.nodes[id][d] += amplitude * h[d] * u[d];
      }
  m.finalize();
}

// proj/src/msh_io.cpp:63-175 (MSH 2.2 ASCII reader)
TetMesh load_msh(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw ParseError("cannot open mesh file: " + path);
  long line_no = 0;
  auto next = [&](std::string& line) {
    while (std::getline(is, line)) {
      ++line_no;
      while (!line.empty() && (line.back() == '\r' || line.back() == '\n')) line.pop_back();
      if (!line.empty()) return true;
    }
    return false;
  };
  auto need = [&](const std::string& ctx) {
    std::string l;
    if (!next(l)) throw ParseError("unexpected end of file in " + ctx);
    return l;
  };
  auto count = [&](const std::string& l) {
    try {
      long n = std::stol(l);
      if (n < 0) throw std::invalid_argument("neg");
      return n;
    } catch (const std::exception&) {
      throw ParseError("bad count: '" + l + "'");
    }
  };
  std::string line = need("$MeshFormat");
  if (line != "$MeshFormat") throw ParseError("expected $MeshFormat header");
  line = need("$MeshFormat");
  {
    std::istringstream ss(line);
    std::string version;
    int ft = -1, ds = -1;
    ss >> version >> ft >> ds;
    if (version.rfind("2.2", 0) != 0 || ft != 0) throw ParseError("unsupported mesh format");
  }
  if (need("$MeshFormat") != "$EndMeshFormat") throw ParseError("expected $EndMeshFormat");
  std::map<int, std::string> surface_names;
  std::map<long, int> node_of_id;
  TetMesh mesh;
  std::map<std::string, std::set<int>> sets;
  while (next(line)) {
    if (line == "$PhysicalNames") {
      const long n = count(need("$PhysicalNames"));
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$PhysicalNames"));
        int dim = 0, id = 0;
        ss >> dim >> id;
        std::string name;
        std::getline(ss, name);
        const auto a = name.find('"');
        const auto b = name.rfind('"');
        if (a == std::string::npos || b <= a) throw ParseError("malformed physical name");
        if (dim == 2) surface_names[id] = name.substr(a + 1, b - a - 1);
      }
      if (need("$PhysicalNames") != "$EndPhysicalNames") throw ParseError("expected $EndPhysicalNames");
    } else if (line == "$Nodes") {
      const long n = count(need("$Nodes"));
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$Nodes"));
        long id = 0;
        double x = 0, y = 0, z = 0;
        if (!(ss >> id >> x >> y >> z)) throw ParseError("malformed node line in $Nodes");
        node_of_id[id] = mesh.n_nodes();
        mesh.nodes.push_back({x, y, z});
      }
      if (need("$Nodes") != "$EndNodes") throw ParseError("expected $EndNodes");
    } else if (line == "$Elements") {
      const long n = count(need("$Elements"));
      auto node = [&](long id) {
        auto it = node_of_id.find(id);
        if (it == node_of_id.end()) throw ParseError("element references unknown node");
        return it->second;
      };
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$Elements"));
        long id = 0;
        int type = 0, ntags = 0;
        if (!(ss >> id >> type >> ntags)) throw ParseError("malformed element line");
        int phys = 0;
        for (int t = 0; t < ntags; ++t) {
          int tag = 0;
          if (!(ss >> tag)) throw ParseError("missing element tag");
          if (t == 0) phys = tag;
        }
        if (type == 4) {
          long a, b, c, d;
          if (!(ss >> a >> b >> c >> d)) throw ParseError("tetrahedron with missing nodes");
          mesh.tets.push_back({node(a), node(b), node(c), node(d)});
          mesh.region_id.push_back(phys);
        } else if (type == 2) {
          long a, b, c;
          if (!(ss >> a >> b >> c)) throw ParseError("triangle with missing nodes");
          auto it = surface_names.find(phys);
          const std::string name = it != surface_names.end() ? it->second : "surface_" + std::to_string(phys);
          auto& s = sets[name];
          s.insert(node(a));
          s.insert(node(b));
          s.insert(node(c));
        }
      }
      if (need("$Elements") != "$EndElements") throw ParseError("expected $EndElements");
    } else if (!line.empty() && line[0] == '$' && line.rfind("$End", 0) != 0) {
      const std::string end = "$End" + line.substr(1);
      std::string skip;
      while (next(skip))
        if (skip == end) break;
    }
  }
  for (auto& [name, s] : sets) mesh.boundary_sets[name] = {s.begin(), s.end()};
  if (mesh.tets.empty()) throw GeometryError("mesh file contains no tetrahedra: " + path);
  mesh.finalize();
  return mesh;
}

// proj/src/dofmap.cpp:11-20
void DofMap::lift(const Vec& x_free, const Vec& x_fixed, Vec& x_full) const {
  x_full.resize(n_dofs);
  for (int i = 0; i < n_free(); ++i) x_full[free_dofs[i]] = x_free[i];
  for (int i = 0; i < n_fixed(); ++i) x_full[fixed_dofs[i]] = x_fixed[i];
}
void DofMap::restrict_free(const Vec& x_full, Vec& x_free) const {
  x_free.resize(n_free());
  for (int i = 0; i < n_free(); ++i) x_free[i] = x_full[free_dofs[i]];
}

// proj/src/dofmap.cpp:22-91
DofMap build_dof_map(const TetMesh& mesh, int order, const std::vector<std::string>& dirichlet_sets) {
  if (order != 1 && order != 2) throw ConfigError("element order must be 1 or 2");
  DofMap dm;
  dm.order = order;
  dm.n_local = order == 1 ? 4 : 10;
  dm.dof_coords = mesh.nodes;
  std::map<std::pair<int, int>, int> edge_id;
  dm.element_dofs.resize(mesh.n_tets());
  for (int t = 0; t < mesh.n_tets(); ++t) {
    auto& ed = dm.element_dofs[t];
    ed.fill(-1);
    for (int v = 0; v < 4; ++v) ed[v] = mesh.tets[t][v];
    if (order == 2) {
      for (int e = 0; e < 6; ++e) {
        int a = mesh.tets[t][kTetEdgeVertices[e][0]];
        int b = mesh.tets[t][kTetEdgeVertices[e][1]];
        if (a > b) std::swap(a, b);
        auto [it, inserted] = edge_id.try_emplace({a, b}, (int)edge_id.size());
        ed[4 + e] = mesh.n_nodes() + it->second;
      }
    }
  }
  dm.n_dofs = mesh.n_nodes() + (int)edge_id.size();
  if (order == 2) {
    dm.dof_coords.resize(dm.n_dofs);
    for (const auto& [pair, id] : edge_id) {
      const auto& a = mesh.nodes[pair.first];
      const auto& b = mesh.nodes[pair.second];
      dm.dof_coords[mesh.n_nodes() + id] = {0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1]), 0.5 * (a[2] + b[2])};
    }
  }
  std::vector<int> node_set(mesh.n_nodes(), -1);
  for (const auto& name : dirichlet_sets) {
    auto it = mesh.boundary_sets.find(name);
    if (it == mesh.boundary_sets.end()) throw ConfigError("unknown boundary set '" + name + "'");
    const int set_idx = (int)dm.set_names.size();
    dm.set_names.push_back(name);
    for (int n : it->second) node_set[n] = set_idx;
  }
  dm.fixed_set.assign(dm.n_dofs, -1);
  for (int n = 0; n < mesh.n_nodes(); ++n) dm.fixed_set[n] = node_set[n];
  if (order == 2)
    for (const auto& [pair, id] : edge_id) {
      const int sa = node_set[pair.first], sb = node_set[pair.second];
      if (sa >= 0 && sa == sb) dm.fixed_set[mesh.n_nodes() + id] = sa;
    }
  dm.free_index.assign(dm.n_dofs, -1);
  dm.fixed_index.assign(dm.n_dofs, -1);
  for (int d = 0; d < dm.n_dofs; ++d) {
    if (dm.fixed_set[d] >= 0) {
      dm.fixed_index[d] = (int)dm.fixed_dofs.size();
      dm.fixed_dofs.push_back(d);
    } else {
      dm.free_index[d] = (int)dm.free_dofs.size();
      dm.free_dofs.push_back(d);
    }
  }
  return dm;
}

// proj/src/materials.cpp:10-23
void MaterialModel::validate() const {
  if (!(eps_r > 0.0)) throw ConfigError("material: eps_r must be positive");
  if (const auto* c = std::get_if<ConstantConductivity>(&conductivity)) {
    if (!(c->kappa >= 0.0)) throw ConfigError("material: kappa must be non-negative");
  } else {
    const auto& mv = std::get<MicrovaristorConductivity>(conductivity);
    if (!(mv.kappa_lo > 0.0 && mv.kappa_hi > 0.0)) throw ConfigError("microvaristor: conductivities must be positive");
    if (!(mv.kappa_hi >= mv.kappa_lo)) throw ConfigError("microvaristor: kappa_hi must be >= kappa_lo");
    if (!(mv.e_switch > 0.0)) throw ConfigError("microvaristor: e_switch must be positive");
    if (!(mv.width > 0.0)) throw ConfigError("microvaristor: width must be positive");
  }
}

// proj/src/materials.cpp:25-33
double kappa_of_e(const MaterialModel& m, double e_mag) {
  if (!(e_mag >= 0.0)) throw std::invalid_argument("kappa_of_e: negative field magnitude");
  if (const auto* c = std::get_if<ConstantConductivity>(&m.conductivity)) return c->kappa;
  const auto& mv = std::get<MicrovaristorConductivity>(m.conductivity);
  const double lo = std::log10(mv.kappa_lo);
  const double hi = std::log10(mv.kappa_hi);
  const double s = 0.5 * (1.0 + std::tanh((e_mag - mv.e_switch) / mv.width));
  return std::pow(10.0, lo + (hi - lo) * s);
}

// proj/src/excitation.cpp:10-26
double waveform_value(const Waveform& w, double t) {
  if (const auto* s = std::get_if<SinusoidWaveform>(&w))
    return s->amplitude * std::sin(2.0 * std::numbers::pi * s->frequency * t + s->phase);
  if (const auto* r = std::get_if<RampWaveform>(&w))
    return t >= r->rise_time ? r->amplitude : r->amplitude * t / r->rise_time;
  return std::get<ConstantWaveform>(w).value;
}
double waveform_rate(const Waveform& w, double t) {
  if (const auto* s = std::get_if<SinusoidWaveform>(&w)) {
    const double om = 2.0 * std::numbers::pi * s->frequency;
    return s->amplitude * om * std::cos(om * t + s->phase);
  }
  if (const auto* r = std::get_if<RampWaveform>(&w)) return t >= r->rise_time ? 0.0 : r->amplitude / r->rise_time;
  return 0.0;
}
// proj/src/excitation.cpp:28-54
double BoundaryExcitation::value(const std::string& set, double t) const {
  auto it = per_set.find(set);
  if (it == per_set.end()) throw ConfigError("no excitation for boundary set '" + set + "'");
  return waveform_value(it->second, t);
}
double BoundaryExcitation::rate(const std::string& set, double t) const {
  auto it = per_set.find(set);
  if (it == per_set.end()) throw ConfigError("no excitation for boundary set '" + set + "'");
  return waveform_rate(it->second, t);
}
Vec BoundaryExcitation::boundary_values(const DofMap& dm, double t) const {
  Vec xb(dm.n_fixed());
  std::vector<double> per(dm.set_names.size());
  for (size_t s = 0; s < dm.set_names.size(); ++s) per[s] = value(dm.set_names[s], t);
  for (int i = 0; i < dm.n_fixed(); ++i) xb[i] = per[dm.fixed_set[dm.fixed_dofs[i]]];
  return xb;
}
Vec BoundaryExcitation::boundary_rates(const DofMap& dm, double t) const {
  Vec xb(dm.n_fixed());
  std::vector<double> per(dm.set_names.size());
  for (size_t s = 0; s < dm.set_names.size(); ++s) per[s] = rate(dm.set_names[s], t);
  for (int i = 0; i < dm.n_fixed(); ++i) xb[i] = per[dm.fixed_set[dm.fixed_dofs[i]]];
  return xb;
}

// proj/tests/support/test_helpers.hpp:15-21
Vec random_vec(int n, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  Vec v(n);
  for (int i = 0; i < n; ++i) v[i] = uni(rng);
  return v;
}

}  // namespace ora
