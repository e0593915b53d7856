// Host mesh + dof setup. Bit-exact with the reference generator
// (proj/src/mesh.cpp:93-154), finalize (:57-91), MSH 2.2 reader
// (proj/src/msh_io.cpp:63-175) and build_dof_map (proj/src/dofmap.cpp:22-91),
// but written for 10^8-tet meshes: flat arrays, OpenMP over independent cells
// and tets, no per-node std::vector.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <fstream>
#include <random>
#include <set>
#include <sstream>
#include <unordered_map>

#include "eqs_internal.hpp"

namespace eqsb {

namespace {
inline double signed_volume(const double* a, const double* b, const double* c, const double* d) {
  const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const double e3[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                     e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
  return det / 6.0;
}
}  // namespace

// proj/src/mesh.cpp:57-91
void Mesh::finalize() {
  if (n_tets == 0) throw GeometryError("mesh has no tetrahedra");
  if ((int)region.size() != n_tets) throw GeometryError("region_id size does not match tet count");
  const int nn = n_nodes;
  long bad_range = -1, bad_degen = -1;
#pragma omp parallel for schedule(static) reduction(max : bad_range, bad_degen)
  for (long t = 0; t < n_tets; ++t) {
    int* k = &tets[4 * t];
    bool ok = true;
    for (int i = 0; i < 4; ++i)
      if (k[i] < 0 || k[i] >= nn) ok = false;
    if (!ok) {
      bad_range = std::max(bad_range, (long)n_tets - t);  // smallest t wins
      continue;
    }
    double v = signed_volume(&nodes[3 * k[0]], &nodes[3 * k[1]], &nodes[3 * k[2]], &nodes[3 * k[3]]);
    if (v < 0.0) {
      std::swap(k[2], k[3]);
      v = -v;
    }
    double h = 0.0;
    for (int i = 0; i < 4; ++i)
      for (int j = i + 1; j < 4; ++j) {
        const double* a = &nodes[3 * k[i]];
        const double* b = &nodes[3 * k[j]];
        const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
        h = std::max(h, std::sqrt(dx * dx + dy * dy + dz * dz));
      }
    if (!(v > 1e-14 * h * h * h)) bad_degen = std::max(bad_degen, (long)n_tets - t);
  }
  if (bad_range >= 0 || bad_degen >= 0) {
    const long tr = bad_range >= 0 ? n_tets - bad_range : n_tets;
    const long td = bad_degen >= 0 ? n_tets - bad_degen : n_tets;
    if (tr <= td) throw GeometryError("tet " + std::to_string(tr) + " references node out of range");
    throw GeometryError("tet " + std::to_string(td) + " is degenerate");
  }
  std::map<int, std::string> owner;
  for (auto& [name, set] : boundary_sets) {
    std::sort(set.begin(), set.end());
    set.erase(std::unique(set.begin(), set.end()), set.end());
    for (int n : set) {
      if (n < 0 || n >= nn) throw GeometryError("boundary set '" + name + "' references node out of range");
      auto [it, inserted] = owner.emplace(n, name);
      if (!inserted)
        throw GeometryError("boundary sets '" + it->second + "' and '" + name + "' overlap at node " +
                            std::to_string(n));
    }
  }
}

// proj/src/mesh.cpp:93-154
Mesh generate_box_mesh(int nx, int ny, int nz, double lx, double ly, double lz, const LayerSpec& layers) {
  if (nx < 1 || ny < 1 || nz < 1) throw std::invalid_argument("generate_box_mesh: cell counts must be >= 1");
  if (!(lx > 0.0 && ly > 0.0 && lz > 0.0)) throw std::invalid_argument("generate_box_mesh: extents must be positive");
  if (layers.regions.size() != layers.z_planes.size() + 1)
    throw std::invalid_argument("generate_box_mesh: need one region per layer");
  for (double z : layers.z_planes)
    if (!(z > 0.0 && z < lz)) throw std::invalid_argument("generate_box_mesh: layer plane outside (0, lz)");
  const long n_nodes = (long)(nx + 1) * (ny + 1) * (nz + 1);
  const long n_tets = 6L * nx * ny * nz;
  if (n_nodes >= (1L << 31) || n_tets >= (1L << 31)) throw std::invalid_argument("generate_box_mesh: mesh too large");
  Mesh m;
  m.n_nodes = (int)n_nodes;
  m.n_tets = (int)n_tets;
  m.nodes.resize(3 * n_nodes);
  m.tets.resize(4 * n_tets);
  m.region.resize(n_tets);
  auto node_id = [&](int i, int j, int k) { return (k * (ny + 1) + j) * (nx + 1) + i; };
#pragma omp parallel for schedule(static)
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        double* p = &m.nodes[3L * node_id(i, j, k)];
        p[0] = lx * i / nx;
        p[1] = ly * j / ny;
        p[2] = lz * k / nz;
      }
  static const int paths[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
#pragma omp parallel for schedule(static)
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const long cell = ((long)k * ny + j) * nx + i;
        for (int pi = 0; pi < 6; ++pi) {
          const long t = 6 * cell + pi;
          int pos[3] = {i, j, k};
          int* tet = &m.tets[4 * t];
          tet[0] = node_id(pos[0], pos[1], pos[2]);
          for (int s = 0; s < 3; ++s) {
            ++pos[paths[pi][s]];
            tet[s + 1] = node_id(pos[0], pos[1], pos[2]);
          }
          double zc = 0.0;  // TetMesh::tet_centroid (mesh.cpp:48-53), same summation order
          for (int v = 0; v < 4; ++v) zc += 0.25 * m.nodes[3L * tet[v] + 2];
          size_t layer = 0;
          while (layer < layers.z_planes.size() && zc >= layers.z_planes[layer]) ++layer;
          m.region[t] = layers.regions[layer];
        }
      }
  const double ztol = 1e-12 * lz;
  std::vector<int> ground, hv;
  for (long n = 0; n < n_nodes; ++n) {
    const double z = m.nodes[3 * n + 2];
    if (std::abs(z) <= ztol) ground.push_back((int)n);
    if (std::abs(z - lz) <= ztol) hv.push_back((int)n);
  }
  m.boundary_sets["ground"] = std::move(ground);
  m.boundary_sets["hv"] = std::move(hv);
  m.finalize();
  return m;
}

// Additive interior jitter; identical to oracle/mesh_dof.cpp.
void jitter_box_mesh(Mesh& m, int nx, int ny, int nz, double lx, double ly, double lz, double amplitude,
                     unsigned seed) {
  if (amplitude == 0.0) return;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  const int n[3] = {nx, ny, nz};
  const double h[3] = {lx / nx, ly / ny, lz / nz};
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const long id = ((long)k * (ny + 1) + j) * (nx + 1) + i;
        const int idx[3] = {i, j, k};
        double u[3];
        for (int d = 0; d < 3; ++d) u[d] = uni(rng);
        for (int d = 0; d < 3; ++d)
          if (idx[d] > 0 && idx[d] < n[d]) m.nodes[3 * id + d] += amplitude * h[d] * u[d];
      }
  m.finalize();
}

// proj/src/msh_io.cpp:63-175
Mesh load_msh(const std::string& path) {
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
    if (!next(l)) throw ParseError("unexpected end of file in " + ctx + " (line " + std::to_string(line_no) + ")");
    return l;
  };
  auto count = [&](const std::string& l, const std::string& sec) {
    try {
      long n = std::stol(l);
      if (n < 0) throw std::invalid_argument("negative");
      return n;
    } catch (const std::exception&) {
      throw ParseError("bad count in " + sec + ": '" + l + "' (line " + std::to_string(line_no) + ")");
    }
  };
  std::string line = need("$MeshFormat");
  if (line != "$MeshFormat") throw ParseError("expected $MeshFormat header, got '" + line + "'");
  line = need("$MeshFormat");
  {
    std::istringstream ss(line);
    std::string version;
    int ft = -1, ds = -1;
    ss >> version >> ft >> ds;
    if (version.rfind("2.2", 0) != 0 || ft != 0)
      throw ParseError("unsupported mesh format '" + line + "' (need MSH 2.2 ASCII)");
  }
  if (need("$MeshFormat") != "$EndMeshFormat") throw ParseError("expected $EndMeshFormat");
  std::map<int, std::string> surface_names;
  std::unordered_map<long, int> node_of_id;
  Mesh mesh;
  std::map<std::string, std::set<int>> sets;
  while (next(line)) {
    if (line == "$PhysicalNames") {
      const long n = count(need("$PhysicalNames"), "$PhysicalNames");
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$PhysicalNames"));
        int dim = 0, id = 0;
        ss >> dim >> id;
        std::string name;
        std::getline(ss, name);
        const auto a = name.find('"');
        const auto b = name.rfind('"');
        if (a == std::string::npos || b <= a) throw ParseError("malformed physical name '" + name + "'");
        if (dim == 2) surface_names[id] = name.substr(a + 1, b - a - 1);
      }
      if (need("$PhysicalNames") != "$EndPhysicalNames") throw ParseError("expected $EndPhysicalNames");
    } else if (line == "$Nodes") {
      const long n = count(need("$Nodes"), "$Nodes");
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$Nodes"));
        long id = 0;
        double x = 0, y = 0, z = 0;
        if (!(ss >> id >> x >> y >> z)) throw ParseError("malformed node line in $Nodes");
        node_of_id[id] = mesh.n_nodes++;
        mesh.nodes.insert(mesh.nodes.end(), {x, y, z});
      }
      if (need("$Nodes") != "$EndNodes") throw ParseError("expected $EndNodes");
    } else if (line == "$Elements") {
      const long n = count(need("$Elements"), "$Elements");
      auto node = [&](long id) {
        auto it = node_of_id.find(id);
        if (it == node_of_id.end()) throw ParseError("element references unknown node " + std::to_string(id));
        return it->second;
      };
      for (long i = 0; i < n; ++i) {
        std::istringstream ss(need("$Elements"));
        long id = 0;
        int type = 0, ntags = 0;
        if (!(ss >> id >> type >> ntags)) throw ParseError("malformed element line in $Elements");
        int phys = 0;
        for (int t = 0; t < ntags; ++t) {
          int tag = 0;
          if (!(ss >> tag)) throw ParseError("missing element tag in $Elements");
          if (t == 0) phys = tag;
        }
        if (type == 4) {
          long a, b, c, d;
          if (!(ss >> a >> b >> c >> d)) throw ParseError("tetrahedron with missing nodes in $Elements");
          mesh.tets.insert(mesh.tets.end(), {node(a), node(b), node(c), node(d)});
          mesh.region.push_back(phys);
          ++mesh.n_tets;
        } else if (type == 2) {
          long a, b, c;
          if (!(ss >> a >> b >> c)) throw ParseError("triangle with missing nodes in $Elements");
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
  if (mesh.n_tets == 0) throw GeometryError("mesh file contains no tetrahedra: " + path);
  mesh.finalize();
  return mesh;
}

// proj/src/dofmap.cpp:22-91. Edge ids are assigned in first-encounter order
// (dofmap.cpp:42-43); a hash map gives the same ids as the reference's std::map
// because the id is the map size at insertion.
Dofs build_dof_map(const Mesh& mesh, int order, const std::vector<std::string>& dirichlet_sets) {
  if (order != 1 && order != 2) throw ConfigError("element order must be 1 or 2");
  Dofs dm;
  dm.order = order;
  dm.n_local = order == 1 ? 4 : 10;
  const int nt = mesh.n_tets, nn = mesh.n_nodes;
  dm.element_dofs.resize((size_t)dm.n_local * nt);
  std::vector<std::pair<int, int>> edges;  // edge id -> sorted node pair
  if (order == 1) {
    std::copy(mesh.tets.begin(), mesh.tets.end(), dm.element_dofs.begin());
  } else {
    std::unordered_map<uint64_t, int> edge_id;
    edge_id.reserve((size_t)nt * 2);
    for (int t = 0; t < nt; ++t) {
      int* ed = &dm.element_dofs[(size_t)10 * t];
      for (int v = 0; v < 4; ++v) ed[v] = mesh.tets[4L * t + v];
      for (int e = 0; e < 6; ++e) {
        int a = mesh.tets[4L * t + kTetEdgeVertices[e][0]];
        int b = mesh.tets[4L * t + kTetEdgeVertices[e][1]];
        if (a > b) std::swap(a, b);
        const uint64_t key = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
        auto [it, inserted] = edge_id.try_emplace(key, (int)edges.size());
        if (inserted) edges.emplace_back(a, b);
        ed[4 + e] = nn + it->second;
      }
    }
  }
  dm.n_dofs = nn + (int)edges.size();
  std::vector<int> node_set(nn, -1);
  for (const auto& name : dirichlet_sets) {
    auto it = mesh.boundary_sets.find(name);
    if (it == mesh.boundary_sets.end()) throw ConfigError("unknown boundary set '" + name + "'");
    const int set_idx = (int)dm.set_names.size();
    dm.set_names.push_back(name);
    for (int n : it->second) node_set[n] = set_idx;
  }
  dm.fixed_set.assign(dm.n_dofs, -1);
  std::copy(node_set.begin(), node_set.end(), dm.fixed_set.begin());
  for (size_t e = 0; e < edges.size(); ++e) {
    const int sa = node_set[edges[e].first], sb = node_set[edges[e].second];
    if (sa >= 0 && sa == sb) dm.fixed_set[nn + e] = sa;
  }
  for (int d = 0; d < dm.n_dofs; ++d) {
    if (dm.fixed_set[d] >= 0) dm.fixed_dofs.push_back(d);
    else dm.free_dofs.push_back(d);
  }
  return dm;
}

// proj/src/materials.cpp:10-23
void Material::validate() const {
  if (!(eps_r > 0.0)) throw ConfigError("material: eps_r must be positive");
  if (kind == 0) {
    if (!(kappa >= 0.0)) throw ConfigError("material: kappa must be non-negative");
  } else {
    if (!(kappa_lo > 0.0 && kappa_hi > 0.0)) throw ConfigError("microvaristor: conductivities must be positive");
    if (!(kappa_hi >= kappa_lo)) throw ConfigError("microvaristor: kappa_hi must be >= kappa_lo");
    if (!(e_switch > 0.0)) throw ConfigError("microvaristor: e_switch must be positive");
    if (!(width > 0.0)) throw ConfigError("microvaristor: width must be positive");
  }
}

// proj/src/excitation.cpp:10-26
double Waveform::value_at(double t) const {
  if (kind == 0) return amplitude * std::sin(2.0 * M_PI * frequency * t + phase);
  if (kind == 1) return t >= rise_time ? amplitude : amplitude * t / rise_time;
  return value;
}
double Waveform::rate_at(double t) const {
  if (kind == 0) {
    const double om = 2.0 * M_PI * frequency;
    return amplitude * om * std::cos(om * t + phase);
  }
  if (kind == 1) return t >= rise_time ? 0.0 : amplitude / rise_time;
  return 0.0;
}

}  // namespace eqsb
