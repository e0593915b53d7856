// Element geometry and local weighted Laplacian, host + device. Same operation
// order as proj/src/assembly.cpp:34-116 so that host-assembled matrices are
// bit-identical to the reference restatement (compiled with FMA contraction
// off on the host).
#pragma once

#ifdef __CUDACC__
#define EQS_HD __host__ __device__ __forceinline__
#else
#define EQS_HD inline
#endif

namespace eqsb {

// proj/src/assembly.cpp:13-18
constexpr double kQa = 0.58541019662496845446;
constexpr double kQb = 0.13819660112501051518;

struct TetGeo {
  double g[4][3] = {};  // barycentric gradients grad(lambda_i)
  double volume = 0.0;
  double det = 0.0;
};

// proj/src/assembly.cpp:34-61. Returns false for det == 0 (GeometryError).
EQS_HD bool tet_geometry(const double p[4][3], TetGeo& geo) {
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
  geo.det = det;
  if (det == 0.0) return false;
  geo.volume = det / 6.0;
  for (int i = 0; i < 3; ++i)
    for (int d = 0; d < 3; ++d) geo.g[i + 1][d] = cr[i][d] / det;
  for (int d = 0; d < 3; ++d) geo.g[0][d] = -geo.g[1][d] - geo.g[2][d] - geo.g[3][d];
  return true;
}

// proj/src/assembly.cpp:69-85 for order 2 at quadrature point q.
EQS_HD void p2_gradients(const TetGeo& geo, int q, double grads[10][3]) {
  double lam[4];
  for (int i = 0; i < 4; ++i) lam[i] = (i == q) ? kQa : kQb;
  for (int i = 0; i < 4; ++i) {
    const double f = 4.0 * lam[i] - 1.0;
    for (int d = 0; d < 3; ++d) grads[i][d] = f * geo.g[i][d];
  }
  const int ev[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  for (int e = 0; e < 6; ++e) {
    const int a = ev[e][0], b = ev[e][1];
    for (int d = 0; d < 3; ++d) grads[4 + e][d] = 4.0 * (lam[a] * geo.g[b][d] + lam[b] * geo.g[a][d]);
  }
}

// Lower triangle of S = sum_q w_q c_q grad N_i . grad N_j (proj/src/assembly.cpp:97-116),
// packed row-major: S[i*(i+1)/2 + j], j <= i.
EQS_HD void element_laplacian_p1(const TetGeo& geo, double coeff, double S[10]) {
  const double wc = geo.volume * coeff;
  int k = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j <= i; ++j) {
      const double gij = geo.g[i][0] * geo.g[j][0] + geo.g[i][1] * geo.g[j][1] + geo.g[i][2] * geo.g[j][2];
      S[k++] = 0.0 + wc * gij;
    }
}

EQS_HD void element_laplacian_p2(const TetGeo& geo, const double coeff[4], double S[55]) {
  for (int k = 0; k < 55; ++k) S[k] = 0.0;
  double grads[10][3];
  for (int q = 0; q < 4; ++q) {
    p2_gradients(geo, q, grads);
    const double wc = 0.25 * geo.volume * coeff[q];
    int k = 0;
    for (int i = 0; i < 10; ++i)
      for (int j = 0; j <= i; ++j) {
        const double gij = grads[i][0] * grads[j][0] + grads[i][1] * grads[j][1] + grads[i][2] * grads[j][2];
        S[k++] += wc * gij;
      }
  }
}

EQS_HD int tri_index(int i, int j) { return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i; }

}  // namespace eqsb
