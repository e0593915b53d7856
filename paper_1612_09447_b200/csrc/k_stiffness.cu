// K1: fused matrix-free stiffness product y = K(x_state) v
// (proj/src/matfree.cpp:65-117 with tet_geometry / gradient_magnitude /
// kappa_of_e / element_laplacian inlined, proj/src/assembly.cpp:34-116,
// proj/src/materials.cpp:25-33).
//
// One thread per tetrahedron: gather 4 vertex coordinates (32 B padded rows)
// and the local x / v values, form the barycentric gradients in registers,
// evaluate kappa(|grad x_h|) per quadrature point and apply the local matrix
// without materialising it:  (S v)_i = sum_q w_q kappa_q grad N_i(q) . grad v_h(q)
// (for P1 that is V kappa g_i . grad v_h: 24 flops instead of the 4x4 matrix).
//
// Scatter is deterministic in both modes:
//  * gather mode (default): pass 1 writes the local products per tet, pass 2
//    sums them per dof over a fixed ascending-tet slot list (no atomics);
//  * coloured mode: one launch per colour of the reference colouring
//    (matfree.cpp:100-117): tets of one colour share no dof, so y[dof] +=
//    is race-free and the per-dof summation order equals the reference's.
#include <cuda_runtime.h>

#include "dev.cuh"
#include "element.hpp"

namespace eqsb {

namespace {

__constant__ DevMaterial c_mat[kMaxMaterials];

// kappa_of_e (proj/src/materials.cpp:25-33) with log10(kappa_lo/hi) hoisted.
__device__ __forceinline__ double kappa_dev(const DevMaterial& m, double e) {
  if (m.kind == 0) return m.kappa;
  const double s = 0.5 * (1.0 + tanh((e - m.e_switch) * m.inv_width));
  return exp10(m.lo + (m.hi - m.lo) * s);
}

__device__ __forceinline__ void load_xyz(const double* __restrict__ coords, int d, double p[3]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(coords + 4L * d));
  const double b = __ldg(coords + 4L * d + 2);
  p[0] = a.x;
  p[1] = a.y;
  p[2] = b;
}

// barycentric gradients + volume (proj/src/assembly.cpp:34-61), reciprocal of det once.
__device__ __forceinline__ bool geometry(const double p[4][3], double g[4][3], double& vol) {
  double e[3][3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
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
  const double inv = 1.0 / det;
  vol = det / 6.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int d = 0; d < 3; ++d) g[i + 1][d] = cr[i][d] * inv;
#pragma unroll
  for (int d = 0; d < 3; ++d) g[0][d] = -g[1][d] - g[2][d] - g[3][d];
  return det != 0.0;
}

// local product of one P1 tet; returns false on a degenerate tet
__device__ __forceinline__ void p1_local(int4 n, int m, const double* __restrict__ coords,
                                         const double* __restrict__ x, const double* __restrict__ v, bool same,
                                         double y[4], int* err) {
  double p[4][3];
  load_xyz(coords, n.x, p[0]);
  load_xyz(coords, n.y, p[1]);
  load_xyz(coords, n.z, p[2]);
  load_xyz(coords, n.w, p[3]);
  double g[4][3], vol;
  if (!geometry(p, g, vol)) atomicOr(err, 1);
  const double xl[4] = {__ldg(x + n.x), __ldg(x + n.y), __ldg(x + n.z), __ldg(x + n.w)};
  double gx[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int d = 0; d < 3; ++d) gx[d] += xl[i] * g[i][d];
  const double e = sqrt(gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2]);
  if (!(e >= 0.0)) atomicOr(err, 2);  // kappa_of_e: invalid_argument (materials.cpp:26)
  const double kap = kappa_dev(c_mat[m], e);
  double gv[3];
  if (same) {
    gv[0] = gx[0];
    gv[1] = gx[1];
    gv[2] = gx[2];
  } else {
    const double vl[4] = {__ldg(v + n.x), __ldg(v + n.y), __ldg(v + n.z), __ldg(v + n.w)};
    gv[0] = gv[1] = gv[2] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) gv[d] += vl[i] * g[i][d];
  }
  const double c = vol * kap;
#pragma unroll
  for (int i = 0; i < 4; ++i) y[i] = c * (g[i][0] * gv[0] + g[i][1] * gv[1] + g[i][2] * gv[2]);
}

// P2: 10 dofs, 4-point degree-2 rule (assembly.cpp:13-18, 69-85, 97-116)
__device__ __forceinline__ void p2_local(const int* __restrict__ dofs, int m, const double* __restrict__ coords,
                                         const double* __restrict__ x, const double* __restrict__ v, bool same,
                                         double y[10], int* err) {
  double p[4][3];
#pragma unroll
  for (int k = 0; k < 4; ++k) load_xyz(coords, dofs[k], p[k]);
  double g[4][3], vol;
  if (!geometry(p, g, vol)) atomicOr(err, 1);
  double xl[10], vl[10];
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    xl[i] = __ldg(x + dofs[i]);
    vl[i] = same ? xl[i] : __ldg(v + dofs[i]);
  }
#pragma unroll
  for (int i = 0; i < 10; ++i) y[i] = 0.0;
  const int ev[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll 1
  for (int q = 0; q < 4; ++q) {
    double lam[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) lam[i] = (i == q) ? kQa : kQb;
    double gr[10][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double f = 4.0 * lam[i] - 1.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) gr[i][d] = f * g[i][d];
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int a = ev[e][0], b = ev[e][1];
#pragma unroll
      for (int d = 0; d < 3; ++d) gr[4 + e][d] = 4.0 * (lam[a] * g[b][d] + lam[b] * g[a][d]);
    }
    double gx[3] = {0.0, 0.0, 0.0}, gv[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 10; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        gx[d] += xl[i] * gr[i][d];
        gv[d] += vl[i] * gr[i][d];
      }
    const double e = sqrt(gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2]);
    if (!(e >= 0.0)) atomicOr(err, 2);
    const double c = 0.25 * vol * kappa_dev(c_mat[m], e);
#pragma unroll
    for (int i = 0; i < 10; ++i) y[i] += c * (gr[i][0] * gv[0] + gr[i][1] * gv[1] + gr[i][2] * gv[2]);
  }
}

__global__ void __launch_bounds__(kBlock) k_kx_p1(int nt, const int4* __restrict__ tets,
                                                  const unsigned char* __restrict__ mat,
                                                  const double* __restrict__ coords, const double* __restrict__ x,
                                                  const double* __restrict__ v, double* __restrict__ ytet, int* err) {
  const int t = blockIdx.x * kBlock + threadIdx.x;
  if (t >= nt) return;
  const int4 n = __ldg(tets + t);
  double y[4];
  p1_local(n, mat[t], coords, x, v, x == v, y, err);
  double2* out = reinterpret_cast<double2*>(ytet + 4L * t);
  out[0] = make_double2(y[0], y[1]);
  out[1] = make_double2(y[2], y[3]);
}

__global__ void __launch_bounds__(kBlock) k_kx_p2(int nt, const int* __restrict__ tet_dofs,
                                                  const unsigned char* __restrict__ mat,
                                                  const double* __restrict__ coords, const double* __restrict__ x,
                                                  const double* __restrict__ v, double* __restrict__ ytet, int* err) {
  const int t = blockIdx.x * kBlock + threadIdx.x;
  if (t >= nt) return;
  int dofs[10];
#pragma unroll
  for (int i = 0; i < 10; ++i) dofs[i] = __ldg(tet_dofs + 10L * t + i);
  double y[10];
  p2_local(dofs, mat[t], coords, x, v, x == v, y, err);
#pragma unroll
  for (int i = 0; i < 10; ++i) ytet[10L * t + i] = y[i];
}

__global__ void __launch_bounds__(kBlock) k_kx_gather(int n, const long* __restrict__ ptr,
                                                      const int* __restrict__ slots, const double* __restrict__ ytet,
                                                      const double* __restrict__ base, double sign,
                                                      double* __restrict__ out) {
  const int d = blockIdx.x * kBlock + threadIdx.x;
  if (d >= n) return;
  double s = 0.0;
  for (long k = ptr[d]; k < ptr[d + 1]; ++k) s += __ldg(ytet + slots[k]);
  out[d] = base ? base[d] + sign * s : sign * s;
}

__global__ void __launch_bounds__(kBlock) k_kx_colored_p1(int nb, const int* __restrict__ batch,
                                                          const int4* __restrict__ tets,
                                                          const unsigned char* __restrict__ mat,
                                                          const double* __restrict__ coords,
                                                          const double* __restrict__ x, const double* __restrict__ v,
                                                          double* __restrict__ y, int* err) {
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= nb) return;
  const int t = batch[k];
  const int4 n = __ldg(tets + t);
  double yl[4];
  p1_local(n, mat[t], coords, x, v, x == v, yl, err);
  y[n.x] += yl[0];
  y[n.y] += yl[1];
  y[n.z] += yl[2];
  y[n.w] += yl[3];
}

__global__ void __launch_bounds__(kBlock) k_kx_colored_p2(int nb, const int* __restrict__ batch,
                                                          const int* __restrict__ tet_dofs,
                                                          const unsigned char* __restrict__ mat,
                                                          const double* __restrict__ coords,
                                                          const double* __restrict__ x, const double* __restrict__ v,
                                                          double* __restrict__ y, int* err) {
  const int k = blockIdx.x * kBlock + threadIdx.x;
  if (k >= nb) return;
  const int t = batch[k];
  int dofs[10];
#pragma unroll
  for (int i = 0; i < 10; ++i) dofs[i] = __ldg(tet_dofs + 10L * t + i);
  double yl[10];
  p2_local(dofs, mat[t], coords, x, v, x == v, yl, err);
#pragma unroll
  for (int i = 0; i < 10; ++i) y[dofs[i]] += yl[i];
}

}  // namespace

void set_materials(const DevMaterial* mats, int n, cudaStream_t s) {
  cudaMemcpyToSymbolAsync(c_mat, mats, sizeof(DevMaterial) * n, 0, cudaMemcpyHostToDevice, s);
}

void launch_kx_tets(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                    const double* x_state, const double* v, double* ytet, int* geo_error, cudaStream_t s) {
  ++g_launch_count;
  if (n_tets == 0) return;
  const int g = (n_tets + kBlock - 1) / kBlock;
  if (order == 1)
    k_kx_p1<<<g, kBlock, 0, s>>>(n_tets, reinterpret_cast<const int4*>(tet_dofs), tet_mat, coords, x_state, v, ytet,
                                 geo_error);
  else
    k_kx_p2<<<g, kBlock, 0, s>>>(n_tets, tet_dofs, tet_mat, coords, x_state, v, ytet, geo_error);
}

void launch_kx_gather(int n_rows, const long* slot_ptr, const int* slots, const double* ytet, const double* base,
                      double sign, double* out, cudaStream_t s) {
  ++g_launch_count;
  if (n_rows == 0) return;
  k_kx_gather<<<(n_rows + kBlock - 1) / kBlock, kBlock, 0, s>>>(n_rows, slot_ptr, slots, ytet, base, sign, out);
}

void launch_kx_colored(int order, int n_batch, const int* batch_tets, const int* tet_dofs,
                       const unsigned char* tet_mat, const double* coords, const double* x_state, const double* v,
                       double* y, int* geo_error, cudaStream_t s) {
  ++g_launch_count;
  if (n_batch == 0) return;
  const int g = (n_batch + kBlock - 1) / kBlock;
  if (order == 1)
    k_kx_colored_p1<<<g, kBlock, 0, s>>>(n_batch, batch_tets, reinterpret_cast<const int4*>(tet_dofs), tet_mat,
                                         coords, x_state, v, y, geo_error);
  else
    k_kx_colored_p2<<<g, kBlock, 0, s>>>(n_batch, batch_tets, tet_dofs, tet_mat, coords, x_state, v, y, geo_error);
}

}  // namespace eqsb
