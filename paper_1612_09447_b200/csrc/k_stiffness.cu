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

// out-of-line field-dependent branch: keeps the tanh / exp10 registers out
// of the element loop of k_kx_block4 (linear materials never call it)
__device__ __noinline__ double kappa_nl(const DevMaterial& m, double e) { return kappa_dev(m, e); }

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

// local product of one P1 tet from its vertex coordinates and x / v values
__device__ __forceinline__ void p1_compute(const double p[4][3], const double xl[4], const double vl[4], bool same,
                                           int m, double y[4], int* err) {
  double g[4][3], vol;
  if (!geometry(p, g, vol)) atomicOr(err, 1);
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

// local product of one P1 tet gathered from global memory
__device__ __forceinline__ void p1_local(int4 n, int m, const double* __restrict__ coords,
                                         const double* __restrict__ x, const double* __restrict__ v, bool same,
                                         double y[4], int* err) {
  double p[4][3];
  load_xyz(coords, n.x, p[0]);
  load_xyz(coords, n.y, p[1]);
  load_xyz(coords, n.z, p[2]);
  load_xyz(coords, n.w, p[3]);
  const double xl[4] = {__ldg(x + n.x), __ldg(x + n.y), __ldg(x + n.z), __ldg(x + n.w)};
  double vl[4] = {0.0, 0.0, 0.0, 0.0};
  if (!same) {
    vl[0] = __ldg(v + n.x);
    vl[1] = __ldg(v + n.y);
    vl[2] = __ldg(v + n.z);
    vl[3] = __ldg(v + n.w);
  }
  p1_compute(p, xl, vl, same, m, y, err);
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

// Blocked deterministic scatter (kxblock.hpp): one CTA per tet block. The
// block's dof lists (slot ranges, slots, outputs) are staged into shared
// memory first, overlapping the element phase; the element phase computes the
// local products into shared memory (next tet's indices prefetched); the sum
// phase adds them per block-dof in slot order. Interior dofs are final (out =
// base + sign * sum for dofs < n_out), boundary dofs leave a partial for pass 2.
template <int NL>
__global__ void __launch_bounds__(kBlock, NL == 4 ? 4 : 1) k_kx_block(const int* __restrict__ blk_tet0, const int* __restrict__ tets,
                                                     const unsigned char* __restrict__ mat,
                                                     const double* __restrict__ coords, const double* __restrict__ x,
                                                     const double* __restrict__ v, const int* __restrict__ blk_dof0,
                                                     const int* __restrict__ sptr, const uint16_t* __restrict__ slots,
                                                     const int* __restrict__ lout, double* __restrict__ partials,
                                                     const double* __restrict__ base, double sign, int n_out,
                                                     double* __restrict__ out, int* err, int max_tets, int max_dofs,
                                                     int max_slots, const int* __restrict__ ldof_dof) {
  // shared memory: [NL][max_tets] products; P1: staged coordinates [max_dofs][3],
  // x and v [max_dofs]; then the dof lists (slot ranges, outputs, slots)
  extern __shared__ double ysm[];
  double* s_xyz = ysm + (size_t)max_tets * NL;
  double* s_x = s_xyz + 3L * max_dofs;
  int* s_sptr = reinterpret_cast<int*>(NL == 4 ? s_x + 2L * max_dofs : s_xyz);  // [max_dofs + 1]
  int* s_out = s_sptr + max_dofs + 1;                                             // [max_dofs]
  uint16_t* s_slot = reinterpret_cast<uint16_t*>(s_out + max_dofs);               // [max_slots]
  const int b = blockIdx.x;
  const int t0 = blk_tet0[b], nt = blk_tet0[b + 1] - t0;
  const int d0 = blk_dof0[b], nd = blk_dof0[b + 1] - d0;
  const int sbase = sptr[d0], nsl = sptr[d0 + nd] - sbase;
  // stage the dof lists (independent loads, in flight during the element phase)
  for (int i = threadIdx.x; i <= nd; i += kBlock) s_sptr[i] = __ldcs(sptr + d0 + i) - sbase;
  for (int i = threadIdx.x; i < nd; i += kBlock) s_out[i] = __ldcs(lout + d0 + i);
  for (int i = threadIdx.x; i < nsl; i += kBlock) s_slot[i] = __ldcs(slots + sbase + i);
  const bool same = x == v;
  if constexpr (NL == 4) {
    // stage the block-dofs' coordinates and x (v) values once per dof; the
    // element phase then reads them through the tets' 16-bit block-local ids
    double* s_v = same ? s_x : s_x + max_dofs;
    for (int i = threadIdx.x; i < nd; i += kBlock) {
      const int gd = __ldcs(ldof_dof + d0 + i);
      double p[3];
      load_xyz(coords, gd, p);
      s_xyz[3 * i] = p[0];
      s_xyz[3 * i + 1] = p[1];
      s_xyz[3 * i + 2] = p[2];
      s_x[i] = __ldg(x + gd);
      if (!same) s_v[i] = __ldg(v + gd);
    }
    __syncthreads();
    const ushort4* tt = reinterpret_cast<const ushort4*>(tets) + t0;
    for (int tl = threadIdx.x; tl < nt; tl += kBlock) {
      const ushort4 n = __ldcs(tt + tl);
      const int li[4] = {n.x, n.y, n.z, n.w};
      double p[4][3], xl[4], vl[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
#pragma unroll
        for (int d = 0; d < 3; ++d) p[k][d] = s_xyz[3 * li[k] + d];
        xl[k] = s_x[li[k]];
        vl[k] = s_v[li[k]];
      }
      double y[4];
      p1_compute(p, xl, vl, same, __ldcs(mat + t0 + tl), y, err);
#pragma unroll
      for (int i = 0; i < 4; ++i) ysm[i * max_tets + tl] = y[i];
    }
  } else {
    for (int tl = threadIdx.x; tl < nt; tl += kBlock) {
      const long t = (long)t0 + tl;
      int dofs[10];
#pragma unroll
      for (int i = 0; i < 10; ++i) dofs[i] = __ldg(tets + 10L * t + i);
      double y[10];
      p2_local(dofs, mat[t], coords, x, v, same, y, err);
#pragma unroll
      for (int i = 0; i < 10; ++i) ysm[i * max_tets + tl] = y[i];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nd; e += kBlock) {
    double s = 0.0;
    const int k1 = s_sptr[e + 1];
    for (int k = s_sptr[e]; k < k1; ++k) s += ysm[s_slot[k]];
    const int o = s_out[e];
    if (o >= 0) {
      if (o < n_out) out[o] = base ? base[o] + sign * s : sign * s;
    } else {
      partials[-o - 1] = s;
    }
  }
}

// P1 blocked K(x)v, latency-lean form. Differences from the
// generic k_kx_block<4>:
//  * every global load is issued before the first barrier: the thread's tets
//    (ushort4 block-local ids + material byte, TPT per thread, in registers),
//    the dof lists, the block-dof coordinates (stored per block-dof, streamed
//    instead of gathered) and the x (v) gathers; the element phase reads
//    registers and shared memory only;
//  * the element arithmetic uses the unscaled cofactor rows cr_k (g_k =
//    cr_k / det): w = sum_k (x_k - x_0) cr_k, |grad x_h| = |w| / |det|,
//    y_k = kappa / (6 det) cr_k . w_v (k = 1..3), y_0 = -(y_1 + y_2 + y_3);
//    the sqrt runs for field-dependent materials only;
//  * the per-dof sums load four products ahead of the (sequential, fixed
//    order) additions.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

#ifndef KX4_MINB
#define KX4_MINB 4
#endif
template <bool SAME>
__global__ void __launch_bounds__(kBlock, KX4_MINB) k_kx_block4(const int* __restrict__ blk_tet0, const ushort4* __restrict__ tets,
                                                        const unsigned char* __restrict__ mat,
                                                        const double2* __restrict__ bxy, const double* __restrict__ bz,
                                                        const double* __restrict__ coords, const double* __restrict__ x,
                                                        const double* __restrict__ v, const int* __restrict__ blk_dof0,
                                                        const int* __restrict__ sptr, const uint16_t* __restrict__ slots,
                                                        const int* __restrict__ lout, double* __restrict__ partials,
                                                        const double* __restrict__ base, double sign, int n_out,
                                                        double* __restrict__ out, int* err, int max_tets, int max_dofs,
                                                        const int* __restrict__ ldof_dof) {
  // shared memory: products [4][max_tets] (the first quarter doubles as the
  // staged tets: thread-private slot tl is read before it is overwritten),
  // block-dof records {x, y, z, x_state} (32 B: two 16-byte loads per
  // vertex), v [max_dofs] when v != x, slot ranges, outputs, material bytes,
  // slots
  extern __shared__ double ysm[];
  ushort4* s_tet = reinterpret_cast<ushort4*>(ysm);
  // {x, y} and {z, x_state} of each block-dof in two arrays of 16-byte
  // records: a 16-byte load then starts on one of 8 bank groups (one of 4
  // with 32-byte records), halving the structural bank conflicts
  double* s_p = ysm + (size_t)max_tets * 4;  // [max_dofs][2] {x, y}, then [max_dofs][2] {z, x_state}
  double* s_q = s_p + 2L * max_dofs;
  double* s_v = SAME ? nullptr : s_p + 4L * max_dofs;
  int* s_sptr = reinterpret_cast<int*>(s_p + (SAME ? 4L : 5L) * max_dofs);  // [max_dofs + 1]
  int* s_out = s_sptr + max_dofs + 1;                      // [max_dofs]
  unsigned* s_matw = reinterpret_cast<unsigned*>(s_out + max_dofs);  // [max_tets / 4 + 2] words
  uint16_t* s_slot = reinterpret_cast<uint16_t*>(s_matw + max_tets / 4 + 2);
  const int b = blockIdx.x;
  const int t0 = __ldg(blk_tet0 + b), nt = __ldg(blk_tet0 + b + 1) - t0;
  const int d0 = __ldg(blk_dof0 + b), nd = __ldg(blk_dof0 + b + 1) - d0;
  // asynchronous copies of the streamed per-tet data (no registers held)
  for (int tl = threadIdx.x; tl < nt; tl += kBlock) cp_async8(s_tet + tl, tets + t0 + tl);
  {
    const unsigned* mw = reinterpret_cast<const unsigned*>(mat);
    const int w0 = t0 >> 2, w1 = (t0 + nt + 3) >> 2;
    for (int w = w0 + threadIdx.x; w < w1; w += kBlock) cp_async4(s_matw + (w - w0), mw + w);
  }
  const int sbase = __ldg(sptr + d0);
  const int nsl = __ldg(sptr + d0 + nd) - sbase;
  for (int i = threadIdx.x; i < nd; i += kBlock) {
    const int gd = __ldcs(ldof_dof + d0 + i);
    if (bz) {  // coordinates streamed from the per-block-dof copy
      cp_async16(s_p + 2 * i, bxy + d0 + i);
      cp_async8(s_q + 2 * i, bz + d0 + i);
    } else {  // gathered from the padded [x, y, z, 0] rows (fewer DRAM bytes, longer chain)
      cp_async16(s_p + 2 * i, coords + 4L * gd);
      cp_async8(s_q + 2 * i, coords + 4L * gd + 2);
    }
    cp_async4(s_sptr + i, sptr + d0 + i);
    cp_async4(s_out + i, lout + d0 + i);
    cp_async8(s_q + 2 * i + 1, x + gd);
    if (!SAME) cp_async8(s_v + i, v + gd);
  }
  for (int i = threadIdx.x; i < nsl; i += kBlock) s_slot[i] = __ldcs(slots + sbase + i);
  if (threadIdx.x == 0) s_sptr[nd] = sbase + nsl;
  cp_async_wait_all();
  __syncthreads();
  const unsigned char* s_mat = reinterpret_cast<const unsigned char*>(s_matw) + (t0 & 3);
  for (int tl = threadIdx.x; tl < nt; tl += kBlock) {
    const ushort4 q = s_tet[tl];
    const int li[4] = {q.x, q.y, q.z, q.w};
    double2 pa[4], pb[4];  // {x, y}, {z, x_state} of the four vertices
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pa[k] = reinterpret_cast<const double2*>(s_p)[li[k]];
      pb[k] = reinterpret_cast<const double2*>(s_q)[li[k]];
    }
    double e[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      e[c][0] = pa[c + 1].x - pa[0].x;
      e[c][1] = pa[c + 1].y - pa[0].y;
      e[c][2] = pb[c + 1].x - pb[0].x;
    }
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
    if (det == 0.0) atomicOr(err, 1);
    const double x0 = pb[0].y;
    const double dx[3] = {pb[1].y - x0, pb[2].y - x0, pb[3].y - x0};
    double w[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) w[d] = dx[0] * cr[0][d] + dx[1] * cr[1][d] + dx[2] * cr[2][d];
    const double s2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    if (!(s2 >= 0.0)) atomicOr(err, 2);  // kappa_of_e: invalid_argument (materials.cpp:26)
    const double inv = 1.0 / det;
    const DevMaterial& m = c_mat[s_mat[tl]];
    const double kap = m.kind == 0 ? m.kappa : kappa_nl(m, sqrt(s2) * fabs(inv));
    double wv[3] = {w[0], w[1], w[2]};
    if (!SAME) {
      const double v0 = s_v[li[0]];
      const double dv[3] = {s_v[li[1]] - v0, s_v[li[2]] - v0, s_v[li[3]] - v0};
#pragma unroll
      for (int d = 0; d < 3; ++d) wv[d] = dv[0] * cr[0][d] + dv[1] * cr[1][d] + dv[2] * cr[2][d];
    }
    const double c = kap * inv * (1.0 / 6.0);
    double y[4];
#pragma unroll
    for (int i = 0; i < 3; ++i) y[i + 1] = c * (cr[i][0] * wv[0] + cr[i][1] * wv[1] + cr[i][2] * wv[2]);
    y[0] = -(y[1] + y[2] + y[3]);
#pragma unroll
    for (int i = 0; i < 4; ++i) ysm[i * max_tets + tl] = y[i];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nd; e += kBlock) {
    int k = s_sptr[e] - sbase;
    const int k1 = s_sptr[e + 1] - sbase;
    double s = 0.0;
    for (; k + 4 <= k1; k += 4) {
      const double a0 = ysm[s_slot[k]], a1 = ysm[s_slot[k + 1]], a2 = ysm[s_slot[k + 2]], a3 = ysm[s_slot[k + 3]];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; k < k1; ++k) s += ysm[s_slot[k]];
    const int o = s_out[e];
    if (o >= 0) {
      if (o < n_out) out[o] = base ? base[o] + sign * s : sign * s;
    } else {
      partials[-o - 1] = s;
    }
  }
}

// pass 2: boundary dofs, partials summed in block order
__global__ void __launch_bounds__(kBlock) k_kx_partials(int nb, const int* __restrict__ bdof,
                                                        const int* __restrict__ bptr, const int* __restrict__ bpart,
                                                        const double* __restrict__ partials,
                                                        const double* __restrict__ base, double sign, int n_out,
                                                        double* __restrict__ out) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i >= nb) return;
  const int d = bdof[i];
  if (d >= n_out) return;
  double s = 0.0;
  for (int k = bptr[i]; k < bptr[i + 1]; ++k) s += partials[bpart[k]];
  out[d] = base ? base[d] + sign * s : sign * s;
}

}  // namespace

void launch_kx_blocked(const KxDev& k, const double* coords, const double* x_state, const double* v,
                       const double* base, double sign, int n_out, double* out, int* geo_error, cudaStream_t s) {
  if (k.n_blocks == 0) return;
  g_launch_count += 2;
  size_t smem = sizeof(double) * k.nl * k.max_block_tets + sizeof(int) * (2L * k.max_block_dofs + 1) +
                sizeof(uint16_t) * k.max_block_slots + 16;
  if (k.nl == 4) smem += sizeof(double) * 5L * k.max_block_dofs;  // staged coordinates, x, v
  if (k.nl == 4 && k.bxy) {
    const bool same = x_state == v;
    const size_t sm4 = sizeof(double) * (4L * k.max_block_tets + (same ? 4L : 5L) * k.max_block_dofs) +
                       sizeof(int) * (2L * k.max_block_dofs + 1) + sizeof(unsigned) * (k.max_block_tets / 4 + 2) +
                       sizeof(uint16_t) * k.max_block_slots + 16;
    static bool attr4 = false;
    if (!attr4) {
      cudaFuncSetAttribute(k_kx_block4<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_kx_block4<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr4 = true;
    }
    auto kern = same ? k_kx_block4<true> : k_kx_block4<false>;
    kern<<<k.n_blocks, kBlock, sm4, s>>>(k.blk_tet0, reinterpret_cast<const ushort4*>(k.tets), k.mat,
                                         reinterpret_cast<const double2*>(k.bxy), k.bz, coords, x_state, v, k.blk_dof0,
                                         k.sptr, k.slots, k.lout, k.partials, base, sign, n_out, out, geo_error,
                                         k.max_block_tets, k.max_block_dofs, k.ldof_dof);
  } else if (k.nl == 4) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_kx_block<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    k_kx_block<4><<<k.n_blocks, kBlock, smem, s>>>(k.blk_tet0, k.tets, k.mat, coords, x_state, v, k.blk_dof0, k.sptr,
                                                   k.slots, k.lout, k.partials, base, sign, n_out, out, geo_error,
                                                   k.max_block_tets, k.max_block_dofs, k.max_block_slots, k.ldof_dof);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_kx_block<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    k_kx_block<10><<<k.n_blocks, kBlock, smem, s>>>(k.blk_tet0, k.tets, k.mat, coords, x_state, v, k.blk_dof0,
                                                    k.sptr, k.slots, k.lout, k.partials, base, sign, n_out, out,
                                                    geo_error, k.max_block_tets, k.max_block_dofs, k.max_block_slots, k.ldof_dof);
  }
  if (k.n_bdof > 0)
    k_kx_partials<<<(k.n_bdof + kBlock - 1) / kBlock, kBlock, 0, s>>>(k.n_bdof, k.bdof, k.bptr, k.bpart, k.partials,
                                                                      base, sign, n_out, out);
}

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

// Element matrices of K(x) for the SDIRK Newton matrix (assemble_stiffness,
// proj/src/assembly.cpp:97-116,178-186): packed lower triangle per tet (10 for
// P1, 55 for P2), kappa at |grad x_h| per quadrature point
// (gradient_magnitude, assembly.cpp:87-95), element.hpp's reference-order
// geometry and Laplacian.
__global__ void __launch_bounds__(kBlock) k_kelem(int nt, int nl, const int* __restrict__ tet_dofs,
                                                  const unsigned char* __restrict__ tet_mat,
                                                  const double* __restrict__ coords, const double* __restrict__ x,
                                                  double* __restrict__ S, int* __restrict__ err) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int dofs[10];
  for (int i = 0; i < nl; ++i) dofs[i] = tet_dofs[(long)nl * t + i];
  double p[4][3];
  for (int v = 0; v < 4; ++v) load_xyz(coords, dofs[v], p[v]);
  TetGeo geo;
  if (!tet_geometry(p, geo)) {
    atomicExch(err, 1);
    return;
  }
  double xl[10];
  for (int i = 0; i < nl; ++i) xl[i] = x[dofs[i]];
  const DevMaterial& m = c_mat[tet_mat[t]];
  if (nl == 4) {
    double g[3] = {0.0, 0.0, 0.0};
    for (int i = 0; i < 4; ++i)
      for (int d = 0; d < 3; ++d) g[d] = __dadd_rn(g[d], __dmul_rn(xl[i], geo.g[i][d]));
    const double e = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])), __dmul_rn(g[2], g[2])));
    double Sl[10];
    element_laplacian_p1(geo, kappa_dev(m, e), Sl);
    for (int k = 0; k < 10; ++k) S[10L * t + k] = Sl[k];
  } else {
    double coeff[4], grads[10][3];
    for (int q = 0; q < 4; ++q) {
      p2_gradients(geo, q, grads);
      double g[3] = {0.0, 0.0, 0.0};
      for (int i = 0; i < 10; ++i)
        for (int d = 0; d < 3; ++d) g[d] = __dadd_rn(g[d], __dmul_rn(xl[i], grads[i][d]));
      coeff[q] = kappa_dev(m, sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])),
                                             __dmul_rn(g[2], g[2]))));
    }
    double Sl[55];
    element_laplacian_p2(geo, coeff, Sl);
    for (int k = 0; k < 55; ++k) S[55L * t + k] = Sl[k];
  }
}

// per-cell kappa of the VTK dump (vtk_writer.cpp:38-46): kappa at |grad x_h|
// of the first quadrature point
__global__ void __launch_bounds__(kBlock) k_cell_kappa(int nt, int nl, const int* __restrict__ tet_dofs,
                                                       const unsigned char* __restrict__ tet_mat,
                                                       const double* __restrict__ coords, const double* __restrict__ x,
                                                       double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  int dofs[10];
  for (int i = 0; i < nl; ++i) dofs[i] = tet_dofs[(long)nl * t + i];
  double p[4][3];
  for (int v = 0; v < 4; ++v) load_xyz(coords, dofs[v], p[v]);
  TetGeo geo;
  tet_geometry(p, geo);
  double grads[10][3];
  if (nl == 4) {
    for (int i = 0; i < 4; ++i)
      for (int d = 0; d < 3; ++d) grads[i][d] = geo.g[i][d];
  } else {
    p2_gradients(geo, 0, grads);
  }
  double g[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < nl; ++i) {
    const double xi = x[dofs[i]];
    for (int d = 0; d < 3; ++d) g[d] = __dadd_rn(g[d], __dmul_rn(xi, grads[i][d]));
  }
  out[t] = kappa_dev(c_mat[tet_mat[t]],
                     sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])), __dmul_rn(g[2], g[2]))));
}

void launch_cell_kappa(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                       const double* x_full, double* kappa, cudaStream_t s) {
  ++g_launch_count;
  if (n_tets == 0) return;
  k_cell_kappa<<<(n_tets + kBlock - 1) / kBlock, kBlock, 0, s>>>(n_tets, order == 1 ? 4 : 10, tet_dofs, tet_mat,
                                                                 coords, x_full, kappa);
}

void launch_k_element(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                      const double* x_full, double* S, int* geo_error, cudaStream_t s) {
  ++g_launch_count;
  if (n_tets == 0) return;
  k_kelem<<<(n_tets + kBlock - 1) / kBlock, kBlock, 0, s>>>(n_tets, order == 1 ? 4 : 10, tet_dofs, tet_mat, coords,
                                                            x_full, S, geo_error);
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
