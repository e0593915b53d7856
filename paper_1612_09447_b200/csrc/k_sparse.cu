// Vector kernels of the M-solve (AMG-PCG), the SPE estimator and the RKC
// recurrence (the matrix row kernels are in k_rows.cu). All HBM-bound,
// grid-stride; reductions are fused into the producing kernel and finished
// deterministically (fixed grid, last-block ordered sum).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>
#include <unordered_map>

#include "dev.cuh"
#include "reduce.cuh"

namespace eqsb {

long g_launch_count = 0;
double g_algo_bytes = 0.0;
bool g_pdl = true;

namespace {

template <class XT>
__global__ void k_dense_solve(int n, const double* __restrict__ ainv, const XT* __restrict__ b,
                              XT* __restrict__ z) {
  pdl_entry();
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sb[i] = (double)b[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int row = w; row < n; row += nw) {
    double s = 0.0;
    for (int k = l; k < n; k += 32) s += ainv[(size_t)row * n + k] * sb[k];
    s = warp_sum(s);
    if (l == 0) z[row] = (XT)s;
  }
}

// z = Ainv b for the larger dense coarse levels: one warp per row, coalesced
// row reads (fp32 inverse for the fp32 V-cycle), fp64 accumulation
template <class MT, class XT>
__global__ void __launch_bounds__(kBlock) k_dense_gemv(int n, const MT* __restrict__ a, const XT* __restrict__ b,
                                                      XT* __restrict__ z) {
  pdl_entry();
  const int row = (int)((blockIdx.x * (long)kBlock + threadIdx.x) >> 5), l = threadIdx.x & 31;
  if (row >= n) return;
  const MT* ar = a + (size_t)row * n;
  double s = 0.0;
#pragma unroll 8
  for (int k = l; k < n; k += 32) s += (double)__ldcs(ar + k) * (double)__ldg(b + k);
  s = warp_sum(s);
  if (l == 0) z[row] = (XT)s;
}

__global__ void k_jacobi(int n, const double* __restrict__ invd, const double* __restrict__ r,
                         double* __restrict__ z, Reducer red, int slot, int do_red) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double zi = invd[i] * r[i];
    z[i] = zi;
    acc += r[i] * zi;
  }
  if (do_red) reduce_finish(acc, red, slot);
}

// x += alpha p ; r -= alpha q ; r.r ; r32 = (float) r for an fp32 V-cycle
// x += alpha p ; r -= alpha q ; r.r ; and for an fp32 V-cycle r32 = (float) r,
// d32 = invd32 .* r32 (its fine-level b and D^-1 b). VEC: pairs of entries per
// thread with 16-byte loads (all arrays 16-byte aligned); the odd tail entry
// is handled by thread 0.
// WX false (graph-resident loop): x is not touched here; its update by this
// iteration's alpha p happens in the next direction kernel (or k_pcg_xfinal),
// which reads p anyway.
template <bool F32, bool VEC, bool WX>
__global__ void __launch_bounds__(kBlock, 6)
    k_pcg_update(int n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                 const double* __restrict__ q, float* __restrict__ r32, const float* __restrict__ invd32,
                 float* __restrict__ d32, Reducer red) {
  pdl_entry();
  const double alpha = red.scal[S_RZ] / red.scal[S_PQ];
  double acc = 0.0;
  auto one = [&](long i) {
    if constexpr (WX) x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    if constexpr (F32) {
      const float rf = (float)ri;
      r32[i] = rf;
      d32[i] = invd32[i] * rf;
    }
    acc += ri * ri;
  };
  if constexpr (VEC) {
    const long n2 = n / 2;
    const bool x_al = ((uintptr_t)x & 15) == 0;
    for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
      const double2 qi = reinterpret_cast<const double2*>(q)[i];
      double2 ri = reinterpret_cast<double2*>(r)[i];
      if constexpr (WX) {
        const double2 pi = reinterpret_cast<const double2*>(p)[i];
        if (x_al) {
          double2 xi = reinterpret_cast<double2*>(x)[i];
          xi.x += alpha * pi.x;
          xi.y += alpha * pi.y;
          reinterpret_cast<double2*>(x)[i] = xi;
        } else {  // a caller's 8-byte-aligned x: same values, scalar accesses
          x[2 * i] += alpha * pi.x;
          x[2 * i + 1] += alpha * pi.y;
        }
      }
      ri.x -= alpha * qi.x;
      ri.y -= alpha * qi.y;
      reinterpret_cast<double2*>(r)[i] = ri;
      if constexpr (F32) {
        const float2 w = reinterpret_cast<const float2*>(invd32)[i];
        const float2 rf = make_float2((float)ri.x, (float)ri.y);
        reinterpret_cast<float2*>(r32)[i] = rf;
        reinterpret_cast<float2*>(d32)[i] = make_float2(w.x * rf.x, w.y * rf.y);
      }
      acc += ri.x * ri.x;
      acc += ri.y * ri.y;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) one(n - 1);
  } else {
    for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) one(i);
  }
  reduce_finish(acc, red, S_RR);
}

__global__ void k_to_f32(long n, const double* __restrict__ x, float* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = (float)x[i];
}
__global__ void k_to_f32_scaled(long n, const double* __restrict__ x, const float* __restrict__ invd,
                                float* __restrict__ y, float* __restrict__ d) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const float f = (float)x[i];
    y[i] = f;
    d[i] = invd[i] * f;
  }
}
// z64 = z32 ; slot <- b.z64
__global__ void k_to_f64_dot(int n, const float* __restrict__ z32, double* __restrict__ z64,
                             const double* __restrict__ b, Reducer red, int slot, int do_red) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double zi = (double)z32[i];
    z64[i] = zi;
    acc += b[i] * zi;
  }
  if (do_red) reduce_finish(acc, red, slot);
}

__global__ void k_pcg_direction(int n, double* __restrict__ p, const double* __restrict__ z,
                                const double* __restrict__ scal, const double* __restrict__ stat,
                                double* __restrict__ x, int vec) {
  pdl_entry();
  // graph-resident loop: before the first iteration (stat[0] == 0) p = z,
  // exactly the host loop's copy
  if (stat && stat[0] == 0.0) {
    for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) p[i] = z[i];
    return;
  }
  const double beta = scal[S_RZ] / scal[S_RZ_OLD];
  if (x) {  // the previous iteration's x += alpha p (alpha = rz_old / pq), deferred from its update
    const double alpha = scal[S_RZ_OLD] / scal[S_PQ];
    const long n2 = vec ? n / 2 : 0;  // element pairs, 16-byte accesses
    for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
      const double2 pi = reinterpret_cast<const double2*>(p)[i], zi = reinterpret_cast<const double2*>(z)[i];
      double2 xi = reinterpret_cast<const double2*>(x)[i];
      xi.x += alpha * pi.x;
      xi.y += alpha * pi.y;
      reinterpret_cast<double2*>(x)[i] = xi;
      reinterpret_cast<double2*>(p)[i] = make_double2(zi.x + beta * pi.x, zi.y + beta * pi.y);
    }
    for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
      const double pi = p[i];
      x[i] += alpha * pi;
      p[i] = z[i] + beta * pi;
    }
    return;
  }
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    p[i] = z[i] + beta * p[i];
}

// the last iteration's deferred x += alpha p (alpha = rz / pq)
__global__ void k_pcg_xfinal(int n, double* __restrict__ x, const double* __restrict__ p,
                             const double* __restrict__ scal) {
  pdl_entry();
  const double alpha = scal[S_RZ] / scal[S_PQ];
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) x[i] += alpha * p[i];
}

// Initial residual test of the graph-resident loop (pcg.cpp:19-31): rr from
// stat[7] (zero start: b.b) or S_RR (x0 start), rel = sqrt(rr) / bnorm.
__global__ void k_pcg_check0(double* __restrict__ scal, double* __restrict__ stat, cudaGraphConditionalHandle h) {
  const double rr = stat[7] < 0.0 ? scal[S_RR] : stat[7];
  const double rel = sqrt(rr) / stat[4];
  int status = PCG_CONTINUE;
  if (!isfinite(rel))
    status = PCG_BAD_INIT;
  else if (rel <= stat[5])
    status = PCG_CONVERGED;
  stat[1] = status;
  stat[2] = rel;
  stat[8] = rel;
  cudaGraphSetConditional(h, status == PCG_CONTINUE ? 1u : 0u);
}

// Same tests, same order and same arithmetic as the host loop in
// GpuSystem::pcg_dev (sqrt and division are correctly rounded on both sides).
__global__ void k_pcg_check(double* __restrict__ scal, double* __restrict__ stat, cudaGraphConditionalHandle h) {
  const double pq = scal[S_PQ], rr = scal[S_RR], rz = scal[S_RZ];
  const double k = stat[0] + 1.0;
  const double rel = sqrt(rr) / stat[4];
  int status = PCG_CONTINUE;
  if (!isfinite(rz))
    status = PCG_BAD_RZ;
  else if (!(pq > 0.0) || !isfinite(pq))
    status = PCG_BAD_PQ;
  else if (!isfinite(rel))
    status = PCG_BAD_REL;
  else if (rel <= stat[5])
    status = PCG_CONVERGED;
  else if (k >= stat[6])
    status = PCG_MAX_ITER;
  stat[0] = k;
  stat[1] = status;
  stat[2] = rel;
  stat[3] = pq;
  if (status == PCG_CONTINUE) scal[S_RZ_OLD] = rz;
  cudaGraphSetConditional(h, status == PCG_CONTINUE ? 1u : 0u);
}

__global__ void k_dot(int n, const double* __restrict__ a, const double* __restrict__ b, Reducer red, int slot) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) acc += a[i] * b[i];
  reduce_finish(acc, red, slot);
}

struct PtrPack {
  const double* p[kMaxMulti];
};

// 16-byte loads over element pairs; an odd last element goes to thread 0 of block 0
__global__ void k_multi_dot(int n, int m, PtrPack V, const double* __restrict__ w, Reducer red, int slot0,
                            int vec) {
  pdl_entry();
  double acc[kMaxMulti];
#pragma unroll
  for (int k = 0; k < kMaxMulti; ++k) acc[k] = 0.0;
  const long n2 = vec ? n / 2 : 0;  // vec: every vector 16-byte aligned
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
    const double2 wi = w2[i];
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)
      if (k < m) {
        const double2 v = reinterpret_cast<const double2*>(V.p[k])[i];
        acc[k] += v.x * wi.x;
        acc[k] += v.y * wi.y;
      }
  }
  for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double wi = w[i];
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)
      if (k < m) acc[k] += V.p[k][i] * wi;
  }
#pragma unroll
  for (int k = 0; k < kMaxMulti; ++k)  // constant indices keep acc in registers
    if (k < m) reduce_finish(acc[k], red, slot0 + k);
}
template <bool ACC>
__global__ void k_lincomb(int n, int m, PtrPack V, CoefPack c, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double s = ACC ? y[i] : 0.0;
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)  // constant indices: the packs stay in parameter space
      if (k < m) s += V.p[k][i] * c.c[k];
    y[i] = s;
  }
}

// w -= sum_j c_j Q_j ; slot <- w.w   (one Gram-Schmidt projection pass)
__global__ void k_orth_update(int n, int m, PtrPack Q, CoefPack c, double* __restrict__ w, Reducer red, int slot) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double s = w[i];
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)
      if (k < m) s -= c.c[k] * Q.p[k][i];
    w[i] = s;
    acc += s * s;
  }
  reduce_finish(acc, red, slot);
}

// the same pass with the coefficients read from device memory (the multi-dot
// slots), so no host round trip sits between the two kernels
__global__ void k_orth_update_dev(int n, int m, PtrPack Q, const double* __restrict__ dcoef,
                                  double* __restrict__ w, Reducer red, int slot) {
  pdl_entry();
  double c[kMaxMulti];
#pragma unroll
  for (int k = 0; k < kMaxMulti; ++k) c[k] = k < m ? dcoef[k] : 0.0;
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double s = w[i];
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)
      if (k < m) s -= c[k] * Q.p[k][i];
    w[i] = s;
    acc += s * s;
  }
  reduce_finish(acc, red, slot);
}

__global__ void k_scale_rsqrt(int n, const double* __restrict__ nrm2, const double* __restrict__ x,
                              double* __restrict__ y) {
  pdl_entry();
  const double a = 1.0 / sqrt(*nrm2);  // the host's 1.0 / std::sqrt(.)
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = a * x[i];
}

// out_j = sum_i T[i][j] in_i  (basis rotation of the SPE window, T by value)
// KIN inputs held in registers (a runtime-indexed array would live in local
// memory); element pairs with 16-byte loads and stores
template <int KIN>
__global__ void k_lincomb_multi(int n, int kout, PtrPack in, PtrPack out, RotPack T, int vec) {
  pdl_entry();
  const long n2 = vec ? n / 2 : 0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
    double2 v[KIN];
#pragma unroll
    for (int a = 0; a < KIN; ++a) v[a] = reinterpret_cast<const double2*>(in.p[a])[i];
#pragma unroll
    for (int b = 0; b < KIN; ++b)
      if (b < kout) {
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int a = 0; a < KIN; ++a) {
          sx += T.t[a][b] * v[a].x;
          sy += T.t[a][b] * v[a].y;
        }
        reinterpret_cast<double2*>(const_cast<double*>(out.p[b]))[i] = make_double2(sx, sy);
      }
  }
  for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double v[KIN];
#pragma unroll
    for (int a = 0; a < KIN; ++a) v[a] = in.p[a][i];
#pragma unroll
    for (int b = 0; b < KIN; ++b)
      if (b < kout) {
        double sv = 0.0;
#pragma unroll
        for (int a = 0; a < KIN; ++a) sv += T.t[a][b] * v[a];
        const_cast<double*>(out.p[b])[i] = sv;
      }
  }
}


// Window kernels of the SPE / POD estimators, templated on the window size M
// (loads unpredicated, accumulators and coefficients in registers) and run on
// element pairs with 16-byte accesses when every vector is 16-byte aligned
// (vec); the remaining elements take a scalar grid-stride loop.
template <int M>
__global__ void k_multi_dot_t(int n, PtrPack V, const double* __restrict__ w, Reducer red, int slot0, int vec) {
  pdl_entry();
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) acc[k] = 0.0;
  const long n2 = vec ? n / 2 : 0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
    const double2 wi = reinterpret_cast<const double2*>(w)[i];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double2 v = reinterpret_cast<const double2*>(V.p[k])[i];
      acc[k] += v.x * wi.x;
      acc[k] += v.y * wi.y;
    }
  }
  for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double wi = w[i];
#pragma unroll
    for (int k = 0; k < M; ++k) acc[k] += V.p[k][i] * wi;
  }
#pragma unroll
  for (int k = 0; k < M; ++k) reduce_finish(acc[k], red, slot0 + k);
}

template <int M, bool ACC>
__global__ void k_lincomb_t(int n, PtrPack V, CoefPack c, double* __restrict__ y, int vec) {
  pdl_entry();
  const long n2 = vec ? n / 2 : 0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
    double2 sacc = ACC ? reinterpret_cast<const double2*>(y)[i] : make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double2 v = reinterpret_cast<const double2*>(V.p[k])[i];
      sacc.x += v.x * c.c[k];
      sacc.y += v.y * c.c[k];
    }
    reinterpret_cast<double2*>(y)[i] = sacc;
  }
  for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double sv = ACC ? y[i] : 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) sv += V.p[k][i] * c.c[k];
    y[i] = sv;
  }
}

template <int M>
__global__ void k_orth_update_t(int n, PtrPack Q, const double* __restrict__ dcoef, double* __restrict__ w,
                                Reducer red, int slot, int vec) {
  pdl_entry();
  double c[M];
#pragma unroll
  for (int k = 0; k < M; ++k) c[k] = dcoef[k];
  double acc = 0.0;
  const long n2 = vec ? n / 2 : 0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n2; i += (long)gridDim.x * kBlock) {
    double2 sv = reinterpret_cast<const double2*>(w)[i];
#pragma unroll
    for (int k = 0; k < M; ++k) {
      const double2 q = reinterpret_cast<const double2*>(Q.p[k])[i];
      sv.x -= c[k] * q.x;
      sv.y -= c[k] * q.y;
    }
    reinterpret_cast<double2*>(w)[i] = sv;
    acc += sv.x * sv.x;
    acc += sv.y * sv.y;
  }
  for (long i = 2 * n2 + (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double sv = w[i];
#pragma unroll
    for (int k = 0; k < M; ++k) sv -= c[k] * Q.p[k][i];
    w[i] = sv;
    acc += sv * sv;
  }
  reduce_finish(acc, red, slot);
}

#define WIN_SWITCH_(m, X) \
  switch (m) {            \
    X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) \
    default: throw std::invalid_argument("estimator window kernels: at most kMaxMulti vectors"); \
  }

// SDIRK Newton matrix values on the M_II pattern: k_e = sum of the element
// contributions in ascending tet order from 0.0 (assemble_matrix), then
// shifted_e = 1.0 m_e + gdt k_e (csr.cpp:168-195 with equal patterns)
__global__ void k_shift_gather(long nnz, const long* __restrict__ ptr, const long* __restrict__ src,
                               const double* __restrict__ S, const double* __restrict__ m, double gdt,
                               double* __restrict__ shifted) {
  pdl_entry();
  for (long e = (long)blockIdx.x * kBlock + threadIdx.x; e < nnz; e += (long)gridDim.x * kBlock) {
    double k = 0.0;
    for (long c = ptr[e]; c < ptr[e + 1]; ++c) k = __dadd_rn(k, S[src[c]]);
    shifted[e] = __dadd_rn(m[e], __dmul_rn(gdt, k));
  }
}
// diag[i] = a_ii (CSR with sorted columns)
__global__ void k_csr_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                           double* __restrict__ d) {
  pdl_entry();
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
    double s = 0.0;
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i) s = v[k];
    d[i] = s;
  }
}
// z = r / d (JacobiPreconditioner, preconditioners.cpp:22-32) ; slot <- r.z
__global__ void k_jacobi_div(int n, const double* __restrict__ d, const double* __restrict__ r, double* __restrict__ z,
                             Reducer red, int slot) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double zi = r[i] / d[i];
    z[i] = zi;
    acc += r[i] * zi;
  }
  reduce_finish(acc, red, slot);
}
// weighted_rms (integrators.cpp:20-31) sum: (est_i / (atol + rtol max(|x_i|, |xn_i|)))^2
__global__ void k_weighted_sq(int n, const double* __restrict__ est, const double* __restrict__ x,
                              const double* __restrict__ xn, double atol, double rtol, Reducer red, int slot) {
  pdl_entry();
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double w = atol + rtol * fmax(fabs(x[i]), fabs(xn[i]));
    const double e = est[i] / w;
    acc += e * e;
  }
  reduce_finish(acc, red, slot);
}

__global__ void k_axpy(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] += a * x[i];
}
__global__ void k_axpy_dev(int n, const double* __restrict__ coef, double sign, const double* __restrict__ x,
                           double* __restrict__ y) {
  pdl_entry();
  const double a = sign * coef[0];
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] += a * x[i];
}
template <class XT>
__global__ void k_diag_scale(int n, const XT* __restrict__ invd, const XT* __restrict__ b, double a,
                             XT* __restrict__ z) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    z[i] = (XT)(a * invd[i] * b[i]);
}
__global__ void k_scale(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = a * x[i];
}
__global__ void k_fill(long n, double v, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = v;
}

__global__ void k_rkc_stage(int n, double a0, double mu, double nu, double mt, double gt,
                            const double* __restrict__ y0, const double* __restrict__ y1,
                            const double* __restrict__ y2, const double* __restrict__ f,
                            const double* __restrict__ f0, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    y[i] = a0 * y0[i] + mu * y1[i] + nu * y2[i] + mt * f[i] + gt * f0[i];
}
__global__ void k_axpby_into(int n, const double* __restrict__ y0, double c, const double* __restrict__ f,
                             double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = y0[i] + c * f[i];
}

__global__ void k_rkc_error(int n, const double* __restrict__ x, const double* __restrict__ xn,
                            const double* __restrict__ f0, const double* __restrict__ fn, double dt, double atol,
                            double rtol, Reducer red, int slot) {
  pdl_entry();
  const double c = 0.4 * dt;
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double xo = x[i], xv = xn[i];
    const double est = 0.8 * (xo - xv) + c * (f0[i] + fn[i]);
    const double w = atol + rtol * fmax(fabs(xo), fabs(xv));
    const double e = est / w;
    acc += e * e;
  }
  reduce_finish(acc, red, slot);
}

template <class T>
__global__ void k_gather(int n, const int* __restrict__ idx, const T* __restrict__ x, T* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = x[idx[i]];
}
__global__ void k_scatter(int n, const int* __restrict__ idx, const double* __restrict__ x, double* __restrict__ y) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[idx[i]] = x[i];
}
__global__ void k_lift_fixed(int n, const int* __restrict__ set_of, SetVals vals, double* __restrict__ out) {
  pdl_entry();
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    out[i] = vals.v[set_of[i]];
}
__global__ void k_boundary_load(int n, const int* __restrict__ rows, const double* __restrict__ coef, int ns,
                                SetVals rates, double* __restrict__ r) {
  pdl_entry();
  for (long k = (long)blockIdx.x * kBlock + threadIdx.x; k < n; k += (long)gridDim.x * kBlock) {
    double s = 0.0;
    for (int j = 0; j < ns; ++j) s += coef[k * ns + j] * rates.v[j];
    r[rows[k]] += -s;
  }
}

}  // namespace

void launch_pcg_update(int n, double* x, double* r, const double* p, const double* q, Reducer red, cudaStream_t s,
                       float* r32, const float* invd32, float* d32) {
  ++g_launch_count;
  auto al = [](const void* ptr, int a) { return ((uintptr_t)ptr % a) == 0; };
  // the paired path (and so the r.r summation order) is chosen from r/p/q
  // only: the host loop (x given) and the graph loop (x deferred) must sum
  // r.r identically whatever the caller's x alignment
  const bool vec = al(r, 16) && al(p, 16) && al(q, 16) && (!r32 || (al(r32, 8) && al(invd32, 8) && al(d32, 8)));
  const long work = vec ? std::max(1, n / 2) : n;
  // r, q in, r out (+ x, p in, x out; + invd32 in, r32 and D^-1 r32 out)
  g_algo_bytes += (24.0 + (x ? 24.0 : 0.0) + (r32 ? 12.0 : 0.0)) * n;
#define U_(F, V, W)                                                                                              \
  launch_pdl(k_pcg_update<F, V, W>, red_grid(k_pcg_update<F, V, W>, work), kBlock, 0, s, n, x, r, p, q, r32, invd32, \
             d32, red)
#define UW_(F, V) \
  if (x) U_(F, V, true); else U_(F, V, false);
  if (r32) {
    if (vec) { UW_(true, true) } else { UW_(true, false) }
  } else {
    if (vec) { UW_(false, true) } else { UW_(false, false) }
  }
#undef UW_
#undef U_
}
void launch_to_f32_scaled(long n, const double* x, const float* invd, float* y, float* d, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  g_algo_bytes += 20.0 * n;
  launch_pdl(k_to_f32_scaled, grid_for(n), kBlock, 0, s, n, x, invd, y, d);
}
void launch_to_f32(long n, const double* x, float* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  g_algo_bytes += 12.0 * n;
  launch_pdl(k_to_f32, grid_for(n), kBlock, 0, s, n, x, y);
}
void launch_to_f64_dot(int n, const float* z32, double* z64, const double* b, Reducer* red, int slot, cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += (red ? 20.0 : 12.0) * n;
  Reducer rr = red ? *red : Reducer{};
  launch_pdl(k_to_f64_dot, red_grid(k_to_f64_dot, n), kBlock, 0, s, n, z32, z64, b, rr, slot, red ? 1 : 0);
}
void launch_pcg_direction(int n, double* p, const double* z, const double* scal, cudaStream_t s,
                          const double* stat, double* x) {
  ++g_launch_count;
  const bool vec = x && aligned16(x) && aligned16(p) && aligned16(z);
  g_algo_bytes += (24.0 + (x ? 16.0 : 0.0)) * n;  // z, p in, p out (+ the deferred x += alpha p: x in and out)
  launch_pdl(k_pcg_direction, grid_for(vec ? n / 2 + 1 : n), kBlock, 0, s, n, p, z, scal, stat, x, vec ? 1 : 0);
}
void launch_pcg_xfinal(int n, double* x, const double* p, const double* scal, cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += 24.0 * n;
  launch_pdl(k_pcg_xfinal, grid_for(n), kBlock, 0, s, n, x, p, scal);
}
void launch_pcg_check0(double* scal, double* stat, cudaGraphConditionalHandle h, cudaStream_t s) {
  ++g_launch_count;
  k_pcg_check0<<<1, 1, 0, s>>>(scal, stat, h);
}
void launch_pcg_check(double* scal, double* stat, cudaGraphConditionalHandle h, cudaStream_t s) {
  ++g_launch_count;
  k_pcg_check<<<1, 1, 0, s>>>(scal, stat, h);
}
template <class XT>
void launch_dense_solve(int n, const double* ainv, const float* ainv32, const XT* b, XT* z, cudaStream_t s) {
  ++g_launch_count;
  if (n <= 256) {  // the hierarchy's own <= 64-row coarsest (amg.hpp:17): one block
    g_algo_bytes += 8.0 * n * n;
    launch_pdl(k_dense_solve<XT>, 1, 1024, n * sizeof(double), s, n, ainv, b, z);
    return;
  }
  const int g = (int)(((long)n * 32 + kBlock - 1) / kBlock);
  if (std::is_same_v<XT, float> && ainv32) {
    g_algo_bytes += 4.0 * n * n + 8.0 * n;
    launch_pdl(k_dense_gemv<float, XT>, g, kBlock, 0, s, n, ainv32, b, z);
  } else {
    g_algo_bytes += 8.0 * n * n + 2.0 * sizeof(XT) * n;
    launch_pdl(k_dense_gemv<double, XT>, g, kBlock, 0, s, n, ainv, b, z);
  }
}
template void launch_dense_solve<double>(int, const double*, const float*, const double*, double*, cudaStream_t);
template void launch_dense_solve<float>(int, const double*, const float*, const float*, float*, cudaStream_t);
void launch_jacobi(int n, const double* invd, const double* r, double* z, Reducer* red, int slot, cudaStream_t s) {
  ++g_launch_count;
  Reducer rr = red ? *red : Reducer{};
  launch_pdl(k_jacobi, red_grid(k_jacobi, n), kBlock, 0, s, n, invd, r, z, rr, slot, red ? 1 : 0);
}
__global__ void __launch_bounds__(kBlock) k_recip(int n, const double* __restrict__ d, double* __restrict__ inv) {
  const int i = blockIdx.x * kBlock + threadIdx.x;
  if (i < n) inv[i] = 1.0 / d[i];
}
void launch_recip(int n, const double* d, double* inv, cudaStream_t s) {
  ++g_launch_count;
  if (n > 0) k_recip<<<(n + kBlock - 1) / kBlock, kBlock, 0, s>>>(n, d, inv);
}
void launch_dot(int n, const double* a, const double* b, Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_dot, red_grid(k_dot, n), kBlock, 0, s, n, a, b, red, slot);
}
void launch_multi_dot(int n, int m, const double* const* V, const double* w, Reducer red, int slot0, cudaStream_t s) {
  if (m <= 0) return;
  ++g_launch_count;
  g_algo_bytes += 8.0 * n * (m + 1);
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = V[k];
  bool vec = aligned16(w);
  for (int k = 0; k < m; ++k) vec = vec && aligned16(V[k]);
#define MD_(M)                                                                                                 \
  case M:                                                                                                      \
    launch_pdl(k_multi_dot_t<M>, red_grid(k_multi_dot_t<M>, n), kBlock, 0, s, n, pk, w, red, slot0, vec ? 1 : 0); \
    break;
  WIN_SWITCH_(m, MD_)
#undef MD_
}
template <bool ACC>
static void lincomb_any(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s) {
  if (m <= 0) {
    if (!ACC) launch_fill(n, 0.0, y, s);
    return;
  }
  ++g_launch_count;
  g_algo_bytes += 8.0 * n * (m + (ACC ? 2 : 1));
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = V[k];
  bool vec = aligned16(y);
  for (int k = 0; k < m; ++k) vec = vec && aligned16(V[k]);
  const int g = grid_for(vec ? n / 2 + 1 : n);
#define LC_(M)                                                                   \
  case M: launch_pdl(k_lincomb_t<M, ACC>, g, kBlock, 0, s, n, pk, c, y, vec ? 1 : 0); break;
  WIN_SWITCH_(m, LC_)
#undef LC_
}
void launch_lincomb(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s) {
  lincomb_any<false>(n, m, V, c, y, s);
}
void launch_lincomb_acc(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s) {
  lincomb_any<true>(n, m, V, c, y, s);
}
void launch_orth_update(int n, int m, const double* const* Q, CoefPack c, double* w, Reducer red, int slot,
                        cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += 8.0 * n * (m + 2);
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = Q[k];
  launch_pdl(k_orth_update, red_grid(k_orth_update, n), kBlock, 0, s, n, m, pk, c, w, red, slot);
}
void launch_orth_update_dev(int n, int m, const double* const* Q, const double* dcoef, double* w, Reducer red,
                            int slot, cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += 8.0 * n * (m > 0 ? m + 2 : 1);
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = Q[k];
  if (m <= 0) {  // no projection: the pass only produces w.w
    launch_pdl(k_orth_update_dev, red_grid(k_orth_update_dev, n), kBlock, 0, s, n, m, pk, dcoef, w, red, slot);
    return;
  }
  bool vec = aligned16(w);
  for (int k = 0; k < m; ++k) vec = vec && aligned16(Q[k]);
#define OU_(M)                                                                                                  \
  case M:                                                                                                       \
    launch_pdl(k_orth_update_t<M>, red_grid(k_orth_update_t<M>, n), kBlock, 0, s, n, pk, dcoef, w, red, slot, \
               vec ? 1 : 0);                                                                                    \
    break;
  WIN_SWITCH_(m, OU_)
#undef OU_
}
void launch_scale_rsqrt(int n, const double* nrm2, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += 16.0 * n;
  launch_pdl(k_scale_rsqrt, grid_for(n), kBlock, 0, s, n, nrm2, x, y);
}
void launch_lincomb_multi(int n, int kin, int kout, const double* const* in, double* const* out, const RotPack& T,
                          cudaStream_t s) {
  ++g_launch_count;
  g_algo_bytes += 8.0 * n * (kin + kout);
  PtrPack pi{}, po{};
  for (int k = 0; k < kin && k < kMaxMulti; ++k) pi.p[k] = in[k];
  for (int k = 0; k < kout && k < kMaxMulti; ++k) po.p[k] = out[k];
  bool vec = true;
  for (int k = 0; k < kin; ++k) vec = vec && aligned16(in[k]);
  for (int k = 0; k < kout; ++k) vec = vec && aligned16(out[k]);
  const int g = grid_for(vec ? n / 2 + 1 : n);
  switch (kin) {
#define LM_(K) \
  case K: launch_pdl(k_lincomb_multi<K>, g, kBlock, 0, s, n, kout, pi, po, T, vec ? 1 : 0); break;
    LM_(1) LM_(2) LM_(3) LM_(4) LM_(5) LM_(6) LM_(7) LM_(8) LM_(9)
#undef LM_
    default: throw std::invalid_argument("lincomb_multi: at most kMaxWin inputs");
  }
}
void launch_shift_gather(long nnz, const long* ptr, const long* src, const double* S, const double* m, double gdt,
                         double* shifted, cudaStream_t s) {
  ++g_launch_count;
  if (nnz == 0) return;
  launch_pdl(k_shift_gather, (int)std::min<long>((nnz + kBlock - 1) / kBlock, 148L * 32), kBlock, 0, s, nnz, ptr, src, S, m,
                                                                                              gdt, shifted);
}
void launch_csr_diag(int n, const int* rp, const int* ci, const double* v, double* d, cudaStream_t s) {
  ++g_launch_count;
  if (n == 0) return;
  launch_pdl(k_csr_diag, grid_for(n), kBlock, 0, s, n, rp, ci, v, d);
}
void launch_jacobi_div(int n, const double* d, const double* r, double* z, Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_jacobi_div, red_grid(k_jacobi_div, n), kBlock, 0, s, n, d, r, z, red, slot);
}
void launch_weighted_sq(int n, const double* est, const double* x, const double* xn, double atol, double rtol,
                        Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_weighted_sq, red_grid(k_weighted_sq, n), kBlock, 0, s, n, est, x, xn, atol, rtol, red, slot);
}
void launch_axpy(int n, double a, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_axpy, grid_for(n), kBlock, 0, s, n, a, x, y);
}
void launch_axpy_dev(int n, const double* coef, double sign, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_axpy_dev, grid_for(n), kBlock, 0, s, n, coef, sign, x, y);
}
template <class XT>
void launch_diag_scale(int n, const XT* invd, const XT* b, double a, XT* z, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  g_algo_bytes += 3.0 * sizeof(XT) * n;
  launch_pdl(k_diag_scale<XT>, grid_for(n), kBlock, 0, s, n, invd, b, a, z);
}
template void launch_diag_scale<double>(int, const double*, const double*, double, double*, cudaStream_t);
template void launch_diag_scale<float>(int, const float*, const float*, double, float*, cudaStream_t);
void launch_scale(int n, double a, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_scale, grid_for(n), kBlock, 0, s, n, a, x, y);
}
void launch_fill(long n, double v, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  launch_pdl(k_fill, grid_for(n), kBlock, 0, s, n, v, y);
}
void launch_rkc_stage(int n, double a0, double mu, double nu, double mt, double gt, const double* y0,
                      const double* y1, const double* y2, const double* f, const double* f0, double* y,
                      cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_rkc_stage, grid_for(n), kBlock, 0, s, n, a0, mu, nu, mt, gt, y0, y1, y2, f, f0, y);
}
void launch_axpby_into(int n, const double* y0, double c, const double* f, double* y, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_axpby_into, grid_for(n), kBlock, 0, s, n, y0, c, f, y);
}
void launch_rkc_error(int n, const double* x, const double* xn, const double* f0, const double* fn, double dt,
                      double atol, double rtol, Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  launch_pdl(k_rkc_error, red_grid(k_rkc_error, n), kBlock, 0, s, n, x, xn, f0, fn, dt, atol, rtol, red, slot);
}
void launch_gather(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  launch_pdl(k_gather<double>, grid_for(n), kBlock, 0, s, n, idx, x, y);
}
void launch_gather_f(int n, const int* idx, const float* x, float* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  launch_pdl(k_gather<float>, grid_for(n), kBlock, 0, s, n, idx, x, y);
}
void launch_scatter(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  launch_pdl(k_scatter, grid_for(n), kBlock, 0, s, n, idx, x, y);
}
void launch_lift_fixed(int n_fixed, const int* set_of_fixed, SetVals set_vals, double* fixed_part, cudaStream_t s) {
  if (n_fixed <= 0) return;
  ++g_launch_count;
  launch_pdl(k_lift_fixed, grid_for(n_fixed), kBlock, 0, s, n_fixed, set_of_fixed, set_vals, fixed_part);
}
void launch_boundary_load(int n_rows, const int* rows, const double* coef, int n_sets, SetVals rates, double* r,
                          cudaStream_t s) {
  if (n_rows <= 0) return;
  ++g_launch_count;
  launch_pdl(k_boundary_load, grid_for(n_rows), kBlock, 0, s, n_rows, rows, coef, n_sets, rates, r);
}

}  // namespace eqsb

