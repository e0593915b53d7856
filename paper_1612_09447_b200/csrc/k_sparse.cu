// Sparse / vector kernels of the M-solve (AMG-PCG) and the RKC recurrence.
// All HBM-bound: CSR rows are read by TPR-thread groups (TPR chosen per
// matrix from the mean row length) so that a warp streams contiguous
// col_idx/values; gathered vectors hit L2. Reductions are fused into the
// producing kernel and finished deterministically (fixed grid, last-block
// ordered sum). V-cycle matrices may be stored with fp32 values (the
// preconditioner only; PCG itself is fp64 throughout).
#include <cuda_runtime.h>

#include <algorithm>
#include <unordered_map>

#include "dev.cuh"

namespace eqsb {

long g_launch_count = 0;

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[kBlock / 32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = l < (kBlock / 32) ? sh[l] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// Store this block's partial; the last block to arrive sums all partials in
// block order and writes the result (deterministic for a fixed grid).
__device__ __forceinline__ void reduce_finish(double v, Reducer red, int slot) {
  __shared__ bool last;
  const double bs = block_sum(v);
  double* part = red.partials + (size_t)slot * kRedGrid;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = bs;
    __threadfence();
    const unsigned prev = atomicAdd(red.counters + slot, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    double acc = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kBlock) acc += __ldcg(part + i);
    acc = block_sum(acc);
    if (threadIdx.x == 0) {
      red.scal[slot] = acc;
      red.counters[slot] = 0u;
    }
  }
}

// Grid of a grid-stride reduction kernel: exactly one wave of resident blocks
// (SMs x blocks-per-SM at this kernel's register use), so no tail wave; the
// grid (hence the summation order) is fixed per kernel: deterministic.
template <class K>
int red_grid(K kernel, long work_items) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  static std::unordered_map<const void*, int> bps_cache;
  const void* key = (const void*)kernel;
  auto it = bps_cache.find(key);
  int bps;
  if (it == bps_cache.end()) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, kBlock, 0) != cudaSuccess || bps < 1) bps = 1;
    bps_cache[key] = bps;
  } else {
    bps = it->second;
  }
  long g = (work_items + kBlock - 1) / kBlock;
  g = std::min<long>(g, std::min<long>((long)sms * bps, kRedGrid));
  return (int)std::max<long>(g, 1);
}

// matrix entries are streamed once per pass: evict-first loads keep L2 for
// the gathered vectors (ld.global.cs)
__device__ __forceinline__ double ldv(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double ldv(const float* p) { return (double)__ldcs(p); }

constexpr int kUnroll = 8;  // independent entries in flight per thread

// Row-group SpMV core: returns sum_k A_ik x_k (x_k w_k when SCALED) for `row`
// in lane 0 of the group. Entries are fetched kUnroll at a time (indices and
// values first, then the gathers) so each thread keeps several independent
// loads in flight. All lanes of the warp must call it (shuffles); rows >= n
// contribute nothing.
template <int TPR, class VT, bool SCALED>
__device__ __forceinline__ double row_dot(const int* __restrict__ rp, const int* __restrict__ ci,
                                          const VT* __restrict__ v, const double* __restrict__ x,
                                          const double* __restrict__ w, int row, int lane, int n) {
  const bool ok = row < n;
  const int beg = ok ? __ldg(rp + row) : 0, end = ok ? __ldg(rp + row + 1) : 0;
  double s = 0.0;
  for (int k0 = beg + lane; k0 < end; k0 += TPR * kUnroll) {
    int c[kUnroll];
    double a[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + u * TPR;
      const bool in = k < end;
      c[u] = in ? __ldcs(ci + k) : 0;
      a[u] = in ? ldv(v + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const double xv = SCALED ? __ldg(x + c[u]) * __ldg(w + c[u]) : __ldg(x + c[u]);
      s += a[u] * xv;
    }
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, TPR);
  return s;
}

// Generic row kernel (one pass over a matrix), warp-uniform early exit.
// OP 0: y = A x                       (restriction, plain SpMV)
// OP 1: y = b - A x                   (residual)
// OP 2: z += A zc                     (prolongation + correction; v = P)
// OP 3: z = c0 D^-1 b + c1 D^-1 (b - A D^-1 b / theta)          (Chebyshev(2) pre-smoothing from 0)
// OP 4: z = D^-1 b / theta ; t = b - A z                         (Chebyshev(1) pre-smoothing + residual)
// OP 5: zo = z + D^-1 (b - A z) / theta                          (Chebyshev(1) post-smoothing, out of place)
// OP 6: w = D^-1 A x                                             (power iteration on D^-1 A)
template <int TPR, class VT, int OP>
__global__ void __launch_bounds__(kBlock) k_row(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const VT* __restrict__ v, const double* __restrict__ x,
                                                const double* __restrict__ b, const double* __restrict__ invd,
                                                double* __restrict__ y, double* __restrict__ y2, ChebCoef c) {
  const long tid = (long)blockIdx.x * kBlock + threadIdx.x;
  const int row = (int)(tid / TPR), lane = (int)(tid % TPR);
  if ((tid & ~31L) / TPR >= n) return;  // warp-uniform exit
  constexpr bool SC = (OP == 3 || OP == 4);
  const double s = row_dot<TPR, VT, SC>(rp, ci, v, SC ? b : x, invd, row, lane, n);
  if (lane != 0 || row >= n) return;
  if (OP == 0) y[row] = s;
  if (OP == 1) y[row] = b[row] - s;
  if (OP == 2) y[row] += s;
  if (OP == 3) {
    const double bi = b[row], di = invd[row];
    y[row] = c.c0 * bi * di + c.c1 * di * (bi - s * c.inv_theta);
  }
  if (OP == 4) {
    const double bi = b[row];
    y[row] = bi * invd[row] * c.inv_theta;
    y2[row] = bi - s * c.inv_theta;
  }
  if (OP == 5) y2[row] = x[row] + invd[row] * (b[row] - s) * c.inv_theta;
  if (OP == 6) y[row] = s * invd[row];
}

// grid-stride row kernels with a fused reduction.
// MODE 0: q = A p,  sum p.q
// MODE 1: y = b - A x, sum y.y
// MODE 2: z += c0 D^-1 r0 + c1 D^-1 (r0 - A D^-1 r0 / theta), sum b.z  (Chebyshev(2) post step 2)
template <int TPR, class VT, int MODE>
__global__ void __launch_bounds__(kBlock) k_row_red(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const VT* __restrict__ v, const double* __restrict__ x,
                                                    const double* __restrict__ b, const double* __restrict__ invd,
                                                    double* __restrict__ y, ChebCoef c, Reducer red, int slot,
                                                    int do_red) {
  const int lane = threadIdx.x % TPR;
  const long groups_per_grid = (long)gridDim.x * (kBlock / TPR);
  // every group iterates the same number of times (shuffles need full warps)
  const long n_pad = ((n + (long)(kBlock / TPR) - 1) / (kBlock / TPR)) * (kBlock / TPR);
  double acc = 0.0;
  for (long row = (long)blockIdx.x * (kBlock / TPR) + threadIdx.x / TPR; row < n_pad; row += groups_per_grid) {
    const double s = row_dot<TPR, VT, MODE == 2>(rp, ci, v, x, invd, (int)row, lane, n);
    if (lane == 0 && row < n) {
      if (MODE == 0) {
        y[row] = s;
        acc += x[row] * s;
      } else if (MODE == 1) {
        const double r = b[row] - s;
        y[row] = r;
        acc += r * r;
      } else {
        const double ri = x[row], di = invd[row];
        const double zn = y[row] + (c.c0 * ri * di + c.c1 * di * (ri - s * c.inv_theta));
        y[row] = zn;
        if (do_red) acc += b[row] * zn;
      }
    }
  }
  if (do_red) reduce_finish(acc, red, slot);
}

__global__ void k_dense_solve(int n, const double* __restrict__ ainv, const double* __restrict__ b,
                              double* __restrict__ z) {
  extern __shared__ double sb[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sb[i] = b[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int row = w; row < n; row += nw) {
    double s = 0.0;
    for (int k = l; k < n; k += 32) s += ainv[(size_t)row * n + k] * sb[k];
    s = warp_sum(s);
    if (l == 0) z[row] = s;
  }
}

__global__ void k_jacobi(int n, const double* __restrict__ invd, const double* __restrict__ r,
                         double* __restrict__ z, Reducer red, int slot, int do_red) {
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double zi = invd[i] * r[i];
    z[i] = zi;
    acc += r[i] * zi;
  }
  if (do_red) reduce_finish(acc, red, slot);
}

__global__ void k_pcg_update(int n, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                             const double* __restrict__ q, Reducer red) {
  const double alpha = red.scal[S_RZ] / red.scal[S_PQ];
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    acc += ri * ri;
  }
  reduce_finish(acc, red, S_RR);
}

__global__ void k_pcg_direction(int n, double* __restrict__ p, const double* __restrict__ z,
                                const double* __restrict__ scal) {
  const double beta = scal[S_RZ] / scal[S_RZ_OLD];
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    p[i] = z[i] + beta * p[i];
}

__global__ void k_dot(int n, const double* __restrict__ a, const double* __restrict__ b, Reducer red, int slot) {
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) acc += a[i] * b[i];
  reduce_finish(acc, red, slot);
}

struct PtrPack {
  const double* p[kMaxMulti];
};

__global__ void k_multi_dot(int n, int m, PtrPack V, const double* __restrict__ w, Reducer red, int slot0) {
  double acc[kMaxMulti];
#pragma unroll
  for (int k = 0; k < kMaxMulti; ++k) acc[k] = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    const double wi = w[i];
#pragma unroll
    for (int k = 0; k < kMaxMulti; ++k)
      if (k < m) acc[k] += V.p[k][i] * wi;
  }
  for (int k = 0; k < m; ++k) reduce_finish(acc[k], red, slot0 + k);
}

__global__ void k_lincomb(int n, int m, PtrPack V, CoefPack c, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double s = 0.0;
    for (int k = 0; k < m; ++k) s += V.p[k][i] * c.c[k];
    y[i] = s;
  }
}

// w -= sum_j c_j Q_j ; slot <- w.w   (one Gram-Schmidt projection pass)
__global__ void k_orth_update(int n, int m, PtrPack Q, CoefPack c, double* __restrict__ w, Reducer red, int slot) {
  double acc = 0.0;
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double s = w[i];
    for (int k = 0; k < m; ++k) s -= c.c[k] * Q.p[k][i];
    w[i] = s;
    acc += s * s;
  }
  reduce_finish(acc, red, slot);
}

// out_j = sum_i T[i][j] in_i  (basis rotation of the SPE window, T by value)
__global__ void k_lincomb_multi(int n, int kin, int kout, PtrPack in, PtrPack out, RotPack T) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) {
    double v[kMaxMulti];
    for (int a = 0; a < kin; ++a) v[a] = in.p[a][i];
    for (int b = 0; b < kout; ++b) {
      double s = 0.0;
      for (int a = 0; a < kin; ++a) s += T.t[a][b] * v[a];
      const_cast<double*>(out.p[b])[i] = s;
    }
  }
}

__global__ void k_axpy(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] += a * x[i];
}
__global__ void k_axpy_dev(int n, const double* __restrict__ coef, double sign, const double* __restrict__ x,
                           double* __restrict__ y) {
  const double a = sign * coef[0];
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] += a * x[i];
}
__global__ void k_diag_scale(int n, const double* __restrict__ invd, const double* __restrict__ b, double a,
                             double* __restrict__ z) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) z[i] = a * invd[i] * b[i];
}
__global__ void k_scale(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = a * x[i];
}
__global__ void k_fill(long n, double v, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = v;
}

__global__ void k_rkc_stage(int n, double a0, double mu, double nu, double mt, double gt,
                            const double* __restrict__ y0, const double* __restrict__ y1,
                            const double* __restrict__ y2, const double* __restrict__ f,
                            const double* __restrict__ f0, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    y[i] = a0 * y0[i] + mu * y1[i] + nu * y2[i] + mt * f[i] + gt * f0[i];
}
__global__ void k_axpby_into(int n, const double* __restrict__ y0, double c, const double* __restrict__ f,
                             double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = y0[i] + c * f[i];
}

__global__ void k_rkc_error(int n, const double* __restrict__ x, const double* __restrict__ xn,
                            const double* __restrict__ f0, const double* __restrict__ fn, double dt, double atol,
                            double rtol, Reducer red, int slot) {
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

__global__ void k_gather(int n, const int* __restrict__ idx, const double* __restrict__ x, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[i] = x[idx[i]];
}
__global__ void k_scatter(int n, const int* __restrict__ idx, const double* __restrict__ x, double* __restrict__ y) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock) y[idx[i]] = x[i];
}
__global__ void k_lift_fixed(int n, const int* __restrict__ set_of, SetVals vals, double* __restrict__ out) {
  for (long i = (long)blockIdx.x * kBlock + threadIdx.x; i < n; i += (long)gridDim.x * kBlock)
    out[i] = vals.v[set_of[i]];
}
__global__ void k_boundary_load(int n, const int* __restrict__ rows, const double* __restrict__ coef, int ns,
                                SetVals rates, double* __restrict__ r) {
  for (long k = (long)blockIdx.x * kBlock + threadIdx.x; k < n; k += (long)gridDim.x * kBlock) {
    double s = 0.0;
    for (int j = 0; j < ns; ++j) s += coef[k * ns + j] * rates.v[j];
    r[rows[k]] += -s;
  }
}

inline int grid_for(long n) {
  long g = (n + kBlock - 1) / kBlock;
  const long cap = 148L * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}
inline int grid_rows(long n_rows, int tpr) {
  long g = (n_rows * tpr + kBlock - 1) / kBlock;
  return (int)(g < 1 ? 1 : g);
}

template <int OP>
void row_launch(const DevCsr& a, const double* x, const double* b, const double* invd, double* y, double* y2,
                ChebCoef c, cudaStream_t s) {
  if (a.n_rows == 0) return;
  ++g_launch_count;
  const int g = grid_rows(a.n_rows, a.tpr);
#define L_(T, VT, V) \
  k_row<T, VT, OP><<<g, kBlock, 0, s>>>(a.n_rows, a.row_ptr, a.col_idx, V, x, b, invd, y, y2, c)
#define D_(VT, V)                \
  switch (a.tpr) {               \
    case 1: L_(1, VT, V); break;   \
    case 2: L_(2, VT, V); break;   \
    case 4: L_(4, VT, V); break;   \
    case 8: L_(8, VT, V); break;   \
    case 16: L_(16, VT, V); break; \
    default: L_(32, VT, V); break; \
  }
  if (a.values_f) {
    D_(float, a.values_f)
  } else {
    D_(double, a.values)
  }
#undef D_
#undef L_
}

template <int MODE>
void row_red_launch(const DevCsr& a, const double* x, const double* b, const double* invd, double* y, ChebCoef c,
                    Reducer* red, int slot, cudaStream_t s) {
  if (a.n_rows == 0) return;
  ++g_launch_count;
  const long work = (long)a.n_rows * a.tpr;
  Reducer r = red ? *red : Reducer{};
  const int dr = red ? 1 : 0;
#define L_(T, VT, V)                                                                                       \
  k_row_red<T, VT, MODE><<<red_grid(k_row_red<T, VT, MODE>, work), kBlock, 0, s>>>(                         \
      a.n_rows, a.row_ptr, a.col_idx, V, x, b, invd, y, c, r, slot, dr)
#define D_(VT, V)                \
  switch (a.tpr) {               \
    case 1: L_(1, VT, V); break;   \
    case 2: L_(2, VT, V); break;   \
    case 4: L_(4, VT, V); break;   \
    case 8: L_(8, VT, V); break;   \
    case 16: L_(16, VT, V); break; \
    default: L_(32, VT, V); break; \
  }
  if (a.values_f) {
    D_(float, a.values_f)
  } else {
    D_(double, a.values)
  }
#undef D_
#undef L_
}

}  // namespace

void launch_spmv(const DevCsr& a, const double* x, double* y, cudaStream_t s) {
  row_launch<0>(a, x, nullptr, nullptr, y, nullptr, ChebCoef{}, s);
}
void launch_residual(const DevCsr& a, const double* b, const double* x, double* y, Reducer* red, int slot,
                     cudaStream_t s) {
  if (red) row_red_launch<1>(a, x, b, nullptr, y, ChebCoef{}, red, slot, s);
  else row_launch<1>(a, x, b, nullptr, y, nullptr, ChebCoef{}, s);
}
void launch_spmv_dot(const DevCsr& a, const double* p, double* q, Reducer red, int slot, cudaStream_t s) {
  row_red_launch<0>(a, p, nullptr, nullptr, q, ChebCoef{}, &red, slot, s);
}
void launch_prolong_add(const DevCsr& p, const double* zc, double* z, cudaStream_t s) {
  row_launch<2>(p, zc, nullptr, nullptr, z, nullptr, ChebCoef{}, s);
}
void launch_cheb_pre(const DevCsr& a, const double* invd, const double* b, double* z, ChebCoef c, cudaStream_t s) {
  row_launch<3>(a, nullptr, b, invd, z, nullptr, c, s);
}
void launch_cheb_post2(const DevCsr& a, const double* invd, const double* r0, double* z, ChebCoef c,
                       const double* b_dot, Reducer* red, int slot, cudaStream_t s) {
  row_red_launch<2>(a, r0, b_dot, invd, z, c, red, slot, s);
}
void launch_cheb1_pre_resid(const DevCsr& a, const double* invd, const double* b, double* z, double* t, ChebCoef c,
                            cudaStream_t s) {
  row_launch<4>(a, nullptr, b, invd, z, t, c, s);
}
void launch_cheb1_post(const DevCsr& a, const double* invd, const double* b, const double* z, double* z_out,
                       ChebCoef c, cudaStream_t s) {
  row_launch<5>(a, z, b, invd, nullptr, z_out, c, s);
}
void launch_scaled_spmv(const DevCsr& a, const double* invd, const double* v, double* w, cudaStream_t s) {
  row_launch<6>(a, v, nullptr, invd, w, nullptr, ChebCoef{}, s);
}

void launch_pcg_update(int n, double* x, double* r, const double* p, const double* q, Reducer red, cudaStream_t s) {
  ++g_launch_count;
  k_pcg_update<<<red_grid(k_pcg_update, n), kBlock, 0, s>>>(n, x, r, p, q, red);
}
void launch_pcg_direction(int n, double* p, const double* z, const double* scal, cudaStream_t s) {
  ++g_launch_count;
  k_pcg_direction<<<grid_for(n), kBlock, 0, s>>>(n, p, z, scal);
}
void launch_dense_solve(int n, const double* ainv, const double* b, double* z, cudaStream_t s) {
  ++g_launch_count;
  k_dense_solve<<<1, 1024, n * sizeof(double), s>>>(n, ainv, b, z);
}
void launch_jacobi(int n, const double* invd, const double* r, double* z, Reducer* red, int slot, cudaStream_t s) {
  ++g_launch_count;
  Reducer rr = red ? *red : Reducer{};
  k_jacobi<<<red_grid(k_jacobi, n), kBlock, 0, s>>>(n, invd, r, z, rr, slot, red ? 1 : 0);
}
void launch_dot(int n, const double* a, const double* b, Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  k_dot<<<red_grid(k_dot, n), kBlock, 0, s>>>(n, a, b, red, slot);
}
void launch_multi_dot(int n, int m, const double* const* V, const double* w, Reducer red, int slot0, cudaStream_t s) {
  ++g_launch_count;
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = V[k];
  k_multi_dot<<<red_grid(k_multi_dot, n), kBlock, 0, s>>>(n, m, pk, w, red, slot0);
}
void launch_lincomb(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s) {
  ++g_launch_count;
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = V[k];
  k_lincomb<<<grid_for(n), kBlock, 0, s>>>(n, m, pk, c, y);
}
void launch_orth_update(int n, int m, const double* const* Q, CoefPack c, double* w, Reducer red, int slot,
                        cudaStream_t s) {
  ++g_launch_count;
  PtrPack pk{};
  for (int k = 0; k < m && k < kMaxMulti; ++k) pk.p[k] = Q[k];
  k_orth_update<<<red_grid(k_orth_update, n), kBlock, 0, s>>>(n, m, pk, c, w, red, slot);
}
void launch_lincomb_multi(int n, int kin, int kout, const double* const* in, double* const* out, const RotPack& T,
                          cudaStream_t s) {
  ++g_launch_count;
  PtrPack pi{}, po{};
  for (int k = 0; k < kin && k < kMaxMulti; ++k) pi.p[k] = in[k];
  for (int k = 0; k < kout && k < kMaxMulti; ++k) po.p[k] = out[k];
  k_lincomb_multi<<<grid_for(n), kBlock, 0, s>>>(n, kin, kout, pi, po, T);
}
void launch_axpy(int n, double a, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  k_axpy<<<grid_for(n), kBlock, 0, s>>>(n, a, x, y);
}
void launch_axpy_dev(int n, const double* coef, double sign, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  k_axpy_dev<<<grid_for(n), kBlock, 0, s>>>(n, coef, sign, x, y);
}
void launch_diag_scale(int n, const double* invd, const double* b, double a, double* z, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  k_diag_scale<<<grid_for(n), kBlock, 0, s>>>(n, invd, b, a, z);
}
void launch_scale(int n, double a, const double* x, double* y, cudaStream_t s) {
  ++g_launch_count;
  k_scale<<<grid_for(n), kBlock, 0, s>>>(n, a, x, y);
}
void launch_fill(long n, double v, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  k_fill<<<grid_for(n), kBlock, 0, s>>>(n, v, y);
}
void launch_rkc_stage(int n, double a0, double mu, double nu, double mt, double gt, const double* y0,
                      const double* y1, const double* y2, const double* f, const double* f0, double* y,
                      cudaStream_t s) {
  ++g_launch_count;
  k_rkc_stage<<<grid_for(n), kBlock, 0, s>>>(n, a0, mu, nu, mt, gt, y0, y1, y2, f, f0, y);
}
void launch_axpby_into(int n, const double* y0, double c, const double* f, double* y, cudaStream_t s) {
  ++g_launch_count;
  k_axpby_into<<<grid_for(n), kBlock, 0, s>>>(n, y0, c, f, y);
}
void launch_rkc_error(int n, const double* x, const double* xn, const double* f0, const double* fn, double dt,
                      double atol, double rtol, Reducer red, int slot, cudaStream_t s) {
  ++g_launch_count;
  k_rkc_error<<<red_grid(k_rkc_error, n), kBlock, 0, s>>>(n, x, xn, f0, fn, dt, atol, rtol, red, slot);
}
void launch_gather(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  k_gather<<<grid_for(n), kBlock, 0, s>>>(n, idx, x, y);
}
void launch_scatter(int n, const int* idx, const double* x, double* y, cudaStream_t s) {
  if (n <= 0) return;
  ++g_launch_count;
  k_scatter<<<grid_for(n), kBlock, 0, s>>>(n, idx, x, y);
}
void launch_lift_fixed(int n_fixed, const int* set_of_fixed, SetVals set_vals, double* fixed_part, cudaStream_t s) {
  if (n_fixed <= 0) return;
  ++g_launch_count;
  k_lift_fixed<<<grid_for(n_fixed), kBlock, 0, s>>>(n_fixed, set_of_fixed, set_vals, fixed_part);
}
void launch_boundary_load(int n_rows, const int* rows, const double* coef, int n_sets, SetVals rates, double* r,
                          cudaStream_t s) {
  if (n_rows <= 0) return;
  ++g_launch_count;
  k_boundary_load<<<grid_for(n_rows), kBlock, 0, s>>>(n_rows, rows, coef, n_sets, rates, r);
}

}  // namespace eqsb
