// Device SA-AMG setup kernels: strength graph, greedy
// aggregation, tentative prolongator, lambda_max power iteration, transposition
// and the diagonal check. Every result is bit-identical to the sequential
// reference algorithm (proj/src/amg.cpp:15-143, csr.cpp:52-70,
// preconditioners.cpp:7-20); tests/test_gpu_amg_setup.py compares the whole
// hierarchy with the host build and the reference fixtures.
//
// Aggregation (amg.cpp:49-88) is three sequential greedy passes in index order.
// The device computes the same result without a sequential sweep:
//
// * Pass 1 makes i a root iff S(i) is non-empty and no earlier root claims a
//   node that i would claim (claimed(i) = {i} U S(i)): the lexicographically
//   first maximal set of candidates with pairwise disjoint claimed sets. It is
//   resolved in rounds over the undecided candidates: a candidate that meets a
//   node already taken by a root is not a root; every other candidate writes
//   atomicMin(m[k], i) on its claimed nodes, and a candidate that is the
//   smallest live claimant of all of its nodes becomes a root (every smaller
//   conflicting candidate has been decided "not a root"). Roots are numbered
//   in index order by a scan, which is the order the sequential loop uses.
// * Pass 2 attaches a leftover node to the aggregate of its strongest
//   aggregated neighbour (first maximum in row order). Earlier leftovers count
//   as aggregated once they are attached. Node i is resolved in the first
//   round in which none of its unresolved smaller leftover neighbours could
//   still be the first maximum of its row scan.
// * Pass 3 numbers the remaining nodes in index order (scan).
//
// The round loops run until their worklists are empty; the result does not
// depend on the order threads run in.
#include <cub/cub.cuh>

#include <climits>
#include <cmath>
#include <random>
#include <string>

#include "amg_device.hpp"

namespace eqsb {

double seq_norm(const std::vector<double>& v);  // host_setup.cpp (Eigen's reduction order)

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("amg setup: ") + what + ": " + cudaGetErrorString(e));
}

inline int blocks_for(long long n, int bs = 256) { return (int)std::max<long long>(1, (n + bs - 1) / bs); }

__global__ void k_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                       double* __restrict__ d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] == i) {
      x = v[k];
      break;
    }
  d[i] = x;
}

// first row with a missing or zero diagonal (preconditioners.cpp:7-20)
__global__ void k_check_diag(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                             const double* __restrict__ v, int* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int pos = -1;
  for (int k = rp[i]; k < rp[i + 1]; ++k)
    if (ci[k] == i) {
      pos = k;
      break;
    }
  if (pos < 0 || v[pos] == 0.0) atomicMin(bad, i);
}

// |a_ij| >= theta sqrt(|a_ii a_jj|), j != i (amg.cpp:15-26), in the host's expression order
__device__ __forceinline__ bool is_strong(double a, double di, double dj, double theta) {
  return fabs(a) >= __dmul_rn(theta, __dsqrt_rn(fabs(__dmul_rn(di, dj))));
}

__global__ void k_strong_count(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                               const double* __restrict__ v, const double* __restrict__ d, double theta,
                               int* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  const double di = d[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    if (j != i && is_strong(v[k], di, d[j], theta)) ++c;
  }
  cnt[i] = c;
}

__global__ void k_strong_fill(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, const double* __restrict__ d, double theta,
                              const int* __restrict__ srp, int* __restrict__ sci) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int pos = srp[i];
  const double di = d[i];
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    if (j != i && is_strong(v[k], di, d[j], theta)) sci[pos++] = j;
  }
}

enum : unsigned char { kUndecided = 0, kRoot = 1, kNotRoot = 2 };

// candidates (non-empty S(i)) in index order
__global__ void k_pass1_init(int n, const int* __restrict__ srp, unsigned char* __restrict__ st,
                             int* __restrict__ taken, int* __restrict__ m, int* __restrict__ list,
                             int* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  taken[i] = -1;
  m[i] = INT_MAX;
  const bool cand = srp[i + 1] > srp[i];
  st[i] = cand ? kUndecided : kNotRoot;
  if (cand) list[atomicAdd(count, 1)] = i;
}

// a candidate meeting a taken node is not a root; the others bid for their claimed nodes
__global__ void k_pass1_bid(int nl, const int* __restrict__ list, const int* __restrict__ srp,
                            const int* __restrict__ sci, unsigned char* __restrict__ st,
                            const int* __restrict__ taken, int* __restrict__ m) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const int i = list[t];
  const int k0 = srp[i], k1 = srp[i + 1];
  bool hit = taken[i] >= 0;
  for (int k = k0; k < k1 && !hit; ++k) hit = taken[sci[k]] >= 0;
  if (hit) {
    st[i] = kNotRoot;
    return;
  }
  atomicMin(&m[i], i);
  for (int k = k0; k < k1; ++k) atomicMin(&m[sci[k]], i);
}

// the smallest live claimant of every claimed node becomes a root and takes them
__global__ void k_pass1_claim(int nl, const int* __restrict__ list, const int* __restrict__ srp,
                              const int* __restrict__ sci, unsigned char* __restrict__ st, int* __restrict__ taken,
                              const int* __restrict__ m) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const int i = list[t];
  if (st[i] != kUndecided) return;
  const int k0 = srp[i], k1 = srp[i + 1];
  bool min_all = m[i] == i;
  for (int k = k0; k < k1 && min_all; ++k) min_all = m[sci[k]] == i;
  if (!min_all) return;
  st[i] = kRoot;
  taken[i] = i;
  for (int k = k0; k < k1; ++k) taken[sci[k]] = i;
}

// reset the bids of this round and keep the undecided candidates
__global__ void k_pass1_next(int nl, const int* __restrict__ list, const int* __restrict__ srp,
                             const int* __restrict__ sci, const unsigned char* __restrict__ st, int* __restrict__ m,
                             int* __restrict__ next, int* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const int i = list[t];
  m[i] = INT_MAX;
  for (int k = srp[i]; k < srp[i + 1]; ++k) m[sci[k]] = INT_MAX;
  if (st[i] == kUndecided) next[atomicAdd(count, 1)] = i;
}

__global__ void k_root_flags(int n, const unsigned char* __restrict__ st, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = st[i] == kRoot ? 1 : 0;
}

// pass-1 aggregate of every node; pass-2 worklist (nodes no root took)
__global__ void k_pass1_agg(int n, const int* __restrict__ taken, const int* __restrict__ rid, int* __restrict__ agg,
                            int* __restrict__ code, int* __restrict__ list, int* __restrict__ count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int r = taken[i];
  agg[i] = r >= 0 ? rid[r] : -1;
  code[i] = 0;
  if (r < 0) list[atomicAdd(count, 1)] = i;
}

// pass 2 (amg.cpp:69-83). code[j] of a leftover j: 0 unresolved, 1 resolved
// without an aggregate, a + 2 attached to aggregate a. Earlier leftovers are
// visible to i only once resolved; later ones are not aggregated yet. Row i is
// decided as soon as no unresolved earlier leftover could be its first
// maximum (mu_k, mu below), so chains resolve in a few rounds.
__global__ void k_pass2(int nl, const int* __restrict__ list, const int* __restrict__ rp, const int* __restrict__ ci,
                        const double* __restrict__ v, const int* __restrict__ agg1, int* code, int* __restrict__ next,
                        int* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nl) return;
  const int i = list[t];
  int best = -1, best_k = INT_MAX;
  double best_w = -1.0;
  // unresolved earlier leftovers: the largest weight and its first position
  double mu = -1.0;
  int mu_k = INT_MAX;
  for (int k = rp[i]; k < rp[i + 1]; ++k) {
    const int j = ci[k];
    if (j == i) continue;
    int aj = agg1[j];
    if (aj < 0) {
      if (j > i) continue;
      const int c = ((volatile int*)code)[j];
      if (c == 0) {
        const double w = fabs(v[k]);
        if (w > mu) {
          mu = w;
          mu_k = k;
        }
        continue;
      }
      aj = c - 2;
      if (aj < 0) continue;
    }
    const double w = fabs(v[k]);
    if (w > best_w) {
      best_w = w;
      best = aj;
      best_k = k;
    }
  }
  // the row scan keeps the first maximum: an unresolved leftover changes the
  // outcome only if it could be that maximum; otherwise i is decided now
  if (mu > best_w || (mu == best_w && mu_k < best_k)) {
    next[atomicAdd(count, 1)] = i;
    return;
  }
  ((volatile int*)code)[i] = best >= 0 ? best + 2 : 1;
}

__global__ void k_pass2_merge(int n, int* __restrict__ agg, const int* __restrict__ code, int* __restrict__ flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int a = agg[i];
  if (a < 0 && code[i] >= 2) a = code[i] - 2;
  agg[i] = a;
  flag[i] = a < 0 ? 1 : 0;
}

__global__ void k_pass3(int n, int n_root, const int* __restrict__ rank, int* __restrict__ agg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && agg[i] < 0) agg[i] = n_root + rank[i];
}

__global__ void k_agg_size(int n, const int* __restrict__ agg, int* __restrict__ size) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(&size[agg[i]], 1);
}

__global__ void k_tentative(int n, const int* __restrict__ agg, const int* __restrict__ size, int* __restrict__ rp,
                            int* __restrict__ ci, double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  rp[i] = i;
  if (i == n) return;
  ci[i] = agg[i];
  v[i] = __ddiv_rn(1.0, __dsqrt_rn((double)size[agg[i]]));
}

// w_i = (sum_k a_ik v_k in row order) / d_i (amg.cpp:38-39, products and sums rounded separately)
__global__ void k_spmv_div(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ a,
                           const double* __restrict__ x, const double* __restrict__ d, double* __restrict__ w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = rp[i]; k < rp[i + 1]; ++k) s = __dadd_rn(s, __dmul_rn(a[k], x[ci[k]]));
  w[i] = __ddiv_rn(s, d[i]);
}

__global__ void k_div_scalar(int n, const double* __restrict__ w, double lambda, double* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = __ddiv_rn(w[i], lambda);
}

__global__ void k_row_of(int n, const int* __restrict__ rp, int* __restrict__ row) {
  const int i = blockIdx.x;
  for (int k = rp[i] + threadIdx.x; k < rp[i + 1]; k += blockDim.x) row[k] = i;
}

__global__ void k_iota(long long n, int* __restrict__ x) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    x[t] = (int)t;
}

__global__ void k_col_count(long long nnz, const int* __restrict__ ci, int* __restrict__ cnt) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
       t += (long long)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ci[t] + 1], 1);
}

__global__ void k_transpose_fill(long long nnz, const int* __restrict__ perm, const int* __restrict__ row,
                                 const double* __restrict__ v, int* __restrict__ tci, double* __restrict__ tv) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
       t += (long long)gridDim.x * blockDim.x) {
    const int k = perm[t];
    tci[t] = row[k];
    tv[t] = v[k];
  }
}

int bits_for_int(int v) {
  int b = 1;
  while (b < 31 && (1 << b) <= v) ++b;
  return b;
}

// exclusive scan of n ints into out (out may alias nothing); returns the total
int scan_total(const int* in, int* out, int n, cudaStream_t s) {
  if (n <= 0) return 0;
  size_t bytes = 0;
  ck(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s), "scan size");
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(1, bytes));
  ck(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, s), "scan");
  int last_in = 0, last_out = 0;
  ck(cudaMemcpyAsync(&last_in, in + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaMemcpyAsync(&last_out, out + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "scan sync");
  return last_in + last_out;
}

int read_int(const int* p, cudaStream_t s) {
  int h = 0;
  ck(cudaMemcpyAsync(&h, p, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  return h;
}

}  // namespace

void dev_diagonal(const DCsr& a, DevBuf<double>& d, cudaStream_t s) {
  d.alloc(std::max(1, a.rows));
  if (a.rows > 0) k_diag<<<blocks_for(a.rows), 256, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.v.p, d.p);
  ck(cudaGetLastError(), "diag");
}

void dev_check_diagonal(const DCsr& a, cudaStream_t s) {
  if (a.rows == 0) return;
  DevBuf<int> bad;
  bad.alloc(1);
  const int big = INT_MAX;
  bad.upload(&big, 1, s);
  k_check_diag<<<blocks_for(a.rows), 256, 0, s>>>(a.rows, a.rp.p, a.ci.p, a.v.p, bad.p);
  ck(cudaGetLastError(), "check diag");
  const int row = read_int(bad.p, s);
  if (row != INT_MAX)
    throw NumericalError("matrix has a missing or zero diagonal entry at row " + std::to_string(row));
}

int dev_aggregate(const DCsr& a, const double* d, double theta, DevBuf<int>& agg, cudaStream_t s,
                  DevAggStats* stats) {
  const int n = a.rows;
  agg.alloc(std::max(1, n));
  if (n == 0) return 0;
  const int nb = blocks_for(n);
  // strength graph S as CSR (strong columns in row order)
  DevBuf<int> srp, cnt, sci;
  cnt.alloc(n);
  srp.alloc(n + 1);
  k_strong_count<<<nb, 256, 0, s>>>(n, a.rp.p, a.ci.p, a.v.p, d, theta, cnt.p);
  ck(cudaGetLastError(), "strength");
  const int snnz = scan_total(cnt.p, srp.p, n, s);
  ck(cudaMemcpyAsync(srp.p + n, &snnz, sizeof(int), cudaMemcpyHostToDevice, s), "h2d");
  sci.alloc(std::max(1, snnz));
  k_strong_fill<<<nb, 256, 0, s>>>(n, a.rp.p, a.ci.p, a.v.p, d, theta, srp.p, sci.p);
  ck(cudaGetLastError(), "strength fill");
  // pass 1
  DevBuf<unsigned char> st;
  DevBuf<int> taken, m, la, lb, counter;
  st.alloc(n);
  taken.alloc(n);
  m.alloc(n);
  la.alloc(n);
  lb.alloc(n);
  counter.alloc(2);
  ck(cudaMemsetAsync(counter.p, 0, 2 * sizeof(int), s), "memset");
  k_pass1_init<<<nb, 256, 0, s>>>(n, srp.p, st.p, taken.p, m.p, la.p, counter.p);
  int nl = read_int(counter.p, s);
  int rounds1 = 0;
  while (nl > 0) {
    ++rounds1;
    const int lb_ = blocks_for(nl);
    k_pass1_bid<<<lb_, 256, 0, s>>>(nl, la.p, srp.p, sci.p, st.p, taken.p, m.p);
    k_pass1_claim<<<lb_, 256, 0, s>>>(nl, la.p, srp.p, sci.p, st.p, taken.p, m.p);
    ck(cudaMemsetAsync(counter.p, 0, sizeof(int), s), "memset");
    k_pass1_next<<<lb_, 256, 0, s>>>(nl, la.p, srp.p, sci.p, st.p, m.p, lb.p, counter.p);
    ck(cudaGetLastError(), "pass 1");
    std::swap(la, lb);
    nl = read_int(counter.p, s);
  }
  // roots numbered in index order
  DevBuf<int>& flag = cnt;
  DevBuf<int>& rid = m;
  k_root_flags<<<nb, 256, 0, s>>>(n, st.p, flag.p);
  const int n_root = scan_total(flag.p, rid.p, n, s);
  // pass 2
  DevBuf<int>& code = srp;  // strength graph no longer needed
  ck(cudaMemsetAsync(counter.p, 0, sizeof(int), s), "memset");
  k_pass1_agg<<<nb, 256, 0, s>>>(n, taken.p, rid.p, agg.p, code.p, la.p, counter.p);
  nl = read_int(counter.p, s);
  const int n_left = nl;
  int rounds2 = 0;
  while (nl > 0) {
    ++rounds2;
    ck(cudaMemsetAsync(counter.p, 0, sizeof(int), s), "memset");
    k_pass2<<<blocks_for(nl), 256, 0, s>>>(nl, la.p, a.rp.p, a.ci.p, a.v.p, agg.p, code.p, lb.p, counter.p);
    ck(cudaGetLastError(), "pass 2");
    std::swap(la, lb);
    nl = read_int(counter.p, s);
  }
  // pass 3
  k_pass2_merge<<<nb, 256, 0, s>>>(n, agg.p, code.p, flag.p);
  const int n_new = scan_total(flag.p, rid.p, n, s);
  k_pass3<<<nb, 256, 0, s>>>(n, n_root, rid.p, agg.p);
  ck(cudaGetLastError(), "pass 3");
  if (stats) *stats = {rounds1, rounds2, n_root, n_left - n_new, n_new};
  return n_root + n_new;
}

void dev_tentative(const DevBuf<int>& agg, int n, int n_agg, DCsr& pt, cudaStream_t s) {
  pt.rows = n;
  pt.cols = n_agg;
  pt.nnz = n;
  pt.rp.alloc(n + 1);
  pt.ci.alloc(std::max(1, n));
  pt.v.alloc(std::max(1, n));
  DevBuf<int> size;
  size.alloc(std::max(1, n_agg));
  ck(cudaMemsetAsync(size.p, 0, sizeof(int) * std::max(1, n_agg), s), "memset");
  if (n > 0) k_agg_size<<<blocks_for(n), 256, 0, s>>>(n, agg.p, size.p);
  k_tentative<<<blocks_for(n + 1), 256, 0, s>>>(n, agg.p, size.p, pt.rp.p, pt.ci.p, pt.v.p);
  ck(cudaGetLastError(), "tentative");
  ck(cudaStreamSynchronize(s), "tentative sync");
}

double dev_lambda_max(const DCsr& a, const double* d, int iters, unsigned seed, cudaStream_t s) {
  const int n = a.rows;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<double> h(n);
  for (int i = 0; i < n; ++i) h[i] = uni(rng);
  const double nv = seq_norm(h);
  for (double& e : h) e /= nv;
  DevBuf<double> v, w;
  v.alloc(std::max(1, n));
  w.alloc(std::max(1, n));
  v.upload(h.data(), n, s);
  double lambda = 1.0;
  for (int it = 0; it < iters; ++it) {
    k_spmv_div<<<blocks_for(n), 256, 0, s>>>(n, a.rp.p, a.ci.p, a.v.p, v.p, d, w.p);
    ck(cudaGetLastError(), "lambda spmv");
    w.download(h.data(), n, s);
    ck(cudaStreamSynchronize(s), "lambda sync");
    lambda = seq_norm(h);
    if (lambda == 0.0) return 1.0;
    k_div_scalar<<<blocks_for(n), 256, 0, s>>>(n, w.p, lambda, v.p);
  }
  ck(cudaStreamSynchronize(s), "lambda");
  return lambda;
}

void dev_transpose(const DCsr& a, DCsr& t, cudaStream_t s) {
  const long long nnz = a.nnz;
  t.rows = a.cols;
  t.cols = a.rows;
  t.nnz = nnz;
  t.rp.alloc(t.rows + 1);
  ck(cudaMemsetAsync(t.rp.p, 0, sizeof(int) * (t.rows + 1), s), "memset");
  t.ci.alloc(std::max<long long>(1, nnz));
  t.v.alloc(std::max<long long>(1, nnz));
  if (nnz == 0) return;
  if (nnz >= (1ll << 31)) throw CudaError("transpose: more than 2^31 entries");
  const int grid = (int)std::min<long long>((nnz + 255) / 256, 148 * 16);
  DevBuf<int> row, keys_out, idx_in, idx_out;
  row.alloc(nnz);
  if (a.rows > 0) k_row_of<<<a.rows, 32, 0, s>>>(a.rows, a.rp.p, row.p);
  idx_in.alloc(nnz);
  idx_out.alloc(nnz);
  keys_out.alloc(nnz);
  k_iota<<<grid, 256, 0, s>>>(nnz, idx_in.p);
  // stable sort of the entry indices by column: each column keeps ascending rows
  size_t bytes = 0;
  const int end_bit = bits_for_int(std::max(1, a.cols - 1));
  ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, a.ci.p, keys_out.p, idx_in.p, idx_out.p, (int)nnz, 0, end_bit, s),
     "sort size");
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(1, bytes));
  ck(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, a.ci.p, keys_out.p, idx_in.p, idx_out.p, (int)nnz, 0, end_bit, s),
     "sort");
  k_transpose_fill<<<grid, 256, 0, s>>>(nnz, idx_out.p, row.p, a.v.p, t.ci.p, t.v.p);
  k_col_count<<<grid, 256, 0, s>>>(nnz, a.ci.p, t.rp.p);
  size_t sb = 0;
  ck(cub::DeviceScan::InclusiveSum(nullptr, sb, t.rp.p, t.rp.p, t.rows + 1, s), "scan size");
  tmp.alloc(std::max<size_t>(1, sb));
  ck(cub::DeviceScan::InclusiveSum(tmp.p, sb, t.rp.p, t.rp.p, t.rows + 1, s), "scan");
  ck(cudaGetLastError(), "transpose");
  ck(cudaStreamSynchronize(s), "transpose sync");
}

}  // namespace eqsb
