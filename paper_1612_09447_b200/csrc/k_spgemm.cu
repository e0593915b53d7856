// Device Galerkin products for the SA-AMG setup:
// C = A B with the reference's per-row arithmetic (proj/src/csr.cpp:133-166),
// bit-identical to the host Gustavson product.
//
// The host accumulates row i as accum[j] += a_ik * b_kj in encounter order
// (ka ascending, then kb ascending), starting from 0.0, products and sums
// rounded separately (-ffp-contract=off). The device reproduces exactly that
// order with expand-sort-compress:
//   1. expand: one warp per row writes every product (key = local row << jbits
//      | j, value = __dmul_rn(a, b)) at its encounter position;
//   2. a stable LSD radix sort on the key (cub::DeviceRadixSort) groups equal
//      (row, j) while keeping encounter order inside each group, and orders
//      the columns of each row ascending, as the host's std::sort does;
//   3. compress: the first entry of every group sums its group sequentially
//      with __dadd_rn from 0.0.
// Rows are processed in batches that bound the product buffers. Optionally A
// is replaced on the fly by the damped-Jacobi smoother I - omega D^-1 A with
// the host's expression order ((-omega * a) / d, then + 1 on the diagonal;
// amg.cpp:121-126), so P = (I - omega D^-1 A) P_tent needs no host copy of A.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "amg_device.hpp"

namespace eqsb {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("spgemm: ") + what + ": " + cudaGetErrorString(e));
}

__global__ void k_spgemm_count(int m, const int* __restrict__ arp, const int* __restrict__ aci,
                               const int* __restrict__ brp, long long* __restrict__ cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  long long s = 0;
  for (int ka = arp[i]; ka < arp[i + 1]; ++ka) {
    const int k = aci[ka];
    s += brp[k + 1] - brp[k];
  }
  cnt[i] = s;
}

// wpr warps per row of A (rows with many products, e.g. the dense coarse
// Galerkin products, would otherwise leave most SMs idle): warp w of a row
// takes the w-th contiguous share of its A entries and starts writing after
// the products of the entries before it (same positions as one warp).
template <bool SCALED>
__global__ void k_spgemm_expand(int r0, int r1, long long base, const long long* __restrict__ off,
                                const int* __restrict__ arp, const int* __restrict__ aci,
                                const double* __restrict__ av, const int* __restrict__ brp,
                                const int* __restrict__ bci, const double* __restrict__ bv,
                                const double* __restrict__ diag, double neg_omega, int jbits,
                                unsigned long long* __restrict__ keys, double* __restrict__ vals, int wpr) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int i = r0 + gw / wpr, w = gw % wpr;
  if (i >= r1) return;
  const int a0 = arp[i], a1 = arp[i + 1], share = (a1 - a0 + wpr - 1) / wpr;
  const int kb = min(a1, a0 + w * share), ke = min(a1, kb + share);
  long long pre = 0;  // products of the row's A entries before this warp's share
  for (int ka = a0 + lane; ka < kb; ka += 32) pre += brp[aci[ka] + 1] - brp[aci[ka]];
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  long long pos = off[i] - base + pre;
  const unsigned long long rowkey = (unsigned long long)(i - r0) << jbits;
  for (int ka = kb; ka < ke; ++ka) {
    const int k = aci[ka];
    double a = av[ka];
    if (SCALED) {
      a = __ddiv_rn(__dmul_rn(neg_omega, a), diag[i]);
      if (k == i) a = __dadd_rn(a, 1.0);
    }
    const int b0 = brp[k], len = brp[k + 1] - b0;
    for (int t = lane; t < len; t += 32) {
      keys[pos + t] = rowkey | (unsigned)bci[b0 + t];
      vals[pos + t] = __dmul_rn(a, bv[b0 + t]);
    }
    pos += len;
  }
}

__global__ void k_spgemm_heads(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ head) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    head[t] = (t == 0 || keys[t] != keys[t - 1]) ? 1 : 0;
}

__global__ void k_spgemm_reduce(long long n, const unsigned long long* __restrict__ keys,
                                const double* __restrict__ vals, const int* __restrict__ head,
                                const int* __restrict__ idx, int jbits, int* __restrict__ out_col,
                                double* __restrict__ out_val, int* __restrict__ row_cnt) {
  const unsigned long long jmask = (1ull << jbits) - 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // warp-uniform trip count (the per-row output counts are aggregated per warp)
  for (long long t0 = (long long)blockIdx.x * blockDim.x; t0 < n; t0 += stride) {
    const long long t = t0 + threadIdx.x;
    const bool h = t < n && head[t];
    unsigned row = 0;
    if (h) {
      const unsigned long long key = keys[t];
      double s = 0.0;
      for (long long u = t; u < n && keys[u] == key; ++u) s = __dadd_rn(s, vals[u]);
      out_col[idx[t]] = (int)(key & jmask);
      out_val[idx[t]] = s;
      row = (unsigned)(key >> jbits);
    }
    // one atomic per row and warp (dense coarse rows have thousands of
    // outputs: one atomic per output serialised on the row's counter)
    const unsigned act = __ballot_sync(0xffffffffu, h);
    if (h) {
      const unsigned peers = __match_any_sync(act, row);
      if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&row_cnt[row], __popc(peers));  // batch-relative row
    }
  }
}

int bits_for(long long v) {  // bits to represent 0..v
  int b = 1;
  while (b < 62 && (1ll << b) <= v) ++b;
  return b;
}

}  // namespace

template <class T>
void up(DevBuf<T>& d, const std::vector<T>& h, cudaStream_t s) {
  d.alloc(std::max<size_t>(1, h.size()));
  if (!h.empty()) d.upload(h.data(), h.size(), s);
}
template void up(DevBuf<double>&, const std::vector<double>&, cudaStream_t);

// ---------------------------------------------------------------- device CSR products (amg_device.hpp)
void SpgemmDevice::init(int device) {
  device_ = device;
  ck(cudaSetDevice(device), "set device");
  ck(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking), "stream");
}
SpgemmDevice::~SpgemmDevice() {
  if (s_) cudaStreamDestroy(s_);
}

void SpgemmDevice::upload(const HostCsr& h, DCsr& d) {
  d.rows = h.n_rows;
  d.cols = h.n_cols;
  d.nnz = h.nnz();
  up(d.rp, h.row_ptr, s_);
  up(d.ci, h.col_idx, s_);
  up(d.v, h.values, s_);
}

void SpgemmDevice::download(const DCsr& d, HostCsr& h) {
  h.n_rows = d.rows;
  h.n_cols = d.cols;
  h.row_ptr.resize(d.rows + 1);
  h.col_idx.resize(d.nnz);
  h.values.resize(d.nnz);
  d.rp.download(h.row_ptr.data(), d.rows + 1, s_);
  d.ci.download(h.col_idx.data(), d.nnz, s_);
  d.v.download(h.values.data(), d.nnz, s_);
  ck(cudaStreamSynchronize(s_), "download");
}

void SpgemmDevice::multiply(const DCsr& a, const DCsr& b, DCsr& c, const double* diag_dev, double omega,
                            long long batch_products) {
  if (a.cols != b.rows) throw NumericalError("csr multiply: dimension mismatch");
  cudaStream_t s = s_;
  const int m = a.rows;
  static const bool trace = getenv("EQS_SPGEMM_TRACE") != nullptr;
  auto T0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what, long long v) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[spgemm] %dx%d * %dx%d %-10s %.3f s (%lld)\n", a.rows, a.cols, b.rows, b.cols, what,
            std::chrono::duration<double>(now - T0).count(), v);
    T0 = now;
  };
  c.rows = m;
  c.cols = b.cols;
  // per-row product counts -> offsets
  DevBuf<long> cnt, off;
  cnt.alloc(std::max(1, m));
  off.alloc(m + 1);
  if (m > 0) k_spgemm_count<<<(m + 255) / 256, 256, 0, s>>>(m, a.rp.p, a.ci.p, b.rp.p, (long long*)cnt.p);
  ck(cudaMemsetAsync(off.p, 0, sizeof(long), s), "memset");
  size_t tmp_bytes = 0;
  ck(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, (long long*)cnt.p, (long long*)off.p + 1, m, s), "scan size");
  DevBuf<unsigned char> tmp;
  tmp.alloc(std::max<size_t>(1, tmp_bytes));
  if (m > 0) ck(cub::DeviceScan::InclusiveSum(tmp.p, tmp_bytes, (long long*)cnt.p, (long long*)off.p + 1, m, s), "scan");
  std::vector<long> hoff(m + 1);
  off.download(hoff.data(), m + 1, s);
  ck(cudaStreamSynchronize(s), "offsets");
  const int jbits = bits_for(std::max(1, b.cols - 1));
  const int kMaxBatchRows = 1 << 22;
  long long max_batch = 0;
  std::vector<std::pair<int, int>> batches;
  for (int r0 = 0; r0 < m;) {
    int r1 = r0 + 1;
    while (r1 < m && r1 - r0 < kMaxBatchRows && hoff[r1 + 1] - hoff[r0] <= batch_products) ++r1;
    batches.push_back({r0, r1});
    max_batch = std::max<long long>(max_batch, hoff[r1] - hoff[r0]);
    r0 = r1;
  }
  lap("offsets", hoff[m]);
  if (max_batch >= (1ll << 31)) throw CudaError("spgemm: a single row has more than 2^31 products");
  const size_t cap = std::max<long long>(1, max_batch);
  DevBuf<unsigned long long> k_in, k_out;
  DevBuf<double> v_in, v_out;
  DevBuf<int> head, idx, rcnt;
  k_in.alloc(cap);
  k_out.alloc(cap);
  v_in.alloc(cap);
  v_out.alloc(cap);
  head.alloc(cap);
  idx.alloc(cap);
  rcnt.alloc(m + 1);
  ck(cudaMemsetAsync(rcnt.p, 0, sizeof(int) * (m + 1), s), "memset");
  size_t sort_bytes = 0, scan_bytes = 0;
  ck(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, k_in.p, k_out.p, v_in.p, v_out.p, (int)cap, 0, 64, s),
     "sort size");
  ck(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head.p, idx.p, (int)cap, s), "scan size");
  tmp.alloc(std::max<size_t>({1, sort_bytes, scan_bytes}));
  lap("alloc", (long long)batches.size());
  // batch outputs (compressed entries in row-major, column-sorted order)
  std::vector<DevBuf<int>> out_c;
  std::vector<DevBuf<double>> out_v;
  std::vector<long long> out_n;
  long long total = 0;
  for (auto [r0, r1] : batches) {
    const long long base = hoff[r0], n = hoff[r1] - base;
    const int nr = r1 - r0;
    if (n == 0) continue;
    const int warps_per_block = 8;
    // enough warps to fill the GPU when the batch has few (heavy) rows
    int wpr = 1;
    while (wpr < 32 && (long long)nr * wpr < 148L * 48) wpr <<= 1;
    const long long warps = (long long)nr * wpr;
    const int blocks = (int)((warps + warps_per_block - 1) / warps_per_block);
    if (diag_dev)
      k_spgemm_expand<true><<<blocks, 32 * warps_per_block, 0, s>>>(r0, r1, base, (const long long*)off.p, a.rp.p,
                                                                    a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p, diag_dev,
                                                                    -omega, jbits, k_in.p, v_in.p, wpr);
    else
      k_spgemm_expand<false><<<blocks, 32 * warps_per_block, 0, s>>>(r0, r1, base, (const long long*)off.p, a.rp.p,
                                                                     a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p, nullptr,
                                                                     0.0, jbits, k_in.p, v_in.p, wpr);
    ck(cudaGetLastError(), "expand");
    lap("expand", n);
    const int end_bit = jbits + bits_for(std::max(1, nr - 1));
    size_t tb = tmp.n;
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k_in.p, k_out.p, v_in.p, v_out.p, (int)n, 0, end_bit, s), "sort");
    lap("sort", end_bit);
    const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 16);
    k_spgemm_heads<<<grid, 256, 0, s>>>(n, k_out.p, head.p);
    tb = tmp.n;
    ck(cub::DeviceScan::ExclusiveSum(tmp.p, tb, head.p, idx.p, (int)n, s), "scan");
    int last_idx = 0, last_head = 0;
    ck(cudaMemcpyAsync(&last_idx, idx.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaMemcpyAsync(&last_head, head.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    ck(cudaStreamSynchronize(s), "batch");
    const long long nu = (long long)last_idx + last_head;
    out_c.emplace_back();
    out_v.emplace_back();
    out_c.back().alloc(nu);
    out_v.back().alloc(nu);
    k_spgemm_reduce<<<grid, 256, 0, s>>>(n, k_out.p, v_out.p, head.p, idx.p, jbits, out_c.back().p, out_v.back().p,
                                         rcnt.p + 1 + r0);
    ck(cudaGetLastError(), "reduce");
    lap("reduce", nu);
    out_n.push_back(nu);
    total += nu;
  }
  if (total >= (1ll << 31)) throw CudaError("spgemm: product has more than 2^31 entries");
  // free the batch work space before the result is assembled
  k_in.alloc(0);
  k_out.alloc(0);
  v_in.alloc(0);
  v_out.alloc(0);
  head.alloc(0);
  idx.alloc(0);
  c.nnz = total;
  c.ci.alloc(std::max<long long>(1, total));
  c.v.alloc(std::max<long long>(1, total));
  long long at = 0;
  for (size_t q = 0; q < out_n.size(); ++q) {
    if (out_n[q] == 0) continue;
    ck(cudaMemcpyAsync(c.ci.p + at, out_c[q].p, sizeof(int) * out_n[q], cudaMemcpyDeviceToDevice, s), "d2d");
    ck(cudaMemcpyAsync(c.v.p + at, out_v[q].p, sizeof(double) * out_n[q], cudaMemcpyDeviceToDevice, s), "d2d");
    at += out_n[q];
  }
  // row_ptr = inclusive scan of the per-row counts (rcnt[0] = 0)
  c.rp.alloc(m + 1);
  size_t sb = 0;
  ck(cub::DeviceScan::InclusiveSum(nullptr, sb, rcnt.p, c.rp.p, m + 1, s), "scan size");
  tmp.alloc(std::max<size_t>(1, sb));
  ck(cub::DeviceScan::InclusiveSum(tmp.p, sb, rcnt.p, c.rp.p, m + 1, s), "row_ptr");
  ck(cudaStreamSynchronize(s), "assemble");
}

struct AmgDeviceBuilder::Impl {
  SpgemmDevice sd;
  DCsr fine, p;
  bool has_fine = false;
};
AmgDeviceBuilder::AmgDeviceBuilder(int device) : impl_(std::make_unique<Impl>()) { impl_->sd.init(device); }
AmgDeviceBuilder::~AmgDeviceBuilder() = default;

HostCsr AmgDeviceBuilder::prolongator(const HostCsr& fine, const HostCsr& p_tent, const std::vector<double>& d,
                                      double omega, long long batch) {
  Impl& m = *impl_;
  if (!m.has_fine) m.sd.upload(fine, m.fine);  // level 0; coarser levels are the previous R A P
  m.has_fine = true;
  DCsr pt;
  m.sd.upload(p_tent, pt);
  DevBuf<double> dg;
  up(dg, d, m.sd.stream());
  m.sd.multiply(m.fine, pt, m.p, dg.p, omega, batch);
  HostCsr p;
  m.sd.download(m.p, p);
  return p;
}

HostCsr AmgDeviceBuilder::galerkin(const HostCsr& r, long long batch) {
  Impl& m = *impl_;
  DCsr ap, dr, coarse;
  m.sd.multiply(m.fine, m.p, ap, nullptr, 0.0, batch);
  m.p = DCsr();
  m.sd.upload(r, dr);
  m.sd.multiply(dr, ap, coarse, nullptr, 0.0, batch);
  HostCsr c;
  m.sd.download(coarse, c);
  m.fine = std::move(coarse);  // next level's fine operator stays resident
  return c;
}

bool AmgDeviceBuilder::next_level(const HostCsr& fine, const SolverParams& sp, long long batch, AmgHostLevel& lv,
                                  HostCsr& coarse_out) {
  Impl& m = *impl_;
  cudaStream_t s = m.sd.stream();
  static const bool trace = getenv("EQS_MEMTRACE") != nullptr;
  auto T0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[amg]   %-10s %.3f s\n", what, std::chrono::duration<double>(now - T0).count());
    T0 = now;
  };
  if (!m.has_fine) m.sd.upload(fine, m.fine);
  m.has_fine = true;
  const int n = m.fine.rows;
  DevBuf<double> d;
  dev_diagonal(m.fine, d, s);
  DevBuf<int> agg;
  DevAggStats st;
  lap("upload");
  const int n_agg = dev_aggregate(m.fine, d.p, sp.amg_theta, agg, s, &st);
  lap("aggregate");
  if (getenv("EQS_MEMTRACE"))
    fprintf(stderr, "[amg] device aggregation: %d rows -> %d aggregates (%d roots in %d rounds, %d attached in %d rounds, %d new)\n",
            n, n_agg, st.roots, st.rounds_pass1, st.pass2, st.rounds_pass2, st.pass3);
  if (n_agg >= n) return false;  // coarsening stalled (amg.cpp:102)
  lv.aggregates.resize(n);
  agg.download(lv.aggregates.data(), n, s);
  DCsr pt;
  dev_tentative(agg, n, n_agg, pt, s);
  lap("p_tent");
  lv.lambda_max_scaled = dev_lambda_max(m.fine, d.p, 10, 20240811u, s);
  lap("lambda");
  const double omega = sp.amg_omega / lv.lambda_max_scaled;
  m.sd.multiply(m.fine, pt, m.p, d.p, omega, batch);  // P = (I - omega D^-1 A) P_tent
  pt = DCsr();
  lap("P");
  DCsr r, ap, coarse;
  dev_transpose(m.p, r, s);
  lap("R");
  m.sd.multiply(m.fine, m.p, ap, nullptr, 0.0, batch);
  lap("AP");
  m.sd.multiply(r, ap, coarse, nullptr, 0.0, batch);
  ap = DCsr();
  dev_check_diagonal(coarse, s);
  lap("RAP");
  m.sd.download(m.p, lv.P);
  m.sd.download(r, lv.R);
  m.sd.download(coarse, coarse_out);
  lap("download");
  m.p = DCsr();
  m.fine = std::move(coarse);
  return true;
}

HostCsr spgemm_device(const HostCsr& a, const HostCsr& b, int device, const std::vector<double>* diag,
                      double omega, long long batch_products) {
  SpgemmDevice sd;
  sd.init(device);
  DCsr da, db, dc;
  sd.upload(a, da);
  sd.upload(b, db);
  DevBuf<double> dg;
  if (diag) up(dg, *diag, sd.stream());
  sd.multiply(da, db, dc, diag ? dg.p : nullptr, omega, batch_products);
  HostCsr c;
  sd.download(dc, c);
  return c;
}

// Galerkin chain A_{k+1} = R_k (A_k P_k) with every operand and the running
// coarse operator resident on the device; only the coarse operators return
std::vector<HostCsr> galerkin_chain_device(const HostCsr& fine, const std::vector<const HostCsr*>& p,
                                           const std::vector<const HostCsr*>& r, int device) {
  SpgemmDevice sd;
  sd.init(device);
  DCsr a;
  sd.upload(fine, a);
  std::vector<HostCsr> out;
  for (size_t k = 0; k < p.size(); ++k) {
    DCsr dp, dr, ap, c;
    sd.upload(*p[k], dp);
    sd.multiply(a, dp, ap, nullptr, 0.0, 1ll << 28);
    dp = DCsr();
    sd.upload(*r[k], dr);
    sd.multiply(dr, ap, c, nullptr, 0.0, 1ll << 28);
    HostCsr hc;
    sd.download(c, hc);
    out.push_back(std::move(hc));
    a = std::move(c);
  }
  return out;
}

}  // namespace eqsb
