// Device element colouring and fine-dof partition,
// bit-identical to the sequential host/reference algorithms.
//
// Colouring (proj/src/matfree.cpp:11-38): tet t takes the smallest colour not
// used by any earlier tet sharing a dof. The colour of t depends only on the
// colours of its earlier neighbours, so the device walks the "earlier
// neighbour" DAG in topological waves (Kahn): cnt[t] = number of earlier
// neighbours (counted once per shared dof); a wave colours its tets from their
// neighbours' final colours, then decrements the counters of the later
// neighbours, and a tet whose counter reaches zero joins the next wave. Each
// incidence is visited twice in total, and the number of waves is the depth of
// the DAG (O(nx + ny + nz) cells on the box meshes).
//
// Partition (host_partition.cpp partition_free_dofs): a stable radix sort of
// the free dofs by their coordinate along the longest axis, then contiguous
// equal chunks.
#include <cub/cub.cuh>

#include <string>

#include "amg_device.hpp"

namespace eqsb {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string("device setup: ") + what + ": " + cudaGetErrorString(e));
}

inline int blocks_for(long long n, int bs = 256) { return (int)std::max<long long>(1, (n + bs - 1) / bs); }
inline int grid_for(long long n) { return (int)std::min<long long>(std::max<long long>(1, (n + 255) / 256), 148 * 16); }

__global__ void k_iota_l(long long n, int* __restrict__ x) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    x[t] = (int)t;
}

__global__ void k_dof_count(long long ne, const int* __restrict__ ed, int* __restrict__ cnt) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ne; t += (long long)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ed[t] + 1], 1);
}

// incidence entry p of dof d: tet = e / nl (ascending inside a dof after the
// stable sort); its rank inside the dof's list = number of earlier tets there
__global__ void k_incidence(long long ne, int nl, const int* __restrict__ dof_sorted, const int* __restrict__ e_sorted,
                            const int* __restrict__ ptr, int* __restrict__ tet, int* __restrict__ cnt) {
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < ne;
       p += (long long)gridDim.x * blockDim.x) {
    const int t = e_sorted[p] / nl;
    tet[p] = t;
    atomicAdd(&cnt[t], (int)(p - ptr[dof_sorted[p]]));
  }
}

__global__ void k_wave0(int n_tets, const int* __restrict__ cnt, int* __restrict__ color, int* __restrict__ list,
                        int* __restrict__ count) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tets) return;
  color[t] = -1;
  if (cnt[t] == 0) list[atomicAdd(count, 1)] = t;
}

constexpr int kMaskWords = 8;  // up to 512 colours (P1 Kuhn boxes use ~30)

__global__ void k_color_wave(int nw, const int* __restrict__ list, int nl, const int* __restrict__ ed,
                             const int* __restrict__ ptr, const int* __restrict__ tet, int* __restrict__ color,
                             int* __restrict__ cnt, int* __restrict__ next, int* __restrict__ count,
                             int* __restrict__ overflow) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  const int t = list[w];
  unsigned long long used[kMaskWords];
#pragma unroll
  for (int q = 0; q < kMaskWords; ++q) used[q] = 0ull;
  // earlier neighbours: the prefix of each dof's ascending list
  for (int i = 0; i < nl; ++i) {
    const int d = ed[(long long)nl * t + i];
    for (int p = ptr[d]; p < ptr[d + 1]; ++p) {
      const int u = tet[p];
      if (u >= t) break;
      const int c = color[u];
      if (c >= kMaskWords * 64) {
        atomicExch(overflow, 1);
        continue;
      }
#pragma unroll
      for (int q = 0; q < kMaskWords; ++q)
        if ((c >> 6) == q) used[q] |= 1ull << (c & 63);
    }
  }
  int c = kMaskWords * 64;
#pragma unroll
  for (int q = kMaskWords - 1; q >= 0; --q)
    if (~used[q]) c = q * 64 + __ffsll((long long)~used[q]) - 1;
  if (c >= kMaskWords * 64) atomicExch(overflow, 1);
  color[t] = c;
  __threadfence();
  // later neighbours: the suffix of each list
  for (int i = 0; i < nl; ++i) {
    const int d = ed[(long long)nl * t + i];
    for (int p = ptr[d + 1] - 1; p >= ptr[d]; --p) {
      const int u = tet[p];
      if (u <= t) break;
      if (atomicSub(&cnt[u], 1) == 1) next[atomicAdd(count, 1)] = u;
    }
  }
}

__global__ void k_max_color(int n, const int* __restrict__ color, int* __restrict__ mx) {
  int m = -1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) m = max(m, color[t]);
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 16));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 8));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 4));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
  m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

__global__ void k_owner(int nf, int nranks, const int* __restrict__ order, int* __restrict__ owner) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nf) owner[order[k]] = (int)((long long)k * nranks / max(1, nf));
}

int read_int(const int* p, cudaStream_t s) {
  int h = 0;
  ck(cudaMemcpyAsync(&h, p, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  ck(cudaStreamSynchronize(s), "sync");
  return h;
}

}  // namespace

std::vector<int> dev_color_elements(const Dofs& dm, int n_tets, int* n_colors_out, int device, int* waves_out) {
  ck(cudaSetDevice(device), "set device");
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  const int nl = dm.n_local;
  const long long ne = (long long)n_tets * nl;
  std::vector<int> color(n_tets, -1);
  int n_colors = 0, waves = 0;
  if (n_tets > 0) {
    if (ne >= (1ll << 31)) throw CudaError("colouring: more than 2^31 element dofs");
    DevBuf<int> ed, ptr, e_in, e_out, d_out, tet, cnt, col, la, lb, counter;
    ed.alloc(ne);
    ed.upload(dm.element_dofs.data(), ne, s);
    // dof -> incident tets (ascending): stable sort of the element-dof slots by dof
    ptr.alloc(dm.n_dofs + 1);
    ck(cudaMemsetAsync(ptr.p, 0, sizeof(int) * (dm.n_dofs + 1), s), "memset");
    k_dof_count<<<grid_for(ne), 256, 0, s>>>(ne, ed.p, ptr.p);
    size_t bytes = 0, sb = 0;
    ck(cub::DeviceScan::InclusiveSum(nullptr, sb, ptr.p, ptr.p, dm.n_dofs + 1, s), "scan size");
    e_in.alloc(ne);
    e_out.alloc(ne);
    d_out.alloc(ne);
    int end_bit = 1;
    while (end_bit < 31 && (1 << end_bit) <= std::max(1, dm.n_dofs - 1)) ++end_bit;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ed.p, d_out.p, e_in.p, e_out.p, (int)ne, 0, end_bit, s),
       "sort size");
    DevBuf<unsigned char> tmp;
    tmp.alloc(std::max<size_t>({1, bytes, sb}));
    ck(cub::DeviceScan::InclusiveSum(tmp.p, sb, ptr.p, ptr.p, dm.n_dofs + 1, s), "scan");
    k_iota_l<<<grid_for(ne), 256, 0, s>>>(ne, e_in.p);
    bytes = tmp.n;
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, ed.p, d_out.p, e_in.p, e_out.p, (int)ne, 0, end_bit, s), "sort");
    e_in.alloc(0);
    tet.alloc(ne);
    cnt.alloc(n_tets);
    ck(cudaMemsetAsync(cnt.p, 0, sizeof(int) * n_tets, s), "memset");
    k_incidence<<<grid_for(ne), 256, 0, s>>>(ne, nl, d_out.p, e_out.p, ptr.p, tet.p, cnt.p);
    ck(cudaGetLastError(), "incidence");
    d_out.alloc(0);
    e_out.alloc(0);
    col.alloc(n_tets);
    la.alloc(n_tets);
    lb.alloc(n_tets);
    counter.alloc(2);
    ck(cudaMemsetAsync(counter.p, 0, 2 * sizeof(int), s), "memset");
    k_wave0<<<blocks_for(n_tets), 256, 0, s>>>(n_tets, cnt.p, col.p, la.p, counter.p);
    int nw = read_int(counter.p, s);
    int done = 0;
    while (nw > 0) {
      ++waves;
      done += nw;
      ck(cudaMemsetAsync(counter.p, 0, sizeof(int), s), "memset");
      k_color_wave<<<blocks_for(nw, 128), 128, 0, s>>>(nw, la.p, nl, ed.p, ptr.p, tet.p, col.p, cnt.p, lb.p,
                                                        counter.p, counter.p + 1);
      ck(cudaGetLastError(), "colour wave");
      std::swap(la, lb);
      nw = read_int(counter.p, s);
    }
    if (read_int(counter.p + 1, s)) throw CudaError("colouring: more than 512 colours");
    if (done != n_tets) throw std::logic_error("colouring: waves did not reach every tet");
    k_max_color<<<148, 256, 0, s>>>(n_tets, col.p, counter.p);
    n_colors = read_int(counter.p, s) + 1;
    col.download(color.data(), n_tets, s);
    ck(cudaStreamSynchronize(s), "colour download");
  }
  cudaStreamDestroy(s);
  if (n_colors_out) *n_colors_out = n_colors;
  if (waves_out) *waves_out = waves;
  return color;
}

// owner[k] of free dof k from its coordinate along `axis` (stable by free index)
std::vector<int> dev_partition_owner(const std::vector<double>& key, int nranks, int device) {
  const int nf = (int)key.size();
  std::vector<int> owner(nf, 0);
  if (nranks == 1 || nf == 0) return owner;
  ck(cudaSetDevice(device), "set device");
  cudaStream_t s;
  ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  {
    std::vector<double> k2(key);
    for (double& v : k2) v += 0.0;  // -0.0 == +0.0 for std::stable_sort's operator<
    DevBuf<double> kin, kout;
    DevBuf<int> iin, iout, own;
    kin.alloc(nf);
    kout.alloc(nf);
    iin.alloc(nf);
    iout.alloc(nf);
    own.alloc(nf);
    kin.upload(k2.data(), nf, s);
    k_iota_l<<<grid_for(nf), 256, 0, s>>>(nf, iin.p);
    size_t bytes = 0;
    ck(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin.p, kout.p, iin.p, iout.p, nf, 0, 64, s), "sort size");
    DevBuf<unsigned char> tmp;
    tmp.alloc(std::max<size_t>(1, bytes));
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin.p, kout.p, iin.p, iout.p, nf, 0, 64, s), "sort");
    k_owner<<<blocks_for(nf), 256, 0, s>>>(nf, nranks, iout.p, own.p);
    ck(cudaGetLastError(), "owner");
    own.download(owner.data(), nf, s);
    ck(cudaStreamSynchronize(s), "owner download");
  }
  cudaStreamDestroy(s);
  return owner;
}

}  // namespace eqsb
