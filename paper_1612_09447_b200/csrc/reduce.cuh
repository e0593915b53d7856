// Deterministic reduction helpers and grid sizing shared by the kernel files
// (fixed grid, last-block ordered sum: the summation order never changes).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <unordered_map>
#include <utility>

#include "dev.cuh"

namespace eqsb {

// Programmatic dependent launch (PDL). Every kernel of k_rows.cu / k_sparse.cu
// starts with pdl_entry(): griddepcontrol.wait blocks until the preceding
// kernel on the stream has completed and its writes are visible (a no-op
// when the launch carried no PDL attribute), then launch_dependents lets the
// next PDL launch start its CTAs on SMs freed by this grid's last wave. The
// next kernel's launch latency and ramp thus overlap this kernel's tail;
// ordering and results are unchanged (each wait covers the whole chain).

__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

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

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline int grid_for(long n) {
  long g = (n + kBlock - 1) / kBlock;
  const long cap = 148L * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}
inline int grid_rows(long n_rows, int tpr) {
  long g = (n_rows * tpr + kBlock - 1) / kBlock;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace
}  // namespace eqsb
