// Matrix row kernels: one pass over a sparse operator with the AMG/PCG
// epilogue fused (SpMV, residual, Chebyshev smoothing steps, prolongation,
// fused dot products). HBM-bound. Two resident formats:
//   * CSR: TPR-thread groups per row (TPR from the mean row length);
//   * SELL-16 (sell.hpp): one warp per chunk of 32/TPR rows, slice-major
//     storage so every load instruction reads 32 consecutive entries, 16-bit
//     packed columns decoded through per-chunk window bases.
// Matrix values are fp64, fp32 or bf16 (DevCsr::prec); the vector type XT is
// fp64 for the PCG operator and fp32 (default) or fp64 inside the V-cycle.
// Row operands of the epilogue are loaded before the matrix pass so that
// their latency overlaps it.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "dev.cuh"
#include "reduce.cuh"

namespace eqsb {

// Algorithmic HBM bytes of one pass over `a` in its resident format: matrix
// stream (indices + values + row/chunk pointers), the gathered vector(s) once
// (n_cols each) and the streamed row vectors (n_rows each).
double matrix_pass_bytes(const DevCsr& a, int gathered, int streamed, int xbytes) {
  double m;
  if (a.stencil64() && a.st.sym) {  // upper slots only (lower values are re-reads of them)
    m = 8.0 * 8.0 * 32.0 * a.st.n_chunks + 32.0 * a.st.n_chunks + 128.0 * a.st.P;
  } else if (a.stencil64()) {
    m = 8.0 * 8.0 * 32.0 * a.st.G * a.st.n_chunks + 32.0 * a.st.n_chunks + 32.0 * a.st.G * a.st.P;
  } else if (a.stencil() && a.st.sym) {
    m = 2.0 * 8.0 * 32.0 * a.st.n_chunks + 32.0 * a.st.n_chunks + 128.0 * a.st.P;
  } else if (a.stencil()) {
    m = 16.0 * 32.0 * a.st.G * a.st.n_chunks + 32.0 * a.st.n_chunks + 32.0 * a.st.G * a.st.P;
  } else if (a.packed()) {
    m = 4.0 * (double)a.pk.padded + (4.0 + 4.0 * a.pk.windows) * a.pk.n_chunks + (a.pk.perm ? 4.0 * a.n_rows : 0.0);
  } else if (a.sell16()) {
    const double vs = a.prec == 2 ? 2.0 : a.prec == 1 ? 4.0 : 8.0;
    m = (double)a.sell.padded * (2.0 + vs) + 40.0 * a.sell.n_chunks;  // padded entries are read too
  } else {
    const double vs = (a.prec >= 1 && a.values_f) ? 4.0 : 8.0;
    m = (double)a.nnz * (4.0 + vs) + 4.0 * (a.n_rows + 1);
  }
  return m + (double)xbytes * ((double)gathered * a.n_cols + (double)streamed * a.n_rows);
}

namespace {

constexpr int kUnroll = 8;  // independent entries in flight per lane
#ifndef SELL_UNROLL1
#define SELL_UNROLL1 8
#endif
#ifndef SELL_MINB
#define SELL_MINB 1
#endif
#ifndef SELLS_RED_MINB
#define SELLS_RED_MINB 5  // k_sells_red: 48 registers, 5 CTAs per SM (A/B at C3: V-cycle -1.9%)
#endif
#ifndef SELLS_MINB
#define SELLS_MINB 6  // k_sells: 40 registers, 6 CTAs per SM (A/B at C3: V-cycle -2.8%)
#endif
constexpr int kSellUnroll1 = SELL_UNROLL1;
constexpr int kSymSlotsDev = 8;  // sell.hpp kSymSlots

// matrix entries are streamed once per pass: evict-first loads keep L2 for
// the gathered vectors (ld.global.cs). bf16 values are stored as uint16 bit
// patterns; bf16 -> fp32 is a 16-bit shift.
__device__ __forceinline__ double ldv(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float ldv(const float* p) { return __ldcs(p); }
__device__ __forceinline__ float ldv(const uint16_t* p) { return __uint_as_float((unsigned)__ldcs(p) << 16); }

// CSR row-group core: sum_k A_ik x_k (x_k w_k when SCALED) in lane 0 of the
// group. All lanes of the warp must call it (shuffles); rows >= n contribute nothing.
template <int TPR, class VT, class XT, bool SCALED>
__device__ __forceinline__ XT row_dot(const int* __restrict__ rp, const int* __restrict__ ci,
                                      const VT* __restrict__ v, const XT* __restrict__ x, const XT* __restrict__ w,
                                      int row, int lane, int n) {
  const bool ok = row < n;
  const int beg = ok ? __ldg(rp + row) : 0, end = ok ? __ldg(rp + row + 1) : 0;
  XT s = 0;
  for (int k0 = beg + lane; k0 < end; k0 += TPR * kUnroll) {
    int c[kUnroll];
    XT a[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int k = k0 + u * TPR;
      const bool in = k < end;
      c[u] = in ? __ldcs(ci + k) : 0;
      a[u] = in ? (XT)ldv(v + k) : (XT)0;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const XT xv = SCALED ? __ldg(x + c[u]) * __ldg(w + c[u]) : __ldg(x + c[u]);
      s += a[u] * xv;
    }
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, TPR);
  return s;
}

// SELL core: the chunk's slices are read with 32-bit offsets from the chunk
// base (immediate-offset loads inside a batch); window bases sit in lanes 0..7
// and are fetched per entry by a shuffle. Result in lane (row_in_chunk * TPR).
template <int TPR, class VT, class XT, bool SCALED>
__device__ __forceinline__ XT sell_dot(const DevSell& m, const VT* __restrict__ v, int chunk, int lane,
                                       const XT* __restrict__ x, const XT* __restrict__ w) {
  const long beg = __ldg(m.chunk_ptr + chunk);
  const int S = (int)((__ldg(m.chunk_ptr + chunk + 1) - beg) >> 5);  // slices (warp-uniform)
  const int mybase = lane < 8 ? __ldg(m.bases + 8L * chunk + lane) : 0;
  const uint16_t* cp = m.code + beg + lane;
  const VT* vp = v + beg + lane;
  // one batch covers a whole fine-level row (<= 16 slices at TPR 1)
  constexpr int U = TPR == 1 ? kSellUnroll1 : kUnroll;
  XT s = 0;
  for (int s0 = 0; s0 < S; s0 += U) {
    unsigned cd[U];
    XT a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool in = s0 + u < S;
      cd[u] = in ? (unsigned)__ldcs(cp + 32 * (s0 + u)) : 0u;
      a[u] = in ? (XT)ldv(vp + 32 * (s0 + u)) : (XT)0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = __shfl_sync(0xffffffffu, mybase, (int)(cd[u] >> 13)) + (int)(cd[u] & 0x1fffu);
      if (s0 + u < S) {
        const XT xv = SCALED ? __ldg(x + c) * __ldg(w + c) : __ldg(x + c);
        s += a[u] * xv;
      }
    }
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, TPR);
  return s;
}

// SELL-P core (sell.hpp): per step every lane reads one 16-byte group of four
// packed entries (bf16 value in the high half: decoding is a mask). Steps are
// batched by 4 (a whole fine-level row per batch at TPR 1). Result in lane
// (row_in_chunk * TPR).
// CG: gathers bypass L1 (for vectors written earlier in the same kernel)
template <bool CG, class T>
__device__ __forceinline__ T ldvec(const T* p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

template <int TPR, class XT, bool SCALED, bool CG = false>
__device__ __forceinline__ XT sellp_dot(const DevSellP& m, int chunk, int lane, const XT* __restrict__ x,
                                        const XT* __restrict__ w) {
  const int beg = m.uniform ? chunk * m.uniform * 32 : __ldg(m.chunk_ptr + chunk);
  const int S = m.uniform ? m.uniform : (__ldg(m.chunk_ptr + chunk + 1) - beg) >> 5;  // steps (warp-uniform)
  const int mybase = lane < m.windows ? __ldg(m.bases + (long)m.windows * chunk + lane) : 0;
  const unsigned mask = (1u << m.shift) - 1u;
  const int shift = m.shift;
  const uint4* p = m.words + beg + lane;
  constexpr int U = 4;
  XT s = 0;
  for (int s0 = 0; s0 < S; s0 += U) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; ++u) q[u] = s0 + u < S ? __ldcs(p + 32 * (s0 + u)) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned wd[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const unsigned code = wd[e] & 0xffffu;
        const int c = __shfl_sync(0xffffffffu, mybase, (int)(code >> shift)) + (int)(code & mask);
        if (s0 + u < S) {
          const XT a = (XT)__uint_as_float(wd[e] & 0xffff0000u);
          const XT xv = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
          s += a * xv;
        }
      }
    }
  }
#pragma unroll
  for (int o = TPR / 2; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, TPR);
  return s;
}

// Stencil-coded rows (TPR 1, one row per lane): the pattern table is staged in
// shared memory (spat); slot j of the row holds the value of its j-th CSR
// entry, so the products are summed in the same order as the TPR-1 SELL-P pass.
// G = 2 (up to 16 slots, the Kuhn-box fine level): the columns of the most
// frequent pattern are gathered speculatively together with the pattern id
// and the values, so no load waits on another; rows with another pattern
// gather again. Same products, same order.
template <class XT, bool SCALED, bool CG = false>
__device__ __forceinline__ XT sells_dot_g2(const DevSellS& m, const int* __restrict__ spat, int chunk, int lane,
                                           int row, const XT* __restrict__ x, const XT* __restrict__ w) {
  const int p = (int)__ldcs(m.pid + 32L * chunk + lane);
  const uint4* v = m.vals + (long)chunk * 2 * 32 + lane;
  const uint4 q0 = __ldcs(v), q1 = __ldcs(v + 32);
  const int cmax = m.n_cols - 1;
  XT xs[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {  // clamped: rows with another pattern may point outside
    const int c = min(max(row + (m.stage ? spat[m.common * 16 + j] : m.coff[j]), 0), cmax);
    xs[j] = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
  }
  if (p != m.common) {
    const int* off = (m.stage ? spat : m.pat) + p * 16;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = row + off[j];
      xs[j] = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
    }
  }
  const unsigned wd[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
  XT s = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    s += (XT)__uint_as_float(wd[e] << 16) * xs[2 * e];
    s += (XT)__uint_as_float(wd[e] & 0xffff0000u) * xs[2 * e + 1];
  }
  return s;
}

template <class XT, bool SCALED, bool CG = false>
__device__ __forceinline__ XT sells_dot(const DevSellS& m, const int* __restrict__ spat, int chunk, int lane,
                                        int row, const XT* __restrict__ x, const XT* __restrict__ w) {
  if (m.G == 2) return sells_dot_g2<XT, SCALED, CG>(m, spat, chunk, lane, row, x, w);
  const int G = m.G;
  const int* off = spat + (int)__ldcs(m.pid + 32L * chunk + lane) * (8 * G);
  const uint4* v = m.vals + (long)chunk * G * 32 + lane;
  uint4 qs[4];  // all value groups in flight before the gathers (G <= 4)
#pragma unroll
  for (int g = 0; g < 4; ++g) qs[g] = g < G ? __ldcs(v + 32 * g) : make_uint4(0u, 0u, 0u, 0u);
  XT s = 0;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (g >= G) break;
    const uint4 q = qs[g];
    const unsigned wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
      for (int hbit = 0; hbit < 2; ++hbit) {
        const int c = row + off[8 * g + 2 * e + hbit];
        const XT a = (XT)__uint_as_float(hbit ? (wd[e] & 0xffff0000u) : (wd[e] << 16));
        const XT xv = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
        s += a * xv;
      }
    }
  }
  return s;
}

// fp64 values (the PCG operator M_II): slot j of the chunk's lanes is one
// 256-byte warp load; products summed in CSR order
__device__ __forceinline__ double sells_dot64(const DevSellS& m, const int* __restrict__ spat, int chunk, int lane,
                                              int row, const double* __restrict__ x) {
  const int L = 8 * m.G;
  if (L == 16) {  // speculative gathers of the most frequent pattern (see sells_dot_g2)
    const int p = (int)__ldcs(m.pid + 32L * chunk + lane);
    const double* v = m.vals64 + (long)chunk * 16 * 32 + lane;
    double a[16], xs[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = __ldcs(v + 32 * j);
    const int cmax = m.n_cols - 1;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      xs[j] = __ldg(x + min(max(row + (m.stage ? spat[m.common * 16 + j] : m.coff[j]), 0), cmax));
    if (p != m.common) {
      const int* off = (m.stage ? spat : m.pat) + p * 16;
#pragma unroll
      for (int j = 0; j < 16; ++j) xs[j] = __ldg(x + row + off[j]);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j] * xs[j];
    return s;
  }
  const int* off = spat + (int)__ldcs(m.pid + 32L * chunk + lane) * L;
  const double* v = m.vals64 + (long)chunk * L * 32 + lane;
  double s = 0.0;
  for (int j0 = 0; j0 < L; j0 += 8) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = __ldcs(v + 32 * (j0 + u));
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u] * __ldg(x + row + off[j0 + u]);
  }
  return s;
}

__device__ __forceinline__ void stage_patterns(const DevSellS& m, int* spat) {
  for (int i = threadIdx.x; i < m.P * 8 * m.G; i += blockDim.x) spat[i] = __ldg(m.pat + i);
  __syncthreads();
}

// SELL-SH (sell.hpp, symmetric half storage; 16 slots): the pattern offsets
// [P][16] and slot kinds [P][16] in shared memory, then for the common
// pattern the element index of every (slot, lane) relative to the lane's
// chunk base (own upper slot: u 32 + lane; lower slot: the mirror row's upper
// slot in its chunk) and the pattern's padding mask
constexpr int kSymSmemInts(int P) { return P * 32 + 16 * 32 + 1; }
__device__ __forceinline__ void stage_sym(const DevSellS& m, int* spat) {
  const int np = m.P * 16;
  for (int i = threadIdx.x; i < np; i += blockDim.x) {
    spat[i] = __ldg(m.pat + i);
    spat[np + i] = __ldg(m.sinfo + i);
  }
  int* dtab = spat + 2 * np;
  for (int i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
    const int j = i >> 5, lane = i & 31;
    const int off = __ldg(m.pat + m.common * 16 + j), kind = __ldg(m.sinfo + m.common * 16 + j);
    int d = lane;  // padding: the row's first upper value (masked out)
    if (kind >= 0 && kind < 8) d = kind * 32 + lane;
    if (kind >= 8) {
      const int t = lane + off;  // mirror row = chunk * 32 + t
      d = (t >> 5) * (kSymSlotsDev * 32) + (kind - 8) * 32 + (t & 31);
    }
    dtab[i] = d;
  }
  if (threadIdx.x == 0) {
    unsigned pad = 0;
    for (int j = 0; j < 16; ++j) pad |= (__ldg(m.sinfo + m.common * 16 + j) < 0 ? 1u : 0u) << j;
    spat[2 * np + 16 * 32] = (int)pad;
  }
  __syncthreads();
}

__device__ __forceinline__ float sym_cvt(uint16_t v) { return __uint_as_float((unsigned)v << 16); }
__device__ __forceinline__ double sym_cvt(double v) { return v; }

// SELL-SH row dot: the 16 slots summed in CSR order, a[j] x[row + off_j]
// (x_j w_j when SCALED); a lower slot's value is the mirror row's upper value.
// Warps whose rows all have the common pattern and common-pattern lower
// neighbours (spid bit 7) use the warp-uniform slot kinds of the common
// pattern. Other warps take each lane's own pattern; a lane whose row lacks
// bit 7 reads its mirror slots from the slow-row table (16 bytes per row,
// located by a ballot over the chunk).
template <class T, class XT, bool SCALED, bool CG>
__device__ __forceinline__ XT sym_dot(const DevSellS& m, const T* __restrict__ U, const int* spat, int chunk, int lane,
                                      int row, const XT* __restrict__ x, const XT* __restrict__ w) {
  const unsigned pf = __ldcs(m.spid + 32L * chunk + lane);
  // speculative pass with the common pattern, issued before the pattern id
  // arrives (no pid -> address -> load chain); indices are clamped because a
  // row of another pattern may point outside the arrays, and such a warp
  // redoes its slots below. Every load is issued before the first use.
  T raw[16];
  XT xs[16];
  {
    const int* offc = spat + m.common * 16;
    const int* dtab = spat + m.P * 32 + lane;
    const long base = (long)chunk * kSymSlotsDev * 32;
    const long emax = (long)m.n_chunks * kSymSlotsDev * 32 - 1;
    const int cmax = m.n_cols - 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = min(max(row + offc[j], 0), cmax);
      xs[j] = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
      raw[j] = __ldg(U + min(max(base + dtab[32 * j], 0L), emax));
    }
  }
  unsigned pad = (unsigned)spat[m.P * 32 + 16 * 32];
  const int p = pf & 127;
  const bool fast = p == m.common && (pf & 0x80u);
  const unsigned slow = __ballot_sync(0xffffffffu, !fast);
  if (slow != 0) {
    // rows of another pattern or next to one: each lane's own pattern; a lane
    // whose row lacks bit 7 reads its mirror slots from the slow-row table
    const unsigned tab = __ballot_sync(0xffffffffu, !(pf & 0x80u));
    const T* own = U + (long)chunk * kSymSlotsDev * 32 + lane;
    const int* po = spat + p * 16;
    const int* pk = spat + m.P * 16 + p * 16;
    uint4 sc = make_uint4(0u, 0u, 0u, 0u);
    if (!(pf & 0x80u)) sc = __ldg(m.slow_code + __ldg(m.slow_base + chunk) + __popc(tab & ((1u << lane) - 1u)));
    const unsigned scw[4] = {sc.x, sc.y, sc.z, sc.w};
    pad = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int kind = pk[j];
      const int c = row + po[j];
      xs[j] = SCALED ? ldvec<CG>(x + c) * ldvec<CG>(w + c) : ldvec<CG>(x + c);
      const int u = (pf & 0x80u) ? kind - 8 : (int)((scw[j >> 2] >> (8 * (j & 3))) & 0xffu);
      const T* mirror = U + ((long)(c >> 5) * kSymSlotsDev + u) * 32 + (c & 31);
      raw[j] = __ldg(kind >= 8 ? mirror : own + 32 * max(kind, 0));
      pad |= (kind < 0 ? 1u : 0u) << j;
    }
  }
  XT s = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const XT a = (pad >> j) & 1u ? (XT)0 : (XT)sym_cvt(raw[j]);
    s += a * xs[j];
  }
  return s;
}

// Row epilogues (load before the pass, store after).
// Row ops (MODE < 0):
// OP 0: y = A x                       (restriction, plain SpMV)
// OP 1: y = b - A x                   (residual)
// OP 2: z += A zc                     (prolongation + correction; v = P)
// OP 3: z = c0 D^-1 b + c1 D^-1 (b - A D^-1 b / theta)          (Chebyshev(2) pre-smoothing from 0)
// OP 4: z = D^-1 b / theta ; t = b - A z                         (Chebyshev(1) pre-smoothing + residual)
// OP 5: zo = z + D^-1 (b - A z) / theta                          (Chebyshev(1) post-smoothing, out of place)
// OP 6: w = D^-1 A x                                             (power iteration on D^-1 A)
// OP 8: y = b - A x ; y2 = D^-1 y                                (residual + its scaled copy)
// OP 9: y = A x ; y2 = W y  (W: the next level's D^-1)          (restriction + its scaled copy)
// The scaled copies feed the PRE kernels: ops that gather D^-1 v (OP 3, 4,
// MODE 2, 3) then gather the one prescaled vector instead of v and D^-1,
// with bit-identical products.
// Reduction modes (MODE >= 0; the dot is accumulated in fp64):
// MODE 0: q = A p,  p.q
// MODE 1: y = b - A x, y.y
// MODE 2: z += c0 D^-1 r0 + c1 D^-1 (r0 - A D^-1 r0 / theta), b.z   (Chebyshev(2) post step 2; x = r0)
// MODE 3: as MODE 2 but z_out64 = z + ... in fp64 and b64.z_out64   (fine level of the fp32 V-cycle)
template <int OP, int MODE, class XT, bool CG = false>
struct Epi {
  XT p0 = 0, p1 = 0, p2 = 0, p3 = 0;
  double q = 0.0;
  static __device__ __forceinline__ XT ld(const XT* p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
  }
  __device__ __forceinline__ void load(int row, const XT* __restrict__ x, const XT* __restrict__ b,
                                       const XT* __restrict__ invd, const XT* y, const double* __restrict__ b64,
                                       int do_red) {
    if constexpr (MODE < 0) {
      if (OP == 1 || OP == 3 || OP == 4 || OP == 5 || OP == 8) p0 = ld(b + row);
      if (OP == 3 || OP == 4 || OP == 5 || OP == 6 || OP == 8 || OP == 9) p1 = ld(invd + row);
      if (OP == 5) p2 = ld(x + row);
      if (OP == 2) p2 = ld(y + row);
    } else {
      if (MODE == 0 || MODE >= 2) p0 = x[row];
      if (MODE == 1 || (MODE == 2 && do_red)) p1 = b[row];
      if (MODE == 3 && do_red) q = b64[row];
      if (MODE >= 2) {
        p2 = invd[row];
        p3 = y[row];
      }
    }
  }
  __device__ __forceinline__ double store(int row, XT s, XT* __restrict__ y, XT* __restrict__ y2,
                                          double* __restrict__ out64, const ChebCoef& c, int do_red) const {
    const XT c0 = (XT)c.c0, c1 = (XT)c.c1, it = (XT)c.inv_theta;
    if constexpr (MODE < 0) {
      if (OP == 0) y[row] = s;
      if (OP == 1) y[row] = p0 - s;
      if (OP == 2) y[row] = p2 + s;
      if (OP == 3) y[row] = c0 * p0 * p1 + c1 * p1 * (p0 - s * it);
      if (OP == 4) {
        y[row] = p0 * p1 * it;
        y2[row] = p0 - s * it;
      }
      if (OP == 5) y2[row] = p2 + p1 * (p0 - s) * it;
      if (OP == 6) y[row] = s * p1;
      if (OP == 8) {
        const XT r = p0 - s;
        y[row] = r;
        y2[row] = p1 * r;
      }
      if (OP == 9) {
        y[row] = s;
        y2[row] = p1 * s;
      }
      return 0.0;
    } else if (MODE == 0) {
      y[row] = s;
      return (double)p0 * (double)s;
    } else if (MODE == 1) {
      const XT r = p1 - s;
      y[row] = r;
      return (double)r * (double)r;
    } else if (MODE == 2) {
      const XT zn = p3 + (c0 * p0 * p2 + c1 * p2 * (p0 - s * it));
      y[row] = zn;
      return do_red ? (double)p1 * (double)zn : 0.0;
    } else {
      const double zn = (double)p3 + (double)(c0 * p0 * p2 + c1 * p2 * (p0 - s * it));
      out64[row] = zn;
      return do_red ? q * zn : 0.0;
    }
  }
};
template <int OP, int MODE>
constexpr bool kScaled = MODE < 0 ? (OP == 3 || OP == 4) : (MODE >= 2);

template <int TPR, class VT, class XT, int OP>
__global__ void __launch_bounds__(kBlock) k_row(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const VT* __restrict__ v, const XT* __restrict__ x,
                                                const XT* __restrict__ b, const XT* __restrict__ invd,
                                                XT* __restrict__ y, XT* __restrict__ y2, ChebCoef c) {
  pdl_entry();
  const long tid = (long)blockIdx.x * kBlock + threadIdx.x;
  const int row = (int)(tid / TPR), lane = (int)(tid % TPR);
  if ((tid & ~31L) / TPR >= n) return;  // warp-uniform exit
  constexpr bool SC = kScaled<OP, -1>;
  const bool act = lane == 0 && row < n;
  Epi<OP, -1, XT> e;
  if (act) e.load(row, x, b, invd, y, nullptr, 0);
  const XT s = row_dot<TPR, VT, XT, SC>(rp, ci, v, SC ? b : x, invd, row, lane, n);
  if (act) e.store(row, s, y, y2, nullptr, c, 0);
}

template <int TPR, class VT, class XT, int OP>
__global__ void __launch_bounds__(kBlock, SELL_MINB) k_sell(int n, DevSell m, const VT* __restrict__ v,
                                                 const XT* __restrict__ x, const XT* __restrict__ b,
                                                 const XT* __restrict__ invd, XT* __restrict__ y,
                                                 XT* __restrict__ y2, ChebCoef c) {
  pdl_entry();
  const int chunk = (int)(((long)blockIdx.x * kBlock + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (chunk >= m.n_chunks) return;  // warp-uniform exit
  constexpr bool SC = kScaled<OP, -1>;
  const int row = chunk * (32 / TPR) + lane / TPR;
  const bool act = lane % TPR == 0 && row < n;
  Epi<OP, -1, XT> e;
  if (act) e.load(row, x, b, invd, y, nullptr, 0);
  const XT s = sell_dot<TPR, VT, XT, SC>(m, v, chunk, lane, SC ? b : x, invd);
  if (act) e.store(row, s, y, y2, nullptr, c, 0);
}

template <int TPR, class XT, int OP, bool PRE>
__global__ void __launch_bounds__(kBlock) k_sellp(int n, DevSellP m, const XT* __restrict__ x,
                                                  const XT* __restrict__ b, const XT* __restrict__ invd,
                                                  XT* __restrict__ y, XT* __restrict__ y2, ChebCoef c,
                                                  const XT* __restrict__ pre) {
  pdl_entry();
  const int chunk = (int)(((long)blockIdx.x * kBlock + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (chunk >= m.n_chunks) return;  // warp-uniform exit
  constexpr bool SC = kScaled<OP, -1>;
  const int slot = chunk * (32 / TPR) + lane / TPR;
  const bool act = lane % TPR == 0 && slot < n;
  const int row = act && m.perm ? __ldg(m.perm + slot) : slot;  // sorted rows (SELL-C-sigma)
  Epi<OP, -1, XT> e;
  if (act) e.load(row, x, b, invd, y, nullptr, 0);
  const XT s = sellp_dot<TPR, XT, SC && !PRE>(m, chunk, lane, SC ? (PRE ? pre : b) : x, invd);
  if (act) e.store(row, s, y, y2, nullptr, c, 0);
}

template <class XT, int OP, bool PRE, bool SYM>
__global__ void __launch_bounds__(kBlock, SELLS_MINB) k_sells(int n, DevSellS m, const XT* __restrict__ x,
                                                  const XT* __restrict__ b, const XT* __restrict__ invd,
                                                  XT* __restrict__ y, XT* __restrict__ y2, ChebCoef c,
                                                  const XT* __restrict__ pre) {
  extern __shared__ int spat[];
  if (SYM) stage_sym(m, spat);
  else if (m.G != 2 || m.stage) stage_patterns(m, spat);  // m.stage = 0: offsets from the parameters
  pdl_entry();
  const int chunk = (int)(((long)blockIdx.x * kBlock + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (chunk >= m.n_chunks) return;  // warp-uniform exit
  constexpr bool SC = kScaled<OP, -1>;
  const int row = chunk * 32 + lane;
  const bool act = row < n;
  Epi<OP, -1, XT> e;
  if (act) e.load(row, x, b, invd, y, nullptr, 0);
  XT s;
  if constexpr (SYM)
    s = sym_dot<uint16_t, XT, SC && !PRE, false>(m, m.u16, spat, chunk, lane, act ? row : 0,
                                                 SC ? (PRE ? pre : b) : x, invd);
  else
    s = sells_dot<XT, SC && !PRE>(m, spat, chunk, lane, act ? row : 0, SC ? (PRE ? pre : b) : x, invd);
  if (act) e.store(row, s, y, y2, nullptr, c, 0);
}

template <class XT, int MODE, bool PRE, bool SYM>
__global__ void __launch_bounds__(kBlock, SELLS_RED_MINB) k_sells_red(int n, DevSellS m, const XT* __restrict__ x,
                                                      const XT* __restrict__ b, const XT* __restrict__ invd,
                                                      XT* __restrict__ y, double* __restrict__ out64,
                                                      const double* __restrict__ b64, ChebCoef c, Reducer red,
                                                      int slot, int do_red, const XT* __restrict__ pre) {
  extern __shared__ int spat[];
  if (SYM) stage_sym(m, spat);
  else if (m.G != 2 || m.stage) stage_patterns(m, spat);  // m.stage = 0: offsets from the parameters
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kBlock / 32);
  double acc = 0.0;
  for (int chunk = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); chunk < m.n_chunks; chunk += warps) {
    const int row = chunk * 32 + lane;
    const bool act = row < n;
    Epi<0, MODE, XT> e;
    if (act) e.load(row, x, b, invd, y, b64, do_red);
    XT s;
    if constexpr (SYM)
      s = sym_dot<uint16_t, XT, kScaled<0, MODE> && !PRE, false>(m, m.u16, spat, chunk, lane, act ? row : 0,
                                                                 PRE ? pre : x, invd);
    else
      s = sells_dot<XT, kScaled<0, MODE> && !PRE>(m, spat, chunk, lane, act ? row : 0, PRE ? pre : x, invd);
    if (act) acc += e.store(row, s, y, nullptr, out64, c, do_red);
  }
  reduce_finish(acc, red, slot);
}

// q = A p (MODE -1) / q = A p, p.q (MODE 0) / r = b - A x, r.r (MODE 1) with
// the fp64 stencil-coded operator
template <int MODE, bool SYM>
__global__ void __launch_bounds__(kBlock) k_sells64(int n, DevSellS m, const double* __restrict__ x,
                                                    double* __restrict__ y, Reducer red, int slot, int do_red,
                                                    const double* __restrict__ b) {
  extern __shared__ int spat[];
  if (SYM) stage_sym(m, spat);
  else if (m.G != 2 || m.stage) stage_patterns(m, spat);  // m.stage = 0: offsets from the parameters
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kBlock / 32);
  double acc = 0.0;
  for (int chunk = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); chunk < m.n_chunks; chunk += warps) {
    const int row = chunk * 32 + lane;
    const bool act = row < n;
    const double s = SYM ? sym_dot<double, double, false, false>(m, m.u64, spat, chunk, lane, act ? row : 0, x, nullptr)
                         : sells_dot64(m, spat, chunk, lane, act ? row : 0, x);
    if (act) {
      if (MODE == 1) {
        const double r = b[row] - s;
        y[row] = r;
        acc += r * r;
      } else {
        y[row] = s;
        if (MODE == 0) acc += x[row] * s;
      }
    }
  }
  if (MODE >= 0 && do_red) reduce_finish(acc, red, slot);
}

template <int TPR, class XT, int MODE, bool PRE>
__global__ void __launch_bounds__(kBlock) k_sellp_red(int n, DevSellP m, const XT* __restrict__ x,
                                                      const XT* __restrict__ b, const XT* __restrict__ invd,
                                                      XT* __restrict__ y, double* __restrict__ out64,
                                                      const double* __restrict__ b64, ChebCoef c, Reducer red,
                                                      int slot, int do_red, const XT* __restrict__ pre) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kBlock / 32);
  double acc = 0.0;
  for (int chunk = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); chunk < m.n_chunks; chunk += warps) {
    const int slot = chunk * (32 / TPR) + lane / TPR;
    const bool act = lane % TPR == 0 && slot < n;
    const int row = act && m.perm ? __ldg(m.perm + slot) : slot;  // sorted rows (SELL-C-sigma)
    Epi<0, MODE, XT> e;
    if (act) e.load(row, x, b, invd, y, b64, do_red);
    const XT s = sellp_dot<TPR, XT, kScaled<0, MODE> && !PRE>(m, chunk, lane, PRE ? pre : x, invd);
    if (act) acc += e.store(row, s, y, nullptr, out64, c, do_red);
  }
  if (do_red) reduce_finish(acc, red, slot);
}

// grid-stride kernels with a fused reduction (fixed grid: deterministic)
template <int TPR, class VT, class XT, int MODE>
__global__ void __launch_bounds__(kBlock) k_row_red(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const VT* __restrict__ v, const XT* __restrict__ x,
                                                    const XT* __restrict__ b, const XT* __restrict__ invd,
                                                    XT* __restrict__ y, double* __restrict__ out64,
                                                    const double* __restrict__ b64, ChebCoef c, Reducer red,
                                                    int slot, int do_red) {
  pdl_entry();
  const int lane = threadIdx.x % TPR;
  const long groups_per_grid = (long)gridDim.x * (kBlock / TPR);
  // every group iterates the same number of times (shuffles need full warps)
  const long n_pad = ((n + (long)(kBlock / TPR) - 1) / (kBlock / TPR)) * (kBlock / TPR);
  double acc = 0.0;
  for (long row = (long)blockIdx.x * (kBlock / TPR) + threadIdx.x / TPR; row < n_pad; row += groups_per_grid) {
    const bool act = lane == 0 && row < n;
    Epi<0, MODE, XT> e;
    if (act) e.load((int)row, x, b, invd, y, b64, do_red);
    const XT s = row_dot<TPR, VT, XT, kScaled<0, MODE>>(rp, ci, v, x, invd, (int)row, lane, n);
    if (act) acc += e.store((int)row, s, y, nullptr, out64, c, do_red);
  }
  if (do_red) reduce_finish(acc, red, slot);
}

template <int TPR, class VT, class XT, int MODE>
__global__ void __launch_bounds__(kBlock) k_sell_red(int n, DevSell m, const VT* __restrict__ v,
                                                     const XT* __restrict__ x, const XT* __restrict__ b,
                                                     const XT* __restrict__ invd, XT* __restrict__ y,
                                                     double* __restrict__ out64, const double* __restrict__ b64,
                                                     ChebCoef c, Reducer red, int slot, int do_red) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (kBlock / 32);
  double acc = 0.0;
  for (int chunk = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); chunk < m.n_chunks; chunk += warps) {
    const int row = chunk * (32 / TPR) + lane / TPR;
    const bool act = lane % TPR == 0 && row < n;
    Epi<0, MODE, XT> e;
    if (act) e.load(row, x, b, invd, y, b64, do_red);
    const XT s = sell_dot<TPR, VT, XT, kScaled<0, MODE>>(m, v, chunk, lane, x, invd);
    if (act) acc += e.store(row, s, y, nullptr, out64, c, do_red);
  }
  if (do_red) reduce_finish(acc, red, slot);
}

#define TPR_SWITCH_(tpr, L_, VT, V) \
  switch (tpr) {                    \
    case 1: L_(1, VT, V); break;    \
    case 2: L_(2, VT, V); break;    \
    case 4: L_(4, VT, V); break;    \
    case 8: L_(8, VT, V); break;    \
    case 16: L_(16, VT, V); break;  \
    default: L_(32, VT, V); break;  \
  }

// value array per format and precision; fp32 vectors never read fp64 values
// (the V-cycle then uses the fp32 copy)
template <class XT>
int eff_prec(const DevCsr& a) {
  int p = a.prec;
  if (std::is_same_v<XT, float> && p == 0) p = 1;
  const bool has16 = a.use_sell && a.sell.tpr > 0, hasp = a.use_sell && a.pk.tpr > 0;
  if (p == 2 && !has16 && !hasp) p = 1;  // CSR has no bf16 copy
  if (p == 1 && !has16 && !a.values_f) p = 0;
  return p;
}

template <class XT, int OP>
void row_launch(const DevCsr& a, const XT* x, const XT* b, const XT* invd, XT* y, XT* y2, ChebCoef c, cudaStream_t s,
                const XT* pre = nullptr) {
  if (a.n_rows == 0) return;
  ++g_launch_count;
  // gathered / streamed row vectors per op (Epi)
  constexpr int kG[10] = {1, 1, 1, 2, 2, 1, 1, 0, 1, 1}, kS[10] = {1, 2, 2, 1, 2, 3, 2, 0, 4, 3};
  const int p = eff_prec<XT>(a);
  DevCsr view = a;
  view.prec = p;
  if constexpr (std::is_same_v<XT, double> && OP == 0) {
    if (view.stencil64()) {
      const DevSellS& m = a.st;
      g_algo_bytes += matrix_pass_bytes(view, 1, 1, 8);
      if (m.sym)
        launch_pdl(k_sells64<-1, true>, red_grid(k_sells64<-1, true>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * kSymSmemInts(m.P), s, a.n_rows, m, x, y, Reducer{}, 0, 0, (const double*)nullptr);
      else
        launch_pdl(k_sells64<-1, false>, red_grid(k_sells64<-1, false>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * m.P * 8 * m.G, s, a.n_rows, m, x, y, Reducer{}, 0, 0, (const double*)nullptr);
      return;
    }
  }
  if (view.stencil()) {
    const DevSellS& m = a.st;
    const int g = (int)(((long)m.n_chunks * 32 + kBlock - 1) / kBlock);
    const size_t smem = m.sym ? sizeof(int) * kSymSmemInts(m.P) : sizeof(int) * m.P * 8 * m.G;
    if (pre && kScaled<OP, -1>) {
      g_algo_bytes += matrix_pass_bytes(view, 1, kS[OP] + 2, sizeof(XT));
      if (m.sym) launch_pdl(k_sells<XT, OP, true, true>, g, kBlock, smem, s, a.n_rows, m, x, b, invd, y, y2, c, pre);
      else launch_pdl(k_sells<XT, OP, true, false>, g, kBlock, smem, s, a.n_rows, m, x, b, invd, y, y2, c, pre);
    } else {
      g_algo_bytes += matrix_pass_bytes(view, kG[OP], kS[OP], sizeof(XT));
      if (m.sym)
        launch_pdl(k_sells<XT, OP, false, true>, g, kBlock, smem, s, a.n_rows, m, x, b, invd, y, y2, c, nullptr);
      else
        launch_pdl(k_sells<XT, OP, false, false>, g, kBlock, smem, s, a.n_rows, m, x, b, invd, y, y2, c, nullptr);
    }
    return;
  }
  if (view.packed()) {
    const DevSellP& m = a.pk;
    const int g = (int)(((long)m.n_chunks * 32 + kBlock - 1) / kBlock);
    if (pre && kScaled<OP, -1>) {  // one prescaled gather; b and D^-1 read per row
      g_algo_bytes += matrix_pass_bytes(view, 1, kS[OP] + 2, sizeof(XT));
#define P_(T, VT, V) launch_pdl(k_sellp<T, XT, OP, true>, g, kBlock, 0, s, a.n_rows, m, x, b, invd, y, y2, c, pre)
      TPR_SWITCH_(m.tpr, P_, void, 0)
#undef P_
      return;
    }
    g_algo_bytes += matrix_pass_bytes(view, kG[OP], kS[OP], sizeof(XT));
#define P_(T, VT, V) launch_pdl(k_sellp<T, XT, OP, false>, g, kBlock, 0, s, a.n_rows, m, x, b, invd, y, y2, c, nullptr)
    TPR_SWITCH_(m.tpr, P_, void, 0)
#undef P_
    return;
  }
  if (view.sell16()) {
    const DevSell& m = a.sell;
    g_algo_bytes += matrix_pass_bytes(view, kG[OP], kS[OP], sizeof(XT));
    const int g = (int)(((long)m.n_chunks * 32 + kBlock - 1) / kBlock);
#define S_(T, VT, V) launch_pdl(k_sell<T, VT, XT, OP>, g, kBlock, 0, s, a.n_rows, m, V, x, b, invd, y, y2, c)
    if (p == 2) {
      TPR_SWITCH_(m.tpr, S_, uint16_t, m.v16)
    } else if (p == 1 || std::is_same_v<XT, float>) {
      TPR_SWITCH_(m.tpr, S_, float, m.v32)
    } else {
      if constexpr (std::is_same_v<XT, double>) TPR_SWITCH_(m.tpr, S_, double, m.v64)
    }
#undef S_
    return;
  }
  g_algo_bytes += matrix_pass_bytes(view, kG[OP], kS[OP], sizeof(XT));
  const int g = grid_rows(a.n_rows, a.tpr);
#define L_(T, VT, V) launch_pdl(k_row<T, VT, XT, OP>, g, kBlock, 0, s, a.n_rows, a.row_ptr, a.col_idx, V, x, b, invd, y, y2, c)
  if (p >= 1 || std::is_same_v<XT, float>) {
    TPR_SWITCH_(a.tpr, L_, float, a.values_f)
  } else {
    if constexpr (std::is_same_v<XT, double>) TPR_SWITCH_(a.tpr, L_, double, a.values)
  }
#undef L_
}

template <class XT, int MODE>
void row_red_launch(const DevCsr& a, const XT* x, const XT* b, const XT* invd, XT* y, double* out64,
                    const double* b64, ChebCoef c, Reducer* red, int slot, cudaStream_t s, const XT* pre = nullptr) {
  if (a.n_rows == 0) return;
  ++g_launch_count;
  Reducer r = red ? *red : Reducer{};
  const int dr = red ? 1 : 0;
  constexpr int kG[4] = {1, 1, 2, 2}, kS[4] = {1, 2, 3, 2};
  const int p = eff_prec<XT>(a);
  DevCsr view = a;
  view.prec = p;
  const bool use_pre = pre && kScaled<0, MODE> && (view.packed() || view.stencil());
  double bytes = use_pre ? matrix_pass_bytes(view, 1, kS[MODE] + 2, sizeof(XT))
                         : matrix_pass_bytes(view, kG[MODE], kS[MODE], sizeof(XT));
  if (MODE == 2 && red) bytes += sizeof(XT) * (double)a.n_rows;
  if (MODE == 3) bytes += (red ? 16.0 : 8.0) * a.n_rows;
  if constexpr (std::is_same_v<XT, double> && MODE == 1) {
    if (view.stencil64()) {  // fp64 residual + r.r (PCG start with x0 != 0)
      const DevSellS& m = a.st;
      g_algo_bytes += matrix_pass_bytes(view, 1, 2, 8);
      if (m.sym)
        launch_pdl(k_sells64<1, true>, red_grid(k_sells64<1, true>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * kSymSmemInts(m.P), s, a.n_rows, m, x, y, r, slot, dr, b);
      else
        launch_pdl(k_sells64<1, false>, red_grid(k_sells64<1, false>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * m.P * 8 * m.G, s, a.n_rows, m, x, y, r, slot, dr, b);
      return;
    }
  }
  if constexpr (std::is_same_v<XT, double> && MODE == 0) {
    if (view.stencil64()) {
      const DevSellS& m = a.st;
      g_algo_bytes += matrix_pass_bytes(view, 1, 1, 8);
      if (m.sym)
        launch_pdl(k_sells64<0, true>, red_grid(k_sells64<0, true>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * kSymSmemInts(m.P), s, a.n_rows, m, x, y, r, slot, dr, (const double*)nullptr);
      else
        launch_pdl(k_sells64<0, false>, red_grid(k_sells64<0, false>, (long)m.n_chunks * 32), kBlock,
                   sizeof(int) * m.P * 8 * m.G, s, a.n_rows, m, x, y, r, slot, dr, (const double*)nullptr);
      return;
    }
  }
  g_algo_bytes += bytes;
  if (view.stencil()) {
    const DevSellS& m = a.st;
    const long work = (long)m.n_chunks * 32;
    const size_t smem = m.sym ? sizeof(int) * kSymSmemInts(m.P) : sizeof(int) * m.P * 8 * m.G;
#define R_(PRE, SYM, PP)                                                                                      \
  launch_pdl(k_sells_red<XT, MODE, PRE, SYM>, red_grid(k_sells_red<XT, MODE, PRE, SYM>, work), kBlock, smem, s, \
             a.n_rows, m, x, b, invd, y, out64, b64, c, r, slot, dr, PP)
    if (use_pre) {
      if (m.sym) R_(true, true, pre);
      else R_(true, false, pre);
    } else {
      if (m.sym) R_(false, true, nullptr);
      else R_(false, false, nullptr);
    }
#undef R_
    return;
  }
  if (view.packed()) {
    const DevSellP& m = a.pk;
    const long work = (long)m.n_chunks * 32;
    if (use_pre) {
#define P_(T, VT, V)                                                                                   \
  launch_pdl(k_sellp_red<T, XT, MODE, true>, red_grid(k_sellp_red<T, XT, MODE, true>, work), kBlock, 0, s,      \
      a.n_rows, m, x, b, invd, y, out64, b64, c, r, slot, dr, pre)
      TPR_SWITCH_(m.tpr, P_, void, 0)
#undef P_
      return;
    }
#define P_(T, VT, V)                                                                                   \
  launch_pdl(k_sellp_red<T, XT, MODE, false>, red_grid(k_sellp_red<T, XT, MODE, false>, work), kBlock, 0, s,    \
      a.n_rows, m, x, b, invd, y, out64, b64, c, r, slot, dr, nullptr)
    TPR_SWITCH_(m.tpr, P_, void, 0)
#undef P_
    return;
  }
  if (view.sell16()) {
    const DevSell& m = a.sell;
    const long work = (long)m.n_chunks * 32;
#define S_(T, VT, V)                                                                                              \
  launch_pdl(k_sell_red<T, VT, XT, MODE>, red_grid(k_sell_red<T, VT, XT, MODE>, work), kBlock, 0, s,                       \
      a.n_rows, m, V, x, b, invd, y, out64, b64, c, r, slot, dr)
    if (p == 2) {
      TPR_SWITCH_(m.tpr, S_, uint16_t, m.v16)
    } else if (p == 1 || std::is_same_v<XT, float>) {
      TPR_SWITCH_(m.tpr, S_, float, m.v32)
    } else {
      if constexpr (std::is_same_v<XT, double>) TPR_SWITCH_(m.tpr, S_, double, m.v64)
    }
#undef S_
    return;
  }
  const long work = (long)a.n_rows * a.tpr;
#define L_(T, VT, V)                                                                                             \
  launch_pdl(k_row_red<T, VT, XT, MODE>, red_grid(k_row_red<T, VT, XT, MODE>, work), kBlock, 0, s,                        \
      a.n_rows, a.row_ptr, a.col_idx, V, x, b, invd, y, out64, b64, c, r, slot, dr)
  if (p >= 1 || std::is_same_v<XT, float>) {
    TPR_SWITCH_(a.tpr, L_, float, a.values_f)
  } else {
    if constexpr (std::is_same_v<XT, double>) TPR_SWITCH_(a.tpr, L_, double, a.values)
  }
#undef L_
}

}  // namespace

namespace {
// one thread per row; the first padded slot is the second slot whose column
// offset is 0 (a row's real entries have distinct columns, padding follows them)
__global__ void __launch_bounds__(kBlock) k_sells_rowsum(int n, DevSellS m, uint16_t* __restrict__ vals, int on) {
  const int row = blockIdx.x * kBlock + threadIdx.x;
  if (row >= n) return;
  const int L = 8 * m.G, chunk = row / 32, lane = row % 32;
  const int* off = m.pat + (int)m.pid[row] * L;
  double e = 0.0;
  int slot = -1;
  bool diag = false;
  for (int j = 0; j < L; ++j) {
    const size_t at = (((size_t)chunk * m.G + j / 8) * 32 + lane) * 8 + j % 8;
    if (off[j] == 0) {
      if (diag && slot < 0) slot = (int)j;
      diag = true;
    }
    const double a = m.vals64[((size_t)chunk * L + j) * 32 + lane];
    if (a != 0.0) e += a - (double)__uint_as_float((unsigned)vals[at] << 16);
  }
  if (slot >= 0) {
    const size_t at = (((size_t)chunk * m.G + slot / 8) * 32 + lane) * 8 + slot % 8;
    vals[at] = on ? __bfloat16_as_ushort(__float2bfloat16_rn((float)e)) : (uint16_t)0;
  }
}
}  // namespace

void launch_sells_rowsum(int n_rows, const DevSellS& m, uint16_t* vals, bool on, cudaStream_t s) {
  if (n_rows == 0 || !m.vals64 || m.sym) return;
  ++g_launch_count;
  k_sells_rowsum<<<(n_rows + kBlock - 1) / kBlock, kBlock, 0, s>>>(n_rows, m, vals, on ? 1 : 0);
}

template <class XT>
void launch_spmv(const DevCsr& a, const XT* x, XT* y, cudaStream_t s) {
  row_launch<XT, 0>(a, x, nullptr, nullptr, y, nullptr, ChebCoef{}, s);
}
template <class XT>
void launch_residual(const DevCsr& a, const XT* b, const XT* x, XT* y, Reducer* red, int slot, cudaStream_t s) {
  if (red) row_red_launch<XT, 1>(a, x, b, nullptr, y, nullptr, nullptr, ChebCoef{}, red, slot, s);
  else row_launch<XT, 1>(a, x, b, nullptr, y, nullptr, ChebCoef{}, s);
}
void launch_spmv_dot(const DevCsr& a, const double* p, double* q, Reducer red, int slot, cudaStream_t s) {
  row_red_launch<double, 0>(a, p, nullptr, nullptr, q, nullptr, nullptr, ChebCoef{}, &red, slot, s);
}
template <class XT>
void launch_prolong_add(const DevCsr& p, const XT* zc, XT* z, cudaStream_t s) {
  row_launch<XT, 2>(p, zc, nullptr, nullptr, z, nullptr, ChebCoef{}, s);
}
template <class XT>
void launch_residual_scaled(const DevCsr& a, const XT* b, const XT* x, const XT* invd, XT* y, XT* y2, cudaStream_t s) {
  row_launch<XT, 8>(a, x, b, invd, y, y2, ChebCoef{}, s);
}
template <class XT>
void launch_spmv_scaled(const DevCsr& a, const XT* x, const XT* w, XT* y, XT* y2, cudaStream_t s) {
  row_launch<XT, 9>(a, x, nullptr, w, y, y2, ChebCoef{}, s);
}
template <class XT>
void launch_cheb_pre(const DevCsr& a, const XT* invd, const XT* b, XT* z, ChebCoef c, cudaStream_t s, const XT* pre) {
  row_launch<XT, 3>(a, nullptr, b, invd, z, nullptr, c, s, pre);
}
template <class XT>
void launch_cheb_post2(const DevCsr& a, const XT* invd, const XT* r0, XT* z, ChebCoef c, const XT* b_dot,
                       Reducer* red, int slot, cudaStream_t s, const XT* pre) {
  row_red_launch<XT, 2>(a, r0, b_dot, invd, z, nullptr, nullptr, c, red, slot, s, pre);
}
void launch_cheb_post2_out64(const DevCsr& a, const float* invd, const float* r0, const float* z, ChebCoef c,
                             double* z_out, const double* b_dot, Reducer* red, int slot, cudaStream_t s,
                             const float* pre) {
  row_red_launch<float, 3>(a, r0, nullptr, invd, const_cast<float*>(z), z_out, b_dot, c, red, slot, s, pre);
}
template <class XT>
void launch_cheb1_pre_resid(const DevCsr& a, const XT* invd, const XT* b, XT* z, XT* t, ChebCoef c, cudaStream_t s,
                            const XT* pre) {
  row_launch<XT, 4>(a, nullptr, b, invd, z, t, c, s, pre);
}
template <class XT>
void launch_cheb1_post(const DevCsr& a, const XT* invd, const XT* b, const XT* z, XT* z_out, ChebCoef c,
                       cudaStream_t s) {
  row_launch<XT, 5>(a, z, b, invd, nullptr, z_out, c, s);
}
void launch_scaled_spmv(const DevCsr& a, const double* invd, const double* v, double* w, cudaStream_t s) {
  row_launch<double, 6>(a, v, nullptr, invd, w, nullptr, ChebCoef{}, s);
}

#define INST_(XT)                                                                                              \
  template void launch_spmv<XT>(const DevCsr&, const XT*, XT*, cudaStream_t);                                  \
  template void launch_residual<XT>(const DevCsr&, const XT*, const XT*, XT*, Reducer*, int, cudaStream_t);     \
  template void launch_prolong_add<XT>(const DevCsr&, const XT*, XT*, cudaStream_t);                           \
  template void launch_residual_scaled<XT>(const DevCsr&, const XT*, const XT*, const XT*, XT*, XT*, cudaStream_t); \
  template void launch_spmv_scaled<XT>(const DevCsr&, const XT*, const XT*, XT*, XT*, cudaStream_t);          \
  template void launch_cheb_pre<XT>(const DevCsr&, const XT*, const XT*, XT*, ChebCoef, cudaStream_t, const XT*); \
  template void launch_cheb_post2<XT>(const DevCsr&, const XT*, const XT*, XT*, ChebCoef, const XT*, Reducer*,  \
                                      int, cudaStream_t, const XT*);                                           \
  template void launch_cheb1_pre_resid<XT>(const DevCsr&, const XT*, const XT*, XT*, XT*, ChebCoef, cudaStream_t, \
                                           const XT*);                                                         \
  template void launch_cheb1_post<XT>(const DevCsr&, const XT*, const XT*, const XT*, XT*, ChebCoef, cudaStream_t);
INST_(double)
INST_(float)
#undef INST_

}  // namespace eqsb
