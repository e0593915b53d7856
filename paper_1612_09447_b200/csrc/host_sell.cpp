// SELL-16 encoder (sell.hpp). Deterministic; chunks are independent, so the
// window search and the per-chunk layout run in parallel.
#include <omp.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "sell.hpp"

namespace eqsb {

int choose_sell_tpr(const HostCsr& a, int per_lane) {
  if (a.n_rows == 0) return 1;
  const double avg = (double)a.nnz() / a.n_rows;
  int t = 1;
  while (t < 32 && t * per_lane < avg) t <<= 1;
  return t;
}

int choose_sellp_tpr(const HostCsr& a) {
  static const int per_lane = getenv("EQS_SELLP_LANE_ENTRIES") ? atoi(getenv("EQS_SELLP_LANE_ENTRIES")) : 32;
  return choose_sell_tpr(a, per_lane);
}

bool build_sell(const HostCsr& a, int tpr, HostSell& out) {
  const int rows_per_chunk = 32 / tpr;
  const int n_chunks = (a.n_rows + rows_per_chunk - 1) / rows_per_chunk;
  std::vector<long> len(n_chunks + 1, 0);
  std::vector<int> bases((size_t)n_chunks * kSellWindows, 0);
  int fail = 0;
#pragma omp parallel
  {
    std::vector<int> cols;
#pragma omp for schedule(static) reduction(max : fail)
    for (int c = 0; c < n_chunks; ++c) {
      const int r0 = c * rows_per_chunk, r1 = std::min(a.n_rows, r0 + rows_per_chunk);
      int maxlen = 0;
      cols.assign(a.col_idx.begin() + a.row_ptr[r0], a.col_idx.begin() + a.row_ptr[r1]);
      for (int r = r0; r < r1; ++r) maxlen = std::max(maxlen, a.row_ptr[r + 1] - a.row_ptr[r]);
      std::sort(cols.begin(), cols.end());
      int w = 0;
      for (size_t i = 0; i < cols.size();) {
        if (w == kSellWindows) {
          fail = 1;
          break;
        }
        const int b = cols[i];
        bases[(size_t)c * kSellWindows + w++] = b;
        while (i < cols.size() && cols[i] < b + kSellSpan) ++i;
      }
      for (int k = w; k < kSellWindows; ++k) bases[(size_t)c * kSellWindows + k] = INT_MAX;  // unused
      len[c + 1] = 32L * ((maxlen + tpr - 1) / tpr);
    }
  }
  if (fail) return false;
  for (int c = 0; c < n_chunks; ++c) len[c + 1] += len[c];
  HostSell s;
  s.tpr = tpr;
  s.n_rows = a.n_rows;
  s.n_chunks = n_chunks;
  s.chunk_ptr = std::move(len);
  s.bases = std::move(bases);
  s.code.assign(s.padded(), 0);
  s.src.assign(s.padded(), -1);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < n_chunks; ++c) {
    const int* wb = &s.bases[(size_t)c * kSellWindows];
    const int r0 = c * rows_per_chunk, r1 = std::min(a.n_rows, r0 + rows_per_chunk);
    for (int r = r0; r < r1; ++r) {
      const int q = r - r0;
      for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
        const int j = k - a.row_ptr[r], col = a.col_idx[k];
        // windows ascend (unused ones are INT_MAX): the owner is the last base <= col
        int w = kSellWindows - 1;
        while (w > 0 && wb[w] > col) --w;
        const long pos = s.chunk_ptr[c] + 32L * (j / tpr) + q * tpr + j % tpr;
        s.code[pos] = (uint16_t)((w << kSellShift) | (col - wb[w]));
        s.src[pos] = k;
      }
    }
  }
  out = std::move(s);
  return true;
}


uint16_t to_bf16(double d) {
  const float f = (float)d;
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

namespace {
// windows of `span` columns covering the sorted columns of one chunk; false if
// more than `max_w` are needed
bool chunk_windows(std::vector<int>& cols, int span, int max_w, int* out) {
  std::sort(cols.begin(), cols.end());
  int w = 0;
  for (size_t i = 0; i < cols.size();) {
    if (w == max_w) return false;
    const int b = cols[i];
    out[w++] = b;
    while (i < cols.size() && cols[i] < b + span) ++i;
  }
  for (int k = w; k < max_w; ++k) out[k] = INT_MAX;  // unused
  return true;
}
}  // namespace

bool build_sell_packed(const HostCsr& a, int tpr, HostSellP& out, int sigma) {
  const int rows_per_chunk = 32 / tpr;
  const int n_chunks = (a.n_rows + rows_per_chunk - 1) / rows_per_chunk;
  // slot row -> matrix row (identity unless sorted)
  std::vector<int> perm;
  if (sigma > 0) {
    perm.resize(a.n_rows);
    for (int i = 0; i < a.n_rows; ++i) perm[i] = i;
    for (int w0 = 0; w0 < a.n_rows; w0 += sigma) {
      const int w1 = std::min(a.n_rows, w0 + sigma);
      std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int x, int y) {
        return a.row_ptr[x + 1] - a.row_ptr[x] > a.row_ptr[y + 1] - a.row_ptr[y];
      });
    }
  }
  auto row_of = [&](int i) { return perm.empty() ? i : perm[i]; };
  for (int shift = 13; shift >= 11; --shift) {
    const int windows = 1 << (16 - shift), span = 1 << shift;
    std::vector<int> len(n_chunks + 1, 0);
    std::vector<int> bases((size_t)n_chunks * windows, 0);
    int fail = 0;
#pragma omp parallel
    {
      std::vector<int> cols;
#pragma omp for schedule(static) reduction(max : fail)
      for (int c = 0; c < n_chunks; ++c) {
        const int r0 = c * rows_per_chunk, r1 = std::min(a.n_rows, r0 + rows_per_chunk);
        int maxlen = 0;
        cols.clear();
        for (int i = r0; i < r1; ++i) {
          const int r = row_of(i);
          maxlen = std::max(maxlen, a.row_ptr[r + 1] - a.row_ptr[r]);
          cols.insert(cols.end(), a.col_idx.begin() + a.row_ptr[r], a.col_idx.begin() + a.row_ptr[r + 1]);
        }
        if (!chunk_windows(cols, span, windows, &bases[(size_t)c * windows])) fail = 1;
        const int groups = (maxlen + kPackGroup - 1) / kPackGroup;
        len[c + 1] = 32 * ((groups + tpr - 1) / tpr);
      }
    }
    if (fail) continue;
    // uniform chunks when padding every chunk to the longest costs <= 5% more entries
    long tot = 0;
    int smax = 0;
    for (int c = 0; c < n_chunks; ++c) {
      tot += len[c + 1];
      smax = std::max(smax, len[c + 1] / 32);
    }
    const bool uni = smax > 0 && (double)smax * 32 * n_chunks <= 1.05 * (double)tot;
    if (uni)
      for (int c = 0; c < n_chunks; ++c) len[c + 1] = 32 * smax;
    for (int c = 0; c < n_chunks; ++c) len[c + 1] += len[c];
    HostSellP s;
    s.uniform = uni ? smax : 0;
    s.tpr = tpr;
    s.n_rows = a.n_rows;
    s.n_chunks = n_chunks;
    s.shift = shift;
    s.windows = windows;
    s.chunk_ptr = std::move(len);
    s.bases = std::move(bases);
    s.perm = perm;
    s.words.assign(s.padded(), 0u);
#pragma omp parallel for schedule(static)
    for (int c = 0; c < n_chunks; ++c) {
      const int* wb = &s.bases[(size_t)c * windows];
      const int r0 = c * rows_per_chunk, r1 = std::min(a.n_rows, r0 + rows_per_chunk);
      for (int i = r0; i < r1; ++i) {
        const int q = i - r0, r = row_of(i);
        for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
          const int j = k - a.row_ptr[r], col = a.col_idx[k];
          // entry j of the (column-sorted) row goes to lane j % tpr, slot
          // (j / tpr) % 4 of step j / (4 tpr): one gather instruction of the
          // row's lanes reads tpr consecutive columns
          const int sub = j % tpr, rest = j / tpr, e = rest % kPackGroup, st = rest / kPackGroup;
          int w = windows - 1;  // windows ascend: the owner is the last base <= col
          while (w > 0 && wb[w] > col) --w;
          const long pos = 4L * (s.chunk_ptr[c] + 32L * st + q * tpr + sub) + e;
          const uint32_t code = ((uint32_t)w << shift) | (uint32_t)(col - wb[w]);
          s.words[pos] = ((uint32_t)to_bf16(a.values[k]) << 16) | code;
        }
      }
    }
    out = std::move(s);
    return true;
  }
  return false;
}


// SELL-SH (sell.hpp): upper slots only, lower slots read from the mirror row.
// Leaves s.sym false when the operator does not qualify (not square, more than
// 127 patterns, not 16 slots wide, more than kSymSlots upper slots in a
// pattern, or not bitwise symmetric).
void build_stencil_sym(const HostCsr& a, HostSellS& s) {
  const int n = a.n_rows, L = 8 * s.G;
  s.sym = false;
  if (a.n_cols != n || s.P > 127 || L != 16) return;
  std::vector<int> uslot((size_t)s.P * L, -1);
  for (int p = 0; p < s.P; ++p) {
    int nu = 0;
    for (int j = 0; j < s.plen[p]; ++j)
      if (s.pat[(size_t)p * L + j] >= 0) uslot[(size_t)p * L + j] = nu++;
    if (nu > kSymSlots) return;
  }
  // slot j' of pattern p holding offset `off` (upper slots only), -1 if none
  auto find_upper = [&](int p, int off) {
    for (int j = 0; j < s.plen[p]; ++j)
      if (s.pat[(size_t)p * L + j] == off) return uslot[(size_t)p * L + j];
    return -1;
  };
  const int cm = s.common;
  s.sinfo.assign((size_t)s.P * L, -1);
  std::vector<int> mirror_common((size_t)s.P * L, -1);
  for (int p = 0; p < s.P; ++p)
    for (int j = 0; j < s.plen[p]; ++j) {
      const int off = s.pat[(size_t)p * L + j];
      if (off >= 0) {
        s.sinfo[(size_t)p * L + j] = uslot[(size_t)p * L + j];
      } else {
        const int m = find_upper(cm, -off);
        mirror_common[(size_t)p * L + j] = m;
        s.sinfo[(size_t)p * L + j] = m >= 0 ? 8 + m : 16;
      }
    }
  std::vector<uint16_t> uv((size_t)s.n_chunks * kSymSlots * 32, 0);
  std::vector<double> uv64((size_t)s.n_chunks * kSymSlots * 32, 0.0);
  std::vector<uint8_t> spid(s.pid.size(), 0);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < n; ++r) {
    const int p = s.pid[r], c = r / 32, lane = r % 32;
    for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
      const int u = uslot[(size_t)p * L + (k - a.row_ptr[r])];
      if (u < 0) continue;
      const size_t at = ((size_t)c * kSymSlots + u) * 32 + lane;
      uv[at] = to_bf16(a.values[k]);
      uv64[at] = a.values[k];
    }
  }
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(max : bad)
  for (int r = 0; r < n; ++r) {
    const int p = s.pid[r];
    bool fast = true;
    for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
      const int j = k - a.row_ptr[r], off = s.pat[(size_t)p * L + j];
      if (off >= 0) continue;
      const int col = r + off, pc = s.pid[col];
      const int m = find_upper(pc, -off);
      if (m < 0) {
        bad = 1;
        continue;
      }
      const double mirror = uv64[((size_t)(col / 32) * kSymSlots + m) * 32 + col % 32];
      if (std::memcmp(&mirror, &a.values[k], sizeof(double)) != 0) bad = 1;  // not bitwise symmetric
      if (pc != cm || mirror_common[(size_t)p * L + j] < 0) fast = false;
    }
    spid[r] = (uint8_t)(p | (fast ? 0x80 : 0));
  }
  if (bad) {
    s.sinfo.clear();
    return;
  }
  s.slow_base.assign(s.n_chunks + 1, 0);
  for (int r = 0; r < n; ++r) s.slow_base[r / 32 + 1] += !(spid[r] & 0x80);
  for (int c = 0; c < s.n_chunks; ++c) s.slow_base[c + 1] += s.slow_base[c];
  s.slow_code.assign((size_t)s.slow_base[s.n_chunks] * 16, 0);
#pragma omp parallel for schedule(static)
  for (int c = 0; c < s.n_chunks; ++c) {
    long at = s.slow_base[c];
    for (int r = 32 * c; r < std::min(n, 32 * c + 32); ++r) {
      if (spid[r] & 0x80) continue;
      const int p = s.pid[r];
      for (int j = 0; j < s.plen[p]; ++j) {
        const int off = s.pat[(size_t)p * L + j];
        if (off < 0) s.slow_code[at * 16 + j] = (uint8_t)find_upper(s.pid[r + off], -off);
      }
      ++at;
    }
  }
  s.uvals = std::move(uv);
  s.uvals64 = std::move(uv64);
  s.spid = std::move(spid);
  s.sym = true;
}

bool build_sell_stencil(const HostCsr& a, HostSellS& out, bool with_fp64, bool with_sym) {
  const int n = a.n_rows;
  int lmax = 0;
  for (int r = 0; r < n; ++r) lmax = std::max(lmax, a.row_ptr[r + 1] - a.row_ptr[r]);
  const int L = std::max(8, (lmax + 7) / 8 * 8);
  if (L > 32 || n == 0) return false;
  // row signature hash (length + offsets), then ids in row order with an exact check
  std::vector<uint64_t> h(n);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < n; ++r) {
    uint64_t x = 1469598103934665603ull ^ (uint64_t)(a.row_ptr[r + 1] - a.row_ptr[r]);
    for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
      x ^= (uint64_t)(uint32_t)(a.col_idx[k] - r);
      x *= 1099511628211ull;
    }
    h[r] = x;
  }
  HostSellS s;
  s.n_rows = n;
  s.n_chunks = (n + 31) / 32;
  s.G = L / 8;
  s.pid.assign((size_t)s.n_chunks * 32, 0);
  std::vector<uint64_t> keys;
  std::vector<int> rep;  // representative row per pattern
  auto same = [&](int r, int q) {
    const int lr = a.row_ptr[r + 1] - a.row_ptr[r];
    if (lr != a.row_ptr[q + 1] - a.row_ptr[q]) return false;
    for (int k = 0; k < lr; ++k)
      if (a.col_idx[a.row_ptr[r] + k] - r != a.col_idx[a.row_ptr[q] + k] - q) return false;
    return true;
  };
  for (int r = 0; r < n; ++r) {
    int id = -1;
    if (r > 0 && keys[s.pid[r - 1]] == h[r] && same(r, rep[s.pid[r - 1]])) id = s.pid[r - 1];  // common case
    for (size_t p = 0; p < keys.size() && id < 0; ++p)
      if (keys[p] == h[r] && same(r, rep[p])) {
        id = (int)p;
        break;
      }
    if (id < 0) {
      if (keys.size() == 255) return false;
      id = (int)keys.size();
      keys.push_back(h[r]);
      rep.push_back(r);
    }
    s.pid[r] = (uint8_t)id;
  }
  s.P = (int)keys.size();
  {
    std::vector<long> freq(s.P, 0);
    for (int r = 0; r < n; ++r) ++freq[s.pid[r]];
    s.common = (int)(std::max_element(freq.begin(), freq.end()) - freq.begin());
  }
  s.pat.assign((size_t)s.P * L, 0);
  s.plen.assign(s.P, 0);
  for (int p = 0; p < s.P; ++p) {
    const int r = rep[p];
    s.plen[p] = a.row_ptr[r + 1] - a.row_ptr[r];
    for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) s.pat[(size_t)p * L + (k - a.row_ptr[r])] = a.col_idx[k] - r;
  }
  s.vals.assign((size_t)s.n_chunks * 32 * L, 0);
#pragma omp parallel for schedule(static)
  for (int r = 0; r < n; ++r) {
    const int c = r / 32, lane = r % 32;
    for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
      const int j = k - a.row_ptr[r];
      s.vals[(((size_t)c * s.G + j / 8) * 32 + lane) * 8 + j % 8] = to_bf16(a.values[k]);
    }
  }
  if (with_fp64) {
    s.vals64.assign((size_t)s.n_chunks * 32 * L, 0.0);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) {
      const int c = r / 32, lane = r % 32;
      for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k)
        s.vals64[((size_t)c * L + (k - a.row_ptr[r])) * 32 + lane] = a.values[k];
    }
  }
  if (with_sym) build_stencil_sym(a, s);
  out = std::move(s);
  return true;
}

}  // namespace eqsb
