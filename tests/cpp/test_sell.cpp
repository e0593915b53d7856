// CPU check of the SELL-16 and packed SELL-P encoders (sell.hpp): every CSR
// entry is recovered bit-exactly (column) / as its bf16 rounding (value) by
// the same index arithmetic the kernels use (k_rows.cu sell_dot / sellp_dot),
// and padding decodes to value 0 at a valid column. Built and run by
// tests/test_sell_format.py.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <random>

#include "sell.hpp"

using namespace eqsb;

static float bf16_to_float(uint32_t hi) {
  float f;
  uint32_t u = hi & 0xffff0000u;
  std::memcpy(&f, &u, 4);
  return f;
}

static int check_packed(const HostCsr& a, const HostSellP& p) {
  const int rpc = 32 / p.tpr;
  const unsigned mask = (1u << p.shift) - 1u;
  std::vector<char> seen(a.nnz(), 0);
  for (int c = 0; c < p.n_chunks; ++c) {
    const int S = (p.chunk_ptr[c + 1] - p.chunk_ptr[c]) / 32;
    for (int lane = 0; lane < 32; ++lane) {
      const int q = lane / p.tpr, sub = lane % p.tpr, i = c * rpc + q;
      const int r = i < a.n_rows && !p.perm.empty() ? p.perm[i] : i;  // sorted rows (SELL-C-sigma)
      for (int st = 0; st < S; ++st)
        for (int e = 0; e < 4; ++e) {
          const uint32_t w = p.words[4L * (p.chunk_ptr[c] + 32L * st + lane) + e];
          const unsigned code = w & 0xffffu;
          const int col = p.bases[(size_t)c * p.windows + (code >> p.shift)] + (int)(code & mask);
          const int j = (st * 4 + e) * p.tpr + sub;  // entry index within the row
          if (r < a.n_rows && j < a.row_ptr[r + 1] - a.row_ptr[r]) {
            const long k = a.row_ptr[r] + j;
            if (col != a.col_idx[k]) return printf("col mismatch c%d lane%d st%d e%d\n", c, lane, st, e), 1;
            if (bf16_to_float(w) != bf16_to_float((uint32_t)to_bf16(a.values[k]) << 16)) return printf("val\n"), 1;
            seen[k] = 1;
          } else {
            if ((w >> 16) != 0) return printf("padding value nonzero\n"), 1;
            if (col < 0 || col >= a.n_cols) return printf("padding column out of range\n"), 1;
          }
        }
    }
  }
  for (char s : seen)
    if (!s) return printf("entry not encoded\n"), 1;
  return 0;
}

static int check_sell16(const HostCsr& a, const HostSell& h) {
  const int rpc = 32 / h.tpr;
  for (int c = 0; c < h.n_chunks; ++c) {
    const long beg = h.chunk_ptr[c];
    const int S = (int)((h.chunk_ptr[c + 1] - beg) >> 5);
    for (int lane = 0; lane < 32; ++lane)
      for (int s = 0; s < S; ++s) {
        const long pos = beg + 32L * s + lane;
        const unsigned code = h.code[pos];
        const int col = h.bases[(size_t)c * kSellWindows + (code >> kSellShift)] + (int)(code & (kSellSpan - 1));
        if (h.src[pos] >= 0 && col != a.col_idx[h.src[pos]]) return printf("sell16 col mismatch\n"), 1;
        const int r = c * rpc + lane / h.tpr;
        if (h.src[pos] >= 0 && (h.src[pos] < a.row_ptr[r] || h.src[pos] >= a.row_ptr[r + 1]))
          return printf("sell16 row mismatch\n"), 1;
      }
  }
  return 0;
}

// SELL-S: slot j of row r decodes to the row's j-th CSR entry (column row +
// pat[pid][j], bf16 value), padding slots to value 0 at column row
static int check_stencil(const HostCsr& a, const HostSellS& h) {
  const int L = 8 * h.G;
  int bad = 0;
  for (int r = 0; r < a.n_rows; ++r) {
    const int c = r / 32, lane = r % 32, len = a.row_ptr[r + 1] - a.row_ptr[r];
    for (int j = 0; j < L; ++j) {
      const uint16_t v = h.vals[(((size_t)c * h.G + j / 8) * 32 + lane) * 8 + j % 8];
      const int col = r + h.pat[(size_t)h.pid[r] * L + j];
      if (j < len) {
        const int k = a.row_ptr[r] + j;
        bad += col != a.col_idx[k] || v != to_bf16(a.values[k]);
      } else {
        bad += v != 0 || col != r;
      }
    }
  }
  return bad;
}

// SELL-SH: emulate the kernel's slot resolution (sym_dot in k_rows.cu): the
// common pattern's slot kinds for fast rows, the row's own pattern plus a
// search of the mirror row's pattern otherwise; every slot must decode to the
// row's CSR value (fp64 bitwise, bf16 rounded) and padding to 0
static int check_sym(const HostCsr& a, const HostSellS& h, long* fast_rows) {
  int bad = 0;
  long fast = 0;
  auto U64 = [&](int row, int u) { return h.uvals64[((size_t)(row / 32) * kSymSlots + u) * 32 + row % 32]; };
  auto U16 = [&](int row, int u) { return h.uvals[((size_t)(row / 32) * kSymSlots + u) * 32 + row % 32]; };
  long slow_rank = -1;
  for (int r = 0; r < a.n_rows; ++r) {
    const int pf = h.spid[r], p = pf & 127, len = a.row_ptr[r + 1] - a.row_ptr[r];
    const bool spec = p == h.common && (pf & 0x80);
    fast += spec;
    if (r % 32 == 0 && h.slow_base[r / 32] != slow_rank + 1) ++bad;
    if (!(pf & 0x80)) ++slow_rank;
    for (int j = 0; j < 16; ++j) {
      const int off = h.pat[(size_t)p * 16 + j], kind = h.sinfo[(size_t)(spec ? h.common : p) * 16 + j];
      double v64 = 0.0;
      uint16_t v16 = 0;
      if (kind >= 0 && kind < 8) {
        v64 = U64(r, kind);
        v16 = U16(r, kind);
      } else if (kind >= 8) {
        const int c = r + off;
        int u = -1;
        if (pf & 0x80) {
          u = kind - 8;  // every lower neighbour has the common pattern
        } else {         // slow-row table: rows without bit 7 in order (k_rows.cu sym_dot)
          u = h.slow_code[(size_t)slow_rank * 16 + j];
        }
        if (u < 0) {
          ++bad;
          continue;
        }
        v64 = U64(c, u);
        v16 = U16(c, u);
      }
      if (j < len) {
        const int k = a.row_ptr[r] + j;
        bad += std::memcmp(&v64, &a.values[k], 8) != 0 || v16 != to_bf16(a.values[k]) || r + off != a.col_idx[k];
      } else {
        bad += v64 != 0.0 || v16 != 0;
      }
    }
  }
  *fast_rows = fast;
  return bad;
}

// structured 15-point rows (Kuhn-box M_II-like): 3D grid with offsets
// (di, dj, dk) in {-1,0,1}^3 restricted to the 15 Kuhn-mesh neighbours
static HostCsr kuhn_like(int nx, int ny, int nz) {
  const int off[15][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0}, {0, 0, 1},  {0, 0, -1}, {1, 1, 0},
                          {-1, -1, 0}, {1, 0, 1},  {-1, 0, -1}, {0, 1, 1}, {0, -1, -1}, {1, 1, 1}, {-1, -1, -1}};
  HostCsr a;
  a.n_rows = a.n_cols = nx * ny * nz;
  a.row_ptr.push_back(0);
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        std::vector<int> cols;
        for (auto& o : off) {
          const int ii = i + o[0], jj = j + o[1], kk = k + o[2];
          if (ii >= 0 && ii < nx && jj >= 0 && jj < ny && kk >= 0 && kk < nz) cols.push_back((kk * ny + jj) * nx + ii);
        }
        std::sort(cols.begin(), cols.end());
        for (int col : cols) {
          a.col_idx.push_back(col);
          a.values.push_back(0.25 + 1e-3 * (col % 97) - (col == (int)a.row_ptr.size() - 1 ? 0.0 : 0.5));
        }
        a.row_ptr.push_back((int)a.col_idx.size());
      }
  return a;
}

int main() {
  std::mt19937 g(20261017u);
  int fails = 0;
  // row lengths: fine-level like (15), ragged, empty rows, long coarse rows;
  // column spread: local (one window) to wide (needs 16 or 32 windows)
  const int lens[] = {15, 40, 0, 200, 7};
  const int spreads[] = {3000, 30000, 60000, 120000};
  for (int li = 0; li < 5; ++li)
    for (int si = 0; si < 4; ++si) {
      HostCsr a;
      a.n_rows = 3000 + 97 * li + 13 * si;
      a.n_cols = 400000;
      a.row_ptr.push_back(0);
      for (int i = 0; i < a.n_rows; ++i) {
        const int len = lens[li] == 0 ? (i % 5 == 0 ? 0 : (int)(g() % 20)) : lens[li] - (int)(g() % 3);
        std::vector<int> cols;
        for (int k = 0; k < len; ++k) cols.push_back((i * 97 + (int)(g() % spreads[si])) % a.n_cols);
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        for (int col : cols) {
          a.col_idx.push_back(col);
          a.values.push_back(std::uniform_real_distribution<double>(-1.0, 1.0)(g));
        }
        a.row_ptr.push_back((int)a.col_idx.size());
      }
      const int tpr = choose_sell_tpr(a);
      HostSellP p;
      const bool okp = build_sell_packed(a, tpr, p);
      HostSell h;
      const bool ok16 = build_sell(a, tpr, h);
      const int fp = okp ? check_packed(a, p) : 0;
      const int f16 = ok16 ? check_sell16(a, h) : 0;
      printf("len %3d spread %6d tpr %2d packed %d (shift %d, uniform %d, padded %ld / nnz %ld) sell16 %d -> %s\n",
             lens[li], spreads[si], tpr, okp, p.shift, p.uniform, p.padded(), a.nnz(), ok16, fp || f16 ? "FAIL" : "ok");
      fails += fp + f16;
      if (okp && lens[li] == 15 && p.uniform != 4) ++fails, printf("fine-level-like rows should be uniform\n");
      if (okp && p.uniform && p.padded() != 128L * p.uniform * p.n_chunks) ++fails, printf("uniform size\n");
      if (!okp && spreads[si] <= 30000) ++fails, printf("packed encoding unexpectedly failed\n");
    }
  // rows of irregular length (transfer-operator-like): sorting within windows
  // of 256 rows (SELL-C-sigma) keeps every entry and cuts the padding
  {
    HostCsr a;
    a.n_rows = 5000;
    a.n_cols = 40000;
    a.row_ptr.push_back(0);
    for (int i = 0; i < a.n_rows; ++i) {
      const int len = 2 + (int)(g() % 11);
      std::vector<int> cols;
      for (int k = 0; k < len; ++k) cols.push_back(8 * i + (int)(g() % 64));
      std::sort(cols.begin(), cols.end());
      cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      for (int col : cols) {
        a.col_idx.push_back(col);
        a.values.push_back(0.5 + col % 5);
      }
      a.row_ptr.push_back((int)a.col_idx.size());
    }
    HostSellP p0, p1;
    const bool ok0 = build_sell_packed(a, 1, p0), ok1 = build_sell_packed(a, 1, p1, 256);
    int bad = !ok0 || !ok1 || p1.perm.size() != (size_t)a.n_rows;
    if (!bad) {
      std::vector<int> seen(a.n_rows, 0);
      for (int r : p1.perm) bad |= r < 0 || r >= a.n_rows || seen[r]++;
      for (int w0 = 0; w0 < a.n_rows && !bad; w0 += 256)  // a permutation within each window
        for (int i = w0; i < std::min(a.n_rows, w0 + 256); ++i) bad |= p1.perm[i] / 256 != w0 / 256;
      bad |= check_packed(a, p0) + check_packed(a, p1);
    }
    printf("irregular rows: padded %ld unsorted, %ld sorted (nnz %ld) -> %s\n", p0.padded(), p1.padded(), a.nnz(),
           bad || p1.padded() >= p0.padded() ? "FAIL" : "ok");
    fails += bad || p1.padded() >= p0.padded();
  }
  // clustered columns (restriction-like rows: a few node planes each): 12
  // clusters 20000 apart need 16 windows of 4096 (shift 12), 24 need 32 (shift 11)
  for (int nclus : {12, 24}) {
    HostCsr a;
    a.n_rows = 2000;
    a.n_cols = 600000;
    a.row_ptr.push_back(0);
    for (int i = 0; i < a.n_rows; ++i) {
      std::vector<int> cols;
      for (int cl = 0; cl < nclus; ++cl)
        for (int k = 0; k < 4; ++k) cols.push_back(cl * 20000 + (i / 8) * 4 + (int)(g() % 1000));
      std::sort(cols.begin(), cols.end());
      cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      for (int col : cols) {
        a.col_idx.push_back(col);
        a.values.push_back(1.0 + col % 7);
      }
      a.row_ptr.push_back((int)a.col_idx.size());
    }
    HostSellP p;
    const int tpr = choose_sell_tpr(a);
    const bool okp = build_sell_packed(a, tpr, p);
    const int want_shift = nclus == 12 ? 12 : 11;
    const int fp = okp ? check_packed(a, p) : 1;
    printf("clusters %d tpr %d packed %d shift %d -> %s\n", nclus, tpr, okp, p.shift,
           fp || p.shift != want_shift ? "FAIL" : "ok");
    fails += fp + (p.shift != want_shift);
  }
  // SELL-S on structured rows (27 patterns for a box interior + faces/edges/corners)
  {
    const HostCsr a = kuhn_like(13, 11, 9);
    HostSellS h;
    const bool ok = build_sell_stencil(a, h);
    const int fs = ok ? check_stencil(a, h) : 1;
    printf("stencil kuhn-like %d rows: ok %d patterns %d G %d -> %s\n", a.n_rows, ok, h.P, h.G,
           fs || h.P != 27 || h.G != 2 ? "FAIL" : "ok");
    fails += fs + (h.P != 27) + (h.G != 2);
  }
  // SELL-SH on symmetric structured rows; an asymmetric value set keeps the full copy
  for (int symmetric : {1, 0}) {
    HostCsr a = kuhn_like(13, 11, 9);
    for (int r = 0; r < a.n_rows; ++r)
      for (int k = a.row_ptr[r]; k < a.row_ptr[r + 1]; ++k) {
        const int c = a.col_idx[k], lo = std::min(r, c), hi = std::max(r, c);
        a.values[k] = (c == r ? 6.0 : -0.1) + 1e-3 * ((lo * 31 + hi * 7) % 101) + (symmetric ? 0.0 : 1e-9 * (r > c));
      }
    HostSellS h;
    const bool ok = build_sell_stencil(a, h, true, true);
    long fast = 0;
    const int fs = ok && h.sym ? check_sym(a, h, &fast) : 0;
    const bool pass = ok && (symmetric ? h.sym && fs == 0 && fast > a.n_rows / 4 : !h.sym);
    printf("stencil sym (symmetric %d): built %d sym %d fast rows %ld -> %s\n", symmetric, ok, (int)h.sym, fast,
           pass ? "ok" : "FAIL");
    fails += !pass;
  }
  {  // random columns: too many patterns -> no stencil copy
    HostCsr a;
    a.n_rows = a.n_cols = 5000;
    a.row_ptr.push_back(0);
    for (int i = 0; i < a.n_rows; ++i) {
      std::vector<int> cols = {i, (int)(g() % 5000), (int)(g() % 5000)};
      std::sort(cols.begin(), cols.end());
      cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
      for (int col : cols) {
        a.col_idx.push_back(col);
        a.values.push_back(1.0);
      }
      a.row_ptr.push_back((int)a.col_idx.size());
    }
    HostSellS h;
    const bool ok = build_sell_stencil(a, h);
    printf("stencil random rows: built %d -> %s\n", ok, ok ? "FAIL" : "ok");
    fails += ok;
  }
  return fails ? 1 : 0;
}
