// Sliced-ELL copy of a CSR operator with packed 16-bit column indices
// (DESIGN.md §3 "SELL-16"). The fine-level operators are read 5-6 times per
// PCG iteration and their 32-bit column indices are half of every V-cycle
// pass, so the resident format trades them for 16-bit codes:
//   - a chunk is the 32/tpr consecutive rows one warp processes (tpr lanes per
//     row); its rows are padded to the chunk's longest row (rounded up to tpr)
//     and stored slice-major, so every warp load reads 32 consecutive entries;
//   - the chunk's columns are covered by at most kSellWindows windows of
//     kSellSpan columns starting at `bases`; an entry stores
//     (window << kSellShift) | (column - base);
//   - padding entries hold code 0 (column = bases[0], a valid column) and value 0.
// A matrix that has a chunk needing more windows keeps the plain CSR kernels.
#pragma once

#include <cstdint>
#include <vector>

#include "eqs_internal.hpp"

namespace eqsb {

constexpr int kSellWindows = 8;
constexpr int kSellShift = 13;
constexpr int kSellSpan = 1 << kSellShift;

struct HostSell {
  int tpr = 0, n_rows = 0, n_chunks = 0;
  std::vector<long> chunk_ptr;   // [n_chunks + 1] entry offsets (multiples of 32)
  std::vector<int> bases;        // [n_chunks][kSellWindows]
  std::vector<uint16_t> code;    // packed column per entry
  std::vector<long> src;         // CSR entry of every position (-1: padding)
  long padded() const { return chunk_ptr.empty() ? 0 : chunk_ptr.back(); }
};

// lanes per row: each lane handles about `per_lane` entries of the mean row
int choose_sell_tpr(const HostCsr& a, int per_lane = 16);
// false (and `out` untouched) when some chunk's columns need more than kSellWindows windows
bool build_sell(const HostCsr& a, int tpr, HostSell& out);
// values in SELL order (padding 0), as T
template <class T>
std::vector<T> sell_values(const HostSell& s, const std::vector<double>& v) {
  std::vector<T> out(s.src.size());
#pragma omp parallel for schedule(static)
  for (long k = 0; k < (long)s.src.size(); ++k) out[k] = s.src[k] >= 0 ? (T)v[s.src[k]] : (T)0.0;
  return out;
}

}  // namespace eqsb

namespace eqsb {

// Packed SELL ("SELL-P") for the bf16 V-cycle operators: one
// 32-bit word per entry, bf16 value in the high half and the 16-bit column
// code in the low half. Four consecutive entries of a row form a 16-byte
// group, so each lane reads a whole group with one vector load and a warp
// load instruction moves 512 contiguous bytes (SELL-16 moves 64). Entry j of
// row q of a chunk sits in lane q * tpr + j % tpr, slot (j / tpr) % 4 of step
// j / (4 tpr), so the tpr lanes of a row gather consecutive columns; a chunk
// is `steps` x 32 groups. The column code is (window << shift) | (column - base)
// with shift 13, 12 or 11 (8, 16 or 32 windows per chunk, the first that fits).
constexpr int kPackGroup = 4;

struct HostSellP {
  int tpr = 0, n_rows = 0, n_chunks = 0, shift = 13, windows = 8;
  int uniform = 0;  // > 0: every chunk has this many steps (chunk c starts at c * uniform * 32):
                    // the kernels skip the chunk-pointer load (one dependent round trip less)
  std::vector<int> chunk_ptr;    // [n_chunks + 1] offsets in 16-byte groups (multiples of 32)
  std::vector<int> bases;        // [n_chunks][windows]
  std::vector<uint32_t> words;   // 4 * chunk_ptr.back() packed entries (padding: 0)
  // row sorting (SELL-C-sigma): slot row i of the chunks holds matrix row
  // perm[i]; rows are sorted by length (descending, stable) within windows of
  // sigma rows, so a chunk's rows have similar lengths and little padding.
  // Empty: identity. The kernels read and write the epilogue rows at perm[i].
  std::vector<int> perm;
  long padded() const { return chunk_ptr.empty() ? 0 : 4L * chunk_ptr.back(); }
};

// Stencil-coded SELL ("SELL-S") for operators whose rows share a few
// column-offset lists (the fine level of structured meshes): pattern table
// [P][L] of offsets col - row (P <= 255, L = 8 G <= 32 slots, padding offset
// 0 with value 0), one pattern id per row and only the bf16 values, row r
// (chunk c = r / 32, lane r % 32) slot j at ((c G + j / 8) 32 + lane) 8 + j % 8:
// one 16-byte load gives a lane 8 values. Entries keep the CSR (column) order,
// so a TPR-1 SELL-P pass and a SELL-S pass sum the same products in the same
// order. 2 B per entry + 1 B per row instead of 4 B per entry.
struct HostSellS {
  int n_rows = 0, n_chunks = 0, G = 0, P = 0;
  int common = 0;               // most frequent pattern (the kernels gather its columns speculatively)
  std::vector<uint16_t> vals;   // [n_chunks][G][32][8]
  std::vector<double> vals64;   // [n_chunks][8 G][32] fp64 values (the PCG operator), slot-major per chunk
  std::vector<uint8_t> pid;     // [n_chunks * 32]
  std::vector<int> pat;         // [P][8 G]
  std::vector<int> plen;        // [P] entries per pattern (slots >= plen are padding)
  // Symmetric half storage ("SELL-SH"), built when the operator
  // is square, bitwise symmetric, 16 slots wide and has <= 127 patterns: a row
  // stores only its upper slots (offset >= 0, at most kSymSlots) and reads the
  // value of a lower slot (column c = row + offset < row) from row c's upper
  // slot for -offset, i.e. from data streamed shortly before (L2). Products
  // are still summed in CSR order, so a pass is bit-identical to the full
  // stencil-coded pass.
  bool sym = false;
  std::vector<uint16_t> uvals;  // [n_chunks][kSymSlots][32] bf16 upper values (slot-major)
  std::vector<double> uvals64;  // [n_chunks][kSymSlots][32] fp64 upper values
  std::vector<uint8_t> spid;    // [n_chunks * 32] pattern id | 0x80 when every lower slot's row has the
                                // common pattern and the common pattern holds the mirror slot
  std::vector<int> sinfo;       // [P][16] slot kind: u (0..7) own upper slot u; 8 + m lower slot whose
                                // mirror is upper slot m of the common pattern; 16 lower slot without
                                // such a mirror; -1 padding
  // rows without bit 0x80 ("slow" rows, next to faces/edges): the mirror
  // upper slot of each lower slot, 16 bytes per row, rows in order;
  // slow_base[c] = slow rows before chunk c (a lane finds its row by a ballot)
  std::vector<uint8_t> slow_code;  // [n_slow][16]
  std::vector<int> slow_base;      // [n_chunks + 1]
};
constexpr int kSymSlots = 8;
// false when the rows need more than 255 patterns or more than 32 slots
bool build_sell_stencil(const HostCsr& a, HostSellS& out, bool with_fp64 = false, bool with_sym = false);

uint16_t to_bf16(double d);  // round to nearest even
// lanes per row of the packed format: about 32 entries per lane (fewer
// shuffle-reduction steps and more loads in flight per lane on coarse levels)
int choose_sellp_tpr(const HostCsr& a);
// false when some chunk's columns need more than 32 windows; sigma > 0 sorts
// the rows by length within windows of sigma rows (HostSellP::perm)
bool build_sell_packed(const HostCsr& a, int tpr, HostSellP& out, int sigma = 0);

}  // namespace eqsb
