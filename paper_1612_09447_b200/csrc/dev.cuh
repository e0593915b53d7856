// Device-side helpers and kernel launcher declarations (sm_100a, fp64 CUDA
// cores; no tensor cores — the path is sparse and HBM-bound).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace eqsb {

constexpr int kBlock = 256;

// number of kernels this library has launched (bench.py's gpu_launches)
extern long g_launch_count;
// algorithmic HBM bytes of the sparse row kernels launched so far (roofline accounting)
extern double g_algo_bytes;
// programmatic dependent launch on for the row/vector kernels (eqs_set_option 21)
extern bool g_pdl;
// Reduction kernels run grid-stride on a fixed grid so that the partial-sum
// count (and therefore the summation order) is fixed: deterministic results.
constexpr int kRedGrid = 148 * 8;

// device scalar slots (double) used by the fused PCG / RKC kernels
enum Slot : int {
  S_PQ = 0,   // p.q
  S_RR,       // r.r
  S_RZ,       // r.z (current)
  S_RZ_OLD,   // r.z (previous iteration)
  S_BB,       // b.b
  S_X0X0,     // x0.x0
  S_DOT,      // generic dot
  S_ERR,      // RKC weighted error sum
  S_NORM,     // generic norm^2
  S_MDOT,     // first of kMaxMulti multi-dot slots
  kMaxMulti = 16,
  // SPE append (one host read per append): |h|^2, |w|^2 after each
  // Gram-Schmidt pass, the two passes' coefficients, the new G column
  S_APP = S_MDOT + kMaxMulti,
  S_APP_NRM = S_APP + 1,
  S_APP_C = S_APP + 3,
  S_APP_G = S_APP_C + 2 * kMaxMulti,
  S_COUNT = S_APP_G + kMaxMulti
};

struct Reducer {
  double* partials;   // [S_COUNT][kRedGrid]
  unsigned* counters; // [S_COUNT]
  double* scal;       // [S_COUNT] results
};

// Sliced-ELL copy with packed 16-bit columns (sell.hpp); tpr == 0: absent.
struct DevSell {
  int tpr = 0, n_chunks = 0;
  long padded = 0;                   // stored entries (nnz + padding)
  const long* chunk_ptr = nullptr;   // [n_chunks + 1]
  const int* bases = nullptr;        // [n_chunks][8]
  const uint16_t* code = nullptr;    // (window << 13) | (column - base)
  const double* v64 = nullptr;
  const float* v32 = nullptr;
  const uint16_t* v16 = nullptr;     // bf16 bit patterns
};

// Packed SELL copy (sell.hpp "SELL-P"): bf16 value | 16-bit column code per
// 32-bit word, 16-byte groups; tpr == 0: absent.
struct DevSellP {
  int tpr = 0, n_chunks = 0, shift = 13, windows = 8;
  int uniform = 0;                  // > 0: steps of every chunk (no chunk-pointer load)
  long padded = 0;                  // stored entries (nnz + padding)
  const int* chunk_ptr = nullptr;   // [n_chunks + 1] in 16-byte groups
  const int* bases = nullptr;       // [n_chunks][windows]
  const uint4* words = nullptr;
  const int* perm = nullptr;        // [n_rows] slot row -> matrix row (sell.hpp HostSellP::perm) or null
};

// Stencil-coded SELL (sell.hpp HostSellS): per row a pattern id, per entry the
// bf16 value; column = row + pat[pid][slot]
struct DevSellS {
  int n_chunks = 0, G = 0, P = 0, common = 0;
  int n_cols = 0;                        // length of the gathered vectors (speculative gathers are clamped to it)
  const uint4* vals = nullptr;           // [n_chunks][G][32] x 8 bf16
  const unsigned char* pid = nullptr;    // [n_chunks * 32]
  const int* pat = nullptr;              // [P][8 G]
  int coff[16] = {};                     // G = 2: offsets of the common pattern (kernel parameters)
  int stage = 1;                         // G = 2: 1 = pattern table staged in shared memory, 0 = parameters + L1
  const double* vals64 = nullptr;        // [n_chunks][8 G][32] fp64 values (PCG operator) or null
  // symmetric half storage (sell.hpp SELL-SH); used instead of vals/vals64 when sym
  bool sym = false;
  const uint16_t* u16 = nullptr;         // [n_chunks][8][32] bf16 upper values
  const double* u64 = nullptr;           // [n_chunks][8][32] fp64 upper values
  const unsigned char* spid = nullptr;   // [n_chunks * 32] pattern | 0x80 (fast row)
  const int* sinfo = nullptr;            // [P][16] slot kinds
  const uint4* slow_code = nullptr;      // [n_slow] 16 mirror slots of each slow row
  const int* slow_base = nullptr;        // [n_chunks + 1] slow rows before each chunk
};

// CSR matrix resident in HBM (int32 indices, fp64 values, sorted columns),
// optionally with reduced-precision value copies and a SELL copy that the
// kernels use instead when `use_sell` is set.
struct DevCsr {
  int n_rows = 0, n_cols = 0;
  long nnz = 0;
  int* row_ptr = nullptr;
  int* col_idx = nullptr;
  double* values = nullptr;
  float* values_f = nullptr;  // fp32 copy (V-cycle operators only)
  int tpr = 4;                // threads per row used by the CSR kernels
  int prec = 0;               // values read by the kernels: 0 fp64, 1 fp32, 2 bf16 (SELL only; CSR reads fp32)
  bool use_sell = false;
  DevSell sell;
  DevSellP pk;  // used instead of `sell` for bf16 values (prec 2) when present
  DevSellS st;  // used instead of `pk` when present and use_stencil (fine level, structured meshes)
  bool use_stencil = true;
  bool packed() const { return use_sell && prec == 2 && pk.tpr > 0; }
  bool stencil() const { return use_sell && prec == 2 && use_stencil && st.G > 0; }
  bool stencil64() const { return use_sell && prec == 0 && use_stencil && st.vals64 != nullptr; }
  bool sell16() const { return use_sell && sell.tpr > 0 && !packed(); }
  int lanes() const { return packed() ? pk.tpr : sell16() ? sell.tpr : tpr; }
};

struct ChebCoef {
  double c0, c1, inv_theta;
};

// Material table in constant memory (kappa_of_e, proj/src/materials.cpp:25-33)
struct DevMaterial {
  int kind;         // 0 constant, 1 microvaristor
  double kappa;     // constant
  double lo, hi;    // log10(kappa_lo), log10(kappa_hi) hoisted per material
  double e_switch, inv_width;
};
constexpr int kMaxMaterials = 64;

// ---- stiffness (k_stiffness.cu)
void set_materials(const DevMaterial* mats, int n, cudaStream_t s);
// pass 1: per-tet local products (ytet[t][n_local]); x_state and v in device
// dof numbering; coords [n_dofs][4] (x, y, z, pad)
void launch_kx_tets(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                    const double* x_state, const double* v, double* ytet, int* geo_error, cudaStream_t s);
// pass 2: out[d] = base[d] + sign * sum over incident slots (ascending tet)
void launch_kx_gather(int n_rows, const long* slot_ptr, const int* slots, const double* ytet, const double* base,
                      double sign, double* out, cudaStream_t s);
// blocked single pass + boundary partials (kxblock.hpp): out[d] = base[d] +
// sign * (K(x) v)[d] for d < n_out (base may be null)
struct KxDev {
  int nl = 4, n_blocks = 0, max_block_tets = 0, max_block_dofs = 0, max_block_slots = 0, n_bdof = 0;
  const int* blk_tet0 = nullptr;
  const int* tets = nullptr;           // blocked order: P1 ushort4 block-local dof ids, P2 [tets][10] dof ids
  const int* ldof_dof = nullptr;       // dof of every block-dof entry
  const unsigned char* mat = nullptr;  // blocked order
  const int* blk_dof0 = nullptr;
  const int* sptr = nullptr;
  const uint16_t* slots = nullptr;
  const int* lout = nullptr;
  double* partials = nullptr;
  const int *bdof = nullptr, *bptr = nullptr, *bpart = nullptr;
  const double *bxy = nullptr, *bz = nullptr;  // P1: coordinates per block-dof entry ({x, y} pairs, z)
};
void launch_kx_blocked(const KxDev& k, const double* coords, const double* x_state, const double* v,
                       const double* base, double sign, int n_out, double* out, int* geo_error, cudaStream_t s);
// coloured single pass: y[dof] += local product for one colour batch
void launch_kx_colored(int order, int n_batch, const int* batch_tets, const int* tet_dofs,
                       const unsigned char* tet_mat, const double* coords, const double* x_state, const double* v,
                       double* y, int* geo_error, cudaStream_t s);

// ---- matrix row kernels (k_rows.cu). XT is the vector type: fp64 for the PCG
// operator, fp32 or fp64 for the V-cycle; matrix values per
// DevCsr::prec. Every launcher adds its algorithmic bytes to g_algo_bytes.
// algorithmic bytes of one pass over `a` (resident format) with `gathered`
// column vectors and `streamed` row vectors of `xbytes` each
double matrix_pass_bytes(const DevCsr& a, int gathered, int streamed, int xbytes = 8);
// Row-sum correction of the stencil-coded bf16 V-cycle operator (DESIGN.md
// §4.12): writes sum_k (a_k - bf16(a_k)) of each row (from the fp64 copy) as
// bf16 into the row's first padded slot (column offset 0, the diagonal), or 0
// when on = false. vals is the mutable [n_chunks][G][32] x 8 bf16 array of m.
void launch_sells_rowsum(int n_rows, const DevSellS& m, uint16_t* vals, bool on, cudaStream_t s);

template <class XT>
void launch_spmv(const DevCsr& a, const XT* x, XT* y, cudaStream_t s);
// y = b - A x, and (if red) ||y||^2 into slot
template <class XT>
void launch_residual(const DevCsr& a, const XT* b, const XT* x, XT* y, Reducer* red, int slot, cudaStream_t s);
// q = A p ; slot <- p.q
void launch_spmv_dot(const DevCsr& a, const double* p, double* q, Reducer red, int slot, cudaStream_t s);
// y = b - A x and y2 = D^-1 y ; y = A x and y2 = W y (restriction with the
// next level's D^-1): the scaled copies are the `pre` inputs below
template <class XT>
void launch_residual_scaled(const DevCsr& a, const XT* b, const XT* x, const XT* invd, XT* y, XT* y2, cudaStream_t s);
template <class XT>
void launch_spmv_scaled(const DevCsr& a, const XT* x, const XT* w, XT* y, XT* y2, cudaStream_t s);
// Chebyshev(2) smoother pieces. `pre` (optional) = D^-1 of the
// vector the op scales (b for the pre-smoother, r0 for the post step): the
// packed kernels then gather it instead of the vector and D^-1.
template <class XT>
void launch_cheb_pre(const DevCsr& a, const XT* invd, const XT* b, XT* z, ChebCoef c, cudaStream_t s,
                     const XT* pre = nullptr);
template <class XT>
void launch_cheb_post2(const DevCsr& a, const XT* invd, const XT* r0, XT* z, ChebCoef c, const XT* b_dot,
                       Reducer* red, int slot, cudaStream_t s, const XT* pre = nullptr);
// fp32 V-cycle, fine level: z_out (fp64) = z + Chebyshev(2) post step ; slot <- b64.z_out
void launch_cheb_post2_out64(const DevCsr& a, const float* invd, const float* r0, const float* z, ChebCoef c,
                             double* z_out, const double* b_dot, Reducer* red, int slot, cudaStream_t s,
                             const float* pre = nullptr);
// Chebyshev(1): z = D^-1 b / theta and t = b - A z in one pass
template <class XT>
void launch_cheb1_pre_resid(const DevCsr& a, const XT* invd, const XT* b, XT* z, XT* t, ChebCoef c, cudaStream_t s,
                            const XT* pre = nullptr);
// Chebyshev(1) post: z_out = z + D^-1 (b - A z) / theta (z_out != z)
template <class XT>
void launch_cheb1_post(const DevCsr& a, const XT* invd, const XT* b, const XT* z, XT* z_out, ChebCoef c,
                       cudaStream_t s);
// z += P zc
template <class XT>
void launch_prolong_add(const DevCsr& p, const XT* zc, XT* z, cudaStream_t s);
// w = invd .* (A v)   (power iteration on D^-1 A for the smoother bounds)
void launch_scaled_spmv(const DevCsr& a, const double* invd, const double* v, double* w, cudaStream_t s);

// ---- PCG / dense (k_sparse.cu)
// x += alpha p (skipped for x == nullptr) ; r -= alpha q ; slot_rr <- r.r ; alpha = scal[S_RZ]/scal[S_PQ];
// r32 (optional) = (float) r
// and d32 = invd32 .* r32 (the next fp32 V-cycle's inputs)
void launch_pcg_update(int n, double* x, double* r, const double* p, const double* q, Reducer red, cudaStream_t s,
                       float* r32 = nullptr, const float* invd32 = nullptr, float* d32 = nullptr);
// w -= sum_j dcoef[j] Q_j ; slot <- w.w   (coefficients read from device memory)
void launch_orth_update_dev(int n, int m, const double* const* Q, const double* dcoef, double* w, Reducer red,
                            int slot, cudaStream_t s);
// y = x / sqrt(*nrm2)  (device-resident norm^2)
void launch_scale_rsqrt(int n, const double* nrm2, const double* x, double* y, cudaStream_t s);
// p = z + beta p, beta = scal[S_RZ]/scal[S_RZ_OLD]; p = z when stat && stat[0] == 0;
// x (optional): first x += (scal[S_RZ_OLD]/scal[S_PQ]) p, the update deferred from
// the previous iteration (launch_pcg_update with x == nullptr)
void launch_pcg_direction(int n, double* p, const double* z, const double* scal, cudaStream_t s,
                          const double* stat = nullptr, double* x = nullptr);
// x += (scal[S_RZ]/scal[S_PQ]) p: the deferred update of the last iteration
void launch_pcg_xfinal(int n, double* x, const double* p, const double* scal, cudaStream_t s);
// Device-side PCG stopping rule (pcg.cpp:40-66) for the graph-resident
// iteration loop. stat = [k, status, rel, pq, bnorm, tol, max_iter, rr0 (< 0:
// read S_RR), initial rel]: advances
// k, sets status 0 continue / 1 converged / 2 rz non-finite / 3 p'Ap <= 0 or
// non-finite / 4 rel non-finite / 5 max_iter reached, copies r.z to S_RZ_OLD
// when continuing and sets the loop's conditional handle to (status == 0).
enum PcgStatus : int {
  PCG_CONTINUE = 0, PCG_CONVERGED, PCG_BAD_RZ, PCG_BAD_PQ, PCG_BAD_REL, PCG_MAX_ITER, PCG_BAD_INIT
};
void launch_pcg_check(double* scal, double* stat, cudaGraphConditionalHandle h, cudaStream_t s);
// initial residual test (status PCG_BAD_INIT / PCG_CONVERGED / PCG_CONTINUE), sets the loop condition
void launch_pcg_check0(double* scal, double* stat, cudaGraphConditionalHandle h, cudaStream_t s);
// z = Ainv b (dense, n <= 1024, fp64 inverse)
template <class XT>
void launch_dense_solve(int n, const double* ainv, const float* ainv32, const XT* b, XT* z, cudaStream_t s);
// Jacobi: z = invd .* r (+ dot r.z into slot when red)
void launch_jacobi(int n, const double* invd, const double* r, double* z, Reducer* red, int slot, cudaStream_t s);
// precision conversions at the fp32 V-cycle boundary
void launch_to_f32(long n, const double* x, float* y, cudaStream_t s);
// y = (float) x and d = invd .* y (the fine level's b and D^-1 b of an fp32 V-cycle)
void launch_to_f32_scaled(long n, const double* x, const float* invd, float* y, float* d, cudaStream_t s);
void launch_to_f64_dot(int n, const float* z32, double* z64, const double* b, Reducer* red, int slot, cudaStream_t s);

// ---- vector kernels (k_sparse.cu)
void launch_dot(int n, const double* a, const double* b, Reducer red, int slot, cudaStream_t s);
// slot+k <- V_k . w for k < m (V column-major with leading dim ld)
void launch_multi_dot(int n, int m, const double* const* V, const double* w, Reducer red, int slot0, cudaStream_t s);
void launch_axpy(int n, double a, const double* x, double* y, cudaStream_t s);            // y += a x
void launch_scale(int n, double a, const double* x, double* y, cudaStream_t s);           // y = a x
template <class XT>
void launch_diag_scale(int n, const XT* invd, const XT* b, double a, XT* z, cudaStream_t s);  // z = a D^-1 b
void launch_axpy_dev(int n, const double* coef, double sign, const double* x, double* y, cudaStream_t s);  // y += sign*(*coef) x
// y = sum_k c[k] V_k  (coefficients by value)
struct CoefPack {
  double c[kMaxMulti];
};
void launch_lincomb(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s);
// per-cell kappa (VTK dump)
void launch_cell_kappa(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                       const double* x_full, double* kappa, cudaStream_t s);
// SDIRK Newton matrix (k_sparse.cu / k_stiffness.cu)
void launch_k_element(int order, int n_tets, const int* tet_dofs, const unsigned char* tet_mat, const double* coords,
                      const double* x_full, double* S, int* geo_error, cudaStream_t s);
void launch_shift_gather(long nnz, const long* ptr, const long* src, const double* S, const double* m, double gdt,
                         double* shifted, cudaStream_t s);
void launch_csr_diag(int n, const int* rp, const int* ci, const double* v, double* d, cudaStream_t s);
void launch_recip(int n, const double* d, double* inv, cudaStream_t s);  // inv = 1 / d

void launch_jacobi_div(int n, const double* d, const double* r, double* z, Reducer red, int slot, cudaStream_t s);
void launch_weighted_sq(int n, const double* est, const double* x, const double* xn, double atol, double rtol,
                        Reducer red, int slot, cudaStream_t s);
// y += sum_k c[k] V_k
void launch_lincomb_acc(int n, int m, const double* const* V, CoefPack c, double* y, cudaStream_t s);
// SPE basis maintenance: w -= sum_j c_j Q_j with ||w||^2 into slot; and a
// kin -> kout basis rotation out_j = sum_i T[i][j] in_i (kin, kout <= 9)
constexpr int kMaxWin = 9;
struct RotPack {
  double t[kMaxWin][kMaxWin];
};
void launch_orth_update(int n, int m, const double* const* Q, CoefPack c, double* w, Reducer red, int slot,
                        cudaStream_t s);
void launch_lincomb_multi(int n, int kin, int kout, const double* const* in, double* const* out, const RotPack& T,
                          cudaStream_t s);
// w = invd .* (A v)   (power iteration on D^-1 A for the smoother bounds)
void launch_scaled_spmv(const DevCsr& a, const double* invd, const double* v, double* w, cudaStream_t s);
void launch_fill(long n, double v, double* y, cudaStream_t s);
// RKC stage (proj/src/integrators.cpp:167-168): y = a0 y0 + mu y1 + nu y2 + mt f + gt f0
void launch_rkc_stage(int n, double a0, double mu, double nu, double mt, double gt, const double* y0,
                      const double* y1, const double* y2, const double* f, const double* f0, double* y,
                      cudaStream_t s);
// y = y0 + c f
void launch_axpby_into(int n, const double* y0, double c, const double* f, double* y, cudaStream_t s);
// RKC error estimate + weighted RMS sum (integrators.cpp:20-31,201-202)
void launch_rkc_error(int n, const double* x, const double* xn, const double* f0, const double* fn, double dt,
                      double atol, double rtol, Reducer red, int slot, cudaStream_t s);
// permutations: y[i] = x[idx[i]] / y[idx[i]] = x[i]
void launch_gather(int n, const int* idx, const double* x, double* y, cudaStream_t s);
void launch_gather_f(int n, const int* idx, const float* x, float* y, cudaStream_t s);
void launch_scatter(int n, const int* idx, const double* x, double* y, cudaStream_t s);
// per-boundary-set scalars passed by value (no H2D copy per stage)
constexpr int kMaxSets = 16;
struct SetVals {
  double v[kMaxSets];
};
// boundary lift: full[n_free + i] = set_vals[set_of_fixed[i]]
void launch_lift_fixed(int n_fixed, const int* set_of_fixed, SetVals vals, double* fixed_part, cudaStream_t s);
// r[row_k] -= sum_s coef[k][s] * rate[s]  (compressed M_IB xdot_B, fem_system.cpp:65)
void launch_boundary_load(int n_rows, const int* rows, const double* coef, int n_sets, SetVals rates, double* r,
                          cudaStream_t s);

}  // namespace eqsb
