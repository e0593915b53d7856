// Device-resident pieces of the SA-AMG setup (proj/src/amg.cpp:15-143,
// proj/src/csr.cpp:52-70,133-166), all bit-identical to the host/reference
// algorithm: Galerkin products (k_spgemm.cu) and the strength
// graph, greedy aggregation, tentative prolongator, lambda_max power
// iteration, transposition and diagonal check (k_amgsetup.cu).
#pragma once

#include <cuda_runtime.h>

#include "eqs_internal.hpp"
#include "gpu_system.hpp"

namespace eqsb {

struct DCsr {
  int rows = 0, cols = 0;
  long long nnz = 0;
  DevBuf<int> rp, ci;
  DevBuf<double> v;
};

class SpgemmDevice {
 public:
  SpgemmDevice() = default;
  ~SpgemmDevice();
  void init(int device);
  cudaStream_t stream() const { return s_; }
  void upload(const HostCsr& h, DCsr& d);
  void download(const DCsr& d, HostCsr& h);
  // C = A B (with diag: A replaced by I - omega D^-1 A on the fly)
  void multiply(const DCsr& a, const DCsr& b, DCsr& c, const double* diag_dev, double omega, long long batch);

 private:
  int device_ = -1;
  cudaStream_t s_ = nullptr;
};

struct DevAggStats {
  int rounds_pass1 = 0, rounds_pass2 = 0, roots = 0, pass2 = 0, pass3 = 0;
};

// d_i = a_ii (coeff(a, i, i); 0 when the row has no diagonal entry)
void dev_diagonal(const DCsr& a, DevBuf<double>& d, cudaStream_t s);
// proj/src/preconditioners.cpp:7-20 (throws NumericalError naming the first bad row)
void dev_check_diagonal(const DCsr& a, cudaStream_t s);
// proj/src/amg.cpp:15-26 + 49-88; returns the number of aggregates
int dev_aggregate(const DCsr& a, const double* d, double theta, DevBuf<int>& agg, cudaStream_t s,
                  DevAggStats* stats = nullptr);
// P_tent (amg.cpp:104-118): unit-normalised indicator columns
void dev_tentative(const DevBuf<int>& agg, int n, int n_agg, DCsr& pt, cudaStream_t s);
// proj/src/amg.cpp:28-45 (mt19937 start vector and Eigen-order norms on the host)
double dev_lambda_max(const DCsr& a, const double* d, int iters, unsigned seed, cudaStream_t s);
// proj/src/csr.cpp:52-70 (entries of each column in ascending row order)
void dev_transpose(const DCsr& a, DCsr& t, cudaStream_t s);

}  // namespace eqsb
