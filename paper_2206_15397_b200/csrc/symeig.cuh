// symeig.cuh -- full symmetric eigendecomposition on the GPU, FP64 (see symeig.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace rkfac_b200 {

// Grouped FP64 GEMM: C = alpha * A B + beta * C with A(i, k) = A[i*rsA + k*csA], B(k, j) = B[k*rsB + j*csB],
// C(i, j) = C[i*ldc + j] (transposes by strides).
struct DGemmDesc {
    int M, N, K;
    const double* A; long long rsA, csA;
    const double* B; long long rsB, csB;
    double* C; long long ldc;
    double alpha, beta;
    int tiles_n, tile_off;
    int ksplit = 1, kchunk = 0;  // split-K (single-problem launches with few tiles): partial sums + reduction
    double* partial = nullptr;
};

class DGemmBatch {
  public:
    void clear() { descs_.clear(); tiles_ = 0; }
    void add(DGemmDesc d);
    void launch(cudaStream_t s);  // uploads the descriptors (async from pinned staging) and launches
    bool empty() const { return descs_.empty(); }

  private:
    std::vector<DGemmDesc> descs_;
    int tiles_ = 0;
    DevBuf d_, part_;
    size_t cap_ = 0;
};

// eig.hpp:210-237 sym_eig on a device matrix: S (n x n FP32, pitch lds) -> eigenvalues descending (dvals, n FP32;
// dvals64 optional FP64 copy) and eigenvectors as the COLUMNS of P (n x n FP32, pitch ldp; P may be null).
class SymEig {
  public:
    // Returns the max asymmetry |S - S^T| / max(1, |S|max) found (the caller decides whether to reject).
    double run(const float* S, long long lds, int n, float* P, long long ldp, float* dvals, double* dvals64,
               cudaStream_t s);

  private:
    void reserve(int n);
    void tridiagonalize(cudaStream_t s);
    void divide_and_conquer(cudaStream_t s, bool vectors);
    void back_transform(cudaStream_t s);
    int n_ = 0, cap_n_ = 0;
    long long ld_ = 0;
    DevBuf A_, V_, W_, tau_, dv_, ev_, part_, vbuf_, ybuf_, QT_, QgT_, UT_, ws_, meta_, stat_;
    DGemmBatch gemm_;
};

}  // namespace rkfac_b200
