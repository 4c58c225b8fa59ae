// dmma.cuh -- the FP64 orthonormalisation of the first sketch on the FP64 tensor cores (DMMA m8n8k4).
//
// Y0 = X Omega is conditioned like X itself (kappa ~ lambda_1 / lambda_w), so its Gram matrix
// (kappa^2) is formed and factored in FP64 (rnla.hpp:47-60 does the whole range finder in FP64):
//   Gram64Batch:  G = Y^T Y      from the FP32 sketch Y^T (w x d, rows contiguous), FP64 accumulation,
//                                upper tiles only + mirrored stores (G exactly symmetric), deterministic split-K
//   Tri64Batch:   Q^T = Linv Y^T  Linv lower triangular (FP64), K range cut at the tile's diagonal, FP64
//                                accumulation, FP32 result + its TF32 lo plane (the operands of the next X*Q)
// FP32 inputs are widened exactly when the fragments are loaded (shared memory keeps them in FP32).
#pragma once

#include <vector>

#include "common.cuh"

namespace rkfac_b200 {

struct Gram64Desc {
    int w, d;
    const float* T;    // w x d, pitch ldt (rows = sketch columns)
    long long ldt;
    double* G;         // w x w, pitch ldg
    long long ldg;
    int ksplit;
    int tiles_m;       // ceil(w / 64)
    int tile_offset;   // prefix over problems (CTAs)
    long long elem_offset;  // prefix of w*w over problems (reduction)
    double* partial;   // [ksplit][w][w] when ksplit > 1
};

class Gram64Batch {
  public:
    void add(int w, int d, const float* T, long long ldt, double* G, long long ldg);
    void finalize();
    void launch(cudaStream_t s) const;
    double flops() const;

  private:
    std::vector<Gram64Desc> descs_;
    DevBuf d_descs_, partials_;
    int total_tiles_ = 0;
    long long total_elems_ = 0;
    bool any_split_ = false;
};

struct Tri64Desc {
    int w, d;
    const double* L;   // w x w lower triangular (zeros above the diagonal), pitch ldl (multiple of 2)
    long long ldl;
    const float* Yt;   // w x d, pitch ldy
    long long ldy;
    float* Qt;         // w x d, pitch ldq
    float* Qtlo;       // TF32 lo plane of Qt (same pitch)
    long long ldq;
    int tiles_n;       // ceil(d / 64)
    int tile_offset;
};

class Tri64Batch {
  public:
    void add(int w, int d, const double* L, long long ldl, const float* Yt, long long ldy, float* Qt, float* Qtlo,
             long long ldq);
    void finalize();
    void launch(cudaStream_t s) const;

  private:
    std::vector<Tri64Desc> descs_;
    DevBuf d_descs_;
    int total_tiles_ = 0;
};

}  // namespace rkfac_b200
