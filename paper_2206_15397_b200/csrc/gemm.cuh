// gemm.cuh -- grouped ("batched over factors/layers") dense GEMM with fused epilogues.
//
// One launch covers every problem of a stage (all factors, or all layers): the tile space of all problems is
// flattened and each CTA finds its problem by binary search over the prefix table.  Descriptors live in device
// memory and are built once per plan, so every stage launch is pointer-free and graph-capturable.
//
// C(m,n) = alpha * rs[m] * cs[n] * sum_k A(m,k) B(k,n)  + beta * Cin(m,n) + gamma * D(m,n)
//   A(m,k) = ta ? A[k*lda + m] : A[m*lda + k]       (ta=1: A stored K x M)
//   B(k,n) = tb ? B[n*ldb + k] : B[k*ldb + n]       (tb=1: B stored N x K)
//   C(m,n) -> tc ? C[n*ldc + m] : C[m*ldc + n]      (same for Cin, D)
// sym=1 (M==N): only tiles with tile_m <= tile_n are computed; off-diagonal tiles store both (m,n) and (n,m),
// which keeps EA factors exactly symmetric (kfactor.hpp:39 symmetrize_in_place) at half the flops.
// ksplit>1: deterministic split-K -- each K slice writes raw partials, a second kernel sums the slices in fixed
// order and applies the epilogue (results do not depend on how many problems share the launch).
#pragma once

#include <vector>

#include "common.cuh"

namespace rkfac_b200 {

enum class GemmKind : int {
    F32 = 0,        // float x float -> float, float accumulate
    F32_ACC64 = 1,  // float x float -> double, double accumulate (FP64 Gram of the first sketch)
    F64_F32 = 2,    // double x float -> float, double accumulate (Q0 = Y0 L^-T in FP64)
};

struct GemmDesc {
    int M, N, K;
    int ta, tb, tc;
    int sym;
    int ksplit;
    int tiles_m, tiles_n;
    int tiles_total;  // tiles incl. K slices
    int pad_;
    const void* A; long long lda;
    const void* B; long long ldb;
    void* C; long long ldc;
    const void* Cin; long long ldcin;
    const float* D; long long ldd;
    const float* rs; const float* cs;
    double alpha, beta, gamma;
    void* partial;  // accumulator-typed [ksplit][M*N]
};

// Host-side builder + launcher of one grouped GEMM stage.
class GemmBatch {
  public:
    explicit GemmBatch(GemmKind kind) : kind_(kind) {}
    // Adds a problem; returns its index.  Workspace for split-K is allocated at finalize().
    int add(GemmDesc d);
    void finalize();  // uploads descriptors & prefix table, allocates split-K partials
    void launch(cudaStream_t s) const;
    bool empty() const { return descs_.empty(); }
    std::vector<GemmDesc>& descs() { return descs_; }
    double flops() const;  // 2*M*N*K summed (algorithmic)

    static GemmDesc make(int M, int N, int K, const void* A, long long lda, int ta, const void* B, long long ldb,
                         int tb, void* C, long long ldc, int tc) {
        GemmDesc d{};
        d.M = M; d.N = N; d.K = K;
        d.A = A; d.lda = lda; d.ta = ta;
        d.B = B; d.ldb = ldb; d.tb = tb;
        d.C = C; d.ldc = ldc; d.tc = tc;
        d.alpha = 1.0; d.beta = 0.0; d.gamma = 0.0;
        d.ksplit = 1;
        return d;
    }

  private:
    GemmKind kind_;
    std::vector<GemmDesc> descs_;
    DevBuf d_descs_, d_prefix_, partials_;
    int total_tiles_ = 0;
    int total_partial_elems_ = 0;
    int bm_ = 128, bn_ = 128;
};

// Picks a deterministic split factor for skinny-output / long-K problems (fixed per shape, never per batch).
int choose_ksplit(int M, int N, int K, int bm, int bn);

}  // namespace rkfac_b200
