// tc_gemm.cuh -- tcgen05/TMEM/TMA grouped 3xTF32 GEMM for Y^T = (X Q)^T (see tc_gemm.cu).
#pragma once

#include <cuda.h>

#include <vector>

#include "common.cuh"

namespace rkfac_b200 {

struct TcProblem {
    int M, N, K, kblocks;
    float* Yt;       // N x M output (ld = ldy)
    long long ldy;
};

struct TcTile {
    int prob, m0, n0, n_tile;
};

// A K-major FP32 operand split into TF32 hi/lo planes (rows x K, row pitch ld elements, ld*4 % 16 == 0).
struct TcOperand {
    const float* hi;
    const float* lo;
    long long ld;
};

class TcXQ {
  public:
    // Y^T (N x M) = (A (M x K) * B^T)^T where B is given as N x K (i.e. Q^T); all K-major.
    void add(const TcOperand& a, const TcOperand& b, int M, int N, int K, float* Yt, long long ldy);
    void finalize();
    void launch(cudaStream_t s) const;
    bool empty() const { return tiles_.empty(); }
    double flops() const;
    static size_t smem_bytes();

  private:
    std::vector<TcProblem> probs_;
    std::vector<CUtensorMap> maps_;
    std::vector<TcTile> tiles_;
    int nctas_ = 0;
    DevBuf d_probs_, d_maps_, d_tiles_, d_begin_;
};

// hi/lo TF32 split of row-major matrices (rows x cols, source pitch lds, destination pitch ldd), all problems in
// one launch; offset = prefix of rows*cols.
struct SplitDesc {
    const float* src;
    float* hi;
    float* lo;
    int rows, cols;
    long long lds, ldd;
    long long offset;
};
void launch_split(const SplitDesc* d_descs, int n, long long total, cudaStream_t s);

}  // namespace rkfac_b200
