// tc_gemm.cuh -- tcgen05/TMEM/TMA grouped 3xTF32 GEMM engine (see tc_gemm.cu).
//
//   D(m, n) = sum_k A(m, k) B(n, k)     A: M x K, B: N x K, both K-major FP32 (row pitch % 16 bytes == 0)
//   v(m, n) = alpha * rs[m] * cs[n] * D + beta * Cin(m, n) + gamma * Din(m, n)
//   outputs (each optional, each row-major [m][n] (t=0) or transposed [n][m] (t=1)):
//     out0 = v, out1 = v, lo0 = v - tf32(v), lo1 = v - tf32(v)
// 3xTF32: the tensor core reads FP32 operands as TF32 by ignoring the low 13 mantissa bits (verified on B200:
// results with explicitly truncated operands are bitwise identical), so operand "hi" = the raw FP32 array and only
// the lo plane (x - tf32(x)) is stored separately; D = A*B_lo + A_lo*B + A*B (three MMAs into one TMEM tile).
#pragma once

#include <cuda.h>

#include <utility>
#include <vector>

#include "common.cuh"

namespace rkfac_b200 {

struct TcOut {
    float* p = nullptr;
    long long ld = 0;
    int t = 0;
};

struct TcProblemDesc {
    int M = 0, N = 0, K = 0;
    const float* A = nullptr; const float* A_lo = nullptr; long long lda = 0;  // A_lo null: formed in smem
    const float* B = nullptr; const float* B_lo = nullptr; long long ldb = 0;  // B_lo null: formed in smem
    float alpha = 1.f, beta = 0.f, gamma = 0.f;
    const float* rs = nullptr;
    const float* cs = nullptr;
    const float* Cin = nullptr; long long ldcin = 0; int cin_t = 0;
    const float* Din = nullptr; long long lddin = 0; int din_t = 0;
    TcOut out0, out1, lo0, lo1;
    int sym = 0;       // M == N: upper tiles only, mirrored stores (exactly symmetric result)
    int ksplit = 0;    // 0 = choose automatically
    int slice_k = 0;   // > 0: split K so no TMEM accumulation chain is longer than slice_k (accuracy)
    int single = 0;    // 1: one TF32 MMA per product (no lo terms) -- for products that only carry a subspace
    int max_n_tile = 0;  // > 0: N tiles of at most this many columns (more, shorter tiles; same arithmetic)
};

struct TcProb {  // device copy
    int M, N, K, kblocks, ksplit, sym, n_tile, a_conv;  // a_conv: A lo plane formed in shared memory
    float alpha, beta, gamma;
    int b_conv;  // B lo plane formed in shared memory
    int single, pad3_;
    const float* rs; const float* cs;
    const float* Cin; long long ldcin; int cin_t, din_t;
    const float* Din; long long lddin;
    float* o[4]; long long ldo[4]; int to[4]; int is_lo[4];
    float* partial;
};

struct TcTile {
    int prob, m0, n0, kb0, kb1, slice, pair, pad_;  // pair: rows m0 .. m0+255 as two accumulators sharing B
};

struct TcRed {  // split-K reduction map: first 32x32 output tile of a split problem in the flattened reduction
    long long off;
    int prob, tiles_m;
};

class TcGemm {
  public:
    int add(const TcProblemDesc& d);
    // CTA pairs (cta_group::2): every tile is 256 rows over the two SMs of a TPC, each holding half of the B tile --
    // for the long-K products whose single-CTA mainloop is bound by shared-memory bandwidth.  Call before add().
    void set_two_cta(bool on) { two_cta_ = on; }
    void set_max_ctas(int n) { cap_ = n; }  // persistent-grid cap (0: all SMs); leaves SMs to concurrent streams
    // the consumer reduces the split-K partials itself (launch() skips the reduction kernel); after finalize(),
    // split_of(prob) gives the partial buffer and slice count of a problem ({nullptr, 1} when it was not split)
    void set_defer_reduce(bool on) { defer_reduce_ = on; }
    bool defer_reduce() const { return defer_reduce_; }
    std::pair<const float*, int> split_of(int prob) const {
        const TcProb& p = probs_[prob];
        return p.ksplit > 1 ? std::make_pair((const float*)p.partial, p.ksplit) : std::make_pair((const float*)nullptr, 1);
    }
    void finalize();
    void launch(cudaStream_t s) const;
    bool empty() const { return tiles_.empty(); }
    double flops() const;  // algorithmic 2*M*N*K (sym: half)
    static size_t smem_bytes();
    static int pair_slots();

  private:
    std::vector<TcProb> probs_;
    std::vector<TcProblemDesc> descs_;  // as added (with the resolved K split), for finalize's N split
    std::vector<CUtensorMap> maps_;
    std::vector<TcTile> tiles_;
    std::vector<size_t> partial_off_;
    int nctas_ = 0;
    bool any_split_ = false;
    int cfg_ = 0;
    int cap_ = 0;
    bool two_cta_ = false;
    bool defer_reduce_ = false;  // shared-memory configuration of the launch (tc_gemm.cu StageCfg: single / paired / EA)
    int nred_ = 0;
    long long red_total_ = 0;
    DevBuf d_probs_, d_maps_, d_tiles_, d_begin_, partials_, d_red_;
};

// TF32 lo plane (and optional padded copy) of row-major matrices, all problems in one launch.
struct SplitDesc {
    const float* src;
    float* hi;   // optional padded copy of src (nullptr: not written)
    float* lo;
    int rows, cols;
    long long lds, ldd;
    long long offset;
};
void launch_split(const SplitDesc* d_descs, int n, long long total, cudaStream_t s);

}  // namespace rkfac_b200
