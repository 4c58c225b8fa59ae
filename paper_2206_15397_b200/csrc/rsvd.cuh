// rsvd.cuh -- rnla.hpp:62-77 rsvd on a general rectangular matrix (see rsvd.cu).
#pragma once

#include <cstdint>

#include "common.cuh"

namespace rkfac_b200 {

class Rsvd {
  public:
    Rsvd();
    ~Rsvd();
    // x: m x n (pitch ldx); u: m x r (ldu), s: r, v: n x r (ldv); Omega from (seed, ctr0); *rank_out = clamped r.
    void run(const float* x, long long ldx, int m, int n, int r, int p, int q, uint64_t seed, uint64_t ctr0, float* u,
             long long ldu, float* s, float* v, long long ldv, int* rank_out, cudaStream_t st);

  private:
    struct Side;
    DevBuf ws_;
};

}  // namespace rkfac_b200
