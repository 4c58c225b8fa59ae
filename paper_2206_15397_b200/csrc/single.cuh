// single.cuh -- cached tcgen05 stages of the single-factor C-ABI operators (see single.cu).
#pragma once

#include <list>
#include <memory>

#include "common.cuh"

namespace rkfac_b200 {

class SingleOps {
  public:
    SingleOps();
    ~SingleOps();
    // kfactor.hpp:33-41: x (d x d, pitch ldx) <- rho x + (1-rho) scale^2 m m^T, m d x n (pitch ldm); exactly symmetric
    void ea_update(float* x, long long ldx, int d, const float* m, long long ldm, int n, double rho, double scale,
                   cudaStream_t s);
    // kfactor.hpp:134-161: out = LEFT / RIGHT Eq. 11 of v (rows x cols) with u (dim x r), dvals (r), lambda > 0
    void apply(const float* u, long long ldu, const float* dv, int dim, int r, double lam, const float* v,
               long long ldv, int rows, int cols, int side, float* out, long long ldo, cudaStream_t s);

  private:
    struct Ea;
    struct Apply;
    std::list<std::unique_ptr<Ea>> ea_;
    std::list<std::unique_ptr<Apply>> ap_;
};

}  // namespace rkfac_b200
