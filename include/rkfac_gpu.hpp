// rkfac_gpu.hpp -- header-only C++ drop-in for the reference operator API (/root/reference/proj/include/rkfac),
// implemented over the C-ABI in rkfac_b200.h.  Include it AFTER the reference headers; the call sites of the
// reference compile unchanged once `rkfac::` is replaced by `rkfac::gpu::` (or brought in with a using-declaration):
//
//   reference                                              drop-in (same signature)
//   void ea_update(EAKFactor&, const DenseMatrix&)          rkfac::gpu::ea_update        (kfactor.hpp:33-41)
//   LowRankEig srevd(const DenseMatrix&, const SketchParams&, RngState&)
//                                                          rkfac::gpu::srevd            (rnla.hpp:90-105)
//   LowRankEig rsvd_psd(...same...)                        rkfac::gpu::rsvd_psd         (rnla.hpp:81-85)
//   DenseMatrix apply_lowrank_damped_inverse(const LowRankEig&, double, const DenseMatrix&, ApplySide)
//                                                          rkfac::gpu::apply_lowrank_damped_inverse (kfactor.hpp:134-161)
//   SvdResult rsvd(const DenseMatrix&, const SketchParams&, RngState&)   rkfac::gpu::rsvd  (rnla.hpp:62-77)
//   SymEigResult sym_eig(const DenseMatrix&)                rkfac::gpu::sym_eig          (eig.hpp:210-237)
//   DenseMatrix apply_eig_damped_inverse(const SymEigResult&, double, const DenseMatrix&, ApplySide)
//                                                          rkfac::gpu::apply_eig_damped_inverse (kfactor.hpp:182-185)
//
// Value semantics as in the reference: inputs by const&, outputs by value, EAKFactor mutated in place, RngState&
// advanced by 2*d*w exactly like sample_gaussian (rng.hpp:59-63).  FP64 host data is converted to FP32 for the
// device and back.  Status codes are rethrown as the reference exception types (errors.hpp:8-34).
// Link with librkfac_b200.so and libcudart.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "rkfac_b200.h"

namespace rkfac {
namespace gpu {

namespace detail {

inline rkfac_context_t context() {
    static rkfac_context_t ctx = [] {
        rkfac_context_t c = nullptr;
        const int st = rkfac_create(&c, 0, nullptr);
        if (st != RKFAC_OK) throw std::runtime_error(std::string("rkfac_create: ") + rkfac_last_error(nullptr));
        return c;
    }();
    return ctx;
}

inline void check(int st, const char* what) {
    if (st == RKFAC_OK) return;
    const std::string msg = std::string(what) + ": " + rkfac_last_error(context());
    switch (st) {
        case RKFAC_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case RKFAC_RANK_DEFICIENT: throw RankDeficient(msg);
        case RKFAC_NO_CONVERGENCE: throw NoConvergence(msg);
        case RKFAC_DAMPING_NONPOSITIVE: throw DampingNonpositive(msg);
        default: throw std::runtime_error(msg);
    }
}

// FP32 device copy of a FP64 row-major matrix (RAII).
struct DevMat {
    float* p = nullptr;
    std::size_t rows = 0, cols = 0;
    DevMat(std::size_t r, std::size_t c) : rows(r), cols(c) {
        if (r * c && cudaMalloc(&p, sizeof(float) * r * c) != cudaSuccess) throw std::bad_alloc();
    }
    explicit DevMat(const DenseMatrix& m) : DevMat(m.rows(), m.cols()) { upload(m.data(), m.size()); }
    DevMat(const std::vector<double>& v) : DevMat(v.size(), 1) { upload(v.data(), v.size()); }
    ~DevMat() { if (p) cudaFree(p); }
    DevMat(const DevMat&) = delete;
    DevMat& operator=(const DevMat&) = delete;
    void upload(const double* src, std::size_t n) {
        std::vector<float> h(src, src + n);
        if (n) cudaMemcpy(p, h.data(), sizeof(float) * n, cudaMemcpyHostToDevice);
    }
    void download(double* dst, std::size_t n) const {
        std::vector<float> h(n);
        if (n) cudaMemcpy(h.data(), p, sizeof(float) * n, cudaMemcpyDeviceToHost);
        for (std::size_t i = 0; i < n; ++i) dst[i] = h[i];
    }
};

template <class Fn>
LowRankEig decompose(Fn fn, const char* name, const DenseMatrix& x, const SketchParams& p, RngState& rng,
                     DecompMethod method) {
    if (x.rows() != x.cols()) throw DimensionMismatch(std::string(name) + ": factor must be square");
    const std::size_t d = x.rows();
    const std::size_t rmax = std::max<std::size_t>(1, std::min(p.target_rank, d));
    DevMat dx(x), du(d, rmax), dv(rmax, 1);
    uint64_t counter = rng.counter;
    int64_t rank = 0;
    check(fn(context(), dx.p, (int64_t)d, (int64_t)d, (int64_t)p.target_rank, (int64_t)p.oversampling,
             (int64_t)p.power_iters, rng.seed, &counter, du.p, (int64_t)rmax, dv.p, &rank),
          name);
    check(rkfac_synchronize(context()), name);
    rng.counter = counter;
    const std::size_t r = (std::size_t)rank;
    LowRankEig out;
    out.method = method;
    std::vector<double> u(d * rmax);
    du.download(u.data(), u.size());
    out.u = DenseMatrix(d, r);
    for (std::size_t i = 0; i < d; ++i)
        for (std::size_t j = 0; j < r; ++j) out.u(i, j) = u[i * rmax + j];
    out.d.resize(r);
    std::vector<double> dd(rmax);
    dv.download(dd.data(), rmax);
    for (std::size_t j = 0; j < r; ++j) out.d[j] = dd[j];
    return out;
}

}  // namespace detail

inline void ea_update(EAKFactor& f, const DenseMatrix& m) {
    if (m.rows() != f.dim()) throw DimensionMismatch("ea_update: update row count != factor dimension");
    detail::DevMat dx(f.mbar), dm(m);
    detail::check(rkfac_ea_update(detail::context(), dx.p, (int64_t)f.dim(), (int64_t)f.dim(), dm.p,
                                  (int64_t)m.cols(), (int64_t)m.rows(), (int64_t)m.cols(), f.rho, 1.0),
                  "ea_update");
    detail::check(rkfac_synchronize(detail::context()), "ea_update");
    dx.download(f.mbar.data(), f.mbar.size());
    ++f.steps;
}

inline LowRankEig srevd(const DenseMatrix& x, const SketchParams& p, RngState& rng) {
    return detail::decompose(rkfac_srevd, "srevd", x, p, rng, DecompMethod::SREVD);
}

inline LowRankEig rsvd_psd(const DenseMatrix& x, const SketchParams& p, RngState& rng) {
    return detail::decompose(rkfac_rsvd_psd, "rsvd_psd", x, p, rng, DecompMethod::RSVD);
}

inline DenseMatrix apply_lowrank_damped_inverse(const LowRankEig& lr, double lambda, const DenseMatrix& v,
                                               ApplySide side) {
    if (lambda <= 0.0) throw DampingNonpositive("apply_lowrank_damped_inverse: lambda must be > 0");
    const std::size_t r = lr.rank(), dim = lr.dim();
    detail::DevMat du(lr.u), dd(lr.d), dv(v), dout(v.rows(), v.cols());
    detail::check(rkfac_apply_lowrank_damped_inverse(detail::context(), du.p, (int64_t)std::max<std::size_t>(r, 1),
                                                     dd.p, (int64_t)dim, (int64_t)r, lambda, dv.p,
                                                     (int64_t)v.cols(), (int64_t)v.rows(), (int64_t)v.cols(),
                                                     side == ApplySide::LEFT ? RKFAC_LEFT : RKFAC_RIGHT, dout.p,
                                                     (int64_t)v.cols()),
                  "apply_lowrank_damped_inverse");
    detail::check(rkfac_synchronize(detail::context()), "apply_lowrank_damped_inverse");
    DenseMatrix out(v.rows(), v.cols());
    dout.download(out.data(), out.size());
    return out;
}

// eig.hpp:210-237: full symmetric eigendecomposition (FP64 on the GPU: Householder + divide and conquer), eigenvectors
// as the columns of p, eigenvalues descending; asymmetry -> DimensionMismatch, a non-converging leaf -> NoConvergence.
inline SymEigResult sym_eig(const DenseMatrix& s) {
    if (s.rows() != s.cols()) throw DimensionMismatch("sym_eig: matrix must be square");
    const std::size_t n = s.rows();
    detail::DevMat ds(s), dp(n, n);
    double* d64 = nullptr;
    if (cudaMalloc(&d64, sizeof(double) * std::max<std::size_t>(n, 1)) != cudaSuccess) throw std::bad_alloc();
    const int st = rkfac_sym_eig(detail::context(), ds.p, (int64_t)n, (int64_t)n, dp.p, (int64_t)n, nullptr, d64);
    SymEigResult out;
    out.d.resize(n);
    if (st == RKFAC_OK) cudaMemcpy(out.d.data(), d64, sizeof(double) * n, cudaMemcpyDeviceToHost);
    cudaFree(d64);
    detail::check(st, "sym_eig");
    out.p = DenseMatrix(n, n);
    dp.download(out.p.data(), out.p.size());
    return out;
}

// kfactor.hpp:165-186: the exact damped inverse through the low-rank kernels (Eq. 11 with a complete orthonormal
// basis is exactly (U D U^T + lambda I)^{-1}).
inline DenseMatrix apply_eig_damped_inverse(const SymEigResult& eig, double lambda, const DenseMatrix& v,
                                            ApplySide side) {
    if (lambda <= 0.0) throw DampingNonpositive("apply_eig_damped_inverse: lambda must be > 0");
    LowRankEig lr;
    lr.u = eig.p;
    lr.d = eig.d;
    lr.method = DecompMethod::SREVD;
    return rkfac::gpu::apply_lowrank_damped_inverse(lr, lambda, v, side);
}

// rnla.hpp:62-77 on a general rows x cols matrix.
inline SvdResult rsvd(const DenseMatrix& x, const SketchParams& p, RngState& rng) {
    const std::size_t rows = x.rows(), cols = x.cols();
    const std::size_t rmax = std::max<std::size_t>(1, std::min({p.target_rank, rows, cols}));
    detail::DevMat dx(x), du(rows, rmax), ds(rmax, 1), dv(cols, rmax);
    uint64_t counter = rng.counter;
    int64_t rank = 0;
    detail::check(rkfac_rsvd(detail::context(), dx.p, (int64_t)cols, (int64_t)rows, (int64_t)cols,
                             (int64_t)p.target_rank, (int64_t)p.oversampling, (int64_t)p.power_iters, rng.seed,
                             &counter, du.p, (int64_t)rmax, ds.p, dv.p, (int64_t)rmax, &rank),
                  "rsvd");
    rng.counter = counter;
    const std::size_t r = (std::size_t)rank;
    std::vector<double> u(rows * rmax), s(rmax), v(cols * rmax);
    du.download(u.data(), u.size());
    ds.download(s.data(), s.size());
    dv.download(v.data(), v.size());
    SvdResult out;
    out.u = DenseMatrix(rows, r);
    out.v = DenseMatrix(cols, r);
    for (std::size_t i = 0; i < rows; ++i)
        for (std::size_t j = 0; j < r; ++j) out.u(i, j) = u[i * rmax + j];
    for (std::size_t i = 0; i < cols; ++i)
        for (std::size_t j = 0; j < r; ++j) out.v(i, j) = v[i * rmax + j];
    out.s.assign(s.begin(), s.begin() + r);
    return out;
}

}  // namespace gpu
}  // namespace rkfac
