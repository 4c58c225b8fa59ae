// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-linkage wrappers around the UNMODIFIED reference headers (/root/reference/proj/include/rkfac,
// compiled where they lie by oracle/Makefile into oracle/_ref/librkfac_ref.so).  No reference source
// is copied into this repository: this file only includes the headers and marshals plain arrays.
// Used (a) to pin the C restatement in rkfac_oracle.c bit-for-bit, (b) to generate the golden
// fixtures under tests/golden/, and (c) as bench.py's "reference" CPU baseline
// (cpu_baseline.kind = "reference"), threaded one factor per std::thread as SPEC.md:94,162,251 allow.
#include <rkfac/kfactor.hpp>
#include <rkfac/rnla.hpp>
#include <rkfac/rng.hpp>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

using namespace rkfac;

namespace {

DenseMatrix to_mat(const double* p, std::size_t r, std::size_t c) {
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const DimensionMismatch&) {
        return 1;
    } catch (const RankDeficient&) {
        return 2;
    } catch (const NoConvergence&) {
        return 3;
    } catch (const DampingNonpositive&) {
        return 4;
    } catch (...) {
        return 7;
    }
}

}  // namespace

extern "C" {

int ref_sample_gaussian(std::uint64_t seed, std::uint64_t counter, std::size_t m, std::size_t n,
                        double* out, std::uint64_t* counter_out) {
    return guarded([&] {
        RngState rng(seed);
        rng.counter = counter;
        DenseMatrix x = sample_gaussian(rng, m, n);
        std::memcpy(out, x.data(), sizeof(double) * m * n);
        *counter_out = rng.counter;
    });
}

std::uint64_t ref_substream(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {
    return RngState(seed).substream(a, b).seed;
}

int ref_qr_thin(const double* x, std::size_t m, std::size_t n, int strict, double* q, double* r) {
    return guarded([&] {
        QrResult res = qr_thin(to_mat(x, m, n), strict != 0);
        std::memcpy(q, res.q.data(), sizeof(double) * m * n);
        if (r) std::memcpy(r, res.r.data(), sizeof(double) * n * n);
    });
}

int ref_sym_eig(const double* s, std::size_t n, double* p, double* d) {
    return guarded([&] {
        SymEigResult e = sym_eig(to_mat(s, n, n));
        std::memcpy(p, e.p.data(), sizeof(double) * n * n);
        std::copy(e.d.begin(), e.d.end(), d);
    });
}

int ref_ea_update(double* mbar, std::size_t d, const double* m, std::size_t rows, std::size_t n,
                  double rho) {
    return guarded([&] {
        EAKFactor f;
        f.mbar = to_mat(mbar, d, d);
        f.rho = rho;
        ea_update(f, to_mat(m, rows, n));
        std::memcpy(mbar, f.mbar.data(), sizeof(double) * d * d);
    });
}

// method 0 = srevd (rnla.hpp:90), 1 = rsvd_psd (rnla.hpp:81).
int ref_decompose(int method, const double* x, std::size_t d, std::size_t r, std::size_t p,
                  std::size_t q, std::uint64_t seed, std::uint64_t* counter, double* u, double* dv,
                  std::size_t* r_out) {
    return guarded([&] {
        RngState rng(seed);
        rng.counter = *counter;
        const SketchParams sk{r, p, q};
        LowRankEig lr = method == 0 ? srevd(to_mat(x, d, d), sk, rng) : rsvd_psd(to_mat(x, d, d), sk, rng);
        std::memcpy(u, lr.u.data(), sizeof(double) * lr.u.size());
        std::copy(lr.d.begin(), lr.d.end(), dv);
        *r_out = lr.d.size();
        *counter = rng.counter;
    });
}

// rnla.hpp:62-77 rsvd on a general rows x cols matrix: u (rows x r), s (r), v (cols x r), row-major.
int ref_rsvd(const double* x, std::size_t rows, std::size_t cols, std::size_t r, std::size_t p, std::size_t q,
             std::uint64_t seed, std::uint64_t* counter, double* u, double* s, double* v, std::size_t* r_out) {
    return guarded([&] {
        RngState rng(seed);
        rng.counter = *counter;
        const SketchParams sk{r, p, q};
        SvdResult res = rsvd(to_mat(x, rows, cols), sk, rng);
        std::memcpy(u, res.u.data(), sizeof(double) * res.u.size());
        std::copy(res.s.begin(), res.s.end(), s);
        std::memcpy(v, res.v.data(), sizeof(double) * res.v.size());
        *r_out = res.s.size();
        *counter = rng.counter;
    });
}

// side 0 = LEFT, 1 = RIGHT (kfactor.hpp:134).
int ref_apply_lowrank(const double* u, const double* dv, std::size_t dim, std::size_t r, double lambda,
                      const double* v, std::size_t rows, std::size_t cols, int side, double* out) {
    return guarded([&] {
        LowRankEig lr{to_mat(u, dim, r), std::vector<double>(dv, dv + r), DecompMethod::RSVD};
        DenseMatrix o = apply_lowrank_damped_inverse(lr, lambda, to_mat(v, rows, cols),
                                                     side == 0 ? ApplySide::LEFT : ApplySide::RIGHT);
        std::memcpy(out, o.data(), sizeof(double) * rows * cols);
    });
}

// The reference's full preconditioned step for a list of layers (optimizer.hpp:139-167 semantics:
// decompose A (which=0) and G (which=1) with substream(step, 2l+which), then LEFT_G(RIGHT_A(J))),
// plus one EA update per factor beforehand.  Work is spread one factor (then one layer) per
// std::thread over `threads` workers.  Pointers are per factor / per layer arrays.  Used as the
// timed CPU baseline; times are reported back per phase in seconds.  us/dvs (optional, per factor,
// d x r_f row-major and r_f) receive the decompositions for parity checks.
int ref_step_threaded(int method, int threads, std::size_t nlayers, const std::size_t* dims_a,
                      const std::size_t* dims_g, double* const* factors, const double* const* ms,
                      const std::size_t* ns, double rho, std::size_t r, std::size_t p, std::size_t q,
                      std::uint64_t rng_root, std::uint64_t step, double lambda,
                      const double* const* grads, double* const* outs, double* phase_seconds,
                      double* const* us, double* const* dvs) {
    using Clock = std::chrono::steady_clock;
    const std::size_t nf = 2 * nlayers;
    std::vector<int> status(nf + nlayers, 0);
    std::vector<LowRankEig> dec(nf);
    auto run_pool = [&](std::size_t count, auto&& body) {
        std::atomic<std::size_t> next{0};
        std::vector<std::thread> pool;
        const int nt = std::max(1, threads);
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&] {
                for (std::size_t i = next++; i < count; i = next++) body(i);
            });
        for (auto& th : pool) th.join();
    };
    auto dim_of = [&](std::size_t f) { return (f % 2 == 0) ? dims_a[f / 2] : dims_g[f / 2]; };

    auto t0 = Clock::now();
    if (ms) {
        run_pool(nf, [&](std::size_t f) {
            status[f] = guarded([&] {
                const std::size_t d = dim_of(f);
                EAKFactor fac;
                fac.mbar = to_mat(factors[f], d, d);
                fac.rho = rho;
                ea_update(fac, to_mat(ms[f], d, ns[f]));
                std::memcpy(factors[f], fac.mbar.data(), sizeof(double) * d * d);
            });
        });
    }
    auto t1 = Clock::now();
    run_pool(nf, [&](std::size_t f) {
        if (status[f]) return;
        status[f] = guarded([&] {
            const std::size_t d = dim_of(f);
            RngState sub = RngState(rng_root).substream(step, f);
            const SketchParams sk{r, p, q};
            dec[f] = method == 0 ? srevd(to_mat(factors[f], d, d), sk, sub)
                                 : rsvd_psd(to_mat(factors[f], d, d), sk, sub);
            if (us && us[f]) std::memcpy(us[f], dec[f].u.data(), sizeof(double) * dec[f].u.size());
            if (dvs && dvs[f]) std::copy(dec[f].d.begin(), dec[f].d.end(), dvs[f]);
        });
    });
    auto t2 = Clock::now();
    if (grads) {
        run_pool(nlayers, [&](std::size_t l) {
            status[nf + l] = guarded([&] {
                const std::size_t dA = dims_a[l], dG = dims_g[l];
                DenseMatrix m = apply_lowrank_damped_inverse(dec[2 * l], lambda, to_mat(grads[l], dG, dA),
                                                             ApplySide::RIGHT);
                DenseMatrix s = apply_lowrank_damped_inverse(dec[2 * l + 1], lambda, m, ApplySide::LEFT);
                if (outs) std::memcpy(outs[l], s.data(), sizeof(double) * dG * dA);
            });
        });
    }
    auto t3 = Clock::now();
    if (phase_seconds) {
        phase_seconds[0] = std::chrono::duration<double>(t1 - t0).count();
        phase_seconds[1] = std::chrono::duration<double>(t2 - t1).count();
        phase_seconds[2] = std::chrono::duration<double>(t3 - t2).count();
    }
    for (int s : status)
        if (s) return s;
    return 0;
}

}  // extern "C"
