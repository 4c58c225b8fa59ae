// dropin_test.cpp -- the C++ drop-in (include/rkfac_gpu.hpp) exercised against the UNMODIFIED reference headers:
// the same inputs and RngState go through rkfac::X (reference, FP64 CPU) and rkfac::gpu::X (B200), and the
// sign-invariant reconstruction, eigenvalues and preconditioned gradient are compared (test infrastructure;
// built by oracle/Makefile into oracle/_ref/dropin_test, run by tests/test_gpu_dropin.py on the GPU box).
#include <rkfac/kfactor.hpp>
#include <rkfac/network.hpp>
#include <rkfac/optimizer.hpp>
#include <rkfac/rnla.hpp>
#include <rkfac/rng.hpp>

#include <cmath>
#include <cstdio>

#include "rkfac_gpu.hpp"
#include "rkfac_gpu_optimizer.hpp"

using namespace rkfac;

static double rel(const DenseMatrix& a, const DenseMatrix& b) {
    return frobenius_norm(subtract(a, b)) / std::max(1e-300, frobenius_norm(b));
}

int main() {
    // config-1-like factor: zero-init EA of 12 steps of X^T X / n with column decay i^-1
    const std::size_t d = 384, n = 192;
    EAKFactor f_cpu(d, 0.95, /*zero_init=*/true), f_gpu(d, 0.95, true);
    for (std::size_t k = 0; k < 12; ++k) {
        RngState g = RngState(220615397).substream(k, 0);
        DenseMatrix z = sample_gaussian(g, n, d);
        DenseMatrix m(d, n);
        for (std::size_t i = 0; i < d; ++i)
            for (std::size_t s = 0; s < n; ++s) m(i, s) = z(s, i) / double(i + 1) / std::sqrt(double(n));
        ea_update(f_cpu, m);
        gpu::ea_update(f_gpu, m);
    }
    const double e_ea = rel(f_gpu.mbar, f_cpu.mbar);
    int fails = e_ea < 1e-5 ? 0 : 1;
    std::printf("{\"ea_rel\": %.3e", e_ea);

    const SketchParams sk{48, 8, 2};
    RngState g_j = RngState(99).substream(0, 0);
    const DenseMatrix j = sample_gaussian(g_j, d, d);
    for (int meth = 0; meth < 2; ++meth) {
        RngState r0 = RngState(7).substream(0, 0), r1 = r0;
        LowRankEig a = meth == 0 ? srevd(f_cpu.mbar, sk, r0) : rsvd_psd(f_cpu.mbar, sk, r0);
        LowRankEig b = meth == 0 ? gpu::srevd(f_cpu.mbar, sk, r1) : gpu::rsvd_psd(f_cpu.mbar, sk, r1);
        const double e_rec = rel(lowrank_reconstruct(b), lowrank_reconstruct(a));
        double e_eig = 0.0;
        for (std::size_t i = 0; i < a.d.size(); ++i) e_eig = std::max(e_eig, std::abs(a.d[i] - b.d[i]) / a.d[i]);
        const DenseMatrix sa = apply_lowrank_damped_inverse(
            a, 0.1, apply_lowrank_damped_inverse(a, 0.1, j, ApplySide::RIGHT), ApplySide::LEFT);
        const DenseMatrix sb = gpu::apply_lowrank_damped_inverse(
            b, 0.1, gpu::apply_lowrank_damped_inverse(b, 0.1, j, ApplySide::RIGHT), ApplySide::LEFT);
        const double e_s = rel(sb, sa);
        const bool ok = r0.counter == r1.counter && e_rec < 1e-4 && e_eig < 1e-4 && e_s < 1e-4 &&
                        b.method == a.method && b.rank() == a.rank();
        fails += ok ? 0 : 1;
        std::printf(", \"%s\": {\"recon\": %.3e, \"eig\": %.3e, \"precond\": %.3e, \"counter_match\": %d}",
                    meth == 0 ? "srevd" : "rsvd_psd", e_rec, e_eig, e_s, int(r0.counter == r1.counter));
    }
    // exact K-FAC (eig.hpp:210-237 + kfactor.hpp:182-185) and the general rsvd (rnla.hpp:62-77)
    {
        const SymEigResult ea = sym_eig(f_cpu.mbar), eb = gpu::sym_eig(f_cpu.mbar);
        double e_eig = 0.0;
        for (std::size_t i = 0; i < 40; ++i) e_eig = std::max(e_eig, std::abs(ea.d[i] - eb.d[i]) / std::abs(ea.d[i]));
        const DenseMatrix sa = apply_eig_damped_inverse(ea, 0.1, j, ApplySide::LEFT);
        const DenseMatrix sb = gpu::apply_eig_damped_inverse(eb, 0.1, j, ApplySide::LEFT);
        const double e_s = rel(sb, sa);
        const bool ok = e_eig < 1e-6 && e_s < 1e-4;
        fails += ok ? 0 : 1;
        std::printf(", \"sym_eig\": {\"eig_top40\": %.3e, \"precond\": %.3e}", e_eig, e_s);
        RngState g_x = RngState(5).substream(0, 0);
        const DenseMatrix xr = sample_gaussian(g_x, 150, 100);
        DenseMatrix xs(150, 100);  // geometric column decay so the sketch is well posed
        for (std::size_t i = 0; i < 150; ++i)
            for (std::size_t c = 0; c < 100; ++c) xs(i, c) = xr(i, c) * std::pow(0.9, double(c));
        RngState r0 = RngState(7).substream(0, 3), r1 = r0;
        const SvdResult a = rsvd(xs, SketchParams{12, 4, 2}, r0), b = gpu::rsvd(xs, SketchParams{12, 4, 2}, r1);
        DenseMatrix pa(150, 100), pb(150, 100);
        for (std::size_t i = 0; i < 150; ++i)
            for (std::size_t c = 0; c < 100; ++c)
                for (std::size_t k = 0; k < a.s.size(); ++k) {
                    pa(i, c) += a.u(i, k) * a.s[k] * a.v(c, k);
                    pb(i, c) += b.u(i, k) * b.s[k] * b.v(c, k);
                }
        const double e_p = rel(pb, pa);
        const bool ok2 = r0.counter == r1.counter && e_p < 1e-4 && b.s.size() == a.s.size();
        fails += ok2 ? 0 : 1;
        std::printf(", \"rsvd\": {\"usv\": %.3e, \"counter_match\": %d}", e_p, int(r0.counter == r1.counter));
    }
    // the batched optimizer step (optimizer.hpp:139-222) through the plan: two identical nets, the reference's
    // optimizer_step on one and rkfac::gpu::optimizer_step on the other, over the T_KI cache schedule
    // (step 0 decomposes, step 1 reuses, step 2 decomposes again), for SRE-KFAC and RS-KFAC
    {
        const std::size_t d_in = 72, n = 96;
        double worst = 0.0, worst_cache = 0.0;
        int cache_ok = 1;
        for (Method method : {Method::SRE_KFAC, Method::RS_KFAC}) {
            RngState init_a(11), init_b(11);
            Mlp net_cpu(d_in, {96, 64}, 10, 0.95, init_a), net_gpu(d_in, {96, 64}, 10, 0.95, init_b);
            for (Mlp* net : {&net_cpu, &net_gpu})
                for (LayerState& L : net->layers()) {  // zero-init EA (parity fixtures)
                    L.a_factor = EAKFactor(L.a_factor.dim(), 0.95, true);
                    L.g_factor = EAKFactor(L.g_factor.dim(), 0.95, true);
                }
            OptimizerConfig cfg;
            cfg.method = method;
            cfg.n_pwr_it = 2;
            ResolvedSchedule sch;
            sch.lambda = 0.1; sch.target_rank = 24; sch.oversampling = 8; sch.t_ki = 2;
            const RngState rng(4242);
            for (std::size_t step = 0; step < 3; ++step) {
                Batch b;
                RngState g = RngState(77).substream(step, 0);
                b.x = sample_gaussian(g, d_in, n);
                for (std::size_t i = 0; i < d_in; ++i)
                    for (std::size_t c = 0; c < n; ++c) b.x(i, c) /= double(i + 1);
                for (std::size_t c = 0; c < n; ++c) b.y.push_back(int(g.next_u64() % 10));
                const ForwardResult fw = net_cpu.forward(b);
                const BackwardResult bw = net_cpu.backward(b);
                net_cpu.accumulate_factors(fw.a_matrices, bw.g_matrices);
                gpu::accumulate_factors(net_gpu, fw.a_matrices, bw.g_matrices);
                const StepResult ra = optimizer_step(net_cpu, bw.gradients, cfg, sch, step, rng);
                const StepResult rb = gpu::optimizer_step(net_gpu, bw.gradients, cfg, sch, step, rng);
                for (std::size_t l = 0; l < ra.updates.size(); ++l) worst = std::max(worst, rel(rb.updates[l], ra.updates[l]));
                for (std::size_t l = 0; l < net_cpu.n_layers(); ++l) {  // the mirrored caches follow the reference's
                    const LowRankEig &ca = *net_cpu.layers()[l].cached_a_decomp, &cb = *net_gpu.layers()[l].cached_a_decomp;
                    cache_ok &= int(ca.method == cb.method && ca.rank() == cb.rank());
                    worst_cache = std::max(worst_cache, rel(lowrank_reconstruct(cb), lowrank_reconstruct(ca)));
                }
            }
        }
        const bool ok = worst < 1e-4 && worst_cache < 1e-4 && cache_ok;
        fails += ok ? 0 : 1;
        std::printf(", \"optimizer_step\": {\"updates\": %.3e, \"cached_recon\": %.3e, \"cache_ok\": %d}", worst,
                    worst_cache, cache_ok);
    }
    // error behaviour mirrors the reference exceptions
    bool threw = false;
    try {
        LowRankEig lr{DenseMatrix::identity(2), {1.0, 1.0}, DecompMethod::RSVD};
        gpu::apply_lowrank_damped_inverse(lr, 0.0, DenseMatrix(2, 1, 1.0), ApplySide::LEFT);
    } catch (const DampingNonpositive&) {
        threw = true;
    }
    fails += threw ? 0 : 1;
    std::printf(", \"damping_throws\": %d, \"fails\": %d}\n", int(threw), fails);
    return fails == 0 ? 0 : 1;
}
