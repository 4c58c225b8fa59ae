// capi.cu -- the extern "C" boundary (include/rkfac_b200.h).  No exception crosses it: every entry point maps
// internal errors to an rkfac_status mirroring the reference's exception types (errors.hpp:8-34).
#include <cstring>
#include <string>

#include "engine.cuh"

using namespace rkfac_b200;

struct rkfac_context {
    Context c;
};
struct rkfac_plan {
    std::unique_ptr<Plan> p;
    rkfac_context* ctx;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(rkfac_context* ctx, F&& f) {
    try {
        f();
        return RKFAC_OK;
    } catch (const Error& e) {
        if (ctx) ctx->c.last_error = e.what(); else g_err = e.what();
        return e.status;
    } catch (const std::exception& e) {
        if (ctx) ctx->c.last_error = e.what(); else g_err = e.what();
        return RKFAC_INVALID_ARGUMENT;
    }
}

void check_device() {
    int dev = -1;
    RKFAC_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop{};
    RKFAC_CUDA(cudaGetDeviceProperties(&prop, dev));
    RKFAC_REQUIRE(prop.major == 10, RKFAC_CUDA_ERROR,
                  "rkfac_b200 requires an sm_100 (B200) device; found sm_" + std::to_string(prop.major) +
                      std::to_string(prop.minor));
}

Plan& cached_plan(Context& c, int d, int r, int p, int q, int method) {
    for (auto& e : c.cache)
        if (e.d == d && e.r == r && e.p == p && e.q == q && e.method == method) return *e.plan;
    rkfac_factor_desc ds{d, r, p, q};
    Context::Cached e{d, r, p, q, method, std::make_unique<Plan>(&c, &ds, 1, method), DevBuf(), DevBuf()};
    const int rr = e.plan->factor(0).r;
    e.ut.alloc(sizeof(float) * (size_t)rr * d);
    e.dv.alloc(sizeof(float) * (size_t)rr);
    c.cache.push_back(std::move(e));
    if (c.cache.size() > 16) c.cache.erase(c.cache.begin());
    return *c.cache.back().plan;
}

Context::Cached& cached_entry(Context& c, const Plan& p) {
    for (auto& e : c.cache)
        if (e.plan.get() == &p) return e;
    throw Error(RKFAC_INVALID_ARGUMENT, "plan cache corrupted");
}

int decompose_single(rkfac_context* ctx, int method, const float* x, int64_t ldx, int64_t d, int64_t r, int64_t p,
                     int64_t q, uint64_t seed, uint64_t* counter, float* u, int64_t ldu, float* dvals,
                     int64_t* rank_out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && x && u && dvals && counter, RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(d >= 1 && r >= 1 && p >= 0 && q >= 0 && ldx >= d, RKFAC_INVALID_ARGUMENT, "bad sizes");
        Context& c = ctx->c;
        Plan& plan = cached_plan(c, (int)d, (int)r, (int)p, (int)q, method);
        auto& entry = cached_entry(c, plan);
        FactorState& F = plan.factor(0);
        RKFAC_REQUIRE(ldu >= F.r, RKFAC_INVALID_ARGUMENT, "ld_u < clamped rank");
        float* X = const_cast<float*>(x);
        float* ut = entry.ut.as<float>();
        float* dv = dvals;
        const long long lx = ldx, lu = d;
        plan.bind_factors(&X, &lx, &ut, &lu, &dv);
        plan.set_explicit_seed(0, seed, *counter);
        plan.decompose(0, 0, 0);
        launch_transpose(ut, d, F.r, (int)d, u, ldu, c.stream);
        *counter += 2ULL * (uint64_t)d * (uint64_t)F.w;  // rng.hpp:59-63 advances 2 per draw
        if (rank_out) *rank_out = F.r;
    });
}

}  // namespace

extern "C" {

const char* rkfac_status_string(int s) {
    switch (s) {
        case RKFAC_OK: return "OK";
        case RKFAC_DIMENSION_MISMATCH: return "DimensionMismatch";
        case RKFAC_RANK_DEFICIENT: return "RankDeficient";
        case RKFAC_NO_CONVERGENCE: return "NoConvergence";
        case RKFAC_DAMPING_NONPOSITIVE: return "DampingNonpositive";
        case RKFAC_CUDA_ERROR: return "CudaError";
        case RKFAC_NCCL_ERROR: return "NcclError";
        case RKFAC_INVALID_ARGUMENT: return "InvalidArgument";
    }
    return "Unknown";
}

int rkfac_create(rkfac_context_t* out, int device, void* stream) {
    return guarded(nullptr, [&] {
        RKFAC_REQUIRE(out, RKFAC_INVALID_ARGUMENT, "null context pointer");
        RKFAC_CUDA(cudaSetDevice(device));
        check_device();
        auto* ctx = new rkfac_context();
        ctx->c.device = device;
        ctx->c.stream = static_cast<cudaStream_t>(stream);
        ctx->c.launches_at_create = launch_counter();
        *out = ctx;
    });
}

int rkfac_destroy(rkfac_context_t ctx) {
    return guarded(nullptr, [&] { delete ctx; });
}

int rkfac_set_stream(rkfac_context_t ctx, void* stream) {
    return guarded(ctx, [&] { ctx->c.stream = static_cast<cudaStream_t>(stream); });
}

int rkfac_synchronize(rkfac_context_t ctx) {
    return guarded(ctx, [&] { RKFAC_CUDA(cudaStreamSynchronize(ctx->c.stream)); });
}

const char* rkfac_last_error(rkfac_context_t ctx) { return ctx ? ctx->c.last_error.c_str() : g_err.c_str(); }

uint64_t rkfac_launch_count(rkfac_context_t ctx) { return launch_counter() - (ctx ? ctx->c.launches_at_create : 0); }

int rkfac_ea_update(rkfac_context_t ctx, float* mbar, int64_t ld_mbar, int64_t d, const float* m, int64_t ld_m,
                    int64_t m_rows, int64_t n, double rho, double scale) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(m_rows == d, RKFAC_DIMENSION_MISMATCH, "ea_update: update row count != factor dimension");
        RKFAC_REQUIRE(ctx && mbar && (m || n == 0), RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(ld_mbar >= d && ld_m >= n, RKFAC_INVALID_ARGUMENT, "leading dimension too small");
        GemmBatch b(GemmKind::F32);
        GemmDesc g = GemmBatch::make((int)d, (int)d, (int)n, m, ld_m, 0, m, ld_m, 1, mbar, ld_mbar, 0);
        g.sym = 1;
        g.alpha = (1.0 - rho) * scale * scale;
        g.beta = rho;
        g.Cin = mbar;
        g.ldcin = ld_mbar;
        b.add(g);
        b.finalize();
        b.launch(ctx->c.stream);  // n == 0 gives K = 0: mbar <- rho * mbar
        RKFAC_CUDA(cudaStreamSynchronize(ctx->c.stream));  // descriptors are freed on return
    });
}

int rkfac_sample_gaussian(rkfac_context_t ctx, uint64_t seed, uint64_t* counter, int64_t m, int64_t n, float* out,
                          int64_t ld_out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && counter && (out || m * n == 0) && ld_out >= n, RKFAC_INVALID_ARGUMENT, "bad argument");
        OmegaDesc o{};
        o.d = (int)m; o.w = (int)n; o.ld = ld_out; o.out = out; o.seed = seed; o.ctr0 = *counter; o.offset = 0;
        o.rowmajor = 1;
        DevBuf b(sizeof(OmegaDesc));
        RKFAC_CUDA(cudaMemcpy(b.p, &o, sizeof(o), cudaMemcpyHostToDevice));
        launch_omega(b.as<OmegaDesc>(), 1, m * n, 0, 0, 0, ctx->c.stream);
        RKFAC_CUDA(cudaStreamSynchronize(ctx->c.stream));
        *counter += 2ULL * (uint64_t)(m * n);
    });
}

int rkfac_srevd(rkfac_context_t ctx, const float* x, int64_t ldx, int64_t d, int64_t r, int64_t p, int64_t q,
                uint64_t seed, uint64_t* counter, float* u, int64_t ldu, float* dvals, int64_t* rank_out) {
    return decompose_single(ctx, RKFAC_SREVD, x, ldx, d, r, p, q, seed, counter, u, ldu, dvals, rank_out);
}

int rkfac_rsvd_psd(rkfac_context_t ctx, const float* x, int64_t ldx, int64_t d, int64_t r, int64_t p, int64_t q,
                   uint64_t seed, uint64_t* counter, float* u, int64_t ldu, float* dvals, int64_t* rank_out) {
    return decompose_single(ctx, RKFAC_RSVD, x, ldx, d, r, p, q, seed, counter, u, ldu, dvals, rank_out);
}

int rkfac_apply_lowrank_damped_inverse(rkfac_context_t ctx, const float* u, int64_t ldu, const float* dvals,
                                       int64_t dim, int64_t r, double lambda, const float* v, int64_t ldv,
                                       int64_t rows, int64_t cols, int side, float* out, int64_t ldo) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
        RKFAC_REQUIRE(side == RKFAC_LEFT || side == RKFAC_RIGHT, RKFAC_INVALID_ARGUMENT, "bad side");
        if (side == RKFAC_LEFT)
            RKFAC_REQUIRE(rows == dim, RKFAC_DIMENSION_MISMATCH, "apply_lowrank_damped_inverse: rows(V) != dim");
        else
            RKFAC_REQUIRE(cols == dim, RKFAC_DIMENSION_MISMATCH, "apply_lowrank_damped_inverse: cols(V) != dim");
        RKFAC_REQUIRE(ctx && u && dvals && v && out && out != v, RKFAC_INVALID_ARGUMENT, "null/aliased argument");
        Context& c = ctx->c;
        const size_t wsz = (size_t)r * (side == RKFAC_LEFT ? cols : rows) + (size_t)r;
        if (c.apply_ws.bytes < wsz * sizeof(float)) c.apply_ws.alloc(wsz * sizeof(float));
        float* W = c.apply_ws.as<float>();
        float* br = W + (size_t)r * (side == RKFAC_LEFT ? cols : rows);
        DevBuf bd;
        {
            BracketDesc b{(int)r, dvals, br};
            bd.alloc(sizeof(BracketDesc));
            RKFAC_CUDA(cudaMemcpy(bd.p, &b, sizeof(b), cudaMemcpyHostToDevice));
            launch_bracket(bd.as<BracketDesc>(), 1, lambda, c.stream);
        }
        GemmBatch g1(GemmKind::F32), g2(GemmKind::F32);
        const double inv = 1.0 / lambda;
        if (side == RKFAC_LEFT) {
            // W = diag(bracket) U^T V (r x cols); out = U W + V / lambda   (kfactor.hpp:147-152)
            GemmDesc a = GemmBatch::make((int)r, (int)cols, (int)dim, u, ldu, 1, v, ldv, 0, W, cols, 0);
            a.rs = br;
            g1.add(a);
            GemmDesc b = GemmBatch::make((int)dim, (int)cols, (int)r, u, ldu, 0, W, cols, 0, out, ldo, 0);
            b.D = v; b.ldd = ldv; b.gamma = inv;
            g2.add(b);
        } else {
            // W = V U diag(bracket) (rows x r); out = W U^T + V / lambda   (kfactor.hpp:156-160)
            GemmDesc a = GemmBatch::make((int)rows, (int)r, (int)dim, v, ldv, 0, u, ldu, 0, W, r, 0);
            a.cs = br;
            g1.add(a);
            GemmDesc b = GemmBatch::make((int)rows, (int)dim, (int)r, W, r, 0, u, ldu, 1, out, ldo, 0);
            b.D = v; b.ldd = ldv; b.gamma = inv;
            g2.add(b);
        }
        g1.finalize();
        g2.finalize();
        g1.launch(c.stream);
        g2.launch(c.stream);
        RKFAC_CUDA(cudaStreamSynchronize(c.stream));
    });
}

int rkfac_plan_create(rkfac_context_t ctx, const rkfac_factor_desc* descs, int n, int method, rkfac_plan_t* out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && out && (descs || n == 0), RKFAC_INVALID_ARGUMENT, "null argument");
        auto* p = new rkfac_plan();
        p->ctx = ctx;
        p->p = std::make_unique<Plan>(&ctx->c, descs, n, method);
        *out = p;
    });
}

int rkfac_plan_destroy(rkfac_plan_t plan) {
    return guarded(nullptr, [&] { delete plan; });
}

int64_t rkfac_plan_rank(rkfac_plan_t plan, int f) {
    if (!plan || f < 0 || f >= plan->p->nfactors()) return -1;
    return plan->p->factor(f).r;
}

int rkfac_plan_bind_factors(rkfac_plan_t plan, float* const* factors, float* const* bases_t, float* const* dvals) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(plan && factors && bases_t && dvals, RKFAC_INVALID_ARGUMENT, "null argument");
        plan->p->bind_factors(factors, nullptr, bases_t, nullptr, dvals);
    });
}

int rkfac_plan_bind_factors_ld(rkfac_plan_t plan, float* const* factors, const int64_t* ld_factors,
                               float* const* bases_t, const int64_t* ld_bases, float* const* dvals) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(plan && factors && bases_t && dvals, RKFAC_INVALID_ARGUMENT, "null argument");
        const int n = plan->p->nfactors();
        std::vector<long long> lx(n), lu(n);
        for (int i = 0; i < n; ++i) {
            lx[i] = ld_factors ? ld_factors[i] : plan->p->factor(i).d;
            lu[i] = ld_bases ? ld_bases[i] : plan->p->factor(i).d;
        }
        plan->p->bind_factors(factors, lx.data(), bases_t, lu.data(), dvals);
    });
}

int rkfac_plan_bind_samples(rkfac_plan_t plan, const float* const* samples, const int64_t* n) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(plan && samples && n, RKFAC_INVALID_ARGUMENT, "null argument");
        plan->p->bind_samples(samples, n);
    });
}

int rkfac_plan_bind_layers(rkfac_plan_t plan, int nlayers, const int* a_idx, const int* g_idx,
                           const float* const* grads, float* const* outs, float* const* mids) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(plan && (nlayers == 0 || (a_idx && g_idx && grads && outs && mids)), RKFAC_INVALID_ARGUMENT,
                      "null argument");
        plan->p->bind_layers(nlayers, a_idx, g_idx, grads, outs, mids);
    });
}

int rkfac_plan_set_tags(rkfac_plan_t plan, const uint64_t* tags) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_tags(tags); });
}

int rkfac_plan_ea_update(rkfac_plan_t plan, double rho, double scale) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->ea_update(rho, scale); });
}

int rkfac_plan_decompose(rkfac_plan_t plan, uint64_t root, uint64_t step) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->decompose(1, root, step); });
}

int rkfac_plan_precondition(rkfac_plan_t plan, double lambda) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->precondition(lambda); });
}

int rkfac_plan_step(rkfac_plan_t plan, double rho, double scale, uint64_t root, uint64_t step, double lambda) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->step(rho, scale, root, step, lambda); });
}

int rkfac_plan_timing(rkfac_plan_t plan, float* sums_ms, int* counts) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->timing_report(sums_ms, counts); });
}

int rkfac_plan_prepare(rkfac_plan_t plan, double rho, double scale, double lambda) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->prepare(rho, scale, lambda); });
}

int rkfac_plan_set_max_ctas(rkfac_plan_t plan, int ctas) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(ctas >= 0, RKFAC_INVALID_ARGUMENT, "negative CTA cap");
        plan->p->set_max_ctas(ctas);
    });
}

int rkfac_plan_set_ea_lo_mode(rkfac_plan_t plan, int mode) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_ea_lo_mode(mode); });
}

int rkfac_plan_set_timing(rkfac_plan_t plan, int enabled) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_timing(enabled != 0); });
}

}  // extern "C"
