// capi.cu -- the extern "C" boundary (include/rkfac_b200.h).  No exception crosses it: every entry point maps
// internal errors to an rkfac_status mirroring the reference's exception types (errors.hpp:8-34).
#include <cstring>
#include <string>

#include "comm.cuh"
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
    return guarded(nullptr, [&] {
        if (ctx && ctx->c.nccl_owned) nccl_comm_destroy(ctx->c.nccl_comm);
        delete ctx;
    });
}

int rkfac_nccl_unique_id(void* id_out) {
    return guarded(nullptr, [&] {
        RKFAC_REQUIRE(id_out, RKFAC_INVALID_ARGUMENT, "null id buffer");
        nccl_unique_id(id_out);
    });
}

int rkfac_nccl_init(rkfac_context_t ctx, const void* unique_id, int nranks, int rank) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && unique_id, RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_CUDA(cudaSetDevice(ctx->c.device));
        void* comm = nccl_comm_init(unique_id, nranks, rank);
        if (ctx->c.nccl_owned) nccl_comm_destroy(ctx->c.nccl_comm);
        ctx->c.nccl_comm = comm;
        ctx->c.nccl_rank = rank;
        ctx->c.nccl_nranks = nranks;
        ctx->c.nccl_owned = true;
    });
}

int rkfac_set_nccl_comm(rkfac_context_t ctx, void* nccl_comm, int nranks, int rank) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx, RKFAC_INVALID_ARGUMENT, "null context");
        RKFAC_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, RKFAC_INVALID_ARGUMENT, "bad NCCL rank / size");
        if (ctx->c.nccl_owned) nccl_comm_destroy(ctx->c.nccl_comm);
        ctx->c.nccl_comm = nccl_comm;
        ctx->c.nccl_rank = rank;
        ctx->c.nccl_nranks = nranks;
        ctx->c.nccl_owned = false;
    });
}

int rkfac_allgather(rkfac_context_t ctx, const float* send, float* recv, int64_t count) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && (count == 0 || (send && recv)), RKFAC_INVALID_ARGUMENT, "null argument");
        if (count == 0) return;
        nccl_allgather(ctx->c.nccl_comm, send, recv, count, ctx->c.stream);
    });
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
        if (d == 0) return;
        // tcgen05 symmetric SYRK + axpy; stages cached per operand set (single.cu), asynchronous on the stream
        ctx->c.single.ea_update(mbar, ld_mbar, (int)d, m, ld_m, (int)n, rho, scale, ctx->c.stream);
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

int rkfac_rsvd(rkfac_context_t ctx, const float* x, int64_t ldx, int64_t rows, int64_t cols, int64_t r, int64_t p,
               int64_t q, uint64_t seed, uint64_t* counter, float* u, int64_t ldu, float* s, float* v, int64_t ldv,
               int64_t* rank_out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && x && u && s && v && counter, RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(rows >= 1 && cols >= 1 && r >= 1 && p >= 0 && q >= 0 && ldx >= cols, RKFAC_INVALID_ARGUMENT,
                      "bad sizes");
        const int64_t dim = std::min(rows, cols);
        const int64_t rc = std::min(r, dim), pc = r > dim ? 0 : std::min(p, dim - rc);
        RKFAC_REQUIRE(ldu >= rc && ldv >= rc, RKFAC_INVALID_ARGUMENT, "ld_u / ld_v < clamped rank");
        int rk = 0;
        ctx->c.rsvd.run(x, ldx, (int)rows, (int)cols, (int)r, (int)p, (int)q, seed, *counter, u, ldu, s, v, ldv, &rk,
                        ctx->c.stream);
        *counter += 2ULL * (uint64_t)cols * (uint64_t)(rc + pc);  // sample_gaussian(rng, cols, width), rng.hpp:59-63
        if (rank_out) *rank_out = rk;
    });
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
        RKFAC_REQUIRE(ldu >= r && ldv >= cols && ldo >= cols, RKFAC_INVALID_ARGUMENT, "leading dimension too small");
        Context& c = ctx->c;
        if (rows == 0 || cols == 0) return;
        if (r == 0) {  // no retained modes: out = V / lambda
            CopyDesc cd{v, out, (int)rows, (int)cols, ldv, ldo, 0};
            DevBuf b(sizeof(cd));
            RKFAC_CUDA(cudaMemcpy(b.p, &cd, sizeof(cd), cudaMemcpyHostToDevice));
            launch_copy(b.as<CopyDesc>(), 1, rows * cols, c.stream);
            launch_scale(out, ldo, (int)rows, (int)cols, (float)(1.0 / lambda), c.stream);
            RKFAC_CUDA(cudaStreamSynchronize(c.stream));  // b is freed on return (degenerate case only)
            return;
        }
        // two tcgen05 GEMMs, bracket scale and +V/lambda fused; stages cached per operand set (single.cu)
        c.single.apply(u, ldu, dvals, (int)dim, (int)r, lambda, v, ldv, (int)rows, (int)cols, side, out, ldo, c.stream);
    });
}

int rkfac_conv_patches(rkfac_context_t ctx, const float* x, int64_t B, int64_t C, int64_t H, int64_t W, int64_t kh,
                       int64_t kw, int64_t sh, int64_t sw, int64_t ph, int64_t pw, int64_t dh, int64_t dw, int ones_row,
                       double scale, float* out, int64_t ld_out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && x && out, RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(B >= 0 && C >= 1 && H >= 1 && W >= 1 && kh >= 1 && kw >= 1 && sh >= 1 && sw >= 1 && ph >= 0 &&
                          pw >= 0 && dh >= 1 && dw >= 1,
                      RKFAC_INVALID_ARGUMENT, "conv_patches: bad geometry");
        const int64_t Ho = (H + 2 * ph - dh * (kh - 1) - 1) / sh + 1, Wo = (W + 2 * pw - dw * (kw - 1) - 1) / sw + 1;
        RKFAC_REQUIRE(Ho >= 1 && Wo >= 1, RKFAC_DIMENSION_MISMATCH, "conv_patches: empty output");
        RKFAC_REQUIRE(ld_out >= B * Ho * Wo, RKFAC_INVALID_ARGUMENT, "conv_patches: ld_out < B*Ho*Wo");
        ConvPatchDesc p{x, (int)B, (int)C, (int)H, (int)W, (int)kh, (int)kw, (int)sh, (int)sw, (int)ph, (int)pw,
                        (int)dh, (int)dw, (int)Ho, (int)Wo, ones_row ? 1 : 0, (float)scale, out, ld_out};
        launch_conv_patches(p, ctx->c.stream);
    });
}

int rkfac_conv_grads(rkfac_context_t ctx, const float* dy, int64_t B, int64_t Co, int64_t Ho, int64_t Wo,
                     double scale, float* out, int64_t ld_out) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && dy && out, RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(B >= 0 && Co >= 1 && Ho >= 1 && Wo >= 1 && ld_out >= B * Ho * Wo, RKFAC_INVALID_ARGUMENT,
                      "conv_grads: bad sizes");
        launch_conv_grads(dy, (int)B, (int)Co, Ho * Wo, (float)scale, out, ld_out, ctx->c.stream);
    });
}

int rkfac_sym_eig(rkfac_context_t ctx, const float* s, int64_t lds, int64_t n, float* p, int64_t ldp, float* dvals,
                  double* dvals64) {
    return guarded(ctx, [&] {
        RKFAC_REQUIRE(ctx && s && (dvals || dvals64), RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(n >= 1 && lds >= n && (!p || ldp >= n), RKFAC_INVALID_ARGUMENT, "bad sizes");
        const double asym = ctx->c.symeig.run(s, lds, (int)n, p, ldp, dvals, dvals64, ctx->c.stream);
        // eig.hpp:213-215 rejects asymmetry above 1e-8 max(1, |S|max) in FP64; FP32 storage rounds at 6e-8, so the
        // bar is 1e4 times that (an FP32 matrix formed as A B^T without symmetrisation passes, a wrong one does not)
        RKFAC_REQUIRE(asym <= 1e-4, RKFAC_DIMENSION_MISMATCH, "sym_eig: matrix is not symmetric");
        RKFAC_CUDA(cudaStreamSynchronize(ctx->c.stream));
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

int rkfac_plan_ea_decompose(rkfac_plan_t plan, double rho, double scale, uint64_t root, uint64_t step) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->ea_decompose(rho, scale, root, step); });
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

int rkfac_plan_set_overlap(rkfac_plan_t plan, int enabled) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_overlap(enabled != 0); });
}

int rkfac_plan_set_step_seed(rkfac_plan_t plan, uint64_t root, uint64_t step) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_step_seed(root, step); });
}

int rkfac_plan_set_max_ctas(rkfac_plan_t plan, int ctas) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(ctas >= 0, RKFAC_INVALID_ARGUMENT, "negative CTA cap");
        plan->p->set_max_ctas(ctas);
    });
}

int rkfac_plan_set_gather(rkfac_plan_t plan, int64_t chunk_elems, const int64_t* offsets, float* gathered) {
    return guarded(plan ? plan->ctx : nullptr, [&] {
        RKFAC_REQUIRE(plan && (!gathered || offsets), RKFAC_INVALID_ARGUMENT, "null argument");
        RKFAC_REQUIRE(!gathered || plan->ctx->c.nccl_comm, RKFAC_INVALID_ARGUMENT,
                      "set_gather: attach an NCCL communicator to the context first (rkfac_nccl_init)");
        std::vector<long long> off;
        if (offsets) off.assign(offsets, offsets + plan->p->nlayers());
        plan->p->set_gather(chunk_elems, off.data(), gathered);
    });
}

int rkfac_plan_gather(rkfac_plan_t plan) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->gather(); });
}

size_t rkfac_plan_workspace_size(rkfac_plan_t plan) { return plan ? plan->p->workspace_bytes() : 0; }

int rkfac_plan_set_ea_lo_mode(rkfac_plan_t plan, int mode) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_ea_lo_mode(mode); });
}

int rkfac_plan_set_timing(rkfac_plan_t plan, int enabled) {
    return guarded(plan ? plan->ctx : nullptr, [&] { plan->p->set_timing(enabled != 0); });
}

}  // extern "C"
