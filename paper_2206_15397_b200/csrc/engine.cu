// engine.cu -- Plan: workspace layout and stage orchestration of the batched rand-K-FAC step.
//
// Data layout in HBM (per factor f, d = dim, w = r + p after clamping, rnla.hpp:35-43):
//   X_f        d x d FP32 EA factor (caller-owned, exactly symmetric)
//   B0, B1     w x d FP32: the sketch Y^T and the orthonormal basis Q^T, ping-ponged (basis vectors contiguous:
//              coalesced epilogue stores, K-major operands for the next product)
//   G, Linv    w x w Gram and inverse Cholesky factor (FP64 for the first orthonormalisations, FP32 after)
//   core       w x w FP32 projected matrix (srevd: Q^T X Q, rnla.hpp:97; rsvd_psd: B B^T, eig.hpp:251)
//   eig        FP64 tridiagonal workspace, P (w x r FP32) eigenvectors of the core
//   Ut         r x d FP32 caller-owned U^T, dvals r FP32 (LowRankEig, rnla.hpp:17-24)
#include <algorithm>
#include <cstring>

#include "engine.cuh"

#include <cstdlib>

namespace rkfac_b200 {

namespace {

struct Carver {
    size_t off = 0;
    template <class T>
    size_t take(size_t count) {
        const size_t o = (off + 255) & ~size_t(255);
        off = o + count * sizeof(T);
        return o;
    }
};

template <class T>
T* at(const DevBuf& b, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(b.p) + off);
}

template <class T>
void upload(DevBuf& buf, const std::vector<T>& v) {
    buf.alloc(sizeof(T) * std::max<size_t>(1, v.size()));
    if (!v.empty()) RKFAC_CUDA(cudaMemcpy(buf.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
}

constexpr double kTol64 = 1e-13;  // relative pivot floor for rank deficiency, FP64 Gram
constexpr double kTol32 = 1e-5;   // FP32 Gram (see cholqr.cu)

}  // namespace

Plan::Plan(Context* ctx, const rkfac_factor_desc* descs, int n, int method) : ctx_(ctx), method_(method) {
    RKFAC_REQUIRE(n >= 0, RKFAC_INVALID_ARGUMENT, "negative factor count");
    RKFAC_REQUIRE(method == RKFAC_SREVD || method == RKFAC_RSVD, RKFAC_INVALID_ARGUMENT, "unknown method");
    f_.resize(n);
    const char* simt = std::getenv("RKFAC_SIMT_XQ");
    use_tc_ = !(simt && simt[0] == '1');
    if (const char* nf = std::getenv("RKFAC_FP64_ORTHS")) n_fp64_orth_ = std::atoi(nf);
    Carver c;
    struct Offs {
        size_t B0, B1, Qh, Ql, Xh, Xl, G64, G32, L64, L32, flags, chol, core, esc, refl, tau, dvec, evec, evals, scr, piv, z, P,
            scale, zflags, bracket;
    };
    std::vector<Offs> offs(n);
    for (int i = 0; i < n; ++i) {
        const auto& ds = descs[i];
        RKFAC_REQUIRE(ds.dim >= 1 && ds.rank >= 1 && ds.oversampling >= 0 && ds.power_iters >= 0,
                      RKFAC_INVALID_ARGUMENT, "invalid factor descriptor");
        FactorState& F = f_[i];
        F.d = (int)ds.dim;
        // rnla.hpp:35-43 clamp_sketch
        long long r = ds.rank, p = ds.oversampling;
        if (r > ds.dim) { r = ds.dim; p = 0; }
        else if (r + p > ds.dim) p = ds.dim - r;
        F.r = (int)r; F.p = (int)p; F.q = (int)ds.power_iters; F.w = (int)(r + p);
        F.tag = (uint64_t)i;
        const size_t w = F.w, d = F.d, rr = F.r;
        RKFAC_REQUIRE(w <= 512, RKFAC_INVALID_ARGUMENT, "sketch width r+p above 512 is not supported");
        wmax_ = std::max(wmax_, F.w);
        rmax_ = std::max(rmax_, F.r);
        Offs& o = offs[i];
        F.dp = (int)((d + 31) / 32 * 32);
        const size_t dp = F.dp;
        o.B0 = c.take<float>(w * dp);
        o.B1 = c.take<float>(w * dp);
        o.Qh = c.take<float>(w * dp);
        o.Ql = c.take<float>(w * dp);
        o.Xh = c.take<float>(d * dp);
        o.Xl = c.take<float>(d * dp);
        o.G64 = c.take<double>(w * w);
        o.G32 = c.take<float>(w * w);
        o.L64 = c.take<double>(w * w);
        o.L32 = c.take<float>(w * w);
        o.flags = c.take<int>(w + 1);
        o.chol = c.take<double>(w * (w + 1) / 2 + w * 8);
        o.core = c.take<float>(w * w);
        o.esc = c.take<double>(w * (w + 1) / 2);
        o.refl = c.take<double>(w * w);
        o.tau = c.take<double>(w);
        o.dvec = c.take<double>(w);
        o.evec = c.take<double>(w);
        o.evals = c.take<double>(w);
        o.scr = c.take<double>(4 * w * rr);
        o.piv = c.take<unsigned char>(w * rr);
        o.z = c.take<double>(w * rr);
        o.P = c.take<float>(w * rr);
        o.scale = c.take<float>(rr);
        o.zflags = c.take<int>(rr + 1);
        o.bracket = c.take<float>(rr);
    }
    arena_.alloc(c.off);
    for (int i = 0; i < n; ++i) {
        FactorState& F = f_[i];
        const Offs& o = offs[i];
        F.B0 = at<float>(arena_, o.B0); F.B1 = at<float>(arena_, o.B1);
        F.Qh = at<float>(arena_, o.Qh); F.Ql = at<float>(arena_, o.Ql);
        F.Xh = at<float>(arena_, o.Xh); F.Xl = at<float>(arena_, o.Xl);
        F.G64 = at<double>(arena_, o.G64); F.G32 = at<float>(arena_, o.G32);
        F.Linv64 = at<double>(arena_, o.L64); F.Linv32 = at<float>(arena_, o.L32);
        F.flags = at<int>(arena_, o.flags);
        F.chol_scratch = at<double>(arena_, o.chol);
        F.core = at<float>(arena_, o.core);
        F.eig_scratch = at<double>(arena_, o.esc);
        F.refl = at<double>(arena_, o.refl); F.tau = at<double>(arena_, o.tau);
        F.dvec = at<double>(arena_, o.dvec); F.evec = at<double>(arena_, o.evec);
        F.evals = at<double>(arena_, o.evals); F.scr = at<double>(arena_, o.scr);
        F.piv = at<unsigned char>(arena_, o.piv); F.z = at<double>(arena_, o.z);
        F.P = at<float>(arena_, o.P); F.scale = at<float>(arena_, o.scale);
        F.zflags = at<int>(arena_, o.zflags); F.bracket = at<float>(arena_, o.bracket);
    }
}

Plan::~Plan() {
    for (auto& e : pool_) cudaEventDestroy(e);
}

double Plan::xq_flops() const {
    double fl = 0;
    for (const auto& F : f_) fl += (2.0 * F.q + 2.0) * 2.0 * F.d * (double)F.d * F.w;
    return fl;
}

void Plan::set_tags(const uint64_t* tags) {
    for (size_t i = 0; i < f_.size(); ++i) f_[i].tag = tags[i];
    if (!omega_.empty()) {
        for (size_t i = 0; i < f_.size(); ++i) omega_[i].tag = tags[i];
        upload(d_omega_, omega_);
    }
}

void Plan::set_explicit_seed(int f, uint64_t seed, uint64_t ctr0) {
    RKFAC_REQUIRE(!omega_.empty(), RKFAC_INVALID_ARGUMENT, "factors not bound");
    omega_[f].seed = seed;
    omega_[f].ctr0 = ctr0;
    upload(d_omega_, omega_);
}

void Plan::bind_factors(float* const* X, const long long* ldx, float* const* Ut, const long long* ldu,
                        float* const* dvals) {
    for (size_t i = 0; i < f_.size(); ++i) {
        FactorState& F = f_[i];
        F.X = X[i];
        F.ldx = ldx ? ldx[i] : F.d;
        F.Ut = Ut[i];
        F.ldu = ldu ? ldu[i] : F.d;
        F.dvals = dvals[i];
        RKFAC_REQUIRE(F.X && F.Ut && F.dvals, RKFAC_INVALID_ARGUMENT, "null factor/basis pointer");
        RKFAC_REQUIRE(F.ldx >= F.d && F.ldu >= F.d, RKFAC_INVALID_ARGUMENT, "leading dimension too small");
    }
    factors_bound_ = true;
    build_decomp_stages();
    ea_rho_ = -1;
    ap_lambda_ = -1;
}

void Plan::bind_samples(const float* const* M, const int64_t* n) {
    for (size_t i = 0; i < f_.size(); ++i) {
        f_[i].M = M[i];
        f_[i].n = n[i];
        RKFAC_REQUIRE(n[i] >= 0, RKFAC_INVALID_ARGUMENT, "negative sample count");
    }
    samples_bound_ = true;
    ea_rho_ = -1;
}

void Plan::bind_layers(int nl, const int* a, const int* g, const float* const* J, float* const* out,
                       float* const* mid) {
    layers_.assign(nl, LayerState{});
    Carver c;
    std::vector<size_t> o1(nl), o2(nl);
    for (int l = 0; l < nl; ++l) {
        RKFAC_REQUIRE(a[l] >= 0 && a[l] < nfactors() && g[l] >= 0 && g[l] < nfactors(), RKFAC_INVALID_ARGUMENT,
                      "layer factor index out of range");
        LayerState& L = layers_[l];
        L.a = a[l]; L.g = g[l];
        L.J = J[l]; L.out = out[l]; L.mid = mid[l];
        const FactorState &A = f_[L.a], &G = f_[L.g];
        o1[l] = c.take<float>((size_t)G.d * A.r);
        o2[l] = c.take<float>((size_t)G.r * A.d);
    }
    layer_arena_.alloc(c.off);
    for (int l = 0; l < nl; ++l) {
        layers_[l].W1 = at<float>(layer_arena_, o1[l]);
        layers_[l].W2 = at<float>(layer_arena_, o2[l]);
    }
    ap_lambda_ = -1;
}

void Plan::build_decomp_stages() {
    const int n = nfactors();
    // Omega descriptors: Omega^T written into B1 (the initial "Q").
    omega_.resize(n);
    long long off = 0;
    for (int i = 0; i < n; ++i) {
        FactorState& F = f_[i];
        OmegaDesc o{};
        o.d = F.d; o.w = F.w; o.ld = F.dp; o.out = F.B1; o.tag = F.tag; o.seed = 0; o.ctr0 = 0; o.offset = off;
        off += (long long)F.d * F.w;
        omega_[i] = o;
    }
    omega_total_ = off;
    upload(d_omega_, omega_);
    std::vector<SplitDesc> sx;
    long long sx_off = 0;
    for (auto& F : f_) {
        sx.push_back(SplitDesc{F.X, F.Xh, F.Xl, F.d, F.d, F.ldx, F.dp, sx_off});
        sx_off += (long long)F.d * F.d;
    }
    upload(d_split_x_, sx);
    split_x_total_ = sx_off;

    for (int dir = 0; dir < 2; ++dir) {
        xq_[dir] = std::make_unique<GemmBatch>(GemmKind::F32);
        gram64_[dir] = std::make_unique<GemmBatch>(GemmKind::F32_ACC64);
        tri64_[dir] = std::make_unique<GemmBatch>(GemmKind::F64_F32);
        gram32_[dir] = std::make_unique<GemmBatch>(GemmKind::F32);
        tri32_[dir] = std::make_unique<GemmBatch>(GemmKind::F32);
        core_[dir] = std::make_unique<GemmBatch>(GemmKind::F32);
        lift_[dir] = std::make_unique<GemmBatch>(GemmKind::F32);
        xq_tc_[dir] = std::make_unique<TcXQ>();
        std::vector<CompleteDesc> comp;
        std::vector<SplitDesc> sq;
        long long sq_off = 0;
        for (auto& F : f_) {
            float* Bd = dir == 0 ? F.B0 : F.B1;  // Y (output of xq_[dir]); src of orth_[dir]
            float* Bo = dir == 0 ? F.B1 : F.B0;  // Q
            // Y^T = (X Q)^T : M=d, N=w, K=d
            xq_[dir]->add(GemmBatch::make(F.d, F.w, F.d, F.X, F.ldx, 0, Bo, F.dp, 1, Bd, F.dp, 1));
            xq_tc_[dir]->add(TcOperand{F.Xh, F.Xl, F.dp}, TcOperand{F.Qh, F.Ql, F.dp}, F.d, F.w, F.d, Bd, F.dp);
            sq.push_back(SplitDesc{Bo, F.Qh, F.Ql, F.w, F.d, F.dp, F.dp, sq_off});
            sq_off += (long long)F.w * F.d;
            // orth of B[dir] into B[dir^1]: G = Y^T Y (w x w), then Q^T = Linv Y^T
            GemmDesc g64 = GemmBatch::make(F.w, F.w, F.d, Bd, F.dp, 0, Bd, F.dp, 1, F.G64, F.w, 0);
            g64.ksplit = choose_ksplit(F.w, F.w, F.d, 64, 64);
            gram64_[dir]->add(g64);
            tri64_[dir]->add(GemmBatch::make(F.w, F.d, F.w, F.Linv64, F.w, 0, Bd, F.dp, 0, Bo, F.dp, 0));
            GemmDesc g32 = GemmBatch::make(F.w, F.w, F.d, Bd, F.dp, 0, Bd, F.dp, 1, F.G32, F.w, 0);
            g32.ksplit = choose_ksplit(F.w, F.w, F.d, 128, 128);
            gram32_[dir]->add(g32);
            tri32_[dir]->add(GemmBatch::make(F.w, F.d, F.w, F.Linv32, F.w, 0, Bd, F.dp, 0, Bo, F.dp, 0));
            comp.push_back(CompleteDesc{F.w, F.d, F.dp, Bo, F.flags, F.flags + F.w});
            // core: srevd C = Q^T (X Q) (rnla.hpp:97); rsvd_psd Gram B B^T = Y^T Y (eig.hpp:251)
            const float* Aop = method_ == RKFAC_SREVD ? Bo : Bd;
            GemmDesc cd = GemmBatch::make(F.w, F.w, F.d, Aop, F.dp, 0, Bd, F.dp, 1, F.core, F.w, 0);
            cd.ksplit = choose_ksplit(F.w, F.w, F.d, 128, 128);
            core_[dir]->add(cd);
            // lift: srevd U^T = P_r^T Q^T (rnla.hpp:101); rsvd U^T = diag(1/s) P_r^T Y^T (eig.hpp:260-266)
            const float* Bop = method_ == RKFAC_SREVD ? Bo : Bd;
            GemmDesc ld = GemmBatch::make(F.r, F.d, F.w, F.P, F.r, 1, Bop, F.dp, 0, F.Ut, F.ldu, 0);
            if (method_ == RKFAC_RSVD) ld.rs = F.scale;
            lift_[dir]->add(ld);
        }
        // complete_[dir] completes the output of orth_from(dir) (which is B[dir^1]).
        upload(d_complete_[dir], comp);
        upload(d_split_q_[dir], sq);
        split_q_total_ = sq_off;
        xq_tc_[dir]->finalize();
        xq_[dir]->finalize(); gram64_[dir]->finalize(); tri64_[dir]->finalize();
        gram32_[dir]->finalize(); tri32_[dir]->finalize(); core_[dir]->finalize(); lift_[dir]->finalize();
    }
    std::vector<CholDesc> c64, c32;
    std::vector<EigDesc> eg;
    std::vector<PostDesc> po;
    std::vector<CompleteDesc> cu;
    std::vector<BracketDesc> br;
    for (auto& F : f_) {
        c64.push_back(CholDesc{F.w, F.G64, F.Linv64, F.flags, F.flags + F.w, F.chol_scratch});
        c32.push_back(CholDesc{F.w, F.G32, F.Linv32, F.flags, F.flags + F.w, F.chol_scratch});
        EigDesc e{};
        e.n = F.w; e.r = F.r; e.A = F.core; e.lda = F.w; e.scratch = F.eig_scratch; e.refl = F.refl;
        e.tau = F.tau; e.dvec = F.dvec; e.evec = F.evec; e.evals = F.evals; e.scr = F.scr; e.piv = F.piv;
        e.z = F.z; e.P = F.P; e.ldp = F.r;
        eg.push_back(e);
        po.push_back(PostDesc{F.r, method_, F.evals, F.dvals, F.scale, F.zflags, F.zflags + F.r});
        cu.push_back(CompleteDesc{F.r, F.d, F.ldu, F.Ut, F.zflags, F.zflags + F.r});
        br.push_back(BracketDesc{F.r, F.dvals, F.bracket});
    }
    upload(d_chol64_, c64);
    upload(d_chol32_, c32);
    upload(d_eig_, eg);
    upload(d_post_, po);
    upload(d_complete_u_, cu);
    upload(d_bracket_, br);
}

void Plan::build_ea_stage(double rho, double scale) {
    ea_ = std::make_unique<GemmBatch>(GemmKind::F32);
    for (auto& F : f_) {
        if (!F.M || F.n == 0) continue;
        GemmDesc d = GemmBatch::make(F.d, F.d, (int)F.n, F.M, F.n, 0, F.M, F.n, 1, F.X, F.ldx, 0);
        d.sym = 1;
        d.alpha = (1.0 - rho) * scale * scale;
        d.beta = rho;
        d.Cin = F.X;
        d.ldcin = F.ldx;
        ea_->add(d);
    }
    ea_->finalize();
    ea_rho_ = rho;
    ea_scale_ = scale;
}

void Plan::build_apply_stages(double lambda) {
    for (auto& a : ap_) a = std::make_unique<GemmBatch>(GemmKind::F32);
    const double inv = 1.0 / lambda;
    for (auto& L : layers_) {
        const FactorState &A = f_[L.a], &G = f_[L.g];
        // RIGHT (kfactor.hpp:156-160): W1 = J U_A diag(bracket_A); mid = W1 U_A^T + J / lambda
        GemmDesc d0 = GemmBatch::make(G.d, A.r, A.d, L.J, A.d, 0, A.Ut, A.ldu, 1, L.W1, A.r, 0);
        d0.cs = A.bracket;
        ap_[0]->add(d0);
        GemmDesc d1 = GemmBatch::make(G.d, A.d, A.r, L.W1, A.r, 0, A.Ut, A.ldu, 0, L.mid, A.d, 0);
        d1.D = L.J; d1.ldd = A.d; d1.gamma = inv;
        ap_[1]->add(d1);
        // LEFT (kfactor.hpp:147-152): W2 = diag(bracket_G) U_G^T mid; out = U_G W2 + mid / lambda
        GemmDesc d2 = GemmBatch::make(G.r, A.d, G.d, G.Ut, G.ldu, 0, L.mid, A.d, 0, L.W2, A.d, 0);
        d2.rs = G.bracket;
        d2.ksplit = choose_ksplit(G.r, A.d, G.d, 128, 128);
        ap_[2]->add(d2);
        GemmDesc d3 = GemmBatch::make(G.d, A.d, G.r, G.Ut, G.ldu, 1, L.W2, A.d, 0, L.out, A.d, 0);
        d3.D = L.mid; d3.ldd = A.d; d3.gamma = inv;
        ap_[3]->add(d3);
    }
    for (auto& a : ap_) a->finalize();
    ap_lambda_ = lambda;
}

void Plan::orth(int src, int dst, bool fp64, cudaStream_t s) {
    (void)dst;
    const int n = nfactors();
    if (fp64) {
        gram64_[src]->launch(s);
        launch_cholinv(d_chol64_.as<CholDesc>(), n, wmax_, true, true, kTol64, s);
        tri64_[src]->launch(s);
    } else {
        gram32_[src]->launch(s);
        launch_cholinv(d_chol32_.as<CholDesc>(), n, wmax_, false, false, kTol32, s);
        tri32_[src]->launch(s);
    }
    launch_complete(d_complete_[src].as<CompleteDesc>(), n, s);
}

// ---- stage timing: CUDA events from a pool, recorded on the context stream, harvested after the caller syncs
// (no host synchronisation inside a step).  Kinds: see TimingKind.
void Plan::mark(int kind, bool begin) {
    if (!timing_) return;
    if (pool_used_ == pool_.size()) {
        cudaEvent_t e;
        RKFAC_CUDA(cudaEventCreate(&e));
        pool_.push_back(e);
    }
    const size_t idx = pool_used_++;
    RKFAC_CUDA(cudaEventRecord(pool_[idx], ctx_->stream));
    if (begin) open_[kind] = idx;
    else recs_.push_back({kind, open_[kind], idx});
}

void Plan::timing_reset() {
    pool_used_ = 0;
    recs_.clear();
}

void Plan::timing_report(float* sums, int* counts) const {
    for (int k = 0; k < kTimingKinds; ++k) { sums[k] = 0.f; counts[k] = 0; }
    for (const auto& r : recs_) {
        float t = 0.f;
        RKFAC_CUDA(cudaEventElapsedTime(&t, pool_[r.b], pool_[r.e]));
        sums[r.kind] += t;
        counts[r.kind] += 1;
    }
}

void Plan::ea_update(double rho, double scale) {
    RKFAC_REQUIRE(factors_bound_ && samples_bound_, RKFAC_INVALID_ARGUMENT, "factors/samples not bound");
    if (rho != ea_rho_ || scale != ea_scale_) build_ea_stage(rho, scale);
    mark(kEA, true);
    ea_->launch(ctx_->stream);
    mark(kEA, false);
}

void Plan::decompose(int mode, uint64_t root, uint64_t step) {
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    cudaStream_t s = ctx_->stream;
    const int n = nfactors();
    if (n == 0) return;
    int qmax = 0;
    for (auto& F : f_) qmax = std::max(qmax, F.q);
    for (auto& F : f_)
        RKFAC_REQUIRE(F.q == qmax, RKFAC_INVALID_ARGUMENT, "all factors of a plan share power_iters");
    mark(kDecompose, true);
    launch_omega(d_omega_.as<OmegaDesc>(), n, omega_total_, mode, root, step, s);
    int cur_q = 1;  // Q lives in B[cur_q]
    const int north = 2 * qmax + 1;
    bool last_fp64 = false;
    if (use_tc_) launch_split(d_split_x_.as<SplitDesc>(), n, split_x_total_, s);
    auto timed_xq = [&](int y) {
        if (use_tc_) launch_split(d_split_q_[y].as<SplitDesc>(), n, split_q_total_, s);
        mark(kXQ, true);
        if (use_tc_) xq_tc_[y]->launch(s); else xq_[y]->launch(s);
        mark(kXQ, false);
    };
    for (int o = 0; o < north; ++o) {
        const int y = cur_q ^ 1;
        timed_xq(y);
        last_fp64 = o < n_fp64_orth_;
        mark(kOrth, true);
        orth(y, cur_q, last_fp64, s);
        mark(kOrth, false);
    }
    if (!last_fp64) {  // CholeskyQR2: second pass so the final basis is orthonormal to FP32 rounding
        mark(kOrth, true);
        orth(cur_q, cur_q ^ 1, false, s);
        mark(kOrth, false);
        cur_q ^= 1;
    }
    const int y = cur_q ^ 1;
    timed_xq(y);
    mark(kEig, true);
    core_[y]->launch(s);
    launch_eig(d_eig_.as<EigDesc>(), n, wmax_, rmax_, s);
    launch_post(d_post_.as<PostDesc>(), n, s);
    lift_[y]->launch(s);
    if (method_ == RKFAC_RSVD) launch_complete(d_complete_u_.as<CompleteDesc>(), n, s);
    mark(kEig, false);
    mark(kDecompose, false);
}

void Plan::precondition(double lambda) {
    RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    if (layers_.empty()) return;
    if (lambda != ap_lambda_) build_apply_stages(lambda);
    cudaStream_t s = ctx_->stream;
    mark(kApply, true);
    launch_bracket(d_bracket_.as<BracketDesc>(), nfactors(), lambda, s);
    for (auto& a : ap_) a->launch(s);
    mark(kApply, false);
}

void Plan::step(double rho, double scale, uint64_t root, uint64_t stp, double lambda) {
    RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
    mark(kStep, true);
    if (samples_bound_) ea_update(rho, scale);
    decompose(1, root, stp);
    precondition(lambda);
    mark(kStep, false);
}

}  // namespace rkfac_b200
