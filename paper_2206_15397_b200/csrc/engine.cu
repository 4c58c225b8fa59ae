// engine.cu -- Plan: workspace layout and stage orchestration of the batched rand-K-FAC step.
//
// Data layout in HBM (per factor f, d = dim, w = r + p after clamping, rnla.hpp:35-43; dp = d rounded up to 32,
// wp = w rounded up to 4 so every row pitch is a legal TMA stride):
//   X_f        d x d FP32 EA factor (caller-owned, exactly symmetric); its TF32 lo plane is never stored: the
//              X*Q products form it in shared memory from each TMA-loaded tile (tc_gemm.cu converter warps)
//   S[0],S[1]  ping-pong sketch / basis roles, each in four planes: T = w x d (basis vectors contiguous: the
//              K-major operand of X*Q, Y^T Y and Q^T Y), R = d x w (the K-major operand of Y L^-T), and the TF32
//              lo planes of both (3xTF32 operands); every producer writes all four in its epilogue
//   G, Linv    w x w Gram and inverse Cholesky factor (FP64 for the first orthonormalisation, FP32 after)
//   core       w x w FP32 projected matrix (srevd: Q^T X Q, rnla.hpp:97; rsvd_psd: B B^T, eig.hpp:251)
//   eig        FP64 tridiagonal workspace, P (w x r FP32) eigenvectors of the core
//   Ut         r x d FP32 caller-owned U^T, dvals r FP32 (LowRankEig, rnla.hpp:17-24)
#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>

#include "comm.cuh"
#include "engine.cuh"

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

TcOut out_t(float* p, long long ld) { TcOut o; o.p = p; o.ld = ld; o.t = 1; return o; }
// The tensor core's FP32 accumulation truncates: the error of one TMEM accumulation chain grows linearly with its
// length (tools/tc_acc.cu, 3xTF32: 7.5e-6 at K = 1024, 2.9e-5 at K = 4096, 1.2e-4 at K = 16384).  The products
// whose accuracy reaches the outputs -- the Gram matrices of the orthonormalisation, the final X*Q, the core
// Q^T X Q and the two long-K products of the apply stage -- are split into K slices of at most kSliceK (partials
// summed in FP32 by the deterministic split-K reduction).  The intermediate power products only carry a subspace
// and stay unsplit.  Measured on d = 16384 (config 5) against an FP64 restatement: eigenvalue error 1.8e-4 ->
// 1.4e-5, orthonormality 1.1e-4 -> 7.8e-6.
constexpr int kSliceK = 512;
constexpr int kSliceKFinal = 1024;
// EA updates with more samples than this (convolution statistics) run as K-sliced products + a symmetrize pass
constexpr int kEaLongK = 512;
// The apply's long-K products: at most 8 slices of at least 512 (a slice is one TMEM chain: its length is the
// latency of the product -- 2048-long slices put ~100 us on a VGG16 group's critical path -- while more slices write
// more d_G x r partials: 1 GB per layer at d = 16384 with 512-slices)
static int apply_slice(int K) { return std::max(512, (K + 7) / 8); }

TcOut out_r(float* p, long long ld) { TcOut o; o.p = p; o.ld = ld; o.t = 0; return o; }

}  // namespace

Plan::Plan(Context* ctx, const rkfac_factor_desc* descs, int n, int method) : ctx_(ctx), method_(method) {
    RKFAC_REQUIRE(n >= 0, RKFAC_INVALID_ARGUMENT, "negative factor count");
    RKFAC_REQUIRE(method == RKFAC_SREVD || method == RKFAC_RSVD, RKFAC_INVALID_ARGUMENT, "unknown method");
    f_.resize(n);
    if (const char* nf = std::getenv("RKFAC_FP64_ORTHS")) n_fp64_orth_ = std::atoi(nf);
    if (const char* ov = std::getenv("RKFAC_OVERLAP_ORTH")) overlap_orth_ = std::atoi(ov) != 0;
    if (const char* et = std::getenv("RKFAC_EXPLICIT_TAIL")) explicit_tail_ = std::max(0, std::atoi(et));
    {
        // side stream of the overlapped power iteration (Gram + Cholesky-inverse next to the product): the latency-
        // bound chain gets the highest priority so its small grids take SMs as soon as they drain
        int lo_pri = 0, hi_pri = 0;
        RKFAC_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        RKFAC_CUDA(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, hi_pri));
        RKFAC_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
        RKFAC_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
        RKFAC_CUDA(cudaEventCreateWithFlags(&ev_pre_, cudaEventDisableTiming));
        RKFAC_CUDA(cudaEventCreateWithFlags(&ev_copy_, cudaEventDisableTiming));
    }
    // The side stream doubles the streams of a multi-group step; with the driver's default of 8 hardware work queues
    // streams then share queues and serialise falsely (measured: 5 groups eager 7.3 -> 11.0 ms), so the overlap is
    // on only when the process raised CUDA_DEVICE_MAX_CONNECTIONS (the Python package sets 32 at import).
    if (const char* mc = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS")) step_overlap_ = std::atoi(mc) >= 16;
    if (const char* so = std::getenv("RKFAC_STEP_OVERLAP")) step_overlap_ = std::atoi(so) != 0;
    Carver c;
    struct Offs {
        size_t S[2][4], Xc, G64, G32, L64, L32, L32lo, flags, chol, core, esc, refl, tau, dvec, evec, evals,
            scr, piv, z, Pt, Ptlo, scale, zflags, bracket, Uti, Utilo, Ui, Uilo;
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
        F.dp = (F.d + 31) / 32 * 32;
        F.wp = (F.w + 3) / 4 * 4;
        RKFAC_REQUIRE(F.w <= 512, RKFAC_INVALID_ARGUMENT, "sketch width r+p above 512 is not supported");
        wmax_ = std::max(wmax_, F.w);
        rmax_ = std::max(rmax_, F.r);
        const size_t w = F.w, d = F.d, rr = F.r, dp = F.dp, wp = F.wp;
        Offs& o = offs[i];
        for (int s = 0; s < 2; ++s) {
            o.S[s][0] = c.take<float>(w * dp);
            o.S[s][1] = c.take<float>(w * dp);
            o.S[s][2] = c.take<float>(d * wp);
            o.S[s][3] = c.take<float>(d * wp);
        }
        o.Xc = c.take<float>(d * dp);
        o.G64 = c.take<double>(w * wp);
        o.G32 = c.take<float>(w * wp);
        o.L64 = c.take<double>(w * wp);
        o.L32 = c.take<float>(w * wp);
        o.L32lo = c.take<float>(w * wp);
        o.flags = c.take<int>(w + 1);
        o.chol = c.take<double>(w * (w + 1) / 2 + 8 * w + 16);  // padded, skewed packed triangle (cholqr.cu prow)
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
        o.Pt = c.take<float>(rr * wp);
        o.Ptlo = c.take<float>(rr * wp);
        o.scale = c.take<float>(rr);
        o.zflags = c.take<int>(rr + 1);
        o.bracket = c.take<float>(rr);
        F.rp = (F.r + 3) / 4 * 4;
        o.Uti = c.take<float>(rr * dp);
        o.Utilo = c.take<float>(rr * dp);
        o.Ui = c.take<float>(d * F.rp);
        o.Uilo = c.take<float>(d * F.rp);
    }
    arena_.alloc(c.off);
    RKFAC_CUDA(cudaMemset(arena_.p, 0, c.off));
    for (int i = 0; i < n; ++i) {
        FactorState& F = f_[i];
        const Offs& o = offs[i];
        for (int s = 0; s < 2; ++s) {
            F.S[s].T = at<float>(arena_, o.S[s][0]);
            F.S[s].Tlo = at<float>(arena_, o.S[s][1]);
            F.S[s].R = at<float>(arena_, o.S[s][2]);
            F.S[s].Rlo = at<float>(arena_, o.S[s][3]);
        }
        F.Xc = at<float>(arena_, o.Xc);
        F.G64 = at<double>(arena_, o.G64); F.G32 = at<float>(arena_, o.G32);
        F.Linv64 = at<double>(arena_, o.L64); F.Linv32 = at<float>(arena_, o.L32);
        F.Linv32lo = at<float>(arena_, o.L32lo);
        F.flags = at<int>(arena_, o.flags);
        F.chol_scratch = at<double>(arena_, o.chol);
        F.core = at<float>(arena_, o.core);
        F.eig_scratch = at<double>(arena_, o.esc);
        F.refl = at<double>(arena_, o.refl); F.tau = at<double>(arena_, o.tau);
        F.dvec = at<double>(arena_, o.dvec); F.evec = at<double>(arena_, o.evec);
        F.evals = at<double>(arena_, o.evals); F.scr = at<double>(arena_, o.scr);
        F.piv = at<unsigned char>(arena_, o.piv); F.z = at<double>(arena_, o.z);
        F.Pt = at<float>(arena_, o.Pt); F.Ptlo = at<float>(arena_, o.Ptlo); F.scale = at<float>(arena_, o.scale);
        F.zflags = at<int>(arena_, o.zflags); F.bracket = at<float>(arena_, o.bracket);
        F.Uti = at<float>(arena_, o.Uti); F.Utilo = at<float>(arena_, o.Utilo);
        F.Ui = at<float>(arena_, o.Ui); F.Uilo = at<float>(arena_, o.Uilo);
    }
}

Plan::~Plan() {
    for (auto& e : pool_) cudaEventDestroy(e);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_pre_) cudaEventDestroy(ev_pre_);
    if (ev_copy_) cudaEventDestroy(ev_copy_);
    if (side_) cudaStreamDestroy(side_);
    if (h_seed_) cudaFreeHost(h_seed_);
}

double Plan::xq_flops() const {
    double fl = 0;
    for (const auto& F : f_) fl += 2.0 * F.d * (double)F.d * F.w;
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
    if (factors_bound_) {  // re-binding the same buffers (repeated single-factor calls): the stages are still valid
        bool same = true;
        for (size_t i = 0; i < f_.size() && same; ++i) {
            const FactorState& F = f_[i];
            same = F.X == X[i] && F.ldx == (ldx ? ldx[i] : F.d) && F.Ut == Ut[i] && F.ldu == (ldu ? ldu[i] : F.d) &&
                   F.dvals == dvals[i];
        }
        if (same) return;
    }
    x_tma_ok_ = true;
    for (size_t i = 0; i < f_.size(); ++i) {
        FactorState& F = f_[i];
        F.X = X[i];
        F.ldx = ldx ? ldx[i] : F.d;
        F.Ut = Ut[i];
        F.ldu = ldu ? ldu[i] : F.d;
        F.dvals = dvals[i];
        RKFAC_REQUIRE(F.X && F.Ut && F.dvals, RKFAC_INVALID_ARGUMENT, "null factor/basis pointer");
        RKFAC_REQUIRE(F.ldx >= F.d && F.ldu >= F.d, RKFAC_INVALID_ARGUMENT, "leading dimension too small");
        x_tma_ok_ = x_tma_ok_ && tc_operand_ok(F.X, F.ldx) && F.ldx <= F.dp;
    }
    for (auto& F : f_) F.ldxa = x_tma_ok_ ? F.ldx : F.dp;
    factors_bound_ = true;
    build_decomp_stages();
    ea_rho_ = -1;
    ap_lambda_ = -1;
}

void Plan::set_ea_lo_mode(int mode) {
    RKFAC_REQUIRE(mode >= -1 && mode <= 1, RKFAC_INVALID_ARGUMENT, "EA lo mode must be -1, 0 or 1");
    ea_lo_mode_ = mode;
    ea_rho_ = -1;  // rebuilt on the next EA update
}

void Plan::bind_samples(const float* const* M, const int64_t* n) {
    bool ok = true;
    Carver c;
    std::vector<size_t> off(f_.size());
    for (size_t i = 0; i < f_.size(); ++i) {
        FactorState& F = f_[i];
        F.M = M[i];
        F.n = n[i];
        F.ldm = n[i];
        RKFAC_REQUIRE(n[i] >= 0, RKFAC_INVALID_ARGUMENT, "negative sample count");
        ok = ok && (F.n == 0 || tc_operand_ok(F.M, F.ldm));
        off[i] = c.take<float>((size_t)F.d * std::max<long long>(F.n, 1));
    }
    ml_arena_.alloc(c.off);
    for (size_t i = 0; i < f_.size(); ++i) f_[i].Ml = at<float>(ml_arena_, off[i]);
    samples_tma_ok_ = ok;
    samples_bound_ = true;
    ea_rho_ = -1;
}

void Plan::bind_layers(int nl, const int* a, const int* g, const float* const* J, float* const* out,
                       float* const* mid) {
    layers_.assign(nl, LayerState{});
    Carver c;
    std::vector<std::array<size_t, 8>> o(nl);
    for (int l = 0; l < nl; ++l) {
        RKFAC_REQUIRE(a[l] >= 0 && a[l] < nfactors() && g[l] >= 0 && g[l] < nfactors(), RKFAC_INVALID_ARGUMENT,
                      "layer factor index out of range");
        LayerState& L = layers_[l];
        L.a = a[l]; L.g = g[l];
        L.J = J[l]; L.out = out[l]; L.mid = mid[l];
        const FactorState &A = f_[L.a], &G = f_[L.g];
        const size_t dAp = (A.d + 3) / 4 * 4, dGp = (G.d + 3) / 4 * 4;
        o[l][0] = c.take<float>((size_t)G.d * dAp);
        o[l][1] = c.take<float>((size_t)G.d * dAp);
        o[l][2] = c.take<float>((size_t)G.d * A.rp);
        o[l][3] = c.take<float>((size_t)G.d * A.rp);
        o[l][4] = c.take<float>((size_t)A.d * dGp);
        o[l][5] = c.take<float>((size_t)A.d * dGp);
        o[l][6] = c.take<float>((size_t)A.d * G.rp);
        o[l][7] = c.take<float>((size_t)A.d * G.rp);
    }
    layer_arena_.alloc(c.off);
    std::vector<SplitDesc> sj;
    long long off = 0;
    for (int l = 0; l < nl; ++l) {
        LayerState& L = layers_[l];
        L.Jc = at<float>(layer_arena_, o[l][0]); L.Jlo = at<float>(layer_arena_, o[l][1]);
        L.W1 = at<float>(layer_arena_, o[l][2]); L.W1lo = at<float>(layer_arena_, o[l][3]);
        L.Mt = at<float>(layer_arena_, o[l][4]); L.Mtlo = at<float>(layer_arena_, o[l][5]);
        L.W2t = at<float>(layer_arena_, o[l][6]); L.W2tlo = at<float>(layer_arena_, o[l][7]);
        const FactorState &A = f_[L.a], &G = f_[L.g];
        const long long dAp = (A.d + 3) / 4 * 4;
        sj.push_back(SplitDesc{L.J, L.Jc, nullptr, G.d, A.d, A.d, dAp, off});  // aligned copy (lo formed in smem)
        off += (long long)G.d * A.d;
    }
    upload(d_split_j_, sj);
    split_j_total_ = off;
    ap_lambda_ = -1;
}

void Plan::build_decomp_stages() {
    const int n = nfactors();
    // Omega^T written into S[1].T (the initial basis role) together with its TF32 lo plane.
    omega_.resize(n);
    long long off = 0;
    std::vector<SplitDesc> so;
    for (int i = 0; i < n; ++i) {
        FactorState& F = f_[i];
        OmegaDesc o{};
        o.d = F.d; o.w = F.w; o.ld = F.dp; o.out = F.S[1].T; o.tag = F.tag; o.seed = 0; o.ctr0 = 0; o.offset = off;
        o.out_lo = F.S[1].Tlo;
        so.push_back(SplitDesc{F.S[1].T, nullptr, F.S[1].Tlo, F.w, F.d, F.dp, F.dp, off});
        off += (long long)F.d * F.w;
        omega_[i] = o;
    }
    omega_total_ = off;
    upload(d_omega_, omega_);
    upload(d_split_omega_, so);
    // padded copy of X when X itself is not a legal TMA operand
    std::vector<SplitDesc> sx;
    long long sx_off = 0;
    for (auto& F : f_) {
        sx.push_back(SplitDesc{F.X, F.Xc, nullptr, F.d, F.d, F.ldx, F.ldxa, sx_off});
        sx_off += (long long)F.d * F.d;
    }
    upload(d_split_x_, sx);
    split_x_total_ = sx_off;

    for (int dir = 0; dir < 2; ++dir) {
        xq_[dir] = new_tc();
        xqf_[dir] = new_tc();
        xq_t_[dir] = new_tc();
        xq_tl_[dir] = new_tc();
        xz_[dir] = new_tc();
        // the long-K products run on CTA pairs (cta_group::2; tc_gemm.cu kCfg 3): RKFAC_XQ_PAIR=0 disables
        static const bool pair_xq = [] {
            const char* e = std::getenv("RKFAC_XQ_PAIR");
            return !(e && e[0] == '0');
        }();
        for (TcGemm* g : {xq_[dir].get(), xqf_[dir].get(), xq_t_[dir].get(), xq_tl_[dir].get(), xz_[dir].get()})
            g->set_two_cta(pair_xq);
        gram_[dir] = new_tc();
        tri_[dir] = new_tc();
        tri_t_[dir] = new_tc();
        core_[dir] = new_tc();
        gram64_[dir] = std::make_unique<Gram64Batch>();
        tri64_[dir] = std::make_unique<Tri64Batch>();
        lift_[dir] = new_tc();
        std::vector<CompleteDesc> comp;
        for (auto& F : f_) {
            Role& Y = F.S[dir];      // written by xq_[dir]; source of the orthonormalisation indexed dir
            Role& Q = F.S[dir ^ 1];  // basis read by xq_[dir]; destination of orth(src = dir)
            const float* Xop = x_tma_ok_ ? F.X : F.Xc;
            // Y = X Q (Y^T with its TF32 lo plane for the Gram and the core; Y row-major without: the Y L^-T and lift
            // products form that lo plane in smem -- measured: forming Y^T's lo plane in the Gram too is slower):
            // A = X (d x d), B = Q^T (w x d)
            {
                TcProblemDesc p;
                p.M = F.d; p.N = F.w; p.K = F.d;
                p.A = Xop; p.A_lo = nullptr; p.lda = F.ldxa;  // X's lo plane is formed in shared memory
                p.B = Q.T; p.B_lo = Q.Tlo; p.ldb = F.dp;
                p.out0 = out_t(Y.T, F.dp); p.lo0 = out_t(Y.Tlo, F.dp);
                p.out1 = out_r(Y.R, F.wp);
                // unsplit: K slices of 1-2K for the power products were measured 30-40 % slower (partials + the
                // 4-output reduction) without shortening the step
                // (N tiles of 128 instead of one 240-column tile: measured 46 % slower; splitting only the d >= 4096
                // factors' K in two: X*Q stage 3.28 -> 4.18 ms)
                xq_[dir]->add(p);
                // the products whose Y planes feed only T-plane consumers: before an FP64 orthonormalisation (its Gram
                // and Y L^-T read Y^T) and, for srevd, the final product (the core reads Y^T; the lift reads Q)
                TcProblemDesc pt = p;
                pt.out1 = TcOut{};
                pt.lo0 = TcOut{};  // the FP64 Gram and Y L^-T read Y^T itself (FP64 DMMA), not its TF32 lo plane
                xq_t_[dir]->add(pt);
                // the overlapped power iteration (decompose): Y1 = X Q0 feeds the Gram and the next product (Y^T and
                // its lo plane only); Z = X Y is read by Z L^-T as a row-major operand only
                TcProblemDesc ptl = p;
                ptl.out1 = TcOut{};
                xq_tl_[dir]->add(ptl);
                TcProblemDesc pz = p;
                pz.out0 = out_r(Y.R, F.wp);
                pz.out1 = TcOut{};
                pz.lo0 = TcOut{};
                xz_[dir]->add(pz);
                p.slice_k = kSliceKFinal;
                if (method_ == RKFAC_SREVD) p.out1 = TcOut{};
                xqf_[dir]->add(p);

            }
            // FP32 CholeskyQR of Y into Q:  G = Y^T Y (A = B = Y^T), then Q = Y L^-T (A = Y, B = Linv)
            {
                TcProblemDesc g;
                g.M = F.w; g.N = F.w; g.K = F.d;
                g.A = Y.T; g.A_lo = Y.Tlo; g.lda = F.dp;
                g.B = Y.T; g.B_lo = Y.Tlo; g.ldb = F.dp;
                g.out0 = out_r(F.G32, F.wp);
                g.slice_k = kSliceK;  // (256 / 128 measured slower: more partials summed by the Cholesky-inverse)
                gram_[dir]->add(g);
                TcProblemDesc t;
                t.M = F.d; t.N = F.w; t.K = F.w;
                t.A = Y.R; t.A_lo = nullptr; t.lda = F.wp;
                t.B = F.Linv32; t.B_lo = F.Linv32lo; t.ldb = F.wp;
                t.out0 = out_t(Q.T, F.dp); t.lo0 = out_t(Q.Tlo, F.dp);
                tri_t_[dir]->add(t);  // intermediate bases: only the X*Q operand planes (Q^T and its lo plane)
                t.out1 = out_r(Q.R, F.wp);
                tri_[dir]->add(t);
            }
            // FP64 CholeskyQR of Y into Q (DMMA): G = Y^T Y in FP64, Q^T = Linv Y^T with FP64 accumulation
            gram64_[dir]->add(F.w, F.d, Y.T, F.dp, F.G64, F.wp);
            tri64_[dir]->add(F.w, F.d, F.Linv64, F.wp, Y.T, F.dp, Q.T, Q.Tlo, F.dp);
            comp.push_back(CompleteDesc{F.w, F.d, F.dp, Q.T, F.flags, F.flags + F.w, Q.Tlo, Q.R, Q.Rlo, F.wp});
            // core: srevd C = Q^T (X Q) (rnla.hpp:97); rsvd_psd B B^T = Y^T Y (eig.hpp:251)
            {
                TcProblemDesc cc;
                cc.M = F.w; cc.N = F.w; cc.K = F.d;
                const Role& Aop = method_ == RKFAC_SREVD ? Q : Y;
                cc.A = Aop.T; cc.A_lo = Aop.Tlo; cc.lda = F.dp;
                cc.B = Y.T; cc.B_lo = Y.Tlo; cc.ldb = F.dp;
                cc.out0 = out_r(F.core, F.w);
                cc.slice_k = kSliceK;
                core_[dir]->add(cc);
            }
            // lift: srevd U = Q P_r (rnla.hpp:101); rsvd U = Y P_r diag(1/s) (eig.hpp:260-266); both layouts of U
            // (+ lo planes) for the apply stage, U^T copied out to the caller afterwards
            {
                TcProblemDesc lf;
                lf.M = F.d; lf.N = F.r; lf.K = F.w;
                const Role& Aop = method_ == RKFAC_SREVD ? Q : Y;
                lf.A = Aop.R; lf.A_lo = nullptr; lf.lda = F.wp;
                lf.B = F.Pt; lf.B_lo = F.Ptlo; lf.ldb = F.wp;
                if (method_ == RKFAC_RSVD) lf.cs = F.scale;
                lf.out0 = out_t(F.Uti, F.dp); lf.lo0 = out_t(F.Utilo, F.dp);
                lf.out1 = out_r(F.Ui, F.rp); lf.lo1 = out_r(F.Uilo, F.rp);
                lift_[dir]->add(lf);
            }
        }
        // complete_[dir] completes the output of orth(src = dir), i.e. role S[dir ^ 1]
        upload(d_complete_[dir], comp);
        static const bool fuse_gram = [] {
            const char* e = std::getenv("RKFAC_GRAM_FUSED");
            return !(e && e[0] == '0');
        }();
        gram_[dir]->set_defer_reduce(fuse_gram);  // the Cholesky-inverse sums the Gram's K slices while loading it
        xq_[dir]->finalize(); xqf_[dir]->finalize(); xq_t_[dir]->finalize(); xq_tl_[dir]->finalize();
        xz_[dir]->finalize(); gram_[dir]->finalize(); tri_[dir]->finalize(); tri_t_[dir]->finalize(); core_[dir]->finalize();
        gram64_[dir]->finalize(); tri64_[dir]->finalize(); lift_[dir]->finalize();
    }
    std::vector<CopyDesc> cp;
    long long cp_off = 0;
    for (auto& F : f_) {
        cp.push_back(CopyDesc{F.Uti, F.Ut, F.r, F.d, F.dp, F.ldu, cp_off});
        cp_off += (long long)F.r * F.d;
    }
    upload(d_copy_ut_, cp);
    copy_ut_total_ = cp_off;
    std::vector<CholDesc> c64, c32[2];
    std::vector<EigDesc> eg;
    std::vector<PostDesc> po;
    std::vector<CompleteDesc> cu;
    std::vector<BracketDesc> br;
    for (auto& F : f_) {
        c64.push_back(CholDesc{F.w, F.G64, F.wp, F.Linv64, F.wp, nullptr, F.flags, F.flags + F.w, F.chol_scratch,
                               nullptr, 1});
        for (int dir = 0; dir < 2; ++dir) {
            auto sp = gram_[dir]->split_of((int)(&F - f_.data()));
            if (!gram_[dir]->defer_reduce()) sp = {nullptr, 1};
            c32[dir].push_back(CholDesc{F.w, F.G32, F.wp, F.Linv32, F.wp, F.Linv32lo, F.flags, F.flags + F.w,
                                        F.chol_scratch, sp.first, sp.second});
        }
        EigDesc e{};
        e.n = F.w; e.r = F.r; e.A = F.core; e.lda = F.w; e.scratch = F.eig_scratch; e.refl = F.refl;
        e.tau = F.tau; e.dvec = F.dvec; e.evec = F.evec; e.evals = F.evals; e.scr = F.scr; e.piv = F.piv;
        e.z = F.z; e.Pt = F.Pt; e.Ptlo = F.Ptlo; e.ldpt = F.wp;
        eg.push_back(e);
        po.push_back(PostDesc{F.r, method_, F.evals, F.dvals, F.scale, F.zflags, F.zflags + F.r});
        cu.push_back(CompleteDesc{F.r, F.d, F.dp, F.Uti, F.zflags, F.zflags + F.r, F.Utilo, F.Ui, F.Uilo, F.rp});
        br.push_back(BracketDesc{F.r, F.dvals, F.bracket});
    }
    upload(d_chol64_, c64);
    upload(d_chol32_[0], c32[0]);
    upload(d_chol32_[1], c32[1]);
    upload(d_eig_, eg);
    upload(d_post_, po);
    upload(d_complete_u_, cu);
    upload(d_bracket_, br);
}

std::unique_ptr<TcGemm> Plan::new_tc() const {
    auto g = std::make_unique<TcGemm>();
    g->set_max_ctas(tc_cap_);
    return g;
}

void Plan::set_max_ctas(int n) {
    tc_cap_ = n;
    if (factors_bound_) build_decomp_stages();
    ea_rho_ = -1;  // EA and apply stages are rebuilt on their next use
    ap_lambda_ = -1;
}

void Plan::build_ea_stage(double rho, double scale) {
    ea_tc_stage_.reset();
    ea_long_stage_.reset();
    ea_simt_.reset();
    std::vector<SplitDesc> sm;
    long long off = 0;
    ea_split_n_ = 0;
    // decided from the operands bound NOW (factors and samples may be re-bound in either order)
    ea_tc_ = x_tma_ok_ && samples_tma_ok_;
    if (ea_tc_) {
        // the samples' lo planes: formed in smem by the converter warps for short K (VGG16, n = 128: 0.218 vs
        // 0.256 ms with the split pass), stored by a split pass for long K, where the converters bound the mainloop
        // (config 5, n = 512: 7.8 vs 12.1 ms); RKFAC_EA_STORED_LO=0/1 forces either
        long long nmax = 0;
        for (auto& F : f_) nmax = std::max<long long>(nmax, F.M ? F.n : 0);
        bool stored_lo = nmax >= 512;
        if (const char* e = std::getenv("RKFAC_EA_STORED_LO")) stored_lo = std::atoi(e) != 0;
        if (ea_lo_mode_ >= 0) stored_lo = ea_lo_mode_ == 1;
        ea_tc_stage_ = new_tc();
        ea_long_stage_ = new_tc();
        std::vector<SymDesc> sym;
        long long sym_off = 0;
        for (auto& F : f_) {
            if (!F.M || F.n == 0) continue;
            TcProblemDesc p;
            p.M = F.d; p.N = F.d; p.K = (int)F.n;
            p.A = F.M; p.A_lo = stored_lo ? F.Ml : nullptr; p.lda = F.ldm;  // default: both lo planes formed in smem
            p.B = F.M; p.B_lo = stored_lo ? F.Ml : nullptr; p.ldb = F.ldm;
            p.alpha = (float)((1.0 - rho) * scale * scale);
            p.beta = (float)rho;
            p.Cin = F.X; p.ldcin = F.ldx; p.cin_t = 0;
            p.out0 = out_r(F.X, F.ldx);
            if (F.n <= kEaLongK) {
                p.sym = 1;  // upper tiles, mirrored: exactly symmetric; one TMEM chain of n <= 512
                ea_tc_stage_->add(p);
            } else {
                // long K (convolution statistics, n = B*H*W): the truncating TMEM accumulation would grow the error
                // linearly with n (tools/tc_acc.cu), so K is cut into slices of kEaLongK summed in FP32 by the
                // deterministic split-K reduction, which applies the axpy epilogue; the full square is computed and
                // symmetrised afterwards, exactly the reference's symmetrize_in_place (kfactor.hpp:39)
                p.sym = 0;
                p.slice_k = kEaLongK;
                ea_long_stage_->add(p);
                sym.push_back(SymDesc{F.X, F.ldx, F.d, sym_off});
                sym_off += (long long)F.d * (F.d - 1) / 2;
            }
            sm.push_back(SplitDesc{F.M, nullptr, F.Ml, F.d, (int)F.n, F.ldm, F.ldm, off});
            off += (long long)F.d * F.n;
        }
        ea_tc_stage_->finalize();
        ea_long_stage_->finalize();
        upload(d_sym_, sym);
        sym_n_ = (int)sym.size();
        sym_total_ = sym_off;
        if (stored_lo) ea_split_n_ = (int)sm.size();
    } else {
        ea_simt_ = std::make_unique<GemmBatch>(GemmKind::F32);
        for (auto& F : f_) {
            if (!F.M || F.n == 0) continue;
            GemmDesc d = GemmBatch::make(F.d, F.d, (int)F.n, F.M, F.ldm, 0, F.M, F.ldm, 1, F.X, F.ldx, 0);
            d.sym = 1;
            d.alpha = (1.0 - rho) * scale * scale;
            d.beta = rho;
            d.Cin = F.X;
            d.ldcin = F.ldx;
            ea_simt_->add(d);
        }
        ea_simt_->finalize();
    }
    upload(d_split_m_, sm);
    split_m_total_ = off;
    ea_rho_ = rho;
    ea_scale_ = scale;
}

void Plan::build_apply_stages(double lambda) {
    // Four grouped 3xTF32 tcgen05 GEMMs over all layers, every operand K-major (intermediates are written in the
    // layout their consumer needs, with their TF32 lo planes):
    //   RIGHT (kfactor.hpp:156-160):  W1 = J U_A diag(b_A)           (M=dG, N=rA, K=dA)
    //                                 mid^T = (W1 U_A^T + J/lambda)^T (M=dG, N=dA, K=rA)
    //   LEFT  (kfactor.hpp:147-152):  W2^T = (diag(b_G) U_G^T mid)^T  (M=rG, N=dA, K=dG)
    //                                 out = U_G W2 + mid/lambda        (M=dG, N=dA, K=rG)
    for (auto& a : ap_) a = new_tc();
    const float inv = (float)(1.0 / lambda);
    for (auto& L : layers_) {
        const FactorState &A = f_[L.a], &G = f_[L.g];
        const long long dAp = (A.d + 3) / 4 * 4, dGp = (G.d + 3) / 4 * 4;
        TcProblemDesc p0;
        p0.M = G.d; p0.N = A.r; p0.K = A.d;
        p0.A = L.Jc; p0.A_lo = nullptr; p0.lda = dAp;
        p0.B = A.Uti; p0.B_lo = A.Utilo; p0.ldb = A.dp;
        p0.cs = A.bracket;
        p0.out0 = out_r(L.W1, A.rp); p0.lo0 = out_r(L.W1lo, A.rp);
        p0.slice_k = apply_slice(A.d);
        ap_[0]->add(p0);
        TcProblemDesc p1;
        p1.M = G.d; p1.N = A.d; p1.K = A.r;
        p1.A = L.W1; p1.A_lo = L.W1lo; p1.lda = A.rp;
        p1.B = A.Ui; p1.B_lo = A.Uilo; p1.ldb = A.rp;
        p1.gamma = inv; p1.Din = L.Jc; p1.lddin = dAp; p1.din_t = 0;
        p1.out0 = out_t(L.Mt, dGp); p1.lo0 = out_t(L.Mtlo, dGp);
        ap_[1]->add(p1);
        TcProblemDesc p2;
        p2.M = G.r; p2.N = A.d; p2.K = G.d;
        p2.A = G.Uti; p2.A_lo = G.Utilo; p2.lda = G.dp;
        p2.B = L.Mt; p2.B_lo = L.Mtlo; p2.ldb = dGp;
        p2.rs = G.bracket;
        p2.out0 = out_t(L.W2t, G.rp); p2.lo0 = out_t(L.W2tlo, G.rp);
        p2.slice_k = apply_slice(G.d);
        ap_[2]->add(p2);
        TcProblemDesc p3;
        p3.M = G.d; p3.N = A.d; p3.K = G.r;
        p3.A = G.Ui; p3.A_lo = G.Uilo; p3.lda = G.rp;
        p3.B = L.W2t; p3.B_lo = L.W2tlo; p3.ldb = G.rp;
        p3.gamma = inv; p3.Din = L.Mt; p3.lddin = dGp; p3.din_t = 1;
        p3.out0 = out_r(L.out, A.d);
        ap_[3]->add(p3);
    }
    for (auto& a : ap_) a->finalize();
    ap_lambda_ = lambda;
}

// Orthonormalise role S[src] into S[src ^ 1].
void Plan::orth(int src, bool fp64, cudaStream_t s, bool need_r) {
    const int n = nfactors();
    if (fp64) {
        gram64_[src]->launch(s);
        launch_cholinv(d_chol64_.as<CholDesc>(), n, wmax_, true, true, kTol64, s);
        tri64_[src]->launch(s);
    } else {
        gram_[src]->launch(s);
        launch_cholinv(d_chol32_[src].as<CholDesc>(), n, wmax_, false, false, kTol32, s);
        (need_r ? tri_ : tri_t_)[src]->launch(s);
    }
    // rank-deficient columns stay zero here; the final basis is completed in decompose()
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
    cudaStream_t s = ctx_->stream;
    mark(kEA, true);
    if (ea_tc_) {
        if (ea_split_n_ > 0) launch_split(d_split_m_.as<SplitDesc>(), ea_split_n_, split_m_total_, s);
        ea_tc_stage_->launch(s);
        if (ea_long_stage_ && !ea_long_stage_->empty()) {
            ea_long_stage_->launch(s);
            launch_symmetrize(d_sym_.as<SymDesc>(), sym_n_, sym_total_, s);
        }
    } else {
        ea_simt_->launch(s);
    }
    mark(kEA, false);
}

void Plan::decompose(int mode, uint64_t root, uint64_t step, bool x_lo_fresh, int flags) {
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    cudaStream_t s = ctx_->stream;
    const int n = nfactors();
    if (n == 0) return;
    int qmax = 0;
    for (auto& F : f_) qmax = std::max(qmax, F.q);
    for (auto& F : f_)
        RKFAC_REQUIRE(F.q == qmax, RKFAC_INVALID_ARGUMENT, "all factors of a plan share power_iters");
    mark(kDecompose, true);
    (void)x_lo_fresh;
    if (!x_tma_ok_) launch_split(d_split_x_.as<SplitDesc>(), n, split_x_total_, s);  // padded TMA copy of X
    if (flags & kOmegaAhead) RKFAC_CUDA(cudaStreamWaitEvent(s, ev_pre_, 0));  // generated next to the EA update
    else launch_omega(d_omega_.as<OmegaDesc>(), n, omega_total_, mode, root, step, s,
                      mode == 1 ? captured_seed(root, step, s) : nullptr);
    int cur_q = 1;  // the basis lives in S[cur_q]
    const int north = 2 * qmax + 1;
    bool last_fp64 = false;
    // Every power product runs in 3xTF32: 1xTF32 intermediate products (0.7 ms faster per VGG16 step) were measured
    // to move the poorly converged Ritz values near the cut-off by up to 6e-3 (d = 16384) -- first order in the
    // perturbation of the subspace -- so the reference's randomized answer is not reproduced to 1e-4.
    auto timed_xq = [&](int y, int o) {
        mark(kXQ, true);
        (o < n_fp64_orth_ ? xq_t_ : xq_)[y]->launch(s);  // an FP64 orthonormalisation reads only Y^T
        mark(kXQ, false);
    };
    // Every product is orthonormalised, as in the reference: skipping alternate orthonormalisations (X X Q, same
    // span) was measured to lose the tail of the spectrum in FP32 (eigenvalue errors ~0.9 at index r-1).
    // Optional overlapped power iteration (RKFAC_OVERLAP_ORTH=1; default off).  The reference orthonormalises every
    // product: Y' = X (Y L^-T), L = chol(Y^T Y) (rnla.hpp:47-56).  By associativity Y' = (X Y) L^-T, and X Y depends
    // only on Y -- like the Gram and its Cholesky-inverse -- so the product can run NEXT to the latency-bound Gram +
    // Cholesky-inverse (side stream) and one skinny product Z L^-T joins them.  Measured on B200:
    // a lone 4609-wide layer's chain shortens, the 5-group VGG16 step gains 3 % (it is throughput-bound), and the
    // rounding of the Gram coefficients is amplified by lambda_1 / lambda_j in column j (the reference's order keeps
    // it inside the span of the earlier columns): the last Ritz values move by ~(6e-8 lambda_1 / lambda_r)^2, i.e.
    // 2.8e-5 at VGG16's spectrum (bar met) but 1.2e-3 at config 5's (lambda_r / lambda_1 = 1.6e-6, bar missed; an
    // FP64 Gram / Cholesky / Z L^-T restores 4e-5 but costs more than the overlap gains).  Hence off by default.
    const bool overlap = overlap_orth_ && n_fp64_orth_ == 1 && north >= 3;
    for (int o = 0; o < north && !(overlap && o >= 1); ++o) {
        const int y = cur_q ^ 1;
        timed_xq(y, o);
        last_fp64 = o < n_fp64_orth_;
        mark(kOrth, true);
        // S[y] -> S[cur_q]; the row-major planes of Q are read only by the CholeskyQR2 pass and the lift
        orth(y, last_fp64, s, o == north - 1);
        mark(kOrth, false);
    }
    if (overlap) {
        const int y = cur_q ^ 1;  // Y lives in S[y] throughout, Z in S[cur_q].R
        const int n_over = std::max(0, north - 2 - explicit_tail_);
        mark(kXQ, true);
        (n_over == 0 ? xq_ : xq_tl_)[y]->launch(s);  // Y1 = X Q0
        mark(kXQ, false);
        // with stage timing on, the side chain is issued on the main stream (every stage timed alone)
        cudaStream_t side = timing_ ? s : side_;
        for (int o = 1; o <= n_over; ++o) {
            if (side != s) {
                RKFAC_CUDA(cudaEventRecord(ev_fork_, s));
                RKFAC_CUDA(cudaStreamWaitEvent(side, ev_fork_, 0));
            }
            mark(kXQ, true);
            xz_[cur_q]->launch(s);  // Z = X Y (row-major only)
            mark(kXQ, false);
            mark(kOrth, true);
            gram_[y]->launch(side);
            launch_cholinv(d_chol32_[y].as<CholDesc>(), n, wmax_, false, false, kTol32, side);
            if (side != s) {
                RKFAC_CUDA(cudaEventRecord(ev_join_, side));
                RKFAC_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
            }
            // Y' = Z L^-T back into S[y] (the last iterate with its row-major plane, for the explicit CholeskyQR2)
            (o == n_over ? tri_ : tri_t_)[cur_q]->launch(s);
            mark(kOrth, false);
        }
        // the last explicit_tail_ products in the reference's order (orthonormalise, then multiply)
        for (int o = 0; o < std::min(explicit_tail_, std::max(0, north - 2)); ++o) {
            mark(kOrth, true);
            orth(y, false, s, false);
            mark(kOrth, false);
            mark(kXQ, true);
            xq_[y]->launch(s);
            mark(kXQ, false);
        }
        mark(kOrth, true);
        orth(y, false, s, true);
        mark(kOrth, false);
        last_fp64 = false;
    }
    if (!last_fp64) {  // CholeskyQR2: second pass so the final basis is orthonormal to FP32 rounding
        mark(kOrth, true);
        launch_fill(d_complete_[cur_q ^ 1].as<CompleteDesc>(), n, s);  // candidates for flagged columns
        orth(cur_q, false, s);
        launch_complete(d_complete_[cur_q].as<CompleteDesc>(), n, s);  // last resort (normally nothing flagged)
        mark(kOrth, false);
        cur_q ^= 1;
    } else {
        launch_complete(d_complete_[cur_q ^ 1].as<CompleteDesc>(), n, s);
    }
    const int y = cur_q ^ 1;
    mark(kXQ, true);
    xqf_[y]->launch(s);
    mark(kXQ, false);
    mark(kEig, true);
    core_[y]->launch(s);
    launch_eig(d_eig_.as<EigDesc>(), n, wmax_, rmax_, s);
    launch_post(d_post_.as<PostDesc>(), n, s);
    lift_[y]->launch(s);
    if (method_ == RKFAC_RSVD) launch_complete(d_complete_u_.as<CompleteDesc>(), n, s);
    if (flags & kDeferUtCopy) {  // U^T leaves next to the preconditioning (which reads the plan's own copies)
        RKFAC_CUDA(cudaEventRecord(ev_fork_, s));
        RKFAC_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
        launch_copy(d_copy_ut_.as<CopyDesc>(), n, copy_ut_total_, side_);
        RKFAC_CUDA(cudaEventRecord(ev_copy_, side_));
    } else {
        launch_copy(d_copy_ut_.as<CopyDesc>(), n, copy_ut_total_, s);
    }
    mark(kEig, false);
    mark(kDecompose, false);
}

void Plan::precondition(double lambda, bool j_copied) {
    RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    if (layers_.empty()) return;
    if (lambda != ap_lambda_) build_apply_stages(lambda);
    cudaStream_t s = ctx_->stream;
    mark(kApply, true);
    launch_bracket(d_bracket_.as<BracketDesc>(), nfactors(), lambda, s);
    if (!j_copied)
        launch_split(d_split_j_.as<SplitDesc>(), (int)layers_.size(), split_j_total_, s);  // J -> aligned TMA copy
    for (auto& a : ap_) a->launch(s);
    mark(kApply, false);
}

void Plan::prepare(double rho, double scale, double lambda) {
    RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
    if (samples_bound_ && (rho != ea_rho_ || scale != ea_scale_)) build_ea_stage(rho, scale);
    if (!layers_.empty() && lambda != ap_lambda_) build_apply_stages(lambda);
    if (!h_seed_) set_step_seed(0, 0);  // allocated here: no allocation while a stream is being captured
}

// The pieces of a step that depend on neither the EA update nor the decomposition run next to them on the side
// stream: Omega (FP64 transcendental math: ~0.1 ms per VGG16 group) and, for step(), the aligned copy of the
// gradients next to the EA update; U^T's copy-out next to the preconditioning.  Stage timing keeps everything in line.
// While the stream is being captured into a CUDA graph, (root, step) go through a pinned host pair that a copy node
// brings to the device at every replay, so one captured step serves every step id: rkfac_plan_set_step_seed before the
// replay.  Eager launches pass them as kernel arguments (returns nullptr).
const uint64_t* Plan::captured_seed(uint64_t root, uint64_t stp, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    RKFAC_CUDA(cudaStreamIsCapturing(s, &st));
    if (st != cudaStreamCaptureStatusActive) return nullptr;
    set_step_seed(root, stp);
    RKFAC_CUDA(cudaMemcpyAsync(d_seed_.p, h_seed_, 2 * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    return d_seed_.as<uint64_t>();
}

void Plan::set_step_seed(uint64_t root, uint64_t stp) {
    if (!h_seed_) {
        RKFAC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_seed_), 2 * sizeof(uint64_t), cudaHostAllocDefault));
        d_seed_.alloc(2 * sizeof(uint64_t));
    }
    h_seed_[0] = root;
    h_seed_[1] = stp;
}

bool Plan::launch_ahead(uint64_t root, uint64_t stp, bool with_grads) {
    if (!step_overlap_ || timing_ || nfactors() == 0) return false;
    cudaStream_t s = ctx_->stream;
    RKFAC_CUDA(cudaEventRecord(ev_fork_, s));
    RKFAC_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    launch_omega(d_omega_.as<OmegaDesc>(), nfactors(), omega_total_, 1, root, stp, side_,
                 captured_seed(root, stp, side_));
    if (with_grads && !layers_.empty())
        launch_split(d_split_j_.as<SplitDesc>(), (int)layers_.size(), split_j_total_, side_);
    RKFAC_CUDA(cudaEventRecord(ev_pre_, side_));
    return true;
}

void Plan::ea_decompose(double rho, double scale, uint64_t root, uint64_t stp) {
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    const bool over = launch_ahead(root, stp, false);
    bool fresh = false;
    if (samples_bound_) {
        ea_update(rho, scale);
        bool all = true;  // the tensor-core EA epilogue wrote every factor's lo plane
        for (auto& F : f_) all = all && F.M && F.n > 0;
        fresh = ea_tc_ && all;
    }
    decompose(1, root, stp, fresh, over ? kOmegaAhead : 0);
}

void Plan::step(double rho, double scale, uint64_t root, uint64_t stp, double lambda) {
    RKFAC_REQUIRE(lambda > 0.0, RKFAC_DAMPING_NONPOSITIVE, "apply_lowrank_damped_inverse: lambda must be > 0");
    RKFAC_REQUIRE(factors_bound_, RKFAC_INVALID_ARGUMENT, "factors not bound");
    mark(kStep, true);
    const bool over = launch_ahead(root, stp, true);
    bool fresh = false;
    if (samples_bound_) {
        ea_update(rho, scale);
        bool all = true;
        for (auto& F : f_) all = all && F.M && F.n > 0;
        fresh = ea_tc_ && all;
    }
    decompose(1, root, stp, fresh, over ? (kOmegaAhead | kDeferUtCopy) : 0);
    precondition(lambda, over);
    if (over) RKFAC_CUDA(cudaStreamWaitEvent(ctx_->stream, ev_copy_, 0));
    if (gathered_) gather();
    mark(kStep, false);
}

void Plan::set_gather(long long chunk, const long long* offsets, float* gathered) {
    RKFAC_REQUIRE(!layers_.empty(), RKFAC_INVALID_ARGUMENT, "set_gather: no layers bound");
    if (!gathered) {
        gathered_ = nullptr;
        return;
    }
    std::vector<CopyDesc> cp;
    long long off = 0;
    for (size_t l = 0; l < layers_.size(); ++l) {
        const LayerState& L = layers_[l];
        const int dG = f_[L.g].d, dA = f_[L.a].d;
        RKFAC_REQUIRE(offsets[l] >= 0 && offsets[l] + (long long)dG * dA <= chunk, RKFAC_INVALID_ARGUMENT,
                      "set_gather: layer output outside the chunk");
        // the output is dG x dA contiguous: one row of dG*dA floats into the chunk
        cp.push_back(CopyDesc{L.out, nullptr, 1, dG * dA, (long long)dG * dA, (long long)dG * dA, off});
        off += (long long)dG * dA;
    }
    gather_send_.alloc(sizeof(float) * (size_t)std::max<long long>(1, chunk));
    RKFAC_CUDA(cudaMemset(gather_send_.p, 0, sizeof(float) * (size_t)std::max<long long>(1, chunk)));
    for (size_t l = 0; l < cp.size(); ++l) cp[l].dst = gather_send_.as<float>() + offsets[l];
    upload(d_pack_, cp);
    pack_total_ = off;
    gather_chunk_ = chunk;
    gathered_ = gathered;
}

void Plan::gather() {
    RKFAC_REQUIRE(gathered_, RKFAC_INVALID_ARGUMENT, "gather: set_gather was not called");
    cudaStream_t s = ctx_->stream;
    launch_copy(d_pack_.as<CopyDesc>(), (int)layers_.size(), pack_total_, s);
    nccl_allgather(ctx_->nccl_comm, gather_send_.as<float>(), gathered_, gather_chunk_, s);
}

}  // namespace rkfac_b200
