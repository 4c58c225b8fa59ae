// rsvd.cu -- rnla.hpp:62-77 rsvd on a general (rectangular) matrix: SvdResult {u (rows x r), s (r), v (cols x r)}.
//
// The same building blocks as the batched plan (engine.cu), on the two sides of a rectangular X (m x n):
//   Q  = orth(X Omega)                                 (m-side; Omega^T: w x n from the reference stream)
//   q x { Z = orth(X^T Q) (n-side);  Q = orth(X Z) (m-side) }     randomized_range, rnla.hpp:47-56
//   B^T = X^T Q (n x w), core = B B^T (w x w)          svd_small(B^T) by the Gram route, eig.hpp:243-270
//   core = P diag(s^2) P^T; u_x = Q P_r, s_r, v_x = B^T P_r / s_r (zero modes completed)
// Products are tcgen05 3xTF32; the first orthonormalisation is FP64 (DMMA Gram + Cholesky-inverse + TRSM) and the
// final basis gets a second CholeskyQR pass, exactly as the square path; the w x w eigensolver is eig.cu.  X^T is
// formed once by a transposed copy (the K-major operand of X^T Q).  Not on the optimizer path (which uses the square
// PSD specialisation rsvd_psd); single problem, synchronous, workspace cached per shape.
#include <algorithm>

#include "dmma.cuh"
#include "engine.cuh"
#include "rsvd.cuh"

namespace rkfac_b200 {

namespace {

constexpr double kTol64 = 1e-13;
constexpr double kTol32 = 1e-5;
constexpr int kSliceK = 512;

TcOut to_t(float* p, long long ld) { TcOut o; o.p = p; o.ld = ld; o.t = 1; return o; }
TcOut to_r(float* p, long long ld) { TcOut o; o.p = p; o.ld = ld; o.t = 0; return o; }

template <class T>
void up(DevBuf& b, const T& v) {
    b.alloc(sizeof(T));
    RKFAC_CUDA(cudaMemcpy(b.p, &v, sizeof(T), cudaMemcpyHostToDevice));
}

}  // namespace

struct Rsvd::Side {  // a tall-skinny d x w basis in the four layouts its consumers read (cf. Role, engine.cuh)
    int d = 0, dp = 0;
    float *T = nullptr, *Tlo = nullptr, *R = nullptr, *Rlo = nullptr;
};

Rsvd::Rsvd() = default;
Rsvd::~Rsvd() = default;

void Rsvd::run(const float* x, long long ldx, int m, int n, int r_in, int p_in, int q, uint64_t seed, uint64_t ctr0,
               float* u, long long ldu, float* s, float* v, long long ldv, int* rank_out, cudaStream_t st) {
    // clamp_sketch with dim = min(rows, cols) (rnla.hpp:63)
    const int dim = std::min(m, n);
    long long r = r_in, p = p_in;
    if (r > dim) { r = dim; p = 0; }
    else if (r + p > dim) p = dim - r;
    const int w = (int)(r + p), rr = (int)r;
    RKFAC_REQUIRE(w >= 1 && w <= 512, RKFAC_INVALID_ARGUMENT, "rsvd: sketch width r+p must be in [1, 512]");
    const int wp = (w + 3) / 4 * 4, rp = (rr + 3) / 4 * 4;
    const int mp = (m + 31) / 32 * 32, np = (n + 31) / 32 * 32;
    // ---- workspace (one arena)
    size_t off = 0;
    auto take = [&](size_t bytes) { const size_t o = (off + 255) & ~size_t(255); off = o + bytes; return o; };
    const size_t oX = take(sizeof(float) * (size_t)m * np), oXt = take(sizeof(float) * (size_t)n * mp);
    size_t oS[4][4];
    for (int k = 0; k < 4; ++k) {  // sides: 0, 1 = m-side raw / basis; 2, 3 = n-side raw / basis
        const int d = k < 2 ? m : n, dpk = k < 2 ? mp : np;
        oS[k][0] = take(sizeof(float) * (size_t)w * dpk);
        oS[k][1] = take(sizeof(float) * (size_t)w * dpk);
        oS[k][2] = take(sizeof(float) * (size_t)d * wp);
        oS[k][3] = take(sizeof(float) * (size_t)d * wp);
    }
    const size_t oG64 = take(sizeof(double) * w * wp), oG32 = take(sizeof(float) * w * wp),
                 oL64 = take(sizeof(double) * w * wp), oL32 = take(sizeof(float) * w * wp),
                 oL32lo = take(sizeof(float) * w * wp), oFl = take(sizeof(int) * (w + 1)),
                 oCh = take(sizeof(double) * ((size_t)w * (w + 1) / 2 + 8 * w + 16)),
                 oCore = take(sizeof(float) * w * w), oEsc = take(sizeof(double) * w * (w + 1) / 2),
                 oRefl = take(sizeof(double) * w * w), oTau = take(sizeof(double) * w),
                 oDv = take(sizeof(double) * w), oEv = take(sizeof(double) * w), oEvals = take(sizeof(double) * w),
                 oScr = take(sizeof(double) * 4 * w * rr), oPiv = take((size_t)w * rr), oZ = take(sizeof(double) * w * rr),
                 oPt = take(sizeof(float) * rr * wp), oPtlo = take(sizeof(float) * rr * wp),
                 oScale = take(sizeof(float) * rr), oZf = take(sizeof(int) * (rr + 1)),
                 oUt = take(sizeof(float) * (size_t)rr * mp), oVt = take(sizeof(float) * (size_t)rr * np),
                 oVtlo = take(sizeof(float) * (size_t)rr * np), oVr = take(sizeof(float) * (size_t)n * rp),
                 oVrlo = take(sizeof(float) * (size_t)n * rp);
    if (ws_.bytes < off) ws_.alloc(off);
    RKFAC_CUDA(cudaMemsetAsync(ws_.p, 0, off, st));
    char* base = static_cast<char*>(ws_.p);
    auto F = [&](size_t o) { return reinterpret_cast<float*>(base + o); };
    auto D = [&](size_t o) { return reinterpret_cast<double*>(base + o); };
    Side S[4];
    for (int k = 0; k < 4; ++k) {
        S[k].d = k < 2 ? m : n;
        S[k].dp = k < 2 ? mp : np;
        S[k].T = F(oS[k][0]); S[k].Tlo = F(oS[k][1]); S[k].R = F(oS[k][2]); S[k].Rlo = F(oS[k][3]);
    }
    // X (pitch np) and X^T (pitch mp): TMA-legal K-major operands of X Z and X^T Q
    float* X = F(oX);
    float* Xt = F(oXt);
    {
        CopyDesc cd{x, X, m, n, ldx, np, 0};
        DevBuf b;
        up(b, cd);
        launch_copy(b.as<CopyDesc>(), 1, (long long)m * n, st);
        launch_transpose(x, ldx, m, n, Xt, mp, st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    }
    // Omega^T (w x n) into the n-side basis role S[3] (+ TF32 lo plane), the reference stream (rng.hpp:59-63)
    {
        OmegaDesc o{};
        o.d = n; o.w = w; o.ld = np; o.out = S[3].T; o.out_lo = S[3].Tlo; o.seed = seed; o.ctr0 = ctr0; o.offset = 0;
        DevBuf b;
        up(b, o);
        launch_omega(b.as<OmegaDesc>(), 1, (long long)n * w, 0, 0, 0, st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    }
    double* G64 = D(oG64);
    float* G32 = F(oG32);
    double* L64 = D(oL64);
    float* L32 = F(oL32);
    float* L32lo = F(oL32lo);
    int* flags = reinterpret_cast<int*>(base + oFl);
    void* chs = base + oCh;
    // product: Y (side dst) = op (A-operand) . basis^T (side src): Y^T (+lo) and Y row-major
    auto product = [&](const float* Aop, long long lda, int M, int K, Side& src, Side& dst, int slice) {
        TcGemm g;
        TcProblemDesc pd;
        pd.M = M; pd.N = w; pd.K = K;
        pd.A = Aop; pd.lda = lda;
        pd.B = src.T; pd.B_lo = src.Tlo; pd.ldb = src.dp;
        pd.out0 = to_t(dst.T, dst.dp); pd.lo0 = to_t(dst.Tlo, dst.dp);
        pd.out1 = to_r(dst.R, wp);
        pd.slice_k = slice;
        g.add(pd);
        g.finalize();
        g.launch(st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    };
    // orthonormalise side src (Y) into side dst (Q): CholeskyQR, FP64 or FP32
    auto orth = [&](Side& y, Side& qd, bool fp64) {
        if (fp64) {
            Gram64Batch gb;
            gb.add(w, y.d, y.T, y.dp, G64, wp);
            gb.finalize();
            gb.launch(st);
            CholDesc c{w, G64, wp, L64, wp, nullptr, flags, flags + w, chs, nullptr, 1};
            DevBuf b;
            up(b, c);
            launch_cholinv(b.as<CholDesc>(), 1, w, true, true, kTol64, st);
            Tri64Batch tb;
            tb.add(w, y.d, L64, wp, y.T, y.dp, qd.T, qd.Tlo, qd.dp);
            tb.finalize();
            tb.launch(st);
            // the row-major planes of Q for the consumers that read them (the X^T Q / X Z products read Q^T)
            launch_transpose(qd.T, qd.dp, w, y.d, qd.R, wp, st);
            RKFAC_CUDA(cudaStreamSynchronize(st));
        } else {
            TcGemm g;
            TcProblemDesc gd;
            gd.M = w; gd.N = w; gd.K = y.d;
            gd.A = y.T; gd.A_lo = y.Tlo; gd.lda = y.dp;
            gd.B = y.T; gd.B_lo = y.Tlo; gd.ldb = y.dp;
            gd.out0 = to_r(G32, wp);
            gd.slice_k = kSliceK;
            g.add(gd);
            g.finalize();
            g.launch(st);
            CholDesc c{w, G32, wp, L32, wp, L32lo, flags, flags + w, chs, nullptr, 1};
            DevBuf b;
            up(b, c);
            launch_cholinv(b.as<CholDesc>(), 1, w, false, false, kTol32, st);
            TcGemm t;
            TcProblemDesc td;
            td.M = y.d; td.N = w; td.K = w;
            td.A = y.R; td.lda = wp;
            td.B = L32; td.B_lo = L32lo; td.ldb = wp;
            td.out0 = to_t(qd.T, qd.dp); td.lo0 = to_t(qd.Tlo, qd.dp);
            td.out1 = to_r(qd.R, wp);
            t.add(td);
            t.finalize();
            t.launch(st);
            RKFAC_CUDA(cudaStreamSynchronize(st));
        }
    };
    auto complete = [&](Side& qd, bool fill) {
        CompleteDesc cd{w, qd.d, qd.dp, qd.T, flags, flags + w, qd.Tlo, qd.R, qd.Rlo, wp};
        DevBuf b;
        up(b, cd);
        if (fill) launch_fill(b.as<CompleteDesc>(), 1, st);
        else launch_complete(b.as<CompleteDesc>(), 1, st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    };
    // ---- randomized_range (rnla.hpp:47-56)
    product(X, np, m, n, S[3], S[0], 0);  // Y0 = X Omega
    orth(S[0], S[1], true);               // Q (m-side), FP64
    for (int t = 0; t < q; ++t) {
        product(Xt, mp, n, m, S[1], S[2], 0);  // X^T Q
        orth(S[2], S[3], false);               // Z
        product(X, np, m, n, S[3], S[0], 0);   // X Z
        orth(S[0], S[1], false);               // Q
    }
    // CholeskyQR2 pass on the final basis (completion of rank-deficient columns first)
    RKFAC_CUDA(cudaMemcpyAsync(S[0].T, S[1].T, sizeof(float) * (size_t)w * mp, cudaMemcpyDeviceToDevice, st));
    RKFAC_CUDA(cudaMemcpyAsync(S[0].Tlo, S[1].Tlo, sizeof(float) * (size_t)w * mp, cudaMemcpyDeviceToDevice, st));
    RKFAC_CUDA(cudaMemcpyAsync(S[0].R, S[1].R, sizeof(float) * (size_t)m * wp, cudaMemcpyDeviceToDevice, st));
    complete(S[0], true);
    orth(S[0], S[1], false);
    complete(S[1], false);
    // ---- B^T = X^T Q (n x w, row-major in S[2].R) and B = its transpose (S[2].T + lo); core = B B^T
    product(Xt, mp, n, m, S[1], S[2], kSliceK);
    float* core = F(oCore);
    {
        TcGemm g;
        TcProblemDesc cd;
        cd.M = w; cd.N = w; cd.K = n;
        cd.A = S[2].T; cd.A_lo = S[2].Tlo; cd.lda = np;
        cd.B = S[2].T; cd.B_lo = S[2].Tlo; cd.ldb = np;
        cd.out0 = to_r(core, w);
        cd.slice_k = kSliceK;
        g.add(cd);
        g.finalize();
        g.launch(st);
    }
    // ---- core = P diag(mu) P^T (eig.cu), s = sqrt(max(0, mu)), zero modes flagged (eig.hpp:255-270)
    float* Pt = F(oPt);
    float* Ptlo = F(oPtlo);
    float* scale = F(oScale);
    int* zf = reinterpret_cast<int*>(base + oZf);
    {
        EigDesc e{};
        e.n = w; e.r = rr; e.A = core; e.lda = w; e.scratch = D(oEsc); e.refl = D(oRefl); e.tau = D(oTau);
        e.dvec = D(oDv); e.evec = D(oEv); e.evals = D(oEvals); e.scr = D(oScr);
        e.piv = reinterpret_cast<unsigned char*>(base + oPiv); e.z = D(oZ); e.Pt = Pt; e.Ptlo = Ptlo; e.ldpt = wp;
        DevBuf b;
        up(b, e);
        launch_eig(b.as<EigDesc>(), 1, w, rr, st);
        PostDesc pd{rr, RKFAC_RSVD, D(oEvals), s, scale, zf, zf + rr};
        DevBuf b2;
        up(b2, pd);
        launch_post(b2.as<PostDesc>(), 1, st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    }
    // ---- u_x = Q P_r (m x r); v_x = B^T P_r diag(1/s) (n x r), zero modes completed to orthonormal directions
    float* Ut = F(oUt);
    float* Vt = F(oVt);
    {
        TcGemm g;
        TcProblemDesc a;
        a.M = m; a.N = rr; a.K = w;
        a.A = S[1].R; a.lda = wp;
        a.B = Pt; a.B_lo = Ptlo; a.ldb = wp;
        a.out0 = to_t(Ut, mp);
        g.add(a);
        TcProblemDesc b;
        b.M = n; b.N = rr; b.K = w;
        b.A = S[2].R; b.lda = wp;
        b.B = Pt; b.B_lo = Ptlo; b.ldb = wp;
        b.cs = scale;
        b.out0 = to_t(Vt, np); b.lo0 = to_t(F(oVtlo), np);
        b.out1 = to_r(F(oVr), rp); b.lo1 = to_r(F(oVrlo), rp);
        g.add(b);
        g.finalize();
        g.launch(st);
        CompleteDesc cu{rr, n, np, Vt, zf, zf + rr, F(oVtlo), F(oVr), F(oVrlo), rp};
        DevBuf bc;
        up(bc, cu);
        launch_complete(bc.as<CompleteDesc>(), 1, st);
        launch_transpose(Ut, mp, rr, m, u, ldu, st);
        launch_transpose(Vt, np, rr, n, v, ldv, st);
        RKFAC_CUDA(cudaStreamSynchronize(st));
    }
    if (rank_out) *rank_out = rr;
}

}  // namespace rkfac_b200
