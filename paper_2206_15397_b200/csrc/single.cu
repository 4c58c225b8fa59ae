// single.cu -- the single-factor operators of the C-ABI on the tcgen05 engine:
//
//   rkfac_ea_update                     (kfactor.hpp:33-41)   symmetric 3xTF32 SYRK + axpy, mirrored upper tiles
//   rkfac_apply_lowrank_damped_inverse  (kfactor.hpp:134-161) two 3xTF32 GEMMs with the bracket scale and +V/lambda
//                                                             fused into their epilogues
//
// A call's stages (TMA descriptors, tile schedules, padded-operand copies) depend on its pointers and shapes, so they
// are built on the first call with a given operand set and kept in a small LRU cache per context: a repeated call
// (the reference's optimizer calls ea_update / apply every step on the same buffers) only enqueues its kernels -- no
// allocation, no descriptor upload, no host synchronisation.  Operands that are not valid TMA operands (row pitch not
// a multiple of 16 bytes, or a misaligned base) are copied into padded workspaces first.
#include <list>

#include "engine.cuh"
#include "single.cuh"

namespace rkfac_b200 {

namespace {

constexpr size_t kCacheEntries = 8;

long long pad4(long long x) { return (x + 3) / 4 * 4; }

// The apply's long-K product (K = dim) is split into slices of at most 512 for accuracy (engine.cu, kSliceK).
int apply_slice(long long K) { return (int)std::max<long long>(512, (K + 7) / 8); }

TcOut out_of(float* p, long long ld, int t) { TcOut o; o.p = p; o.ld = ld; o.t = t; return o; }

struct Copy {  // one grouped copy launch (device descriptors kept for the entry's lifetime)
    DevBuf d;
    long long total = 0;
    int n = 0;
    void set(const std::vector<CopyDesc>& v) {
        n = (int)v.size();
        total = 0;
        for (const auto& c : v) total = std::max(total, c.offset + (long long)c.rows * c.cols);
        d.alloc(sizeof(CopyDesc) * std::max<size_t>(1, v.size()));
        if (!v.empty()) RKFAC_CUDA(cudaMemcpy(d.p, v.data(), sizeof(CopyDesc) * v.size(), cudaMemcpyHostToDevice));
    }
    void launch(cudaStream_t s) const { if (n) launch_copy(d.as<CopyDesc>(), n, total, s); }
};

}  // namespace

struct SingleOps::Ea {
    // key
    float* x; long long ldx; int d; const float* m; long long ldm; int n; double rho, scale;
    // stage
    std::unique_ptr<TcGemm> g;
    DevBuf xp, mp;
    Copy in, out;
    cudaEvent_t done = nullptr;
    bool same(float* x_, long long ldx_, int d_, const float* m_, long long ldm_, int n_, double rho_,
              double scale_) const {
        return x == x_ && ldx == ldx_ && d == d_ && m == m_ && ldm == ldm_ && n == n_ && rho == rho_ &&
               scale == scale_;
    }
    ~Ea() { if (done) cudaEventDestroy(done); }
};

struct SingleOps::Apply {
    const float* u; long long ldu; const float* dv; int dim, r; double lam; const float* v; long long ldv;
    int rows, cols, side; float* out; long long ldo;
    std::unique_ptr<TcGemm> g1, g2;
    DevBuf ws, bd;
    Copy in;
    float *Ut = nullptr, *Uc = nullptr, *Vop = nullptr, *W = nullptr, *br = nullptr;
    long long ldvop = 0;
    bool vt = false;  // LEFT: V^T formed by a transpose
    cudaEvent_t done = nullptr;
    bool same(const Apply& o) const {
        return u == o.u && ldu == o.ldu && dv == o.dv && dim == o.dim && r == o.r && lam == o.lam && v == o.v &&
               ldv == o.ldv && rows == o.rows && cols == o.cols && side == o.side && out == o.out && ldo == o.ldo;
    }
    ~Apply() { if (done) cudaEventDestroy(done); }
};

SingleOps::SingleOps() = default;
SingleOps::~SingleOps() = default;

template <class T>
static void evict(std::list<std::unique_ptr<T>>& l) {
    while (l.size() > kCacheEntries) {  // the evicted stage may still be in flight: wait for its last launch
        if (l.back()->done) cudaEventSynchronize(l.back()->done);
        l.pop_back();
    }
}

void SingleOps::ea_update(float* x, long long ldx, int d, const float* m, long long ldm, int n, double rho,
                          double scale, cudaStream_t s) {
    if (n == 0) {  // m m^T = 0: mbar <- rho * mbar
        launch_scale(x, ldx, d, d, (float)rho, s);
        return;
    }
    Ea* e = nullptr;
    for (auto it = ea_.begin(); it != ea_.end(); ++it)
        if ((*it)->same(x, ldx, d, m, ldm, n, rho, scale)) {
            ea_.splice(ea_.begin(), ea_, it);
            e = ea_.front().get();
            break;
        }
    if (!e) {
        auto ne = std::make_unique<Ea>();
        e = ne.get();
        e->x = x; e->ldx = ldx; e->d = d; e->m = m; e->ldm = ldm; e->n = n; e->rho = rho; e->scale = scale;
        RKFAC_CUDA(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
        float* xop = x;
        long long ldxop = ldx;
        if (!tc_operand_ok(x, ldx)) {  // padded copy of the factor, updated in place, copied back
            ldxop = pad4(d);
            e->xp.alloc(sizeof(float) * (size_t)d * ldxop);
            xop = e->xp.as<float>();
            e->in.set({CopyDesc{x, xop, d, d, ldx, ldxop, 0}});
            e->out.set({CopyDesc{xop, x, d, d, ldxop, ldx, 0}});
        }
        const float* mop = m;
        long long ldmop = ldm;
        if (!tc_operand_ok(m, ldm)) {
            ldmop = pad4(n);
            e->mp.alloc(sizeof(float) * (size_t)d * ldmop);
            RKFAC_CUDA(cudaMemset(e->mp.p, 0, sizeof(float) * (size_t)d * ldmop));
            float* mp = e->mp.as<float>();
            std::vector<CopyDesc> c;
            if (e->in.n) c.push_back(CopyDesc{x, xop, d, d, ldx, ldxop, 0});
            c.push_back(CopyDesc{m, mp, d, n, ldm, ldmop, c.empty() ? 0 : (long long)d * d});
            e->in.set(c);
            mop = mp;
        }
        e->g = std::make_unique<TcGemm>();
        TcProblemDesc p;
        p.M = d; p.N = d; p.K = n;
        p.A = mop; p.lda = ldmop;  // both lo planes formed in shared memory
        p.B = mop; p.ldb = ldmop;
        p.sym = 1;
        p.alpha = (float)((1.0 - rho) * scale * scale);
        p.beta = (float)rho;
        p.Cin = xop; p.ldcin = ldxop; p.cin_t = 0;
        p.out0 = out_of(xop, ldxop, 0);
        e->g->add(p);
        e->g->finalize();
        ea_.push_front(std::move(ne));
        evict(ea_);
    }
    e->in.launch(s);
    e->g->launch(s);
    e->out.launch(s);
    RKFAC_CUDA(cudaEventRecord(e->done, s));
}

void SingleOps::apply(const float* u, long long ldu, const float* dv, int dim, int r, double lam, const float* v,
                      long long ldv, int rows, int cols, int side, float* out, long long ldo, cudaStream_t s) {
    Apply key;
    key.u = u; key.ldu = ldu; key.dv = dv; key.dim = dim; key.r = r; key.lam = lam; key.v = v; key.ldv = ldv;
    key.rows = rows; key.cols = cols; key.side = side; key.out = out; key.ldo = ldo;
    Apply* e = nullptr;
    for (auto it = ap_.begin(); it != ap_.end(); ++it)
        if ((*it)->same(key)) {
            ap_.splice(ap_.begin(), ap_, it);
            e = ap_.front().get();
            break;
        }
    if (!e) {
        auto ne = std::make_unique<Apply>();
        e = ne.get();
        e->u = u; e->ldu = ldu; e->dv = dv; e->dim = dim; e->r = r; e->lam = lam; e->v = v; e->ldv = ldv;
        e->rows = rows; e->cols = cols; e->side = side; e->out = out; e->ldo = ldo;
        RKFAC_CUDA(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming));
        const long long dimp = pad4(dim), rp = pad4(r);
        const bool left = side == RKFAC_LEFT;
        // workspace: U^T (r x dim), U (dim x r), the V operand (RIGHT: a padded copy when V is not a TMA operand;
        // LEFT: V^T, cols x rows), W (RIGHT: rows x r; LEFT: W^T, cols x r), the brackets (r)
        const bool vcopy = !left && !tc_operand_ok(v, ldv);
        const long long ldvop = left ? pad4(rows) : (vcopy ? pad4(cols) : ldv);
        const size_t nUt = (size_t)r * dimp, nUc = (size_t)dim * rp;
        const size_t nV = left ? (size_t)cols * ldvop : (vcopy ? (size_t)rows * ldvop : 0);
        const size_t nW = (size_t)(left ? cols : rows) * rp;
        e->ws.alloc(sizeof(float) * (nUt + nUc + nV + nW + rp) + 256);
        float* base = e->ws.as<float>();
        e->Ut = base;
        e->Uc = e->Ut + nUt;
        e->Vop = nV ? e->Uc + nUc : const_cast<float*>(v);
        e->W = e->Uc + nUc + nV;
        e->br = e->W + nW;
        e->ldvop = ldvop;
        e->vt = left;
        std::vector<CopyDesc> c{CopyDesc{u, e->Uc, dim, r, ldu, rp, 0}};
        if (vcopy) c.push_back(CopyDesc{v, e->Vop, rows, cols, ldv, ldvop, (long long)dim * r});
        e->in.set(c);
        BracketDesc b{r, dv, e->br};
        e->bd.alloc(sizeof(BracketDesc));
        RKFAC_CUDA(cudaMemcpy(e->bd.p, &b, sizeof(b), cudaMemcpyHostToDevice));
        const float inv = (float)(1.0 / lam);
        e->g1 = std::make_unique<TcGemm>();
        e->g2 = std::make_unique<TcGemm>();
        if (!left) {
            // RIGHT (kfactor.hpp:156-160): W = V U diag(b) (rows x r); out = W U^T + V / lambda
            TcProblemDesc p1;
            p1.M = rows; p1.N = r; p1.K = dim;
            p1.A = e->Vop; p1.lda = ldvop;
            p1.B = e->Ut; p1.ldb = dimp;
            p1.cs = e->br;
            p1.out0 = out_of(e->W, rp, 0);
            p1.slice_k = apply_slice(dim);
            e->g1->add(p1);
            TcProblemDesc p2;
            p2.M = rows; p2.N = dim; p2.K = r;
            p2.A = e->W; p2.lda = rp;
            p2.B = e->Uc; p2.ldb = rp;
            p2.gamma = inv; p2.Din = v; p2.lddin = ldv; p2.din_t = 0;
            p2.out0 = out_of(out, ldo, 0);
            e->g2->add(p2);
        } else {
            // LEFT (kfactor.hpp:147-152): W^T = (diag(b) U^T V)^T (cols x r); out = U W + V / lambda
            TcProblemDesc p1;
            p1.M = r; p1.N = cols; p1.K = dim;
            p1.A = e->Ut; p1.lda = dimp;
            p1.B = e->Vop; p1.ldb = ldvop;
            p1.rs = e->br;
            p1.out0 = out_of(e->W, rp, 1);
            p1.slice_k = apply_slice(dim);
            e->g1->add(p1);
            TcProblemDesc p2;
            p2.M = dim; p2.N = cols; p2.K = r;
            p2.A = e->Uc; p2.lda = rp;
            p2.B = e->W; p2.ldb = rp;
            p2.gamma = inv; p2.Din = v; p2.lddin = ldv; p2.din_t = 0;
            p2.out0 = out_of(out, ldo, 0);
            e->g2->add(p2);
        }
        e->g1->finalize();
        e->g2->finalize();
        ap_.push_front(std::move(ne));
        evict(ap_);
    }
    launch_bracket(e->bd.as<BracketDesc>(), 1, lam, s);
    launch_transpose(u, ldu, dim, r, e->Ut, pad4(dim), s);  // U^T: the K-major operand of the long-K product
    if (e->vt) launch_transpose(v, ldv, rows, cols, e->Vop, e->ldvop, s);
    e->in.launch(s);
    e->g1->launch(s);
    e->g2->launch(s);
    RKFAC_CUDA(cudaEventRecord(e->done, s));
}

}  // namespace rkfac_b200
