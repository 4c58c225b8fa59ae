// engine.cuh -- the batched rand-K-FAC step: every factor of every layer in single launches per stage.
//
//   EA update      (kfactor.hpp:33-41)   one grouped symmetric 3xTF32 tcgen05 SYRK over all factors (upper tiles,
//                                        mirrored stores), epilogue rho*old + c*acc fused, TF32 lo plane of X fused
//   decomposition  (rnla.hpp:47-105)     Omega -> [X Q -> CholeskyQR] x (2q+1) -> core -> eig -> lift
//   precondition   (kfactor.hpp:134-161, optimizer.hpp:159-162)  RIGHT(A) then LEFT(Gamma), 4 grouped GEMMs
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "dmma.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "rsvd.cuh"
#include "single.cuh"
#include "symeig.cuh"
#include "tc_gemm.cuh"

namespace rkfac_b200 {

struct Context;

// A w x d tall-skinny matrix kept in the four layouts its consumers read as K-major TMA operands.
struct Role {
    float* T = nullptr;    // w x d, pitch dp (basis vectors contiguous)
    float* Tlo = nullptr;  // TF32 lo plane of T
    float* R = nullptr;    // d x w row-major, pitch wp
    float* Rlo = nullptr;
};

struct FactorState {
    int d = 0, r = 0, p = 0, q = 0, w = 0;  // clamped r, p; w = r + p
    int dp = 0;                              // d rounded up to 32 (pitch of internal w x d buffers)
    int wp = 0;                              // w rounded up to 4 (pitch of internal d x w / w x w buffers)
    // bound (caller-owned)
    float* X = nullptr;     // d x d
    long long ldx = 0;
    float* Ut = nullptr;    // r x d  (U^T)
    long long ldu = 0;
    float* dvals = nullptr; // r
    const float* M = nullptr;  // d x n samples
    long long n = 0, ldm = 0;
    uint64_t tag = 0;
    // plan-owned workspace (carved from the arena)
    Role S[2];                           // ping-pong sketch / basis
    float* Xc = nullptr;                 // padded copy of X (only when X itself is not a valid TMA operand)
    long long ldxa = 0;                  // pitch of the X operand actually fed to TMA (ldx or dp)
    float* Ml = nullptr;                 // TF32 lo plane of the samples (d x n, pitch ldm)
    double* G64 = nullptr;               // w x w
    float* G32 = nullptr;                // w x wp
    double* Linv64 = nullptr;            // w x wp
    float* Linv32 = nullptr;             // w x wp
    float* Linv32lo = nullptr;
    int* flags = nullptr;                // w + 1
    void* chol_scratch = nullptr;
    float* core = nullptr;               // w x w
    double *eig_scratch = nullptr, *refl = nullptr, *tau = nullptr, *dvec = nullptr, *evec = nullptr,
           *evals = nullptr, *scr = nullptr, *z = nullptr;
    unsigned char* piv = nullptr;
    float *Pt = nullptr, *Ptlo = nullptr;  // r x w (pitch wp): eigenvectors of the core, transposed
    float* scale = nullptr;              // r
    int* zflags = nullptr;               // r + 1
    float* bracket = nullptr;            // r
    int rp = 0;                          // r rounded up to 4
    // the basis in both K-major layouts (+ TF32 lo planes) for the tensor-core apply stage
    float *Uti = nullptr, *Utilo = nullptr;  // r x d, pitch dp
    float *Ui = nullptr, *Uilo = nullptr;    // d x r, pitch rp
};

struct LayerState {
    int a = 0, g = 0;
    const float* J = nullptr;  // dG x dA (caller pitch dA)
    float* out = nullptr;
    float* mid = nullptr;
    // plan-owned, TMA-aligned (pitches rounded up to 4 floats)
    float *Jc = nullptr, *Jlo = nullptr;       // dG x dA, pitch dAp
    float *W1 = nullptr, *W1lo = nullptr;      // dG x rA, pitch rAp
    float *Mt = nullptr, *Mtlo = nullptr;      // mid^T: dA x dG, pitch dGp
    float *W2t = nullptr, *W2tlo = nullptr;    // W2^T: dA x rG, pitch rGp
};

class Plan {
  public:
    Plan(Context* ctx, const rkfac_factor_desc* descs, int n, int method);
    ~Plan();

    int nfactors() const { return (int)f_.size(); }
    int nlayers() const { return (int)layers_.size(); }
    // device bytes the plan owns (rkfac_plan_workspace_size): per-factor arena, layer arena, sample lo planes, gather
    size_t workspace_bytes() const {
        return arena_.bytes + layer_arena_.bytes + ml_arena_.bytes + gather_send_.bytes;
    }
    FactorState& factor(int i) { return f_[i]; }
    int method() const { return method_; }

    void bind_factors(float* const* X, const long long* ldx, float* const* Ut, const long long* ldu,
                      float* const* dvals);
    void bind_samples(const float* const* M, const int64_t* n);
    void bind_layers(int nl, const int* a, const int* g, const float* const* J, float* const* out,
                     float* const* mid);
    void set_tags(const uint64_t* tags);
    void set_explicit_seed(int f, uint64_t seed, uint64_t ctr0);
    // EA operands' TF32 lo planes: -1 automatic (stored by a split pass when n >= 512), 0 formed in shared memory,
    // 1 stored by a split pass (arithmetic identical; rkfac_plan_set_ea_lo_mode)
    void set_ea_lo_mode(int mode);
    // overlapped power iteration (see decompose()): off by default
    void set_overlap(bool on) { overlap_orth_ = on; }

    void ea_update(double rho, double scale);
    // mode 1: seeds from substream(root, step, tag); mode 0: explicit seeds.
    // flags / j_copied: set by step() and ea_decompose(), which run Omega (and the gradient copy) next to the EA update
    enum DecompFlags { kOmegaAhead = 1, kDeferUtCopy = 2 };
    void decompose(int mode, uint64_t root, uint64_t step, bool x_lo_fresh = false, int flags = 0);
    void precondition(double lambda, bool j_copied = false);
    // EA update + decomposition of the same step (Omega generated next to the EA update)
    void ea_decompose(double rho, double scale, uint64_t root, uint64_t step);
    void step(double rho, double scale, uint64_t root, uint64_t step, double lambda);
    // Multi-GPU (config 4): step() ends with packing this rank's layer outputs at offsets[l] of a chunk of chunk
    // floats and all-gathering the chunks over the context's NCCL communicator into gathered (nranks * chunk).
    void set_gather(long long chunk, const long long* offsets, float* gathered);
    void gather();
    // Builds every stage a step with these parameters uses (descriptor uploads), so that the step itself only
    // enqueues kernels and can be captured into a CUDA graph.
    void prepare(double rho, double scale, double lambda);
    // (root, step) of the next replay of a captured step / decomposition (see captured_seed in engine.cu)
    void set_step_seed(uint64_t root, uint64_t step);

    enum TimingKind { kEA = 0, kDecompose = 1, kApply = 2, kXQ = 3, kOrth = 4, kEig = 5, kStep = 6, kTimingKinds = 7 };
    void set_timing(bool on) { timing_ = on; timing_reset(); }
    void set_max_ctas(int n);
    void timing_reset();
    // Sums (ms) and counts of each timed region since the last reset; call after the stream is synchronised.
    void timing_report(float* sums, int* counts) const;
    bool has_samples() const { return samples_bound_; }
    bool has_layers() const { return !layers_.empty(); }

    // Algorithmic FLOPs of one grouped X*Q launch (all factors), for roofline reporting.
    double xq_flops() const;

  private:
    void build_decomp_stages();
    std::unique_ptr<TcGemm> new_tc() const;
    void build_ea_stage(double rho, double scale);
    void build_apply_stages(double lambda);
    void orth(int src, bool fp64, cudaStream_t s, bool need_r = true);
    void mark(int kind, bool begin);
    bool launch_ahead(uint64_t root, uint64_t step, bool with_grads);
    const uint64_t* captured_seed(uint64_t root, uint64_t step, cudaStream_t s);

    Context* ctx_;
    int method_;
    std::vector<FactorState> f_;
    std::vector<LayerState> layers_;
    DevBuf arena_, layer_arena_, ml_arena_;
    DevBuf gather_send_, d_pack_;  // packed chunk of this rank's outputs and its copy descriptors
    float* gathered_ = nullptr;
    long long gather_chunk_ = 0, pack_total_ = 0;
    bool factors_bound_ = false, samples_bound_ = false;
    bool x_tma_ok_ = true;   // every bound X is a valid TMA operand (else a padded copy is made per decomposition)
    bool samples_tma_ok_ = false;  // every bound sample matrix is a valid TMA operand
    bool ea_tc_ = false;     // EA runs on the tensor-core path (needs TMA-valid X and samples; set by build_ea_stage)
    int ea_lo_mode_ = -1;    // see set_ea_lo_mode
    int ea_split_n_ = 0;     // > 0: the samples' TF32 lo planes are stored by a split pass (RKFAC_EA_STORED_LO=1)

    // Stage objects, indexed by the role buffer they write (xq, core: Y in S[dir]) or read (orth: src).
    // xqf_: the final X*Q (input of the core) with short accumulation chains (see kSliceK in engine.cu)
    // xq_tl_ / xz_: the overlapped power iteration's products (Y^T + lo plane only; Z row-major only)
    std::unique_ptr<TcGemm> xq_tl_[2], xz_[2];
    std::unique_ptr<TcGemm> xq_[2], xq_t_[2], xqf_[2], gram_[2], tri_[2], tri_t_[2], core_[2], lift_[2];
    std::unique_ptr<Gram64Batch> gram64_[2];
    std::unique_ptr<Tri64Batch> tri64_[2];
    std::unique_ptr<TcGemm> ea_tc_stage_, ea_long_stage_;
    DevBuf d_sym_;  // symmetrize descriptors of the long-K EA factors
    int sym_n_ = 0;
    long long sym_total_ = 0;
    std::unique_ptr<GemmBatch> ea_simt_;
    std::unique_ptr<TcGemm> ap_[4];
    DevBuf d_omega_, d_chol64_, d_chol32_[2], d_complete_[2], d_eig_, d_post_, d_complete_u_, d_bracket_;
    DevBuf d_split_x_, d_split_m_, d_split_omega_, d_split_j_, d_copy_ut_;
    long long split_x_total_ = 0, split_m_total_ = 0, split_j_total_ = 0, copy_ut_total_ = 0;
    std::vector<OmegaDesc> omega_;
    long long omega_total_ = 0;
    int wmax_ = 0, rmax_ = 0;
    double ea_rho_ = -1, ea_scale_ = -1, ap_lambda_ = -1;
    // Orthonormalisations done in FP64 (Gram, Cholesky, Y L^-T): only the first sketch Y0 = X Omega is
    // ill-conditioned enough (kappa ~1e4) to break FP32 CholeskyQR; measured on B200: 1 vs 2 FP64
    // orths give the same parity error, 0 gives eigenvalue errors of ~5e-2.
    int n_fp64_orth_ = 1;
    int tc_cap_ = 0;  // persistent tensor-core grid cap (0: all SMs)
    // overlapped power iteration (decompose): Gram + Cholesky-inverse on side_ next to the product X Y
    bool overlap_orth_ = false;  // opt-in (RKFAC_OVERLAP_ORTH=1): see decompose()
    int explicit_tail_ = 1;  // trailing products kept in the reference's order
    uint64_t* h_seed_ = nullptr;  // pinned (root, step) read by captured steps at replay
    DevBuf d_seed_;
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_pre_ = nullptr, ev_copy_ = nullptr;
    bool step_overlap_ = false;  // step(): Omega / gradient copy next to the EA update, U^T copy-out next to the apply

    bool timing_ = false;
    struct Rec { int kind; size_t b, e; };
    std::vector<cudaEvent_t> pool_;
    size_t pool_used_ = 0;
    size_t open_[kTimingKinds] = {};
    std::vector<Rec> recs_;
};

struct Context {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::string last_error;
    uint64_t launches_at_create = 0;
    // single-factor API plan cache
    struct Cached {
        int d, r, p, q, method;
        std::unique_ptr<Plan> plan;
        DevBuf ut, dv;
    };
    std::vector<Cached> cache;
    // cached tcgen05 stages of the single-factor ea_update / apply_lowrank_damped_inverse (single.cu)
    SingleOps single;
    // full d x d eigensolver of the exact K-FAC comparator and the spectrum snapshots (symeig.cu), workspace kept
    SymEig symeig;
    // general rectangular rsvd (rsvd.cu), workspace kept
    Rsvd rsvd;
    // optional NCCL communicator (ncclComm_t, caller-owned) for the plan's all-gather (comm.cu)
    void* nccl_comm = nullptr;
    int nccl_rank = 0, nccl_nranks = 1;
    bool nccl_owned = false;  // created by rkfac_nccl_init: destroyed with the context
};

bool tc_operand_ok(const float* p, long long ld);

}  // namespace rkfac_b200
