/*
 * rkfac_b200.h -- C-ABI of the B200-native randomized K-FAC hot path.
 *
 * Drop-in boundary for the reference's operator API (/root/reference/proj/include/rkfac):
 *
 *   reference (C++, FP64, CPU)                                   this ABI (FP32 device buffers, sm_100a)
 *   ------------------------------------------------------------ ------------------------------------------
 *   void ea_update(EAKFactor&, const DenseMatrix& m)             rkfac_ea_update           (kfactor.hpp:33-41)
 *   LowRankEig srevd(const DenseMatrix&, const SketchParams&,    rkfac_srevd               (rnla.hpp:90-105)
 *                    RngState&)
 *   LowRankEig rsvd_psd(const DenseMatrix&, const SketchParams&, rkfac_rsvd_psd            (rnla.hpp:81-85)
 *                       RngState&)
 *   DenseMatrix apply_lowrank_damped_inverse(const LowRankEig&,  rkfac_apply_lowrank_damped_inverse
 *                    double, const DenseMatrix&, ApplySide)                                 (kfactor.hpp:134-161)
 *   preconditioned_step's per-layer loop (optimizer.hpp:139-167) rkfac_plan_* (batched: every factor of every
 *                                                                 layer in single launches)
 *
 * Conventions
 *   - Every pointer argument named *_dev is a device pointer; matrices are row-major FP32 with an explicit
 *     leading dimension (elements), exactly the reference's DenseMatrix layout (matrix.hpp:47-48).
 *   - Calls are asynchronous on the context's CUDA stream (rkfac_set_stream), except where noted.
 *   - No C++ exception crosses this ABI: every entry point returns an rkfac_status that mirrors the reference
 *     exception types (errors.hpp:8-34); rkfac_last_error() gives the message.
 *   - RngState& is passed as (seed, *counter).  Like sample_gaussian (rng.hpp:59-63) the counter advances by
 *     2*d*w, so a caller that keeps a reference RngState stays bit-compatible with the CPU stream.
 *   - There is no CPU fallback: without a usable sm_100 device every call returns RKFAC_CUDA_ERROR.
 */
#ifndef RKFAC_B200_H
#define RKFAC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RKFAC_OK = 0,
    RKFAC_DIMENSION_MISMATCH = 1,  /* errors.hpp:8   DimensionMismatch  */
    RKFAC_RANK_DEFICIENT = 2,      /* errors.hpp:12  RankDeficient      */
    RKFAC_NO_CONVERGENCE = 3,      /* errors.hpp:16  NoConvergence      */
    RKFAC_DAMPING_NONPOSITIVE = 4, /* errors.hpp:20  DampingNonpositive */
    RKFAC_CUDA_ERROR = 5,
    RKFAC_NCCL_ERROR = 6,
    RKFAC_INVALID_ARGUMENT = 7
} rkfac_status;

typedef enum { RKFAC_RSVD = 0, RKFAC_SREVD = 1 } rkfac_method; /* DecompMethod, rnla.hpp:14 */
typedef enum { RKFAC_LEFT = 0, RKFAC_RIGHT = 1 } rkfac_side;   /* ApplySide, kfactor.hpp:128 */

typedef struct rkfac_context* rkfac_context_t;
typedef struct rkfac_plan* rkfac_plan_t;

/* ---- context ------------------------------------------------------------------------------------------ */
int rkfac_create(rkfac_context_t* ctx, int device, void* cuda_stream);
int rkfac_destroy(rkfac_context_t ctx);
int rkfac_set_stream(rkfac_context_t ctx, void* cuda_stream);
int rkfac_synchronize(rkfac_context_t ctx);
const char* rkfac_last_error(rkfac_context_t ctx);
const char* rkfac_status_string(int status);
/* Kernels launched by this library since the context was created (the bench's gpu_launches count). */
uint64_t rkfac_launch_count(rkfac_context_t ctx);

/* ---- single-factor operators (the reference signatures) ---------------------------------------------- */

/* rng.hpp:59-63 sample_gaussian: out (m x n row-major, FP32) = N(0,1) draws of RngState(seed) starting at
 * *counter (Box-Muller, cos branch, FP64 math); *counter advances by 2*m*n.  Omega of srevd/rsvd_psd is this. */
int rkfac_sample_gaussian(rkfac_context_t ctx, uint64_t seed, uint64_t* counter, int64_t m, int64_t n, float* out_dev,
                          int64_t ld_out);

/* kfactor.hpp:33-41: mbar (d x d) <- rho*mbar + (1-rho) * scale^2 * m m^T, m is d x n; mbar stays exactly
 * symmetric (upper tiles computed, mirrored).  Rows of m != d -> RKFAC_DIMENSION_MISMATCH. */
int rkfac_ea_update(rkfac_context_t ctx, float* mbar_dev, int64_t ld_mbar, int64_t d, const float* m_dev,
                    int64_t ld_m, int64_t m_rows, int64_t n, double rho, double scale);

/* rnla.hpp:90-105 srevd and rnla.hpp:81-85 rsvd_psd on a symmetric PSD x (d x d).
 * Sketch clamping as rnla.hpp:35-43; *rank_out = clamped r.  u_dev: d x rank_out row-major (ld_u >= rank_out),
 * dvals_dev: rank_out floats, descending.  Omega is drawn from (seed, *counter) exactly like the reference. */
int rkfac_srevd(rkfac_context_t ctx, const float* x_dev, int64_t ld_x, int64_t d, int64_t r, int64_t p, int64_t q,
                uint64_t seed, uint64_t* counter, float* u_dev, int64_t ld_u, float* dvals_dev, int64_t* rank_out);
int rkfac_rsvd_psd(rkfac_context_t ctx, const float* x_dev, int64_t ld_x, int64_t d, int64_t r, int64_t p,
                   int64_t q, uint64_t seed, uint64_t* counter, float* u_dev, int64_t ld_u, float* dvals_dev,
                   int64_t* rank_out);

/* rnla.hpp:62-77 rsvd on a general x (rows x cols): SvdResult {u: rows x rank_out (ld_u), s: rank_out (descending),
 * v: cols x rank_out (ld_v)}.  Sketch clamping with dim = min(rows, cols) (rnla.hpp:63); Omega (cols x w) is drawn
 * from (seed, *counter), which advances by 2*cols*w.  Synchronous; not on the optimizer path (which uses the square
 * PSD specialisation rkfac_rsvd_psd). */
int rkfac_rsvd(rkfac_context_t ctx, const float* x_dev, int64_t ld_x, int64_t rows, int64_t cols, int64_t r,
               int64_t p, int64_t q, uint64_t seed, uint64_t* counter, float* u_dev, int64_t ld_u, float* s_dev,
               float* v_dev, int64_t ld_v, int64_t* rank_out);

/* kfactor.hpp:134-161.  u: dim x r (row-major, orthonormal columns), dvals: r.  LEFT needs rows == dim,
 * RIGHT needs cols == dim.  lambda <= 0 -> RKFAC_DAMPING_NONPOSITIVE.  out may not alias v. */
int rkfac_apply_lowrank_damped_inverse(rkfac_context_t ctx, const float* u_dev, int64_t ld_u,
                                       const float* dvals_dev, int64_t dim, int64_t r, double lambda,
                                       const float* v_dev, int64_t ld_v, int64_t rows, int64_t cols, int side,
                                       float* out_dev, int64_t ld_out);

/* ---- factor statistics of convolution layers -------------------------------------------
 * The reference's MLP forms A_l = [a_{l-1}; 1] (with_ones_row, network.hpp:94-95) and G_l = delta_l
 * (network.hpp:134), and accumulate_factors feeds M = X / sqrt(n) to ea_update (network.hpp:155-165).  For a
 * convolution the statistics run over every output location: A is the patch matrix with a ones row,
 * d = C*kh*kw + 1 rows, n = B*Ho*Wo columns; G is the output gradient, Co rows, n columns.  Both write the EA operand
 * M = X * scale directly (row-major, pitch ld_out >= n); pass scale = 1/sqrt(n) and then rkfac_plan_ea_update(rho, 1).
 * Long n (> 512) is handled by the plan's EA as K slices of 512 + the symmetrize pass (accuracy). */
/* x: B x C x H x W (NCHW, contiguous); out[(c*kh + ky)*kw + kx][(b*Ho + oy)*Wo + ox]; ones_row appends a row of
 * `scale`.  Ho = (H + 2 ph - dh (kh-1) - 1) / sh + 1, likewise Wo. */
int rkfac_conv_patches(rkfac_context_t ctx, const float* x_dev, int64_t batch, int64_t channels, int64_t height,
                       int64_t width, int64_t kh, int64_t kw, int64_t stride_h, int64_t stride_w, int64_t pad_h,
                       int64_t pad_w, int64_t dil_h, int64_t dil_w, int ones_row, double scale, float* out_dev,
                       int64_t ld_out);
/* dy: B x Co x Ho x Wo (NCHW, contiguous); out[co][b*Ho*Wo + q] = scale * dy[b][co][q]. */
int rkfac_conv_grads(rkfac_context_t ctx, const float* dy_dev, int64_t batch, int64_t channels, int64_t out_h,
                     int64_t out_w, double scale, float* out_dev, int64_t ld_out);

/* eig.hpp:210-237 sym_eig: S (n x n symmetric, FP32, pitch lds) = P diag(d) P^T with the eigenvalues descending
 * (dvals: n FP32, and/or dvals64: n FP64; either may be NULL but not both) and the eigenvectors as the columns of P
 * (n x n FP32, pitch ldp; NULL: eigenvalues only).  FP64 Householder tridiagonalisation + divide and conquer +
 * back-transformation on the GPU.  Asymmetry above 1e-4 * max(1, |S|max) -> RKFAC_DIMENSION_MISMATCH
 * (eig.hpp:213-215's 1e-8 scaled for FP32 storage); no convergence of a leaf QL -> RKFAC_NO_CONVERGENCE.
 * Synchronous.  The exact K-FAC comparator (kfactor.hpp:165-186) and spectrum (kfactor.hpp:56-63) use it. */
int rkfac_sym_eig(rkfac_context_t ctx, const float* s_dev, int64_t lds, int64_t n, float* p_dev, int64_t ldp,
                  float* dvals_dev, double* dvals64_dev);

/* ---- batched plan: every factor of every layer in single launches ------------------------------------ */

typedef struct {
    int64_t dim;          /* d */
    int64_t rank;         /* r  (target_rank, before clamping) */
    int64_t oversampling; /* p  (r_l)                            */
    int64_t power_iters;  /* q  (n_pwr_it)                       */
} rkfac_factor_desc;

/* Creates a plan over nfactors factors decomposed with `method`.  The plan owns its workspaces; the caller
 * owns factors, bases, eigenvalues, samples, gradients and outputs (bound below). */
int rkfac_plan_create(rkfac_context_t ctx, const rkfac_factor_desc* descs, int nfactors, int method,
                      rkfac_plan_t* plan);
int rkfac_plan_destroy(rkfac_plan_t plan);
/* Clamped rank of factor f (rnla.hpp:35-43). */
int64_t rkfac_plan_rank(rkfac_plan_t plan, int f);

/* factors[f]: d_f x d_f (ld = d_f).  bases_t[f]: Ut, rank_f x d_f (ld = d_f), i.e. U^T (the basis vectors
 * contiguous).  dvals[f]: rank_f floats. */
int rkfac_plan_bind_factors(rkfac_plan_t plan, float* const* factors_dev, float* const* bases_t_dev,
                            float* const* dvals_dev);
/* As rkfac_plan_bind_factors with explicit row pitches (elements).  Pitches that are multiples of 4 with 16-byte
 * aligned bases let the EA update and the X*Q products feed the factor to TMA directly (no padded copy). */
int rkfac_plan_bind_factors_ld(rkfac_plan_t plan, float* const* factors_dev, const int64_t* ld_factors,
                               float* const* bases_t_dev, const int64_t* ld_bases, float* const* dvals_dev);
/* samples[f]: d_f x n_f (ld = n_f), the m argument of ea_update. */
int rkfac_plan_bind_samples(rkfac_plan_t plan, const float* const* samples_dev, const int64_t* n);
/* Layer l preconditions grads[l] (d_G x d_A, ld = d_A) with A-factor a_idx[l] and G-factor g_idx[l] into
 * outs[l] (d_G x d_A); mids[l] is caller scratch of the same shape (RIGHT(A) result). */
int rkfac_plan_bind_layers(rkfac_plan_t plan, int nlayers, const int* a_idx, const int* g_idx,
                           const float* const* grads_dev, float* const* outs_dev, float* const* mids_dev);

/* How the EA update gets the samples' TF32 lo planes (3xTF32 operands): -1 automatic (default: stored by a split
 * pass when some n >= 512, else formed in shared memory), 0 formed in shared memory, 1 stored.  Same arithmetic. */
int rkfac_plan_set_ea_lo_mode(rkfac_plan_t plan, int mode);
/* All factors: mbar <- rho*mbar + (1-rho)*scale^2 * m m^T (one launch). */
int rkfac_plan_ea_update(rkfac_plan_t plan, double rho, double scale);
/* All factors: rand-EVD with Omega_f from RngState(rng_root).substream(step, tag_f) (optimizer.hpp:189, 202),
 * tag_f = f unless rkfac_plan_set_tags was called. */
int rkfac_plan_decompose(rkfac_plan_t plan, uint64_t rng_root, uint64_t step);
int rkfac_plan_set_tags(rkfac_plan_t plan, const uint64_t* tags);
/* rkfac_plan_ea_update followed by rkfac_plan_decompose of the same step, as rkfac_plan_step runs them (Omega is
 * generated next to the EA update); bitwise the two separate calls. */
int rkfac_plan_ea_decompose(rkfac_plan_t plan, double rho, double scale, uint64_t rng_root, uint64_t step);
/* All layers: outs = LEFT_G(RIGHT_A(grads)) (optimizer.hpp:159-162). */
int rkfac_plan_precondition(rkfac_plan_t plan, double lambda);
/* EA (if samples bound) -> decompose -> precondition (if layers bound) -> all-gather (if rkfac_plan_set_gather). */
int rkfac_plan_step(rkfac_plan_t plan, double rho, double scale, uint64_t rng_root, uint64_t step, double lambda);
/* Device bytes the plan owns (the reference has no workspace: every op returns new matrices, matrix.hpp:14-65). */
size_t rkfac_plan_workspace_size(rkfac_plan_t plan);

/* ---- multi-GPU (BASELINE config 4): layers sharded over ranks, one NCCL all-gather ----------- */
/* The reference is single-process (optimizer.hpp:145-165 loops over independent layers; SPEC.md:391 allows them to
 * run concurrently): a rank decomposes and preconditions its own layers, then the packed preconditioned gradients
 * are all-gathered over NVLink/NVSwitch.  NCCL (libnccl.so.2) is loaded on first use; its errors are
 * RKFAC_NCCL_ERROR. */
/* Writes a new clique's 128-byte ncclUniqueId to id_out (rank 0; ship it to the other ranks out of band). */
int rkfac_nccl_unique_id(void* id_out);
/* Joins the clique as `rank` of `nranks` (ncclCommInitRank: blocks until every rank joined) and attaches the
 * communicator to the context, which owns it from then on. */
int rkfac_nccl_init(rkfac_context_t ctx, const void* unique_id, int nranks, int rank);
/* Attaches a caller-owned ncclComm_t instead. */
int rkfac_set_nccl_comm(rkfac_context_t ctx, void* nccl_comm, int nranks, int rank);
/* recv_dev (nranks * count floats, rank-major) <- every rank's send_dev (count floats), on the context stream. */
int rkfac_allgather(rkfac_context_t ctx, const float* send_dev, float* recv_dev, int64_t count);
/* rkfac_plan_step ends with the all-gather: layer l's output (d_G x d_A) is packed at offsets[l] (floats) of this
 * rank's chunk of chunk_elems floats, and the chunks of all ranks land in gathered_dev (nranks * chunk_elems).
 * gathered_dev = NULL turns it off. */
int rkfac_plan_set_gather(rkfac_plan_t plan, int64_t chunk_elems, const int64_t* offsets, float* gathered_dev);
/* The pack + all-gather alone (after rkfac_plan_precondition). */
int rkfac_plan_gather(rkfac_plan_t plan);

/* Stage timing with CUDA events on the context stream, recorded inside the calls and harvested after the caller
 * synchronises (no host sync inside a step).  set_timing(1) enables and resets.  rkfac_plan_timing fills 7 sums (ms)
 * and 7 counts indexed: 0 EA update, 1 decomposition, 2 preconditioning, 3 X*Q products (the GEMM stage),
 * 4 orthonormalisations, 5 core + eigensolve + lift, 6 whole step. */
int rkfac_plan_set_timing(rkfac_plan_t plan, int enabled);
/* Build every stage rkfac_plan_step(rho, scale, *, *, lambda) uses without launching anything, so the step only
 * enqueues kernels and may be captured into a CUDA graph.  A captured step reads (rng_root, step) from a pinned host
 * pair at every replay: rkfac_plan_set_step_seed before the replay gives that replay its Omega (optimizer.hpp:189:
 * the reference draws a fresh substream per step), so one graph serves every step id.  The pair is read by a copy
 * node of the replay, asynchronously: write a new pair only after the previous replay has consumed the old one (e.g.
 * after an event recorded behind that replay). */
int rkfac_plan_prepare(rkfac_plan_t plan, double rho, double scale, double lambda);
int rkfac_plan_set_step_seed(rkfac_plan_t plan, uint64_t rng_root, uint64_t step);
/* Overlapped power iteration (off by default): the middle products of randomized_range (rnla.hpp:47-56) are formed
 * as Y' = (X Y) L^-T, L = chol(Y^T Y), so the product runs next to the Gram + Cholesky-inverse instead of after them
 * (same iterate in exact arithmetic; the last product keeps the reference's order).  It shortens the per-factor
 * latency chain (a lone 4609-wide layer: 4.7 -> 3.7 ms), but the rounding of the Gram coefficients reaches the last
 * Ritz values as ~(6e-8 * lambda_1 / lambda_r)^2: within the 1e-4 bar while lambda_r / lambda_1 >~ 1e-5 (configs
 * 1-3 pass their parity tests with it), beyond it below that (config 5: 3e-4).  Enable it for factors whose retained
 * spectrum spans less than five decades. */
int rkfac_plan_set_overlap(rkfac_plan_t plan, int enabled);
/* Cap the persistent tensor-core grids of this plan at `ctas` CTAs (0: one per SM), leaving SMs to the
 * latency-bound per-factor kernels of plans running concurrently on other streams (StreamedStep). */
int rkfac_plan_set_max_ctas(rkfac_plan_t plan, int ctas);
int rkfac_plan_timing(rkfac_plan_t plan, float* sums_ms7, int* counts7);

#ifdef __cplusplus
}
#endif
#endif /* RKFAC_B200_H */
