// kernels.cuh -- per-factor descriptors and launchers of the non-GEMM kernels of the path.
#pragma once

#include "common.cuh"

namespace rkfac_b200 {

// Omega^T (w x d) for factor f: Omega_ij = gaussian(seed_f, ctr0_f + 2(i*w + j)), stored at out[j*ld + i]
// (rng.hpp:59-63 fills row-major d x w; the transpose keeps the basis vectors contiguous).
struct OmegaDesc {
    int d, w;
    long long ld;
    float* out;
    uint64_t tag;       // substream tag (factor index f in optimizer.hpp:189)
    uint64_t seed;      // used when seeds are explicit
    uint64_t ctr0;
    long long offset;   // prefix of d*w over factors
    int rowmajor;       // 1: out[i*ld + j] (rng.hpp layout, used by rkfac_sample_gaussian)
    float* out_lo;      // optional TF32 lo plane (same layout): the 3xTF32 operand of the first X*Omega
};
// mode 0: seed_f = desc.seed; mode 1: seed_f = substream(root, step, tag_f)
void launch_omega(const OmegaDesc* d_descs, int nfactors, long long total, int mode, uint64_t root, uint64_t step,
                  cudaStream_t s, const uint64_t* seed_src = nullptr);

struct CholDesc {
    int w;
    const void* G;   // w x w Gram (double or float), row pitch ldg
    long long ldg;
    void* Linv;      // w x ldl output (double or float), lower triangular, zero-padded to a multiple of 4 columns
    long long ldl;
    void* Linv_lo;   // optional FP32 TF32-lo plane of Linv (same pitch)
    int* flags;      // w rank-deficiency flags
    int* nflags;     // any flag
    void* scratch;   // global fallback for the packed triangle
    // Split-K Gram (FP32 only): when part != nullptr, G is the fixed-order sum of nslices column-major w x w partials
    // (slice s, element (m, n) at part[s * w * w + n * w + m]; tc_gemm.cu's reduction order), formed while loading
    const float* part;
    int nslices;
};
size_t cholinv_smem_bytes(int wmax, bool fp64);
void launch_cholinv(const CholDesc* d_descs, int nfactors, int wmax, bool fp64, bool gram64, double tol,
                    cudaStream_t s);

struct CompleteDesc {
    int w, d;
    long long ldq;       // pitch of Qt / Qt_lo (w x d)
    float* Qt;
    const int* flags;
    const int* nflags;
    float* Qt_lo;        // optional derived planes refreshed for completed rows
    float* Q;            // optional row-major copy (d x w, pitch ldr)
    float* Q_lo;
    long long ldr;
};
void launch_complete(const CompleteDesc* d_descs, int nfactors, cudaStream_t s);
// Pseudo-random candidates into the flagged rows of a basis (before the final CholeskyQR2 pass).
void launch_fill(const CompleteDesc* d_descs, int nfactors, cudaStream_t s);

struct EigDesc {
    int n, r;            // core size (w) and number of eigenpairs wanted
    const float* A;      // n x n core (FP32, symmetric up to rounding)
    long long lda;
    double* scratch;     // packed triangle fallback (n(n+1)/2)
    double* refl;        // n x n reflectors
    double* tau;         // n
    double* dvec;        // n
    double* evec;        // n
    double* evals;       // r, descending
    double* scr;         // 4*n*r inverse-iteration LU
    unsigned char* piv;  // n*r
    double* z;           // n x r tridiagonal eigenvectors
    float* Pt;           // r x n eigenvectors of the core, transposed (row c = eigenvector c), pitch ldpt
    float* Ptlo;         // TF32 lo plane of Pt
    long long ldpt;
};
size_t tridiag_smem_bytes(int nmax);
void launch_eig(const EigDesc* d_descs, int nfactors, int nmax, int rmax, cudaStream_t s);

// Post-processing of the eigenvalues into the LowRankEig d-vector and the U-lift scales.
//   srevd (rnla.hpp:102-104): dvals = max(0, lam[:r]); colscale = 1.
//   rsvd_psd (eig.hpp:256-270): s = sqrt(max(0, mu)); zero modes (s <= tiny) get s = 0, scale 0 and a flag so
//   the lifted column is completed to an orthonormal direction.
struct PostDesc {
    int r;
    int method;          // RKFAC_SREVD / RKFAC_RSVD
    const double* evals; // r
    float* dvals;        // r (output)
    float* scale;        // r (U-lift row scale)
    int* flags;          // r zero-mode flags (rsvd)
    int* nflags;
};
void launch_post(const PostDesc* d_descs, int nfactors, cudaStream_t s);

// bracket_i = 1/(d_i + lambda) - 1/lambda = -d_i / (lambda (lambda + d_i)) (kfactor.hpp:140-142), FP64 math.
struct BracketDesc {
    int r;
    const float* dvals;
    float* out;
};
void launch_bracket(const BracketDesc* d_descs, int n, double lambda, cudaStream_t s);

// Grouped 2-D copy (all problems in one launch): dst[r*ldd + c] = src[r*lds + c], offset = prefix of rows*cols.
struct CopyDesc {
    const float* src;
    float* dst;
    int rows, cols;
    long long lds, ldd;
    long long offset;
};
void launch_copy(const CopyDesc* d_descs, int n, long long total, cudaStream_t s);

// Transposed copy: out[j*ldo + i] = in[i*ldi + j] for an rows x cols input (used by the single-factor API to
// return U in the reference's d x r layout).
void launch_transpose(const float* in, long long ldi, int rows, int cols, float* out, long long ldo, cudaStream_t s);

// x (rows x cols, pitch ld) *= a (ea_update with an empty update, kfactor.hpp:33-41 with n = 0).
void launch_scale(float* x, long long ld, int rows, int cols, float a, cudaStream_t s);

// x <- (x + x^T) / 2 for every descriptor's square matrix (kfactor.hpp:39 symmetrize_in_place), one launch.
struct SymDesc {
    float* x;
    long long ld;
    int d;
    long long offset;  // prefix of d*(d-1)/2 (strictly-lower pairs) over descriptors
};
void launch_symmetrize(const SymDesc* d_descs, int n, long long total, cudaStream_t s);

// Convolution factor statistics (stats.cu): the patch matrix of x (B x C x H x W, NCHW) scaled by `scale`,
// out[(c*kh + ky)*kw + kx][(b*Ho + oy)*Wo + ox], plus a row of `scale` when `ones`.
struct ConvPatchDesc {
    const float* x;
    int B, C, H, W, kh, kw, sh, sw, ph, pw, dh, dw, Ho, Wo, ones;
    float scale;
    float* out;
    long long ld;
};
void launch_conv_patches(const ConvPatchDesc& p, cudaStream_t s);
// out[co][b*hw + q] = scale * dy[b][co][q] (dy: B x Co x hw).
void launch_conv_grads(const float* dy, int B, int Co, long long hw, float scale, float* out, long long ld,
                       cudaStream_t s);

}  // namespace rkfac_b200
