// eig.cu -- symmetric eigensolver for the projected w x w core (replaces sym_eig, eig.hpp:210-237, as called by
// srevd rnla.hpp:99 and svd_small eig.hpp:253).
//
// The reference reduces to tridiagonal form (tred2, eig.hpp:33-124) and runs implicit QL (tql2, eig.hpp:131-193).
// QL's rotation chain is serial, so on the GPU the tridiagonal problem is solved with two embarrassingly parallel
// methods instead, all in FP64:
//   tridiag_kernel   -- Householder tridiagonalisation, one CTA per factor, packed lower triangle in shared
//                       memory (FP64 keeps the normwise backward error ~1e-16*||C||, i.e. ~1e-12 relative on the
//                       smallest retained eigenvalue of config 2).
//   tdeig_kernel     -- one thread per wanted eigenpair: bisection with Sturm counts (the k-th largest
//                       eigenvalue, so the output is already sorted descending like sort_desc_stable,
//                       eig.hpp:197-203), then inverse iteration with partial-pivoting LU; clusters of (near)
//                       equal eigenvalues are re-orthogonalised (modified Gram-Schmidt).
//   backxform_kernel -- P = H_0 ... H_{n-3} Z, the eigenvectors of the core.
// The cost is O(w^3) FP64 once (tridiagonalisation) instead of O(sweeps * w^3) for Jacobi; see DESIGN.md.
#include <cfloat>
#include <cmath>

#include "kernels.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kMaxN = 512;

__device__ __forceinline__ long long pk(int i, int j) { return (long long)i * (i + 1) / 2 + j; }

__device__ double block_sum_d(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        double s = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// ---------------------------------------------------------------------------------------------- tridiag
template <bool kSmem>  // compile-time storage choice: LDS/STS instead of generic LD/ST
__global__ void __launch_bounds__(1024) tridiag_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.x];
    const int n = ed.n;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* A;
    if constexpr (kSmem) A = reinterpret_cast<double*>(smem_raw);
    else A = ed.scratch;
    __shared__ double v[kMaxN], p[kMaxN], red[33];

    // Load the symmetrised lower triangle of the FP32 core.
    for (int i = warp; i < n; i += nwarp)
        for (int j = lane; j <= i; j += 32)
            A[pk(i, j)] = 0.5 * ((double)ed.A[(long long)i * ed.lda + j] + (double)ed.A[(long long)j * ed.lda + i]);
    __syncthreads();

    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;  // length of the column below the diagonal
        __syncthreads();
        // x = A[k+1:n, k]
        double sig = 0.0;
        for (int t = tid; t < m; t += nthr) {
            const double x = A[pk(k + 1 + t, k)];
            v[t] = x;
            if (t > 0) sig += x * x;
        }
        sig = block_sum_d(sig, red);
        const double alpha = v[0];
        double tau = 0.0, beta = alpha;
        if (sig > 0.0) {
            const double nrm = sqrt(alpha * alpha + sig);
            beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
        }
        const double scale = (sig > 0.0) ? 1.0 / (alpha - beta) : 0.0;
        __syncthreads();
        for (int t = tid; t < m; t += nthr) v[t] = (t == 0) ? 1.0 : v[t] * scale;
        if (tid == 0) {
            ed.dvec[k] = A[pk(k, k)];
            ed.evec[k] = beta;
            ed.tau[k] = tau;
        }
        __syncthreads();
        // Reflector storage (row k of refl, length m).
        for (int t = tid; t < m; t += nthr) ed.refl[(long long)k * n + t] = v[t];
        if (tau == 0.0) continue;

        // p = tau * A22 v  (A22 = A[k+1:, k+1:], lower-packed)
        int g = 1;
        while (g < 32 && g * 2 * m <= nthr) g *= 2;
        {
            const int row = tid / g, seg = tid % g;
            double acc = 0.0;
            if (row < m) {
                const int ii = k + 1 + row;
                for (int j = seg; j < m; j += g) {
                    const int jj = k + 1 + j;
                    const double a = (jj <= ii) ? A[pk(ii, jj)] : A[pk(jj, ii)];
                    acc += a * v[j];
                }
            }
            for (int off = g / 2; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off, g);
            if (row < m && seg == 0) p[row] = tau * acc;
        }
        __syncthreads();
        double pv = 0.0;
        for (int t = tid; t < m; t += nthr) pv += p[t] * v[t];
        pv = block_sum_d(pv, red);
        const double alpha2 = -0.5 * tau * pv;
        for (int t = tid; t < m; t += nthr) p[t] += alpha2 * v[t];  // p := w
        __syncthreads();
        // A22 -= v w^T + w v^T (lower triangle); rows paired (i, m-1-i) per warp for balance.
        for (int pr = warp; pr < (m + 1) / 2; pr += nwarp) {
            for (int h = 0; h < 2; ++h) {
                const int row = h == 0 ? pr : m - 1 - pr;
                if (h == 1 && row == pr) break;
                const int ii = k + 1 + row;
                const double vi = v[row], wi = p[row];
                for (int j = lane; j <= row; j += 32) {
                    const int jj = k + 1 + j;
                    A[pk(ii, jj)] -= vi * p[j] + wi * v[j];
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        if (n >= 2) {
            ed.dvec[n - 2] = A[pk(n - 2, n - 2)];
            ed.dvec[n - 1] = A[pk(n - 1, n - 1)];
            ed.evec[n - 2] = A[pk(n - 1, n - 2)];
            ed.tau[n - 2] = 0.0;
        } else {
            ed.dvec[0] = A[0];
        }
        ed.evec[n - 1] = 0.0;
        if (n >= 1) ed.tau[n - 1] = 0.0;
    }
}

// ------------------------------------------------------------------------------------- tridiagonal eig
// Number of eigenvalues of T strictly less than x (Sturm count, LAPACK dstebz style with pivmin guard).
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    if (q < 0.0) ++cnt;
    for (int i = 1; i < n; ++i) {
        q = d[i] - x - e2[i - 1] / q;
        if (fabs(q) < pivmin) q = -pivmin;
        if (q < 0.0) ++cnt;
    }
    return cnt;
}

__global__ void __launch_bounds__(256) tdeig_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.x];
    const int n = ed.n, r = ed.r;
    __shared__ double d[kMaxN], e[kMaxN], e2[kMaxN], lam[kMaxN];
    __shared__ double s_lo, s_hi, s_pivmin, s_tnorm;
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += blockDim.x) {
        d[i] = ed.dvec[i];
        e[i] = (i < n - 1) ? ed.evec[i] : 0.0;
        e2[i] = e[i] * e[i];
    }
    __syncthreads();
    if (tid == 0) {
        double lo = DBL_MAX, hi = -DBL_MAX, emax2 = 0.0, tn = 0.0;
        for (int i = 0; i < n; ++i) {
            const double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0);
            lo = fmin(lo, d[i] - off);
            hi = fmax(hi, d[i] + off);
            emax2 = fmax(emax2, e2[i]);
            tn = fmax(tn, fabs(d[i]) + off);
        }
        const double pivmin = DBL_MIN * fmax(1.0, emax2);
        const double pad = 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + 4.0 * pivmin;
        s_lo = lo - pad;
        s_hi = hi + pad;
        s_pivmin = pivmin;
        s_tnorm = fmax(tn, DBL_MIN);
    }
    __syncthreads();
    const double pivmin = s_pivmin, tnorm = s_tnorm;

    // Multisection for the k-th largest eigenvalue (ascending index n-1-k): 4 Sturm counts per iteration run as
    // independent chains (their divisions overlap), shrinking the bracket 5x per iteration instead of 2x.
    for (int k = tid; k < r; k += blockDim.x) {
        const int idx = n - 1 - k;
        double lo = s_lo, hi = s_hi;
        const double abstol = 4.0 * DBL_EPSILON * tnorm;
        for (int it = 0; it < 100; ++it) {
            if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + abstol) break;
            const double h = (hi - lo) * 0.2;
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = lo + h * (u + 1);
            if (x[0] <= lo || x[3] >= hi) {  // bracket at the resolution of doubles: plain bisection step
                const double mid = 0.5 * (lo + hi);
                if (mid == lo || mid == hi) break;
                if (sturm_count(d, e2, n, mid, pivmin) <= idx) lo = mid; else hi = mid;
                continue;
            }
            double q[4];
            int cnt[4] = {0, 0, 0, 0};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                q[u] = d[0] - x[u];
                if (fabs(q[u]) < pivmin) q[u] = -pivmin;
                cnt[u] += q[u] < 0.0;
            }
            for (int i = 1; i < n; ++i) {
                const double di = d[i], ei = e2[i - 1];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    q[u] = di - x[u] - ei / q[u];
                    if (fabs(q[u]) < pivmin) q[u] = -pivmin;
                    cnt[u] += q[u] < 0.0;
                }
            }
            // counts are nondecreasing in x: the eigenvalue lies in the first sub-interval whose right end has
            // more than idx eigenvalues below it
            double nlo = lo, nhi = hi;
#pragma unroll
            for (int u = 3; u >= 0; --u)
                if (cnt[u] <= idx) { nlo = x[u]; break; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (cnt[u] > idx) { nhi = x[u]; break; }
            lo = nlo;
            hi = nhi;
        }
        lam[k] = 0.5 * (lo + hi);
    }
    __syncthreads();
    for (int k = tid; k < r; k += blockDim.x) ed.evals[k] = lam[k];

    // Inverse iteration: (T - lam I) z = b, LU with partial pivoting.  Scratch layout [i][k] (coalesced).
    const long long S = r;
    double* U1 = ed.scr;             // diagonal of U
    double* U2 = ed.scr + n * S;     // first superdiagonal
    double* U3 = ed.scr + 2 * n * S; // second superdiagonal
    double* ML = ed.scr + 3 * n * S; // multipliers (sign bit unused), pivot flag in PV
    double* Z = ed.z;                // n x r (row-major, column k = eigenvector k)
    unsigned char* PV = ed.piv;      // n x r
    for (int k = tid; k < r; k += blockDim.x) {
        const double lmb = lam[k];
        const double eps_piv = DBL_EPSILON * tnorm;
        // Factor.
        double a = d[0] - lmb;
        double b = (n > 1) ? e[0] : 0.0;
        for (int i = 0; i < n - 1; ++i) {
            const double c = e[i];              // sub-diagonal entry T[i+1][i]
            const double anext = d[i + 1] - lmb; // diagonal of row i+1
            const double bnext = (i + 1 < n - 1) ? e[i + 1] : 0.0;
            if (fabs(a) >= fabs(c)) {
                double piv = a;
                if (piv == 0.0) piv = eps_piv;
                const double mult = c / piv;
                U1[i * S + k] = piv; U2[i * S + k] = b; U3[i * S + k] = 0.0;
                ML[i * S + k] = mult; PV[i * S + k] = 0;
                a = anext - mult * b;
                b = bnext;
            } else {
                const double mult = a / c;
                U1[i * S + k] = c; U2[i * S + k] = anext; U3[i * S + k] = bnext;
                ML[i * S + k] = mult; PV[i * S + k] = 1;
                a = b - mult * anext;
                b = -mult * bnext;
            }
        }
        U1[(n - 1) * S + k] = (a == 0.0) ? eps_piv : a;
        // Start vector: deterministic pseudo-random, then 3 solves.
        for (int i = 0; i < n; ++i) {
            const uint64_t h = splitmix64(0x5EEDULL ^ ((uint64_t)k << 32) ^ (uint64_t)i);
            Z[i * S + k] = (double)(h >> 11) * 0x1.0p-53 - 0.5;
        }
        for (int iter = 0; iter < 3; ++iter) {
            // forward: apply L^{-1} P
            for (int i = 0; i < n - 1; ++i) {
                const double zi = Z[i * S + k], zi1 = Z[(i + 1) * S + k];
                const double mult = ML[i * S + k];
                if (PV[i * S + k]) { Z[i * S + k] = zi1; Z[(i + 1) * S + k] = zi - mult * zi1; }
                else { Z[(i + 1) * S + k] = zi1 - mult * zi; }
            }
            // back substitution with U (diag, super1, super2)
            double z2 = 0.0, z1 = 0.0;  // z[i+2], z[i+1]
            double nrm = 0.0;
            for (int i = n - 1; i >= 0; --i) {
                double s = Z[i * S + k];
                if (i + 1 < n) s -= U2[i * S + k] * z1;
                if (i + 2 < n) s -= U3[i * S + k] * z2;
                const double zi = s / U1[i * S + k];
                Z[i * S + k] = zi;
                z2 = z1; z1 = zi;
                nrm = fmax(nrm, fabs(zi));
            }
            // rescale (avoid overflow) and normalise to unit 2-norm at the end
            const double inv = (nrm > 0.0) ? 1.0 / nrm : 1.0;
            double s2 = 0.0;
            for (int i = 0; i < n; ++i) { const double z = Z[i * S + k] * inv; Z[i * S + k] = z; s2 += z * z; }
            const double inv2 = 1.0 / sqrt(s2);
            for (int i = 0; i < n; ++i) Z[i * S + k] *= inv2;
        }
    }
    __syncthreads();
    // Re-orthogonalise clusters of (numerically) equal eigenvalues: MGS by one warp per cluster.
    const double clus = 1e-10 * tnorm;
    if (tid < 32) {
        int k = 0;
        while (k < r) {
            int k1 = k + 1;
            while (k1 < r && fabs(lam[k1 - 1] - lam[k1]) <= clus) ++k1;
            for (int pass = 0; pass < 2 && k1 - k > 1; ++pass) {
                for (int j = k; j < k1; ++j) {
                    for (int i = k; i < j; ++i) {
                        double dot = 0.0;
                        for (int t = tid; t < n; t += 32) dot += Z[t * S + i] * Z[t * S + j];
                        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                        for (int t = tid; t < n; t += 32) Z[t * S + j] -= dot * Z[t * S + i];
                        __syncwarp();
                    }
                    double nn = 0.0;
                    for (int t = tid; t < n; t += 32) nn += Z[t * S + j] * Z[t * S + j];
                    for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
                    const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
                    for (int t = tid; t < n; t += 32) Z[t * S + j] *= inv;
                    __syncwarp();
                }
            }
            k = k1;
        }
    }
}

// ------------------------------------------------------------------------------ back transformation
// Grid: (factor, column chunk of 32).  P[:, cols] = H_0 ... H_{n-3} Z[:, cols]; written as FP32 n x r.
constexpr int kBxCols = 32;
__global__ void __launch_bounds__(256) backxform_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.y];
    const int n = ed.n, r = ed.r;
    const int c0 = blockIdx.x * kBxCols;
    if (c0 >= r) return;
    const int nc = min(kBxCols, r - c0);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* Zs = reinterpret_cast<double*>(smem_raw);  // [n][kBxCols]
    __shared__ double vk[2][kMaxN], dots[kBxCols];
    const int tid = threadIdx.x;  // blockDim.x == 256: two reflector entries per thread (n <= 512)
    for (long long e = tid; e < (long long)n * kBxCols; e += blockDim.x) {
        const int i = (int)(e / kBxCols), c = (int)(e % kBxCols);
        Zs[e] = (c < nc) ? ed.z[(long long)i * r + c0 + c] : 0.0;
    }
    // The reflector of step k-1 is fetched into registers while step k computes (its global load latency was
    // the serial critical path: one L2 round trip per reflector).
    int buf = 0;
    double tau = 0.0;
    if (n >= 3) {
        const int k0 = n - 3, m0 = n - k0 - 1;
        for (int t = tid; t < m0; t += blockDim.x) vk[0][t] = ed.refl[(long long)k0 * n + t];
        tau = ed.tau[k0];
    }
    __syncthreads();
    for (int k = n - 3; k >= 0; --k) {
        const int m = n - k - 1;
        double pf0 = 0.0, pf1 = 0.0, tau_next = 0.0;
        if (k > 0) {
            const long long base = (long long)(k - 1) * n;
            if (tid < m + 1) pf0 = ed.refl[base + tid];
            if (tid + 256 < m + 1) pf1 = ed.refl[base + tid + 256];
            tau_next = ed.tau[k - 1];
        }
        if (tau != 0.0) {
            const double* v = vk[buf];
            // dots[c] = v^T Z[k+1:, c]; 8 threads per column.
            {
                const int c = tid / 8, seg = tid % 8;
                double s = 0.0;
                for (int t = seg; t < m; t += 8) s += v[t] * Zs[(long long)(k + 1 + t) * kBxCols + c];
                for (int o = 4; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o, 8);
                if (seg == 0) dots[c] = tau * s;
            }
            __syncthreads();
            for (long long e = tid; e < (long long)m * kBxCols; e += blockDim.x) {
                const int t = (int)(e / kBxCols), c = (int)(e % kBxCols);
                Zs[(long long)(k + 1 + t) * kBxCols + c] -= dots[c] * v[t];
            }
        }
        vk[buf ^ 1][tid] = pf0;
        if (tid + 256 < kMaxN) vk[buf ^ 1][tid + 256] = pf1;
        __syncthreads();
        buf ^= 1;
        tau = tau_next;
    }
    for (long long e = tid; e < (long long)n * kBxCols; e += blockDim.x) {
        const int i = (int)(e / kBxCols), c = (int)(e % kBxCols);
        if (c < nc) {
            const float v = (float)Zs[e];
            ed.Pt[(long long)(c0 + c) * ed.ldpt + i] = v;
            ed.Ptlo[(long long)(c0 + c) * ed.ldpt + i] = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
        }
    }
}

}  // namespace

size_t tridiag_smem_bytes(int nmax) { return (size_t)nmax * (nmax + 1) / 2 * 8; }

void launch_eig(const EigDesc* d_descs, int nfactors, int nmax, int rmax, cudaStream_t s) {
    if (nfactors == 0) return;
    RKFAC_REQUIRE(nmax <= kMaxN, RKFAC_INVALID_ARGUMENT, "core size above 512 is not supported");
    const size_t bytes = tridiag_smem_bytes(nmax);
    const bool use_smem = bytes <= max_dynamic_smem((const void*)tridiag_kernel<true>);
    auto k = use_smem ? tridiag_kernel<true> : tridiag_kernel<false>;
    const size_t dyn = use_smem ? bytes : 0;
    RKFAC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k<<<nfactors, 1024, dyn, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
    tdeig_kernel<<<nfactors, 256, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
    const size_t bx = (size_t)nmax * kBxCols * 8;
    RKFAC_CUDA(cudaFuncSetAttribute(backxform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bx));
    dim3 grid((unsigned)ceil_div(std::max(rmax, 1), kBxCols), (unsigned)nfactors);
    backxform_kernel<<<grid, 256, bx, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
