// eig.cu -- symmetric eigensolver for the projected w x w core (replaces sym_eig, eig.hpp:210-237, as called by
// srevd rnla.hpp:99 and svd_small eig.hpp:253).
//
// The reference reduces to tridiagonal form (tred2, eig.hpp:33-124) and runs implicit QL (tql2, eig.hpp:131-193).
// QL's rotation chain is serial, so on the GPU the tridiagonal problem is solved with two embarrassingly parallel
// methods instead, all in FP64:
//   tridiag_kernel   -- Householder tridiagonalisation, one CTA per factor, packed lower triangle in shared
//                       memory (FP64 keeps the normwise backward error ~1e-16*||C||, i.e. ~1e-12 relative on the
//                       smallest retained eigenvalue of config 2).
//   bisect_kernel    -- 4 threads per wanted eigenvalue (5-section per step), grid (eigenvalue chunk, factor):
//                       division-free Sturm counts for the k-th largest eigenvalue, so the output is already
//                       sorted descending like sort_desc_stable (eig.hpp:197-203).
//   eigvec_kernel    -- one thread per eigenpair: twisted factorisation (one solve) for isolated eigenvalues,
//                       inverse iteration (partial-pivoting LU) for members of clusters.
//   reorth_kernel    -- modified Gram-Schmidt over clusters of (near) equal eigenvalues.
//   backxform_kernel -- P = H_0 ... H_{n-3} Z, the eigenvectors of the core.
// The cost is O(w^3) FP64 once (tridiagonalisation) instead of O(sweeps * w^3) for Jacobi; see DESIGN.md.
#include <cfloat>
#include <cmath>

#include <cooperative_groups.h>
#include <cstdlib>

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

// ------------------------------------------------------------------------------ tridiag on a CTA cluster
// The same reduction spread over a cluster of 4 CTAs per factor (4 SMs; the 32 single-CTA factors left 116 SMs
// idle).  CTA q owns the full rows i = q (mod 4) of the symmetric matrix (no packing, contiguous row dots), so:
//   (B) p_i = tau A_i,: v is a local row dot (8 threads per row, shuffle tree), broadcast to the 4 CTAs through
//       distributed shared memory together with per-warp partials of p^T v;
//   (C) A_ij -= v_i w_j + w_i v_j on the owned rows (explicitly rounded products: row j's owner computes the
//       mirror element bit-identically, the matrix stays exactly symmetric); the owners of the next column
//       broadcast its entries and partial norms.
// Two cluster barriers per column step; the reflector (beta, tau, v) is derived redundantly by every thread.
constexpr int kTcC = 4;
constexpr int kTcThreads = 512;
constexpr int kTcWarps = kTcThreads / 32;
constexpr int kTcG = 8;  // threads per row
constexpr int kTcMaxN = 320;

#ifdef RKFAC_TRC_TIMING  // per-phase clock64 stamps of one step (tools/eig_bench.cu)
__device__ long long g_trc[16];
#define TRC_PHASE(k, slot)                                                                     \
    do {                                                                                       \
        const long long t_ = clock64();                                                        \
        if ((k) == RKFAC_TRC_TIMING && threadIdx.x == 0 && blockIdx.x == 0) g_trc[slot] = t_; \
        __syncwarp();                                                                          \
    } while (0)
#else
#define TRC_PHASE(k, slot)
#endif

size_t tridiag_cluster_smem_bytes(int n) {
    const int nloc = (n + kTcC - 1) / kTcC;
    return ((size_t)nloc * n + 5 * (size_t)n + 3 * kTcC * kTcWarps) * sizeof(double);
}

// Cluster barrier with release/acquire at cluster scope (the cooperative-groups sync adds a GPU-scope fence).
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __cluster_dims__(kTcC, 1, 1) __launch_bounds__(kTcThreads)
    tridiag_cluster_kernel(const EigDesc* __restrict__ descs) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();
    const EigDesc& ed = descs[blockIdx.x / kTcC];
    const int n = ed.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nloc = (n - q + kTcC - 1) / kTcC;  // rows i = q + 4 li, li < nloc
    extern __shared__ __align__(16) double tsm[];
    double* R = tsm;                                   // nloc x n
    double* const xbuf0 = R + (size_t)((n + kTcC - 1) / kTcC) * n;  // column below the diagonal (double-buffered)
    double* const xbuf1 = xbuf0 + n;
    double* pbuf = xbuf0 + 2 * n;                      // p (relative index)
    double* vs = xbuf0 + 3 * n;                        // v of this step
    double* ws = xbuf0 + 4 * n;                        // w of this step
    double* sigp = xbuf0 + 5 * n;                      // [2][kTcC][kTcWarps]
    double* pvp = sigp + 2 * kTcC * kTcWarps;          // [kTcC][kTcWarps]
    // distributed-smem stores: element e of buffer buf in all 4 CTAs of the cluster
    auto bcast = [&](double* buf, int e, double v) {
#pragma unroll
        for (int r = 0; r < kTcC; ++r) cluster.map_shared_rank(buf, r)[e] = v;
    };
    // owned rows, symmetrised from the FP32 core
    for (int li = warp; li < nloc; li += kTcWarps) {
        const int i = q + kTcC * li;
        for (int j = lane; j < n; j += 32)
            R[(size_t)li * n + j] =
                0.5 * ((double)ed.A[(long long)i * ed.lda + j] + (double)ed.A[(long long)j * ed.lda + i]);
    }
    cluster.sync();  // every CTA of the cluster is running: distributed smem may be written
    // first column: x_t = A[1 + t][0]
    if (n >= 3) {
        double s = 0.0;
        for (int li = tid; li < nloc; li += kTcThreads) {
            const int i = q + kTcC * li;
            if (i >= 1) {
                const double a = R[(size_t)li * n];
                bcast(xbuf0, i - 1, a);
                if (i >= 2) s += a * a;
            }
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) bcast(sigp, q * kTcWarps + warp, s);
    }
    cluster_barrier();

    const int g = tid / kTcG, sub = tid % kTcG;
    const unsigned gmask = 0xFFu << (lane & ~(kTcG - 1));  // the row's 8 lanes (groups diverge in trip count)
    constexpr int kGroups = kTcThreads / kTcG;
    for (int k = 0; k + 2 < n; ++k) {
        const int base = k + 1, m = n - base, cur = k & 1, nxt = cur ^ 1;
        const double* x = cur ? xbuf1 : xbuf0;
        double* xnext = cur ? xbuf0 : xbuf1;
        TRC_PHASE(k, 0);
        // (A) reflector (fixed-order sums of the 32 partials), v into smem
        double sig = 0.0;
#pragma unroll
        for (int e = lane; e < kTcC * kTcWarps; e += 32) sig += sigp[cur * kTcC * kTcWarps + e];
        for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
        const double alpha = x[0];
        double tau = 0.0, beta = alpha;
        if (sig > 0.0) {
            const double nrm = sqrt(alpha * alpha + sig);
            beta = alpha >= 0.0 ? -nrm : nrm;
            tau = (beta - alpha) / beta;
        }
        const double scale = (sig > 0.0) ? 1.0 / (alpha - beta) : 0.0;
        for (int t = tid; t < m; t += kTcThreads) {
            const double v = t == 0 ? 1.0 : x[t] * scale;
            vs[t] = v;
            if (q == 0) ed.refl[(long long)k * n + t] = v;
        }
        if (q == 0 && tid == 0) {
            ed.evec[k] = beta;
            ed.tau[k] = tau;
        }
        if (q == (k & (kTcC - 1)) && tid == 0) ed.dvec[k] = R[(size_t)(k / kTcC) * n + k];
        __syncthreads();
        TRC_PHASE(k, 1);
        // (B) p_i = tau sum_j A_ij v_j over the owned rows i >= base
        const int li0 = (base - q + kTcC - 1) / kTcC;  // first owned row >= base
        double pvpart = 0.0;
        for (int li = li0 + g; li < nloc; li += kGroups) {
            const int i = q + kTcC * li;
            const double* row = R + (size_t)li * n + base;
            double a0 = 0.0, a1 = 0.0;
            int t = sub;
            for (; t + kTcG < m; t += 2 * kTcG) {
                a0 += row[t] * vs[t];
                a1 += row[t + kTcG] * vs[t + kTcG];
            }
            if (t < m) a0 += row[t] * vs[t];
            double acc = a0 + a1;
#pragma unroll
            for (int o = kTcG / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(gmask, acc, o);
            const double p = tau * acc;
            if (sub == 0) {
                bcast(pbuf, i - base, p);
                pvpart += p * vs[i - base];
            }
        }
        for (int o = 16; o > 0; o >>= 1) pvpart += __shfl_xor_sync(0xffffffffu, pvpart, o);
        if (lane == 0) bcast(pvp, q * kTcWarps + warp, pvpart);
        TRC_PHASE(k, 2);
        cluster_barrier();
        TRC_PHASE(k, 3);
        // (C) rank-2 update of the owned rows; the next column's entries and partial norms are broadcast
        double pv = 0.0;
#pragma unroll
        for (int e = lane; e < kTcC * kTcWarps; e += 32) pv += pvp[e];
        for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
        const double alpha2 = -0.5 * tau * pv;
        for (int t = tid; t < m; t += kTcThreads) ws[t] = pbuf[t] + alpha2 * vs[t];
        __syncthreads();
        double s2 = 0.0;
        for (int li = li0 + g; li < nloc; li += kGroups) {
            const int i = q + kTcC * li;
            double* row = R + (size_t)li * n + base;
            const double vr = vs[i - base], wr = ws[i - base];
            // explicitly rounded products: row j's owner computes the mirror element bit-identically
            auto upd = [&](int t) {
                const double a = __dsub_rn(row[t], __dadd_rn(__dmul_rn(vr, ws[t]), __dmul_rn(wr, vs[t])));
                row[t] = a;
                return a;
            };
            int t = sub;
            if (sub == 0) {  // column base: the next x
                const double a = upd(0);
                if (i >= base + 1) {
                    bcast(xnext, i - base - 1, a);
                    if (i >= base + 2) s2 += a * a;
                }
                t = kTcG;
            }
            for (; t + kTcG < m; t += 2 * kTcG) {
                upd(t);
                upd(t + kTcG);
            }
            if (t < m) upd(t);
        }
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0) bcast(sigp, (nxt * kTcC + q) * kTcWarps + warp, s2);
        TRC_PHASE(k, 4);
        cluster_barrier();
        TRC_PHASE(k, 5);
    }
    // trailing 2 x 2 (or 1 x 1)
    if (tid == 0) {
        if (n >= 2) {
            if (q == ((n - 2) & (kTcC - 1))) ed.dvec[n - 2] = R[(size_t)((n - 2) / kTcC) * n + (n - 2)];
            if (q == ((n - 1) & (kTcC - 1))) {
                ed.dvec[n - 1] = R[(size_t)((n - 1) / kTcC) * n + (n - 1)];
                ed.evec[n - 2] = R[(size_t)((n - 1) / kTcC) * n + (n - 2)];
            }
            if (q == 0) {
                ed.tau[n - 2] = 0.0;
                ed.evec[n - 1] = 0.0;
                ed.tau[n - 1] = 0.0;
            }
        } else if (q == 0) {
            ed.dvec[0] = R[0];
            ed.evec[0] = 0.0;
            ed.tau[0] = 0.0;
        }
    }
    cluster.sync();  // no CTA leaves while others may still write into its shared memory
}

// --------------------------------------------------------- tridiag on a CTA cluster, one barrier per column
// Same reduction, same cluster shape (CTA q owns the full rows i = q mod 4), restructured so that each column step
// costs ONE cluster barrier and ONE pass over the owned rows:
//   * every warp holds the reflector v_k, w_k and the next reflector v_{k+1} in registers, indexed by absolute
//     column (lane + 32 t), and derives them redundantly: after the barrier of step k it has p_k (pushed by the row
//     owners) and the entries of column k+1 as they were before update k (pushed one step early), so
//     w_k = p_k - (tau_k/2)(p_k.v_k) v_k and column k+1 after update k, hence v_{k+1}, need no further exchange;
//   * the pass over an owned row i applies update k (A_ij -= v_i w_j + w_i v_j, explicitly rounded products so
//     that row j's owner and the redundant column computation agree bit for bit) and accumulates
//     p_{k+1,i} = tau_{k+1} A_i. v_{k+1} from the updated values, then pushes (p_{k+1,i}, A_{i,k+2}) to every CTA
//     as one 16-byte store (double-buffered by step parity: with one barrier per step no CTA is more than one
//     step ahead of another).
template <int NT>
__device__ __forceinline__ double sel_slot(const double (&a)[NT], int s) {
    double r = 0.0;
#pragma unroll
    for (int t = 0; t < NT; ++t) r = (t == s) ? a[t] : r;
    return r;
}
// element j of a register vector held as v[t] at lane j % 32, slot j / 32 (uniform j across the warp)
template <int NT>
__device__ __forceinline__ double vget(const double (&a)[NT], int j) {
    return __shfl_sync(0xffffffffu, sel_slot<NT>(a, j >> 5), j & 31);
}
// 1/x and 1/sqrt(x) for the per-column reflector: hardware approximations (rcp/rsqrt.approx.f64, ~2^-23) refined by
// two Newton steps (~2^-92 before rounding): within an ulp of the IEEE results at a fraction of their latency, which
// sits on the serial chain of every column (x > 0, normal).
__device__ __forceinline__ double rcp_fast(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = fma(y, fma(-x, y, 1.0), y);
    y = fma(y, fma(-x, y, 1.0), y);
    return y;
}
__device__ __forceinline__ double rsqrt_fast(double x) {
    double y;
    asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    y = y * fma(-h * y, y, 1.5);
    y = y * fma(-h * y, y, 1.5);
    return y;
}

template <int NT>
__device__ __forceinline__ double tree_sum(const double (&a)[NT]) {
    double t[NT];
#pragma unroll
    for (int i = 0; i < NT; ++i) t[i] = a[i];
#pragma unroll
    for (int w = 1; w < NT; w *= 2)
#pragma unroll
        for (int i = 0; i + w < NT; i += 2 * w) t[i] += t[i + w];
    return t[0];
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double rank2(double a, double vi, double wj, double wi, double vj) {
    return __dsub_rn(a, __dadd_rn(__dmul_rn(vi, wj), __dmul_rn(wi, vj)));
}

#ifndef RKFAC_T1B_THREADS
#define RKFAC_T1B_THREADS 256
#endif
#ifndef RKFAC_T1B_U
#define RKFAC_T1B_U 1
#endif
#ifndef RKFAC_T1B_LOADFIRST
#define RKFAC_T1B_LOADFIRST 1
#endif
constexpr int kT2Threads = RKFAC_T1B_THREADS;
constexpr int kT2Warps = kT2Threads / 32;

size_t tridiag1b_smem_bytes(int n) {
    const int nloc = (n + kTcC - 1) / kTcC;
    const int nt = n <= 256 ? 8 : 10;  // the kernel's NT
    const int rmax = (32 * nt / kTcC + kT2Warps - 1) / kT2Warps;  // per-warp row partials of the deferred reduction
    return ((((size_t)nloc * n + 1) & ~(size_t)1) + 4 * (size_t)n + (size_t)kT2Warps * rmax * 34 +
            (size_t)kT2Warps * 64 * nt) * sizeof(double);
}

template <int NT, int U>
__global__ void __cluster_dims__(kTcC, 1, 1) __launch_bounds__(kT2Threads)
    tridiag1b_kernel(const EigDesc* __restrict__ descs) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();
    const EigDesc& ed = descs[blockIdx.x / kTcC];
    const int n = ed.n;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nloc = (n - q + kTcC - 1) / kTcC;  // rows i = q + 4 li
    const bool writer = q == 0 && warp == 0;     // global outputs of the reflectors
    extern __shared__ __align__(16) double tsm[];
    double* R = tsm;                                                       // nloc x n
    double2* pc = reinterpret_cast<double2*>(R + (((size_t)((n + kTcC - 1) / kTcC) * n + 1) & ~(size_t)1));
    // pc: [2][n] of (p_i, A_{i,next column}), pushed by the row owners
    constexpr int kRowsPerWarp = (32 * NT / kTcC + kT2Warps - 1) / kT2Warps;  // owned rows per warp, at most
    double* wpart = reinterpret_cast<double*>(pc + 2 * n) + warp * (kRowsPerWarp * 33 + kRowsPerWarp);
    double* wcn = wpart + kRowsPerWarp * 33;
    // per-warp copy of v_k and w_k (the pass reads v_i, w_i of each owned row with one broadcast load each)
    double* sV = reinterpret_cast<double*>(pc + 2 * n) + kT2Warps * (kRowsPerWarp * 33 + kRowsPerWarp) + warp * 64 * NT;
    double* sW = sV + 32 * NT;
    auto push = [&](int buf, int i, double p, double c) {  // lanes 0..3 store into CTA `lane`
        if (lane < kTcC) cluster.map_shared_rank(pc, lane)[buf * n + i] = make_double2(p, c);
    };
    for (int li = warp; li < nloc; li += kT2Warps) {
        const int i = q + kTcC * li;
        for (int j = lane; j < n; j += 32)
            R[(size_t)li * n + j] =
                0.5 * ((double)ed.A[(long long)i * ed.lda + j] + (double)ed.A[(long long)j * ed.lda + i]);
    }
    __syncthreads();
    if (n < 3) {  // nothing to reduce
        if (q == 0 && tid == 0) {
            ed.dvec[0] = R[0];
            ed.evec[0] = 0.0;
            ed.tau[0] = 0.0;
            if (n == 2) {
                ed.evec[0] = R[1];
                ed.tau[1] = 0.0;
                ed.evec[1] = 0.0;
            }
        }
        if (q == 1 && tid == 0 && n == 2) ed.dvec[1] = R[1];
        return;
    }
    cluster.sync();  // every CTA runs: distributed shared memory may be written
    // columns 0 and 1 (rows i >= 1) into buffer 1
    for (int li = warp; li < nloc; li += kT2Warps) {
        const int i = q + kTcC * li;
        if (i >= 1) push(1, i, R[(size_t)li * n], R[(size_t)li * n + 1]);
    }
    if (q == 0 && tid == 0) ed.dvec[0] = R[0];
    cluster_barrier();

    // reflector from a column x (entries j >= b; x_b = alpha): v_b = 1, v_j = x_j / (alpha - beta)
    double V[NT], W[NT], Vn[NT];
    double tau = 0.0, taun = 0.0;
    auto reflector = [&](const double (&x)[NT], int b, double (&v)[NT], double& t) {
        double sq[NT];
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            sq[s] = (j > b && j < n) ? x[s] * x[s] : 0.0;
        }
        double sig = tree_sum<NT>(sq);  // pairwise within the lane: a 3-deep chain instead of NT
        sig = warp_sum_d(sig);
        const double alpha = vget<NT>(x, b);
        double beta = alpha;
        t = 0.0;
        double scale = 0.0;
        if (sig > 0.0) {
            // one square root and one division: with beta = -sign(alpha) nrm, tau = (beta - alpha) / beta
            // = 1 + |alpha| / nrm and 1 / (alpha - beta) = sign(alpha) / (|alpha| + nrm)
            const double s2 = alpha * alpha + sig;
            const double rn = rsqrt_fast(s2);  // 1 / nrm
            const double nrm = s2 * rn;
            const double aa = fabs(alpha);
            beta = alpha >= 0.0 ? -nrm : nrm;
            t = 1.0 + aa * rn;
            scale = (alpha >= 0.0 ? 1.0 : -1.0) * rcp_fast(aa + nrm);
        }
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            v[s] = (j == b) ? 1.0 : ((j > b && j < n) ? x[s] * scale : 0.0);
        }
        return beta;
    };
    // the reflector's global copy: slot s written by warp s % kT2Warps of CTA 0 (one store per lane and warp, so no
    // warp carries the writes on the step's critical path)
    auto write_refl = [&](int k, const double (&v)[NT], double beta, double t) {
        if (q != 0) return;
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            if (s % kT2Warps == warp && j > k && j < n) ed.refl[(long long)k * n + (j - k - 1)] = v[s];
        }
        if (warp == kT2Warps - 1 && lane == 0) {
            ed.evec[k] = beta;
            ed.tau[k] = t;
        }
    };
    {
        double x[NT];
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            x[s] = (j >= 1 && j < n) ? pc[n + j].x : 0.0;
        }
        const double beta = reflector(x, 1, V, tau);
        write_refl(0, V, beta, tau);
    }
    // p_0 over the owned rows i >= 1, with column 1 (rows >= 1) re-pushed alongside into buffer 0
    for (int li = warp; li < nloc; li += kT2Warps) {
        const int i = q + kTcC * li;
        if (i < 1) continue;
        const double* row = R + (size_t)li * n;
        double dot = 0.0;
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            if (j >= 1 && j < n) dot += row[j] * V[s];
        }
        dot = warp_sum_d(dot);
        push(0, i, tau * dot, row[1]);
    }
    cluster_barrier();

    for (int k = 0; k + 2 < n; ++k) {
        const int b = k + 1;  // update k acts on indices >= b
        const double2* cur = pc + (k & 1) * n;
        TRC_PHASE(k, 8);
        // w_k = p_k - (tau_k / 2)(p_k . v_k) v_k
        double P[NT], pvs[NT];
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            P[s] = (j >= b && j < n) ? cur[j].x : 0.0;
            pvs[s] = P[s] * V[s];
        }
        double pv = warp_sum_d(tree_sum<NT>(pvs));
        const double alpha2 = -0.5 * tau * pv;
        TRC_PHASE(k, 12);
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            W[s] = P[s] + alpha2 * V[s];
            sV[lane + 32 * s] = V[s];
            sW[lane + 32 * s] = W[s];
        }
        __syncwarp();
        // column b+... : x = column b after update k (entries j >= b; j = b is the diagonal d_b)
        const double vb = sV[b], wb = sW[b];  // the per-warp copy written just above
        double x[NT];
#pragma unroll
        for (int s = 0; s < NT; ++s) {
            const int j = lane + 32 * s;
            x[s] = (j >= b && j < n) ? rank2(cur[j].y, V[s], wb, W[s], vb) : 0.0;
        }
        TRC_PHASE(k, 13);
        const bool more = k + 3 < n;  // reflector b exists
        if (q == 0 && warp == kT2Warps - 2) {
            const double db = vget<NT>(x, b);
            if (lane == 0) ed.dvec[b] = db;
        }
        if (more) {
            const double beta = reflector(x, b + 1, Vn, taun);
            TRC_PHASE(k, 14);
            write_refl(b, Vn, beta, taun);
        } else {
            // last 2 x 2: d_{n-1} comes from the pushed diagonal after this update; e_{n-2} = x_{n-1}
            const double e = vget<NT>(x, n - 1);
            if (writer && lane == 0) {
                ed.evec[n - 2] = e;
                ed.tau[n - 2] = 0.0;
                ed.evec[n - 1] = 0.0;
                ed.tau[n - 1] = 0.0;
            }
#pragma unroll
            for (int s = 0; s < NT; ++s) Vn[s] = 0.0;
            taun = 0.0;
        }
        TRC_PHASE(k, 9);
        // one pass over the owned rows i >= b + 1: apply update k, accumulate p_{k+1,i}, push with A_{i,b+1};
        // U rows of the warp at a time (independent chains overlap; the loop over row chunks stays rolled so the
        // step's code fits the instruction cache)
        {
            const int li_first = max(0, (b + 1 - q + kTcC - 1) / kTcC);  // first owned row >= b + 1
#pragma unroll 1
            for (int l0 = li_first + warp; l0 < nloc; l0 += U * kT2Warps) {
                double vi[U], wi[U], dot[U], cn[U];
                double* row[U];
                bool ok[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    ok[u] = l0 + u * kT2Warps < nloc;
                    const int li = min(l0 + u * kT2Warps, nloc - 1);
                    const int i = q + kTcC * li;
                    vi[u] = sV[i];
                    wi[u] = sW[i];
                    dot[u] = 0.0;
                    cn[u] = 0.0;
                    row[u] = R + (size_t)li * n;
                }
#if RKFAC_T1B_LOADFIRST
                // all loads first (stores to one row must not order the loads of another), then the updates,
                // then the stores
                double a[U][NT];
#pragma unroll
                for (int s = 0; s < NT; ++s) {
                    const int j = lane + 32 * s;
#pragma unroll
                    for (int u = 0; u < U; ++u) a[u][s] = (ok[u] && j >= b + 1 && j < n) ? row[u][j] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    double pr[NT];
#pragma unroll
                    for (int s = 0; s < NT; ++s) {
                        const int j = lane + 32 * s;
                        a[u][s] = rank2(a[u][s], vi[u], W[s], wi[u], V[s]);
                        pr[s] = a[u][s] * Vn[s];  // Vn is zero outside [b + 1, n)
                        if (j == b + 1) cn[u] = a[u][s];
                    }
                    dot[u] = tree_sum<NT>(pr);
                }
#pragma unroll
                for (int s = 0; s < NT; ++s) {
                    const int j = lane + 32 * s;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (ok[u] && j >= b + 1 && j < n) row[u][j] = a[u][s];
                }
#else
#pragma unroll
                for (int s = 0; s < NT; ++s) {
                    const int j = lane + 32 * s;
                    if (j >= b + 1 && j < n) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (ok[u]) {
                                const double a = rank2(row[u][j], vi[u], W[s], wi[u], V[s]);
                                row[u][j] = a;
                                dot[u] += a * Vn[s];
                                if (j == b + 1) cn[u] = a;
                            }
                        }
                    }
                }
#endif
                if constexpr (true) {
                    // deferred: the lane partials of every row go to shared memory and are summed after the loop,
                    // all rows at once (one short transposed reduction instead of a 5-level butterfly per row)
                    const int rr = (l0 - li_first - warp) / kT2Warps;
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (ok[u]) {
                            wpart[(rr + u) * 33 + lane] = dot[u];
                            if (((b + 1) & 31) == lane) wcn[rr + u] = cn[u];
                        }
                } else {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int u = 0; u < U; ++u) dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int li = l0 + u * kT2Warps;
                        const double c = __shfl_sync(0xffffffffu, cn[u], (b + 1) & 31);
                        if (li < nloc) push((k + 1) & 1, q + kTcC * li, taun * dot[u], c);
                    }
                }
            }
            if constexpr (true) {
                __syncwarp();
                const int nrows = nloc > li_first + warp ? (nloc - li_first - warp + kT2Warps - 1) / kT2Warps : 0;
                if (lane < nrows) {
                    const double* pr = wpart + lane * 33;
                    double t8[8];
#pragma unroll
                    for (int a8 = 0; a8 < 8; ++a8) t8[a8] = (pr[a8] + pr[a8 + 8]) + (pr[a8 + 16] + pr[a8 + 24]);
                    const double dsum = tree_sum<8>(t8);
                    const int i = q + kTcC * (li_first + warp + lane * kT2Warps);
                    const double2 val = make_double2(taun * dsum, wcn[lane]);
#pragma unroll
                    for (int r = 0; r < kTcC; ++r) cluster.map_shared_rank(pc, r)[((k + 1) & 1) * n + i] = val;
                }
                __syncwarp();
            }
        }
        TRC_PHASE(k, 10);
        cluster_barrier();
        TRC_PHASE(k, 11);
        if (!more) {
            if (writer && lane == 0) ed.dvec[n - 1] = pc[((k + 1) & 1) * n + (n - 1)].y;
            break;
        }
#pragma unroll
        for (int s = 0; s < NT; ++s) V[s] = Vn[s];
        tau = taun;
    }
    cluster.sync();  // no CTA leaves while others may still write into its shared memory
}

// ------------------------------------------------------------------------------------- tridiagonal eig
// Spread over the whole GPU: grid (eigenvalue chunk, factor) for both the bisection and the vectors.

// Sturm count (eigenvalues of T strictly below x) with the division-free three-term recurrence of the leading
// principal minors p_i = (d_i - x) p_{i-1} - e_{i-1}^2 p_{i-2}; the count is the number of sign changes, i.e. of
// negative pivots q_i = p_i / p_{i-1} of the LDL^T recurrence LAPACK dstebz uses.  d, e2 are pre-scaled to
// ||T|| ~ 1 and negligible e are zero (dstebz's relative splitting test).  The fast loop has a single FMA on its
// dependence chain: e^2 p_{i-2} is formed a step ahead, the sign bookkeeping runs on the integer pipe, and every 4
// steps both minors are renormalised by the power of two that brings p_{i-1} (known a step early) to [1, 2).
// An exactly zero minor (x on an eigenvalue of a leading block) is only flagged in the fast loop; the rare flagged
// count is redone with dstebz's guard (a zero pivot becomes -pivmin: here p_i = -2^-200 p_{i-1}).
__device__ __forceinline__ double pow2_inverse_of(double v) {  // 2^-floor(log2|v|), clamped to the normal range
    const int eb = (__double2hiint(v) >> 20) & 0x7ff;
    return __hiloint2double((2046 - max(1, min(eb, 2045))) << 20, 0);
}

template <bool kGuard>
__device__ __forceinline__ void sturm_step(double dx, double e2, double& p0, double& p1, int& cnt, int& zero) {
    double pn = fma(dx, p1, -e2 * p0);
    if (kGuard) {
        if (pn == 0.0) pn = -0x1p-200 * p1;
    } else {
        zero |= (__double2hiint(pn) << 1) == 0;  // +-0 (or a denormal: harmless, just takes the guarded path)
    }
    cnt += (int)((unsigned)(__double2hiint(pn) ^ __double2hiint(p1)) >> 31);
    p0 = p1;
    p1 = pn;
}

template <bool kGuard>
__device__ __forceinline__ int sturm_count_impl(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                                double x, int& zero) {
    double p0 = 1.0, p1 = d[0] - x;
    if (p1 == 0.0) p1 = -0x1p-200;
    int cnt = p1 < 0.0;
    int i = 1;
    for (; i + 3 < n; i += 4) {
        const double d0 = d[i], d1 = d[i + 1], d2 = d[i + 2], d3 = d[i + 3];
        const double f0 = e2[i - 1], f1 = e2[i], f2 = e2[i + 1], f3 = e2[i + 2];
        sturm_step<kGuard>(d0 - x, f0, p0, p1, cnt, zero);
        sturm_step<kGuard>(d1 - x, f1, p0, p1, cnt, zero);
        sturm_step<kGuard>(d2 - x, f2, p0, p1, cnt, zero);
        const double f = pow2_inverse_of(p1);  // p1 here is p0 after the next step
        sturm_step<kGuard>(d3 - x, f3, p0, p1, cnt, zero);
        p0 *= f;
        p1 *= f;
    }
    for (; i < n; ++i) sturm_step<kGuard>(d[i] - x, e2[i - 1], p0, p1, cnt, zero);
    return cnt;
}

__device__ __forceinline__ int sturm_count_p(const double* __restrict__ d, const double* __restrict__ e2, int n,
                                             double x) {
    int zero = 0;
    const int c = sturm_count_impl<false>(d, e2, n, x, zero);
    if (!zero) return c;
    return sturm_count_impl<true>(d, e2, n, x, zero);
}

#ifndef RKFAC_BIS_G
#define RKFAC_BIS_G 4
#endif
constexpr int kBisG = RKFAC_BIS_G;  // threads per eigenvalue: (kBisG+1)-section per iteration
constexpr int kBisE = 32;   // eigenvalues per CTA
constexpr int kBisThreads = kBisG * kBisE;

// Gershgorin interval and norm of T, computed by the first W lanes of warp 0 (n <= 512).
template <int W = 32>
__device__ void tri_bounds(const double* d, const double* e, int n, double* out /* lo, hi, tnorm */) {
    constexpr unsigned mask = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
    const int lane = threadIdx.x & 31;
    double lo = DBL_MAX, hi = -DBL_MAX, tn = 0.0;
    for (int i = lane; i < n; i += W) {
        const double off = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i < n - 1 ? fabs(e[i]) : 0.0);
        lo = fmin(lo, d[i] - off);
        hi = fmax(hi, d[i] + off);
        tn = fmax(tn, fabs(d[i]) + off);
    }
    for (int o = W / 2; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(mask, lo, o));
        hi = fmax(hi, __shfl_xor_sync(mask, hi, o));
        tn = fmax(tn, __shfl_xor_sync(mask, tn, o));
    }
    if (lane == 0) { out[0] = lo; out[1] = hi; out[2] = fmax(tn, DBL_MIN); }
}

__global__ void __launch_bounds__(kBisThreads) bisect_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.y];
    const int n = ed.n, r = ed.r;
    const int kbase = blockIdx.x * kBisE;
    if (kbase >= r) return;
    __shared__ double d[kMaxN], e2[kMaxN], ev[kMaxN], bnd[3];
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += blockDim.x) {
        d[i] = ed.dvec[i];
        ev[i] = (i < n - 1) ? ed.evec[i] : 0.0;
    }
    __syncthreads();
    if (tid < 32) tri_bounds(d, ev, n, bnd);
    __syncthreads();
    int ex;
    frexp(bnd[2], &ex);
    const double sc = ldexp(1.0, -ex);  // exact: ||T|| sc in [0.5, 1)
    const double lo0 = bnd[0], hi0 = bnd[1], tnorm = bnd[2];
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
        const double di = d[i] * sc;
        double t = 0.0;
        if (i < n - 1) {
            const double ei = ev[i] * sc, dn = ed.dvec[i + 1] * sc;
            t = ei * ei;
            if (t <= DBL_EPSILON * DBL_EPSILON * fabs(di * dn) + DBL_MIN) t = 0.0;  // dstebz split test
        }
        d[i] = di;
        e2[i] = t;
    }
    __syncthreads();

    const int grp = tid / kBisG, u = tid % kBisG;
    const int k = kbase + grp;  // k-th largest eigenvalue
    if (k >= r) return;         // whole groups leave together
    const unsigned gmask = ((1u << kBisG) - 1u) << ((tid & 31) & ~(kBisG - 1));
    const int idx = n - 1 - k;
    const double pad = 2.0 * DBL_EPSILON * fmax(fabs(lo0), fabs(hi0)) * sc + 4.0 * DBL_MIN;
    double lo = lo0 * sc - pad, hi = hi0 * sc + pad;
    const double abstol = 4.0 * DBL_EPSILON * tnorm * sc;
    for (int it = 0; it < 100; ++it) {
        if (hi - lo <= 2.0 * DBL_EPSILON * fmax(fabs(lo), fabs(hi)) + abstol) break;
        const double h = (hi - lo) * (1.0 / (kBisG + 1));
        const double x0 = lo + h, xl = lo + h * kBisG;
        if (!(x0 > lo) || !(xl < hi)) {  // at the resolution of doubles: one plain bisection step
            const double mid = 0.5 * (lo + hi);
            if (mid == lo || mid == hi) break;
            const bool above = sturm_count_p(d, e2, n, mid) > idx;  // same on every lane of the group
            if (above) hi = mid; else lo = mid;
            continue;
        }
        const double x = lo + h * (u + 1);
        const bool above = sturm_count_p(d, e2, n, x) > idx;
        const unsigned b = __ballot_sync(gmask, above) & gmask;
        const int first = b ? (__ffs(b) - 1) - ((tid & 31) & ~(kBisG - 1)) : kBisG;  // first point above
        const double nhi = first < kBisG ? lo + h * (first + 1) : hi;
        const double nlo = first > 0 ? lo + h * first : lo;
        lo = nlo;
        hi = nhi;
    }
    if (u == 0) ed.evals[k] = 0.5 * (lo + hi) / sc;
}

// Inverse iteration from a pseudo-random start (LU with partial pivoting, 3 solves): used for members of
// clusters of (numerically) equal eigenvalues, whose vectors must span the cluster before the MGS pass.
__device__ void inverse_iteration(const double* d, const double* e, int n, double lmb, double tnorm, int k,
                                  const EigDesc& ed) {
    const long long S = ed.r;
    double* U1 = ed.scr;
    double* U2 = ed.scr + n * S;
    double* U3 = ed.scr + 2 * n * S;
    double* ML = ed.scr + 3 * n * S;
    double* Z = ed.z;
    unsigned char* PV = ed.piv;
    const double eps_piv = DBL_EPSILON * tnorm;
    double a = d[0] - lmb;
    double b = (n > 1) ? e[0] : 0.0;
    for (int i = 0; i < n - 1; ++i) {
        const double c = e[i];
        const double anext = d[i + 1] - lmb;
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
    for (int i = 0; i < n; ++i) {
        const uint64_t h = splitmix64(0x5EEDULL ^ ((uint64_t)k << 32) ^ (uint64_t)i);
        Z[i * S + k] = (double)(h >> 11) * 0x1.0p-53 - 0.5;
    }
    for (int iter = 0; iter < 3; ++iter) {
        for (int i = 0; i < n - 1; ++i) {
            const double zi = Z[i * S + k], zi1 = Z[(i + 1) * S + k];
            const double mult = ML[i * S + k];
            if (PV[i * S + k]) { Z[i * S + k] = zi1; Z[(i + 1) * S + k] = zi - mult * zi1; }
            else { Z[(i + 1) * S + k] = zi1 - mult * zi; }
        }
        double z2 = 0.0, z1 = 0.0, nrm = 0.0;
        for (int i = n - 1; i >= 0; --i) {
            double s = Z[i * S + k];
            if (i + 1 < n) s -= U2[i * S + k] * z1;
            if (i + 2 < n) s -= U3[i * S + k] * z2;
            const double zi = s / U1[i * S + k];
            Z[i * S + k] = zi;
            z2 = z1; z1 = zi;
            nrm = fmax(nrm, fabs(zi));
        }
        const double inv = (nrm > 0.0) ? 1.0 / nrm : 1.0;
        double s2 = 0.0;
        for (int i = 0; i < n; ++i) { const double z = Z[i * S + k] * inv; Z[i * S + k] = z; s2 += z * z; }
        const double inv2 = 1.0 / sqrt(s2);
        for (int i = 0; i < n; ++i) Z[i * S + k] *= inv2;
    }
}

// 1/x from the MUFU approximation and two Newton steps (full double precision; x is a normal number here).
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double t = fma(-x, r, 1.0);
    r = fma(r, t, r);
    t = fma(-x, r, 1.0);
    return fma(r, t, r);
}

// Eigenvectors of isolated eigenvalues from the twisted factorisation T - lam I = N_t Delta_t N_t^T (the stationary
// L+ D+ L+^T and progressive U- D- U-^T recurrences, twist t = argmin |gamma_t|, gamma_t = D+_t + D-_t - (d_t - lam)),
// then z_t = 1, z_i = -L+_i z_{i+1} (i < t), z_{i+1} = -U-_i z_i (i >= t): one solve, no start vector.  Cluster
// members (gap <= 1e-10 ||T||, the MGS threshold below) take the inverse-iteration path instead.
// One thread per eigenpair, 16 per CTA; the recurrences live in shared memory ([i][thread], conflict-free):
// L+ (later overwritten by z_i, i < t) and D+ (overwritten by U- in the backward sweep, then by z_{i+1}, i >= t).
constexpr int kVecThreads = 16;
size_t eigvec_smem_bytes(int nmax) { return (size_t)2 * nmax * kVecThreads * sizeof(double); }

__global__ void __launch_bounds__(kVecThreads) eigvec_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.y];
    const int n = ed.n, r = ed.r;
    const int tid = threadIdx.x;
    const int k = blockIdx.x * kVecThreads + tid;
    __shared__ double d[kMaxN], e[kMaxN], bnd[3];
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* Ls = reinterpret_cast<double*>(smem_raw);  // [n][kVecThreads]
    double* Ws = Ls + (size_t)n * kVecThreads;
    if (blockIdx.x * kVecThreads >= r) return;
    for (int i = tid; i < n; i += kVecThreads) {
        d[i] = ed.dvec[i];
        e[i] = (i < n - 1) ? ed.evec[i] : 0.0;
    }
    __syncwarp(0xffffu);
    tri_bounds<kVecThreads>(d, e, n, bnd);
    __syncwarp(0xffffu);
    const double tnorm = bnd[2];
    if (k >= r) return;
    const double lmb = ed.evals[k];
    const double clus = 1e-10 * tnorm;
    const bool clustered = (k > 0 && fabs(ed.evals[k - 1] - lmb) <= clus) ||
                           (k + 1 < r && fabs(ed.evals[k + 1] - lmb) <= clus);
    if (clustered) {
        inverse_iteration(d, e, n, lmb, tnorm, k, ed);
        return;
    }
    const double eps_piv = DBL_EPSILON * tnorm;
#define L_(i) Ls[(i) * kVecThreads + tid]
#define W_(i) Ws[(i) * kVecThreads + tid]
    // stationary: D+_{i+1} = (d_{i+1} - lam) - e_i^2 / D+_i
    double dp = d[0] - lmb;
    if (fabs(dp) < DBL_MIN) dp = eps_piv;
    int i = 0;
    for (; i + 4 < n; i += 4) {
        double ee[4], dd[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { ee[u] = e[i + u]; dd[u] = d[i + 1 + u] - lmb; }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            W_(i + u) = dp;
            const double l = ee[u] * rcp_nr(dp);
            L_(i + u) = l;
            dp = dd[u] - l * ee[u];
            if (fabs(dp) < DBL_MIN) dp = eps_piv;
        }
    }
    for (; i < n - 1; ++i) {
        W_(i) = dp;
        const double l = e[i] * rcp_nr(dp);
        L_(i) = l;
        dp = (d[i + 1] - lmb) - l * e[i];
        if (fabs(dp) < DBL_MIN) dp = eps_piv;
    }
    W_(n - 1) = dp;
    // progressive: D-_i = (d_i - lam) - e_i^2 / D-_{i+1}; gamma_i = D+_i + D-_i - (d_i - lam)
    double dm = d[n - 1] - lmb;
    if (fabs(dm) < DBL_MIN) dm = eps_piv;
    int t = n - 1;
    double best = fabs(dp + dm - (d[n - 1] - lmb));
    i = n - 2;
    for (; i >= 3; i -= 4) {
        double ee[4], dd[4], pp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) { ee[u] = e[i - u]; dd[u] = d[i - u] - lmb; pp[u] = W_(i - u); }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double um = ee[u] * rcp_nr(dm);
            W_(i - u) = um;
            dm = dd[u] - um * ee[u];
            if (fabs(dm) < DBL_MIN) dm = eps_piv;
            const double g = fabs(pp[u] + dm - dd[u]);
            if (g < best) { best = g; t = i - u; }
        }
    }
    for (; i >= 0; --i) {
        const double dd = d[i] - lmb, pp = W_(i);
        const double um = e[i] * rcp_nr(dm);
        W_(i) = um;
        dm = dd - um * e[i];
        if (fabs(dm) < DBL_MIN) dm = eps_piv;
        const double g = fabs(pp + dm - dd);
        if (g < best) { best = g; t = i; }
    }
    // z: z_t = 1; z_i (i < t) into L_(i), z_{i+1} (i >= t) into W_(i)
    double s2 = 1.0, z = 1.0;
    for (i = t - 1; i >= 0; --i) {
        z = -L_(i) * z;
        L_(i) = z;
        s2 += z * z;
    }
    z = 1.0;
    for (i = t; i < n - 1; ++i) {
        z = -W_(i) * z;
        W_(i) = z;
        s2 += z * z;
    }
    const double inv = 1.0 / sqrt(s2);
    const long long S = r;
    for (i = 0; i < n; ++i) {
        const double zi = i < t ? L_(i) : (i == t ? 1.0 : W_(i - 1));
        ed.z[i * S + k] = zi * inv;
    }
#undef L_
#undef W_
}

// Re-orthogonalise clusters of (numerically) equal eigenvalues, one CTA per factor.  Clusters are rare in general
// but large right after a zero-init EA (rank(X) < w: ~w - rank eigenvalues at 0), so every vector of a
// cluster is orthogonalised against all earlier ones at once -- classical Gram-Schmidt applied twice (CGS2): thread
// per earlier vector for the coefficients, thread per component for the update -- O(c) block steps instead of the
// O(c^2) dependent warp dot products of MGS.  The cluster is staged in shared memory when it fits (n*c <= kRoElems).
constexpr int kRoThreads = 256;
constexpr int kRoElems = 24576;  // 192 KB of FP64

__global__ void __launch_bounds__(kRoThreads) reorth_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.x];
    const int n = ed.n, r = ed.r;
    __shared__ double d[kMaxN], e[kMaxN], lam[kMaxN], coef[kMaxN], bnd[3], red[33];
    __shared__ int any_s;
    extern __shared__ double zc[];  // staged cluster, [t][c] (row t = component)
    const int tid = threadIdx.x;
    for (int i = tid; i < n; i += kRoThreads) {
        d[i] = ed.dvec[i];
        e[i] = (i < n - 1) ? ed.evec[i] : 0.0;
    }
    for (int i = tid; i < r; i += kRoThreads) lam[i] = ed.evals[i];
    if (tid == 0) any_s = 0;
    __syncthreads();
    if (tid < 32) tri_bounds(d, e, n, bnd);
    __syncthreads();
    const double clus = 1e-10 * bnd[2];
    for (int i = tid + 1; i < r; i += kRoThreads)
        if (fabs(lam[i - 1] - lam[i]) <= clus) any_s = 1;
    __syncthreads();
    if (!any_s) return;
    const long long S = r;
    double* Z = ed.z;
    int k = 0;
    while (k < r) {
        int k1 = k + 1;
        while (k1 < r && fabs(lam[k1 - 1] - lam[k1]) <= clus) ++k1;
        const int c = k1 - k;
        if (c > 1) {
            const bool staged = (long long)n * c <= kRoElems;
            // element (t, i) of the cluster (i relative to k)
            auto at = [&](int t, int i) -> double& { return staged ? zc[t * c + i] : Z[t * S + k + i]; };
            if (staged)
                for (int x = tid; x < n * c; x += kRoThreads) zc[x] = Z[(x / c) * S + k + (x % c)];
            __syncthreads();
            for (int j = 0; j < c; ++j) {
                for (int pass = 0; pass < 2 && j > 0; ++pass) {
                    for (int i = tid; i < j; i += kRoThreads) {
                        double s0 = 0.0, s1 = 0.0;
                        int t = 0;
                        for (; t + 1 < n; t += 2) { s0 += at(t, i) * at(t, j); s1 += at(t + 1, i) * at(t + 1, j); }
                        if (t < n) s0 += at(t, i) * at(t, j);
                        coef[i] = s0 + s1;
                    }
                    __syncthreads();
                    for (int t = tid; t < n; t += kRoThreads) {
                        double acc = at(t, j);
                        for (int i = 0; i < j; ++i) acc -= coef[i] * at(t, i);
                        at(t, j) = acc;
                    }
                    __syncthreads();
                }
                double nn = 0.0;
                for (int t = tid; t < n; t += kRoThreads) nn += at(t, j) * at(t, j);
                nn = block_sum_d(nn, red);
                const double inv = nn > 0.0 ? 1.0 / sqrt(nn) : 0.0;
                for (int t = tid; t < n; t += kRoThreads) at(t, j) *= inv;
                __syncthreads();
            }
            if (staged)
                for (int x = tid; x < n * c; x += kRoThreads) Z[(x / c) * S + k + (x % c)] = zc[x];
            __syncthreads();
        }
        k = k1;
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

// Blocked back transformation with the compact WY form (LAPACK dlarft/dlarfb, forward columnwise): the 32
// reflectors k0..k0+31 act as I - V T V^T, applied to the CTA's 32 eigenvector columns from the last block to
// the first, so 8 blocks of three small products (W = V^T Z, W = T W, Z -= V W) replace 228 dependent reflector
// steps.  T is formed in the CTA from G = V^T V (upper triangle): T_ii = tau_i, T(0:i, i) = -tau_i T G(0:i, i).
#ifdef RKFAC_TRC_TIMING
__device__ long long g_bx[8][8];
#define BX_PHASE(b, slot)                                                                       \
    do {                                                                                        \
        const long long t_ = clock64();                                                         \
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && (b) < 8) g_bx[b][slot] = t_; \
        __syncwarp();                                                                           \
    } while (0)
#else
#define BX_PHASE(b, slot)
#endif
constexpr int kWyB = 32;          // reflectors per block
constexpr int kWyC = 64;          // eigenvector columns per CTA (2 per lane)
constexpr int kWyThreads = 512;
constexpr int kWyWarps = kWyThreads / 32;
constexpr int kWyMaxN = 256;
constexpr int kWyP = kWyB + 2;    // padded pitch of V and G (doubles; even: 16-byte pairs)
constexpr int kWyWP = kWyC + 1;   // padded pitch of W

size_t backxform_wy_smem_bytes(int n) {
    return ((size_t)n * kWyC + (size_t)n * kWyP + 2 * kWyB * kWyP + kWyB * kWyWP + kWyB) * sizeof(double);
}

__global__ void __launch_bounds__(kWyThreads) backxform_wy_kernel(const EigDesc* __restrict__ descs) {
    const EigDesc& ed = descs[blockIdx.y];
    const int n = ed.n, r = ed.r;
    const int c0 = blockIdx.x * kWyC;
    if (c0 >= r) return;
    const int nc = min(kWyC, r - c0);
    extern __shared__ __align__(16) double wsm[];
    double* Zs = wsm;                          // [n][64]
    double* V = Zs + (size_t)n * kWyC;         // [M][kWyP]
    double* G = V + (size_t)n * kWyP;          // [32][kWyP]
    double* T = G + kWyB * kWyP;               // [32][kWyP]
    double* W = T + kWyB * kWyP;               // [32][kWyWP]
    double* taus = W + kWyB * kWyWP;           // [32]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int e = tid; e < n * kWyC; e += kWyThreads) {
        const int i = e / kWyC, c = e % kWyC;
        Zs[e] = (c < nc) ? ed.z[(long long)i * r + c0 + c] : 0.0;
    }
    const int nref = n - 2;  // reflectors 0 .. n-3
    const int nblk = nref > 0 ? (nref + kWyB - 1) / kWyB : 0;
    for (int b = nblk - 1; b >= 0; --b) {
        const int k0 = b * kWyB, nb = min(kWyB, nref - k0);
        const int r0 = k0 + 1, M = n - r0;  // rows r0 .. n-1
        __syncthreads();
        BX_PHASE(b, 0);
        // V[rel][j] = v_{k0+j}[rel - j] (rel >= j), unit at rel == j, zero above; 4 independent loads per thread
        for (int e0 = tid; e0 < M * kWyB; e0 += 4 * kWyThreads) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * kWyThreads, rel = e / kWyB, j = e % kWyB;
                v[u] = (e < M * kWyB && j < nb && rel >= j) ? ed.refl[(long long)(k0 + j) * n + (rel - j)] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * kWyThreads;
                if (e < M * kWyB) V[(e / kWyB) * kWyP + e % kWyB] = v[u];
            }
        }
        if (tid < kWyB) taus[tid] = (tid < nb) ? ed.tau[k0 + tid] : 0.0;
        __syncthreads();
        BX_PHASE(b, 1);
        // G = V^T V (upper triangle) and W = V^T Z: warp -> rows jj, jj+1 of G/W (a 16-byte broadcast pair of V),
        // lane -> column i of G and columns lane, lane + 32 of W; six independent chains per thread
        {
            const int jj = 2 * warp;  // kWyWarps * 2 == kWyB
            const int i = lane;
            double g0 = 0.0, g1 = 0.0, w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0;
            for (int rel = jj; rel < M; ++rel) {
                const double2 vp = *reinterpret_cast<const double2*>(&V[rel * kWyP + jj]);
                const double vi = V[rel * kWyP + i];
                const double z0 = Zs[(r0 + rel) * kWyC + lane], z1 = Zs[(r0 + rel) * kWyC + lane + 32];
                g0 += vp.x * vi;
                g1 += vp.y * vi;
                w00 += vp.x * z0;
                w01 += vp.x * z1;
                w10 += vp.y * z0;
                w11 += vp.y * z1;
            }
            G[jj * kWyP + i] = (jj < i) ? g0 : 0.0;
            G[(jj + 1) * kWyP + i] = (jj + 1 < i) ? g1 : 0.0;
            W[jj * kWyWP + lane] = w00;
            W[jj * kWyWP + lane + 32] = w01;
            W[(jj + 1) * kWyWP + lane] = w10;
            W[(jj + 1) * kWyWP + lane + 32] = w11;
        }
        __syncthreads();
        BX_PHASE(b, 2);
        // W <- T W with T = (diag(1/tau) + striu(V^T V))^{-1} (compact WY, forward columnwise), as one triangular
        // solve (diag(1/tau) + striu(G)) X = W: a thread per eigenvector column back-substitutes, x_i =
        // tau_i (w_i - sum_{l>i} G(i, l) x_l), right-looking (after x_i, every w_l, l < i, loses G(l, i) x_i), so
        // neither T nor the T W product is formed (tau_i = 0 gives x_i = 0: the identity reflector)
        BX_PHASE(b, 3);
        if (tid < kWyC) {
            const int c = tid;
            double x[kWyB];
#pragma unroll
            for (int i = 0; i < kWyB; ++i) x[i] = W[i * kWyWP + c];
#pragma unroll
            for (int i = kWyB - 1; i >= 0; --i) {
                x[i] *= taus[i];
#pragma unroll
                for (int l = 0; l < i; ++l) x[l] -= G[l * kWyP + i] * x[i];
            }
#pragma unroll
            for (int i = 0; i < kWyB; ++i) W[i * kWyWP + c] = x[i];
        }
        __syncthreads();
        BX_PHASE(b, 4);
        // Z -= V W: a warp takes 4 rows at a time (the W loads are shared), lanes over 2 columns
        for (int rel0 = 4 * warp; rel0 < M; rel0 += 4 * kWyWarps) {
            double acc[4][2] = {};
#pragma unroll 4
            for (int j = 0; j < kWyB; j += 2) {
                const double wa0 = W[j * kWyWP + lane], wb0 = W[j * kWyWP + lane + 32];
                const double wa1 = W[(j + 1) * kWyWP + lane], wb1 = W[(j + 1) * kWyWP + lane + 32];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int rel = min(rel0 + u, M - 1);
                    const double2 vp = *reinterpret_cast<const double2*>(&V[rel * kWyP + j]);
                    acc[u][0] += vp.x * wa0 + vp.y * wa1;
                    acc[u][1] += vp.x * wb0 + vp.y * wb1;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (rel0 + u < M) {
                    Zs[(r0 + rel0 + u) * kWyC + lane] -= acc[u][0];
                    Zs[(r0 + rel0 + u) * kWyC + lane + 32] -= acc[u][1];
                }
        }
        __syncthreads();
        BX_PHASE(b, 5);
    }
    __syncthreads();
    for (long long e = tid; e < (long long)n * kWyC; e += kWyThreads) {
        const int i = (int)(e / kWyC), c = (int)(e % kWyC);
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
    static const bool old_tridiag = [] {
        const char* e = getenv("RKFAC_TRIDIAG_TWO_BARRIER");
        return e && e[0] == '1';
    }();
    const size_t b1 = tridiag1b_smem_bytes(nmax);
    auto k1 = nmax <= 256 ? tridiag1b_kernel<8, RKFAC_T1B_U> : tridiag1b_kernel<10, RKFAC_T1B_U>;
    const size_t cbytes = tridiag_cluster_smem_bytes(nmax);
    if (!old_tridiag && nmax <= 320 && b1 <= max_dynamic_smem((const void*)k1)) {
        RKFAC_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b1));
        k1<<<nfactors * kTcC, kT2Threads, b1, s>>>(d_descs);
    } else if (nmax <= kTcMaxN && cbytes <= max_dynamic_smem((const void*)tridiag_cluster_kernel)) {
        RKFAC_CUDA(cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)cbytes));
        tridiag_cluster_kernel<<<nfactors * kTcC, kTcThreads, cbytes, s>>>(d_descs);
    } else {
        const size_t bytes = tridiag_smem_bytes(nmax);
        const bool use_smem = bytes <= max_dynamic_smem((const void*)tridiag_kernel<true>);
        auto k = use_smem ? tridiag_kernel<true> : tridiag_kernel<false>;
        const size_t dyn = use_smem ? bytes : 0;
        RKFAC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        k<<<nfactors, 1024, dyn, s>>>(d_descs);
    }
    count_launch();
    RKFAC_CHECK_LAUNCH();
    const unsigned rchunks = (unsigned)std::max<int64_t>(1, ceil_div(std::max(rmax, 1), kBisE));
    bisect_kernel<<<dim3(rchunks, (unsigned)nfactors), kBisThreads, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
    const size_t evb = eigvec_smem_bytes(nmax);
    RKFAC_CUDA(cudaFuncSetAttribute(eigvec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)evb));
    eigvec_kernel<<<dim3((unsigned)ceil_div(std::max(rmax, 1), kVecThreads), (unsigned)nfactors), kVecThreads, evb,
                    s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
    RKFAC_CUDA(cudaFuncSetAttribute(reorth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kRoElems * sizeof(double))));
    reorth_kernel<<<nfactors, kRoThreads, kRoElems * sizeof(double), s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
    dim3 grid((unsigned)ceil_div(std::max(rmax, 1), kBxCols), (unsigned)nfactors);
    const size_t wyb = backxform_wy_smem_bytes(nmax);
    if (nmax <= kWyMaxN && wyb <= max_dynamic_smem((const void*)backxform_wy_kernel)) {
        RKFAC_CUDA(cudaFuncSetAttribute(backxform_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wyb));
        dim3 gwy((unsigned)ceil_div(std::max(rmax, 1), kWyC), (unsigned)nfactors);
        backxform_wy_kernel<<<gwy, kWyThreads, wyb, s>>>(d_descs);
    } else {
        const size_t bx = (size_t)nmax * kBxCols * 8;
        RKFAC_CUDA(cudaFuncSetAttribute(backxform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bx));
        backxform_kernel<<<grid, 256, bx, s>>>(d_descs);
    }
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
