// cholqr.cu -- CholeskyQR building blocks for the orthonormalisation of the sketch (replaces qr_thin,
// qr.hpp:23-87, inside randomized_range, rnla.hpp:47-56).
//
//   G = Y^T Y (grouped GEMM)  ->  cholinv_kernel: G = L L^T, Linv = L^{-1}  ->  Q = Y L^{-T} (grouped GEMM)
//   -> complete_kernel (only when a column was rank deficient)
//
// The reference's Householder QR forces diag(R) >= 0, so its thin Q is unique for full-rank input and
// CholeskyQR (R = L^T has a positive diagonal) yields the same Q up to rounding.  Only span(Q) matters
// downstream (C = Q^T X Q and U = Q P are basis independent), so rank-deficient columns -- which the
// reference skips (qr.hpp:35-45, H = I) -- are replaced here by any unit vector orthogonal to the others.
//
// cholinv_kernel: one CTA (512 threads) per factor.  The lower triangle lives in shared memory in a
// "padded packed" layout: row i starts at a 16-byte aligned offset and is zero-padded to a multiple of 4 entries,
// so every inner loop is a 4x4 register tile fed by LDS.128 and the zero padding doubles as the upper-triangle
// zeros of L^{-1}.  w <= 230 fits in FP64 (w <= 330 in FP32); larger w uses a global scratch.  Latency matters
// more than the w^3/3 flops, so:
//   Cholesky   right-looking over 32-wide panels: the 32x32 diagonal block is factored by one warp in registers
//              (pivot chain on shuffles, the rest of each column software-pipelined through shared memory), the
//              panel below by a row-parallel TRSM, the trailing update by 4x4 register tiles;
//   inverse    all 32x32 diagonal blocks inverted concurrently (one warp each), then recursive doubling over block
//              segments, B <- -C^{-1} B A^{-1}, as passes of register tiles (log2(w/32) levels, 4 barriers each).
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kNB = 32;

// Optional per-phase clock64 stamps (tools/chol_bench.cu builds with -DRKFAC_PHASE_TIMING).
#ifdef RKFAC_PHASE_TIMING
__device__ long long g_chol_phase[64 * 64];
#define CHOL_PHASE(k)                                                                     \
    do {                                                                                  \
        const long long t_ = clock64();                                                   \
        if (threadIdx.x == 0 && blockIdx.x < 64) g_chol_phase[blockIdx.x * 64 + (k)] = t_; \
        __syncwarp(); /* reconverge warp 0: a split warp would run the shuffles emulated */ \
    } while (0)
#else
#define CHOL_PHASE(k)
#endif
constexpr int kMaxW = 512;
constexpr int kCholThreads = 512;  // 128-register budget: the unrolled 32-wide row arrays stay in registers

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__host__ __device__ __forceinline__ int rup4(int x) { return (x + 3) & ~3; }
__host__ __device__ __forceinline__ int rup8(int x) { return (x + 7) & ~7; }

// Offset of row i in the padded packed layout: sum_{t<i} rup4(t+1) plus 4 skew elements after every block of 4
// rows.  rup4(t+1) for t = 4a+b is 4a+4, so block a starts at 8a(a+1); without the skew the rows 4a (the first rows
// of the 4x4 register tiles that consecutive threads take) all start in the same two 16-byte bank groups (16-way
// conflicts on LDS.128); with it, 8 consecutive blocks start in 8 distinct groups.
__host__ __device__ __forceinline__ int prow(int i) {
    const int a = i >> 2, b = i & 3;
    return 8 * a * (a + 1) + b * (4 * a + 4) + 4 * a;
}

// bytes of the small per-factor state carved at the start of the dynamic smem (16-byte multiple)
__host__ __device__ __forceinline__ int cholinv_state_bytes(int n, int es) {
    return (es * (kNB * (kNB + 1) + kNB) + 4 * rup4(n) + rup4(n) + 15) & ~15;
}

// G(i, j) (the element itself: the Gram is not exactly symmetric, and for factors with a 1e-6 spectral range using
// the mirror element was measured to move the smallest eigenvalues by 3e-3) from split-K partials (column-major,
// so consecutive i are contiguous); the association ((s0 + s1) + (s2 + s3)) with s_r summing slices r, r+4, ... is
// the one of tc_gemm.cu's tc_reduce_kernel.
__device__ __forceinline__ float gram_from_parts(const CholDesc& cd, int i, int j) {
    const long long ww = (long long)cd.w * cd.w;
    const float* p = cd.part + (long long)j * cd.w + i;
    float s0 = p[0], s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int k = 1;
    for (; k + 3 < cd.nslices; k += 4) {
        s0 += p[k * ww]; s1 += p[(k + 1) * ww]; s2 += p[(k + 2) * ww]; s3 += p[(k + 3) * ww];
    }
    for (; k < cd.nslices; ++k) s0 += p[k * ww];
    return (s0 + s1) + (s2 + s3);
}

template <class T> struct Vec4T;
template <> struct Vec4T<float> { using type = float4; };
template <> struct Vec4T<double> { using type = double4; };

template <class T>
__device__ __forceinline__ void st4(T* p, T a, T b, T c, T d) {
    using V = typename Vec4T<T>::type;
    V x;
    x.x = a; x.y = b; x.z = c; x.w = d;
    *reinterpret_cast<V*>(p) = x;
}

template <class T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[4]) {
    using V = typename Vec4T<T>::type;
    const V x = *reinterpret_cast<const V*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}

// kSmem selects the storage of the triangle at compile time: a pointer chosen at run time between shared and
// global memory compiles to generic LD/ST (measured ~2.5x slower than LDS/STS on this kernel).
template <class T>
__device__ __forceinline__ T rsqrt_t(T x);
template <>
__device__ __forceinline__ float rsqrt_t<float>(float x) { return rsqrtf(x); }
template <>
__device__ __forceinline__ double rsqrt_t<double>(double x) { return rsqrt(x); }

// Lower-triangular tile enumeration of a trapezoid, row-major: row tiles I in [0, TR), column tiles J in
// [0, min(I + 1, CJ)).  Consecutive threads take consecutive J of the same row tile, so the A operand rows are
// broadcast and the read-modify-write of the output is contiguous within a warp.
__device__ __forceinline__ void trap_tile(int t, int CJ, int& I, int& J) {
    const int tri = CJ * (CJ + 1) / 2;
    if (t < tri) {
        int i = (int)((sqrtf(8.f * (float)t + 1.f) - 1.f) * 0.5f);
        while (i * (i + 1) / 2 > t) --i;
        while ((i + 1) * (i + 2) / 2 <= t) ++i;
        I = i;
        J = t - i * (i + 1) / 2;
    } else {
        const int u = t - tri;
        I = CJ + u / CJ;
        J = u - (I - CJ) * CJ;
    }
}

template <class TG, class T, bool kSmem>
__global__ void __launch_bounds__(kCholThreads) cholinv_kernel(const CholDesc* __restrict__ descs, double tol) {
    const CholDesc& cd = descs[blockIdx.x];
    const int n = cd.w;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // dynamic smem: [small per-factor state][padded packed triangle (kSmem only)]
    T* colbuf = reinterpret_cast<T*>(smem_raw);                                   // column broadcast (warp 0)
    T* dinv = colbuf + 2 * kNB;                                                    // reciprocal diagonal of L_bb
    float* diag0 = reinterpret_cast<float*>(smem_raw + sizeof(T) * (kNB * (kNB + 1) + kNB));  // diag of G
    unsigned char* defic = reinterpret_cast<unsigned char*>(diag0 + rup4(n));    // rank-deficiency flags
    __shared__ int any_defic;
    T* L;
    if constexpr (kSmem) L = reinterpret_cast<T*>(smem_raw + cholinv_state_bytes(n, sizeof(T)));
    else L = static_cast<T*>(cd.scratch);
    const T tolT = T(tol);

    CHOL_PHASE(0);
    // Lower triangle of G (the Gram matrix is symmetric; its upper half is not read).  Same element type and a
    // 16-byte aligned pitch: asynchronous 16-byte copies straight into the packed rows (all in flight at once),
    // then the few upper entries a copy brought into the zero padding are cleared.
    const TG* G = static_cast<const TG*>(cd.G);
    bool async_load = false;
    if constexpr (kSmem && sizeof(TG) == sizeof(T)) {
        async_load = !cd.part && ((cd.ldg * (long long)sizeof(T)) & 15) == 0 && (((uintptr_t)G) & 15) == 0 &&
                     cd.ldg >= rup4(n);
        if (async_load) {
            constexpr int E = 16 / sizeof(T);
            for (int i = warp; i < n; i += nwarp) {
                const int nch = rup4(i + 1) / E;
                for (int c = lane; c < nch; c += 32) {
                    const unsigned dst = (unsigned)__cvta_generic_to_shared(L + prow(i) + c * E);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst),
                                 "l"(G + (long long)i * cd.ldg + c * E));
                }
            }
            asm volatile("cp.async.wait_all;\n" ::);
            __syncthreads();
            for (int i = tid; i < n; i += nthr)
                for (int j = i + 1; j < rup4(i + 1); ++j) L[prow(i) + j] = T(0);
        }
    }
    if (!async_load) {
        for (int i = warp; i < n; i += nwarp) {
            T* row = L + prow(i);
            for (int j = lane; j < rup4(i + 1); j += 32)
                row[j] = (j <= i) ? (cd.part ? T(gram_from_parts(cd, i, j)) : T(G[(long long)i * cd.ldg + j])) : T(0);
        }
    }
    for (int i = tid; i < n; i += nthr) defic[i] = 0;
    if (tid == 0) any_defic = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nthr) diag0[i] = (float)L[prow(i) + i];
    __syncthreads();
    CHOL_PHASE(1);

    const int nblk = (n + kNB - 1) / kNB;

    // 32x32 diagonal block b, one warp, lane = row, right-looking: the pivot is read by shuffle, the scaled column
    // is broadcast through shared memory.  Deficient pivots (<= tol * G_kk) give L_kk = 1 and a zero column.
    auto factor_diag = [&](int b) {
        const int J0 = b * kNB, nb = min(kNB, n - J0);
        T a[kNB];
        const int rl = min(lane, nb - 1);
        const T* rowp = L + prow(J0 + rl) + J0;
#pragma unroll
        for (int c4 = 0; c4 < kNB; c4 += 4) {
            T v4[4] = {T(0), T(0), T(0), T(0)};
            if (c4 <= rl) ld4(rowp + c4, v4);  // row J0+rl holds rup4(J0+rl+1) >= J0+c4+4 entries
#pragma unroll
            for (int u = 0; u < 4; ++u) a[c4 + u] = (lane < nb && c4 + u <= lane) ? v4[u] : T(0);
        }
        // Lanes above the diagonal only touch their (never stored) upper part, so loads and FMAs need no per-lane
        // predicate (a predicated load would put its latency on the chain of every update).  Step k's pivot is
        // read by shuffle; the entry the next pivot depends on, L(k+1, k), is shuffled too and applied first,
        // while the rest of column k goes through shared memory and is applied one step later (FP32: software
        // pipelined, so the shared-memory round trip leaves the pivot chain).
        T tp[kNB];  // column k-1, entries j >= k+1 (pipelined remainder)
        auto step = [&](int k, int nbv, bool defer) {
            const T piv = __shfl_sync(0xffffffffu, a[k], k);
            const T g = T(diag0[J0 + k]);
            const bool def = !(piv > tolT * g) || g == T(0);
            const T inv = def ? T(0) : rsqrt_t(piv);
            const T lkk = def ? T(1) : piv * inv;
            a[k] = lane == k ? lkk : (lane > k ? a[k] * inv : a[k]);
            if (lane == 0) dinv[k] = inv;
            if (def && lane == 0) { defic[J0 + k] = 1; any_defic = 1; }
            if (k + 1 < nbv) {
                const T tn = __shfl_sync(0xffffffffu, a[k], k + 1);
                T* cb = colbuf + (k & 1) * kNB;  // double-buffered: one __syncwarp per step
                cb[lane] = a[k];
                __syncwarp();
                if (defer) {
                    T tc[kNB];
#pragma unroll
                    for (int q4 = (k + 2) & ~3; q4 < kNB; q4 += 4) {
                        T v4[4];
                        ld4(cb + q4, v4);
#pragma unroll
                        for (int u = 0; u < 4; ++u) tc[q4 + u] = v4[u];
                    }
                    if (k >= 1) {  // remainder of column k-1 (j >= k+1), loaded one step ago
#pragma unroll
                        for (int j = k + 1; j < kNB; ++j) a[j] -= a[k - 1] * tp[j];
                    }
                    a[k + 1] -= a[k] * tn;
#pragma unroll
                    for (int j = k + 2; j < kNB; ++j) tp[j] = tc[j];
                } else {
                    a[k + 1] -= a[k] * tn;
#pragma unroll
                    for (int q4 = (k + 2) & ~3; q4 < kNB; q4 += 4) {
                        T v4[4];
                        ld4(cb + q4, v4);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (q4 + u >= k + 2) a[q4 + u] -= a[k] * v4[u];
                    }
                }
            } else if (defer && k >= 1) {
#pragma unroll
                for (int j = k + 1; j < kNB; ++j) a[j] -= a[k - 1] * tp[j];
            }
        };
        constexpr bool kDefer = sizeof(T) == 4;  // FP64: the second column buffer would exceed the register budget
        if (nb == kNB) {
#pragma unroll
            for (int k = 0; k < kNB; ++k) step(k, kNB, kDefer);
        } else {
#pragma unroll
            for (int k = 0; k < kNB; ++k)
                if (k < nb) step(k, nb, false);
        }
        if (lane < nb) {
            T* wrow = L + prow(J0 + lane) + J0;
#pragma unroll
            for (int c = 0; c < kNB; ++c)
                if (c <= lane) wrow[c] = a[c];
        }
    };

    // Trailing update A(i, j) -= sum_c L(i, J0+c) L(j, J0+c) over the lower trapezoid with columns [c0, c1) and
    // rows [c0, n), 4x4 register tiles (LDS.128 along the panel), tiles spread over threads [t0, t0 + nt).
    auto update = [&](int J0, int nb, int c0, int c1, int t0, int nt) {
        if (c0 >= c1 || tid < t0 || tid >= t0 + nt) return;
        const int TR = (n - c0 + 3) / 4, CJ = (c1 - c0 + 3) / 4;
        const int ntiles = CJ * TR - CJ * (CJ - 1) / 2;
        for (int t = tid - t0; t < ntiles; t += nt) {
            int I, J;
            trap_tile(t, CJ, I, J);
            const T* ra[4];
            const T* rb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                ra[u] = L + prow(min(c0 + I * 4 + u, n - 1)) + J0;
                rb[u] = L + prow(min(c0 + J * 4 + u, n - 1)) + J0;
            }
            T acc[4][4] = {};
            if (nb == kNB) {  // full panel: branch-free K loop, all loads can be hoisted by the scheduler
#pragma unroll
                for (int c4 = 0; c4 < kNB; c4 += 4) {
                    T av[4][4], bv[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) { ld4(ra[u] + c4, av[u]); ld4(rb[u] + c4, bv[u]); }
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int v = 0; v < 4; ++v) acc[u][v] += av[u][c] * bv[v][c];
                }
            } else {
#pragma unroll
                for (int c4 = 0; c4 < kNB; c4 += 4) {
                    if (c4 < nb) {
                        T av[4][4], bv[4][4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) { ld4(ra[u] + c4, av[u]); ld4(rb[u] + c4, bv[u]); }
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (c4 + c < nb)
#pragma unroll
                                for (int u = 0; u < 4; ++u)
#pragma unroll
                                    for (int v = 0; v < 4; ++v) acc[u][v] += av[u][c] * bv[v][c];
                    }
                }
            }
            const int j0 = c0 + J * 4;
            const bool full = I > J && j0 + 3 < c1;  // strictly below the diagonal, whole column group in range
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int ii = c0 + I * 4 + u;
                if (ii >= n) continue;
                T* wr = L + prow(ii) + j0;
                if (full) {
                    T w4[4];
                    ld4(wr, w4);
                    st4(wr, w4[0] - acc[u][0], w4[1] - acc[u][1], w4[2] - acc[u][2], w4[3] - acc[u][3]);
                } else {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        if (j0 + v <= ii && j0 + v < c1) wr[v] -= acc[u][v];
                }
            }
        }
    };

    // ------------------------------------------------------------------ Cholesky, right-looking with look-ahead
    if (warp == 0) factor_diag(0);
    __syncthreads();
    CHOL_PHASE(2);
    for (int b = 0; b < nblk; ++b) {
        const int J0 = b * kNB, nb = min(kNB, n - J0);
        // panel TRSM: rows below the block, one thread per row, forward substitution with 4 partial sums
        const int rows = n - J0 - nb;
        for (int t = tid; t < rows; t += nthr) {
            const int i = J0 + nb + t;
            T* rp = L + prow(i) + J0;
            T x[kNB];
#pragma unroll
            for (int c4 = 0; c4 < kNB; c4 += 4) {
                T v4[4];
                ld4(rp + c4, v4);
#pragma unroll
                for (int u = 0; u < 4; ++u) x[c4 + u] = v4[u];
            }
#pragma unroll
            for (int c = 0; c < kNB; ++c) {
                if (c < nb) {
                    const T* lc = L + prow(J0 + c) + J0;
                    T s0 = x[c], s1 = T(0), s2 = T(0), s3 = T(0);
#pragma unroll
                    for (int q = 0; q < c; q += 4) {
                        T l4[4];
                        ld4(lc + q, l4);
                        s0 -= x[q] * l4[0];
                        if (q + 1 < c) s1 -= x[q + 1] * l4[1];
                        if (q + 2 < c) s2 -= x[q + 2] * l4[2];
                        if (q + 3 < c) s3 -= x[q + 3] * l4[3];
                    }
                    x[c] = ((s0 + s1) + (s2 + s3)) * dinv[c];
                }
            }
#pragma unroll
            for (int c = 0; c < kNB; ++c)
                if (c < nb) rp[c] = x[c];
        }
        __syncthreads();
        CHOL_PHASE(3 + 3 * b);
        if (b + 1 < nblk) {
            // trailing update of everything right of the panel (all warps), then the next diagonal block (warp 0;
            // overlapping it with the update was measured slower: the update's shared-memory traffic stalls the
            // factorisation's latency-bound chain)
            update(J0, nb, J0 + kNB, n, 0, nthr);
            __syncthreads();
            CHOL_PHASE(4 + 3 * b);
            if (warp == 0) factor_diag(b + 1);
            __syncthreads();
            CHOL_PHASE(5 + 3 * b);
        }
    }

    // ------------------------------------------------------------------ triangular inverse, in place
    // (a) all diagonal blocks concurrently: warp b inverts block b; lane j computes column j (broadcast loads).
    for (int b = warp; b < nblk; b += nwarp) {
        const int J0 = b * kNB, nb = min(kNB, n - J0);
        T x[kNB];
        const int j = lane;
#pragma unroll
        for (int i = 0; i < kNB; ++i) {
            if (i < nb) {
                const T* li = L + prow(J0 + i) + J0;
                const T di = defic[J0 + i] ? T(1) : T(1) / li[i];
                // x[k] = 0 for k < j, so the sums need no predicate (and the loads no per-lane condition)
                T s0 = T(0), s1 = T(0), s2 = T(0), s3 = T(0);
#pragma unroll
                for (int k = 0; k < i; k += 4) {
                    T l4[4];
                    ld4(li + k, l4);
                    s0 += l4[0] * x[k];
                    if (k + 1 < i) s1 += l4[1] * x[k + 1];
                    if (k + 2 < i) s2 += l4[2] * x[k + 2];
                    if (k + 3 < i) s3 += l4[3] * x[k + 3];
                }
                x[i] = (i < j) ? T(0) : (i == j ? di : -((s0 + s1) + (s2 + s3)) * di);
            } else {
                x[i] = T(0);
            }
        }
        __syncwarp();
        if (lane < nb) {
#pragma unroll
            for (int i = 0; i < kNB; ++i)
                if (i < nb && i >= lane) L[prow(J0 + i) + J0 + lane] = x[i];
        }
    }
    __syncthreads();
    CHOL_PHASE(51);
    // (b) recursive doubling over block segments: for [A 0; B C] with A^-1, C^-1 in place,
    //     B <- -C^-1 (B A^-1).  Both products run as passes of 4x4 tiles held in registers (all reads of a pass
    //     precede its writes); product 1 goes by increasing column (T_ij reads B_ik, k >= j), product 2 by
    //     decreasing row (R_ij reads T_kj, k <= i), so no pass overwrites what a later pass reads.
    for (int s = 1; s < nblk; s *= 2) {
        const int nseg = (nblk + 2 * s - 1) / (2 * s);
        // tiles per segment: rows of C x columns of A (in 4-tiles)
        int total = 0;
        for (int g = 0; g < nseg; ++g) {
            const int cs = (2 * g + 1) * s * kNB, ce = min((2 * g + 2) * s * kNB, n);
            if (cs < n) total += ((ce - cs + 3) / 4) * (s * kNB / 4);
        }
        for (int prod = 0; prod < 2; ++prod) {
            for (int base = 0; base < total; base += nthr) {
                const int t = base + tid;
                T acc[4][4] = {};
                int r0 = 0, c0 = 0;
                bool have = false;
                if (t < total) {
                    // locate the segment
                    int g = 0, rem = t, RT = 0, CT = s * kNB / 4, cs = 0, as = 0, ae = 0;
                    for (;; ++g) {
                        cs = (2 * g + 1) * s * kNB;
                        const int ce = min((2 * g + 2) * s * kNB, n);
                        RT = (ce - cs + 3) / 4;
                        if (rem < RT * CT) break;
                        rem -= RT * CT;
                    }
                    as = 2 * g * s * kNB;
                    ae = cs;
                    int rt, ct;
                    if (prod == 0) { ct = rem / RT; rt = rem - ct * RT; }                // column-major, increasing c
                    else { const int q = rem / CT; ct = rem - q * CT; rt = RT - 1 - q; }  // row-major, decreasing r
                    r0 = cs + rt * 4;
                    c0 = as + ct * 4;
                    have = true;
                    const T* rr[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) rr[u] = L + prow(min(r0 + u, n - 1));
                    if (prod == 0) {
                        // T(r, c) = sum_{k=c}^{ae-1} B(r, k) Ainv(k, c)
                        for (int k4 = c0; k4 < ae; k4 += 4) {
                            T bv[4][4], xv[4][4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) ld4(rr[u] + k4, bv[u]);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) ld4(L + prow(k4 + kk) + c0, xv[kk]);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                                for (int u = 0; u < 4; ++u)
#pragma unroll
                                    for (int v = 0; v < 4; ++v) acc[u][v] += bv[u][kk] * xv[kk][v];
                        }
                    } else {
                        // R(r, c) = -sum_{k=cs}^{r} Cinv(r, k) T(k, c)  (Cinv zero-padded past the diagonal)
                        const int kend = min(r0 + 4, n);
                        for (int k4 = cs; k4 < kend; k4 += 4) {
                            T cv[4][4], xv[4][4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) ld4(rr[u] + k4, cv[u]);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) ld4(L + prow(min(k4 + kk, n - 1)) + c0, xv[kk]);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                if (k4 + kk < n)
#pragma unroll
                                    for (int u = 0; u < 4; ++u)
#pragma unroll
                                        for (int v = 0; v < 4; ++v) acc[u][v] -= cv[u][kk] * xv[kk][v];
                        }
                    }
                }
                __syncthreads();
                if (have) {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (r0 + u < n) st4(L + prow(r0 + u) + c0, acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
                }
                __syncthreads();
            }
        }
    }

    CHOL_PHASE(56);
    // ------------------------------------------------------------------ outputs
    // Only the lower triangle (and its zero padding to a multiple of 4) is stored, 4 elements per thread: the
    // strictly upper part of Linv / Linv_lo is zero from the workspace's creation and never written.
    T* out = static_cast<T*>(cd.Linv);
    float* lo = static_cast<float*>(cd.Linv_lo);
    const bool vec_out = (cd.ldl & 3) == 0 && (((uintptr_t)out) & (4 * sizeof(T) - 1)) == 0 &&
                         (!lo || (((uintptr_t)lo) & 15) == 0);
    for (int i = warp; i < n; i += nwarp) {
        const T* row = L + prow(i);
        const bool z = defic[i];
        const int len = min(rup4(i + 1), (int)cd.ldl);
        if (vec_out) {
            for (int c = lane * 4; c < len; c += 128) {
                T v[4];
                ld4(row + c, v);
                if (z) v[0] = v[1] = v[2] = v[3] = T(0);
                T* o = out + (long long)i * cd.ldl + c;
                if constexpr (sizeof(T) == 4) {
                    *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
                    reinterpret_cast<double2*>(o)[0] = make_double2(v[0], v[1]);
                    reinterpret_cast<double2*>(o)[1] = make_double2(v[2], v[3]);
                }
                if (lo) {
                    float f[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) { const float x = (float)v[u]; f[u] = x - tf32_trunc(x); }
                    *reinterpret_cast<float4*>(lo + (long long)i * cd.ldl + c) = make_float4(f[0], f[1], f[2], f[3]);
                }
            }
        } else {
            for (int j = lane; j < len; j += 32) {
                const T v = z ? T(0) : row[j];
                out[(long long)i * cd.ldl + j] = v;
                if (lo) {
                    const float f = (float)v;
                    lo[(long long)i * cd.ldl + j] = f - tf32_trunc(f);
                }
            }
        }
    }
    for (int i = tid; i < n; i += nthr) cd.flags[i] = defic[i];
    if (tid == 0) *cd.nflags = any_defic;
    __syncthreads();
    CHOL_PHASE(57);
}

// ------------------------------------------------------------------------------ Cholesky-inverse on a CTA cluster
// cholinv_cluster_kernel: the same G = L L^T, Linv = L^{-1} (same deficiency semantics) spread over a cluster of 4
// CTAs per factor.  L itself is never stored: the inverse is accumulated by the same right-looking sweep, so there is
// no separate inversion phase.  32-row blocks are owned in snake order (0,1,2,3,3,2,1,0,0,...), each owned row i kept
// in the owner's shared memory as ONE row of (block+1)*32 entries: columns left of the current panel hold the
// partial inverse row R_i = e_i - sum_{c<=b} L_ic X_c, columns right of it the trailing Schur complement.
// Step b (panel of block b, J0 = 32b):
//   1. owner(b): L_bb = chol(A_bb) by one warp (pivot chain on shuffles), then X_b = L_bb^{-1} [R_b | I] by one
//      thread per column -- X_b is the final block row b of Linv (written to global at once);        barrier
//   2. all: X_b copied from the owner (distributed shared memory), panel rows of the owned rows below,
//      P_i = A_i(:, J0:J0+32) L_bb^{-T} (L_bb^{-1} is X_b's last 32 columns), pushed to every CTA's panel;  barrier
//   3. all, owned rows below block b, 4x4 register tiles with k-major operands (conflict-free LDS.128):
//      trailing A_ic -= P_i . P_c (J0+32 <= c <= i) and inverse R_i(:, 0:J0+32) -= P_i X_b.
// Two cluster barriers per 32 columns (16 for w = 230) instead of the single CTA's serial TRSM and log-depth
// inversion; every product has a fixed order (deterministic).
#ifndef RKFAC_CC_CTAS
#define RKFAC_CC_CTAS 4  // CTAs per cluster (per factor); 2 / 4 / 8 measured (tools/chol_cc_sweep.sh): FP32 123 / 115 / 234 us at w = 230, 26 factors (8: two waves)
#endif
constexpr int kCC = RKFAC_CC_CTAS;
#ifndef RKFAC_CC_THREADS
#define RKFAC_CC_THREADS 256  // 192 / 256 / 384 / 512 measured: 256 best (FP32 113 us, FP64 193 us at w = 230)
#endif
#ifndef RKFAC_CC_DEFER64
#define RKFAC_CC_DEFER64 0
#endif
#ifndef RKFAC_CC_TW32
// columns per register tile of the trailing / inverse update; 4 or 8. 8 measured slower (tools/chol_tw_sweep.sh,
// w = 230: 122 vs 115 us FP32, 219 vs 195 us FP64): the update is latency-bound, fewer tiles leave threads idle
#define RKFAC_CC_TW32 4
#endif
#ifndef RKFAC_CC_TW64
#define RKFAC_CC_TW64 4
#endif
constexpr int kCcThreads = RKFAC_CC_THREADS;
constexpr int kCcMaxBlk = 16;

__host__ __device__ __forceinline__ int cc_owner(int b) {
    const int r = b % (2 * kCC);
    return r < kCC ? r : 2 * kCC - 1 - r;
}
__host__ __device__ __forceinline__ int cc_pitch(int b) { return (b + 1) * kNB + 4; }  // odd in 16-byte units

__host__ __device__ inline int cc_rows_elems(int n, int q) {
    const int nblk = (n + kNB - 1) / kNB;
    int e = 0;
    for (int b = 0; b < nblk; ++b)
        if (cc_owner(b) == q) e += min(kNB, n - b * kNB) * cc_pitch(b);
    return e;
}

__host__ __device__ inline size_t cc_smem_bytes(int n, int es) {
    int rows = 0;
    for (int q = 0; q < kCC; ++q) rows = max(rows, cc_rows_elems(n, q));
    rows = (rows + 3) & ~3;
    const int np = rup8(n) + 4, xbp = rup8(n) + 4, lp = kNB + 4;  // odd multiples of 16 bytes
    size_t b = (size_t)es * ((size_t)rows + (size_t)kNB * np + (size_t)kNB * xbp + (size_t)kNB * lp + 3 * kNB);
    b = (b + 15) & ~(size_t)15;
    b += 4 * (size_t)rup4(n) + (size_t)rup4(n) + 16 + 64;  // diag0 (float), defic, flags
    return (b + 15) & ~(size_t)15;
}

__device__ __forceinline__ void cc_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <class TG, class T>
__global__ void __cluster_dims__(kCC, 1, 1) __launch_bounds__(kCcThreads)
    cholinv_cluster_kernel(const CholDesc* __restrict__ descs, double tol) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int q = (int)cluster.block_rank();
    const CholDesc& cd = descs[blockIdx.x / kCC];
    const int n = cd.w, nblk = (n + kNB - 1) / kNB;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int np = rup8(n) + 4, xbp = rup8(n) + 4, lp = kNB + 4;  // odd multiples of 16 bytes
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* rows = reinterpret_cast<T*>(smem_raw);
    // the row storage differs per CTA; everything after it sits at the same offset in every CTA (pushed remotely)
    int mxrows = 0;
    for (int qq = 0; qq < kCC; ++qq) mxrows = max(mxrows, cc_rows_elems(n, qq));
    T* panel = rows + ((mxrows + 3) & ~3);  // k-major [kNB][np]: panel[k][i] = P_ik
    T* xb = panel + kNB * np;      // X_b, k-major [kNB][xbp]
    T* lbbT = xb + kNB * xbp;      // L_bb transposed: lbbT[c][i] = L_ic
    T* dinv = lbbT + kNB * lp;     // 1 / L_kk (0 for a deficient pivot)
    T* colbuf = dinv + kNB;        // 2 x kNB column broadcast of the factorisation
    float* diag0 = reinterpret_cast<float*>(
        reinterpret_cast<unsigned char*>(smem_raw) +
        ((sizeof(T) * ((size_t)(panel - rows) + (size_t)kNB * np + (size_t)kNB * xbp + (size_t)kNB * lp + 3 * kNB) +
          15) & ~(size_t)15));
    unsigned char* defic = reinterpret_cast<unsigned char*>(diag0 + rup4(n));
    int* cflags = reinterpret_cast<int*>(defic + ((rup4(n) + 15) & ~15));  // [kCC] any-deficiency per CTA (CTA 0)
    __shared__ int boff[kCcMaxBlk];
    __shared__ int any_defic;
    const T tolT = T(tol);

    // ---- layout of the owned blocks, zeroed panel / X_b buffers, owned rows of G (lower triangle)
    if (tid == 0) {
        int e = 0;
        for (int b = 0; b < nblk; ++b) {
            if (cc_owner(b) == q) { boff[b] = e; e += min(kNB, n - b * kNB) * cc_pitch(b); }
            else boff[b] = -1;
        }
        any_defic = 0;
    }
    for (int i = tid; i < kNB * np; i += kCcThreads) panel[i] = T(0);
    for (int i = tid; i < kNB * xbp; i += kCcThreads) xb[i] = T(0);
    __syncthreads();
    const TG* G = static_cast<const TG*>(cd.G);
    for (int b = 0; b < nblk; ++b) {
        if (boff[b] < 0) continue;
        const int J0 = b * kNB, nb = min(kNB, n - J0), pb = cc_pitch(b);
        T* rb = rows + boff[b];
        if (cd.part) {  // lane = row: the column-major partials are read 128 bytes per warp access
            const int r = lane, i = J0 + r;
            for (int j = warp; j < pb; j += kCcThreads / 32) {
                if (r < nb) {
                    const T g = (j <= i) ? T(gram_from_parts(cd, i, j)) : T(0);
                    rb[r * pb + j] = g;
                    if (j == i) { diag0[i] = (float)g; defic[i] = 0; }
                }
            }
        } else {
            for (int r = warp; r < nb; r += kCcThreads / 32) {
                const int i = J0 + r;
                for (int j = lane; j < pb; j += 32) {
                    const T g = (j <= i) ? T(G[(long long)i * cd.ldg + j]) : T(0);
                    rb[r * pb + j] = g;
                    if (j == i) { diag0[i] = (float)g; defic[i] = 0; }
                }
            }
        }
    }
    CHOL_PHASE(0);
    cluster.sync();  // every CTA runs: distributed shared memory may be accessed
    CHOL_PHASE(1);

    T* out = static_cast<T*>(cd.Linv);
    float* lo = static_cast<float*>(cd.Linv_lo);
    const bool vec_out = (cd.ldl & 3) == 0 && (((uintptr_t)out) & (4 * sizeof(T) - 1)) == 0 &&
                         (!lo || (((uintptr_t)lo) & 15) == 0);

    // 32x32 diagonal block fb of the owner, one warp: L_bb into lbbT (transposed), 1/L_kk into dinv
    auto factor_block = [&](int fb) {
        const int J0 = fb * kNB, nb = min(kNB, n - J0), pb = cc_pitch(fb);
        const T* rb = rows + boff[fb];
            T a[kNB];
            const int rl = min(lane, nb - 1);
#pragma unroll
            for (int c4 = 0; c4 < kNB; c4 += 4) {
                T v4[4];
                ld4(rb + rl * pb + J0 + c4, v4);
#pragma unroll
                for (int u = 0; u < 4; ++u) a[c4 + u] = (lane < nb && c4 + u <= lane) ? v4[u] : T(0);
            }
            // right-looking, lane = row: the pivot and the next pivot's multiplier by shuffle, the rest of the
            // column through shared memory (double-buffered, one __syncwarp per step); FP32 applies that rest one
            // step late (software pipelined: the shared-memory round trip leaves the pivot chain)
            T tp[kNB];
            auto step = [&](int k, int nbv, bool defer) {
                const T piv = __shfl_sync(0xffffffffu, a[k], k);
                const T g = T(diag0[J0 + k]);
                const bool def = !(piv > tolT * g) || g == T(0);
                const T inv = def ? T(0) : rsqrt_t(piv);
                const T lkk = def ? T(1) : piv * inv;
                a[k] = lane == k ? lkk : (lane > k ? a[k] * inv : a[k]);
                if (lane == 0) dinv[k] = inv;
                if (def && lane == 0) { defic[J0 + k] = 1; any_defic = 1; }
                if (k + 1 < nbv) {
                    const T tn = __shfl_sync(0xffffffffu, a[k], k + 1);
                    T* cb = colbuf + (k & 1) * kNB;
                    cb[lane] = a[k];
                    __syncwarp();
                    if (defer) {
                        T tc[kNB];
#pragma unroll
                        for (int q4 = (k + 2) & ~3; q4 < kNB; q4 += 4) {
                            T v4[4];
                            ld4(cb + q4, v4);
#pragma unroll
                            for (int u = 0; u < 4; ++u) tc[q4 + u] = v4[u];
                        }
                        if (k >= 1) {
#pragma unroll
                            for (int j = k + 1; j < kNB; ++j) a[j] -= a[k - 1] * tp[j];
                        }
                        a[k + 1] -= a[k] * tn;
#pragma unroll
                        for (int j = k + 2; j < kNB; ++j) tp[j] = tc[j];
                    } else {
                        a[k + 1] -= a[k] * tn;
#pragma unroll
                        for (int q4 = (k + 2) & ~3; q4 < kNB; q4 += 4) {
                            T v4[4];
                            ld4(cb + q4, v4);
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                if (q4 + u >= k + 2) a[q4 + u] -= a[k] * v4[u];
                        }
                    }
                } else if (defer && k >= 1) {
#pragma unroll
                    for (int j = k + 1; j < kNB; ++j) a[j] -= a[k - 1] * tp[j];
                }
            };
            constexpr bool kDefer = sizeof(T) == 4 || RKFAC_CC_DEFER64;
            if (nb == kNB) {
#pragma unroll
                for (int k = 0; k < kNB; ++k) step(k, kNB, kDefer);
            } else {
#pragma unroll
                for (int k = 0; k < kNB; ++k)
                    if (k < nb) step(k, nb, false);
            }
#pragma unroll
            for (int c = 0; c < kNB; ++c) lbbT[c * lp + lane] = (lane < nb && c <= lane) ? a[c] : T(0);
    };
    // block row b of Linv is final: store it (rows of deficient pivots are zero) and its deficiency flags
    auto store_block = [&](int sb, int w0) {  // by warps w0 ..
        const int J0 = sb * kNB, nb = min(kNB, n - J0), pb = cc_pitch(sb);
        const T* rb = rows + boff[sb];
        for (int r = warp - w0; r < nb; r += kCcThreads / 32 - w0) {
            const int i = J0 + r;
            const T* row = rb + r * pb;
            const int len = min(rup4(i + 1), (int)cd.ldl);
            const bool z = defic[i];
            if (vec_out) {
                for (int c = lane * 4; c < len; c += 128) {
                    T v[4];
                    ld4(row + c, v);
                    if (z) v[0] = v[1] = v[2] = v[3] = T(0);
                    T* o = out + (long long)i * cd.ldl + c;
                    if constexpr (sizeof(T) == 4) {
                        *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
                    } else {
                        reinterpret_cast<double2*>(o)[0] = make_double2(v[0], v[1]);
                        reinterpret_cast<double2*>(o)[1] = make_double2(v[2], v[3]);
                    }
                    if (lo) {
                        float f[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) { const float x = (float)v[u]; f[u] = x - tf32_trunc(x); }
                        *reinterpret_cast<float4*>(lo + (long long)i * cd.ldl + c) =
                            make_float4(f[0], f[1], f[2], f[3]);
                    }
                }
            } else {
                for (int j = lane; j < len; j += 32) {
                    const T v = z ? T(0) : row[j];
                    out[(long long)i * cd.ldl + j] = v;
                    if (lo) {
                        const float f = (float)v;
                        lo[(long long)i * cd.ldl + j] = f - tf32_trunc(f);
                    }
                }
            }
            if (lane == 0) cd.flags[i] = z;
        }
    };

    for (int b = 0; b < nblk; ++b) {
        const int J0 = b * kNB, nb = min(kNB, n - J0), own = cc_owner(b);
        const int ncols = rup4(J0 + nb);  // columns of X_b (lower triangle, zero padded to a multiple of 4)
        // ------------------------------------------------ 1. owner: factor the diagonal block, X_b = L_bb^-1 [R_b|I]
        if (own == q) {
            const int pb = cc_pitch(b);
            T* rb = rows + boff[b];
            if (b == 0 && warp == 0) factor_block(0);  // later blocks were factored during the previous step
            __syncthreads();
            CHOL_PHASE(30 + b);
            // X_b = L_bb^{-1} [R_b(:, 0:J0) | I]: one thread per column, forward substitution in registers
            for (int c = tid; c < ncols; c += kCcThreads) {
                T acc[kNB];
#pragma unroll
                for (int i = 0; i < kNB; ++i)
                    acc[i] = (i < nb) ? (c < J0 ? rb[i * pb + c] : (c - J0 == i ? T(1) : T(0))) : T(0);
#pragma unroll
                for (int k = 0; k < kNB; ++k) {
                    const T x = acc[k] * dinv[k];
                    acc[k] = x;
#pragma unroll
                    for (int i4 = (k + 1) & ~3; i4 < kNB; i4 += 4) {
                        T l4[4];
                        ld4(lbbT + k * lp + i4, l4);
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i4 + u > k) acc[i4 + u] -= l4[u] * x;
                    }
                }
#pragma unroll
                for (int i = 0; i < kNB; ++i)
                    if (i < nb) rb[i * pb + c] = acc[i];
            }
            __syncthreads();
            CHOL_PHASE(40 + b);
            if (b + 1 == nblk) store_block(b, 0);
        }
        CHOL_PHASE(2 + 3 * b);
        if (b + 1 == nblk) break;
        cc_barrier();  // (1) X_b published
        // ------------------------------------------------ 2. X_b from the owner; panel rows of the owned rows below
        {
            const T* src = cluster.map_shared_rank(rows, own);
            // the owner's block-b offset: recomputed (boff is per CTA)
            int ob = 0;
            for (int bb = 0; bb < b; ++bb)
                if (cc_owner(bb) == own) ob += min(kNB, n - bb * kNB) * cc_pitch(bb);
            const int pb = cc_pitch(b);
            const int c4n = ncols / 4;
            for (int t = tid; t < nb * c4n; t += kCcThreads) {
                const int r = t / c4n, c = (t - r * c4n) * 4;
                T v[4];
                ld4(src + ob + r * pb + c, v);
                st4(xb + r * xbp + c, v[0], v[1], v[2], v[3]);
            }
        }
        __syncthreads();
        CHOL_PHASE(50 + b);
        // owned rows below block b: thread = (4 rows, one panel column k), one 16-byte store into every CTA
        for (int gbase = tid >> 5;; gbase += kCcThreads / 32) {
            int g = gbase, ob = b + 1;
            for (; ob < nblk; ++ob) {
                if (boff[ob] < 0) continue;
                const int G4 = (min(kNB, n - ob * kNB) + 3) / 4;
                if (g < G4) break;
                g -= G4;
            }
            if (ob >= nblk) break;
            const int k = lane, pbo = cc_pitch(ob), nbo = min(kNB, n - ob * kNB);
            const T* ar = rows + boff[ob] + g * 4 * pbo + J0;
            const T* xr = xb + k * xbp + J0;
            T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
            for (int m4 = 0; m4 < kNB; m4 += 4) {
                T x4[4];
                ld4(xr + m4, x4);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (g * 4 + u < nbo) {
                        T a4[4];
                        ld4(ar + u * pbo + m4, a4);
#pragma unroll
                        for (int m = 0; m < 4; ++m) acc[u] += a4[m] * x4[m];
                    }
                }
            }
            const int i0 = ob * kNB + g * 4;
#pragma unroll
            for (int r = 0; r < kCC; ++r) st4(cluster.map_shared_rank(panel, r) + k * np + i0, acc[0], acc[1], acc[2], acc[3]);
        }
        CHOL_PHASE(3 + 3 * b);
        cc_barrier();  // (2) panel complete in every CTA
        // ------------------------------------------------ 3. trailing update and inverse update of the owned rows
        {
            // row groups of 4 owned rows below block b; group at row i0 has i0/4 + 1 column tiles (0 .. i0)
            // tiles are 4 rows x kTW columns; group g of block ob covers columns 0 .. ob*kNB + 4g + 3
            constexpr int kTW = sizeof(T) == 4 ? RKFAC_CC_TW32 : RKFAC_CC_TW64;
            auto ntile = [&](int ob, int g) { return ob * (kNB / kTW) + (4 * g + 4 + kTW - 1) / kTW; };
            auto ntiles_blk = [&](int ob) {
                const int G4 = (min(kNB, n - ob * kNB) + 3) / 4;
                int t = 0;
                for (int g = 0; g < G4; ++g) t += ntile(ob, g);
                return t;
            };
            int total = 0;
            for (int ob = b + 1; ob < nblk; ++ob)
                if (boff[ob] >= 0) total += ntiles_blk(ob);
            const int jb = J0 + kNB;  // first trailing column
            // look-ahead: the owner of block b+1 updates that block's diagonal tiles first, then one warp factors it
            // while the others finish the update
            const bool ahead = cc_owner(b + 1) == q;
            auto tile = [&](int t, bool& diag_next, int& obo, int& go, int& c0o) {
                int rem = t, ob = b + 1, g = 0;
                for (; ob < nblk; ++ob) {
                    if (boff[ob] < 0) continue;
                    const int tiles = ntiles_blk(ob);
                    if (rem < tiles) break;
                    rem -= tiles;
                }
                for (;; ++g) {
                    const int tg = ntile(ob, g);
                    if (rem < tg) break;
                    rem -= tg;
                }
                obo = ob; go = g; c0o = rem * kTW;
                diag_next = ob == b + 1 && c0o >= jb;
            };
            auto run = [&](int ob, int g, int c0) {
                const int i0 = ob * kNB + g * 4;
                const int pbo = cc_pitch(ob);
                T* rr = rows + boff[ob] + g * 4 * pbo;
                const bool inv_tile = c0 < jb;
                const T* bop = inv_tile ? (xb + c0) : (panel + c0);
                const int bld = inv_tile ? xbp : np;
                T acc[4][kTW] = {};
#pragma unroll 8
                for (int k = 0; k < kNB; ++k) {  // nb == kNB: every block but the last has a trailing update
                    T av[4], bv[kTW];
                    ld4(panel + k * np + i0, av);
#pragma unroll
                    for (int v4 = 0; v4 < kTW; v4 += 4) {
                        T t4[4];
                        ld4(bop + k * bld + v4, t4);
#pragma unroll
                        for (int e = 0; e < 4; ++e) bv[v4 + e] = t4[e];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < kTW; ++v) acc[u][v] += av[u] * bv[v];
                }
                // panel columns become inverse columns: old value 0. Columns of a tile right of its rows' diagonal
                // (kTW > 4) receive values that are never read: X_b's substitution rewrites the block from I
                const bool fresh = c0 >= J0 && c0 < jb;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (i0 + u >= n) continue;
#pragma unroll
                    for (int v4 = 0; v4 < kTW; v4 += 4) {
                        T* w = rr + u * pbo + c0 + v4;
                        T o4[4] = {T(0), T(0), T(0), T(0)};
                        if (!fresh) ld4(w, o4);
                        st4(w, o4[0] - acc[u][v4], o4[1] - acc[u][v4 + 1], o4[2] - acc[u][v4 + 2],
                            o4[3] - acc[u][v4 + 3]);
                    }
                }
            };
            if (ahead) {
                const int G4 = (min(kNB, n - (b + 1) * kNB) + 3) / 4;
                auto ndg = [&](int g) { return (4 * g + 4 + kTW - 1) / kTW; };  // diagonal-block tiles of group g
                int nd = 0;
                for (int g = 0; g < G4; ++g) nd += ndg(g);
                for (int t = tid; t < nd; t += kCcThreads) {
                    int g = 0, rem = t;
                    while (rem >= ndg(g)) { rem -= ndg(g); ++g; }
                    run(b + 1, g, jb + rem * kTW);
                }
                __syncthreads();
                if (warp == 0) factor_block(b + 1);
            }
            if (!ahead || warp > 0) {
                const int t0 = ahead ? tid - 32 : tid, nt = ahead ? kCcThreads - 32 : kCcThreads;
                for (int t = t0; t < total; t += nt) {
                    bool dn;
                    int ob, g, c0;
                    tile(t, dn, ob, g, c0);
                    if (ahead && dn) continue;
                    run(ob, g, c0);
                }
                // block row b of Linv: stored off the critical path (not by the warp factoring block b+1)
                if (own == q) store_block(b, ahead ? 1 : 0);
            }
        }
        __syncthreads();
        CHOL_PHASE(4 + 3 * b);
    }
    // ---- any-deficiency flag: gathered in CTA 0
    if (tid == 0) cluster.map_shared_rank(cflags, 0)[q] = any_defic;
    cc_barrier();
    if (q == 0 && tid == 0) {
        int a = 0;
        for (int r = 0; r < kCC; ++r) a |= cflags[r];
        *cd.nflags = a;
    }
    CHOL_PHASE(60);
}

// Deterministic pseudo-random candidate for completing a rank-deficient column.
__device__ __forceinline__ float cand_value(int k, int attempt, int i) {
    const uint64_t h = splitmix64(0xC0FFEEULL ^ ((uint64_t)k << 40) ^ ((uint64_t)attempt << 32) ^ (uint64_t)i);
    return (float)((double)(h >> 11) * 0x1.0p-53 - 0.5);
}

__device__ float block_sum(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.f;
    if (threadIdx.x < 32) {
        s = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) red[32] = s;
    }
    __syncthreads();
    return red[32];
}

// Fills each flagged (zeroed) row k of Qt (w x d) with a unit vector orthogonal to all other rows, then refreshes
// the derived planes (Q row-major copy and TF32 lo planes) of those rows.
__global__ void __launch_bounds__(1024) complete_kernel(const CompleteDesc* __restrict__ descs) {
    const CompleteDesc& cd = descs[blockIdx.x];
    if (*cd.nflags == 0) return;
    __shared__ float red[33];
    const int w = cd.w, d = cd.d;
    float* Qt = cd.Qt;
    for (int k = 0; k < w; ++k) {
        if (!cd.flags[k]) continue;
        for (int attempt = 0; attempt < 8; ++attempt) {
            float n0 = 0.f;
            for (int i = threadIdx.x; i < d; i += blockDim.x) {
                const float v = cand_value(k, attempt, i);
                Qt[(long long)k * cd.ldq + i] = v;
                n0 += v * v;
            }
            n0 = block_sum(n0, red);
            for (int pass = 0; pass < 2; ++pass) {
                for (int j = 0; j < w; ++j) {
                    if (j == k || (cd.flags[j] && j > k)) continue;  // later flagged rows are still zero
                    float dot = 0.f;
                    for (int i = threadIdx.x; i < d; i += blockDim.x)
                        dot += Qt[(long long)k * cd.ldq + i] * Qt[(long long)j * cd.ldq + i];
                    dot = block_sum(dot, red);
                    for (int i = threadIdx.x; i < d; i += blockDim.x)
                        Qt[(long long)k * cd.ldq + i] -= dot * Qt[(long long)j * cd.ldq + i];
                    __syncthreads();
                }
            }
            float nn = 0.f;
            for (int i = threadIdx.x; i < d; i += blockDim.x) {
                const float v = Qt[(long long)k * cd.ldq + i];
                nn += v * v;
            }
            nn = block_sum(nn, red);
            if (nn > 1e-8f * n0) {
                const float inv = rsqrtf(nn);
                for (int i = threadIdx.x; i < d; i += blockDim.x) Qt[(long long)k * cd.ldq + i] *= inv;
                __syncthreads();
                break;
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            const float v = Qt[(long long)k * cd.ldq + i];
            const float l = v - tf32_trunc(v);
            if (cd.Qt_lo) cd.Qt_lo[(long long)k * cd.ldq + i] = l;
            if (cd.Q) cd.Q[(long long)i * cd.ldr + k] = v;
            if (cd.Q_lo) cd.Q_lo[(long long)i * cd.ldr + k] = l;
        }
        __syncthreads();
    }
}

// Rank-deficient columns of the final basis: the flagged (zero) rows of Qt get deterministic pseudo-random
// candidates, which the CholeskyQR2 pass that follows orthonormalises together with the good columns (span of the
// good columns unchanged).  Intermediate bases simply keep their zero columns: X maps them to zero, so they stay
// flagged and never perturb the power iteration (rank(X) < w means the good columns already span range(X)).
__global__ void __launch_bounds__(256) fill_kernel(const CompleteDesc* __restrict__ descs) {
    const CompleteDesc& cd = descs[blockIdx.y];
    if (*cd.nflags == 0) return;
    const int w = cd.w, d = cd.d;
    const float unit = sqrtf(12.f / (float)d);  // candidates of about unit norm: the CholeskyQR that follows sees a
                                                // well-conditioned Gram (good columns are unit norm too)
    for (int k = 0; k < w; ++k) {
        if (!cd.flags[k]) continue;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
            const float v = unit * cand_value(k, 0, i);
            const float l = v - tf32_trunc(v);
            cd.Qt[(long long)k * cd.ldq + i] = v;
            if (cd.Qt_lo) cd.Qt_lo[(long long)k * cd.ldq + i] = l;
            if (cd.Q) cd.Q[(long long)i * cd.ldr + k] = v;
            if (cd.Q_lo) cd.Q_lo[(long long)i * cd.ldr + k] = l;
        }
    }
}

}  // namespace

// RKFAC_CHOLINV_SINGLE=1 forces the single-CTA kernel (A/B checks and tools/chol_bench)
static bool cholinv_single_cta() {
    static const bool v = [] {
        const char* e = getenv("RKFAC_CHOLINV_SINGLE");
        return e && e[0] == '1';
    }();
    return v;
}

size_t cholinv_smem_bytes(int wmax, bool fp64) {
    const int es = fp64 ? 8 : 4;
    return (size_t)cholinv_state_bytes(wmax, es) + (size_t)prow(wmax) * es;
}

void launch_cholinv(const CholDesc* d_descs, int nfactors, int wmax, bool fp64, bool gram64, double tol,
                    cudaStream_t s) {
    if (nfactors == 0) return;
    RKFAC_REQUIRE(wmax <= kMaxW, RKFAC_INVALID_ARGUMENT, "sketch width above 512 is not supported");
    if (wmax > kNB && !cholinv_single_cta()) {
        auto kc = fp64 ? (gram64 ? cholinv_cluster_kernel<double, double> : cholinv_cluster_kernel<float, double>)
                       : (gram64 ? cholinv_cluster_kernel<double, float> : cholinv_cluster_kernel<float, float>);
        const size_t cb = cc_smem_bytes(wmax, fp64 ? 8 : 4);
        if (cb <= max_dynamic_smem((const void*)kc)) {
            RKFAC_CUDA(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cb));
            kc<<<nfactors * kCC, kCcThreads, cb, s>>>(d_descs, tol);
            count_launch();
            RKFAC_CHECK_LAUNCH();
            return;
        }
    }
    const size_t bytes = cholinv_smem_bytes(wmax, fp64);
    auto ks = fp64 ? (gram64 ? cholinv_kernel<double, double, true> : cholinv_kernel<float, double, true>)
                   : (gram64 ? cholinv_kernel<double, float, true> : cholinv_kernel<float, float, true>);
    auto kg = fp64 ? (gram64 ? cholinv_kernel<double, double, false> : cholinv_kernel<float, double, false>)
                   : (gram64 ? cholinv_kernel<double, float, false> : cholinv_kernel<float, float, false>);
    const bool use_smem = bytes <= max_dynamic_smem((const void*)ks);
    auto k = use_smem ? ks : kg;
    const size_t dyn = use_smem ? bytes : (size_t)cholinv_state_bytes(wmax, fp64 ? 8 : 4);
    RKFAC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k<<<nfactors, kCholThreads, dyn, s>>>(d_descs, tol);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_fill(const CompleteDesc* d_descs, int nfactors, cudaStream_t s) {
    if (nfactors == 0) return;
    fill_kernel<<<dim3(8, nfactors), 256, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_complete(const CompleteDesc* d_descs, int nfactors, cudaStream_t s) {
    if (nfactors == 0) return;
    complete_kernel<<<nfactors, 1024, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
