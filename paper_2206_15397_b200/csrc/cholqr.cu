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
// cholinv_kernel: one CTA (1024 threads) per factor.  The lower triangle lives in shared memory in a
// "padded packed" layout: row i starts at a 16-byte aligned offset and is zero-padded to a multiple of 4 entries,
// so every inner loop is a 4x4 register tile fed by LDS.128 and the zero padding doubles as the upper-triangle
// zeros of L^{-1}.  w <= 230 fits in FP64 (w <= 330 in FP32); larger w uses a global scratch.  Latency matters
// more than the w^3/3 flops, so:
//   Cholesky   right-looking over 32-wide panels: the 32x32 diagonal block is factored by one warp in registers
//              (shuffles, no block barrier), the panel below by a row-parallel TRSM, the trailing update by 4x4
//              register tiles -- 3 barriers per panel;
//   inverse    all 32x32 diagonal blocks inverted concurrently (one warp each), then block rows
//              X_I = -(D_I^{-1} L_I,<I) X_<I in place, 4x4 register tiles -- 3 barriers per block row.
#include <cmath>

#include "kernels.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kNB = 32;
constexpr int kMaxW = 512;
constexpr int kCholThreads = 512;  // 128-register budget: the unrolled 32-wide row arrays stay in registers

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__host__ __device__ __forceinline__ int rup4(int x) { return (x + 3) & ~3; }

// Offset of row i in the padded packed layout: sum_{t<i} rup4(t+1).
__host__ __device__ __forceinline__ int prow(int i) {
    // rup4(t+1) for t = 4a+b (b=0..3) is 4a+4 => a block of 4 rows [4a, 4a+4) occupies 16a+16
    const int a = i >> 2, b = i & 3;
    return 8 * a * (a + 1) + b * (4 * a + 4);
}

// bytes of the small per-factor state carved at the start of the dynamic smem (16-byte multiple)
__host__ __device__ __forceinline__ int cholinv_state_bytes(int n, int es) {
    return (es * (kNB * (kNB + 1) + kNB) + 4 * rup4(n) + rup4(n) + 15) & ~15;
}

template <class T> struct Vec4T;
template <> struct Vec4T<float> { using type = float4; };
template <> struct Vec4T<double> { using type = double4; };

template <class T>
__device__ __forceinline__ void ld4(const T* p, T (&v)[4]) {
    using V = typename Vec4T<T>::type;
    const V x = *reinterpret_cast<const V*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}

// kSmem selects the storage of the triangle at compile time: a pointer chosen at run time between shared and
// global memory compiles to generic LD/ST (measured ~2.5x slower than LDS/STS on this kernel).
template <class TG, class T, bool kSmem>
__global__ void __launch_bounds__(kCholThreads) cholinv_kernel(const CholDesc* __restrict__ descs, double tol) {
    const CholDesc& cd = descs[blockIdx.x];
    const int n = cd.w;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // dynamic smem: [small per-factor state][padded packed triangle (kSmem only)]
    T (*l11t)[kNB + 1] = reinterpret_cast<T (*)[kNB + 1]>(smem_raw);          // transposed diagonal block
    T* dinv = reinterpret_cast<T*>(smem_raw + sizeof(T) * kNB * (kNB + 1));    // its reciprocal diagonal
    float* diag0 = reinterpret_cast<float*>(dinv + kNB);                       // original diagonal of G
    unsigned char* defic = reinterpret_cast<unsigned char*>(diag0 + rup4(n));  // rank-deficiency flags
    __shared__ int any_defic;
    T* L;
    if constexpr (kSmem) L = reinterpret_cast<T*>(smem_raw + cholinv_state_bytes(n, sizeof(T)));
    else L = static_cast<T*>(cd.scratch);
    const T tolT = T(tol);

    const TG* G = static_cast<const TG*>(cd.G);
    for (int i = warp; i < n; i += nwarp) {
        T* row = L + prow(i);
        for (int j = lane; j < rup4(i + 1); j += 32)
            row[j] = (j <= i) ? T(0.5) * (T(G[(long long)i * cd.ldg + j]) + T(G[(long long)j * cd.ldg + i])) : T(0);
    }
    for (int i = tid; i < n; i += nthr) defic[i] = 0;
    if (tid == 0) any_defic = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nthr) diag0[i] = (float)L[prow(i) + i];
    __syncthreads();

    const int nblk = (n + kNB - 1) / kNB;
    // ------------------------------------------------------------------ blocked right-looking Cholesky
    for (int b = 0; b < nblk; ++b) {
        const int J0 = b * kNB, nb = min(kNB, n - J0);
        if (warp == 0) {
            // (1) 32x32 diagonal block in registers, lane i owns row J0+i.  Step k broadcasts column k by
            //     shuffles issued in batches of 8 before their FMAs (a SHFL->FFMA chain per element serialises on
            //     the shuffle latency).
            T a[kNB];
            const T* rowp = L + prow(J0 + min(lane, nb - 1)) + J0;
#pragma unroll
            for (int c = 0; c < kNB; ++c) a[c] = (lane < nb && c <= lane) ? rowp[c] : T(0);
#pragma unroll
            for (int k = 0; k < kNB; ++k) {
                if (k < nb) {
                    const T piv = __shfl_sync(0xffffffffu, a[k], k);
                    const T g = T(diag0[J0 + k]);
                    const bool def = !(piv > tolT * g) || g == T(0);
                    const T lkk = def ? T(1) : sqrt(piv);
                    const T inv = def ? T(0) : T(1) / lkk;
                    if (lane == k) {
                        a[k] = lkk;
                        dinv[k] = inv;
                        if (def) { defic[J0 + k] = 1; any_defic = 1; }
                    } else if (lane > k) {
                        a[k] *= inv;
                    }
#pragma unroll
                    for (int j0 = k + 1; j0 < kNB; j0 += 8) {
                        T t[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (j0 + u < kNB) t[u] = __shfl_sync(0xffffffffu, a[k], j0 + u);
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (j0 + u < kNB && lane >= j0 + u) a[j0 + u] -= a[k] * t[u];
                    }
                }
            }
            if (lane < nb) {
                T* wrow = L + prow(J0 + lane) + J0;
#pragma unroll
                for (int c = 0; c < kNB; ++c)
                    if (c <= lane) wrow[c] = a[c];
            }
        }
        __syncthreads();
        // (2) panel TRSM (left-looking per row, 4 partial sums per dot, reciprocal diagonal); rows below the
        //     block, one thread per row; L11 rows are broadcast from smem.  Deficient columns give 0.
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
                        s0 -= x[q] * lc[q];
                        if (q + 1 < c) s1 -= x[q + 1] * lc[q + 1];
                        if (q + 2 < c) s2 -= x[q + 2] * lc[q + 2];
                        if (q + 3 < c) s3 -= x[q + 3] * lc[q + 3];
                    }
                    x[c] = ((s0 + s1) + (s2 + s3)) * dinv[c];
                }
            }
#pragma unroll
            for (int c = 0; c < kNB; ++c)
                if (c < nb) rp[c] = x[c];
        }
        __syncthreads();
        // (3) trailing update A22 -= L21 L21^T (lower triangle), 4x4 tiles, LDS.128 along the panel columns
        const int t0 = J0 + nb, m = n - t0;
        if (m > 0) {
            const int TI = (m + 3) / 4;
            const int ntiles = TI * (TI + 1) / 2;
            for (int t = tid; t < ntiles; t += nthr) {
                int I = (int)((sqrtf(8.f * (float)t + 1.f) - 1.f) * 0.5f);
                while (I * (I + 1) / 2 > t) --I;
                while ((I + 1) * (I + 2) / 2 <= t) ++I;
                const int J = t - I * (I + 1) / 2;
                const T* ra[4];
                const T* rb[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    ra[u] = L + prow(min(t0 + I * 4 + u, n - 1)) + J0;
                    rb[u] = L + prow(min(t0 + J * 4 + u, n - 1)) + J0;
                }
                T acc[4][4] = {};
#pragma unroll
                for (int c4 = 0; c4 < kNB; c4 += 4) {
                    if (c4 < nb) {  // panel columns beyond nb are zero padding / next rows: masked below
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
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int ii = t0 + I * 4 + u;
                    if (ii >= n) continue;
                    T* wr = L + prow(ii);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int jj = t0 + J * 4 + v;
                        if (jj <= ii) wr[jj] -= acc[u][v];
                    }
                }
            }
        }
        __syncthreads();
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
                T s0 = T(0), s1 = T(0);
#pragma unroll
                for (int k = 0; k < i; k += 2) {
                    if (k >= j) s0 += li[k] * x[k];
                    if (k + 1 < i && k + 1 >= j) s1 += li[k + 1] * x[k + 1];
                }
                x[i] = (i < j) ? T(0) : (i == j ? di : -(s0 + s1) * di);
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
    // (b) block rows I = 1..nblk-1: X_I,<i0 = -(D_I^{-1} L_I,<i0) X_<i0,<i0
    for (int I = 1; I < nblk; ++I) {
        const int i0 = I * kNB, nbI = min(kNB, n - i0);
        // step 1 (in place): B = D_I^{-1} L_I,<i0, one thread per column c < i0 (D_I entries broadcast)
        for (int c = tid; c < i0; c += nthr) {
            T col[kNB];
#pragma unroll
            for (int s = 0; s < kNB; ++s) col[s] = (s < nbI) ? L[prow(i0 + s) + c] : T(0);
#pragma unroll
            for (int r = kNB - 1; r >= 0; --r) {  // descending r: col[s] for s <= r is still the input
                if (r < nbI) {
                    const T* dr = L + prow(i0 + r) + i0;
                    T acc = T(0);
#pragma unroll
                    for (int s = 0; s <= r; ++s) acc += dr[s] * col[s];
                    col[r] = acc;
                }
            }
#pragma unroll
            for (int r = 0; r < kNB; ++r)
                if (r < nbI) L[prow(i0 + r) + c] = col[r];
        }
        __syncthreads();
        // step 2: X(i0+r, c) = -sum_{k=c}^{i0-1} B(r, k) X(k, c); 4x4 tiles; X rows are zero-padded past the
        // diagonal, so whole LDS.128 groups can be used from k = c0 on
        // Tiles are processed in passes of increasing column c0: a tile reads B(r, k) only for k >= c0 and writes
        // columns c0..c0+3, so writing a pass in place never clobbers what a later pass still has to read.
        const int rg = (nbI + 3) / 4, cgs = i0 / 4;
        const int ntl = rg * cgs;
        for (int pass = 0; pass * nthr < ntl; ++pass) {
        const int tt = pass * nthr + tid;
        T res[4][4];
        int r0 = 0, c0 = 0;
        const bool have = tt < ntl;
        if (have) {
            r0 = (tt % rg) * 4;
            c0 = (tt / rg) * 4;
            const T* rb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) rb[u] = L + prow(i0 + min(r0 + u, nbI - 1));
            T acc[4][4] = {};
            for (int k4 = c0; k4 < i0; k4 += 4) {
                T bv[4][4], xv[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) ld4(rb[u] + k4, bv[u]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) ld4(L + prow(k4 + kk) + c0, xv[kk]);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[u][v] += bv[u][kk] * xv[kk][v];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) res[u][v] = -acc[u][v];
        }
        __syncthreads();
        if (have) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (r0 + u < nbI) {
                    T* wr = L + prow(i0 + r0 + u) + c0;
#pragma unroll
                    for (int v = 0; v < 4; ++v) wr[v] = res[u][v];
                }
        }
        __syncthreads();
        }  // pass
    }

    // ------------------------------------------------------------------ outputs
    T* out = static_cast<T*>(cd.Linv);
    float* lo = static_cast<float*>(cd.Linv_lo);
    const int wcols = (int)min((long long)rup4(n), cd.ldl);
    for (int i = warp; i < n; i += nwarp) {
        const T* row = L + prow(i);
        for (int j = lane; j < wcols; j += 32) {
            const T v = (j <= i && !defic[i]) ? row[j] : T(0);
            out[(long long)i * cd.ldl + j] = v;
            if (lo) {
                const float f = (float)v;
                lo[(long long)i * cd.ldl + j] = f - tf32_trunc(f);
            }
        }
    }
    for (int i = tid; i < n; i += nthr) cd.flags[i] = defic[i];
    if (tid == 0) *cd.nflags = any_defic;
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

}  // namespace

size_t cholinv_smem_bytes(int wmax, bool fp64) {
    const int es = fp64 ? 8 : 4;
    return (size_t)cholinv_state_bytes(wmax, es) + (size_t)prow(wmax) * es;
}

void launch_cholinv(const CholDesc* d_descs, int nfactors, int wmax, bool fp64, bool gram64, double tol,
                    cudaStream_t s) {
    if (nfactors == 0) return;
    RKFAC_REQUIRE(wmax <= kMaxW, RKFAC_INVALID_ARGUMENT, "sketch width above 512 is not supported");
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

void launch_complete(const CompleteDesc* d_descs, int nfactors, cudaStream_t s) {
    if (nfactors == 0) return;
    complete_kernel<<<nfactors, 1024, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
