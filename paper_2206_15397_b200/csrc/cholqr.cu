// cholqr.cu -- CholeskyQR building blocks for the orthonormalisation of the sketch (replaces qr_thin,
// qr.hpp:23-87, inside randomized_range, rnla.hpp:47-56).
//
//   G = Y^T Y (grouped GEMM)  ->  cholinv_kernel: G = L L^T, Linv = L^{-1}  ->  Q^T = Linv Y^T (grouped GEMM)
//   -> complete_kernel (only when a column was rank deficient)
//
// The reference's Householder QR forces diag(R) >= 0, so its thin Q is unique for full-rank input and
// CholeskyQR (R = L^T has a positive diagonal) yields the same Q up to rounding.  Only span(Q) matters
// downstream (C = Q^T X Q and U = Q P are basis independent), so rank-deficient columns -- which the
// reference skips (qr.hpp:35-45, H = I) -- are replaced here by any unit vector orthogonal to the others.
//
// cholinv_kernel: one CTA per factor; the packed lower triangle lives in shared memory when it fits (w <= 230
// in FP64), else in a global scratch.  Blocked right-looking Cholesky (panel width 8, 4x4 register tiles for
// the trailing update) followed by an in-place triangular inversion with row-parallel dot products.
#include <cmath>

#include "kernels.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kPanel = 8;
constexpr int kMaxW = 512;

__device__ __forceinline__ long long pk(int i, int j) { return (long long)i * (i + 1) / 2 + j; }

template <class T>
__device__ __forceinline__ T my_sqrt(T x) { return sqrt(x); }

template <class TG, class T>
__global__ void __launch_bounds__(1024) cholinv_kernel(const CholDesc* __restrict__ descs, int use_smem,
                                                       double tol) {
    const CholDesc& cd = descs[blockIdx.x];
    const int n = cd.w;
    const int tid = threadIdx.x, nthr = blockDim.x;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* L = use_smem ? reinterpret_cast<T*>(smem_raw) : static_cast<T*>(cd.scratch);
    __shared__ T diag0[kMaxW];
    __shared__ T xs[kMaxW];
    __shared__ T prow[kPanel];
    __shared__ int defic[kMaxW];
    __shared__ int any_defic;

    const TG* G = static_cast<const TG*>(cd.G);
    // Load the symmetrised lower triangle.
    for (int i = tid / 32; i < n; i += nthr / 32)
        for (int j = tid % 32; j <= i; j += 32)
            L[pk(i, j)] = T(0.5) * (T(G[(long long)i * n + j]) + T(G[(long long)j * n + i]));
    for (int i = tid; i < n; i += nthr) defic[i] = 0;
    if (tid == 0) any_defic = 0;
    __syncthreads();
    for (int i = tid; i < n; i += nthr) diag0[i] = L[pk(i, i)];
    __syncthreads();

    // ---- blocked right-looking Cholesky ----
    for (int p0 = 0; p0 < n; p0 += kPanel) {
        const int nb = min(kPanel, n - p0);
        const int rows = n - p0;
        // Panel: thread t owns row i = p0 + t (rows <= n <= kMaxW <= 1024 threads... loop for safety).
        T r[kPanel];
        const int i = p0 + tid;
        const bool own = tid < rows;
#pragma unroll
        for (int c = 0; c < kPanel; ++c) r[c] = (own && c < nb && p0 + c <= i) ? L[pk(i, p0 + c)] : T(0);
        for (int c = 0; c < nb; ++c) {
            const int pc = p0 + c;
            if (own && i == pc) {
                T s = r[c];
#pragma unroll
                for (int t = 0; t < kPanel; ++t)
                    if (t < c) s -= r[t] * r[t];
                T lcc;
                const T g = diag0[pc];
                if (!(s > T(tol) * g) || g == T(0)) {  // rank-deficient column (also catches NaN)
                    defic[pc] = 1;
                    any_defic = 1;
                    lcc = T(1);
#pragma unroll
                    for (int t = 0; t < kPanel; ++t)
                        if (t < c) r[t] = T(0);
                } else {
                    lcc = my_sqrt(s);
                }
                r[c] = lcc;
#pragma unroll
                for (int t = 0; t < kPanel; ++t) prow[t] = (t <= c) ? r[t] : T(0);
            }
            __syncthreads();
            if (own && i > pc) {
                if (defic[pc]) {
                    r[c] = T(0);
                } else {
                    T s = r[c];
#pragma unroll
                    for (int t = 0; t < kPanel; ++t)
                        if (t < c) s -= r[t] * prow[t];
                    r[c] = s / prow[c];
                }
            }
            __syncthreads();
        }
        if (own) {
#pragma unroll
            for (int c = 0; c < kPanel; ++c) {
                if (c < nb && p0 + c <= i) L[pk(i, p0 + c)] = r[c];

            }
        }
        __syncthreads();
        // Trailing update with 4x4 register tiles over the lower triangle of rows/cols >= p0+nb.
        const int t0 = p0 + nb;
        const int m = n - t0;
        if (m > 0) {
            const int TI = (m + 3) / 4;
            const int ntiles = TI * (TI + 1) / 2;
            for (int t = tid; t < ntiles; t += nthr) {
                int I = (int)((sqrtf(8.f * (float)t + 1.f) - 1.f) * 0.5f);
                while ((long long)I * (I + 1) / 2 > t) --I;
                while ((long long)(I + 1) * (I + 2) / 2 <= t) ++I;
                const int J = t - I * (I + 1) / 2;
                T acc[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = T(0);
#pragma unroll
                for (int c = 0; c < kPanel; ++c) {
                    T a[4], b[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int ii = t0 + I * 4 + u, jj = t0 + J * 4 + u;
                        a[u] = (ii < n && c < nb) ? L[pk(ii, p0 + c)] : T(0);
                        b[u] = (jj < n && c < nb) ? L[pk(jj, p0 + c)] : T(0);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int v = 0; v < 4; ++v) acc[u][v] += a[u] * b[v];
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int ii = t0 + I * 4 + u;
                    if (ii >= n) continue;
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const int jj = t0 + J * 4 + v;
                        if (jj > ii) continue;
                        L[pk(ii, jj)] -= acc[u][v];
                    }
                }
            }
        }
        __syncthreads();
    }

    // ---- in-place inversion of the lower-triangular L (LAPACK trti2 order: last column first) ----
    for (int j = n - 1; j >= 0; --j) {
        const T ljj_inv = T(1) / L[pk(j, j)];
        const int cnt = n - 1 - j;
        for (int k = tid; k < cnt; k += nthr) xs[k] = L[pk(j + 1 + k, j)];
        __syncthreads();
        // y_i = sum_{k=j+1}^{i} Linv[i][k] x_k, rows i = j+1..n-1; G threads per row.
        int g = 1;
        while (g < 8 && g * 2 * cnt <= nthr) g *= 2;
        T y = T(0);
        const int row = tid / g, seg = tid % g;
        const int ii = j + 1 + row;
        if (row < cnt) {
            for (int k = j + 1 + seg; k <= ii; k += g) y += L[pk(ii, k)] * xs[k - j - 1];
        }
        for (int off = g / 2; off > 0; off /= 2) y += __shfl_down_sync(0xffffffffu, y, off, g);
        __syncthreads();
        if (row < cnt && seg == 0) L[pk(ii, j)] = -ljj_inv * y;
        if (tid == 0) L[pk(j, j)] = ljj_inv;
        __syncthreads();
    }

    // ---- write Linv (full w x w, zero upper part; rank-deficient rows zeroed so Q's column is 0) ----
    T* out = static_cast<T*>(cd.Linv);
    for (long long e = tid; e < (long long)n * n; e += nthr) {
        const int i = (int)(e / n), j = (int)(e - (long long)i * n);
        out[e] = (j <= i && !defic[i]) ? L[pk(i, j)] : T(0);
    }
    for (int i = tid; i < n; i += nthr) cd.flags[i] = defic[i];
    if (tid == 0) *cd.nflags = any_defic;
}

// Deterministic pseudo-random unit-ish candidate for completing a rank-deficient column.
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

// Fills each flagged (zeroed) row k of Qt (w x d) with a unit vector orthogonal to all other rows.
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
    }
}

}  // namespace

size_t cholinv_smem_bytes(int wmax, bool fp64) {
    const size_t es = fp64 ? 8 : 4;
    return (size_t)wmax * (wmax + 1) / 2 * es;
}

void launch_cholinv(const CholDesc* d_descs, int nfactors, int wmax, bool fp64, bool gram64, double tol,
                    cudaStream_t s) {
    if (nfactors == 0) return;
    RKFAC_REQUIRE(wmax <= kMaxW, RKFAC_INVALID_ARGUMENT, "sketch width above 512 is not supported");
    const size_t bytes = cholinv_smem_bytes(wmax, fp64);
    const int threads = 1024;
    auto k = fp64 ? (gram64 ? cholinv_kernel<double, double> : cholinv_kernel<float, double>)
                  : (gram64 ? cholinv_kernel<double, float> : cholinv_kernel<float, float>);
    const bool use_smem = bytes <= max_dynamic_smem((const void*)k);
    const size_t dyn = use_smem ? bytes : 0;
    RKFAC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    k<<<nfactors, threads, dyn, s>>>(d_descs, use_smem ? 1 : 0, tol);
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
