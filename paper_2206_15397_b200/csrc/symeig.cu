// symeig.cu -- full symmetric eigendecomposition S = P diag(d) P^T of a d x d factor, FP64, on the GPU: the exact
// K-FAC comparator (kfactor.hpp:165-186 apply_eig_damped_inverse over eig.hpp:210-237 sym_eig,
// harness.hpp:402-478 bench-inverse) and the spectrum snapshots (8(f) #4: kfactor.hpp:56-63).
//
// The reference tridiagonalises with Householder reflections (tred2) and diagonalises the tridiagonal with the
// implicit QL iteration (tql2), eig.hpp:33-193 -- O(n^3) serial loops.  Same mathematics here, organised for the GPU:
//   1. Householder tridiagonalisation blocked like LAPACK's sytrd/latrd.  A panel of 32 columns runs on a cooperative
//      grid (one CTA per SM): per column the update from the panel's earlier reflectors, the reflector, the symmetric
//      matrix-vector product over the trailing matrix by every SM (the memory-bound half of the flops), and the panel
//      corrections -- four grid barriers per column.  The trailing matrix then takes the rank-64 update as two FP64
//      GEMMs.  The full symmetric matrix is kept (both triangles), so every matrix-vector row is a coalesced stream.
//   2. The tridiagonal eigenproblem by Cuppen's divide and conquer: leaves of <= 32 by implicit QL with Wilkinson
//      shifts in one warp; each merge T = diag(T1, T2) + rho u u^T by deflation (small z components; close poles
//      rotated out), the secular equation 1 + rho sum z_i^2 / (d_i - lambda) = 0 by bisection (one warp per root,
//      each root kept as an offset from its nearer pole), the Gu-Eisenstat recomputed z-hat (numerically orthogonal
//      eigenvectors in working precision) and the eigenvector update as an FP64 GEMM.
//   3. Back-transformation P = H_0 ... H_{n-2} Z in compact-WY blocks of 32 reflectors (dlarft forward columnwise),
//      three GEMMs per block.
// Eigenvectors are kept eigenvector-major (row c = eigenvector c) so every column operation of the merges is a
// contiguous row operation.  Output: eigenvalues descending, eigenvectors as the columns of P (eig.hpp:197-203).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "symeig.cuh"

namespace cg = cooperative_groups;

namespace rkfac_b200 {

namespace {

constexpr int kNB = 32;           // panel width (reflectors per block)
constexpr int kPS = 72;           // per-CTA partials of the panel kernel: [0] ssq, [1..32] W^T v, [33..64] V^T v, [65] w.v
constexpr int kPanelThreads = 256;
constexpr int kLeaf = 32;
constexpr double kEps = 1.1102230246251565e-16;  // 2^-53

// ------------------------------------------------------------------------------------------- FP64 GEMM
constexpr int kGT = 64, kGK = 16;

// nd == 0: the single problem `one` (passed by value: no descriptor upload)
__global__ void __launch_bounds__(256) dgemm_kernel(const DGemmDesc* __restrict__ descs, int nd, DGemmDesc one) {
    int lo = 0, hi = nd - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (descs[mid].tile_off <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    const DGemmDesc g = nd ? descs[lo] : one;
    int t = blockIdx.x - g.tile_off;
    int kbeg = 0, kend = g.K, slice = 0;
    if (g.ksplit > 1) {  // tiles of slice s are [s * tiles_mn, (s + 1) * tiles_mn)
        const int tiles_mn = ((g.M + kGT - 1) / kGT) * g.tiles_n;
        slice = t / tiles_mn;
        t -= slice * tiles_mn;
        kbeg = slice * g.kchunk;
        kend = min(g.K, kbeg + g.kchunk);
    }
    const int i0 = (t / g.tiles_n) * kGT, j0 = (t % g.tiles_n) * kGT;
    __shared__ double As[kGK][kGT + 4], Bs[kGK][kGT + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    double acc[4][4] = {};
    const bool a_kfast = g.csA == 1, b_jfast = g.csB == 1;
    for (int k0 = kbeg; k0 < kend; k0 += kGK) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = tid + 256 * u;
            int i, kk;
            if (a_kfast) { i = e / kGK; kk = e % kGK; } else { i = e % kGT; kk = e / kGT; }
            const int gi = i0 + i, gk = k0 + kk;
            As[kk][i] = (gi < g.M && gk < kend) ? g.A[gi * g.rsA + gk * g.csA] : 0.0;
            int j;
            if (b_jfast) { kk = e / kGT; j = e % kGT; } else { kk = e % kGK; j = e / kGK; }
            const int gj = j0 + j, gk2 = k0 + kk;
            Bs[kk][j] = (gj < g.N && gk2 < kend) ? g.B[gk2 * g.rsB + gj * g.csB] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kGK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { a[q] = As[kk][ty * 4 + q]; b[q] = Bs[kk][tx * 4 + q]; }
#pragma unroll
            for (int p = 0; p < 4; ++p)
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
        }
        __syncthreads();
    }
    // epilogue: every C element of the thread loaded first (16 independent loads in flight), then the stores
    if (g.ksplit > 1) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int gi = i0 + ty * 4 + p;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int gj = j0 + tx * 4 + q;
                if (gi < g.M && gj < g.N) g.partial[((long long)slice * g.M + gi) * g.N + gj] = acc[p][q];
            }
        }
        return;
    }
    double cv[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gi = i0 + ty * 4 + p, gj = j0 + tx * 4 + q;
            cv[p][q] = (g.beta != 0.0 && gi < g.M && gj < g.N) ? g.C[(long long)gi * g.ldc + gj] : 0.0;
        }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int gi = i0 + ty * 4 + p, gj = j0 + tx * 4 + q;
            if (gi < g.M && gj < g.N) g.C[(long long)gi * g.ldc + gj] = fma(g.alpha, acc[p][q], g.beta * cv[p][q]);
        }
}

// split-K reduction in a fixed slice order: C = alpha * sum_s partial[s] + beta * C
__global__ void dgemm_reduce_kernel(DGemmDesc g) {
    const long long mn = (long long)g.M * g.N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mn; e += (long long)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int s = 0; s < g.ksplit; ++s) acc += g.partial[s * mn + e];
        const long long i = e / g.N, j = e - i * g.N;
        double* c = g.C + i * g.ldc + j;
        *c = g.beta == 0.0 ? g.alpha * acc : fma(g.alpha, acc, g.beta * *c);
    }
}

// --------------------------------------------------------------------------------- input and output
// A = (S + S^T) / 2 in FP64 (eig.hpp:216 symmetrises); stats[0] = max |S - S^T|, stats[1] = max |S| (as ordered
// bit patterns of non-negative doubles).
__global__ void widen_kernel(const float* __restrict__ S, long long lds, int n, double* __restrict__ A, long long lda,
                             unsigned long long* stats) {
    double asym = 0.0, amax = 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n * n;
         e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e / n), c = (int)(e - (long long)r * n);
        const double x = S[(long long)r * lds + c], y = S[(long long)c * lds + r];
        A[(long long)r * lda + c] = 0.5 * (x + y);
        asym = fmax(asym, fabs(x - y));
        amax = fmax(amax, fabs(x));
    }
    for (int o = 16; o; o >>= 1) {
        asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
        amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&stats[0], (unsigned long long)__double_as_longlong(asym));
        atomicMax(&stats[1], (unsigned long long)__double_as_longlong(amax));
    }
}

// P[r][c] = X[n-1-c][r] (eigenvector-major, ascending -> eigenvectors as columns, descending), dvals likewise.
__global__ void output_kernel(const double* __restrict__ X, long long ldx, const double* __restrict__ D, int n,
                              float* __restrict__ P, long long ldp, float* __restrict__ dv, double* __restrict__ dv64) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;  // bx: component r, by: output column c
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = by + y, r = bx + threadIdx.x;
        if (c < n && r < n) tile[y][threadIdx.x] = X[(long long)(n - 1 - c) * ldx + r];
    }
    __syncthreads();
    if (P)
        for (int y = threadIdx.y; y < 32; y += blockDim.y) {
            const int r = bx + y, c = by + threadIdx.x;
            if (c < n && r < n) P[(long long)r * ldp + c] = (float)tile[threadIdx.x][y];
        }
    if (blockIdx.x == 0 && threadIdx.y == 0) {
        const int c = by + threadIdx.x;
        if (c < n) {
            if (dv) dv[c] = (float)D[n - 1 - c];
            if (dv64) dv64[c] = D[n - 1 - c];
        }
    }
}

// ------------------------------------------------------------------------------ tridiagonalisation
struct PanelArgs {
    double* A; long long lda; int n, k, nbp;
    double* V; double* W;  // n x 32 row-major
    double* tau; double* d; double* e;
    double* part;          // gridDim.x x kPS
    double* vbuf; double* ybuf;
};

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    return s;
}

// sum over CTAs of part[b * kPS + idx] by warp 0, broadcast through shared memory
__device__ __forceinline__ double grid_partial_sum(const double* part, int idx, double* slot) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (int b = threadIdx.x; b < (int)gridDim.x; b += 32) s += part[b * kPS + idx];
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *slot = s;
    }
    __syncthreads();
    const double r = *slot;
    __syncthreads();
    return r;
}

// One panel of 32 columns (latrd): reflectors v_j (stored in A below the subdiagonal, implicit 1 at j+1), tau_j,
// d_j, e_j, and the panel's V, W (n x 32) for the trailing update A -= V W^T + W V^T.
//
// Thread tid owns row tid (the grid has >= n threads).  Three grid barriers per column j:
//   X  the previous column's w correction alpha (w = w_raw + alpha v, from the partials of w_raw . v); own row:
//      a_r = b_r + alpha c_r (the column updated by the panel's earlier reflectors, b and c prepared in Z), the
//      previous column's final w; partial |a|^2 below the subdiagonal
//   Y  the reflector (dlarfg) from |a|^2; y = A22 v with v = scal (a - a_{j+1} e_{j+1}) + e_{j+1}, formed as
//      scal A22 a + (1 - scal a_{j+1}) A22 e_{j+1} (warp per row, coalesced rows of the full symmetric matrix), so
//      the matrix-vector product needs no barrier after the reflector; partial W^T a, V^T a
//   Z  W^T v, V^T v from those; own row: v_r, w_raw = tau (y - V (W^T v) - W (V^T v)), partial w_raw . v; the next
//      column's b_r, c_r (its panel term t = i split into the raw part and the alpha part)
enum { kWV = 0, kSS = 1, kDots = 8 };  // part layout: [kDots, kDots+64) = W^T a, V^T a

__global__ void __launch_bounds__(kPanelThreads) sytrd_panel_kernel(PanelArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[2][kPanelThreads / 32];
    __shared__ double bc[2];
    __shared__ double cwv[2 * kNB];
    __shared__ double accs[kPanelThreads / 32][2 * kNB];
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int gw = blockIdx.x * nw + warp, GW = gridDim.x * nw;
    const long long lda = a.lda;
    const int n = a.n, r = tid;  // the row this thread owns
    const bool own = r < n;
    double* pub = a.part + gridDim.x * kPS;  // a_{j+1}, published by its owner
    double* abuf = a.vbuf;
    auto cta_reduce = [&](double v, int idx) {
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[0][warp] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += red[0][w];
            a.part[blockIdx.x * kPS + idx] = t;
        }
        __syncthreads();
    };
    auto grid_sum = [&](int idx) {
        if (warp == 0) {
            double t = 0.0;
            for (int b2 = lane; b2 < (int)gridDim.x; b2 += 32) t += a.part[b2 * kPS + idx];
            for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) bc[0] = t;
        }
        __syncthreads();
        const double t = bc[0];
        __syncthreads();
        return t;
    };
    if (own && r >= a.k)
        for (int t = 0; t < kNB; ++t) { a.V[r * kNB + t] = 0.0; a.W[r * kNB + t] = 0.0; }
    // column k has no panel updates: b = A(:, k), c = 0
    double b_r = (own && r >= a.k) ? a.A[r * lda + a.k] : 0.0, c_r = 0.0;
    if (threadIdx.x == 0) a.part[blockIdx.x * kPS + kWV] = 0.0;
    double tau_prev = 0.0;
    for (int i = 0; i < a.nbp; ++i) {
        const int j = a.k + i;
        grid.sync();  // X
        const double alpha2 = i > 0 ? -0.5 * tau_prev * grid_sum(kWV) : 0.0;
        double a_r = 0.0;
        if (own && r >= j) {
            a_r = b_r + alpha2 * c_r;
            if (i > 0) a.W[r * kNB + i - 1] += alpha2 * a.V[r * kNB + i - 1];  // final w of the previous column
            abuf[r] = a_r;
            if (r == j) { a.A[r * lda + j] = a_r; a.d[j] = a_r; }
            if (r == j + 1) pub[0] = a_r;
        }
        cta_reduce((own && r >= j + 2) ? a_r * a_r : 0.0, kSS);
        grid.sync();  // Y
        const double ssq = grid_sum(kSS);
        const double a1 = pub[0];
        double beta, tj, scal;
        if (ssq <= 0.0) { beta = a1; tj = 0.0; scal = 0.0; }
        else {
            const double nrm = sqrt(a1 * a1 + ssq);
            beta = a1 >= 0.0 ? -nrm : nrm;
            tj = (beta - a1) / beta;
            scal = 1.0 / (a1 - beta);
        }
        if (tid == 0) { a.tau[j] = tj; a.e[j] = beta; }
        {
            const double corr = 1.0 - scal * a1;
            double aw = 0.0, av = 0.0;  // lane t accumulates column t of W^T a and V^T a
            for (int rr = j + 1 + gw; rr < n; rr += GW) {
                const double* row = a.A + rr * lda;
                double y = 0.0;
                for (int c = j + 1 + lane; c < n; c += 32) y = fma(row[c], abuf[c], y);
                for (int o = 16; o; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
                if (lane == 0) a.ybuf[rr] = scal * y + corr * row[j + 1];
                const double ar = abuf[rr];
                if (lane < i) { aw = fma(a.W[rr * kNB + lane], ar, aw); av = fma(a.V[rr * kNB + lane], ar, av); }
            }
            accs[warp][lane] = aw;
            accs[warp][kNB + lane] = av;
            __syncthreads();
            if (threadIdx.x < 2 * kNB) {
                double sum = 0.0;
                for (int w = 0; w < nw; ++w) sum += accs[w][threadIdx.x];
                a.part[blockIdx.x * kPS + kDots + threadIdx.x] = sum;
            }
        }
        grid.sync();  // Z
        if (threadIdx.x < 2 * kNB) {
            const int t = threadIdx.x & (kNB - 1);
            double sum = 0.0;
            if (t < i) {
                for (int b2 = 0; b2 < (int)gridDim.x; ++b2) sum += a.part[b2 * kPS + kDots + threadIdx.x];
                // W^T v = W(j+1,:) + scal (W^T a - W(j+1,:) a_{j+1})   (v_{j+1} = 1, v_r = scal a_r below)
                const double wj = threadIdx.x < kNB ? a.W[(j + 1) * kNB + t] : a.V[(j + 1) * kNB + t];
                sum = wj + scal * (sum - wj * a1);
            }
            cwv[threadIdx.x] = sum;
        }
        __syncthreads();
        auto w_raw_of = [&](int row) {
            double y = a.ybuf[row];
            for (int t = 0; t < i; ++t) y -= a.V[row * kNB + t] * cwv[t] + a.W[row * kNB + t] * cwv[kNB + t];
            return tj * y;
        };
        double wv = 0.0, wr = 0.0, v_r = 0.0;
        if (own && r >= j + 1) {
            v_r = (r == j + 1) ? 1.0 : scal * a_r;
            a.V[r * kNB + i] = v_r;
            if (r >= j + 2) a.A[r * lda + j] = v_r;  // reflector storage (the 1 at j+1 is implicit)
            wr = w_raw_of(r);
            a.W[r * kNB + i] = wr;
            wv = wr * v_r;
        }
        if (i + 1 < a.nbp && own && r >= j + 1) {
            // next column j+1: a_r = b_r + alpha c_r, its panel term t = i split into the raw and the alpha part
            const int jn = j + 1;
            const double wj1 = w_raw_of(jn);  // row j+1's raw w (its owner computes the same value)
            double x = a.A[r * lda + jn];
            for (int t = 0; t < i; ++t)
                x -= a.V[r * kNB + t] * a.W[jn * kNB + t] + a.W[r * kNB + t] * a.V[jn * kNB + t];
            x -= v_r * wj1 + wr;  // V(j+1, i) = 1
            b_r = x;
            c_r = -2.0 * v_r;
        }
        cta_reduce(wv, kWV);
        tau_prev = tj;
    }
    grid.sync();
    const double alpha2 = -0.5 * tau_prev * grid_sum(kWV);
    const int jl = a.k + a.nbp - 1;
    if (own && r >= jl + 1) a.W[r * kNB + a.nbp - 1] += alpha2 * a.V[r * kNB + a.nbp - 1];  // last w column
}

__global__ void last_diag_kernel(const double* A, long long lda, int n, double* d, double* e) {
    d[n - 1] = A[(long long)(n - 1) * lda + (n - 1)];
    if (n >= 1) e[n - 1] = 0.0;
}

// ------------------------------------------------------------------------------ divide and conquer
struct MergeDesc {
    int s, m, m1;
    double rho, theta;  // T = diag(T1', T2') + rho u u^T, u = e_{m1-1} + theta e_{m1} (block-local)
};

struct MergeMeta {
    int k, kd, nrot, pad;
    double rhon;
};

// Per-index work arrays (length n each, a merge uses [s, s+m)).
struct DcArrays {
    double* ds;   // sorted d
    double* zs;   // sorted normalized z
    int* perm;    // sorted index -> block column
    int* ndidx;   // nondeflated sorted indices (ascending d)
    int* dfidx;   // deflated sorted indices
    int* rp; int* rq; double* rc; double* rs;  // rotations (sorted-index space)
    double* dnd; double* znd;                  // compact nondeflated d, z
    int* org; double* tau; double* zhat;       // roots: lambda_j = dnd[org_j] + tau_j
    MergeMeta* meta;                           // per merge
};

// Cuppen coupling: the children solve T1 with its last diagonal and T2 with its first diagonal reduced by |beta|.
__global__ void adjust_kernel(const MergeDesc* md, int nm, double* d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nm) return;
    const MergeDesc m = md[i];
    d[m.s + m.m1 - 1] -= m.rho;
    d[m.s + m.m1] -= m.rho;
}

// Leaves (<= 32): implicit QL with Wilkinson shifts, one warp per leaf.  Lane 0 runs the scalar sweep and records
// its rotations; every lane then applies them to its own row of Z (Z[row][col], columns = eigenvectors).
constexpr int kLeafWarps = 4;
__global__ void __launch_bounds__(kLeafWarps * 32) leaf_kernel(const int* starts, const int* sizes, int nleaves, double* d,
                                                   const double* e, double* QT, long long ldq, int* fail) {
    __shared__ double Zs[kLeafWarps][kLeaf][kLeaf + 1];
    __shared__ double dd[kLeafWarps][kLeaf], ee[kLeafWarps][kLeaf], rc[kLeafWarps][kLeaf], rs[kLeafWarps][kLeaf];
    __shared__ int ctl[kLeafWarps][4];
    __shared__ int perm[kLeafWarps][kLeaf];
    const int wb = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int leaf = blockIdx.x * kLeafWarps + wb;
    if (leaf >= nleaves) return;
    const int s = starts[leaf], m = sizes[leaf];
    double (*Z)[kLeaf + 1] = Zs[wb];
    for (int c = 0; c < kLeaf; ++c) Z[lane][c] = (lane == c) ? 1.0 : 0.0;
    dd[wb][lane] = lane < m ? d[s + lane] : 0.0;
    ee[wb][lane] = lane < m - 1 ? e[s + lane] : 0.0;
    __syncwarp();
    for (int l = 0; l < m; ++l) {
        for (int iter = 0;; ++iter) {
            if (lane == 0) {
                double* D = dd[wb];
                double* E = ee[wb];
                int mm = l;
                for (; mm < m - 1; ++mm) {
                    const double dsum = fabs(D[mm]) + fabs(D[mm + 1]);
                    if (fabs(E[mm]) <= kEps * dsum) break;
                }
                int nr = 0, lo = l;
                if (mm != l && iter < 60) {
                    double g = (D[l + 1] - D[l]) / (2.0 * E[l]);
                    double r = hypot(g, 1.0);
                    g = D[mm] - D[l] + E[l] / (g + copysign(r, g));
                    double sn = 1.0, cs = 1.0, p = 0.0;
                    bool early = false;
                    for (int i = mm - 1; i >= l; --i) {
                        const double f = sn * E[i], b = cs * E[i];
                        r = hypot(f, g);
                        E[i + 1] = r;
                        if (r == 0.0) {  // underflow: split here
                            D[i + 1] -= p;
                            E[mm] = 0.0;
                            early = true;
                            lo = i + 1;
                            break;
                        }
                        sn = f / r;
                        cs = g / r;
                        g = D[i + 1] - p;
                        r = (D[i] - g) * sn + 2.0 * cs * b;
                        p = sn * r;
                        D[i + 1] = g + p;
                        g = cs * r - b;
                        rc[wb][nr] = cs;
                        rs[wb][nr] = sn;
                        ++nr;
                    }
                    if (!early) {
                        D[l] -= p;
                        E[l] = g;
                        E[mm] = 0.0;
                    }
                }
                if (mm != l && iter >= 60) atomicExch(fail, 1);
                ctl[wb][0] = (mm == l || iter >= 60) ? 1 : 0;
                ctl[wb][1] = mm;
                ctl[wb][2] = nr;
                ctl[wb][3] = lo;
            }
            __syncwarp();
            if (ctl[wb][0]) break;
            const int mm = ctl[wb][1], nr = ctl[wb][2];
            for (int q = 0; q < nr; ++q) {  // rotation q acts on columns (i, i+1), i = mm-1-q
                const int i = mm - 1 - q;
                const double cs = rc[wb][q], sn = rs[wb][q];
                const double fz = Z[lane][i + 1];
                Z[lane][i + 1] = sn * Z[lane][i] + cs * fz;
                Z[lane][i] = cs * Z[lane][i] - sn * fz;
            }
            __syncwarp();
        }
        __syncwarp();
    }
    // ascending order (selection by lane 0), then rows out, eigenvector-major
    if (lane == 0) {
        for (int c = 0; c < m; ++c) perm[wb][c] = c;
        for (int c = 0; c < m; ++c) {
            int best = c;
            for (int q = c + 1; q < m; ++q)
                if (dd[wb][perm[wb][q]] < dd[wb][perm[wb][best]]) best = q;
            const int t = perm[wb][c]; perm[wb][c] = perm[wb][best]; perm[wb][best] = t;
        }
    }
    __syncwarp();
    if (lane < m)
        for (int c = 0; c < m; ++c) QT[(long long)(s + c) * ldq + s + lane] = Z[lane][perm[wb][c]];
    if (lane < m) d[s + lane] = dd[wb][perm[wb][lane]];
}

// M1 (one CTA per merge): z, the merged sort, deflation (small z; close poles rotated out, dlaed2's tests).
__global__ void __launch_bounds__(1024) merge_setup_kernel(const MergeDesc* md, const double* QT, long long ldq,
                                                           const double* d, DcArrays w) {
    const MergeDesc g = md[blockIdx.x];
    const int s = g.s, m = g.m, m1 = g.m1;
    __shared__ double red[32];
    double zz = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double z = i < m1 ? QT[(long long)(s + i) * ldq + s + m1 - 1] : g.theta * QT[(long long)(s + i) * ldq + s + m1];
        zz += z * z;
    }
    for (int o = 16; o; o >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = zz;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
        red[0] = t;
    }
    __syncthreads();
    zz = red[0];
    const double zn = zz > 0.0 ? 1.0 / sqrt(zz) : 0.0;
    const double rhon = g.rho * zz;
    const double* D1 = d + s;
    const double* D2 = d + s + m1;
    const int m2 = m - m1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        int rank;
        double di;
        if (i < m1) {
            di = D1[i];
            int lo = 0, hi = m2;  // # of D2 < di
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (D2[mid] < di) lo = mid + 1; else hi = mid; }
            rank = i + lo;
        } else {
            di = D2[i - m1];
            int lo = 0, hi = m1;  // # of D1 <= di
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (D1[mid] <= di) lo = mid + 1; else hi = mid; }
            rank = (i - m1) + lo;
        }
        const double z = i < m1 ? QT[(long long)(s + i) * ldq + s + m1 - 1] : g.theta * QT[(long long)(s + i) * ldq + s + m1];
        w.perm[s + rank] = i;
        w.ds[s + rank] = di;
        w.zs[s + rank] = z * zn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double* ds = w.ds + s;
        double* zs = w.zs + s;
        const double dmax = fmax(fabs(ds[0]), fabs(ds[m - 1]));
        const double tol = 8.0 * kEps * fmax(dmax, fabs(rhon));
        int k = 0, kd = 0, nrot = 0, p = -1;
        for (int q = 0; q < m; ++q) {
            if (fabs(rhon * zs[q]) <= tol) {  // small z: (d_q, e_q) is an eigenpair
                w.dfidx[s + kd++] = q;
                continue;
            }
            if (p < 0) { p = q; continue; }
            const double S0 = zs[p], C0 = zs[q];
            const double tn = hypot(C0, S0);
            const double c = C0 / tn, sn = -S0 / tn;
            const double t = ds[q] - ds[p];
            if (fabs(t * c * sn) <= tol) {  // close poles: rotate z_p out, p deflates
                zs[q] = tn;
                zs[p] = 0.0;
                const double tp = ds[p] * c * c + ds[q] * sn * sn;
                ds[q] = ds[p] * sn * sn + ds[q] * c * c;
                ds[p] = tp;
                w.rp[s + nrot] = p; w.rq[s + nrot] = q; w.rc[s + nrot] = c; w.rs[s + nrot] = sn;
                ++nrot;
                w.dfidx[s + kd++] = p;
                p = q;
            } else {
                w.ndidx[s + k] = p;
                w.dnd[s + k] = ds[p];
                w.znd[s + k] = zs[p];
                ++k;
                p = q;
            }
        }
        if (p >= 0) {
            w.ndidx[s + k] = p;
            w.dnd[s + k] = ds[p];
            w.znd[s + k] = zs[p];
            ++k;
        }
        MergeMeta mt;
        mt.k = k; mt.kd = kd; mt.nrot = nrot; mt.pad = 0; mt.rhon = rhon;
        w.meta[blockIdx.x] = mt;
    }
}

__device__ __forceinline__ int find_merge(const MergeDesc* md, int nm, int gidx) {
    int lo = 0, hi = nm - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (md[mid].s <= gidx) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// M2 (thread per block row r = eigenvector component): gather the sorted columns, apply the rotations in order,
// write the nondeflated eigenvectors to QT rows s..s+k-1 and the deflated ones to rows s+k.. (eigenvector-major).
__global__ void merge_gather_kernel(const MergeDesc* md, int nm, double* __restrict__ QT, double* __restrict__ QgT,
                                    long long ldq, DcArrays w) {
    const int gidx = blockIdx.x * blockDim.x + threadIdx.x;  // global component index
    const int mi = find_merge(md, nm, gidx);
    const MergeDesc g = md[mi];
    if (gidx >= g.s + g.m) return;
    const int s = g.s, m = g.m, r = gidx - s;
    const MergeMeta mt = w.meta[mi];
    constexpr int U = 8;  // loads in flight per thread
    for (int i0 = 0; i0 < m; i0 += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            v[u] = i0 + u < m ? QT[(long long)(s + w.perm[s + i0 + u]) * ldq + s + r] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u < m) QgT[(long long)(s + i0 + u) * ldq + s + r] = v[u];
    }
    for (int q = 0; q < mt.nrot; ++q) {
        const int p = w.rp[s + q], qq = w.rq[s + q];
        const double c = w.rc[s + q], sn = w.rs[s + q];
        double* xp = QgT + (long long)(s + p) * ldq + s + r;
        double* xq = QgT + (long long)(s + qq) * ldq + s + r;
        const double x = *xp, y = *xq;
        *xp = c * x + sn * y;
        *xq = c * y - sn * x;
    }
    const int k = mt.k, kd = mt.kd;
    for (int i0 = 0; i0 < k + kd; i0 += U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int e = i0 + u;
            v[u] = e < k + kd ? QgT[(long long)(s + (e < k ? w.ndidx[s + e] : w.dfidx[s + e - k])) * ldq + s + r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u < k + kd) QT[(long long)(s + i0 + u) * ldq + s + r] = v[u];
    }
}

// M3 (warp per root): the secular equation f(lambda) = 1/rho + sum z_i^2 / (d_i - lambda) = 0 (f/rho: same sign),
// lambda = d_org + tau with org the nearer pole, so every d_i - lambda = (d_i - d_org) - tau is formed without
// cancellation.  A bracket [lo, hi] (f(lo) < 0 <= f(hi); f increases) is kept; each iteration takes the root of the
// two-pole rational model of f at the current point (psi and phi -- the sums over the poles left and right of the
// root -- each matched in value and slope by a constant plus one pole: the classic scheme behind LAPACK's dlaed4),
// falling back to bisection whenever the model's root leaves the bracket.  Converges in a handful of iterations;
// the bracket alone bounds the worst case.
__global__ void secular_kernel(const MergeDesc* md, int nm, DcArrays w, int total) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= total) return;
    const int mi = find_merge(md, nm, gw);
    const MergeDesc g = md[mi];
    const MergeMeta mt = w.meta[mi];
    const int s = g.s, j = gw - s, k = mt.k;
    if (j >= k) return;
    const double* dn = w.dnd + s;
    const double* zn = w.znd + s;
    const double irho = 1.0 / mt.rhon;
    // sums at offset t from pole o: psi (i <= j), dpsi, phi (i > j), dphi
    auto sums = [&](int o, double t, double& psi, double& dpsi, double& phi, double& dphi) {
        psi = dpsi = phi = dphi = 0.0;
        const double dor = dn[o];
        for (int i = lane; i < k; i += 32) {
            const double r = 1.0 / ((dn[i] - dor) - t);
            const double q = zn[i] * zn[i] * r;
            if (i <= j) { psi += q; dpsi += q * r; } else { phi += q; dphi += q * r; }
        }
        for (int q = 16; q; q >>= 1) {
            psi += __shfl_xor_sync(0xffffffffu, psi, q);
            dpsi += __shfl_xor_sync(0xffffffffu, dpsi, q);
            phi += __shfl_xor_sync(0xffffffffu, phi, q);
            dphi += __shfl_xor_sync(0xffffffffu, dphi, q);
        }
    };
    double psi, dpsi, phi, dphi;
    int o;
    double lo, hi, t;
    if (j < k - 1) {
        const double half = 0.5 * (dn[j + 1] - dn[j]);
        sums(j, half, psi, dpsi, phi, dphi);
        if (irho + psi + phi >= 0.0) { o = j; lo = 0.0; hi = half; }  // root in (d_j, midpoint]
        else { o = j + 1; lo = -half; hi = 0.0; }                      // root in (midpoint, d_{j+1})
    } else {
        double zz = 0.0;
        for (int i = lane; i < k; i += 32) zz += zn[i] * zn[i];
        for (int q = 16; q; q >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, q);
        o = j; lo = 0.0; hi = zz / irho;
    }
    t = 0.5 * (lo + hi);
    for (int it = 0; it < 100; ++it) {
        sums(o, t, psi, dpsi, phi, dphi);
        const double f = irho + psi + phi;
        if (f < 0.0) lo = t; else hi = t;
        if (f == 0.0 || hi - lo <= 2.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
        // two-pole model around the poles j (left) and j+1 (right) of the root
        const double dj = (dn[j] - dn[o]) - t;
        double tn;
        if (j < k - 1) {
            const double dj1 = (dn[j + 1] - dn[o]) - t;
            const double sl = dpsi * dj * dj, sr = dphi * dj1 * dj1;
            const double c = f - dpsi * dj - dphi * dj1;
            // c eta^2 - B eta + C = 0, eta the move of lambda
            const double B = c * (dj + dj1) + sl + sr, C = c * dj * dj1 + sl * dj1 + sr * dj;
            const double disc = fmax(0.0, B * B - 4.0 * c * C);
            double e1, e2;
            if (c == 0.0) { e1 = e2 = C / B; }
            else {
                const double qq = 0.5 * (B + copysign(sqrt(disc), B));
                e1 = qq / c;
                e2 = qq != 0.0 ? C / qq : e1;
            }
            const double t1 = t + e1, t2 = t + e2;
            tn = (t1 > lo && t1 < hi) ? t1 : ((t2 > lo && t2 < hi) ? t2 : 0.5 * (lo + hi));
        } else {
            const double sl = dpsi * dj * dj;
            const double c = f - dpsi * dj;  // c + sl / (dj - eta) = 0
            tn = c != 0.0 ? t + dj + sl / c : 0.5 * (lo + hi);
            if (!(tn > lo && tn < hi)) tn = 0.5 * (lo + hi);
        }
        if (fabs(tn - t) <= 2.0 * kEps * fabs(t)) { t = tn; break; }
        t = tn;
    }
    if (lane == 0) {
        w.org[s + j] = o;
        w.tau[s + j] = (t == 0.0) ? (o == j ? hi : lo) : t;
    }
}

// M4 (warp per i): Gu-Eisenstat z-hat_i^2 = prod_j (lambda_j - d_i) / (rho prod_{j != i} (d_j - d_i)).
__global__ void zhat_kernel(const MergeDesc* md, int nm, DcArrays w, int total) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= total) return;
    const int mi = find_merge(md, nm, gw);
    const MergeDesc g = md[mi];
    const MergeMeta mt = w.meta[mi];
    const int s = g.s, i = gw - s, k = mt.k;
    if (i >= k) return;
    const double* dn = w.dnd + s;
    const double di = dn[i];
    double prod = 1.0;
    for (int j = lane; j < k; j += 32) {
        const double lmd = (dn[w.org[s + j]] - di) + w.tau[s + j];  // lambda_j - d_i
        double den;
        if (j == k - 1) den = mt.rhon;
        else den = (j < i) ? (dn[j] - di) : (dn[j + 1] - di);
        prod *= lmd / den;
    }
    for (int q = 16; q; q >>= 1) prod *= __shfl_xor_sync(0xffffffffu, prod, q);
    if (lane == 0) w.zhat[s + i] = copysign(sqrt(fabs(prod)), w.znd[s + i]);
}

// M5 (warp per root j): U row j = normalized (z-hat_i / (d_i - lambda_j))_i.
__global__ void evec_kernel(const MergeDesc* md, int nm, DcArrays w, double* UT, long long ldq, int total) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= total) return;
    const int mi = find_merge(md, nm, gw);
    const MergeDesc g = md[mi];
    const MergeMeta mt = w.meta[mi];
    const int s = g.s, j = gw - s, k = mt.k;
    if (j >= k) return;
    const double* dn = w.dnd + s;
    const double dor = dn[w.org[s + j]], t = w.tau[s + j];
    double* row = UT + (long long)(s + j) * ldq + s;
    double ss = 0.0;
    for (int i = lane; i < k; i += 32) {
        const double u = w.zhat[s + i] / ((dn[i] - dor) - t);
        row[i] = u;
        ss += u * u;
    }
    for (int q = 16; q; q >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, q);
    const double inv = 1.0 / sqrt(ss);
    for (int i = lane; i < k; i += 32) row[i] *= inv;
}

// M7 (thread per output): merge the roots (ascending by construction) with the deflated values into ascending
// order; eigenvalue -> d, eigenvector row -> OUT (eigenvector-major).  Ties: roots first, then deflated by index.
__global__ void assemble_kernel(const MergeDesc* md, int nm, DcArrays w, const double* NEW, const double* QT,
                                double* OUT, long long ldq, double* d) {
    const int gidx = blockIdx.x;  // one CTA per (block row) element
    const int mi = find_merge(md, nm, gidx);
    const MergeDesc g = md[mi];
    const MergeMeta mt = w.meta[mi];
    const int s = g.s, m = g.m, e = gidx - s, k = mt.k, kd = mt.kd;
    __shared__ int rank_s;
    __shared__ double val_s;
    if (threadIdx.x == 0) {
        double v;
        int rank;
        if (e < k) {
            v = w.dnd[s + w.org[s + e]] + w.tau[s + e];
            int c = 0;
            for (int b = 0; b < kd; ++b) c += w.ds[s + w.dfidx[s + b]] < v;
            rank = e + c;
        } else {
            const int b = e - k;
            v = w.ds[s + w.dfidx[s + b]];
            int c = 0;
            for (int j = 0; j < k; ++j) c += (w.dnd[s + w.org[s + j]] + w.tau[s + j]) <= v;
            for (int b2 = 0; b2 < kd; ++b2) {
                const double u = w.ds[s + w.dfidx[s + b2]];
                c += (u < v) || (u == v && b2 < b);
            }
            rank = c;
        }
        rank_s = rank;
        val_s = v;
    }
    __syncthreads();
    const int rank = rank_s;
    const double* src = e < k ? NEW + (long long)(s + e) * ldq + s : QT + (long long)(s + e) * ldq + s;
    double* dst = OUT + (long long)(s + rank) * ldq + s;
    for (int r = threadIdx.x; r < m; r += blockDim.x) dst[r] = src[r];
    if (threadIdx.x == 0) d[s + rank] = val_s;
}

// ------------------------------------------------------------------------------ back-transformation
// V_p (n x 32, rows >= k+1): V[r][t] = 1 at r = k+t+1, A[r][k+t] below, 0 above.
__global__ void build_v_kernel(const double* A, long long lda, int n, int k, int nbp, double* V) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (n - k - 1) * kNB; e += gridDim.x * blockDim.x) {
        const int r = k + 1 + e / kNB, t = e % kNB;
        double v = 0.0;
        if (t < nbp) {
            if (r == k + t + 1) v = 1.0;
            else if (r > k + t + 1) v = A[(long long)r * lda + k + t];
        }
        V[(long long)r * kNB + t] = v;
    }
}

// T (32 x 32 upper triangular, row-major): T(t,t) = tau_t, T(0:t, t) = -tau_t T(0:t, 0:t) G(0:t, t), G = V^T V.
__global__ void build_t_kernel(const double* G, const double* tau, int k, int nbp, double* T) {
    __shared__ double Ts[kNB][kNB + 1], Gs[kNB][kNB + 1];
    const int lane = threadIdx.x;
    for (int r = 0; r < kNB; ++r) { Ts[r][lane] = 0.0; Gs[r][lane] = G[r * kNB + lane]; }
    __syncwarp();
    for (int t = 0; t < nbp; ++t) {
        const double tt = tau[k + t];
        double acc = 0.0;
        if (lane < t)
            for (int c = lane; c < t; ++c) acc += Ts[lane][c] * Gs[c][t];
        __syncwarp();
        if (lane < t) Ts[lane][t] = -tt * acc;
        if (lane == 0) Ts[t][t] = tt;
        __syncwarp();
    }
    for (int r = 0; r < kNB; ++r) T[r * kNB + lane] = Ts[r][lane];
}

void check_launch() { RKFAC_CHECK_LAUNCH(); }

}  // namespace

// ---------------------------------------------------------------------------------------------- host
void DGemmBatch::add(DGemmDesc d) {
    if (d.M <= 0 || d.N <= 0) return;
    d.tiles_n = (int)ceil_div(d.N, kGT);
    d.tile_off = tiles_;
    tiles_ += (int)ceil_div(d.M, kGT) * d.tiles_n;
    descs_.push_back(d);
}

void DGemmBatch::launch(cudaStream_t s) {
    if (descs_.empty()) return;
    if (descs_.size() == 1) {  // by value: fully asynchronous
        DGemmDesc g = descs_[0];
        const int tiles_mn = (int)ceil_div(g.M, kGT) * g.tiles_n;
        // few output tiles and a long K (the skinny products of the back-transformation): split K
        if (tiles_mn < 2 * kNumSMs && g.K >= 512) {
            const int ks = (int)std::min<long long>(ceil_div(g.K, 256), ceil_div(4 * kNumSMs, tiles_mn));
            if (ks > 1) {
                g.ksplit = ks;
                g.kchunk = (int)(ceil_div(ceil_div(g.K, ks), kGK) * kGK);
                g.ksplit = (int)ceil_div(g.K, g.kchunk);
                const size_t bytes = sizeof(double) * (size_t)g.ksplit * g.M * g.N;
                if (part_.bytes < bytes) part_.alloc(bytes);
                g.partial = part_.as<double>();
            }
        }
        dgemm_kernel<<<tiles_mn * g.ksplit, 256, 0, s>>>(nullptr, 0, g);
        count_launch();
        if (g.ksplit > 1) {
            dgemm_reduce_kernel<<<(int)std::min<long long>(ceil_div((long long)g.M * g.N, 256), 1184), 256, 0, s>>>(g);
            count_launch();
        }
        check_launch();
        clear();
        return;
    }
    const size_t bytes = sizeof(DGemmDesc) * descs_.size();
    if (cap_ < bytes) {
        d_.alloc(std::max<size_t>(bytes, 4096));
        cap_ = d_.bytes;
    }
    RKFAC_CUDA(cudaMemcpyAsync(d_.p, descs_.data(), bytes, cudaMemcpyHostToDevice, s));
    dgemm_kernel<<<tiles_, 256, 0, s>>>(d_.as<DGemmDesc>(), (int)descs_.size(), descs_[0]);
    count_launch();
    check_launch();
    // the host vector is the source of an async copy: keep it until the copy is done
    RKFAC_CUDA(cudaStreamSynchronize(s));
    clear();
}

void SymEig::reserve(int n) {
    n_ = n;
    ld_ = (n + 3) / 4 * 4;
    if (n <= cap_n_) return;
    cap_n_ = n;
    const size_t nn = (size_t)n * ld_;
    A_.alloc(sizeof(double) * nn);
    QT_.alloc(sizeof(double) * nn);
    QgT_.alloc(sizeof(double) * nn);
    UT_.alloc(sizeof(double) * nn);
    V_.alloc(sizeof(double) * (size_t)n * kNB);
    W_.alloc(sizeof(double) * (size_t)n * kNB);
    tau_.alloc(sizeof(double) * (n + 1));
    dv_.alloc(sizeof(double) * (n + 1));
    ev_.alloc(sizeof(double) * (n + 1));
    vbuf_.alloc(sizeof(double) * (n + 1));
    ybuf_.alloc(sizeof(double) * (n + 1));
    part_.alloc(sizeof(double) * (kNumSMs + 1) * kPS);
    ws_.alloc(sizeof(double) * (size_t)(n + 1) * 24 + sizeof(MergeMeta) * (n + 1) + 4096);
    meta_.alloc(sizeof(double) * 4096);
    stat_.alloc(64);
}

void SymEig::tridiagonalize(cudaStream_t s) {
    const int n = n_;
    double* A = A_.as<double>();
    int grid = (int)std::min<long long>(kNumSMs, std::max(ceil_div(n, kPanelThreads), ceil_div(n, 32)));
    if (const char* e = std::getenv("RKFAC_SYMEIG_GRID")) grid = std::max<int>((int)ceil_div(n, kPanelThreads), std::atoi(e));
    RKFAC_REQUIRE((long long)grid * kPanelThreads >= n, RKFAC_INVALID_ARGUMENT,
                  "sym_eig: n above the panel kernel's row capacity (37888)");
    for (int k = 0; k < n - 1; k += kNB) {
        const int nbp = std::min(kNB, n - 1 - k);
        PanelArgs a{A, ld_, n, k, nbp, V_.as<double>(), W_.as<double>(), tau_.as<double>(), dv_.as<double>(),
                    ev_.as<double>(), part_.as<double>(), vbuf_.as<double>(), ybuf_.as<double>()};
        void* args[] = {&a};
        RKFAC_CUDA(cudaLaunchCooperativeKernel((const void*)sytrd_panel_kernel, grid, kPanelThreads, args, 0, s));
        count_launch();
        const int k2 = k + nbp;
        if (k2 < n) {  // trailing update A(k2:, k2:) -= V W^T + W V^T (two launches: both write A)
            const double* V = V_.as<double>() + (long long)k2 * kNB;
            const double* W = W_.as<double>() + (long long)k2 * kNB;
            double* C = A + (long long)k2 * ld_ + k2;
            const int m = n - k2;
            gemm_.add(DGemmDesc{m, m, nbp, V, kNB, 1, W, 1, kNB, C, ld_, -1.0, 1.0, 0, 0});
            gemm_.launch(s);
            gemm_.add(DGemmDesc{m, m, nbp, W, kNB, 1, V, 1, kNB, C, ld_, -1.0, 1.0, 0, 0});
            gemm_.launch(s);
        }
    }
    last_diag_kernel<<<1, 1, 0, s>>>(A, ld_, n, dv_.as<double>(), ev_.as<double>());
    count_launch();
    check_launch();
}

void SymEig::divide_and_conquer(cudaStream_t s, bool) {
    const int n = n_;
    const long long ldq = ld_;
    // tree: depth D so that leaves have <= 32 rows; levels of merges bottom-up
    int D = 0;
    while ((n + (1 << D) - 1) / (1 << D) > kLeaf) ++D;
    std::vector<std::vector<MergeDesc>> levels(D);
    std::vector<int> lstart, lsize;
    std::vector<double> e_h(n);
    RKFAC_CUDA(cudaMemcpyAsync(e_h.data(), ev_.p, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    RKFAC_CUDA(cudaStreamSynchronize(s));
    struct Node { int s, m, depth; };
    std::vector<Node> stack{{0, n, 0}};
    std::vector<MergeDesc> all;
    while (!stack.empty()) {
        const Node nd = stack.back();
        stack.pop_back();
        if (nd.depth == D || nd.m <= 1) {
            lstart.push_back(nd.s);
            lsize.push_back(nd.m);
            continue;
        }
        const int m1 = nd.m / 2;
        const double beta = e_h[nd.s + m1 - 1];
        MergeDesc md{nd.s, nd.m, m1, fabs(beta), beta < 0.0 ? -1.0 : 1.0};
        levels[D - 1 - nd.depth].push_back(md);
        all.push_back(md);
        stack.push_back({nd.s, m1, nd.depth + 1});
        stack.push_back({nd.s + m1, nd.m - m1, nd.depth + 1});
    }
    for (auto& l : levels) std::sort(l.begin(), l.end(), [](const MergeDesc& a, const MergeDesc& b) { return a.s < b.s; });
    DevBuf d_all, d_leaf;
    {
        d_all.alloc(sizeof(MergeDesc) * std::max<size_t>(1, all.size()));
        if (!all.empty()) {
            RKFAC_CUDA(cudaMemcpy(d_all.p, all.data(), sizeof(MergeDesc) * all.size(), cudaMemcpyHostToDevice));
            adjust_kernel<<<(int)ceil_div((long long)all.size(), 256), 256, 0, s>>>(d_all.as<MergeDesc>(), (int)all.size(),
                                                                                 dv_.as<double>());
            count_launch();
            check_launch();
        }
        std::vector<int> lb(lstart);
        lb.insert(lb.end(), lsize.begin(), lsize.end());
        d_leaf.alloc(sizeof(int) * lb.size() + 16);
        RKFAC_CUDA(cudaMemcpy(d_leaf.p, lb.data(), sizeof(int) * lb.size(), cudaMemcpyHostToDevice));
    }
    RKFAC_CUDA(cudaMemsetAsync(QT_.p, 0, sizeof(double) * (size_t)n * ldq, s));
    RKFAC_CUDA(cudaMemsetAsync(QgT_.p, 0, sizeof(double) * (size_t)n * ldq, s));
    RKFAC_CUDA(cudaMemsetAsync(UT_.p, 0, sizeof(double) * (size_t)n * ldq, s));
    RKFAC_CUDA(cudaMemsetAsync(stat_.p, 0, 64, s));
    const int nl = (int)lstart.size();
    leaf_kernel<<<(int)ceil_div(nl, kLeafWarps), kLeafWarps * 32, 0, s>>>(d_leaf.as<int>(), d_leaf.as<int>() + nl, nl, dv_.as<double>(),
                                                    ev_.as<double>(), QT_.as<double>(), ldq, stat_.as<int>());
    count_launch();
    check_launch();
    // per-index work arrays carved from ws_
    char* base = static_cast<char*>(ws_.p);
    auto take = [&](size_t bytes) { char* p = base; base += (bytes + 255) & ~size_t(255); return p; };
    DcArrays w;
    w.ds = (double*)take(sizeof(double) * n); w.zs = (double*)take(sizeof(double) * n);
    w.perm = (int*)take(sizeof(int) * n); w.ndidx = (int*)take(sizeof(int) * n); w.dfidx = (int*)take(sizeof(int) * n);
    w.rp = (int*)take(sizeof(int) * n); w.rq = (int*)take(sizeof(int) * n);
    w.rc = (double*)take(sizeof(double) * n); w.rs = (double*)take(sizeof(double) * n);
    w.dnd = (double*)take(sizeof(double) * n); w.znd = (double*)take(sizeof(double) * n);
    w.org = (int*)take(sizeof(int) * n); w.tau = (double*)take(sizeof(double) * n);
    w.zhat = (double*)take(sizeof(double) * n);
    w.meta = (MergeMeta*)take(sizeof(MergeMeta) * (n + 1));
    double* QT = QT_.as<double>();
    double* QgT = QgT_.as<double>();
    double* UT = UT_.as<double>();
    DevBuf d_lvl;
    for (int L = 0; L < D; ++L) {
        const auto& ms = levels[L];
        const int nm = (int)ms.size();
        if (!nm) continue;
        d_lvl.alloc(sizeof(MergeDesc) * nm);
        RKFAC_CUDA(cudaMemcpy(d_lvl.p, ms.data(), sizeof(MergeDesc) * nm, cudaMemcpyHostToDevice));
        const MergeDesc* dm = d_lvl.as<MergeDesc>();
        merge_setup_kernel<<<nm, 1024, 0, s>>>(dm, QT, ldq, dv_.as<double>(), w);
        count_launch();
        check_launch();
        merge_gather_kernel<<<(int)ceil_div(n, 128), 128, 0, s>>>(dm, nm, QT, QgT, ldq, w);
        count_launch();
        check_launch();
        const int warps_blocks = (int)ceil_div((long long)n * 32, 256);
        secular_kernel<<<warps_blocks, 256, 0, s>>>(dm, nm, w, n);
        count_launch();
        zhat_kernel<<<warps_blocks, 256, 0, s>>>(dm, nm, w, n);
        count_launch();
        evec_kernel<<<warps_blocks, 256, 0, s>>>(dm, nm, w, UT, ldq, n);
        count_launch();
        check_launch();
        // eigenvector update NEW (k x m) = U (k x k) * Qnd^T (k x m) per merge (k known after the setup)
        std::vector<MergeMeta> mt(nm);
        RKFAC_CUDA(cudaMemcpyAsync(mt.data(), w.meta, sizeof(MergeMeta) * nm, cudaMemcpyDeviceToHost, s));
        RKFAC_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < nm; ++i) {
            const MergeDesc& g = ms[i];
            const int k = mt[i].k;
            if (k == 0) continue;
            gemm_.add(DGemmDesc{k, g.m, k, UT + (long long)g.s * ldq + g.s, ldq, 1, QT + (long long)g.s * ldq + g.s, ldq,
                                1, QgT + (long long)g.s * ldq + g.s, ldq, 1.0, 0.0, 0, 0});
        }
        gemm_.launch(s);
        assemble_kernel<<<n, 128, 0, s>>>(dm, nm, w, QgT, QT, UT, ldq, dv_.as<double>());
        count_launch();
        check_launch();
        std::swap(QT, UT);  // the assembled eigenvectors are the next level's input
    }
    if (QT != QT_.as<double>()) std::swap(QT_, UT_);
}

void SymEig::back_transform(cudaStream_t s) {
    const int n = n_;
    const long long ldq = ld_;
    double* X = QT_.as<double>();  // eigenvectors of T, eigenvector-major: X <- X B_p^T, p from last to first
    double* V = V_.as<double>();
    double* G = ybuf_.as<double>();  // 32 x 32 Gram (n >= 1024 floats of scratch needed: use W_ instead when small)
    double* T = W_.as<double>();
    double* Y = UT_.as<double>();    // n x 32
    double* Y2 = QgT_.as<double>();  // n x 32
    DevBuf gbuf(sizeof(double) * kNB * kNB * 2);
    G = gbuf.as<double>();
    T = G + kNB * kNB;
    const int npan = (n - 1 + kNB - 1) / kNB;
    for (int p = npan - 1; p >= 0; --p) {
        const int k = p * kNB;
        const int nbp = std::min(kNB, n - 1 - k);
        if (nbp <= 0) continue;
        const int mrows = n - k - 1;
        build_v_kernel<<<(int)std::min<long long>(ceil_div((long long)mrows * kNB, 256), 1184), 256, 0, s>>>(
            A_.as<double>(), ld_, n, k, nbp, V);
        count_launch();
        const double* Vk = V + (long long)(k + 1) * kNB;
        gemm_.add(DGemmDesc{kNB, kNB, mrows, Vk, 1, kNB, Vk, kNB, 1, G, kNB, 1.0, 0.0, 0, 0});  // G = V^T V
        gemm_.launch(s);
        build_t_kernel<<<1, 32, 0, s>>>(G, tau_.as<double>(), k, nbp, T);
        count_launch();
        gemm_.add(DGemmDesc{n, kNB, mrows, X + (k + 1), ldq, 1, Vk, kNB, 1, Y, kNB, 1.0, 0.0, 0, 0});    // Y = X V
        gemm_.launch(s);
        gemm_.add(DGemmDesc{n, kNB, kNB, Y, kNB, 1, T, 1, kNB, Y2, kNB, 1.0, 0.0, 0, 0});               // Y2 = Y T^T
        gemm_.launch(s);
        gemm_.add(DGemmDesc{n, mrows, kNB, Y2, kNB, 1, Vk, 1, kNB, X + (k + 1), ldq, -1.0, 1.0, 0, 0});  // X -= Y2 V^T
        gemm_.launch(s);
    }
    check_launch();
}

double SymEig::run(const float* S, long long lds, int n, float* P, long long ldp, float* dvals, double* dvals64,
                   cudaStream_t s) {
    RKFAC_REQUIRE(n >= 1, RKFAC_INVALID_ARGUMENT, "sym_eig: empty matrix");
    reserve(n);
    RKFAC_CUDA(cudaMemsetAsync(stat_.p, 0, 64, s));
    widen_kernel<<<(int)std::min<long long>(ceil_div((long long)n * n, 256), 4096), 256, 0, s>>>(
        S, lds, n, A_.as<double>(), ld_, stat_.as<unsigned long long>() + 1);
    count_launch();
    check_launch();
    unsigned long long st[3] = {0, 0, 0};
    RKFAC_CUDA(cudaMemcpyAsync(st, stat_.p, sizeof(st), cudaMemcpyDeviceToHost, s));
    RKFAC_CUDA(cudaStreamSynchronize(s));
    double asym, amax;
    std::memcpy(&asym, &st[1], 8);
    std::memcpy(&amax, &st[2], 8);
    const double rel = asym / std::max(1.0, amax);
    // RKFAC_SYMEIG_TIMING=1: phase times (CUDA events) to stderr
    static const bool timing = std::getenv("RKFAC_SYMEIG_TIMING") != nullptr;
    cudaEvent_t ev[4] = {};
    if (timing)
        for (auto& e : ev) { RKFAC_CUDA(cudaEventCreate(&e)); }
    if (timing) RKFAC_CUDA(cudaEventRecord(ev[0], s));
    if (n > 1) tridiagonalize(s);
    else {
        RKFAC_CUDA(cudaMemcpyAsync(dv_.p, A_.p, sizeof(double), cudaMemcpyDeviceToDevice, s));
        RKFAC_CUDA(cudaMemsetAsync(ev_.p, 0, sizeof(double), s));
    }
    if (timing) RKFAC_CUDA(cudaEventRecord(ev[1], s));
    divide_and_conquer(s, true);
    if (timing) RKFAC_CUDA(cudaEventRecord(ev[2], s));
    int fail = 0;
    RKFAC_CUDA(cudaMemcpyAsync(&fail, stat_.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    RKFAC_CUDA(cudaStreamSynchronize(s));
    RKFAC_REQUIRE(!fail, RKFAC_NO_CONVERGENCE, "sym_eig: QL iteration did not converge (eig.hpp:147-148)");
    if (n > 1) back_transform(s);
    if (timing) {
        RKFAC_CUDA(cudaEventRecord(ev[3], s));
        RKFAC_CUDA(cudaEventSynchronize(ev[3]));
        float t[3];
        for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
        std::fprintf(stderr, "symeig n=%d: tridiagonalisation %.2f ms, divide and conquer %.2f ms, back-transformation "
                     "%.2f ms\n", n, t[0], t[1], t[2]);
        for (auto& e : ev) cudaEventDestroy(e);
    }
    dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
    output_kernel<<<grid, dim3(32, 8), 0, s>>>(QT_.as<double>(), ld_, dv_.as<double>(), n, P, ldp, dvals, dvals64);
    count_launch();
    check_launch();
    return rel;
}

}  // namespace rkfac_b200
