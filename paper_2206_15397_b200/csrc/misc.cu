// misc.cu -- small elementwise kernels of the path: Gaussian test matrix, eigenvalue post-processing, damping
// brackets, transposes.
#include <cmath>

#include "kernels.cuh"

namespace rkfac_b200 {

uint64_t& launch_counter() {
    static uint64_t c = 0;
    return c;
}

namespace {

__device__ __forceinline__ int find_desc(const OmegaDesc* descs, int n, long long e) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (descs[mid].offset <= e) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// K1: rng.hpp:59-63 sample_gaussian, every factor in one launch; FP64 transcendental math, FP32 store.
// Threads walk Omega^T (w x d) in storage order: consecutive threads -> consecutive i -> coalesced stores.
__global__ void omega_kernel(const OmegaDesc* __restrict__ descs, int n, long long total, int mode, uint64_t root,
                             uint64_t step, const uint64_t* __restrict__ seed_src) {
    if (seed_src) {  // a captured step: (root, step) are read at replay time (rkfac_plan_set_step_seed)
        root = seed_src[0];
        step = seed_src[1];
    }
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int f = find_desc(descs, n, e);
        const OmegaDesc& od = descs[f];
        const long long local = e - od.offset;
        const int j = (int)(local / od.d), i = (int)(local - (long long)j * od.d);
        const uint64_t seed = mode ? substream(root, step, od.tag) : od.seed;
        const uint64_t ctr = od.ctr0 + 2ULL * ((uint64_t)i * (uint64_t)od.w + (uint64_t)j);
        const float g = (float)gaussian_at(seed, ctr);
        const long long o = od.rowmajor ? (long long)i * od.ld + j : (long long)j * od.ld + i;
        od.out[o] = g;
        if (od.out_lo) od.out_lo[o] = g - __uint_as_float(__float_as_uint(g) & 0xFFFFE000u);
    }
}

__global__ void post_kernel(const PostDesc* __restrict__ descs) {
    const PostDesc& pd = descs[blockIdx.x];
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    if (pd.method == RKFAC_SREVD) {
        for (int k = threadIdx.x; k < pd.r; k += blockDim.x) {
            pd.dvals[k] = (float)fmax(0.0, pd.evals[k]);
            if (pd.scale) pd.scale[k] = 1.f;
            if (pd.flags) pd.flags[k] = 0;
        }
    } else {
        const double smax = pd.r > 0 ? sqrt(fmax(0.0, pd.evals[0])) : 0.0;
        // FP32 Gram => singular values below ~1e-6*smax carry no information (the reference uses 1e-13 in FP64,
        // eig.hpp:258); such modes have d ~ 0, so only their basis direction (completed below) is affected.
        const double tiny = fmax(smax * 1e-6, 1e-300);
        for (int k = threadIdx.x; k < pd.r; k += blockDim.x) {
            const double s = sqrt(fmax(0.0, pd.evals[k]));
            const bool zero = !(s > tiny);
            pd.dvals[k] = zero ? 0.f : (float)s;
            pd.scale[k] = zero ? 0.f : (float)(1.0 / s);
            pd.flags[k] = zero ? 1 : 0;
            if (zero) any = 1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && pd.nflags) *pd.nflags = any;
}

__global__ void bracket_kernel(const BracketDesc* __restrict__ descs, double lambda) {
    const BracketDesc& bd = descs[blockIdx.x];
    for (int k = threadIdx.x; k < bd.r; k += blockDim.x) {
        const double d = (double)bd.dvals[k];
        bd.out[k] = (float)(-d / (lambda * (lambda + d)));
    }
}

// One descriptor per blockIdx.y; work items are (row, 2 KB chunk) pairs spread over the warps of the descriptor's
// blocks, four 16-byte loads in flight per lane (a few long rows -- a 512 x 4609 gradient -- still fill the GPU).
__global__ void copy_kernel(const CopyDesc* __restrict__ descs) {
    const CopyDesc cd = descs[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const bool vec = ((reinterpret_cast<uintptr_t>(cd.src) | reinterpret_cast<uintptr_t>(cd.dst) |
                       (uintptr_t)(cd.lds * 4) | (uintptr_t)(cd.ldd * 4)) & 15) == 0;
    const int c4 = vec ? cd.cols / 4 : 0;
    // chunks: 2 KB float4 chunks, then 1 KB scalar chunks for the rest (a whole unaligned row), 8 loads in flight
    const int nvec = (c4 + 127) / 128, nsc = (cd.cols - 4 * c4 + 255) / 256, chunks = nvec + nsc;
    const long long items = (long long)cd.rows * chunks;
    for (long long it = blockIdx.x * wpb + warp; it < items; it += (long long)gridDim.x * wpb) {
        const int r = (int)(it / chunks), ch = (int)(it - (long long)r * chunks);
        const float* s = cd.src + (long long)r * cd.lds;
        float* d = cd.dst + (long long)r * cd.ldd;
        if (ch >= nvec) {
            const int cb = 4 * c4 + (ch - nvec) * 256 + lane;
            float xs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cb + 32 * u < cd.cols) xs[u] = s[cb + 32 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cb + 32 * u < cd.cols) d[cb + 32 * u] = xs[u];
            continue;
        }
        const int c0 = ch * 128 + lane;
        float4 xs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (c0 + 32 * u < c4) xs[u] = reinterpret_cast<const float4*>(s)[c0 + 32 * u];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (c0 + 32 * u < c4) reinterpret_cast<float4*>(d)[c0 + 32 * u] = xs[u];
    }
}

__global__ void scale_kernel(float* __restrict__ x, long long ld, int rows, int cols, float a) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)rows * cols;
         e += (long long)gridDim.x * blockDim.x) {
        const long long r = e / cols, c = e - r * cols;
        x[r * ld + c] *= a;
    }
}

__global__ void transpose_kernel(const float* __restrict__ in, long long ldi, int rows, int cols,
                                 float* __restrict__ out, long long ldo) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int r = by + y, c = bx + threadIdx.x;
        if (r < rows && c < cols) tile[y][threadIdx.x] = in[(long long)r * ldi + c];
    }
    __syncthreads();
    for (int y = threadIdx.y; y < 32; y += blockDim.y) {
        const int c = bx + y, r = by + threadIdx.x;
        if (r < rows && c < cols) out[(long long)c * ldo + r] = tile[threadIdx.x][y];
    }
}

}  // namespace

void launch_omega(const OmegaDesc* d_descs, int nfactors, long long total, int mode, uint64_t root, uint64_t step,
                  cudaStream_t s, const uint64_t* seed_src) {
    if (total == 0) return;
    const int blocks = (int)std::min<long long>(ceil_div(total, 256), kNumSMs * 16);
    omega_kernel<<<blocks, 256, 0, s>>>(d_descs, nfactors, total, mode, root, step, seed_src);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_post(const PostDesc* d_descs, int nfactors, cudaStream_t s) {
    if (nfactors == 0) return;
    post_kernel<<<nfactors, 256, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_bracket(const BracketDesc* d_descs, int n, double lambda, cudaStream_t s) {
    if (n == 0) return;
    bracket_kernel<<<n, 256, 0, s>>>(d_descs, lambda);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_copy(const CopyDesc* d_descs, int n, long long total, cudaStream_t s) {
    if (total == 0 || n == 0) return;
    // ~8 row-blocks of 8 warps per SM over all descriptors; blocks past a descriptor's rows exit at once
    const int bx = (int)std::max<long long>(1, std::min<long long>(512, ceil_div(kNumSMs * 8, n)));
    copy_kernel<<<dim3(bx, n), 256, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

__global__ void symmetrize_kernel(const SymDesc* __restrict__ descs, int n, long long total) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (descs[mid].offset <= e) lo = mid; else hi = mid - 1;
        }
        const SymDesc sd = descs[lo];
        // strictly-lower pair index -> (i, j), i > j: i = floor((1 + sqrt(1 + 8q)) / 2)
        const long long q = e - sd.offset;
        long long i = (long long)((1.0 + sqrt(1.0 + 8.0 * (double)q)) * 0.5);
        while (i * (i - 1) / 2 > q) --i;
        while ((i + 1) * i / 2 <= q) ++i;
        const long long j = q - i * (i - 1) / 2;
        float* a = sd.x + i * sd.ld + j;
        float* b = sd.x + j * sd.ld + i;
        const float v = 0.5f * (*a + *b);
        *a = v;
        *b = v;
    }
}

void launch_symmetrize(const SymDesc* d_descs, int n, long long total, cudaStream_t s) {
    if (total == 0 || n == 0) return;
    const int blocks = (int)std::min<long long>(ceil_div(total, 256), kNumSMs * 8);
    symmetrize_kernel<<<blocks, 256, 0, s>>>(d_descs, n, total);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_scale(float* x, long long ld, int rows, int cols, float a, cudaStream_t s) {
    if (rows == 0 || cols == 0) return;
    const int blocks = (int)std::min<long long>(ceil_div((long long)rows * cols, 256), kNumSMs * 8);
    scale_kernel<<<blocks, 256, 0, s>>>(x, ld, rows, cols, a);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

void launch_transpose(const float* in, long long ldi, int rows, int cols, float* out, long long ldo, cudaStream_t s) {
    if (rows == 0 || cols == 0) return;
    dim3 grid((unsigned)ceil_div(cols, 32), (unsigned)ceil_div(rows, 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(in, ldi, rows, cols, out, ldo);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
