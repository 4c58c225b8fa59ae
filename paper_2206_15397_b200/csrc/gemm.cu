// gemm.cu -- grouped SIMT GEMM (FP32 / FP64-accumulate) with fused epilogues; see gemm.cuh.
//
// This is the general-purpose engine behind every contraction of the path whose shape or precision does not
// go to the tcgen05 kernels (gram/trsm products of the orthonormalisation, the w x w cores, the basis lift and
// the apply stage).  128x128x16 tiles, 8x8 register micro-tiles split in 4x4 quadrants (conflict-free LDS.128),
// register-staged double buffering.
#include <algorithm>

#include "gemm.cuh"

namespace rkfac_b200 {

namespace {

template <class T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };

template <class TA, class TB, class TC, class TACC, int BM, int BN, int BK, int TM, int TN>
struct GemmCfg {
    static constexpr int NTX = BN / TN;
    static constexpr int NTY = BM / TM;
    static constexpr int NT = NTX * NTY;
    static constexpr int A_PER = BM * BK / NT;
    static constexpr int B_PER = BN * BK / NT;
    static_assert(A_PER * NT == BM * BK, "A tile must divide");
    static_assert(B_PER * NT == BN * BK, "B tile must divide");
};

__device__ __forceinline__ int find_problem(const int* prefix, int n, int tile) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// Upper-triangle tile enumeration for sym problems: l -> (tm, tn) with tm <= tn, row-major over tm.
__device__ __forceinline__ void sym_tile(int l, int T, int& tm, int& tn) {
    int row = 0, remaining = l;
    while (remaining >= T - row) { remaining -= T - row; ++row; }
    tm = row;
    tn = row + remaining;
}

template <class T>
__device__ __forceinline__ double as_double(T v) { return static_cast<double>(v); }

template <class TC>
__device__ __forceinline__ void epilogue_store(const GemmDesc& d, int m, int n, double v) {
    double out = d.alpha * v;
    if (d.rs) out *= static_cast<double>(d.rs[m]);
    if (d.cs) out *= static_cast<double>(d.cs[n]);
    const long long ic = d.tc ? (long long)n * d.ldc + m : (long long)m * d.ldc + n;
    if (d.beta != 0.0) {
        const long long ii = d.tc ? (long long)n * d.ldcin + m : (long long)m * d.ldcin + n;
        out += d.beta * as_double(static_cast<const TC*>(d.Cin)[ii]);
    }
    if (d.gamma != 0.0) {
        const long long id = d.tc ? (long long)n * d.ldd + m : (long long)m * d.ldd + n;
        out += d.gamma * static_cast<double>(d.D[id]);
    }
    static_cast<TC*>(d.C)[ic] = static_cast<TC>(out);
}

// FP32 epilogue keeps FP32 arithmetic (the accumulate precision of the F32 kind).
template <>
__device__ __forceinline__ void epilogue_store<float>(const GemmDesc& d, int m, int n, double vd) {
    float v = static_cast<float>(vd);
    float out = static_cast<float>(d.alpha) * v;
    if (d.rs) out *= d.rs[m];
    if (d.cs) out *= d.cs[n];
    const long long ic = d.tc ? (long long)n * d.ldc + m : (long long)m * d.ldc + n;
    if (d.beta != 0.0) {
        const long long ii = d.tc ? (long long)n * d.ldcin + m : (long long)m * d.ldcin + n;
        out = fmaf(static_cast<float>(d.beta), static_cast<const float*>(d.Cin)[ii], out);
    }
    if (d.gamma != 0.0) {
        const long long id = d.tc ? (long long)n * d.ldd + m : (long long)m * d.ldd + n;
        out = fmaf(static_cast<float>(d.gamma), d.D[id], out);
    }
    static_cast<float*>(d.C)[ic] = out;
}

template <class TA, class TB, class TC, class TACC, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__(GemmCfg<TA, TB, TC, TACC, BM, BN, BK, TM, TN>::NT)
grouped_gemm_kernel(const GemmDesc* __restrict__ descs, const int* __restrict__ prefix, int nprob) {
    using Cfg = GemmCfg<TA, TB, TC, TACC, BM, BN, BK, TM, TN>;
    constexpr int NT = Cfg::NT, NTX = Cfg::NTX;
    __shared__ __align__(16) TACC As[2][BK][BM];
    __shared__ __align__(16) TACC Bs[2][BK][BN];

    const int tile = blockIdx.x;
    const int p = find_problem(prefix, nprob, tile);
    const GemmDesc& d = descs[p];
    int local = tile - prefix[p];
    const int tiles_mn = d.sym ? d.tiles_m * (d.tiles_m + 1) / 2 : d.tiles_m * d.tiles_n;
    const int slice = local / tiles_mn;
    local -= slice * tiles_mn;
    int tm, tn;
    if (d.sym) sym_tile(local, d.tiles_m, tm, tn);
    else { tm = local / d.tiles_n; tn = local - tm * d.tiles_n; }
    const int m0 = tm * BM, n0 = tn * BN;

    // K range of this slice (slices are multiples of BK; fixed by the descriptor => deterministic).
    const int kchunks = (d.K + BK - 1) / BK;
    const int per = (kchunks + d.ksplit - 1) / d.ksplit;
    const int kb_begin = slice * per;
    const int kb_end = min(kchunks, kb_begin + per);

    const TA* __restrict__ A = static_cast<const TA*>(d.A);
    const TB* __restrict__ B = static_cast<const TB*>(d.B);
    const int tid = threadIdx.x;
    const int tx = tid % NTX, ty = tid / NTX;

    TACC ra[Cfg::A_PER], rb[Cfg::B_PER];
    auto load_regs = [&](int kb) {
        const int k0 = kb * BK;
#pragma unroll
        for (int i = 0; i < Cfg::A_PER; ++i) {
            const int idx = tid + i * NT;
            int mm, kk;
            if (d.ta) { mm = idx % BM; kk = idx / BM; } else { kk = idx % BK; mm = idx / BK; }
            const int gm = m0 + mm, gk = k0 + kk;
            TACC v = TACC(0);
            if (gm < d.M && gk < d.K)
                v = static_cast<TACC>(d.ta ? A[(long long)gk * d.lda + gm] : A[(long long)gm * d.lda + gk]);
            ra[i] = v;
        }
#pragma unroll
        for (int i = 0; i < Cfg::B_PER; ++i) {
            const int idx = tid + i * NT;
            int nn, kk;
            if (d.tb) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            const int gn = n0 + nn, gk = k0 + kk;
            TACC v = TACC(0);
            if (gn < d.N && gk < d.K)
                v = static_cast<TACC>(d.tb ? B[(long long)gn * d.ldb + gk] : B[(long long)gk * d.ldb + gn]);
            rb[i] = v;
        }
    };
    auto store_smem = [&](int buf) {
#pragma unroll
        for (int i = 0; i < Cfg::A_PER; ++i) {
            const int idx = tid + i * NT;
            int mm, kk;
            if (d.ta) { mm = idx % BM; kk = idx / BM; } else { kk = idx % BK; mm = idx / BK; }
            As[buf][kk][mm] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < Cfg::B_PER; ++i) {
            const int idx = tid + i * NT;
            int nn, kk;
            if (d.tb) { kk = idx % BK; nn = idx / BK; } else { nn = idx % BN; kk = idx / BN; }
            Bs[buf][kk][nn] = rb[i];
        }
    };

    // Row/col ownership: TM/4 (TN/4) quadrants spaced BM/(TM/4) apart.
    constexpr int QM = TM / 4, QN = TN / 4;
    constexpr int SM = BM / QM, SN = BN / QN;
    TACC acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = TACC(0);

    if (kb_begin < kb_end) {
        load_regs(kb_begin);
        store_smem(0);
        __syncthreads();
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            const int buf = (kb - kb_begin) & 1;
            const bool more = kb + 1 < kb_end;
            if (more) load_regs(kb + 1);
#pragma unroll
            for (int kk = 0; kk < BK; ++kk) {
                TACC a[TM], b[TN];
#pragma unroll
                for (int q = 0; q < QM; ++q)
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[q * 4 + i] = As[buf][kk][q * SM + ty * 4 + i];
#pragma unroll
                for (int q = 0; q < QN; ++q)
#pragma unroll
                    for (int j = 0; j < 4; ++j) b[q * 4 + j] = Bs[buf][kk][q * SN + tx * 4 + j];
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
            if (more) store_smem(buf ^ 1);
            __syncthreads();
        }
    }

    // Epilogue.
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int m = m0 + (i / 4) * SM + ty * 4 + (i % 4);
        if (m >= d.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + (j / 4) * SN + tx * 4 + (j % 4);
            if (n >= d.N) continue;
            if (d.ksplit > 1) {
                static_cast<TACC*>(d.partial)[(long long)slice * d.M * d.N + (long long)m * d.N + n] = acc[i][j];
                continue;
            }
            epilogue_store<TC>(d, m, n, as_double(acc[i][j]));
            if (d.sym && tm != tn) epilogue_store<TC>(d, n, m, as_double(acc[i][j]));
        }
    }
}

// Split-K reduction: fixed slice order => bitwise reproducible.
template <class TC, class TACC>
__global__ void splitk_reduce_kernel(const GemmDesc* __restrict__ descs, int nprob) {
    for (int p = 0; p < nprob; ++p) {
        const GemmDesc& d = descs[p];
        if (d.ksplit <= 1) continue;
        const long long mn = (long long)d.M * d.N;
        const TACC* part = static_cast<const TACC*>(d.partial);
        for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mn;
             e += (long long)gridDim.x * blockDim.x) {
            TACC s = part[e];
            for (int k = 1; k < d.ksplit; ++k) s += part[(long long)k * mn + e];
            const int m = (int)(e / d.N), n = (int)(e - (long long)m * d.N);
            epilogue_store<TC>(d, m, n, as_double(s));
        }
    }
}

}  // namespace

int choose_ksplit(int M, int N, int K, int bm, int bn) {
    const int tiles = (int)(ceil_div(M, bm) * ceil_div(N, bn));
    const int kchunks = (int)ceil_div(K, 16);
    // Aim for >= 16 CTAs per problem on skinny outputs, each slice >= 16 K-chunks.
    int s = 1;
    while (tiles * s < 16 && kchunks / (2 * s) >= 16) s *= 2;
    return s;
}

int GemmBatch::add(GemmDesc d) {
    descs_.push_back(d);
    return (int)descs_.size() - 1;
}

double GemmBatch::flops() const {
    double f = 0;
    for (const auto& d : descs_) f += 2.0 * d.M * (double)d.N * d.K * (d.sym ? 0.5 : 1.0);
    return f;
}

void GemmBatch::finalize() {
    if (kind_ == GemmKind::F32) { bm_ = 128; bn_ = 128; } else { bm_ = 64; bn_ = 64; }
    std::vector<int> prefix;
    size_t partial_elems = 0;
    total_tiles_ = 0;
    for (auto& d : descs_) {
        d.tiles_m = (int)ceil_div(d.M, bm_);
        d.tiles_n = (int)ceil_div(d.N, bn_);
        if (d.sym) RKFAC_REQUIRE(d.M == d.N && d.ksplit == 1, RKFAC_INVALID_ARGUMENT, "sym gemm needs M==N, no split");
        const int mn = d.sym ? d.tiles_m * (d.tiles_m + 1) / 2 : d.tiles_m * d.tiles_n;
        d.tiles_total = (d.M > 0 && d.N > 0) ? mn * d.ksplit : 0;
        prefix.push_back(total_tiles_);
        total_tiles_ += d.tiles_total;
        if (d.ksplit > 1) partial_elems += (size_t)d.ksplit * d.M * d.N;
    }
    const size_t acc_bytes = (kind_ == GemmKind::F32) ? 4 : 8;
    partials_.alloc(partial_elems * acc_bytes);
    size_t off = 0;
    for (auto& d : descs_) {
        if (d.ksplit > 1) {
            d.partial = static_cast<char*>(partials_.p) + off * acc_bytes;
            off += (size_t)d.ksplit * d.M * d.N;
        }
    }
    d_descs_.alloc(sizeof(GemmDesc) * std::max<size_t>(1, descs_.size()));
    d_prefix_.alloc(sizeof(int) * std::max<size_t>(1, prefix.size()));
    if (!descs_.empty()) {
        RKFAC_CUDA(cudaMemcpy(d_descs_.p, descs_.data(), sizeof(GemmDesc) * descs_.size(), cudaMemcpyHostToDevice));
        RKFAC_CUDA(cudaMemcpy(d_prefix_.p, prefix.data(), sizeof(int) * prefix.size(), cudaMemcpyHostToDevice));
    }
}

void GemmBatch::launch(cudaStream_t s) const {
    if (total_tiles_ == 0) return;
    const int n = (int)descs_.size();
    const auto* dd = d_descs_.as<GemmDesc>();
    const auto* pp = d_prefix_.as<int>();
    bool any_split = false;
    for (const auto& d : descs_) any_split |= d.ksplit > 1;
    switch (kind_) {
        case GemmKind::F32:
            grouped_gemm_kernel<float, float, float, float, 128, 128, 16, 8, 8><<<total_tiles_, 256, 0, s>>>(dd, pp, n);
            count_launch();
            if (any_split) { splitk_reduce_kernel<float, float><<<296, 256, 0, s>>>(dd, n); count_launch(); }
            break;
        case GemmKind::F32_ACC64:
            grouped_gemm_kernel<float, float, double, double, 64, 64, 16, 4, 4><<<total_tiles_, 256, 0, s>>>(dd, pp, n);
            count_launch();
            if (any_split) { splitk_reduce_kernel<double, double><<<296, 256, 0, s>>>(dd, n); count_launch(); }
            break;
        case GemmKind::F64_F32:
            grouped_gemm_kernel<double, float, float, double, 64, 64, 16, 4, 4><<<total_tiles_, 256, 0, s>>>(dd, pp, n);
            count_launch();
            if (any_split) { splitk_reduce_kernel<float, double><<<296, 256, 0, s>>>(dd, n); count_launch(); }
            break;
    }
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
