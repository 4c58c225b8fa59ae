// dmma.cu -- FP64 tensor-core (DMMA m8n8k4) Gram and triangular products of the first orthonormalisation.
//
// 128 threads per CTA, 64 x 64 output tile, 2 x 2 warps of 32 x 32 (4 x 4 DMMA tiles of 8 x 8 per warp, 32 FP64
// accumulators per thread).  Operands stream through a 3-stage cp.async pipeline in 32-wide K chunks.
// Fragment layouts of mma.m8n8k4.f64 (g = lane / 4, t = lane % 4):  A(g, t), B(t, g), C(g, 2t + {0,1}).
// Shared-memory row pitches are chosen so every fragment load of a warp touches 32 distinct banks:
//   K-major float rows  pitch 36 floats:  bank = 4g + t
//   K-major double rows pitch 36 doubles: bank = 8g + 2t (+1)
//   N-major float rows  pitch 72 floats:  bank = 8t + g
#include "dmma.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kTile = 64;
constexpr int kBK = 32;
constexpr int kStages = 3;
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ void sym_tile(int l, int T, int& tm, int& tn) {
    int row = 0, remaining = l;
    while (remaining >= T - row) { remaining -= T - row; ++row; }
    tm = row;
    tn = row + remaining;
}

template <class D>
__device__ __forceinline__ int find_by_tile(const D* descs, int n, int tile) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (descs[mid].tile_offset <= tile) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------------------------------------------ Gram
constexpr int kGP = 36;  // float pitch of a K-major 64 x 32 stage
struct GramSmem {
    float a[kStages][kTile][kGP];
    float b[kStages][kTile][kGP];
};

__global__ void __launch_bounds__(kThreads) gram64_kernel(const Gram64Desc* __restrict__ descs, int nprob) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GramSmem& sm = *reinterpret_cast<GramSmem*>(smem_raw);
    const int p = find_by_tile(descs, nprob, blockIdx.x);
    const Gram64Desc& D = descs[p];
    const int ntri = D.tiles_m * (D.tiles_m + 1) / 2;
    int local = blockIdx.x - D.tile_offset;
    const int slice = local / ntri;
    local -= slice * ntri;
    int tm, tn;
    sym_tile(local, D.tiles_m, tm, tn);
    const bool diag = tm == tn;
    const int m0 = tm * kTile, n0 = tn * kTile;
    const int kchunks = (D.d + kBK - 1) / kBK;
    const int per = (kchunks + D.ksplit - 1) / D.ksplit;
    const int kb0 = slice * per, kb1 = min(kchunks, kb0 + per);
    const int nk = max(0, kb1 - kb0);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;

    auto load_stage = [&](int st, int kb) {
        const int k0 = kb * kBK;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = tid + i * kThreads;
            const int row = c >> 3, col = (c & 7) * 4;
            const int k = k0 + col;
            const int kbytes = max(0, min(16, (D.d - k) * 4));
            {
                const int r = m0 + row;
                const bool ok = r < D.w && kbytes > 0;
                cp_async16(&sm.a[st][row][col], ok ? (const void*)(D.T + (long long)r * D.ldt + k) : (const void*)D.T,
                           ok ? kbytes : 0);
            }
            if (!diag) {
                const int r = n0 + row;
                const bool ok = r < D.w && kbytes > 0;
                cp_async16(&sm.b[st][row][col], ok ? (const void*)(D.T + (long long)r * D.ldt + k) : (const void*)D.T,
                           ok ? kbytes : 0);
            }
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load_stage(s, kb0 + s);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nxt = it + kStages - 1;
            if (nxt < nk) load_stage(nxt % kStages, kb0 + nxt);
            cp_async_commit();
        }
        const int st = it % kStages;
        const float(*As)[kGP] = sm.a[st];
        const float(*Bs)[kGP] = diag ? sm.a[st] : sm.b[st];
#pragma unroll
        for (int ks = 0; ks < kBK / 4; ++ks) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = (double)As[wm * 32 + i * 8 + g][ks * 4 + t];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = (double)Bs[wn * 32 + j * 8 + g][ks * 4 + t];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();

    double* out = D.ksplit > 1 ? D.partial + (long long)slice * D.w * D.w : D.G;
    const long long ld = D.ksplit > 1 ? D.w : D.ldg;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + wm * 32 + i * 8 + g;
        if (m >= D.w) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int n = n0 + wn * 32 + j * 8 + 2 * t + e;
                if (n >= D.w) continue;
                out[(long long)m * ld + n] = acc[i][j][e];
                if (D.ksplit == 1 && !diag) out[(long long)n * ld + m] = acc[i][j][e];
            }
    }
}

// Split-K reduction in fixed slice order over the upper triangle (m <= n always lies in a computed tile), mirrored.
__global__ void gram64_reduce_kernel(const Gram64Desc* __restrict__ descs, int nprob, long long total) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = nprob - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (descs[mid].elem_offset <= e) lo = mid; else hi = mid - 1;
        }
        const Gram64Desc& D = descs[lo];
        if (D.ksplit <= 1) continue;
        const long long local = e - D.elem_offset;
        const int m = (int)(local / D.w), n = (int)(local - (long long)m * D.w);
        if (m > n) continue;
        const long long ww = (long long)D.w * D.w;
        double s = D.partial[local];
        for (int k = 1; k < D.ksplit; ++k) s += D.partial[k * ww + local];
        D.G[(long long)m * D.ldg + n] = s;
        D.G[(long long)n * D.ldg + m] = s;
    }
}

// -------------------------------------------------------------------------------------------- Triangular
constexpr int kAP = 36;  // double pitch of the K-major 64 x 32 Linv stage
constexpr int kBP = 72;  // float pitch of the N-major 32 x 64 Y^T stage
struct TriSmem {
    double a[kStages][kTile][kAP];
    float b[kStages][kBK][kBP];
};

__global__ void __launch_bounds__(kThreads) tri64_kernel(const Tri64Desc* __restrict__ descs, int nprob) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TriSmem& sm = *reinterpret_cast<TriSmem*>(smem_raw);
    const int p = find_by_tile(descs, nprob, blockIdx.x);
    const Tri64Desc& D = descs[p];
    const int local = blockIdx.x - D.tile_offset;
    const int tm = local / D.tiles_n, tn = local - tm * D.tiles_n;
    const int m0 = tm * kTile, n0 = tn * kTile;
    const int kmax = min(D.w, m0 + kTile);  // Linv(m, k) = 0 for k > m
    const int nk = (kmax + kBK - 1) / kBK;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp >> 1, wn = warp & 1;

    auto load_stage = [&](int st, int kb) {
        const int k0 = kb * kBK;
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // Linv: 64 rows x 32 doubles = 1024 16-byte chunks
            const int c = tid + i * kThreads;
            const int row = c >> 4, col = (c & 15) * 2;
            const int r = m0 + row, k = k0 + col;
            const int kbytes = max(0, min(16, (D.w - k) * 8));
            const bool ok = r < D.w && kbytes > 0;
            cp_async16(&sm.a[st][row][col], ok ? (const void*)(D.L + (long long)r * D.ldl + k) : (const void*)D.L,
                       ok ? kbytes : 0);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // Y^T: 32 rows x 64 floats = 512 chunks
            const int c = tid + i * kThreads;
            const int row = c >> 4, col = (c & 15) * 4;
            const int k = k0 + row, n = n0 + col;
            const int nbytes = max(0, min(16, (D.d - n) * 4));
            const bool ok = k < D.w && nbytes > 0;
            cp_async16(&sm.b[st][row][col], ok ? (const void*)(D.Yt + (long long)k * D.ldy + n) : (const void*)D.Yt,
                       ok ? nbytes : 0);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nxt = it + kStages - 1;
            if (nxt < nk) load_stage(nxt % kStages, nxt);
            cp_async_commit();
        }
        const int st = it % kStages;
#pragma unroll
        for (int ks = 0; ks < kBK / 4; ++ks) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sm.a[st][wm * 32 + i * 8 + g][ks * 4 + t];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = (double)sm.b[st][ks * 4 + t][wn * 32 + j * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + wm * 32 + i * 8 + g;
        if (m >= D.w) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + wn * 32 + j * 8 + 2 * t;
            const float v0 = (float)acc[i][j][0], v1 = (float)acc[i][j][1];
            float* q = D.Qt + (long long)m * D.ldq + n;
            float* ql = D.Qtlo + (long long)m * D.ldq + n;
            if (n + 1 < D.d) {
                *reinterpret_cast<float2*>(q) = make_float2(v0, v1);
                *reinterpret_cast<float2*>(ql) = make_float2(v0 - tf32_trunc(v0), v1 - tf32_trunc(v1));
            } else if (n < D.d) {
                q[0] = v0;
                ql[0] = v0 - tf32_trunc(v0);
            }
        }
    }
}

template <class Desc>
void upload_descs(DevBuf& buf, const std::vector<Desc>& v) {
    buf.alloc(sizeof(Desc) * std::max<size_t>(1, v.size()));
    if (!v.empty()) RKFAC_CUDA(cudaMemcpy(buf.p, v.data(), sizeof(Desc) * v.size(), cudaMemcpyHostToDevice));
}

}  // namespace

// ------------------------------------------------------------------------------------------------ host
void Gram64Batch::add(int w, int d, const float* T, long long ldt, double* G, long long ldg) {
    RKFAC_REQUIRE(((uintptr_t)T & 15) == 0 && ldt % 4 == 0, RKFAC_INVALID_ARGUMENT, "gram64: T must be 16B aligned");
    Gram64Desc g{};
    g.w = w; g.d = d; g.T = T; g.ldt = ldt; g.G = G; g.ldg = ldg;
    g.tiles_m = (int)ceil_div(w, kTile);
    const int kchunks = (int)ceil_div(d, kBK);
    // Split K so every problem has >= ~96 CTAs with >= 6 chunks each; fixed per shape => deterministic.
    const int ntri = g.tiles_m * (g.tiles_m + 1) / 2;
    int ks = 1;
    while (ks < 32 && ntri * ks < 96 && kchunks / (2 * ks) >= 6) ks *= 2;
    g.ksplit = ks;
    descs_.push_back(g);
}

void Gram64Batch::finalize() {
    total_tiles_ = 0;
    total_elems_ = 0;
    size_t part = 0;
    any_split_ = false;
    for (auto& g : descs_) {
        g.tile_offset = total_tiles_;
        g.elem_offset = total_elems_;
        const int ntri = g.tiles_m * (g.tiles_m + 1) / 2;
        total_tiles_ += (g.w > 0 && g.d > 0) ? ntri * g.ksplit : 0;
        total_elems_ += (long long)g.w * g.w;
        if (g.ksplit > 1) { part += (size_t)g.ksplit * g.w * g.w; any_split_ = true; }
    }
    partials_.alloc(part * sizeof(double));
    size_t off = 0;
    for (auto& g : descs_)
        if (g.ksplit > 1) {
            g.partial = static_cast<double*>(partials_.p) + off;
            off += (size_t)g.ksplit * g.w * g.w;
        }
    upload_descs(d_descs_, descs_);
    RKFAC_CUDA(cudaFuncSetAttribute(gram64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(GramSmem)));
}

double Gram64Batch::flops() const {
    double f = 0;
    for (const auto& g : descs_) f += (double)g.w * g.w * g.d;  // half of 2 w^2 d (symmetric)
    return f;
}

void Gram64Batch::launch(cudaStream_t s) const {
    if (total_tiles_ == 0) return;
    const int n = (int)descs_.size();
    gram64_kernel<<<total_tiles_, kThreads, sizeof(GramSmem), s>>>(d_descs_.as<Gram64Desc>(), n);
    count_launch();
    if (any_split_) {
        const int blocks = (int)std::min<long long>(ceil_div(total_elems_, 256), 148 * 8);
        gram64_reduce_kernel<<<blocks, 256, 0, s>>>(d_descs_.as<Gram64Desc>(), n, total_elems_);
        count_launch();
    }
    RKFAC_CHECK_LAUNCH();
}

void Tri64Batch::add(int w, int d, const double* L, long long ldl, const float* Yt, long long ldy, float* Qt,
                     float* Qtlo, long long ldq) {
    RKFAC_REQUIRE(((uintptr_t)L & 15) == 0 && ldl % 2 == 0 && ((uintptr_t)Yt & 15) == 0 && ldy % 4 == 0 &&
                      ((uintptr_t)Qt & 7) == 0 && ((uintptr_t)Qtlo & 7) == 0 && ldq % 2 == 0,
                  RKFAC_INVALID_ARGUMENT, "tri64: misaligned operands");
    Tri64Desc t{};
    t.w = w; t.d = d; t.L = L; t.ldl = ldl; t.Yt = Yt; t.ldy = ldy; t.Qt = Qt; t.Qtlo = Qtlo; t.ldq = ldq;
    t.tiles_n = (int)ceil_div(d, kTile);
    descs_.push_back(t);
}

void Tri64Batch::finalize() {
    total_tiles_ = 0;
    for (auto& t : descs_) {
        t.tile_offset = total_tiles_;
        total_tiles_ += (t.w > 0 && t.d > 0) ? (int)ceil_div(t.w, kTile) * t.tiles_n : 0;
    }
    upload_descs(d_descs_, descs_);
    RKFAC_CUDA(cudaFuncSetAttribute(tri64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(TriSmem)));
}

void Tri64Batch::launch(cudaStream_t s) const {
    if (total_tiles_ == 0) return;
    tri64_kernel<<<total_tiles_, kThreads, sizeof(TriSmem), s>>>(d_descs_.as<Tri64Desc>(), (int)descs_.size());
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
