// tc_gemm.cu -- tcgen05 / TMEM / TMA grouped GEMM in 3xTF32 for the sketch and power-iteration products
// Y = X Q of every factor (rnla.hpp:50-53, 97).  sm_100a only.
//
// Per problem f:   Y_f^T (w x d) = (X_f (d x d) * Q_f (d x w))^T,  Q stored as Q^T (w x d).
// Both operands are K-major (rows of X and rows of Q^T are contiguous along the contraction index), so the UMMA
// canonical K-major SWIZZLE_64B layout is exactly what TMA writes for a {16 floats x rows} box.
//
// 3xTF32: x = hi + lo with hi = tf32(x) (low 13 mantissa bits cleared) and lo = x - hi, both stored as FP32 in
// global memory by the producers of X and Q.  D += Ah*Bh + Ah*Bl + Al*Bh accumulates in one FP32 TMEM tile, which
// keeps the product within ~2^-21 relative of FP32 (1xTF32 fails the parity bar, 3xTF32 passes).
//
// Structure (one CTA per SM, persistent over an LPT tile schedule built on the host):
//   warp 0        TMA producer: 4 loads (Ah, Al, Bh, Bl) per 16-wide K block into a 4-stage smem ring
//   warp 1        TMEM allocator + single-thread MMA issuer: 6 x tcgen05.mma.kind::tf32 (M=128, N<=256, K=8)
//                 per K block, tcgen05.commit -> "stage empty"; after the last K block -> "accumulator full"
//   warps 2..5    epilogue: tcgen05.ld 32x32b (one TMEM lane = one output row) -> coalesced stores of Y^T
//                 (32 consecutive rows m per store instruction); two TMEM accumulators (2 x 256 columns) so the
//                 epilogue of tile i overlaps the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "tc_gemm.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 16;          // floats per K block (64 bytes per row => SWIZZLE_64B)
constexpr int kStages = 4;
constexpr int kMaxBN = 256;
constexpr int kATileBytes = kBM * kBK * 4;     // 8 KB
constexpr int kBTileBytes = kMaxBN * kBK * 4;  // 16 KB
constexpr int kStageBytes = 2 * kATileBytes + 2 * kBTileBytes;  // 48 KB
constexpr int kThreads = 192;
constexpr int kEpiWarp0 = 2;

struct __align__(8) SmemBarriers {
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_base;
};

// ------------------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_64B UMMA shared-memory descriptor (rows of 64 bytes, 8-row atoms of 512 bytes).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                        // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;               // stride byte offset: 8 rows x 64 B
    d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;                        // layout: SWIZZLE_64B
    return d;
}

// Instruction descriptor: D=F32, A=B=TF32, both K-major, M=128, N.
__device__ __forceinline__ uint32_t idesc_tf32(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ------------------------------------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(kThreads, 1)
xq_tc_kernel(const TcProblem* __restrict__ probs, const CUtensorMap* __restrict__ maps,
             const TcTile* __restrict__ tiles, const int* __restrict__ cta_begin) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte alignment of the stage ring (swizzle atoms need >= 512 B).
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                           ~uintptr_t(1023));
    SmemBarriers* bars = reinterpret_cast<SmemBarriers*>(smem + kStages * kStageBytes);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int t_begin = cta_begin[blockIdx.x], t_end = cta_begin[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 2 accumulators x 256 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&bars->tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_base;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < t_end; ++t) {
                const TcTile tl = tiles[t];
                const TcProblem& pr = probs[tl.prob];
                const CUtensorMap* mAh = maps + 4 * tl.prob;
                const uint32_t bytes = 2u * kATileBytes + 2u * (uint32_t)tl.n_tile * kBK * 4u;
                for (int kb = 0; kb < pr.kblocks; ++kb) {
                    mbar_wait(&bars->empty[stage], phase ^ 1);
                    unsigned char* st = smem + stage * kStageBytes;
                    mbar_expect_tx(&bars->full[stage], bytes);
                    const int k0 = kb * kBK;
                    tma_load_2d(st, mAh + 0, &bars->full[stage], k0, tl.m0);
                    tma_load_2d(st + kATileBytes, mAh + 1, &bars->full[stage], k0, tl.m0);
                    tma_load_2d(st + 2 * kATileBytes, mAh + 2, &bars->full[stage], k0, tl.n0);
                    tma_load_2d(st + 2 * kATileBytes + kBTileBytes, mAh + 3, &bars->full[stage], k0, tl.n0);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = t_begin; t < t_end; ++t, ++it) {
                const TcTile tl = tiles[t];
                const TcProblem& pr = probs[tl.prob];
                const int acc = it & 1;
                const uint32_t acc_phase = (it >> 1) & 1;
                mbar_wait(&bars->tmem_empty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * kMaxBN;
                const uint32_t idesc = idesc_tf32(tl.n_tile);
                for (int kb = 0; kb < pr.kblocks; ++kb) {
                    mbar_wait(&bars->full[stage], phase);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + stage * kStageBytes);
                    const uint32_t a_hi = st, a_lo = st + kATileBytes;
                    const uint32_t b_hi = st + 2 * kATileBytes, b_lo = b_hi + kBTileBytes;
#pragma unroll
                    for (int kk = 0; kk < kBK / 8; ++kk) {
                        const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along K inside the 64-byte row
                        const uint32_t first = (kb == 0 && kk == 0) ? 0u : 1u;
                        mma_tf32(tmem_d, umma_desc_sw64(a_lo + off), umma_desc_sw64(b_hi + off), idesc, first);
                        mma_tf32(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_lo + off), idesc, 1u);
                        mma_tf32(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_hi + off), idesc, 1u);
                    }
                    mma_commit(&bars->empty[stage]);  // frees the smem stage once these MMAs retire
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                mma_commit(&bars->tmem_full[acc]);
            }
        }
    } else {
        // ---------------- epilogue: TMEM -> registers -> Y^T (coalesced along m) ----------------
        const int q = warp % 4;  // TMEM lane quadrant this warp may access
        int it = 0;
        for (int t = t_begin; t < t_end; ++t, ++it) {
            const TcTile tl = tiles[t];
            const TcProblem& pr = probs[tl.prob];
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            mbar_wait(&bars->tmem_full[acc], acc_phase);
            tc_fence_after();
            const int m = tl.m0 + q * 32 + lane;
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kMaxBN;
            for (int c0 = 0; c0 < tl.n_tile; c0 += 32) {
                uint32_t r[32];
                tmem_ld32(tbase + c0, r);
                if (m < pr.M) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int n = tl.n0 + c0 + j;
                        if (c0 + j < tl.n_tile && n < pr.N) pr.Yt[(long long)n * pr.ldy + m] = __uint_as_float(r[j]);
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&bars->tmem_empty[acc]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// ------------------------------------------------------------------------------ hi/lo split producers
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void split_kernel(const SplitDesc* __restrict__ descs, int n, long long total, int raw_hi) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (descs[mid].offset <= e) lo = mid; else hi = mid - 1;
        }
        const SplitDesc& sd = descs[lo];
        const long long local = e - sd.offset;
        const int r = (int)(local / sd.cols), c = (int)(local - (long long)r * sd.cols);
        const float x = sd.src[(long long)r * sd.lds + c];
        const float h = tf32_trunc(x);
        sd.hi[(long long)r * sd.ldd + c] = raw_hi ? x : h;
        sd.lo[(long long)r * sd.ldd + c] = x - h;
    }
}

// --------------------------------------------------------------------------------------- host helpers
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        RKFAC_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q));
        RKFAC_REQUIRE(p && q == cudaDriverEntryPointSuccess, RKFAC_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

CUtensorMap make_map(const float* base, int inner, int outer, long long ld_elems, int box_inner, int box_outer) {
    RKFAC_REQUIRE((ld_elems * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0, RKFAC_INVALID_ARGUMENT,
                  "TMA operand needs 16-byte aligned base and row pitch");
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RKFAC_REQUIRE(r == CUDA_SUCCESS, RKFAC_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace

void TcXQ::add(const TcOperand& a, const TcOperand& b, int M, int N, int K, float* Yt, long long ldy) {
    RKFAC_REQUIRE(M > 0 && N > 0 && K > 0, RKFAC_INVALID_ARGUMENT, "empty tc problem");
    TcProblem p{};
    p.M = M; p.N = N; p.K = K; p.kblocks = (int)ceil_div(K, kBK);
    p.Yt = Yt; p.ldy = ldy;
    const int prob = (int)probs_.size();
    probs_.push_back(p);
    // B tile rows: N split into <=256-row tiles, each a multiple of 16 (UMMA M=128 needs N % 16 == 0).
    const int ntiles = (int)ceil_div(N, kMaxBN);
    const int per = (int)ceil_div(ceil_div(N, ntiles), 16) * 16;
    maps_.push_back(make_map(a.hi, K, M, a.ld, kBK, kBM));
    maps_.push_back(make_map(a.lo, K, M, a.ld, kBK, kBM));
    maps_.push_back(make_map(b.hi, K, N, b.ld, kBK, per));
    maps_.push_back(make_map(b.lo, K, N, b.ld, kBK, per));
    for (int nt = 0; nt < ntiles; ++nt)
        for (int m0 = 0; m0 < M; m0 += kBM) {
            TcTile t{};
            t.prob = prob; t.m0 = m0; t.n0 = nt * per;
            t.n_tile = per;
            tiles_.push_back(t);
        }
}

void TcXQ::finalize() {
    // LPT over persistent CTAs: cost of a tile ~ K * n_tile.
    const int ntiles = (int)tiles_.size();
    nctas_ = std::max(1, std::min(ntiles, kNumSMs));
    std::vector<int> order(ntiles);
    std::iota(order.begin(), order.end(), 0);
    auto cost = [&](int i) { return (double)probs_[tiles_[i].prob].kblocks * (tiles_[i].n_tile + 32); };
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
    std::vector<double> load(nctas_, 0.0);
    std::vector<std::vector<int>> lists(nctas_);
    for (int i : order) {
        const int k = (int)(std::min_element(load.begin(), load.end()) - load.begin());
        lists[k].push_back(i);
        load[k] += cost(i);
    }
    std::vector<TcTile> sched;
    std::vector<int> begin(nctas_ + 1, 0);
    for (int c = 0; c < nctas_; ++c) {
        begin[c] = (int)sched.size();
        for (int i : lists[c]) sched.push_back(tiles_[i]);
    }
    begin[nctas_] = (int)sched.size();
    auto up = [](DevBuf& b, const void* src, size_t bytes) {
        b.alloc(std::max<size_t>(bytes, 64));
        if (bytes) RKFAC_CUDA(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice));
    };
    up(d_probs_, probs_.data(), sizeof(TcProblem) * probs_.size());
    up(d_maps_, maps_.data(), sizeof(CUtensorMap) * maps_.size());
    up(d_tiles_, sched.data(), sizeof(TcTile) * sched.size());
    up(d_begin_, begin.data(), sizeof(int) * begin.size());
}

size_t TcXQ::smem_bytes() { return (size_t)kStages * kStageBytes + sizeof(SmemBarriers) + 1024; }

void TcXQ::launch(cudaStream_t s) const {
    if (tiles_.empty()) return;
    const size_t smem = smem_bytes();
    RKFAC_CUDA(cudaFuncSetAttribute(xq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    xq_tc_kernel<<<nctas_, kThreads, smem, s>>>(d_probs_.as<TcProblem>(), d_maps_.as<CUtensorMap>(),
                                                d_tiles_.as<TcTile>(), d_begin_.as<int>());
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

double TcXQ::flops() const {
    double f = 0;
    for (const auto& p : probs_) f += 2.0 * p.M * (double)p.N * p.K;
    return f;
}

void launch_split(const SplitDesc* d_descs, int n, long long total, cudaStream_t s) {
    if (total == 0) return;
    const int blocks = (int)std::min<long long>(ceil_div(total, 256), kNumSMs * 8);
    static const int raw_hi = [] { const char* e = std::getenv("RKFAC_RAW_HI"); return e && e[0] == '1'; }();
    split_kernel<<<blocks, 256, 0, s>>>(d_descs, n, total, raw_hi);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
