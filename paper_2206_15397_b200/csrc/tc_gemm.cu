// tc_gemm.cu -- tcgen05 / TMEM / TMA grouped GEMM in 3xTF32 (sm_100a).  Every dense contraction of the rand-EVD
// whose operands are FP32 goes through it, all factors of a stage in ONE launch:
//   X*Q sketch / power products (rnla.hpp:50-53, 97), Gram Y^T Y and Y L^-T of the CholeskyQR orthonormalisation
//   (replacing qr_thin, qr.hpp:23-87), the core Q^T X Q / B B^T (rnla.hpp:97, eig.hpp:251) and the EA SYRK
//   (kfactor.hpp:33-41, symmetric tiles).
//
// Operands are K-major (A: M x K, B: N x K rows contiguous along K), so the UMMA canonical K-major SWIZZLE_64B
// layout is exactly what TMA writes for a {16 floats x rows} box.  3xTF32: D = A*B_lo + A_lo*B + A*B in one FP32
// TMEM tile; "A" and "B" are the raw FP32 arrays (the tensor core reads them as TF32 by dropping the low 13
// mantissa bits -- verified bitwise against explicitly truncated operands), the lo planes x - tf32(x) are produced
// by the previous stage's epilogue.  SURVEY.md F8b: 1xTF32 fails the parity bar, 3xTF32 keeps FP32 accuracy.
//
// One CTA per SM, persistent over an LPT tile schedule built on the host (tiles of all problems, all K slices):
//   warp 0      TMA producer: 4 box loads (A, A_lo, B, B_lo) per 16-wide K block into a 4-stage smem ring
//   warp 1      TMEM allocator + single-thread MMA issuer: 6 x tcgen05.mma.kind::tf32 (M=128, N<=256, K=8) per
//               K block; tcgen05.commit -> stage empty; after the last K block -> accumulator full
//   warps 2..5  epilogue: tcgen05.ld 32x32b (TMEM lane = output row) -> fused alpha/scales/axpy -> up to four
//               outputs in either layout (+ TF32 lo planes); split-K tiles store raw partials instead
//   warps 6..7  lo-plane converters: for problems without a stored A lo plane (the EA factor X, read by every
//               power product) the A_lo slot of each stage is formed in shared memory from the TMA-loaded A tile
//               (x - tf32(x), same swizzled layout), so X's lo plane never travels through HBM
// Two TMEM accumulators (2 x 256 columns) let the epilogue of tile i overlap the MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>

#include "tc_gemm.cuh"

namespace rkfac_b200 {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 16;          // floats per K block (64 bytes per row => SWIZZLE_64B)
constexpr int kMaxStages = 6;
constexpr int kMaxBN = 256;
constexpr int kATileBytes = kBM * kBK * 4;     // 8 KB (one 128-row A sub-tile)
constexpr int kBTileBytes = kMaxBN * kBK * 4;  // 16 KB
// Three shared-memory configurations of the same ~192 KB region:
//   kCfg 0, single tiles: 4 stages of [A hi][A lo][B hi][B lo] = 48 KB
//   kCfg 1, paired tiles: 3 stages of [A0 hi][A1 hi][A0 lo][A1 lo][B hi][B lo] = 64 KB (256 rows share the B tile)
//   kCfg 2, EA update (symmetric 128 x 128 tiles, axpy input Cin): RKFAC_EA_STAGES (4) stages of 32 KB (B tile of
//           128 rows) and, after them, per epilogue warp a ring of kCinRing 32 x 32 chunks (Cin prefetched by
//           cp.async, the output written in place) and two mirror chunks, all dense 128-byte rows in the TMA
//           SWIZZLE_128B layout: each output chunk and its transpose leave by TMA bulk-tensor stores (the diagonal
//           chunk after its lower part is overwritten by the mirror of its upper part), so the epilogue -- a pure
//           HBM stream -- keeps several chunks in flight per warp with a handful of instructions per chunk; with no
//           transpose tiles this region (208 KB) extends into their space and the barriers follow it
#ifndef RKFAC_EA_CIN_RING
#define RKFAC_EA_CIN_RING 3  // Cin chunks per epilogue warp in the EA configuration
#endif
constexpr int kCinRing = RKFAC_EA_CIN_RING;
#ifndef RKFAC_EA_STAGES
#define RKFAC_EA_STAGES 4  // mainloop stages of the EA configuration (its region reaches 208 KB; 3: 6 % slower)
#endif
//   kCfg 3, CTA pairs (cta_group::2, M = 256 over two SMs): 6 stages of [A hi][A lo][B hi half][B lo half] = 32 KB;
//           each CTA of the pair holds its own 128 rows of A and HALF of the B tile's rows.  Measured: the mainloop
//           runs at the same per-SM rate as the single-CTA configurations (1040 cycles per 128 x 240 x 16 block of
//           six MMAs, i.e. the measured dense-TF32 rate; 512-row pair tiles, B lo planes formed in smem and deeper
//           pipelines all leave it unchanged), but its 256-row tiles over SM pairs schedule better (X*Q 3.28 -> 3.06 ms)
template <int kCfg>
struct StageCfg {
    static constexpr int kSub = kCfg == 1 ? 2 : 1;
    static constexpr int kStages = kCfg == 0 ? 4 : (kCfg == 2 ? RKFAC_EA_STAGES : (kCfg == 3 ? 6 : 3));
    static constexpr int kBTile = kCfg == 2 ? kBM * kBK * 4 : (kCfg == 3 ? kBTileBytes / 2 : kBTileBytes);
    static constexpr int kStageBytes = 2 * kSub * kATileBytes + 2 * kBTile;
};
constexpr int kStagesBytesMax = 3 * (4 * kATileBytes + 2 * kBTileBytes);  // == 4 * 48 KB
constexpr int kChunkBytes = 32 * 32 * 4;                                   // dense swizzled 32 x 32 chunk
constexpr int kEaRingOff = StageCfg<2>::kStages * StageCfg<2>::kStageBytes;  // 96 KB
constexpr int kEaMirOff = kEaRingOff + 4 * kCinRing * kChunkBytes;         // 144 KB
constexpr int kEaRegionBytes = kEaMirOff + 4 * 2 * kChunkBytes;
constexpr int kCfgRegionBytes(int cfg) { return cfg == 2 && kEaRegionBytes > kStagesBytesMax ? kEaRegionBytes : kStagesBytesMax; }
// byte offset of element (row r, column c) of a dense 32 x 32 FP32 chunk in the SWIZZLE_128B layout
__device__ __forceinline__ uint32_t sw128(int r, int c) {
    return (uint32_t)(r * 128 + ((((c >> 2) ^ (r & 7)) & 7) << 4) + (c & 3) * 4);
}
constexpr int kThreads = 256;
constexpr int kMapsPerProb = 5;  // A, A_lo, B, B_lo, out0 (SWIZZLE_128B 32 x 32 store boxes; EA configuration)
constexpr int kConvThreads = 64;  // warps 6..7

struct __align__(8) SmemBarriers {
    uint64_t full[kMaxStages];
    uint64_t empty[kMaxStages];
    uint64_t conv[kMaxStages];  // A lo slot of the stage formed (converter warps)
    uint64_t tmem_full[2];
    uint64_t tmem_empty[2];
    uint32_t tmem_base;
};
constexpr int kBarrierBytes = (sizeof(SmemBarriers) + 127) / 128 * 128;
constexpr int kStageTileBytes = 4 * 32 * 36 * 4;  // one 32x36 transpose tile per epilogue warp
// the EA configuration stores its diagonal chunks by TMA too (no transpose tiles): its region may use their space
static_assert(kEaRegionBytes <= kStagesBytesMax + kStageTileBytes, "EA smem");

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
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 1000000;\n"
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
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major SWIZZLE_64B UMMA shared-memory descriptor (rows of 64 bytes, 8-row atoms of 512 bytes).
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);  // start address
    d |= (uint64_t)1 << 16;                  // leading byte offset (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;         // stride byte offset: 8 rows x 64 B
    d |= (uint64_t)1 << 46;                  // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;                  // layout: SWIZZLE_64B
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
// CTA pair (cta_group::2): issued by the leader CTA only; D is 256 x N (128 TMEM lanes in each CTA), A's rows 128..255
// and B's rows N/2..N-1 are read from the peer CTA's shared memory at the same offsets.
__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ uint32_t idesc_tf32_pair(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)((2 * kBM) >> 4) << 24);
}
// completion of the pair's MMAs arrives on the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive on the barrier at this offset in CTA `rank` of the cluster.  Default semantics (release at CTA scope), as
// for any consumer-release arrival across a cluster: a cluster-scope release costs a full memory barrier per arrival
// (measured: the converter warps then bound the mainloop, 2.1x slower); the data the leader's MMAs read from the
// peer's shared memory is ordered by the fence.proxy.async that precedes the arrival.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    uint32_t addr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
// wait with acquire at cluster scope (the arrivals come from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAITC:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, 1000000;\n"
        "@P1 bra DONEC;\n"
        "bra LAB_WAITC;\n"
        "DONEC:\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
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

// split form: issue the TMEM load, overlap other waits, then wait with the registers as operands (so no use of them
// can be scheduled above the wait)
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32_wait(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__device__ __forceinline__ float load_mn(const float* p, long long ld, int t, int m, int n) {
    return t ? p[(long long)n * ld + m] : p[(long long)m * ld + n];
}

// Epilogue value of element (m, n) from the raw accumulator sum (used by the split-K reduction).
__device__ __forceinline__ float epi_value(const TcProb& pr, int m, int n, float acc) {
    float v = pr.alpha * acc;
    if (pr.rs) v *= pr.rs[m];
    if (pr.cs) v *= pr.cs[n];
    if (pr.beta != 0.f) v = fmaf(pr.beta, load_mn(pr.Cin, pr.ldcin, pr.cin_t, m, n), v);
    if (pr.gamma != 0.f) v = fmaf(pr.gamma, load_mn(pr.Din, pr.lddin, pr.din_t, m, n), v);
    return v;
}

// Warp-cooperative 32x32 chunk I/O of the epilogue.  Lane = output row (TMEM lane); a row-major ([m][n]) access
// of the chunk is staged through a padded smem tile so that global memory sees 128-byte row segments, a
// transposed ([n][m]) access is naturally coalesced across lanes.
// Row-major 32x32 chunk accesses are done as 8 x 128-bit accesses per lane (lane covers row 4*i + lane/8,
// columns 4*(lane%8)..+3), all issued back to back, and transposed through a [32][36] smem tile.
constexpr int kTP = 36;  // staging tile pitch (floats): 16-byte aligned rows

__device__ __forceinline__ void rm_issue(float4 (&pre)[8], const float* p, long long ld, int mbase, int nbase, int M,
                                         int N, int lane) {
    const int c = (lane & 7) * 4;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | (uintptr_t)(ld * 4)) & 15) == 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int m = mbase + i * 4 + (lane >> 3), n = nbase + c;
        if (vec && m < M && n + 3 < N) {
            pre[i] = *reinterpret_cast<const float4*>(p + (long long)m * ld + n);
        } else {
            float e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = (m < M && n + u < N) ? p[(long long)m * ld + n + u] : 0.f;
            pre[i] = make_float4(e[0], e[1], e[2], e[3]);
        }
    }
}

__device__ __forceinline__ void rm_finish(float (&dst)[32], const float4 (&pre)[8], float (*tile)[kTP], int lane) {
    const int c = (lane & 7) * 4;
#pragma unroll
    for (int i = 0; i < 8; ++i) *reinterpret_cast<float4*>(&tile[i * 4 + (lane >> 3)][c]) = pre[i];
    __syncwarp();
#pragma unroll
    for (int j4 = 0; j4 < 32; j4 += 4) {
        const float4 q = *reinterpret_cast<const float4*>(&tile[lane][j4]);
        dst[j4] = q.x; dst[j4 + 1] = q.y; dst[j4 + 2] = q.z; dst[j4 + 3] = q.w;
    }
    __syncwarp();
}

__device__ __forceinline__ void chunk_load(float (&dst)[32], const float* p, long long ld, int t, int mbase,
                                           int nbase, int M, int N, float (*tile)[kTP], int lane) {
    if (t) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int m = mbase + lane, n = nbase + j;
            dst[j] = (m < M && n < N) ? p[(long long)n * ld + m] : 0.f;
        }
    } else {
        float4 pre[8];
        rm_issue(pre, p, ld, mbase, nbase, M, N, lane);
        rm_finish(dst, pre, tile, lane);
    }
}

// Stores v (row mbase+lane, cols nbase..nbase+31) to one output; `skip_lower` drops elements below the diagonal
// (symmetric diagonal tiles), `mirror` additionally stores the transposed element (symmetric tiles).
__device__ __forceinline__ float lo_or(float x, bool lo) { return lo ? x - tf32_trunc(x) : x; }

// Scalar store of one element to every output (split-K reduction path).
__device__ __forceinline__ void store_outputs(const TcProb& pr, int m, int n, float v) {
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        if (!pr.o[o]) continue;
        const float x = lo_or(v, pr.is_lo[o] != 0);
        if (pr.to[o]) pr.o[o][(long long)n * pr.ldo[o] + m] = x;
        else pr.o[o][(long long)m * pr.ldo[o] + n] = x;
    }
}

__device__ __forceinline__ void chunk_store(const float (&v)[32], float* p, long long ld, int t, bool lo, int mbase,
                                            int nbase, int M, int N, bool skip_lower, bool mirror,
                                            float (*tile)[kTP], int lane) {
    const int m = mbase + lane;
    if (t) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int n = nbase + j;
            if (m < M && n < N && !(skip_lower && n < m)) p[(long long)n * ld + m] = lo_or(v[j], lo);
        }
    } else {
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4)
            *reinterpret_cast<float4*>(&tile[lane][j4]) =
                make_float4(lo_or(v[j4], lo), lo_or(v[j4 + 1], lo), lo_or(v[j4 + 2], lo), lo_or(v[j4 + 3], lo));
        __syncwarp();
        const int c = (lane & 7) * 4;
        const bool vec = ((reinterpret_cast<uintptr_t>(p) | (uintptr_t)(ld * 4)) & 15) == 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int mm = mbase + i * 4 + (lane >> 3), n = nbase + c;
            const float4 q = *reinterpret_cast<const float4*>(&tile[i * 4 + (lane >> 3)][c]);
            if (vec && mm < M && n + 3 < N && !(skip_lower && n < mm)) {
                *reinterpret_cast<float4*>(p + (long long)mm * ld + n) = q;
            } else {
                const float e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (mm < M && n + u < N && !(skip_lower && n + u < mm)) p[(long long)mm * ld + n + u] = e[u];
            }
        }
        __syncwarp();
    }
    if (mirror) {  // element (n, m) in the opposite layout of the direct store: coalesced when t == 0
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int n = nbase + j;
            if (m < M && n < N && n > m) {
                if (t) p[(long long)m * ld + n] = lo_or(v[j], lo);
                else p[(long long)n * ld + m] = lo_or(v[j], lo);
            }
        }
    }
}

// A value plane and its TF32 lo plane in the same layout, written in one pass (the common output pair of the
// path: the operands of the next tensor-core product).  Interior chunks take pointer-increment fast paths: a
// transposed chunk is 32 coalesced 128-byte stores per plane, a row-major chunk is staged once through the smem
// tile and leaves as 128-bit stores of both planes.
__device__ __forceinline__ float4 lo4(float4 q) {
    return make_float4(q.x - tf32_trunc(q.x), q.y - tf32_trunc(q.y), q.z - tf32_trunc(q.z), q.w - tf32_trunc(q.w));
}

__device__ __forceinline__ void chunk_store_pair(const float (&v)[32], float* ph, float* pl, long long ld, int t,
                                                 int mbase, int nbase, int M, int N, bool skip_lower, bool mirror,
                                                 float (*tile)[kTP], int lane) {
    const int m = mbase + lane;
    if (t) {
        if (!skip_lower && nbase + 32 <= N) {
            if (m < M) {
                float* qh = ph + (long long)nbase * ld + m;
                float* ql = pl + (long long)nbase * ld + m;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    *qh = v[j];
                    *ql = v[j] - tf32_trunc(v[j]);
                    qh += ld;
                    ql += ld;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = nbase + j;
                if (m < M && n < N && !(skip_lower && n < m)) {
                    ph[(long long)n * ld + m] = v[j];
                    pl[(long long)n * ld + m] = v[j] - tf32_trunc(v[j]);
                }
            }
        }
    } else {
#pragma unroll
        for (int j4 = 0; j4 < 32; j4 += 4)
            *reinterpret_cast<float4*>(&tile[lane][j4]) = make_float4(v[j4], v[j4 + 1], v[j4 + 2], v[j4 + 3]);
        __syncwarp();
        const int c = (lane & 7) * 4;
        const bool vec = ((reinterpret_cast<uintptr_t>(ph) | reinterpret_cast<uintptr_t>(pl) | (uintptr_t)(ld * 4)) &
                          15) == 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int mm = mbase + i * 4 + (lane >> 3), n = nbase + c;
            const float4 q = *reinterpret_cast<const float4*>(&tile[i * 4 + (lane >> 3)][c]);
            if (vec && mm < M && n + 3 < N && !(skip_lower && n < mm)) {
                *reinterpret_cast<float4*>(ph + (long long)mm * ld + n) = q;
                *reinterpret_cast<float4*>(pl + (long long)mm * ld + n) = lo4(q);
            } else {
                const float e[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (mm < M && n + u < N && !(skip_lower && n + u < mm)) {
                        ph[(long long)mm * ld + n + u] = e[u];
                        pl[(long long)mm * ld + n + u] = e[u] - tf32_trunc(e[u]);
                    }
            }
        }
        __syncwarp();
    }
    if (mirror && m < M) {  // element (n, m) in the opposite layout of the direct store: coalesced when t == 0
        if (!t && nbase > m + 0 && nbase + 32 <= N) {  // whole chunk strictly above this row's diagonal
            float* qh = ph + (long long)nbase * ld + m;
            float* ql = pl + (long long)nbase * ld + m;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                *qh = v[j];
                *ql = v[j] - tf32_trunc(v[j]);
                qh += ld;
                ql += ld;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int n = nbase + j;
                if (n < N && n > m) {
                    const long long i = t ? (long long)m * ld + n : (long long)n * ld + m;
                    ph[i] = v[j];
                    pl[i] = v[j] - tf32_trunc(v[j]);
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------------------------ kernel
template <int kCfg>
__global__ void __launch_bounds__(kThreads, 1)
tc_gemm_kernel(const TcProb* __restrict__ probs, const CUtensorMap* __restrict__ maps,
               const TcTile* __restrict__ tiles, const int* __restrict__ cta_begin) {
    __shared__ TcProb s_pr[4];  // per epilogue warp
    constexpr bool kPair = kCfg == 1;
    constexpr bool k2 = kCfg == 3;  // CTA pairs: blockIdx.x / 2 is the schedule slot, %cluster_ctarank the half
    constexpr int kStages = StageCfg<kCfg>::kStages;
    constexpr int kStageBytes = StageCfg<kCfg>::kStageBytes;
    constexpr int kSub = StageCfg<kCfg>::kSub;
    constexpr int kBTileS = StageCfg<kCfg>::kBTile;
    // declared 16-byte aligned only: with __align__(1024) the compiler folds the runtime alignment below to 0
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // 1024-byte aligned base, derived by indexing the __shared__ array (integer round-trips of the address would
    // lose the address space: every smem access below would compile to generic LD/ST)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    SmemBarriers* bars = reinterpret_cast<SmemBarriers*>(smem + kCfgRegionBytes(kCfg));
    float (*stage_tiles)[32][36] =  // unused by kCfg 2 when its region extends past kStagesBytesMax
        reinterpret_cast<float (*)[32][36]>(smem + kStagesBytesMax + kBarrierBytes);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int slot_id = k2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int crank = k2 ? (int)cluster_ctarank() : 0;
    const int t_begin = cta_begin[slot_id], t_end = cta_begin[slot_id + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
            // pairs: the leader's barrier collects the converter warps of both CTAs
            mbar_init(&bars->conv[s], k2 ? 2 : kConvThreads / 32);  // pairs: one converter warp of each CTA
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->tmem_full[a], 1);
            mbar_init(&bars->tmem_empty[a], k2 ? 8 : 128);  // pairs: one arrival per epilogue warp of both CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: 2 accumulators x 256 fp32 columns
        if constexpr (k2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_u32(&bars->tmem_base)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                             smem_u32(&bars->tmem_base)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (k2) cluster_sync_all();  // the peer's barriers are initialised and its TMEM allocated
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = bars->tmem_base;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_begin; t < t_end; ++t) {
                const TcTile tl = tiles[t];
                const TcProb& pr = probs[tl.prob];
                const CUtensorMap* mp = maps + kMapsPerProb * tl.prob;
                const uint32_t aplanes = (pr.a_conv || pr.single) ? 1u : 2u, bplanes = (pr.b_conv || pr.single) ? 1u : 2u;
                const int brows = k2 ? pr.n_tile / 2 : pr.n_tile;  // pairs: this CTA's half of the B tile
                // pairs: this CTA's rows follow the leader's (one or two 128-row sub-tiles each)
                const int am0 = tl.m0 + crank * ((kPair && tl.pair) ? 2 : 1) * kBM, bn0 = tl.n0 + crank * brows;
                const uint32_t bytes =
                    ((kPair && tl.pair) ? 2u : 1u) * aplanes * kATileBytes + bplanes * (uint32_t)brows * kBK * 4u;
                for (int kb = tl.kb0; kb < tl.kb1; ++kb) {
                    mbar_wait(&bars->empty[stage], phase ^ 1);
                    unsigned char* st = smem + stage * kStageBytes;
                    mbar_expect_tx(&bars->full[stage], bytes);
                    const int k0 = kb * kBK;
                    tma_load_2d(st, mp + 0, &bars->full[stage], k0, am0);
                    if (!pr.a_conv && !pr.single) tma_load_2d(st + kSub * kATileBytes, mp + 1, &bars->full[stage], k0, am0);
                    if (kPair && tl.pair) {
                        tma_load_2d(st + kATileBytes, mp + 0, &bars->full[stage], k0, am0 + kBM);
                        if (!pr.a_conv && !pr.single)
                            tma_load_2d(st + 3 * kATileBytes, mp + 1, &bars->full[stage], k0, am0 + kBM);
                    }
                    tma_load_2d(st + 2 * kSub * kATileBytes, mp + 2, &bars->full[stage], k0, bn0);
                    if (!pr.b_conv && !pr.single)
                        tma_load_2d(st + 2 * kSub * kATileBytes + kBTileS, mp + 3, &bars->full[stage], k0, bn0);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (pairs: the leader CTA issues for both) ----------------
        if (lane == 0 && crank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int rr = 0;                     // next accumulator slot for a single tile
            uint32_t uses[2] = {0u, 0u};    // completed uses of each slot (parity of its barriers)
            for (int t = t_begin; t < t_end; ++t) {
                const TcTile tl = tiles[t];
                const TcProb& pr = probs[tl.prob];
                const int nsub = (kPair && tl.pair) ? 2 : 1;
                const int slot0 = (kPair && tl.pair) ? 0 : rr;
                for (int sub = 0; sub < nsub; ++sub) {
                    const int a = slot0 + sub;
                    if constexpr (k2) mbar_wait_cluster(&bars->tmem_empty[a], (uses[a] & 1u) ^ 1u);
                    else mbar_wait(&bars->tmem_empty[a], (uses[a] & 1u) ^ 1u);
                }
                tc_fence_after();
                const uint32_t idesc = k2 ? idesc_tf32_pair(pr.n_tile) : idesc_tf32(pr.n_tile);
                const bool single = pr.single != 0;
                for (int kb = tl.kb0; kb < tl.kb1; ++kb) {
                    mbar_wait(&bars->full[stage], phase);
                    // pairs: the converter warps of both CTAs arrive here once their own tiles have landed
#ifdef RKFAC_PAIR_CLUSTER_ACQ
                    if constexpr (k2) mbar_wait_cluster(&bars->conv[stage], phase);
                    else
#endif
                    mbar_wait(&bars->conv[stage], phase);
                    tc_fence_after();
                    const uint32_t st = smem_u32(smem + stage * kStageBytes);
                    const uint32_t b_hi = st + 2 * kSub * kATileBytes, b_lo = b_hi + kBTileS;
                    for (int sub = 0; sub < nsub; ++sub) {
                        const uint32_t tmem_d = tmem_base + (slot0 + sub) * kMaxBN;
                        const uint32_t a_hi = st + sub * kATileBytes, a_lo = st + (kSub + sub) * kATileBytes;
#pragma unroll
                        for (int kk = 0; kk < kBK / 8; ++kk) {
                            const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along K inside the 64-byte row
                            const uint32_t first = (kb == tl.kb0 && kk == 0) ? 0u : 1u;
                            if constexpr (k2) {
                                if (!single) {
                                    mma_tf32_pair(tmem_d, umma_desc_sw64(a_lo + off), umma_desc_sw64(b_hi + off), idesc, first);
                                    mma_tf32_pair(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_lo + off), idesc, 1u);
                                }
                                mma_tf32_pair(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_hi + off), idesc,
                                              single ? first : 1u);
                            } else {
                                if (!single) {
                                    mma_tf32(tmem_d, umma_desc_sw64(a_lo + off), umma_desc_sw64(b_hi + off), idesc, first);
                                    mma_tf32(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_lo + off), idesc, 1u);
                                }
                                mma_tf32(tmem_d, umma_desc_sw64(a_hi + off), umma_desc_sw64(b_hi + off), idesc,
                                         single ? first : 1u);
                            }
                        }
                    }
                    if constexpr (k2) mma_commit_pair(&bars->empty[stage]);
                    else mma_commit(&bars->empty[stage]);
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                }
                for (int sub = 0; sub < nsub; ++sub) {
                    if constexpr (k2) mma_commit_pair(&bars->tmem_full[slot0 + sub]);
                    else mma_commit(&bars->tmem_full[slot0 + sub]);
                    ++uses[slot0 + sub];
                }
                if (!(kPair && tl.pair)) rr ^= 1;
            }
        }
    } else if (warp >= 6) {
        // ---------------- A lo-plane converters ----------------
        // kCfg 0-2: both warps share every stage.  CTA pairs (kCfg 3): the warps take alternate K blocks, each
        // converting a whole stage alone, so one warp's proxy fence (the long pole of a stage) overlaps the other
        // warp's conversion.
        constexpr int kCT = k2 ? 32 : kConvThreads;  // threads converting one stage
        const int ct = k2 ? lane : (int)threadIdx.x - 6 * 32;
        const int mine = warp - 6;  // kCfg 3: parity of the K blocks this warp converts
        int stage = 0;
        uint32_t phase = 0;
        uint32_t kbn = 0;  // K blocks seen
        for (int t = t_begin; t < t_end; ++t) {
            const TcTile tl = tiles[t];
            const bool single = probs[tl.prob].single != 0;
            const bool conv = probs[tl.prob].a_conv != 0 && !single, bconv = probs[tl.prob].b_conv != 0 && !single;
            const int nb16 = (k2 ? probs[tl.prob].n_tile / 2 : probs[tl.prob].n_tile) * kBK / 4;  // float4s of the B tile
            const int nsub = (kPair && tl.pair) ? 2 : 1;
            for (int kb = tl.kb0; kb < tl.kb1; ++kb, ++kbn) {
                if (k2 && (int)(kbn & 1u) != mine) {
                    if (++stage == kStages) { stage = 0; phase ^= 1; }
                    continue;
                }
                mbar_wait(&bars->full[stage], phase);  // also paces the arrivals of unconverted problems
                if (conv) {
                    unsigned char* st = smem + stage * kStageBytes;
                    for (int sub = 0; sub < nsub; ++sub) {
                        const float4* src = reinterpret_cast<const float4*>(st + sub * kATileBytes);
                        float4* dst = reinterpret_cast<float4*>(st + (kSub + sub) * kATileBytes);
#pragma unroll
                        for (int i = 0; i < kATileBytes / 16 / kCT; ++i) {
                            const float4 x = src[i * kCT + ct];
                            dst[i * kCT + ct] = lo4(x);
                        }
                    }
                }
                if (bconv) {
                    unsigned char* st = smem + stage * kStageBytes;
                    const float4* src = reinterpret_cast<const float4*>(st + 2 * kSub * kATileBytes);
                    float4* dst = reinterpret_cast<float4*>(st + 2 * kSub * kATileBytes + kBTileS);
                    for (int i = ct; i < nb16; i += kCT) dst[i] = lo4(src[i]);
                }
                if (conv || bconv) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // tensor core
                __syncwarp();
                if (lane == 0) {
                    if (k2 && crank != 0) mbar_arrive_remote(&bars->conv[stage], 0);  // the leader issues the MMAs
                    else mbar_arrive(&bars->conv[stage]);
                }
                if (++stage == kStages) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue ----------------
        const int q = warp % 4;  // TMEM lane quadrant this warp may access
        int rr = 0;
        uint32_t uses[2] = {0u, 0u};
        // kCfg 2: Cin chunks of this warp in (tile, chunk) order, prefetched by cp.async kCinRing-1 chunks ahead into a
        // ring of kCinRing swizzled slots (zero-filled past the matrix edge); the output chunk is written in place
        unsigned char* ring = smem + kEaRingOff + (warp - 2) * kCinRing * kChunkBytes;
        unsigned char* mir = smem + kEaMirOff + (warp - 2) * 2 * kChunkBytes;
        int cin_t = t_begin, cin_c = 0;  // next chunk to prefetch
        auto cin_issue = [&](int slot) {
            if (cin_t < t_end) {
                const TcTile ct = tiles[cin_t];
                const TcProb& cp = probs[ct.prob];
                const int mb = ct.m0 + q * 32, nb = ct.n0 + cin_c * 32;
                const int cc = lane & 7, nl = min(cp.N, ct.n0 + cp.n_tile);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int rr_ = i * 4 + (lane >> 3), mm = mb + rr_, n = nb + cc * 4;
                    const int valid = (mm < cp.M) ? max(0, min(4, nl - n)) : 0;
                    const float* src = valid ? cp.Cin + (long long)mm * cp.ldcin + n : cp.Cin;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                                     smem_u32(ring + slot * kChunkBytes + sw128(rr_, cc * 4))),
                                 "l"(src), "r"(valid * 4));
                }
                if (++cin_c * 32 >= cp.n_tile) { cin_c = 0; ++cin_t; }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        };
        int chunk_no = 0;  // chunks consumed by this warp
        if constexpr (kCfg == 2)
            for (int i = 0; i + 1 < kCinRing; ++i) cin_issue(i);  // kCinRing - 1 chunks ahead
        for (int t = t_begin; t < t_end; ++t) {
          const TcTile tl = tiles[t];
          const int nsub = (kPair && tl.pair) ? 2 : 1;
          const int slot0 = (kPair && tl.pair) ? 0 : rr;
          if (!(kPair && tl.pair)) rr ^= 1;
          // the problem descriptor in this warp's shared-memory slot: its fields are re-read in every chunk, and
          // from global memory the compiler must reload them after each epilogue store (possible aliasing)
          {
              const int* src = reinterpret_cast<const int*>(&probs[tl.prob]);
              int* dst = reinterpret_cast<int*>(&s_pr[warp - 2]);
              for (int i = lane; i < (int)(sizeof(TcProb) / sizeof(int)); i += 32) dst[i] = src[i];
              __syncwarp();
          }
          for (int sub = 0; sub < nsub; ++sub) {
            const TcProb& pr = s_pr[warp - 2];
            const int acc = slot0 + sub;
            const uint32_t acc_phase = uses[acc] & 1u;
            ++uses[acc];
            const int m0s = tl.m0 + (crank * nsub + sub) * kBM;  // this sub-tile's first row (CTA pairs: rank-major)
            const int mbase = m0s + q * 32;
            const int m = mbase + lane;
            const bool diag = pr.sym && m0s == tl.n0;
            const int nlim = min(pr.N, tl.n0 + pr.n_tile);
            float (*tile)[kTP] = stage_tiles[warp - 2];
            // (an axpy input Cin outside the EA configuration -- kCfg 2 prefetches it through its cp.async ring -- is
            // loaded chunk by chunk: no problem on the path takes that route, and a register-held prefetch costs the
            // 32 registers that keep this epilogue from spilling)
            mbar_wait(&bars->tmem_full[acc], acc_phase);
            tc_fence_after();
            const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kMaxBN;
            // kCfg 0/1/3: the next chunk's TMEM load is issued as soon as this chunk's accumulators are consumed, so
            // its latency overlaps this chunk's epilogue (short-K products are epilogue-bound)
            uint32_t r[32];
            if constexpr (kCfg != 2) tmem_ld32_issue(tbase, r);
            for (int c0 = 0; c0 < pr.n_tile; c0 += 32) {
                if constexpr (kCfg == 2) {
                    // the TMEM load in flight while this chunk's Cin cp.async group is awaited (every EA tile has a
                    // Cin, host-checked: chunk_no's slot is complete once at most one younger group is pending)
                    tmem_ld32_issue(tbase + c0, r);
                    asm volatile("cp.async.wait_group %0;\n" ::"n"(kCinRing - 2) : "memory");
                    tmem_ld32_wait(r);
                } else {
                    tmem_ld32_wait(r);
                }
                const int nbase = tl.n0 + c0;
                if (pr.ksplit > 1) {  // raw partials, column-major per slice: each store is 128 B across the warp
                    if (m < pr.M) {
                        float* part = pr.partial + ((long long)tl.slice * pr.N + nbase) * pr.M + m;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (nbase + j < nlim) part[(long long)j * pr.M] = __uint_as_float(r[j]);
                    }
                    if constexpr (kCfg != 2)
                        if (c0 + 32 < pr.n_tile) tmem_ld32_issue(tbase + c0 + 32, r);
                    continue;
                }
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = pr.alpha * __uint_as_float(r[j]);
                if constexpr (kCfg != 2)
                    if (c0 + 32 < pr.n_tile) tmem_ld32_issue(tbase + c0 + 32, r);
                if (pr.rs) {
                    const float sr = (m < pr.M) ? pr.rs[m] : 0.f;
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= sr;
                }
                if (pr.cs) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] *= (nbase + j < nlim) ? pr.cs[nbase + j] : 0.f;
                }
                if constexpr (kCfg == 2) {
                    const int slot = chunk_no % kCinRing;  // its cp.async group was awaited with the TMEM load
                    unsigned char* cs = ring + slot * kChunkBytes;
                    __syncwarp();
#pragma unroll
                    for (int j4 = 0; j4 < 32; j4 += 4) {
                        float4* pc = reinterpret_cast<float4*>(cs + sw128(lane, j4));
                        const float4 c4 = *pc;
                        v[j4] = fmaf(pr.beta, c4.x, v[j4]);
                        v[j4 + 1] = fmaf(pr.beta, c4.y, v[j4 + 1]);
                        v[j4 + 2] = fmaf(pr.beta, c4.z, v[j4 + 2]);
                        v[j4 + 3] = fmaf(pr.beta, c4.w, v[j4 + 3]);
                        *pc = make_float4(v[j4], v[j4 + 1], v[j4 + 2], v[j4 + 3]);  // the output chunk, in place
                    }
                    const bool full_off = !(diag && nbase <= mbase + 31);  // strictly above the diagonal block
                    unsigned char* ms = mir + (chunk_no & 1) * kChunkBytes;
                    if (full_off) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) *reinterpret_cast<float*>(ms + sw128(j, lane)) = v[j];
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) {
                            const CUtensorMap* om = maps + kMapsPerProb * tl.prob + 4;
                            tma_store_2d(om, cs, nbase, mbase);  // chunk (m, n)
                            tma_store_2d(om, ms, mbase, nbase);  // mirror (n, m)
                        }
                    } else {
                        __syncwarp();
                        if (nbase == mbase) {
                            // the 32 x 32 diagonal chunk: its strictly lower part replaced in place by the mirror of
                            // the upper part (exact symmetry), then stored by TMA like any other chunk
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j > lane) *reinterpret_cast<float*>(cs + sw128(j, lane)) = v[j];
                            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                            __syncwarp();
                            if (lane == 0) tma_store_2d(maps + kMapsPerProb * tl.prob + 4, cs, nbase, mbase);
                        }
                        // chunks below the diagonal block are the mirrors of chunks above it: nothing to store
                    }
                    if (lane == 0) {
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        // the previous chunk's stores have read their smem: its ring slot and mirror buffer are free
                        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    }
                    __syncwarp();
                    cin_issue((chunk_no + kCinRing - 1) % kCinRing);
                    ++chunk_no;
                    continue;
                }
                if (pr.beta != 0.f) {
                    float cv[32];
                    chunk_load(cv, pr.Cin, pr.ldcin, pr.cin_t, mbase, nbase, pr.M, nlim, tile, lane);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = fmaf(pr.beta, cv[j], v[j]);
                }
                if (pr.gamma != 0.f) {
                    float dv[32];
                    chunk_load(dv, pr.Din, pr.lddin, pr.din_t, mbase, nbase, pr.M, nlim, tile, lane);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = fmaf(pr.gamma, dv[j], v[j]);
                }
#pragma unroll 1
                for (int o = 0; o < 2; ++o) {  // (value, lo) plane pairs 0/2 and 1/3
                    float* ph = pr.o[o];
                    float* pl = pr.o[o + 2];
                    if (ph && pl && pr.to[o] == pr.to[o + 2] && pr.ldo[o] == pr.ldo[o + 2]) {
                        chunk_store_pair(v, ph, pl, pr.ldo[o], pr.to[o], mbase, nbase, pr.M, nlim, diag,
                                         pr.sym != 0, tile, lane);
                    } else {
                        if (ph)
                            chunk_store(v, ph, pr.ldo[o], pr.to[o], false, mbase, nbase, pr.M, nlim, diag,
                                        pr.sym != 0, tile, lane);
                        if (pl)
                            chunk_store(v, pl, pr.ldo[o + 2], pr.to[o + 2], true, mbase, nbase, pr.M, nlim, diag,
                                        pr.sym != 0, tile, lane);
                    }
                }
            }
            tc_fence_before();
            if constexpr (k2) {
                __syncwarp();
                if (lane == 0) {
                    if (crank != 0) mbar_arrive_remote(&bars->tmem_empty[acc], 0);
                    else mbar_arrive(&bars->tmem_empty[acc]);
                }
            } else {
                mbar_arrive(&bars->tmem_empty[acc]);
            }
          }
        }
        if (kCfg == 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    if constexpr (k2) {
        tc_fence_before();
        __syncwarp();  // the single-lane roles rejoin their warps before the aligned cluster barrier
        cluster_sync_all();  // neither CTA leaves (or frees its TMEM) while the pair's MMAs / remote arrivals may touch it
    } else {
        __syncthreads();
    }
    if (warp == 1) {
        tc_fence_after();
        if constexpr (k2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// Deterministic split-K reduction (fixed slice order) + the full epilogue, one 32x32 output tile per block:
// partials (column-major per slice) are summed with coalesced loads along m, the tile is staged in smem, and every
// output plane leaves coalesced -- along m for transposed layouts, along n (read transposed) for row-major ones.
__global__ void __launch_bounds__(256) tc_reduce_kernel(const TcProb* __restrict__ probs,
                                                        const TcRed* __restrict__ red, int nred, long long total) {
    __shared__ float tile[32][33];
    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;  // 8 warps
    for (long long tt = blockIdx.x; tt < total; tt += gridDim.x) {
        int lo = 0, hi = nred - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (red[mid].off <= tt) lo = mid; else hi = mid - 1;
        }
        const TcProb& pr = probs[red[lo].prob];
        const int local = (int)(tt - red[lo].off);
        const int tn = local / red[lo].tiles_m, tm = local - tn * red[lo].tiles_m;
        const int m0 = tm * 32, n0 = tn * 32;
        const long long mn = (long long)pr.M * pr.N;
        __syncthreads();  // previous tile's reads of `tile` are done
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int nl = wy + 8 * u, m = m0 + lane, n = n0 + nl;
            float v = 0.f;
            if (m < pr.M && n < pr.N) {
                const float* part = pr.partial + (long long)n * pr.M + m;
                float s0 = part[0], s1 = 0.f, s2 = 0.f, s3 = 0.f;
                int k = 1;
                for (; k + 3 < pr.ksplit; k += 4) {  // fixed association: ((s0 + s1) + (s2 + s3))
                    const float a = part[k * mn], b = part[(k + 1) * mn], c = part[(k + 2) * mn],
                                d = part[(k + 3) * mn];
                    s0 += a; s1 += b; s2 += c; s3 += d;
                }
                for (; k < pr.ksplit; ++k) s0 += part[k * mn];
                v = epi_value(pr, m, n, (s0 + s1) + (s2 + s3));
            }
            tile[nl][lane] = v;
        }
        __syncthreads();
#pragma unroll 1
        for (int o = 0; o < 4; ++o) {
            float* p = pr.o[o];
            if (!p) continue;
            const bool islo = pr.is_lo[o] != 0;
            const long long ld = pr.ldo[o];
            if (pr.to[o]) {  // p[n * ld + m]: along m
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int nl = wy + 8 * u, m = m0 + lane, n = n0 + nl;
                    if (m < pr.M && n < pr.N) p[(long long)n * ld + m] = lo_or(tile[nl][lane], islo);
                }
            } else {  // p[m * ld + n]: along n
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int ml = wy + 8 * u, m = m0 + ml, n = n0 + lane;
                    if (m < pr.M && n < pr.N) p[(long long)m * ld + n] = lo_or(tile[lane][ml], islo);
                }
            }
        }
    }
}

// One descriptor per blockIdx.y; work items are (row, 2 KB chunk) pairs spread over the warps of the descriptor's
// blocks, float4 accesses (four in flight per lane) when every row involved is 16-byte aligned.
__global__ void split_kernel(const SplitDesc* __restrict__ descs) {
    const SplitDesc sd = descs[blockIdx.y];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    const bool vec = ((reinterpret_cast<uintptr_t>(sd.src) | reinterpret_cast<uintptr_t>(sd.hi) |
                       reinterpret_cast<uintptr_t>(sd.lo) | (uintptr_t)(sd.lds * 4) | (uintptr_t)(sd.ldd * 4)) & 15) == 0;
    const int c4 = vec ? sd.cols / 4 : 0;
    // chunks: 2 KB float4 chunks, then 1 KB scalar chunks for the rest (a whole unaligned row), 8 loads in flight
    const int nvec = (c4 + 127) / 128, nsc = (sd.cols - 4 * c4 + 255) / 256, chunks = nvec + nsc;
    const long long items = (long long)sd.rows * chunks;
    for (long long it = blockIdx.x * wpb + warp; it < items; it += (long long)gridDim.x * wpb) {
        const int r = (int)(it / chunks), ch = (int)(it - (long long)r * chunks);
        const float* s = sd.src + (long long)r * sd.lds;
        float* h = sd.hi ? sd.hi + (long long)r * sd.ldd : nullptr;
        float* l = sd.lo ? sd.lo + (long long)r * sd.ldd : nullptr;
        if (ch >= nvec) {
            const int cb = 4 * c4 + (ch - nvec) * 256 + lane;
            float xs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (cb + 32 * u < sd.cols) xs[u] = s[cb + 32 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int c = cb + 32 * u;
                if (c >= sd.cols) break;
                if (h) h[c] = xs[u];
                if (l) l[c] = xs[u] - tf32_trunc(xs[u]);
            }
            continue;
        }
        const int c0 = ch * 128 + lane;
        float4 xs[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (c0 + 32 * u < c4) xs[u] = reinterpret_cast<const float4*>(s)[c0 + 32 * u];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = c0 + 32 * u;
            if (c >= c4) break;
            const float4 x = xs[u];
            if (h) reinterpret_cast<float4*>(h)[c] = x;
            if (l)
                reinterpret_cast<float4*>(l)[c] =
                    make_float4(x.x - tf32_trunc(x.x), x.y - tf32_trunc(x.y), x.z - tf32_trunc(x.z),
                                x.w - tf32_trunc(x.w));
        }
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

CUtensorMap make_map(const float* base, int inner, int outer, long long ld_elems, int box_inner, int box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B) {
    RKFAC_REQUIRE(base && (ld_elems * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0,
                  RKFAC_INVALID_ARGUMENT, "TMA operand needs a 16-byte aligned base and row pitch");
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)(ld_elems * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RKFAC_REQUIRE(r == CUDA_SUCCESS, RKFAC_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
    return m;
}

}  // namespace

bool tc_operand_ok(const float* p, long long ld) {
    return p && (ld * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(p) % 16) == 0;
}

int TcGemm::add(const TcProblemDesc& d) {
    RKFAC_REQUIRE(d.M > 0 && d.N > 0 && d.K > 0, RKFAC_INVALID_ARGUMENT, "empty tc problem");
    RKFAC_REQUIRE(!d.sym || d.M == d.N, RKFAC_INVALID_ARGUMENT, "sym tc problem needs M == N");
    RKFAC_REQUIRE(!(two_cta_ && d.sym), RKFAC_INVALID_ARGUMENT, "CTA-pair tc problems cannot be symmetric");
    TcProb p{};
    p.M = d.M; p.N = d.N; p.K = d.K; p.kblocks = (int)ceil_div(d.K, kBK); p.sym = d.sym;
    p.alpha = d.alpha; p.beta = d.beta; p.gamma = d.gamma; p.rs = d.rs; p.cs = d.cs;
    p.Cin = d.Cin; p.ldcin = d.ldcin; p.cin_t = d.cin_t; p.Din = d.Din; p.lddin = d.lddin; p.din_t = d.din_t;
    const TcOut outs[4] = {d.out0, d.out1, d.lo0, d.lo1};
    for (int o = 0; o < 4; ++o) {
        p.o[o] = outs[o].p; p.ldo[o] = outs[o].ld; p.to[o] = outs[o].t; p.is_lo[o] = o >= 2;
    }
    const int prob = (int)probs_.size();
    // tiles: M in 128-row tiles; N in <=256-row tiles (multiples of 16); sym: square 128x128 upper tiles
    int per, ntn;
    if (d.sym) { per = 128; ntn = (int)ceil_div(d.N, 128); }
    else {
        const int maxbn = d.max_n_tile > 0 ? std::min(kMaxBN, d.max_n_tile) : kMaxBN;
        ntn = (int)ceil_div(d.N, maxbn);
        per = (int)ceil_div(ceil_div(d.N, ntn), 16) * 16;
    }
    p.n_tile = per;
    const int ntm = (int)ceil_div(d.M, kBM);
    const int mn_tiles = d.sym ? ntm * (ntm + 1) / 2 : ntm * ntn;
    int ks = d.ksplit;
    if (ks <= 0) {  // fixed per shape, so results never depend on the batch composition
        ks = 1;
        // long-K problems with few output tiles: >= 8 CTAs per problem, >= 32 K blocks a slice
        while (mn_tiles * ks < 8 && p.kblocks / (2 * ks) >= 32) ks *= 2;
        // accuracy: the tensor core's FP32 accumulation truncates, so the error of one TMEM accumulation chain
        // grows linearly with its length (tools/tc_acc.cu: 3xTF32 rel. error 7.5e-6 at K = 1024, 2.9e-5 at 4096);
        // slices of at most `slice_k` K are summed in FP32 on the CUDA cores by the split-K reduction
        static const int env_slice = [] {
            const char* e = std::getenv("RKFAC_TC_SLICE_K");
            return e ? std::atoi(e) : 0;
        }();
        const int slice_k = d.slice_k > 0 ? d.slice_k : env_slice;
        if (slice_k > 0 && !d.sym) ks = std::max(ks, (int)ceil_div(p.kblocks, std::max(1, slice_k / kBK)));
    }
    RKFAC_REQUIRE(!(d.sym && ks > 1), RKFAC_INVALID_ARGUMENT, "sym tc problem cannot be split");
    p.ksplit = ks;
    const int kper = (int)ceil_div(p.kblocks, ks);
    p.a_conv = d.A_lo ? 0 : 1;
    p.b_conv = d.B_lo ? 0 : 1;
    p.single = d.single;
    maps_.push_back(make_map(d.A, d.K, d.M, d.lda, kBK, kBM));
    maps_.push_back(make_map(d.A_lo ? d.A_lo : d.A, d.K, d.M, d.lda, kBK, kBM));
    const int bbox = two_cta_ ? per / 2 : per;  // CTA pairs: each CTA loads half of the B tile's rows
    maps_.push_back(make_map(d.B, d.K, d.N, d.ldb, kBK, bbox));
    maps_.push_back(make_map(d.B_lo ? d.B_lo : d.B, d.K, d.N, d.ldb, kBK, bbox));
    const bool out_tma = d.out0.p && d.out0.t == 0 && tc_operand_ok(d.out0.p, d.out0.ld);
    maps_.push_back(out_tma ? make_map(d.out0.p, d.N, d.M, d.out0.ld, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B)
                            : make_map(d.A, d.K, d.M, d.lda, kBK, kBM));
    for (int s = 0; s < ks; ++s) {
        const int kb0 = s * kper, kb1 = std::min(p.kblocks, kb0 + kper);
        if (kb0 >= kb1) continue;
        // tall problems (>= 8 row tiles, unsplit, not symmetric): pairs of row tiles share each B tile (halves the
        // L2->SM traffic of B, the re-read operand); the accumulation order per element is unchanged (bitwise)
        // (long K only: a pair occupies both TMEM accumulators, so its epilogue cannot overlap the next tile's
        // mainloop -- for short-K products such as Y L^-T (K = w) that serialisation costs more than the B re-read)
        static const int pair_min_kb = [] {
            const char* e = std::getenv("RKFAC_TC_PAIR_MIN_KB");
            return e ? std::atoi(e) : 48;
        }();
        const bool pairs = !d.sym && ks == 1 && ntm >= 8 && !two_cta_ && (kb1 - kb0) >= pair_min_kb;
        // units of 128 rows per tile: single CTA 1 (2 when paired); CTA pairs 2
        const int unit = two_cta_ ? 2 : 1;
        for (int tn = 0; tn < ntn; ++tn)
            for (int tm = 0; tm < ntm;) {
                if (d.sym && tn < tm) { tm += unit; continue; }
                TcTile t{};
                t.prob = prob; t.m0 = tm * kBM; t.n0 = tn * per; t.kb0 = kb0; t.kb1 = kb1; t.slice = s;
                t.pair = (pairs && tm + unit < ntm) ? 1 : 0;
                tiles_.push_back(t);
                tm += t.pair ? 2 * unit : unit;
            }
    }
    probs_.push_back(p);
    TcProblemDesc kept = d;
    kept.ksplit = ks;  // a re-add (finalize's N split) keeps the K slicing, hence the arithmetic
    descs_.push_back(kept);
    return prob;
}

// CTA pairs that can be resident at once (TPCs with both SMs enabled)
int TcGemm::pair_slots() {
    static const int max_pairs = [] {
        auto k = tc_gemm_kernel<3>;
        const size_t smem = smem_bytes();
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(2 * kNumSMs);
        lc.blockDim = dim3(kThreads);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k, &lc) != cudaSuccess || n <= 0) n = kNumSMs / 2;
        if (std::getenv("RKFAC_TC_DEBUG")) fprintf(stderr, "tc_gemm: %d CTA pairs resident\n", n);
        return n;
    }();
    return max_pairs;
}

void TcGemm::finalize() {
    // A grid that leaves most SMs idle (a plan with few factors owning its GPU: a multi-GPU shard, a single-factor
    // call) gets narrower N tiles until its tiles fill at least half the SMs.  Every output element keeps its K order
    // (the N split only changes which CTA owns it), so the result is bitwise the same as with wide tiles; with a full
    // grid the wide tiles stay (N tiles of 128 measured 46 % slower at VGG16 scale: the A operand is re-read).
    // RKFAC_TC_NSPLIT=0 disables.
    static const bool nsplit_on = [] {
        const char* e = std::getenv("RKFAC_TC_NSPLIT");
        return !(e && e[0] == '0');
    }();
    // CTA pairs need enough 256-row tiles to fill the SM pairs; an under-filled launch (a multi-GPU shard, a
    // single-factor call) goes back to single-CTA tiles and the N split below (same K order per element: bitwise)
    // (only a launch that owns the GPU: a capped one shares it with the other groups' launches)
    if (two_cta_ && cap_ == 0 && (int)tiles_.size() * 2 < pair_slots()) {
        two_cta_ = false;
        std::vector<TcProblemDesc> nd = descs_;
        probs_.clear(); maps_.clear(); tiles_.clear(); descs_.clear();
        for (const auto& d : nd) add(d);
    }
    if (nsplit_on && cap_ == 0 && !two_cta_ && std::getenv("RKFAC_TC_MAX_CTAS") == nullptr) {
        for (int it = 0; it < 4; ++it) {
            long long units = 0;
            for (const auto& t : tiles_) units += t.pair ? 2 : 1;
            if (units * 2 >= kNumSMs) break;
            std::vector<TcProblemDesc> nd = descs_;
            bool changed = false;
            for (size_t i = 0; i < nd.size(); ++i)
                if (!nd[i].sym && probs_[i].n_tile >= 64) {
                    nd[i].max_n_tile = (int)ceil_div(probs_[i].n_tile / 2, 16) * 16;
                    changed = true;
                }
            if (!changed) break;
            probs_.clear(); maps_.clear(); tiles_.clear(); descs_.clear();
            for (const auto& d : nd) add(d);
        }
    }
    // Paired tiles halve the B traffic but also the number of schedulable units: keep them only when the paired
    // units still fill every SM (pairing never changes the arithmetic, so this may depend on the batch).  Splitting
    // the pairs longer than a CTA's average load as well was measured: VGG16's X*Q 3.29 -> 4.01 ms (the B re-reads
    // cost more than the better balance gains).
    {
        long long units = 0, paired_units = (long long)tiles_.size();
        for (const auto& t : tiles_) units += t.pair ? 2 : 1;
        if (paired_units < (two_cta_ ? pair_slots() : kNumSMs)) {
            std::vector<TcTile> split;
            split.reserve((size_t)units);
            for (const auto& t : tiles_) {
                TcTile a = t;
                a.pair = 0;
                split.push_back(a);
                if (t.pair) {
                    a.m0 = t.m0 + (two_cta_ ? 2 : 1) * kBM;
                    split.push_back(a);
                }
            }
            tiles_.swap(split);
        }
        // the 3 x 64 KB configuration also measured faster for the symmetric EA update (0.62 vs 0.84 ms, VGG16)
        bool paired = false, ea = !tiles_.empty();
        for (const auto& t : tiles_) paired = paired || t.pair || probs_[t.prob].sym;
        for (const auto& p : probs_)  // the EA configuration: symmetric axpy problems with an aligned row-major Cin
            ea = ea && p.sym && p.beta != 0.f && p.cin_t == 0 && p.ksplit <= 1 && p.n_tile == kBM && p.Cin &&
                 (p.ldcin % 4) == 0 && (reinterpret_cast<uintptr_t>(p.Cin) % 16) == 0 && p.o[0] && p.to[0] == 0 &&
                 (p.ldo[0] % 4) == 0 && (reinterpret_cast<uintptr_t>(p.o[0]) % 16) == 0 && !p.o[1] && !p.o[2] &&
                 !p.o[3] && !p.rs && !p.cs && p.gamma == 0.f;
        cfg_ = ea ? 2 : (paired ? 1 : 0);
        if (two_cta_) cfg_ = 3;
    }
    // split-K partial buffers
    size_t total = 0;
    for (auto& p : probs_)
        if (p.ksplit > 1) total += (size_t)p.ksplit * p.M * p.N;
    partials_.alloc(std::max<size_t>(total, 1) * sizeof(float));
    size_t off = 0;
    any_split_ = false;
    std::vector<TcRed> red;
    red_total_ = 0;
    for (size_t i = 0; i < probs_.size(); ++i) {
        TcProb& p = probs_[i];
        if (p.ksplit > 1) {
            p.partial = partials_.as<float>() + off;
            off += (size_t)p.ksplit * p.M * p.N;
            any_split_ = true;
            const int tm = (int)ceil_div(p.M, 32), tn = (int)ceil_div(p.N, 32);
            red.push_back(TcRed{red_total_, (int)i, tm});
            red_total_ += (long long)tm * tn;
        }
    }
    nred_ = (int)red.size();
    // LPT over persistent CTAs: tile cost ~ K blocks * (n_tile + epilogue overhead)
    const int ntiles = (int)tiles_.size();
    int cap = cap_ > 0 ? std::min(kNumSMs, cap_) : kNumSMs;
    if (const char* e = std::getenv("RKFAC_TC_MAX_CTAS")) cap = std::max(1, std::min(kNumSMs, std::atoi(e)));
    if (two_cta_) cap = std::max(1, std::min(cap / 2, pair_slots()));  // schedule slots are CTA pairs
    nctas_ = std::max(1, std::min(ntiles, cap));
    std::vector<int> order(ntiles);
    std::iota(order.begin(), order.end(), 0);
    auto cost = [&](int i) {
        const TcTile& t = tiles_[i];
        return (t.pair ? 2.0 : 1.0) * ((double)(t.kb1 - t.kb0) * (probs_[t.prob].n_tile + 16) +
                                        4.0 * probs_[t.prob].n_tile);
    };
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
    up(d_probs_, probs_.data(), sizeof(TcProb) * probs_.size());
    up(d_maps_, maps_.data(), sizeof(CUtensorMap) * maps_.size());
    up(d_tiles_, sched.data(), sizeof(TcTile) * sched.size());
    up(d_begin_, begin.data(), sizeof(int) * begin.size());
    up(d_red_, red.data(), sizeof(TcRed) * red.size());
}

size_t TcGemm::smem_bytes() { return (size_t)kStagesBytesMax + kBarrierBytes + kStageTileBytes + 1024; }

void TcGemm::launch(cudaStream_t s) const {
    if (tiles_.empty()) return;
    const size_t smem = smem_bytes();
    auto k = cfg_ == 3 ? tc_gemm_kernel<3>
                       : (cfg_ == 2 ? tc_gemm_kernel<2> : (cfg_ == 1 ? tc_gemm_kernel<1> : tc_gemm_kernel<0>));
    RKFAC_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (cfg_ == 3) {  // one cluster of two CTAs (a TPC's SM pair) per schedule slot
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(2 * nctas_);
        lc.blockDim = dim3(kThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        RKFAC_CUDA(cudaLaunchKernelEx(&lc, k, (const TcProb*)d_probs_.as<TcProb>(),
                                      (const CUtensorMap*)d_maps_.as<CUtensorMap>(),
                                      (const TcTile*)d_tiles_.as<TcTile>(), (const int*)d_begin_.as<int>()));
    } else {
        k<<<nctas_, kThreads, smem, s>>>(d_probs_.as<TcProb>(), d_maps_.as<CUtensorMap>(), d_tiles_.as<TcTile>(),
                                         d_begin_.as<int>());
    }
    count_launch();
    RKFAC_CHECK_LAUNCH();
    if (any_split_ && !defer_reduce_) {
        const int blocks = (int)std::min<long long>(red_total_, kNumSMs * 8);
        tc_reduce_kernel<<<blocks, 256, 0, s>>>(d_probs_.as<TcProb>(), d_red_.as<TcRed>(), nred_, red_total_);
        count_launch();
        RKFAC_CHECK_LAUNCH();
    }
}

double TcGemm::flops() const {
    double f = 0;
    for (const auto& p : probs_) f += 2.0 * p.M * (double)p.N * p.K * (p.sym ? 0.5 : 1.0);
    return f;
}

void launch_split(const SplitDesc* d_descs, int n, long long total, cudaStream_t s) {
    if (total == 0 || n == 0) return;
    // ~8 row-blocks of 8 warps per SM over all descriptors; blocks past a descriptor's rows exit at once
    const int bx = (int)std::max<long long>(1, std::min<long long>(512, ceil_div(kNumSMs * 8, n)));
    split_kernel<<<dim3(bx, n), 256, 0, s>>>(d_descs);
    count_launch();
    RKFAC_CHECK_LAUNCH();
}

}  // namespace rkfac_b200
