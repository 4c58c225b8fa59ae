// chol_bench.cu -- per-phase clock64 profile of cholinv_kernel on VGG16-shaped problems (w = 230, 32 factors).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_PHASE_TIMING -lineinfo \
//        tools/chol_bench.cu -o gpurun_out/chol_bench && gpurun_out/chol_bench [w] [nfactors] [fp64]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2206_15397_b200/csrc/cholqr.cu"

namespace rkfac_b200 {
uint64_t& launch_counter() {
    static uint64_t c = 0;
    return c;
}
}  // namespace rkfac_b200

using namespace rkfac_b200;

__global__ void make_gram(float* G, double* G64, int w, int wp, int d, int nf) {
    // G = Y^T Y / d + 1e-3 I for a deterministic pseudo-random Y (w x d), one CTA row per (factor, i)
    const int f = blockIdx.y, i = blockIdx.x;
    for (int j = threadIdx.x; j < w; j += blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            const double a = (double)((splitmix64((uint64_t)f * 1000003ULL + (uint64_t)i * 7919ULL + k) >> 11)) *
                                 0x1.0p-53 - 0.5;
            const double b = (double)((splitmix64((uint64_t)f * 1000003ULL + (uint64_t)j * 7919ULL + k) >> 11)) *
                                 0x1.0p-53 - 0.5;
            s += a * b;
        }
        s = s / d + (i == j ? 1e-3 : 0.0);
        G[((size_t)f * w + i) * wp + j] = (float)s;
        G64[((size_t)f * w + i) * wp + j] = s;
    }
}

__global__ void spin(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
}

int main(int argc, char** argv) {
    const int w = argc > 1 ? atoi(argv[1]) : 230;
    const int nf = argc > 2 ? atoi(argv[2]) : 32;
    const bool fp64 = argc > 3 && atoi(argv[3]) != 0;
    const int wp = (w + 3) / 4 * 4;
    float *G, *Li, *Llo;
    double *G64, *L64;
    int* flags;
    void* scratch;
    cudaMalloc(&G, sizeof(float) * nf * w * wp);
    cudaMalloc(&G64, sizeof(double) * nf * w * wp);
    cudaMalloc(&Li, sizeof(float) * nf * w * wp);
    cudaMalloc(&Llo, sizeof(float) * nf * w * wp);
    cudaMalloc(&L64, sizeof(double) * nf * w * wp);
    cudaMalloc(&flags, sizeof(int) * nf * (w + 1));
    cudaMalloc(&scratch, sizeof(double) * nf * (size_t)prow(w + 4));
    cudaMemset(Li, 0, sizeof(float) * nf * w * wp);
    cudaMemset(L64, 0, sizeof(double) * nf * w * wp);
    make_gram<<<dim3(w, nf), 128>>>(G, G64, w, wp, 256, nf);
    std::vector<CholDesc> h(nf);
    for (int f = 0; f < nf; ++f) {
        CholDesc& c = h[f];
        c.w = w;
        c.G = fp64 ? (const void*)(G64 + (size_t)f * w * wp) : (const void*)(G + (size_t)f * w * wp);
        c.ldg = wp;
        c.Linv = fp64 ? (void*)(L64 + (size_t)f * w * wp) : (void*)(Li + (size_t)f * w * wp);
        c.ldl = wp;
        c.Linv_lo = fp64 ? nullptr : (void*)(Llo + (size_t)f * w * wp);
        c.flags = flags + f * (w + 1);
        c.nflags = flags + f * (w + 1) + w;
        c.scratch = (char*)scratch + (size_t)f * prow(w + 4) * 8;
    }
    CholDesc* d;
    cudaMalloc(&d, sizeof(CholDesc) * nf);
    cudaMemcpy(d, h.data(), sizeof(CholDesc) * nf, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 3; ++it) launch_cholinv(d, nf, w, fp64, fp64, fp64 ? 1e-13 : 1e-5, 0);
#ifdef RKFAC_PHASE_TIMING
    {
        std::vector<long long> z(64 * 64, 0);
        cudaMemcpyToSymbol(g_chol_phase, z.data(), sizeof(long long) * 64 * 64);
        launch_cholinv(d, nf, w, fp64, fp64, fp64 ? 1e-13 : 1e-5, 0);
        cudaDeviceSynchronize();
    }
#endif
    // per-launch device time (the launcher's host work must not be what is measured)
    const int reps = 20;
    float ms = 0.f;
    for (int it = 0; it < reps; ++it) {
        spin<<<1, 32>>>(200000);  // keeps the GPU busy while the host enqueues the launch below
        cudaEventRecord(e0);
        launch_cholinv(d, nf, w, fp64, fp64, fp64 ? 1e-13 : 1e-5, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float m = 0.f;
        cudaEventElapsedTime(&m, e0, e1);
        ms += m;
    }
    const cudaError_t err = cudaGetLastError();
    printf("w=%d nf=%d fp64=%d: %.1f us per launch (%s)\n", w, nf, (int)fp64, 1e3f * ms / reps, cudaGetErrorString(err));
#ifdef RKFAC_PHASE_TIMING
    std::vector<long long> ph(64 * 64);  // stamps of the single launch above
    cudaMemcpyFromSymbol(ph.data(), g_chol_phase, sizeof(long long) * 64 * 64);
    // phase stamps of blocks 0..3 (one cluster, or four single-CTA factors) in time order, cycles since block 0's mark 0
    for (int blk = 0; blk < 4; ++blk) {
        const long long* p = ph.data() + blk * 64;
        const long long t0 = ph[0];
        std::vector<std::pair<long long, int>> ev;
        for (int k = 0; k < 64; ++k)
            if (p[k] >= t0 && p[k] > 0) ev.push_back({p[k], k});
        std::sort(ev.begin(), ev.end());
        printf("block %d:", blk);
        long long prev = t0;
        for (auto& e : ev) {
            printf(" %d:+%lld", e.second, e.first - prev);
            prev = e.first;
        }
        printf("  (total %lld)\n", ev.empty() ? 0 : ev.back().first - t0);
    }
#endif
    // verify: max |Linv G Linv^T - I| on the first and last factor
    for (int f : {0, nf - 1}) {
        std::vector<double> hg((size_t)w * w), hl((size_t)w * wp);
        if (fp64) {
            std::vector<double> a((size_t)w * wp), l((size_t)w * wp);
            cudaMemcpy(a.data(), G64 + (size_t)f * w * wp, sizeof(double) * w * wp, cudaMemcpyDeviceToHost);
            cudaMemcpy(l.data(), L64 + (size_t)f * w * wp, sizeof(double) * w * wp, cudaMemcpyDeviceToHost);
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j) hg[(size_t)i * w + j] = a[(size_t)i * wp + j];
            hl = l;
        } else {
            std::vector<float> a((size_t)w * wp), l((size_t)w * wp);
            cudaMemcpy(a.data(), G + (size_t)f * w * wp, sizeof(float) * w * wp, cudaMemcpyDeviceToHost);
            cudaMemcpy(l.data(), Li + (size_t)f * w * wp, sizeof(float) * w * wp, cudaMemcpyDeviceToHost);
            for (int i = 0; i < w; ++i)
                for (int j = 0; j < w; ++j) hg[(size_t)i * w + j] = a[(size_t)i * wp + j];
            for (size_t i = 0; i < l.size(); ++i) hl[i] = l[i];
        }
        std::vector<double> t((size_t)w * w, 0.0);
        for (int i = 0; i < w; ++i)
            for (int k = 0; k < w; ++k) {
                double s = 0;
                for (int j = 0; j <= i; ++j) s += hl[(size_t)i * wp + j] * hg[(size_t)j * w + k];
                t[(size_t)i * w + k] = s;
            }
        double err2 = 0, upper = 0;
        for (int i = 0; i < w; ++i)
            for (int k = 0; k < w; ++k) {
                double s = 0;
                for (int j = 0; j < w; ++j) s += t[(size_t)i * w + j] * hl[(size_t)k * wp + j];
                err2 = fmax(err2, fabs(s - (i == k ? 1.0 : 0.0)));
                if (k > i && k < wp) upper = fmax(upper, fabs(hl[(size_t)i * wp + k]));
            }
        printf("factor %d: max |Linv G Linv^T - I| = %.3e, max |upper(Linv)| = %.1e\n", f, err2, upper);
    }
    return 0;
}
