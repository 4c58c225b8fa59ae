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
    cudaEventRecord(e0);
    const int reps = 20;
    for (int it = 0; it < reps; ++it) launch_cholinv(d, nf, w, fp64, fp64, fp64 ? 1e-13 : 1e-5, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const cudaError_t err = cudaGetLastError();
    printf("w=%d nf=%d fp64=%d: %.1f us per launch (%s)\n", w, nf, (int)fp64, 1e3f * ms / reps, cudaGetErrorString(err));
#ifdef RKFAC_PHASE_TIMING
    std::vector<long long> ph(64 * 64);
    cudaMemcpyFromSymbol(ph.data(), g_chol_phase, sizeof(long long) * 64 * 64);
    // phase stamps of block 0 in time order (cycles since mark 0)
    const long long* p = ph.data();
    std::vector<std::pair<long long, int>> ev;
    for (int k = 1; k < 64; ++k)
        if (p[k] > p[0]) ev.push_back({p[k], k});
    std::sort(ev.begin(), ev.end());
    long long prev = p[0];
    printf("phase cycles (block 0):\n");
    for (auto& e : ev) {
        printf("  mark %2d: +%7lld  (cum %7lld)\n", e.second, e.first - prev, e.first - p[0]);
        prev = e.first;
    }
#endif
    // verify: max |Linv G Linv^T - I| on factor 0 (FP32 only)
    if (!fp64) {
        std::vector<float> hg((size_t)w * w), hl((size_t)w * wp);
        std::vector<float> hgp((size_t)w * wp);
        cudaMemcpy(hgp.data(), G, sizeof(float) * w * wp, cudaMemcpyDeviceToHost);
        for (int i = 0; i < w; ++i)
            for (int j = 0; j < w; ++j) hg[(size_t)i * w + j] = hgp[(size_t)i * wp + j];
        cudaMemcpy(hl.data(), Li, sizeof(float) * w * wp, cudaMemcpyDeviceToHost);
        std::vector<double> t((size_t)w * w, 0.0);
        for (int i = 0; i < w; ++i)
            for (int k = 0; k < w; ++k) {
                double s = 0;
                for (int j = 0; j < w; ++j) s += (double)hl[(size_t)i * wp + j] * hg[(size_t)j * w + k];
                t[(size_t)i * w + k] = s;
            }
        double err2 = 0;
        for (int i = 0; i < w; ++i)
            for (int k = 0; k < w; ++k) {
                double s = 0;
                for (int j = 0; j < w; ++j) s += t[(size_t)i * w + j] * hl[(size_t)k * wp + j];
                err2 = fmax(err2, fabs(s - (i == k ? 1.0 : 0.0)));
            }
        printf("max |Linv G Linv^T - I| = %.3e\n", err2);
    }
    return 0;
}
