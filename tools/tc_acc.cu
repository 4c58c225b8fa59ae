// tc_acc.cu -- accuracy of the 3xTF32 tcgen05 grouped GEMM against an FP64 host product, as a function of K and of
// the split-K factor (FP32 partial sums reduced on the CUDA cores).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tc_acc.cu -lcuda -o gpurun_out/tc_acc
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../paper_2206_15397_b200/csrc/tc_gemm.cu"

namespace rkfac_b200 {
uint64_t& launch_counter() {
    static uint64_t c = 0;
    return c;
}
}  // namespace rkfac_b200
using namespace rkfac_b200;

int main() {
    const int M = 256, N = 240;
    for (int K : {1024, 4096, 16384}) {
        std::mt19937_64 rng(K);
        std::uniform_real_distribution<float> U(-1.f, 1.f);
        std::vector<float> A((size_t)M * K), B((size_t)N * K), Al(A.size()), Bl(B.size());
        for (auto& v : A) v = U(rng);
        for (auto& v : B) v = U(rng) + 0.25f;  // non-zero mean: sums do not cancel
        auto lo = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float h; memcpy(&h, &u, 4); return x - h; };
        for (size_t i = 0; i < A.size(); ++i) Al[i] = lo(A[i]);
        for (size_t i = 0; i < B.size(); ++i) Bl[i] = lo(B[i]);
        auto hi = [](float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float h; memcpy(&h, &u, 4); return h; };
        // accumulation-only error: 1xTF32 products (lo planes zero) against the exact FP64 sum of TF32 products
        std::vector<double> T64((size_t)M * N, 0.0);
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) s += (double)hi(A[(size_t)m * K + k]) * hi(B[(size_t)n * K + k]);
                T64[(size_t)m * N + n] = s;
            }
        std::vector<double> C64((size_t)M * N, 0.0);
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < K; ++k) s += (double)A[(size_t)m * K + k] * B[(size_t)n * K + k];
                C64[(size_t)m * N + n] = s;
            }
        float *dA, *dB, *dAl, *dBl, *dC;
        cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
        cudaMalloc(&dAl, A.size() * 4); cudaMalloc(&dBl, B.size() * 4);
        cudaMalloc(&dC, (size_t)M * N * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dAl, Al.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dBl, Bl.data(), B.size() * 4, cudaMemcpyHostToDevice);
        {
            float* dZ;
            cudaMalloc(&dZ, std::max(A.size(), B.size()) * 4);
            cudaMemset(dZ, 0, std::max(A.size(), B.size()) * 4);
            TcGemm g;
            TcProblemDesc p;
            p.M = M; p.N = N; p.K = K;
            p.A = dA; p.A_lo = dZ; p.lda = K;
            p.B = dB; p.B_lo = dZ; p.ldb = K;
            p.out0.p = dC; p.out0.ld = N; p.out0.t = 0;
            p.ksplit = 1;
            g.add(p);
            g.finalize();
            g.launch(0);
            cudaDeviceSynchronize();
            std::vector<float> C((size_t)M * N);
            cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
            double num = 0, den = 0, bias = 0;
            for (size_t i = 0; i < C.size(); ++i) {
                const double e = (double)C[i] - T64[i];
                num += e * e; den += T64[i] * T64[i]; bias += e;
            }
            printf("K=%6d 1xTF32 accumulation only: rel fro err %.3e  mean err %.3e\n", K, std::sqrt(num / den),
                   bias / C.size());
            cudaFree(dZ);
        }
        for (int ks : {1, 4, 16}) {
            for (int conv = 0; conv < 1; ++conv) {
                TcGemm g;
                TcProblemDesc p;
                p.M = M; p.N = N; p.K = K;
                p.A = dA; p.A_lo = conv ? nullptr : dAl; p.lda = K;
                p.B = dB; p.B_lo = dBl; p.ldb = K;
                p.out0.p = dC; p.out0.ld = N; p.out0.t = 0;
                p.ksplit = ks;
                g.add(p);
                g.finalize();
                g.launch(0);
                cudaDeviceSynchronize();
                std::vector<float> C((size_t)M * N);
                cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
                double num = 0, den = 0, mx = 0, bias = 0;
                for (size_t i = 0; i < C.size(); ++i) {
                    const double e = (double)C[i] - C64[i];
                    num += e * e; den += C64[i] * C64[i]; bias += e;
                    mx = std::max(mx, std::fabs(e) / std::sqrt((double)K));
                }
                printf("K=%6d ksplit=%2d conv=%d: rel fro err %.3e  mean err %.3e  (%s)\n", K, ks, conv,
                       std::sqrt(num / den), bias / C.size(), cudaGetErrorString(cudaGetLastError()));
            }
        }
        cudaFree(dA); cudaFree(dB); cudaFree(dAl); cudaFree(dBl); cudaFree(dC);
    }
    return 0;
}
