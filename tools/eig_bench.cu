// eig_bench.cu -- times the eigensolver kernels on VGG16-shaped cores (32 factors, w = 230) and prints the
// per-phase clock64 stamps of one tridiagonalisation step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_TRC_TIMING=50 tools/eig_bench.cu \
//        paper_2206_15397_b200/csrc/misc.cu -o build/eig_bench
#include <cstdio>
#include <vector>

#include "../paper_2206_15397_b200/csrc/eig.cu"

using namespace rkfac_b200;

__global__ void make_core(float* A, int n, int nf) {
    const int f = blockIdx.y, i = blockIdx.x;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const int a = min(i, j), b = max(i, j);
        const double u = (double)(splitmix64((uint64_t)f * 977ULL + (uint64_t)a * 131071ULL + b) >> 11) * 0x1.0p-53;
        A[((size_t)f * n + i) * n + j] = (float)((i == j ? 1.0 / (1 + i) : 0.0) + 1e-3 * (u - 0.5));
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 230, nf = argc > 2 ? atoi(argv[2]) : 32, r = n - 10;
    const int np = (n + 3) / 4 * 4;
    float* A;
    cudaMalloc(&A, sizeof(float) * nf * n * n);
    make_core<<<dim3(n, nf), 128>>>(A, n, nf);
    std::vector<EigDesc> h(nf);
    std::vector<void*> bufs;
    auto alloc = [&](size_t b) { void* p; cudaMalloc(&p, b); bufs.push_back(p); return p; };
    for (int f = 0; f < nf; ++f) {
        EigDesc& e = h[f];
        e.n = n; e.r = r; e.A = A + (size_t)f * n * n; e.lda = n;
        e.scratch = (double*)alloc(sizeof(double) * n * (n + 1) / 2);
        e.refl = (double*)alloc(sizeof(double) * n * n);
        e.tau = (double*)alloc(sizeof(double) * n);
        e.dvec = (double*)alloc(sizeof(double) * n);
        e.evec = (double*)alloc(sizeof(double) * n);
        e.evals = (double*)alloc(sizeof(double) * n);
        e.scr = (double*)alloc(sizeof(double) * 4 * n * r);
        e.piv = (unsigned char*)alloc(n * r);
        e.z = (double*)alloc(sizeof(double) * n * r);
        e.Pt = (float*)alloc(sizeof(float) * r * np);
        e.Ptlo = (float*)alloc(sizeof(float) * r * np);
        e.ldpt = np;
    }
    EigDesc* d;
    cudaMalloc(&d, sizeof(EigDesc) * nf);
    cudaMemcpy(d, h.data(), sizeof(EigDesc) * nf, cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) launch_eig(d, nf, n, r, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) launch_eig(d, nf, n, r, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("launch_eig n=%d nf=%d: %.1f us (%s)\n", n, nf, 1e3f * ms / 10, cudaGetErrorString(cudaGetLastError()));
#ifdef RKFAC_TRC_TIMING
    long long t[16];
    cudaMemcpyFromSymbol(t, g_trc, sizeof(t));
    printf("one-barrier step %d: vectors %lld (pv %lld, x %lld, reflector %lld, write %lld), pass %lld, barrier %lld "
           "cycles\n", RKFAC_TRC_TIMING, t[9] - t[8], t[12] - t[8], t[13] - t[12], t[14] - t[13], t[9] - t[14],
           t[10] - t[9], t[11] - t[10]);
    printf("step %d: reflector %lld, B %lld, sync1 %lld, C %lld, sync2 %lld cycles\n", RKFAC_TRC_TIMING, t[1] - t[0],
           t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4]);
    long long bx[8][8];
    cudaMemcpyFromSymbol(bx, g_bx, sizeof(bx));
    for (int b = 7; b >= 0; --b)
        printf("wy block %d: V %lld, G/W %lld, T %lld, TW %lld, Z %lld\n", b, bx[b][1] - bx[b][0], bx[b][2] - bx[b][1],
               bx[b][3] - bx[b][2], bx[b][4] - bx[b][3], bx[b][5] - bx[b][4]);
#endif
    std::vector<double> dv(n);
    cudaMemcpy(dv.data(), h[0].evals, sizeof(double) * 5, cudaMemcpyDeviceToHost);
    printf("evals[0..4] of factor 0: %.6g %.6g %.6g %.6g %.6g\n", dv[0], dv[1], dv[2], dv[3], dv[4]);
    return 0;
}
