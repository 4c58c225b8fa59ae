// common.cuh -- shared helpers for the rkfac B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/rkfac_b200.h"

namespace rkfac_b200 {

// Internal error type; converted to an rkfac_status at the C-ABI boundary (capi.cu).
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& what) : std::runtime_error(what), status(s) {}
};

#define RKFAC_CUDA(expr)                                                                       \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            throw ::rkfac_b200::Error(RKFAC_CUDA_ERROR, std::string(#expr) + ": " +            \
                                                            cudaGetErrorString(_e));           \
    } while (0)

#define RKFAC_CHECK_LAUNCH() RKFAC_CUDA(cudaGetLastError())

#define RKFAC_REQUIRE(cond, status, msg)                     \
    do {                                                     \
        if (!(cond)) throw ::rkfac_b200::Error(status, msg); \
    } while (0)

constexpr int kNumSMs = 148;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch counter shared by every kernel launch site (reported as gpu_launches by the bench).
uint64_t& launch_counter();
inline void count_launch(uint64_t n = 1) { launch_counter() += n; }

// ---- counter-based RNG, device side (rng.hpp:13-55) ----------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t substream(uint64_t seed, uint64_t a, uint64_t b) {
    return splitmix64(seed ^ splitmix64(a ^ splitmix64(b)));
}

// uniform in (0,1]: ((u >> 11) + 1) * 2^-53 (rng.hpp:42-45)
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t ctr) {
    const uint64_t u = splitmix64(seed ^ splitmix64(ctr));
    return (double)((u >> 11) + 1ULL) * 0x1.0p-53;
}

// Box-Muller, cos branch, counters (ctr, ctr+1) (rng.hpp:51-55); FP64 transcendental math.
__device__ __forceinline__ double gaussian_at(uint64_t seed, uint64_t ctr) {
    const double u1 = uniform_at(seed, ctr);
    const double u2 = uniform_at(seed, ctr + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

// Largest dynamic shared memory a launch of `kernel` may request on the current device
// (opt-in per-block limit minus the kernel's static shared memory).
inline size_t max_dynamic_smem(const void* kernel) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes attr{};
    if (cudaFuncGetAttributes(&attr, kernel) != cudaSuccess) return 0;
    return optin > (int)attr.sharedSizeBytes ? (size_t)(optin - (int)attr.sharedSizeBytes) : 0;
}

// Device buffer with RAII (plan workspaces).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    explicit DevBuf(size_t b) { alloc(b); }
    void alloc(size_t b) {
        release();
        bytes = b;
        if (b) RKFAC_CUDA(cudaMalloc(&p, b));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0;
        return *this;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace rkfac_b200
