// Helpers shared by the CUDA translation units (kernels.cu, kernels_act.cu).
// Each TU defines its own copy of the constant tables (no relocatable device
// code) before including this header; dev::upload_constants() fills both.
#pragma once
#include <mutex>
#include <unordered_map>

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "dash_prim.cuh"

namespace dashgpu {

// Warps per CTA of the activation kernels (one CTA per SM).  Garbling is
// latency-bound and gains from every extra warp up to the shared-memory cap
// (64 KB AES tables + 28 x 5.5 KB label buffers = 218 KB); evaluation is
// fastest at 24 (measured on B200: garble 59.1 -> 55.9 ms from 24 to 28
// warps, eval 13.7 -> 15.2 ms).
#ifndef DASH_GARBLE_WARPS
#define DASH_GARBLE_WARPS 28
#endif
constexpr int kActWarpsGarble = DASH_GARBLE_WARPS;
#ifndef DASH_EVAL_WARPS
#define DASH_EVAL_WARPS 24
#endif
constexpr int kActWarpsEval = DASH_EVAL_WARPS;
constexpr int kTWords = 256 * 32;

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA ") + what + ": " + cudaGetErrorString(e));
}
inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel and size:
// the call costs microseconds, and small launches are latency-bound
inline void smem_attr(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& v = done[fn];
    if (v >= bytes) return;
    ck(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "attr");
    v = bytes;
}

// ---- per-kind CUDA-event timing on the launching stream (kernels.cu owns it)
struct ProfData {
    int on = 0;
    double ms[K_NKINDS] = {};
    uint64_t n[K_NKINDS] = {};
    struct Pending {
        int kind;
        cudaEvent_t a, b;
    };
    std::vector<Pending> pending;
};
ProfData& prof();

struct ProfScope {
    int kind;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(int k, cudaStream_t st) : kind(k), s(st) {
        if (prof().on) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope() {
        if (prof().on) {
            cudaEventRecord(b, s);
            prof().pending.push_back({kind, a, b});
        }
    }
};

// Fills the AES tables at the start of dynamic shared memory (layout in
// dash_device.cuh: 256-byte rows of 32 T0 replicas then 32 T2 replicas).
__device__ __forceinline__ void fill_T(const uint32_t* T0) {
    for (int i = threadIdx.x; i < kTabWords; i += blockDim.x) {
        const uint32_t v = T0[i >> 6];
        s_dyn[i] = (i & 32) ? __funnelshift_l(v, v, 16) : v;
    }
    __syncthreads();
}
constexpr size_t kTabBytes = sizeof(uint32_t) * kTabWords;

}  // namespace dashgpu
