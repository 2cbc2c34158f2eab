// Activation-layer kernels (ReLU / SignAct gadget tapes), garble and eval.
// One thread = one (inference, element); a warp = 32 consecutive elements of
// one inference, so every tape branch, modulus and offset load is warp-uniform.
// CTA = 8 warps; shared memory = replicated AES T-table (32 KB) + per-lane
// compressed label slots.
#include "dash_common.hpp"

namespace dashgpu {
__constant__ ModC c_mod[MAXMOD + 1];
__constant__ uint32_t c_pi_rk[44];
__constant__ uint16_t c_modslot[MAXMOD + 1];
__device__ uint32_t g_T0[256];
}  // namespace dashgpu
#define DASH_CONST_DEFINED 1
#include <algorithm>
#include <cstring>

#include "kernels_common.cuh"

namespace dashgpu {

namespace {

// Dynamic shared memory per CTA: AES tables (64 KB) + per-lane label
// buffers X (NWMAX words), K (4 words: the Z_2-sized y operand of half
// gates, checked by the tape builder), A (NWMAX words); word w of a buffer at
// base + w*32 + lane.  28 warps x 5.5 KB + 64 KB = 218 KB.
constexpr int kLaneWords = 2 * NWMAX + 4;
constexpr int kBufWords = kLaneWords * 32;

template <bool G>
__global__ void __launch_bounds__(kActWarps * 32, 1)
    act_kernel(const ActParams* __restrict__ layers, ItemMap map, uint32_t* counter) {
    uint32_t* L = s_dyn + kTabWords;
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t total = map.base[map.n];
    uint32_t* lb = L + (uint64_t)warp * kBufWords + lane;
    Elt e;
    e.X = LB{lb, 32};
    e.K = LB{lb + NWMAX * 32, 32};
    e.A = LB{lb + (NWMAX + 4) * 32, 32};
    e.t = make_tab(nullptr, lane);
    // first round: item = warp * grid + cta spreads small launches over all
    // SMs; afterwards warps pull items from the counter (balanced tail)
    uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t first = kActWarps * gridDim.x;
    for (;;) {
        if (item >= total) break;
        uint32_t li = 0;
        while (li + 1 < map.n && item >= map.base[li + 1]) ++li;
        const uint32_t local = item - map.base[li];
        const ActParams& P = layers[li];
        e.b = local / map.wpi[li];
        e.u = (local % map.wpi[li]) * 32 + lane;
        e.rk = nullptr;
        e.mult = nullptr;
        if (e.u < P.E) act_element<G>(P, e);
        __syncwarp();
        uint32_t next = 0;
        if (lane == 0) next = first + atomicAdd(counter, 1u);
        item = __shfl_sync(0xffffffffu, next, 0);
    }
}

// All k lanes of one layer in one launch: thread (lane i, element u) of
// inference blockIdx.y; elements are padded to whole warps per lane so the
// modulus is warp-uniform.
struct Primes {
    uint16_t p[MAXK];
};
__global__ void __launch_bounds__(256) act_out_kernel(ActParams P, Primes pr, uint32_t epad) {
    fill_T(g_T0);
    const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t i = idx / epad, u = idx % epad;
    if (i >= (uint32_t)P.k || u >= P.E) return;
    uint32_t buf[2][NWMAX];
    act_output_thread(P, blockIdx.y, u, (int)i, pr.p[i], LB{buf[0], 1}, LB{buf[1], 1},
                      make_tab(nullptr, threadIdx.x & 31u));
}

}  // namespace

void upload_act(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0) {
    ck(cudaMemcpyToSymbol(c_mod, mods, sizeof(ModC) * (MAXMOD + 1)), "c_mod(act)");
    ck(cudaMemcpyToSymbol(c_pi_rk, pi_rk, sizeof(uint32_t) * 44), "c_pi_rk(act)");
    ck(cudaMemcpyToSymbol(c_modslot, modslot, sizeof(uint16_t) * (MAXMOD + 1)), "c_modslot(act)");
    ck(cudaMemcpyToSymbol(g_T0, T0, sizeof(uint32_t) * 256), "g_T0(act)");
}

static uint32_t* act_counter() {
    static uint32_t* counter = nullptr;
    if (!counter) ck(cudaMalloc(&counter, 64 * sizeof(uint32_t)), "counter");
    return counter;
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        ck(cudaGetDevice(&dev), "dev");
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    }
    return sms;
}

void launch_act_multi(const ActParams* dev_layers, const ActParams* host_layers, int n, bool garble, void* st) {
    if (n > MAXACT) throw std::runtime_error("too many activation layers for one launch");
    ItemMap map;
    std::memset(&map, 0, sizeof map);
    map.n = (uint32_t)n;
    for (int i = 0; i < n; ++i) {
        map.wpi[i] = (host_layers[i].E + 31) / 32;
        map.base[i + 1] = map.base[i] + host_layers[i].B * map.wpi[i];
    }
    if (map.base[n] == 0) return;
    ProfScope ps(garble ? K_ACT_GARBLE : K_ACT_EVAL, S(st));
    // one CTA per SM (the first round strides items across SMs), never fewer
    // CTAs than needed to give every item its own SM when items < #SMs
    const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)sm_count(), map.base[n]);
    const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)kActWarps * kBufWords;
    uint32_t* counter = act_counter();
    ck(cudaMemsetAsync(counter, 0, sizeof(uint32_t), S(st)), "counter reset");
    if (garble) {
        ck(cudaFuncSetAttribute(act_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        act_kernel<true><<<grid, kActWarps * 32, smem, S(st)>>>(dev_layers, map, counter);
    } else {
        ck(cudaFuncSetAttribute(act_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        act_kernel<false><<<grid, kActWarps * 32, smem, S(st)>>>(dev_layers, map, counter);
    }
    ck(cudaGetLastError(), "act launch");
}

void launch_act_outputs(const ActParams& P, const uint16_t* primes, void* st) {
    if (P.B == 0 || P.E == 0) return;
    ProfScope ps(K_SETUP, S(st));
    Primes pr;
    for (int i = 0; i < MAXK; ++i) pr.p[i] = i < P.k ? primes[i] : 0;
    const uint32_t epad = (P.E + 31) / 32 * 32;
    ck(cudaFuncSetAttribute(act_out_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTabBytes), "attr");
    act_out_kernel<<<dim3(cdiv((uint64_t)epad * P.k, 256), P.B), 256, kTabBytes, S(st)>>>(P, pr, epad);
    ck(cudaGetLastError(), "act outputs launch");
}

}  // namespace dashgpu
