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
#include "kernels_common.cuh"

namespace dashgpu {

namespace {

// Shared memory per CTA: static T-table s_T (32 KB) + dynamic: 4 label buffers of NWMAX words
// per lane (word w of buffer j for lane l at L[((warp*4 + j)*NWMAX + w)*32 + l]).
constexpr int kBufWords = 4 * NWMAX * 32;

template <bool G>
__global__ void __launch_bounds__(kActWarps * 32, 2) act_kernel(ActParams P) {
    extern __shared__ uint4 smem4[];
    uint32_t* L = reinterpret_cast<uint32_t*>(smem4);
    fill_T(s_T, g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t wpi = (P.E + 31) / 32;
    const uint64_t gw = (uint64_t)blockIdx.x * kActWarps + warp;
    const uint32_t b = (uint32_t)(gw / wpi);
    const uint32_t u = (uint32_t)(gw % wpi) * 32 + lane;
    if (b >= P.B || u >= P.E) return;
    uint32_t* lb = L + (uint64_t)warp * kBufWords + lane;
    Elt e;
    e.b = b;
    e.u = u;
    e.X = LB{lb, 32};
    e.K = LB{lb + NWMAX * 32, 32};
    e.A = LB{lb + 2 * NWMAX * 32, 32};
    e.T = LB{lb + 3 * NWMAX * 32, 32};
    e.t = make_tab(s_T, lane);
    e.rk = nullptr;
    e.mult = nullptr;
    act_element<G>(P, e);
}

}  // namespace

void upload_act(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0) {
    ck(cudaMemcpyToSymbol(c_mod, mods, sizeof(ModC) * (MAXMOD + 1)), "c_mod(act)");
    ck(cudaMemcpyToSymbol(c_pi_rk, pi_rk, sizeof(uint32_t) * 44), "c_pi_rk(act)");
    ck(cudaMemcpyToSymbol(c_modslot, modslot, sizeof(uint16_t) * (MAXMOD + 1)), "c_modslot(act)");
    ck(cudaMemcpyToSymbol(g_T0, T0, sizeof(uint32_t) * 256), "g_T0(act)");
}

void launch_act(const ActParams& P, bool garble, int nslots, void* st) {
    if (P.B == 0 || P.E == 0) return;
    ProfScope ps(garble ? K_ACT_GARBLE : K_ACT_EVAL, S(st));
    const uint64_t warps = (uint64_t)P.B * ((P.E + 31) / 32);
    const uint32_t grid = cdiv(warps, kActWarps);
    (void)nslots;  // slots live in global memory (P.slots)
    const size_t smem = sizeof(uint32_t) * (size_t)kActWarps * kBufWords;  // + static s_T (32 KB)
    if (garble) {
        ck(cudaFuncSetAttribute(act_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        act_kernel<true><<<grid, kActWarps * 32, smem, S(st)>>>(P);
    } else {
        ck(cudaFuncSetAttribute(act_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "attr");
        act_kernel<false><<<grid, kActWarps * 32, smem, S(st)>>>(P);
    }
    ck(cudaGetLastError(), "act launch");
}

}  // namespace dashgpu
