// Activation-layer kernels (ReLU / SignAct gadget tapes), garble and eval.
// act_kernel: one thread = one (inference, element); a warp = 32 consecutive
// elements of one inference, so every tape branch, modulus and offset load is
// warp-uniform.  One persistent CTA per SM (28 warps garbling, 24 evaluating);
// shared memory = the replicated AES T-tables (64 KB) + per-lane label
// buffers.  Garbling work items are (tape chunk, layer, inference, block).
// act_wpe_kernel / act_wpe_eval_kernel: one warp per element for small
// launches (wpe.cuh, level-scheduled evaluation tape).  act_out_kernel: the
// garbler's output labels of a layer (pure PRF functions).
#include "dash_common.hpp"

namespace dashgpu {
__constant__ ModC c_mod[MAXMOD + 1];
__constant__ uint32_t c_pi_rk[44];
__constant__ uint16_t c_modslot[MAXMOD + 1];
__device__ uint32_t g_T0[256];
}  // namespace dashgpu
#define DASH_CONST_DEFINED 1
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels_common.cuh"
#include "wpe.cuh"

namespace dashgpu {

namespace {

// Dynamic shared memory per CTA: AES tables (64 KB) + per-lane label
// buffers X (NWMAX words), K (4 words: the Z_2-sized y operand of half
// gates, checked by the tape builder), A (NWMAX words); word w of a buffer at
// base + w*32 + lane.  28 warps x 5.5 KB + 64 KB = 218 KB.
constexpr int kLaneWords = 2 * NWMAX + 4;
constexpr int kBufWords = kLaneWords * 32;

// Work item = (tape chunk c, layer, inference, 32-element block), chunk-major:
// every element's tape is split into nchunks op ranges of similar cost, so the
// last wave of the persistent launch holds short items (the tail of a launch
// with whole-tape items idles ~10 % of the warp slots).  Chunks of one
// element communicate through the global label slots; chunk c waits for the
// done flag of chunk c-1 (dequeued earlier, so it is running or finished).
template <bool G>
__global__ void __launch_bounds__((G ? kActWarpsGarble : kActWarpsEval) * 32, 1)
    act_kernel(const ActParams* __restrict__ layers, ItemMap map, uint32_t* counter, uint32_t* flags,
               uint32_t nchunks) {
    uint32_t* L = s_dyn + kTabWords;
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per_chunk = map.base[map.n], total = per_chunk * nchunks;
    uint32_t* lb = L + (uint64_t)warp * kBufWords + lane;
    Elt e;
    e.X = LB{lb, 32};
    e.K = LB{lb + NWMAX * 32, 32};
    e.A = LB{lb + (NWMAX + 4) * 32, 32};
    e.t = make_tab(nullptr, lane);
    // first round: item = warp * grid + cta spreads small launches over all
    // SMs; afterwards warps pull items from the counter (balanced tail)
    uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t first = (G ? kActWarpsGarble : kActWarpsEval) * gridDim.x;
    for (;;) {
        if (item >= total) break;
        const uint32_t c = item / per_chunk, it = item - c * per_chunk;
        uint32_t li = 0;
        while (li + 1 < map.n && it >= map.base[li + 1]) ++li;
        const uint32_t local = it - map.base[li];
        const ActParams& P = layers[li];
        e.b = local / map.wpi[li];
        e.u = (local % map.wpi[li]) * 32 + lane;
        e.rk = nullptr;
        e.mult = nullptr;
        if (c > 0) {
            if (lane == 0) {
                uint32_t v;
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + it) : "memory");
                    if (v >= c) break;
                    __nanosleep(2000);
                }
            }
            __syncwarp();
        }
        const int op0 = nchunks > 1 ? P.chunk_op[c] : 0, op1 = nchunks > 1 ? P.chunk_op[c + 1] : P.n_ops;
        if (e.u < P.E) act_element<G>(P, e, op0, op1);
        __syncwarp();
        uint32_t next = 0;
        if (lane == 0) {
            if (nchunks > 1) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + it), "r"(c + 1) : "memory");
            }
            next = first + atomicAdd(counter, 1u);
        }
        item = __shfl_sync(0xffffffffu, next, 0);
    }
}

// Small garbling launches (few elements in total): one warp per element
// (wpe.cuh), every activation layer in one persistent launch.
constexpr int kWpeWarps = 16;
// Lane groups win while the per-thread launch would be latency-bound: G
// lanes per element cut an element's latency ~G-fold but idle lanes on small
// gates cost throughput (whole-warp groups for Model A b64 = 16k elements
// were 23.5 ms vs 13.8 ms per-thread); G is chosen so the warps fit
// kWpeGarbleWaves waves.
#ifndef DASH_WPE_GARBLE_WAVES
#define DASH_WPE_GARBLE_WAVES 1
#endif
constexpr uint64_t kWpeGarbleWaves = DASH_WPE_GARBLE_WAVES;
// evaluation: lane groups of G >= 2 while elements * G fits one wave of
// 16-warp CTAs (<= 148 * 512 / 2 = 37,888 elements; engine.cpp sizes the
// level-tape slots for it: dev::lane_group_eval_max())

__global__ void __launch_bounds__(kWpeWarps * 32, 1)
    act_wpe_kernel(const ActParams* __restrict__ layers, ItemMap map, uint32_t* counter, uint32_t G) {
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per = 32 / G, grp = lane / G, j = lane & (G - 1);
    uint32_t* wb = s_dyn + kTabWords + warp * kWpeWords;
    uint32_t* gb = wb + NWMAX * 32 + grp * kWpeShared;  // this group's shared labels
    WpeBufs w;
    w.X = LB{gb, 1};
    w.A = LB{gb + NWMAX, 1};
    w.K = LB{gb + 2 * NWMAX, 1};
    w.KEY = LB{wb + lane, 32};
    Elt e;
    e.X = w.X;
    e.K = w.K;
    e.A = w.A;
    e.t = make_tab(nullptr, lane);
    const uint32_t total = map.base[map.n];
    uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t first = kWpeWarps * gridDim.x;
    while (item < total) {
        uint32_t li = 0;
        while (li + 1 < map.n && item >= map.base[li + 1]) ++li;
        const ActParams& P = layers[li];
        const uint32_t local = item - map.base[li];
        e.b = local / map.wpi[li];
        e.u = (local - e.b * map.wpi[li]) * per + grp;
        // a group past the layer's last element repeats that element (same
        // values written twice) so every group stays in step with the syncs
        if (e.u >= P.E) e.u = P.E - 1;
        e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
        e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
        e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
        e.sstride = (uint64_t)P.B * P.E;
        e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
        e.rk = P.rk + (uint64_t)e.b * 44;
        e.mult = P.mult + (uint64_t)e.b * P.mult_stride;
        for (int i = 0; i < P.n_ops; ++i) garble_op_w(P, e, P.tape[i], w, j, G);
        uint32_t next = 0;
        if (lane == 0) next = first + atomicAdd(counter, 1u);
        item = __shfl_sync(0xffffffffu, next, 0);
    }
}

// Small garbling launches (batch-1 latency): W warps per element run the
// level-scheduled tape (ActParams::lv_tape).  Warp w of an element takes ops
// w, w+W, ... of every level, each op row-parallel over its 32 lanes
// (garble_op_w with G = 32), and the element's warps meet at a named barrier
// between levels.  The wide first levels (an element's k x t projections)
// then run W ops at a time instead of one.
constexpr int kLvWords = kWpeShared + NWMAX * 32;  // one lane group (G = 32) per warp
__global__ void __launch_bounds__(kWpeWarps * 32, 1)
    act_lv_garble_kernel(const ActParams* __restrict__ layers, ItemMap map, uint32_t W) {
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t grp = warp / W, wi = warp - grp * W, epc = kWpeWarps / W;
    uint32_t* wb = s_dyn + kTabWords + warp * kLvWords;
    uint32_t* gb = wb + NWMAX * 32;
    WpeBufs w;
    w.X = LB{gb, 1};
    w.A = LB{gb + NWMAX, 1};
    w.K = LB{gb + 2 * NWMAX, 1};
    w.KEY = LB{wb + lane, 32};
    Elt e;
    e.X = w.X;
    e.K = w.K;
    e.A = w.A;
    e.t = make_tab(nullptr, lane);
    const uint32_t item = blockIdx.x * epc + grp;
    if (item >= map.base[map.n]) return;  // the whole element group leaves together
    uint32_t li = 0;
    while (li + 1 < map.n && item >= map.base[li + 1]) ++li;
    const ActParams& P = layers[li];
    const uint32_t local = item - map.base[li];
    e.b = local / P.E;
    e.u = local - e.b * P.E;
    e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
    e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
    e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
    e.sstride = (uint64_t)P.B * P.E;
    e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
    e.rk = P.rk + (uint64_t)e.b * 44;
    e.mult = P.mult + (uint64_t)e.b * P.mult_stride;
    for (int L = 0; L < P.n_levels; ++L) {
        for (int i = P.lv_start[L] + (int)wi; i < P.lv_start[L + 1]; i += (int)W)
            garble_op_w(P, e, P.lv_tape[i], w, lane, 32);
        // slots written by this level are read by the next one (bar.sync
        // orders the element's global-memory accesses among its warps)
        asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(W * 32) : "memory");
    }
}

// Small evaluation launches: one warp per element, the level-scheduled tape
// (ActParams::lv_tape), lane t takes ops t, t+32, ... of every level.  Each
// lane keeps its own X / K / A buffers (lane-interleaved, as act_kernel).
constexpr int kWpeEvalWarps = 16;
constexpr int kLaneWordsEval = 2 * NWMAX + 4;

// Lanes form groups of G (a power of two): a warp evaluates 32/G elements, the
// G lanes of a group take ops j, j+G, ... of every level of their element;
// lane j of every group runs the same tape op (SIMT-uniform across groups).
__global__ void __launch_bounds__(kWpeEvalWarps * 32, 1)
    act_wpe_eval_kernel(const ActParams* __restrict__ layers, ItemMap map, uint32_t* counter, uint32_t G) {
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* lb = s_dyn + kTabWords + warp * kLaneWordsEval * 32 + lane;
    Elt e;
    e.X = LB{lb, 32};
    e.K = LB{lb + NWMAX * 32, 32};
    e.A = LB{lb + (NWMAX + 4) * 32, 32};
    e.t = make_tab(nullptr, lane);
    e.rk = nullptr;
    e.mult = nullptr;
    const uint32_t total = map.base[map.n];
    uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t first = kWpeEvalWarps * gridDim.x;
    const uint32_t per = 32 / G, grp = lane / G, j = lane & (G - 1);
    while (item < total) {
        uint32_t li = 0;
        while (li + 1 < map.n && item >= map.base[li + 1]) ++li;
        const ActParams& P = layers[li];
        const uint32_t local = item - map.base[li];
        e.b = local / map.wpi[li];
        e.u = (local - e.b * map.wpi[li]) * per + grp;
        const bool active = e.u < P.E;
        if (!active) e.u = P.E - 1;  // idle group: stays in step with the warp's level syncs
        e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
        e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
        e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
        e.sstride = (uint64_t)P.B * P.E;
        e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
        for (int L = 0; L < P.n_levels; ++L) {
            const int end = P.lv_start[L + 1];
            if (active)
                for (int i = P.lv_start[L] + (int)j; i < end; i += (int)G) eval_op<true>(P, e, P.lv_tape[i]);
            __syncwarp();
        }
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

// Small launches: one warp per (inference, element, lane) output label, the
// PRF counter blocks split over the 32 lanes (prf_coop); lane 0 finishes the
// label.  Same values as act_output_thread.
constexpr int kOutWarps = 8;
__global__ void __launch_bounds__(kOutWarps * 32) act_out_warp_kernel(ActParams P, Primes pr) {
    fill_T(g_T0);
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint32_t idx = blockIdx.x * kOutWarps + wl;
    const uint32_t i = idx % (uint32_t)P.k, u = idx / (uint32_t)P.k, b = blockIdx.y;
    if (u >= P.E) return;  // whole warp
    LB A{s_dyn + kTabWords + wl * 2 * NWMAX, 1}, T{s_dyn + kTabWords + wl * 2 * NWMAX + NWMAX, 1};
    const AesTab t = make_tab(nullptr, lane);
    const uint32_t p = pr.p[i];
    const ModC& M = c_mod[p];
    const uint32_t* rk = P.rk + (uint64_t)b * 44;
    const uint64_t w = P.wire_base + (uint64_t)u * P.uc_wires + P.out_wire[i];
    prf_coop(A, w, 0, p, rk, t, lane, 32);
    const bool mm = P.out_kind[i] == OP_MMHALF;
    if (mm) prf_coop(T, w + 1, 0, p, rk, t, lane, 32);
    if (lane == 0) {
        if (mm) {  // out = v0 - u0 (gadgets.hpp:354)
            if (P.mmlab) {
                U4* ml = P.mmlab + (((uint64_t)b * P.E + u) * P.k + i) * 2;
                ml[0] = lb_compress(A, M);
                ml[1] = lb_compress(T, M);
            }
            lb_sub(T, A, M);
            lb_store_rows(T, P.out[i] + ((uint64_t)b * M.nw) * P.E + u, P.E, M);
        } else {
            lb_store_rows(A, P.out[i] + ((uint64_t)b * M.nw) * P.E + u, P.E, M);
        }
    }
}

}  // namespace

void upload_act(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0) {
    ck(cudaMemcpyToSymbol(c_mod, mods, sizeof(ModC) * (MAXMOD + 1)), "c_mod(act)");
    ck(cudaMemcpyToSymbol(c_pi_rk, pi_rk, sizeof(uint32_t) * 44), "c_pi_rk(act)");
    ck(cudaMemcpyToSymbol(c_modslot, modslot, sizeof(uint16_t) * (MAXMOD + 1)), "c_modslot(act)");
    ck(cudaMemcpyToSymbol(g_T0, T0, sizeof(uint32_t) * 256), "g_T0(act)");
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

static dev::ActShape g_shape[2];

static void note_shape(bool garble, uint32_t variant, uint32_t nchunks, uint32_t grid, uint64_t items, uint32_t group) {
    g_shape[garble ? 1 : 0] = dev::ActShape{variant, nchunks, grid, (uint32_t)items, group};
}

namespace dev {
ActShape last_act_shape(bool garble) { return g_shape[garble ? 1 : 0]; }
uint64_t chunk_min_items() {
    const char* e = std::getenv("DASH_CHUNK_MIN_ITEMS");
    return e ? (uint64_t)std::atol(e) : (uint64_t)sm_count() * kActWarpsGarble;
}
bool force_thread_shape() {
    const char* e = std::getenv("DASH_ACT_SHAPE");
    return e && std::strcmp(e, "thread") == 0;
}
uint64_t lane_group_eval_max() { return (uint64_t)sm_count() * kWpeEvalWarps * 32 / 2; }
// warps per element of the level-parallel garbling launch (0: not used): the
// largest power of two <= 8 whose warps still fit one wave of 16-warp CTAs
uint32_t garble_lv_warps(uint64_t elements) {
    static const uint32_t wmax = [] {  // DASH_LV_WARPS: A/B knob for the cap
        const char* e = std::getenv("DASH_LV_WARPS");
        return e ? (uint32_t)std::atoi(e) : 8u;
    }();
    static const uint32_t ctas = [] {  // DASH_LV_CTAS: resident 16-warp CTAs per SM assumed
        const char* e = std::getenv("DASH_LV_CTAS");
        return e ? (uint32_t)std::atoi(e) : 1u;
    }();
    uint32_t W = wmax;
    while (W >= 2 && elements * W > (uint64_t)sm_count() * kWpeWarps * ctas) W >>= 1;
    return W >= 2 ? W : 0;
}
}  // namespace dev

void launch_act_multi(const ActParams* dev_layers, const ActParams* host_layers, int n, bool garble, void* st,
                      const Sched& q) {
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
    uint64_t elements = 0;
    for (int i = 0; i < n; ++i) elements += (uint64_t)host_layers[i].B * host_layers[i].E;
    // evaluation lane groups: the largest G whose warps still fit one wave
    uint32_t G = 32;
    const uint64_t wave = (uint64_t)sm_count() * kWpeEvalWarps * 32;
    while (G > 1 && elements * G > wave) G >>= 1;
    const bool thread_only = dev::force_thread_shape();
    if (!garble && G >= 2 && !thread_only) {
        ItemMap wm;
        std::memset(&wm, 0, sizeof wm);
        wm.n = (uint32_t)n;
        const uint32_t per = 32 / G;
        for (int i = 0; i < n; ++i) {
            wm.wpi[i] = (host_layers[i].E + per - 1) / per;
            wm.base[i + 1] = wm.base[i] + host_layers[i].B * wm.wpi[i];
        }
        const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)sm_count(), wm.base[n]);  // spread: latency-bound
        const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)kWpeEvalWarps * kLaneWordsEval * 32;
        ck(cudaMemsetAsync(q.counter, 0, sizeof(uint32_t), S(st)), "counter reset");
        smem_attr((const void*)act_wpe_eval_kernel, smem);
        act_wpe_eval_kernel<<<grid, kWpeEvalWarps * 32, smem, S(st)>>>(dev_layers, wm, q.counter, G);
        ck(cudaGetLastError(), "act wpe eval launch");
        note_shape(false, dev::ACT_SHAPE_WPE_EVAL, 1, grid, wm.base[n], G);
        return;
    }
    // level-parallel garbling: W warps per element when the launch is small
    // enough and every layer's slot region holds the level tape's slots
    if (garble && !thread_only) {
        bool lv_ok = true;
        for (int i = 0; i < n; ++i) lv_ok = lv_ok && host_layers[i].lv_ok;
        const uint32_t W = lv_ok ? dev::garble_lv_warps(elements) : 0;
        if (W >= 2) {
            ItemMap lm;
            std::memset(&lm, 0, sizeof lm);
            lm.n = (uint32_t)n;
            for (int i = 0; i < n; ++i) {
                lm.wpi[i] = host_layers[i].E;
                lm.base[i + 1] = lm.base[i] + host_layers[i].B * host_layers[i].E;
            }
            const uint32_t epc = kWpeWarps / W;
            const uint32_t grid = (uint32_t)((lm.base[n] + epc - 1) / epc);
            const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)kWpeWarps * kLvWords;
            smem_attr((const void*)act_lv_garble_kernel, smem);
            act_lv_garble_kernel<<<grid, kWpeWarps * 32, smem, S(st)>>>(dev_layers, lm, W);
            ck(cudaGetLastError(), "act lv garble launch");
            note_shape(true, dev::ACT_SHAPE_LV_GARBLE, 1, grid, lm.base[n], 32 * W);
            return;
        }
    }
    // garbling lane groups: the largest G whose warps fit one wave of 16-warp
    // CTAs; G = 1 is the per-thread kernel below
    uint32_t Gg = 32;
    while (Gg > 1 && elements * Gg > (uint64_t)sm_count() * kWpeWarps * 32 * kWpeGarbleWaves) Gg >>= 1;
    if (garble && Gg >= 2 && !thread_only) {
        ItemMap wm;
        std::memset(&wm, 0, sizeof wm);
        wm.n = (uint32_t)n;
        const uint32_t per = 32 / Gg;
        for (int i = 0; i < n; ++i) {
            wm.wpi[i] = (host_layers[i].E + per - 1) / per;
            wm.base[i + 1] = wm.base[i] + host_layers[i].B * wm.wpi[i];
        }
        const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)sm_count(), wm.base[n]);  // spread: latency-bound
        const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)kWpeWarps * kWpeWords;
        ck(cudaMemsetAsync(q.counter, 0, sizeof(uint32_t), S(st)), "counter reset");
        smem_attr((const void*)act_wpe_kernel, smem);
        act_wpe_kernel<<<grid, kWpeWarps * 32, smem, S(st)>>>(dev_layers, wm, q.counter, Gg);
        ck(cudaGetLastError(), "act wpe launch");
        note_shape(true, dev::ACT_SHAPE_WPE_GARBLE, 1, grid, wm.base[n], Gg);
        return;
    }
    // one CTA per SM (the first round strides items across SMs), never fewer
    // CTAs than needed to give every item its own SM when items < #SMs
    const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)sm_count(), map.base[n]);
    const int warps = garble ? kActWarpsGarble : kActWarpsEval;
    const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)warps * kBufWords;
    uint32_t* counter = q.counter;
    ck(cudaMemsetAsync(counter, 0, sizeof(uint32_t), S(st)), "counter reset");
    // garbling: chunked tapes (host_layers[].chunk_op); evaluation: whole tapes
    uint32_t nchunks = 1;
    // chunked tapes only pay when the launch has more warp items than warp
    // slots (the last wave); below that every chunk would just wait in turn
    if (garble && map.base[n] > dev::chunk_min_items()) {
        for (int i = 0; i < n; ++i)
            for (int c = 1; c <= MAXCHUNK; ++c)
                if (host_layers[i].chunk_op[c] == host_layers[i].n_ops) {
                    nchunks = std::max<uint32_t>(nchunks, (uint32_t)c);
                    break;
                }
    }
    uint32_t* flags = q.flags;
    if (nchunks > 1) {
        if (q.flags_cap < map.base[n]) throw std::runtime_error("work-queue flags too small");
        ck(cudaMemsetAsync(flags, 0, sizeof(uint32_t) * map.base[n], S(st)), "flags reset");
    }
    if (garble) {
        smem_attr((const void*)act_kernel<true>, smem);
        act_kernel<true><<<grid, warps * 32, smem, S(st)>>>(dev_layers, map, counter, flags, nchunks);
    } else {
        smem_attr((const void*)act_kernel<false>, smem);
        act_kernel<false><<<grid, warps * 32, smem, S(st)>>>(dev_layers, map, counter, flags, 1);
    }
    ck(cudaGetLastError(), "act launch");
    note_shape(garble, dev::ACT_SHAPE_THREAD, nchunks, grid, map.base[n], 1);
}

void launch_act_outputs(const ActParams& P, const uint16_t* primes, void* st) {
    if (P.B == 0 || P.E == 0) return;
    ProfScope ps(K_SETUP, S(st));
    Primes pr;
    for (int i = 0; i < MAXK; ++i) pr.p[i] = i < P.k ? primes[i] : 0;
    const uint64_t labels = (uint64_t)P.B * P.E * P.k;
    if (labels <= (uint64_t)sm_count() * 24 * 2) {  // <= two waves of warps: one warp per label
        const size_t smem = kTabBytes + sizeof(uint32_t) * kOutWarps * 2 * NWMAX;
        smem_attr((const void*)act_out_warp_kernel, smem);
        act_out_warp_kernel<<<dim3(cdiv((uint64_t)P.E * P.k, kOutWarps), P.B), kOutWarps * 32, smem, S(st)>>>(P, pr);
        ck(cudaGetLastError(), "act outputs launch");
        return;
    }
    const uint32_t epad = (P.E + 31) / 32 * 32;
    smem_attr((const void*)act_out_kernel, kTabBytes);
    act_out_kernel<<<dim3(cdiv((uint64_t)epad * P.k, 256), P.B), 256, kTabBytes, S(st)>>>(P, pr, epad);
    ck(cudaGetLastError(), "act outputs launch");
}

}  // namespace dashgpu
