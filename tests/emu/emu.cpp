// TEST INFRASTRUCTURE ONLY — CPU emulation of the device side of libdashgpu.
//
// Compiles the *same* per-thread kernel logic (dash_device.cuh,
// dash_layers.cuh, dash_prim.cuh) with g++ and runs every "launch" as a host
// loop over the grid, so kernel logic can be debugged against the oracle on a
// machine without a GPU.  Linked with engine.cpp into tests/emu/libdashemu.so.
// The product package never loads this library; on a GPU box the tests run
// the real CUDA library (paper_2302_06361_b200/libdashgpu.so).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "dash_common.hpp"

namespace dashgpu {
ModC c_mod[MAXMOD + 1];
uint32_t c_pi_rk[44];
uint16_t c_modslot[MAXMOD + 1];
}  // namespace dashgpu
#define DASH_CONST_DEFINED 1
#include "dash_prim.cuh"

namespace dashgpu {

static uint32_t g_T[256 * 64];
static uint32_t g_T0plain[256];

static AesTab tab() { return make_tab(g_T, 0); }

namespace dev {
void set_device(int) {}
int get_device() { return 0; }
int backend() { return 2; }
void* alloc(size_t n) {
    void* p = std::calloc(1, n ? n : 16);
    if (!p) throw std::runtime_error("emu alloc failed");
    return p;
}
void release(void* p) { std::free(p); }
void* host_alloc(size_t n) { return alloc(n); }
void host_release(void* p) { std::free(p); }
void h2d(void* d, const void* s, size_t n, void*) { std::memcpy(d, s, n); }
void d2h(void* d, const void* s, size_t n, void*) { std::memcpy(d, s, n); }
void d2d(void* d, const void* s, size_t n, void*) { std::memmove(d, s, n); }
void memset0(void* p, size_t n, void*) { std::memset(p, 0, n); }
void sync(void*) {}
void check() {}
size_t free_bytes() { return (size_t)8 << 30; }
void upload_constants(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0) {
    std::memcpy(c_mod, mods, sizeof(ModC) * (MAXMOD + 1));
    std::memcpy(c_pi_rk, pi_rk, sizeof(uint32_t) * 44);
    std::memcpy(c_modslot, modslot, sizeof(uint16_t) * (MAXMOD + 1));
    std::memcpy(g_T0plain, T0, sizeof g_T0plain);
    for (int i = 0; i < 256 * 64; ++i) {
        const uint32_t v = T0[i >> 6];
        g_T[i] = (i & 32) ? ((v << 16) | (v >> 16)) : v;
    }
}
uint64_t lane_group_eval_max() { return 148 * 16 * 32 / 2; }
uint32_t garble_lv_warps(uint64_t elements) {  // kernels_act.cu, 148 SMs x 16 warps
    uint32_t W = 8;
    while (W >= 2 && elements * W > 148ull * 16) W >>= 1;
    return W >= 2 ? W : 0;
}
void* stream_create() { return nullptr; }
void stream_destroy(void*) {}
void* event_create() { return nullptr; }
void event_destroy(void*) {}
void event_sync(void*) {}
void event_record(void*, void*) {}
void stream_wait(void*, void*) {}
void prof_enable(int) {}
void prof_reset() {}
int prof_read(double*, uint64_t*, int) { return 0; }
}  // namespace dev

namespace dev {
static ActShape g_shape[2];
ActShape last_act_shape(bool garble) { return g_shape[garble ? 1 : 0]; }
uint64_t chunk_min_items() {  // kernels_act.cu: one wave of 28-warp garbling CTAs on 148 SMs
    const char* e = std::getenv("DASH_CHUNK_MIN_ITEMS");
    return e ? (uint64_t)std::atol(e) : 148ull * 28;
}
bool force_thread_shape() {
    const char* e = std::getenv("DASH_ACT_SHAPE");
    return e && std::strcmp(e, "thread") == 0;
}
}  // namespace dev

static const uint32_t kPoison = 0xA5C3E1F7u;

// Runs ops [op0, op1) of every element's tape.  chunk > 0 emulates a chunked
// work item of the persistent garbling kernel (kernels_act.cu act_kernel): it
// runs on whatever warp dequeues it, so its shared-memory label buffers hold
// garbage from other work -- they are poisoned here, and every value a chunk
// needs must come from the global label slots.
static void act_layer(const ActParams& P, bool garble, bool lv_garble, int chunk = -1, bool thread_eval = false) {
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t b = 0; b < (int64_t)P.B; ++b)
        for (int64_t u = 0; u < (int64_t)P.E; ++u) {
            uint32_t buf[3][NWMAX];
            if (chunk >= 0)
                for (int j = 0; j < 3; ++j)
                    for (int w = 0; w < NWMAX; ++w) buf[j][w] = kPoison ^ (uint32_t)(u * 131 + w * 7 + j);
            Elt e;
            e.b = (uint32_t)b;
            e.u = (uint32_t)u;
            e.X = LB{buf[0], 1};
            e.K = LB{buf[1], 1};
            e.A = LB{buf[2], 1};
            e.t = tab();
            e.rk = nullptr;
            e.mult = nullptr;
            if (chunk >= 0) {
                act_element<true>(P, e, P.chunk_op[chunk], P.chunk_op[chunk + 1]);
            } else if (garble && lv_garble) {
                // level-parallel garbling (act_lv_garble_kernel): the level
                // tape, ops of a level in reverse order (they are independent)
                e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
                e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
                e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
                e.sstride = (uint64_t)P.B * P.E;
                e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
                e.rk = P.rk + (uint64_t)e.b * 44;
                e.mult = P.mult + (uint64_t)e.b * P.mult_stride;
                for (int L = 0; L < P.n_levels; ++L)
                    for (int i = P.lv_start[L + 1] - 1; i >= P.lv_start[L]; --i) garble_op(P, e, P.lv_tape[i]);
            } else if (garble) {
                act_element<true>(P, e, 0, P.n_ops);
            } else if (!thread_eval && (uint64_t)P.B * P.E <= dev::lane_group_eval_max() && P.n_levels > 0) {
                // small launches: the level-scheduled tape, as the CUDA
                // warp-per-element evaluation runs it (levels in order;
                // the ops of a level are independent)
                e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
                e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
                e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
                e.sstride = (uint64_t)P.B * P.E;
                e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
                for (int L = 0; L < P.n_levels; ++L)
                    for (int i = P.lv_start[L + 1] - 1; i >= P.lv_start[L]; --i) eval_op<true>(P, e, P.lv_tape[i]);
            } else {
                act_element<false>(P, e, 0, P.n_ops);
            }
        }
}

// Mirrors the launch-shape choice of kernels_act.cu launch_act_multi (148 SMs).
void launch_act_multi(const ActParams* dev_layers, const ActParams* host_layers, int n, bool garble, void*,
                      const Sched&) {
    uint64_t elements = 0, items = 0;
    bool lv_ok = true;
    for (int i = 0; i < n; ++i) {
        elements += (uint64_t)host_layers[i].B * host_layers[i].E;
        items += (uint64_t)host_layers[i].B * ((host_layers[i].E + 31) / 32);
        lv_ok = lv_ok && host_layers[i].lv_ok;
    }
    const bool thread_only = dev::force_thread_shape();
    if (!garble) {
        uint32_t G = 32;
        while (G > 1 && elements * G > 148ull * 16 * 32) G >>= 1;
        if (thread_only) G = 1;
        dev::g_shape[0] = G >= 2 ? dev::ActShape{dev::ACT_SHAPE_WPE_EVAL, 1, 148, (uint32_t)elements, G}
                                 : dev::ActShape{dev::ACT_SHAPE_THREAD, 1, 148, (uint32_t)items, 1};
        for (int i = 0; i < n; ++i) act_layer(dev_layers[i], false, false, -1, thread_only);
        return;
    }
    const bool lv = !thread_only && lv_ok && dev::garble_lv_warps(elements) >= 2;
    if (lv) {
        dev::g_shape[1] = dev::ActShape{dev::ACT_SHAPE_LV_GARBLE, 1, 0, (uint32_t)elements,
                                        32 * dev::garble_lv_warps(elements)};
        for (int i = 0; i < n; ++i) act_layer(dev_layers[i], true, true);
        return;
    }
    uint32_t Gg = 32;
    while (Gg > 1 && elements * Gg > 148ull * 16 * 32) Gg >>= 1;
    if (Gg >= 2 && !thread_only) {
        dev::g_shape[1] = dev::ActShape{dev::ACT_SHAPE_WPE_GARBLE, 1, 148, (uint32_t)elements, Gg};
        for (int i = 0; i < n; ++i) act_layer(dev_layers[i], true, false);
        return;
    }
    uint32_t nchunks = 1;
    if (items > dev::chunk_min_items())
        for (int i = 0; i < n; ++i)
            for (int c = 1; c <= MAXCHUNK; ++c)
                if (host_layers[i].chunk_op[c] == host_layers[i].n_ops) {
                    nchunks = std::max<uint32_t>(nchunks, (uint32_t)c);
                    break;
                }
    dev::g_shape[1] = dev::ActShape{dev::ACT_SHAPE_THREAD, nchunks, 148, (uint32_t)items, 1};
    if (nchunks == 1) {
        for (int i = 0; i < n; ++i) act_layer(dev_layers[i], true, false);
        return;
    }
    // chunk-major, as the persistent kernel dequeues its items
    for (uint32_t c = 0; c < nchunks; ++c)
        for (int i = 0; i < n; ++i) act_layer(dev_layers[i], true, false, (int)c);
}

void launch_act_outputs(const ActParams& P, const uint16_t* primes, void*) {
#pragma omp parallel for collapse(2)
    for (int64_t b = 0; b < (int64_t)P.B; ++b)
        for (int64_t u = 0; u < (int64_t)P.E; ++u) {
            uint32_t buf[2][NWMAX];
            for (int i = 0; i < P.k; ++i)
                act_output_thread(P, (uint32_t)b, (uint32_t)u, i, primes[i], LB{buf[0], 1}, LB{buf[1], 1}, tab());
        }
}

void make_weight_map(TcLinear&) {}

// the tensor-core GEMM (tc_linear.cuh) has no CPU emulation; the emulation
// runs the same arithmetic per output word (dash_layers.cuh linear_thread)
void launch_linear(const LinParams* Ls, int n, const TcLinear&, void*) {
    for (int i = 0; i < n; ++i) {
        const LinParams& L = Ls[i];
#pragma omp parallel for collapse(3)
        for (int64_t b = 0; b < (int64_t)L.B; ++b)
            for (int64_t w = 0; w < (int64_t)L.nw; ++w)
                for (int64_t u = 0; u < (int64_t)L.M; ++u) linear_thread(L, (uint32_t)b, (uint32_t)w, (uint32_t)u);
    }
}

void launch_pad_add(const PadAddParams& P, void*) {
#pragma omp parallel for collapse(2)
    for (int64_t b = 0; b < (int64_t)P.B; ++b)
        for (int64_t wi = 0; wi < (int64_t)P.wbase[P.k]; ++wi)
            for (uint32_t u = 0; u < P.E_out; ++u) pad_add_thread(P, (uint32_t)b, (uint32_t)wi, u);
}

void launch_expand(const uint8_t* seeds, uint32_t* rk, uint32_t B, void*) {
    for (uint32_t b = 0; b < B; ++b) expand_thread(seeds + (uint64_t)b * 16, rk + (uint64_t)b * 44, g_T0plain);
}

void launch_proj(const ProjParams& P, void*) {
#pragma omp parallel for
    for (int64_t i = 0; i < (int64_t)P.n; ++i) {
        uint32_t buf[2][NWMAX] = {};
        proj_thread(P, (uint32_t)i, tab(), LB{buf[0], 1}, LB{buf[1], 1});
    }
}

void launch_private(const PrivParams& P, void*, const Sched&) {
#pragma omp parallel for collapse(2)
    for (int64_t b = 0; b < (int64_t)P.B; ++b)
        for (int64_t u = 0; u < (int64_t)P.M; ++u) private_thread(P, (uint32_t)b, (uint32_t)u, tab());
}

void launch_setup(const SetupParams& S, void*) {
    for (uint32_t b = 0; b < S.B; ++b)
        for (uint32_t si = 0; si < S.nslot; ++si)
            for (uint32_t x = 0; x < 128; ++x) setup_offsets_thread(S, b, si, x, tab());
#pragma omp parallel for collapse(2)
    for (int64_t b = 0; b < (int64_t)S.B; ++b)
        for (int64_t e = 0; e <= (int64_t)S.n_in; ++e)
            for (int i = 0; i < S.k; ++i) setup_labels_thread(S, (uint32_t)b, (uint32_t)e, i, tab());
}

void launch_encode(const EncodeParams& P, void*) {
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t e = 0; e < P.n_in; ++e)
            for (int i = 0; i < P.k; ++i) encode_thread(P, b, e, i);
}

void launch_dectable(const DecodeParams& P, void*) {
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t e = 0; e < P.n_out; ++e)
            for (int i = 0; i < P.k; ++i) dectable_thread(P, b, e, i);
}

void launch_decode(const DecodeParams& P, void*) {
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t e = 0; e < P.n_out; ++e) decode_thread(P, b, e);
}

void launch_compress(const CompressParams& P, void*) {
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t e = 0; e < P.n; ++e) compress_thread(P, b, e);
}

void launch_decompress(const CompressParams& P, uint32_t* lane_out, void*) {
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t e = 0; e < P.n; ++e) decompress_thread(P, b, e, lane_out);
}

void launch_rows_permute(const RowsPermuteParams& P, void*) {
#pragma omp parallel for
    for (int64_t r = 0; r < (int64_t)(P.E * P.uc); ++r) rows_permute_thread(P, (uint64_t)r);
}

void launch_digest(const DigestParams& P, uint32_t* roots, void*) {
#pragma omp parallel for collapse(2)
    for (uint32_t b = 0; b < P.B; ++b)
        for (uint32_t l = 0; l < P.leaves; ++l) digest_leaf_thread(P, b, l);
    for (uint32_t b = 0; b < P.B; ++b) digest_root_thread(P, b, roots);
}

void launch_prim(const PrimParams& P, void*) {
    for (uint32_t i = 0; i < P.n; ++i) prim_thread(P, i, tab());
}

}  // namespace dashgpu
