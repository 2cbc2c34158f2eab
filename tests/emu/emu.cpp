// TEST INFRASTRUCTURE ONLY — CPU emulation of the device side of libdashgpu.
//
// Compiles the *same* per-thread kernel logic (dash_device.cuh,
// dash_layers.cuh, dash_prim.cuh) with g++ and runs every "launch" as a host
// loop over the grid, so kernel logic can be debugged against the oracle on a
// machine without a GPU.  Linked with engine.cpp into tests/emu/libdashemu.so.
// The product package never loads this library; on a GPU box the tests run
// the real CUDA library (paper_2302_06361_b200/libdashgpu.so).
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
void event_record(void*, void*) {}
void stream_wait(void*, void*) {}
void prof_enable(int) {}
void prof_reset() {}
int prof_read(double*, uint64_t*, int) { return 0; }
}  // namespace dev

static void act_layer(const ActParams& P, bool garble, bool lv_garble) {
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t b = 0; b < (int64_t)P.B; ++b)
        for (int64_t u = 0; u < (int64_t)P.E; ++u) {
            uint32_t buf[3][NWMAX];
            Elt e;
            e.b = (uint32_t)b;
            e.u = (uint32_t)u;
            e.X = LB{buf[0], 1};
            e.K = LB{buf[1], 1};
            e.A = LB{buf[2], 1};
            e.t = tab();
            e.rk = nullptr;
            e.mult = nullptr;
            if (garble && lv_garble) {
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
            } else if ((uint64_t)P.B * P.E <= dev::lane_group_eval_max() && P.n_levels > 0) {
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

void launch_act_multi(const ActParams* dev_layers, const ActParams* host_layers, int n, bool garble, void*,
                      const Sched&) {
    uint64_t elements = 0;
    bool lv_ok = true;
    for (int i = 0; i < n; ++i) {
        elements += (uint64_t)host_layers[i].B * host_layers[i].E;
        lv_ok = lv_ok && host_layers[i].lv_ok;
    }
    const bool lv = garble && lv_ok && dev::garble_lv_warps(elements) >= 2;
    for (int i = 0; i < n; ++i) act_layer(dev_layers[i], garble, lv);
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

void launch_prim(const PrimParams& P, void*) {
    for (uint32_t i = 0; i < P.n; ++i) prim_thread(P, i, tab());
}

}  // namespace dashgpu
