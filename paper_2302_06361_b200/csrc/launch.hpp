// Seam between the host engine (engine.cpp, plain C++) and the device side
// (kernels.cu: CUDA for sm_100a).  The engine never includes CUDA headers; all
// device memory, streams and kernel launches go through these functions.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "dash_layers.cuh"

namespace dashgpu {
namespace dev {

void set_device(int device);
int get_device();  // current device of the calling host thread (-1 = none)
int backend();  // 1 = CUDA
void* alloc(size_t bytes);
void release(void* p);
void* host_alloc(size_t bytes);  // pinned
void host_release(void* p);
void h2d(void* dst, const void* src, size_t n, void* stream);
void d2h(void* dst, const void* src, size_t n, void* stream);
void d2d(void* dst, const void* src, size_t n, void* stream);
void memset0(void* p, size_t n, void* stream);
void sync(void* stream);
void check();  // raise on a pending device error
size_t free_bytes();
void upload_constants(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0);
// elements up to which an evaluation launch runs in lane groups on the level
// tape (kernels_act.cu; the engine sizes the level tape's slots for it)
uint64_t lane_group_eval_max();
uint32_t garble_lv_warps(uint64_t elements);  // level-parallel garbling (0 = not used)
// Launch shape of the most recent activation launch (garble / eval), so tests
// can pin the configuration a benchmark times: variant (ACT_SHAPE_*), tape
// chunks per element, grid, work items (warps or lane groups), lanes per element.
enum { ACT_SHAPE_NONE = 0, ACT_SHAPE_WPE_EVAL = 1, ACT_SHAPE_LV_GARBLE = 2, ACT_SHAPE_WPE_GARBLE = 3, ACT_SHAPE_THREAD = 4 };
struct ActShape {
    uint32_t variant, nchunks, grid, items, group;
};
ActShape last_act_shape(bool garble);
// warp items above which the per-thread garbling launch splits element tapes
// into chunks (default: one wave of garbling warps; DASH_CHUNK_MIN_ITEMS overrides)
uint64_t chunk_min_items();
// DASH_ACT_SHAPE=thread: activation launches always take the per-thread
// kernels (tests pin the chunked garbling path on small circuits)
bool force_thread_shape();
// streams / events
void* stream_create();
void stream_destroy(void* s);
void* event_create();
void event_destroy(void* e);
void event_record(void* e, void* stream);
void event_sync(void* e);  // host waits for the event
void stream_wait(void* stream, void* e);

// per-kernel-kind event timing on the launching stream (bench roofline)
void prof_enable(int on);
void prof_reset();
int prof_read(double* ms, uint64_t* launches, int max_kinds);

}  // namespace dev

enum KernelKind {
    K_ACT_GARBLE = 0,
    K_ACT_EVAL = 1,
    K_LINEAR = 2,
    K_PRIV_GARBLE = 3,
    K_PRIV_EVAL = 4,
    K_SETUP = 5,
    K_ENCODE = 6,
    K_DECODE = 7,
    K_MISC = 8,
    K_NKINDS = 9
};

// Work-queue state of the persistent kernels (one per stream that launches
// them concurrently): item counter + per-item chunk flags.
struct Sched {
    uint32_t* counter = nullptr;  // >= 2 words: [0] activation, [1] private kernel
    uint32_t* flags = nullptr;
    size_t flags_cap = 0;         // words
};

// Activation tapes of n layers in one persistent launch (dev_layers: the same
// ActParams array in device memory).
void launch_act_multi(const ActParams* dev_layers, const ActParams* host_layers, int n, bool garble, void* stream,
                      const Sched& q);
// Garbler-side output labels of an activation layer (pure PRF functions).
void launch_act_outputs(const ActParams& P, const uint16_t* primes, void* stream);
// Tensor-core form of one public linear layer (tc_linear.cuh): the weight
// residues of all k lanes, [k][Npad][Kpad] u8 K-major (row oc, column =
// window index i), the window offset table and the TMA descriptor of the
// weights.
struct TcLinear {
    alignas(64) uint8_t tmap[128];
    const uint8_t* wexp = nullptr;
    const int32_t* koff = nullptr;  // [kblocks * 128] element offsets, -1 = padding
    uint32_t kblocks = 0, Npad = 0, Kpad = 0, BN = 0, nout = 0, k = 0;
    int fold = 0;  // zero-wire / bias terms are window columns K, K + 1 (tc_linear.cuh)
    enum { DIGIT_ROWS = 0, EXPANDED = 1 };
    int mode = DIGIT_ROWS;  // DIGIT_ROWS: tc_linear.cuh (aligned dense); EXPANDED: tc_linear_exp.cuh
};
void make_weight_map(TcLinear& t);  // encodes t.tmap for t.wexp
// all lanes of a public linear layer in one launch
void launch_linear(const LinParams* Ls, int n, const TcLinear& tc, void* stream);
void launch_private(const PrivParams& P, void* stream, const Sched& q);
void launch_pad_add(const PadAddParams& P, void* stream);  // extension layers
void launch_proj(const ProjParams& P, void* stream);        // t_proj primitive
void launch_setup(const SetupParams& S, void* stream);
void launch_expand(const uint8_t* seeds, uint32_t* rk, uint32_t B, void* stream);  // device AES key schedules
void launch_encode(const EncodeParams& P, void* stream);
void launch_dectable(const DecodeParams& P, void* stream);
void launch_decode(const DecodeParams& P, void* stream);
void launch_compress(const CompressParams& P, void* stream);
void launch_decompress(const CompressParams& P, uint32_t* lane_out, void* stream);
void launch_rows_permute(const RowsPermuteParams& P, void* stream);  // GC export / import row order
// streamed-garbling layer digests: leaves into P.out, then the roots [B][8] state words
void launch_digest(const DigestParams& P, uint32_t* roots, void* stream);

// primitive kernels for parity tests: op 0 decompress+compress, 1 aes_pi,
// 2 aes with key, 3 prf label, 4 encrypt_label, 5 decrypt_label
struct PrimParams {
    int op;
    uint32_t n;
    uint32_t m, q;
    const U4* in;       // [n]
    U4* out;            // [n]
    uint32_t* digits;   // [n][LABW] byte-digit words
    const uint32_t* rk; // [44]
    const uint64_t* wires;
    uint64_t gate;
};
void launch_prim(const PrimParams& P, void* stream);

}  // namespace dashgpu
