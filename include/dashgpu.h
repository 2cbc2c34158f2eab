/*
 * libdashgpu — B200-native LabelTensor garble/evaluate engine for the
 * arithmetic garbled-circuit scheme of arXiv 2302.06361 ("Dash").
 *
 * C-ABI drop-in boundary.  Each entry point replaces one call of the
 * reference's dash:: C++ API (paths under /root/reference/proj/core/):
 *
 *   dashgpu_garble          <- dash::garble          include/dash/garble.hpp:93-94
 *   dashgpu_garble_inputs   <- dash::garble_inputs   include/dash/garble.hpp:97-99
 *   dashgpu_evaluate        <- dash::evaluate        include/dash/garble.hpp:103-105
 *   dashgpu_decode_outputs  <- dash::decode_outputs  include/dash/garble.hpp:110-112
 *   dashgpu_export_gc       <- dash::serialize_garbled_circuit  garble.hpp:116
 *   dashgpu_export_encoding <- dash::serialize_encoding         garble.hpp:119
 *   dashgpu_export_decoding <- dash::serialize_decoding         garble.hpp:122
 *   dashgpu_export_bundle   <- dash::bundle_payload             garble.hpp:131
 *   dashgpu_import_bundle   <- dash::bundle_from_payload        garble.hpp:132-134
 *   dashgpu_import_gc       <- dash::parse_garbled_circuit      garble.hpp:117 (garble.cpp:368-403)
 *   dashgpu_circuit_create  <- dash::validate_circuit + circuit_layout   circuit.hpp:26, garble.hpp:86-88
 *   dashgpu_circuit_info    <- dash::count_circuit / GarbleStats         circuit.hpp:61-62, garble.hpp:36-41
 *
 * Differences by design: every call is batched over `batch` independent
 * inferences (one 16-byte seed each, garbled circuits are single-use), all
 * label material stays resident in HBM (one structure-of-arrays buffer per
 * CRT modulus), and errors are status codes instead of exceptions:
 * DASHGPU_ERR_DATA <-> dash::DataError (CLI exit 3), DASHGPU_ERR_AUTH <->
 * dash::AuthenticityError (exit 4), DASHGPU_ERR_OVERFLOW <-> dash::OverflowError.
 * dashgpu_last_error() returns the thread-local message of the last failure.
 * There is no CPU fallback: without a CUDA device every call returns
 * DASHGPU_ERR_CUDA.
 */
#ifndef DASHGPU_H
#define DASHGPU_H

#include <stddef.h>
#include <stdint.h>

#include "dash_circuit_desc.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DASHGPU_OK 0
#define DASHGPU_ERR 1
#define DASHGPU_ERR_CUDA 2
#define DASHGPU_ERR_DATA 3
#define DASHGPU_ERR_AUTH 4
#define DASHGPU_ERR_OVERFLOW 5

typedef struct dashgpu_circuit dashgpu_circuit;
typedef struct dashgpu_network dashgpu_network;
typedef struct dashgpu_bundle dashgpu_bundle;

typedef struct dashgpu_circuit_info {
    int32_t k;
    uint32_t n_layers;
    uint64_t n_in, n_out;
    uint64_t cts, gates, wires;      /* per inference (GarbleStats, garble.hpp:36-41) */
    uint32_t sign_t;                 /* mixed-radix digits (0 when no activation) */
    uint16_t radices[32];
    uint64_t relu_elements;          /* activation elements per inference */
    uint64_t linear_macs;            /* digit multiply-accumulates per inference and pass */
    uint64_t act_uc_cts;             /* ciphertexts per ReLU element (garbler writes) */
    uint64_t act_eval_rows;          /* ciphertext rows one ReLU evaluation reads */
    uint32_t max_slots;
} dashgpu_circuit_info;

/* dashgpu_infer enqueues a whole sub-batch without host syncs, so it reports
 * the sub-batch wall time in ms_garble (the other phase fields stay 0);
 * dashgpu_infer_stream fills every phase. */
typedef struct dashgpu_timing {
    double ms_garble, ms_encode, ms_evaluate, ms_decode, ms_total;
    uint64_t h2d_bytes, d2h_bytes;
    uint32_t sub_batches;
    uint32_t layerwise; /* dashgpu_infer: 1 = layer-windowed sub-batches */
} dashgpu_timing;

const char* dashgpu_last_error(void);
int dashgpu_version(void);
/* Selects the CUDA device and uploads the constant tables. */
/* 1 = the CUDA engine (this library); anything else is a test build. */
int dashgpu_backend(void);
int dashgpu_init(int device);
/* Stream all work of the calling host thread is enqueued on (a cudaStream_t;
 * NULL = legacy default).  Thread-local: each host thread drives its own. */
int dashgpu_set_stream(void* stream);
/* Per-call device and stream: selects `device` for the calling
 * host thread (uploading the constant tables on first use of that device)
 * and sets the thread's stream.  Circuits and networks are bound to the
 * device they were first used on; dashgpu_infer keeps one workspace per
 * stream, so threads on different streams run one circuit concurrently. */
int dashgpu_use(int device, void* stream);

/* ---- circuits (host) ---- */
int dashgpu_circuit_create(const dash_circuit_desc* desc, dashgpu_circuit** out);
void dashgpu_circuit_destroy(dashgpu_circuit* c);
int dashgpu_circuit_info_get(const dashgpu_circuit* c, dashgpu_circuit_info* out);
/* Deterministic synthetic models: the reference test builders
 * (tests/support/test_models.hpp: model_a, model_c, model_d, model_f_dims,
 * model_tiny) plus "lenet5", "minionn" (paper Model F) and "relu<N>" /
 * "sign<N>" single-layer sweeps. */
int dashgpu_model_build(const char* name, uint32_t seed, int k, int private_weights,
                        dashgpu_circuit** out);
/* View of the circuit's quantized parameters (valid while c lives). */
int dashgpu_circuit_desc_view(const dashgpu_circuit* c, dash_circuit_desc* out);
/* testsupport::random_input(c, rng(seed), lo, hi) */
int dashgpu_random_input(const dashgpu_circuit* c, uint32_t seed, int lo, int hi, int64_t* out);
/* circuit_plain_forward (circuit.hpp:48-50), host reference semantics. */
int dashgpu_plain_forward(const dashgpu_circuit* c, const int64_t* in, int64_t* out);

/* ---- garbling / evaluation (device) ---- */
/* seeds: batch*16 bytes (host).  The network keeps the garbled circuit,
 * encoding and decoding information of every inference in HBM. */
int dashgpu_garble(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch,
                   dashgpu_network** out);
void dashgpu_network_destroy(dashgpu_network* n);
/* Garbler side, once the GCs have been exported (serialize_garbled_circuit
 * handed them to the evaluator): frees the ciphertexts, gadget slots and
 * per-layer planes, keeping only what garble_inputs and decode_outputs need
 * (offsets and their multiples, input base labels, decoding tables) -- the
 * reference garbler likewise keeps only EncodingInfo / DecodingInfo.  Later
 * export_gc / evaluate / layer calls on n fail with DASHGPU_ERR_DATA. */
int dashgpu_network_release_gc(dashgpu_network* n);
/* values: host [batch][n_in] signed quantized inputs */
int dashgpu_garble_inputs(dashgpu_network* n, const int64_t* values, dashgpu_bundle** out);
int dashgpu_evaluate(dashgpu_network* n, const dashgpu_bundle* in, dashgpu_bundle** out);
/* values: host [batch][n_out]; DASHGPU_ERR_AUTH if any label misses its table */
int dashgpu_decode_outputs(dashgpu_network* n, const dashgpu_bundle* out, int64_t* values);
void dashgpu_bundle_destroy(dashgpu_bundle* b);

/* ---- layer level (reference layer.hpp:79-97) ----
 * dashgpu_network_setup: the garbling environment of garble() without any
 * layer (offsets R_m and their multiples, zero-wire and input base labels,
 * seed commitment; garble.cpp:134-204).  dashgpu_input_base: the input base
 * labels (EncodingInfo::input_labels).  dashgpu_layer_garble = garble_layer
 * (layer.hpp:85-90): base labels of layer li's input (in2: second operand of
 * the Add extension, else NULL) -> base labels of its output; the layer's
 * rows land at layer_ct_base[li] of every inference's GC.
 * dashgpu_layer_eval = eval_layer (layer.hpp:93-97) on active labels.
 * dashgpu_network_finish: decoding tables from the final base labels, after
 * which the network equals the one dashgpu_garble builds.
 * dashgpu_layer_count = count_layer (layer.hpp:79-80): cts, gates, wires. */
int dashgpu_network_setup(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch,
                          dashgpu_network** out);
int dashgpu_input_base(dashgpu_network* n, dashgpu_bundle** out);
int dashgpu_layer_garble(dashgpu_network* n, uint32_t layer, const dashgpu_bundle* in,
                         const dashgpu_bundle* in2, dashgpu_bundle** out);
int dashgpu_layer_eval(dashgpu_network* n, uint32_t layer, const dashgpu_bundle* in,
                       const dashgpu_bundle* in2, dashgpu_bundle** out);
int dashgpu_network_finish(dashgpu_network* n, const dashgpu_bundle* final_base);
int dashgpu_layer_count(const dashgpu_circuit* c, uint32_t layer, uint64_t* cts_gates_wires3);

/* ---- t_proj primitive (gadgets.hpp:146-176) over n independent gates ----
 * garble: seed = the PRF seed (offsets R_p, R_q and the fresh out0 labels,
 * prf.cpp:11-32); in: n compressed base labels mod p (u128 as 2 x u64 LE);
 * phi: p table values mod q; gates / wires: gate ids and fresh wire ids;
 * rows: [n][p] u128 (row (color + a) mod p = Enc_{in + aR_p}(out0 + phi(a) R_q));
 * out0: [n] compressed fresh labels mod q; offsets (may be NULL): R_p, R_q.
 * eval: active labels in + rows -> active out labels (compressed). */
int dashgpu_proj_garble(const uint8_t* seed16, uint32_t n, int p, int q, const uint8_t* phi,
                        const uint64_t* in, const uint64_t* gates, const uint64_t* wires,
                        uint64_t* rows, uint64_t* out0, uint64_t* offsets);
int dashgpu_proj_eval(uint32_t n, int p, int q, const uint64_t* in, const uint64_t* gates,
                      const uint64_t* rows, uint64_t* out);
/* Device-resident form for throughput (the raw t_proj sweep of SURVEY 8(d)
 * (ii); the reference times one gate at a time, bench_main.cpp:40-74):
 * a context holds the PRF key schedule, R_p / R_q multiples and phi; every
 * buffer is a DEVICE pointer with the layouts above (in / out0 / out: n x
 * 16 B, gates / wires: n x u64, rows: n x p x 16 B); calls are enqueued on
 * the calling thread's stream without a host sync. */
typedef struct dashgpu_proj_ctx dashgpu_proj_ctx;
int dashgpu_proj_ctx_create(const uint8_t* seed16, int p, int q, const uint8_t* phi, dashgpu_proj_ctx** out);
void dashgpu_proj_ctx_destroy(dashgpu_proj_ctx* c);
int dashgpu_proj_garble_dev(const dashgpu_proj_ctx* c, uint32_t n, const void* in, const void* gates,
                            const void* wires, void* rows, void* out0);
int dashgpu_proj_eval_dev(const dashgpu_proj_ctx* c, uint32_t n, const void* in, const void* gates,
                          const void* rows, void* out);

/* ---- LabelTensor images (label_tensor.hpp:14-42: per lane, label-major
 * u16 digits [batch][elements][n_p]) <-> device bundles (u8 SoA planes) ---- */
int dashgpu_bundle_info(const dashgpu_bundle* b, uint32_t* batch, uint64_t* elements);
int dashgpu_bundle_from_labels(dashgpu_network* n, uint64_t elements, const uint16_t* const* lanes,
                               int output, dashgpu_bundle** out);
int dashgpu_bundle_labels(const dashgpu_bundle* b, int lane, uint16_t* out);

/* ---- reference wire formats (byte-identical to the reference) ---- */
int dashgpu_export_gc(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len);
int dashgpu_export_encoding(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len);
int dashgpu_export_decoding(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len);
int dashgpu_export_bundle(const dashgpu_bundle* bd, uint32_t b, uint8_t* buf, size_t cap, size_t* len);
/* payload of every inference concatenated ([batch][k][n][16] bytes) */
int dashgpu_import_bundle(dashgpu_network* n, const uint8_t* data, size_t len, int output,
                          dashgpu_bundle** out);
/* evaluator side (EvaluatorService GC_TRANSFER, protocol.cpp:309-316):
 * batch serialized GCs (export_gc format) of one circuit -> a network that
 * evaluates them as inferences 0..batch-1 (garbling it returns
 * DASHGPU_ERR_DATA: private weights are not in a GC).  Owns its circuit. */
int dashgpu_import_gc(const uint8_t* const* gcs, const size_t* lens, uint32_t batch, dashgpu_network** out);
/* The same with the ciphertexts kept in pinned HOST memory (reference cts
 * order) instead of HBM: dashgpu_evaluate moves each layer's rows into a
 * one-layer device window just before evaluating it, so an
 * evaluator holds GCs larger than HBM.  Everything else is dashgpu_import_gc's
 * (checks, export_gc, tamper, release). */
int dashgpu_import_gc_host(const uint8_t* const* gcs, const size_t* lens, uint32_t batch, dashgpu_network** out);
/* the circuit a network garbles / evaluates (borrowed: lives as long as the network) */
int dashgpu_network_circuit(const dashgpu_network* n, const dashgpu_circuit** out);
/* fault injection for tests: XOR `mask` (16 bytes) into ciphertext `index` of inference b */
int dashgpu_tamper_ct(dashgpu_network* n, uint32_t b, uint64_t index, const uint8_t* mask16);

/* ---- fused pipeline: garble + garble_inputs + evaluate + decode_outputs ----
 * inputs [batch][n_in], outputs [batch][n_out].  on_device=0: host buffers
 * (copies inside the call); on_device=1: device pointers (seeds too).
 * Sub-batches automatically when the garbled circuits exceed free HBM; such
 * sub-batches are garbled and evaluated layer by layer through a one-layer
 * ciphertext window when that admits more inferences per pass
 * (t->layerwise; DASHGPU_LAYERWISE=0/1 forces the schedule). */
int dashgpu_infer(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch,
                  const int64_t* inputs, int64_t* outputs, int on_device, dashgpu_timing* t);

/* Digest parity mode of streamed whole-network garbling:
 * garbles the batch layer by layer through a one-layer ciphertext window
 * (no whole GC is held) and writes, per inference and layer, the tree
 * SHA-256 of the layer's ciphertexts in GarbledCircuit::cts order
 * (garble.hpp:46-53): SHA-256 over the SHA-256 digests of its 64 KiB leaves;
 * a layer without ciphertexts gets SHA-256 of the empty string.
 * seeds [batch][16] (host), digests [batch][n_layers][32] (host). */
int dashgpu_garble_digest(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch, uint8_t* digests);
/* The same digests of a network's held GC (garbled whole, or imported into
 * HBM or host memory), inference b: digests [n_layers][32] (host).  An
 * evaluator checks a received GC against the garbler's digest list. */
int dashgpu_network_digest(const dashgpu_network* n, uint32_t b, uint8_t* digests);

/* Streamed serialize_garbled_circuit (garble.cpp:347-403):
 * garbles the batch layer by layer through a one-layer ciphertext window and
 * calls sink(user, b, data, len) with inference b's GC bytes in order --
 * header, every layer's rows in GarbledCircuit::cts order, commitment -- so
 * the concatenation for each b equals dashgpu_export_gc(net, b) of a whole
 * garbling, while the device never holds a whole GC.  A nonzero sink return
 * aborts with DASHGPU_ERR_DATA.  *out (optional) receives the network with
 * its encoding / decoding material, as after dashgpu_network_release_gc. */
typedef int (*dashgpu_gc_sink)(void* user, uint32_t b, const uint8_t* data, size_t len);
int dashgpu_garble_stream(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch, dashgpu_gc_sink sink,
                          void* user, dashgpu_network** out);

/* Streamed inference of a single activation-layer circuit (the label-ops
 * sweep: {input_shape={N}, layers={relu()}}, reference bench_main.cpp:156-162,
 * garble_layer/eval_layer layer.hpp:85-97 over element ranges).  Element
 * chunks of chunk_elems are garbled, encoded, evaluated and decoded in turn
 * with the reference's gate/wire/ciphertext numbering, so the tables of the
 * whole layer (1.8 TB at N = 2^26, k = 8) never exist at once.  Host buffers:
 * seeds [batch][16], inputs [batch][N], outputs [batch][N]; gc_out (optional,
 * may be NULL) receives every chunk's ciphertexts, [batch][N*uc_cts][16]
 * bytes = the layer's GarbledCircuit::cts (garble.hpp:46-53). */
int dashgpu_infer_stream(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch,
                         const int64_t* inputs, int64_t* outputs, uint64_t chunk_elems,
                         uint8_t* gc_out, dashgpu_timing* t);
/* The same over elements [u_begin, u_end) only (a layer shards
 * by element range across GPUs with no exchange -- gate / wire / row ids are
 * affine in the element index).  inputs / outputs / gc_out keep the full-layer
 * indexing; only the range is read / written. */
int dashgpu_infer_stream_range(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch,
                               const int64_t* inputs, int64_t* outputs, uint64_t chunk_elems,
                               uint64_t u_begin, uint64_t u_end, uint8_t* gc_out, dashgpu_timing* t);

/* ---- per-kernel CUDA-event timing on the launching stream ---- */
int dashgpu_profile(int enable);
/* kinds: 0 act-garble 1 act-eval 2 linear 3 priv-garble 4 priv-eval 5 setup 6 encode 7 decode 8 misc */
int dashgpu_profile_read(double* ms, uint64_t* launches, int max_kinds);
/* Shape of the most recent activation-layer launch (garble = 1: the combined
 * garbling launch; 0: the last evaluation launch): out[0] variant (0 none,
 * 1 lane-group evaluation, 2 level-parallel garbling, 3 lane-group garbling,
 * 4 one element per thread), out[1] tape chunks per element, out[2] grid,
 * out[3] work items, out[4] lanes per element.  Lets parity tests pin the
 * launch configuration a benchmark times. */
int dashgpu_last_act_launch(int garble, uint32_t out[5]);
/* The element tape of the circuit's ReLU (kind 3) or SignAct (kind 4)
 * gadget as recorded from the reference gadget DAG (gadgets.hpp:146-481):
 * per op its kind (1 proj, 2 grr, 3 half, 4 mm-half, 5 add, 6 add-const,
 * 7 output, 8 fused add), input / output moduli and gate / wire / ciphertext
 * offsets inside the element.  ops == NULL: *n = op count only. */
typedef struct {
    uint32_t kind, pm, qm, gate_off, wire_off, ct_off;
} dashgpu_tape_op;
int dashgpu_activation_tape(const dashgpu_circuit* c, int kind, dashgpu_tape_op* ops, uint32_t cap, uint32_t* n);

/* ---- primitive kernels (parity tests) ----
 * op 0: decompress_mod(in[i], m) -> digits (u16), then compress -> out[i]
 * op 1: AES-128 under the all-zero key (fixed permutation pi)
 * op 2: AES-128 under key16
 * op 3: LabelPrf::draw(wires[i], stream=q, m) -> digits
 * op 4: out[i] = encrypt_label(key=decompress(in[i], m), tweak{gate, i%7, i%3}, msg=decompress(out[i], q))
 * op 5: digits = decrypt_label(key=decompress(in[i], m), tweak{gate, i%7, i%3}, ct=out[i], q)
 * in/out: n u128 as (lo, hi) u64 pairs; digits: n*128 u16. */
int dashgpu_prim(int op, uint32_t n, int m, int q, const uint64_t* in, uint64_t* out, uint16_t* digits,
                 const uint8_t* key16, const uint64_t* wires, uint64_t gate);

#ifdef __cplusplus
}
#endif
#endif
