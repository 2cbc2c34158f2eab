// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI harness around the UNMODIFIED reference library (the dash_core
// sources under /root/reference/proj/core/src, compiled in place by
// oracle/Makefile into oracle/_ref/libdashref.so).  It exposes the reference's
// own public API (proj/core/include/dash/garble.hpp:93-136, cipher.hpp,
// label.hpp, prf.hpp, mixed_radix.hpp) through plain pointers so that the
// Python tests, the golden-fixture generator and bench.py's reference arm can
// drive the real reference implementation.  Nothing here re-implements the
// algorithm; every function forwards to dash::.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <omp.h>

#include "dash/cipher.hpp"
#include "dash/circuit.hpp"
#include "dash/crt.hpp"
#include "dash/gadgets.hpp"
#include "dash/garble.hpp"
#include "dash/label.hpp"
#include "dash/mixed_radix.hpp"
#include "dash/prf.hpp"
#include "test_models.hpp"  // reference tests/support (deterministic builders)

#include "dash_circuit_desc.h"

using namespace dash;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const AuthenticityError& e) {
        g_err = e.what();
        return 4;
    } catch (const DataError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

u128 load_u128(const uint64_t* p) { return make_u128(p[1], p[0]); }
void store_u128(uint64_t* p, u128 v) {
    p[0] = lo64(v);
    p[1] = hi64(v);
}

Label label_from(const uint16_t* d, crt_val_t m) {
    Label l = Label::shape(m);
    for (int i = 0; i < l.n; ++i) l.d[i] = d[i];
    return l;
}
void label_to(const Label& l, uint16_t* d) {
    for (int i = 0; i < l.n; ++i) d[i] = l.d[i];
}

Seed seed_from_bytes(const uint8_t* s) {
    Seed seed;
    std::memcpy(seed.data(), s, 16);
    return seed;
}

struct CircuitHandle {
    Circuit c;
    std::vector<dash_layer_desc> layer_descs;
    dash_circuit_desc desc{};
};

size_t copy_out(const std::vector<uint8_t>& v, uint8_t* buf, size_t cap) {
    if (buf && cap >= v.size()) std::memcpy(buf, v.data(), v.size());
    return v.size();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ----- circuits --------------------------------------------------------------

void* ref_circuit_from_desc(const dash_circuit_desc* d) {
    auto* h = new CircuitHandle;
    h->c.k = d->k;
    h->c.input_shape.assign(d->input_shape, d->input_shape + d->rank);
    h->c.sign_target = d->sign_target;
    h->c.quant.alpha = d->alpha;
    for (uint32_t i = 0; i < d->n_layers; ++i) {
        const dash_layer_desc& s = d->layers[i];
        if (s.kind > DASH_LAYER_FLATTEN || s.src || s.src2 || s.pad) {
            // Pad2d / Add / DAG inputs are extensions of this repo (dash_circuit_desc.h)
            delete h;
            g_err = "circuit uses layer extensions the reference does not have";
            return nullptr;
        }
        Layer l;
        l.kind = static_cast<LayerKind>(s.kind);
        l.private_weights = s.private_weights != 0;
        l.in_dim = s.in_dim;
        l.out_dim = s.out_dim;
        l.in_ch = s.in_ch;
        l.out_ch = s.out_ch;
        l.filter = s.filter;
        l.stride = s.stride;
        if (s.q_weights) l.q_weights.assign(s.q_weights, s.q_weights + s.n_weights);
        if (s.q_biases) l.q_biases.assign(s.q_biases, s.q_biases + s.n_biases);
        h->c.layers.push_back(std::move(l));
    }
    return h;
}

// Reference test-support builders (tests/support/test_models.hpp:79-140).
void* ref_model(const char* name, uint32_t seed, int k, int priv) {
    auto* h = new CircuitHandle;
    const std::string n = name;
    if (n == "model_a") h->c = testsupport::model_a(seed, k);
    else if (n == "model_c") h->c = testsupport::model_c(seed, k);
    else if (n == "model_d") h->c = testsupport::model_d(seed, k);
    else if (n == "model_f_dims") h->c = testsupport::model_f_dims(seed, k);
    else if (n == "model_tiny") h->c = testsupport::model_tiny(seed, k, priv != 0);
    else {
        delete h;
        g_err = "unknown model";
        return nullptr;
    }
    return h;
}

// Exposes a handle's circuit as a desc (pointers valid while the handle lives).
const dash_circuit_desc* ref_circuit_desc(void* hv) {
    auto* h = static_cast<CircuitHandle*>(hv);
    h->layer_descs.clear();
    for (const auto& l : h->c.layers) {
        dash_layer_desc s{};
        s.kind = static_cast<int32_t>(l.kind);
        s.private_weights = l.private_weights;
        s.in_dim = l.in_dim;
        s.out_dim = l.out_dim;
        s.in_ch = l.in_ch;
        s.out_ch = l.out_ch;
        s.filter = l.filter;
        s.stride = l.stride;
        s.q_weights = l.q_weights.empty() ? nullptr : l.q_weights.data();
        s.n_weights = l.q_weights.size();
        s.q_biases = l.q_biases.empty() ? nullptr : l.q_biases.data();
        s.n_biases = l.q_biases.size();
        h->layer_descs.push_back(s);
    }
    h->desc.k = h->c.k;
    h->desc.rank = static_cast<uint32_t>(h->c.input_shape.size());
    for (size_t i = 0; i < h->c.input_shape.size(); ++i)
        h->desc.input_shape[i] = h->c.input_shape[i];
    h->desc.sign_target = h->c.sign_target;
    h->desc.alpha = h->c.quant.alpha;
    h->desc.n_layers = static_cast<uint32_t>(h->layer_descs.size());
    h->desc.layers = h->layer_descs.data();
    return &h->desc;
}

void ref_circuit_free(void* h) { delete static_cast<CircuitHandle*>(h); }

// testsupport::random_input(c, rng(seed), lo, hi)
int ref_random_input(void* hv, uint32_t seed, int lo, int hi, int64_t* out) {
    auto* h = static_cast<CircuitHandle*>(hv);
    auto g = testsupport::rng(seed);
    auto v = testsupport::random_input(h->c, g, lo, hi);
    std::copy(v.begin(), v.end(), out);
    return static_cast<int>(v.size());
}

int ref_plain_forward(void* hv, const int64_t* in, int64_t* out) {
    auto* h = static_cast<CircuitHandle*>(hv);
    return guard([&] {
        const CrtBase base = crt_base(h->c.k);
        std::vector<q_val_t> x(in, in + size_of(h->c.input_shape));
        auto y = circuit_plain_forward(h->c, x, base);
        std::copy(y.begin(), y.end(), out);
    });
}

// ----- whole-network API (garble.hpp:93-112) ---------------------------------

void* ref_garble(void* hv, const uint8_t* seed16, int threads) {
    auto* h = static_cast<CircuitHandle*>(hv);
    GarbledNetwork* net = nullptr;
    int rc = guard([&] {
        net = new GarbledNetwork(garble(h->c, seed_from_bytes(seed16), threads));
    });
    return rc == 0 ? net : nullptr;
}
void ref_net_free(void* n) { delete static_cast<GarbledNetwork*>(n); }

size_t ref_net_gc_bytes(void* n, uint8_t* buf, size_t cap) {
    return copy_out(serialize_garbled_circuit(static_cast<GarbledNetwork*>(n)->gc), buf, cap);
}
size_t ref_net_enc_bytes(void* n, uint8_t* buf, size_t cap) {
    return copy_out(serialize_encoding(static_cast<GarbledNetwork*>(n)->enc), buf, cap);
}
size_t ref_net_dec_bytes(void* n, uint8_t* buf, size_t cap) {
    return copy_out(serialize_decoding(static_cast<GarbledNetwork*>(n)->dec), buf, cap);
}
uint64_t ref_net_cts_count(void* n) {
    return static_cast<GarbledNetwork*>(n)->gc.cts.size();
}
// Raw ciphertext blob as (lo, hi) u64 pairs.
void ref_net_cts(void* n, uint64_t* out) {
    const auto& cts = static_cast<GarbledNetwork*>(n)->gc.cts;
    for (size_t i = 0; i < cts.size(); ++i) store_u128(out + 2 * i, cts[i]);
}
int ref_net_layer_ct_base(void* n, uint64_t* out) {
    const auto& v = static_cast<GarbledNetwork*>(n)->gc.layer_ct_base;
    std::copy(v.begin(), v.end(), out);
    return static_cast<int>(v.size());
}
void ref_net_stats(void* n, uint64_t* out3) {
    const auto& s = static_cast<GarbledNetwork*>(n)->stats;
    out3[0] = s.ciphertexts;
    out3[1] = s.gates;
    out3[2] = s.wires;
}

void* ref_garble_inputs(void* n, const int64_t* values, size_t count) {
    auto* net = static_cast<GarbledNetwork*>(n);
    std::vector<LabelTensor>* out = nullptr;
    int rc = guard([&] {
        const CrtBase base = crt_base(net->enc.k);
        out = new std::vector<LabelTensor>(
            garble_inputs(net->enc, std::span<const q_val_t>(values, count), base));
    });
    return rc == 0 ? out : nullptr;
}

void* ref_evaluate(void* n, void* bundle, int threads) {
    auto* net = static_cast<GarbledNetwork*>(n);
    auto* in = static_cast<std::vector<LabelTensor>*>(bundle);
    std::vector<LabelTensor>* out = nullptr;
    int rc = guard([&] {
        out = new std::vector<LabelTensor>(evaluate(net->gc, *in, threads));
    });
    return rc == 0 ? out : nullptr;
}

int ref_decode(void* n, void* bundle, int64_t* values) {
    auto* net = static_cast<GarbledNetwork*>(n);
    auto* out = static_cast<std::vector<LabelTensor>*>(bundle);
    return guard([&] {
        const CrtBase base = crt_base(net->dec.k);
        auto v = decode_outputs(net->dec, *out, base);
        std::copy(v.begin(), v.end(), values);
    });
}

// Parses a (possibly tampered) GC and evaluates it: DataError/Authenticity
// behaviour of the reference for fault-injection tests.
int ref_eval_gc_bytes(const uint8_t* gc, size_t len, void* bundle, int threads,
                      void** out_bundle) {
    auto* in = static_cast<std::vector<LabelTensor>*>(bundle);
    return guard([&] {
        GarbledCircuit parsed = parse_garbled_circuit(std::span<const uint8_t>(gc, len));
        *out_bundle = new std::vector<LabelTensor>(evaluate(parsed, *in, threads));
    });
}

size_t ref_bundle_payload(void* bundle, uint8_t* buf, size_t cap) {
    return copy_out(bundle_payload(*static_cast<std::vector<LabelTensor>*>(bundle)), buf, cap);
}
void ref_bundle_free(void* b) { delete static_cast<std::vector<LabelTensor>*>(b); }

// ----- primitives ------------------------------------------------------------

void ref_aes_fixed(const uint64_t* in, uint64_t* out) {
    store_u128(out, fixed_permutation().encrypt(load_u128(in)));
}
void ref_aes_key(const uint8_t* key16, const uint64_t* in, uint64_t* out) {
    std::array<uint8_t, 16> k;
    std::memcpy(k.data(), key16, 16);
    Aes128 a(k);
    store_u128(out, a.encrypt(load_u128(in)));
}
void ref_davies_meyer(const uint64_t* in, uint64_t* out) {
    store_u128(out, davies_meyer(load_u128(in)));
}
int ref_n_digits(int m) { return n_digits(static_cast<crt_val_t>(m)); }
void ref_compress(int m, const uint16_t* d, uint64_t* out) {
    store_u128(out, compress(label_from(d, static_cast<crt_val_t>(m))));
}
void ref_decompress_mod(const uint64_t* c, int m, uint16_t* d) {
    label_to(decompress_mod(load_u128(c), static_cast<crt_val_t>(m)), d);
}
void ref_seed_from_string(const char* s, uint8_t* out16) {
    Seed seed = seed_from_string(s);
    std::memcpy(out16, seed.data(), 16);
}
void ref_prf_label(const uint8_t* seed16, uint64_t wire, int m, uint16_t* d) {
    LabelPrf prf(seed_from_bytes(seed16));
    label_to(prf.label(wire, static_cast<crt_val_t>(m)), d);
}
void ref_prf_offset(const uint8_t* seed16, int m, uint16_t* d) {
    LabelPrf prf(seed_from_bytes(seed16));
    label_to(prf.offset(static_cast<crt_val_t>(m)), d);
}
void ref_pad_bits(int m, const uint16_t* k1, uint64_t gate, uint32_t row,
                  uint32_t slot, uint64_t* out) {
    store_u128(out, pad_bits(label_from(k1, static_cast<crt_val_t>(m)),
                             Tweak{gate, row, slot}));
}
void ref_pad_bits2(int m1, const uint16_t* k1, int m2, const uint16_t* k2,
                   uint64_t gate, uint32_t row, uint32_t slot, uint64_t* out) {
    store_u128(out, pad_bits(label_from(k1, static_cast<crt_val_t>(m1)),
                             label_from(k2, static_cast<crt_val_t>(m2)),
                             Tweak{gate, row, slot}));
}
void ref_encrypt_label(int mk, const uint16_t* k1, uint64_t gate, uint32_t row,
                       uint32_t slot, int mq, const uint16_t* msg, uint64_t* out) {
    store_u128(out, encrypt_label(label_from(k1, static_cast<crt_val_t>(mk)),
                                  Tweak{gate, row, slot},
                                  label_from(msg, static_cast<crt_val_t>(mq))));
}
void ref_decrypt_label(int mk, const uint16_t* k1, uint64_t gate, uint32_t row,
                       uint32_t slot, const uint64_t* ct, int q, uint16_t* out) {
    label_to(decrypt_label(label_from(k1, static_cast<crt_val_t>(mk)),
                           Tweak{gate, row, slot}, load_u128(ct),
                           static_cast<crt_val_t>(q)),
             out);
}

// Full-accuracy (target>=1) or reduced spec; returns t, radices into out.
int ref_choose_mixed_radix(int k, double target, uint16_t* radices) {
    int t = 0;
    int rc = guard([&] {
        const CrtBase base = crt_base(k);
        MixedRadixSpec s = target < 1.0 ? choose_mixed_radix(base, target)
                                        : choose_mixed_radix(base);
        t = s.t();
        for (int j = 0; j < t; ++j) radices[j] = s.radices[j];
    });
    return rc == 0 ? t : -rc;
}

// Per-element gadget costs {cts, gates, wires} for ReLU (kind 3) / SignAct (4).
int ref_element_cost(int k, double target, int kind, uint64_t* out3) {
    return guard([&] {
        Circuit c;
        c.k = k;
        c.input_shape = {1};
        c.sign_target = target;
        Layer l;
        l.kind = static_cast<LayerKind>(kind);
        c.layers = {l};
        const CrtBase base = crt_base(k);
        SignContext s = make_sign_context(base, target);
        CountCtx ctx = count_circuit(c, base, &s.plan);
        out3[0] = ctx.cts;
        out3[1] = ctx.gates;
        out3[2] = ctx.wires;
    });
}

// ----- CPU baseline timing (reference arm of bench.py) ------------------------
//
// One inference = garble + garble_inputs + evaluate + decode_outputs with a
// fresh seed.  mode 0: OpenMP intra-layer (threads inside,
// sequential over inferences); mode 1: inference-parallel (one inference per
// thread, threads=1 inside).  seeds: n*16 bytes; inputs: n*n_in values;
// outputs: n*n_out decoded values.  Returns wall seconds.
double ref_bench_infer(void* hv, int n, const uint8_t* seeds, const int64_t* inputs,
                       int64_t* outputs, int mode, int threads) {
    auto* h = static_cast<CircuitHandle*>(hv);
    const Circuit& c = h->c;
    const CrtBase base = crt_base(c.k);
    const size_t n_in = size_of(c.input_shape);
    const auto shapes = circuit_shapes(c);
    const size_t n_out = size_of(shapes.back());
    auto one = [&](int b, int inner) {
        GarbledNetwork net = garble(c, seed_from_bytes(seeds + 16 * b), inner);
        auto lanes = garble_inputs(net.enc,
                                   std::span<const q_val_t>(inputs + b * n_in, n_in), base);
        auto out = evaluate(net.gc, lanes, inner);
        auto v = decode_outputs(net.dec, out, base);
        std::copy(v.begin(), v.end(), outputs + b * n_out);
    };
    const auto t0 = std::chrono::steady_clock::now();
    int rc = guard([&] {
        if (mode == 0) {
            for (int b = 0; b < n; ++b) one(b, threads);
        } else {
            std::string err;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
            for (int b = 0; b < n; ++b) {
                try {
                    one(b, 1);
                } catch (const std::exception& e) {
#pragma omp critical
                    err = e.what();
                }
            }
            if (!err.empty()) throw Error(err);
        }
    });
    const auto t1 = std::chrono::steady_clock::now();
    if (rc != 0) return -1.0;
    return std::chrono::duration<double>(t1 - t0).count();
}

int ref_max_threads() { return omp_get_max_threads(); }

}  // extern "C"
