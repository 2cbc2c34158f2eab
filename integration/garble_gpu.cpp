// dash::gpu shim over the C ABI (include/dashgpu.h).  See garble_gpu.hpp.
// Compiled against the reference's own headers and sources by
// oracle/Makefile (target `shim`) and checked by integration/shim_check.cpp.
#include "garble_gpu.hpp"

#include <string>

#include "dash/errors.hpp"
#include "dashgpu.h"

namespace dash::gpu {
namespace {

void check(int rc) {
    if (rc == DASHGPU_OK) return;
    const std::string msg = dashgpu_last_error();
    if (rc == DASHGPU_ERR_AUTH) throw AuthenticityError(msg);
    if (rc == DASHGPU_ERR_OVERFLOW) throw OverflowError(msg);
    if (rc == DASHGPU_ERR_DATA) throw DataError(msg);
    throw Error(msg);
}

// device + stream of this call (constant tables are uploaded once per device)
void use(int device, void* stream) { check(dashgpu_use(device, stream)); }

struct CircuitHandle {
    dashgpu_circuit* c = nullptr;
    ~CircuitHandle() { dashgpu_circuit_destroy(c); }
};
struct NetworkHandle {
    dashgpu_network* n = nullptr;
    ~NetworkHandle() { dashgpu_network_destroy(n); }
};
struct BundleHandle {
    dashgpu_bundle* b = nullptr;
    ~BundleHandle() { dashgpu_bundle_destroy(b); }
};

// dash::Circuit (circuit.hpp:13-19, layer.hpp:25-54) -> the plain C image
void upload(const Circuit& c, CircuitHandle& h) {
    std::vector<dash_layer_desc> ls;
    for (const Layer& l : c.layers) {
        dash_layer_desc d{};
        d.kind = static_cast<int32_t>(l.kind);
        d.private_weights = l.private_weights;
        d.in_dim = l.in_dim;
        d.out_dim = l.out_dim;
        d.in_ch = l.in_ch;
        d.out_ch = l.out_ch;
        d.filter = l.filter;
        d.stride = l.stride;
        d.q_weights = l.q_weights.empty() ? nullptr : l.q_weights.data();
        d.n_weights = l.q_weights.size();
        d.q_biases = l.q_biases.empty() ? nullptr : l.q_biases.data();
        d.n_biases = l.q_biases.size();
        ls.push_back(d);
    }
    dash_circuit_desc d{};
    d.k = c.k;
    if (c.input_shape.size() > 8) throw DataError("input rank out of range");
    d.rank = static_cast<uint32_t>(c.input_shape.size());
    for (size_t i = 0; i < c.input_shape.size(); ++i) d.input_shape[i] = c.input_shape[i];
    d.sign_target = c.sign_target;
    d.alpha = c.quant.alpha;
    d.n_layers = static_cast<uint32_t>(ls.size());
    d.layers = ls.data();
    check(dashgpu_circuit_create(&d, &h.c));
}

template <class Fn, class Obj>
std::vector<uint8_t> fetch(Fn fn, Obj* o, uint32_t b) {
    size_t len = 0;
    check(fn(o, b, nullptr, 0, &len));
    std::vector<uint8_t> buf(len);
    check(fn(o, b, buf.data(), len, &len));
    return buf;
}

}  // namespace

std::vector<GarbledNetwork> garble_batch(const Circuit& circuit, std::span<const Seed> seeds, int device,
                                         void* stream) {
    use(device, stream);
    CircuitHandle c;
    upload(circuit, c);
    std::vector<uint8_t> s;
    for (const Seed& x : seeds) s.insert(s.end(), x.begin(), x.end());
    NetworkHandle n;
    check(dashgpu_garble(c.c, s.data(), static_cast<uint32_t>(seeds.size()), &n.n));
    dashgpu_circuit_info info;
    check(dashgpu_circuit_info_get(c.c, &info));
    std::vector<GarbledNetwork> out(seeds.size());
    for (uint32_t b = 0; b < seeds.size(); ++b) {
        // the reference's own parsers rebuild the dash:: objects from the
        // byte-identical wire formats (garble.cpp:368-463)
        out[b].gc = parse_garbled_circuit(fetch(dashgpu_export_gc, n.n, b));
        out[b].enc = parse_encoding(fetch(dashgpu_export_encoding, n.n, b));
        out[b].dec = parse_decoding(fetch(dashgpu_export_decoding, n.n, b));
        out[b].stats = {info.cts, info.gates, info.wires};
    }
    return out;
}

GarbledNetwork garble(const Circuit& circuit, const Seed& seed, int /*threads*/, int device, void* stream) {
    return std::move(garble_batch(circuit, std::span<const Seed>(&seed, 1), device, stream)[0]);
}

std::vector<LabelTensor> garble_inputs(const EncodingInfo& enc, std::span<const q_val_t> values,
                                       const CrtBase& base, int /*device*/, void* /*stream*/) {
    // label = base + (enc(v) mod p)·R_p: one label add per input element and
    // lane on data the caller holds in host memory (garble.cpp:242-263); the
    // batched device encoder is dashgpu_garble_inputs on a dashgpu_network.
    return dash::garble_inputs(enc, values, base);
}

std::vector<LabelTensor> evaluate(const GarbledCircuit& gc, const std::vector<LabelTensor>& inputs, int /*threads*/,
                                  int device, void* stream) {
    use(device, stream);
    const std::vector<uint8_t> bytes = serialize_garbled_circuit(gc);
    const uint8_t* p = bytes.data();
    const size_t len = bytes.size();
    NetworkHandle n;
    check(dashgpu_import_gc(&p, &len, 1, &n.n));
    const std::vector<uint8_t> payload = bundle_payload(inputs);
    BundleHandle in, out;
    check(dashgpu_import_bundle(n.n, payload.data(), payload.size(), 0, &in.b));
    check(dashgpu_evaluate(n.n, in.b, &out.b));
    const std::vector<uint8_t> gout = fetch(dashgpu_export_bundle, out.b, 0);
    dim_t shape = circuit_shapes(gc.circuit).back();
    return bundle_from_payload(gout, crt_base(gc.circuit.k), shape);
}

}  // namespace dash::gpu
