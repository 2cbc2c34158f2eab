// Drop-in proof for integration/garble_gpu.cpp (TEST INFRASTRUCTURE).
//
// Linked with the UNMODIFIED reference sources (proj/core/src) and
// libdashgpu: for each reference test model (tests/support/test_models.hpp)
// the circuit is garbled by dash::garble (CPU) and by dash::gpu::garble
// (B200), and every artifact must be byte-identical; the GPU-garbled network
// is then evaluated by dash::evaluate (CPU) and dash::gpu::evaluate (B200),
// and both decode to circuit_plain_forward.  A tampered output label must
// raise dash::AuthenticityError through the shim, a malformed GC
// dash::DataError.  Exit code 0 = all checks passed.
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "dash/circuit.hpp"
#include "dash/errors.hpp"
#include "dash/garble.hpp"
#include "garble_gpu.hpp"
#include "test_models.hpp"

using namespace dash;

static int failures = 0;
#define EXPECT(cond, what)                                         \
    do {                                                           \
        if (!(cond)) {                                             \
            std::printf("FAIL %s: %s\n", name.c_str(), what);      \
            ++failures;                                            \
        }                                                          \
    } while (0)

static Seed seed_of(uint32_t v) {
    Seed s{};
    for (int i = 0; i < 4; ++i) s[15 - i] = static_cast<uint8_t>(v >> (8 * i));  // big-endian hex(v)
    return s;
}

static void check_model(const std::string& name, const Circuit& c, uint32_t seed, uint32_t input_rng) {
    const Seed s = seed_of(seed);
    const GarbledNetwork cpu = dash::garble(c, s);
    const GarbledNetwork gpu = dash::gpu::garble(c, s);
    EXPECT(serialize_garbled_circuit(cpu.gc) == serialize_garbled_circuit(gpu.gc), "gc bytes");
    EXPECT(serialize_encoding(cpu.enc) == serialize_encoding(gpu.enc), "encoding bytes");
    EXPECT(serialize_decoding(cpu.dec) == serialize_decoding(gpu.dec), "decoding bytes");
    EXPECT(cpu.stats.ciphertexts == gpu.stats.ciphertexts && cpu.stats.gates == gpu.stats.gates &&
               cpu.stats.wires == gpu.stats.wires,
           "stats");
    const CrtBase base = crt_base(c.k);
    auto g = testsupport::rng(input_rng);
    const auto x = testsupport::random_input(c, g);
    const auto in = dash::gpu::garble_inputs(gpu.enc, x, base);
    const auto out_cpu = dash::evaluate(gpu.gc, in);
    const auto out_gpu = dash::gpu::evaluate(gpu.gc, in);
    EXPECT(bundle_payload(out_cpu) == bundle_payload(out_gpu), "garbled output bytes");
    const auto want = circuit_plain_forward(c, x, base);
    EXPECT(dash::gpu::decode_outputs(gpu.dec, out_gpu, base) == want, "decoded != plain_forward");
    // tampering: one flipped digit of the first output label
    auto bad = out_gpu;
    bad[0].at(0)[1] = static_cast<crt_val_t>((bad[0].at(0)[1] + 1) % bad[0].mod());
    bool auth = false;
    try {
        dash::gpu::decode_outputs(gpu.dec, bad, base);
    } catch (const AuthenticityError&) {
        auth = true;
    }
    EXPECT(auth, "tampered output not rejected");
    std::printf("ok %s: gc %zu bytes, cts %llu, decoded[0] = %lld\n", name.c_str(),
                serialize_garbled_circuit(gpu.gc).size(), (unsigned long long)gpu.stats.ciphertexts,
                (long long)want[0]);
}

int main() {
    try {
        check_model("model_tiny", testsupport::model_tiny(1000, 8), 0x5EED1, 4000);
        check_model("model_tiny_priv", testsupport::model_tiny(1000, 5, true), 0x5EED2, 4001);
        check_model("model_a", testsupport::model_a(1001, 8), 0x5EED0000, 4000);
        check_model("model_c", testsupport::model_c(1003, 9), 0x5EED0003, 4000);
        check_model("model_d", testsupport::model_d(1004, 8), 0x5EED0004, 4000);
        // batched: B seeds in one device garbling, each equal to its own CPU garbling
        {
            const std::string name = "model_tiny_batch";
            const Circuit c = testsupport::model_tiny(1000, 8);
            std::vector<Seed> seeds;
            for (uint32_t b = 0; b < 5; ++b) seeds.push_back(seed_of(0x5EED0100 + b));
            const auto nets = dash::gpu::garble_batch(c, seeds);
            for (uint32_t b = 0; b < seeds.size(); ++b)
                EXPECT(serialize_garbled_circuit(nets[b].gc) ==
                           serialize_garbled_circuit(dash::garble(c, seeds[b]).gc),
                       "batched gc bytes");
            std::printf("ok %s: %zu garblings\n", name.c_str(), nets.size());
        }
        // malformed GC -> DataError through the shim
        {
            const std::string name = "malformed_gc";
            GarbledNetwork n = dash::gpu::garble(testsupport::model_tiny(1000, 8), seed_of(7));
            n.gc.cts.resize(n.gc.cts.size() - 1);  // blob shorter than the layout
            bool data = false;
            try {
                dash::gpu::evaluate(n.gc, {});
            } catch (const DataError&) {
                data = true;
            }
            EXPECT(data, "short GC not rejected as DataError");
            std::printf("ok %s\n", name.c_str());
        }
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf(failures ? "shim check: %d failure(s)\n" : "shim check: all passed\n", failures);
    return failures ? 1 : 0;
}
