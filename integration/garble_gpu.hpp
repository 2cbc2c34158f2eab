// dash::gpu — the reference's whole-network garbling API served by the B200
// engine (libdashgpu, include/dashgpu.h).  Drop-in for the four hot-path
// calls of proj/core/include/dash/garble.hpp:93-112: same types, same
// exceptions (dash::DataError / AuthenticityError / OverflowError / Error,
// errors.hpp:9-34), byte-identical artifacts.  A maintainer adds this file
// pair to proj/core/src and links -ldashgpu; callers (protocol.cpp:211,252,
// 267,331, tools/dash.cpp:334-338) switch by namespace.
//
// Extra parameters beyond the reference signatures are trailing and
// defaulted: the CUDA device and stream (a cudaStream_t, nullptr = the
// legacy default stream) every call is enqueued on.
#pragma once

#include <span>
#include <vector>

#include "dash/garble.hpp"

namespace dash::gpu {

// dash::garble (garble.hpp:93-94) — `threads` is accepted for signature
// compatibility and ignored (the device runs every element in parallel).
GarbledNetwork garble(const Circuit& circuit, const Seed& seed, int threads = 0, int device = 0,
                      void* stream = nullptr);

// B independent garblings of one circuit in one device launch sequence.
std::vector<GarbledNetwork> garble_batch(const Circuit& circuit, std::span<const Seed> seeds, int device = 0,
                                         void* stream = nullptr);

// dash::garble_inputs (garble.hpp:97-99)
std::vector<LabelTensor> garble_inputs(const EncodingInfo& enc, std::span<const q_val_t> values,
                                       const CrtBase& base, int device = 0, void* stream = nullptr);

// dash::evaluate (garble.hpp:103-105): the GC is imported into HBM
// (dashgpu_import_gc), evaluated there and the output labels copied back.
std::vector<LabelTensor> evaluate(const GarbledCircuit& gc, const std::vector<LabelTensor>& inputs,
                                  int threads = 0, int device = 0, void* stream = nullptr);

// dash::decode_outputs (garble.hpp:110-112) is a table lookup on the host
// data the caller already holds; the reference implementation is kept.
using dash::decode_outputs;

}  // namespace dash::gpu
