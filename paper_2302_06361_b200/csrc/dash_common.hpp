// Shared host/device definitions for the B200 Dash engine.
//
// Everything that runs per element on the GPU is written as DASH_HD
// (__host__ __device__ under nvcc) so that the same code can be compiled by
// g++ into the TEST-ONLY emulation library tests/emu/libdashemu.so (used to
// debug kernel logic on a machine without a GPU).  The product library
// libdashgpu.so is always built by nvcc for sm_100a.
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DASH_HD __host__ __device__ __forceinline__
#define DASH_CONST __constant__
#else
#define DASH_HD inline
#define DASH_CONST
#endif

namespace dashgpu {

typedef unsigned __int128 u128;

// Largest digit count of a non-power-of-two modulus (m = 3: 80 digits) in
// u32 words of four u8 digits.  Power-of-two moduli use a packed-bit form
// (4 words) that is identical to their compressed value.
constexpr int NWMAX = 20;
// Words of one label row in global memory (128 u8 digits, modulus 2).
constexpr int LABW = 32;
constexpr int MAXMOD = 128;  // kMaxModulus (reference label.hpp:15)
constexpr int MAXK = 16;     // kMaxCrtPrimes (reference crt.hpp:11)
constexpr int MAXSLOTS = 48; // activation tape slots per element

// Per-modulus constants, built on the host (engine.cpp: make_modc) and kept
// in __constant__ memory; every access is warp-uniform.
struct ModC {
    uint16_t m;
    uint8_t n;        // digits n_m (reference label.cpp:15-29)
    uint8_t nw;       // words of four digits
    uint8_t pow2;     // power of two: packed-bit representation
    uint8_t e;        // log2 m (pow2)
    uint8_t full;     // pow2 with e*n == 128 (no reduction, label.cpp:43)
    uint8_t W;        // words per decomposition chunk (non-pow2)
    uint8_t nchunks;  // ceil(nw / W)
    uint8_t limbs[21];// significant 32-bit limbs of the value before chunk j
    uint32_t m4;      // m^4
    uint32_t D;       // m^(4W) < 2^30: chunk divisor
    uint32_t negD;    // (uint32_t)-D
    uint32_t mag_m, sh_m;    // x/m  = umulhi(x, mag_m)  >> sh_m  (x < 2^31)
    uint32_t mag_m4, sh_m4;  // x/m^4 = umulhi(x, mag_m4) >> sh_m4 (x < 2^31)
    uint32_t spread;  // m * 0x01010101 (SWAR)
    uint32_t addc;    // (128 - m) * 0x01010101 (SWAR compare)
    uint64_t invD;    // floor((2^64 - 1) / D)
    uint64_t mag64;   // ceil(2^64 / m): exact x mod m for 32-bit PRF words
    uint32_t bits[4]; // pow2: low e*n bits
    uint32_t hi[4];   // pow2: top bit of every field
    uint32_t lo[4];   // pow2: bottom bit of every field
    // word values by byte dot products (dash_device.cuh wval):
    // d0 + m d1 = dp4a(x, wlo), d2 + m d3 = dp4a(x, whi)
    uint32_t wlo, whi, m2;
    uint32_t negm, negm4;  // (uint32_t)-m, -m^4: x - q m as one multiply-add
    // Horner compress (dash_device.cuh horner): hp words per step (2 when
    // m^8 < 2^32), step multiplier m8 = m^(4 hp), htop words in the top step,
    // hlim[L-1] steps whose partial value fits L 32-bit limbs
    uint32_t m8;
    uint8_t hp, htop, hlim[4];
    // chunk recombination (lb_enc / lb_dec_c): limbs of D^(j+1) per chunk j
    uint8_t climbs[21];
};

// Activation-tape operations (one per gadget call of the reference's
// t_approx_sign_bit / relu_element / sign_act_element, gadgets.hpp:146-481,
// layer.cpp:214-236).
enum OpKind : uint8_t {
    OP_PROJ = 1,     // t_proj: p rows
    OP_GRR = 2,      // t_proj_grr: p-1 rows
    OP_HALF = 3,     // t_half_gate: 2p rows
    OP_MMHALF = 4,   // t_mm_half_gate: p+q+1 rows
    OP_ADD = 5,      // free_add (binary step)
    OP_ADDCONST = 6, // add_public_constant
    OP_OUTPUT = 7,   // element result for lane `cst`
    OP_ADDACC = 8,   // running sum of a fused free-add chain: A += b (OP_ADD / OP_ADDACC with
                     // cst & kKeep leave the sum in A instead of storing it)
};

constexpr uint16_t kKeep = 0x8000;  // fused add chain: result stays in the A buffer

// Operand encoding: < 240 -> slot index; >= 240 -> input lane (v - 240).
constexpr uint8_t IN_LANE = 240;

struct TapeOp {
    uint8_t kind;
    uint8_t a, b, out;    // operands / output slot
    uint16_t pm, qm;      // modulus of a (p) and of the output / b (q)
    uint16_t cst;         // ADDCONST constant, OUTPUT lane
    uint32_t gate_off;    // relative to the element's first gate
    uint32_t wire_off;    // relative to the element's first fresh wire
    uint32_t ct_off;      // relative to the element's first ciphertext
    uint32_t phi_off;     // offset into the phi pool (p entries)
};

// Status codes of the C ABI (mirror dash:: exceptions, errors.hpp:9-34).
enum Status : int {
    ST_OK = 0,
    ST_ERR = 1,
    ST_CUDA = 2,
    ST_DATA = 3,
    ST_AUTH = 4,
    ST_OVERFLOW = 5,
};

}  // namespace dashgpu
