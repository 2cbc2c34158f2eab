// Per-thread logic of the non-tape kernels: public-weight linear lanes,
// private-weight (projection) linear lanes, PRF setup, input encoding,
// decoding tables / decode and label export.
#pragma once

#include "dash_device.cuh"
#include "sha256.hpp"

namespace dashgpu {

// ---------------------------------------------------------------------------
// Public-weight linear lane (reference layer.cpp:122-191):
//   out[u][d] = (sum_{i: w!=0 mod p} (w mod p) x_i[d] + z_u zero[d] - [garbler] b_u R_p[d]) mod p
// One thread = four digits (one word w) of one output unit of one inference.
struct LinParams {
    int conv;
    uint32_t K;          // in_dim or in_ch*f*f
    uint32_t M;          // output units
    uint32_t E_in;
    uint32_t in_ch, H, W, f, stride, OH, OW;
    const uint8_t* wres; // dense: [K][M]; conv: [out_ch][K]   (w mod p)
    const uint8_t* zt;   // [M] (dense) / [out_ch] (conv): #zero-residue weights mod p
    const uint8_t* bres; // [M] / [out_ch]: bias residue (garbler only)
    const uint32_t* in;  // [B][nw][E_in]
    uint32_t* out;       // [B][nw][M]
    const uint32_t* zero;// zero-wire label of this lane (byte digits), inference b at zero[b*zstride]
    const uint32_t* R;   // offset R_p (byte digits), garbler only, same stride
    uint32_t zstride;
    uint32_t p, nw, B;
    uint32_t n, mag, sh;  // digits n_p and the x/p magic (tensor-core epilogue)
    int garbler;
};

DASH_HD void linear_thread(const LinParams& L, uint32_t b, uint32_t w, uint32_t u) {
    const ModC& M = c_mod[L.p];
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    const uint32_t* xin = L.in + ((uint64_t)b * L.nw + w) * L.E_in;
    uint32_t oc = 0;
    if (!L.conv) {
        for (uint32_t i = 0; i < L.K; ++i) {
            const uint32_t wv = L.wres[(uint64_t)i * L.M + u];
            const uint32_t x = xin[i];
            acc0 += wv * (x & 0xffu);
            acc1 += wv * ((x >> 8) & 0xffu);
            acc2 += wv * ((x >> 16) & 0xffu);
            acc3 += wv * (x >> 24);
        }
    } else {
        oc = u / (L.OH * L.OW);
        const uint32_t oy = (u / L.OW) % L.OH, ox = u % L.OW;
        const uint8_t* wr = L.wres + (uint64_t)oc * L.K;
        uint32_t i = 0;
        for (uint32_t ic = 0; ic < L.in_ch; ++ic)
            for (uint32_t ky = 0; ky < L.f; ++ky) {
                const uint32_t* row = xin + ((uint64_t)ic * L.H + (oy * L.stride + ky)) * L.W + ox * L.stride;
                for (uint32_t kx = 0; kx < L.f; ++kx, ++i) {
                    const uint32_t wv = wr[i];
                    const uint32_t x = row[kx];
                    acc0 += wv * (x & 0xffu);
                    acc1 += wv * ((x >> 8) & 0xffu);
                    acc2 += wv * ((x >> 16) & 0xffu);
                    acc3 += wv * (x >> 24);
                }
            }
    }
    const uint32_t idx = L.conv ? oc : u;
    const uint32_t z = L.zt[idx];
    const uint32_t nb = L.garbler ? (L.bres[idx] ? L.p - L.bres[idx] : 0u) : 0u;
    const uint32_t zw = L.zero[(uint64_t)b * L.zstride + w];
    const uint32_t rw = L.garbler ? L.R[(uint64_t)b * L.zstride + w] : 0u;
    uint32_t accs[4] = {acc0, acc1, acc2, acc3};
    const uint32_t c31 = 0x7fffffffu - fdiv(0x7fffffffu, M.mag_m, M.sh_m) * L.p + 1u;  // == 2^31 mod p (up to one p)
    uint32_t o = 0;
    for (int j = 0; j < 4; ++j) {
        // u32 wrap-around as the reference's accumulator (layer.cpp:116-118);
        // the 31-bit-exact magic sees the low 31 bits plus 2^31 mod p
        const uint32_t lo = accs[j] & 0x7fffffffu;
        const uint32_t s = lo - fdiv(lo, M.mag_m, M.sh_m) * L.p + (accs[j] >> 31) * c31;
        const uint32_t t = s + z * ((zw >> (8 * j)) & 0xffu) + nb * ((rw >> (8 * j)) & 0xffu);
        const uint32_t d = t - fdiv(t, M.mag_m, M.sh_m) * L.p;
        o |= d << (8 * j);
    }
    // digits beyond n in the top word stay zero (inputs are zero there)
    if (4 * w + 4 > M.n) o &= 0xffffffffu >> (8 * (4 * w + 4 - M.n));
    L.out[((uint64_t)b * L.nw + w) * L.M + u] = o;
}

// ---------------------------------------------------------------------------
// Private-weight linear lane (layer.cpp:195-212, 456-507): per weight one
// projection x -> w*x mod p, free add, then add_public_constant(bias).
struct PrivParams {
    int conv;
    uint32_t win;            // window
    uint32_t M;              // units
    uint32_t E_in;
    uint32_t in_ch, H, W, f, stride, OH, OW;
    const uint8_t* wres;     // [M][win] (dense) / [out_ch][win] (conv)
    const uint8_t* bres;     // [M] / [out_ch]
    const uint32_t* in;      // [B][nw][E_in]
    uint32_t* out;           // [B][nw][M]
    uint32_t p, B;
    uint64_t gate_base, wire_base;   // layer base + lane offset
    U4* blob;                // layer blob of inference 0, already offset by the lane's ct offset
    uint64_t blob_stride;
    const uint32_t* rk;      // [B][44]
    const uint32_t* mult;    // [B][...]
    uint64_t mult_stride;
    int garbler;
};

DASH_HD void private_thread(const PrivParams& P, uint32_t b, uint32_t u, const AesTab& t) {
    const ModC& M = c_mod[P.p];
    const uint32_t p = P.p;
    Elt e;
    e.b = b;
    e.u = u;
    e.rk = P.rk + (uint64_t)b * 44;
    e.mult = P.mult + (uint64_t)b * P.mult_stride;
    e.t = t;
    U4* rows = P.blob + (uint64_t)b * P.blob_stride + (uint64_t)u * P.win * p;
    uint32_t oc = 0, oy = 0, ox = 0;
    if (P.conv) {
        oc = u / (P.OH * P.OW);
        oy = (u / P.OW) % P.OH;
        ox = u % P.OW;
    }
    const uint8_t* wr = P.wres + (uint64_t)(P.conv ? oc : u) * P.win;
    const uint32_t* Rp = P.garbler ? mult_row(e, p, 1) : nullptr;
    uint32_t buf[3][NWMAX];
    const LB X{buf[0], 1}, term{buf[1], 1}, sum{buf[2], 1};
    for (uint32_t j = 0; j < P.win; ++j) {
        uint64_t xi;
        if (!P.conv) {
            xi = j;
        } else {
            const uint32_t ic = j / (P.f * P.f), ky = (j / P.f) % P.f, kx = j % P.f;
            xi = ((uint64_t)ic * P.H + (oy * P.stride + ky)) * P.W + (ox * P.stride + kx);
        }
        lb_load_rows(X, P.in + ((uint64_t)b * M.nw) * P.E_in + xi, P.E_in, M);
        const uint64_t g = P.gate_base + (uint64_t)u * P.win + j;
        U4* R = rows + (uint64_t)j * p;
        const uint32_t c = lb_color(X, M);
        if (P.garbler) {
            lb_prf(term, P.wire_base + (uint64_t)u * P.win + j, 0, M, e.rk, t);
            const uint32_t w = wr[j];
            for (uint32_t a = 0; a < p; ++a) {
                uint32_t row = c + a;
                row = row >= p ? row - p : row;
                const U4 H = hash_tw(lb_key_step(X, Rp, M), g, row, 0, t);
                R[row] = lb_enc(H, term, mult_row(e, p, (w * a) % p), nullptr, 0, M);
            }
        } else {
            lb_dec(term, R[c], hash_tw(lb_compress(X, M), g, c, 0, t), M);
        }
        if (j == 0) lb_copy(sum, term, M);
        else lb_add(sum, term, M);
    }
    if (P.garbler) {
        const uint32_t bb = P.bres[P.conv ? oc : u];
        if (bb) lb_sub_g(sum, mult_row(e, p, bb), M);
    }
    lb_store_rows(sum, P.out + ((uint64_t)b * M.nw) * P.M + u, P.M, M);
}

// ---------------------------------------------------------------------------
// Garbling setup: offsets R_m and their multiples v*R_m (prf.hpp:28-32,
// gadgets.hpp:20-34), zero-wire / input base labels (garble.cpp:155-173) and
// the seed commitment (garble.cpp:199-204).
struct SetupParams {
    uint32_t B;
    int k;
    uint16_t primes[MAXK];
    uint32_t nslot;
    uint16_t slot_mod[MAXMOD + 1];
    const uint32_t* rk;        // [B][44]
    const uint8_t* seeds;      // [B][16]
    uint32_t* mult;            // [B][nslot][128][NWMAX]
    uint64_t mult_stride;
    uint32_t n_in;
    uint64_t e0;               // first input element of this launch (streamed layers)
    uint32_t* base_planes[MAXK]; // [B][nw][n_in] input base labels (encoding info)
    uint32_t* zero;            // [B][k][LABW] byte-digit words
    uint32_t* Rb;              // [B][k][LABW] offsets of the primes, byte-digit words
    U4* commit;                // [B]
};

// One thread per (modulus slot, multiple x): R_m is drawn by every thread of
// the slot (a few AES blocks), so the m multiples are written in parallel.
DASH_HD void setup_offsets_thread(const SetupParams& S, uint32_t b, uint32_t si, uint32_t x, const AesTab& t) {
    const uint32_t m = S.slot_mod[si];
    if (x >= m) return;
    const ModC& M = c_mod[m];
    uint32_t buf[2][NWMAX] = {};
    const LB R{buf[0], 1}, v{buf[1], 1};
    lb_prf(R, m, 1, M, S.rk + (uint64_t)b * 44, t);
    // digit 0 forced to 1 (prf.hpp:28-32)
    if (M.pow2) R[0] = (R[0] & ~(M.m - 1u)) | 1u;
    else R[0] = (R[0] & ~0xffu) | 1u;
    uint32_t* base = S.mult + (uint64_t)b * S.mult_stride + (uint64_t)c_modslot[m] * 128 * NWMAX;
    lb_scale(v, R, x, M);
    for (int w = 0; w < NWMAX; ++w) base[(uint64_t)x * NWMAX + w] = v[w];
    if (x == 1)
        for (int i = 0; i < S.k; ++i)
            if (S.primes[i] == m) lb_store_rows(R, S.Rb + ((uint64_t)b * S.k + i) * LABW, 1, M);
}

DASH_HD void setup_labels_thread(const SetupParams& S, uint32_t b, uint32_t e, int i, const AesTab& t) {
    // e < n_in: input base of element e, lane i (wire k + e*k + i); e == n_in: zero wire i
    const uint32_t p = S.primes[i];
    const ModC& M = c_mod[p];
    uint32_t buf[NWMAX];
    const LB L{buf, 1};
    const uint32_t* rk = S.rk + (uint64_t)b * 44;
    if (e < S.n_in) {
        lb_prf(L, (uint64_t)S.k + (S.e0 + e) * S.k + (uint64_t)i, 0, M, rk, t);
        lb_store_rows(L, S.base_planes[i] + ((uint64_t)b * M.nw) * S.n_in + e, S.n_in, M);
    } else {
        lb_prf(L, (uint64_t)i, 0, M, rk, t);
        lb_store_rows(L, S.zero + ((uint64_t)b * S.k + i) * LABW, 1, M);
    }
    if (e == S.n_in && i == 0) {
        // seed commitment = davies_meyer(seed bytes read little-endian)
        const uint8_t* sd = S.seeds + (uint64_t)b * 16;
        U4 v;
        for (int j = 0; j < 4; ++j)
            v.x[j] = (uint32_t)sd[4 * j] | ((uint32_t)sd[4 * j + 1] << 8) | ((uint32_t)sd[4 * j + 2] << 16) |
                     ((uint32_t)sd[4 * j + 3] << 24);
        U4 h = aes_pi(v, t);
        for (int j = 0; j < 4; ++j) h.x[j] ^= v.x[j];
        S.commit[b] = h;
    }
}

// AES-128 key schedule of a 16-byte seed (aes.cpp:32-46) on the device, so a
// batch whose seeds are already in HBM needs no host round trip.  S-box =
// byte 1 of T0 (T0[x] = (2S, S, S, 3S) little-endian).
DASH_HD void expand_thread(const uint8_t* key, uint32_t* rk, const uint32_t* T0) {
    const uint8_t rcon[10] = {1, 2, 4, 8, 16, 32, 64, 128, 0x1b, 0x36};
    for (int i = 0; i < 4; ++i)
        rk[i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) | ((uint32_t)key[4 * i + 2] << 16) |
                ((uint32_t)key[4 * i + 3] << 24);
    for (int i = 4; i < 44; ++i) {
        uint32_t t = rk[i - 1];
        if (i % 4 == 0) {
            auto sb = [&](uint32_t x) { return (T0[x & 0xffu] >> 8) & 0xffu; };
            // RotWord + SubWord + Rcon on the little-endian word
            t = (sb(t >> 8) ^ rcon[i / 4 - 1]) | (sb(t >> 16) << 8) | (sb(t >> 24) << 16) | (sb(t) << 24);
        }
        rk[i] = rk[i - 4] ^ t;
    }
}

// ---------------------------------------------------------------------------
// garble_inputs (garble.cpp:242-263): label = base + (enc(v) mod p) R_p
struct EncodeParams {
    uint32_t B, n_in;
    int k;
    uint16_t primes[MAXK];
    const int64_t* values;     // [B][n_in]
    const uint32_t* base[MAXK];// [B][nw][n_in]
    uint32_t* out[MAXK];       // [B][nw][n_in]
    const uint32_t* mult;
    uint64_t mult_stride;
    uint64_t half_up_lo, half_up_hi;  // ceil(P/2) as u128
    uint64_t half_dn_lo, half_dn_hi;  // floor(P/2)
    int* err;
};

DASH_HD void encode_thread(const EncodeParams& P, uint32_t b, uint32_t e, int i) {
    const uint32_t p = P.primes[i];
    const ModC& M = c_mod[p];
    const int64_t v = P.values[(uint64_t)b * P.n_in + e];
    const u128 half_up = ((u128)P.half_up_hi << 64) | P.half_up_lo;
    const u128 half_dn = ((u128)P.half_dn_hi << 64) | P.half_dn_lo;
    uint32_t r;
    if (v >= 0) {
        if ((u128)(uint64_t)v >= half_up) {
            *P.err = ST_DATA;
            return;
        }
        r = (uint32_t)((uint64_t)v % p);
    } else {
        const uint64_t mag = (uint64_t)(-(v + 1)) + 1;
        if ((u128)mag > half_dn) {
            *P.err = ST_DATA;
            return;
        }
        const uint32_t mr = (uint32_t)(mag % p);
        r = mr ? p - mr : 0;
    }
    uint32_t buf[NWMAX];
    const LB L{buf, 1};
    lb_load_rows(L, P.base[i] + ((uint64_t)b * M.nw) * P.n_in + e, P.n_in, M);
    Elt ex;
    ex.mult = P.mult + (uint64_t)b * P.mult_stride;
    lb_add_g(L, mult_row(ex, p, r), M);
    lb_store_rows(L, P.out[i] + ((uint64_t)b * M.nw) * P.n_in + e, P.n_in, M);
}

// ---------------------------------------------------------------------------
// Decoding tables (garble.cpp:208-231) and decode_outputs (314-343)
struct DecodeParams {
    uint32_t B, n_out;
    int k;
    uint16_t primes[MAXK];
    uint16_t poff[MAXK + 1];   // prefix sums of the primes
    const uint32_t* lanes[MAXK];  // [B][nw][n_out] base (tables) or active (decode) labels
    U4* table;                 // [B][n_out][sum_p]
    const uint32_t* mult;
    uint64_t mult_stride;
    uint8_t* residues;         // [B][n_out][k]
    int* err;
    // crt_reconstruct + decode_signed on the device (crt.cpp:63-101):
    // values[b][e] = signed(sum_i coeff_i r_i mod P); coeff_i = (P/p_i) * inv
    int64_t* values;           // [B][n_out] (nullptr: residues only)
    uint64_t coeff_lo[MAXK], coeff_hi[MAXK];  // coeff_i mod P
    uint64_t P_lo, P_hi;
}; 

DASH_HD void dectable_thread(const DecodeParams& P, uint32_t b, uint32_t e, int i) {
    const uint32_t p = P.primes[i];
    const ModC& M = c_mod[p];
    uint32_t buf[2][NWMAX];
    const LB base{buf[0], 1}, c{buf[1], 1};
    lb_load_rows(base, P.lanes[i] + ((uint64_t)b * M.nw) * P.n_out + e, P.n_out, M);
    Elt ex;
    ex.mult = P.mult + (uint64_t)b * P.mult_stride;
    U4* row = P.table + ((uint64_t)b * P.n_out + e) * P.poff[P.k] + P.poff[i];
    for (uint32_t v = 0; v < p; ++v) {
        lb_copy(c, base, M);
        lb_add_g(c, mult_row(ex, p, v), M);
        row[v] = lb_compress(c, M);
    }
}

// error flag, the most severe code wins (AuthenticityError over DataError)
DASH_HD void flag_err(int* err, int code) {
#if defined(__CUDA_ARCH__)
    atomicMax(err, code);
#else
    if (*err < code) *err = code;
#endif
}

DASH_HD void decode_thread(const DecodeParams& P, uint32_t b, uint32_t e) {
    uint8_t res[MAXK];
    uint32_t buf[NWMAX];
    const LB L{buf, 1};
    for (int i = 0; i < P.k; ++i) {
        const uint32_t p = P.primes[i];
        const ModC& M = c_mod[p];
        lb_load_rows(L, P.lanes[i] + ((uint64_t)b * M.nw) * P.n_out + e, P.n_out, M);
        const U4 c = lb_compress(L, M);
        const U4* row = P.table + ((uint64_t)b * P.n_out + e) * P.poff[P.k] + P.poff[i];
        int found = -1;
        for (uint32_t v = 0; v < p; ++v) {
            const U4 t = row[v];
            if (found < 0 && t.x[0] == c.x[0] && t.x[1] == c.x[1] && t.x[2] == c.x[2] && t.x[3] == c.x[3])
                found = (int)v;
        }
        if (found < 0) {
            flag_err(P.err, ST_AUTH);
            found = 0;
        }
        P.residues[((uint64_t)b * P.n_out + e) * P.k + i] = (uint8_t)found;
        res[i] = (uint8_t)found;
    }
    if (!P.values) return;
    const u128 Pm = ((u128)P.P_hi << 64) | P.P_lo;
    u128 acc = 0;
    for (int i = 0; i < P.k; ++i) {
        const u128 c = ((u128)P.coeff_hi[i] << 64) | P.coeff_lo[i];  // < P
        acc += c * res[i] % Pm;  // c * r < 2^128 for the CRT bases (P < 2^66, r < 64)
        if (acc >= Pm) acc -= Pm;
    }
    const u128 half_up = (Pm + 1) / 2;
    int64_t v;
    if (acc < half_up) {
        if (acc > (u128)INT64_MAX) {
            flag_err(P.err, ST_DATA);
            return;
        }
        v = (int64_t)acc;
    } else {
        const u128 mag = Pm - acc;
        if (mag > (u128)INT64_MAX) {
            flag_err(P.err, ST_DATA);
            return;
        }
        v = -(int64_t)mag;
    }
    P.values[(uint64_t)b * P.n_out + e] = v;
}

// ---------------------------------------------------------------------------
// Extension layers (include/dash_circuit_desc.h): Pad2d writes the zero-wire
// label (garble.cpp:157) into the pad cells of a [C][H][W] plane; Add is the
// lane-wise label sum (free, like free_add, gadgets.hpp:108-118).  Garbler
// and evaluator run the same code (the zero wire's active label is its base
// label).  One thread = one digit word of one element of one inference.
struct PadAddParams {
    int add;                   // 0: Pad2d, 1: Add
    uint32_t B, E_out;
    uint32_t C, H, W, pad, OH, OW;
    int k;
    uint16_t primes[MAXK];
    uint32_t wbase[MAXK + 1];  // prefix sums of nw over the lanes
    const uint32_t* in[MAXK];  // [B][nw][E_in]
    const uint32_t* in2[MAXK]; // Add: second operand [B][nw][E_out]
    uint32_t* out[MAXK];       // [B][nw][E_out]
    const uint32_t* zero;      // [B][k][LABW]
};

DASH_HD void pad_add_thread(const PadAddParams& P, uint32_t b, uint32_t wi, uint32_t u) {
    int i = 0;
    while (i + 1 < P.k && wi >= P.wbase[i + 1]) ++i;
    const uint32_t nw = P.wbase[i + 1] - P.wbase[i], w = wi - P.wbase[i];
    uint32_t* o = P.out[i] + ((uint64_t)b * nw + w) * P.E_out + u;
    if (P.add) {
        const uint64_t at = ((uint64_t)b * nw + w) * P.E_out + u;
        *o = swar_add(P.in[i][at], P.in2[i][at], c_mod[P.primes[i]]);
        return;
    }
    const uint32_t ch = u / (P.OH * P.OW), y = (u / P.OW) % P.OH, x = u % P.OW;
    const bool inside = y >= P.pad && y < P.pad + P.H && x >= P.pad && x < P.pad + P.W;
    *o = inside ? P.in[i][((uint64_t)b * nw + w) * ((uint64_t)P.C * P.H * P.W) +
                          ((uint64_t)ch * P.H + (y - P.pad)) * P.W + (x - P.pad)]
                : P.zero[((uint64_t)b * P.k + i) * LABW + w];
}

// ---------------------------------------------------------------------------
// t_proj primitive (gadgets.hpp:146-176) over n independent gates, one thread
// per gate: garbler rows [n][p] + fresh out0, or evaluator output labels.
struct ProjParams {
    uint32_t n, p, q;
    const uint8_t* phi;      // [p] values mod q
    const U4* in;            // [n] compressed labels mod p (garbler: base, evaluator: active)
    const uint64_t* gates;   // [n] gate ids (tweak g)
    const uint64_t* wires;   // [n] fresh output wire ids (garbler)
    U4* rows;                // [n][p]
    U4* out;                 // [n] compressed labels mod q (garbler: out0, evaluator: active)
    const uint32_t* rk;      // [44] PRF key schedule
    const uint32_t* mult;    // multiples table of the PRF's offsets
    int garbler;
};

// X, A: label buffers (shared memory on the device: garble_rows_n assumes it)
DASH_HD void proj_thread(const ProjParams& P, uint32_t i, const AesTab& t, LB X, LB A) {
    const ModC& Mp = c_mod[P.p];
    const ModC& Mq = c_mod[P.q];
    lb_decompress(X, P.in[i], Mp);
    const uint32_t c = lb_color(X, Mp);
    U4* R = P.rows + (uint64_t)i * P.p;
    if (P.garbler) {
        lb_prf(A, P.wires[i], 0, Mq, P.rk, t);
        garble_rows_n(X, A, t, P.mult, P.p, P.q, c, P.gates[i], P.phi, 0, R, 0, 1);
    } else {
        lb_dec(A, R[c], hash_tw(lb_compress(X, Mp), P.gates[i], c, 0, t), Mq);
    }
    P.out[i] = lb_compress(A, Mq);
}

// compress every label of a lane plane: out[b][e] (bundle payload / tensor_write)
struct CompressParams {
    uint32_t B, n;
    uint32_t p;
    const uint32_t* lane;  // [B][nw][n]
    U4* out;               // [B][n] strided: out[b*ostride + e]
    uint64_t ostride;
};

DASH_HD void compress_thread(const CompressParams& P, uint32_t b, uint32_t e) {
    const ModC& M = c_mod[P.p];
    uint32_t buf[NWMAX];
    const LB L{buf, 1};
    lb_load_rows(L, P.lane + ((uint64_t)b * M.nw) * P.n + e, P.n, M);
    P.out[(uint64_t)b * P.ostride + e] = lb_compress(L, M);
}

// parse side of the bundle format: decompress_mod every chunk into a lane plane
DASH_HD void decompress_thread(const CompressParams& P, uint32_t b, uint32_t e, uint32_t* lane_out) {
    const ModC& M = c_mod[P.p];
    uint32_t buf[NWMAX];
    const LB L{buf, 1};
    lb_decompress(L, P.out[(uint64_t)b * P.ostride + e], M);
    lb_store_rows(L, lane_out + ((uint64_t)b * M.nw) * P.n + e, P.n, M);
}

// Activation-layer rows between the device layout (act_rows: blocks of 32
// elements, row-major inside a block) and the reference's element-major
// GarbledCircuit::cts order (layer.cpp:537-541), for GC export / import.
// Thread r handles reference row r = e * uc + j of the layer.
struct RowsPermuteParams {
    const U4* src;
    U4* dst;
    uint64_t E, uc;
    int to_ref;  // 1: device -> reference order, 0: reference -> device
};

DASH_HD void rows_permute_thread(const RowsPermuteParams& P, uint64_t r) {
    const uint64_t e = r / P.uc, j = r - e * P.uc;
    const uint64_t blk = e >> 5, left = P.E - (blk << 5), w = left < 32 ? left : 32;
    const uint64_t d = blk * 32 * P.uc + j * w + (e & 31);
    if (P.to_ref) P.dst[r] = P.src[d];
    else P.dst[d] = P.src[r];
}

// Streamed-garbling digest mode (sha256.hpp): one 64 KiB leaf of one
// inference's layer rows, read in reference order straight from the garbling
// window (activation rows through the rows_permute mapping above).
struct DigestParams {
    const U4* src;    // window: inference b's rows at src + b * stride
    uint64_t stride;  // rows per inference in the window
    uint64_t rows;    // ciphertext rows of the layer per inference
    uint64_t E, uc;   // activation layer (device row order); uc == 0: reference order
    uint32_t B, leaves;
    uint32_t* out;    // [B][leaves][8] SHA-256 state words
};

DASH_HD void digest_leaf_thread(const DigestParams& P, uint32_t b, uint32_t leaf) {
    const U4* src = P.src + (uint64_t)b * P.stride;
    const uint64_t r0 = (uint64_t)leaf * kDigestLeafRows;
    const uint64_t n = P.rows - r0 < kDigestLeafRows ? P.rows - r0 : kDigestLeafRows;
    auto row = [&](uint64_t i, uint32_t* w) {
        uint64_t r = r0 + i;
        if (P.uc) {
            const uint64_t e = r / P.uc, j = r - e * P.uc;
            const uint64_t blk = e >> 5, left = P.E - (blk << 5), wd = left < 32 ? left : 32;
            r = blk * 32 * P.uc + j * wd + (e & 31);
        }
        const U4 v = src[r];
        for (int t = 0; t < 4; ++t) w[t] = v.x[t];
    };
    sha256_rows(n, row, P.out + ((uint64_t)b * P.leaves + leaf) * 8);
}

// The root of one inference's layer: SHA-256 over its leaf digests as bytes
// (state words big-endian), read as 16-byte rows: row i = half (i & 1) of
// leaf i >> 1.  out: [B][8] state words.
DASH_HD void digest_root_thread(const DigestParams& P, uint32_t b, uint32_t* out) {
    const uint32_t* lv = P.out + (uint64_t)b * P.leaves * 8;
    auto row = [&](uint64_t i, uint32_t* w) {
        const uint32_t* d = lv + (i >> 1) * 8 + (i & 1) * 4;
        for (int t = 0; t < 4; ++t) w[t] = sha_bswap(d[t]);
    };
    sha256_rows((uint64_t)P.leaves * 2, row, out + (uint64_t)b * 8);
}

}  // namespace dashgpu
