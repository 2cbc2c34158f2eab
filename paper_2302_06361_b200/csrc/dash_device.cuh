// Per-thread device logic of the B200 Dash engine: label codec, fixed-key
// AES (T-table in shared memory), label PRF, garbled-row encryption and the
// activation-tape interpreter.  One thread = one (inference, element).
//
// Reference behaviour followed (paths under /root/reference/proj/core/):
//   label codec      src/label.cpp:101-232  (compress / decompose / decompress_mod)
//   AES-128          src/aes.cpp:32-90      (FIPS-197; u128 LE bytes are the block)
//   PRF              src/prf.cpp:11-27, include/dash/prf.hpp:24-32
//   hash / cipher    src/cipher.cpp:8-69, include/dash/cipher.hpp:13-26,62-66
//   gadgets          include/dash/gadgets.hpp:127-358
//
// Design: labels of non-power-of-two moduli live in per-lane
// shared-memory buffers as packed u8 digits (four per u32 word); power-of-two
// moduli use the packed bit form, which *is* their compressed value.  Compression works word by
// word (Horner in base m^4); decompression divides the 128-bit value by
// D = m^(4W) <= 2^31 with a precomputed 64-bit reciprocal, then splits each
// chunk into digits with 32-bit magic multiplies.  Every modulus-dependent
// branch is warp-uniform (all lanes run the same tape), only data differs.
#pragma once

#include "dash_common.hpp"

namespace dashgpu {

// loop unrolling knobs (tuning builds: -DDASH_AES_UNROLL=n / -DDASH_CODEC_UNROLL=n)
#ifndef DASH_AES_UNROLL
#define DASH_AES_UNROLL 1
#endif
#ifndef DASH_CODEC_UNROLL
#define DASH_CODEC_UNROLL 1
#endif
constexpr int kAesUnroll = DASH_AES_UNROLL;
constexpr int kCodecUnroll = DASH_CODEC_UNROLL;

// ---------------------------------------------------------------- intrinsics
#if defined(__CUDA_ARCH__)
DASH_HD uint32_t umulhi32(uint32_t a, uint32_t b) { return __umulhi(a, b); }
DASH_HD uint64_t umulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }
DASH_HD uint32_t rotl32(uint32_t x, int s) { return __funnelshift_l(x, x, s); }
#else
DASH_HD uint32_t umulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * b) >> 32); }
DASH_HD uint64_t umulhi64(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }
DASH_HD uint32_t rotl32(uint32_t x, int s) { return (x << s) | (x >> ((32 - s) & 31)); }
#endif

// Constant tables (filled by the host: engine.cpp upload_constants()).  The
// translation unit that owns them (kernels*.cu, or the emulation library)
// defines DASH_CONST_DEFINED before including this header.
#if !defined(DASH_CONST_DEFINED)
extern DASH_CONST ModC c_mod[MAXMOD + 1];
extern DASH_CONST uint32_t c_pi_rk[44];           // all-zero-key AES schedule
extern DASH_CONST uint16_t c_modslot[MAXMOD + 1];  // modulus -> mult-table slot
#endif


struct alignas(16) U4 {  // 16-byte aligned: one 128-bit load / store per garbled row
    uint32_t x[4];
};

// --------------------------------------------------------------- AES-128
// T0[x] = (2S, S, S, 3S) as little-endian bytes; T1..T3 are byte rotations.
// The table is replicated 32x in shared memory (entry x of lane l at
// T[x*32 + l]) so the 32 lanes of a warp never bank-conflict.
// T-tables in shared memory, 256-byte rows: row x holds 32 lane replicas of
// T0[x] (bytes 0..127) and of T2[x] = rot16(T0[x]) (bytes 128..255), so
//  * one PRMT turns state byte r into the row offset (byte << 8) | lane*4
//    (| 128 for T2) -- no shift/mask pair per lookup;
//  * T0[a] ^ T1[b] ^ T2[c] ^ T3[d] = T0[a] ^ T2[c] ^ rot8(T0[b] ^ T2[d]),
//    one rotation per column instead of three;
//  * the 32 replicas keep every warp-wide lookup bank-conflict free.
// The table is the first 64 KB of dynamic shared memory of every kernel
// that hashes (link-time-constant base: LDS [R + 0]).
constexpr int kTabWords = 256 * 64;
#if defined(__CUDACC__)
extern __shared__ uint32_t s_dyn[];
#endif

struct AesTab {
    const uint32_t* T;  // host emulation only
    uint32_t l4;        // 4 * lane
};

DASH_HD AesTab make_tab(const uint32_t* T, uint32_t lane) {
    AesTab t;
    t.T = T;
    t.l4 = 4u * lane;
    return t;
}

DASH_HD uint32_t bperm(uint32_t x, uint32_t y, uint32_t sel) {
#if defined(__CUDA_ARCH__)
    return __byte_perm(x, y, sel);
#else
    const uint64_t v = ((uint64_t)y << 32) | x;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)((v >> (8 * ((sel >> (4 * i)) & 7))) & 0xff) << (8 * i);
    return r;
#endif
}

DASH_HD uint32_t tlo(const AesTab& t, uint32_t off) {
#if defined(__CUDA_ARCH__)
    (void)t;
    return *reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(s_dyn) + off);
#else
    return t.T[off >> 2];
#endif
}

template <class RK>
DASH_HD U4 aes_core(U4 s, const RK& rk, const AesTab& t) {
    const uint32_t L0 = t.l4, L2 = t.l4 | 0x80u;
#define P0(v, r) bperm((v), L0, 0x5504u | ((r) << 4))
#define P2(v, r) bperm((v), L2, 0x5504u | ((r) << 4))
#define COL(a, b, c, d, k) \
    (tlo(t, P0(a, 0)) ^ tlo(t, P2(c, 2)) ^ rotl32(tlo(t, P0(b, 1)) ^ tlo(t, P2(d, 3)), 8) ^ (k))
    const U4 k0 = rk.round(0);
    uint32_t s0 = s.x[0] ^ k0.x[0], s1 = s.x[1] ^ k0.x[1], s2 = s.x[2] ^ k0.x[2], s3 = s.x[3] ^ k0.x[3];
#if defined(__CUDA_ARCH__)
#pragma unroll kAesUnroll
#endif
    for (int r = 1; r < 10; ++r) {
        const U4 k = rk.round(r);  // one 128-bit load per round for keyed AES
        const uint32_t t0 = COL(s0, s1, s2, s3, k.x[0]);
        const uint32_t t1 = COL(s1, s2, s3, s0, k.x[1]);
        const uint32_t t2 = COL(s2, s3, s0, s1, k.x[2]);
        const uint32_t t3 = COL(s3, s0, s1, s2, k.x[3]);
        s0 = t0;
        s1 = t1;
        s2 = t2;
        s3 = t3;
    }
    // last round: S-box = byte 1 of T0 (no MixColumns); three PRMTs gather
    // the four S-box bytes of a column
#define SB(v, r) tlo(t, P0(v, r))
#define GATHER(a, b, c, d) \
    bperm(bperm(SB(a, 0), SB(b, 1), 0x0051u), bperm(SB(c, 2), SB(d, 3), 0x5100u), 0x7610u)
    const U4 k10 = rk.round(10);
    U4 o;
    o.x[0] = GATHER(s0, s1, s2, s3) ^ k10.x[0];
    o.x[1] = GATHER(s1, s2, s3, s0) ^ k10.x[1];
    o.x[2] = GATHER(s2, s3, s0, s1) ^ k10.x[2];
    o.x[3] = GATHER(s3, s0, s1, s2) ^ k10.x[3];
#undef GATHER
#undef SB
#undef COL
#undef P2
#undef P0
    return o;
}

struct RkConst {
    DASH_HD U4 round(int r) const {
        U4 k;
        for (int i = 0; i < 4; ++i) k.x[i] = c_pi_rk[4 * r + i];
        return k;
    }
};
struct RkPtr {  // 16-byte aligned schedule (44 words per inference)
    const uint32_t* p;
    DASH_HD U4 round(int r) const {
        U4 k;
#if defined(__CUDA_ARCH__)
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + r);
        k.x[0] = v.x;
        k.x[1] = v.y;
        k.x[2] = v.z;
        k.x[3] = v.w;
#else
        for (int i = 0; i < 4; ++i) k.x[i] = p[4 * r + i];
#endif
        return k;
    }
};

#if defined(__CUDA_ARCH__)
__device__ __noinline__ U4 aes_pi(U4 s, AesTab t) { return aes_core(s, RkConst{}, t); }
__device__ __noinline__ U4 aes_key(U4 s, const uint32_t* rk, AesTab t) { return aes_core(s, RkPtr{rk}, t); }
#else
static inline U4 aes_pi(U4 s, AesTab t) { return aes_core(s, RkConst{}, t); }
static inline U4 aes_key(U4 s, const uint32_t* rk, AesTab t) { return aes_core(s, RkPtr{rk}, t); }
#endif

// Davies-Meyer of K = Kc ^ tweak(g, row, slot)   (cipher.cpp:8-12, cipher.hpp:23-26).
// INLINE: the AES rounds are inlined at the call site (the garbling row loop,
// one copy) instead of calling aes_pi: a call spills the caller's live
// registers to local memory, which misses the small L1 left next to 218 KB
// of shared memory.
template <bool INLINE = false>
DASH_HD U4 hash_tw(const U4& Kc, uint64_t g, uint32_t row, uint32_t slot, const AesTab& t) {
    U4 K;
    K.x[0] = Kc.x[0] ^ (uint32_t)g;
    K.x[1] = Kc.x[1] ^ (uint32_t)(g >> 32);
    K.x[2] = Kc.x[2] ^ row;
    K.x[3] = Kc.x[3] ^ slot;
    U4 H = INLINE ? aes_core(K, RkConst{}, t) : aes_pi(K, t);
    H.x[0] ^= K.x[0];
    H.x[1] ^= K.x[1];
    H.x[2] ^= K.x[2];
    H.x[3] ^= K.x[3];
    return H;
}

// ------------------------------------------------------------ label codec
DASH_HD uint32_t fdiv(uint32_t x, uint32_t mag, uint32_t sh) { return umulhi32(x, mag) >> sh; }

// 128-bit value c (4 limbs, c[0] least significant) divided in place by D,
// returning c mod D.  `limbs` bounds the nonzero limbs (host-computed).
// Each limb step divides cur = rem 2^32 + c_i (rem < D < 2^30) by D with the
// reciprocal invD = ih 2^32 + il = floor((2^64 - 1) / D) using 32-bit
// multiplies only: q~ = rem ih + hi32(rem il + c_i ih) drops the c_i il
// partial product and the reciprocal's truncation, so q - 2 <= q~ <= q; the
// low word r~ = c_i - q~ D is then exact (r~ < 3D < 2^32) and two
// conditional subtractions finish (no 64 x 64 multiply-high, no branches).
// One limb step: (rem 2^32 + ci) = q D + r, rem < D
DASH_HD void dm_step(uint32_t rem, uint32_t ci, uint32_t il, uint32_t ih, uint32_t negD, uint32_t D, uint32_t& q,
                     uint32_t& r) {
#if defined(__CUDA_ARCH__)
    asm("{\n\t.reg .u64 t;\n\t.reg .u32 lo, hi;\n\t.reg .pred p;\n\t"
        "mul.wide.u32 t, %2, %4;\n\t"
        "mad.wide.u32 t, %3, %5, t;\n\t"
        "mov.b64 {lo, hi}, t;\n\t"
        "mad.lo.u32 %1, %2, %5, hi;\n\t"
        "mad.lo.u32 %0, %1, %6, %3;\n\t"
        "setp.ge.u32 p, %0, %7;\n\t@p sub.u32 %0, %0, %7;\n\t@p add.u32 %1, %1, 1;\n\t"
        "setp.ge.u32 p, %0, %7;\n\t@p sub.u32 %0, %0, %7;\n\t@p add.u32 %1, %1, 1;\n\t}"
        : "=&r"(r), "=&r"(q)  // early clobber: q is written before ci is read
        : "r"(rem), "r"(ci), "r"(il), "r"(ih), "r"(negD), "r"(D));
#else
    const uint64_t t = (uint64_t)rem * il + (uint64_t)ci * ih;
    q = rem * ih + (uint32_t)(t >> 32);
    r = q * negD + ci;
    for (int k = 0; k < 2; ++k)
        if (r >= D) {
            r -= D;
            ++q;
        }
#endif
}
DASH_HD uint32_t divmod_D(uint32_t c[4], const ModC& M, int limbs) {
    uint32_t rem = 0;
    const uint32_t il = (uint32_t)M.invD, ih = (uint32_t)(M.invD >> 32), D = M.D, negD = M.negD;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 3; i >= 0; --i) {
        if (i < limbs) {
            uint32_t q, r;
            dm_step(rem, c[i], il, ih, negD, D, q, r);
            c[i] = q;
            rem = r;
        }
    }
    return rem;
}

// Four base-m digits of v < m^4 packed as bytes.
DASH_HD uint32_t split4(uint32_t v, const ModC& M) {
    const uint32_t q1 = fdiv(v, M.mag_m, M.sh_m);
    const uint32_t d0 = q1 * M.negm + v;  // v - q1 m
    const uint32_t q2 = fdiv(q1, M.mag_m, M.sh_m);
    const uint32_t d1 = q2 * M.negm + q1;
    const uint32_t q3 = fdiv(q2, M.mag_m, M.sh_m);
    const uint32_t d2 = q3 * M.negm + q2;
    return d0 | (d1 << 8) | (d2 << 16) | (q3 << 24);
}

DASH_HD void mul_add_128(uint32_t c[4], uint32_t m, uint32_t add) {
    uint64_t t = (uint64_t)c[0] * m + add;
    c[0] = (uint32_t)t;
    t = (uint64_t)c[1] * m + (t >> 32);
    c[1] = (uint32_t)t;
    t = (uint64_t)c[2] * m + (t >> 32);
    c[2] = (uint32_t)t;
    t = (uint64_t)c[3] * m + (t >> 32);
    c[3] = (uint32_t)t;
}

// compress (label.cpp:208-219): Horner, one word (four digits) per step.

// ---- componentwise arithmetic (label.cpp:144-206) ----
DASH_HD uint32_t swar_add(uint32_t a, uint32_t b, const ModC& M) {
    const uint32_t s = a + b;
    const uint32_t ge = ((s + M.addc) >> 7) & 0x01010101u;
    return ge * M.negm + s;  // s - ge * m in one IMAD
}

DASH_HD void p2_add(uint32_t a[4], const uint32_t b[4], const ModC& M) {
    // fieldwise add mod 2^e: ((a & ~H) + (b & ~H)) ^ ((a ^ b) & H)
    uint64_t carry = 0;
    uint32_t x[4];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 4; ++i) {
        const uint64_t s = (uint64_t)(a[i] & ~M.hi[i]) + (b[i] & ~M.hi[i]) + carry;
        x[i] = (uint32_t)s;
        carry = s >> 32;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 4; ++i) a[i] = (x[i] ^ ((a[i] ^ b[i]) & M.hi[i])) & M.bits[i];
}

DASH_HD void p2_neg(uint32_t a[4], const ModC& M) {
    uint32_t n[4];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 4; ++i) n[i] = ~a[i] & M.bits[i];
    p2_add(n, M.lo, M);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 4; ++i) a[i] = n[i];
}


DASH_HD uint32_t field_width(uint32_t p) {
    uint32_t w = 0;
    while ((1u << w) < p) ++w;
    return w == 0 ? 1 : w;
}

// u128 helpers on U4
DASH_HD void u4_or_shl(U4& a, uint32_t v, uint32_t sh) {
    const uint32_t limb = sh >> 5, off = sh & 31;
    const uint32_t lo = v << off;
    const uint32_t hi = off ? (v >> (32 - off)) : 0u;
    a.x[0] |= limb == 0 ? lo : 0u;
    a.x[1] |= limb == 1 ? lo : (limb == 0 ? hi : 0u);
    a.x[2] |= limb == 2 ? lo : (limb == 1 ? hi : 0u);
    a.x[3] |= limb == 3 ? lo : (limb == 2 ? hi : 0u);
}
DASH_HD uint32_t u4_shr_low(const U4& a, uint32_t sh) {
    const uint32_t limb = sh >> 5, off = sh & 31;
    uint32_t v = a.x[0];
    v = limb == 1 ? a.x[1] : v;
    v = limb == 2 ? a.x[2] : v;
    v = limb == 3 ? a.x[3] : v;
    const uint32_t nx = limb == 0 ? a.x[1] : (limb == 1 ? a.x[2] : (limb == 2 ? a.x[3] : 0u));
    return (v >> off) | (off ? (nx << (32 - off)) : 0u);
}


// ---- PRF (prf.cpp:11-27): digit i = (u32 word i of AES_seed(wire|stream<<64|(i/4)<<96)) mod m
DASH_HD uint32_t mod32(uint32_t x, const ModC& M) {
    const uint64_t q = umulhi64((uint64_t)x, M.mag64);
    return x - (uint32_t)q * M.m;
}


// =================================================== label buffers
// A label lives in a per-lane buffer: word w at p[w * s].  In the
// activation kernel the buffers are in shared memory, lane-interleaved
// (s = 32), so a warp touching word w of its 32 labels hits 32 banks once.
// Non-power-of-two moduli: u8 digits, four per word (nw words).  Powers of
// two: the packed-bit form in 4 words, which equals the compressed value.
// All loops are runtime loops: one compact copy of every routine.
struct LB {
    uint32_t* p;
    uint32_t s;
    DASH_HD uint32_t& operator[](int w) const { return p[(uint32_t)w * s]; }
};

DASH_HD int lb_words(const ModC& M) { return M.pow2 ? 4 : M.nw; }

DASH_HD U4 lb_u4(LB a) {
    U4 r;
    r.x[0] = a[0];
    r.x[1] = a[1];
    r.x[2] = a[2];
    r.x[3] = a[3];
    return r;
}
DASH_HD void lb_set_u4(LB a, const U4& v) {
    a[0] = v.x[0];
    a[1] = v.x[1];
    a[2] = v.x[2];
    a[3] = v.x[3];
}

DASH_HD void lb_copy(LB d, LB s, const ModC& M) {
    const int n = lb_words(M);
    for (int w = 0; w < n; ++w) d[w] = s[w];
}

DASH_HD uint32_t lb_color(LB a, const ModC& M) { return M.pow2 ? (a[0] & (M.m - 1u)) : (a[0] & 0xffu); }

DASH_HD uint32_t top_keep(const ModC& M) {
    const int extra = M.nw * 4 - M.n;
    return extra ? (0xffffffffu >> (8 * extra)) : 0xffffffffu;
}

// digit-wise (x * s) mod m of one word (non-pow2)
DASH_HD uint32_t scale_word(uint32_t x, uint32_t s, const ModC& M) {
    uint32_t r = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int j = 0; j < 4; ++j) {
        const uint32_t t = ((x >> (8 * j)) & 0xffu) * s;
        r |= (t - fdiv(t, M.mag_m, M.sh_m) * M.m) << (8 * j);
    }
    return r;
}

DASH_HD U4 p2_scale(U4 x, uint32_t s, const ModC& M) {
    uint32_t acc[4] = {0, 0, 0, 0};
    for (int bit = 0; bit < 7; ++bit) {
        if ((s >> bit) & 1u) p2_add(acc, x.x, M);
        const uint32_t c0 = x.x[0] >> 31, c1 = x.x[1] >> 31, c2 = x.x[2] >> 31;
        x.x[0] = (x.x[0] << 1) & ~M.lo[0] & M.bits[0];
        x.x[1] = ((x.x[1] << 1) | c0) & ~M.lo[1] & M.bits[1];
        x.x[2] = ((x.x[2] << 1) | c1) & ~M.lo[2] & M.bits[2];
        x.x[3] = ((x.x[3] << 1) | c2) & ~M.lo[3] & M.bits[3];
    }
    U4 r;
    r.x[0] = acc[0];
    r.x[1] = acc[1];
    r.x[2] = acc[2];
    r.x[3] = acc[3];
    return r;
}

DASH_HD U4 p2_sub(U4 a, U4 b, const ModC& M) {
    p2_neg(b.x, M);
    p2_add(a.x, b.x, M);
    return a;
}

// a += b
DASH_HD void lb_add(LB a, LB b, const ModC& M) {
    if (M.pow2) {
        U4 x = lb_u4(a), y = lb_u4(b);
        p2_add(x.x, y.x, M);
        lb_set_u4(a, x);
        return;
    }
    for (int w = 0; w < M.nw; ++w) a[w] = swar_add(a[w], b[w], M);
}
// a += g (label words in global memory, same form)
DASH_HD void lb_add_g(LB a, const uint32_t* g, const ModC& M) {
    if (M.pow2) {
        U4 x = lb_u4(a);
        uint32_t y[4] = {g[0], g[1], g[2], g[3]};
        p2_add(x.x, y, M);
        lb_set_u4(a, x);
        return;
    }
    for (int w = 0; w < M.nw; ++w) a[w] = swar_add(a[w], g[w], M);
}
DASH_HD void lb_sub(LB a, LB b, const ModC& M) {
    if (M.pow2) {
        lb_set_u4(a, p2_sub(lb_u4(a), lb_u4(b), M));
        return;
    }
    for (int w = 0; w < M.nw; ++w) a[w] = swar_add(a[w], M.spread - b[w], M);
}
DASH_HD void lb_sub_g(LB a, const uint32_t* g, const ModC& M) {
    if (M.pow2) {
        U4 y;
        y.x[0] = g[0];
        y.x[1] = g[1];
        y.x[2] = g[2];
        y.x[3] = g[3];
        lb_set_u4(a, p2_sub(lb_u4(a), y, M));
        return;
    }
    for (int w = 0; w < M.nw; ++w) a[w] = swar_add(a[w], M.spread - g[w], M);
}
DASH_HD void lb_neg(LB a, const ModC& M) {
    if (M.pow2) {
        U4 x = lb_u4(a);
        p2_neg(x.x, M);
        lb_set_u4(a, x);
        return;
    }
    for (int w = 0; w < M.nw; ++w) a[w] = swar_add(M.spread - a[w], 0u, M);
}
// o = s * a (o may alias a)
DASH_HD void lb_scale(LB o, LB a, uint32_t s, const ModC& M) {
    if (M.pow2) {
        lb_set_u4(o, p2_scale(lb_u4(a), s, M));
        return;
    }
    for (int w = 0; w < M.nw; ++w) o[w] = scale_word(a[w], s, M);
}

// ---- multi-limb helpers of the codec: c = c * mul + v on L limbs (the
// result is known to fit L limbs; higher limbs stay zero) ----
DASH_HD void mad_l2(uint32_t& c0, uint32_t& c1, uint32_t mul, uint32_t v) {
    const uint64_t t = (uint64_t)c0 * mul + v;
    c0 = (uint32_t)t;
    c1 = c1 * mul + (uint32_t)(t >> 32);
}
DASH_HD void mad_l3(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t mul, uint32_t v) {
#if defined(__CUDA_ARCH__)
    uint32_t h0, h1;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(h0) : "r"(c0), "r"(mul));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(h1) : "r"(c1), "r"(mul));
    asm("mad.lo.cc.u32 %0, %0, %3, %4;\n\t"
        "madc.lo.cc.u32 %1, %1, %3, %5;\n\t"
        "madc.lo.u32 %2, %2, %3, %6;"
        : "+r"(c0), "+r"(c1), "+r"(c2)
        : "r"(mul), "r"(v), "r"(h0), "r"(h1));
#else
    uint64_t t = (uint64_t)c0 * mul + v;
    c0 = (uint32_t)t;
    t = (uint64_t)c1 * mul + (t >> 32);
    c1 = (uint32_t)t;
    c2 = c2 * mul + (uint32_t)(t >> 32);
#endif
}
DASH_HD void mad_l4(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t mul, uint32_t v) {
#if defined(__CUDA_ARCH__)
    uint32_t h0, h1, h2;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(h0) : "r"(c0), "r"(mul));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(h1) : "r"(c1), "r"(mul));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(h2) : "r"(c2), "r"(mul));
    asm("mad.lo.cc.u32 %0, %0, %4, %5;\n\t"
        "madc.lo.cc.u32 %1, %1, %4, %6;\n\t"
        "madc.lo.cc.u32 %2, %2, %4, %7;\n\t"
        "madc.lo.u32 %3, %3, %4, %8;"
        : "+r"(c0), "+r"(c1), "+r"(c2), "+r"(c3)
        : "r"(mul), "r"(v), "r"(h0), "r"(h1), "r"(h2));
#else
    uint64_t t = (uint64_t)c0 * mul + v;
    c0 = (uint32_t)t;
    t = (uint64_t)c1 * mul + (t >> 32);
    c1 = (uint32_t)t;
    t = (uint64_t)c2 * mul + (t >> 32);
    c2 = (uint32_t)t;
    c3 = c3 * mul + (uint32_t)(t >> 32);
#endif
}
// c += v * p on L limbs (p = D^j, c + v p fits L limbs)
DASH_HD void mac_l(uint32_t c[4], const uint32_t p[4], uint32_t v, int L) {
    uint64_t t = (uint64_t)p[0] * v + c[0];
    c[0] = (uint32_t)t;
    if (L < 2) return;
    t = (uint64_t)p[1] * v + c[1] + (t >> 32);
    c[1] = (uint32_t)t;
    if (L < 3) return;
    t = (uint64_t)p[2] * v + c[2] + (t >> 32);
    c[2] = (uint32_t)t;
    if (L < 4) return;
    c[3] = (uint32_t)((uint64_t)p[3] * v + c[3] + (t >> 32));
}

DASH_HD uint32_t dp4a_u8(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
    return __dp4a(a, b, c);
#else
    for (int i = 0; i < 4; ++i) c += ((a >> (8 * i)) & 0xffu) * ((b >> (8 * i)) & 0xffu);
    return c;
#endif
}
// value of one word of four base-m digits, d0 + m d1 + m^2 (d2 + m d3) < m^4
DASH_HD uint32_t wval(uint32_t x, const ModC& M) { return dp4a_u8(x, M.wlo, dp4a_u8(x, M.whi, 0u) * M.m2); }

// compress (label.cpp:208-219) as a Horner over the label's words, top
// down: word(w) yields word w (called once per word, nw-1 .. 0).  Two words
// per step when m^8 < 2^32, and each step only touches the 32-bit limbs its
// partial value can occupy (ModC::hlim, host-computed).
template <class F>
DASH_HD U4 horner(const ModC& M, F&& word) {
    int w = M.nw - 1;
    uint32_t c0 = wval(word(w), M), c1 = 0, c2 = 0, c3 = 0;
    --w;
    if (M.htop == 2) {
        c0 = c0 * M.m4 + wval(word(w), M);
        --w;
    }
    const uint32_t mul = M.m8, m4 = M.m4;
    const bool two = M.hp == 2;
    auto stepv = [&]() {
        uint32_t v = wval(word(w), M);
        --w;
        if (two) {
            v = v * m4 + wval(word(w), M);
            --w;
        }
        return v;
    };
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
    for (int i = M.hlim[0]; i > 0; --i) c0 = c0 * mul + stepv();
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
    for (int i = M.hlim[1]; i > 0; --i) {
        const uint32_t v = stepv();
        mad_l2(c0, c1, mul, v);
    }
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
    for (int i = M.hlim[2]; i > 0; --i) {
        const uint32_t v = stepv();
        mad_l3(c0, c1, c2, mul, v);
    }
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
    for (int i = M.hlim[3]; i > 0; --i) {
        const uint32_t v = stepv();
        mad_l4(c0, c1, c2, c3, mul, v);
    }
    U4 o;
    o.x[0] = c0;
    o.x[1] = c1;
    o.x[2] = c2;
    o.x[3] = c3;
    return o;
}

// compress (label.cpp:208-219)
DASH_HD U4 lb_compress(LB a, const ModC& M) {
    if (M.pow2) return lb_u4(a);
    return horner(M, [&](int w) { return a[w]; });
}

// Returns compress(key), then key += R (the per-row key step of every
// garbling loop: rows a and a+1 use keys in + aR and in + (a+1)R).
DASH_HD U4 lb_key_step(LB key, const uint32_t* R, const ModC& M) {
    if (M.pow2) {
        U4 k = lb_u4(key), r = k;
        uint32_t y[4] = {R[0], R[1], R[2], R[3]};
        p2_add(k.x, y, M);
        lb_set_u4(key, k);
        return r;
    }
    return horner(M, [&](int w) {
        const uint32_t x = key[w];
        key[w] = swar_add(x, R[w], M);
        return x;
    });
}

// Streams the base-m words of decompress_mod(cin, m) (label.cpp:228-232)
// to f(word_index, packed_digits); digits beyond n are zeroed.
template <class F>
DASH_HD void digits_stream(const U4& cin, const ModC& M, F&& f) {
    uint32_t c[4] = {cin.x[0], cin.x[1], cin.x[2], cin.x[3]};
    const uint32_t keep = top_keep(M);
    int w = 0;
    for (int j = 0; j < M.nchunks; ++j) {
        uint32_t chunk = divmod_D(c, M, M.limbs[j]);
#if defined(__CUDA_ARCH__)
#pragma unroll kCodecUnroll
#endif
        for (int ww = 0; ww < M.W && w < M.nw; ++ww, ++w) {
            const uint32_t q = fdiv(chunk, M.mag_m4, M.sh_m4);
            uint32_t v = split4(q * M.negm4 + chunk, M);
            chunk = q;
            if (w == M.nw - 1) v &= keep;
            f(w, v);
        }
    }
}

// digits_stream with a callback after every chunk of W words (fc(j))
template <class F, class G>
DASH_HD void digits_stream_c(const U4& cin, const ModC& M, F&& f, G&& fc) {
    uint32_t c[4] = {cin.x[0], cin.x[1], cin.x[2], cin.x[3]};
    const uint32_t keep = top_keep(M);
    int w = 0;
    for (int j = 0; j < M.nchunks; ++j) {
        uint32_t chunk = divmod_D(c, M, M.limbs[j]);
        for (int ww = 0; ww < M.W && w < M.nw; ++ww, ++w) {
            const uint32_t q = fdiv(chunk, M.mag_m4, M.sh_m4);
            uint32_t v = split4(q * M.negm4 + chunk, M);
            chunk = q;
            if (w == M.nw - 1) v &= keep;
            f(w, v);
        }
        fc(j);
    }
}

// Accumulates a label's compressed value low chunk first: word values are
// combined inside a chunk in 32 bits (the chunk's value < D < 2^31), and
// chunk j enters the 128-bit sum as chunk * D^j on the limbs it can reach.
struct ChunkAcc {
    uint32_t c[4] = {0, 0, 0, 0}, pd[4] = {1, 0, 0, 0};
    uint32_t acc = 0, pw = 1;
    DASH_HD void word(uint32_t t, const ModC& M) {
        acc += wval(t, M) * pw;
        pw *= M.m4;
    }
    DASH_HD void chunk(int j, const ModC& M) {
        const int L = M.climbs[j];
        mac_l(c, pd, acc, L);
        acc = 0;
        pw = 1;
        if (j + 1 < M.nchunks) {  // pd *= D
            uint64_t t = (uint64_t)pd[0] * M.D;
            pd[0] = (uint32_t)t;
            t = (uint64_t)pd[1] * M.D + (t >> 32);
            pd[1] = (uint32_t)t;
            t = (uint64_t)pd[2] * M.D + (t >> 32);
            pd[2] = (uint32_t)t;
            pd[3] = pd[3] * M.D + (uint32_t)(t >> 32);
        }
    }
    DASH_HD U4 value() const {
        U4 o;
        o.x[0] = c[0];
        o.x[1] = c[1];
        o.x[2] = c[2];
        o.x[3] = c[3];
        return o;
    }
};

// digits_stream of two values in one loop: two independent division chains
// interleave (evaluation decrypts ct - pad; its latency is this chain)
struct NoChunk {
    DASH_HD void operator()(int) const {}
};
template <class F, class G = NoChunk>
DASH_HD void digits_stream2(const U4& x, const U4& y, const ModC& M, F&& f, G&& fc = G()) {
    uint32_t a[4] = {x.x[0], x.x[1], x.x[2], x.x[3]}, b[4] = {y.x[0], y.x[1], y.x[2], y.x[3]};
    const uint32_t keep = top_keep(M);
    int w = 0;
    for (int j = 0; j < M.nchunks; ++j) {
        uint32_t ca = divmod_D(a, M, M.limbs[j]);
        uint32_t cb = divmod_D(b, M, M.limbs[j]);
#if defined(__CUDA_ARCH__)
#pragma unroll kCodecUnroll
#endif
        for (int ww = 0; ww < M.W && w < M.nw; ++ww, ++w) {
            const uint32_t qa = fdiv(ca, M.mag_m4, M.sh_m4), qb = fdiv(cb, M.mag_m4, M.sh_m4);
            uint32_t va = split4(qa * M.negm4 + ca, M), vb = split4(qb * M.negm4 + cb, M);
            ca = qa;
            cb = qb;
            if (w == M.nw - 1) {
                va &= keep;
                vb &= keep;
            }
            f(w, va, vb);
        }
        fc(j);
    }
}

DASH_HD void lb_decompress(LB out, const U4& c, const ModC& M) {
    if (M.pow2) {
        U4 v;
        for (int i = 0; i < 4; ++i) v.x[i] = c.x[i] & M.bits[i];
        lb_set_u4(out, v);
        return;
    }
    digits_stream(c, M, [&](int w, uint32_t v) { out[w] = v; });
}

// Row encryption (cipher.cpp:27-29 with the payload of gadgets.hpp):
//   ct = compress(decompress_mod(H, q) + base [+ g] [- s*sub])
// The pad digits stream out low word first; the ciphertext is accumulated
// low chunk first (ChunkAcc), so no scratch label is needed.
// G: payload adds the global label g; SUB: payload subtracts s * sub
template <bool G, bool SUB>
DASH_HD U4 lb_enc_t(const U4& H, LB base, const uint32_t* g, LB sub, uint32_t s, const ModC& M) {
    if (M.pow2) {
        U4 t;
        for (int i = 0; i < 4; ++i) t.x[i] = H.x[i] & M.bits[i];
        U4 b = lb_u4(base);
        p2_add(t.x, b.x, M);
        if (G) {
            uint32_t y[4] = {g[0], g[1], g[2], g[3]};
            p2_add(t.x, y, M);
        }
        if (SUB) t = p2_sub(t, p2_scale(lb_u4(sub), s, M), M);
        return t;
    }
    ChunkAcc A;
    digits_stream_c(
        H, M,
        [&](int w, uint32_t v) {
            uint32_t t = swar_add(v, base[w], M);
            if (G) t = swar_add(t, g[w], M);
            if (SUB) t = swar_add(t, M.spread - scale_word(sub[w], s, M), M);
            A.word(t, M);
        },
        [&](int j) { A.chunk(j, M); });
    return A.value();
}
DASH_HD U4 lb_enc(const U4& H, LB base, const uint32_t* g, LB* sub, uint32_t s, const ModC& M) {
    if (sub) return g ? lb_enc_t<true, true>(H, base, g, *sub, s, M) : lb_enc_t<false, true>(H, base, g, *sub, s, M);
    return g ? lb_enc_t<true, false>(H, base, g, base, s, M) : lb_enc_t<false, false>(H, base, g, base, s, M);
}

// out += digits(c)  (componentwise, streamed: no scratch label)
DASH_HD void lb_add_c(LB out, const U4& c, const ModC& M) {
    if (M.pow2) {
        U4 a = lb_u4(out);
        uint32_t y[4];
        for (int i = 0; i < 4; ++i) y[i] = c.x[i] & M.bits[i];
        p2_add(a.x, y, M);
        lb_set_u4(out, a);
        return;
    }
    digits_stream(c, M, [&](int w, uint32_t v) { out[w] = swar_add(out[w], v, M); });
}
// out -= digits(c)
DASH_HD void lb_sub_c(LB out, const U4& c, const ModC& M) {
    if (M.pow2) {
        U4 y;
        for (int i = 0; i < 4; ++i) y.x[i] = c.x[i] & M.bits[i];
        lb_set_u4(out, p2_sub(lb_u4(out), y, M));
        return;
    }
    digits_stream(c, M, [&](int w, uint32_t v) { out[w] = swar_add(out[w], M.spread - v, M); });
}
// out += s * x
DASH_HD void lb_add_scaled(LB out, LB x, uint32_t s, const ModC& M) {
    if (M.pow2) {
        U4 a = lb_u4(out);
        const U4 y = p2_scale(lb_u4(x), s, M);
        p2_add(a.x, y.x, M);
        lb_set_u4(out, a);
        return;
    }
    for (int w = 0; w < M.nw; ++w) out[w] = swar_add(out[w], scale_word(x[w], s, M), M);
}

// Row decryption (cipher.cpp:36-38): out = decompress_mod(ct) - decompress_mod(H)
DASH_HD void lb_dec(LB out, const U4& ct, const U4& H, const ModC& M) {
    if (M.pow2) {
        U4 a, b;
        for (int i = 0; i < 4; ++i) {
            a.x[i] = ct.x[i] & M.bits[i];
            b.x[i] = H.x[i] & M.bits[i];
        }
        lb_set_u4(out, p2_sub(a, b, M));
        return;
    }
    digits_stream2(ct, H, M, [&](int w, uint32_t a, uint32_t h) { out[w] = swar_add(a, M.spread - h, M); });
}

// compress(decompress_mod(ct) - decompress_mod(H)): the decrypted label
// straight into its compressed slot form, accumulated low word first in the
// decryption loop (no digit buffer, no second Horner pass)
DASH_HD U4 lb_dec_c(const U4& ct, const U4& H, const ModC& M) {
    if (M.pow2) {
        U4 a, b;
        for (int i = 0; i < 4; ++i) {
            a.x[i] = ct.x[i] & M.bits[i];
            b.x[i] = H.x[i] & M.bits[i];
        }
        return p2_sub(a, b, M);
    }
    ChunkAcc A;
    digits_stream2(
        ct, H, M, [&](int, uint32_t a, uint32_t h) { A.word(swar_add(a, M.spread - h, M), M); },
        [&](int j) { A.chunk(j, M); });
    return A.value();
}

// ---- global label rows: u8 digits, four per word, word stride `stride` ----
// Words are fetched kRowBatch at a time into registers before any of them is
// used: L is a generic pointer (shared memory), so a load / store per word
// would serialise one global-memory latency per word (the compiler cannot
// prove p and L do not alias).
constexpr int kRowBatch = 4;
// (The garbling tape keeps batch 1: it is issue-bound and at its register
// cap, and its operand loads are a small share of its time.)
template <int NB = kRowBatch, class F>
DASH_HD void rows_batched(const uint32_t* p, uint64_t stride, int nw, F&& f) {
    for (int w0 = 0; w0 < nw; w0 += NB) {
        uint32_t v[NB];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int j = 0; j < NB; ++j) v[j] = w0 + j < nw ? p[(uint64_t)(w0 + j) * stride] : 0u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int j = 0; j < NB; ++j)
            if (w0 + j < nw) f(w0 + j, v[j]);
    }
}

// Power-of-two labels: a word of four byte digits (each < 2^e) <-> the
// 4e-bit field of the packed form (digit j at bit e j)
DASH_HD uint32_t pack_digits(uint32_t x, uint32_t e) {
    if (e == 1) return ((x & 0x01010101u) * 0x10204080u) >> 28;  // bit 8j -> bit 28 + j, no carries
    return (x & 0xffu) | (((x >> 8) & 0xffu) << e) | (((x >> 16) & 0xffu) << (2 * e)) | ((x >> 24) << (3 * e));
}
DASH_HD uint32_t unpack_digits(uint32_t c, uint32_t e, uint32_t mask) {
    if (e == 1) return ((c & 0xfu) * 0x00204081u) & 0x01010101u;  // bit j -> bit 8j
    return (c & mask) | (((c >> e) & mask) << 8) | (((c >> (2 * e)) & mask) << 16) | (((c >> (3 * e)) & mask) << 24);
}
// byte mask of the digits of word w that exist (i < n)
DASH_HD uint32_t live_bytes(int w, const ModC& M) {
    const int left = M.n - 4 * w;
    return left >= 4 ? 0xffffffffu : (1u << (8 * left)) - 1u;
}

template <int NB = kRowBatch>
DASH_HD void lb_load_rows(LB L, const uint32_t* p, uint64_t stride, const ModC& M) {
    if (!M.pow2) {
        rows_batched<NB>(p, stride, M.nw, [&](int w, uint32_t x) { L[w] = x; });
        return;
    }
    U4 acc;
    acc.x[0] = acc.x[1] = acc.x[2] = acc.x[3] = 0;
    rows_batched<NB>(p, stride, M.nw, [&](int w, uint32_t x) {
        u4_or_shl(acc, pack_digits(x & live_bytes(w, M), M.e), (uint32_t)(4 * M.e * w));
    });
    for (int i = 0; i < 4; ++i) acc.x[i] &= M.bits[i];
    lb_set_u4(L, acc);
}

DASH_HD void lb_store_rows(LB L, uint32_t* p, uint64_t stride, const ModC& M) {
    if (!M.pow2) {
        for (int w = 0; w < M.nw; ++w) p[(uint64_t)w * stride] = L[w];
        return;
    }
    const U4 v = lb_u4(L);
    const uint32_t mask = M.m - 1u;
    for (int w = 0; w < M.nw; ++w)
        p[(uint64_t)w * stride] = unpack_digits(u4_shr_low(v, (uint32_t)(4 * M.e * w)), M.e, mask) & live_bytes(w, M);
}

// LabelPrf::draw (prf.cpp:11-27): digit i = (u32 word i of
// AES_seed(wire | stream<<64 | (i/4)<<96)) mod m; one AES block per word.
DASH_HD void lb_prf(LB L, uint64_t wire, uint32_t stream, const ModC& M, const uint32_t* rk, const AesTab& t) {
    const int nb = (M.n + 3) / 4;
    U4 acc;
    acc.x[0] = acc.x[1] = acc.x[2] = acc.x[3] = 0;
    const uint32_t mask = M.m - 1u;
    for (int b = 0; b < nb; ++b) {
        U4 s;
        s.x[0] = (uint32_t)wire;
        s.x[1] = (uint32_t)(wire >> 32);
        s.x[2] = stream;
        s.x[3] = (uint32_t)b;
        const U4 o = aes_key(s, rk, t);
        if (!M.pow2) {
            uint32_t x = 0;
            for (int j = 0; j < 4; ++j)
                if (4 * b + j < M.n) x |= mod32(o.x[j], M) << (8 * j);
            L[b] = x;
        } else {
            // four e-bit digits (words of the block mod 2^e) -> one 4e-bit field;
            // digits past n fall beyond bit 128 or under the final mask
            const uint32_t e = M.e;
            const uint32_t c = (o.x[0] & mask) | ((o.x[1] & mask) << e) | ((o.x[2] & mask) << (2 * e)) |
                               ((o.x[3] & mask) << (3 * e));
            u4_or_shl(acc, c, (uint32_t)(4 * e * b));
        }
    }
    if (M.pow2) {
        for (int i = 0; i < 4; ++i) acc.x[i] &= M.bits[i];
        lb_set_u4(L, acc);
    }
}

// ------------------------------------------------------------ element tape
constexpr int MAXCHUNK = 8;  // tape chunks per element in the garbling launch
struct ActParams {
    const TapeOp* tape;
    int n_ops;
    // level-scheduled evaluation tape (warp-per-element evaluation of small
    // launches): ops of level L are lv_tape[lv_start[L] .. lv_start[L+1]),
    // mutually independent, slots never reused inside a level
    const TapeOp* lv_tape;
    const uint16_t* lv_start;
    int n_levels;
    // op boundaries of the tape chunks (garbling launch: chunk c of every
    // element is a separate work item, run after chunk c-1 of that element)
    uint16_t chunk_op[MAXCHUNK + 1];
    const uint8_t* phi;        // phi pool (values already reduced mod q)
    int k;
    uint32_t E;                // elements per inference in this layer
    uint32_t B;                // inferences in this launch
    uint64_t gate_base, wire_base;
    uint64_t uc_cts, uc_gates, uc_wires;
    U4* blob;                  // ciphertexts of this layer, inference 0
    uint64_t blob_stride;      // ciphertexts between inferences
    const uint32_t* in[MAXK];  // input lane planes [B][nw][E]
    uint32_t* out[MAXK];       // output lane planes [B][nw][E]
    const uint32_t* rk;        // PRF round keys [B][44] (garble)
    const uint32_t* mult;      // multiples v*R_m [B][127][128][NWMAX] (garble)
    uint64_t mult_stride;      // words per inference
    U4* slots;                 // compressed label slots [nslots][B*E]
    // garble-side outputs are pure PRF functions of the element's wire ids:
    // ReLU lane i = v0 - u0 of its mm half gate, SignAct lane i = out0 of its
    // projection; act_output_thread writes them before the tape runs.
    uint8_t out_kind[MAXK];    // OP_MMHALF or OP_PROJ
    uint32_t out_wire[MAXK];   // wire offset of that gadget within the element
    // compressed u0, v0 of the output mm half gates ([B][E][k][2], garbling):
    // act_output_thread draws them once, the tape's MMHALF (cst = lane + 1)
    // reads them instead of drawing the same PRF labels again
    U4* mmlab;
    // garbling: `slots` holds max(nslots, nslots_lv) per element, so a small
    // launch may run the level tape with several warps per element
    int lv_ok;
};

// Work map of a multi-layer launch: layer li owns items [base[li], base[li+1]),
// item -> (b, 32-element block) with wpi[li] blocks per inference.
constexpr int MAXACT = 64;  // activation layers garbled in one launch (circuits have <= 64 layers)
struct ItemMap {
    uint32_t n;
    uint32_t base[MAXACT + 1];
    uint32_t wpi[MAXACT];
};

// Working buffers of one element: X (first operand / running key), K (the
// Z_2-sized second operand of half gates), A (fresh / accumulated label).
struct Elt {
    uint32_t b, u;
    uint64_t gate0, wire0;
    U4* rows;           // row j of this element at rows[j * rs] (act_rows)
    uint32_t rs;
    const uint32_t* rk;
    const uint32_t* mult;
    U4* slot0;          // slot s at slot0[s * sstride]
    uint64_t sstride;
    LB X, K, A;
    AesTab t;
};

// Garbled rows of an activation layer in HBM: blocks of 32 consecutive
// elements, row-major inside a block (row j of the block's element l at
// block + j*w + l, w = block width, 32 except a ragged last block), so the 32
// lanes of a warp write one contiguous 512-byte run per row instead of 32
// scattered half-sectors.  dashgpu_export_gc restores the reference order
// (element-major, layer.cpp:537-541).
DASH_HD U4* act_rows(U4* layer_blob, uint32_t E, uint64_t uc_cts, uint32_t u, uint32_t& rs) {
    const uint32_t blk = u >> 5, left = E - (blk << 5);
    rs = left < 32 ? left : 32;
    return layer_blob + (uint64_t)blk * 32 * uc_cts + (u & 31);
}

// Garbled rows are written once and read much later (evaluation): streaming
// stores keep them from evicting the kernels' L2 working set (label slots,
// multiples tables, register spills).
DASH_HD void store_row(U4* p, const U4& v) {
#if defined(__CUDA_ARCH__)
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]),
                 "r"(v.x[3])
                 : "memory");
#else
    *p = v;
#endif
}

DASH_HD const uint32_t* mult_row(const Elt& e, uint32_t m, uint32_t v) {
    return e.mult + ((uint64_t)c_modslot[m] * 128u + v) * NWMAX;
}

#if defined(__CUDA_ARCH__)
#define DASH_NI __device__ __noinline__
#else
#define DASH_NI static inline
#endif
// The out-of-line tape helpers only ever see label buffers in shared memory
// (act / wpe / lv kernels): telling the compiler so turns their generic
// LD/ST into LDS/STS (the provenance is lost at the call boundary).
#if defined(__CUDA_ARCH__)
#define DASH_SHARED(lb) __builtin_assume(__isShared((lb).p))
#else
#define DASH_SHARED(lb) ((void)0)
#endif
template <int NB>
DASH_NI void operand_n(LB L, const uint32_t* rows, uint32_t E, const U4* slot, uint32_t m);
DASH_NI void store_n(U4* slot, LB L, uint32_t m);

// NB: words of an input-lane operand fetched per batch (rows_batched)
template <int NB = 1>
DASH_HD void load_operand(LB L, const ActParams& P, const Elt& e, uint8_t v, const ModC& M) {
    if (v >= IN_LANE) operand_n<NB>(L, P.in[v - IN_LANE] + ((uint64_t)e.b * M.nw) * P.E + e.u, P.E, nullptr, M.m);
    else operand_n<NB>(L, nullptr, 0, e.slot0 + (uint64_t)v * e.sstride, M.m);
}

DASH_HD void store_slot(const Elt& e, uint8_t s, LB L, const ModC& M) {
    store_n(e.slot0 + (uint64_t)s * e.sstride, L, M.m);
}

// L += operand v (streamed, no scratch label)
template <int NB>
DASH_NI void add_operand_n(LB L, const uint32_t* rows, uint32_t E, const U4* slot, uint32_t m) {
    DASH_SHARED(L);
    const ModC& M = c_mod[m];
    if (!rows) {
        lb_add_c(L, *slot, M);
    } else if (!M.pow2) {
        rows_batched<NB>(rows, E, M.nw, [&](int w, uint32_t x) { L[w] = swar_add(L[w], x, M); });
    } else {
        uint32_t tmp[4];
        const LB T{tmp, 1};
        lb_load_rows<NB>(T, rows, E, M);
        lb_add(L, T, M);
    }
}
template <int NB = 1>
DASH_HD void add_operand(LB L, const ActParams& P, const Elt& e, uint8_t v, const ModC& M) {
    if (v >= IN_LANE) add_operand_n<NB>(L, P.in[v - IN_LANE] + ((uint64_t)e.b * M.nw) * P.E + e.u, P.E, nullptr, M.m);
    else add_operand_n<NB>(L, nullptr, 0, e.slot0 + (uint64_t)v * e.sstride, M.m);
}

// Single-copy helpers (called once per gadget, not per row): keeps the
// instruction working set of 24 co-resident warps inside the I-cache.
DASH_NI void prf_n(LB L, uint64_t wire, uint32_t stream, uint32_t m, const uint32_t* rk, AesTab t) {
    DASH_SHARED(L);
    lb_prf(L, wire, stream, c_mod[m], rk, t);
}
// operand from an input lane (row pointer of this element) or from a slot
template <int NB>
DASH_NI void operand_n(LB L, const uint32_t* rows, uint32_t E, const U4* slot, uint32_t m) {
    DASH_SHARED(L);
    if (rows) lb_load_rows<NB>(L, rows, E, c_mod[m]);
    else lb_decompress(L, *slot, c_mod[m]);
}
DASH_NI void store_n(U4* slot, LB L, uint32_t m) {
    DASH_SHARED(L);
    *slot = lb_compress(L, c_mod[m]);
}

// The garbling row loop of every projection / half gate (one copy).  Row
// r = (cin + a) mod p holds key X + aR_p and payload base + phi(a) R_q (phi
// table) or base + (a r mod p) R_p (phi == nullptr); GRR stores row j at
// R[j-1] and has no row 0 (gadgets.hpp:156-175, 195-219, 244-252).  The loop
// runs in ROW order (a = (r - cin) mod p, the key starts at X + a(r0) R_p and
// steps by R_p, wrapping since p R_p = 0): every lane of a warp writes the
// same row of its element, so a warp's stores fill whole 512-byte lines of
// the interleaved table, and GRR's row 0 is never computed.  X advances.
DASH_NI void garble_rows_n(LB X, LB base, AesTab t, const uint32_t* mult, uint32_t p, uint32_t q, uint32_t cin,
                           uint64_t g, const uint8_t* phi, uint32_t r, U4* R, int grr, uint32_t rs) {
    DASH_SHARED(X);
    DASH_SHARED(base);
    const ModC& Mp = c_mod[p];
    const ModC& Mq = c_mod[q];
    const uint32_t* Mp0 = mult + (uint64_t)c_modslot[p] * 128u * NWMAX;
    const uint32_t* Rp = Mp0 + NWMAX;
    const uint32_t* Mrow = mult + (uint64_t)c_modslot[q] * 128u * NWMAX;
    const uint32_t r0 = grr ? 1u : 0u;
    uint32_t a = r0 + p - cin;
    a = a >= p ? a - p : a;
    if (a) lb_add_g(X, Mp0 + (uint64_t)a * NWMAX, Mp);
    U4* out = R;  // row r0 goes to R[0] (GRR: row j at R[j-1])
    for (uint32_t row = r0; row < p; ++row) {
        const U4 H = hash_tw<true>(lb_key_step(X, Rp, Mp), g, row, 0, t);
        const uint32_t v = phi ? phi[a] : (a * r) % p;
        const U4 ct = lb_enc_t<true, false>(H, base, Mrow + (uint64_t)v * NWMAX, base, 0, Mq);
        store_row(out, ct);
        out += rs;
        a = a + 1 == p ? 0 : a + 1;
    }
}

// ---- garbling of one op (gadgets.hpp) ----
DASH_HD void garble_op(const ActParams& P, const Elt& e, const TapeOp& op) {
    switch (op.kind) {
        case OP_PROJ:
        case OP_GRR: {  // t_proj (gadgets.hpp:146-176), t_proj_grr (181-221)
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint32_t p = op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            const uint8_t* phi = P.phi + op.phi_off;
            U4* R = e.rows + (uint64_t)op.ct_off * e.rs;
            load_operand(e.X, P, e, op.a, Mp);
            const uint32_t cin = lb_color(e.X, Mp);
            if (op.kind == OP_PROJ) {
                prf_n(e.A, e.wire0 + op.wire_off, 0, op.qm, e.rk, e.t);
            } else {
                // out0 = -pad(key0, {g,0,0}) - phi(a0) R_q, key0 = in + a0 R_p
                const uint32_t a0 = cin == 0 ? 0 : p - cin;
                lb_copy(e.A, e.X, Mp);
                lb_add_g(e.A, mult_row(e, p, a0), Mp);
                const U4 H0 = hash_tw(lb_compress(e.A, Mp), g, 0, 0, e.t);
                lb_decompress(e.A, H0, Mq);
                lb_neg(e.A, Mq);
                lb_sub_g(e.A, mult_row(e, op.qm, phi[a0]), Mq);
            }
            garble_rows_n(e.X, e.A, e.t, e.mult, p, op.qm, cin, g, phi, 0, R, op.kind == OP_GRR, e.rs);
            store_slot(e, op.out, e.A, Mq);
            break;
        }
        case OP_HALF:      // t_half_gate (gadgets.hpp:230-282): x, y mod p
        case OP_MMHALF: {  // t_mm_half_gate (gadgets.hpp:292-358): x mod p, y mod q
            const bool mm = op.kind == OP_MMHALF;
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[mm ? op.qm : op.pm];
            const uint32_t p = op.pm, q = mm ? op.qm : op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            U4* R = e.rows + (uint64_t)op.ct_off * e.rs;
            load_operand(e.K, P, e, op.b, Mq);
            const uint32_t cy = lb_color(e.K, Mq);
            load_operand(e.X, P, e, op.a, Mp);
            const uint32_t cx = lb_color(e.X, Mp);
            const uint32_t r = mm ? cx : cy;
            // garbler rows: key x + aR_p, payload u0 + (a r mod p) R_p, slot 0
            const U4* ml = (op.cst && P.mmlab) ? P.mmlab + (((uint64_t)e.b * P.E + e.u) * P.k + (op.cst - 1)) * 2
                                               : nullptr;
            U4 u0c;
            if (ml) {
                u0c = ml[0];
                lb_decompress(e.A, u0c, Mp);
            } else {
                prf_n(e.A, e.wire0 + op.wire_off, 0, op.pm, e.rk, e.t);
                u0c = lb_compress(e.A, Mp);
            }
            // X is the running key here (K only holds the Z_2-sized y operand)
            garble_rows_n(e.X, e.A, e.t, e.mult, p, p, cx, g, nullptr, r, R, 0, e.rs);
            // evaluator rows: key y + bR_q, payload v0 - s x, slot 1
            load_operand(e.X, P, e, op.a, Mp);
            if (ml) lb_decompress(e.A, ml[1], Mp);
            else prf_n(e.A, e.wire0 + op.wire_off + 1, 0, op.pm, e.rk, e.t);
            load_operand(e.K, P, e, op.b, Mq);
            const uint32_t* Rq = mult_row(e, q, 1);
            const uint32_t fw = field_width(p);
            const uint32_t fmask = (1u << fw) - 1u;
            U4 sb;
            sb.x[0] = sb.x[1] = sb.x[2] = sb.x[3] = 0;
            // row order as in garble_rows_n: b = (row - cy) mod q, key y + bR_q
            uint32_t b = cy ? q - cy : 0;
            if (b) lb_add_g(e.K, mult_row(e, q, b), Mq);
            for (uint32_t row = 0; row < q; ++row, b = b + 1 == q ? 0 : b + 1) {
                uint32_t s = r + b;
                s = s >= p ? s - p : s;
                const U4 Kc = lb_key_step(e.K, Rq, Mq);
                const U4 H = hash_tw(Kc, g, row, 1, e.t);
                LB X = e.X;
                store_row(R + (uint64_t)(p + row) * e.rs, lb_enc_t<false, true>(H, e.A, nullptr, X, mm ? s : row, Mp));
                if (mm) {  // encrypt_short field of this row (cipher.cpp:45-60)
                    const U4 Hs = hash_tw(Kc, g, 0, 2, e.t);
                    u4_or_shl(sb, (s ^ (Hs.x[0] & fmask)) & fmask, fw * row);
                }
            }
            if (mm) store_row(R + (uint64_t)(p + q) * e.rs, sb);
            lb_sub_c(e.A, u0c, Mp);  // out = v0 - u0
            store_slot(e, op.out, e.A, Mp);
            break;
        }
        case OP_ADD:
        case OP_ADDACC: {  // free_add; fused chains keep the running sum in A
            const ModC& M = c_mod[op.qm];
            if (op.kind == OP_ADD) load_operand(e.A, P, e, op.a, M);
            add_operand(e.A, P, e, op.b, M);
            if (!(op.cst & kKeep)) store_slot(e, op.out, e.A, M);
            break;
        }
        case OP_ADDCONST: {  // add_public_constant (gadgets.hpp:127-139)
            const ModC& M = c_mod[op.qm];
            load_operand(e.A, P, e, op.a, M);
            const uint32_t c = op.cst % op.qm;
            if (c) lb_sub_g(e.A, mult_row(e, op.qm, c), M);
            store_slot(e, op.out, e.A, M);
            break;
        }
        case OP_OUTPUT:  // written up front by act_output_thread (same value)
            break;
    }
}

// Garbler-side output base label of lane i of element (b, u): for ReLU the
// mm half gate's v0 - u0 (gadgets.hpp:354), for SignAct the fresh out0 of the
// Z_2 -> Z_p projection (gadgets.hpp:172).  Both depend only on wire ids, so
// every activation layer's outputs exist before any gadget is garbled.
DASH_HD void act_output_thread(const ActParams& P, uint32_t b, uint32_t u, int i, uint32_t p, LB A, LB T,
                               const AesTab& t) {
    const ModC& M = c_mod[p];
    const uint32_t* rk = P.rk + (uint64_t)b * 44;
    const uint64_t w = P.wire_base + (uint64_t)u * P.uc_wires + P.out_wire[i];
    lb_prf(A, w, 0, M, rk, t);
    if (P.out_kind[i] == OP_MMHALF) {  // out = v0 - u0, v0 drawn at the next wire id
        lb_prf(T, w + 1, 0, M, rk, t);
        if (P.mmlab) {
            U4* ml = P.mmlab + (((uint64_t)b * P.E + u) * P.k + i) * 2;
            ml[0] = lb_compress(A, M);
            ml[1] = lb_compress(T, M);
        }
        lb_sub(T, A, M);
        lb_store_rows(T, P.out[i] + ((uint64_t)b * M.nw) * P.E + u, P.E, M);
    } else {
        lb_store_rows(A, P.out[i] + ((uint64_t)b * M.nw) * P.E + u, P.E, M);
    }
}

// ---- evaluation of one op ----
// c mod m of a compressed label (its colour digit) without unpacking digits
DASH_HD uint32_t colour_c(const U4& c, const ModC& M) {
    if (M.pow2) return c.x[0] & (M.m - 1u);
    uint64_t r = c.x[3] - (uint32_t)umulhi64((uint64_t)c.x[3], M.mag64) * M.m;
    for (int i = 2; i >= 0; --i) {
        const uint64_t x = (r << 32) | c.x[i];  // < m * 2^32: the magic quotient is exact
        r = x - umulhi64(x, M.mag64) * M.m;
    }
    return (uint32_t)r;
}

// Compressed operand (a slot already holds compress(label) < m^n, so a
// slot operand is used as is; an input lane is loaded and compressed) and
// its colour.  digits: also unpack the digits into L (needed by half gates).
DASH_HD U4 operand_c(LB L, const ActParams& P, const Elt& e, uint8_t v, const ModC& M, uint32_t& colour,
                     bool digits) {
    if (v < IN_LANE) {
        const U4 c = e.slot0[(uint64_t)v * e.sstride];
        colour = colour_c(c, M);
        if (digits) load_operand<kRowBatch>(L, P, e, v, M);
        return c;
    }
    load_operand<kRowBatch>(L, P, e, v, M);
    colour = lb_color(L, M);
    return lb_compress(L, M);
}

// LAT: latency-bound small launches (act_wpe_eval_kernel) also decompress
// both slot operands of an add in one loop; the throughput-bound per-thread
// kernel keeps the smaller code
template <bool LAT = false>
DASH_HD void eval_op(const ActParams& P, const Elt& e, const TapeOp& op) {
    switch (op.kind) {
        case OP_PROJ:
        case OP_GRR: {
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint64_t g = e.gate0 + op.gate_off;
            const U4* R = e.rows + (uint64_t)op.ct_off * e.rs;
            uint32_t row;
            const U4 Xc = operand_c(e.X, P, e, op.a, Mp, row, false);
            U4 ct;
            if (op.kind == OP_PROJ) {
                ct = R[(uint64_t)row * e.rs];
            } else if (row == 0) {
                ct.x[0] = ct.x[1] = ct.x[2] = ct.x[3] = 0;
            } else {
                ct = R[(uint64_t)(row - 1) * e.rs];
            }
            const U4 H = hash_tw(Xc, g, row, 0, e.t);
            e.slot0[(uint64_t)op.out * e.sstride] = lb_dec_c(ct, H, Mq);  // compressed, no digit buffer
            break;
        }
        case OP_HALF:
        case OP_MMHALF: {
            const bool mm = op.kind == OP_MMHALF;
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[mm ? op.qm : op.pm];
            const uint32_t p = op.pm, q = mm ? op.qm : op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            const U4* R = e.rows + (uint64_t)op.ct_off * e.rs;
            uint32_t cx, cy;
            const U4 Xc = operand_c(e.X, P, e, op.a, Mp, cx, true);
            const U4 Ky = operand_c(e.K, P, e, op.b, Mq, cy, false);
            // u = Dec(x, {g,cx,0}); out = Dec(y, {g,cy,1}) (+ s x) - u, all streamed
            const U4 Hx = hash_tw(Xc, g, cx, 0, e.t);
            const U4 Hy = hash_tw(Ky, g, cy, 1, e.t);
            const U4 cty = R[(uint64_t)(p + cy) * e.rs], ctx = R[(uint64_t)cx * e.rs];
            uint32_t s = cy;
            if (mm) {  // decrypt_short (cipher.cpp:62-69)
                const uint32_t fw = field_width(p);
                const uint32_t fmask = (1u << fw) - 1u;
                const U4 Hs = hash_tw(Ky, g, 0, 2, e.t);
                const uint32_t field = u4_shr_low(R[(uint64_t)(p + q) * e.rs], fw * cy) & fmask;
                s = ((field ^ (Hs.x[0] & fmask)) & fmask) % p;
            }
            if (Mp.pow2) {
                lb_dec(e.A, cty, Hy, Mp);
                lb_add_scaled(e.A, e.X, s, Mp);
                lb_sub_c(e.A, ctx, Mp);  // - u = - (decompress(ct_x) - pad_x)
                lb_add_c(e.A, Hx, Mp);
            } else {  // the same sums, two decryptions per loop (digits_stream2)
                digits_stream2(cty, Hy, Mp, [&](int w, uint32_t a, uint32_t h) {
                    e.A[w] = swar_add(swar_add(a, Mp.spread - h, Mp), scale_word(e.X[w], s, Mp), Mp);
                });
                digits_stream2(ctx, Hx, Mp, [&](int w, uint32_t c, uint32_t h) {
                    e.A[w] = swar_add(e.A[w], swar_add(h, Mp.spread - c, Mp), Mp);
                });
            }
            store_slot(e, op.out, e.A, Mp);
            break;
        }
        case OP_ADD:
        case OP_ADDACC: {
            const ModC& M = c_mod[op.qm];
            if (LAT && op.kind == OP_ADD && op.a < IN_LANE && op.b < IN_LANE && !M.pow2) {
                // two slot operands: both decompressed in one loop
                const U4 ca = e.slot0[(uint64_t)op.a * e.sstride], cb = e.slot0[(uint64_t)op.b * e.sstride];
                digits_stream2(ca, cb, M, [&](int w, uint32_t a, uint32_t b) { e.A[w] = swar_add(a, b, M); });
                if (!(op.cst & kKeep)) store_slot(e, op.out, e.A, M);
                break;
            }
            if (op.kind == OP_ADD) load_operand<kRowBatch>(e.A, P, e, op.a, M);
            add_operand<kRowBatch>(e.A, P, e, op.b, M);
            if (!(op.cst & kKeep)) store_slot(e, op.out, e.A, M);
            break;
        }
        case OP_ADDCONST: {
            if (op.a != op.out) {
                const ModC& M = c_mod[op.qm];
                load_operand<kRowBatch>(e.A, P, e, op.a, M);
                store_slot(e, op.out, e.A, M);
            }
            break;
        }
        case OP_OUTPUT: {
            const ModC& M = c_mod[op.qm];
            load_operand<kRowBatch>(e.A, P, e, op.a, M);
            lb_store_rows(e.A, P.out[op.cst] + ((uint64_t)e.b * M.nw) * P.E + e.u, P.E, M);
            break;
        }
    }
}

template <bool GARBLE>
DASH_HD void act_element(const ActParams& P, Elt& e, int op0, int op1) {
    e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
    e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
    e.rows = act_rows(P.blob + (uint64_t)e.b * P.blob_stride, P.E, P.uc_cts, e.u, e.rs);
    e.sstride = (uint64_t)P.B * P.E;
    e.slot0 = P.slots + (uint64_t)e.b * P.E + e.u;
    if (GARBLE) {
        e.rk = P.rk + (uint64_t)e.b * 44;
        e.mult = P.mult + (uint64_t)e.b * P.mult_stride;
    }
    for (int i = op0; i < op1; ++i) {
        const TapeOp op = P.tape[i];
        if (GARBLE) garble_op(P, e, op);
        else eval_op(P, e, op);
    }
}

}  // namespace dashgpu
