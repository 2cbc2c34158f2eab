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
// Design: labels of non-power-of-two moduli live in registers
// as packed u8 digits (four per u32 word); power-of-two moduli use the packed
// bit form, which *is* their compressed value.  Compression works word by
// word (Horner in base m^4); decompression divides the 128-bit value by
// D = m^(4W) <= 2^31 with a precomputed 64-bit reciprocal, then splits each
// chunk into digits with 32-bit magic multiplies.  Every modulus-dependent
// branch is warp-uniform (all lanes run the same tape), only data differs.
#pragma once

#include "dash_common.hpp"

namespace dashgpu {

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

struct Lab {
    uint32_t w[NWMAX];
};

struct U4 {
    uint32_t x[4];
};

// --------------------------------------------------------------- AES-128
// T0[x] = (2S, S, S, 3S) as little-endian bytes; T1..T3 are byte rotations.
// The table is replicated 32x in shared memory (entry x of lane l at
// T[x*32 + l]) so the 32 lanes of a warp never bank-conflict.
struct AesTab {
    const uint32_t* T;
    uint32_t lane;
};

DASH_HD uint32_t tl(const AesTab& t, uint32_t x) { return t.T[(x << 5) | t.lane]; }

template <class RK>
DASH_HD U4 aes_core(U4 s, const RK& rk, const AesTab& t) {
    uint32_t s0 = s.x[0] ^ rk(0), s1 = s.x[1] ^ rk(1), s2 = s.x[2] ^ rk(2), s3 = s.x[3] ^ rk(3);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int r = 1; r < 10; ++r) {
        const uint32_t t0 = tl(t, s0 & 0xff) ^ rotl32(tl(t, (s1 >> 8) & 0xff), 8) ^
                            rotl32(tl(t, (s2 >> 16) & 0xff), 16) ^ rotl32(tl(t, s3 >> 24), 24) ^ rk(4 * r);
        const uint32_t t1 = tl(t, s1 & 0xff) ^ rotl32(tl(t, (s2 >> 8) & 0xff), 8) ^
                            rotl32(tl(t, (s3 >> 16) & 0xff), 16) ^ rotl32(tl(t, s0 >> 24), 24) ^
                            rk(4 * r + 1);
        const uint32_t t2 = tl(t, s2 & 0xff) ^ rotl32(tl(t, (s3 >> 8) & 0xff), 8) ^
                            rotl32(tl(t, (s0 >> 16) & 0xff), 16) ^ rotl32(tl(t, s1 >> 24), 24) ^
                            rk(4 * r + 2);
        const uint32_t t3 = tl(t, s3 & 0xff) ^ rotl32(tl(t, (s0 >> 8) & 0xff), 8) ^
                            rotl32(tl(t, (s1 >> 16) & 0xff), 16) ^ rotl32(tl(t, s2 >> 24), 24) ^
                            rk(4 * r + 3);
        s0 = t0;
        s1 = t1;
        s2 = t2;
        s3 = t3;
    }
#define DASH_SB(v) ((tl(t, (v)) >> 8) & 0xff)
    U4 o;
    o.x[0] = (DASH_SB(s0 & 0xff) | (DASH_SB((s1 >> 8) & 0xff) << 8) | (DASH_SB((s2 >> 16) & 0xff) << 16) |
              (DASH_SB(s3 >> 24) << 24)) ^ rk(40);
    o.x[1] = (DASH_SB(s1 & 0xff) | (DASH_SB((s2 >> 8) & 0xff) << 8) | (DASH_SB((s3 >> 16) & 0xff) << 16) |
              (DASH_SB(s0 >> 24) << 24)) ^ rk(41);
    o.x[2] = (DASH_SB(s2 & 0xff) | (DASH_SB((s3 >> 8) & 0xff) << 8) | (DASH_SB((s0 >> 16) & 0xff) << 16) |
              (DASH_SB(s1 >> 24) << 24)) ^ rk(42);
    o.x[3] = (DASH_SB(s3 & 0xff) | (DASH_SB((s0 >> 8) & 0xff) << 8) | (DASH_SB((s1 >> 16) & 0xff) << 16) |
              (DASH_SB(s2 >> 24) << 24)) ^ rk(43);
#undef DASH_SB
    return o;
}

struct RkConst {
    DASH_HD uint32_t operator()(int i) const { return c_pi_rk[i]; }
};
struct RkPtr {
    const uint32_t* p;
    DASH_HD uint32_t operator()(int i) const {
#if defined(__CUDA_ARCH__)
        return __ldg(p + i);
#else
        return p[i];
#endif
    }
};

#if defined(__CUDA_ARCH__)
__device__ __noinline__ U4 aes_pi(U4 s, AesTab t) { return aes_core(s, RkConst{}, t); }
__device__ __noinline__ U4 aes_key(U4 s, const uint32_t* rk, AesTab t) { return aes_core(s, RkPtr{rk}, t); }
#else
static inline U4 aes_pi(U4 s, AesTab t) { return aes_core(s, RkConst{}, t); }
static inline U4 aes_key(U4 s, const uint32_t* rk, AesTab t) { return aes_core(s, RkPtr{rk}, t); }
#endif

// Davies-Meyer of K = Kc ^ tweak(g, row, slot)   (cipher.cpp:8-12, cipher.hpp:23-26)
DASH_HD U4 hash_tw(const U4& Kc, uint64_t g, uint32_t row, uint32_t slot, const AesTab& t) {
    U4 K;
    K.x[0] = Kc.x[0] ^ (uint32_t)g;
    K.x[1] = Kc.x[1] ^ (uint32_t)(g >> 32);
    K.x[2] = Kc.x[2] ^ row;
    K.x[3] = Kc.x[3] ^ slot;
    U4 H = aes_pi(K, t);
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
DASH_HD uint32_t divmod_D(uint32_t c[4], const ModC& M, int limbs) {
    uint64_t rem = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 3; i >= 0; --i) {
        if (i < limbs) {
            const uint64_t cur = (rem << 32) | c[i];
            uint64_t q = umulhi64(cur, M.invD);
            uint64_t r = cur - q * M.D;
            if (r >= M.D) {
                r -= M.D;
                ++q;
            }
            c[i] = (uint32_t)q;
            rem = r;
        }
    }
    return (uint32_t)rem;
}

// Four base-m digits of v < m^4 packed as bytes.
DASH_HD uint32_t split4(uint32_t v, const ModC& M) {
    const uint32_t q1 = fdiv(v, M.mag_m, M.sh_m);
    const uint32_t d0 = v - q1 * M.m;
    const uint32_t q2 = fdiv(q1, M.mag_m, M.sh_m);
    const uint32_t d1 = q1 - q2 * M.m;
    const uint32_t q3 = fdiv(q2, M.mag_m, M.sh_m);
    const uint32_t d2 = q2 - q3 * M.m;
    return d0 | (d1 << 8) | (d2 << 16) | (q3 << 24);
}

// decompress_mod (label.cpp:228-232): the first n base-m digits of c.
DASH_HD void decompress(Lab& L, const U4& cin, const ModC& M) {
    if (M.pow2) {
        L.w[0] = cin.x[0] & M.bits[0];
        L.w[1] = cin.x[1] & M.bits[1];
        L.w[2] = cin.x[2] & M.bits[2];
        L.w[3] = cin.x[3] & M.bits[3];
        return;
    }
    uint32_t c[4] = {cin.x[0], cin.x[1], cin.x[2], cin.x[3]};
    uint32_t chunk = 0;
    int left = 0, j = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w) {
        if (w < M.nw) {
            if (left == 0) {
                chunk = divmod_D(c, M, M.limbs[j]);
                ++j;
                left = M.W;
            }
            --left;
            const uint32_t q = fdiv(chunk, M.mag_m4, M.sh_m4);
            const uint32_t v = chunk - q * M.m4;
            chunk = q;
            L.w[w] = split4(v, M);
        } else {
            L.w[w] = 0;
        }
    }
    // digits beyond n in the top word must be zero
    const int extra = M.nw * 4 - M.n;
    if (extra) {
        const uint32_t keep = 0xffffffffu >> (8 * extra);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int w = 0; w < NWMAX; ++w)
            if (w == M.nw - 1) L.w[w] &= keep;
    }
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
DASH_HD U4 compress(const Lab& L, const ModC& M) {
    U4 o;
    if (M.pow2) {
        o.x[0] = L.w[0];
        o.x[1] = L.w[1];
        o.x[2] = L.w[2];
        o.x[3] = L.w[3];
        return o;
    }
    uint32_t c[4] = {0, 0, 0, 0};
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = NWMAX - 1; w >= 0; --w) {
        if (w < M.nw) {
            const uint32_t x = L.w[w];
            const uint32_t cv = (x & 0xff) + M.m * (((x >> 8) & 0xff) + M.m * (((x >> 16) & 0xff) + M.m * (x >> 24)));
            mul_add_128(c, M.m4, cv);
        }
    }
    o.x[0] = c[0];
    o.x[1] = c[1];
    o.x[2] = c[2];
    o.x[3] = c[3];
    return o;
}

DASH_HD uint32_t color(const Lab& L, const ModC& M) { return M.pow2 ? (L.w[0] & (M.m - 1u)) : (L.w[0] & 0xffu); }

// ---- componentwise arithmetic (label.cpp:144-206) ----
DASH_HD uint32_t swar_add(uint32_t a, uint32_t b, const ModC& M) {
    const uint32_t s = a + b;
    const uint32_t ge = ((s + M.addc) >> 7) & 0x01010101u;
    return s - ge * M.m;
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

DASH_HD void lab_add(Lab& a, const Lab& b, const ModC& M) {
    if (M.pow2) {
        p2_add(a.w, b.w, M);
        return;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w)
        if (w < M.nw) a.w[w] = swar_add(a.w[w], b.w[w], M);
}

// a += label stored in global memory (word form)
DASH_HD void lab_add_g(Lab& a, const uint32_t* g, const ModC& M) {
    if (M.pow2) {
        uint32_t b[4] = {g[0], g[1], g[2], g[3]};
        p2_add(a.w, b, M);
        return;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w)
        if (w < M.nw) a.w[w] = swar_add(a.w[w], g[w], M);
}

DASH_HD void lab_neg(Lab& a, const ModC& M) {
    if (M.pow2) {
        p2_neg(a.w, M);
        return;
    }
    // (m - d) mod m per digit: m - d, then fold m -> 0 via the SWAR add of 0
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w)
        if (w < M.nw) a.w[w] = swar_add(M.spread - a.w[w], 0u, M);
    const int extra = M.nw * 4 - M.n;
    if (extra) {
        const uint32_t keep = 0xffffffffu >> (8 * extra);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int w = 0; w < NWMAX; ++w)
            if (w == M.nw - 1) a.w[w] &= keep;
    }
}

DASH_HD void lab_sub(Lab& a, const Lab& b, const ModC& M) {
    if (M.pow2) {
        uint32_t n[4] = {b.w[0], b.w[1], b.w[2], b.w[3]};
        p2_neg(n, M);
        p2_add(a.w, n, M);
        return;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w)
        if (w < M.nw) a.w[w] = swar_add(a.w[w], M.spread - b.w[w], M);
    // padding digits: 0 + (m - 0) folds to 0 in swar_add
}

DASH_HD void lab_sub_g(Lab& a, const uint32_t* g, const ModC& M) {
    if (M.pow2) {
        uint32_t n[4] = {g[0], g[1], g[2], g[3]};
        p2_neg(n, M);
        p2_add(a.w, n, M);
        return;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w)
        if (w < M.nw) a.w[w] = swar_add(a.w[w], M.spread - g[w], M);
}

// s*a mod m componentwise, s per lane (label.cpp:167-175)
DASH_HD void lab_scale(Lab& o, const Lab& a, uint32_t s, const ModC& M) {
    if (M.pow2) {
        uint32_t acc[4] = {0, 0, 0, 0};
        uint32_t x[4] = {a.w[0], a.w[1], a.w[2], a.w[3]};
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int bit = 0; bit < 7; ++bit) {
            if ((s >> bit) & 1u) p2_add(acc, x, M);
            // double each field: shift left, drop bits that crossed a field boundary
            const uint32_t c0 = x[0] >> 31, c1 = x[1] >> 31, c2 = x[2] >> 31;
            x[0] = (x[0] << 1) & ~M.lo[0] & M.bits[0];
            x[1] = ((x[1] << 1) | c0) & ~M.lo[1] & M.bits[1];
            x[2] = ((x[2] << 1) | c1) & ~M.lo[2] & M.bits[2];
            x[3] = ((x[3] << 1) | c2) & ~M.lo[3] & M.bits[3];
        }
        o.w[0] = acc[0];
        o.w[1] = acc[1];
        o.w[2] = acc[2];
        o.w[3] = acc[3];
        return;
    }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w) {
        if (w < M.nw) {
            const uint32_t x = a.w[w];
            uint32_t r = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
            for (int j = 0; j < 4; ++j) {
                const uint32_t t = ((x >> (8 * j)) & 0xffu) * s;
                const uint32_t q = fdiv(t, M.mag_m, M.sh_m);
                r |= (t - q * M.m) << (8 * j);
            }
            o.w[w] = r;
        } else {
            o.w[w] = 0;
        }
    }
}

DASH_HD void lab_zero(Lab& a) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int w = 0; w < NWMAX; ++w) a.w[w] = 0;
}

// ---- global label rows: u8 digits, four per word, word stride `stride` ----
DASH_HD void lab_load_rows(Lab& L, const uint32_t* p, uint64_t stride, const ModC& M) {
    if (!M.pow2) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int w = 0; w < NWMAX; ++w) L.w[w] = (w < M.nw) ? p[(uint64_t)w * stride] : 0u;
        return;
    }
    uint32_t acc[4] = {0, 0, 0, 0};
    for (int w = 0; w < M.nw; ++w) {
        const uint32_t x = p[(uint64_t)w * stride];
        for (int j = 0; j < 4; ++j) {
            const int i = 4 * w + j;
            if (i < M.n) {
                const uint32_t d = (x >> (8 * j)) & 0xffu;
                const int pos = M.e * i;
                const int limb = pos >> 5, off = pos & 31;
                const uint32_t lo = d << off;
                const uint32_t hi = off ? (d >> (32 - off)) : 0u;
                acc[0] |= limb == 0 ? lo : 0u;
                acc[1] |= limb == 1 ? lo : (limb == 0 ? hi : 0u);
                acc[2] |= limb == 2 ? lo : (limb == 1 ? hi : 0u);
                acc[3] |= limb == 3 ? lo : (limb == 2 ? hi : 0u);
            }
        }
    }
    L.w[0] = acc[0];
    L.w[1] = acc[1];
    L.w[2] = acc[2];
    L.w[3] = acc[3];
}

DASH_HD void lab_store_rows(const Lab& L, uint32_t* p, uint64_t stride, const ModC& M) {
    if (!M.pow2) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int w = 0; w < NWMAX; ++w)
            if (w < M.nw) p[(uint64_t)w * stride] = L.w[w];
        return;
    }
    const uint32_t mask = M.m - 1u;
    for (int w = 0; w < M.nw; ++w) {
        uint32_t x = 0;
        for (int j = 0; j < 4; ++j) {
            const int i = 4 * w + j;
            if (i < M.n) {
                const int pos = M.e * i;
                const int limb = pos >> 5, off = pos & 31;
                uint32_t v = L.w[0];
                v = limb == 1 ? L.w[1] : v;
                v = limb == 2 ? L.w[2] : v;
                v = limb == 3 ? L.w[3] : v;
                uint32_t nx = limb == 0 ? L.w[1] : (limb == 1 ? L.w[2] : (limb == 2 ? L.w[3] : 0u));
                uint32_t d = (v >> off) | (off ? (nx << (32 - off)) : 0u);
                x |= (d & mask) << (8 * j);
            }
        }
        p[(uint64_t)w * stride] = x;
    }
}

// ---- PRF (prf.cpp:11-27): digit i = (u32 word i of AES_seed(wire|stream<<64|(i/4)<<96)) mod m
DASH_HD uint32_t mod32(uint32_t x, const ModC& M) {
    const uint64_t q = umulhi64((uint64_t)x, M.mag64);
    return x - (uint32_t)q * M.m;
}

DASH_HD void prf_label(Lab& L, uint64_t wire, uint32_t stream, const ModC& M, const uint32_t* rk, const AesTab& t) {
    if (!M.pow2) {
        uint32_t tmp[NWMAX];
        for (int w = 0; w < M.nw; ++w) {
            U4 s;
            s.x[0] = (uint32_t)wire;
            s.x[1] = (uint32_t)(wire >> 32);
            s.x[2] = stream;
            s.x[3] = (uint32_t)w;
            const U4 o = aes_key(s, rk, t);
            uint32_t x = 0;
            for (int j = 0; j < 4; ++j)
                if (4 * w + j < M.n) x |= mod32(o.x[j], M) << (8 * j);
            tmp[w] = x;
        }
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
        for (int w = 0; w < NWMAX; ++w) L.w[w] = (w < M.nw) ? tmp[w] : 0u;
        return;
    }
    uint32_t acc[4] = {0, 0, 0, 0};
    const int nb = (M.n + 3) / 4;
    const uint32_t mask = M.m - 1u;
    for (int b = 0; b < nb; ++b) {
        U4 s;
        s.x[0] = (uint32_t)wire;
        s.x[1] = (uint32_t)(wire >> 32);
        s.x[2] = stream;
        s.x[3] = (uint32_t)b;
        const U4 o = aes_key(s, rk, t);
        for (int j = 0; j < 4; ++j) {
            const int i = 4 * b + j;
            if (i < M.n) {
                const uint32_t d = o.x[j] & mask;
                const int pos = M.e * i;
                const int limb = pos >> 5, off = pos & 31;
                const uint32_t lo = d << off;
                const uint32_t hi = off ? (d >> (32 - off)) : 0u;
                acc[0] |= limb == 0 ? lo : 0u;
                acc[1] |= limb == 1 ? lo : (limb == 0 ? hi : 0u);
                acc[2] |= limb == 2 ? lo : (limb == 1 ? hi : 0u);
                acc[3] |= limb == 3 ? lo : (limb == 2 ? hi : 0u);
            }
        }
    }
    L.w[0] = acc[0] & M.bits[0];
    L.w[1] = acc[1] & M.bits[1];
    L.w[2] = acc[2] & M.bits[2];
    L.w[3] = acc[3] & M.bits[3];
}

// ---- row encryption (cipher.cpp:27-43) ----
// ct = compress(payload + decompress_mod(H, q))
DASH_HD U4 enc_with(const U4& H, const Lab& payload, const ModC& Q) {
    Lab pad;
    decompress(pad, H, Q);
    lab_add(pad, payload, Q);
    return compress(pad, Q);
}
// m = decompress_mod(ct, q) - decompress_mod(H, q)
DASH_HD void dec_with(Lab& out, const U4& ct, const U4& H, const ModC& Q) {
    Lab pad;
    decompress(out, ct, Q);
    decompress(pad, H, Q);
    lab_sub(out, pad, Q);
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

// ------------------------------------------------------------ element tape
struct ActParams {
    const TapeOp* tape;
    int n_ops;
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
    uint16_t lane_mod[MAXK];
    const uint32_t* rk;        // PRF round keys [B][44] (garble)
    const uint32_t* mult;      // multiples v*R_m [B][nslot][128][NWMAX] (garble)
    uint64_t mult_stride;      // words per inference
};

struct Elt {
    uint32_t b, u;
    uint64_t gate0, wire0;
    U4* rows;
    const uint32_t* rk;
    const uint32_t* mult;
    U4* slots;      // slot s at slots[s * sstride]
    uint32_t sstride;
    AesTab t;
};

DASH_HD const uint32_t* mult_row(const Elt& e, uint32_t m, uint32_t v) {
    return e.mult + ((uint64_t)c_modslot[m] * 128u + v) * NWMAX;
}

DASH_HD void load_operand(Lab& L, const ActParams& P, const Elt& e, uint8_t v, const ModC& M) {
    if (v >= IN_LANE) {
        const int lane = v - IN_LANE;
        const uint32_t* base = P.in[lane] + ((uint64_t)e.b * M.nw) * P.E + e.u;
        lab_load_rows(L, base, P.E, M);
    } else {
        decompress(L, e.slots[(uint32_t)v * e.sstride], M);
    }
}

DASH_HD void store_slot(const Elt& e, uint8_t s, const Lab& L, const ModC& M) {
    e.slots[(uint32_t)s * e.sstride] = compress(L, M);
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
            U4* R = e.rows + op.ct_off;
            Lab x;
            load_operand(x, P, e, op.a, Mp);
            const uint32_t cin = color(x, Mp);
            Lab out0;
            if (op.kind == OP_PROJ) {
                prf_label(out0, e.wire0 + op.wire_off, 0, Mq, e.rk, e.t);
            } else {
                // out0 = -pad(key0, {g,0,0}) - phi(a0) R_q, key0 = in + a0 R_p
                const uint32_t a0 = cin == 0 ? 0 : p - cin;
                Lab key0 = x;
                lab_add_g(key0, mult_row(e, p, a0), Mp);
                const U4 H0 = hash_tw(compress(key0, Mp), g, 0, 0, e.t);
                decompress(out0, H0, Mq);
                lab_neg(out0, Mq);
                lab_sub_g(out0, mult_row(e, op.qm, phi[a0]), Mq);
            }
            const uint32_t* Rp = mult_row(e, p, 1);
            for (uint32_t a = 0; a < p; ++a) {
                uint32_t row = cin + a;
                row = row >= p ? row - p : row;
                const U4 H = hash_tw(compress(x, Mp), g, row, 0, e.t);
                Lab pay = out0;
                lab_add_g(pay, mult_row(e, op.qm, phi[a]), Mq);
                const U4 ct = enc_with(H, pay, Mq);
                if (op.kind == OP_PROJ) R[row] = ct;
                else if (row != 0) R[row - 1] = ct;
                lab_add_g(x, Rp, Mp);
            }
            store_slot(e, op.out, out0, Mq);
            break;
        }
        case OP_HALF: {  // t_half_gate (gadgets.hpp:230-282)
            const ModC& M = c_mod[op.pm];
            const uint32_t p = op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            U4* R = e.rows + op.ct_off;
            Lab x, key;
            load_operand(x, P, e, op.a, M);
            const uint32_t* Rp = mult_row(e, p, 1);
            const uint32_t cx = color(x, M);
            uint32_t r;
            {
                Lab y;
                load_operand(y, P, e, op.b, M);
                r = color(y, M);
                key = y;
            }
            Lab u0;
            prf_label(u0, e.wire0 + op.wire_off, 0, M, e.rk, e.t);
            const U4 u0c = compress(u0, M);
            {
                Lab kx = x;
                for (uint32_t a = 0; a < p; ++a) {
                    uint32_t row = cx + a;
                    row = row >= p ? row - p : row;
                    const U4 H = hash_tw(compress(kx, M), g, row, 0, e.t);
                    Lab pay = u0;
                    lab_add_g(pay, mult_row(e, p, (a * r) % p), M);
                    R[row] = enc_with(H, pay, M);
                    lab_add_g(kx, Rp, M);
                }
            }
            Lab v0;
            prf_label(v0, e.wire0 + op.wire_off + 1, 0, M, e.rk, e.t);
            for (uint32_t b = 0; b < p; ++b) {
                uint32_t row = r + b;
                row = row >= p ? row - p : row;
                const U4 H = hash_tw(compress(key, M), g, row, 1, e.t);
                Lab pay = v0, sx;
                lab_scale(sx, x, row, M);
                lab_sub(pay, sx, M);
                R[p + row] = enc_with(H, pay, M);
                lab_add_g(key, Rp, M);
            }
            decompress(u0, u0c, M);
            lab_sub(v0, u0, M);
            store_slot(e, op.out, v0, M);
            break;
        }
        case OP_MMHALF: {  // t_mm_half_gate (gadgets.hpp:292-358)
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint32_t p = op.pm, q = op.qm;
            const uint64_t g = e.gate0 + op.gate_off;
            U4* R = e.rows + op.ct_off;
            Lab x;
            load_operand(x, P, e, op.a, Mp);
            const uint32_t r = color(x, Mp);
            Lab u0;
            prf_label(u0, e.wire0 + op.wire_off, 0, Mp, e.rk, e.t);
            const U4 u0c = compress(u0, Mp);
            {
                const uint32_t* Rp = mult_row(e, p, 1);
                Lab kx = x;
                for (uint32_t a = 0; a < p; ++a) {
                    uint32_t row = r + a;
                    row = row >= p ? row - p : row;
                    const U4 H = hash_tw(compress(kx, Mp), g, row, 0, e.t);
                    Lab pay = u0;
                    lab_add_g(pay, mult_row(e, p, (a * r) % p), Mp);
                    R[row] = enc_with(H, pay, Mp);
                    lab_add_g(kx, Rp, Mp);
                }
            }
            Lab v0;
            prf_label(v0, e.wire0 + op.wire_off + 1, 0, Mp, e.rk, e.t);
            const uint32_t fw = field_width(p);
            const uint32_t fmask = (1u << fw) - 1u;
            U4 sb;
            sb.x[0] = sb.x[1] = sb.x[2] = sb.x[3] = 0;
            {
                Lab key;
                load_operand(key, P, e, op.b, Mq);
                const uint32_t cy = color(key, Mq);
                const uint32_t* Rq = mult_row(e, q, 1);
                for (uint32_t b = 0; b < q; ++b) {
                    uint32_t row = cy + b;
                    row = row >= q ? row - q : row;
                    uint32_t s = r + b;
                    s = s >= p ? s - p : s;
                    const U4 Kc = compress(key, Mq);
                    const U4 H = hash_tw(Kc, g, row, 1, e.t);
                    Lab pay = v0, sx;
                    lab_scale(sx, x, s, Mp);
                    lab_sub(pay, sx, Mp);
                    R[p + row] = enc_with(H, pay, Mp);
                    const U4 Hs = hash_tw(Kc, g, 0, 2, e.t);
                    u4_or_shl(sb, (s ^ (Hs.x[0] & fmask)) & fmask, fw * row);
                    lab_add_g(key, Rq, Mq);
                }
            }
            R[p + q] = sb;
            decompress(u0, u0c, Mp);
            lab_sub(v0, u0, Mp);
            store_slot(e, op.out, v0, Mp);
            break;
        }
        case OP_ADD: {
            const ModC& M = c_mod[op.qm];
            Lab a, b;
            load_operand(a, P, e, op.a, M);
            load_operand(b, P, e, op.b, M);
            lab_add(a, b, M);
            store_slot(e, op.out, a, M);
            break;
        }
        case OP_ADDCONST: {  // add_public_constant (gadgets.hpp:127-139)
            const ModC& M = c_mod[op.qm];
            Lab a;
            load_operand(a, P, e, op.a, M);
            const uint32_t c = op.cst % op.qm;
            if (c) lab_sub_g(a, mult_row(e, op.qm, c), M);
            store_slot(e, op.out, a, M);
            break;
        }
        case OP_OUTPUT: {
            const ModC& M = c_mod[op.qm];
            Lab a;
            load_operand(a, P, e, op.a, M);
            uint32_t* base = P.out[op.cst] + ((uint64_t)e.b * M.nw) * P.E + e.u;
            lab_store_rows(a, base, P.E, M);
            break;
        }
    }
}

// decrypt_label (cipher.cpp:36-38): key label -> payload label mod q
DASH_HD void dec_row(Lab& out, const Lab& key, const ModC& Mk, uint64_t g, uint32_t row, uint32_t slot,
                     const U4& ct, const ModC& Mq, const AesTab& t) {
    const U4 H = hash_tw(compress(key, Mk), g, row, slot, t);
    dec_with(out, ct, H, Mq);
}

// ---- evaluation of one op ----
DASH_HD void eval_op(const ActParams& P, const Elt& e, const TapeOp& op) {
    switch (op.kind) {
        case OP_PROJ:
        case OP_GRR: {
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint64_t g = e.gate0 + op.gate_off;
            const U4* R = e.rows + op.ct_off;
            Lab x, out;
            load_operand(x, P, e, op.a, Mp);
            const uint32_t row = color(x, Mp);
            U4 ct;
            if (op.kind == OP_PROJ) {
                ct = R[row];
            } else if (row == 0) {
                ct.x[0] = ct.x[1] = ct.x[2] = ct.x[3] = 0;
            } else {
                ct = R[row - 1];
            }
            dec_row(out, x, Mp, g, row, 0, ct, Mq, e.t);
            store_slot(e, op.out, out, Mq);
            break;
        }
        case OP_HALF: {
            const ModC& M = c_mod[op.pm];
            const uint32_t p = op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            const U4* R = e.rows + op.ct_off;
            Lab x, y, u, out, sx;
            load_operand(x, P, e, op.a, M);
            load_operand(y, P, e, op.b, M);
            const uint32_t cx = color(x, M), cy = color(y, M);
            dec_row(u, x, M, g, cx, 0, R[cx], M, e.t);
            dec_row(out, y, M, g, cy, 1, R[p + cy], M, e.t);
            lab_scale(sx, x, cy, M);
            lab_add(out, sx, M);
            lab_sub(out, u, M);
            store_slot(e, op.out, out, M);
            break;
        }
        case OP_MMHALF: {
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint32_t p = op.pm, q = op.qm;
            const uint64_t g = e.gate0 + op.gate_off;
            const U4* R = e.rows + op.ct_off;
            Lab x, y, u, out, sx;
            load_operand(x, P, e, op.a, Mp);
            load_operand(y, P, e, op.b, Mq);
            const uint32_t cx = color(x, Mp), cy = color(y, Mq);
            dec_row(u, x, Mp, g, cx, 0, R[cx], Mp, e.t);
            const U4 Ky = compress(y, Mq);
            const U4 H = hash_tw(Ky, g, cy, 1, e.t);
            dec_with(out, R[p + cy], H, Mp);
            // decrypt_short (cipher.cpp:62-69)
            const uint32_t fw = field_width(p);
            const uint32_t fmask = (1u << fw) - 1u;
            const U4 Hs = hash_tw(Ky, g, 0, 2, e.t);
            const uint32_t field = u4_shr_low(R[p + q], fw * cy) & fmask;
            const uint32_t s = ((field ^ (Hs.x[0] & fmask)) & fmask) % p;
            lab_scale(sx, x, s, Mp);
            lab_add(out, sx, Mp);
            lab_sub(out, u, Mp);
            store_slot(e, op.out, out, Mp);
            break;
        }
        case OP_ADD: {
            const ModC& M = c_mod[op.qm];
            Lab a, b;
            load_operand(a, P, e, op.a, M);
            load_operand(b, P, e, op.b, M);
            lab_add(a, b, M);
            store_slot(e, op.out, a, M);
            break;
        }
        case OP_ADDCONST: {
            if (op.a != op.out) {
                const ModC& M = c_mod[op.qm];
                Lab a;
                load_operand(a, P, e, op.a, M);
                store_slot(e, op.out, a, M);
            }
            break;
        }
        case OP_OUTPUT: {
            const ModC& M = c_mod[op.qm];
            Lab a;
            load_operand(a, P, e, op.a, M);
            uint32_t* base = P.out[op.cst] + ((uint64_t)e.b * M.nw) * P.E + e.u;
            lab_store_rows(a, base, P.E, M);
            break;
        }
    }
}

template <bool GARBLE>
DASH_HD void act_element(const ActParams& P, Elt& e) {
    e.gate0 = P.gate_base + (uint64_t)e.u * P.uc_gates;
    e.wire0 = P.wire_base + (uint64_t)e.u * P.uc_wires;
    e.rows = P.blob + (uint64_t)e.b * P.blob_stride + (uint64_t)e.u * P.uc_cts;
    if (GARBLE) {
        e.rk = P.rk + (uint64_t)e.b * 44;
        e.mult = P.mult + (uint64_t)e.b * P.mult_stride;
    }
    for (int i = 0; i < P.n_ops; ++i) {
        const TapeOp op = P.tape[i];
        if (GARBLE) garble_op(P, e, op);
        else eval_op(P, e, op);
    }
}

}  // namespace dashgpu
