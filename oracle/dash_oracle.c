/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the Dash LabelTensor garble/eval
 * path.  Plain C restatement of the reference algorithm; every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/core/).  Pinned by tests/test_oracle.py against golden
 * vectors generated from the compiled reference (tests/golden/).
 *
 * Deliberately simple: one label = up to 128 u16 digits, u128 via the GNU
 * extension, byte-wise AES.  Element loops are OpenMP-parallel with the same
 * per-element gate/wire/ct strides the reference uses (layer.cpp:516-550),
 * so results are thread-count independent.
 */
#include "dash_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

#define MAXD 128  /* kMaxLabelDigits (label.hpp:13) */
#define MAXM 128  /* kMaxModulus (label.hpp:15) */
#define MAXK 16   /* kMaxCrtPrimes (crt.hpp:11) */

static __thread char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

static u128 ld128(const uint64_t* p) { return ((u128)p[1] << 64) | p[0]; }
static void st128(uint64_t* p, u128 v) {
    p[0] = (uint64_t)v;
    p[1] = (uint64_t)(v >> 64);
}

/* ===================== AES-128 (aes.cpp:32-90, FIPS-197) ===================== */

static uint8_t SBOX[256];
static int sbox_ready = 0;

static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t r = 0;
    while (b) {
        if (b & 1) r ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
        b >>= 1;
    }
    return r;
}
static uint8_t rotl8(uint8_t x, int s) { return (uint8_t)((x << s) | (x >> (8 - s))); }

static void sbox_init(void) {
    if (sbox_ready) return;
    for (int x = 0; x < 256; ++x) {
        uint8_t inv = 0;
        if (x) {
            for (int y = 1; y < 256; ++y)
                if (gmul((uint8_t)x, (uint8_t)y) == 1) {
                    inv = (uint8_t)y;
                    break;
                }
        }
        SBOX[x] = (uint8_t)(inv ^ rotl8(inv, 1) ^ rotl8(inv, 2) ^ rotl8(inv, 3) ^
                            rotl8(inv, 4) ^ 0x63);
    }
    sbox_ready = 1;
}

typedef struct {
    uint8_t rk[176];
} aes_key;

static void aes_expand(aes_key* k, const uint8_t key[16]) {
    static const uint8_t rcon[10] = {1, 2, 4, 8, 16, 32, 64, 128, 0x1b, 0x36};
    sbox_init();
    memcpy(k->rk, key, 16);
    for (int i = 4; i < 44; ++i) {
        uint8_t t[4];
        memcpy(t, k->rk + 4 * (i - 1), 4);
        if (i % 4 == 0) {
            uint8_t t0 = t[0];
            t[0] = (uint8_t)(SBOX[t[1]] ^ rcon[i / 4 - 1]);
            t[1] = SBOX[t[2]];
            t[2] = SBOX[t[3]];
            t[3] = SBOX[t0];
        }
        for (int j = 0; j < 4; ++j) k->rk[4 * i + j] = (uint8_t)(k->rk[4 * (i - 4) + j] ^ t[j]);
    }
}

/* The u128's little-endian bytes are the AES block (aes.cpp:48-57). */
static u128 aes_enc(const aes_key* k, u128 block) {
    uint8_t s[16];
    memcpy(s, &block, 16);
    for (int i = 0; i < 16; ++i) s[i] ^= k->rk[i];
    for (int r = 1; r <= 10; ++r) {
        uint8_t t[16];
        for (int i = 0; i < 16; ++i) t[i] = SBOX[s[i]];
        /* ShiftRows: state[row][col] = s[row + 4col] */
        for (int c = 0; c < 4; ++c)
            for (int row = 0; row < 4; ++row) s[row + 4 * c] = t[row + 4 * ((c + row) & 3)];
        if (r != 10) {
            for (int c = 0; c < 4; ++c) {
                uint8_t a0 = s[4 * c], a1 = s[4 * c + 1], a2 = s[4 * c + 2], a3 = s[4 * c + 3];
                s[4 * c] = (uint8_t)(gmul(a0, 2) ^ gmul(a1, 3) ^ a2 ^ a3);
                s[4 * c + 1] = (uint8_t)(a0 ^ gmul(a1, 2) ^ gmul(a2, 3) ^ a3);
                s[4 * c + 2] = (uint8_t)(a0 ^ a1 ^ gmul(a2, 2) ^ gmul(a3, 3));
                s[4 * c + 3] = (uint8_t)(gmul(a0, 3) ^ a1 ^ a2 ^ gmul(a3, 2));
            }
        }
        for (int i = 0; i < 16; ++i) s[i] ^= k->rk[16 * r + i];
    }
    u128 out;
    memcpy(&out, s, 16);
    return out;
}

static aes_key g_pi; /* fixed_permutation(): all-zero key (aes.cpp:142-145) */
static int g_pi_ready = 0;
static const aes_key* fixed_pi(void) {
    if (!g_pi_ready) {
        uint8_t z[16] = {0};
        aes_expand(&g_pi, z);
        g_pi_ready = 1;
    }
    return &g_pi;
}

/* cipher.cpp:8 */
static u128 davies_meyer(u128 x) { return aes_enc(fixed_pi(), x) ^ x; }

/* ===================== labels (label.cpp) ===================== */

typedef struct {
    uint16_t m, n;
    uint16_t d[MAXD];
} olabel;

typedef struct {
    int n, pow2, log2m, full_range;
    u128 mn;
    int r;
    uint64_t mr;
} modinfo;

static modinfo MI[MAXM + 1];
static int mi_ready = 0;

/* label.cpp:15-29 */
static int compute_n_digits(int m) {
    const u128 limit = ((u128)0 - 1) / (u128)m;
    u128 acc = 1;
    int n = 0;
    while (acc <= limit) {
        acc *= (u128)m;
        ++n;
    }
    if ((m & (m - 1)) == 0) {
        int e = 0;
        while ((1 << e) < m) ++e;
        if (e * (n + 1) == 128) ++n;
    }
    return n;
}

/* label.cpp:31-64 */
static void mi_init(void) {
    if (mi_ready) return;
    for (int m = 2; m <= MAXM; ++m) {
        modinfo* I = &MI[m];
        I->n = compute_n_digits(m);
        I->pow2 = (m & (m - 1)) == 0;
        I->log2m = 0;
        if (I->pow2)
            while ((1 << (I->log2m + 1)) <= m) ++I->log2m;
        u128 mn = 1;
        for (int i = 0; i < I->n; ++i) mn *= (u128)m;
        I->full_range = mn == 0;
        I->mn = mn;
        uint64_t mr = 1;
        int r = 0;
        while (mr <= ((uint64_t)1 << 31) / (uint64_t)m) {
            mr *= (uint64_t)m;
            ++r;
        }
        I->r = r;
        I->mr = mr;
    }
    mi_ready = 1;
}

static olabel lshape(int m) {
    olabel l;
    mi_init();
    l.m = (uint16_t)m;
    l.n = (uint16_t)MI[m].n;
    return l;
}
static olabel lzeros(int m) {
    olabel l = lshape(m);
    memset(l.d, 0, sizeof l.d);
    return l;
}
static int color(const olabel* l) { return l->d[0]; }

/* label.cpp:208-219 */
static u128 compress(const olabel* l) {
    const modinfo* I = &MI[l->m];
    u128 acc = 0;
    if (I->pow2) {
        for (int i = l->n - 1; i >= 0; --i) acc = (acc << I->log2m) | l->d[i];
        return acc;
    }
    for (int i = l->n - 1; i >= 0; --i) acc = acc * l->m + l->d[i];
    return acc;
}

/* label.cpp:101-123 + 228-232: reduce mod m^n (unless full range), then digits */
static olabel decompress_mod(u128 c, int m) {
    mi_init();
    const modinfo* I = &MI[m];
    olabel l = lshape(m);
    if (!I->full_range && c >= I->mn) c %= I->mn;
    if (I->pow2) {
        for (int i = 0; i < I->n; ++i) {
            l.d[i] = (uint16_t)(c & (u128)(m - 1));
            c >>= I->log2m;
        }
        return l;
    }
    for (int i = 0; i < I->n; ++i) {
        l.d[i] = (uint16_t)(c % (u128)m);
        c /= (u128)m;
    }
    return l;
}

/* label.cpp:144-206 */
static void ladd_into(olabel* a, const olabel* b) {
    for (int i = 0; i < a->n; ++i) a->d[i] = (uint16_t)((a->d[i] + b->d[i]) % a->m);
}
static void lsub_into(olabel* a, const olabel* b) {
    for (int i = 0; i < a->n; ++i) a->d[i] = (uint16_t)((a->d[i] + a->m - b->d[i]) % a->m);
}
static olabel ladd(olabel a, const olabel* b) {
    ladd_into(&a, b);
    return a;
}
static olabel lsub(olabel a, const olabel* b) {
    lsub_into(&a, b);
    return a;
}
static olabel lneg(olabel a) {
    for (int i = 0; i < a.n; ++i) a.d[i] = (uint16_t)(a.d[i] ? a.m - a.d[i] : 0);
    return a;
}
static olabel lscale(olabel a, uint32_t c) {
    for (int i = 0; i < a.n; ++i) a.d[i] = (uint16_t)((a.d[i] * c) % a.m);
    return a;
}
static void ladd_scaled(olabel* a, const olabel* b, uint32_t c) {
    for (int i = 0; i < a->n; ++i) a->d[i] = (uint16_t)((a->d[i] + b->d[i] * c) % a->m);
}
static int leq(const olabel* a, const olabel* b) {
    if (a->m != b->m) return 0;
    for (int i = 0; i < a->n; ++i)
        if (a->d[i] != b->d[i]) return 0;
    return 1;
}

/* ===================== PRF (prf.cpp:11-27, prf.hpp:24-32) ===================== */

typedef struct {
    aes_key k;
} oprf;

static olabel prf_draw(const oprf* p, uint64_t wire, uint32_t stream, int m) {
    olabel l = lshape(m);
    const int nb = (l.n + 3) / 4;
    u128 blocks[32];
    for (int b = 0; b < nb; ++b)
        blocks[b] = aes_enc(&p->k, (u128)wire | ((u128)stream << 64) | ((u128)(uint32_t)b << 96));
    for (int i = 0; i < l.n; ++i) {
        uint32_t w = (uint32_t)(blocks[i / 4] >> (32 * (i % 4)));
        l.d[i] = (uint16_t)(w % (uint32_t)m);
    }
    return l;
}
static olabel prf_label(const oprf* p, uint64_t wire, int m) { return prf_draw(p, wire, 0, m); }
static olabel prf_offset(const oprf* p, int m) {
    olabel r = prf_draw(p, (uint64_t)m, 1, m);
    r.d[0] = 1;
    return r;
}

/* ===================== cipher (cipher.cpp:8-69, cipher.hpp:13-26,62-66) ===================== */

static u128 tweak(uint64_t g, uint32_t row, uint32_t slot) {
    return (u128)g | ((u128)row << 64) | ((u128)slot << 96);
}
static u128 pad_bits(const olabel* k1, u128 tw) { return davies_meyer(compress(k1) ^ tw); }
static olabel pad_label(const olabel* k1, u128 tw, int q) { return decompress_mod(pad_bits(k1, tw), q); }
static u128 encrypt_label(const olabel* k1, u128 tw, const olabel* msg) {
    olabel pad = pad_label(k1, tw, msg->m);
    olabel s = ladd(*msg, &pad);
    return compress(&s);
}
static olabel decrypt_label(const olabel* k1, u128 tw, u128 ct, int q) {
    olabel c = decompress_mod(ct, q);
    olabel pad = pad_label(k1, tw, q);
    return lsub(c, &pad);
}
static int field_width(int p) {
    int w = 0;
    while ((1 << w) < p) ++w;
    return w == 0 ? 1 : w;
}
static u128 encrypt_short(const olabel* keys, u128 tw, const uint16_t* vals, int count, int p) {
    const int w = field_width(p);
    const u128 fm = ((u128)1 << w) - 1;
    u128 ct = 0;
    for (int j = 0; j < count; ++j) {
        u128 mask = pad_bits(&keys[j], tw) & fm;
        u128 field = ((u128)vals[j] ^ mask) & fm;
        ct |= field << (w * j);
    }
    return ct;
}
static int decrypt_short(const olabel* key, u128 tw, u128 ct, int index, int p) {
    const int w = field_width(p);
    const u128 fm = ((u128)1 << w) - 1;
    u128 field = (ct >> (w * index)) & fm;
    u128 mask = pad_bits(key, tw) & fm;
    return (int)((uint32_t)(field ^ mask) % (uint32_t)p);
}

/* ===================== CRT (crt.cpp:22-101) ===================== */

static const int PRIMES[MAXK] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53};

typedef struct {
    int k;
    int primes[MAXK];
    u128 P;
    u128 coeffs[MAXK];
} ocrt;

static ocrt crt_base(int k) {
    ocrt b;
    b.k = k;
    b.P = 1;
    for (int i = 0; i < k; ++i) {
        b.primes[i] = PRIMES[i];
        b.P *= (u128)PRIMES[i];
    }
    for (int i = 0; i < k; ++i) {
        const int p = PRIMES[i];
        u128 A = b.P / (u128)p;
        uint64_t base = (uint64_t)(A % (u128)p), r = 1;
        for (int e = p - 2; e > 0; e >>= 1) {
            if (e & 1) r = r * base % (uint64_t)p;
            base = base * base % (uint64_t)p;
        }
        b.coeffs[i] = A * (u128)r;
    }
    return b;
}

static int encode_signed(int64_t v, const ocrt* b, u128* out) {
    const u128 half_up = (b->P + 1) / 2, half_down = b->P / 2;
    if (v >= 0) {
        if ((u128)v >= half_up) return fail(ORC_DATA, "encode_signed: value above range");
        *out = (u128)v;
        return 0;
    }
    u128 mag = (u128)(uint64_t)(-(v + 1)) + 1;
    if (mag > half_down) return fail(ORC_DATA, "encode_signed: value below range");
    *out = b->P - mag;
    return 0;
}
static int64_t decode_signed(u128 x, const ocrt* b) {
    const u128 half_up = (b->P + 1) / 2;
    if (x < half_up) return (int64_t)x;
    return -(int64_t)(b->P - x);
}
static u128 crt_reconstruct(const uint16_t* r, const ocrt* b) {
    u128 acc = 0;
    for (int i = 0; i < b->k; ++i) acc += b->coeffs[i] % b->P * r[i] % b->P;
    return acc % b->P;
}
static int64_t max_signed(const ocrt* b) {
    u128 hi = (b->P + 1) / 2 - 1;
    return hi > (u128)INT64_MAX ? INT64_MAX : (int64_t)hi;
}
static int64_t min_signed(const ocrt* b) {
    u128 mag = b->P / 2;
    return mag > (u128)INT64_MAX ? INT64_MIN : -(int64_t)mag;
}

/* ===================== mixed radix (mixed_radix.cpp:59-235, gadgets.cpp:5-28) ===================== */

typedef struct {
    int t;
    int radices[32];
} ospec;

static u128 spec_M(const ospec* s) {
    u128 M = 1;
    for (int j = 0; j < s->t; ++j) M *= (u128)s->radices[j];
    return M;
}

/* exact floor((2·M·y + P) / (2P)) with a 256-bit numerator (mixed_radix.cpp:59-63) */
static u128 round_scaled(u128 M, u128 y, u128 P) {
    const u128 a = 2 * M, b = y;
    const u128 al = (uint64_t)a, ah = a >> 64, bl = (uint64_t)b, bh = b >> 64;
    const u128 ll = al * bl, lh = al * bh, hl = ah * bl, hh = ah * bh;
    u128 lo = ll + (lh << 64);
    u128 carry = lo < ll;
    u128 lo2 = lo + (hl << 64);
    carry += lo2 < lo;
    lo = lo2;
    u128 hi = hh + (lh >> 64) + (hl >> 64) + carry;
    u128 lo3 = lo + P;
    hi += lo3 < lo;
    lo = lo3;
    const u128 d = 2 * P;
    u128 q = 0, rem = 0;
    for (int i = 255; i >= 0; --i) {
        u128 bit = i >= 128 ? (hi >> (i - 128)) & 1 : (lo >> i) & 1;
        rem = (rem << 1) | bit;
        if (rem >= d) {
            rem -= d;
            if (i < 128) q |= (u128)1 << i;
        }
    }
    return q;
}

/* d_tables (mixed_radix.cpp:130-142) */
static void d_tables(const ocrt* b, u128 M, u128 d[MAXK][64]) {
    for (int i = 0; i < b->k; ++i) {
        const u128 alpha = b->coeffs[i] % b->P;
        for (int x = 0; x < b->primes[i]; ++x) d[i][x] = round_scaled(M, alpha * (u128)x % b->P, b->P) % M;
    }
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* measure_sign_accuracy (mixed_radix.cpp:214-235); returns correct/total */
static double sign_accuracy(const ocrt* b, const ospec* s) {
    const u128 M = spec_M(s);
    static __thread u128 d[MAXK][64];
    d_tables(b, M, d);
    uint64_t ok = 0, total;
    if (b->P <= ((u128)1 << 20)) {
        total = (uint64_t)b->P;
        for (u128 x = 0; x < b->P; ++x) {
            u128 sum = 0;
            for (int i = 0; i < b->k; ++i) sum += d[i][(int)(x % (u128)b->primes[i])];
            sum %= M;
            ok += ((2 * sum >= M) == (2 * x >= b->P));
        }
    } else {
        total = 100000;
        for (uint64_t i = 0; i < total; ++i) {
            u128 x = (((u128)splitmix64(2 * i) << 64) | splitmix64(2 * i + 1)) % b->P;
            u128 sum = 0;
            for (int j = 0; j < b->k; ++j) sum += d[j][(int)(x % (u128)b->primes[j])];
            sum %= M;
            ok += ((2 * sum >= M) == (2 * x >= b->P));
        }
    }
    return total ? (double)ok / (double)total : 0.0;
}

typedef struct {
    int found;
    u128 M;
    int t, m1;
    ospec spec;
} osearch;

/* consider / dfs (mixed_radix.cpp:84-125) */
static void consider(osearch* best, int m1, const int* tr, int nt, u128 bound) {
    u128 M = (u128)m1;
    for (int i = 0; i < nt; ++i) M *= (u128)tr[i];
    if (M <= bound) return;
    const int t = 1 + nt;
    int better = !best->found || M < best->M || (M == best->M && t < best->t) ||
                 (M == best->M && t == best->t && m1 > best->m1);
    if (!better) return;
    best->found = 1;
    best->M = M;
    best->t = t;
    best->m1 = m1;
    best->spec.t = t;
    best->spec.radices[0] = m1;
    for (int i = 0; i < nt; ++i) best->spec.radices[1 + i] = tr[i];
}
static void dfs(osearch* best, int* seq, int nseq, u128 q, int last, u128 bound, u128 qmax) {
    if (nseq > 0) {
        const u128 need = bound / q + 1;
        u128 m1 = need + (need & 1);
        if (m1 < 50) m1 = 50;
        if (m1 <= 128) consider(best, (int)m1, seq, nseq, bound);
    }
    for (int d = last < 8 ? last : 8; d >= 2; --d) {
        if (q * (u128)d <= qmax && nseq < 30) {
            seq[nseq] = d;
            dfs(best, seq, nseq + 1, q * (u128)d, d, bound, qmax);
        }
    }
}
static int choose_full(const ocrt* b, ospec* out) {
    const u128 bound = (u128)b->k * b->P / 2;
    osearch best;
    memset(&best, 0, sizeof best);
    for (int m1 = 2; m1 <= 128; m1 += 2) consider(&best, m1, NULL, 0, bound);
    u128 qmax = bound / 25 + 1;
    int seq[32];
    dfs(&best, seq, 0, 1, 8, bound, qmax);
    if (!best.found) return fail(ORC_DATA, "no mixed-radix spec reaches the required M");
    *out = best.spec;
    return 0;
}
/* mixed_radix.cpp:171-189 */
static int choose_spec(const ocrt* b, double target, ospec* out) {
    ospec cur;
    int rc = choose_full(b, &cur);
    if (rc) return rc;
    if (target >= 1.0) {
        *out = cur;
        return 0;
    }
    if (sign_accuracy(b, &cur) < target) {
        *out = cur;
        return 0;
    }
    ospec last = cur;
    for (;;) {
        ospec next = cur;
        if (next.t > 1)
            next.t--;
        else if (next.radices[0] > 2)
            next.radices[0] -= 2;
        else {
            *out = last;
            return 0;
        }
        if (sign_accuracy(b, &next) < target) {
            *out = last;
            return 0;
        }
        last = next;
        cur = next;
    }
}

typedef struct {
    int m, b_mod, carry_in, carry_out;
} opos;

typedef struct {
    ospec spec;
    int k;
    int npos;
    opos pos[32];
    int msd_carry;
    /* sign tables: digits[i][j][x] (mixed_radix.cpp:191-212) */
    uint16_t digits[MAXK][32][64];
} osign;

static int make_sign(const ocrt* b, const ospec* spec, osign* s) {
    memset(s, 0, sizeof *s);
    s->spec = *spec;
    s->k = b->k;
    const int t = spec->t;
    if (spec->radices[0] % 2) return fail(ORC_DATA, "mixed-radix m_1 must be even");
    if (b->k > 1 && t > 1) {
        int carry = 0;
        for (int j = t - 1; j >= 1; --j) {
            opos p;
            p.m = spec->radices[j];
            p.carry_in = carry;
            p.b_mod = b->k * (p.m - 1) + (carry ? carry - 1 : 0) + 1;
            if (p.b_mod > MAXM) return fail(ORC_DATA, "mixed-radix digit sum exceeds the modulus limit");
            const int maxcarry = (p.b_mod - 1) / p.m;
            p.carry_out = maxcarry > 0 ? maxcarry + 1 : 0;
            carry = p.carry_out;
            s->pos[s->npos++] = p;
        }
        s->msd_carry = carry;
    }
    const u128 M = spec_M(spec);
    static __thread u128 d[MAXK][64];
    d_tables(b, M, d);
    for (int i = 0; i < b->k; ++i)
        for (int x = 0; x < b->primes[i]; ++x) {
            u128 v = d[i][x];
            for (int j = t - 1; j >= 0; --j) {
                s->digits[i][j][x] = (uint16_t)(v % (u128)spec->radices[j]);
                v /= (u128)spec->radices[j];
            }
        }
    return 0;
}

/* ===================== gadget contexts (gadgets.hpp:20-98) ===================== */

enum { M_GARBLE = 0, M_EVAL = 1, M_COUNT = 2 };

typedef struct {
    olabel r[MAXM + 1];
    int present[MAXM + 1];
} ooffsets;

typedef struct {
    int mode;
    /* garble */
    const oprf* prf;
    const ooffsets* offs;
    u128* out;
    uint64_t out_pos;
    uint64_t next_gate, next_wire;
    /* eval */
    const u128* in;
    uint64_t in_len, in_pos;
    int err;
    /* count */
    uint64_t cts, gates, wires;
    int moduli[MAXM + 1];
} octx;

static uint64_t cgate(octx* c) {
    if (c->mode == M_COUNT) return c->gates++;
    return c->next_gate++;
}
static olabel cfresh(octx* c, int m) {
    if (c->mode == M_COUNT) {
        c->wires++;
        c->moduli[m] = 1;
        return lzeros(m);
    }
    return prf_label(c->prf, c->next_wire++, m);
}
static const olabel* coffset(octx* c, int m) {
    if (c->mode == M_COUNT) {
        c->moduli[m] = 1;
        return NULL;
    }
    return &c->offs->r[m];
}
static void cemit(octx* c, u128 ct) { c->out[c->out_pos++] = ct; }
static const u128* ctake(octx* c, uint64_t n) {
    static const u128 zero[256] = {0};
    if (c->in_pos + n > c->in_len) {
        c->err = ORC_DATA;
        return zero;
    }
    const u128* p = c->in + c->in_pos;
    c->in_pos += n;
    return p;
}

/* phi functions of the gadget call sites */
enum {
    PHI_TABLE,    /* sign-table digit (gadgets.hpp:453-457) */
    PHI_LIFT,     /* identity cast (gadgets.hpp:398) */
    PHI_DIV,      /* carry a / m (gadgets.hpp:415-418) */
    PHI_MOD,      /* c % m1 (gadgets.hpp:430-432) */
    PHI_GE,       /* s >= half (gadgets.hpp:464-466) */
    PHI_NONZERO,  /* a != 0 (gadgets.hpp:469-471) */
    PHI_GE1,      /* c >= 1 (gadgets.hpp:477-479) */
    PHI_SIGNACT,  /* b != 0 ? 1 : p-1 (layer.cpp:231-233) */
    PHI_WMUL      /* w·a mod p (layer.cpp:203-206) */
};
typedef struct {
    int kind;
    int param;
    const uint16_t* table;
} ophi;
static uint32_t phi_eval(const ophi* f, int a) {
    switch (f->kind) {
        case PHI_TABLE: return f->table[a];
        case PHI_LIFT: return (uint32_t)a;
        case PHI_DIV: return (uint32_t)(a / f->param);
        case PHI_MOD: return (uint32_t)(a % f->param);
        case PHI_GE: return a >= f->param ? 1u : 0u;
        case PHI_NONZERO: return a != 0;
        case PHI_GE1: return a >= 1;
        case PHI_SIGNACT: return a != 0 ? 1u : (uint32_t)(f->param - 1);
        case PHI_WMUL: return (uint32_t)(f->param * a) % (uint32_t)f->table[0];
    }
    return 0;
}

/* add_public_constant (gadgets.hpp:127-139) */
static olabel g_add_const(octx* c, const olabel* l, int cst) {
    if (c->mode == M_GARBLE) {
        if (cst % l->m == 0) return *l;
        olabel s = lscale(c->offs->r[l->m], (uint32_t)(cst % l->m));
        return lsub(*l, &s);
    }
    if (c->mode == M_COUNT) coffset(c, l->m);
    return *l;
}

/* t_proj (gadgets.hpp:146-176) */
static olabel g_proj(octx* c, const olabel* in, int q, const ophi* phi) {
    const uint64_t g = cgate(c);
    const int p = in->m;
    if (c->mode == M_GARBLE) {
        const olabel* rp = coffset(c, p);
        const olabel* rq = coffset(c, q);
        const olabel out0 = cfresh(c, q);
        u128 rows[MAXM];
        olabel key = *in;
        for (int a = 0; a < p; ++a) {
            const int row = (color(in) + a) % p;
            olabel sc = lscale(*rq, phi_eval(phi, a) % (uint32_t)q);
            olabel payload = ladd(out0, &sc);
            rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 0), &payload);
            ladd_into(&key, rp);
        }
        for (int row = 0; row < p; ++row) cemit(c, rows[row]);
        return out0;
    }
    if (c->mode == M_EVAL) {
        const u128* rows = ctake(c, (uint64_t)p);
        const int row = color(in);
        return decrypt_label(in, tweak(g, (uint32_t)row, 0), rows[row], q);
    }
    c->cts += (uint64_t)p;
    coffset(c, p);
    return cfresh(c, q);
}

/* t_proj_grr (gadgets.hpp:181-221) */
static olabel g_proj_grr(octx* c, const olabel* in, int q, const ophi* phi) {
    const uint64_t g = cgate(c);
    const int p = in->m;
    if (c->mode == M_GARBLE) {
        const olabel* rp = coffset(c, p);
        const olabel* rq = coffset(c, q);
        const int a0 = (p - color(in)) % p;
        olabel s0 = lscale(*rp, (uint32_t)a0);
        olabel key0 = ladd(*in, &s0);
        olabel pad0 = pad_label(&key0, tweak(g, 0, 0), q);
        olabel sc0 = lscale(*rq, phi_eval(phi, a0) % (uint32_t)q);
        olabel out0 = lsub(lneg(pad0), &sc0);
        u128 rows[MAXM];
        olabel key = *in;
        for (int a = 0; a < p; ++a) {
            const int row = (color(in) + a) % p;
            if (row != 0) {
                olabel sc = lscale(*rq, phi_eval(phi, a) % (uint32_t)q);
                olabel payload = ladd(out0, &sc);
                rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 0), &payload);
            }
            ladd_into(&key, rp);
        }
        for (int row = 1; row < p; ++row) cemit(c, rows[row]);
        return out0;
    }
    if (c->mode == M_EVAL) {
        const u128* rows = ctake(c, (uint64_t)(p - 1));
        const int row = color(in);
        const u128 ct = row == 0 ? 0 : rows[row - 1];
        return decrypt_label(in, tweak(g, (uint32_t)row, 0), ct, q);
    }
    c->cts += (uint64_t)(p - 1);
    coffset(c, p);
    coffset(c, q);
    return lzeros(q);
}

/* t_half_gate (gadgets.hpp:230-282) */
static olabel g_half(octx* c, const olabel* x, const olabel* y) {
    const uint64_t g = cgate(c);
    const int p = x->m;
    if (c->mode == M_GARBLE) {
        const olabel* rp = coffset(c, p);
        const olabel u0 = cfresh(c, p);
        const olabel v0 = cfresh(c, p);
        const int r = color(y);
        u128 rows[MAXM];
        olabel key = *x;
        for (int a = 0; a < p; ++a) {
            const int row = (color(x) + a) % p;
            olabel sc = lscale(*rp, (uint32_t)(a * r % p));
            olabel payload = ladd(u0, &sc);
            rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 0), &payload);
            ladd_into(&key, rp);
        }
        for (int row = 0; row < p; ++row) cemit(c, rows[row]);
        key = *y;
        for (int b = 0; b < p; ++b) {
            const int row = (r + b) % p;
            olabel sx = lscale(*x, (uint32_t)row);
            olabel payload = lsub(v0, &sx);
            rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 1), &payload);
            ladd_into(&key, rp);
        }
        for (int row = 0; row < p; ++row) cemit(c, rows[row]);
        return lsub(v0, &u0);
    }
    if (c->mode == M_EVAL) {
        const u128* gr = ctake(c, (uint64_t)p);
        const u128* er = ctake(c, (uint64_t)p);
        const int cx = color(x), cy = color(y);
        olabel u = decrypt_label(x, tweak(g, (uint32_t)cx, 0), gr[cx], p);
        olabel out = decrypt_label(y, tweak(g, (uint32_t)cy, 1), er[cy], p);
        ladd_scaled(&out, x, (uint32_t)cy);
        lsub_into(&out, &u);
        return out;
    }
    c->cts += 2u * (uint64_t)p;
    coffset(c, p);
    cfresh(c, p);
    return cfresh(c, p);
}

/* t_mm_half_gate (gadgets.hpp:292-358) */
static olabel g_mm_half(octx* c, const olabel* x, const olabel* y) {
    const int p = x->m, q = y->m;
    const uint64_t g = cgate(c);
    if (c->mode == M_GARBLE) {
        const olabel* rp = coffset(c, p);
        const olabel* rq = coffset(c, q);
        const olabel u0 = cfresh(c, p);
        const olabel v0 = cfresh(c, p);
        const int r = color(x);
        u128 rows[MAXM];
        olabel key = *x;
        for (int a = 0; a < p; ++a) {
            const int row = (color(x) + a) % p;
            olabel sc = lscale(*rp, (uint32_t)(a * r % p));
            olabel payload = ladd(u0, &sc);
            rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 0), &payload);
            ladd_into(&key, rp);
        }
        for (int row = 0; row < p; ++row) cemit(c, rows[row]);
        static __thread olabel fkeys[MAXM];
        uint16_t fvals[MAXM];
        key = *y;
        for (int b = 0; b < q; ++b) {
            const int row = (color(y) + b) % q;
            const int s = (r + b) % p;
            olabel sx = lscale(*x, (uint32_t)s);
            olabel payload = lsub(v0, &sx);
            rows[row] = encrypt_label(&key, tweak(g, (uint32_t)row, 1), &payload);
            fkeys[row] = key;
            fvals[row] = (uint16_t)s;
            ladd_into(&key, rq);
        }
        for (int row = 0; row < q; ++row) cemit(c, rows[row]);
        cemit(c, encrypt_short(fkeys, tweak(g, 0, 2), fvals, q, p));
        return lsub(v0, &u0);
    }
    if (c->mode == M_EVAL) {
        const u128* gr = ctake(c, (uint64_t)p);
        const u128* er = ctake(c, (uint64_t)q);
        const u128 sb = *ctake(c, 1);
        const int cx = color(x), cy = color(y);
        olabel u = decrypt_label(x, tweak(g, (uint32_t)cx, 0), gr[cx], p);
        olabel out = decrypt_label(y, tweak(g, (uint32_t)cy, 1), er[cy], p);
        const int s = decrypt_short(y, tweak(g, 0, 2), sb, cy, p);
        ladd_scaled(&out, x, (uint32_t)s);
        lsub_into(&out, &u);
        return out;
    }
    c->cts += (uint64_t)p + (uint64_t)q + 1;
    coffset(c, p);
    coffset(c, q);
    cfresh(c, p);
    return cfresh(c, p);
}

/* t_mixed_radix_add (gadgets.hpp:382-435); bundles[s*t + j] */
static olabel g_mixed_radix_add(octx* c, const olabel* bundles, const osign* s) {
    const int k = s->k, t = s->spec.t;
    if (k == 1) return bundles[0];
    olabel carry;
    int carry_mod = 0;
    const ophi lift = {PHI_LIFT, 0, NULL};
    for (int i = 0; i < s->npos; ++i) {
        const opos* pos = &s->pos[i];
        const int j = t - 1 - i;
        olabel sum = g_proj(c, &bundles[0 * t + j], pos->b_mod, &lift);
        for (int r = 1; r < k; ++r) {
            olabel term = g_proj(c, &bundles[r * t + j], pos->b_mod, &lift);
            ladd_into(&sum, &term);
        }
        if (pos->carry_in) {
            olabel term = g_proj(c, &carry, pos->b_mod, &lift);
            ladd_into(&sum, &term);
        }
        if (pos->carry_out) {
            const ophi div = {PHI_DIV, pos->m, NULL};
            carry = g_proj(c, &sum, pos->carry_out, &div);
            carry_mod = pos->carry_out;
        } else {
            carry_mod = 0;
        }
    }
    (void)carry_mod;
    const int m1 = s->spec.radices[0];
    olabel msd = bundles[0];
    for (int r = 1; r < k; ++r) ladd_into(&msd, &bundles[r * t]);
    if (s->msd_carry) {
        const ophi mod = {PHI_MOD, m1, NULL};
        olabel term = g_proj(c, &carry, m1, &mod);
        ladd_into(&msd, &term);
    }
    return msd;
}

/* t_approx_sign_bit (gadgets.hpp:442-481) */
static olabel g_sign_bit(octx* c, const olabel* x, const ocrt* b, const osign* s) {
    const int k = b->k, t = s->spec.t;
    olabel* bundles = (olabel*)malloc(sizeof(olabel) * (size_t)(k * t));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < t; ++j) {
            const ophi tab = {PHI_TABLE, 0, s->digits[i][j]};
            bundles[i * t + j] = g_proj(c, &x[i], s->spec.radices[j], &tab);
        }
    const olabel msd = g_mixed_radix_add(c, bundles, s);
    free(bundles);
    const int m1 = s->spec.radices[0];
    const ophi ge = {PHI_GE, m1 / 2, NULL};
    const olabel negative = g_proj_grr(c, &msd, 2, &ge);
    const olabel nonneg = g_add_const(c, &negative, 1);
    const ophi nzf = {PHI_NONZERO, 0, NULL};
    olabel count = g_proj(c, &x[0], k + 1, &nzf);
    for (int i = 1; i < k; ++i) {
        olabel nz = g_proj(c, &x[i], k + 1, &nzf);
        ladd_into(&count, &nz);
    }
    const ophi ge1 = {PHI_GE1, 0, NULL};
    const olabel nonzero = g_proj(c, &count, 2, &ge1);
    return g_half(c, &nonneg, &nonzero);
}

/* relu_element / sign_act_element (layer.cpp:214-236) */
static void g_act_element(octx* c, int kind, const olabel* in, olabel* out, const ocrt* b,
                          const osign* s) {
    const olabel bit = g_sign_bit(c, in, b, s);
    for (int i = 0; i < b->k; ++i) {
        if (kind == DASH_LAYER_RELU) {
            out[i] = g_mm_half(c, &in[i], &bit);
        } else {
            const ophi sa = {PHI_SIGNACT, b->primes[i], NULL};
            out[i] = g_proj(c, &bit, b->primes[i], &sa);
        }
    }
}

/* ===================== layers (layer.cpp) ===================== */

#define ORC_MAXL 256 /* layers per circuit (ResNet-20 with extensions: 71) */

typedef struct {
    int kind, priv;
    uint32_t in_dim, out_dim, in_ch, out_ch, filter, stride;
    int src, src2; /* extension: DAG inputs (dash_circuit_desc.h) */
    uint32_t pad;  /* extension: PAD2D */
    int64_t* w;
    uint64_t nw;
    int64_t* bias;
    uint64_t nb;
} olayer;

struct orc_circuit {
    int k;
    int rank;
    uint32_t shape[8];
    double sign_target, alpha;
    int nl;
    olayer* layers;
    /* derived: shapes[0] = input, shapes[j + 1] = output of layer j;
     * ishapes[j] = input of layer j (from its DAG source) */
    uint32_t shapes[ORC_MAXL + 1][8];
    int ranks[ORC_MAXL + 1];
    uint32_t ishapes[ORC_MAXL][8];
    int iranks[ORC_MAXL];
};

/* index into shapes[] / the per-layer value list of a layer's DAG source:
 * src 0 = previous layer (the reference's chain), j + 1 = layer j, -1 = input */
static int src_index(int li, int src) { return src == 0 ? li : (src < 0 ? 0 : src); }

typedef struct {
    int n; /* elements */
    int m;
    olabel* l;
} otensor;

static uint64_t shape_size(const uint32_t* s, int r) {
    uint64_t n = 1;
    for (int i = 0; i < r; ++i) n *= s[i];
    return n;
}

static int conv_extent(uint32_t in, uint32_t f, uint32_t s, uint32_t* out) {
    if (f == 0 || s == 0 || f > in) return fail(ORC_DATA, "convolution filter does not fit the input");
    *out = (in - f) / s + 1;
    return 0;
}

/* layer_out_shape (layer.cpp:320-344) */
static int out_shape(const olayer* l, const uint32_t* in, int rin, uint32_t* out, int* rout) {
    switch (l->kind) {
        case DASH_LAYER_DENSE:
            if (rin != 1 || in[0] != l->in_dim) return fail(ORC_DATA, "dense layer input shape mismatch");
            out[0] = l->out_dim;
            *rout = 1;
            return 0;
        case DASH_LAYER_CONV2D: {
            if (rin != 3 || in[0] != l->in_ch) return fail(ORC_DATA, "conv layer input shape mismatch");
            uint32_t oh, ow;
            if (conv_extent(in[1], l->filter, l->stride, &oh) || conv_extent(in[2], l->filter, l->stride, &ow))
                return ORC_DATA;
            out[0] = l->out_ch;
            out[1] = oh;
            out[2] = ow;
            *rout = 3;
            return 0;
        }
        case DASH_LAYER_RELU:
        case DASH_LAYER_SIGNACT:
        case DASH_LAYER_ADD:
            memcpy(out, in, sizeof(uint32_t) * (size_t)rin);
            *rout = rin;
            return 0;
        case DASH_LAYER_PAD2D:
            if (rin != 3) return fail(ORC_DATA, "pad layer needs a [C][H][W] input");
            out[0] = in[0];
            out[1] = in[1] + 2 * l->pad;
            out[2] = in[2] + 2 * l->pad;
            *rout = 3;
            return 0;
        case DASH_LAYER_FLATTEN:
            out[0] = (uint32_t)shape_size(in, rin);
            *rout = 1;
            return 0;
    }
    return fail(ORC_DATA, "unknown layer kind");
}

static uint64_t wcount(const olayer* l) {
    if (l->kind == DASH_LAYER_DENSE) return (uint64_t)l->in_dim * l->out_dim;
    if (l->kind == DASH_LAYER_CONV2D) return (uint64_t)l->out_ch * l->in_ch * l->filter * l->filter;
    return 0;
}
static uint64_t bcount(const olayer* l) {
    if (l->kind == DASH_LAYER_DENSE) return l->out_dim;
    if (l->kind == DASH_LAYER_CONV2D) return l->out_ch;
    return 0;
}
static int is_linear(const olayer* l) { return l->kind == DASH_LAYER_DENSE || l->kind == DASH_LAYER_CONV2D; }

int orc_circuit_new(const dash_circuit_desc* d, orc_circuit** out) {
    mi_init();
    if (d->k < 1 || d->k > MAXK) return fail(ORC_DATA, "CRT base size out of range");
    if (d->rank < 1 || d->rank > 8 || d->n_layers > ORC_MAXL) return fail(ORC_DATA, "bad circuit shape");
    orc_circuit* c = (orc_circuit*)calloc(1, sizeof *c);
    c->k = d->k;
    c->rank = (int)d->rank;
    memcpy(c->shape, d->input_shape, sizeof c->shape);
    c->sign_target = d->sign_target;
    c->alpha = d->alpha;
    c->nl = (int)d->n_layers;
    c->layers = (olayer*)calloc((size_t)c->nl + 1, sizeof(olayer));
    memcpy(c->shapes[0], c->shape, sizeof c->shape);
    c->ranks[0] = c->rank;
    if (shape_size(c->shape, c->rank) == 0) {
        orc_circuit_free(c);
        return fail(ORC_DATA, "circuit has an empty input shape");
    }
    for (int i = 0; i < c->nl; ++i) {
        const dash_layer_desc* s = &d->layers[i];
        olayer* l = &c->layers[i];
        l->kind = s->kind;
        l->priv = s->private_weights;
        l->in_dim = s->in_dim;
        l->out_dim = s->out_dim;
        l->in_ch = s->in_ch;
        l->out_ch = s->out_ch;
        l->filter = s->filter;
        l->stride = s->stride;
        l->src = s->src;
        l->src2 = s->src2;
        l->pad = s->pad;
        if (l->src > i || l->src < -1 || l->src2 > i || l->src2 < -1 ||
            (l->kind == DASH_LAYER_ADD && l->src2 == 0)) {
            orc_circuit_free(c);
            return fail(ORC_DATA, "layer input refers to a later layer");
        }
        if (s->q_weights && s->n_weights) {
            l->nw = s->n_weights;
            l->w = (int64_t*)malloc(sizeof(int64_t) * l->nw);
            memcpy(l->w, s->q_weights, sizeof(int64_t) * l->nw);
        }
        if (s->q_biases && s->n_biases) {
            l->nb = s->n_biases;
            l->bias = (int64_t*)malloc(sizeof(int64_t) * l->nb);
            memcpy(l->bias, s->q_biases, sizeof(int64_t) * l->nb);
        }
        const int si = src_index(i, l->src);
        memcpy(c->ishapes[i], c->shapes[si], sizeof c->ishapes[i]);
        c->iranks[i] = c->ranks[si];
        int rc = out_shape(l, c->ishapes[i], c->iranks[i], c->shapes[i + 1], &c->ranks[i + 1]);
        if (!rc && l->kind == DASH_LAYER_ADD) {
            const int s2 = src_index(i, l->src2);
            if (c->ranks[s2] != c->iranks[i] ||
                memcmp(c->shapes[s2], c->ishapes[i], sizeof(uint32_t) * (size_t)c->iranks[i]))
                rc = fail(ORC_DATA, "add operands differ in shape");
        }
        if (rc) {
            orc_circuit_free(c);
            return rc;
        }
        if (is_linear(l) && ((l->nw && l->nw != wcount(l)) || (l->nb && l->nb != bcount(l)))) {
            orc_circuit_free(c);
            return fail(ORC_DATA, "quantized weight count mismatch");
        }
    }
    *out = c;
    return 0;
}

void orc_circuit_free(orc_circuit* c) {
    if (!c) return;
    for (int i = 0; i < c->nl; ++i) {
        free(c->layers[i].w);
        free(c->layers[i].bias);
    }
    free(c->layers);
    free(c);
}

int orc_circuit_io(const orc_circuit* c, uint64_t* n_in, uint64_t* n_out) {
    *n_in = shape_size(c->shapes[0], c->ranks[0]);
    *n_out = shape_size(c->shapes[c->nl], c->ranks[c->nl]);
    return 0;
}

static int circuit_needs_sign(const orc_circuit* c) {
    for (int i = 0; i < c->nl; ++i)
        if (c->layers[i].kind == DASH_LAYER_RELU || c->layers[i].kind == DASH_LAYER_SIGNACT) return 1;
    return 0;
}

/* plain_forward (layer.cpp:346-376, 56-109), plus the Pad2d / Add / DAG
 * extensions (pad cells are 0, add is the integer sum) */
int orc_plain_forward(const orc_circuit* c, const int64_t* in, int64_t* out) {
    const ocrt b = crt_base(c->k);
    const int64_t hi = max_signed(&b), lo = min_signed(&b);
    int64_t* vals[ORC_MAXL + 1] = {0};
    uint64_t n0 = shape_size(c->shapes[0], c->ranks[0]);
    vals[0] = (int64_t*)malloc(sizeof(int64_t) * n0);
    memcpy(vals[0], in, sizeof(int64_t) * n0);
    int rc = 0;
    for (int li = 0; li < c->nl && !rc; ++li) {
        const olayer* l = &c->layers[li];
        const uint32_t* s = c->ishapes[li];
        const int64_t* x = vals[src_index(li, l->src)];
        const uint64_t no = shape_size(c->shapes[li + 1], c->ranks[li + 1]);
        int64_t* y = (int64_t*)malloc(sizeof(int64_t) * (no ? no : 1));
        vals[li + 1] = y;
        if (l->kind == DASH_LAYER_DENSE || l->kind == DASH_LAYER_CONV2D) {
            for (uint64_t u = 0; u < no; ++u) {
                __int128 acc;
                if (l->kind == DASH_LAYER_DENSE) {
                    acc = l->nb ? l->bias[u] : 0;
                    for (uint32_t i = 0; i < l->in_dim; ++i) acc += (__int128)l->w[u * l->in_dim + i] * x[i];
                } else {
                    const uint32_t h = s[1], w = s[2], oh = c->shapes[li + 1][1], ow = c->shapes[li + 1][2];
                    const uint32_t oc = (uint32_t)(u / ((uint64_t)oh * ow)), oy = (uint32_t)((u / ow) % oh),
                                   ox = (uint32_t)(u % ow);
                    acc = l->nb ? l->bias[oc] : 0;
                    for (uint32_t ic = 0; ic < l->in_ch; ++ic)
                        for (uint32_t ky = 0; ky < l->filter; ++ky)
                            for (uint32_t kx = 0; kx < l->filter; ++kx) {
                                const uint64_t wi = (((uint64_t)oc * l->in_ch + ic) * l->filter + ky) * l->filter + kx;
                                const uint64_t xi = ((uint64_t)ic * h + (oy * l->stride + ky)) * w + (ox * l->stride + kx);
                                acc += (__int128)l->w[wi] * x[xi];
                            }
                }
                if (acc > INT64_MAX || acc < INT64_MIN || (int64_t)acc > hi || (int64_t)acc < lo) {
                    rc = fail(ORC_OVERFLOW, "intermediate value left the signed range of the base");
                    break;
                }
                y[u] = (int64_t)acc;
            }
        } else if (l->kind == DASH_LAYER_PAD2D) {
            const uint32_t H = s[1], W = s[2], OH = H + 2 * l->pad, OW = W + 2 * l->pad;
            for (uint64_t u = 0; u < no; ++u) {
                const uint64_t ch = u / ((uint64_t)OH * OW);
                const uint32_t y0 = (uint32_t)((u / OW) % OH), x0 = (uint32_t)(u % OW);
                const int inside = y0 >= l->pad && y0 < l->pad + H && x0 >= l->pad && x0 < l->pad + W;
                y[u] = inside ? x[(ch * H + (y0 - l->pad)) * W + (x0 - l->pad)] : 0;
            }
        } else if (l->kind == DASH_LAYER_ADD) {
            const int64_t* x2 = vals[src_index(li, l->src2)];
            for (uint64_t u = 0; u < no; ++u) {
                const __int128 acc = (__int128)x[u] + x2[u];
                if (acc > hi || acc < lo) {
                    rc = fail(ORC_OVERFLOW, "intermediate value left the signed range of the base");
                    break;
                }
                y[u] = (int64_t)acc;
            }
        } else {
            for (uint64_t u = 0; u < no; ++u) {
                if (l->kind == DASH_LAYER_RELU) y[u] = x[u] > 0 ? x[u] : 0;
                else if (l->kind == DASH_LAYER_SIGNACT) y[u] = x[u] > 0 ? 1 : -1;
                else y[u] = x[u];
            }
        }
    }
    if (!rc) memcpy(out, vals[c->nl], sizeof(int64_t) * shape_size(c->shapes[c->nl], c->ranks[c->nl]));
    for (int i = 0; i <= c->nl; ++i) free(vals[i]);
    return rc;
}

/* env shared by the layer runners (layer.hpp:67-75) */
typedef struct {
    ocrt base;
    osign* sign; /* NULL when no activation layers */
    olabel zeros[MAXK];
    const oprf* prf;
    const ooffsets* offs;
} oenv;

typedef struct {
    uint64_t cts, gates, wires;
} ocost;

/* element_unit_cost (layer.cpp:239-256) */
static ocost element_cost(int kind, const oenv* e, int* moduli) {
    octx c;
    memset(&c, 0, sizeof c);
    c.mode = M_COUNT;
    olabel in[MAXK], out[MAXK];
    for (int i = 0; i < e->base.k; ++i) in[i] = lzeros(e->base.primes[i]);
    g_act_element(&c, kind, in, out, &e->base, e->sign);
    if (moduli)
        for (int m = 0; m <= MAXM; ++m)
            if (c.moduli[m]) moduli[m] = 1;
    ocost r = {c.cts, c.gates, c.wires};
    return r;
}

static uint64_t private_window(const olayer* l) {
    return l->kind == DASH_LAYER_DENSE ? l->in_dim : (uint64_t)l->in_ch * l->filter * l->filter;
}

/* count_layer (layer.cpp:378-412) */
static void count_layer(const orc_circuit* c, int li, const oenv* e, octx* ctx) {
    const olayer* l = &c->layers[li];
    const uint64_t units = shape_size(c->shapes[li + 1], c->ranks[li + 1]);
    switch (l->kind) {
        case DASH_LAYER_FLATTEN:
        case DASH_LAYER_PAD2D:
        case DASH_LAYER_ADD: return; /* free: no gates, wires or rows */
        case DASH_LAYER_DENSE:
        case DASH_LAYER_CONV2D:
            for (int i = 0; i < e->base.k; ++i) {
                const int p = e->base.primes[i];
                ctx->moduli[p] = 1;
                if (l->priv) {
                    const uint64_t win = private_window(l);
                    ctx->cts += win * (uint64_t)p * units;
                    ctx->gates += win * units;
                    ctx->wires += win * units;
                }
            }
            return;
        default: {
            const ocost uc = element_cost(l->kind, e, ctx->moduli);
            ctx->cts += uc.cts * units;
            ctx->gates += uc.gates * units;
            ctx->wires += uc.wires * units;
        }
    }
}

static int64_t resid(int64_t w, int p) { return ((w % p) + p) % p; }

/* linear_public_lane (layer.cpp:122-191) */
static void linear_lane(const orc_circuit* c, int li, const otensor* in, otensor* out, const olabel* zero,
                        int p, int garbler, const ooffsets* offs) {
    const olayer* l = &c->layers[li];
    const uint32_t* s = c->ishapes[li];
    const int dense = l->kind == DASH_LAYER_DENSE;
    const uint64_t units = (uint64_t)out->n;
    const uint32_t oh = dense ? 0 : c->shapes[li + 1][1], ow = dense ? 0 : c->shapes[li + 1][2];
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)units; ++u) {
        uint32_t acc[MAXD] = {0};
        uint32_t zt = 0;
        int64_t bias = 0;
        const int n = in->l[0].n;
        if (dense) {
            for (uint32_t i = 0; i < l->in_dim; ++i) {
                const uint32_t wv = (uint32_t)resid(l->w[(uint64_t)u * l->in_dim + i], p);
                if (wv == 0) ++zt;
                else for (int d = 0; d < n; ++d) acc[d] += wv * in->l[i].d[d];
            }
            if (l->nb) bias = l->bias[u];
        } else {
            const uint32_t oc = (uint32_t)(u / ((uint64_t)oh * ow)), oy = (uint32_t)((u / ow) % oh), ox = (uint32_t)(u % ow);
            for (uint32_t ic = 0; ic < l->in_ch; ++ic)
                for (uint32_t ky = 0; ky < l->filter; ++ky)
                    for (uint32_t kx = 0; kx < l->filter; ++kx) {
                        const uint64_t wi = (((uint64_t)oc * l->in_ch + ic) * l->filter + ky) * l->filter + kx;
                        const uint64_t xi = ((uint64_t)ic * s[1] + (oy * l->stride + ky)) * s[2] + (ox * l->stride + kx);
                        const uint32_t wv = (uint32_t)resid(l->w[wi], p);
                        if (wv == 0) ++zt;
                        else for (int d = 0; d < n; ++d) acc[d] += wv * in->l[xi].d[d];
                    }
            if (l->nb) bias = l->bias[oc];
        }
        olabel sum = lshape(p);
        for (int d = 0; d < n; ++d) sum.d[d] = (uint16_t)(acc[d] % (uint32_t)p);
        if (zt) ladd_scaled(&sum, zero, zt % (uint32_t)p);
        if (garbler) {
            const int64_t b = resid(bias, p);
            if (b) {
                olabel sb = lscale(offs->r[p], (uint32_t)b);
                lsub_into(&sum, &sb);
            }
        }
        out->l[u] = sum;
    }
}

static otensor tnew(int m, uint64_t n) {
    otensor t;
    t.n = (int)n;
    t.m = m;
    t.l = (olabel*)malloc(sizeof(olabel) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) t.l[i] = lzeros(m);
    return t;
}
static void tfree(otensor* t) {
    free(t->l);
    t->l = NULL;
}

/* run_layer<Garble> (layer.cpp:419-551).  garble: blob = output position (already
 * sized); eval: blob = this layer's ciphertext span. */
static int run_layer(const orc_circuit* c, int li, const oenv* e, int garble, uint64_t gate_base,
                     uint64_t wire_base, u128* blob, uint64_t blob_len, const otensor* in /* k lanes */,
                     const otensor* in2 /* ADD: second operand */, otensor* out /* k lanes */) {
    const olayer* l = &c->layers[li];
    const int k = e->base.k;
    const uint64_t units = shape_size(c->shapes[li + 1], c->ranks[li + 1]);
    for (int i = 0; i < k; ++i) out[i] = tnew(e->base.primes[i], units);
    if (l->kind == DASH_LAYER_FLATTEN) {
        for (int i = 0; i < k; ++i) memcpy(out[i].l, in[i].l, sizeof(olabel) * units);
        return 0;
    }
    if (l->kind == DASH_LAYER_PAD2D) { /* extension: pad cells = zero-wire label */
        const uint32_t H = c->ishapes[li][1], W = c->ishapes[li][2], OH = H + 2 * l->pad, OW = W + 2 * l->pad;
        for (int i = 0; i < k; ++i)
            for (uint64_t u = 0; u < units; ++u) {
                const uint64_t ch = u / ((uint64_t)OH * OW);
                const uint32_t y = (uint32_t)((u / OW) % OH), x = (uint32_t)(u % OW);
                const int inside = y >= l->pad && y < l->pad + H && x >= l->pad && x < l->pad + W;
                out[i].l[u] = inside ? in[i].l[(ch * H + (y - l->pad)) * W + (x - l->pad)] : e->zeros[i];
            }
        return 0;
    }
    if (l->kind == DASH_LAYER_ADD) { /* extension: lane-wise label sum (free_add) */
        for (int i = 0; i < k; ++i)
            for (uint64_t u = 0; u < units; ++u) {
                out[i].l[u] = in[i].l[u];
                ladd_into(&out[i].l[u], &in2[i].l[u]);
            }
        return 0;
    }
    if (is_linear(l) && !l->priv) {
        for (int i = 0; i < k; ++i)
            linear_lane(c, li, &in[i], &out[i], &e->zeros[i], e->base.primes[i], garble, e->offs);
        return 0;
    }
    int err = 0;
    if (is_linear(l)) { /* private weights (layer.cpp:456-507) */
        const uint64_t win = private_window(l);
        uint64_t ct_off = 0, gate_off = 0, wire_off = 0;
        for (int i = 0; i < k; ++i) {
            const int p = e->base.primes[i];
            const ocost uc = {win * (uint64_t)p, win, win};
#pragma omp parallel for schedule(static)
            for (int64_t u = 0; u < (int64_t)units; ++u) {
                octx cx;
                memset(&cx, 0, sizeof cx);
                cx.mode = garble ? M_GARBLE : M_EVAL;
                cx.prf = e->prf;
                cx.offs = e->offs;
                cx.next_gate = gate_base + gate_off + (uint64_t)u * uc.gates;
                cx.next_wire = wire_base + wire_off + (uint64_t)u * uc.wires;
                if (garble) {
                    cx.out = blob + ct_off + (uint64_t)u * uc.cts;
                } else {
                    cx.in = blob + ct_off + (uint64_t)u * uc.cts;
                    cx.in_len = (ct_off + (uint64_t)(u + 1) * uc.cts <= blob_len) ? uc.cts : 0;
                }
                /* collect_private_unit (layer.cpp:271-316) */
                olabel sum;
                int64_t bias = 0;
                uint64_t oc = 0, oy = 0, ox = 0;
                if (l->kind == DASH_LAYER_CONV2D) {
                    const uint32_t oh = c->shapes[li + 1][1], ow = c->shapes[li + 1][2];
                    oc = (uint64_t)u / ((uint64_t)oh * ow);
                    oy = ((uint64_t)u / ow) % oh;
                    ox = (uint64_t)u % ow;
                }
                for (uint64_t j = 0; j < win; ++j) {
                    uint64_t xi, wi;
                    if (l->kind == DASH_LAYER_DENSE) {
                        xi = j;
                        wi = (uint64_t)u * l->in_dim + j;
                    } else {
                        const uint64_t ic = j / ((uint64_t)l->filter * l->filter);
                        const uint64_t ky = (j / l->filter) % l->filter, kx = j % l->filter;
                        wi = ((oc * l->in_ch + ic) * l->filter + ky) * l->filter + kx;
                        xi = (ic * c->ishapes[li][1] + (oy * l->stride + ky)) * c->ishapes[li][2] + (ox * l->stride + kx);
                    }
                    const uint16_t pm = (uint16_t)p;
                    const ophi wm = {PHI_WMUL, l->nw ? (int)resid(l->w[wi], p) : 0, &pm};
                    olabel term = g_proj(&cx, &in[i].l[xi], p, &wm);
                    if (j == 0) sum = term;
                    else ladd_into(&sum, &term);
                }
                if (l->nb) bias = l->bias[l->kind == DASH_LAYER_DENSE ? (uint64_t)u : oc];
                out[i].l[u] = g_add_const(&cx, &sum, (int)resid(bias, p));
                if (cx.err) err = cx.err;
            }
            ct_off += uc.cts * units;
            gate_off += uc.gates * units;
            wire_off += uc.wires * units;
        }
        return err ? fail(ORC_DATA, "ciphertext stream exhausted") : 0;
    }
    /* ReLU / SignAct */
    const ocost uc = element_cost(l->kind, e, NULL);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)units; ++u) {
        octx cx;
        memset(&cx, 0, sizeof cx);
        cx.mode = garble ? M_GARBLE : M_EVAL;
        cx.prf = e->prf;
        cx.offs = e->offs;
        cx.next_gate = gate_base + (uint64_t)u * uc.gates;
        cx.next_wire = wire_base + (uint64_t)u * uc.wires;
        if (garble) cx.out = blob + (uint64_t)u * uc.cts;
        else {
            cx.in = blob + (uint64_t)u * uc.cts;
            cx.in_len = ((uint64_t)(u + 1) * uc.cts <= blob_len) ? uc.cts : 0;
        }
        olabel xin[MAXK], xout[MAXK];
        for (int i = 0; i < k; ++i) xin[i] = in[i].l[u];
        g_act_element(&cx, l->kind, xin, xout, &e->base, e->sign);
        for (int i = 0; i < k; ++i) out[i].l[u] = xout[i];
        if (cx.err) err = cx.err;
    }
    return err ? fail(ORC_DATA, "ciphertext stream exhausted") : 0;
}

/* ===================== whole network (garble.cpp:16-343) ===================== */

struct orc_net {
    const orc_circuit* c;
    ocrt base;
    osign* sign;
    int has_sign;
    uint8_t seed[16];
    ooffsets* offs;
    olabel zeros[MAXK];
    otensor enc_bases[MAXK]; /* input lanes */
    u128* cts;
    uint64_t ncts;
    uint64_t layer_ct_base[ORC_MAXL + 2];
    uint64_t layer_gate[ORC_MAXL + 2], layer_wire[ORC_MAXL + 2];
    u128 commitment;
    u128* dec; /* [elem*k + lane][p] flattened with row offsets */
    uint64_t* dec_off;
    uint64_t n_out;
    uint64_t stats[3];
};

struct orc_bundle {
    int k;
    otensor lanes[MAXK];
};

static void env_init(oenv* e, const orc_net* n) {
    memset(e, 0, sizeof *e);
    e->base = n->base;
    e->sign = n->has_sign ? n->sign : NULL;
    for (int i = 0; i < n->base.k; ++i) e->zeros[i] = n->zeros[i];
    e->offs = n->offs;
}

/* circuit_layout (garble.cpp:16-37) */
static void layout(orc_net* n, const oenv* e, uint64_t wire0) {
    uint64_t g = 0, w = wire0, ct = 0;
    for (int li = 0; li < n->c->nl; ++li) {
        n->layer_gate[li] = g;
        n->layer_wire[li] = w;
        n->layer_ct_base[li] = ct;
        octx cx;
        memset(&cx, 0, sizeof cx);
        cx.mode = M_COUNT;
        count_layer(n->c, li, e, &cx);
        g += cx.gates;
        w += cx.wires;
        ct += cx.cts;
    }
    n->layer_gate[n->c->nl] = g;
    n->layer_wire[n->c->nl] = w;
    n->layer_ct_base[n->c->nl] = ct;
}

int orc_garble(const orc_circuit* c, const uint8_t* seed16, orc_net** out) {
    for (int i = 0; i < c->nl; ++i)
        if (is_linear(&c->layers[i]) && c->layers[i].nw != wcount(&c->layers[i]))
            return fail(ORC_DATA, "circuit must be quantized before garbling");
    orc_net* n = (orc_net*)calloc(1, sizeof *n);
    n->c = c;
    n->base = crt_base(c->k);
    n->sign = (osign*)calloc(1, sizeof(osign));
    n->offs = (ooffsets*)calloc(1, sizeof(ooffsets));
    memcpy(n->seed, seed16, 16);
    n->has_sign = circuit_needs_sign(c);
    int rc = 0;
    if (n->has_sign) {
        ospec spec;
        rc = choose_spec(&n->base, c->sign_target, &spec);
        if (!rc) rc = make_sign(&n->base, &spec, n->sign);
        if (rc) {
            orc_net_free(n);
            return rc;
        }
    }
    oprf prf;
    aes_expand(&prf.k, seed16);
    oenv e;
    env_init(&e, n);
    e.prf = &prf;
    /* count_circuit (circuit.cpp:127-142) */
    octx tot;
    memset(&tot, 0, sizeof tot);
    tot.mode = M_COUNT;
    for (int li = 0; li < c->nl; ++li) count_layer(c, li, &e, &tot);
    for (int i = 0; i < n->base.k; ++i) tot.moduli[n->base.primes[i]] = 1;
    for (int m = 2; m <= MAXM; ++m)
        if (tot.moduli[m]) {
            n->offs->r[m] = prf_offset(&prf, m);
            n->offs->present[m] = 1;
        }
    const int k = n->base.k;
    for (int i = 0; i < k; ++i) n->zeros[i] = prf_label(&prf, (uint64_t)i, n->base.primes[i]);
    env_init(&e, n);
    e.prf = &prf;
    const uint64_t n_in = shape_size(c->shapes[0], c->ranks[0]);
    /* outs[0] = input base labels, outs[j + 1] = base labels out of layer j */
    otensor(*outs)[MAXK] = (otensor(*)[MAXK])calloc((size_t)c->nl + 1, sizeof(otensor[MAXK]));
    for (int i = 0; i < k; ++i) {
        n->enc_bases[i] = tnew(n->base.primes[i], n_in);
        for (uint64_t el = 0; el < n_in; ++el)
            n->enc_bases[i].l[el] = prf_label(&prf, (uint64_t)k + el * (uint64_t)k + (uint64_t)i, n->base.primes[i]);
        outs[0][i] = tnew(n->base.primes[i], n_in);
        memcpy(outs[0][i].l, n->enc_bases[i].l, sizeof(olabel) * n_in);
    }
    layout(n, &e, (uint64_t)k * (1 + n_in));
    n->ncts = tot.cts;
    n->cts = (u128*)calloc(n->ncts ? n->ncts : 1, sizeof(u128));
    {   /* seed commitment (garble.cpp:199-204) */
        u128 v = 0;
        for (int i = 15; i >= 0; --i) v = (v << 8) | seed16[i];
        n->commitment = davies_meyer(v);
    }
    for (int li = 0; li < c->nl; ++li) {
        const olayer* l = &c->layers[li];
        rc = run_layer(c, li, &e, 1, n->layer_gate[li], n->layer_wire[li], n->cts + n->layer_ct_base[li], 0,
                       outs[src_index(li, l->src)], outs[src_index(li, l->src2)], outs[li + 1]);
        if (rc) break;
    }
    otensor* wires = outs[c->nl];
    if (!rc) {
        /* decoding tables (garble.cpp:208-231) */
        n->n_out = shape_size(c->shapes[c->nl], c->ranks[c->nl]);
        uint64_t sum_p = 0;
        for (int i = 0; i < k; ++i) sum_p += (uint64_t)n->base.primes[i];
        n->dec = (u128*)malloc(sizeof(u128) * n->n_out * sum_p + 16);
        n->dec_off = (uint64_t*)malloc(sizeof(uint64_t) * (n->n_out * (uint64_t)k + 1));
        uint64_t pos = 0;
        for (uint64_t el = 0; el < n->n_out; ++el)
            for (int i = 0; i < k; ++i) {
                const int p = n->base.primes[i];
                n->dec_off[el * (uint64_t)k + (uint64_t)i] = pos;
                olabel cand = wires[i].l[el];
                for (int v = 0; v < p; ++v) {
                    n->dec[pos++] = compress(&cand);
                    ladd_into(&cand, &n->offs->r[p]);
                }
            }
        n->dec_off[n->n_out * (uint64_t)k] = pos;
        n->stats[0] = tot.cts;
        n->stats[1] = tot.gates;
        n->stats[2] = tot.wires + (uint64_t)k * (1 + n_in);
    }
    for (int li = 0; li <= c->nl; ++li)
        for (int i = 0; i < k; ++i) tfree(&outs[li][i]);
    free(outs);
    if (rc) {
        orc_net_free(n);
        return rc;
    }
    *out = n;
    return 0;
}

void orc_net_free(orc_net* n) {
    if (!n) return;
    for (int i = 0; i < MAXK; ++i) tfree(&n->enc_bases[i]);
    free(n->cts);
    free(n->dec);
    free(n->dec_off);
    free(n->sign);
    free(n->offs);
    free(n);
}

uint64_t orc_net_cts_count(const orc_net* n) { return n->ncts; }
void orc_net_cts(const orc_net* n, uint64_t* out) {
    for (uint64_t i = 0; i < n->ncts; ++i) st128(out + 2 * i, n->cts[i]);
}
int orc_net_layer_ct_base(const orc_net* n, uint64_t* out) {
    for (int i = 0; i <= n->c->nl; ++i) out[i] = n->layer_ct_base[i];
    return n->c->nl + 1;
}
void orc_net_stats(const orc_net* n, uint64_t* out3) { memcpy(out3, n->stats, sizeof n->stats); }

/* ----- serialization (garble.cpp:56-132, 347-526; serial.hpp) ----- */

typedef struct {
    uint8_t* buf;
    size_t cap, len;
} owriter;
static void w_bytes(owriter* w, const void* p, size_t n) {
    if (w->buf && w->len + n <= w->cap) memcpy(w->buf + w->len, p, n);
    w->len += n;
}
static void w_le(owriter* w, uint64_t v, int nbytes) {
    uint8_t b[8];
    for (int i = 0; i < nbytes; ++i) b[i] = (uint8_t)(v >> (8 * i));
    w_bytes(w, b, (size_t)nbytes);
}
static void w_u128(owriter* w, u128 v) {
    w_le(w, (uint64_t)v, 8);
    w_le(w, (uint64_t)(v >> 64), 8);
}
static void w_header(owriter* w, int kind) {
    w_bytes(w, "DASH", 4);
    w_le(w, 1, 2);
    w_le(w, (uint64_t)kind, 1);
}
static void w_shape(owriter* w, const uint32_t* s, int r) {
    w_le(w, (uint64_t)r, 1);
    for (int i = 0; i < r; ++i) w_le(w, s[i], 4);
}
static uint64_t dbits(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
}

size_t orc_net_gc_bytes(const orc_net* n, uint8_t* buf, size_t cap) {
    owriter w = {buf, cap, 0};
    const orc_circuit* c = n->c;
    w_header(&w, 1);
    w_le(&w, (uint64_t)c->k, 1);
    w_shape(&w, c->shapes[0], c->ranks[0]);
    w_le(&w, dbits(c->alpha), 8);
    w_le(&w, dbits(c->sign_target), 8);
    const int t = n->has_sign ? n->sign->spec.t : 0;
    w_le(&w, (uint64_t)t, 1);
    for (int j = 0; j < t; ++j) w_le(&w, (uint64_t)n->sign->spec.radices[j], 2);
    w_le(&w, (uint64_t)c->nl, 2);
    for (int li = 0; li < c->nl; ++li) {
        const olayer* l = &c->layers[li];
        w_le(&w, (uint64_t)l->kind, 1);
        /* bit 1 of the private byte flags the extension record (dash_circuit_desc.h) */
        const int ext = l->kind > DASH_LAYER_FLATTEN || l->src || l->src2 || l->pad;
        w_le(&w, (uint64_t)(l->priv ? 1 : 0) | (ext ? 2u : 0u), 1);
        w_le(&w, l->in_dim, 4);
        w_le(&w, l->out_dim, 4);
        w_le(&w, l->in_ch, 4);
        w_le(&w, l->out_ch, 4);
        w_le(&w, l->filter, 4);
        w_le(&w, l->stride, 4);
        const int ww = is_linear(l) && !l->priv;
        w_le(&w, ww ? 1 : 0, 1);
        if (ww) {
            w_le(&w, l->nw, 8);
            for (uint64_t i = 0; i < l->nw; ++i) w_le(&w, (uint64_t)l->w[i], 8);
        }
        if (ext) { /* extension record */
            w_le(&w, (uint64_t)(uint32_t)l->src, 4);
            w_le(&w, (uint64_t)(uint32_t)l->src2, 4);
            w_le(&w, l->pad, 4);
        }
    }
    for (int i = 0; i < c->k; ++i) w_u128(&w, compress(&n->zeros[i]));
    w_le(&w, (uint64_t)c->nl + 1, 8);
    for (int i = 0; i <= c->nl; ++i) w_le(&w, n->layer_ct_base[i], 8);
    w_le(&w, n->ncts, 8);
    for (uint64_t i = 0; i < n->ncts; ++i) w_u128(&w, n->cts[i]);
    w_u128(&w, n->commitment);
    return w.len;
}

size_t orc_net_enc_bytes(const orc_net* n, uint8_t* buf, size_t cap) {
    owriter w = {buf, cap, 0};
    const orc_circuit* c = n->c;
    w_header(&w, 2);
    w_le(&w, (uint64_t)c->k, 1);
    w_shape(&w, c->shapes[0], c->ranks[0]);
    for (int i = 0; i < c->k; ++i) w_u128(&w, compress(&n->offs->r[n->base.primes[i]]));
    for (int i = 0; i < c->k; ++i) { /* tensor_write (label_tensor.cpp:95-101) */
        w_le(&w, (uint64_t)n->base.primes[i], 2);
        w_shape(&w, c->shapes[0], c->ranks[0]);
        for (int el = 0; el < n->enc_bases[i].n; ++el) w_u128(&w, compress(&n->enc_bases[i].l[el]));
    }
    return w.len;
}

size_t orc_net_dec_bytes(const orc_net* n, uint8_t* buf, size_t cap) {
    owriter w = {buf, cap, 0};
    const orc_circuit* c = n->c;
    w_header(&w, 3);
    w_le(&w, (uint64_t)c->k, 1);
    w_shape(&w, c->shapes[c->nl], c->ranks[c->nl]);
    for (uint64_t i = 0; i < n->dec_off[n->n_out * (uint64_t)c->k]; ++i) w_u128(&w, n->dec[i]);
    return w.len;
}

/* garble_inputs (garble.cpp:242-263) */
int orc_garble_inputs(const orc_net* n, const int64_t* values, size_t count, orc_bundle** out) {
    const uint64_t n_in = shape_size(n->c->shapes[0], n->c->ranks[0]);
    if (count != n_in) return fail(ORC_DATA, "input element count mismatch");
    orc_bundle* b = (orc_bundle*)calloc(1, sizeof *b);
    b->k = n->base.k;
    for (int i = 0; i < b->k; ++i) {
        const int p = n->base.primes[i];
        b->lanes[i] = tnew(p, n_in);
        for (uint64_t el = 0; el < n_in; ++el) {
            u128 x;
            if (encode_signed(values[el], &n->base, &x)) {
                orc_bundle_free(b);
                return ORC_DATA;
            }
            olabel l = n->enc_bases[i].l[el];
            ladd_scaled(&l, &n->offs->r[p], (uint32_t)(x % (u128)p));
            b->lanes[i].l[el] = l;
        }
    }
    *out = b;
    return 0;
}

/* evaluate (garble.cpp:265-312) */
int orc_evaluate(const orc_net* n, const orc_bundle* in, orc_bundle** out) {
    const int k = n->base.k;
    oenv e;
    env_init(&e, n);
    e.offs = NULL;
    const int nl = n->c->nl;
    otensor(*outs)[MAXK] = (otensor(*)[MAXK])calloc((size_t)nl + 1, sizeof(otensor[MAXK]));
    for (int i = 0; i < k; ++i) {
        outs[0][i] = tnew(in->lanes[i].m, (uint64_t)in->lanes[i].n);
        memcpy(outs[0][i].l, in->lanes[i].l, sizeof(olabel) * (size_t)in->lanes[i].n);
    }
    int rc = 0;
    int done = 0;
    for (int li = 0; li < nl && !rc; ++li) {
        const olayer* l = &n->c->layers[li];
        const uint64_t b0 = n->layer_ct_base[li], b1 = n->layer_ct_base[li + 1];
        rc = run_layer(n->c, li, &e, 0, n->layer_gate[li], 0, n->cts + b0, b1 - b0, outs[src_index(li, l->src)],
                       outs[src_index(li, l->src2)], outs[li + 1]);
        done = li + 1;
    }
    orc_bundle* b = NULL;
    if (!rc) {
        b = (orc_bundle*)calloc(1, sizeof *b);
        b->k = k;
        for (int i = 0; i < k; ++i) {
            b->lanes[i] = outs[nl][i];
            outs[nl][i].l = NULL;
        }
    }
    for (int li = 0; li <= done; ++li)
        for (int i = 0; i < k; ++i)
            if (outs[li][i].l) tfree(&outs[li][i]);
    free(outs);
    if (rc) return rc;
    *out = b;
    return 0;
}

/* decode_outputs (garble.cpp:314-343) */
int orc_decode(const orc_net* n, const orc_bundle* b, int64_t* values) {
    const int k = n->base.k;
    for (uint64_t el = 0; el < n->n_out; ++el) {
        uint16_t res[MAXK];
        for (int i = 0; i < k; ++i) {
            const u128 cand = compress(&b->lanes[i].l[el]);
            const uint64_t o = n->dec_off[el * (uint64_t)k + (uint64_t)i];
            int found = -1;
            for (int v = 0; v < n->base.primes[i]; ++v)
                if (n->dec[o + (uint64_t)v] == cand) {
                    found = v;
                    break;
                }
            if (found < 0) return fail(ORC_AUTH, "output label not present in the decoding table");
            res[i] = (uint16_t)found;
        }
        values[el] = decode_signed(crt_reconstruct(res, &n->base), &n->base);
    }
    return 0;
}

/* bundle_payload (garble.cpp:465-472) */
size_t orc_bundle_payload(const orc_bundle* b, uint8_t* buf, size_t cap) {
    owriter w = {buf, cap, 0};
    for (int i = 0; i < b->k; ++i)
        for (int el = 0; el < b->lanes[i].n; ++el) w_u128(&w, compress(&b->lanes[i].l[el]));
    return w.len;
}

/* bundle_from_payload (garble.cpp:474-490): k lanes over the input (output=0)
 * or output (output=1) shape, chunks reduced mod m^n. */
int orc_bundle_from_payload(const orc_net* n, const uint8_t* data, size_t len, int output, orc_bundle** out) {
    const int li = output ? n->c->nl : 0;
    const uint64_t ne = shape_size(n->c->shapes[li], n->c->ranks[li]);
    if (len != (size_t)n->base.k * ne * 16) return fail(ORC_DATA, "wire payload size mismatch");
    orc_bundle* b = (orc_bundle*)calloc(1, sizeof *b);
    b->k = n->base.k;
    size_t pos = 0;
    for (int i = 0; i < b->k; ++i) {
        b->lanes[i] = tnew(n->base.primes[i], ne);
        for (uint64_t el = 0; el < ne; ++el) {
            uint64_t lo = 0, hi = 0;
            for (int j = 0; j < 8; ++j) lo |= (uint64_t)data[pos + j] << (8 * j);
            for (int j = 0; j < 8; ++j) hi |= (uint64_t)data[pos + 8 + j] << (8 * j);
            pos += 16;
            b->lanes[i].l[el] = decompress_mod(((u128)hi << 64) | lo, n->base.primes[i]);
        }
    }
    *out = b;
    return 0;
}

void orc_bundle_free(orc_bundle* b) {
    if (!b) return;
    for (int i = 0; i < b->k; ++i) tfree(&b->lanes[i]);
    free(b);
}

/* ===================== primitive exports ===================== */

static olabel lfrom(const uint16_t* d, int m) {
    olabel l = lshape(m);
    for (int i = 0; i < l.n; ++i) l.d[i] = d[i];
    return l;
}
static void lto(const olabel* l, uint16_t* d) {
    for (int i = 0; i < l->n; ++i) d[i] = l->d[i];
}

void orc_aes_fixed(const uint64_t* in, uint64_t* out) { st128(out, aes_enc(fixed_pi(), ld128(in))); }
void orc_aes_key(const uint8_t* key16, const uint64_t* in, uint64_t* out) {
    aes_key k;
    aes_expand(&k, key16);
    st128(out, aes_enc(&k, ld128(in)));
}
void orc_davies_meyer(const uint64_t* in, uint64_t* out) { st128(out, davies_meyer(ld128(in))); }
int orc_n_digits(int m) {
    mi_init();
    return (m >= 2 && m <= MAXM) ? MI[m].n : -1;
}
void orc_compress(int m, const uint16_t* d, uint64_t* out) {
    olabel l = lfrom(d, m);
    st128(out, compress(&l));
}
void orc_decompress_mod(const uint64_t* c, int m, uint16_t* d) {
    olabel l = decompress_mod(ld128(c), m);
    lto(&l, d);
}
/* seed_from_string (prf.cpp:42-66) */
int orc_seed_from_string(const char* s, uint8_t* out16) {
    if (s[0] == '0' && (s[1] == 'x' || s[1] == 'X')) s += 2;
    const size_t len = strlen(s);
    if (len == 0 || len > 32) return fail(ORC_DATA, "seed must be 1..32 hex digits");
    u128 v = 0;
    for (size_t i = 0; i < len; ++i) {
        const char ch = s[i];
        int dg;
        if (ch >= '0' && ch <= '9') dg = ch - '0';
        else if (ch >= 'a' && ch <= 'f') dg = ch - 'a' + 10;
        else if (ch >= 'A' && ch <= 'F') dg = ch - 'A' + 10;
        else return fail(ORC_DATA, "seed contains a non-hex character");
        v = (v << 4) | (unsigned)dg;
    }
    for (int i = 15; i >= 0; --i) {
        out16[i] = (uint8_t)v;
        v >>= 8;
    }
    return 0;
}
void orc_prf_label(const uint8_t* seed16, uint64_t wire, int m, uint16_t* d) {
    oprf p;
    aes_expand(&p.k, seed16);
    olabel l = prf_label(&p, wire, m);
    lto(&l, d);
}
void orc_prf_offset(const uint8_t* seed16, int m, uint16_t* d) {
    oprf p;
    aes_expand(&p.k, seed16);
    olabel l = prf_offset(&p, m);
    lto(&l, d);
}
void orc_pad_bits(int m, const uint16_t* k1, uint64_t gate, uint32_t row, uint32_t slot, uint64_t* out) {
    olabel a = lfrom(k1, m);
    st128(out, pad_bits(&a, tweak(gate, row, slot)));
}
/* two-key form (cipher.cpp:14-16) */
void orc_pad_bits2(int m1, const uint16_t* k1, int m2, const uint16_t* k2, uint64_t gate, uint32_t row,
                   uint32_t slot, uint64_t* out) {
    olabel a = lfrom(k1, m1), b = lfrom(k2, m2);
    const u128 cb = compress(&b);
    st128(out, davies_meyer(compress(&a) ^ ((cb << 1) | (cb >> 127)) ^ tweak(gate, row, slot)));
}
void orc_encrypt_label(int mk, const uint16_t* k1, uint64_t gate, uint32_t row, uint32_t slot, int mq,
                       const uint16_t* msg, uint64_t* out) {
    olabel a = lfrom(k1, mk), m = lfrom(msg, mq);
    st128(out, encrypt_label(&a, tweak(gate, row, slot), &m));
}
void orc_decrypt_label(int mk, const uint16_t* k1, uint64_t gate, uint32_t row, uint32_t slot,
                       const uint64_t* ct, int q, uint16_t* out) {
    olabel a = lfrom(k1, mk);
    olabel r = decrypt_label(&a, tweak(gate, row, slot), ld128(ct), q);
    lto(&r, out);
}
int orc_choose_mixed_radix(int k, double target, uint16_t* radices) {
    if (k < 1 || k > MAXK) return -ORC_DATA;
    const ocrt b = crt_base(k);
    ospec s;
    int rc = choose_spec(&b, target, &s);
    if (rc) return -rc;
    for (int j = 0; j < s.t; ++j) radices[j] = (uint16_t)s.radices[j];
    return s.t;
}
int orc_element_cost(int k, double target, int kind, uint64_t* out3) {
    oenv e;
    memset(&e, 0, sizeof e);
    e.base = crt_base(k);
    ospec s;
    int rc = choose_spec(&e.base, target, &s);
    if (rc) return rc;
    e.sign = (osign*)calloc(1, sizeof(osign));
    rc = make_sign(&e.base, &s, e.sign);
    if (!rc) {
        ocost uc = element_cost(kind, &e, NULL);
        out3[0] = uc.cts;
        out3[1] = uc.gates;
        out3[2] = uc.wires;
    }
    free(e.sign);
    return rc;
}

double orc_bench_infer(const orc_circuit* c, int n, const uint8_t* seeds, const int64_t* inputs, int64_t* outputs,
                       int threads) {
    uint64_t n_in, n_out;
    orc_circuit_io(c, &n_in, &n_out);
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    int err = 0;
    /* fewer inferences than threads: one at a time, OpenMP inside the layers
     * (the reference's own intra-layer mode); else one inference per thread */
    const int outer = n >= threads ? threads : 1;
#ifdef _OPENMP
    omp_set_max_active_levels(1);
    if (outer == 1) omp_set_num_threads(threads);
#endif
#pragma omp parallel for schedule(dynamic, 1) num_threads(outer)
    for (int b = 0; b < n; ++b) {
        orc_net* net = NULL;
        orc_bundle *in = NULL, *out = NULL;
        int rc = orc_garble(c, seeds + 16 * b, &net);
        if (!rc) rc = orc_garble_inputs(net, inputs + (uint64_t)b * n_in, n_in, &in);
        if (!rc) rc = orc_evaluate(net, in, &out);
        if (!rc) rc = orc_decode(net, out, outputs + (uint64_t)b * n_out);
        if (rc) err = rc;
        orc_bundle_free(in);
        orc_bundle_free(out);
        orc_net_free(net);
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (err) return -1.0;
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}

/* one-time table setup before any OpenMP region touches them */
__attribute__((constructor)) static void orc_init(void) {
    sbox_init();
    mi_init();
    (void)fixed_pi();
}
