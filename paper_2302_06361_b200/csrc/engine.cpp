// Host engine of the B200 Dash garble/evaluate path (plain C++; all device
// work goes through launch.hpp).
//
//  * host math: digit capacities / codec constants (reference label.cpp:15-64),
//    AES key schedule (aes.cpp:32-46), CRT base (crt.cpp:38-101), mixed-radix
//    spec search and sign tables (mixed_radix.cpp:59-212), sign plan
//    (gadgets.cpp:5-28);
//  * the activation "gadget tape": the reference's t_approx_sign_bit /
//    relu_element / sign_act_element (gadgets.hpp:382-481, layer.cpp:214-236)
//    recorded once in reference order so every gate / fresh wire / ciphertext
//    gets the reference's per-element offset, then re-scheduled depth-first
//    to keep few labels live and mapped onto per-thread label slots;
//  * circuit preparation and layout (circuit.cpp, garble.cpp:16-42);
//  * the batched network driver: garble / garble_inputs / evaluate /
//    decode_outputs over B inferences resident in HBM (garble.cpp:134-343);
//  * reference wire formats (garble.cpp:347-526) and the C ABI (dashgpu.h).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <tuple>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "dashgpu.h"
#include "launch.hpp"

namespace dashgpu {

struct DataError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct OverflowErr : DataError {
    using DataError::DataError;
};
struct AuthError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

static const int kPrimes[MAXK] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53};

// =========================================================== host math

// n_m = max{n : m^n <= 2^128} (label.cpp:15-29)
static int n_digits_host(int m) {
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

static int bitlen(u128 x) {
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

// floor(x / d) = umulhi(x, mag) >> sh for 0 <= x < 2^31 (Granlund-Montgomery)
static void magic31(uint64_t d, uint32_t& mag, uint32_t& sh) {
    int l = 0;
    while (((uint64_t)1 << l) < d) ++l;
    if (l == 0) l = 1;
    const u128 num = (u128)1 << (31 + l);
    const u128 M = (num + d - 1) / d;
    if (M >> 32) throw std::logic_error("magic31 overflow");
    mag = (uint32_t)M;
    sh = (uint32_t)(l - 1);
    // spot-check exactness at the range edges
    const uint64_t probes[] = {0, 1, d - 1, d, d + 1, (1u << 31) - 1, (1u << 31) - d, 12345677};
    for (uint64_t x : probes) {
        if (x >= (1ull << 31)) continue;
        if ((((uint64_t)x * mag) >> 32 >> sh) != x / d) throw std::logic_error("magic31 inexact");
    }
}

static ModC make_modc(int m) {
    ModC c;
    std::memset(&c, 0, sizeof c);
    c.m = (uint16_t)m;
    c.n = (uint8_t)n_digits_host(m);
    c.nw = (uint8_t)((c.n + 3) / 4);
    c.pow2 = (m & (m - 1)) == 0;
    c.e = 0;
    if (c.pow2)
        while ((1 << (c.e + 1)) <= m) ++c.e;
    c.full = c.pow2 && c.e * c.n == 128;
    magic31((uint64_t)m, c.mag_m, c.sh_m);
    c.mag64 = (uint64_t)(~0ull / (uint64_t)m) + 1;
    c.spread = (uint32_t)m * 0x01010101u;
    c.negm = 0u - (uint32_t)m;
    c.negm4 = 0u - (uint32_t)m * m * m * m;
    c.addc = (uint32_t)(128 - (m < 128 ? m : 127)) * 0x01010101u;
    if (c.pow2) {
        u128 bits = 0, hi = 0, lo = 0;
        for (int i = 0; i < c.n; ++i) {
            lo |= (u128)1 << (c.e * i);
            hi |= (u128)1 << (c.e * i + c.e - 1);
        }
        bits = c.e * c.n >= 128 ? ~(u128)0 : (((u128)1 << (c.e * c.n)) - 1);
        for (int j = 0; j < 4; ++j) {
            c.bits[j] = (uint32_t)(bits >> (32 * j));
            c.hi[j] = (uint32_t)(hi >> (32 * j));
            c.lo[j] = (uint32_t)(lo >> (32 * j));
        }
        c.m4 = (uint32_t)m * m * m * m;
        return c;
    }
    c.m4 = (uint32_t)m * m * m * m;
    int W = 1;
    while (true) {
        u128 p = 1;
        for (int i = 0; i < 4 * (W + 1); ++i) p *= (u128)m;
        if (p >= ((u128)1 << 30)) break;  // D < 2^30: divmod_D's r~ < 3D fits 32 bits
        ++W;
    }
    c.W = (uint8_t)W;
    u128 D = 1;
    for (int i = 0; i < 4 * W; ++i) D *= (u128)m;
    c.D = (uint32_t)D;
    c.negD = 0u - c.D;
    c.nchunks = (uint8_t)((c.nw + W - 1) / W);
    u128 bound = ~(u128)0;
    for (int j = 0; j < c.nchunks && j < 21; ++j) {
        const int b = bitlen(bound);
        c.limbs[j] = (uint8_t)((b + 31) / 32);
        if (c.limbs[j] == 0) c.limbs[j] = 1;
        bound /= D;
    }
    magic31(c.m4, c.mag_m4, c.sh_m4);
    c.invD = ~0ull / (uint64_t)c.D;
    // byte dot-product word values and the paired / limb-bounded Horner
    c.wlo = 1u | ((uint32_t)m << 8);
    c.whi = (1u << 16) | ((uint32_t)m << 24);
    c.m2 = (uint32_t)m * m;
    const u128 m8 = (u128)c.m4 * c.m4;
    c.hp = m8 < ((u128)1 << 32) ? 2 : 1;
    c.m8 = c.hp == 2 ? (uint32_t)m8 : c.m4;
    c.htop = (c.hp == 2 && c.nw % 2 == 0) ? 2 : 1;
    auto limbs_of_digits = [&](int digits) {  // limbs of m^digits - 1
        u128 v = 1;
        for (int i = 0; i < digits; ++i) v *= (u128)m;
        const int b = bitlen(v - 1);
        return std::max(1, (b + 31) / 32);
    };
    for (int wlo = c.nw - c.htop - c.hp; wlo >= 0; wlo -= c.hp) {
        const int L = limbs_of_digits(std::min<int>(c.n, c.n - 4 * wlo));
        ++c.hlim[L - 1];
    }
    if (limbs_of_digits(std::min<int>(c.n, 4 * c.htop)) != 1) throw std::logic_error("horner top step overflow");
    for (int j = 0; j < c.nchunks && j < 21; ++j)
        c.climbs[j] = (uint8_t)limbs_of_digits(std::min<int>(c.n, 4 * c.W * (j + 1)));
    return c;
}

// ---- AES-128 key schedule + T0 table (FIPS-197; aes.cpp:32-46) ----
static uint8_t g_sbox[256];
static void sbox_init() {
    static bool done = false;
    if (done) return;
    auto gmul = [](uint8_t a, uint8_t b) {
        uint8_t r = 0;
        while (b) {
            if (b & 1) r ^= a;
            a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
            b >>= 1;
        }
        return r;
    };
    auto rotl8 = [](uint8_t x, int s) { return (uint8_t)((x << s) | (x >> (8 - s))); };
    for (int x = 0; x < 256; ++x) {
        uint8_t inv = 0;
        for (int y = 1; x && y < 256; ++y)
            if (gmul((uint8_t)x, (uint8_t)y) == 1) {
                inv = (uint8_t)y;
                break;
            }
        g_sbox[x] = (uint8_t)(inv ^ rotl8(inv, 1) ^ rotl8(inv, 2) ^ rotl8(inv, 3) ^ rotl8(inv, 4) ^ 0x63);
    }
    done = true;
}

static void aes_expand_host(const uint8_t key[16], uint32_t rk[44]) {
    static const uint8_t rcon[10] = {1, 2, 4, 8, 16, 32, 64, 128, 0x1b, 0x36};
    sbox_init();
    uint8_t w[176];
    std::memcpy(w, key, 16);
    for (int i = 4; i < 44; ++i) {
        uint8_t t[4];
        std::memcpy(t, w + 4 * (i - 1), 4);
        if (i % 4 == 0) {
            const uint8_t t0 = t[0];
            t[0] = (uint8_t)(g_sbox[t[1]] ^ rcon[i / 4 - 1]);
            t[1] = g_sbox[t[2]];
            t[2] = g_sbox[t[3]];
            t[3] = g_sbox[t0];
        }
        for (int j = 0; j < 4; ++j) w[4 * i + j] = (uint8_t)(w[4 * (i - 4) + j] ^ t[j]);
    }
    for (int i = 0; i < 44; ++i)
        rk[i] = (uint32_t)w[4 * i] | ((uint32_t)w[4 * i + 1] << 8) | ((uint32_t)w[4 * i + 2] << 16) |
                ((uint32_t)w[4 * i + 3] << 24);
}

static void t0_table(uint32_t T0[256]) {
    sbox_init();
    for (int x = 0; x < 256; ++x) {
        const uint32_t s = g_sbox[x];
        const uint32_t s2 = ((s << 1) ^ ((s & 0x80) ? 0x1b : 0)) & 0xff;
        const uint32_t s3 = s2 ^ s;
        T0[x] = s2 | (s << 8) | (s << 16) | (s3 << 24);
    }
}

// ---- CRT base (crt.cpp:38-101) ----
struct Crt {
    int k = 0;
    std::vector<int> primes;
    u128 P = 0;
    std::vector<u128> coeffs;
};

static Crt crt_base(int k) {
    if (k < 1 || k > MAXK) throw DataError("crt_base: k must be in [1, 16]");
    Crt b;
    b.k = k;
    b.P = 1;
    for (int i = 0; i < k; ++i) {
        b.primes.push_back(kPrimes[i]);
        b.P *= (u128)kPrimes[i];
    }
    for (int p : b.primes) {
        const u128 A = b.P / (u128)p;
        uint64_t base = (uint64_t)(A % (u128)p), r = 1;
        for (int e = p - 2; e > 0; e >>= 1) {
            if (e & 1) r = r * base % (uint64_t)p;
            base = base * base % (uint64_t)p;
        }
        b.coeffs.push_back(A * (u128)r);
    }
    return b;
}

static int64_t max_signed(const Crt& b) {
    const u128 hi = (b.P + 1) / 2 - 1;
    return hi > (u128)INT64_MAX ? INT64_MAX : (int64_t)hi;
}
static int64_t min_signed(const Crt& b) {
    const u128 mag = b.P / 2;
    return mag > (u128)INT64_MAX ? INT64_MIN : -(int64_t)mag;
}

// ---- mixed radix (mixed_radix.cpp) ----
using Spec = std::vector<int>;

static u128 spec_M(const Spec& s) {
    u128 M = 1;
    for (int r : s) M *= (u128)r;
    return M;
}

// round-half-away(M*y/P) = floor((2My + P) / (2P)) with a 256-bit numerator
static u128 round_scaled(u128 M, u128 y, u128 P) {
    const u128 a = 2 * M;
    const u128 al = (uint64_t)a, ah = a >> 64, bl = (uint64_t)y, bh = y >> 64;
    const u128 ll = al * bl, lh = al * bh, hl = ah * bl, hh = ah * bh;
    u128 lo = ll + (lh << 64);
    u128 carry = lo < ll;
    const u128 lo2 = lo + (hl << 64);
    carry += lo2 < lo;
    lo = lo2;
    u128 hi = hh + (lh >> 64) + (hl >> 64) + carry;
    const u128 lo3 = lo + P;
    hi += lo3 < lo;
    lo = lo3;
    const u128 d = 2 * P;
    u128 q = 0, rem = 0;
    for (int i = 255; i >= 0; --i) {
        const u128 bit = i >= 128 ? (hi >> (i - 128)) & 1 : (lo >> i) & 1;
        rem = (rem << 1) | bit;
        if (rem >= d) {
            rem -= d;
            if (i < 128) q |= (u128)1 << i;
        }
    }
    return q;
}

static std::vector<std::vector<u128>> d_tables(const Crt& b, u128 M) {
    std::vector<std::vector<u128>> d(b.k);
    for (int i = 0; i < b.k; ++i) {
        const u128 alpha = b.coeffs[i] % b.P;
        for (int x = 0; x < b.primes[i]; ++x) d[i].push_back(round_scaled(M, alpha * (u128)x % b.P, b.P) % M);
    }
    return d;
}

static uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

static double sign_accuracy(const Crt& b, const Spec& s) {
    const u128 M = spec_M(s);
    const auto d = d_tables(b, M);
    uint64_t ok = 0, total;
    auto cls = [&](u128 x) {
        u128 sum = 0;
        for (int i = 0; i < b.k; ++i) sum += d[i][(int)(x % (u128)b.primes[i])];
        sum %= M;
        return (2 * sum >= M) == (2 * x >= b.P);
    };
    if (b.P <= ((u128)1 << 20)) {
        total = (uint64_t)b.P;
        for (u128 x = 0; x < b.P; ++x) ok += cls(x);
    } else {
        total = 100000;
        for (uint64_t i = 0; i < total; ++i)
            ok += cls((((u128)splitmix64(2 * i) << 64) | splitmix64(2 * i + 1)) % b.P);
    }
    return (double)ok / (double)total;
}

struct SpecSearch {
    bool found = false;
    u128 M = 0;
    int t = 0, m1 = 0;
    Spec spec;
    void consider(int m1v, const std::vector<int>& tr, u128 bound) {
        u128 Mv = (u128)m1v;
        for (int x : tr) Mv *= (u128)x;
        if (Mv <= bound) return;
        const int tv = 1 + (int)tr.size();
        const bool better = !found || Mv < M || (Mv == M && tv < t) || (Mv == M && tv == t && m1v > m1);
        if (!better) return;
        found = true;
        M = Mv;
        t = tv;
        m1 = m1v;
        spec.assign(1, m1v);
        spec.insert(spec.end(), tr.begin(), tr.end());
    }
    void dfs(std::vector<int>& seq, u128 q, int last, u128 bound, u128 qmax) {
        if (!seq.empty()) {
            const u128 need = bound / q + 1;
            u128 m1v = need + (need & 1);
            if (m1v < 50) m1v = 50;
            if (m1v <= 128) consider((int)m1v, seq, bound);
        }
        for (int d = std::min(last, 8); d >= 2; --d)
            if (q * (u128)d <= qmax) {
                seq.push_back(d);
                dfs(seq, q * (u128)d, d, bound, qmax);
                seq.pop_back();
            }
    }
};

// choose_mixed_radix (mixed_radix.cpp:153-189)
static Spec choose_spec(const Crt& b, double target) {
    const u128 bound = (u128)b.k * b.P / 2;
    SpecSearch s;
    for (int m1 = 2; m1 <= 128; m1 += 2) s.consider(m1, {}, bound);
    std::vector<int> seq;
    s.dfs(seq, 1, 8, bound, bound / 25 + 1);
    if (!s.found) throw DataError("no mixed-radix spec reaches the required M");
    Spec cur = s.spec;
    if (target >= 1.0) return cur;
    if (sign_accuracy(b, cur) < target) return cur;
    Spec last = cur;
    while (true) {
        Spec next = cur;
        if (next.size() > 1) next.pop_back();
        else if (next[0] > 2) next[0] -= 2;
        else return last;
        if (sign_accuracy(b, next) < target) return last;
        last = next;
        cur = next;
    }
}

struct Pos {
    int m, b_mod, carry_in, carry_out;
};
struct SignCtx {
    Spec spec;
    std::vector<Pos> positions;  // make_sign_plan (gadgets.cpp:5-28)
    int msd_carry = 0;
    std::vector<std::vector<std::vector<int>>> digits;  // [i][j][x]
};

static SignCtx make_sign(const Crt& b, const Spec& spec) {
    if (spec.empty() || spec[0] % 2) throw DataError("mixed-radix m_1 must be even");
    for (int r : spec)
        if (r < 2 || r > 128) throw DataError("mixed-radix digit modulus out of range");
    SignCtx s;
    s.spec = spec;
    const int t = (int)spec.size();
    if (b.k > 1 && t > 1) {
        int carry = 0;
        for (int j = t - 1; j >= 1; --j) {
            Pos p;
            p.m = spec[j];
            p.carry_in = carry;
            p.b_mod = b.k * (p.m - 1) + (carry ? carry - 1 : 0) + 1;
            if (p.b_mod > MAXMOD) throw DataError("mixed-radix digit sum exceeds the modulus limit");
            const int maxcarry = (p.b_mod - 1) / p.m;
            p.carry_out = maxcarry > 0 ? maxcarry + 1 : 0;
            carry = p.carry_out;
            s.positions.push_back(p);
        }
        s.msd_carry = carry;
    }
    const auto d = d_tables(b, spec_M(spec));
    s.digits.assign(b.k, std::vector<std::vector<int>>(t));
    for (int i = 0; i < b.k; ++i)
        for (int x = 0; x < b.primes[i]; ++x) {
            u128 v = d[i][x];
            for (int j = t - 1; j >= 0; --j) {
                s.digits[i][j].resize(b.primes[i]);
                s.digits[i][j][x] = (int)(v % (u128)spec[j]);
                v /= (u128)spec[j];
            }
        }
    return s;
}

// ======================================================= activation tape

struct Tape {
    std::vector<TapeOp> ops;
    std::vector<uint8_t> phi;
    uint64_t cts = 0, gates = 0, wires = 0;
    uint64_t eval_rows = 0;  // ciphertext rows one evaluation reads
    int nslots = 0;
    std::set<int> moduli;
    uint8_t out_kind[MAXK] = {};   // gadget producing output lane i (OP_MMHALF / OP_PROJ)
    uint32_t out_wire[MAXK] = {};  // its first fresh wire offset
    // level-scheduled copy for warp-per-element evaluation (see ActParams)
    std::vector<TapeOp> lv_ops;
    std::vector<uint16_t> lv_start;
    int nslots_lv = 0;
};

// Records the gadget DAG in reference order (CountCtx semantics,
// gadgets.hpp:82-98): gate ids, fresh wires and ciphertext positions advance
// exactly as in the reference.
class Recorder {
  public:
    struct ROp {
        int kind;
        int a = -1, b = -1, out = -1;
        int pm = 0, qm = 0, cst = 0;
        uint64_t gate = 0, wire = 0, ct = 0;
        uint32_t phi = 0;
    };
    std::vector<int> vmod;  // modulus per value; values 0..k-1 are the inputs
    std::vector<int> producer;
    std::vector<ROp> ops;
    std::vector<uint8_t> phi;
    uint64_t cts = 0, gates = 0, wires = 0;
    std::set<int> moduli;
    int k;

    explicit Recorder(const Crt& b) : k(b.k) {
        for (int p : b.primes) {
            vmod.push_back(p);
            producer.push_back(-1);
        }
    }
    int newval(int m, int op) {
        vmod.push_back(m);
        producer.push_back(op);
        return (int)vmod.size() - 1;
    }
    uint32_t addphi(const std::vector<int>& f, int q) {
        const uint32_t off = (uint32_t)phi.size();
        for (int v : f) phi.push_back((uint8_t)(v % q));
        return off;
    }
    int proj(int in, int q, const std::vector<int>& f) {  // t_proj
        const int p = vmod[in];
        ROp o;
        o.kind = OP_PROJ;
        o.a = in;
        o.pm = p;
        o.qm = q;
        o.gate = gates++;
        o.ct = cts;
        cts += (uint64_t)p;
        moduli.insert(p);
        o.wire = wires++;
        moduli.insert(q);
        o.phi = addphi(f, q);
        ops.push_back(o);
        return ops.back().out = newval(q, (int)ops.size() - 1);
    }
    int grr(int in, int q, const std::vector<int>& f) {  // t_proj_grr
        const int p = vmod[in];
        ROp o;
        o.kind = OP_GRR;
        o.a = in;
        o.pm = p;
        o.qm = q;
        o.gate = gates++;
        o.ct = cts;
        cts += (uint64_t)(p - 1);
        moduli.insert(p);
        moduli.insert(q);
        o.phi = addphi(f, q);
        ops.push_back(o);
        return ops.back().out = newval(q, (int)ops.size() - 1);
    }
    int half(int x, int y) {  // t_half_gate
        const int p = vmod[x];
        if (vmod[y] != p) throw DataError("half gate modulus mismatch");
        ROp o;
        o.kind = OP_HALF;
        o.a = x;
        o.b = y;
        o.pm = p;
        o.qm = p;
        o.gate = gates++;
        o.ct = cts;
        cts += 2u * (uint64_t)p;
        moduli.insert(p);
        o.wire = wires;
        wires += 2;
        ops.push_back(o);
        return ops.back().out = newval(p, (int)ops.size() - 1);
    }
    int mmhalf(int x, int y) {  // t_mm_half_gate
        const int p = vmod[x], q = vmod[y];
        if (q > p) throw DataError("mixed-modulus half gate needs q <= p");
        int w = 0;
        while ((1 << w) < p) ++w;
        if (w == 0) w = 1;
        if (q * w > 128) throw DataError("mixed-modulus short block exceeds 128 bits");
        ROp o;
        o.kind = OP_MMHALF;
        o.a = x;
        o.b = y;
        o.pm = p;
        o.qm = q;
        o.gate = gates++;
        o.ct = cts;
        cts += (uint64_t)p + (uint64_t)q + 1;
        moduli.insert(p);
        moduli.insert(q);
        o.wire = wires;
        wires += 2;
        ops.push_back(o);
        return ops.back().out = newval(p, (int)ops.size() - 1);
    }
    int add(int a, int b) {  // free_add (one binary step)
        if (vmod[a] != vmod[b]) throw DataError("free_add modulus mismatch");
        ROp o;
        o.kind = OP_ADD;
        o.a = a;
        o.b = b;
        o.pm = o.qm = vmod[a];
        ops.push_back(o);
        return ops.back().out = newval(vmod[a], (int)ops.size() - 1);
    }
    int addconst(int a, int c) {  // add_public_constant
        ROp o;
        o.kind = OP_ADDCONST;
        o.a = a;
        o.pm = o.qm = vmod[a];
        o.cst = c;
        moduli.insert(vmod[a]);
        ops.push_back(o);
        return ops.back().out = newval(vmod[a], (int)ops.size() - 1);
    }
    void output(int v, int lane) {
        ROp o;
        o.kind = OP_OUTPUT;
        o.a = v;
        o.pm = o.qm = vmod[v];
        o.cst = lane;
        ops.push_back(o);
    }
};

static std::vector<int> tabulate(int n, const std::function<int(int)>& f) {
    std::vector<int> v(n);
    for (int i = 0; i < n; ++i) v[i] = f(i);
    return v;
}

// t_approx_sign_bit (gadgets.hpp:442-481) with t_mixed_radix_add (382-435)
static int record_sign_bit(Recorder& r, const Crt& b, const SignCtx& s) {
    const int k = b.k, t = (int)s.spec.size();
    std::vector<std::vector<int>> bundles(k, std::vector<int>(t));
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < t; ++j) bundles[i][j] = r.proj(i, s.spec[j], s.digits[i][j]);
    int msd;
    if (k == 1) {
        msd = bundles[0][0];
    } else {
        int carry = -1;
        for (size_t pi = 0; pi < s.positions.size(); ++pi) {
            const Pos& pos = s.positions[pi];
            const int j = t - 1 - (int)pi;
            auto lift = [&](int m) { return tabulate(m, [](int a) { return a; }); };
            int sum = -1;
            for (int si = 0; si < k; ++si) {
                const int term = r.proj(bundles[si][j], pos.b_mod, lift(s.spec[j]));
                sum = sum < 0 ? term : r.add(sum, term);
            }
            if (pos.carry_in) {
                const int term = r.proj(carry, pos.b_mod, lift(pos.carry_in));
                sum = r.add(sum, term);
            }
            if (pos.carry_out) {
                const int m = pos.m;
                carry = r.proj(sum, pos.carry_out, tabulate(pos.b_mod, [m](int a) { return a / m; }));
            } else {
                carry = -1;
            }
        }
        const int m1 = s.spec[0];
        msd = bundles[0][0];
        for (int si = 1; si < k; ++si) msd = r.add(msd, bundles[si][0]);
        if (s.msd_carry) {
            const int term = r.proj(carry, m1, tabulate(s.msd_carry, [m1](int c) { return c % m1; }));
            msd = r.add(msd, term);
        }
    }
    const int m1 = s.spec[0], half = m1 / 2;
    const int negative = r.grr(msd, 2, tabulate(m1, [half](int v) { return v >= half ? 1 : 0; }));
    const int nonneg = r.addconst(negative, 1);
    int count = -1;
    for (int i = 0; i < k; ++i) {
        const int nz = r.proj(i, k + 1, tabulate(b.primes[i], [](int a) { return a != 0 ? 1 : 0; }));
        count = count < 0 ? nz : r.add(count, nz);
    }
    const int nonzero = r.proj(count, 2, tabulate(k + 1, [](int c) { return c >= 1 ? 1 : 0; }));
    return r.half(nonneg, nonzero);
}

// Depth-first schedule from the outputs + linear-scan slot assignment.
static Tape build_tape(int kind, const Crt& b, const SignCtx& s) {
    Recorder r(b);
    const int bit = record_sign_bit(r, b, s);
    for (int i = 0; i < b.k; ++i) {
        if (kind == DASH_LAYER_RELU) {
            r.output(r.mmhalf(i, bit), i);
        } else {
            const int p = b.primes[i];
            r.output(r.proj(bit, p, tabulate(2, [p](int v) { return v != 0 ? 1 : p - 1; })), i);
        }
    }
    const int nops = (int)r.ops.size();
    std::vector<int> order;
    std::vector<char> done(nops, 0);
    // depth-first, deeper operand first (keeps the live label set small once
    // add chains are fused below: a chain's running-sum terms are produced
    // after the long carry dependency they are added to)
    std::vector<int> depth(r.vmod.size(), 0);
    for (const auto& o : r.ops)
        if (o.out >= 0)
            depth[o.out] = 1 + std::max(o.a >= b.k ? depth[o.a] : 0, o.b >= b.k ? depth[o.b] : 0);
    std::function<void(int)> dfs = [&](int v) {
        if (v < 0 || v < b.k) return;
        const int op = r.producer[v];
        if (done[op]) return;
        int x = r.ops[op].a, y = r.ops[op].b;
        if (y >= b.k && (x < b.k || depth[y] > depth[x])) std::swap(x, y);
        dfs(x);
        dfs(y);
        done[op] = 1;
        order.push_back(op);
    };
    for (int i = 0; i < nops; ++i)
        if (r.ops[i].kind == OP_OUTPUT) {
            dfs(r.ops[i].a);
            done[i] = 1;
            order.push_back(i);
        }
    for (int i = 0; i < nops; ++i)
        if (!done[i]) throw std::logic_error("tape: unreachable gadget");
    // Fuse chains of free adds (the mixed-radix sums, the zero-test count):
    // an ADD whose result only feeds the next ADD's running operand is not
    // stored; the chain runs as OP_ADD(keep) + OP_ADDACC... at the position of
    // its last ADD (all terms are computed before it in DFS order), so the
    // running sum never round-trips through a compressed slot.  Execution
    // order does not change any output: gate / wire / row ids are per op.
    std::vector<int> uses(r.vmod.size(), 0);
    for (const auto& o : r.ops) {
        if (o.a >= 0) ++uses[o.a];
        if (o.b >= 0) ++uses[o.b];
    }
    std::vector<char> inter(nops, 0);  // ADD whose result is the running operand of the next ADD only
    for (int i = 0; i < nops; ++i) {
        const auto& o = r.ops[i];
        if (o.kind != OP_ADD || o.a < b.k) continue;
        const int pa = r.producer[o.a];
        if (r.ops[pa].kind == OP_ADD && uses[o.a] == 1) inter[pa] = 1;
    }
    struct Emit {
        int op, kind, a, b, out;
        bool keep;
    };
    std::vector<Emit> emits;
    for (int t : order) {
        const auto& o = r.ops[t];
        if (o.kind == OP_ADD && inter[t]) continue;  // emitted with its chain
        if (o.kind != OP_ADD || o.a < b.k || !inter[r.producer[o.a]]) {
            emits.push_back({t, o.kind, o.a, o.b, o.out, false});
            continue;
        }
        std::vector<int> chain{t};  // walk back to the chain's first ADD
        while (chain.back() >= 0) {
            const auto& c = r.ops[chain.back()];
            if (c.a < b.k || !inter[r.producer[c.a]]) break;
            chain.push_back(r.producer[c.a]);
        }
        std::reverse(chain.begin(), chain.end());
        const auto& f = r.ops[chain[0]];
        emits.push_back({chain[0], OP_ADD, f.a, f.b, -1, true});
        for (size_t j = 1; j < chain.size(); ++j) {
            const auto& c = r.ops[chain[j]];
            const bool last_add = j + 1 == chain.size();
            emits.push_back({chain[j], OP_ADDACC, -1, c.b, last_add ? c.out : -1, !last_add});
        }
    }
    std::vector<int> last(r.vmod.size(), -1);
    for (int t = 0; t < (int)emits.size(); ++t) {
        if (emits[t].a >= 0) last[emits[t].a] = t;
        if (emits[t].b >= 0) last[emits[t].b] = t;
    }
    std::vector<int> slot(r.vmod.size(), -1);
    std::vector<int> freelist;
    int nslots = 0;
    Tape tp;
    for (int t = 0; t < (int)emits.size(); ++t) {
        const Emit& em = emits[t];
        Recorder::ROp o = r.ops[em.op];
        o.kind = em.kind;
        o.a = em.a;
        o.b = em.b;
        o.out = em.out;
        TapeOp d;
        std::memset(&d, 0, sizeof d);
        d.kind = (uint8_t)o.kind;
        auto enc = [&](int v) -> uint8_t {
            if (v < 0) return 0;
            if (v < b.k) return (uint8_t)(IN_LANE + v);
            if (slot[v] < 0) throw std::logic_error("tape: operand without slot");
            return (uint8_t)slot[v];
        };
        d.a = enc(o.a);
        d.b = enc(o.b);
        d.pm = (uint16_t)o.pm;
        d.qm = (uint16_t)o.qm;
        d.cst = (uint16_t)(o.cst | (em.keep ? kKeep : 0));
        d.gate_off = (uint32_t)o.gate;
        d.wire_off = (uint32_t)o.wire;
        d.ct_off = (uint32_t)o.ct;
        d.phi_off = o.phi;
        for (int v : {o.a, o.b})
            if (v >= b.k && last[v] == t && slot[v] >= 0) {
                freelist.push_back(slot[v]);
                slot[v] = -1;
            }
        if ((o.kind == OP_HALF || o.kind == OP_MMHALF) && (o.qm & (o.qm - 1)) != 0)
            throw DataError("half-gate selector wire must have a power-of-two modulus <= 16");
        if ((o.kind == OP_HALF || o.kind == OP_MMHALF) && o.qm > 16)
            throw DataError("half-gate selector wire must have a power-of-two modulus <= 16");
        if (o.out >= 0) {
            int sidx;
            if (!freelist.empty()) {
                sidx = freelist.back();
                freelist.pop_back();
            } else {
                sidx = nslots++;
            }
            slot[o.out] = sidx;
            d.out = (uint8_t)sidx;
            if (last[o.out] < 0) {  // dead value
                freelist.push_back(sidx);
                slot[o.out] = -1;
            }
        }
        tp.ops.push_back(d);
    }
    if (nslots > MAXSLOTS) throw DataError("activation gadget needs too many label slots");
    tp.nslots = nslots;
    {
        // Level schedule of the same DAG for warp-per-element evaluation:
        // level(op) = 1 + max level of its operands' producers; ops of a level
        // are independent and run on different lanes.  Slots are allocated per
        // level and freed only after the level of a value's last reader, so
        // no op of a level overwrites a slot another op of that level reads.
        std::vector<int> lvl(nops, 0), vlevel(r.vmod.size(), -1), lastlv(r.vmod.size(), -1);
        int nl = 0;
        for (int t : order) {
            const auto& o = r.ops[t];
            int L = 0;
            for (int v : {o.a, o.b})
                if (v >= b.k) L = std::max(L, vlevel[v] + 1);
            lvl[t] = L;
            if (o.out >= 0) vlevel[o.out] = L;
            nl = std::max(nl, L + 1);
        }
        for (int t : order)
            for (int v : {r.ops[t].a, r.ops[t].b})
                if (v >= b.k) lastlv[v] = std::max(lastlv[v], lvl[t]);
        std::vector<std::vector<int>> bylv(nl);
        for (int t : order) bylv[lvl[t]].push_back(t);
        std::vector<int> lslot(r.vmod.size(), -1), lfree;
        int lns = 0;
        for (int L = 0; L < nl; ++L) {
            auto& ops = bylv[L];
            std::stable_sort(ops.begin(), ops.end(), [&](int x, int y) {  // similar gadgets on adjacent lanes
                const auto &ox = r.ops[x], &oy = r.ops[y];
                return std::make_tuple(ox.kind, ox.pm, ox.qm) < std::make_tuple(oy.kind, oy.pm, oy.qm);
            });
            tp.lv_start.push_back((uint16_t)tp.lv_ops.size());
            for (int t : ops) {
                const auto& o = r.ops[t];
                TapeOp d;
                std::memset(&d, 0, sizeof d);
                d.kind = (uint8_t)o.kind;
                d.pm = (uint16_t)o.pm;
                d.qm = (uint16_t)o.qm;
                d.cst = (uint16_t)o.cst;
                d.gate_off = (uint32_t)o.gate;
                d.wire_off = (uint32_t)o.wire;
                d.ct_off = (uint32_t)o.ct;
                d.phi_off = o.phi;
                auto enc = [&](int v) -> uint8_t {
                    if (v < 0) return 0;
                    if (v < b.k) return (uint8_t)(IN_LANE + v);
                    return (uint8_t)lslot[v];
                };
                d.a = enc(o.a);
                d.b = enc(o.b);
                if (o.out >= 0) {
                    int sidx;
                    if (!lfree.empty()) {
                        sidx = lfree.back();
                        lfree.pop_back();
                    } else {
                        sidx = lns++;
                    }
                    lslot[o.out] = sidx;
                    d.out = (uint8_t)sidx;
                }
                tp.lv_ops.push_back(d);
            }
            for (size_t v = b.k; v < r.vmod.size(); ++v)  // free values whose readers are all done
                if (lslot[v] >= 0 && lastlv[v] <= L && vlevel[v] <= L) {
                    lfree.push_back(lslot[v]);
                    lslot[v] = -1;
                }
        }
        tp.lv_start.push_back((uint16_t)tp.lv_ops.size());
        if (lns >= IN_LANE) throw DataError("level schedule needs too many label slots");
        if (std::getenv("DASH_DEBUG_LEVELS")) {
            for (size_t L = 0; L + 1 < tp.lv_start.size(); ++L) {
                double cost = 0, mx = 0;
                for (int i = tp.lv_start[L]; i < tp.lv_start[L + 1]; ++i) {
                    const auto& o = tp.lv_ops[i];
                    double c = o.kind == OP_PROJ ? o.pm + (n_digits_host(o.qm) + 3) / 4 : o.kind == OP_GRR ? o.pm : o.kind == OP_HALF ? 2 * o.pm : o.kind == OP_MMHALF ? o.pm + 2 * o.qm : 0;
                    cost += c;
                    mx = std::max(mx, c);
                }
                fprintf(stderr, "level %zu ops %d cost %.0f max %.0f\n", L, tp.lv_start[L + 1] - tp.lv_start[L], cost, mx);
            }
        }
        tp.nslots_lv = lns;
    }
    tp.phi = r.phi;
    if (tp.phi.empty()) tp.phi.push_back(0);
    for (const auto& o : r.ops)
        if (o.kind == OP_OUTPUT) {
            const auto& prod = r.ops[r.producer[o.a]];
            if (prod.kind != OP_MMHALF && prod.kind != OP_PROJ) throw std::logic_error("tape: unexpected output gadget");
            tp.out_kind[o.cst] = (uint8_t)prod.kind;
            tp.out_wire[o.cst] = (uint32_t)prod.wire;
        }
    // output mm half gates carry their lane (cst = lane + 1): the garbling tape
    // reads their u0 / v0 from act_output_thread instead of drawing them again
    for (const auto& o : r.ops)
        if (o.kind == OP_OUTPUT && r.ops[r.producer[o.a]].kind == OP_MMHALF) {
            const auto& prod = r.ops[r.producer[o.a]];
            for (auto* ops : {&tp.ops, &tp.lv_ops})
                for (auto& d : *ops)
                    if (d.kind == OP_MMHALF && d.wire_off == (uint32_t)prod.wire) d.cst = (uint16_t)(o.cst + 1);
        }
    tp.cts = r.cts;
    for (const auto& o : r.ops)
        tp.eval_rows += o.kind == OP_PROJ || o.kind == OP_GRR ? 1 : o.kind == OP_HALF ? 2 : o.kind == OP_MMHALF ? 3 : 0;
    tp.gates = r.gates;
    tp.wires = r.wires;
    tp.moduli = r.moduli;
    return tp;
}

// ============================================================== circuits

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { dev::release(p); }
    void reset() {
        dev::release(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t bytes) {
        if (bytes <= n && p) return;
        dev::release(p);
        p = dev::alloc(bytes);
        n = bytes;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// pinned host memory (asynchronous uploads of launch parameters)
struct HostBuf {
    void* p = nullptr;
    size_t n = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { dev::host_release(p); }
    void reset() {
        dev::host_release(p);
        p = nullptr;
        n = 0;
    }
    void ensure(size_t bytes) {
        if (bytes <= n && p) return;
        dev::host_release(p);
        p = dev::host_alloc(bytes);
        n = bytes;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Device and stream of this host thread's calls (dashgpu_use /
// dashgpu_set_stream): every entry point enqueues on the calling thread's
// stream, so several host threads can drive several streams (and devices).
static thread_local void* g_stream = nullptr;

struct HLayer {
    int kind = 0;
    bool priv = false;
    uint32_t in_dim = 0, out_dim = 0, in_ch = 0, out_ch = 0, filter = 0, stride = 0;
    int src = 0, src2 = 0;  // extension: DAG inputs (dash_circuit_desc.h)
    uint32_t pad = 0;       // extension: PAD2D
    std::vector<int64_t> w, bias;
    std::vector<uint32_t> in_shape, out_shape;
    uint64_t E_in = 0, E_out = 0;
    // layout (per inference)
    uint64_t gate_base = 0, wire_base = 0, ct_base = 0, cts = 0, gates = 0, wires = 0;
    // public / private linear: per-lane residues (host) and their device copies
    std::vector<std::vector<uint8_t>> wres_h, zt_h, bres_h;
    std::vector<std::shared_ptr<DevBuf>> wres, zt, bres;
    // public linear on the tensor cores: expanded weights + window offsets
    std::vector<uint8_t> wexp_h;
    std::vector<int32_t> koff_h;
    std::shared_ptr<DevBuf> wexp, koff;
    TcLinear tc;
    std::vector<int> tc_primes;  // CRT primes of the lanes (build_tc_linear)
    std::vector<uint64_t> lane_ct_off, lane_gate_off, lane_wire_off;  // private
    uint32_t K = 0;  // window
    // activation
    std::shared_ptr<Tape> tape;
    std::shared_ptr<DevBuf> tape_d, phi_d, lv_tape_d, lv_start_d;
    bool linear() const { return kind == DASH_LAYER_DENSE || kind == DASH_LAYER_CONV2D; }
    uint64_t weight_count() const {
        if (kind == DASH_LAYER_DENSE) return (uint64_t)in_dim * out_dim;
        if (kind == DASH_LAYER_CONV2D) return (uint64_t)out_ch * in_ch * filter * filter;
        return 0;
    }
    uint64_t bias_count() const {
        if (kind == DASH_LAYER_DENSE) return out_dim;
        if (kind == DASH_LAYER_CONV2D) return out_ch;
        return 0;
    }
};

struct Network;
struct StreamWS;

}  // namespace dashgpu

struct dashgpu_circuit {
    int k = 8;
    std::vector<uint32_t> input_shape;
    double sign_target = 1.0, alpha = 1.0;
    std::vector<dashgpu::HLayer> layers;
    dashgpu::Crt base;
    bool needs_sign = false;
    dashgpu::SignCtx sign;
    std::shared_ptr<dashgpu::Tape> relu_tape, sign_tape;
    uint64_t n_in = 0, n_out = 0;
    uint64_t total_cts = 0, total_gates = 0, total_wires = 0, wire0 = 0;
    std::set<int> moduli;
    uint64_t relu_elements = 0, linear_macs = 0;
    std::vector<dash_layer_desc> desc_layers;  // for dashgpu_circuit_desc_view
    // dashgpu_infer caches: one workspace per stream, so concurrent streams
    // (host threads) run the same circuit without serializing on it
    struct Workspace {
        std::unique_ptr<dashgpu::Network> net;
        std::mutex mu;
    };
    std::map<void*, std::unique_ptr<Workspace>> workspaces;
    std::map<void*, std::shared_ptr<dashgpu::StreamWS>> stream_ws;  // dashgpu_infer_stream, per stream
    bool uploaded = false;  // per-layer device buffers created (upload_circuit)
    int device = -1;        // device the per-layer buffers live on
    // evaluator copy parsed from a GC (dashgpu_import_gc): private weights
    // withheld, so it can evaluate but not garble; sign spec taken from the GC
    bool eval_only = false;
    dashgpu::Spec gc_spec;
    std::mutex mu;
    ~dashgpu_circuit();
};

namespace dashgpu {

static void check_constants();

static uint64_t shape_size(const std::vector<uint32_t>& s) {
    uint64_t n = 1;
    for (auto x : s) n *= x;
    return n;
}

static uint32_t conv_extent(uint32_t in, uint32_t f, uint32_t s) {
    if (f == 0 || s == 0 || f > in) throw DataError("convolution filter does not fit the input");
    return (in - f) / s + 1;
}

// layer_out_shape (layer.cpp:320-344)
static std::vector<uint32_t> out_shape_of(const HLayer& l, const std::vector<uint32_t>& in) {
    switch (l.kind) {
        case DASH_LAYER_DENSE:
            if (in.size() != 1 || in[0] != l.in_dim) throw DataError("dense layer input shape mismatch");
            return {l.out_dim};
        case DASH_LAYER_CONV2D:
            if (in.size() != 3 || in[0] != l.in_ch) throw DataError("conv layer input shape mismatch");
            return {l.out_ch, conv_extent(in[1], l.filter, l.stride), conv_extent(in[2], l.filter, l.stride)};
        case DASH_LAYER_RELU:
        case DASH_LAYER_SIGNACT:
        case DASH_LAYER_ADD:
            return in;
        case DASH_LAYER_FLATTEN:
            return {(uint32_t)shape_size(in)};
        case DASH_LAYER_PAD2D:
            if (in.size() != 3) throw DataError("pad layer needs a [C][H][W] input");
            return {in[0], in[1] + 2 * l.pad, in[2] + 2 * l.pad};
    }
    throw DataError("unknown layer kind");
}

// index of a layer's DAG source in the per-layer value list (0 = circuit
// input, j + 1 = output of layer j); src 0 = previous layer (reference chain)
static size_t src_index(size_t li, int src) { return src == 0 ? li : (src < 0 ? 0 : (size_t)src); }

static std::shared_ptr<DevBuf> upload(const void* data, size_t bytes) {
    auto b = std::make_shared<DevBuf>();
    b->ensure(bytes ? bytes : 16);
    dev::h2d(b->p, data, bytes, g_stream);
    return b;
}

static int64_t resid(int64_t w, int p) { return ((w % p) + p) % p; }

// Tensor-core operands of a public linear layer (tc_linear.cuh): expanded
// weights W'[(lane, oc, j')][(i, j)] = wres[oc][i] if j == j', zero padded to
// whole 128-byte K stages and N tiles, and the im2col window offsets
// koff[i] = ic*H*W + ky*W + kx (dense: i).
// tc_linear_exp.cuh: rows (b, w, pos), K' = (window index, digit byte), the
// weight residues expanded block-diagonally over the four digit bytes
static void build_tc_linear_exp(HLayer& l, int k) {
    const bool dense = l.kind == DASH_LAYER_DENSE;
    const uint32_t nout = dense ? l.out_dim : l.out_ch, K = l.K;
    TcLinear& T = l.tc;
    T.mode = TcLinear::EXPANDED;
    T.fold = 0;
    T.k = (uint32_t)k;
    T.nout = nout;
    T.kblocks = (K + 31) / 32;
    T.Kpad = T.kblocks * 128;
    const uint32_t n4 = 4 * nout;
    T.BN = n4 <= 32 ? 32 : n4 <= 64 ? 64 : n4 <= 128 ? 128 : 256;
    T.Npad = (n4 + T.BN - 1) / T.BN * T.BN;
    l.wexp_h.assign((size_t)k * T.Npad * T.Kpad, 0);
    const uint64_t M = l.E_out;
    for (int i = 0; i < k; ++i) {
        const std::vector<uint8_t>& wr = l.wres_h[i];
        for (uint32_t oc = 0; oc < nout; ++oc)
            for (uint32_t j = 0; j < 4; ++j) {
                uint8_t* row = &l.wexp_h[((size_t)i * T.Npad + 4 * oc + j) * T.Kpad];
                for (uint32_t kw = 0; kw < K; ++kw)
                    row[4 * kw + j] = dense ? wr[(uint64_t)kw * M + oc] : wr[(uint64_t)oc * K + kw];
            }
    }
    l.koff_h.assign((size_t)T.kblocks * 32, -1);
    for (uint32_t kw = 0; kw < K; ++kw) {
        if (dense) {
            l.koff_h[kw] = (int32_t)kw;
        } else {
            const uint32_t f = l.filter, ic = kw / (f * f), ky = (kw / f) % f, kx = kw % f;
            l.koff_h[kw] = (int32_t)((ic * l.in_shape[1] + ky) * l.in_shape[2] + kx);
        }
    }
}

static void build_tc_linear(HLayer& l, int k) {
    // convolutions and dense layers over unaligned planes: the expanded-digit
    // kernel (whole-word window gathers); aligned dense layers: the digit-row
    // kernel (no expansion)
    const bool dense = l.kind == DASH_LAYER_DENSE;
    if (!dense || l.K % 4 != 0) {
        build_tc_linear_exp(l, k);
        return;
    }
    // tc_linear.cuh: per lane a plain [Npad][Kpad] u8 K-major weight-residue
    // matrix (row oc, column = window index i), all lanes stacked
    const uint32_t nout = dense ? l.out_dim : l.out_ch, K = l.K;
    TcLinear& T = l.tc;
    T.mode = TcLinear::DIGIT_ROWS;
    T.k = (uint32_t)k;
    T.nout = nout;
    // zero-wire and bias terms folded into the contraction as two extra
    // window columns (A: the zero label / R_p digits of the row's inference,
    // B: z_oc and p - b_oc) when the u32 accumulator provably stays below
    // 2^31: then sum mod p equals the reference's (acc mod p + z zero - b R)
    // mod p (layer.cpp:177-188) and the epilogue is one reduction per digit
    // Folding is kept for small windows (K <= 64, several row tiles per
    // stage, cp.async window copies); larger windows load their window words
    // by TMA straight from the plane, where the extra columns cannot come from.
    T.fold = K <= 64;
    for (int i = 0; i < k; ++i) {
        const uint64_t p = (uint64_t)l.tc_primes[i];
        if ((uint64_t)(K + 2) * (p - 1) * (p - 1) >= (1ull << 31)) T.fold = 0;
    }
    const uint32_t Keff = K + (T.fold ? 2 : 0);
    T.kblocks = (Keff + 127) / 128;
    T.Kpad = T.kblocks * 128;
    static const uint32_t bn_max = [] {  // tuning: DASH_TC_BNMAX=128 caps the column tile
        const char* e = std::getenv("DASH_TC_BNMAX");
        return (e && std::atoi(e) == 128) ? 128u : 256u;
    }();
    T.BN = nout <= 16 ? 16 : nout <= 32 ? 32 : nout <= 64 ? 64 : nout <= 128 ? 128 : bn_max;
    T.Npad = (nout + T.BN - 1) / T.BN * T.BN;
    for (int i = 0; i < k; ++i) {  // the epilogue reads z / bias residues a column tile at a time
        l.zt_h[i].resize(std::max<size_t>(l.zt_h[i].size(), T.Npad), 0);
        l.bres_h[i].resize(std::max<size_t>(l.bres_h[i].size(), T.Npad), 0);
    }
    l.wexp_h.assign((size_t)k * T.Npad * T.Kpad, 0);
    const uint64_t M = l.E_out;
    for (int i = 0; i < k; ++i) {
        const std::vector<uint8_t>& wr = l.wres_h[i];
        for (uint32_t oc = 0; oc < nout; ++oc) {
            uint8_t* row = &l.wexp_h[((size_t)i * T.Npad + oc) * T.Kpad];
            for (uint32_t kw = 0; kw < K; ++kw) row[kw] = dense ? wr[(uint64_t)kw * M + oc] : wr[(uint64_t)oc * K + kw];
            if (T.fold) {
                const uint32_t p = (uint32_t)l.tc_primes[i], b = l.bres_h[i][oc];
                row[K] = l.zt_h[i][oc];                   // x z_oc the zero-wire label
                row[K + 1] = (uint8_t)(b ? p - b : 0u);  // x (p - b_oc) R_p (garbler; the evaluator's column is 0)
            }
        }
    }
    l.koff_h.assign((size_t)T.kblocks * 128, -1);
    if (T.fold) {
        l.koff_h[K] = -2;      // the zero-wire label word of the row's inference
        l.koff_h[K + 1] = -3;  // R_p word (garbler), 0 (evaluator)
    }
    for (uint32_t kw = 0; kw < K; ++kw) {
        if (dense) {
            l.koff_h[kw] = (int32_t)kw;
        } else {
            const uint32_t f = l.filter, ic = kw / (f * f), ky = (kw / f) % f, kx = kw % f;
            l.koff_h[kw] = (int32_t)((ic * l.in_shape[1] + ky) * l.in_shape[2] + kx);
        }
    }
}

// validate_circuit + circuit_layout + per-layer residues and tapes (host only;
// device copies are made lazily by upload_circuit at the first garble)
static void prepare_circuit(dashgpu_circuit& c) {
    c.uploaded = false;
    c.base = crt_base(c.k);
    if (c.input_shape.empty() || c.input_shape.size() > 8 || shape_size(c.input_shape) == 0)
        throw DataError("circuit has an empty input shape");
    c.n_in = shape_size(c.input_shape);
    std::vector<std::vector<uint32_t>> shapes{c.input_shape};
    c.needs_sign = false;
    for (size_t li = 0; li < c.layers.size(); ++li) {
        auto& l = c.layers[li];
        if (l.kind < 1 || l.kind > 7) throw DataError("bad layer kind");
        if (l.src > (int)li || l.src < -1 || l.src2 > (int)li || l.src2 < -1 || (l.kind == DASH_LAYER_ADD && !l.src2))
            throw DataError("layer input refers to a later layer");
        l.in_shape = shapes[src_index(li, l.src)];
        l.out_shape = out_shape_of(l, l.in_shape);
        if (l.kind == DASH_LAYER_ADD && shapes[src_index(li, l.src2)] != l.in_shape)
            throw DataError("add operands differ in shape");
        l.E_in = shape_size(l.in_shape);
        l.E_out = shape_size(l.out_shape);
        if (l.linear()) {
            if (c.eval_only && l.priv && l.w.empty()) l.w.assign(l.weight_count(), 0);  // never read by evaluation
            if (l.w.size() != l.weight_count()) throw DataError("circuit must be quantized before garbling");
            if (!l.bias.empty() && l.bias.size() != l.bias_count()) throw DataError("quantized bias count mismatch");
        }
        if (l.kind == DASH_LAYER_RELU || l.kind == DASH_LAYER_SIGNACT) c.needs_sign = true;
        shapes.push_back(l.out_shape);
    }
    c.n_out = shape_size(shapes.back());
    if (c.n_in > (1u << 26) || c.n_out > (1u << 26)) throw DataError("tensor too large");
    if (c.needs_sign) {
        if (c.eval_only && c.gc_spec.empty()) throw DataError("garbled circuit lacks a sign spec");
        c.sign = make_sign(c.base, c.gc_spec.empty() ? choose_spec(c.base, c.sign_target) : c.gc_spec);
        c.relu_tape = std::make_shared<Tape>(build_tape(DASH_LAYER_RELU, c.base, c.sign));
        c.sign_tape = std::make_shared<Tape>(build_tape(DASH_LAYER_SIGNACT, c.base, c.sign));
    }
    const int k = c.k;
    c.wire0 = (uint64_t)k * (1 + c.n_in);
    uint64_t g = 0, w = c.wire0, ct = 0;
    c.moduli.clear();
    for (int p : c.base.primes) c.moduli.insert(p);
    c.relu_elements = 0;
    c.linear_macs = 0;
    for (auto& l : c.layers) {
        l.gate_base = g;
        l.wire_base = w;
        l.ct_base = ct;
        l.cts = l.gates = l.wires = 0;
        l.wres_h.clear();
        l.wexp_h.clear();
        l.koff_h.clear();
        l.zt_h.clear();
        l.bres_h.clear();
        l.lane_ct_off.clear();
        l.lane_gate_off.clear();
        l.lane_wire_off.clear();
        if (l.linear()) {
            const bool dense = l.kind == DASH_LAYER_DENSE;
            l.K = dense ? l.in_dim : l.in_ch * l.filter * l.filter;
            const uint64_t M = l.E_out;
            const uint64_t nrow = dense ? M : l.out_ch;
            for (int i = 0; i < k; ++i) {
                const int p = c.base.primes[i];
                if (!l.priv) {
                    std::vector<uint8_t> wr(l.w.size()), zt(nrow), br(nrow);
                    for (uint64_t row = 0; row < nrow; ++row) {
                        uint32_t z = 0;
                        for (uint32_t j = 0; j < l.K; ++j) {
                            const int64_t wv = resid(l.w[row * l.K + j], p);
                            if (wv == 0) ++z;
                            if (dense) wr[(uint64_t)j * M + row] = (uint8_t)wv;
                            else wr[row * l.K + j] = (uint8_t)wv;
                        }
                        zt[row] = (uint8_t)(z % (uint32_t)p);
                        br[row] = (uint8_t)resid(l.bias.empty() ? 0 : l.bias[row], p);
                    }
                    l.wres_h.push_back(std::move(wr));
                    l.zt_h.push_back(std::move(zt));
                    l.bres_h.push_back(std::move(br));
                    if (i == k - 1) {
                        l.tc_primes = c.base.primes;
                        build_tc_linear(l, k);
                    }
                } else {
                    std::vector<uint8_t> wr(l.w.size()), br(nrow);
                    for (uint64_t row = 0; row < nrow; ++row) {
                        for (uint32_t j = 0; j < l.K; ++j) wr[row * l.K + j] = (uint8_t)resid(l.w[row * l.K + j], p);
                        br[row] = (uint8_t)resid(l.bias.empty() ? 0 : l.bias[row], p);
                    }
                    l.wres_h.push_back(std::move(wr));
                    l.bres_h.push_back(std::move(br));
                    // count_layer order (layer.cpp:393-404): lane after lane
                    l.lane_ct_off.push_back(l.cts);
                    l.lane_gate_off.push_back(l.gates);
                    l.lane_wire_off.push_back(l.wires);
                    l.cts += (uint64_t)l.K * p * M;
                    l.gates += (uint64_t)l.K * M;
                    l.wires += (uint64_t)l.K * M;
                }
            }
        } else if (l.kind == DASH_LAYER_RELU || l.kind == DASH_LAYER_SIGNACT) {
            l.tape = l.kind == DASH_LAYER_RELU ? c.relu_tape : c.sign_tape;
            l.cts = l.tape->cts * l.E_out;
            l.gates = l.tape->gates * l.E_out;
            l.wires = l.tape->wires * l.E_out;
            for (int m : l.tape->moduli) c.moduli.insert(m);
            c.relu_elements += l.E_out;
        }
        g += l.gates;
        w += l.wires;
        ct += l.cts;
    }
    c.linear_macs = 0;  // digit multiply-accumulates of the public linear lanes
    for (auto& l : c.layers)
        if (l.linear() && !l.priv) {
            uint64_t sum_n = 0;
            for (int p : c.base.primes) sum_n += (uint64_t)n_digits_host(p);
            c.linear_macs += (uint64_t)l.K * l.E_out * sum_n;
        }
    c.total_cts = ct;
    c.total_gates = g;
    c.total_wires = w - c.wire0;
}

static void upload_circuit(dashgpu_circuit& c) {
    check_constants();
    if (c.uploaded) {
        if (c.device != dev::get_device())
            throw DataError("circuit parameters live on device " + std::to_string(c.device) +
                            "; build one circuit per device");
        return;
    }
    for (auto& l : c.layers) {
        l.wres.clear();
        l.zt.clear();
        l.bres.clear();
        for (auto& v : l.wres_h) l.wres.push_back(upload(v.data(), v.size()));
        for (auto& v : l.zt_h) l.zt.push_back(upload(v.data(), v.size()));
        for (auto& v : l.bres_h) l.bres.push_back(upload(v.data(), v.size()));
        if (!l.wexp_h.empty()) {
            l.wexp = upload(l.wexp_h.data(), l.wexp_h.size());
            l.koff = upload(l.koff_h.data(), l.koff_h.size() * sizeof(int32_t));
            l.tc.wexp = l.wexp->as<uint8_t>();
            l.tc.koff = l.koff->as<int32_t>();
            make_weight_map(l.tc);
        }
        if (l.tape) {
            l.tape_d = upload(l.tape->ops.data(), l.tape->ops.size() * sizeof(TapeOp));
            l.phi_d = upload(l.tape->phi.data(), l.tape->phi.size());
            l.lv_tape_d = upload(l.tape->lv_ops.data(), l.tape->lv_ops.size() * sizeof(TapeOp));
            l.lv_start_d = upload(l.tape->lv_start.data(), l.tape->lv_start.size() * sizeof(uint16_t));
        }
    }
    dev::sync(g_stream);
    c.device = dev::get_device();
    c.uploaded = true;
}

// ================================================================ network

struct Lanes {
    std::vector<std::unique_ptr<DevBuf>> lane;  // [k] of [B][nw][E] u32
    uint64_t E = 0;
    void ensure(const Crt& b, uint32_t B, uint64_t E_) {
        E = E_;
        lane.resize(b.k);
        for (int i = 0; i < b.k; ++i) {
            if (!lane[i]) lane[i] = std::make_unique<DevBuf>();
            const uint64_t nw = (n_digits_host(b.primes[i]) + 3) / 4;
            lane[i]->ensure((size_t)B * nw * E * 4);
        }
    }
};

struct Network {
    dashgpu_circuit* c = nullptr;
    uint32_t B = 0, cap = 0;
    DevBuf seeds_d, rk, mult, zero, Rb, commit, blob, dec, vals, resid, err, slots, mmlab, outv;
    Lanes base;  // encoding info: input base labels
    // per-layer output planes (garbler: base labels, evaluator: active labels);
    // at[j + 1] = output of layer j, at[0] = the input; Flatten aliases its input
    struct Outs {
        std::vector<std::unique_ptr<Lanes>> own;
        std::vector<const Lanes*> at;
    } gouts, eouts;
    std::unique_ptr<struct Bundle> bin, bout;  // dashgpu_infer's cached bundles
    // garbling of every activation layer is one launch over these
    std::vector<ActParams> act_host;
    // launch parameters: [0, nact) the garbling launch, [nact + li) the
    // evaluation launch of layer li; staged through pinned memory so that
    // enqueueing never blocks the host on the stream
    DevBuf act_dev;
    HostBuf act_pin, rk_pin, res_pin, err_pin;
    size_t act_cap = 0, nact = 0;
    // work-queue state of this network's persistent kernels
    DevBuf qctr, qflags;
    Sched sched() const {
        Sched q;
        q.counter = qctr.as<uint32_t>();
        q.flags = qflags.as<uint32_t>();
        q.flags_cap = qflags.n / 4;
        return q;
    }
    // dashgpu_network_release_gc: ciphertexts, gadget slots and layer planes
    // freed once the GC has been exported; encoding and decoding remain
    bool gc_released = false;
    void require_gc() const {
        if (gc_released) throw DataError("garbled circuit already released (dashgpu_network_release_gc)");
    }
    // Layer-windowed garbling (infer_layerwise, garble_digest_into): `blob`
    // holds one layer's rows for the batch at a time, [B][layer cts], instead
    // of whole GCs [B][total_cts]
    bool windowed = false;
    // host-resident GC (dashgpu_import_gc_host): rows in the reference's cts
    // order, [B][total_cts] in pinned memory, moved to the window layer by
    // layer during evaluation
    bool host_gc = false;
    HostBuf hblob;
    size_t act_flushed = 0;  // activation layers whose garbling launch is enqueued
    // dashgpu_infer's last sub-batch plan (batch size -> sub-batch, schedule)
    uint32_t plan_batch = 0, plan_chunk = 0;
    bool plan_layerwise = false;
    U4* layer_blob(const HLayer& l) const { return blob.as<U4>() + (windowed ? 0 : l.ct_base); }
    uint64_t layer_blob_stride(const HLayer& l) const { return windowed ? l.cts : c->total_cts; }
    size_t slot_used = 0;  // U4 entries of `slots` handed out to garbled layers
    size_t mm_used = 0;    // U4 entries of `mmlab` handed out to garbled layers
    uint64_t mult_stride = 0;
    uint32_t sum_p = 0;
};

struct Bundle {
    Network* net = nullptr;
    uint32_t B = 0;
    bool output = false;
    Lanes lanes;
};

static void make_lane_ptrs(const Lanes& L, int k, const uint32_t** out) {
    for (int i = 0; i < k; ++i) out[i] = L.lane[i]->as<uint32_t>();
}

static void fill_primes(const Crt& b, uint16_t* out) {
    for (int i = 0; i < b.k; ++i) out[i] = (uint16_t)b.primes[i];
}

// Splits an element's tape into K op ranges of similar garbling cost (rows +
// PRF blocks); the garbling launch runs chunk c of every element as its own
// work item (kernels_act.cu), which keeps the launch's last wave short.
static void fill_chunks(ActParams& P, const Tape& T, int K) {
    const size_t n = T.ops.size();
    std::vector<double> cum(n + 1, 0.0);
    for (size_t i = 0; i < n; ++i) {
        const TapeOp& o = T.ops[i];
        const double pb = (n_digits_host(o.pm) + 3) / 4, qb = (n_digits_host(o.qm ? o.qm : 2) + 3) / 4;
        double c = 0.05;
        switch (o.kind) {
            case OP_PROJ: c = o.pm + qb; break;
            case OP_GRR: c = o.pm; break;
            case OP_HALF: c = 2.0 * o.pm + 2 * pb; break;
            case OP_MMHALF: c = o.pm + 2.0 * o.qm + 2 * pb; break;
            default: break;
        }
        cum[i + 1] = cum[i] + c;
    }
    K = std::max(1, std::min<int>(K, MAXCHUNK));
    P.chunk_op[0] = 0;
    size_t at = 0;
    for (int c = 1; c < K; ++c) {
        const double target = cum[n] * c / K;
        while (at < n && cum[at] < target) ++at;
        while (at < n && T.ops[at].kind == OP_ADDACC) ++at;  // never split a fused add chain
        P.chunk_op[c] = (uint16_t)std::max<size_t>(at, P.chunk_op[c - 1]);
    }
    for (int c = K; c <= MAXCHUNK; ++c) P.chunk_op[c] = (uint16_t)n;
}
// chunks per element tape in the garbling launch (DASH_TAPE_CHUNKS overrides, for tuning)
static int tape_chunks() {
    static int k = [] {
        const char* v = std::getenv("DASH_TAPE_CHUNKS");
        return v ? std::max(1, std::min(MAXCHUNK, std::atoi(v))) : 8;
    }();
    return k;
}

// Runs one layer over B inferences.  garbler: base labels; else active.
// in2: second operand of the Add extension.
// level-parallel garbling of an activation layer of `elements` (B x E)
static bool act_lv_ok(const Tape&, uint64_t elements) { return dev::garble_lv_warps(elements) >= 2; }
static int act_slots(const Tape& T, bool lv) { return lv ? std::max(T.nslots, T.nslots_lv) : T.nslots; }

static void run_layer(Network& n, size_t li, const HLayer& l, bool garbler, const Lanes& in, const Lanes* in2,
                      Lanes& out) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    out.ensure(c.base, n.B, l.E_out);
    if (l.kind == DASH_LAYER_PAD2D || l.kind == DASH_LAYER_ADD) {
        PadAddParams P;
        std::memset(&P, 0, sizeof P);
        P.add = l.kind == DASH_LAYER_ADD;
        P.B = n.B;
        P.E_out = (uint32_t)l.E_out;
        if (!P.add) {
            P.C = l.in_shape[0];
            P.H = l.in_shape[1];
            P.W = l.in_shape[2];
            P.pad = l.pad;
            P.OH = l.out_shape[1];
            P.OW = l.out_shape[2];
        }
        P.k = k;
        fill_primes(c.base, P.primes);
        for (int i = 0; i < k; ++i) {
            P.wbase[i + 1] = P.wbase[i] + (uint32_t)(n_digits_host(c.base.primes[i]) + 3) / 4;
            P.in[i] = in.lane[i]->as<uint32_t>();
            P.in2[i] = in2 ? in2->lane[i]->as<uint32_t>() : nullptr;
            P.out[i] = out.lane[i]->as<uint32_t>();
        }
        P.zero = n.zero.as<uint32_t>();
        launch_pad_add(P, g_stream);
        return;
    }
    if (l.linear() && !l.priv) {
        LinParams Ls[MAXK];
        for (int i = 0; i < k; ++i) {
            LinParams& L = Ls[i];
            std::memset(&L, 0, sizeof L);
            L.conv = l.kind == DASH_LAYER_CONV2D;
            L.K = l.K;
            L.M = (uint32_t)l.E_out;
            L.E_in = (uint32_t)l.E_in;
            if (L.conv) {
                L.in_ch = l.in_ch;
                L.H = l.in_shape[1];
                L.W = l.in_shape[2];
                L.f = l.filter;
                L.stride = l.stride;
                L.OH = l.out_shape[1];
                L.OW = l.out_shape[2];
            }
            L.wres = l.wres[i]->as<uint8_t>();
            L.zt = l.zt[i]->as<uint8_t>();
            L.bres = l.bres[i]->as<uint8_t>();
            L.in = in.lane[i]->as<uint32_t>();
            L.out = out.lane[i]->as<uint32_t>();
            L.zero = n.zero.as<uint32_t>() + (uint64_t)i * LABW;
            L.R = n.Rb.as<uint32_t>() + (uint64_t)i * LABW;
            L.p = (uint32_t)c.base.primes[i];
            L.n = (uint32_t)n_digits_host(L.p);
            L.nw = (L.n + 3) / 4;
            magic31(L.p, L.mag, L.sh);
            L.B = n.B;
            L.zstride = (uint32_t)(k * LABW);  // zero / R rows are [B][k][LABW]
            L.garbler = garbler;
        }
        launch_linear(Ls, k, l.tc, g_stream);
        return;
    }
    if (l.linear()) {
        for (int i = 0; i < k; ++i) {
            PrivParams P;
            std::memset(&P, 0, sizeof P);
            P.conv = l.kind == DASH_LAYER_CONV2D;
            P.win = l.K;
            P.M = (uint32_t)l.E_out;
            P.E_in = (uint32_t)l.E_in;
            if (P.conv) {
                P.in_ch = l.in_ch;
                P.H = l.in_shape[1];
                P.W = l.in_shape[2];
                P.f = l.filter;
                P.stride = l.stride;
                P.OH = l.out_shape[1];
                P.OW = l.out_shape[2];
            }
            P.wres = l.wres[i]->as<uint8_t>();
            P.bres = l.bres[i]->as<uint8_t>();
            P.in = in.lane[i]->as<uint32_t>();
            P.out = out.lane[i]->as<uint32_t>();
            P.p = (uint32_t)c.base.primes[i];
            P.B = n.B;
            P.gate_base = l.gate_base + l.lane_gate_off[i];
            P.wire_base = l.wire_base + l.lane_wire_off[i];
            P.blob = n.layer_blob(l) + l.lane_ct_off[i];
            P.blob_stride = n.layer_blob_stride(l);
            P.rk = n.rk.as<uint32_t>();
            P.mult = n.mult.as<uint32_t>();
            P.mult_stride = n.mult_stride;
            P.garbler = garbler;
            launch_private(P, g_stream, n.sched());
        }
        return;
    }
    ActParams P;
    std::memset(&P, 0, sizeof P);
    P.tape = l.tape_d->as<TapeOp>();
    P.n_ops = (int)l.tape->ops.size();
    P.lv_tape = l.lv_tape_d->as<TapeOp>();
    P.lv_start = l.lv_start_d->as<uint16_t>();
    P.n_levels = (int)l.tape->lv_start.size() - 1;
    fill_chunks(P, *l.tape, tape_chunks());
    P.phi = l.phi_d->as<uint8_t>();
    P.k = k;
    P.E = (uint32_t)l.E_out;
    P.B = n.B;
    P.gate_base = l.gate_base;
    P.wire_base = l.wire_base;
    P.uc_cts = l.tape->cts;
    P.uc_gates = l.tape->gates;
    P.uc_wires = l.tape->wires;
    P.blob = n.layer_blob(l);
    P.blob_stride = n.layer_blob_stride(l);
    for (int i = 0; i < k; ++i) {
        P.out[i] = out.lane[i]->as<uint32_t>();
        P.out_kind[i] = l.tape->out_kind[i];
        P.out_wire[i] = l.tape->out_wire[i];
    }
    P.rk = n.rk.as<uint32_t>();
    P.mult = n.mult.as<uint32_t>();
    P.mult_stride = n.mult_stride;
    if (garbler) {
        // a layer small enough for level-parallel garbling gets room for the
        // level tape's slots too (kernels_act.cu act_lv_garble_kernel)
        const bool lv = act_lv_ok(*l.tape, (uint64_t)n.B * l.E_out);
        const size_t slot_words = (size_t)act_slots(*l.tape, lv) * n.B * l.E_out;
        P.lv_ok = lv;
        // Inputs (per-layer planes) stay resident until the combined tape
        // launch; the outputs (pure PRF functions) are written now so the
        // next layer can proceed.
        for (int i = 0; i < k; ++i) P.in[i] = in.lane[i]->as<uint32_t>();
        P.slots = n.slots.as<U4>() + n.slot_used;
        n.slot_used += slot_words;
        P.mmlab = n.mmlab.as<U4>() + n.mm_used;
        n.mm_used += (size_t)n.B * l.E_out * k * 2;
        uint16_t primes[MAXK];
        fill_primes(c.base, primes);
        launch_act_outputs(P, primes, g_stream);
        n.act_host.push_back(P);
        return;
    }
    for (int i = 0; i < k; ++i) P.in[i] = in.lane[i]->as<uint32_t>();
    P.slots = n.slots.as<U4>();
    ActParams* pin = n.act_pin.as<ActParams>() + n.nact + li;
    ActParams* dp = n.act_dev.as<ActParams>() + n.nact + li;
    *pin = P;
    dev::h2d(dp, pin, sizeof P, g_stream);
    launch_act_multi(dp, pin, 1, false, g_stream, n.sched());
}

static uint64_t max_layer_cts(const dashgpu_circuit& c) {
    uint64_t m = 0;
    for (const auto& l : c.layers) m = std::max<uint64_t>(m, l.cts);
    return m;
}

static void network_reserve(Network& n, uint32_t B, bool windowed = false) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    n.windowed = windowed;
    // ciphertexts, gadget slots and mixed-modulus labels: every layer's
    // region at once, or (windowed) the largest layer's, reused layer by
    // layer.  Sized before the early return: they depend on the schedule.
    n.blob.ensure((size_t)B * std::max<uint64_t>(windowed ? max_layer_cts(c) : c.total_cts, 1) * 16);
    {
        size_t slot_total = 0, slot_eval = 0, mm_total = 0;
        for (const auto& l : c.layers)
            if (l.tape) {
                const size_t sl = (size_t)act_slots(*l.tape, act_lv_ok(*l.tape, (uint64_t)B * l.E_out)) * B * l.E_out;
                const size_t mm = (size_t)B * l.E_out * k * 2;
                slot_total = windowed ? std::max(slot_total, sl) : slot_total + sl;
                mm_total = windowed ? std::max(mm_total, mm) : mm_total + mm;
                // warp-per-element evaluation of a small layer uses the level tape's slots
                if ((uint64_t)B * l.E_out <= dev::lane_group_eval_max())
                    slot_eval = std::max(slot_eval, (size_t)l.tape->nslots_lv * B * l.E_out);
            }
        n.slots.ensure(std::max<size_t>(std::max(slot_total, slot_eval), 1) * 16);
        n.mmlab.ensure(std::max<size_t>(mm_total, 1) * 16);
    }
    if (B <= n.cap && n.cap) {
        n.B = B;
        return;
    }
    n.cap = B;
    n.B = B;
    n.mult_stride = (uint64_t)(MAXMOD - 1) * 128 * NWMAX;
    n.seeds_d.ensure((size_t)B * 16);
    n.rk.ensure((size_t)B * 44 * 4);
    n.mult.ensure((size_t)B * n.mult_stride * 4);
    n.zero.ensure((size_t)B * k * LABW * 4);
    n.Rb.ensure((size_t)B * k * LABW * 4);
    n.commit.ensure((size_t)B * 16);
    n.sum_p = 0;
    for (int p : c.base.primes) n.sum_p += (uint32_t)p;
    n.dec.ensure((size_t)B * c.n_out * n.sum_p * 16);
    n.vals.ensure((size_t)B * std::max(c.n_in, c.n_out) * 8);
    n.resid.ensure((size_t)B * c.n_out * k);
    n.err.ensure(16);
    n.base.ensure(c.base, B, c.n_in);
    size_t nact = 0;
    for (const auto& l : c.layers)
        if (l.tape) ++nact;
    n.nact = nact;
    n.act_cap = nact + c.layers.size();
    n.act_dev.ensure(n.act_cap * sizeof(ActParams));
    n.act_pin.ensure(n.act_cap * sizeof(ActParams));
    n.rk_pin.ensure((size_t)B * (44 * 4 + 16));
    n.res_pin.ensure((size_t)B * c.n_out * 8 + 16);
    n.outv.ensure((size_t)B * c.n_out * 8 + 16);
    n.err_pin.ensure(64);
    size_t items = 0;  // work items per tape chunk of the garbling launch
    for (const auto& l : c.layers)
        if (l.tape) items += (size_t)B * ((l.E_out + 31) / 32);
    n.qctr.ensure(64);
    n.qflags.ensure(std::max<size_t>(items, 1) * 4);
}

// All layers of the circuit in order (DAG inputs per layer, see
// dash_circuit_desc.h); returns the final output planes.
static void outs_begin(Network& n, bool garbler, const Lanes& input) {
    Network::Outs& O = garbler ? n.gouts : n.eouts;
    const size_t L = n.c->layers.size();
    O.own.resize(L + 1);
    O.at.assign(L + 1, nullptr);
    O.at[0] = &input;
}

static void run_layer_at(Network& n, bool garbler, size_t li) {
    Network::Outs& O = garbler ? n.gouts : n.eouts;
    const HLayer& l = n.c->layers[li];
    const Lanes* src = O.at[src_index(li, l.src)];
    if (l.kind == DASH_LAYER_FLATTEN) {  // metadata-only reshape: planes are already flat
        O.at[li + 1] = src;
        return;
    }
    if (!O.own[li + 1]) O.own[li + 1] = std::make_unique<Lanes>();
    const Lanes* src2 = l.kind == DASH_LAYER_ADD ? O.at[src_index(li, l.src2)] : nullptr;
    run_layer(n, li, l, garbler, *src, src2, *O.own[li + 1]);
    O.at[li + 1] = O.own[li + 1].get();
}

static const Lanes* run_layers(Network& n, bool garbler, const Lanes& input) {
    outs_begin(n, garbler, input);
    const size_t L = n.c->layers.size();
    for (size_t li = 0; li < L; ++li) run_layer_at(n, garbler, li);
    return (garbler ? n.gouts : n.eouts).at[L];
}

// garble (garble.cpp:134-240), batched: inference b uses seeds[b].
// garble_setup: offsets, multiples, zero-wire / input base labels, seed
// commitment (garble.cpp:134-204 before the layer loop).
static void garble_setup(Network& n, const uint8_t* seeds, uint32_t B, bool seeds_on_device, bool windowed = false) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    if (c.eval_only) throw DataError("circuit is an evaluator copy (private weights withheld): it cannot garble");
    upload_circuit(c);
    network_reserve(n, B, windowed);
    // seeds -> device, AES key schedules expanded on the device (no host
    // round trip when the seeds are already in HBM)
    if (seeds_on_device) {
        dev::d2d(n.seeds_d.p, seeds, 16 * (size_t)B, g_stream);
    } else {
        std::memcpy(n.rk_pin.p, seeds, 16 * (size_t)B);
        dev::h2d(n.seeds_d.p, n.rk_pin.p, 16 * (size_t)B, g_stream);
    }
    launch_expand(n.seeds_d.as<uint8_t>(), n.rk.as<uint32_t>(), B, g_stream);
    // zero / Rb rows are addressed per lane with stride LABW between inferences
    // in linear_thread; store them lane-major: [k][B][LABW]
    SetupParams S;
    std::memset(&S, 0, sizeof S);
    S.B = B;
    S.k = k;
    fill_primes(c.base, S.primes);
    S.nslot = 0;
    for (int m : c.moduli) S.slot_mod[S.nslot++] = (uint16_t)m;
    S.rk = n.rk.as<uint32_t>();
    S.seeds = n.seeds_d.as<uint8_t>();
    S.mult = n.mult.as<uint32_t>();
    S.mult_stride = n.mult_stride;
    S.n_in = (uint32_t)c.n_in;
    for (int i = 0; i < k; ++i) S.base_planes[i] = n.base.lane[i]->as<uint32_t>();
    S.zero = n.zero.as<uint32_t>();
    S.Rb = n.Rb.as<uint32_t>();
    S.commit = n.commit.as<U4>();
    launch_setup(S, g_stream);
    n.act_host.clear();
    n.act_flushed = 0;
    n.slot_used = 0;
    n.mm_used = 0;
}

// decoding tables (garble.cpp:208-231) from the final output base labels
static void garble_dectables(Network& n, const Lanes& fin) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    DecodeParams D;
    std::memset(&D, 0, sizeof D);
    D.B = n.B;
    D.n_out = (uint32_t)c.n_out;
    D.k = k;
    fill_primes(c.base, D.primes);
    D.poff[0] = 0;
    for (int i = 0; i < k; ++i) D.poff[i + 1] = (uint16_t)(D.poff[i] + c.base.primes[i]);
    make_lane_ptrs(fin, k, D.lanes);
    D.table = n.dec.as<U4>();
    D.mult = n.mult.as<uint32_t>();
    D.mult_stride = n.mult_stride;
    launch_dectable(D, g_stream);
}

// the deferred combined garbling launch of the activation layers recorded in act_host
static void garble_act_flush(Network& n) {
    if (n.act_host.empty()) return;
    // a layer-windowed garbling flushes once per activation layer: each flush
    // stages its parameters in its own pinned / device slot, since the async
    // copy of an earlier flush may not have run yet
    const size_t cnt = n.act_host.size();
    if (cnt > n.nact) throw std::logic_error("activation launch staging overflow");
    if (n.act_flushed + cnt > n.nact) {  // slots exhausted (layer API reuse): drain, then restart
        dev::sync(g_stream);
        n.act_flushed = 0;
    }
    const size_t at = n.act_flushed;
    ActParams* pin = n.act_pin.as<ActParams>() + at;
    ActParams* dp = n.act_dev.as<ActParams>() + at;
    std::memcpy(pin, n.act_host.data(), cnt * sizeof(ActParams));
    dev::h2d(dp, pin, cnt * sizeof(ActParams), g_stream);
    launch_act_multi(dp, n.act_host.data(), (int)cnt, true, g_stream, n.sched());
    n.act_flushed += cnt;
    n.act_host.clear();
    n.slot_used = 0;
    n.mm_used = 0;
}

static void garble_into(Network& n, const uint8_t* seeds, uint32_t B, bool seeds_on_device) {
    garble_setup(n, seeds, B, seeds_on_device);
    n.gc_released = false;
    // run the layers on the input base planes
    const Lanes* cur = run_layers(n, true, n.base);
    garble_act_flush(n);
    garble_dectables(n, *cur);
}

static void encode_enqueue(Network& n, const int64_t* values, bool on_device, Bundle& out) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    const int64_t* vd = values;
    if (!on_device) {
        dev::h2d(n.vals.p, values, (size_t)n.B * c.n_in * 8, g_stream);
        vd = n.vals.as<int64_t>();
    }
    out.net = &n;
    out.B = n.B;
    out.output = false;
    out.lanes.ensure(c.base, n.B, c.n_in);
    dev::memset0(n.err.p, 4, g_stream);
    EncodeParams P;
    std::memset(&P, 0, sizeof P);
    P.B = n.B;
    P.n_in = (uint32_t)c.n_in;
    P.k = k;
    fill_primes(c.base, P.primes);
    P.values = vd;
    for (int i = 0; i < k; ++i) {
        P.base[i] = n.base.lane[i]->as<uint32_t>();
        P.out[i] = out.lanes.lane[i]->as<uint32_t>();
    }
    P.mult = n.mult.as<uint32_t>();
    P.mult_stride = n.mult_stride;
    const u128 half_up = (c.base.P + 1) / 2, half_dn = c.base.P / 2;
    P.half_up_lo = (uint64_t)half_up;
    P.half_up_hi = (uint64_t)(half_up >> 64);
    P.half_dn_lo = (uint64_t)half_dn;
    P.half_dn_hi = (uint64_t)(half_dn >> 64);
    P.err = n.err.as<int>();
    launch_encode(P, g_stream);
    dev::d2h(n.err_pin.as<int>(), n.err.p, 4, g_stream);
}

static void encode_finish(Network& n) {
    if (n.err_pin.as<int>()[0]) throw DataError("encode_signed: value outside the representable range");
}

static void encode_into(Network& n, const int64_t* values, bool on_device, Bundle& out) {
    encode_enqueue(n, values, on_device, out);
    dev::sync(g_stream);
    encode_finish(n);
}

// copies the last layer's evaluator planes into the output bundle
static void eval_output(Network& n, const Lanes& cur, Bundle& out) {
    dashgpu_circuit& c = *n.c;
    out.net = &n;
    out.B = n.B;
    out.output = true;
    out.lanes.ensure(c.base, n.B, c.n_out);
    for (int i = 0; i < c.k; ++i)
        dev::d2d(out.lanes.lane[i]->p, cur.lane[i]->p,
                 (size_t)n.B * ((n_digits_host(c.base.primes[i]) + 3) / 4) * c.n_out * 4, g_stream);
}

// evaluate (garble.cpp:265-312)
static void evaluate_into(Network& n, const Bundle& in, Bundle& out) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    // evaluate's input checks (garble.cpp:265-280): a bundle of another
    // network or element count would make the kernels read out of bounds
    if (in.net != &n || in.B != n.B || in.output) throw DataError("garbled input bundle does not match the network");
    if (in.lanes.E != c.n_in || in.lanes.lane.size() != (size_t)k) throw DataError("garbled input shape mismatch");
    n.require_gc();
    if (n.host_gc) {  // host-resident GC: fill the window layer by layer
        outs_begin(n, false, in.lanes);
        DevBuf ref;
        ref.ensure(std::max<uint64_t>(max_layer_cts(c), 1) * 16);
        for (size_t li = 0; li < c.layers.size(); ++li) {
            const HLayer& l = c.layers[li];
            for (uint32_t b = 0; l.cts && b < n.B; ++b) {
                const U4* h = n.hblob.as<U4>() + (uint64_t)b * c.total_cts + l.ct_base;
                U4* w = n.blob.as<U4>() + (uint64_t)b * l.cts;
                if (!l.tape) {  // private-weight rows are stored in reference order
                    dev::h2d(w, h, l.cts * 16, g_stream);
                    continue;
                }
                dev::h2d(ref.p, h, l.cts * 16, g_stream);
                RowsPermuteParams P;
                P.src = ref.as<U4>();
                P.dst = w;
                P.E = l.E_out;
                P.uc = l.tape->cts;
                P.to_ref = 0;
                launch_rows_permute(P, g_stream);
            }
            run_layer_at(n, false, li);
        }
        eval_output(n, *n.eouts.at[c.layers.size()], out);
        return;
    }
    eval_output(n, *run_layers(n, false, in.lanes), out);
}

// Layer-windowed inference ("tables are streamed per
// layer chunk, not materialised whole"): layer li of the whole sub-batch is
// garbled into the window, evaluated from it, and the window is reused for
// li + 1.  Rows, labels and outputs are those of garble_into + evaluate_into
// (same kernels, same ids; only the row addresses change), but a pass holds
// B x (largest layer) ciphertexts instead of B x (whole GC), so batches whose
// GCs exceed HBM run in fewer, larger sub-batches.  The GC is never whole:
// the network cannot be exported afterwards.
static void infer_layerwise(Network& n, const uint8_t* seeds, uint32_t B, bool on_device, const int64_t* inputs,
                            Bundle& in, Bundle& out) {
    dashgpu_circuit& c = *n.c;
    garble_setup(n, seeds, B, on_device, true);
    n.gc_released = false;
    encode_enqueue(n, inputs, on_device, in);
    outs_begin(n, true, n.base);
    outs_begin(n, false, in.lanes);
    const size_t L = c.layers.size();
    for (size_t li = 0; li < L; ++li) {
        run_layer_at(n, true, li);
        garble_act_flush(n);
        run_layer_at(n, false, li);
    }
    garble_dectables(n, *n.gouts.at[L]);
    eval_output(n, *n.eouts.at[L], out);
    n.gc_released = true;
}

// Digest parity mode: garbles layer by layer into the
// window and reduces each layer's rows to the tree SHA-256 of sha256.hpp
// (the leaves on the device, read in the reference's cts order; the root on
// the host).  digests: [B][layers][32].  A layer's digest equals the one of
// the same layer's bytes in dashgpu_export_gc, so whole-GC parity at sizes
// that never fit HBM reduces to comparing 32 bytes per layer.
static void garble_digest_into(Network& n, const uint8_t* seeds, uint32_t B, uint8_t* digests) {
    dashgpu_circuit& c = *n.c;
    garble_setup(n, seeds, B, false, true);
    n.gc_released = false;
    outs_begin(n, true, n.base);
    const size_t L = c.layers.size();
    // leaf digests of one layer at a time, roots of every layer: [L][B][8]
    // words; one host sync for the whole network
    DevBuf leaves, roots;
    leaves.ensure(std::max<size_t>((size_t)B * ((max_layer_cts(c) + kDigestLeafRows - 1) / kDigestLeafRows), 1) * 32);
    roots.ensure(std::max<size_t>(L, 1) * B * 32);
    for (size_t li = 0; li < L; ++li) {
        run_layer_at(n, true, li);
        garble_act_flush(n);
        const HLayer& l = c.layers[li];
        DigestParams P;
        std::memset(&P, 0, sizeof P);
        P.src = n.blob.as<U4>();
        P.stride = l.cts;
        P.rows = l.cts;
        P.E = l.tape ? l.E_out : 0;
        P.uc = l.tape ? l.tape->cts : 0;
        P.B = B;
        P.leaves = (uint32_t)((l.cts + kDigestLeafRows - 1) / kDigestLeafRows);
        P.out = leaves.as<uint32_t>();
        launch_digest(P, roots.as<uint32_t>() + li * B * 8, g_stream);
    }
    std::vector<uint32_t> hr(L * B * 8);
    dev::d2h(hr.data(), roots.p, hr.size() * 4, g_stream);
    dev::sync(g_stream);
    for (size_t li = 0; li < L; ++li)
        for (uint32_t b = 0; b < B; ++b)
            for (int t = 0; t < 8; ++t)
                for (int q = 0; q < 4; ++q)
                    digests[((size_t)b * L + li) * 32 + 4 * t + q] = (uint8_t)(hr[(li * B + b) * 8 + t] >> (24 - 8 * q));
    n.gc_released = true;
}


// decode_outputs (garble.cpp:314-343): table lookup on the device (enqueued,
// residues + miss flag land in pinned memory), CRT reconstruction on the host
// CRT coefficients of the base, reduced mod P, as the device decode wants them
static void fill_crt(const Crt& base, DecodeParams& D) {
    for (int i = 0; i < base.k; ++i) {
        const u128 cf = base.coeffs[i] % base.P;
        D.coeff_lo[i] = (uint64_t)cf;
        D.coeff_hi[i] = (uint64_t)(cf >> 64);
    }
    D.P_lo = (uint64_t)base.P;
    D.P_hi = (uint64_t)(base.P >> 64);
}

// decode_outputs (garble.cpp:314-343) with crt_reconstruct / decode_signed
// (crt.cpp:63-101) on the device: values go straight to dev_values (device
// outputs) or to the network's buffer and a pinned host copy.
static void decode_enqueue(Network& n, const Bundle& outb, int64_t* dev_values = nullptr) {
    dashgpu_circuit& c = *n.c;
    const int k = c.k;
    if (outb.net != &n || !outb.output || outb.B != n.B) throw DataError("output lane count mismatch");
    if (outb.lanes.E != c.n_out || outb.lanes.lane.size() != (size_t)k)
        throw DataError("output element count mismatch");  // decode_outputs, garble.cpp:318-322
    DecodeParams D;
    std::memset(&D, 0, sizeof D);
    D.B = n.B;
    D.n_out = (uint32_t)c.n_out;
    D.k = k;
    fill_primes(c.base, D.primes);
    for (int i = 0; i < k; ++i) D.poff[i + 1] = (uint16_t)(D.poff[i] + c.base.primes[i]);
    make_lane_ptrs(outb.lanes, k, D.lanes);
    D.table = n.dec.as<U4>();
    D.residues = n.resid.as<uint8_t>();
    D.err = n.err.as<int>();
    D.values = dev_values ? dev_values : n.outv.as<int64_t>();
    fill_crt(c.base, D);
    dev::memset0(n.err.p, 4, g_stream);
    launch_decode(D, g_stream);
    if (!dev_values) dev::d2h(n.res_pin.p, n.outv.p, (size_t)n.B * c.n_out * 8, g_stream);
    dev::d2h(n.err_pin.as<int>() + 1, n.err.p, 4, g_stream);
}

static void decode_finish(Network& n, int64_t* values, bool values_on_device) {
    dashgpu_circuit& c = *n.c;
    const int err = n.err_pin.as<int>()[1];
    if (err == ST_AUTH) throw AuthError("output label not present in the decoding table");
    if (err) throw DataError("decode_signed: value exceeds 64-bit signed range");
    if (!values_on_device) std::memcpy(values, n.res_pin.p, (size_t)n.B * c.n_out * 8);
}

static void decode_into(Network& n, const Bundle& outb, int64_t* values, bool values_on_device) {
    decode_enqueue(n, outb, values_on_device ? values : nullptr);
    dev::sync(g_stream);
    decode_finish(n, values, values_on_device);
}

// Position in HBM of row j of element u of an activation layer, relative to
// the layer's first row (act_rows: 32-element blocks, row-major per block).
static uint64_t act_row_pos(uint64_t E, uint64_t uc, uint64_t u, uint64_t j) {
    const uint64_t blk = u >> 5, w = std::min<uint64_t>(32, E - (blk << 5));
    return blk * 32 * uc + j * w + (u & 31);
}

// ============================================================ streamed layers
//
// The label-ops sweep of SURVEY.md section 8(d) is one activation layer over N
// elements ({input_shape={N}, layers={relu()}}, bench_main.cpp:156-162); at
// N = 2^26, k = 8 its garbled tables are 1.8 TB, so they never exist at once.
// Element chunks [u0, u0 + C) are garbled, encoded, evaluated and decoded in
// turn with the reference's numbering: input wire k + e*k + i
// (garble.cpp:170), gate gate_base + u*uc.gates, wire wire_base + u*uc.wires,
// ciphertext u*uc.cts inside the layer (layer.cpp:531-541).  Every chunk
// buffer is C elements wide; only the id bases move.
struct StreamWS {
    DevBuf rk, seeds, mult, zero, Rb, commit, blob, slots, dec, vals, resid, err, actp, qctr, qflags, mmlab, outv;
    Lanes base, in, gout, eout;
    uint64_t C = 0;  // chunk capacity (elements) the buffers are sized for
    // host staging, double-buffered: chunk i's inputs / decoded outputs go
    // through slot i & 1; the host touches a slot only after the event of
    // the chunk that used it two chunks earlier (no per-chunk stream sync)
    HostBuf in_pin[2], out_pin[2], act_pin, par_pin;
    void* ev[2] = {nullptr, nullptr};
    int64_t* pend_dst[2] = {nullptr, nullptr};
    uint32_t pend_n[2] = {0, 0};
    ~StreamWS() {
        for (void* e : ev) dev::event_destroy(e);
    }
};

static bool streamable(const dashgpu_circuit& c) {
    return c.layers.size() == 1 && c.layers[0].tape != nullptr;
}

// Workspace of (circuit, stream), sized once for chunks of C elements and
// reused by every later call (the sweep's timed calls allocate nothing).
static StreamWS& stream_ws(dashgpu_circuit& c, uint64_t C) {
    auto& slot = c.stream_ws[g_stream];
    if (slot && slot->C >= C) return *slot;
    slot.reset();  // free the smaller workspace before allocating the larger one
    auto w = std::make_shared<StreamWS>();
    const int k = c.k;
    const Tape& T = *c.layers[0].tape;
    const uint64_t mult_stride = (uint64_t)(MAXMOD - 1) * 128 * NWMAX;
    uint32_t sum_p = 0;
    for (int p : c.base.primes) sum_p += (uint32_t)p;
    w->C = C;
    w->rk.ensure(44 * 4);
    w->seeds.ensure(16);
    w->mult.ensure(mult_stride * 4);
    w->zero.ensure((size_t)k * LABW * 4);
    w->Rb.ensure((size_t)k * LABW * 4);
    w->commit.ensure(16);
    w->blob.ensure((size_t)C * T.cts * 16);
    w->slots.ensure(std::max<size_t>((size_t)std::max(T.nslots, T.nslots_lv) * C, 1) * 16);
    w->dec.ensure((size_t)C * sum_p * 16);
    w->vals.ensure((size_t)2 * C * 8);
    w->resid.ensure((size_t)C * k);
    w->outv.ensure((size_t)2 * C * 8);
    w->err.ensure(16);
    w->actp.ensure(2 * sizeof(ActParams));
    w->mmlab.ensure((size_t)C * k * 2 * 16);
    w->qctr.ensure(64);
    w->qflags.ensure(((C + 31) / 32 + 1) * 4);
    w->base.ensure(c.base, 1, C);
    w->in.ensure(c.base, 1, C);
    w->gout.ensure(c.base, 1, C);
    w->eout.ensure(c.base, 1, C);
    for (int i = 0; i < 2; ++i) {
        w->in_pin[i].ensure((size_t)C * 8);
        w->out_pin[i].ensure((size_t)C * 8);
        w->ev[i] = dev::event_create();
    }
    w->act_pin.ensure(4 * sizeof(ActParams));
    w->par_pin.ensure(64 + 44 * 4 + 16 + 8);
    slot = w;
    return *w;
}

// retire the chunk that last used staging slot s: its decoded outputs are
// copied from pinned memory to the caller's buffer
static void stream_retire(StreamWS& w, int s) {
    if (!w.pend_dst[s]) return;
    dev::event_sync(w.ev[s]);
    std::memcpy(w.pend_dst[s], w.out_pin[s].p, (size_t)w.pend_n[s] * 8);
    w.pend_dst[s] = nullptr;
}

static void infer_stream(dashgpu_circuit& c, const uint8_t* seeds, uint32_t batch, const int64_t* inputs,
                         int64_t* outputs, uint64_t chunk, uint8_t* gc_out, dashgpu_timing& tm, uint64_t u_begin,
                         uint64_t u_end) {
    if (!streamable(c)) throw DataError("streamed inference needs a single activation-layer circuit");
    upload_circuit(c);
    const int k = c.k;
    const HLayer& l = c.layers[0];
    const Tape& T = *l.tape;
    const uint64_t N = l.E_out;
    u_end = std::min<uint64_t>(u_end, N);
    if (u_begin > u_end) throw DataError("element range out of order");
    const uint64_t C = std::max<uint64_t>(1, std::min<uint64_t>(chunk, std::max<uint64_t>(u_end - u_begin, 1)));
    StreamWS& w = stream_ws(c, C);
    const uint64_t mult_stride = (uint64_t)(MAXMOD - 1) * 128 * NWMAX;
    Sched q;
    q.counter = w.qctr.as<uint32_t>();
    q.flags = w.qflags.as<uint32_t>();
    q.flags_cap = w.qflags.n / 4;
    uint16_t primes[MAXK];
    fill_primes(c.base, primes);
    // per-chunk launch parameters that do not depend on the chunk
    ActParams P;
    std::memset(&P, 0, sizeof P);
    P.tape = l.tape_d->as<TapeOp>();
    P.n_ops = (int)T.ops.size();
    P.lv_tape = l.lv_tape_d->as<TapeOp>();
    P.lv_start = l.lv_start_d->as<uint16_t>();
    P.n_levels = (int)T.lv_start.size() - 1;
    fill_chunks(P, T, tape_chunks());
    P.phi = l.phi_d->as<uint8_t>();
    P.k = k;
    P.B = 1;
    P.uc_cts = T.cts;
    P.uc_gates = T.gates;
    P.uc_wires = T.wires;
    P.blob = w.blob.as<U4>();
    for (int i = 0; i < k; ++i) {
        P.out_kind[i] = T.out_kind[i];
        P.out_wire[i] = T.out_wire[i];
    }
    P.rk = w.rk.as<uint32_t>();
    P.mult = w.mult.as<uint32_t>();
    P.mult_stride = mult_stride;
    P.slots = w.slots.as<U4>();  // max(nslots, nslots_lv) per element
    P.lv_ok = 1;
    P.mmlab = w.mmlab.as<U4>();
    ActParams* actp = w.actp.as<ActParams>();  // [0] garbling, [1] evaluation of the current chunk
    // the sweep's error flags accumulate over the call (kernels only raise
    // them): [0] encode range, [1] decode miss / range; checked once at the end
    dev::memset0(w.err.p, 8, g_stream);
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    uint64_t ci = 0;  // chunk counter (staging slot = ci & 1)
    for (uint32_t b = 0; b < batch; ++b) {
        uint32_t rk[44];
        aes_expand_host(seeds + 16 * (size_t)b, rk);
        // the previous inference's chunks may still read rk / seeds
        for (int s = 0; s < 2; ++s) stream_retire(w, s);
        dev::sync(g_stream);
        std::memcpy(w.par_pin.p, rk, sizeof rk);
        std::memcpy(w.par_pin.as<uint8_t>() + sizeof rk, seeds + 16 * (size_t)b, 16);
        dev::h2d(w.rk.p, w.par_pin.p, sizeof rk, g_stream);
        dev::h2d(w.seeds.p, w.par_pin.as<uint8_t>() + sizeof rk, 16, g_stream);
        for (uint64_t u0 = u_begin; u0 < u_end; u0 += C, ++ci) {
            const int s = (int)(ci & 1);
            const uint32_t n = (uint32_t)std::min<uint64_t>(C, u_end - u0);
            stream_retire(w, s);  // chunk ci - 2 is done: slot s is free
            // offsets, zero wires and this chunk's input base labels
            SetupParams S;
            std::memset(&S, 0, sizeof S);
            S.B = 1;
            S.k = k;
            fill_primes(c.base, S.primes);
            for (int m : c.moduli) S.slot_mod[S.nslot++] = (uint16_t)m;
            S.rk = w.rk.as<uint32_t>();
            S.seeds = w.seeds.as<uint8_t>();
            S.mult = w.mult.as<uint32_t>();
            S.mult_stride = mult_stride;
            S.n_in = n;
            S.e0 = u0;
            for (int i = 0; i < k; ++i) S.base_planes[i] = w.base.lane[i]->as<uint32_t>();
            S.zero = w.zero.as<uint32_t>();
            S.Rb = w.Rb.as<uint32_t>();
            S.commit = w.commit.as<U4>();
            launch_setup(S, g_stream);
            // garble the chunk: outputs (PRF functions) first, then the tapes
            P.E = n;
            P.gate_base = l.gate_base + u0 * T.gates;
            P.wire_base = l.wire_base + u0 * T.wires;
            P.blob_stride = (uint64_t)n * T.cts;
            for (int i = 0; i < k; ++i) {
                P.in[i] = w.base.lane[i]->as<uint32_t>();
                P.out[i] = w.gout.lane[i]->as<uint32_t>();
            }
            launch_act_outputs(P, primes, g_stream);
            ActParams* pin = w.act_pin.as<ActParams>() + 2 * s;  // pinned launch parameters of slot s
            pin[0] = P;
            dev::h2d(actp, pin, sizeof P, g_stream);
            launch_act_multi(actp, &P, 1, true, g_stream, q);
            DecodeParams D;
            std::memset(&D, 0, sizeof D);
            D.B = 1;
            D.n_out = n;
            D.k = k;
            fill_primes(c.base, D.primes);
            for (int i = 0; i < k; ++i) D.poff[i + 1] = (uint16_t)(D.poff[i] + c.base.primes[i]);
            make_lane_ptrs(w.gout, k, D.lanes);
            D.table = w.dec.as<U4>();
            D.mult = w.mult.as<uint32_t>();
            D.mult_stride = mult_stride;
            launch_dectable(D, g_stream);
            if (gc_out) {  // test path: chunk rows -> reference order (act_rows layout with E = n)
                std::vector<U4> rows((size_t)n * T.cts);
                dev::d2h(rows.data(), w.blob.p, rows.size() * 16, g_stream);
                dev::sync(g_stream);
                U4* dst = reinterpret_cast<U4*>(gc_out) + (uint64_t)b * N * T.cts + u0 * T.cts;
                for (uint64_t u = 0; u < n; ++u)
                    for (uint64_t j = 0; j < T.cts; ++j) dst[u * T.cts + j] = rows[act_row_pos(n, T.cts, u, j)];
            }
            // garble_inputs of the chunk (garble.cpp:242-263), inputs staged in pinned slot s
            std::memcpy(w.in_pin[s].p, inputs + (uint64_t)b * N + u0, (size_t)n * 8);
            int64_t* vals = w.vals.as<int64_t>() + (size_t)s * C;
            dev::h2d(vals, w.in_pin[s].p, (size_t)n * 8, g_stream);
            EncodeParams E;
            std::memset(&E, 0, sizeof E);
            E.B = 1;
            E.n_in = n;
            E.k = k;
            fill_primes(c.base, E.primes);
            E.values = vals;
            for (int i = 0; i < k; ++i) {
                E.base[i] = w.base.lane[i]->as<uint32_t>();
                E.out[i] = w.in.lane[i]->as<uint32_t>();
            }
            E.mult = w.mult.as<uint32_t>();
            E.mult_stride = mult_stride;
            const u128 half_up = (c.base.P + 1) / 2, half_dn = c.base.P / 2;
            E.half_up_lo = (uint64_t)half_up;
            E.half_up_hi = (uint64_t)(half_up >> 64);
            E.half_dn_lo = (uint64_t)half_dn;
            E.half_dn_hi = (uint64_t)(half_dn >> 64);
            E.err = w.err.as<int>();
            launch_encode(E, g_stream);
            // evaluate the chunk on the active labels
            ActParams Pe = P;
            for (int i = 0; i < k; ++i) {
                Pe.in[i] = w.in.lane[i]->as<uint32_t>();
                Pe.out[i] = w.eout.lane[i]->as<uint32_t>();
            }
            pin[1] = Pe;
            dev::h2d(actp + 1, pin + 1, sizeof Pe, g_stream);
            launch_act_multi(actp + 1, &Pe, 1, false, g_stream, q);
            // decode_outputs of the chunk into staging slot s
            make_lane_ptrs(w.eout, k, D.lanes);
            D.residues = w.resid.as<uint8_t>();
            D.err = w.err.as<int>() + 1;
            D.values = w.outv.as<int64_t>() + (size_t)s * C;
            fill_crt(c.base, D);
            launch_decode(D, g_stream);
            dev::d2h(w.out_pin[s].p, D.values, (size_t)n * 8, g_stream);
            dev::event_record(w.ev[s], g_stream);
            w.pend_dst[s] = outputs + (uint64_t)b * N + u0;
            w.pend_n[s] = n;
            tm.sub_batches += 1;
        }
    }
    int err[2] = {0, 0};
    dev::d2h(err, w.err.p, 8, g_stream);
    for (int s = 0; s < 2; ++s) stream_retire(w, s);
    dev::sync(g_stream);
    if (err[0]) throw DataError("encode_signed: value outside the representable range");
    if (err[1] == ST_AUTH) throw AuthError("output label not present in the decoding table");
    if (err[1]) throw DataError("decode_signed: value exceeds 64-bit signed range");
    // one pipelined pass: the phases overlap, so the whole call is reported
    tm.ms_garble = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
    tm.h2d_bytes = (uint64_t)batch * ((u_end - u_begin) * 8 + 16 + 44 * 4);
    tm.d2h_bytes = (uint64_t)batch * (u_end - u_begin) * 8;
}

// ============================================================ exports

struct Writer {
    std::vector<uint8_t> b;
    void le(uint64_t v, int n) {
        for (int i = 0; i < n; ++i) b.push_back((uint8_t)(v >> (8 * i)));
    }
    void u128v(u128 v) {
        le((uint64_t)v, 8);
        le((uint64_t)(v >> 64), 8);
    }
    void bytes(const void* p, size_t n) {
        const uint8_t* q = (const uint8_t*)p;
        b.insert(b.end(), q, q + n);
    }
    void header(int kind) {
        bytes("DASH", 4);
        le(1, 2);
        le((uint64_t)kind, 1);
    }
    void shape(const std::vector<uint32_t>& s) {
        le(s.size(), 1);
        for (auto d : s) le(d, 4);
    }
};

// compress of a byte-digit row (label.cpp:208-219), host side for exports
static u128 host_compress(const uint32_t* words, int m) {
    const int n = n_digits_host(m);
    u128 acc = 0;
    const bool pow2 = (m & (m - 1)) == 0;
    int e = 0;
    while ((1 << e) < m) ++e;
    for (int i = n - 1; i >= 0; --i) {
        const uint32_t d = (words[i / 4] >> (8 * (i % 4))) & 0xff;
        acc = pow2 ? ((acc << e) | d) : (acc * (u128)m + d);
    }
    return acc;
}

static u128 u4_to_u128(const U4& v) {
    return ((u128)v.x[3] << 96) | ((u128)v.x[2] << 64) | ((u128)v.x[1] << 32) | v.x[0];
}
static U4 u128_to_u4(u128 v) {
    U4 r;
    for (int i = 0; i < 4; ++i) r.x[i] = (uint32_t)(v >> (32 * i));
    return r;
}

// device row index of reference ciphertext index idx (one inference's GC)
static uint64_t device_ct_index(const dashgpu_circuit& c, uint64_t idx) {
    for (const auto& l : c.layers)
        if (l.tape && idx >= l.ct_base && idx < l.ct_base + l.cts) {
            const uint64_t r = idx - l.ct_base, uc = l.tape->cts;
            return l.ct_base + act_row_pos(l.E_out, uc, r / uc, r % uc);
        }
    return idx;
}

// One inference's ciphertexts between the device row layout and the
// reference's GarbledCircuit::cts order, on the device (rows_permute_thread):
// activation layers are permuted block by block, everything else copied.
// to_ref: device (src) -> reference (dst); else reference -> device.
static void blob_permute(const dashgpu_circuit& c, const U4* src, U4* dst, bool to_ref) {
    uint64_t at = 0;
    for (const auto& l : c.layers) {
        if (!l.tape || !l.cts) continue;
        if (l.ct_base > at) dev::d2d(dst + at, src + at, (l.ct_base - at) * 16, g_stream);
        RowsPermuteParams P;
        P.src = src + l.ct_base;
        P.dst = dst + l.ct_base;
        P.E = l.E_out;
        P.uc = l.tape->cts;
        P.to_ref = to_ref ? 1 : 0;
        launch_rows_permute(P, g_stream);
        at = l.ct_base + l.cts;
    }
    if (c.total_cts > at) dev::d2d(dst + at, src + at, (c.total_cts - at) * 16, g_stream);
}

static size_t out_bytes(const std::vector<uint8_t>& v, uint8_t* buf, size_t cap, size_t* len) {
    if (len) *len = v.size();
    if (buf && cap >= v.size()) std::memcpy(buf, v.data(), v.size());
    return v.size();
}

// serialize_garbled_circuit (garble.cpp:347-403) up to the ciphertext rows:
// circuit description, zero-wire labels (zero = this inference's [k][LABW]
// words), layer ciphertext bases and the row count
static void gc_header(const dashgpu_circuit& c, const uint32_t* zero, Writer& w) {
    w.header(1);
    w.le((uint64_t)c.k, 1);
    w.shape(c.input_shape);
    uint64_t bits;
    std::memcpy(&bits, &c.alpha, 8);
    w.le(bits, 8);
    std::memcpy(&bits, &c.sign_target, 8);
    w.le(bits, 8);
    const auto& radices = c.needs_sign ? c.sign.spec : Spec{};
    w.le(radices.size(), 1);
    for (int r : radices) w.le((uint64_t)r, 2);
    w.le(c.layers.size(), 2);
    for (const auto& l : c.layers) {
        w.le((uint64_t)l.kind, 1);
        // bit 1 of the private byte flags the extension record, so a reader
        // knows it follows (reference circuits never set it)
        const bool ext = l.kind > DASH_LAYER_FLATTEN || l.src || l.src2 || l.pad;
        w.le((l.priv ? 1 : 0) | (ext ? 2 : 0), 1);
        for (uint32_t v : {l.in_dim, l.out_dim, l.in_ch, l.out_ch, l.filter, l.stride}) w.le(v, 4);
        const bool ww = l.linear() && !l.priv;
        w.le(ww ? 1 : 0, 1);
        if (ww) {
            w.le(l.w.size(), 8);
            for (int64_t v : l.w) w.le((uint64_t)v, 8);
        }
        if (ext) {  // extension record
            w.le((uint32_t)l.src, 4);
            w.le((uint32_t)l.src2, 4);
            w.le(l.pad, 4);
        }
    }
    for (int i = 0; i < c.k; ++i) w.u128v(host_compress(zero + (size_t)i * LABW, c.base.primes[i]));
    w.le(c.layers.size() + 1, 8);
    for (const auto& l : c.layers) w.le(l.ct_base, 8);
    w.le(c.total_cts, 8);
    w.le(c.total_cts, 8);
}

// device rows -> host memory (pageable caller buffer) through two pinned
// chunks: the copy of chunk i + 1 is in flight while chunk i is memcpy'd
static void rows_to_host(const uint8_t* dsrc, size_t bytes, uint8_t* dst) {
    constexpr size_t kChunk = 8u << 20;
    static thread_local HostBuf stage[2];
    struct Ev {
        void* e = dev::event_create();
        ~Ev() { dev::event_destroy(e); }
    } ev[2];
    const size_t n = (bytes + kChunk - 1) / kChunk;
    for (size_t i = 0; i <= n; ++i) {
        if (i < n) {
            const size_t len = std::min(kChunk, bytes - i * kChunk);
            stage[i & 1].ensure(kChunk);
            dev::d2h(stage[i & 1].p, dsrc + i * kChunk, len, g_stream);
            dev::event_record(ev[i & 1].e, g_stream);
        }
        if (i > 0) {
            const size_t j = i - 1, len = std::min(kChunk, bytes - j * kChunk);
            dev::event_sync(ev[j & 1].e);
            std::memcpy(dst + j * kChunk, stage[j & 1].p, len);
        }
    }
}

// serialize_garbled_circuit (garble.cpp:347-403) of inference b straight into
// buf (when cap suffices); *len = the GC's byte count either way
static void export_gc_into(const Network& n, uint32_t b, uint8_t* buf, size_t cap, size_t* len) {
    const dashgpu_circuit& c = *n.c;
    if (b >= n.B) throw DataError("inference index out of range");
    n.require_gc();
    std::vector<uint32_t> zero((size_t)c.k * LABW);
    U4 commit;
    dev::d2h(zero.data(), n.zero.as<uint32_t>() + (uint64_t)b * c.k * LABW, zero.size() * 4, g_stream);
    dev::d2h(&commit, n.commit.as<U4>() + b, 16, g_stream);
    dev::sync(g_stream);
    Writer w;
    gc_header(c, zero.data(), w);
    const size_t rows = c.total_cts * 16, total = w.b.size() + rows + 16;
    if (len) *len = total;
    if (!buf || cap < total) return;
    std::memcpy(buf, w.b.data(), w.b.size());
    // rows -> reference order on the device (little-endian u128 rows == the
    // U4 layout), then to the caller's buffer
    if (n.host_gc) {
        std::memcpy(buf + w.b.size(), n.hblob.as<U4>() + (uint64_t)b * c.total_cts, rows);
    } else {
        DevBuf ref;
        ref.ensure(std::max<uint64_t>(c.total_cts, 1) * 16);
        blob_permute(c, n.blob.as<U4>() + (uint64_t)b * c.total_cts, ref.as<U4>(), true);
        rows_to_host(ref.as<uint8_t>(), rows, buf + w.b.size());
    }
    Writer t;
    t.u128v(u4_to_u128(commit));
    std::memcpy(buf + w.b.size() + rows, t.b.data(), 16);
}

// Streamed serialize_garbled_circuit (SURVEY §8(f) row 1 at GC sizes beyond
// HBM): garbles layer by layer through the one-layer window (§11.1) and hands
// every inference's GC bytes to `sink` in order -- header, each layer's rows
// in the reference's cts order, commitment -- so the concatenation per
// inference is byte-identical to export_gc.  The network keeps its encoding
// and decoding material (as after dashgpu_network_release_gc).
static void garble_stream_into(Network& n, const uint8_t* seeds, uint32_t B, dashgpu_gc_sink sink, void* user) {
    dashgpu_circuit& c = *n.c;
    garble_setup(n, seeds, B, false, true);
    n.gc_released = false;
    auto emit = [&](uint32_t b, const void* p, size_t len) {
        if (len && sink(user, b, static_cast<const uint8_t*>(p), len) != 0)
            throw DataError("garbled-circuit sink aborted the stream");
    };
    std::vector<uint32_t> zero((size_t)B * c.k * LABW);
    std::vector<U4> commit(B);
    dev::d2h(zero.data(), n.zero.p, zero.size() * 4, g_stream);
    dev::d2h(commit.data(), n.commit.p, (size_t)B * 16, g_stream);
    dev::sync(g_stream);
    for (uint32_t b = 0; b < B; ++b) {
        Writer w;
        gc_header(c, zero.data() + (size_t)b * c.k * LABW, w);
        emit(b, w.b.data(), w.b.size());
    }
    outs_begin(n, true, n.base);
    // double-buffered: inference b + 1's rows are permuted and copied while
    // the sink consumes inference b's
    DevBuf ref[2];
    HostBuf host[2];
    struct Ev {
        void* e = dev::event_create();
        ~Ev() { dev::event_destroy(e); }
    } ev[2];
    for (size_t li = 0; li < c.layers.size(); ++li) {
        run_layer_at(n, true, li);
        garble_act_flush(n);
        const HLayer& l = c.layers[li];
        if (!l.cts) continue;
        const size_t bytes = l.cts * 16;
        for (int s = 0; s < 2; ++s) {
            ref[s].ensure(bytes);
            host[s].ensure(bytes);
        }
        for (uint32_t b = 0; b <= B; ++b) {
            if (b < B) {
                const int s = b & 1;
                const U4* src = n.blob.as<U4>() + (uint64_t)b * l.cts;
                if (l.tape) {
                    RowsPermuteParams P;
                    P.src = src;
                    P.dst = ref[s].as<U4>();
                    P.E = l.E_out;
                    P.uc = l.tape->cts;
                    P.to_ref = 1;
                    launch_rows_permute(P, g_stream);
                    src = ref[s].as<U4>();
                }
                dev::d2h(host[s].p, src, bytes, g_stream);
                dev::event_record(ev[s].e, g_stream);
            }
            if (b > 0) {  // hand over inference b - 1 while b is in flight
                const int s = (b - 1) & 1;
                dev::event_sync(ev[s].e);
                emit(b - 1, host[s].p, bytes);
            }
        }
    }
    for (uint32_t b = 0; b < B; ++b) {
        Writer w;
        w.u128v(u4_to_u128(commit[b]));
        emit(b, w.b.data(), w.b.size());
    }
    garble_dectables(n, *n.gouts.at[c.layers.size()]);
    dev::sync(g_stream);
    for (DevBuf* d : {&n.blob, &n.slots, &n.mmlab}) d->reset();
    n.gc_released = true;
}

static std::vector<U4> compress_lanes(const Lanes& L, const Crt& base, uint32_t B, uint32_t b) {
    const uint64_t n = L.E;
    DevBuf tmp;
    tmp.ensure((size_t)B * n * 16);
    std::vector<U4> out((size_t)base.k * n);
    for (int i = 0; i < base.k; ++i) {
        CompressParams P;
        std::memset(&P, 0, sizeof P);
        P.B = B;
        P.n = (uint32_t)n;
        P.p = (uint32_t)base.primes[i];
        P.lane = L.lane[i]->as<uint32_t>();
        P.out = tmp.as<U4>();
        P.ostride = n;
        launch_compress(P, g_stream);
        dev::d2h(out.data() + (size_t)i * n, tmp.as<U4>() + (uint64_t)b * n, n * 16, g_stream);
        dev::sync(g_stream);
    }
    return out;
}

// ---- GC import (evaluator side) ----
struct Reader {
    const uint8_t* p;
    size_t n, at = 0;
    uint64_t le(int w) {
        if (n - at < (size_t)w) throw DataError("truncated garbled circuit");
        uint64_t v = 0;
        for (int i = 0; i < w; ++i) v |= (uint64_t)p[at + i] << (8 * i);
        at += w;
        return v;
    }
    u128 u128v() {
        const uint64_t lo = le(8);
        return ((u128)le(8) << 64) | lo;
    }
};

// decompress_mod (label.cpp:228-232) into byte-digit words
static void host_decompress(u128 v, int m, uint32_t* words) {
    const int n = n_digits_host(m);
    const bool pow2 = (m & (m - 1)) == 0;
    if (!pow2) {
        u128 mn = 1;
        for (int i = 0; i < n; ++i) mn *= (u128)m;
        v %= mn;
    }
    int e = 0;
    while ((1 << e) < m) ++e;
    for (int w = 0; w < LABW; ++w) words[w] = 0;
    for (int i = 0; i < n; ++i) {
        const uint32_t d = pow2 ? (uint32_t)(v & (u128)(m - 1)) : (uint32_t)(v % (u128)m);
        v = pow2 ? v >> e : v / (u128)m;
        words[i / 4] |= d << (8 * (i % 4));
    }
}

struct ParsedGc {
    size_t circuit_bytes = 0;  // prefix holding the circuit description
    std::vector<u128> zero;
    std::vector<uint64_t> bases;
    const uint8_t* cts = nullptr;  // n_cts little-endian u128 rows inside the input
    uint64_t n_cts = 0;
    u128 commit = 0;
};

// parse_garbled_circuit (garble.cpp:368-403) + read_layer (garble.cpp:89-107);
// the circuit is built into c when c is non-null
static ParsedGc parse_gc(const uint8_t* data, size_t len, dashgpu_circuit* c) {
    Reader r{data, len};
    if (len < 4 || std::memcmp(data, "DASH", 4) != 0) throw DataError("bad file magic");
    r.at = 4;
    if (r.le(2) != 1) throw DataError("unsupported format version");
    if (r.le(1) != 1) throw DataError("wrong file kind");
    const int k = (int)r.le(1);
    if (k < 1 || k > MAXK) throw DataError("bad base size");
    const int rank = (int)r.le(1);
    if (rank == 0 || rank > 8) throw DataError("bad tensor rank");
    std::vector<uint32_t> shape(rank);
    uint64_t total = 1;
    for (auto& d : shape) {
        d = (uint32_t)r.le(4);
        if (d == 0) throw DataError("zero tensor dimension");
        total *= d;
        if (total > (1ull << 26)) throw DataError("tensor too large");
    }
    const uint64_t alpha = r.le(8), target = r.le(8);
    const int t = (int)r.le(1);
    Spec spec(t);
    for (auto& m : spec) m = (int)r.le(2);
    const uint32_t nl = (uint32_t)r.le(2);
    std::vector<HLayer> layers(nl);
    for (auto& l : layers) {
        l.kind = (int)r.le(1);
        if (l.kind < 1 || l.kind > 7) throw DataError("bad layer kind");
        const uint32_t flags = (uint32_t)r.le(1);
        l.priv = (flags & 1) != 0;
        l.in_dim = (uint32_t)r.le(4);
        l.out_dim = (uint32_t)r.le(4);
        l.in_ch = (uint32_t)r.le(4);
        l.out_ch = (uint32_t)r.le(4);
        l.filter = (uint32_t)r.le(4);
        l.stride = (uint32_t)r.le(4);
        if (r.le(1) != 0) {
            const uint64_t n = r.le(8);
            if (n != l.weight_count()) throw DataError("bad weight count");
            if (n > (len - r.at) / 8) throw DataError("truncated garbled circuit");
            l.w.resize(n);
            for (auto& v : l.w) v = (int64_t)r.le(8);
        }
        if (flags & 2) {  // extension record (export_gc)
            l.src = (int32_t)(uint32_t)r.le(4);
            l.src2 = (int32_t)(uint32_t)r.le(4);
            l.pad = (uint32_t)r.le(4);
        }
    }
    ParsedGc g;
    g.circuit_bytes = r.at;
    if (c) {
        c->k = k;
        c->input_shape = shape;
        std::memcpy(&c->alpha, &alpha, 8);
        std::memcpy(&c->sign_target, &target, 8);
        c->layers = std::move(layers);
        c->eval_only = true;
        c->gc_spec = spec;
        prepare_circuit(*c);  // validate_circuit + layout + tapes
    }
    for (int i = 0; i < k; ++i) g.zero.push_back(r.u128v());
    const uint64_t nb = r.le(8);
    if (nb != (uint64_t)nl + 1) throw DataError("bad ciphertext index length");
    g.bases.resize(nb);
    for (auto& b : g.bases) b = r.le(8);
    const uint64_t ncts = r.le(8);
    if (ncts > (1ull << 32)) throw DataError("ciphertext blob too large");
    if (ncts > (len - r.at) / 16) throw DataError("truncated garbled circuit");
    g.cts = data + r.at;  // little-endian u128 rows == the U4 layout
    g.n_cts = ncts;
    r.at += 16 * ncts;
    g.commit = r.u128v();
    if (r.at != len) throw DataError("trailing bytes in garbled circuit file");
    return g;
}

static std::vector<uint8_t> export_encoding(const Network& n, uint32_t b) {
    const dashgpu_circuit& c = *n.c;
    if (b >= n.B) throw DataError("inference index out of range");
    Writer w;
    w.header(2);
    w.le((uint64_t)c.k, 1);
    w.shape(c.input_shape);
    std::vector<uint32_t> R((size_t)c.k * LABW);
    dev::d2h(R.data(), n.Rb.as<uint32_t>() + (uint64_t)b * c.k * LABW, R.size() * 4, g_stream);
    dev::sync(g_stream);
    for (int i = 0; i < c.k; ++i) w.u128v(host_compress(R.data() + (size_t)i * LABW, c.base.primes[i]));
    const auto lanes = compress_lanes(n.base, c.base, n.B, b);
    for (int i = 0; i < c.k; ++i) {  // tensor_write (label_tensor.cpp:95-101)
        w.le((uint64_t)c.base.primes[i], 2);
        w.shape(c.input_shape);
        for (uint64_t e = 0; e < c.n_in; ++e) w.u128v(u4_to_u128(lanes[(size_t)i * c.n_in + e]));
    }
    return w.b;
}

static std::vector<uint8_t> export_decoding(const Network& n, uint32_t b) {
    const dashgpu_circuit& c = *n.c;
    if (b >= n.B) throw DataError("inference index out of range");
    Writer w;
    w.header(3);
    w.le((uint64_t)c.k, 1);
    w.shape(c.layers.empty() ? c.input_shape : c.layers.back().out_shape);
    std::vector<U4> t((size_t)c.n_out * n.sum_p);
    dev::d2h(t.data(), n.dec.as<U4>() + (uint64_t)b * t.size(), t.size() * 16, g_stream);
    dev::sync(g_stream);
    for (const auto& v : t) w.u128v(u4_to_u128(v));
    return w.b;
}

// ============================================================ models

namespace models {
using Rng = std::mt19937;

static std::vector<int64_t> random_ints(Rng& g, size_t n, int lo, int hi) {
    std::uniform_int_distribution<int> d(lo, hi);
    std::vector<int64_t> v(n);
    for (auto& x : v) x = d(g);
    return v;
}
static HLayer dense(uint32_t in, uint32_t out, Rng& g, bool priv = false, int wmax = 2, int bmax = 10) {
    HLayer l;
    l.kind = DASH_LAYER_DENSE;
    l.priv = priv;
    l.in_dim = in;
    l.out_dim = out;
    l.w = random_ints(g, (size_t)in * out, -wmax, wmax);
    l.bias = random_ints(g, out, -bmax, bmax);
    return l;
}
static HLayer conv2d(uint32_t ic, uint32_t oc, uint32_t f, uint32_t s, Rng& g, bool priv = false, int wmax = 2,
                     int bmax = 10) {
    HLayer l;
    l.kind = DASH_LAYER_CONV2D;
    l.priv = priv;
    l.in_ch = ic;
    l.out_ch = oc;
    l.filter = f;
    l.stride = s;
    l.w = random_ints(g, (size_t)oc * ic * f * f, -wmax, wmax);
    l.bias = random_ints(g, oc, -bmax, bmax);
    return l;
}
static HLayer simple(int kind) {
    HLayer l;
    l.kind = kind;
    return l;
}

// Builders mirror the reference's tests/support/test_models.hpp:79-145 (same
// mt19937 stream, same draw order) plus the benchmark configurations of
// SURVEY.md section 8(d).
static void build(dashgpu_circuit& c, const std::string& name, uint32_t seed, int k, bool priv) {
    Rng g(seed);
    c.k = k;
    c.layers.clear();
    const HLayer R = simple(DASH_LAYER_RELU), F = simple(DASH_LAYER_FLATTEN), SA = simple(DASH_LAYER_SIGNACT);
    if (name == "model_a") {
        c.input_shape = {784};
        c.layers.push_back(dense(784, 128, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(128, 128, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(128, 10, g));
    } else if (name == "model_c") {
        c.input_shape = {1, 28, 28};
        c.layers.push_back(conv2d(1, 5, 4, 2, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(simple(DASH_LAYER_FLATTEN));
        c.layers.push_back(dense(845, 100, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(100, 10, g));
    } else if (name == "model_d") {
        c.input_shape = {1, 28, 28};
        c.layers.push_back(conv2d(1, 16, 6, 2, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(conv2d(16, 16, 6, 2, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(simple(DASH_LAYER_FLATTEN));
        c.layers.push_back(dense(256, 100, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(100, 10, g));
    } else if (name == "model_f_dims") {
        c.input_shape = {3, 32, 32};
        c.layers.push_back(simple(DASH_LAYER_FLATTEN));
        c.layers.push_back(dense(3072, 16, g));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(16, 10, g));
    } else if (name == "model_tiny") {
        c.input_shape = {2, 6, 6};
        c.layers.push_back(conv2d(2, 3, 3, 1, g, priv));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(conv2d(3, 2, 2, 2, g, priv));
        c.layers.push_back(simple(DASH_LAYER_SIGNACT));
        c.layers.push_back(simple(DASH_LAYER_FLATTEN));
        c.layers.push_back(dense(8, 5, g, priv));
        c.layers.push_back(simple(DASH_LAYER_RELU));
        c.layers.push_back(dense(5, 3, g, priv));
    } else if (name == "lenet5") {
        // LeNet-5 restated in reference ops (pooling -> strided 2x2 conv)
        c.input_shape = {1, 28, 28};
        c.layers.push_back(conv2d(1, 6, 5, 1, g, priv));
        c.layers.push_back(R);
        c.layers.push_back(conv2d(6, 6, 2, 2, g, priv));
        c.layers.push_back(conv2d(6, 16, 5, 1, g, priv));
        c.layers.push_back(R);
        c.layers.push_back(conv2d(16, 16, 2, 2, g, priv));
        c.layers.push_back(F);
        c.layers.push_back(dense(256, 120, g, priv));
        c.layers.push_back(R);
        c.layers.push_back(dense(120, 84, g, priv));
        c.layers.push_back(R);
        c.layers.push_back(dense(84, 10, g, priv));
    } else if (name == "minionn") {
        // paper Model F, Tanh -> ReLU, padding-free
        c.input_shape = {3, 32, 32};
        const uint32_t spec[8][4] = {{3, 32, 3, 1},  {32, 32, 3, 1}, {32, 32, 2, 2},  {32, 64, 3, 1},
                                     {64, 64, 3, 1}, {64, 64, 2, 2}, {64, 128, 3, 1}, {128, 128, 3, 1}};
        for (auto& s : spec) {
            c.layers.push_back(conv2d(s[0], s[1], s[2], s[3], g, priv));
            c.layers.push_back(R);
        }
        c.layers.push_back(F);
        c.layers.push_back(dense(128, 10, g, priv));
    } else if (name == "resnet20" || name == "resnet20s" || name == "resnet_tiny") {
        // ResNet-20 (CIFAR variant) in reference ops + the Pad2d / Add / DAG
        // extensions (include/dash_circuit_desc.h, SURVEY.md 8(d) "ResNet-20
        // extension notes"): 3x3 pad-1 convs with 16/32/64 channels, three
        // basic blocks per stage, 1x1 stride-2 projection shortcuts, residual
        // add, ReLU (resnet20s: SignAct after every add), global sum pool as
        // an identity-channel conv over the final map, FC 64 -> 10.
        // resnet_tiny: the same graph with 4/8/16 channels on 3x8x8, one
        // block per stage (parity tests).
        const bool tiny = name == "resnet_tiny";
        const uint32_t C0 = tiny ? 4 : 16, S = tiny ? 8 : 32;
        const int blocks = tiny ? 1 : 3;
        const HLayer post = name == "resnet20s" ? SA : R;
        c.input_shape = {3, S, S};
        // ids: 0 = circuit input, j + 1 = output of layer j
        auto add_layer = [&](HLayer l, int src_id) {
            const int li = (int)c.layers.size();
            l.src = src_id == li ? 0 : (src_id == 0 ? -1 : src_id);
            c.layers.push_back(std::move(l));
            return li + 1;
        };
        auto padded_conv = [&](int x, uint32_t ci, uint32_t co, uint32_t stride) {
            HLayer pd = simple(DASH_LAYER_PAD2D);
            pd.pad = 1;
            const int p = add_layer(pd, x);
            return add_layer(conv2d(ci, co, 3, stride, g, priv), p);
        };
        int x = add_layer(R, padded_conv(0, 3, C0, 1));
        uint32_t cin = C0;
        for (int st = 0; st < 3; ++st) {
            const uint32_t cout = C0 << st;
            for (int bk = 0; bk < blocks; ++bk) {
                const uint32_t stride = (st > 0 && bk == 0) ? 2 : 1;
                const int r1 = add_layer(R, padded_conv(x, cin, cout, stride));
                const int c2 = padded_conv(r1, cout, cout, 1);
                const int sc = (stride != 1 || cin != cout) ? add_layer(conv2d(cin, cout, 1, stride, g, priv), x) : x;
                HLayer ad = simple(DASH_LAYER_ADD);
                ad.src2 = c2;
                x = add_layer(post, add_layer(ad, sc));
                cin = cout;
            }
        }
        const uint32_t Cf = C0 << 2, Sf = S >> 2;
        HLayer pool = conv2d(Cf, Cf, Sf, 1, g, false);  // global sum pool: w[oc][ic] = [oc == ic]
        for (uint32_t oc = 0; oc < Cf; ++oc)
            for (uint32_t ic = 0; ic < Cf; ++ic)
                for (uint32_t t = 0; t < Sf * Sf; ++t) pool.w[((uint64_t)oc * Cf + ic) * Sf * Sf + t] = oc == ic;
        std::fill(pool.bias.begin(), pool.bias.end(), 0);
        x = add_layer(pool, x);
        x = add_layer(F, x);
        add_layer(dense(Cf, 10, g, priv), x);
    } else if (name.rfind("relu", 0) == 0 || name.rfind("sign", 0) == 0) {
        const long n = std::stol(name.substr(4));
        if (n <= 0) throw DataError("bad sweep size");
        c.input_shape = {(uint32_t)n};
        c.layers.push_back(name[0] == 'r' ? R : SA);
    } else if (name.rfind("dense", 0) == 0) {
        const long n = std::stol(name.substr(5));
        c.input_shape = {(uint32_t)n};
        c.layers.push_back(dense((uint32_t)n, (uint32_t)n, g));
    } else {
        throw DataError("unknown model " + name);
    }
}
}  // namespace models

// ============================================================ constants

static std::atomic<uint64_t> g_constants{0};  // devices whose constant tables are uploaded
static std::mutex g_init_mu;

static void check_constants() {
    const int d = dev::get_device();
    if (d < 0 || d >= 64 || !((g_constants.load() >> d) & 1))
        throw std::runtime_error("dashgpu_init() / dashgpu_use() has not been called for device " +
                                 std::to_string(d));
}

static void init_device(int device) {
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (device < 0 || device >= 64) throw DataError("device index out of range");
    dev::set_device(device);
    if ((g_constants.load() >> device) & 1) return;
    static std::vector<ModC> mods(MAXMOD + 1);
    for (int m = 2; m <= MAXMOD; ++m) mods[m] = make_modc(m);
    uint32_t pi_rk[44];
    const uint8_t zero[16] = {0};
    aes_expand_host(zero, pi_rk);
    uint16_t modslot[MAXMOD + 1] = {0};
    for (int m = 2; m <= MAXMOD; ++m) modslot[m] = (uint16_t)(m - 2);
    uint32_t T0[256];
    t0_table(T0);
    dev::upload_constants(mods.data(), pi_rk, modslot, T0);
    g_constants |= 1ull << device;
}

// plain_forward (layer.cpp:346-376, 56-109) with OverflowError range checks,
// plus the Pad2d / Add / DAG extensions (pad cells 0, add = integer sum)
static std::vector<int64_t> plain_forward(const dashgpu_circuit& c, std::vector<int64_t> x0) {
    const int64_t hi = max_signed(c.base), lo = min_signed(c.base);
    std::vector<std::vector<int64_t>> vals;
    vals.push_back(std::move(x0));
    for (size_t li = 0; li < c.layers.size(); ++li) {
        const auto& l = c.layers[li];
        const std::vector<int64_t>& x = vals[src_index(li, l.src)];
        std::vector<int64_t> y(l.E_out);
        if (l.linear()) {
            for (uint64_t u = 0; u < l.E_out; ++u) {
                __int128 acc;
                if (l.kind == DASH_LAYER_DENSE) {
                    acc = l.bias.empty() ? 0 : l.bias[u];
                    for (uint32_t i = 0; i < l.in_dim; ++i) acc += (__int128)l.w[u * l.in_dim + i] * x[i];
                } else {
                    const uint32_t H = l.in_shape[1], W = l.in_shape[2], OH = l.out_shape[1], OW = l.out_shape[2];
                    const uint32_t oc = (uint32_t)(u / ((uint64_t)OH * OW)), oy = (uint32_t)((u / OW) % OH),
                                   ox = (uint32_t)(u % OW);
                    acc = l.bias.empty() ? 0 : l.bias[oc];
                    for (uint32_t ic = 0; ic < l.in_ch; ++ic)
                        for (uint32_t ky = 0; ky < l.filter; ++ky)
                            for (uint32_t kx = 0; kx < l.filter; ++kx)
                                acc += (__int128)l.w[(((uint64_t)oc * l.in_ch + ic) * l.filter + ky) * l.filter + kx] *
                                       x[((uint64_t)ic * H + (oy * l.stride + ky)) * W + (ox * l.stride + kx)];
                }
                if (acc > hi || acc < lo) throw OverflowErr("intermediate value left the signed range of the base");
                y[u] = (int64_t)acc;
            }
        } else if (l.kind == DASH_LAYER_PAD2D) {
            const uint32_t H = l.in_shape[1], W = l.in_shape[2], OH = l.out_shape[1], OW = l.out_shape[2];
            for (uint64_t u = 0; u < l.E_out; ++u) {
                const uint64_t ch = u / ((uint64_t)OH * OW);
                const uint32_t yy = (uint32_t)((u / OW) % OH), xx = (uint32_t)(u % OW);
                const bool inside = yy >= l.pad && yy < l.pad + H && xx >= l.pad && xx < l.pad + W;
                y[u] = inside ? x[(ch * H + (yy - l.pad)) * W + (xx - l.pad)] : 0;
            }
        } else if (l.kind == DASH_LAYER_ADD) {
            const std::vector<int64_t>& x2 = vals[src_index(li, l.src2)];
            for (uint64_t u = 0; u < l.E_out; ++u) {
                const __int128 acc = (__int128)x[u] + x2[u];
                if (acc > hi || acc < lo) throw OverflowErr("intermediate value left the signed range of the base");
                y[u] = (int64_t)acc;
            }
        } else {
            for (uint64_t u = 0; u < l.E_out; ++u) {
                if (l.kind == DASH_LAYER_RELU) y[u] = x[u] > 0 ? x[u] : 0;
                else if (l.kind == DASH_LAYER_SIGNACT) y[u] = x[u] > 0 ? 1 : -1;
                else y[u] = x[u];
            }
        }
        vals.push_back(std::move(y));
    }
    return vals.back();
}

}  // namespace dashgpu

dashgpu_circuit::~dashgpu_circuit() = default;

struct dashgpu_network {
    std::unique_ptr<dashgpu_circuit> own_c;  // evaluator copy of an imported GC
    std::unique_ptr<dashgpu::Network> net;
};
struct dashgpu_bundle {
    std::unique_ptr<dashgpu::Bundle> b;
};

// ================================================================ C ABI

using namespace dashgpu;

static thread_local std::string g_err;

template <class F>
static int guarded(F&& f) {
    try {
        f();
        return DASHGPU_OK;
    } catch (const OverflowErr& e) {
        g_err = e.what();
        return DASHGPU_ERR_OVERFLOW;
    } catch (const DataError& e) {
        g_err = e.what();
        return DASHGPU_ERR_DATA;
    } catch (const AuthError& e) {
        g_err = e.what();
        return DASHGPU_ERR_AUTH;
    } catch (const std::exception& e) {
        g_err = e.what();
        return std::string(e.what()).rfind("CUDA", 0) == 0 ? DASHGPU_ERR_CUDA : DASHGPU_ERR;
    }
}

// The size query (buf == nullptr) and the copy call of one export come in
// pairs; the query keeps its result for the copy that follows on this thread
// (a GC is ~125 MB for LeNet-5: built once, not twice).
template <class F>
static void export_cached(const dashgpu_network* n, uint32_t b, int kind, uint8_t* buf, size_t cap, size_t* len,
                          F&& make) {
    static thread_local struct {
        const dashgpu_network* n = nullptr;
        uint32_t b = 0;
        int kind = -1;
        std::vector<uint8_t> v;
    } cache;
    const bool hit = cache.n == n && cache.b == b && cache.kind == kind;
    std::vector<uint8_t> v = hit ? std::move(cache.v) : make();
    cache.n = nullptr;
    cache.kind = -1;
    cache.v.clear();
    out_bytes(v, buf, cap, len);
    if (!buf) {
        cache.n = n;
        cache.b = b;
        cache.kind = kind;
        cache.v = std::move(v);
    }
}
extern "C" {

const char* dashgpu_last_error(void) { return g_err.c_str(); }
int dashgpu_version(void) { return 1; }
int dashgpu_backend(void) { return dev::backend(); }

int dashgpu_init(int device) {
    return guarded([&] { init_device(device); });
}

int dashgpu_set_stream(void* stream) {
    g_stream = stream;
    return DASHGPU_OK;
}

int dashgpu_use(int device, void* stream) {
    return guarded([&] {
        init_device(device);  // selects the device for this thread; constants once per device
        g_stream = stream;
    });
}

int dashgpu_circuit_create(const dash_circuit_desc* d, dashgpu_circuit** out) {
    return guarded([&] {
        if (!d || !out) throw DataError("null argument");
        if (d->k < 1 || d->k > MAXK) throw DataError("CRT base size out of range");
        if (d->rank < 1 || d->rank > 8) throw DataError("bad tensor rank");
        auto c = std::make_unique<dashgpu_circuit>();
        c->k = d->k;
        c->input_shape.assign(d->input_shape, d->input_shape + d->rank);
        c->sign_target = d->sign_target;
        c->alpha = d->alpha;
        for (uint32_t i = 0; i < d->n_layers; ++i) {
            const dash_layer_desc& s = d->layers[i];
            HLayer l;
            l.kind = s.kind;
            l.priv = s.private_weights != 0;
            l.in_dim = s.in_dim;
            l.out_dim = s.out_dim;
            l.in_ch = s.in_ch;
            l.out_ch = s.out_ch;
            l.filter = s.filter;
            l.stride = s.stride;
            l.src = s.src;
            l.src2 = s.src2;
            l.pad = s.pad;
            if (s.q_weights) l.w.assign(s.q_weights, s.q_weights + s.n_weights);
            if (s.q_biases) l.bias.assign(s.q_biases, s.q_biases + s.n_biases);
            c->layers.push_back(std::move(l));
        }
        prepare_circuit(*c);
        *out = c.release();
    });
}

void dashgpu_circuit_destroy(dashgpu_circuit* c) { delete c; }

int dashgpu_model_build(const char* name, uint32_t seed, int k, int priv, dashgpu_circuit** out) {
    return guarded([&] {
        auto c = std::make_unique<dashgpu_circuit>();
        models::build(*c, name, seed, k, priv != 0);
        prepare_circuit(*c);
        *out = c.release();
    });
}

int dashgpu_circuit_info_get(const dashgpu_circuit* c, dashgpu_circuit_info* o) {
    return guarded([&] {
        std::memset(o, 0, sizeof *o);
        o->k = c->k;
        o->n_layers = (uint32_t)c->layers.size();
        o->n_in = c->n_in;
        o->n_out = c->n_out;
        o->cts = c->total_cts;
        o->gates = c->total_gates;
        o->wires = c->total_wires + c->wire0;
        if (c->needs_sign) {
            o->sign_t = (uint32_t)c->sign.spec.size();
            for (size_t j = 0; j < c->sign.spec.size() && j < 32; ++j) o->radices[j] = (uint16_t)c->sign.spec[j];
            o->act_uc_cts = c->relu_tape->cts;
            o->act_eval_rows = c->relu_tape->eval_rows;
            o->max_slots = (uint32_t)std::max(c->relu_tape->nslots, c->sign_tape->nslots);
        }
        o->relu_elements = c->relu_elements;
        o->linear_macs = c->linear_macs;
    });
}

int dashgpu_circuit_desc_view(const dashgpu_circuit* cc, dash_circuit_desc* out) {
    return guarded([&] {
        auto* c = const_cast<dashgpu_circuit*>(cc);
        c->desc_layers.clear();
        for (const auto& l : c->layers) {
            dash_layer_desc s;
            std::memset(&s, 0, sizeof s);
            s.kind = l.kind;
            s.private_weights = l.priv;
            s.in_dim = l.in_dim;
            s.out_dim = l.out_dim;
            s.in_ch = l.in_ch;
            s.out_ch = l.out_ch;
            s.filter = l.filter;
            s.stride = l.stride;
            s.src = l.src;
            s.src2 = l.src2;
            s.pad = l.pad;
            s.q_weights = l.w.empty() ? nullptr : l.w.data();
            s.n_weights = l.w.size();
            s.q_biases = l.bias.empty() ? nullptr : l.bias.data();
            s.n_biases = l.bias.size();
            c->desc_layers.push_back(s);
        }
        std::memset(out, 0, sizeof *out);
        out->k = c->k;
        out->rank = (uint32_t)c->input_shape.size();
        for (size_t i = 0; i < c->input_shape.size(); ++i) out->input_shape[i] = c->input_shape[i];
        out->sign_target = c->sign_target;
        out->alpha = c->alpha;
        out->n_layers = (uint32_t)c->desc_layers.size();
        out->layers = c->desc_layers.data();
    });
}

int dashgpu_random_input(const dashgpu_circuit* c, uint32_t seed, int lo, int hi, int64_t* out) {
    return guarded([&] {
        models::Rng g(seed);
        auto v = models::random_ints(g, c->n_in, lo, hi);
        std::copy(v.begin(), v.end(), out);
    });
}

int dashgpu_plain_forward(const dashgpu_circuit* c, const int64_t* in, int64_t* out) {
    return guarded([&] {
        auto y = plain_forward(*c, std::vector<int64_t>(in, in + c->n_in));
        std::copy(y.begin(), y.end(), out);
    });
}

int dashgpu_garble(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch, dashgpu_network** out) {
    return guarded([&] {
        if (batch == 0) throw DataError("empty batch");
        auto n = std::make_unique<dashgpu_network>();
        n->net = std::make_unique<Network>();
        n->net->c = const_cast<dashgpu_circuit*>(c);
        garble_into(*n->net, seeds, batch, false);
        dev::sync(g_stream);
        *out = n.release();
    });
}

int dashgpu_garble_stream(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch, dashgpu_gc_sink sink,
                          void* user, dashgpu_network** out) {
    return guarded([&] {
        if (batch == 0) throw DataError("empty batch");
        if (!sink) throw DataError("null sink");
        auto n = std::make_unique<dashgpu_network>();
        n->net = std::make_unique<Network>();
        n->net->c = const_cast<dashgpu_circuit*>(c);
        garble_stream_into(*n->net, seeds, batch, sink, user);
        if (out) *out = n.release();
    });
}

void dashgpu_network_destroy(dashgpu_network* n) { delete n; }

// ---- layer level (layer.hpp:79-97) ----
int dashgpu_network_setup(const dashgpu_circuit* c, const uint8_t* seeds, uint32_t batch, dashgpu_network** out) {
    return guarded([&] {
        if (batch == 0) throw DataError("empty batch");
        auto n = std::make_unique<dashgpu_network>();
        n->net = std::make_unique<Network>();
        n->net->c = const_cast<dashgpu_circuit*>(c);
        garble_setup(*n->net, seeds, batch, false);
        dev::sync(g_stream);
        *out = n.release();
    });
}

static std::unique_ptr<dashgpu_bundle> new_bundle(Network& N, uint64_t E, bool output) {
    auto bd = std::make_unique<dashgpu_bundle>();
    bd->b = std::make_unique<Bundle>();
    bd->b->net = &N;
    bd->b->B = N.B;
    bd->b->output = output;
    bd->b->lanes.ensure(N.c->base, N.B, E);
    return bd;
}

static void copy_lanes(const Network& N, const Lanes& from, Lanes& to, uint64_t E) {
    for (int i = 0; i < N.c->k; ++i)
        dev::d2d(to.lane[i]->p, from.lane[i]->p,
                 (size_t)N.B * ((n_digits_host(N.c->base.primes[i]) + 3) / 4) * E * 4, g_stream);
}

int dashgpu_input_base(dashgpu_network* n, dashgpu_bundle** out) {
    return guarded([&] {
        Network& N = *n->net;
        auto bd = new_bundle(N, N.c->n_in, false);
        copy_lanes(N, N.base, bd->b->lanes, N.c->n_in);
        dev::sync(g_stream);
        *out = bd.release();
    });
}

static void layer_pass(dashgpu_network* n, uint32_t li, const dashgpu_bundle* in, const dashgpu_bundle* in2,
                       dashgpu_bundle** out, bool garbler) {
    Network& N = *n->net;
    dashgpu_circuit& c = *N.c;
    if (li >= c.layers.size()) throw DataError("layer index out of range");
    N.require_gc();
    const HLayer& l = c.layers[li];
    if (!in || in->b->B != N.B || in->b->lanes.E != l.E_in) throw DataError("layer input shape mismatch");
    if (l.kind == DASH_LAYER_ADD && (!in2 || in2->b->B != N.B || in2->b->lanes.E != l.E_out))
        throw DataError("add layer needs a second operand of the output shape");
    auto bd = new_bundle(N, l.E_out, li + 1 == c.layers.size());
    if (l.kind == DASH_LAYER_FLATTEN) {
        copy_lanes(N, in->b->lanes, bd->b->lanes, l.E_out);
    } else {
        run_layer(N, li, l, garbler, in->b->lanes, in2 ? &in2->b->lanes : nullptr, bd->b->lanes);
        if (garbler) garble_act_flush(N);
    }
    dev::sync(g_stream);
    *out = bd.release();
}

int dashgpu_layer_garble(dashgpu_network* n, uint32_t li, const dashgpu_bundle* in, const dashgpu_bundle* in2,
                         dashgpu_bundle** out) {
    return guarded([&] { layer_pass(n, li, in, in2, out, true); });
}

int dashgpu_layer_eval(dashgpu_network* n, uint32_t li, const dashgpu_bundle* in, const dashgpu_bundle* in2,
                       dashgpu_bundle** out) {
    return guarded([&] { layer_pass(n, li, in, in2, out, false); });
}

int dashgpu_network_release_gc(dashgpu_network* n) {
    return guarded([&] {
        if (!n) throw DataError("null network");
        Network& N = *n->net;
        dev::sync(g_stream);  // nothing in flight may still read them
        for (DevBuf* b : {&N.blob, &N.slots, &N.mmlab, &N.act_dev, &N.qflags}) b->reset();
        N.hblob.reset();
        N.gouts.own.clear();
        N.gouts.at.clear();
        N.eouts.own.clear();
        N.eouts.at.clear();
        N.slot_used = N.mm_used = 0;
        N.gc_released = true;
    });
}

int dashgpu_network_finish(dashgpu_network* n, const dashgpu_bundle* fin) {
    return guarded([&] {
        Network& N = *n->net;
        if (!fin || fin->b->B != N.B || fin->b->lanes.E != N.c->n_out) throw DataError("output shape mismatch");
        garble_dectables(N, fin->b->lanes);
        dev::sync(g_stream);
    });
}

int dashgpu_layer_count(const dashgpu_circuit* c, uint32_t li, uint64_t* cts_gates_wires) {
    return guarded([&] {
        if (li >= c->layers.size()) throw DataError("layer index out of range");
        const HLayer& l = c->layers[li];
        cts_gates_wires[0] = l.cts;
        cts_gates_wires[1] = l.gates;
        cts_gates_wires[2] = l.wires;
    });
}

// ---- LabelTensor upload / download (label_tensor.hpp:14-42: label-major u16 digits) ----
int dashgpu_bundle_info(const dashgpu_bundle* b, uint32_t* batch, uint64_t* elements) {
    return guarded([&] {
        *batch = b->b->B;
        *elements = b->b->lanes.E;
    });
}

int dashgpu_bundle_from_labels(dashgpu_network* n, uint64_t elements, const uint16_t* const* lanes, int output,
                               dashgpu_bundle** out) {
    return guarded([&] {
        Network& N = *n->net;
        const dashgpu_circuit& c = *N.c;
        auto bd = new_bundle(N, elements, output != 0);
        for (int i = 0; i < c.k; ++i) {
            const int p = c.base.primes[i], nd = n_digits_host(p), nw = (nd + 3) / 4;
            std::vector<uint32_t> w((size_t)N.B * nw * elements, 0);
            for (uint32_t b = 0; b < N.B; ++b)
                for (uint64_t e = 0; e < elements; ++e)
                    for (int d = 0; d < nd; ++d) {
                        const uint16_t v = lanes[i][((uint64_t)b * elements + e) * nd + d];
                        if (v >= p) throw DataError("label digit out of range");
                        w[((uint64_t)b * nw + d / 4) * elements + e] |= (uint32_t)v << (8 * (d % 4));
                    }
            dev::h2d(bd->b->lanes.lane[i]->p, w.data(), w.size() * 4, g_stream);
            dev::sync(g_stream);
        }
        *out = bd.release();
    });
}

int dashgpu_bundle_labels(const dashgpu_bundle* bd, int lane, uint16_t* out) {
    return guarded([&] {
        const Bundle& B = *bd->b;
        const dashgpu_circuit& c = *B.net->c;
        if (lane < 0 || lane >= c.k) throw DataError("lane out of range");
        const int p = c.base.primes[lane], nd = n_digits_host(p), nw = (nd + 3) / 4;
        const uint64_t E = B.lanes.E;
        std::vector<uint32_t> w((size_t)B.B * nw * E);
        dev::d2h(w.data(), B.lanes.lane[lane]->p, w.size() * 4, g_stream);
        dev::sync(g_stream);
        for (uint32_t b = 0; b < B.B; ++b)
            for (uint64_t e = 0; e < E; ++e)
                for (int d = 0; d < nd; ++d)
                    out[((uint64_t)b * E + e) * nd + d] =
                        (uint16_t)((w[((uint64_t)b * nw + d / 4) * E + e] >> (8 * (d % 4))) & 0xffu);
    });
}

int dashgpu_garble_inputs(dashgpu_network* n, const int64_t* values, dashgpu_bundle** out) {
    return guarded([&] {
        auto b = std::make_unique<dashgpu_bundle>();
        b->b = std::make_unique<Bundle>();
        encode_into(*n->net, values, false, *b->b);
        *out = b.release();
    });
}

int dashgpu_evaluate(dashgpu_network* n, const dashgpu_bundle* in, dashgpu_bundle** out) {
    return guarded([&] {
        auto b = std::make_unique<dashgpu_bundle>();
        b->b = std::make_unique<Bundle>();
        evaluate_into(*n->net, *in->b, *b->b);
        dev::sync(g_stream);
        *out = b.release();
    });
}

int dashgpu_decode_outputs(dashgpu_network* n, const dashgpu_bundle* out, int64_t* values) {
    return guarded([&] { decode_into(*n->net, *out->b, values, false); });
}

void dashgpu_bundle_destroy(dashgpu_bundle* b) { delete b; }

int dashgpu_export_gc(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len) {
    return guarded([&] { export_gc_into(*n->net, b, buf, cap, len); });
}
int dashgpu_export_encoding(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len) {
    return guarded([&] { export_cached(n, b, 2, buf, cap, len, [&] { return export_encoding(*n->net, b); }); });
}
int dashgpu_export_decoding(const dashgpu_network* n, uint32_t b, uint8_t* buf, size_t cap, size_t* len) {
    return guarded([&] { export_cached(n, b, 3, buf, cap, len, [&] { return export_decoding(*n->net, b); }); });
}
int dashgpu_export_bundle(const dashgpu_bundle* bd, uint32_t b, uint8_t* buf, size_t cap, size_t* len) {
    return guarded([&] {
        const Bundle& B = *bd->b;
        if (b >= B.B) throw DataError("inference index out of range");
        const auto v = compress_lanes(B.lanes, B.net->c->base, B.B, b);
        Writer w;
        for (const auto& x : v) w.u128v(u4_to_u128(x));
        out_bytes(w.b, buf, cap, len);
    });
}

int dashgpu_import_bundle(dashgpu_network* n, const uint8_t* data, size_t len, int output, dashgpu_bundle** out) {
    return guarded([&] {
        Network& N = *n->net;
        const dashgpu_circuit& c = *N.c;
        const uint64_t E = output ? c.n_out : c.n_in;
        if (len != (size_t)N.B * c.k * E * 16) throw DataError("wire payload size mismatch");
        auto bd = std::make_unique<dashgpu_bundle>();
        bd->b = std::make_unique<Bundle>();
        Bundle& B = *bd->b;
        B.net = &N;
        B.B = N.B;
        B.output = output != 0;
        B.lanes.ensure(c.base, N.B, E);
        DevBuf tmp;
        tmp.ensure((size_t)N.B * E * 16);
        for (int i = 0; i < c.k; ++i) {
            std::vector<uint8_t> lane((size_t)N.B * E * 16);
            for (uint32_t b = 0; b < N.B; ++b)
                std::memcpy(lane.data() + (size_t)b * E * 16, data + ((size_t)b * c.k + i) * E * 16, E * 16);
            dev::h2d(tmp.p, lane.data(), lane.size(), g_stream);
            CompressParams P;
            std::memset(&P, 0, sizeof P);
            P.B = N.B;
            P.n = (uint32_t)E;
            P.p = (uint32_t)c.base.primes[i];
            P.out = tmp.as<U4>();
            P.ostride = E;
            launch_decompress(P, B.lanes.lane[i]->as<uint32_t>(), g_stream);
            dev::sync(g_stream);
        }
        *out = bd.release();
    });
}

// EvaluatorService GC_TRANSFER (protocol.cpp:309-316): garbled circuits ->
// an evaluator network, one inference per GC; all GCs of a batch must carry
// the same circuit.  The consistency checks of evaluate (garble.cpp:262-303)
// run here, once.
static void import_gc(const uint8_t* const* gcs, const size_t* lens, uint32_t batch, dashgpu_network** out,
                      bool host) {
    {
        if (!gcs || !lens || !out) throw DataError("null argument");
        if (batch == 0) throw DataError("empty batch");
        auto n = std::make_unique<dashgpu_network>();
        n->own_c = std::make_unique<dashgpu_circuit>();
        dashgpu_circuit& c = *n->own_c;
        std::vector<ParsedGc> gs;
        gs.push_back(parse_gc(gcs[0], lens[0], &c));
        for (uint32_t b = 1; b < batch; ++b) {
            gs.push_back(parse_gc(gcs[b], lens[b], nullptr));
            if (gs[b].circuit_bytes != gs[0].circuit_bytes ||
                std::memcmp(gcs[b], gcs[0], gs[0].circuit_bytes) != 0)
                throw DataError("garbled circuits of a batch differ in their circuit");
        }
        for (const auto& g : gs) {
            if (g.n_cts != c.total_cts) throw DataError("ciphertext blob does not match the circuit");
            for (size_t li = 0; li < c.layers.size(); ++li)
                if (g.bases[li] != c.layers[li].ct_base) throw DataError("ciphertext blob does not match the circuit");
            if (g.bases.back() != c.total_cts) throw DataError("ciphertext blob does not match the circuit");
        }
        n->net = std::make_unique<Network>();
        Network& N = *n->net;
        N.c = &c;
        upload_circuit(c);
        network_reserve(N, batch, host);  // host-resident: a one-layer device window
        N.host_gc = host;
        std::vector<uint32_t> zero((size_t)batch * c.k * LABW);
        std::vector<U4> commit(batch);
        DevBuf ref;  // one inference's rows in the reference order, then permuted on the device
        if (host) N.hblob.ensure(std::max<uint64_t>((uint64_t)batch * c.total_cts, 1) * 16);
        else ref.ensure(std::max<uint64_t>(c.total_cts, 1) * 16);
        for (uint32_t b = 0; b < batch; ++b) {
            for (int i = 0; i < c.k; ++i)
                host_decompress(gs[b].zero[i], c.base.primes[i], zero.data() + ((size_t)b * c.k + i) * LABW);
            if (host) {
                std::memcpy(N.hblob.as<U4>() + (uint64_t)b * c.total_cts, gs[b].cts, c.total_cts * 16);
            } else {
                dev::h2d(ref.p, gs[b].cts, c.total_cts * 16, g_stream);
                blob_permute(c, ref.as<U4>(), N.blob.as<U4>() + (uint64_t)b * c.total_cts, false);
            }
            commit[b] = u128_to_u4(gs[b].commit);
        }
        dev::h2d(N.zero.p, zero.data(), zero.size() * 4, g_stream);
        dev::h2d(N.commit.p, commit.data(), commit.size() * 16, g_stream);
        // garbler-only state stays zero on an evaluator network
        dev::memset0(N.Rb.p, N.Rb.n, g_stream);
        dev::memset0(N.rk.p, N.rk.n, g_stream);
        dev::sync(g_stream);
        *out = n.release();
    }
}

int dashgpu_import_gc(const uint8_t* const* gcs, const size_t* lens, uint32_t batch, dashgpu_network** out) {
    return guarded([&] { import_gc(gcs, lens, batch, out, false); });
}

int dashgpu_import_gc_host(const uint8_t* const* gcs, const size_t* lens, uint32_t batch, dashgpu_network** out) {
    return guarded([&] { import_gc(gcs, lens, batch, out, true); });
}

int dashgpu_network_circuit(const dashgpu_network* n, const dashgpu_circuit** out) {
    return guarded([&] {
        if (!n || !out) throw DataError("null argument");
        *out = n->net->c;
    });
}

int dashgpu_tamper_ct(dashgpu_network* n, uint32_t b, uint64_t index, const uint8_t* mask16) {
    return guarded([&] {
        Network& N = *n->net;
        if (b >= N.B || index >= N.c->total_cts) throw DataError("ciphertext index out of range");
        N.require_gc();
        if (N.host_gc) {
            uint8_t* h = reinterpret_cast<uint8_t*>(N.hblob.as<U4>() + (uint64_t)b * N.c->total_cts + index);
            for (int i = 0; i < 16; ++i) h[i] ^= mask16[i];
            return;
        }
        U4 v;
        U4* p = N.blob.as<U4>() + (uint64_t)b * N.c->total_cts + device_ct_index(*N.c, index);
        dev::d2h(&v, p, 16, g_stream);
        dev::sync(g_stream);
        uint8_t* vb = reinterpret_cast<uint8_t*>(&v);
        for (int i = 0; i < 16; ++i) vb[i] ^= mask16[i];
        dev::h2d(p, &v, 16, g_stream);
        dev::sync(g_stream);
    });
}

// device bytes one inference of dashgpu_infer needs: ciphertexts (whole GC,
// or its largest layer when layer-windowed) + multiples + planes of every
// layer for garbler and evaluator + gadget slots + decode table
static uint64_t per_inference_bytes(const dashgpu_circuit& c, bool windowed) {
    uint64_t planes = 0;
    {
        uint64_t sumE = 3 * c.n_in + 2 * c.n_out;
        for (const auto& l : c.layers)
            if (l.kind != DASH_LAYER_FLATTEN) sumE += 2 * l.E_out;
        for (int p : c.base.primes) planes += (uint64_t)((n_digits_host(p) + 3) / 4) * sumE * 4;
    }
    uint64_t slots = 0;
    for (const auto& l : c.layers)
        if (l.tape) {
            const uint64_t sl = (uint64_t)std::max(l.tape->nslots, l.tape->nslots_lv) * l.E_out * 16 +
                                (uint64_t)l.E_out * c.k * 2 * 16;  // + mixed-modulus labels
            slots = windowed ? std::max(slots, sl) : slots + sl;
        }
    return (windowed ? max_layer_cts(c) : c.total_cts) * 16 + (uint64_t)(MAXMOD - 1) * 128 * NWMAX * 4 + planes +
           slots + c.n_out * 600 * 16 + 4096;
}

// per-layer tree digests of a network's held GC (whole-GC device blob or
// host-resident rows): the evaluator's side of the digest parity mode
static void network_digest(const Network& n, uint32_t b, uint8_t* digests) {
    const dashgpu_circuit& c = *n.c;
    if (b >= n.B) throw DataError("inference index out of range");
    n.require_gc();
    if (n.windowed && !n.host_gc) throw DataError("garbled circuit is not held whole");
    const size_t L = c.layers.size();
    DevBuf leaves, roots, rows;
    leaves.ensure(std::max<size_t>((max_layer_cts(c) + kDigestLeafRows - 1) / kDigestLeafRows, 1) * 32);
    roots.ensure(std::max<size_t>(L, 1) * 32);
    if (n.host_gc) rows.ensure(std::max<uint64_t>(max_layer_cts(c), 1) * 16);
    for (size_t li = 0; li < L; ++li) {
        const HLayer& l = c.layers[li];
        DigestParams P;
        std::memset(&P, 0, sizeof P);
        P.rows = l.cts;
        P.stride = l.cts;
        P.B = 1;
        P.leaves = (uint32_t)((l.cts + kDigestLeafRows - 1) / kDigestLeafRows);
        P.out = leaves.as<uint32_t>();
        if (n.host_gc) {  // reference order already: copy the layer up
            dev::h2d(rows.p, n.hblob.as<U4>() + (uint64_t)b * c.total_cts + l.ct_base, l.cts * 16, g_stream);
            P.src = rows.as<U4>();
        } else {
            P.src = n.blob.as<U4>() + (uint64_t)b * c.total_cts + l.ct_base;
            P.E = l.tape ? l.E_out : 0;
            P.uc = l.tape ? l.tape->cts : 0;
        }
        launch_digest(P, roots.as<uint32_t>() + li * 8, g_stream);
    }
    std::vector<uint32_t> hr(L * 8);
    dev::d2h(hr.data(), roots.p, hr.size() * 4, g_stream);
    dev::sync(g_stream);
    for (size_t i = 0; i < L * 8; ++i)
        for (int q = 0; q < 4; ++q) digests[4 * i + q] = (uint8_t)(hr[i] >> (24 - 8 * q));
}

int dashgpu_network_digest(const dashgpu_network* n, uint32_t b, uint8_t* digests) {
    return guarded([&] {
        if (!n || !digests) throw DataError("null argument");
        network_digest(*n->net, b, digests);
    });
}

int dashgpu_garble_digest(const dashgpu_circuit* cc, const uint8_t* seeds, uint32_t batch, uint8_t* digests) {
    return guarded([&] {
        auto* c = const_cast<dashgpu_circuit*>(cc);
        {
            std::lock_guard<std::mutex> lk(c->mu);
            upload_circuit(*c);
        }
        Network n;
        n.c = c;
        const uint64_t per = per_inference_bytes(*c, true);
        const uint32_t chunk =
            (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(batch, (uint64_t)(dev::free_bytes() * 0.85) / per));
        for (uint32_t b0 = 0; b0 < batch; b0 += chunk) {
            const uint32_t B = std::min(chunk, batch - b0);
            garble_digest_into(n, seeds + (size_t)16 * b0, B, digests + (size_t)b0 * c->layers.size() * 32);
        }
    });
}

int dashgpu_infer(const dashgpu_circuit* cc, const uint8_t* seeds, uint32_t batch, const int64_t* inputs,
                  int64_t* outputs, int on_device, dashgpu_timing* t) {
    return guarded([&] {
        auto* c = const_cast<dashgpu_circuit*>(cc);
        // one workspace per stream: the circuit lock covers the lookup and
        // the one-time parameter upload, the workspace lock this stream's work
        dashgpu_circuit::Workspace* wsp;
        {
            std::lock_guard<std::mutex> lk(c->mu);
            auto& slot = c->workspaces[g_stream];
            if (!slot) slot = std::make_unique<dashgpu_circuit::Workspace>();
            wsp = slot.get();
            upload_circuit(*c);
        }
        std::lock_guard<std::mutex> lk(wsp->mu);
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        auto make_ws = [&](std::unique_ptr<Network>& ws) {
            if (!ws) {
                ws = std::make_unique<Network>();
                ws->c = c;
                ws->bin = std::make_unique<Bundle>();
                ws->bout = std::make_unique<Bundle>();
            }
            return ws.get();
        };
        dashgpu_timing tm;
        std::memset(&tm, 0, sizeof tm);
        // One network, sub-batched to free HBM.  (Running two half-batches on
        // two streams was measured slower: the persistent garbling / eval
        // CTAs hold 196-218 KB of shared memory, so the other stream's
        // kernels cannot co-reside and the halves serialize.)
        Network& n = *make_ws(wsp->net);
        // Whole GCs per sub-batch, or layer-windowed (infer_layerwise) when
        // the batch's GCs exceed the HBM budget and a window admits a larger
        // sub-batch; DASHGPU_LAYERWISE=0/1 forces either schedule.
        const char* force = std::getenv("DASHGPU_LAYERWISE");
        uint32_t chunk = batch;
        bool layerwise = n.windowed;
        if (!force && n.plan_batch == batch && n.plan_chunk) {  // this batch size was planned before
            chunk = n.plan_chunk;
            layerwise = n.plan_layerwise;
        } else if (n.cap < batch || force) {
            // (cudaMemGetInfo is only asked when the workspace must grow: it
            // costs far more than the rest of the host side of a call)
            const uint64_t per = per_inference_bytes(*c, false), per_w = per_inference_bytes(*c, true);
            // free HBM plus what this workspace already holds (its last schedule)
            const uint64_t avail =
                (uint64_t)(dev::free_bytes() * 0.85) + (uint64_t)n.cap * (n.windowed ? per_w : per);
            auto fit = [&](uint64_t p) {
                return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(batch, avail / p));
            };
            chunk = fit(per);
            layerwise = chunk < batch && fit(per_w) > chunk;
            if (force) layerwise = force[0] == '1';
            if (layerwise) chunk = fit(per_w);
        }
        n.plan_batch = force ? 0 : batch;
        n.plan_chunk = chunk;
        n.plan_layerwise = layerwise;
        Bundle& in = *n.bin;
        Bundle& out = *n.bout;
        for (uint32_t b0 = 0; b0 < batch; b0 += chunk) {
            // one host sync per sub-batch: everything up to the decoded
            // residues is enqueued back to back (range / authenticity flags
            // are checked after the sync)
            const uint32_t B = std::min(chunk, batch - b0);
            const auto a = clk::now();
            if (layerwise) {
                infer_layerwise(n, seeds + (size_t)16 * b0, B, on_device != 0, inputs + (size_t)b0 * c->n_in, in, out);
            } else {
                garble_into(n, seeds + (size_t)16 * b0, B, on_device != 0);
                encode_enqueue(n, inputs + (size_t)b0 * c->n_in, on_device != 0, in);
                evaluate_into(n, in, out);
            }
            decode_enqueue(n, out, on_device ? outputs + (size_t)b0 * c->n_out : nullptr);
            dev::sync(g_stream);
            encode_finish(n);
            decode_finish(n, outputs + (size_t)b0 * c->n_out, on_device != 0);
            tm.ms_garble += std::chrono::duration<double, std::milli>(clk::now() - a).count();
            tm.sub_batches += 1;
        }
        tm.layerwise = layerwise ? 1 : 0;
        if (!on_device) {
            // seeds + quantized inputs in, decoded outputs out (AES key
            // schedules are expanded on the device, launch parameters are
            // staged once per network)
            tm.h2d_bytes = (uint64_t)batch * (c->n_in * 8 + 16);
            tm.d2h_bytes = (uint64_t)batch * c->n_out * 8;
        }
        tm.ms_total = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        if (t) *t = tm;
    });
}

int dashgpu_infer_stream(const dashgpu_circuit* cc, const uint8_t* seeds, uint32_t batch, const int64_t* inputs,
                         int64_t* outputs, uint64_t chunk_elems, uint8_t* gc_out, dashgpu_timing* t) {
    return dashgpu_infer_stream_range(cc, seeds, batch, inputs, outputs, chunk_elems, 0, ~0ull, gc_out, t);
}

int dashgpu_infer_stream_range(const dashgpu_circuit* cc, const uint8_t* seeds, uint32_t batch,
                               const int64_t* inputs, int64_t* outputs, uint64_t chunk_elems, uint64_t u_begin,
                               uint64_t u_end, uint8_t* gc_out, dashgpu_timing* t) {
    return guarded([&] {
        auto* c = const_cast<dashgpu_circuit*>(cc);
        std::lock_guard<std::mutex> lk(c->mu);
        dashgpu_timing tm;
        std::memset(&tm, 0, sizeof tm);
        const auto t0 = std::chrono::steady_clock::now();
        infer_stream(*c, seeds, batch, inputs, outputs, chunk_elems, gc_out, tm, u_begin, u_end);
        tm.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (t) *t = tm;
    });
}

int dashgpu_profile(int enable) {
    return guarded([&] {
        dev::prof_enable(enable);
        dev::prof_reset();
    });
}

int dashgpu_profile_read(double* ms, uint64_t* launches, int max_kinds) {
    int k = 0;
    int rc = guarded([&] { k = dev::prof_read(ms, launches, max_kinds); });
    return rc ? -rc : k;
}

int dashgpu_activation_tape(const dashgpu_circuit* c, int kind, dashgpu_tape_op* ops, uint32_t cap, uint32_t* n) {
    return guarded([&] {
        if (!c || !n) throw DataError("null argument");
        const auto& t = kind == DASH_LAYER_SIGNACT ? c->sign_tape : c->relu_tape;
        if (!t) throw DataError("circuit has no activation layer");
        *n = (uint32_t)t->ops.size();
        if (!ops) return;
        for (uint32_t i = 0; i < *n && i < cap; ++i) {
            const TapeOp& o = t->ops[i];
            ops[i] = dashgpu_tape_op{o.kind, o.pm, o.qm, o.gate_off, o.wire_off, o.ct_off};
        }
    });
}

int dashgpu_last_act_launch(int garble, uint32_t out[5]) {
    return guarded([&] {
        const dev::ActShape s = dev::last_act_shape(garble != 0);
        out[0] = s.variant;
        out[1] = s.nchunks;
        out[2] = s.grid;
        out[3] = s.items;
        out[4] = s.group;
    });
}

int dashgpu_prim(int op, uint32_t n, int m, int q, const uint64_t* in, uint64_t* out, uint16_t* digits,
                 const uint8_t* key16, const uint64_t* wires, uint64_t gate) {
    return guarded([&] {
        check_constants();
        if (m < 2 || m > MAXMOD || ((op == 4 || op == 5) && (q < 2 || q > MAXMOD)))
            throw DataError("modulus out of range");
        DevBuf din, dout, ddig, drk, dw;
        din.ensure((size_t)n * 16);
        dout.ensure((size_t)n * 16);
        ddig.ensure((size_t)n * LABW * 4);
        drk.ensure(44 * 4);
        dw.ensure((size_t)n * 8);
        if (in) dev::h2d(din.p, in, (size_t)n * 16, g_stream);
        if (out && (op == 4 || op == 5)) dev::h2d(dout.p, out, (size_t)n * 16, g_stream);
        if (key16) {
            uint32_t rk[44];
            aes_expand_host(key16, rk);
            dev::h2d(drk.p, rk, sizeof rk, g_stream);
        }
        if (wires) dev::h2d(dw.p, wires, (size_t)n * 8, g_stream);
        dev::memset0(ddig.p, (size_t)n * LABW * 4, g_stream);
        PrimParams P;
        std::memset(&P, 0, sizeof P);
        P.op = op;
        P.n = n;
        P.m = (uint32_t)m;
        P.q = (uint32_t)q;
        P.in = din.as<U4>();
        P.out = dout.as<U4>();
        P.digits = ddig.as<uint32_t>();
        P.rk = drk.as<uint32_t>();
        P.wires = dw.as<uint64_t>();
        P.gate = gate;
        launch_prim(P, g_stream);
        if (out) dev::d2h(out, dout.p, (size_t)n * 16, g_stream);
        std::vector<uint32_t> dg((size_t)n * LABW);
        dev::d2h(dg.data(), ddig.p, dg.size() * 4, g_stream);
        dev::sync(g_stream);
        if (digits)
            for (size_t i = 0; i < (size_t)n * 128; ++i) digits[i] = (uint16_t)((dg[i / 4] >> (8 * (i % 4))) & 0xff);
    });
}

// ---- t_proj primitive (gadgets.hpp:146-176) ----
static void proj_setup(const uint8_t* seed16, int p, int q, DevBuf& rk, DevBuf& mult, DevBuf& scratch) {
    uint32_t k44[44];
    aes_expand_host(seed16, k44);
    rk.ensure(sizeof k44);
    dev::h2d(rk.p, k44, sizeof k44, g_stream);
    const uint64_t mult_stride = (uint64_t)(MAXMOD - 1) * 128 * NWMAX;
    mult.ensure(mult_stride * 4);
    scratch.ensure(4096);
    SetupParams S;
    std::memset(&S, 0, sizeof S);
    S.B = 1;
    S.k = 1;
    S.primes[0] = (uint16_t)p;
    S.slot_mod[S.nslot++] = (uint16_t)p;
    if (q != p) S.slot_mod[S.nslot++] = (uint16_t)q;
    S.rk = rk.as<uint32_t>();
    S.seeds = scratch.as<uint8_t>();
    S.mult = mult.as<uint32_t>();
    S.mult_stride = mult_stride;
    S.n_in = 0;
    S.base_planes[0] = scratch.as<uint32_t>();
    S.zero = scratch.as<uint32_t>() + 256;
    S.Rb = scratch.as<uint32_t>() + 512;
    S.commit = scratch.as<U4>() + 64;
    launch_setup(S, g_stream);
}

int dashgpu_proj_garble(const uint8_t* seed16, uint32_t n, int p, int q, const uint8_t* phi, const uint64_t* in,
                        const uint64_t* gates, const uint64_t* wires, uint64_t* rows, uint64_t* out0,
                        uint64_t* offsets) {
    return guarded([&] {
        check_constants();
        if (p < 2 || p > MAXMOD || q < 2 || q > MAXMOD) throw DataError("modulus out of range");
        for (int a = 0; a < p; ++a)
            if (phi[a] >= q) throw DataError("projection table value out of range");
        DevBuf rk, mult, scratch, dphi, din, dg, dw, drows, dout;
        proj_setup(seed16, p, q, rk, mult, scratch);
        dphi.ensure(p);
        dev::h2d(dphi.p, phi, p, g_stream);
        din.ensure((size_t)n * 16);
        dg.ensure((size_t)n * 8);
        dw.ensure((size_t)n * 8);
        drows.ensure((size_t)n * p * 16);
        dout.ensure((size_t)n * 16);
        if (n) {
            dev::h2d(din.p, in, (size_t)n * 16, g_stream);
            dev::h2d(dg.p, gates, (size_t)n * 8, g_stream);
            dev::h2d(dw.p, wires, (size_t)n * 8, g_stream);
        }
        ProjParams P;
        std::memset(&P, 0, sizeof P);
        P.n = n;
        P.p = (uint32_t)p;
        P.q = (uint32_t)q;
        P.phi = dphi.as<uint8_t>();
        P.in = din.as<U4>();
        P.gates = dg.as<uint64_t>();
        P.wires = dw.as<uint64_t>();
        P.rows = drows.as<U4>();
        P.out = dout.as<U4>();
        P.rk = rk.as<uint32_t>();
        P.mult = mult.as<uint32_t>();
        P.garbler = 1;
        launch_proj(P, g_stream);
        if (n) {
            dev::d2h(rows, drows.p, (size_t)n * p * 16, g_stream);
            dev::d2h(out0, dout.p, (size_t)n * 16, g_stream);
        }
        std::vector<uint32_t> R(2 * NWMAX);
        dev::d2h(R.data(), mult.as<uint32_t>() + ((uint64_t)(p - 2) * 128 + 1) * NWMAX, NWMAX * 4, g_stream);
        dev::d2h(R.data() + NWMAX, mult.as<uint32_t>() + ((uint64_t)(q - 2) * 128 + 1) * NWMAX, NWMAX * 4, g_stream);
        dev::sync(g_stream);
        if (offsets) {
            // multiples-table rows: byte digits, or the packed-bit (= compressed) form for powers of two
            auto comp = [](const uint32_t* w, int m) {
                if ((m & (m - 1)) == 0) return ((u128)w[3] << 96) | ((u128)w[2] << 64) | ((u128)w[1] << 32) | w[0];
                return host_compress(w, m);
            };
            const u128 rp = comp(R.data(), p), rq = comp(R.data() + NWMAX, q);
            offsets[0] = (uint64_t)rp;
            offsets[1] = (uint64_t)(rp >> 64);
            offsets[2] = (uint64_t)rq;
            offsets[3] = (uint64_t)(rq >> 64);
        }
    });
}

// Device-resident t_proj over n gates (the raw projection sweep, SURVEY
// 8(d) (ii); bench_main.cpp:40-74 times one gate at a time on the CPU): the
// context holds the PRF key schedule and the multiples tables of R_p / R_q,
// every buffer argument is a device pointer, work is enqueued on the calling
// thread's stream without a host sync.
struct dashgpu_proj_ctx {
    int p = 0, q = 0;
    dashgpu::DevBuf rk, mult, scratch, phi;
};

int dashgpu_proj_ctx_create(const uint8_t* seed16, int p, int q, const uint8_t* phi, dashgpu_proj_ctx** out) {
    return guarded([&] {
        check_constants();
        if (!seed16 || !phi || !out) throw DataError("null argument");
        if (p < 2 || p > MAXMOD || q < 2 || q > MAXMOD) throw DataError("modulus out of range");
        for (int a = 0; a < p; ++a)
            if (phi[a] >= q) throw DataError("projection table value out of range");
        auto c = std::make_unique<dashgpu_proj_ctx>();
        c->p = p;
        c->q = q;
        proj_setup(seed16, p, q, c->rk, c->mult, c->scratch);
        c->phi.ensure(p);
        dev::h2d(c->phi.p, phi, p, g_stream);
        dev::sync(g_stream);
        *out = c.release();
    });
}

void dashgpu_proj_ctx_destroy(dashgpu_proj_ctx* c) { delete c; }

static ProjParams proj_params(const dashgpu_proj_ctx* c, uint32_t n, const void* in, const void* gates, void* rows,
                              void* out) {
    if (!c) throw DataError("null projection context");
    if (n && (!in || !gates || !rows || !out)) throw DataError("null device buffer");
    ProjParams P;
    std::memset(&P, 0, sizeof P);
    P.n = n;
    P.p = (uint32_t)c->p;
    P.q = (uint32_t)c->q;
    P.phi = c->phi.as<uint8_t>();
    P.in = static_cast<const U4*>(in);
    P.gates = static_cast<const uint64_t*>(gates);
    P.rows = static_cast<U4*>(rows);
    P.out = static_cast<U4*>(out);
    P.rk = c->rk.as<uint32_t>();
    P.mult = c->mult.as<uint32_t>();
    return P;
}

int dashgpu_proj_garble_dev(const dashgpu_proj_ctx* c, uint32_t n, const void* in, const void* gates,
                            const void* wires, void* rows, void* out0) {
    return guarded([&] {
        ProjParams P = proj_params(c, n, in, gates, rows, out0);
        if (n && !wires) throw DataError("null device buffer");
        P.wires = static_cast<const uint64_t*>(wires);
        P.garbler = 1;
        if (n) launch_proj(P, g_stream);
    });
}

int dashgpu_proj_eval_dev(const dashgpu_proj_ctx* c, uint32_t n, const void* in, const void* gates,
                          const void* rows, void* out) {
    return guarded([&] {
        ProjParams P = proj_params(c, n, in, gates, const_cast<void*>(rows), out);
        if (n) launch_proj(P, g_stream);
    });
}

int dashgpu_proj_eval(uint32_t n, int p, int q, const uint64_t* in, const uint64_t* gates, const uint64_t* rows,
                      uint64_t* out) {
    return guarded([&] {
        check_constants();
        if (p < 2 || p > MAXMOD || q < 2 || q > MAXMOD) throw DataError("modulus out of range");
        DevBuf din, dg, drows, dout;
        din.ensure((size_t)n * 16);
        dg.ensure((size_t)n * 8);
        drows.ensure((size_t)n * p * 16);
        dout.ensure((size_t)n * 16);
        if (n) {
            dev::h2d(din.p, in, (size_t)n * 16, g_stream);
            dev::h2d(dg.p, gates, (size_t)n * 8, g_stream);
            dev::h2d(drows.p, rows, (size_t)n * p * 16, g_stream);
        }
        ProjParams P;
        std::memset(&P, 0, sizeof P);
        P.n = n;
        P.p = (uint32_t)p;
        P.q = (uint32_t)q;
        P.in = din.as<U4>();
        P.gates = dg.as<uint64_t>();
        P.rows = drows.as<U4>();
        P.out = dout.as<U4>();
        launch_proj(P, g_stream);
        if (n) dev::d2h(out, dout.p, (size_t)n * 16, g_stream);
        dev::sync(g_stream);
    });
}

}  // extern "C"
