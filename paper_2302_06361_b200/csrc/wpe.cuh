// Lane-group garbling for small launches (batch-1 models such as BASELINE
// configs[0], Model A at batch 1: 256 ReLU elements would occupy 8 warps of
// the whole GPU with one element per thread).  A group of G lanes (a power of
// two, up to the whole warp) garbles one element: the rows of every gate are
// split over the group (row a by lane a mod G, key x + a R_p from the
// multiples table instead of the running key step), the fresh output label's
// PRF blocks too, and the operands / labels shared by the rows live in
// group-shared shared memory.
// The ciphertexts, slots and outputs are exactly those of the per-thread tape
// interpreter (dash_device.cuh garble_op), which the gadget semantics follow
// (gadgets.hpp:146-358).
#pragma once

#include "dash_device.cuh"

namespace dashgpu {

// Per-group buffers: X (operand x / GRR scratch), A (fresh or payload label),
// K (operand y of half gates) shared by the group's lanes (stride 1,
// broadcast reads); KEY private per lane (stride 32) for the row key.  A warp
// holds 32 / G groups: kWpeWords covers the worst case G = 1... 32 of them.
constexpr int kWpeShared = 3 * NWMAX;
constexpr int kWpeWords = kWpeShared * 32 + NWMAX * 32;

struct WpeBufs {
    LB X, A, K, KEY;
};

// LabelPrf::draw (prf.cpp:11-27) with the counter blocks split over the lanes
static __device__ void prf_coop(LB L, uint64_t wire, uint32_t stream, uint32_t m, const uint32_t* rk, const AesTab& t,
                         uint32_t j, uint32_t G) {
    const ModC& M = c_mod[m];
    const int nb = (M.n + 3) / 4;
    U4 acc;
    acc.x[0] = acc.x[1] = acc.x[2] = acc.x[3] = 0;
    for (int b = (int)j; b < nb; b += (int)G) {
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
            for (int j = 0; j < 4; ++j) {
                const int i = 4 * b + j;
                if (i < M.n) u4_or_shl(acc, o.x[j] & (M.m - 1u), (uint32_t)(M.e * i));
            }
        }
    }
    if (M.pow2) {
        for (int i = 0; i < 4; ++i) {
            uint32_t v = acc.x[i];
            for (uint32_t off = G >> 1; off > 0; off >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, off);
            acc.x[i] = v & M.bits[i];
        }
        if (j == 0) lb_set_u4(L, acc);
    }
    __syncwarp();
}

// The rows of a projection / half gate (garble_rows_n), lane a mod 32 takes row
// (cin + a) mod p with key X + a R_p and payload base + v(a) R_q.
static __device__ void garble_rows_w(LB X, LB base, LB KEY, const AesTab& t, const uint32_t* mult, uint32_t p, uint32_t q,
                              uint32_t cin, uint64_t g, const uint8_t* phi, uint32_t r, U4* R, int grr,
                              uint32_t rs, uint32_t j, uint32_t G) {
    const ModC& Mp = c_mod[p];
    const ModC& Mq = c_mod[q];
    const uint32_t* Mp0 = mult + (uint64_t)c_modslot[p] * 128u * NWMAX;
    const uint32_t* Mq0 = mult + (uint64_t)c_modslot[q] * 128u * NWMAX;
    for (uint32_t a = j; a < p; a += G) {
        uint32_t row = cin + a;
        row = row >= p ? row - p : row;
        lb_copy(KEY, X, Mp);
        lb_add_g(KEY, Mp0 + (uint64_t)a * NWMAX, Mp);
        const U4 H = hash_tw(lb_compress(KEY, Mp), g, row, 0, t);
        const uint32_t v = phi ? phi[a] : (a * r) % p;
        const U4 ct = lb_enc(H, base, Mq0 + (uint64_t)v * NWMAX, nullptr, 0, Mq);
        if (!grr) R[(uint64_t)row * rs] = ct;
        else if (row != 0) R[(uint64_t)(row - 1) * rs] = ct;
    }
    __syncwarp();
}

static __device__ void load_w(LB L, const ActParams& P, const Elt& e, uint8_t v, const ModC& M, uint32_t j) {
    if (j == 0) load_operand(L, P, e, v, M);
    __syncwarp();
}

static __device__ void garble_op_w(const ActParams& P, Elt& e, const TapeOp& op, const WpeBufs& w, uint32_t j,
                            uint32_t G) {
    switch (op.kind) {
        case OP_PROJ:
        case OP_GRR: {  // t_proj (gadgets.hpp:146-176), t_proj_grr (181-221)
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[op.qm];
            const uint32_t p = op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            const uint8_t* phi = P.phi + op.phi_off;
            load_w(w.X, P, e, op.a, Mp, j);
            const uint32_t cin = lb_color(w.X, Mp);
            if (op.kind == OP_PROJ) {
                prf_coop(w.A, e.wire0 + op.wire_off, 0, op.qm, e.rk, e.t, j, G);
            } else {
                if (j == 0) {  // out0 = -pad(key0, {g,0,0}) - phi(a0) R_q, key0 = in + a0 R_p
                    const uint32_t a0 = cin == 0 ? 0 : p - cin;
                    lb_copy(w.A, w.X, Mp);
                    lb_add_g(w.A, mult_row(e, p, a0), Mp);
                    const U4 H0 = hash_tw(lb_compress(w.A, Mp), g, 0, 0, e.t);
                    lb_decompress(w.A, H0, Mq);
                    lb_neg(w.A, Mq);
                    lb_sub_g(w.A, mult_row(e, op.qm, phi[a0]), Mq);
                }
                __syncwarp();
            }
            garble_rows_w(w.X, w.A, w.KEY, e.t, e.mult, p, op.qm, cin, g, phi, 0,
                          e.rows + (uint64_t)op.ct_off * e.rs, op.kind == OP_GRR, e.rs, j, G);
            if (j == 0) store_slot(e, op.out, w.A, Mq);
            __syncwarp();
            break;
        }
        case OP_HALF:      // t_half_gate (gadgets.hpp:230-282)
        case OP_MMHALF: {  // t_mm_half_gate (gadgets.hpp:292-358)
            const bool mm = op.kind == OP_MMHALF;
            const ModC& Mp = c_mod[op.pm];
            const ModC& Mq = c_mod[mm ? op.qm : op.pm];
            const uint32_t p = op.pm, q = mm ? op.qm : op.pm;
            const uint64_t g = e.gate0 + op.gate_off;
            U4* R = e.rows + (uint64_t)op.ct_off * e.rs;
            if (j == 0) {
                load_operand(w.K, P, e, op.b, Mq);
                load_operand(w.X, P, e, op.a, Mp);
            }
            __syncwarp();
            const uint32_t cy = lb_color(w.K, Mq), cx = lb_color(w.X, Mp);
            const uint32_t r = mm ? cx : cy;
            // garbler rows: key x + aR_p, payload u0 + (a r mod p) R_p
            const U4* ml = (op.cst && P.mmlab) ? P.mmlab + (((uint64_t)e.b * P.E + e.u) * P.k + (op.cst - 1)) * 2
                                               : nullptr;
            if (ml) {
                if (j == 0) lb_decompress(w.A, ml[0], Mp);
                __syncwarp();
            } else {
                prf_coop(w.A, e.wire0 + op.wire_off, 0, op.pm, e.rk, e.t, j, G);
            }
            const U4 u0c = lb_compress(w.A, Mp);
            garble_rows_w(w.X, w.A, w.KEY, e.t, e.mult, p, p, cx, g, nullptr, r, R, 0, e.rs, j, G);
            // evaluator rows: key y + bR_q, payload v0 - s x
            if (ml) {
                if (j == 0) lb_decompress(w.A, ml[1], Mp);
                __syncwarp();
            } else {
                prf_coop(w.A, e.wire0 + op.wire_off + 1, 0, op.pm, e.rk, e.t, j, G);
            }
            const uint32_t fw = field_width(p);
            const uint32_t fmask = (1u << fw) - 1u;
            U4 sb;
            sb.x[0] = sb.x[1] = sb.x[2] = sb.x[3] = 0;
            for (uint32_t b = j; b < q; b += G) {
                uint32_t row = cy + b;
                row = row >= q ? row - q : row;
                uint32_t s = r + b;
                s = s >= p ? s - p : s;
                lb_copy(w.KEY, w.K, Mq);
                lb_add_g(w.KEY, mult_row(e, q, b), Mq);
                const U4 Kc = lb_compress(w.KEY, Mq);
                LB X = w.X;
                R[(uint64_t)(p + row) * e.rs] = lb_enc(hash_tw(Kc, g, row, 1, e.t), w.A, nullptr, &X, mm ? s : row, Mp);
                if (mm) {  // encrypt_short field of this row (cipher.cpp:45-60)
                    const U4 Hs = hash_tw(Kc, g, 0, 2, e.t);
                    u4_or_shl(sb, (s ^ (Hs.x[0] & fmask)) & fmask, fw * row);
                }
            }
            if (mm) {
                for (int i = 0; i < 4; ++i)
                    for (uint32_t off = G >> 1; off > 0; off >>= 1)
                        sb.x[i] |= __shfl_xor_sync(0xffffffffu, sb.x[i], off);
                if (j == 0) R[(uint64_t)(p + q) * e.rs] = sb;
            }
            __syncwarp();
            if (j == 0) {
                lb_sub_c(w.A, u0c, Mp);  // out = v0 - u0
                store_slot(e, op.out, w.A, Mp);
            }
            __syncwarp();
            break;
        }
        case OP_ADD:
        case OP_ADDACC:
        case OP_ADDCONST:
            if (j == 0) garble_op(P, e, op);
            __syncwarp();
            break;
        case OP_OUTPUT:  // written up front by act_output_thread
            break;
    }
}

}  // namespace dashgpu
