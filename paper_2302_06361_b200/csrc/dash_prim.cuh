// Primitive-level entry points used only by the parity tests (they exercise
// the exact device code paths the gadget kernels use).
#pragma once

#include "launch.hpp"

namespace dashgpu {

DASH_HD void prim_thread(const PrimParams& P, uint32_t i, const AesTab& t) {
    uint32_t buf[2][NWMAX] = {};
    const LB A{buf[0], 1}, B{buf[1], 1};
    switch (P.op) {
        case 0: {  // decompress_mod + compress (label.cpp:208-232)
            const ModC& M = c_mod[P.m];
            lb_decompress(A, P.in[i], M);
            lb_store_rows(A, P.digits + (uint64_t)i * LABW, 1, M);
            lb_load_rows(B, P.digits + (uint64_t)i * LABW, 1, M);
            P.out[i] = lb_compress(B, M);
            break;
        }
        case 1:
            P.out[i] = aes_pi(P.in[i], t);
            break;
        case 2:
            P.out[i] = aes_key(P.in[i], P.rk, t);
            break;
        case 3: {  // LabelPrf::label / offset draw (prf.cpp:11-27)
            const ModC& M = c_mod[P.m];
            lb_prf(A, P.wires[i], P.q, M, P.rk, t);
            lb_store_rows(A, P.digits + (uint64_t)i * LABW, 1, M);
            break;
        }
        case 4: {  // encrypt_label with key = decompress(in, m), msg = decompress(out, q)
            const ModC& Mk = c_mod[P.m];
            const ModC& Mq = c_mod[P.q];
            lb_decompress(A, P.in[i], Mk);
            lb_decompress(B, P.out[i], Mq);
            const U4 H = hash_tw(lb_compress(A, Mk), P.gate, i % 7u, i % 3u, t);
            P.out[i] = lb_enc(H, B, nullptr, nullptr, 0, Mq);
            break;
        }
        case 5: {  // decrypt_label
            const ModC& Mk = c_mod[P.m];
            const ModC& Mq = c_mod[P.q];
            lb_decompress(A, P.in[i], Mk);
            const U4 H = hash_tw(lb_compress(A, Mk), P.gate, i % 7u, i % 3u, t);
            lb_dec(B, P.out[i], H, Mq);
            lb_store_rows(B, P.digits + (uint64_t)i * LABW, 1, Mq);
            break;
        }
    }
}

}  // namespace dashgpu
