// Primitive-level entry points used only by the parity tests (they exercise
// the exact device code paths the gadget kernels use).
#pragma once

#include "launch.hpp"

namespace dashgpu {

DASH_HD void prim_thread(const PrimParams& P, uint32_t i, const AesTab& t) {
    switch (P.op) {
        case 0: {  // decompress_mod + compress (label.cpp:208-232)
            const ModC& M = c_mod[P.m];
            Lab L;
            decompress(L, P.in[i], M);
            lab_store_rows(L, P.digits + (uint64_t)i * LABW, 1, M);
            Lab R;
            lab_load_rows(R, P.digits + (uint64_t)i * LABW, 1, M);
            P.out[i] = compress(R, M);
            break;
        }
        case 1:
            P.out[i] = aes_pi(P.in[i], t);
            break;
        case 2:
            P.out[i] = aes_key(P.in[i], P.rk, t);
            break;
        case 3: {  // LabelPrf::label / offset (prf.cpp:11-27)
            const ModC& M = c_mod[P.m];
            Lab L;
            prf_label(L, P.wires[i], P.q, M, P.rk, t);
            lab_store_rows(L, P.digits + (uint64_t)i * LABW, 1, M);
            break;
        }
        case 4: {  // encrypt_label with key = decompress(in, m), msg = decompress(out, q)
            const ModC& Mk = c_mod[P.m];
            const ModC& Mq = c_mod[P.q];
            Lab key, msg;
            decompress(key, P.in[i], Mk);
            decompress(msg, P.out[i], Mq);
            const U4 H = hash_tw(compress(key, Mk), P.gate, i % 7u, i % 3u, t);
            P.out[i] = enc_with(H, msg, Mq);
            break;
        }
        case 5: {  // decrypt_label
            const ModC& Mk = c_mod[P.m];
            const ModC& Mq = c_mod[P.q];
            Lab key, msg;
            decompress(key, P.in[i], Mk);
            dec_row(msg, key, Mk, P.gate, i % 7u, i % 3u, P.out[i], Mq, t);
            lab_store_rows(msg, P.digits + (uint64_t)i * LABW, 1, Mq);
            break;
        }
    }
}

}  // namespace dashgpu
