// SHA-256 (FIPS 180-4) for the streamed-garbling digest mode: the compression
// function is DASH_HD so the leaf and root kernels (dash_layers.cuh
// digest_leaf_thread / digest_root_thread) and the CPU emulation share it.
//
// Layer digest: the layer's ciphertext bytes in the
// reference's GarbledCircuit::cts order (garble.cpp:134-240, 16 little-endian
// bytes per row) are cut into 64 KiB leaves; digest = SHA-256(SHA-256(leaf 0)
// || SHA-256(leaf 1) || ...).  A layer without ciphertexts has SHA-256("").
#pragma once
#include <cstddef>
#include <cstdint>

#include "dash_common.hpp"

namespace dashgpu {

constexpr uint32_t kDigestLeafRows = 4096;  // 64 KiB leaves

DASH_HD uint32_t sha_rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

DASH_HD uint32_t sha_bswap(uint32_t x) {
    return (x >> 24) | ((x >> 8) & 0xff00u) | ((x << 8) & 0xff0000u) | (x << 24);
}

DASH_HD void sha256_init(uint32_t s[8]) {
    s[0] = 0x6a09e667u; s[1] = 0xbb67ae85u; s[2] = 0x3c6ef372u; s[3] = 0xa54ff53au;
    s[4] = 0x510e527fu; s[5] = 0x9b05688cu; s[6] = 0x1f83d9abu; s[7] = 0x5be0cd19u;
}

// one 64-byte block, w = the block's 16 big-endian words (clobbered)
DASH_HD void sha256_block(uint32_t s[8], uint32_t w[16]) {
    constexpr uint32_t K[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
        0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
        0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
        0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
        0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
    uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
    for (int i = 0; i < 64; ++i) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            const uint32_t w15 = w[(i + 1) & 15], w2 = w[(i + 14) & 15];
            wi = w[i & 15] + (sha_rotr(w15, 7) ^ sha_rotr(w15, 18) ^ (w15 >> 3)) + w[(i + 9) & 15] +
                 (sha_rotr(w2, 17) ^ sha_rotr(w2, 19) ^ (w2 >> 10));
            w[i & 15] = wi;
        }
        const uint32_t t1 = h + (sha_rotr(e, 6) ^ sha_rotr(e, 11) ^ sha_rotr(e, 25)) + ((e & f) ^ (~e & g)) + K[i] + wi;
        const uint32_t t2 = (sha_rotr(a, 2) ^ sha_rotr(a, 13) ^ sha_rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// SHA-256 of `rows` 16-byte rows; row(i, out4) yields row i as 4
// little-endian u32 words (the bytes of the U4 in memory)
template <class Row>
DASH_HD void sha256_rows(uint64_t rows, Row row, uint32_t out[8]) {
    uint32_t s[8], w[16], r[4];
    sha256_init(s);
    uint64_t i = 0;
    for (; i + 4 <= rows; i += 4) {
        for (int q = 0; q < 4; ++q) {
            row(i + q, r);
            for (int t = 0; t < 4; ++t) w[4 * q + t] = sha_bswap(r[t]);
        }
        sha256_block(s, w);
    }
    // tail: 0-3 rows (<= 48 bytes), the 0x80 byte and the bit length fit one block
    const int left = (int)(rows - i);
    for (int q = 0; q < 16; ++q) w[q] = 0;
    for (int q = 0; q < left; ++q) {
        row(i + q, r);
        for (int t = 0; t < 4; ++t) w[4 * q + t] = sha_bswap(r[t]);
    }
    w[4 * left] = 0x80000000u;
    const uint64_t bits = rows * 128;
    w[14] = (uint32_t)(bits >> 32);
    w[15] = (uint32_t)bits;
    sha256_block(s, w);
    for (int t = 0; t < 8; ++t) out[t] = s[t];
}

}  // namespace dashgpu
