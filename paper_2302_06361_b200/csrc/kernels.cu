// CUDA side of the B200 Dash engine (sm_100a), non-activation kernels:
// public/private linear lanes, garbling setup (offsets, PRF labels), input
// encoding, decoding tables / decode, label export and primitive parity
// kernels.  Owns device memory, streams and per-kernel event timing.
#include "dash_common.hpp"

namespace dashgpu {
__constant__ ModC c_mod[MAXMOD + 1];
__constant__ uint32_t c_pi_rk[44];
__constant__ uint16_t c_modslot[MAXMOD + 1];
__device__ uint32_t g_T0[256];
}  // namespace dashgpu
#define DASH_CONST_DEFINED 1
#include <cudaTypedefs.h>

#include <algorithm>

#include "dash_prim.cuh"
#include "kernels_common.cuh"
#include "tc_linear.cuh"
#include "tc_linear_exp.cuh"
#include "wpe.cuh"

namespace dashgpu {

void upload_act(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0);

ProfData& prof() {
    static ProfData p;
    return p;
}

namespace {

// all = false: only the events that already completed (a stream sync must
// not wait on another stream's work: pipelined inference runs two streams)
void prof_drain(bool all = true) {
    std::vector<ProfData::Pending> keep;
    for (auto& p : prof().pending) {
        if (!all && cudaEventQuery(p.b) != cudaSuccess) {
            keep.push_back(p);
            continue;
        }
        cudaEventSynchronize(p.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        prof().ms[p.kind] += ms;
        prof().n[p.kind] += 1;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    prof().pending.swap(keep);
}

// Private-weight linear lane (layer.cpp:195-212, 456-507), warp-cooperative:
// one warp = one (inference, output unit); lane t takes window weights
// j = t, t+32, ...: its projection gate x_j -> w_j x_j (p rows, fresh output
// label) is garbled / evaluated independently, then the 32 term labels are
// summed with a shuffle butterfly (free add, digit-wise mod p) and the
// garbler subtracts b R_p (add_public_constant).  Every branch is
// warp-uniform (one lane modulus per launch); labels live in lane-interleaved
// shared memory next to the AES tables; persistent CTAs pull units from a
// counter.  Ciphertext rows keep the reference's order (unit-major, weight,
// row), so the blob is byte-identical to garble_layer's.
constexpr int kPrivWarps = 24;
constexpr int kPrivLaneWords = 2 * NWMAX;  // X, T per lane (lane-interleaved) + one warp-shared sum
constexpr int kPrivWarpWords = kPrivLaneWords * 32 + NWMAX;

DASH_HD void warp_sum_label(LB A, LB T, bool active, const ModC& M) {
#if defined(__CUDA_ARCH__)
    if (M.pow2) {
        U4 v = lb_u4(T);
        if (!active) v.x[0] = v.x[1] = v.x[2] = v.x[3] = 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) o[i] = __shfl_xor_sync(0xffffffffu, v.x[i], off);
            p2_add(v.x, o, M);
        }
        U4 a = lb_u4(A);
        p2_add(a.x, v.x, M);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) lb_set_u4(A, a);
        __syncwarp();
        return;
    }
    for (int w = 0; w < M.nw; ++w) {
        uint32_t v = active ? T[w] : 0u;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v = swar_add(v, __shfl_xor_sync(0xffffffffu, v, off), M);
        const uint32_t s = swar_add(A[w], v, M);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) A[w] = s;
        __syncwarp();
    }
#endif
}

template <bool G>
__global__ void __launch_bounds__(kPrivWarps * 32, 1) private_kernel(const __grid_constant__ PrivParams P,
                                                                      uint32_t* counter) {
    fill_T(g_T0);
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* wb = s_dyn + kTabWords + warp * kPrivWarpWords;
    // the running sum is identical in every lane (butterfly): one warp copy
    const LB X{wb + lane, 32}, T{wb + NWMAX * 32 + lane, 32}, A{wb + kPrivLaneWords * 32, 1};
    const AesTab t = make_tab(nullptr, lane);
    const ModC& M = c_mod[P.p];
    const uint32_t p = P.p, total = P.B * P.M;
    uint32_t item = warp * gridDim.x + blockIdx.x;
    const uint32_t first = kPrivWarps * gridDim.x;
    while (item < total) {
        const uint32_t b = item / P.M, u = item - b * P.M;
        const uint32_t* rk = P.rk + (uint64_t)b * 44;
        const uint32_t* mult = P.mult + (uint64_t)b * P.mult_stride;
        uint32_t oc = 0, oy = 0, ox = 0;
        if (P.conv) {
            oc = u / (P.OH * P.OW);
            oy = (u / P.OW) % P.OH;
            ox = u % P.OW;
        }
        const uint8_t* wr = P.wres + (uint64_t)(P.conv ? oc : u) * P.win;
        if (lane == 0)
            for (int w = 0; w < lb_words(M); ++w) A[w] = 0;
        __syncwarp();
        for (uint32_t j0 = 0; j0 < P.win; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool active = j < P.win;
            if (active) {
                uint64_t xi;
                if (!P.conv) {
                    xi = j;
                } else {
                    const uint32_t ic = j / (P.f * P.f), ky = (j / P.f) % P.f, kx = j % P.f;
                    xi = ((uint64_t)ic * P.H + (oy * P.stride + ky)) * P.W + (ox * P.stride + kx);
                }
                lb_load_rows(X, P.in + ((uint64_t)b * M.nw) * P.E_in + xi, P.E_in, M);
                const uint64_t g = P.gate_base + (uint64_t)u * P.win + j;
                U4* R = P.blob + (uint64_t)b * P.blob_stride + ((uint64_t)u * P.win + j) * p;
                const uint32_t c = lb_color(X, M);
                if (G) {
                    // fresh output label, then the projection x -> w x mod p: row
                    // (c + a) mod p carries payload (w a mod p) R_p -- the act
                    // kernels' single-copy row loop (garble_rows_n, phi = nullptr)
                    prf_n(T, P.wire_base + (uint64_t)u * P.win + j, 0, p, rk, t);
                    garble_rows_n(X, T, t, mult, p, p, c, g, nullptr, wr[j], R, 0, 1);
                } else {
                    lb_dec(T, R[c], hash_tw(lb_compress(X, M), g, c, 0, t), M);
                }
            }
            __syncwarp();
            warp_sum_label(A, T, active, M);
        }
        if (lane == 0) {  // A is one warp-shared copy: lane 0 finishes the unit
            if (G) {
                const uint32_t bb = P.bres[P.conv ? oc : u];
                if (bb) lb_sub_g(A, mult + ((uint64_t)c_modslot[p] * 128u + bb) * NWMAX, M);
            }
            lb_store_rows(A, P.out + ((uint64_t)b * M.nw) * P.M + u, P.M, M);
        }
        __syncwarp();
        uint32_t next = 0;
        if (lane == 0) next = first + atomicAdd(counter, 1u);
        item = __shfl_sync(0xffffffffu, next, 0);
    }
}

__global__ void __launch_bounds__(128) pad_add_kernel(const __grid_constant__ PadAddParams P) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= P.E_out) return;
    pad_add_thread(P, blockIdx.z, blockIdx.y, u);
}

__global__ void __launch_bounds__(128) proj_kernel(const __grid_constant__ ProjParams P) {
    fill_T(g_T0);
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    // per-thread label buffers in shared memory, lane-interleaved (stride 32)
    uint32_t* lb = s_dyn + kTabWords + (threadIdx.x >> 5) * (2 * NWMAX * 32) + (threadIdx.x & 31u);
    proj_thread(P, i, make_tab(nullptr, threadIdx.x & 31u), LB{lb, 32}, LB{lb + NWMAX * 32, 32});
}

__global__ void __launch_bounds__(128) expand_kernel(const uint8_t* seeds, uint32_t* rk, uint32_t B) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) expand_thread(seeds + (uint64_t)b * 16, rk + (uint64_t)b * 44, g_T0);
}

__global__ void __launch_bounds__(128) setup_offsets_kernel(SetupParams Sp) {
    fill_T(g_T0);
    const uint32_t si = blockIdx.x;  // modulus slot; thread = multiple x < 128
    setup_offsets_thread(Sp, blockIdx.y, si, threadIdx.x, make_tab(nullptr, threadIdx.x & 31u));
}

__global__ void __launch_bounds__(128) setup_labels_kernel(SetupParams Sp) {
    fill_T(g_T0);
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e > Sp.n_in) return;
    setup_labels_thread(Sp, blockIdx.z, e, (int)blockIdx.y, make_tab(nullptr, threadIdx.x & 31u));
}

// Small launches: one warp per label (PRF counter blocks over the lanes,
// prf_coop); same values as setup_labels_thread.
constexpr int kLabWarps = 8;
__global__ void __launch_bounds__(kLabWarps * 32) setup_labels_warp_kernel(SetupParams Sp) {
    fill_T(g_T0);
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const uint32_t idx = blockIdx.x * kLabWarps + wl, b = blockIdx.y;
    const uint32_t i = idx % (uint32_t)Sp.k, e = idx / (uint32_t)Sp.k;
    if (e > Sp.n_in) return;  // whole warp
    const LB L{s_dyn + kTabWords + wl * NWMAX, 1};
    const AesTab t = make_tab(nullptr, lane);
    const uint32_t p = Sp.primes[i];
    const ModC& M = c_mod[p];
    const uint32_t* rk = Sp.rk + (uint64_t)b * 44;
    // e < n_in: input base of element e, lane i (wire k + e*k + i); e == n_in: zero wire i
    const uint64_t wire = e < Sp.n_in ? (uint64_t)Sp.k + (Sp.e0 + e) * Sp.k + (uint64_t)i : (uint64_t)i;
    prf_coop(L, wire, 0, p, rk, t, lane, 32);
    if (lane != 0) return;
    if (e < Sp.n_in) lb_store_rows(L, Sp.base_planes[i] + ((uint64_t)b * M.nw) * Sp.n_in + e, Sp.n_in, M);
    else lb_store_rows(L, Sp.zero + ((uint64_t)b * Sp.k + i) * LABW, 1, M);
    if (e == Sp.n_in && i == 0) {  // seed commitment = davies_meyer(seed bytes read little-endian)
        const uint8_t* sd = Sp.seeds + (uint64_t)b * 16;
        U4 v;
        for (int j = 0; j < 4; ++j)
            v.x[j] = (uint32_t)sd[4 * j] | ((uint32_t)sd[4 * j + 1] << 8) | ((uint32_t)sd[4 * j + 2] << 16) |
                     ((uint32_t)sd[4 * j + 3] << 24);
        U4 h = aes_pi(v, t);
        for (int j = 0; j < 4; ++j) h.x[j] ^= v.x[j];
        Sp.commit[b] = h;
    }
}

__global__ void __launch_bounds__(128) encode_kernel(EncodeParams P) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.n_in) return;
    encode_thread(P, blockIdx.z, e, (int)blockIdx.y);
}

__global__ void __launch_bounds__(128) dectable_kernel(DecodeParams P) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.n_out) return;
    dectable_thread(P, blockIdx.z, e, (int)blockIdx.y);
}

__global__ void __launch_bounds__(128) decode_kernel(DecodeParams P) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.n_out) return;
    decode_thread(P, blockIdx.y, e);
}

__global__ void __launch_bounds__(128) compress_kernel(CompressParams P) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.n) return;
    compress_thread(P, blockIdx.y, e);
}

__global__ void __launch_bounds__(128) decompress_kernel(CompressParams P, uint32_t* lane_out) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= P.n) return;
    decompress_thread(P, blockIdx.y, e, lane_out);
}

__global__ void __launch_bounds__(256) rows_permute_kernel(RowsPermuteParams P) {
    const uint64_t n = P.E * P.uc;
    for (uint64_t r = (uint64_t)blockIdx.x * 256 + threadIdx.x; r < n; r += (uint64_t)gridDim.x * 256)
        rows_permute_thread(P, r);
}

__global__ void __launch_bounds__(128) digest_kernel(DigestParams P) {
    const uint32_t leaf = blockIdx.x * blockDim.x + threadIdx.x;
    if (leaf < P.leaves) digest_leaf_thread(P, blockIdx.y, leaf);
}

__global__ void __launch_bounds__(128) prim_kernel(PrimParams P) {
    fill_T(g_T0);
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.n) return;
    prim_thread(P, i, make_tab(nullptr, threadIdx.x & 31u));
}

}  // namespace

namespace dev {

void set_device(int d) { ck(cudaSetDevice(d), "cudaSetDevice"); }
int get_device() {
    int d = -1;
    return cudaGetDevice(&d) == cudaSuccess ? d : -1;
}
int backend() { return 1; }
void* alloc(size_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, n ? n : 16), "cudaMalloc");
    return p;
}
void release(void* p) {
    if (p) cudaFree(p);
}
void* host_alloc(size_t n) {
    void* p = nullptr;
    ck(cudaMallocHost(&p, n ? n : 16), "cudaMallocHost");
    return p;
}
void host_release(void* p) {
    if (p) cudaFreeHost(p);
}
void h2d(void* d, const void* s, size_t n, void* st) {
    if (n) ck(cudaMemcpyAsync(d, s, n, cudaMemcpyHostToDevice, S(st)), "h2d");
}
void d2h(void* d, const void* s, size_t n, void* st) {
    if (n) ck(cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToHost, S(st)), "d2h");
}
void d2d(void* d, const void* s, size_t n, void* st) {
    if (n) ck(cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice, S(st)), "d2d");
}
void memset0(void* p, size_t n, void* st) {
    if (n) ck(cudaMemsetAsync(p, 0, n, S(st)), "memset");
}
void sync(void* st) {
    ck(cudaStreamSynchronize(S(st)), "sync");
    if (prof().on) prof_drain(false);
}
void check() { ck(cudaGetLastError(), "launch"); }
size_t free_bytes() {
    size_t f = 0, t = 0;
    ck(cudaMemGetInfo(&f, &t), "cudaMemGetInfo");
    return f;
}
void upload_constants(const ModC* mods, const uint32_t* pi_rk, const uint16_t* modslot, const uint32_t* T0) {
    ck(cudaMemcpyToSymbol(c_mod, mods, sizeof(ModC) * (MAXMOD + 1)), "c_mod");
    ck(cudaMemcpyToSymbol(c_pi_rk, pi_rk, sizeof(uint32_t) * 44), "c_pi_rk");
    ck(cudaMemcpyToSymbol(c_modslot, modslot, sizeof(uint16_t) * (MAXMOD + 1)), "c_modslot");
    ck(cudaMemcpyToSymbol(g_T0, T0, sizeof(uint32_t) * 256), "g_T0");
    upload_act(mods, pi_rk, modslot, T0);
}
void* stream_create() {
    cudaStream_t s;
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
    return s;
}
void stream_destroy(void* s) {
    if (s) cudaStreamDestroy(S(s));
}
void* event_create() {
    cudaEvent_t e;
    ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    return e;
}
void event_destroy(void* e) {
    if (e) cudaEventDestroy(static_cast<cudaEvent_t>(e));
}
void event_sync(void* e) { ck(cudaEventSynchronize(static_cast<cudaEvent_t>(e)), "event sync"); }
void event_record(void* e, void* st) { ck(cudaEventRecord(static_cast<cudaEvent_t>(e), S(st)), "event record"); }
void stream_wait(void* st, void* e) {
    ck(cudaStreamWaitEvent(S(st), static_cast<cudaEvent_t>(e), 0), "stream wait");
}
void prof_enable(int on) { prof().on = on; }
void prof_reset() {
    prof_drain();
    for (int i = 0; i < K_NKINDS; ++i) {
        prof().ms[i] = 0;
        prof().n[i] = 0;
    }
}
int prof_read(double* ms, uint64_t* n, int maxk) {
    prof_drain();
    const int k = maxk < K_NKINDS ? maxk : K_NKINDS;
    for (int i = 0; i < k; ++i) {
        ms[i] = prof().ms[i];
        n[i] = prof().n[i];
    }
    return k;
}

}  // namespace dev

// 2-D u8 tensor map, K-major rows, 128-byte swizzle (tc_linear.cuh operands)
static void encode_u8_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t rows, uint64_t stride,
                         uint32_t box_inner, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        ck(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q),
           "cuTensorMapEncodeTiled entry point");
        if (q != cudaDriverEntryPointSuccess || !encode) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    }
    const cuuint64_t dims[2] = {inner, rows};
    const cuuint64_t strides[1] = {stride};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

void make_weight_map(TcLinear& T) {
    CUtensorMap m;
    encode_u8_2d(&m, T.wexp, T.Kpad, (uint64_t)T.k * T.Npad, T.Kpad, (uint32_t)tc::BKB, T.BN);  // both kernels: 128-byte K boxes
    static_assert(sizeof(CUtensorMap) == sizeof(T.tmap), "tensor map size");
    memcpy(T.tmap, &m, sizeof m);
}

// expanded-digit kernel (tc_linear_exp.cuh): convolutions, unaligned dense layers
static void launch_linear_exp(const LinParams* Ls, int n, const TcLinear& T, void* st) {
    tcx::TcParams P;
    memset(&P, 0, sizeof P);
    const LinParams& L0 = Ls[0];
    P.nl = n;
    P.kblocks = T.kblocks;
    P.BN = T.BN;
    P.tiles_n = T.Npad / T.BN;
    P.nout = T.nout;
    if (L0.conv) {
        P.P = L0.OH * L0.OW;
        P.OW = L0.OW;
        P.s = L0.stride;
        P.W = L0.W;
    } else {
        P.P = 1;
        P.OW = 1;
    }
    P.E_in = L0.E_in;
    P.M = L0.M;
    P.stages = tcx::stages_for(T.BN);
    P.nowrap = 1;  // the accumulator, z zero and (p - b) R sum below 2^31: no wrap handling
    for (int i = 0; i < n; ++i)
        if ((uint64_t)(L0.K + 3) * Ls[i].p * Ls[i].p >= (1ull << 31)) P.nowrap = 0;
    P.zstride = L0.zstride;
    P.garbler = L0.garbler;
    P.koff = T.koff;
    uint32_t tiles = 0;
    for (int i = 0; i < n; ++i) {
        const LinParams& L = Ls[i];
        tcx::TcLane& l = P.L[i];
        l.in = L.in;
        l.out = L.out;
        l.zt = L.zt;
        l.bres = L.bres;
        l.zero = L.zero;
        l.R = L.R;
        l.p = L.p;
        l.n = L.n;
        l.nw = L.nw;
        l.mag = L.mag;
        l.sh = L.sh;
        l.rows = L.B * L.nw * P.P;
        l.tile_base = tiles;
        l.wrow = (uint32_t)i * T.Npad;
        tiles += cdiv(l.rows, tcx::BM) * P.tiles_n;
    }
    // dense layer over 16-byte-aligned planes: the A tiles are plain 2-D boxes
    // of the [B*nw][4*E_in] digit-byte matrix, loaded by TMA instead of gathered
    tcx::TcAMaps amaps;
    memset(&amaps, 0, sizeof amaps);
    P.a_tma = !L0.conv && (L0.E_in % 4) == 0;
    if (P.a_tma)
        for (int i = 0; i < n; ++i)
            encode_u8_2d(&amaps.m[i], Ls[i].in, (uint64_t)4 * L0.E_in, (uint64_t)Ls[i].B * Ls[i].nw,
                         (uint64_t)4 * L0.E_in, (uint32_t)tcx::BKB, (uint32_t)tcx::BM);
    const size_t smem = tcx::smem_bytes(T.BN);
    smem_attr((const void*)tcx::tc_linear_kernel, smem);
    CUtensorMap map;
    memcpy(&map, T.tmap, sizeof map);
    tcx::tc_linear_kernel<<<tiles, tcx::kThreads, smem, S(st)>>>(map, P, amaps);
    dev::check();
}

void launch_linear(const LinParams* Ls, int n, const TcLinear& T, void* st) {
    if (n <= 0 || Ls[0].B == 0 || Ls[0].M == 0) return;
    ProfScope ps(K_LINEAR, S(st));
    if (T.mode == TcLinear::EXPANDED) {
        launch_linear_exp(Ls, n, T, st);
        return;
    }
    tc::TcParams P;
    memset(&P, 0, sizeof P);
    const LinParams& L0 = Ls[0];
    P.nl = n;
    P.kblocks = T.kblocks;
    P.K = L0.K;
    P.BN = T.BN;
    P.tiles_n = T.Npad / T.BN;
    P.nout = T.nout;
    if (L0.conv) {
        P.P = L0.OH * L0.OW;
        P.OW = L0.OW;
        P.s = L0.stride;
        P.W = L0.W;
    } else {
        P.P = 1;
        P.OW = 1;
    }
    P.E_in = L0.E_in;
    P.M = L0.M;
    uint32_t koff_bytes = (!L0.conv && (L0.E_in % 4) == 0) ? 0u : T.kblocks * tc::BKB * 4;
    if (koff_bytes > 32 * 1024) koff_bytes = 0;  // huge windows read the table from global memory
    P.koff_smem = koff_bytes != 0;

    P.zstride = L0.zstride;
    P.garbler = L0.garbler;
    P.koff = T.koff;
    P.dense_vec = !L0.conv && (L0.E_in % 4) == 0;
    P.fold = T.fold;
    P.nowrap = 2;
    for (int i = 0; i < n; ++i) {
        const uint64_t p = Ls[i].p, bound = (uint64_t)(L0.K + 3) * p * p;  // acc + z zero + nb R
        if (bound >= (1ull << 31)) P.nowrap = 0;
        else if (bound * p >= (1ull << 32) && P.nowrap == 2) P.nowrap = 1;
    }
    // small windows: SUB row tiles share one 128-byte K stage (TMEM: SUB * BN <= 256 columns per buffer)
    P.sub = 1;
    if (T.kblocks == 1) {
        const uint32_t keff = L0.K + (T.fold ? 2u : 0u), k32 = (keff + 31) / 32 * 32;
        uint32_t sub = k32 <= 32 ? 4u : k32 <= 64 ? 2u : 1u;
        while (sub > 1 && sub * T.BN > 256) sub >>= 1;
        P.sub = sub;
    }
    P.ksub = tc::BKB / P.sub;
    // dense window words by TMA: one row tile per stage, no fold columns
    // (the zero-wire / R_p words come from other arrays)
    P.a_tma = P.dense_vec && P.sub == 1 && !T.fold && std::getenv("DASH_TC_NOTMA") == nullptr;
    // CTA pairs (tcgen05.mma.cta_group::2, M = 256) on the TMA window path,
    // opt-in (DASH_TC_CG=2): bit-exact, but measured at half the single-CTA
    // throughput on the Dense 1024^2 sweep
    uint64_t mt_total = 0;
    for (int i = 0; i < n; ++i) mt_total += cdiv((uint64_t)Ls[i].B * Ls[i].nw * P.P, tc::GM);
    const char* cge = std::getenv("DASH_TC_CG");
    const uint32_t CG = (P.a_tma && T.BN >= 32 && mt_total >= 2 * (uint64_t)n && cge && std::atoi(cge) == 2) ? 2u : 1u;
    P.stages = tc::stages_for(T.BN, koff_bytes, P.a_tma, CG);
    uint32_t tiles = 0;
    for (int i = 0; i < n; ++i) {
        const LinParams& L = Ls[i];
        tc::TcLane& l = P.L[i];
        l.in = L.in;
        l.out = L.out;
        l.zt = L.zt;
        l.bres = L.bres;
        l.zero = L.zero;
        l.R = L.R;
        l.p = L.p;
        l.n = L.n;
        l.nw = L.nw;
        l.mag = L.mag;
        l.sh = L.sh;
        l.mag0 = (uint32_t)((0xffffffffull + L.p) / L.p);  // ceil(2^32 / p)
        if (L.nw < 2) throw std::runtime_error("tc_linear: lanes of fewer than 5 digits");
        l.nw_mag = (uint32_t)(0xffffffffull / L.nw + 1);
        if ((uint64_t)L.B * L.nw * P.P >= (1ull << 22))
            throw std::runtime_error("tc_linear: too many row groups per lane for the reciprocal decode");
        l.groups = L.B * L.nw * P.P;
        l.tile_base = tiles;
        l.wrow = (uint32_t)i * T.Npad;
        tiles += cdiv(cdiv(l.groups, tc::GM * P.sub), CG) * P.tiles_n;  // (pairs of) row tiles x column tiles
    }
    P.tiles = tiles;
    P.tn_mag = P.tiles_n > 1 ? (uint32_t)(0xffffffffull / P.tiles_n + 1) : 0u;
    // umulhi(x, floor(2^32 / d) + 1) == x / d whenever x * d < 2^32
    if (tiles >= (1u << 22) || P.tiles_n >= 1024) throw std::runtime_error("tc_linear: tile grid too large for the reciprocal decode");
    P.raw_stages = tc::raw_stages(P.a_tma);
    const size_t smem = tc::smem_bytes(T.BN, P.stages, koff_bytes, P.a_tma, CG);
    CUtensorMap map;
    if (CG == 2)  // each CTA of a pair loads half of the BN weight rows
        encode_u8_2d(&map, T.wexp, T.Kpad, (uint64_t)T.k * T.Npad, T.Kpad, (uint32_t)tc::BKB, T.BN / 2);
    else
        memcpy(&map, T.tmap, sizeof map);
    tc::TcRawMaps rmaps;
    memset(&rmaps, 0, sizeof rmaps);
    if (P.a_tma)
        for (int i = 0; i < n; ++i)  // [B * nw][4 E_in] bytes, boxes of 32 rows x 128 bytes
            encode_u8_2d(&rmaps.m[i], Ls[i].in, (uint64_t)4 * L0.E_in, (uint64_t)Ls[i].B * Ls[i].nw,
                         (uint64_t)4 * L0.E_in, 128u, (uint32_t)tc::GM);
    int sms = 0, dev = 0;
    ck(cudaGetDevice(&dev), "dev");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    if (CG == 2) {
        // persistent CTA pairs: clusters of two, one CTA per SM
        smem_attr((const void*)tc::tc_linear_kernel<2>, smem);
        cudaLaunchConfig_t cfg;
        memset(&cfg, 0, sizeof cfg);
        // persistent: as many pairs as can be resident at once (a GPC with an
        // odd SM count leaves one SM without a partner)
        static int max_pairs = 0;
        if (max_pairs == 0) {
            cudaLaunchConfig_t q;
            memset(&q, 0, sizeof q);
            q.gridDim = dim3(sms);
            q.blockDim = dim3(tc::kThreads);
            q.dynamicSmemBytes = smem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 2;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, (const void*)tc::tc_linear_kernel<2>, &q) != cudaSuccess || nc <= 0)
                nc = sms / 2;
            max_pairs = nc;
            if (std::getenv("DASH_TC_VERBOSE")) fprintf(stderr, "tc_linear: %d resident CTA pairs\n", nc);
        }
        const uint32_t pairs = std::min<uint32_t>(tiles, (uint32_t)max_pairs);
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(tc::kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = S(st);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ck(cudaLaunchKernelEx(&cfg, tc::tc_linear_kernel<2>, map, P, rmaps), "tc_linear pair launch");
    } else {
        smem_attr((const void*)tc::tc_linear_kernel<1>, smem);
        const uint32_t grid = std::min<uint32_t>(tiles, (uint32_t)sms);  // persistent: one CTA per SM
        tc::tc_linear_kernel<1><<<grid, tc::kThreads, smem, S(st)>>>(map, P, rmaps);
    }
    dev::check();
}

void launch_private(const PrivParams& P, void* st, const Sched& q) {
    if (P.B == 0 || P.M == 0) return;
    ProfScope ps(P.garbler ? K_PRIV_GARBLE : K_PRIV_EVAL, S(st));
    uint32_t* counter = q.counter + 1;
    ck(cudaMemsetAsync(counter, 0, sizeof(uint32_t), S(st)), "counter reset");
    int sms = 0, dev = 0;
    ck(cudaGetDevice(&dev), "dev");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sms");
    const size_t smem = kTabBytes + sizeof(uint32_t) * (size_t)kPrivWarps * kPrivWarpWords;
    const uint32_t grid = (uint32_t)std::min<uint64_t>((uint64_t)sms, cdiv((uint64_t)P.B * P.M, 1));
    if (P.garbler) {
        smem_attr((const void*)private_kernel<true>, smem);
        private_kernel<true><<<grid, kPrivWarps * 32, smem, S(st)>>>(P, counter);
    } else {
        smem_attr((const void*)private_kernel<false>, smem);
        private_kernel<false><<<grid, kPrivWarps * 32, smem, S(st)>>>(P, counter);
    }
    dev::check();
}

void launch_pad_add(const PadAddParams& P, void* st) {
    if (P.B == 0 || P.E_out == 0) return;
    ProfScope ps(K_MISC, S(st));
    pad_add_kernel<<<dim3(cdiv(P.E_out, 128), P.wbase[P.k], P.B), 128, 0, S(st)>>>(P);
    dev::check();
}

void launch_proj(const ProjParams& P, void* st) {
    if (P.n == 0) return;
    ProfScope ps(K_MISC, S(st));
    const size_t smem = kTabBytes + sizeof(uint32_t) * 4 * 2 * NWMAX * 32;  // 4 warps x (X, A)
    smem_attr((const void*)proj_kernel, smem);
    proj_kernel<<<cdiv(P.n, 128), 128, smem, S(st)>>>(P);
    dev::check();
}

void launch_expand(const uint8_t* seeds, uint32_t* rk, uint32_t B, void* st) {
    if (!B) return;
    ProfScope ps(K_SETUP, S(st));
    expand_kernel<<<cdiv(B, 128), 128, 0, S(st)>>>(seeds, rk, B);
    dev::check();
}

void launch_setup(const SetupParams& Sp, void* st) {
    ProfScope ps(K_SETUP, S(st));
    smem_attr((const void*)setup_offsets_kernel, kTabBytes);
    setup_offsets_kernel<<<dim3(Sp.nslot, Sp.B), 128, kTabBytes, S(st)>>>(Sp);
    dev::check();
    const uint64_t labels = (uint64_t)(Sp.n_in + 1) * Sp.k * Sp.B;
    static int sms = 0;
    if (!sms) {
        int devi = 0;
        ck(cudaGetDevice(&devi), "dev");
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, devi), "sms");
    }
    if (labels <= (uint64_t)sms * 24 * 2) {  // <= two waves of warps: one warp per label
        const size_t smem = kTabBytes + sizeof(uint32_t) * kLabWarps * NWMAX;
        smem_attr((const void*)setup_labels_warp_kernel, smem);
        setup_labels_warp_kernel<<<dim3(cdiv((uint64_t)(Sp.n_in + 1) * Sp.k, kLabWarps), Sp.B), kLabWarps * 32, smem,
                                   S(st)>>>(Sp);
    } else {
        smem_attr((const void*)setup_labels_kernel, kTabBytes);
        setup_labels_kernel<<<dim3(cdiv(Sp.n_in + 1, 128), Sp.k, Sp.B), 128, kTabBytes, S(st)>>>(Sp);
    }
    dev::check();
}

void launch_encode(const EncodeParams& P, void* st) {
    ProfScope ps(K_ENCODE, S(st));
    encode_kernel<<<dim3(cdiv(P.n_in, 128), P.k, P.B), 128, 0, S(st)>>>(P);
    dev::check();
}

void launch_dectable(const DecodeParams& P, void* st) {
    ProfScope ps(K_DECODE, S(st));
    dectable_kernel<<<dim3(cdiv(P.n_out, 128), P.k, P.B), 128, 0, S(st)>>>(P);
    dev::check();
}

void launch_decode(const DecodeParams& P, void* st) {
    ProfScope ps(K_DECODE, S(st));
    decode_kernel<<<dim3(cdiv(P.n_out, 128), P.B), 128, 0, S(st)>>>(P);
    dev::check();
}

void launch_compress(const CompressParams& P, void* st) {
    ProfScope ps(K_MISC, S(st));
    compress_kernel<<<dim3(cdiv(P.n, 128), P.B), 128, 0, S(st)>>>(P);
    dev::check();
}

void launch_decompress(const CompressParams& P, uint32_t* lane_out, void* st) {
    ProfScope ps(K_MISC, S(st));
    decompress_kernel<<<dim3(cdiv(P.n, 128), P.B), 128, 0, S(st)>>>(P, lane_out);
    dev::check();
}

void launch_rows_permute(const RowsPermuteParams& P, void* st) {
    const uint64_t n = P.E * P.uc;
    if (!n) return;
    ProfScope ps(K_MISC, S(st));
    rows_permute_kernel<<<(uint32_t)std::min<uint64_t>(cdiv(n, 256), 148ull * 16), 256, 0, S(st)>>>(P);
    dev::check();
}

__global__ void __launch_bounds__(32) digest_root_kernel(DigestParams P, uint32_t* roots) {
    const uint32_t b = blockIdx.x * 32 + threadIdx.x;
    if (b < P.B) digest_root_thread(P, b, roots);
}

void launch_digest(const DigestParams& P, uint32_t* roots, void* st) {
    if (!P.B) return;
    ProfScope ps(K_MISC, S(st));
    if (P.leaves) digest_kernel<<<dim3(cdiv(P.leaves, 128), P.B), 128, 0, S(st)>>>(P);
    digest_root_kernel<<<cdiv(P.B, 32), 32, 0, S(st)>>>(P, roots);
    dev::check();
}

void launch_prim(const PrimParams& P, void* st) {
    smem_attr((const void*)prim_kernel, kTabBytes);
    prim_kernel<<<cdiv(P.n, 128), 128, kTabBytes, S(st)>>>(P);
    dev::check();
}

}  // namespace dashgpu
