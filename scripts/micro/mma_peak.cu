// Microbenchmark: tcgen05.mma kind::i8 issue rate, cta_group::1 (M = 128)
// vs cta_group::2 (M = 256, CTA pairs), N = 256, K = 32 per instruction,
// operands resident in shared memory (contents irrelevant).  One CTA per SM,
// persistent; reports int8 ops/s over the whole GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak mma_peak.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int CG>
__global__ void __launch_bounds__(128, 1) mma_peak(int iters, unsigned long long* cyc, int commit_every) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar, sbar;
    const uint32_t warp = threadIdx.x >> 5;
    uint32_t rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint32_t a = smem_u32(base), b = a + 16384;
    const uint32_t idesc = (2u << 4) | ((256u >> 3) << 17) | ((uint32_t)((CG * 128) >> 4) << 24);
    if (threadIdx.x == 0 && rank == 0) {
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int kk = 0; kk < 4; ++kk) {
                if (CG == 2)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(desc(a + kk * 32)), "l"(desc(b + kk * 32)), "r"(idesc), "r"(it | kk));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                                 "l"(desc(a + kk * 32)), "l"(desc(b + kk * 32)), "r"(idesc), "r"(it | kk));
            }
            if (commit_every && (it % commit_every) == 0 && CG == 1)  // per-stage commit, never waited on
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&sbar)) : "memory");
        }
        if (CG == 2)
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        cyc[blockIdx.x] = clock64() - t0;
    }
    if (CG == 2 && threadIdx.x == 0 && rank == 1) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
    }
}

template <int CG>
void run(int iters, int commit_every) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cyc;
    cudaMalloc(&cyc, sms * sizeof(unsigned long long));
    cudaMemset(cyc, 0, sms * sizeof(unsigned long long));
    const size_t smem = 65536 + 1024;
    cudaFuncSetAttribute(mma_peak<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / CG * CG);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, mma_peak<CG>, iters / 10, cyc, commit_every);  // warm-up
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, mma_peak<CG>, iters, cyc, commit_every);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = (double)(sms / CG) * iters * 4 * (CG * 128.0) * 256 * 32;
    printf("cta_group::%d M=%d N=256, commit every %d x 4 MMAs: %.3f ms, %.3g int8 ops/s (%s)\n", CG, CG * 128,
           commit_every, ms, 2 * macs / (ms * 1e-3), cudaGetErrorString(err));
    cudaFree(cyc);
}

int main() {
    run<1>(20000, 0);
    run<1>(20000, 1);
    run<1>(20000, 2);
    run<2>(20000, 0);
    return 0;
}
