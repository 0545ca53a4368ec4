// umma_bench.cu -- microbenchmark: cost of one tcgen05.mma.kind::f16 issued back to back from a
// single thread on static shared-memory operands, for the shapes/layouts the tcgen05 engine
// could use.  Profiling tool only (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/umma_bench tools/umma_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46) | (uint64_t(layout & 7) << 61);
}

__global__ void bench(int iters, uint32_t idesc, uint32_t layout, uint32_t lbo, uint32_t sbo, int nacc,
                      unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    uint16_t* ones = reinterpret_cast<uint16_t*>(sm);
    for (int i = threadIdx.x; i < 48 * 1024 / 2; i += blockDim.x) ones[i] = 0x3C00;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint64_t a = desc(smem_u32(sm), lbo, sbo, layout);
        const uint64_t b = desc(smem_u32(sm + 32768), 128, 256, 0);
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tm + uint32_t(i % nacc) * 32u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(a), "l"(b), "r"(idesc), "r"(0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
        unsigned long long t1 = clock64();
        out[0] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    struct Case {
        const char* name;
        uint32_t M, N, amaj, layout, lbo, sbo;
    } cases[] = {
        {"M128 N16 A MN-major SW32 (engine)", 128, 16, 1, 6, 512, 256},
        {"M128 N16 A MN-major SW32 lbo=32 (dense)", 128, 16, 1, 6, 32, 256},
        {"M128 N16 A K-major none", 128, 16, 0, 0, 128, 256},
        {"M128 N64 A MN-major SW32", 128, 64, 1, 6, 512, 256},
        {"M128 N256 A K-major none", 128, 256, 0, 0, 128, 256},
        {"M128 N32 A MN-major SW32", 128, 32, 1, 6, 512, 256},
        {"M64 N16 A MN-major SW32", 64, 16, 1, 6, 512, 256},
        {"M128 N16 A K-major SW32", 128, 16, 0, 6, 256, 512},
    };
    for (auto& c : cases) {
        const uint32_t idesc = (1u << 4) | (c.amaj << 15) | ((c.N >> 3) << 17) | ((c.M >> 4) << 24);
        for (int nacc : {1, (c.N <= 32 ? 8 : 1)}) {
            const int iters = 4096;
            bench<<<1, 128, 64 * 1024>>>(iters, idesc, c.layout, c.lbo, c.sbo, nacc, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long cyc = 0;
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            printf("%-45s accs=%d: %s %.1f cycles/MMA  (%.1f B/cycle of A)\n", c.name, nacc,
                   e == cudaSuccess ? "ok" : cudaGetErrorString(e), double(cyc) / iters,
                   double(c.M) * 16 * 2 / (double(cyc) / iters));
            if (e != cudaSuccess) return 1;
        }
    }
    // concurrency: grid of 1, 148 and 296 CTAs (<= 2 per SM fit), same per-CTA work; if 296
    // CTAs take ~the time of 148, two issuers on one SM overlap (issue-latency bound)
    for (int grid : {1, 148, 296}) {
        const uint32_t idesc = (1u << 4) | (1u << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        bench<<<grid, 128, 64 * 1024>>>(4096, idesc, 6, 512, 256, 8, d);
        cudaEventRecord(a);
        bench<<<grid, 128, 64 * 1024>>>(4096, idesc, 6, 512, 256, 8, d);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("grid %d: %.3f ms for 4096 MMAs per CTA (M128 N16 MN-major SW32)\n", grid, ms);
    }
    return 0;
}
