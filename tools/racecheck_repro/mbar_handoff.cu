// Minimal known-correct shared-memory handoff through an mbarrier, for compute-sanitizer
// racecheck (profiling / tool-behaviour evidence, not product code).
//
// Warp 0 writes 32 floats to shared memory, __syncwarp (orders the lanes' writes before lane
// 0), lane 0 mbarrier.arrive (release.cta); warp 1 waits with mbarrier.try_wait (acquire.cta)
// and reads them.  This is the pattern the TMA engine's streaming warps use to hand chunk
// tables to the manager warp.  Mode 1 replaces the mbarrier by a named barrier (bar.arrive /
// bar.sync), which racecheck models.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mbar_handoff mbar_handoff.cu
//   compute-sanitizer --tool racecheck ./mbar_handoff 0 ; ... ./mbar_handoff 1
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__global__ void handoff(int mode, float* out) {
    __shared__ float buf[32];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        buf[lane] = float(lane) * 2.0f;
        __syncwarp();
        if (mode == 0) {
            if (lane == 0) asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
        } else {
            asm volatile("bar.arrive 1, 64;" ::: "memory");
        }
    } else {
        if (mode == 0) {
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(b) : "memory");
        } else {
            asm volatile("bar.sync 1, 64;" ::: "memory");
        }
        out[lane] = buf[lane];
    }
}

int main(int argc, char** argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    float* d;
    cudaMalloc(&d, 32 * sizeof(float));
    handoff<<<1, 64>>>(mode, d);
    float h[32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 32; ++i) bad += h[i] != 2.0f * i;
    printf("mode %d (%s): %s\n", mode, mode == 0 ? "mbarrier" : "named barrier", bad ? "WRONG" : "ok");
    return bad != 0;
}
