// Microbenchmark: random 4-byte loads from a 2-CTA cluster's shared memory
// (half local, half remote via mapa + ld.shared::cluster), the access pattern
// an exact filter split across two SMs would have.  Prints loads/s per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int THREADS = 1024, WORDS = 125 * 1024 / 4, ITERS = 4096;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) dsmem(uint32_t *out, int remote_pct) {
    extern __shared__ uint32_t bits[];
    for (int i = threadIdx.x; i < WORDS; i += THREADS) bits[i] = i * 2654435761u;
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    uint32_t rank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(bits);
    uint32_t x = threadIdx.x * 7919u + blockIdx.x * 104729u, acc = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x = x * 1664525u + 1013904223u;
            const uint32_t w = (x >> 8) % WORDS;
            const uint32_t owner = ((x & 127u) < (uint32_t)remote_pct * 128u / 100u) ? (rank ^ 1u) : rank;
            uint32_t addr, v;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(base + 4 * w), "r"(owner));
            asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr));
            acc += v;
        }
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void __launch_bounds__(THREADS, 1) local_only(uint32_t *out) {
    extern __shared__ uint32_t bits[];
    for (int i = threadIdx.x; i < WORDS; i += THREADS) bits[i] = i * 2654435761u;
    __syncthreads();
    uint32_t x = threadIdx.x * 7919u + blockIdx.x * 104729u, acc = 0;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            x = x * 1664525u + 1013904223u;
            acc += bits[(x >> 8) % WORDS];
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out;
    cudaMalloc(&out, 4);
    const size_t smem = WORDS * 4;
    cudaFuncSetAttribute(dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(local_only, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = sms / 2 * 2;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double loads = (double)grid * THREADS * ITERS * 4;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        local_only<<<grid, THREADS, smem>>>(out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("local LDS          : %.3f ms, %.2f G loads/s per SM\n", ms, loads / (ms * 1e-3) / grid / 1e9);
        for (int pct : {0, 50, 100}) {
            cudaEventRecord(a);
            dsmem<<<grid, THREADS, smem>>>(out, pct);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("cluster, %3d%% remote: %.3f ms, %.2f G loads/s per SM (%s)\n", pct, ms,
                   loads / (ms * 1e-3) / grid / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
