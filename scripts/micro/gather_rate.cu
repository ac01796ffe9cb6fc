// Microbenchmark: random 16-byte gathers from an L2-resident 32 MB table, no
// id stream -- the per-SM rate of scattered L2 sector reads (K2's record
// gathers in isolation).  DEPTH independent gathers in flight per lane.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_rate gather_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint32_t NREC = 1u << 21;  // 2M records x 16 B = 32 MB

template <int DEPTH, bool NA>
__global__ void __launch_bounds__(1024, 1) gather(const uint4 *tab, int64_t per_thread, unsigned long long *sink) {
    uint32_t x = (blockIdx.x * 1024u + threadIdx.x) * 2654435761u + 12345u, acc = 0;
    for (int64_t it = 0; it < per_thread; it += DEPTH) {
        uint4 v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            x = x * 1664525u + 1013904223u;
            const uint4 *p = tab + (x >> 11);
            if (NA)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[d].x), "=r"(v[d].y), "=r"(v[d].z), "=r"(v[d].w) : "l"(p));
            else
                v[d] = __ldg(p);
        }
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) acc += v[d].x ^ v[d].w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int DEPTH, bool NA>
void run(const uint4 *tab, unsigned long long *sink, int sms, int threads_per_sm) {
    const int64_t per_thread = 1024;
    const int blocks = sms * (threads_per_sm / 1024 > 0 ? threads_per_sm / 1024 : 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<DEPTH, NA><<<blocks, 1024>>>(tab, per_thread, sink);
    cudaEventRecord(a);
    gather<DEPTH, NA><<<blocks, 1024>>>(tab, per_thread, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double n = (double)blocks * 1024 * per_thread;
    printf("{\"depth\": %d, \"no_allocate\": %d, \"gathers\": %.0f, \"ms\": %.4f, \"G_per_s\": %.1f, \"per_SM_per_ns\": %.3f}\n",
           DEPTH, (int)NA, n, ms, n / ms / 1e6, n / ms / 1e6 / sms);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint4 *tab;
    unsigned long long *sink;
    cudaMalloc(&tab, (size_t)NREC * 16);
    cudaMemset(tab, 1, (size_t)NREC * 16);
    cudaMalloc(&sink, 8);
    run<1, true>(tab, sink, sms, 1024);
    run<2, true>(tab, sink, sms, 1024);
    run<4, true>(tab, sink, sms, 1024);
    run<8, true>(tab, sink, sms, 1024);
    run<4, false>(tab, sink, sms, 1024);
    run<8, false>(tab, sink, sms, 1024);
    return 0;
}
