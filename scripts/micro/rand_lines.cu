// Microbenchmark: random 128-byte line reads from a table larger than L2
// (2M lines x 128 B = 256 MB, the dense kernel's event-major copy at C2/C4).
// Mode 0: one lane per line, 8 x 16-byte loads per lane (k2_dense's pattern).
// Mode 1: 8 lanes per line, one 16-byte load each (4 lines per warp load).
// Prints line bytes per second (GB/s).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int LINES = 2 * 1024 * 1024;

__device__ __forceinline__ uint32_t rnd(uint32_t &x) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    return x;
}

template <int MODE, int DEPTH>
__global__ void __launch_bounds__(256) rl(const double2 *tab, int iters, double *sink) {
    const int lane = threadIdx.x & 31;
    uint32_t x = (blockIdx.x * 256 + threadIdx.x) * 2654435761u + 12345u;
    if (MODE == 1) x = ((blockIdx.x * 256 + threadIdx.x) >> 3) * 2654435761u + 12345u;  // 8 lanes share a stream
    double acc = 0.0;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            const uint32_t l = rnd(x) & (LINES - 1);
            double2 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldg(tab + (size_t)l * 8 + k);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y;
        } else {
            double2 v[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const uint32_t l = rnd(x) & (LINES - 1);
                v[d] = __ldg(tab + (size_t)l * 8 + (lane & 7));
            }
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) acc += v[d].x + v[d].y;
        }
    }
    if (acc == 1.2345) sink[0] = acc;
}

int main() {
    double2 *tab;
    double *sink;
    cudaMalloc(&tab, (size_t)LINES * 128);
    cudaMemset(tab, 0, (size_t)LINES * 128);
    cudaMalloc(&sink, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int blocks_per_sm : {4, 8}) {
        const int grid = sms * blocks_per_sm, iters = 2000;
        for (int mode = 0; mode < 3; ++mode) {
            auto run = [&]() {
                if (mode == 0) rl<0, 1><<<grid, 256>>>(tab, iters, sink);
                else if (mode == 1) rl<1, 8><<<grid, 256>>>(tab, iters, sink);
                else rl<1, 16><<<grid, 256>>>(tab, iters / 2, sink);
            };
            run();
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) run();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            // lines read: mode 0 one per thread-iter; mode 1/2 DEPTH per 8 threads per iter
            const double lines = mode == 0 ? (double)grid * 256 * iters
                                           : (double)grid * 256 / 8 * iters * 8;
            printf("ctas/SM %d mode %d: %.0f GB/s of 128-byte lines (%s)\n", blocks_per_sm, mode,
                   3 * lines * 128 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
