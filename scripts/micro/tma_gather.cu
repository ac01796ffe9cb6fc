// Microbenchmark: random 16-byte record gathers from an L2-resident table
// (2M records x 16 B = 32 MB, the hot-set slot array at C2).
// Mode 0: LDG.128, one record per lane (K2's gather; one L1TEX wavefront per lane).
// Mode 1: TMA tile::gather4 (cp.async.bulk.tensor ... gather4): 8 lanes each
//         fetch 4 records into a per-warp shared buffer (mbarrier, two stages),
//         then every lane reads its record with one LDS.128.
// Prints records per second and records per SM-cycle at the measured clock.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

constexpr uint32_t N = 2u * 1024 * 1024;

__device__ __forceinline__ uint32_t rnd(uint32_t &x) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    return x;
}

template <int DEPTH>
__global__ void __launch_bounds__(1024, 1) g_ldg(const uint4 *tab, int iters, uint32_t *sink) {
    uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 2654435761u + 12345u;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) v[d] = __ldg(tab + (rnd(x) & (N - 1)));
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) acc ^= v[d].x + v[d].w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(a), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(a),
        "r"(parity) : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap *map, uint32_t r0, uint32_t r1, uint32_t r2,
                                        uint32_t r3, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(mbar)
        : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(256, 4) g_tma(const __grid_constant__ CUtensorMap map, int iters, uint32_t *sink) {
    __shared__ __align__(128) uint4 buf[8][STAGES][64];
    __shared__ __align__(8) uint64_t bar[8][STAGES];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = (blockIdx.x * 256 + threadIdx.x) * 2654435761u + 12345u;
    if (lane == 0)
        for (int s = 0; s < STAGES; ++s) mbar_init((uint32_t)__cvta_generic_to_shared(&bar[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t acc = 0;
    auto issue = [&](int s) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[w][s]);
        if (lane == 0) mbar_expect(b, 32 * 16);
        __syncwarp();
        if (lane < 8) {
            const uint32_t r0 = rnd(x) & (N - 1), r1 = rnd(x) & (N - 1), r2 = rnd(x) & (N - 1), r3 = rnd(x) & (N - 1);
            gather4((uint32_t)__cvta_generic_to_shared(&buf[w][s][lane * 8]), &map, r0, r1, r2, r3, b);
        }
    };
    for (int s = 0; s < STAGES; ++s) issue(s);
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        const int s = it % STAGES;
        mbar_wait((uint32_t)__cvta_generic_to_shared(&bar[w][s]), phase);
        const uint4 v = buf[w][s][(lane >> 2) * 8 + (lane & 3)];
        acc ^= v.x + v.w;
        __syncwarp();
        issue(s);
        if (s == STAGES - 1) phase ^= 1;
    }
    for (int s = 0; s < STAGES; ++s) {
        mbar_wait((uint32_t)__cvta_generic_to_shared(&bar[w][(iters + s) % STAGES]), phase ^ ((iters + s) / STAGES != iters / STAGES));
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
    uint4 *tab;
    uint32_t *sink;
    cudaMalloc(&tab, (size_t)N * 16);
    cudaMalloc(&sink, 64);
    cudaMemset(tab, 1, (size_t)N * 16);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    auto report = [&](const char *name, double recs) {
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.3f ms  %7.2f G records/s  %5.2f records/SM-cycle @%d MHz  (%s)\n", name, ms,
               recs / ms / 1e6, recs / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000,
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        g_ldg<4><<<sms, 1024>>>(tab, iters / 4, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        report("LDG.128 depth 4", (double)sms * 1024 * (iters / 4) * 4);
    }
    CUtensorMap map;
    cuuint64_t dims[2] = {4, N};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, tab, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("tensor map encode: %d\n", (int)r);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        g_tma<4><<<4 * sms, 256>>>(map, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        report("TMA gather4, 4 stages", (double)sms * 1024 * iters);
    }
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        g_tma<2><<<4 * sms, 256>>>(map, iters, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        report("TMA gather4, 2 stages", (double)sms * 1024 * iters);
    }
    return 0;
}
