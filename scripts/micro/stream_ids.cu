// Microbenchmark: how fast can one persistent CTA of 32 warps per SM stream
// the YET id array (1M trials x 1000 uint32 ids = 4 GB) with K2's access
// pattern, and test every id against a ~200 KB shared-memory bit filter?
//
//   mode 0: warp per trial (round-robin, as K2), 32-id rows (LDG.32 per
//           lane), 4 rows per chunk, DEPTH chunks in flight (register ring)
//   mode 1: warp per trial, one LDG.128 per lane per 128-id chunk, DEPTH in flight
//   mode 2: warp per trial, TMA bulk copy (cp.async.bulk) of 512-byte chunks
//           into a per-warp shared ring of DEPTH stages (mbarrier per stage)
//   mode 3: warp owns a contiguous block of trials and streams it as one
//           sequence (LDG.128, DEPTH in flight; trial boundaries ignored)
// FILTER=1 adds the filter test per id (hash, LDS, bit test) into a sum.
// GATHER=1 (with FILTER) also gathers a random 16-byte record from a 32 MB
// L2-resident table for every hot id (1 in 8), consumed a chunk later (K2's
// record gathers; tests whether the id stream's path limits them).
// Prints GB/s of ids.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int64_t TRIALS = 1000000, E = 1000;
constexpr int NW = 32;
constexpr uint32_t NBITS = 1600000;

__device__ __forceinline__ uint32_t ftest(const uint32_t *s_f, uint32_t e) {
    const uint32_t h = min(e, e - NBITS);
    return (s_f[h >> 5] >> (h & 31)) & 1u;
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(a),
                 "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(bar) : "memory");
}

template <int MODE, int DEPTH, bool FILTER, bool GATHER = false>
__global__ void __launch_bounds__(NW * 32, 1) stream(const uint32_t *ids, const int64_t *off, uint32_t filter_words,
                                                     unsigned long long *sink, const uint4 *tab) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *s_f = reinterpret_cast<uint32_t *>(smem);
    for (uint32_t i = threadIdx.x; i < filter_words; i += blockDim.x)
        s_f[i] = (i * 2654435761u) & ((i ^ 0x5bd1e995u) * 0x27d4eb2du) & ((i + 0x9e3779b9u) * 0x85ebca6bu);  // ~1/8 hot
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint4 *ring = reinterpret_cast<uint4 *>(smem + filter_words * 4) + warp * DEPTH * 32;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + filter_words * 4 + NW * DEPTH * 512) + warp * DEPTH;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(bars);
    if (MODE == 2 && lane < DEPTH) mbar_init(bar0 + 8 * lane, 1);
    __syncthreads();
    uint32_t acc = 0;
    const int64_t W = (int64_t)gridDim.x * NW;
    uint32_t pend[4] = {0, 0, 0, 0};
    // k: the call site's position in its chunk (a compile-time constant), so
    // pend[k] is a register and the record is consumed a chunk later
    auto use = [&](uint32_t e, int k) {
        if (!GATHER) {
            acc += FILTER ? ftest(s_f, e) : e;
            return;
        }
        const uint32_t hot = ftest(s_f, e);
        acc += pend[k];
        uint32_t r = 0;
        if (hot) r = __ldcg(reinterpret_cast<const unsigned int *>(tab + (e & ((1u << 21) - 1))));
        pend[k] = r;
    };
    if (MODE == 3) {
        const int64_t per = (TRIALS + W - 1) / W;
        const int64_t gw = (int64_t)blockIdx.x * NW + warp;
        const int64_t t0 = min(TRIALS, gw * per), t1 = min(TRIALS, t0 + per);
        const int64_t lo = off[t0], hi = off[t1];
        const uint4 *p = reinterpret_cast<const uint4 *>(ids + lo) + lane;
        const int64_t n = (hi - lo) / 128;
        uint4 buf[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) buf[d] = d < n ? __ldcs(p + 32 * d) : make_uint4(0, 0, 0, 0);
        for (int64_t c = 0; c < n; c += DEPTH) {
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const uint4 v = buf[d];
                if (c + d + DEPTH < n) buf[d] = __ldcs(p + 32 * (c + d + DEPTH));
                use(v.x, 0); use(v.y, 1); use(v.z, 2); use(v.w, 3);
            }
        }
    } else {
        uint32_t phase = 0;
        for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < TRIALS; t += W) {
            const int64_t lo = off[t], hi = off[t + 1];
            const uint32_t skew = (uint32_t)(lo & 31);
            const uint32_t *base = ids + lo - skew;
            const uint32_t len = (uint32_t)(hi - lo);
            const int nch = (int)((len + skew + 127) >> 7);
            if (MODE == 0) {
                uint32_t r[DEPTH][4];
#pragma unroll
                for (int d = 0; d < DEPTH; ++d)
#pragma unroll
                    for (int k = 0; k < 4; ++k) r[d][k] = d < nch ? __ldcs(base + 128 * d + 32 * k + lane) : 0u;
                for (int c = 0; c < nch; c += DEPTH) {
#pragma unroll
                    for (int d = 0; d < DEPTH; ++d) {
                        uint32_t v[4];
#pragma unroll
                        for (int k = 0; k < 4; ++k) v[k] = r[d][k];
                        if (c + d + DEPTH < nch)
#pragma unroll
                            for (int k = 0; k < 4; ++k) r[d][k] = __ldcs(base + 128 * (c + d + DEPTH) + 32 * k + lane);
#pragma unroll
                        for (int k = 0; k < 4; ++k) use(v[k], k);
                    }
                }
            } else if (MODE == 1) {
                const uint4 *p = reinterpret_cast<const uint4 *>(base) + lane;
                uint4 buf[DEPTH];
#pragma unroll
                for (int d = 0; d < DEPTH; ++d) buf[d] = d < nch ? __ldcs(p + 32 * d) : make_uint4(0, 0, 0, 0);
                for (int c = 0; c < nch; c += DEPTH) {
#pragma unroll
                    for (int d = 0; d < DEPTH; ++d) {
                        const uint4 v = buf[d];
                        if (c + d + DEPTH < nch) buf[d] = __ldcs(p + 32 * (c + d + DEPTH));
                        use(v.x, 0); use(v.y, 1); use(v.z, 2); use(v.w, 3);
                    }
                }
            } else {  // MODE 2: TMA ring; stage s holds chunk c with c % DEPTH == s
                const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
                if (lane == 0)
                    for (int d = 0; d < DEPTH && d < nch; ++d) {
                        mbar_expect_tx(bar0 + 8 * d, 512);
                        bulk_g2s(ring_s + 512 * d, base + 128 * d, 512, bar0 + 8 * d);
                    }
                for (int c = 0; c < nch; ++c) {
                    const int s = c % DEPTH;
                    mbar_wait(bar0 + 8 * s, (phase >> s) & 1);
                    phase ^= 1u << s;
                    const uint4 v = ring[s * 32 + lane];
                    __syncwarp();
                    if (lane == 0 && c + DEPTH < nch) {
                        mbar_expect_tx(bar0 + 8 * s, 512);
                        bulk_g2s(ring_s + 512 * s, base + 128 * (c + DEPTH), 512, bar0 + 8 * s);
                    }
                    use(v.x, 0); use(v.y, 1); use(v.z, 2); use(v.w, 3);
                }
            }
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void fill(uint32_t *ids, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        ids[i] = (uint32_t)(((uint64_t)i * 2654435761ull) % 2000000ull) + 1u;
}

template <int MODE, int DEPTH, bool FILTER, bool GATHER = false>
void run(const uint32_t *ids, const int64_t *off, unsigned long long *sink, int sms, const uint4 *tab = nullptr) {
    const size_t ring = MODE == 2 ? NW * DEPTH * 512 + NW * DEPTH * 8 : 0;
    uint32_t fw = 50000;  // 200 KB of filter words (less when the TMA ring needs room)
    if (fw * 4 + ring > 227 * 1024) fw = (uint32_t)((227 * 1024 - ring) / 4) & ~3u;
    const size_t smem = fw * 4 + ring;
    if (smem > 227 * 1024) { printf("mode %d depth %d: smem %zu too large\n", MODE, DEPTH, smem); return; }
    cudaFuncSetAttribute(stream<MODE, DEPTH, FILTER, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) stream<MODE, DEPTH, FILTER, GATHER><<<sms, NW * 32, smem>>>(ids, off, fw, sink, tab);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) stream<MODE, DEPTH, FILTER, GATHER><<<sms, NW * 32, smem>>>(ids, off, fw, sink, tab);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const cudaError_t e = cudaGetLastError();
    printf("{\"mode\": %d, \"depth\": %d, \"filter\": %d, \"gather\": %d, \"ms\": %.4f, \"GBps\": %.1f, \"err\": \"%s\"}\n", MODE, DEPTH,
           (int)FILTER, (int)GATHER, ms, TRIALS * E * 4 / ms / 1e6, cudaGetErrorString(e));
}

// MODE 4 (separate kernel): the same per-trial stream over a packed resident
// layout -- 21-bit ids, three per 64-bit word, stride-major within a 96-id
// block (lane l's word holds positions l, l+32, l+64), each trial padded to
// whole blocks.  2.8 GB instead of 4 GB per 1M x 1000 trials.
constexpr int NBLK = (int)((E + 95) / 96);
template <int DEPTH, bool GATHER>
__global__ void __launch_bounds__(NW * 32, 1) stream_packed(const unsigned long long *pk, uint32_t filter_words,
                                                            unsigned long long *sink, const uint4 *tab) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *s_f = reinterpret_cast<uint32_t *>(smem);
    for (uint32_t i = threadIdx.x; i < filter_words; i += blockDim.x)
        s_f[i] = (i * 2654435761u) & ((i ^ 0x5bd1e995u) * 0x27d4eb2du) & ((i + 0x9e3779b9u) * 0x85ebca6bu);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t acc = 0, pend[3] = {0, 0, 0};
    auto use = [&](uint32_t e, int k) {
        const uint32_t hot = ftest(s_f, e);
        if (!GATHER) { acc += hot; return; }
        acc += pend[k];
        uint32_t r = 0;
        if (hot) r = __ldcg(reinterpret_cast<const unsigned int *>(tab + (e & ((1u << 21) - 1))));
        pend[k] = r;
    };
    const int64_t W = (int64_t)gridDim.x * NW;
    for (int64_t t = (int64_t)blockIdx.x * NW + warp; t < TRIALS; t += W) {
        const unsigned long long *base = pk + t * NBLK * 32 + lane;
        unsigned long long r[DEPTH];
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) r[d] = __ldcs(base + 32 * d);
        for (int c = 0; c < NBLK; c += DEPTH) {
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
                const unsigned long long v = r[d];
                if (c + d + DEPTH < NBLK) r[d] = __ldcs(base + 32 * (c + d + DEPTH));
                if (c + d < NBLK) {
                    use((uint32_t)v & 0x1FFFFFu, 0);
                    use((uint32_t)(v >> 21) & 0x1FFFFFu, 1);
                    use((uint32_t)(v >> 42), 2);
                }
            }
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void pack(const uint32_t *ids, unsigned long long *pk) {
    const int64_t n = TRIALS * NBLK * 32;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / (NBLK * 32), b = (i / 32) % NBLK, l = i % 32;
        unsigned long long w = 0;
        for (int k = 0; k < 3; ++k) {
            const int64_t pos = 96 * b + 32 * k + l;
            const unsigned long long e = pos < E ? ids[t * E + pos] : 0u;
            w |= e << (21 * k);
        }
        pk[i] = w;
    }
}

template <int DEPTH, bool GATHER>
void run_packed(const unsigned long long *pk, unsigned long long *sink, int sms, const uint4 *tab) {
    const uint32_t fw = 50000;
    const size_t smem = fw * 4;
    cudaFuncSetAttribute(stream_packed<DEPTH, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) stream_packed<DEPTH, GATHER><<<sms, NW * 32, smem>>>(pk, fw, sink, tab);
    cudaEventRecord(a);
    const int reps = 5;
    for (int i = 0; i < reps; ++i) stream_packed<DEPTH, GATHER><<<sms, NW * 32, smem>>>(pk, fw, sink, tab);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("{\"mode\": \"packed21\", \"depth\": %d, \"filter\": 1, \"gather\": %d, \"ms\": %.4f, \"GBps_equiv_u32\": %.1f, \"err\": \"%s\"}\n",
           DEPTH, (int)GATHER, ms, TRIALS * E * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *ids;
    int64_t *off;
    unsigned long long *sink;
    cudaMalloc(&ids, TRIALS * E * 4 + 1024);
    cudaMalloc(&off, (TRIALS + 1) * 8);
    cudaMalloc(&sink, 8);
    fill<<<sms * 8, 256>>>(ids, TRIALS * E);
    int64_t *h = new int64_t[TRIALS + 1];
    for (int64_t t = 0; t <= TRIALS; ++t) h[t] = t * E;
    cudaMemcpy(off, h, (TRIALS + 1) * 8, cudaMemcpyHostToDevice);
    uint4 *tab;
    cudaMalloc(&tab, (size_t)(1u << 21) * 16);
    cudaMemset(tab, 0, (size_t)(1u << 21) * 16);
    if (getenv("PACKED")) {
        unsigned long long *pk;
        cudaMalloc(&pk, (size_t)TRIALS * NBLK * 32 * 8);
        pack<<<sms * 8, 256>>>(ids, pk);
        run<0, 2, true>(ids, off, sink, sms);
        run<0, 2, true, true>(ids, off, sink, sms, tab);
        run<0, 3, true, true>(ids, off, sink, sms, tab);
        run_packed<2, false>(pk, sink, sms, tab);
        run_packed<4, false>(pk, sink, sms, tab);
        run_packed<2, true>(pk, sink, sms, tab);
        run_packed<3, true>(pk, sink, sms, tab);
        run_packed<4, true>(pk, sink, sms, tab);
        return 0;
    }
    const bool all = getenv("ALL") != nullptr;
    if (all) {
        run<0, 2, false>(ids, off, sink, sms);
        run<1, 4, true>(ids, off, sink, sms);
        run<3, 4, true>(ids, off, sink, sms);
    }
    run<0, 2, true>(ids, off, sink, sms);
    run<0, 2, true, true>(ids, off, sink, sms, tab);
    run<0, 3, true, true>(ids, off, sink, sms, tab);
    run<2, 2, true>(ids, off, sink, sms);
    run<2, 2, true, true>(ids, off, sink, sms, tab);
    run<2, 3, true, true>(ids, off, sink, sms, tab);
    run<2, 4, true, true>(ids, off, sink, sms, tab);
    run<1, 4, true, true>(ids, off, sink, sms, tab);
    run<3, 4, true, true>(ids, off, sink, sms, tab);
    return 0;
}
