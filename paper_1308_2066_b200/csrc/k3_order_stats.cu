// K3 -- order statistics over a Year Loss Table: PML, TVaR, EP points, and
// the per-trial portfolio roll-up.
//
// Replaces pkg/src/aggrisk/metrics.py:29-133.  PML at return period rp is
// the k-th smallest loss with k = n - floor(n / rp) (metrics.py:29-42,
// computed on the host in the same float64 arithmetic); TVaR is the mean of
// the closed tail, the top m = n - k + 1 order statistics (metrics.py:55-63).
//
// Device algorithm: one cooperative launch.  MSD radix select on the
// order-preserving 64-bit key of each float64 (NaN last, like np.partition),
// 8 passes of 8 bits, all return periods of a call selected together (one
// 256-bin histogram per rp and pass: shared-memory atomics, one global add
// per bin, a grid barrier, then every CTA fixes the next digit itself).  The tail sum is
// then  S = sum of losses strictly above the PML key  (double-double
// accumulation, fixed grid, partials combined in a fixed order, so the
// result is bit-reproducible run to run and for any GPU count) plus
// (m - G) copies of the PML value itself (G = count strictly above):
//     tvar = (S + (m - G) * pml) / m.
// This equals the mean of the closed tail for any ties; it is within a few
// ulp of numpy's pairwise mean (tolerance in tests/test_metrics_gpu.py).
#include "k3_order_stats.cuh"

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <vector>

namespace are {

static constexpr int K3_MAX_RP = 16;
static constexpr int K3_THREADS = 512;

struct DD {
    double hi, lo;
};
__device__ __forceinline__ void dd_add(DD &a, double b) {
    const double s = __dadd_rn(a.hi, b);
    const double bb = __dsub_rn(s, a.hi);
    const double err = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    a.hi = s;
    a.lo = __dadd_rn(a.lo, err);
}

struct TailPartial {
    double hi, lo;
    unsigned long long above;
    unsigned long long pad;
};

// Device workspace of one K3 call; zeroed (hist, barrier) before launch.
struct K3Work {
    unsigned int hist[3][K3_MAX_RP][256];  // triple-buffered pass histograms
    unsigned int bar_count, bar_gen;
    int64_t rank[K3_MAX_RP];               // 1-based ranks k (input)
    int64_t m_tail[K3_MAX_RP];             // n - k + 1 (input)
    double res[2][K3_MAX_RP];              // pml, tvar (output)
};

// Sense-free generation barrier across a co-resident (cooperative) grid.
__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *count = 0;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// One cooperative launch: 8 MSD radix passes (8-bit digits) selecting the
// k-th smallest key for every return period, then the tail sums.
__global__ void __launch_bounds__(K3_THREADS) k3_select(const double *__restrict__ x, int64_t n, int n_rp,
                                                       K3Work *__restrict__ w, TailPartial *__restrict__ part) {
    __shared__ unsigned int sh[K3_MAX_RP * 256];
    __shared__ uint64_t s_prefix[K3_MAX_RP];
    __shared__ uint64_t s_rank[K3_MAX_RP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < n_rp) {
        s_prefix[tid] = 0;
        s_rank[tid] = (uint64_t)w->rank[tid];
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + 8));
        for (int i = tid; i < n_rp * 256; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < n; i += stride) {
            const uint64_t k = order_key(x[i]);
            const unsigned d = (unsigned)(k >> shift) & 255u;
            for (int r = 0; r < n_rp; ++r)
                if (((k ^ s_prefix[r]) & hi_mask) == 0) atomicAdd(&sh[r * 256 + d], 1u);
        }
        __syncthreads();
        unsigned int(*h)[256] = w->hist[pass % 3];
        for (int i = tid; i < n_rp * 256; i += blockDim.x)
            if (sh[i]) atomicAdd(&h[i >> 8][i & 255], sh[i]);
        grid_barrier(&w->bar_count, &w->bar_gen);
        if (blockIdx.x == 0)  // buffer of pass+2 was last read before this barrier
            for (int i = tid; i < n_rp * 256; i += blockDim.x) w->hist[(pass + 2) % 3][i >> 8][i & 255] = 0;
        // every CTA fixes the next digit itself: warp r scans rp r's 256 bins
        if (warp < n_rp) {
            const volatile unsigned int *hr = h[warp];
            uint64_t cnt[8], tot = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                cnt[b] = hr[lane * 8 + b];
                tot += cnt[b];
            }
            uint64_t inc = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            const uint64_t want = s_rank[warp];
            uint64_t run = inc - tot;  // bins before this lane's 8
            const bool mine = run < want && want <= inc;
            const unsigned owner = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                int b = 0;
                for (; b < 7 && run + cnt[b] < want; ++b) run += cnt[b];
                s_rank[warp] = want - run;
                s_prefix[warp] |= (uint64_t)(lane * 8 + b) << shift;
            }
            (void)owner;
        }
        __syncthreads();
    }
    // tail: sum and count of losses strictly above each PML key
    for (int r = 0; r < n_rp; ++r) {
        const uint64_t kp = s_prefix[r];
        DD acc = {0.0, 0.0};
        unsigned long long above = 0;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + tid; i < n; i += stride) {
            const double v = x[i];
            if (order_key(v) > kp) {
                dd_add(acc, v);
                ++above;
            }
        }
        __shared__ double shi[K3_THREADS], slo[K3_THREADS];
        __shared__ unsigned long long sab[K3_THREADS];
        shi[tid] = acc.hi;
        slo[tid] = acc.lo;
        sab[tid] = above;
        __syncthreads();
        if (tid == 0) {  // fixed-order block combine
            DD b = {0.0, 0.0};
            unsigned long long ab = 0;
            for (int i = 0; i < (int)blockDim.x; ++i) {
                dd_add(b, shi[i]);
                b.lo = __dadd_rn(b.lo, slo[i]);
                ab += sab[i];
            }
            part[(int64_t)r * gridDim.x + blockIdx.x] = TailPartial{b.hi, b.lo, ab, 0};
        }
        __syncthreads();
    }
    grid_barrier(&w->bar_count, &w->bar_gen);
    if (blockIdx.x == 0 && tid < n_rp) {  // fixed-order grid combine
        const int r = tid;
        DD s = {0.0, 0.0};
        unsigned long long above = 0;
        for (int b = 0; b < (int)gridDim.x; ++b) {
            const TailPartial p = part[(int64_t)r * gridDim.x + b];
            dd_add(s, p.hi);
            s.lo = __dadd_rn(s.lo, p.lo);
            above += p.above;
        }
        const double pml = key_value(s_prefix[r]);
        const int64_t m = w->m_tail[r];
        const double copies = (double)(m - (int64_t)above);
        const double prod = __dmul_rn(copies, pml);
        double total;
        if (isfinite(prod) && isfinite(s.hi)) {
            const double perr = fma(copies, pml, -prod);  // exact product error
            dd_add(s, prod);
            s.lo = __dadd_rn(s.lo, perr);
            total = __dadd_rn(s.hi, s.lo);
        } else {
            total = __dadd_rn(__dadd_rn(s.hi, s.lo), prod);
        }
        w->res[0][r] = pml;
        w->res[1][r] = __ddiv_rn(total, (double)m);
    }
}

__global__ void k3_rollup(const double *const *__restrict__ ylts, int n_layers, int first_chunk,
                          int64_t n, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double acc = first_chunk ? ylts[0][i] : out[i];
        for (int l = first_chunk ? 1 : 0; l < n_layers; ++l) acc = __dadd_rn(acc, ylts[l][i]);
        out[i] = acc;
    }
}

// metrics.py:29-42 in the same float64 arithmetic Python uses.
int order_stat_k(int64_t n, double rp, int64_t *k) {
    if (!(rp > 1.0)) return fail(ARE_EINVAL, "return_period must exceed 1");
    if (rp > (double)n) return fail(ARE_EINVAL, "return_period exceeds trial count");
    const double q = (double)n / rp;
    *k = n - (int64_t)std::floor(q);
    if (*k < 1 || *k > n) return fail(ARE_EINVAL, "order statistic rank out of range");
    return ARE_OK;
}

// Per-device cached K3 workspace (device K3Work + tail partials + pinned
// host staging), serialised by a mutex.
struct K3Cache {
    std::mutex mu;
    int device = -1;
    K3Work *d_work = nullptr;
    TailPartial *d_part = nullptr;
    K3Work *h_work = nullptr;  // pinned
    int grid = 0;
};
static K3Cache g_k3[64];

int k3_order_stats(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                   double *tvar_out, int sms, cudaStream_t st) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    if (n >= (int64_t)0xFFFFFFFFll) return fail(ARE_EINVAL, "year loss table too long for K3");
    int dev;
    ARE_CUDA(cudaGetDevice(&dev));
    K3Cache &c = g_k3[dev & 63];
    std::lock_guard<std::mutex> guard(c.mu);
    if (!c.d_work) {
        int per_sm = 0;
        ARE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_select, K3_THREADS, 0));
        c.grid = sms * std::max(1, std::min(per_sm, 2));
        ARE_CUDA(cudaMalloc(&c.d_work, sizeof(K3Work)));
        ARE_CUDA(cudaMalloc(&c.d_part, sizeof(TailPartial) * (size_t)c.grid * K3_MAX_RP));
        ARE_CUDA(cudaHostAlloc(&c.h_work, sizeof(K3Work), cudaHostAllocDefault));
    }
    for (int64_t base = 0; base < n_rp; base += K3_MAX_RP) {
        const int R = (int)std::min<int64_t>(K3_MAX_RP, n_rp - base);
        for (int r = 0; r < R; ++r) {
            int64_t k;
            int rc = order_stat_k(n, rps[base + r], &k);
            if (rc) return rc;
            c.h_work->rank[r] = k;
            c.h_work->m_tail[r] = n - k + 1;
        }
        std::memset(c.h_work->hist, 0, sizeof(c.h_work->hist));
        c.h_work->bar_count = c.h_work->bar_gen = 0;
        ARE_CUDA(cudaMemcpyAsync(c.d_work, c.h_work, offsetof(K3Work, res), cudaMemcpyHostToDevice, st));
        int grid = (int)std::min<int64_t>(c.grid, (n + K3_THREADS - 1) / K3_THREADS);
        grid = std::max(grid, 1);
        int nn = R;
        void *args[] = {(void *)&d_x, (void *)&n, (void *)&nn, (void *)&c.d_work, (void *)&c.d_part};
        ARE_CUDA(cudaLaunchCooperativeKernel((void *)k3_select, grid, K3_THREADS, args, 0, st));
        ARE_LAUNCHED();
        ARE_CUDA(cudaMemcpyAsync(c.h_work->res, c.d_work->res, sizeof(c.h_work->res), cudaMemcpyDeviceToHost, st));
        ARE_CUDA(cudaStreamSynchronize(st));
        for (int r = 0; r < R; ++r) {
            pml_out[base + r] = c.h_work->res[0][r];
            tvar_out[base + r] = c.h_work->res[1][r];
        }
    }
    return ARE_OK;
}

int k3_rollup_launch(const double *const *d_ylts_host_array, int64_t n_layers, int64_t n, double *d_out,
                     int sms, cudaStream_t st) {
    if (n_layers < 1) return fail(ARE_EINVAL, "no year loss tables to roll up");
    static constexpr int CH = 64;
    const double **d_ptrs = nullptr;
    ARE_CUDA(cudaMallocAsync((void **)&d_ptrs, sizeof(double *) * n_layers, st));
    ARE_CUDA(cudaMemcpyAsync(d_ptrs, d_ylts_host_array, sizeof(double *) * n_layers, cudaMemcpyHostToDevice, st));
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
    for (int64_t l0 = 0; l0 < n_layers; l0 += CH) {
        const int nl = (int)std::min<int64_t>(CH, n_layers - l0);
        k3_rollup<<<blocks < 1 ? 1 : blocks, 256, 0, st>>>(d_ptrs + l0, nl, l0 == 0, n, d_out);
        ARE_LAUNCHED();
    }
    cudaFreeAsync(d_ptrs, st);
    ARE_CUDA(cudaStreamSynchronize(st));
    return ARE_OK;
}

}  // namespace are
