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
// six passes of 11/11/11/11/11/9 bits, up to 8 return periods selected
// together.  Pass 0 builds ONE histogram all return periods share (no prefix
// yet); later passes build one per distinct prefix (return periods whose
// prefixes agree -- ties, e.g. several PMLs at an aggregate limit -- share
// it).  Shared-memory atomics, one global add per non-empty bin, a grid
// barrier, then every CTA fixes the next digit itself.  One tail pass then
// accumulates, for every return period at once,
//     S = sum of losses strictly above the PML key
// in double-double (warp trees, a block tree, and a last-block combine of
// the per-CTA partials -- a fixed order for a fixed grid, so the result is
// bit-reproducible run to run) plus (m - G) copies of the PML value itself
// (G = count strictly above):
//     tvar = (S + (m - G) * pml) / m.
// This equals the mean of the closed tail for any ties; it is within a few
// ulp of numpy's pairwise mean (tolerance in tests/test_metrics_gpu.py).
#include "k3_order_stats.cuh"

#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <mutex>
#include <vector>

namespace are {

static constexpr int K3_GROUP = 8;       // return periods per launch
static constexpr int K3_THREADS = 512;
static constexpr int K3_BINS = 2048;     // 11-bit digits
static constexpr int K3_PASSES = 6;      // 11, 11, 11, 11, 11, 9 bits
static constexpr int K3_TAIL = 4;        // return periods per tail sweep

__host__ __device__ constexpr int k3_shift(int pass) { return pass < 5 ? 53 - 11 * pass : 0; }
__host__ __device__ constexpr int k3_width(int pass) { return pass < 5 ? 11 : 9; }

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
__device__ __forceinline__ void dd_merge(DD &a, const DD &b) {
    dd_add(a, b.hi);
    a.lo = __dadd_rn(a.lo, b.lo);
}
// Fixed-shape warp tree: lane 0 ends with the combined value.
__device__ __forceinline__ void dd_warp_reduce(DD &a, unsigned long long &cnt) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        DD b;
        b.hi = __shfl_down_sync(0xffffffffu, a.hi, o);
        b.lo = __shfl_down_sync(0xffffffffu, a.lo, o);
        const unsigned long long c = __shfl_down_sync(0xffffffffu, cnt, o);
        dd_merge(a, b);
        cnt += c;
    }
}

struct TailPartial {
    double hi, lo;
    unsigned long long above;
    unsigned long long pad;
};

struct K3Params {
    int64_t rank[K3_GROUP];    // 1-based ranks k
    int64_t m_tail[K3_GROUP];  // n - k + 1
    int n_rp;
    int summary;               // also the mean and the maximum (slot n_rp of the tail pass)
};

// Device workspace of one K3 call; cleared (cudaMemsetAsync) before launch.
struct K3Work {
    unsigned int hist[3][K3_GROUP][K3_BINS];  // triple-buffered pass histograms
    unsigned int bar_count, bar_gen, done, pad;
    double res[2][K3_GROUP];                  // pml, tvar (output)
    double summary[2];                        // mean, max (output, when requested)
};

__global__ void __launch_bounds__(K3_THREADS, 2) k3_select(const double *__restrict__ x, int64_t n, const K3Params prm,
                                                          K3Work *__restrict__ w, TailPartial *__restrict__ part) {
    extern __shared__ unsigned int sh[];  // [K3_GROUP][K3_BINS]
    __shared__ uint64_t s_prefix[K3_GROUP];
    __shared__ uint64_t s_rank[K3_GROUP];
    __shared__ uint64_t s_lpre[K3_GROUP];  // distinct prefixes ("leaders")
    __shared__ int s_slot[K3_GROUP];       // rp -> its leader's histogram row
    __shared__ int s_nlead;
    __shared__ DD s_dd[K3_THREADS / 32][K3_TAIL];
    __shared__ unsigned long long s_cnt[K3_THREADS / 32][K3_TAIL];
    __shared__ int s_last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int R = prm.n_rp;
    if (tid < R) {
        s_prefix[tid] = 0;
        s_rank[tid] = (uint64_t)prm.rank[tid];
        s_slot[tid] = 0;
        s_lpre[tid] = 0;
    }
    if (tid == 0) s_nlead = 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + tid;
    for (int pass = 0; pass < K3_PASSES; ++pass) {
        const int shift = k3_shift(pass), nb = 1 << k3_width(pass);
        const uint64_t hi_mask = pass == 0 ? 0ull : (~0ull << (shift + k3_width(pass)));
        __syncthreads();
        const int rows = s_nlead;
        for (int i = tid; i < rows * nb; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        if (pass == 0) {
            int64_t i = i0;
            for (; i + 3 * stride < n; i += 4 * stride) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(x + i + u * stride);
#pragma unroll
                for (int u = 0; u < 4; ++u) atomicAdd(&sh[(unsigned)(order_key(v[u]) >> shift)], 1u);
            }
            for (; i < n; i += stride) atomicAdd(&sh[(unsigned)(order_key(__ldg(x + i)) >> shift)], 1u);
        } else {
            uint64_t pre[K3_GROUP];
#pragma unroll
            for (int j = 0; j < K3_GROUP; ++j) pre[j] = j < rows ? s_lpre[j] : 0;
            auto count = [&](double v) {
                const uint64_t k = order_key(v);
                const unsigned d = (unsigned)(k >> shift) & (unsigned)(nb - 1);
#pragma unroll
                for (int j = 0; j < K3_GROUP; ++j) {
                    if (j >= rows) break;
                    if (((k ^ pre[j]) & hi_mask) == 0) atomicAdd(&sh[j * nb + d], 1u);
                }
            };
            int64_t i = i0;
            for (; i + 3 * stride < n; i += 4 * stride) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(x + i + u * stride);
#pragma unroll
                for (int u = 0; u < 4; ++u) count(v[u]);
            }
            for (; i < n; i += stride) count(__ldg(x + i));
        }
        __syncthreads();
        unsigned int(*h)[K3_BINS] = w->hist[pass % 3];
        for (int i = tid; i < rows * nb; i += blockDim.x)
            if (sh[i]) atomicAdd(&h[i / nb][i % nb], sh[i]);
        cooperative_groups::this_grid().sync();
        if (blockIdx.x == 0)  // buffer of pass+2 was last read before this barrier
            for (int i = tid; i < R * K3_BINS; i += blockDim.x) w->hist[(pass + 2) % 3][i / K3_BINS][i % K3_BINS] = 0;
        // stage the global histogram rows in shared memory (one round trip)
        {
            const int q = nb >> 2;  // uint4 per row
            for (int i = tid; i < rows * q; i += blockDim.x)
                reinterpret_cast<uint4 *>(sh)[i] = __ldcg(reinterpret_cast<const uint4 *>(h[i / q]) + (i % q));
        }
        __syncthreads();
        // every CTA fixes the next digit itself: warp r scans rp r's row
        if (warp < R) {
            const unsigned int *hr = sh + s_slot[warp] * nb;
            const int per = nb >> 5;  // bins per lane: 64 or 16
            const uint4 *mine = reinterpret_cast<const uint4 *>(hr + lane * per);
            uint64_t tot = 0;
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if (4 * b < per) {
                    const uint4 v = mine[b];
                    tot += (uint64_t)v.x + v.y + v.z + v.w;
                }
            uint64_t inc = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += v;
            }
            const uint64_t want = s_rank[warp];
            // the lane whose bins cross `want`, then the warp searches its
            // bins 32 at a time (shuffle scan, ballot)
            const unsigned owner_mask = __ballot_sync(0xffffffffu, inc - tot < want && want <= inc);
            const int owner = __ffs(owner_mask) - 1;
            uint64_t run = __shfl_sync(0xffffffffu, inc - tot, owner);
            const unsigned int *ob = hr + owner * per;
            for (int b0 = 0; b0 < per; b0 += 32) {
                const uint64_t c = lane < per - b0 ? ob[b0 + lane] : 0u;
                uint64_t ci = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t v = __shfl_up_sync(0xffffffffu, ci, o);
                    if (lane >= o) ci += v;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, run + ci >= want);
                if (hit) {
                    const int l = __ffs(hit) - 1;
                    const uint64_t before = run + __shfl_sync(0xffffffffu, ci - c, l);
                    if (lane == 0) {
                        s_rank[warp] = want - before;
                        s_prefix[warp] |= (uint64_t)(owner * per + b0 + l) << shift;
                    }
                    break;
                }
                run += __shfl_sync(0xffffffffu, ci, 31);
            }
        }
        __syncthreads();
        if (tid == 0) {  // equal prefixes share one histogram row next pass
            int nl = 0;
            for (int r = 0; r < R; ++r) {
                int j = 0;
                while (j < nl && s_lpre[j] != s_prefix[r]) ++j;
                if (j == nl) s_lpre[nl++] = s_prefix[r];
                s_slot[r] = j;
            }
            s_nlead = nl;
        }
    }
    // tail: sum and count of losses strictly above each PML key, K3_TAIL
    // return periods per sweep.  The summary (mean, max) rides along as slot
    // R: key 0 lies below every loss (NaN included), so it sums them all, and
    // the sweep that holds it also tracks the largest key.
    const int RT = R + (prm.summary ? 1 : 0);
    uint64_t kmax = 0;
    for (int r0 = 0; r0 < RT; r0 += K3_TAIL) {
        uint64_t kp[K3_TAIL];
        DD acc[K3_TAIL];
        unsigned long long above[K3_TAIL];
#pragma unroll
        for (int r = 0; r < K3_TAIL; ++r) {
            kp[r] = r0 + r < R ? s_prefix[r0 + r] : (r0 + r == R && prm.summary ? 0ull : ~0ull);  // ~0: nothing is above
            acc[r] = DD{0.0, 0.0};
            above[r] = 0;
        }
        const bool track_max = prm.summary && R >= r0 && R < r0 + K3_TAIL;
        auto tail = [&](double v) {
            const uint64_t k = order_key(v);
            if (track_max) kmax = max(kmax, k);
#pragma unroll
            for (int r = 0; r < K3_TAIL; ++r)
                if (k > kp[r]) {
                    dd_add(acc[r], v);
                    ++above[r];
                }
        };
        int64_t i = i0;
        for (; i + 3 * stride < n; i += 4 * stride) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(x + i + u * stride);
#pragma unroll
            for (int u = 0; u < 4; ++u) tail(v[u]);
        }
        for (; i < n; i += stride) tail(__ldg(x + i));
#pragma unroll
        for (int r = 0; r < K3_TAIL; ++r) {
            dd_warp_reduce(acc[r], above[r]);
            if (lane == 0) {
                s_dd[warp][r] = acc[r];
                s_cnt[warp][r] = above[r];
            }
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll
            for (int r = 0; r < K3_TAIL; ++r) {
                DD a = {0.0, 0.0};
                unsigned long long c = 0;
                if (lane < K3_THREADS / 32) {
                    a = s_dd[lane][r];
                    c = s_cnt[lane][r];
                }
                dd_warp_reduce(a, c);
                if (lane == 0 && r0 + r < RT)
                    part[(int64_t)(r0 + r) * gridDim.x + blockIdx.x] = TailPartial{a.hi, a.lo, c, 0};
            }
        }
        __syncthreads();
    }
    if (prm.summary) {  // the CTA's largest key, next to its summary partial
        unsigned long long m = kmax;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) s_cnt[warp][0] = m;
        __syncthreads();
        if (warp == 0) {
            m = lane < K3_THREADS / 32 ? s_cnt[lane][0] : 0ull;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) part[(int64_t)R * gridDim.x + blockIdx.x].pad = m;
        }
    }
    // the last CTA to finish combines the partials
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(&w->done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (warp < R) {
        const int r = warp;
        DD s = {0.0, 0.0};
        unsigned long long ab = 0;
        for (int b0 = 0; b0 < (int)gridDim.x; b0 += 32 * 8) {  // loads first, then merge
            double2 v[8];
            unsigned long long c[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int b = b0 + 32 * u + lane;
                const TailPartial *pp = part + (int64_t)r * gridDim.x + b;
                v[u] = b < (int)gridDim.x ? __ldcg(reinterpret_cast<const double2 *>(pp)) : make_double2(0.0, 0.0);
                c[u] = b < (int)gridDim.x ? __ldcg(&pp->above) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                dd_merge(s, DD{v[u].x, v[u].y});
                ab += c[u];
            }
        }
        dd_warp_reduce(s, ab);
        if (lane == 0) {
            const double pml = key_value(s_prefix[r]);
            const int64_t m = prm.m_tail[r];
            const double copies = (double)(m - (int64_t)ab);
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
    if (prm.summary && warp == K3_GROUP) {  // mean and max of every loss
        DD s = {0.0, 0.0};
        unsigned long long ab = 0, km = 0;
        for (int b = lane; b < (int)gridDim.x; b += 32) {
            const TailPartial pp = part[(int64_t)R * gridDim.x + b];
            dd_merge(s, DD{pp.hi, pp.lo});
            km = max(km, pp.pad);
        }
        dd_warp_reduce(s, ab);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) km = max(km, __shfl_xor_sync(0xffffffffu, km, o));
        if (lane == 0) {
            w->summary[0] = __ddiv_rn(__dadd_rn(s.hi, s.lo), (double)n);
            w->summary[1] = key_value(km);
        }
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
// result staging), serialised by a mutex.
struct K3Cache {
    std::mutex mu;
    K3Work *d_work = nullptr;
    TailPartial *d_part = nullptr;
    double *h_res = nullptr;  // pinned [2][K3_GROUP] + mean, max
    int grid = 0;
};
static K3Cache g_k3[64];

static K3Cache g_k3_async[64];  // the asynchronous entry's own workspace (one stream per device)

// One K3 launch (<= K3_GROUP return periods) on `st`: clear the work area,
// the cooperative select, no host synchronisation.
static int k3_launch(K3Cache &c, const double *d_x, int64_t n, const double *rps, int64_t n_rp, bool summary,
                     int sms, int max_ctas, cudaStream_t st) {
    constexpr size_t smem = sizeof(unsigned int) * K3_GROUP * K3_BINS;
    if (!c.d_work) {
        ARE_CUDA(cudaFuncSetAttribute(k3_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        ARE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_select, K3_THREADS, smem));
        if (per_sm < 1) return fail(ARE_ECUDA, "K3 does not fit on an SM");
        c.grid = sms * std::min(per_sm, 2);
        ARE_CUDA(cudaMalloc(&c.d_work, sizeof(K3Work)));
        ARE_CUDA(cudaMalloc(&c.d_part, sizeof(TailPartial) * (size_t)c.grid * (K3_GROUP + 1)));
        ARE_CUDA(cudaHostAlloc(&c.h_res, sizeof(double) * (2 * K3_GROUP + 2), cudaHostAllocDefault));
    }
    K3Params prm{};
    prm.n_rp = (int)n_rp;
    prm.summary = summary;
    for (int r = 0; r < prm.n_rp; ++r) {
        int64_t k;
        int rc = order_stat_k(n, rps[r], &k);
        if (rc) return rc;
        prm.rank[r] = k;
        prm.m_tail[r] = n - k + 1;
    }
    ARE_CUDA(cudaMemsetAsync(c.d_work, 0, offsetof(K3Work, res), st));
    int grid = (int)std::min<int64_t>(c.grid, (n + K3_THREADS - 1) / K3_THREADS);
    if (max_ctas > 0) grid = std::min(grid, max_ctas);
    grid = std::max(grid, 1);
    void *args[] = {(void *)&d_x, (void *)&n, (void *)&prm, (void *)&c.d_work, (void *)&c.d_part};
    ARE_CUDA(cudaLaunchCooperativeKernel((void *)k3_select, grid, K3_THREADS, args, smem, st));
    ARE_LAUNCHED();
    return ARE_OK;
}

int k3_order_stats(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                   double *tvar_out, int sms, cudaStream_t st, double *summary) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    if (n >= (int64_t)0xFFFFFFFFll) return fail(ARE_EINVAL, "year loss table too long for K3");
    int dev;
    ARE_CUDA(cudaGetDevice(&dev));
    K3Cache &c = g_k3[dev & 63];
    std::lock_guard<std::mutex> guard(c.mu);
    for (int64_t base = 0; base < std::max<int64_t>(n_rp, summary ? 1 : 0); base += K3_GROUP) {
        const int64_t nr = std::min<int64_t>(K3_GROUP, n_rp - base);
        int rc = k3_launch(c, d_x, n, rps + base, nr > 0 ? nr : 0, summary && base == 0, sms, 0, st);
        if (rc) return rc;
        ARE_CUDA(cudaMemcpyAsync(c.h_res, c.d_work->res, sizeof(double) * (2 * K3_GROUP + 2), cudaMemcpyDeviceToHost,
                                 st));
        ARE_CUDA(cudaStreamSynchronize(st));
        for (int r = 0; r < nr; ++r) {
            pml_out[base + r] = c.h_res[r];
            tvar_out[base + r] = c.h_res[K3_GROUP + r];
        }
        if (summary && base == 0) {
            summary[0] = c.h_res[2 * K3_GROUP];
            summary[1] = c.h_res[2 * K3_GROUP + 1];
        }
    }
    return ARE_OK;
}

int k3_order_stats_async(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *d_res, int sms,
                         int max_ctas, cudaStream_t st) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    if (n >= (int64_t)0xFFFFFFFFll) return fail(ARE_EINVAL, "year loss table too long for K3");
    if (n_rp < 1 || n_rp > K3_GROUP) return fail(ARE_EINVAL, "asynchronous K3 takes 1..8 return periods");
    if (!d_res) return fail(ARE_EINVAL, "null result buffer");
    int dev;
    ARE_CUDA(cudaGetDevice(&dev));
    K3Cache &c = g_k3_async[dev & 63];
    std::lock_guard<std::mutex> guard(c.mu);
    int rc = k3_launch(c, d_x, n, rps, n_rp, false, sms, max_ctas, st);
    if (rc) return rc;
    // pml at d_res[r], tvar at d_res[8 + r]: one device copy, stream-ordered
    ARE_CUDA(cudaMemcpyAsync(d_res, c.d_work->res, sizeof(double) * 2 * K3_GROUP, cudaMemcpyDeviceToDevice, st));
    return ARE_OK;
}

// ---- many return periods, PML only (ep_curve, metrics.py:97-115) --------
// The reference sorts the table once for an EP curve (metrics.py:110); so
// does this: the order-preserving keys (NaN last) are radix-sorted on the
// device and every requested rank is read from the sorted keys in one
// gather, where the select kernel would need ceil(n_rp / 8) launches.
__global__ void k3_keys(const double *__restrict__ x, int64_t n, uint64_t *__restrict__ keys) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = order_key(x[i]);
}
__global__ void k3_gather_ranks(const uint64_t *__restrict__ sorted, const int64_t *__restrict__ ranks, int n_rp,
                                double *__restrict__ out) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rp; r += gridDim.x * blockDim.x)
        out[r] = key_value(sorted[ranks[r] - 1]);
}

// Split keys for the two-pass EP sort: the high and low 32 bits of each
// order-preserving key; the pairs are sorted by the high half only (4 radix
// passes instead of 8), which orders every key except inside runs of equal
// high halves (losses within ~1e-6 of each other, or exactly equal).
__global__ void k3_keys_split(const double *__restrict__ x, int64_t n, uint32_t *__restrict__ hi,
                              uint32_t *__restrict__ lo) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = order_key(x[i]);
        hi[i] = (uint32_t)(k >> 32);
        lo[i] = (uint32_t)k;
    }
}
// One warp per requested rank: the run of equal high halves around it, then
// the rank's low half inside the run (all equal -- ties at a cap -- needs
// nothing more; a short run is resolved by counting; a run longer than
// K3_RUN_MAX sets *fallback and the host re-sorts the full 64-bit keys).
static constexpr int64_t K3_RUN_MAX = 256;
__global__ void k3_select_split(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo, int64_t n,
                                const int64_t *__restrict__ ranks, int n_rp, double *__restrict__ out,
                                unsigned int *__restrict__ fallback) {
    const int lane = threadIdx.x & 31;
    const int r = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (r >= n_rp) return;
    const int64_t k = ranks[r] - 1;  // 0-based position in sorted order
    const uint32_t h = hi[k];
    // a run of one (the usual case for distinct losses): no search
    if ((k == 0 || hi[k - 1] != h) && (k + 1 == n || hi[k + 1] != h)) {
        if (lane == 0) out[r] = key_value(((uint64_t)h << 32) | lo[k]);
        return;
    }
    // run [s, e) of high half h: binary searches (every lane the same)
    int64_t a = 0, b = k;
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (hi[m] < h) a = m + 1; else b = m;
    }
    const int64_t s = a;
    a = k + 1;
    b = n;
    while (a < b) {
        const int64_t m = (a + b) >> 1;
        if (hi[m] <= h) a = m + 1; else b = m;
    }
    const int64_t e = a, len = e - s;
    uint32_t lmin = 0xFFFFFFFFu, lmax = 0u;
    for (int64_t i = s + lane; i < e; i += 32) {
        lmin = min(lmin, lo[i]);
        lmax = max(lmax, lo[i]);
    }
    lmin = __reduce_min_sync(0xffffffffu, lmin);
    lmax = __reduce_max_sync(0xffffffffu, lmax);
    uint32_t want = lmin;
    if (lmin != lmax) {
        if (len > K3_RUN_MAX) {
            if (lane == 0) atomicOr(fallback, 1u);
            return;
        }
        // the low half with exactly (k - s) smaller ones before it in the run
        const int64_t target = k - s;
        want = 0xFFFFFFFFu;
        for (int64_t i = s + lane; i < e; i += 32) {
            const uint32_t v = lo[i];
            int64_t less = 0, leq = 0;
            for (int64_t j = s; j < e; ++j) {
                less += lo[j] < v;
                leq += lo[j] <= v;
            }
            if (less <= target && target < leq) want = v;
        }
        want = __reduce_min_sync(0xffffffffu, want);
    }
    if (lane == 0) out[r] = key_value(((uint64_t)h << 32) | want);
}

struct SortCache {
    std::mutex mu;
    int64_t cap = 0;         // keys
    uint64_t *d_keys = nullptr;  // [2 * cap]
    void *d_tmp = nullptr;
    size_t tmp_bytes = 0;
    int64_t rank_cap = 0;
    int64_t *d_ranks = nullptr;
    double *d_out = nullptr;
    int64_t *h_ranks = nullptr;  // pinned staging: the copies stay asynchronous
    double *h_out = nullptr;
};
static SortCache g_sort[64];

int k3_pml_sorted(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out, int sms,
                  cudaStream_t st) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    if (n_rp <= 0) return ARE_OK;
    std::vector<int64_t> ranks((size_t)n_rp);
    for (int64_t r = 0; r < n_rp; ++r) {
        int rc = order_stat_k(n, rps[r], &ranks[(size_t)r]);
        if (rc) return rc;
    }
    int dev;
    ARE_CUDA(cudaGetDevice(&dev));
    SortCache &c = g_sort[dev & 63];
    std::lock_guard<std::mutex> guard(c.mu);
    if (n > c.cap) {
        cudaFree(c.d_keys);
        cudaFree(c.d_tmp);
        c.d_keys = nullptr;
        c.d_tmp = nullptr;
        c.cap = 0;
        size_t tmp = 0, tmp2 = 0;
        ARE_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, (const uint64_t *)nullptr, (uint64_t *)nullptr, n));
        ARE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp2, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                 (const uint32_t *)nullptr, (uint32_t *)nullptr, n));
        tmp = std::max(tmp, tmp2);
        ARE_CUDA(cudaMalloc(&c.d_keys, sizeof(uint64_t) * 2 * (size_t)n));  // or 4 x n uint32 (split)
        ARE_CUDA(cudaMalloc(&c.d_tmp, tmp));
        c.tmp_bytes = tmp;
        c.cap = n;
    }
    if (n_rp > c.rank_cap) {
        cudaFree(c.d_ranks);
        cudaFree(c.d_out);
        cudaFreeHost(c.h_ranks);
        cudaFreeHost(c.h_out);
        c.d_ranks = nullptr;
        c.d_out = nullptr;
        c.h_ranks = nullptr;
        c.h_out = nullptr;
        c.rank_cap = 0;
        ARE_CUDA(cudaMalloc(&c.d_ranks, sizeof(int64_t) * (size_t)n_rp));
        ARE_CUDA(cudaMalloc(&c.d_out, sizeof(double) * (size_t)(n_rp + 1)));  // + the fallback flag
        ARE_CUDA(cudaHostAlloc(&c.h_ranks, sizeof(int64_t) * (size_t)n_rp, cudaHostAllocDefault));
        ARE_CUDA(cudaHostAlloc(&c.h_out, sizeof(double) * (size_t)(n_rp + 1), cudaHostAllocDefault));
        c.rank_cap = n_rp;
    }
    // every copy from/to pinned staging, the ranks first: nothing waits on the
    // host between the launches (a pageable copy would sync the stream first)
    std::memcpy(c.h_ranks, ranks.data(), sizeof(int64_t) * (size_t)n_rp);
    ARE_CUDA(cudaMemcpyAsync(c.d_ranks, c.h_ranks, sizeof(int64_t) * (size_t)n_rp, cudaMemcpyHostToDevice, st));
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8));
    size_t tmp = c.tmp_bytes;
    // split keys: sort (high half, low half) pairs by the high half
    uint32_t *hi_in = reinterpret_cast<uint32_t *>(c.d_keys), *lo_in = hi_in + c.cap;
    uint32_t *hi_out = lo_in + c.cap, *lo_out = hi_out + c.cap;
    ARE_CUDA(cudaMemsetAsync(c.d_out + n_rp, 0, sizeof(double), st));
    k3_keys_split<<<blocks, 256, 0, st>>>(d_x, n, hi_in, lo_in);
    ARE_LAUNCHED();
    ARE_CUDA(cub::DeviceRadixSort::SortPairs(c.d_tmp, tmp, hi_in, hi_out, lo_in, lo_out, n, 0, 32, st));
    k3_select_split<<<(int)((n_rp * 32 + 255) / 256), 256, 0, st>>>(
        hi_out, lo_out, n, c.d_ranks, (int)n_rp, c.d_out, reinterpret_cast<unsigned int *>(c.d_out + n_rp));
    ARE_LAUNCHED();
    ARE_CUDA(cudaMemcpyAsync(c.h_out, c.d_out, sizeof(double) * (size_t)(n_rp + 1), cudaMemcpyDeviceToHost, st));
    ARE_CUDA(cudaStreamSynchronize(st));
    if (c.h_out[n_rp] != 0.0) {  // a long run of near-equal losses: the full 64-bit sort
        tmp = c.tmp_bytes;
        k3_keys<<<blocks, 256, 0, st>>>(d_x, n, c.d_keys);
        ARE_LAUNCHED();
        ARE_CUDA(cub::DeviceRadixSort::SortKeys(c.d_tmp, tmp, c.d_keys, c.d_keys + c.cap, n, 0, 64, st));
        k3_gather_ranks<<<(int)std::min<int64_t>((n_rp + 255) / 256, 1024), 256, 0, st>>>(c.d_keys + c.cap,
                                                                                           c.d_ranks, (int)n_rp,
                                                                                           c.d_out);
        ARE_LAUNCHED();
        ARE_CUDA(cudaMemcpyAsync(c.h_out, c.d_out, sizeof(double) * (size_t)n_rp, cudaMemcpyDeviceToHost, st));
        ARE_CUDA(cudaStreamSynchronize(st));
    }
    std::memcpy(pml_out, c.h_out, sizeof(double) * (size_t)n_rp);
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
