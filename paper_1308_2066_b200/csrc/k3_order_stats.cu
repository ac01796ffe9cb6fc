// K3 -- order statistics over a Year Loss Table: PML, TVaR, EP points, and
// the per-trial portfolio roll-up.
//
// Replaces pkg/src/aggrisk/metrics.py:29-133.  PML at return period rp is
// the k-th smallest loss with k = n - floor(n / rp) (metrics.py:29-42,
// computed on the host in the same float64 arithmetic); TVaR is the mean of
// the closed tail, the top m = n - k + 1 order statistics (metrics.py:55-63).
//
// Device algorithm: MSD radix select on the order-preserving 64-bit key of
// each float64 (NaN last, like np.partition), 8 passes of 8 bits, all return
// periods of a call selected together (one 256-bin histogram per rp and
// pass, shared-memory atomics then one global add per bin).  The tail sum is
// then  S = sum of losses strictly above the PML key  (double-double
// accumulation, fixed grid, partials combined in a fixed order, so the
// result is bit-reproducible run to run and for any GPU count) plus
// (m - G) copies of the PML value itself (G = count strictly above):
//     tvar = (S + (m - G) * pml) / m.
// This equals the mean of the closed tail for any ties; it is within a few
// ulp of numpy's pairwise mean (tolerance in tests/test_metrics_gpu.py).
#include "k3_order_stats.cuh"

#include <cmath>
#include <vector>

namespace are {

static constexpr int K3_MAX_RP = 32;
static constexpr int K3_THREADS = 256;

struct SelectState {
    uint64_t prefix[K3_MAX_RP];
    uint64_t rank[K3_MAX_RP];  // 1-based rank still to find inside the prefix bucket
};

__global__ void k3_hist(const double *__restrict__ x, int64_t n, const SelectState *__restrict__ st,
                        int n_rp, int shift, unsigned int *__restrict__ hist) {
    extern __shared__ unsigned int sh[];
    for (int i = threadIdx.x; i < n_rp * 256; i += blockDim.x) sh[i] = 0;
    __shared__ uint64_t pre[K3_MAX_RP];
    for (int r = threadIdx.x; r < n_rp; r += blockDim.x) pre[r] = st->prefix[r];
    __syncthreads();
    const uint64_t hi_mask = shift >= 56 ? 0ull : (~0ull << (shift + 8));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = order_key(x[i]);
        const unsigned d = (unsigned)(k >> shift) & 255u;
        for (int r = 0; r < n_rp; ++r)
            if (((k ^ pre[r]) & hi_mask) == 0) atomicAdd(&sh[r * 256 + d], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_rp * 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// One thread per return period: walk the 256 bins, fix the next digit.
__global__ void k3_pick(SelectState *__restrict__ st, int n_rp, int shift, unsigned int *__restrict__ hist) {
    const int r = threadIdx.x;
    if (r < n_rp) {
        uint64_t want = st->rank[r], run = 0;
        unsigned d = 0;
        for (; d < 255; ++d) {
            const uint64_t h = hist[r * 256 + d];
            if (run + h >= want) break;
            run += h;
        }
        st->rank[r] = want - run;
        st->prefix[r] |= (uint64_t)d << shift;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n_rp * 256; i += blockDim.x) hist[i] = 0;
}

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

// blockIdx.y = return period; fixed grid-stride assignment -> deterministic.
__global__ void k3_tail(const double *__restrict__ x, int64_t n, const SelectState *__restrict__ st,
                        TailPartial *__restrict__ part) {
    const int r = blockIdx.y;
    const uint64_t kp = st->prefix[r];
    DD acc = {0.0, 0.0};
    unsigned long long above = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (order_key(v) > kp) {
            dd_add(acc, v);
            ++above;
        }
    }
    __shared__ double shi[K3_THREADS], slo[K3_THREADS];
    __shared__ unsigned long long sab[K3_THREADS];
    shi[threadIdx.x] = acc.hi;
    slo[threadIdx.x] = acc.lo;
    sab[threadIdx.x] = above;
    __syncthreads();
    if (threadIdx.x == 0) {  // fixed-order block combine
        DD b = {0.0, 0.0};
        unsigned long long ab = 0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
            dd_add(b, shi[i]);
            b.lo = __dadd_rn(b.lo, slo[i]);
            ab += sab[i];
        }
        TailPartial p;
        p.hi = b.hi;
        p.lo = b.lo;
        p.above = ab;
        p.pad = 0;
        part[(int64_t)r * gridDim.x + blockIdx.x] = p;
    }
}

__global__ void k3_final(const SelectState *__restrict__ st, const TailPartial *__restrict__ part,
                         int nblocks, int n_rp, const int64_t *__restrict__ m_tail,
                         double *__restrict__ res /* [2][n_rp]: pml, tvar */) {
    const int r = threadIdx.x;
    if (r >= n_rp) return;
    DD s = {0.0, 0.0};
    unsigned long long above = 0;
    for (int b = 0; b < nblocks; ++b) {
        const TailPartial p = part[(int64_t)r * nblocks + b];
        dd_add(s, p.hi);
        s.lo = __dadd_rn(s.lo, p.lo);
        above += p.above;
    }
    const double pml = key_value(st->prefix[r]);
    const int64_t m = m_tail[r];
    const double copies = (double)(m - (int64_t)above);
    double total;
    const double prod = __dmul_rn(copies, pml);
    if (isfinite(prod) && isfinite(s.hi)) {
        const double perr = fma(copies, pml, -prod);  // exact product error
        dd_add(s, prod);
        s.lo = __dadd_rn(s.lo, perr);
        total = __dadd_rn(s.hi, s.lo);
    } else {
        total = __dadd_rn(__dadd_rn(s.hi, s.lo), prod);
    }
    res[r] = pml;
    res[n_rp + r] = __ddiv_rn(total, (double)m);
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

int k3_order_stats(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                   double *tvar_out, int sms, cudaStream_t st) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    if (n >= (int64_t)0xFFFFFFFFll) return fail(ARE_EINVAL, "year loss table too long for K3");
    for (int64_t base = 0; base < n_rp; base += K3_MAX_RP) {
        const int R = (int)std::min<int64_t>(K3_MAX_RP, n_rp - base);
        SelectState hs;
        std::vector<int64_t> m(R);
        for (int r = 0; r < R; ++r) {
            int64_t k;
            int rc = order_stat_k(n, rps[base + r], &k);
            if (rc) return rc;
            hs.prefix[r] = 0;
            hs.rank[r] = (uint64_t)k;
            m[r] = n - k + 1;
        }
        const int hist_blocks = (int)std::min<int64_t>((n + K3_THREADS - 1) / K3_THREADS, (int64_t)sms * 2);
        const int tail_blocks = hist_blocks;
        SelectState *d_st = nullptr;
        unsigned int *d_hist = nullptr;
        TailPartial *d_part = nullptr;
        int64_t *d_m = nullptr;
        double *d_res = nullptr;
        ARE_CUDA(cudaMallocAsync(&d_st, sizeof(SelectState), st));
        ARE_CUDA(cudaMallocAsync(&d_hist, sizeof(unsigned int) * 256 * R, st));
        ARE_CUDA(cudaMallocAsync(&d_part, sizeof(TailPartial) * tail_blocks * R, st));
        ARE_CUDA(cudaMallocAsync(&d_m, sizeof(int64_t) * R, st));
        ARE_CUDA(cudaMallocAsync(&d_res, sizeof(double) * 2 * R, st));
        ARE_CUDA(cudaMemcpyAsync(d_st, &hs, sizeof(SelectState), cudaMemcpyHostToDevice, st));
        ARE_CUDA(cudaMemcpyAsync(d_m, m.data(), sizeof(int64_t) * R, cudaMemcpyHostToDevice, st));
        ARE_CUDA(cudaMemsetAsync(d_hist, 0, sizeof(unsigned int) * 256 * R, st));
        for (int shift = 56; shift >= 0; shift -= 8) {
            k3_hist<<<hist_blocks, K3_THREADS, sizeof(unsigned int) * 256 * R, st>>>(d_x, n, d_st, R, shift, d_hist);
            ARE_LAUNCHED();
            k3_pick<<<1, 256, 0, st>>>(d_st, R, shift, d_hist);
            ARE_LAUNCHED();
        }
        k3_tail<<<dim3(tail_blocks, R), K3_THREADS, 0, st>>>(d_x, n, d_st, d_part);
        ARE_LAUNCHED();
        k3_final<<<1, 32 * ((R + 31) / 32), 0, st>>>(d_st, d_part, tail_blocks, R, d_m, d_res);
        ARE_LAUNCHED();
        std::vector<double> res(2 * R);
        ARE_CUDA(cudaMemcpyAsync(res.data(), d_res, sizeof(double) * 2 * R, cudaMemcpyDeviceToHost, st));
        cudaFreeAsync(d_st, st);
        cudaFreeAsync(d_hist, st);
        cudaFreeAsync(d_part, st);
        cudaFreeAsync(d_m, st);
        cudaFreeAsync(d_res, st);
        ARE_CUDA(cudaStreamSynchronize(st));
        for (int r = 0; r < R; ++r) {
            pml_out[base + r] = res[r];
            tvar_out[base + r] = res[R + r];
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
