// K0 -- device-side validation of a Year Event Table.
//
// Replaces the YET half of validate_portfolio (reference
// pkg/src/aggrisk/model.py:371-395), which costs ~9 s per 1M x 1000 YET in
// numpy on the host: trial lengths in [1, max_len], event ids in [1, catalog],
// timestamps in [0, 1] and non-decreasing inside each trial.  One pass over
// the ids (min/max), one over the offsets, and one warp per trial over the
// timestamps; the host turns the counters into the reference's Violation
// report (categories and messages unchanged).
#include "common.cuh"

namespace are {

static constexpr int K0_THREADS = 256;

__device__ __forceinline__ uint64_t ts_key(double v) {  // order-preserving
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

struct K0Acc {
    unsigned int min_id, max_id;
    unsigned long long bad_trials, first_bad, unsorted, ts_min_key, ts_max_key, ts_nan;
};

__global__ void k0_ids(const uint32_t *__restrict__ ids, int64_t n, K0Acc *acc) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t e = ids[i];
        lo = min(lo, e);
        hi = max(hi, e);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&acc->min_id, lo);
        atomicMax(&acc->max_id, hi);
    }
}

__global__ void k0_trials(const int64_t *__restrict__ offsets, int64_t n_trials, int64_t t_base, int64_t max_len,
                          K0Acc *acc) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_trials;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = offsets[t + 1] - offsets[t];
        if (len < 1 || len > max_len) {
            atomicAdd(&acc->bad_trials, 1ull);
            atomicMin(&acc->first_bad, (unsigned long long)(t + t_base));
        }
    }
}

// one warp per trial: range of every timestamp, drops strictly inside trials
__global__ void k0_timestamps(const double *__restrict__ ts, int64_t ts_base, const int64_t *__restrict__ offsets,
                              int64_t n_trials, K0Acc *acc) {
    const int lane = threadIdx.x & 31;
    uint64_t kmin = ~0ull, kmax = 0;
    unsigned long long drops = 0, nans = 0;
    for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < n_trials;
         t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t lo = offsets[t] - ts_base, hi = offsets[t + 1] - ts_base;
        for (int64_t i = lo + lane; i < hi; i += 32) {
            const double v = ts[i];
            if (v != v) {
                ++nans;
            } else {
                const uint64_t k = ts_key(v);
                kmin = min(kmin, k);
                kmax = max(kmax, k);
            }
            if (i > lo && v < ts[i - 1]) ++drops;  // NaN compares false, as in numpy
        }
    }
    for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, (uint64_t)__shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, (uint64_t)__shfl_xor_sync(0xffffffffu, kmax, o));
        drops += __shfl_xor_sync(0xffffffffu, drops, o);
        nans += __shfl_xor_sync(0xffffffffu, nans, o);
    }
    if (lane == 0) {
        atomicMin(&acc->ts_min_key, (unsigned long long)kmin);
        atomicMax(&acc->ts_max_key, (unsigned long long)kmax);
        if (drops) atomicAdd(&acc->unsorted, drops);
        if (nans) atomicAdd(&acc->ts_nan, nans);
    }
}

static double key_to_double(uint64_t k) {
    const uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    double v;
    std::memcpy(&v, &b, sizeof v);
    return v;
}

}  // namespace are

using namespace are;

extern "C" int are_validate_yet_device(const uint32_t *d_ids, int64_t n_ids, const int64_t *d_offsets,
                                       int64_t n_trials, int64_t t_base, const double *d_ts, int64_t ts_base,
                                       int64_t max_len, are_yet_report_t *out, void *stream) {
    if (!out || n_ids < 0 || n_trials < 0) return fail(ARE_EINVAL, "bad validation arguments");
    cudaStream_t st = (cudaStream_t)stream;
    int dev, sms = 0;
    ARE_CUDA(cudaGetDevice(&dev));
    ARE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    K0Acc h{0xFFFFFFFFu, 0u, 0ull, ~0ull, 0ull, ~0ull, 0ull, 0ull};
    K0Acc *d = nullptr;
    ARE_CUDA(cudaMallocAsync(&d, sizeof(K0Acc), st));
    ARE_CUDA(cudaMemcpyAsync(d, &h, sizeof h, cudaMemcpyHostToDevice, st));
    const unsigned grid = (unsigned)std::max(1, sms * 4);
    if (n_ids > 0) {
        k0_ids<<<grid, K0_THREADS, 0, st>>>(d_ids, n_ids, d);
        ARE_LAUNCHED();
    }
    if (n_trials > 0) {
        k0_trials<<<grid, K0_THREADS, 0, st>>>(d_offsets, n_trials, t_base, max_len, d);
        ARE_LAUNCHED();
        if (d_ts) {
            k0_timestamps<<<grid, K0_THREADS, 0, st>>>(d_ts, ts_base, d_offsets, n_trials, d);
            ARE_LAUNCHED();
        }
    }
    ARE_CUDA(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    cudaFreeAsync(d, st);
    ARE_CUDA(cudaStreamSynchronize(st));
    out->min_id = h.min_id;
    out->max_id = h.max_id;
    out->bad_trials = (int64_t)h.bad_trials;
    out->first_bad_trial = h.bad_trials ? (int64_t)h.first_bad : -1;
    out->unsorted = (int64_t)h.unsorted;
    out->ts_nan = (int64_t)h.ts_nan;
    out->ts_checked = d_ts ? 1 : 0;
    out->ts_min = h.ts_min_key == ~0ull ? 0.0 : key_to_double(h.ts_min_key);
    out->ts_max = h.ts_max_key == 0ull ? 0.0 : key_to_double(h.ts_max_key);
    return ARE_OK;
}
