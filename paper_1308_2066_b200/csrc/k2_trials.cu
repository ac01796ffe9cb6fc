// K2 -- fused per-trial simulation: YET id stream -> Year Loss Table.
//
// Replaces the reference hot loop run_trials (pkg/src/aggrisk/engine/
// _kernel.pyx:17-119).  For every trial t and every occurrence e in trial
// order the reference computes
//     comb = sum_j  share_j * clamp(rate_j * tab_j[e] - ret_j, 0, lim_j)
//     c   += clamp(comb - occ_ret, 0, occ_lim)
// and finally out[t] = clamp(c - agg_ret, 0, agg_lim).
//
// Hot-set kernel (k2_hotset): persistent, one CTA per SM, one warp per trial.
//   * the trial's uint32 ids stream in with coalesced 16-byte loads
//     (L1::no_allocate, L2 evict_first), one chunk of 128 occurrences per
//     warp step (4 per lane, lane-major = trial order), next chunk prefetched;
//   * a bit filter over event ids lives in shared memory (up to ~1.7M bits);
//     events whose bit is clear are absent from every selected table and
//     contribute exactly +-0, so they are
//     skipped;
//   * hot events are compacted, in trial order, into a per-warp queue and
//     processed 32 at a time, one per lane: one 16-byte L2 record read
//     (evict_last), the financial terms in selection order, the occurrence
//     terms;
//   * the trial total is accumulated SEQUENTIALLY in trial order in float64
//     (each occurrence value added once, in order), exactly like the
//     reference, so the YLT is bit-identical to the reference kernel; the
//     skipped +-0 additions cannot change a float64 sum.
// Dense kernel (k2_dense): the literal per-occurrence loop over every selected
//   row of the dense float64 tables; used when the zero-skip precondition
//   does not hold (invalid terms such as negative retentions) and as the
//   uncompacted comparison point.
#include "k2_trials.cuh"

namespace are {

static constexpr int QCAP = 256;  // per-warp hot queue (>= 31 + 128)

__device__ __forceinline__ uint32_t hot_hash(uint32_t e, uint32_t nbits, int mode) {
    if (mode == 0) return e;
    if (mode == 1) return e >= nbits ? e - nbits : e;
    return e % nbits;
}

__device__ __forceinline__ uint4 load_ids4(const uint32_t *ids, int64_t j, int64_t n_ids,
                                           int64_t rlo, int64_t rhi, uint64_t pol) {
    if (j >= 0 && j + 4 <= n_ids) return ld_stream_u4(ids + j, pol);
    uint32_t r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int64_t i = j + k;
        r[k] = (i >= rlo && i < rhi) ? ld_stream_u32(ids + i, pol) : 0u;
    }
    return make_uint4(r[0], r[1], r[2], r[3]);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k2_hotset(const K2Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    Fin *s_fin = reinterpret_cast<Fin *>(smem);
    double *s_occ = reinterpret_cast<double *>(smem + a.fin_bytes);
    uint32_t *s_q = reinterpret_cast<uint32_t *>(s_occ + NW * 32);
    uint32_t *s_filter = s_q + NW * QCAP;

    for (int i = threadIdx.x; i < a.n_sel; i += blockDim.x) s_fin[i] = a.fin[i];
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *ob = s_occ + warp * 32;
    uint32_t *q = s_q + warp * QCAP;
    const uint32_t lt = lanemask_lt();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const int64_t W = (int64_t)gridDim.x * NW;
    bool bad = false;

    // Process `n` queued hot events (uniform n <= 32), then fold their
    // occurrence values into c in queue (= trial) order.
    auto batch = [&](uint32_t qh, uint32_t n, double &c) {
        if ((uint32_t)lane < n) {
            const uint32_t e = q[(qh + lane) & (QCAP - 1)];
            const Slot s = ld_slot(a.slots + e, pol_keep);
            const uint32_t cnt = s.meta >> 16;
            double comb = 0.0;
            if (cnt) {
                comb = __dadd_rn(0.0, fin_term(s_fin[s.meta & 0xFFFFu], s.x));
                for (uint32_t i = 1; i < cnt; ++i) {
                    const Entry en = a.ovf[s.ovf + i - 1];
                    comb = __dadd_rn(comb, fin_term(s_fin[en.j], en.x));
                }
            }
            ob[lane] = clamp_ref(__dsub_rn(comb, a.occ_ret), a.occ_lim);
        }
        __syncwarp();
        if (n == 32) {
            const double2 *ob2 = reinterpret_cast<const double2 *>(ob);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const double2 p = ob2[i];
                c = __dadd_rn(c, p.x);
                c = __dadd_rn(c, p.y);
            }
        } else {
            for (uint32_t i = 0; i < n; ++i) c = __dadd_rn(c, ob[i]);
        }
        __syncwarp();
    };

    int64_t t = a.first + (int64_t)blockIdx.x * NW + warp;
    int64_t lo = 0, hi = 0;
    if (t < a.last) {
        lo = a.offsets[t - a.t_base];
        hi = a.offsets[t - a.t_base + 1];
    }
    for (; t < a.last; t += W) {
        const int64_t tn = t + W;
        int64_t nlo = 0, nhi = 0;
        if (tn < a.last) {  // next trial's bounds, in flight during this trial
            nlo = a.offsets[tn - a.t_base];
            nhi = a.offsets[tn - a.t_base + 1];
        }
        const int64_t rlo = lo - a.id_base, rhi = hi - a.id_base;
        const int64_t mis = (int64_t)((reinterpret_cast<uintptr_t>(a.ids + rlo) >> 2) & 3);
        const int64_t start = rlo - mis;
        const int len = (int)(rhi - rlo);
        double c = 0.0;
        uint32_t qh = 0, qt = 0;

        int64_t j = start + 4 * lane;
        uint4 v = load_ids4(a.ids, j, a.n_ids, rlo, rhi, pol_stream);
        for (int64_t base = start; base < rhi; base += 128) {
            uint4 vn = make_uint4(0u, 0u, 0u, 0u);
            if (base + 128 < rhi) vn = load_ids4(a.ids, j + 128, a.n_ids, rlo, rhi, pol_stream);

            const uint32_t ev[4] = {v.x, v.y, v.z, v.w};
            const int rel = (int)(j - rlo);
            uint32_t hot = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if ((unsigned)(rel + k) < (unsigned)len) {
                    const uint32_t e = ev[k];
                    if (e >= a.row_len) {
                        bad = true;
                    } else {
                        const uint32_t h = hot_hash(e, a.nbits, a.hash_mode);
                        hot |= ((s_filter[h >> 5] >> (h & 31)) & 1u) << k;
                    }
                }
            }
            // lane-major compaction keeps trial order: lane l's hot events
            // follow those of lanes < l
            const uint32_t cnt = __popc(hot);
            const uint32_t b0 = __ballot_sync(0xffffffffu, cnt & 1u);
            const uint32_t b1 = __ballot_sync(0xffffffffu, cnt & 2u);
            const uint32_t b2 = __ballot_sync(0xffffffffu, cnt & 4u);
            const uint32_t tot = __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
            if (tot) {
                uint32_t w = qt + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((hot >> k) & 1u) q[(w++) & (QCAP - 1)] = ev[k];
                qt += tot;
                __syncwarp();
                while (qt - qh >= 32u) {
                    batch(qh, 32u, c);
                    qh += 32u;
                }
            }
            v = vn;
            j += 128;
        }
        if (qt != qh) batch(qh, qt - qh, c);
        if (lane == 0) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
        lo = nlo;
        hi = nhi;
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, 1u);
}

// Literal reference loop: every occurrence, every selected row, in order.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k2_dense(const K2Args a) {
    __shared__ Fin s_fin[ARE_MAX_TABLES];
    __shared__ int64_t s_row[ARE_MAX_TABLES];
    __shared__ double s_occ[NW * 32];
    for (int i = threadIdx.x; i < a.n_sel; i += blockDim.x) {
        s_fin[i] = a.fin[i];
        s_row[i] = a.rows[i] * (int64_t)a.row_len;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *ob = s_occ + warp * 32;
    const uint64_t pol_stream = policy_evict_first();
    bool bad = false;
    for (int64_t t = a.first + (int64_t)blockIdx.x * NW + warp; t < a.last;
         t += (int64_t)gridDim.x * NW) {
        const int64_t rlo = a.offsets[t - a.t_base] - a.id_base;
        const int64_t rhi = a.offsets[t - a.t_base + 1] - a.id_base;
        double c = 0.0;
        for (int64_t base = rlo; base < rhi; base += 32) {
            const int64_t i = base + lane;
            if (i < rhi) {
                const uint32_t e = ld_stream_u32(a.ids + i, pol_stream);
                double comb = 0.0;
                if (e >= a.row_len) {
                    bad = true;
                } else {
                    for (int s = 0; s < a.n_sel; ++s)
                        comb = __dadd_rn(comb, fin_term(s_fin[s], a.stacked[s_row[s] + e]));
                }
                ob[lane] = clamp_ref(__dsub_rn(comb, a.occ_ret), a.occ_lim);
            }
            __syncwarp();
            const int n = (int)min((int64_t)32, rhi - base);
            for (int k = 0; k < n; ++k) c = __dadd_rn(c, ob[k]);
            __syncwarp();
        }
        if (lane == 0) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, 1u);
}

static constexpr int HOT_WARPS = 16;
static constexpr int DENSE_WARPS = 8;

size_t k2_hotset_fixed_smem(int n_sel) {
    return (size_t)n_sel * sizeof(Fin) + (size_t)HOT_WARPS * 32 * sizeof(double) +
           (size_t)HOT_WARPS * QCAP * sizeof(uint32_t);
}

int k2_prepare(int device) {
    (void)device;
    ARE_CUDA(cudaFuncSetAttribute(k2_hotset<HOT_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  k2_max_dynamic_smem()));
    return ARE_OK;
}

int k2_launch(const K2Args &a, int variant, int sms, size_t smem_bytes, cudaStream_t st) {
    if (a.last <= a.first) return ARE_OK;
    const int64_t trials = a.last - a.first;
    if (variant == ARE_VARIANT_DENSE) {
        int64_t g = (trials + DENSE_WARPS - 1) / DENSE_WARPS;
        const int64_t cap = (int64_t)sms * 8;
        k2_dense<DENSE_WARPS><<<(unsigned)(g < cap ? g : cap), DENSE_WARPS * 32, 0, st>>>(a);
        ARE_LAUNCHED();
        return ARE_OK;
    }
    int64_t g = (trials + HOT_WARPS - 1) / HOT_WARPS;
    if (g > sms) g = sms;  // persistent: one CTA per SM (the filter fills shared memory)
    k2_hotset<HOT_WARPS><<<(unsigned)g, HOT_WARPS * 32, smem_bytes, st>>>(a);
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
