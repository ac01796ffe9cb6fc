// K1-L + K2-L pre-combined -- the fused multi-layer pass over a per-event
// table of occurrence values (SURVEY.md §8(f) rows 2 and 4 together; a
// separately reported work unit, never the headline).
//
// For a layer set over one pool plan, an event's occurrence value in layer l
// depends only on the event (its non-zero pool entries, the financial terms,
// l's mask and occurrence terms), not on the trial.  K1-L evaluates it once
// per hot event and layer -- the same float64 sequence k2_layers (and the
// reference, per layer) uses: comb = 0.0 + f_j over the event's entries that
// l selects, in pool order; occ = clamp(comb - occR_l, 0, occL_l), or 0.0 when
// l sees none of them -- into occ[e][0..15] (one 128-byte line per event).
// K2-L-pre then streams the ids exactly like k2_layers (filter, in-order
// queue) and, per 32 queued events, gathers their lines and folds them
// lane-per-layer in trial order: lanes 0-15 take event 2p, lanes 16-31 event
// 2p+1, and lane l adds its own value then its partner's (shuffle).  Every
// layer's YLT is bit-identical to the per-layer kernels.
#include "k2_trials.cuh"

namespace are {

static constexpr int PQCAP = 128;  // per-warp queue (< 32 left + 2 rows of 32)

// ---- K1-L: occ[e * 16 + l] for every event with a non-zero pool entry ------
__global__ void k1_layer_occ(const Slot *__restrict__ slots, const Entry *__restrict__ ovf,
                             const Fin *__restrict__ fin, const uint64_t *__restrict__ masks,
                             const LayerTerm *__restrict__ terms, int n_layers, int64_t row_len,
                             double *__restrict__ occ) {
    __shared__ uint64_t s_mask[K2L_MAX_LAYERS];
    __shared__ double s_ret[K2L_MAX_LAYERS], s_lim[K2L_MAX_LAYERS];
    if (threadIdx.x < K2L_MAX_LAYERS) {
        const bool on = (int)threadIdx.x < n_layers;
        s_mask[threadIdx.x] = on ? masks[threadIdx.x] : 0ull;
        s_ret[threadIdx.x] = on ? terms[threadIdx.x].occ_ret : 0.0;
        s_lim[threadIdx.x] = on ? terms[threadIdx.x].occ_lim : 0.0;
    }
    __syncthreads();
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        const Slot s = slots[e];
        const uint32_t cnt = s.meta >> 16;
        if (!cnt) continue;  // the table is zero-filled: absent events read +0
        double v[K2L_MAX_LAYERS];
#pragma unroll
        for (int l = 0; l < K2L_MAX_LAYERS; ++l) v[l] = 0.0;
        uint32_t seen = 0;
        // entries in pool order: the inline first one, then the overflow
        for (uint32_t k = 0; k < cnt; ++k) {
            const uint32_t j = k ? ovf[s.ovf + k - 1].j : (s.meta & 0xFFFFu);
            const double x = k ? ovf[s.ovf + k - 1].x : s.x;
            const double f = fin_term(fin[j], x);
#pragma unroll
            for (int l = 0; l < K2L_MAX_LAYERS; ++l)
                if ((s_mask[l] >> j) & 1ull) {
                    v[l] = __dadd_rn(v[l], f);  // comb starts at 0.0 (v[l] = 0.0 + f first)
                    seen |= 1u << l;
                }
        }
        double *row = occ + e * K2L_MAX_LAYERS;
#pragma unroll
        for (int l = 0; l < K2L_MAX_LAYERS; ++l)
            row[l] = ((seen >> l) & 1u) ? clamp_ref(__dsub_rn(v[l], s_ret[l]), s_lim[l]) : 0.0;
    }
}

int k1_layer_occ_build(const K2Args &a, const K2Layers &L, double *d_occ, int sms, cudaStream_t st) {
    ARE_CUDA(cudaMemsetAsync(d_occ, 0, (size_t)a.row_len * K2L_MAX_LAYERS * sizeof(double), st));
    const int threads = 256;
    int64_t g = ((int64_t)a.row_len + threads - 1) / threads;
    if (g > (int64_t)sms * 8) g = (int64_t)sms * 8;
    k1_layer_occ<<<(unsigned)g, threads, 0, st>>>(a.slots, a.ovf, a.fin, L.masks, L.terms, L.n_layers,
                                                  (int64_t)a.row_len, d_occ);
    ARE_LAUNCHED();
    return ARE_OK;
}

// ---- K2-L pre-combined -------------------------------------------------------
template <int HASH>
__device__ __forceinline__ uint32_t p_hash(uint32_t e, uint32_t nbits) {
    if (HASH == 0) return e;
    if (HASH == 1) return min(e, e - nbits);
    return e % nbits;
}

template <int HASH, bool CHECK>
__global__ void __launch_bounds__(K2L_THREADS, 1) k2_layers_pre(const K2Args a, const K2Layers L) {
    constexpr int NW = K2L_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *s_q = reinterpret_cast<uint32_t *>(smem);  // [NW][PQCAP]
    uint32_t *s_filter = s_q + NW * PQCAP;
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int half = lane >> 4, ll = lane & 15;  // event parity in a pair, layer
    uint32_t *q = s_q + warp * PQCAP;
    const uint32_t q_saddr = (uint32_t)__cvta_generic_to_shared(q);
    const uint32_t lt = lanemask_lt();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t nbits = a.nbits, last_id = a.row_len - 1;
    const uint32_t *const ids = a.ids;
    const int64_t W = (int64_t)gridDim.x * NW;
    const int nl = L.n_layers;
    const uint32_t pad = cold_pad(s_filter, a.filter_words, nbits, a.row_len);  // out-of-trial lanes
    const double *const occ = L.occ_table + ll;  // this lane's layer column
    const double agg_ret = lane < nl ? L.terms[lane].agg_ret : 0.0;
    const double agg_lim = lane < nl ? L.terms[lane].agg_lim : 0.0;
    uint32_t emax = 0;

    // a batch of n <= 32 queued events: lane (half, l) loads occ[e_{2p+half}][l]
    // for p = 0..15 (events past n read event 0's line: all zero)
    auto gather = [&](uint32_t qh, uint32_t n, double (&v)[16]) {
        const uint32_t mine = (uint32_t)lane < n ? q[(qh + lane) & (PQCAP - 1)] : 0u;
        __syncwarp();  // the ring slot may be rewritten by another lane later
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            const uint32_t e = __shfl_sync(0xffffffffu, mine, 2 * p + half);
            v[p] = ld_nc_f64(occ + (int64_t)e * K2L_MAX_LAYERS, pol_keep);
        }
    };
    // lanes 0..15 fold events 2p (own value) then 2p+1 (the partner's); an
    // absent event adds +0.0, which leaves c unchanged (c is never -0)
    auto fold = [&](const double (&v)[16], double &c) {
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            const double w = __shfl_down_sync(0xffffffffu, v[p], 16);
            c = __dadd_rn(c, v[p]);
            c = __dadd_rn(c, w);
        }
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
        if (tn < a.last) {
            nlo = a.offsets[tn - a.t_base];
            nhi = a.offsets[tn - a.t_base + 1];
        }
        const int64_t rlo = lo - a.id_base;
        const uint32_t len = (uint32_t)(hi - lo);
        const uint32_t skew = (uint32_t)((reinterpret_cast<uintptr_t>(ids + rlo) >> 2) & 31);
        const uint32_t *p = ids + (rlo - skew) + lane;
        const uint32_t rel = (uint32_t)lane - skew;
        const int nchunks = (int)((len + skew + 127) >> 7);
        double c = 0.0;  // lane l < nl: layer l's trial sum
        uint32_t qh = 0, qt = 0;
        // two batch buffers used alternately (renaming, not copying: a copy
        // would wait for the loads in flight); `pend` = which one holds a
        // gathered, unfolded batch: 0 none, 1 va, 2 vb
        int pend = 0;
        double va[16], vb[16];

        uint32_t r0[4], r1[4], r2[4];
        auto issue = [&](uint32_t (&fut)[4], int chn) {
            const uint32_t *pc = p + ((int64_t)chn << 7);
            const uint32_t rc = rel + ((uint32_t)chn << 7);
#pragma unroll
            for (int k = 0; k < 4; ++k) fut[k] = ld_stream_if(pc + 32 * k, rc + 32 * k, len, pol_stream, pad);
        };
        auto filt = [&](const uint32_t (&cur)[4], uint32_t (&ev)[4], uint32_t (&hot)[4]) {
            uint32_t word[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t e = cur[k];
                if (CHECK) {
                    emax = max(emax, e);
                    e = min(e, last_id);
                }
                ev[k] = e;
                word[k] = s_filter[p_hash<HASH>(e, nbits) >> 5];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) hot[k] = (word[k] >> (p_hash<HASH>(ev[k], nbits) & 31)) & 1u;
        };
        issue(r0, 0);
        issue(r1, 1);
        int phase = 0;
        for (int ch = 0; ch < nchunks; ++ch) {
            uint32_t ev[4], hot[4];
            switch (phase) {
                case 0: issue(r2, ch + 2); filt(r0, ev, hot); break;
                case 1: issue(r0, ch + 2); filt(r1, ev, hot); break;
                default: issue(r1, ch + 2); filt(r2, ev, hot); break;
            }
            phase = phase == 2 ? 0 : phase + 1;
#pragma unroll 1
            for (int hf = 0; hf < 2; ++hf) {
                const uint32_t ea = hf ? ev[2] : ev[0], eb = hf ? ev[3] : ev[1];
                const uint32_t ha = hf ? hot[2] : hot[0], hb = hf ? hot[3] : hot[1];
                uint32_t b = ballot_full(ha);
                st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (PQCAP - 1)) << 2), ea, ha);
                qt += __popc(b);
                b = ballot_full(hb);
                st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (PQCAP - 1)) << 2), eb, hb);
                qt += __popc(b);
                __syncwarp();
                while (qt - qh >= 32u) {  // the next gather is in flight while a batch folds
                    if (pend != 1) {
                        gather(qh, 32u, va);
                        if (pend == 2) fold(vb, c);
                        pend = 1;
                    } else {
                        gather(qh, 32u, vb);
                        fold(va, c);
                        pend = 2;
                    }
                    qh += 32u;
                }
            }
        }
        {
            const uint32_t n = qt - qh;  // final partial batch
            if (pend != 1) {
                if (n) gather(qh, n, va);
                if (pend == 2) fold(vb, c);
                if (n) fold(va, c);
            } else {
                if (n) gather(qh, n, vb);
                fold(va, c);
                if (n) fold(vb, c);
            }
        }
        if (lane < nl) a.out[(int64_t)lane * L.out_stride + (t - a.out_base)] = clamp_ref(__dsub_rn(c, agg_ret), agg_lim);
        lo = nlo;
        hi = nhi;
    }
    if (CHECK && __any_sync(0xffffffffu, emax > last_id) && lane == 0) atomicOr(a.err, 1u);
}

size_t k2_layers_pre_smem(int64_t filter_words) {
    constexpr int NW = K2L_THREADS / 32;
    return (size_t)NW * PQCAP * sizeof(uint32_t) + (size_t)filter_words * sizeof(uint32_t);
}

template <int HASH, bool CHECK>
static int pre_prepare_one() {
    ARE_CUDA(cudaFuncSetAttribute(k2_layers_pre<HASH, CHECK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  k2_max_dynamic_smem()));
    return ARE_OK;
}

int k2_layers_pre_prepare() {
    int rc;
    if ((rc = pre_prepare_one<0, true>()) || (rc = pre_prepare_one<1, true>()) ||
        (rc = pre_prepare_one<2, true>()) || (rc = pre_prepare_one<0, false>()) ||
        (rc = pre_prepare_one<1, false>()) || (rc = pre_prepare_one<2, false>()))
        return rc;
    return ARE_OK;
}

int k2_layers_pre_launch(const K2Args &a, const K2Layers &L, bool check, int sms, cudaStream_t st) {
    if (a.last <= a.first) return ARE_OK;
    constexpr int NW = K2L_THREADS / 32;
    const int64_t trials = a.last - a.first;
    int64_t g = (trials + NW - 1) / NW;
    if (g > sms) g = sms;
    const dim3 grid((unsigned)g), block(K2L_THREADS);
    const size_t smem = k2_layers_pre_smem(a.filter_words);
    switch (a.hash_mode * 2 + (check ? 1 : 0)) {
        case 0: k2_layers_pre<0, false><<<grid, block, smem, st>>>(a, L); break;
        case 1: k2_layers_pre<0, true><<<grid, block, smem, st>>>(a, L); break;
        case 2: k2_layers_pre<1, false><<<grid, block, smem, st>>>(a, L); break;
        case 3: k2_layers_pre<1, true><<<grid, block, smem, st>>>(a, L); break;
        case 4: k2_layers_pre<2, false><<<grid, block, smem, st>>>(a, L); break;
        default: k2_layers_pre<2, true><<<grid, block, smem, st>>>(a, L); break;
    }
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
