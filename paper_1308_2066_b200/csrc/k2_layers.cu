// K2-L -- fused multi-layer simulation: one pass over the YET for L layers.
//
// SURVEY.md §8(f) row 2.  The reference runs layers as a sequential outer loop
// (engine/__init__.py:242-253), re-reading the whole event stream per layer.
// Here a layer set whose ELTs come from one pool of P <= 64 tables shares a
// single hot-set plan over the pool (selection = the pool in pool order) and a
// single pass over the ids: the filter flags events present in ANY pool table,
// and each flagged event is evaluated for every layer.
//
// Exactness per layer: layer l's selection must be increasing in pool order
// (checked on the host), so summing the event's non-zero pool entries that are
// in l's bitmask, in pool order, is exactly l's `comb` (zero entries add +-0);
// events absent from l contribute +-0 to l's trial sum; every layer's trial sum
// is folded strictly in trial order.  So each layer's YLT is bit-identical to
// running K2 (and the reference) on that layer alone.
//
// Work mapping (warp per trial, like k2_hotset): queued events are served in
// sub-batches of 8.  Lane (i = lane % 8, g = lane / 8) gathers event i's record
// and evaluates layers g, g+4, g+8, ... for it, writing occ[i][l] to shared
// memory; then lane l (< L) folds occ[0..n)[l] into its own register c_l.  The
// fold is therefore lane-parallel across layers instead of warp-redundant.
// When every event of a sub-batch sits in at most two pool tables (~99% at
// C3) a warp-uniform fast path replaces the general per-layer loop: per pool
// table a word of the layers that contain it, the event's three possible
// combs (first table only, second only, both -- in pool order), layer terms
// in registers.  The row buffers rotate through a phase switch so the append
// and drain code (which inlines the evaluation) exists once: six inlined
// copies thrashed the instruction cache.
#include "k2_trials.cuh"

namespace are {

static constexpr int LQCAP = 128;   // per-warp queue of event ids

// A gathered LRec as loaded: four doubles (the last holds meta | ovf << 32).
struct LRecRaw {
    double fa, fb, x0, mo;
};
static constexpr int LSUB = 8;      // events per sub-batch
static constexpr int LPL = K2L_MAX_LAYERS / 4;  // evaluation layers per lane

template <int HASH>
__device__ __forceinline__ uint32_t l_hash(uint32_t e, uint32_t nbits) {
    if (HASH == 0) return e;
    if (HASH == 1) return min(e, e - nbits);
    return e % nbits;
}

// Evaluate one event (record `s`) for layers sg, sg+4, ... and store each
// layer's occurrence value at out[l].  Kept out of line: the kernel calls it
// from several unrolled sites and an inlined copy each would thrash the
// instruction cache.
__device__ __noinline__ void layer_eval(const Slot s, const Entry *__restrict__ ovf, const Fin *s_fin,
                                        const uint64_t *s_mask, const double *s_occ_ret, const double *s_occ_lim,
                                        int nl, int sg, double *out) {
    // non-zero pool entries of the event in pool order (first inline, the
    // rest in the overflow array); financial terms applied once per entry
    const uint32_t cnt = s.meta >> 16;
    double f[4];
    uint32_t jj[4];
    uint64_t em = 0;  // pool tables the event appears in
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f[k] = 0.0;
        jj[k] = 0;
    }
    if (cnt) {
        jj[0] = s.meta & 0xFFFFu;
        f[0] = fin_term(s_fin[jj[0]], s.x);
        em = 1ull << jj[0];
    }
#pragma unroll 1
    for (uint32_t k = 1; k < cnt && k < 4; ++k) {
        const Entry en = ovf[s.ovf + k - 1];
        jj[k] = en.j;
        f[k] = fin_term(s_fin[en.j], en.x);
        em |= 1ull << en.j;
    }
#pragma unroll 1
    for (uint32_t k = 4; k < cnt; ++k) em |= 1ull << ovf[s.ovf + k - 1].j;
#pragma unroll 1
    for (int l = sg; l < nl; l += 4) {
        const uint64_t m = s_mask[l];
        double o = 0.0;  // layer does not see the event: occ(+0) = +-0, adds nothing
        if (em & m) {
            double comb = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if ((uint32_t)k < cnt && ((m >> jj[k]) & 1ull)) comb = __dadd_rn(comb, f[k]);
#pragma unroll 1
            for (uint32_t k = 4; k < cnt; ++k) {  // events in > 4 pool tables (rare)
                const Entry en = ovf[s.ovf + k - 1];
                if ((m >> en.j) & 1ull) comb = __dadd_rn(comb, fin_term(s_fin[en.j], en.x));
            }
            o = clamp_ref(__dsub_rn(comb, s_occ_ret[l]), s_occ_lim[l]);
        }
        out[l] = o;
    }
}

template <int HASH, bool CHECK>
__global__ void __launch_bounds__(K2L_THREADS, 1) k2_layers(const K2Args a, const K2Layers L) {
    constexpr int NW = K2L_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    Fin *s_fin = reinterpret_cast<Fin *>(smem);
    uint64_t *s_mask = reinterpret_cast<uint64_t *>(smem + a.fin_bytes);  // per layer
    double *s_occ_ret = reinterpret_cast<double *>(s_mask + K2L_MAX_LAYERS);
    double *s_occ_lim = s_occ_ret + K2L_MAX_LAYERS;
    uint32_t *s_lbits = reinterpret_cast<uint32_t *>(s_occ_lim + K2L_MAX_LAYERS);  // [K2L_MAX_POOL]
    double *s_occ = reinterpret_cast<double *>(s_lbits + K2L_MAX_POOL);  // [NW][LSUB][K2L_MAX_LAYERS]
    uint32_t *s_q = reinterpret_cast<uint32_t *>(s_occ + NW * LSUB * K2L_MAX_LAYERS);  // [NW][LQCAP]
    uint32_t *s_filter = s_q + NW * LQCAP;

    for (int i = threadIdx.x; i < a.n_sel; i += blockDim.x) s_fin[i] = a.fin[i];
    for (int i = threadIdx.x; i < L.n_layers; i += blockDim.x) {
        s_mask[i] = L.masks[i];
        s_occ_ret[i] = L.terms[i].occ_ret;
        s_occ_lim[i] = L.terms[i].occ_lim;
    }
    for (int j = threadIdx.x; j < K2L_MAX_POOL; j += blockDim.x) {
        uint32_t b = 0;
        for (int l = 0; l < L.n_layers; ++l) b |= (uint32_t)((L.masks[l] >> j) & 1ull) << l;
        s_lbits[j] = b;
    }
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int si = lane & (LSUB - 1), sg = lane >> 3;  // sub-batch event, layer group
    double *occ = s_occ + warp * LSUB * K2L_MAX_LAYERS;  // occ[i * K2L_MAX_LAYERS + l]
    uint32_t *q = s_q + warp * LQCAP;
    const uint32_t q_saddr = (uint32_t)__cvta_generic_to_shared(q);
    const uint32_t lt = lanemask_lt();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t nbits = a.nbits, last_id = a.row_len - 1;
    const uint32_t *const ids = a.ids;
    const int64_t W = (int64_t)gridDim.x * NW;
    const int nl = L.n_layers;
    const uint32_t pad = cold_pad(s_filter, a.filter_words, nbits, a.row_len);  // out-of-trial lanes
    // this lane's fold layer (lane < nl)
    const double agg_ret = lane < nl ? L.terms[lane].agg_ret : 0.0;
    const double agg_lim = lane < nl ? L.terms[lane].agg_lim : 0.0;
    uint32_t emax = 0;
    // this lane's evaluation layers sg, sg + 4, ... (constants in registers)
    double lret[LPL], llim[LPL];
#pragma unroll
    for (int r = 0; r < LPL; ++r) {
        const int l = sg + 4 * r;
        lret[r] = l < nl ? s_occ_ret[l] : 0.0;
        llim[r] = l < nl ? s_occ_lim[l] : 0.0;
    }

    // one 32-byte record per event (k1_layer_records: the first two entries'
    // financial terms already applied), kept as loaded; lanes past the
    // sub-batch read the always-empty record 0 (an unconditional load: a
    // predicated one would be waited on at once)
    auto gather = [&](uint32_t qh, uint32_t n) -> LRecRaw {
        const uint32_t e = (uint32_t)si < n ? q[(qh + si) & (LQCAP - 1)] : 0u;
        LRecRaw r;
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                     : "=d"(r.fa), "=d"(r.fb), "=d"(r.x0), "=d"(r.mo)
                     : "l"(L.lrec + e), "l"(pol_keep));
        return r;
    };
    // Evaluate a gathered sub-batch of n <= 8 events and fold it per layer.
    // Fast path (warp-uniform): every event of the sub-batch sits in at most
    // two pool tables (~99% of events at C3), so a layer's comb is
    // 0.0 + [j0 in l] f0 + [j1 in l] f1 in pool order (an absent term adds
    // +0.0 to a comb that is never -0: bit-identical to layer_eval).
    auto finish = [&](const LRecRaw &s, uint32_t n, double &c) {
        const uint32_t meta = (uint32_t)__double2loint(s.mo);
        const uint32_t cnt = (uint32_t)si < n ? (meta >> 16) : 0u;
        if (__all_sync(0xffffffffu, cnt <= 2u)) {
            // the three possible combs (layer sees j0 only, j1 only, both)
            // and, per entry, the layers that see it (bit 4r <-> layer sg + 4r)
            double c10 = 0.0, c01 = 0.0, c11 = 0.0;
            uint32_t m0 = 0, m1 = 0;
            if (cnt) {
                c10 = s.fa;  // 0.0 + f_{j0}(x0), taken by K1
                c11 = c10;
                m0 = s_lbits[meta & 0xFFu] >> sg;
            }
            if (cnt == 2u) {
                c01 = __dadd_rn(0.0, s.fb);
                c11 = __dadd_rn(c10, s.fb);
                m1 = s_lbits[(meta >> 8) & 0xFFu] >> sg;
            }
            double *o = occ + si * K2L_MAX_LAYERS;
#pragma unroll
            for (int r = 0; r < LPL; ++r) {
                const int l = sg + 4 * r;
                if (l < nl && (uint32_t)si < n) {
                    const bool b0 = (m0 >> (4 * r)) & 1u, b1 = (m1 >> (4 * r)) & 1u;
                    const double comb = b0 ? (b1 ? c11 : c10) : c01;
                    const double v = clamp_ref(__dsub_rn(comb, lret[r]), llim[r]);
                    o[l] = (b0 || b1) ? v : 0.0;
                }
            }
        } else if ((uint32_t)si < n) {
            const Slot sl{s.x0, (meta & 0xFFu) | (cnt << 16), (uint32_t)__double2hiint(s.mo)};
            layer_eval(sl, a.ovf, s_fin, s_mask, s_occ_ret, s_occ_lim, nl, sg, occ + si * K2L_MAX_LAYERS);
        }
        __syncwarp();
        if (lane < nl) {
            if (n == (uint32_t)LSUB) {  // full sub-batch: all loads first, then the in-order chain
                double v[LSUB];
#pragma unroll
                for (int i = 0; i < LSUB; ++i) v[i] = occ[i * K2L_MAX_LAYERS + lane];
#pragma unroll
                for (int i = 0; i < LSUB; ++i) c = __dadd_rn(c, v[i]);
            } else {
                for (uint32_t i = 0; i < n; ++i) c = __dadd_rn(c, occ[i * K2L_MAX_LAYERS + lane]);
            }
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
        if (tn < a.last) {
            nlo = a.offsets[tn - a.t_base];
            nhi = a.offsets[tn - a.t_base + 1];
        }
        const int64_t rlo = lo - a.id_base;
        const uint32_t len = (uint32_t)(hi - lo);
        const uint32_t skew = (uint32_t)((reinterpret_cast<uintptr_t>(ids + rlo) >> 2) & 31);
        const uint32_t *p = ids + (rlo - skew) + lane;
        uint32_t rel = (uint32_t)lane - skew;
        const int nchunks = (int)((len + skew + 127) >> 7);
        double c = 0.0;  // this lane's layer sum
        uint32_t qh = 0, qt = 0;
        bool pending = false;  // a gathered sub-batch not yet evaluated
        LRecRaw ps{0.0, 0.0, 0.0, 0.0};

        // three row buffers rotate by renaming (chunk ch + 2 loads while ch is
        // filtered); the switch keeps one copy of the append/drain code
        // (inlined once per call site, the drain would thrash the i-cache)
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
                word[k] = s_filter[l_hash<HASH>(e, nbits) >> 5];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) hot[k] = (word[k] >> (l_hash<HASH>(ev[k], nbits) & 31)) & 1u;
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
            for (int half = 0; half < 2; ++half) {
                const uint32_t ea = half ? ev[2] : ev[0], eb = half ? ev[3] : ev[1];
                const uint32_t ha = half ? hot[2] : hot[0], hb = half ? hot[3] : hot[1];
                uint32_t b = ballot_full(ha);
                st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (LQCAP - 1)) << 2), ea, ha);
                qt += __popc(b);
                b = ballot_full(hb);
                st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (LQCAP - 1)) << 2), eb, hb);
                qt += __popc(b);
                __syncwarp();
                while (qt - qh >= (uint32_t)LSUB) {
                    const LRecRaw ns = gather(qh, LSUB);  // in flight while the previous one finishes
                    if (pending) finish(ps, LSUB, c);
                    ps = ns;
                    pending = true;
                    qh += LSUB;
                }
            }
        }
        {
            const uint32_t n = qt - qh;
            const LRecRaw ns = gather(qh, n);
            if (pending) finish(ps, LSUB, c);
            if (n) finish(ns, n, c);
        }
        if (lane < nl) a.out[(int64_t)lane * L.out_stride + (t - a.out_base)] = clamp_ref(__dsub_rn(c, agg_ret), agg_lim);
        lo = nlo;
        hi = nhi;
    }
    if (CHECK && __any_sync(0xffffffffu, emax > last_id) && lane == 0) atomicOr(a.err, 1u);
}

size_t k2_layers_fixed_smem(int n_sel) {
    constexpr int NW = K2L_THREADS / 32;
    return (size_t)n_sel * sizeof(Fin) + 3 * K2L_MAX_LAYERS * sizeof(double) + K2L_MAX_POOL * sizeof(uint32_t) +
           (size_t)NW * LSUB * K2L_MAX_LAYERS * sizeof(double) +
           (size_t)NW * LQCAP * sizeof(uint32_t);
}

template <int HASH, bool CHECK>
static int layers_prepare_one() {
    ARE_CUDA(cudaFuncSetAttribute(k2_layers<HASH, CHECK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  k2_max_dynamic_smem()));
    return ARE_OK;
}

int k2_layers_prepare() {
    int rc;
    if ((rc = layers_prepare_one<0, true>()) || (rc = layers_prepare_one<1, true>()) ||
        (rc = layers_prepare_one<2, true>()) || (rc = layers_prepare_one<0, false>()) ||
        (rc = layers_prepare_one<1, false>()) || (rc = layers_prepare_one<2, false>()))
        return rc;
    return ARE_OK;
}

int k2_layers_launch(const K2Args &a, const K2Layers &L, bool check, int sms, size_t smem_bytes, cudaStream_t st) {
    if (a.last <= a.first) return ARE_OK;
    constexpr int NW = K2L_THREADS / 32;
    const int64_t trials = a.last - a.first;
    int64_t g = (trials + NW - 1) / NW;
    if (g > sms) g = sms;
    const dim3 grid((unsigned)g), block(K2L_THREADS);
    switch (a.hash_mode * 2 + (check ? 1 : 0)) {
        case 0: k2_layers<0, false><<<grid, block, smem_bytes, st>>>(a, L); break;
        case 1: k2_layers<0, true><<<grid, block, smem_bytes, st>>>(a, L); break;
        case 2: k2_layers<1, false><<<grid, block, smem_bytes, st>>>(a, L); break;
        case 3: k2_layers<1, true><<<grid, block, smem_bytes, st>>>(a, L); break;
        case 4: k2_layers<2, false><<<grid, block, smem_bytes, st>>>(a, L); break;
        default: k2_layers<2, true><<<grid, block, smem_bytes, st>>>(a, L); break;
    }
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
