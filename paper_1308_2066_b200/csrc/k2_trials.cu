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
//   * the trial's uint32 ids stream in as coalesced 128-byte rows (one id per
//     lane; L1::no_allocate, L2 evict_first), one chunk of 4 rows = 128
//     occurrences per warp step, two chunks in flight;
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
// Dense kernels (k2_dense, k2_dense_coop): the literal per-occurrence loop over
//   every selected row of the dense float64 tables; used when the zero-skip
//   precondition does not hold (invalid terms such as negative retentions),
//   for dense-overlap plans (several table entries per catalog event), and as
//   the uncompacted comparison point.  From 4 selected rows they read an
//   event-major copy, eight lanes per event line (k2_dense_coop).
#include "k2_trials.cuh"

namespace are {

static constexpr int QCAP = 128;  // per-warp hot queue: < 32 pending + 2 rows of 32
// Build-time variants of k2_hotset (A/B experiments; the defaults are the
// measured choice).
#ifndef ARE_K2_FIN_SOA
#define ARE_K2_FIN_SOA 1      // financial terms as four shared arrays
#endif
#ifndef ARE_K2_VRING
#define ARE_K2_VRING 0        // fold only non-zero values, from a per-warp ring (measured slower)
#endif
#ifndef ARE_K2_FILTER_FIRST
#define ARE_K2_FILTER_FIRST 1 // the filter at shared offset 0
#endif
#ifndef ARE_K2_FOLD_LANE0
#define ARE_K2_FOLD_LANE0 1   // fold on lane 0 only
#endif
#ifndef ARE_K2_INTERIOR
#define ARE_K2_INTERIOR 1     // unpredicated id loads for chunks inside the trial
#endif
#ifndef ARE_K2_L2PF
#define ARE_K2_L2PF 4         // bulk L2 prefetch of the id chunk this many chunks ahead (0: off)
#endif
#if ARE_K2_FIN_SOA
#define FIN_TERM(j, x) fin_term_soa(s_fs, nsel, (j), (x))
#else
#define FIN_TERM(j, x) fin_term(reinterpret_cast<const Fin *>(s_fs)[(j)], (x))
#endif
// per-warp value buffer: the ring of non-zero occurrence values (< 32
// unfolded + one batch), or one batch of values when the ring is off
static constexpr int VRING = ARE_K2_VRING ? 64 : 32;

// Event id -> filter bit.  HASH 0: the filter covers the catalog (exact);
// 1: catalog <= 2 * nbits, fold once (min picks e - nbits iff e >= nbits,
// the unsigned subtraction wraps otherwise); 2: general modulo.
template <int HASH>
__device__ __forceinline__ uint32_t hot_hash(uint32_t e, uint32_t nbits) {
    if (HASH == 0) return e;
    if (HASH == 1) return min(e, e - nbits);
    return e % nbits;
}

// Persistent hot-set kernel.  Each warp owns trials first + gw, first + gw +
// W, ...; a trial's ids are read as 32-id coalesced rows (row k of a 128-id
// chunk is ids [base + 32k, base + 32k + 32), lane l takes one id), two chunks
// kept in flight.  Filter hits are appended, in trial order, to the warp's
// queue; every 32 queued events form one batch: lane i gathers the record of
// the i-th event, applies the financial and occurrence terms, and the warp
// folds the occurrence values into c strictly in order.
// CHECK = false when the caller has validated every id <= catalog (the
// reference's validate_portfolio, or DeviceYearEventTable's upload check).
template <int HASH, bool CHECK, bool PRE>
__global__ void __launch_bounds__(K2_THREADS, 1) k2_hotset(const K2Args a) {
    constexpr int NW = K2_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
#if ARE_K2_FILTER_FIRST
    // the filter at offset 0 (its LDS addresses need no base register); the
    // queues, value buffers and terms after it
    uint32_t *s_filter = reinterpret_cast<uint32_t *>(smem);
    uint32_t *s_q = s_filter + a.filter_words;
    double *s_val = reinterpret_cast<double *>(s_q + NW * QCAP);           // per-warp value buffers
    double *s_fs = s_val + NW * VRING;                                     // financial terms
#else
    double *s_fs = reinterpret_cast<double *>(smem);                      // financial terms
    double *s_val = reinterpret_cast<double *>(smem + a.fin_bytes);        // per-warp value buffers
    uint32_t *s_q = reinterpret_cast<uint32_t *>(s_val + NW * VRING);
    uint32_t *s_filter = s_q + NW * QCAP;
#endif

#if ARE_K2_FIN_SOA
    fin_soa_store(s_fs, a.n_sel, a.fin);
#else
    for (int i = threadIdx.x; i < a.n_sel; i += blockDim.x) reinterpret_cast<Fin *>(s_fs)[i] = a.fin[i];
#endif
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nsel = a.n_sel;
    double *vr = s_val + warp * VRING;
    uint32_t *q = s_q + warp * QCAP;
    const uint32_t q_saddr = (uint32_t)__cvta_generic_to_shared(q);
    const uint32_t lt = lanemask_lt();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t nbits = a.nbits, last_id = a.row_len - 1;
    const double occ_ret = a.occ_ret, occ_lim = a.occ_lim;
    const uint32_t *const ids = a.ids;
    const int64_t W = (int64_t)gridDim.x * NW;
    uint32_t emax = 0;  // largest id seen: ids > catalog are reported, not read
    const uint32_t pad = cold_pad(s_filter, a.filter_words, nbits, a.row_len);

    // A batch is 32 queued events, one per lane.  It runs in two halves so
    // the record gathers of batch j are in flight while batch j-1 is finished
    // (terms, then its non-zero occurrence values appended in order to the
    // warp's value ring) and while the next rows are filtered.  The ring is
    // folded into c strictly in order, 32 values at a time: a value that is
    // +-0 is never appended (c >= +0, so adding it is an exact no-op), which
    // skips the ~45% of queued events that are filter false positives or fall
    // below the occurrence retention.
    uint32_t vh = 0, vt = 0;  // value ring head / tail (uniform); vh % 32 == 0
    auto finish = [&](const Slot &s, uint32_t n, double &c) {
        double v = 0.0;
        if ((uint32_t)lane < n) {
            const uint32_t cnt = s.meta >> 16;
            double comb = 0.0;
            if (PRE) {  // pre-combined plan: x already holds comb
                if (cnt) comb = s.x;
            } else {
                if (cnt) comb = __dadd_rn(0.0, FIN_TERM(s.meta & 0xFFFFu, s.x));
#pragma unroll 1
                for (uint32_t i = 1; i < cnt; ++i) {  // events in several tables (~7%)
                    const Entry en = a.ovf[s.ovf + i - 1];
                    comb = __dadd_rn(comb, FIN_TERM(en.j, en.x));
                }
            }
            v = clamp_ref(__dsub_rn(comb, occ_ret), occ_lim);
        }
#if !ARE_K2_VRING
        // every value of the batch in order (zeros included), as the reference adds them
        vr[lane] = v;
        __syncwarp();
#if ARE_K2_FOLD_LANE0
        // only lane 0 needs c (it writes the trial's result): a one-lane
        // LDS.128 is one shared-memory wavefront, a 32-lane broadcast two
        if (lane == 0)
#endif
        {
            if (n == 32) {
                const double2 *r2 = reinterpret_cast<const double2 *>(vr);
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const double2 w = r2[i];
                    c = __dadd_rn(c, w.x);
                    c = __dadd_rn(c, w.y);
                }
            } else {
                for (uint32_t i = 0; i < n; ++i) c = __dadd_rn(c, vr[i]);
            }
        }
        __syncwarp();
        return;
#endif
        const bool keep = !(v == 0.0);  // NaN is kept, +-0 skipped
        const uint32_t b = ballot_full(keep);
        if (keep) vr[(vt + __popc(b & lt)) & (VRING - 1)] = v;
        vt += __popc(b);
        __syncwarp();
        if (vt - vh >= 32u) {
            const double2 *r2 = reinterpret_cast<const double2 *>(vr + (vh & (VRING - 1)));
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const double2 w = r2[i];
                c = __dadd_rn(c, w.x);
                c = __dadd_rn(c, w.y);
            }
            vh += 32u;
            __syncwarp();
        }
    };
    auto gather = [&](uint32_t qh, uint32_t n) -> Slot {
        Slot s{0.0, 0u, 0u};
        if ((uint32_t)lane < n) s = ld_slot(a.slots + q[(qh + lane) & (QCAP - 1)], pol_keep);
        return s;
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
        const int64_t rlo = lo - a.id_base;
        const uint32_t len = (uint32_t)(hi - lo);
        // rows start on a 128-byte line; `rel` (lane's id index minus the
        // trial start) wraps for the lanes before the trial, so one unsigned
        // compare bounds both ends
        const uint32_t skew = (uint32_t)((reinterpret_cast<uintptr_t>(ids + rlo) >> 2) & 31);
        const uint32_t *p = ids + (rlo - skew) + lane;
        uint32_t rel = (uint32_t)lane - skew;
        const int nchunks = (int)((len + skew + 127) >> 7);
        double c = 0.0;
        uint32_t qh = 0, qt = 0;
        vh = 0;
        vt = 0;
        bool pending = false;  // a gathered, unfinished batch (uniform)
        Slot ps{0.0, 0u, 0u};

        // three row buffers rotate by renaming (a register move would wait
        // for the in-flight load it copies): chunk s+2 loads while s is used
        uint32_t r0[4], r1[4], r2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r0[k] = ld_stream_if(p + 32 * k, rel + 32 * k, len, pol_stream, pad);
#pragma unroll
        for (int k = 0; k < 4; ++k) r1[k] = ld_stream_if(p + 128 + 32 * k, rel + 128 + 32 * k, len, pol_stream, pad);

        auto step = [&](uint32_t (&cur)[4], uint32_t (&fut)[4]) {
#if ARE_K2_L2PF
            // the chunk ARE_K2_L2PF ahead goes to L2 now (one bulk request by
            // lane 0), so its row loads two chunks from now hit L2, not DRAM
            if (lane == 0) {
                const uint32_t ahead = rel - (uint32_t)lane + 128u * ARE_K2_L2PF;  // relative start of that chunk
                if ((int32_t)ahead < (int32_t)len) prefetch_l2_bulk(p - lane + 128 * ARE_K2_L2PF, 512);
            }
#endif
#if ARE_K2_INTERIOR
            // a chunk wholly inside the trial loads without predicates (uniform test)
            const uint32_t rel0 = rel - (uint32_t)lane + 256u;  // chunk start relative to the trial
            if ((int32_t)rel0 >= 0 && rel0 + 128u <= len) {
#pragma unroll
                for (int k = 0; k < 4; ++k) fut[k] = ld_stream_u32(p + 256 + 32 * k, pol_stream);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) fut[k] = ld_stream_if(p + 256 + 32 * k, rel + 256 + 32 * k, len, pol_stream, pad);
            }
#else
#pragma unroll
            for (int k = 0; k < 4; ++k) fut[k] = ld_stream_if(p + 256 + 32 * k, rel + 256 + 32 * k, len, pol_stream, pad);
#endif
            // filter words for all four rows first (independent shared loads)
            uint32_t ev[4], word[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // out-of-trial lanes read `pad`, an id whose bit is clear
                uint32_t e = cur[k];
                if (CHECK) {
                    emax = max(emax, e);
                    e = min(e, last_id);
                }
                ev[k] = e;
                word[k] = s_filter[hot_hash<HASH>(e, nbits) >> 5];
            }
#pragma unroll
            for (int half = 0; half < 2; ++half) {
#pragma unroll
                for (int k = 2 * half; k < 2 * half + 2; ++k) {
                    const bool hot = (word[k] >> (hot_hash<HASH>(ev[k], nbits) & 31)) & 1u;
                    const uint32_t b = ballot_full(hot);
                    st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (QCAP - 1)) << 2), ev[k], hot);
                    qt += __popc(b);
                }
                __syncwarp();
                while (qt - qh >= 32u) {
                    const Slot ns = gather(qh, 32u);
                    if (pending) finish(ps, 32u, c);
                    ps = ns;
                    pending = true;
                    qh += 32u;
                }
            }
            p += 128;
            rel += 128;
        };
        for (int ch = 0; ch < nchunks; ch += 3) {
            step(r0, r2);
            if (ch + 1 >= nchunks) break;
            step(r1, r0);
            if (ch + 2 >= nchunks) break;
            step(r2, r1);
        }
        const uint32_t n = qt - qh;  // final partial batch
        const Slot ns = gather(qh, n);
        if (pending) finish(ps, 32u, c);
        if (n) finish(ns, n, c);
#if ARE_K2_VRING
        {  // the ring's last (< 32) values, in order
            const uint32_t m = vt - vh;
            const double *r = vr + (vh & (VRING - 1));
            uint32_t i = 0;
            for (; i + 1 < m; i += 2) {
                const double2 w = *reinterpret_cast<const double2 *>(r + i);
                c = __dadd_rn(c, w.x);
                c = __dadd_rn(c, w.y);
            }
            if (i < m) c = __dadd_rn(c, r[i]);
            __syncwarp();
        }
#endif
        if (lane == 0) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
        lo = nlo;
        hi = nhi;
    }
    if (CHECK && __any_sync(0xffffffffu, emax > last_id) && lane == 0) atomicOr(a.err, 1u);
}

// ---------------------------------------------------------------------------
// Paired hot-set kernel (k2_pair): two trials per warp, one per half-warp.
// Each lane holds its own half's trial (pointers, counters, running sum), so
// the per-lane state is that of k2_hotset; per step a half filters 4 rows of
// 16 ids (64 ids of its trial) and appends hits to its own 64-entry queue
// (one ballot serves both halves).  A batch takes up to 16 queued events per
// half; lanes past a half's count carry +0.0, so every fold is the unrolled
// 16-value one (8 LDS.128 + 16 DADD) and advances BOTH trials' chains -- half
// the fold instructions of k2_hotset -- and the per-trial setup and final
// flush are shared by the pair.  The float64 sequence per trial is unchanged.
static constexpr int PH_CAP = 64;  // per-half queue: < 16 pending + 2 rows of 16

// REC: the launch gathers the relay records (RSlot, k1_relay_slots: the
// financial terms applied per entry, the first two entries inline) under the
// relay's per-occurrence-terms filter, instead of the hot-set slots.
template <int HASH, bool CHECK, bool PRE, bool REC = false>
__global__ void __launch_bounds__(K2_THREADS, 1) k2_pair(const K2Args a) {
    constexpr int NW = K2_THREADS / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    double *s_fs = reinterpret_cast<double *>(smem);  // financial terms, SoA
    double *s_occ = reinterpret_cast<double *>(smem + a.fin_bytes);
    uint32_t *s_q = reinterpret_cast<uint32_t *>(s_occ + NW * VRING);  // the hot-set kernel's layout
    uint32_t *s_filter = s_q + NW * QCAP;

    fin_soa_store(s_fs, a.n_sel, a.fin);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nsel = a.n_sel;
    const int half = lane >> 4, idx = lane & 15;
    const uint32_t hm = half ? 0xFFFF0000u : 0x0000FFFFu;
    const uint32_t lth = lanemask_lt() & hm;
    double *ob = s_occ + warp * 32 + half * 16;  // this half's 16 values
    const double2 *ob2 = reinterpret_cast<const double2 *>(ob);
    uint32_t *q = s_q + warp * QCAP + half * PH_CAP;
    const uint32_t q_saddr = (uint32_t)__cvta_generic_to_shared(q);
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t nbits = a.nbits, last_id = a.row_len - 1;
    const double occ_ret = a.occ_ret, occ_lim = a.occ_lim;
    const uint32_t *const ids = a.ids;
    const int64_t WP = (int64_t)gridDim.x * NW;  // pairs in flight
    uint32_t emax = 0;
    const uint32_t pad = cold_pad(s_filter, a.filter_words, nbits, a.row_len);

    // this half's next batch entry (record of the idx-th queued event); the
    // ring slot just read may be rewritten by another lane's later append
    auto gather = [&](uint32_t qh, uint32_t n) -> Slot {
        uint32_t ev = 0;
        if ((uint32_t)idx < n) ev = q[(qh + idx) & (PH_CAP - 1)];
        __syncwarp();
        Slot s{0.0, 0u, 0u};
        if (REC) {  // the 16-byte relay record, read as a Slot (x = a, meta|ovf = b)
            if ((uint32_t)idx < n) s = ld_slot(reinterpret_cast<const Slot *>(a.rslots + ev), pol_keep);
        } else if ((uint32_t)idx < n) {
            s = ld_slot(a.slots + ev, pol_keep);
        }
        return s;
    };
    auto finish = [&](const Slot &s, uint32_t n, double &c) {
        double v = 0.0;  // lanes past this half's count add +0 (exact: c is never -0)
        if ((uint32_t)idx < n) {
            const uint32_t cnt = s.meta >> 16;
            double comb = 0.0;
            if (REC) {
                const double ra = s.x, rb = __hiloint2double((int)s.ovf, (int)s.meta);
                if (!rslot_complex(ra)) {
                    comb = __dadd_rn(ra, rb);
                } else {
                    comb = rb;
                    const uint32_t rc = rslot_cnt(ra), ro = rslot_ovf(ra);
#pragma unroll 1
                    for (uint32_t i = 1; i < rc; ++i) comb = __dadd_rn(comb, a.rovf[ro + i - 1]);
                }
            } else if (PRE) {
                if (cnt) comb = s.x;
            } else {
                if (cnt) comb = __dadd_rn(0.0, fin_term_soa(s_fs, nsel, s.meta & 0xFFFFu, s.x));
#pragma unroll 1
                for (uint32_t i = 1; i < cnt; ++i) {
                    const Entry en = a.ovf[s.ovf + i - 1];
                    comb = __dadd_rn(comb, fin_term_soa(s_fs, nsel, en.j, en.x));
                }
            }
            v = clamp_ref(__dsub_rn(comb, occ_ret), occ_lim);
        }
        ob[idx] = v;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double2 w = ob2[i];
            c = __dadd_rn(c, w.x);
            c = __dadd_rn(c, w.y);
        }
        __syncwarp();
    };

    int64_t pr = (int64_t)blockIdx.x * NW + warp;  // pair index
    const int64_t npairs = (a.last - a.first + 1) / 2;
    int64_t lo = 0, hi = 0;
    {
        const int64_t t = a.first + 2 * pr + half;
        if (pr < npairs && t < a.last) {
            lo = a.offsets[t - a.t_base];
            hi = a.offsets[t - a.t_base + 1];
        }
    }
    for (; pr < npairs; pr += WP) {
        const int64_t t = a.first + 2 * pr + half;
        const int64_t tn = t + 2 * WP;
        int64_t nlo = 0, nhi = 0;
        if (pr + WP < npairs && tn < a.last) {  // next pair's bounds, in flight
            nlo = a.offsets[tn - a.t_base];
            nhi = a.offsets[tn - a.t_base + 1];
        }
        const int64_t rlo = lo - a.id_base;
        const uint32_t len = (uint32_t)(hi - lo);
        // this half's rows start on a 64-byte boundary; `rel` wraps before
        // the trial start so one unsigned compare bounds both ends
        const uint32_t skew = (uint32_t)((reinterpret_cast<uintptr_t>(ids + rlo) >> 2) & 15);
        const uint32_t *p = ids + (rlo - skew) + idx;
        uint32_t rel = (uint32_t)idx - skew;
        const int mych = len ? (int)((len + skew + 63) >> 6) : 0;
        const int nchunks = __reduce_max_sync(0xffffffffu, (uint32_t)mych);
        double c = 0.0;
        uint32_t qh = 0, qt = 0;
        bool pending = false;
        Slot ps{0.0, 0u, 0u};
        uint32_t pn = 0;  // this half's count in the pending batch

        // full batches while both halves hold 16; a half past 32 forces one
        // (capacity: 2 more rows add <= 32 to a 64-entry queue); need = 1
        // flushes everything at the end of the pair
        auto drain = [&](uint32_t need) {
            while (need == 1u ? __any_sync(0xffffffffu, qt != qh)
                              : (__all_sync(0xffffffffu, qt - qh >= 16u) || __any_sync(0xffffffffu, qt - qh > 32u))) {
                const uint32_t n = min(qt - qh, 16u);
                const Slot ns = gather(qh, n);
                if (pending) finish(ps, pn, c);
                ps = ns;
                pn = n;
                pending = true;
                qh += n;
            }
        };

        uint32_t r0[4], r1[4], r2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r0[k] = ld_stream_if(p + 16 * k, rel + 16 * k, len, pol_stream, pad);
#pragma unroll
        for (int k = 0; k < 4; ++k) r1[k] = ld_stream_if(p + 64 + 16 * k, rel + 64 + 16 * k, len, pol_stream, pad);

        auto step = [&](uint32_t (&cur)[4], uint32_t (&fut)[4]) {
#pragma unroll
            for (int k = 0; k < 4; ++k) fut[k] = ld_stream_if(p + 128 + 16 * k, rel + 128 + 16 * k, len, pol_stream, pad);
            uint32_t ev[4], word[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t e = cur[k];
                if (CHECK) {
                    emax = max(emax, e);
                    e = min(e, last_id);
                }
                ev[k] = e;
                word[k] = s_filter[hot_hash<HASH>(e, nbits) >> 5];
            }
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
                for (int k = 2 * hf; k < 2 * hf + 2; ++k) {
                    const bool hot = (word[k] >> (hot_hash<HASH>(ev[k], nbits) & 31)) & 1u;
                    const uint32_t b = ballot_full(hot);
                    st_shared_if(q_saddr + (((qt + __popc(b & lth)) & (PH_CAP - 1)) << 2), ev[k], hot);
                    qt += __popc(b & hm);
                }
                __syncwarp();
                drain(16u);
            }
            p += 64;
            rel += 64;
        };
        for (int ch = 0; ch < nchunks; ch += 3) {
            step(r0, r2);
            if (ch + 1 >= nchunks) break;
            step(r1, r0);
            if (ch + 2 >= nchunks) break;
            step(r2, r1);
        }
        drain(1u);  // whatever either half still holds
        if (pending) finish(ps, pn, c);
        if (idx == 0 && t < a.last) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
        lo = nlo;
        hi = nhi;
    }
    if (CHECK && __any_sync(0xffffffffu, emax > last_id) && lane == 0) atomicOr(a.err, 1u);
}

// Literal reference loop: every occurrence, every selected row, in order.
// EM: read the occurrence's selected losses from the event-major copy (one
// 128-byte-aligned line per event when n_sel <= 16) instead of n_sel rows.
// At most 64 registers (4 CTAs of 256 threads per SM), one resident wave;
// the next row's ids load while the current row's lines are in flight.
static constexpr int DENSE_CTAS_PER_SM = 4;
template <int NW, bool EM>
__global__ void __launch_bounds__(NW * 32, DENSE_CTAS_PER_SM) k2_dense(const K2Args a) {
    __shared__ Fin s_fin[ARE_MAX_TABLES];
    __shared__ int64_t s_row[ARE_MAX_TABLES];
    __shared__ __align__(16) double s_occ[NW * 32];
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
        uint32_t e_next = rlo + lane < rhi ? ld_stream_u32(a.ids + rlo + lane, pol_stream) : 0u;
        for (int64_t base = rlo; base < rhi; base += 32) {
            const int64_t i = base + lane;
            const uint32_t e = e_next;
            if (i + 32 < rhi) e_next = ld_stream_u32(a.ids + i + 32, pol_stream);
            if (i < rhi) {
                double comb = 0.0;
                if (e >= a.row_len) {
                    bad = true;
                } else if (EM) {
                    // the whole line in flight at once (<= 16 tables: one
                    // 128-byte line), then the terms in selection order
                    const double2 *line = reinterpret_cast<const double2 *>(a.em + (int64_t)e * a.em_stride);
                    for (int s0 = 0; s0 < a.n_sel; s0 += 16) {
                        double2 v[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if (s0 + 2 * k < a.n_sel) v[k] = line[(s0 >> 1) + k];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const int s = s0 + 2 * k;
                            if (s < a.n_sel) comb = __dadd_rn(comb, fin_term(s_fin[s], v[k].x));
                            if (s + 1 < a.n_sel) comb = __dadd_rn(comb, fin_term(s_fin[s + 1], v[k].y));
                        }
                    }
                } else {
                    for (int s = 0; s < a.n_sel; ++s)
                        comb = __dadd_rn(comb, fin_term(s_fin[s], a.stacked[s_row[s] + e]));
                }
                ob[lane] = clamp_ref(__dsub_rn(comb, a.occ_ret), a.occ_lim);
            }
            __syncwarp();
            const int n = (int)min((int64_t)32, rhi - base);
            if (n == 32) {
                const double2 *ob2 = reinterpret_cast<const double2 *>(ob);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double2 w = ob2[k];
                    c = __dadd_rn(c, w.x);
                    c = __dadd_rn(c, w.y);
                }
            } else {
                for (int k = 0; k < n; ++k) c = __dadd_rn(c, ob[k]);
            }
            __syncwarp();
        }
        if (lane == 0) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, 1u);
}

// Dense kernel over the event-major copy with cooperative line loads: eight
// lanes read one event's 128-byte line (one 16-byte load each), so one warp
// load brings four events' lines, where k2_dense<EM> has every lane load its
// own event's line in eight 16-byte pieces (random 128-byte lines from a
// 256 MB table, scripts/micro/rand_lines.cu: 9.2 vs 4.6 TB/s).  Each lane
// applies the financial terms of its two slots of the line; the values pass
// through shared memory so that the event's own lane adds them in selection
// order -- the reference's comb sequence, bit for bit.  Rows of FS = stride
// + 2 doubles keep the per-event 16-byte reads conflict-free.
static constexpr int COOP_CTAS_PER_SM = 3;  // 85 registers: the eight lines per lane in flight without spills
// FULL: the stride is exactly 16 * PASSES (15-16 or 31-32 selected rows), so
// the line shape is a compile-time constant.
template <int NW, int PASSES, bool FULL>
__global__ void __launch_bounds__(NW * 32, COOP_CTAS_PER_SM) k2_dense_coop(const K2Args a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int S2 = FULL ? 8 * PASSES : a.em_stride >> 1;  // 16-byte pieces per event
    const int FS = 2 * S2 + 2;
    Fin *s_fin = reinterpret_cast<Fin *>(smem);
    double *s_occ = reinterpret_cast<double *>(s_fin + 16 * PASSES);
    double *s_f = s_occ + NW * 32;
    for (int i = threadIdx.x; i < 16 * PASSES; i += blockDim.x) s_fin[i] = i < a.n_sel ? a.fin[i] : Fin{0.0, 0.0, 0.0, 0.0};
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = lane & 7, sub = lane >> 3;  // piece of the line, event within a group of four
    double *ob = s_occ + warp * 32;
    double *fw = s_f + (size_t)warp * 32 * FS;  // fw[event of the row * FS + slot]
    const double2 *em2 = reinterpret_cast<const double2 *>(a.em);
    const uint64_t pol_stream = policy_evict_first();
    const Fin fa = s_fin[2 * k], fb = s_fin[2 * k + 1];  // this lane's slots in pass 0
    const int n_sel = a.n_sel;
    bool bad = false;
    for (int64_t t = a.first + (int64_t)blockIdx.x * NW + warp; t < a.last;
         t += (int64_t)gridDim.x * NW) {
        const int64_t rlo = a.offsets[t - a.t_base] - a.id_base;
        const int64_t rhi = a.offsets[t - a.t_base + 1] - a.id_base;
        double c = 0.0;
        uint32_t e_next = rlo + lane < rhi ? ld_stream_u32(a.ids + rlo + lane, pol_stream) : 0u;
        for (int64_t base = rlo; base < rhi; base += 32) {
            const int64_t i = base + lane;
            uint32_t e = e_next;
            if (i + 32 < rhi) e_next = ld_stream_u32(a.ids + i + 32, pol_stream);
            const bool own = i < rhi;
            const bool ebad = own && e >= a.row_len;
            bad |= ebad;
            if (!own || ebad) e = 0;  // row 0 of the copy: a valid address, result unused
#pragma unroll
            for (int p = 0; p < PASSES; ++p) {
                const int kk = k + 8 * p;
                double2 v[8];
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint32_t eg = __shfl_sync(0xffffffffu, e, 4 * g + sub);
                    if (FULL) {
                        v[g] = __ldg(em2 + (size_t)eg * S2 + kk);
                    } else {
                        v[g] = make_double2(0.0, 0.0);
                        if (kk < S2) v[g] = __ldg(em2 + (size_t)eg * S2 + kk);
                    }
                }
                const Fin &f0 = p == 0 ? fa : s_fin[2 * kk];
                const Fin &f1 = p == 0 ? fb : s_fin[2 * kk + 1];
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    if (FULL || kk < S2) {
                        const double2 f = make_double2(fin_term(f0, v[g].x), fin_term(f1, v[g].y));
                        *reinterpret_cast<double2 *>(fw + (4 * g + sub) * FS + 2 * kk) = f;
                    }
                }
            }
            __syncwarp();
            if (own) {
                const double *row = fw + lane * FS;
                double comb = 0.0;
                if (FULL) {  // n_sel is 2 * S2 - 1 or 2 * S2
                    const double2 *row2 = reinterpret_cast<const double2 *>(row);
#pragma unroll
                    for (int q = 0; q < S2 - 1; ++q) {
                        const double2 w = row2[q];
                        comb = __dadd_rn(comb, w.x);
                        comb = __dadd_rn(comb, w.y);
                    }
                    const double2 w = row2[S2 - 1];
                    comb = __dadd_rn(comb, w.x);
                    if (n_sel == 2 * S2) comb = __dadd_rn(comb, w.y);
                } else {
                    int s = 0;
                    for (; s + 1 < n_sel; s += 2) {
                        const double2 w = *reinterpret_cast<const double2 *>(row + s);
                        comb = __dadd_rn(comb, w.x);
                        comb = __dadd_rn(comb, w.y);
                    }
                    if (s < n_sel) comb = __dadd_rn(comb, row[s]);
                }
                if (ebad) comb = 0.0;
                ob[lane] = clamp_ref(__dsub_rn(comb, a.occ_ret), a.occ_lim);
            }
            __syncwarp();
            const int n = (int)min((int64_t)32, rhi - base);
            if (n == 32) {
                const double2 *ob2 = reinterpret_cast<const double2 *>(ob);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const double2 w = ob2[q];
                    c = __dadd_rn(c, w.x);
                    c = __dadd_rn(c, w.y);
                }
            } else {
                for (int q = 0; q < n; ++q) c = __dadd_rn(c, ob[q]);
            }
            __syncwarp();
        }
        if (lane == 0) a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, a.agg_ret), a.agg_lim);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.err, 1u);
}

static constexpr int DENSE_WARPS = 8;
static size_t dense_coop_smem(int em_stride) {
    const int passes = em_stride > 16 ? 2 : 1;
    return (size_t)16 * passes * sizeof(Fin) + (size_t)DENSE_WARPS * 32 * sizeof(double) +
           (size_t)DENSE_WARPS * 32 * (em_stride + 2) * sizeof(double);
}

size_t k2_hotset_fixed_smem(int n_sel) {
    constexpr int NW = K2_THREADS / 32;
    return (size_t)n_sel * sizeof(Fin) + (size_t)NW * VRING * sizeof(double) + (size_t)NW * QCAP * sizeof(uint32_t);
}

template <int HASH, bool CHECK, bool PRE>
static int prepare_one() {
    ARE_CUDA(cudaFuncSetAttribute(k2_hotset<HASH, CHECK, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  k2_max_dynamic_smem()));
    ARE_CUDA(cudaFuncSetAttribute(k2_pair<HASH, CHECK, PRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  k2_max_dynamic_smem()));
    if (!PRE)
        ARE_CUDA(cudaFuncSetAttribute(k2_pair<HASH, CHECK, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      k2_max_dynamic_smem()));
    return ARE_OK;
}

// k2_pair (reading the relay records under the relay's filter when they
// exist) wins on short trials and loses to the relay kernel from a length
// that falls as more events are hot.  Measured, K2 ms at 1e9 ids, C5 shape,
// k2_pair over relay records vs relay:
//   J=4  (few hot)  E=160 2.00 vs 2.74, E=250 1.80 vs 2.08
//   J=15 (14% hot)  E=200 2.50 vs 2.54, E=250 2.46 vs 2.40
//   J=32 (27% hot)  E=130 3.83 vs 4.18, E=160 3.67 vs 3.66, E=200 3.65 vs 3.30
//   J=64 (48% hot)  E=130 5.76 vs 5.90, E=160 5.69 vs 5.48
// Without relay records the hot-set kernel runs above 320 (round 1: E=250
// 3.04 vs 3.19, E=500 2.89 vs 2.73).  ARE_K2_PAIR=0/1 forces a kernel.
static constexpr double PAIR_MAX_MEAN_LEN_HOTSET = 320.0;
static constexpr double PAIR_MAX_MEAN_LEN_DENSE_HOT = 150.0;  // >= 25% of events hot
static constexpr double PAIR_MAX_MEAN_LEN_MID_HOT = 220.0;    // 6-25% hot
static constexpr double RELAY_MIN_HOT_FRAC_MID = 0.06;
static constexpr double RELAY_HOT_FRAC_DENSE = 0.25;
static bool use_pair(double mean_len, double limit) {
    static const int force = [] {
        const char *e = getenv("ARE_K2_PAIR");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    return force >= 0 ? force == 1 : mean_len <= limit;
}

// ARE_K2_REC_PAIR=0 keeps k2_pair on the hot-set slots (A/B).
static bool rec_pair_off() {
    static const bool off = [] {
        const char *e = getenv("ARE_K2_REC_PAIR");
        return e && e[0] == '0';
    }();
    return off;
}

// ARE_DENSE_COOP=0 runs the lane-per-event event-major kernel instead (A/B).
static bool dense_coop_off() {
    static const bool off = [] {
        const char *e = getenv("ARE_DENSE_COOP");
        return e && e[0] == '0';
    }();
    return off;
}

template <bool PRE>
static int prepare_pre() {
    int rc;
    if ((rc = prepare_one<0, true, PRE>()) || (rc = prepare_one<1, true, PRE>()) ||
        (rc = prepare_one<2, true, PRE>()) || (rc = prepare_one<0, false, PRE>()) ||
        (rc = prepare_one<1, false, PRE>()) || (rc = prepare_one<2, false, PRE>()))
        return rc;
    return ARE_OK;
}

int k2_prepare(int device) {
    (void)device;
    int rc;
    if ((rc = prepare_pre<false>()) || (rc = prepare_pre<true>())) return rc;
    ARE_CUDA(cudaFuncSetAttribute(k2_dense_coop<DENSE_WARPS, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_coop_smem(16)));
    ARE_CUDA(cudaFuncSetAttribute(k2_dense_coop<DENSE_WARPS, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_coop_smem(16)));
    ARE_CUDA(cudaFuncSetAttribute(k2_dense_coop<DENSE_WARPS, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_coop_smem(32)));
    ARE_CUDA(cudaFuncSetAttribute(k2_dense_coop<DENSE_WARPS, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)dense_coop_smem(32)));
    if ((rc = k2_relay_prepare())) return rc;
    if ((rc = k2_layers_prepare())) return rc;
    return k2_layers_pre_prepare();
}

template <bool PRE>
static void launch_hotset(const K2Args &a, int sel, dim3 grid, dim3 block, size_t smem, cudaStream_t st) {
    if (use_pair(a.mean_len, PAIR_MAX_MEAN_LEN_HOTSET)) {
        switch (sel) {
            case 0: k2_pair<0, false, PRE><<<grid, block, smem, st>>>(a); break;
            case 1: k2_pair<0, true, PRE><<<grid, block, smem, st>>>(a); break;
            case 2: k2_pair<1, false, PRE><<<grid, block, smem, st>>>(a); break;
            case 3: k2_pair<1, true, PRE><<<grid, block, smem, st>>>(a); break;
            case 4: k2_pair<2, false, PRE><<<grid, block, smem, st>>>(a); break;
            default: k2_pair<2, true, PRE><<<grid, block, smem, st>>>(a); break;
        }
        return;
    }
    switch (sel) {
        case 0: k2_hotset<0, false, PRE><<<grid, block, smem, st>>>(a); break;
        case 1: k2_hotset<0, true, PRE><<<grid, block, smem, st>>>(a); break;
        case 2: k2_hotset<1, false, PRE><<<grid, block, smem, st>>>(a); break;
        case 3: k2_hotset<1, true, PRE><<<grid, block, smem, st>>>(a); break;
        case 4: k2_hotset<2, false, PRE><<<grid, block, smem, st>>>(a); break;
        default: k2_hotset<2, true, PRE><<<grid, block, smem, st>>>(a); break;
    }
}

int k2_launch(const K2Args &a, int variant, int sms, size_t smem_bytes, cudaStream_t st) {
    if (a.last <= a.first) return ARE_OK;
    const int64_t trials = a.last - a.first;
    const bool check = !(variant & ARE_FLAG_IDS_VALIDATED);
    variant &= 0xFF;
    if (variant == ARE_VARIANT_DENSE) {
        int64_t g = (trials + DENSE_WARPS - 1) / DENSE_WARPS;
        const int64_t cap = (int64_t)sms * DENSE_CTAS_PER_SM;
        const int64_t ccap = (int64_t)sms * COOP_CTAS_PER_SM;
        const unsigned cg = (unsigned)(g < ccap ? g : ccap);
        const size_t csm = dense_coop_smem(a.em_stride);
        if (a.em && !dense_coop_off()) {
            if (a.em_stride == 16)
                k2_dense_coop<DENSE_WARPS, 1, true><<<cg, DENSE_WARPS * 32, csm, st>>>(a);
            else if (a.em_stride < 16)
                k2_dense_coop<DENSE_WARPS, 1, false><<<cg, DENSE_WARPS * 32, csm, st>>>(a);
            else if (a.em_stride == 32)
                k2_dense_coop<DENSE_WARPS, 2, true><<<cg, DENSE_WARPS * 32, csm, st>>>(a);
            else
                k2_dense_coop<DENSE_WARPS, 2, false><<<cg, DENSE_WARPS * 32, csm, st>>>(a);
        } else if (a.em)
            k2_dense<DENSE_WARPS, true><<<(unsigned)(g < cap ? g : cap), DENSE_WARPS * 32, 0, st>>>(a);
        else
            k2_dense<DENSE_WARPS, false><<<(unsigned)(g < cap ? g : cap), DENSE_WARPS * 32, 0, st>>>(a);
        ARE_LAUNCHED();
        return ARE_OK;
    }
    constexpr int NW = K2_THREADS / 32;
    int64_t g = (trials + NW - 1) / NW;
    if (g > sms) g = sms;  // persistent: one CTA per SM (the filter fills shared memory)
    const dim3 grid((unsigned)g), block(K2_THREADS);
    const int sel = a.hash_mode * 2 + (check ? 1 : 0);
    const double pair_limit = a.hot_frac >= RELAY_HOT_FRAC_DENSE ? PAIR_MAX_MEAN_LEN_DENSE_HOT
                              : a.hot_frac >= RELAY_MIN_HOT_FRAC_MID ? PAIR_MAX_MEAN_LEN_MID_HOT
                                                                      : PAIR_MAX_MEAN_LEN_HOTSET;
    if (a.rslots && (a.rtex || !k2_relay_needs_texture()) && !use_pair(a.mean_len, pair_limit)) {
        // the relay kernel, over its own filter
        K2Args b = a;
        b.filter = a.rfilter;
        b.filter_words = a.rfilter_words;
        b.nbits = a.rnbits;
        b.hash_mode = a.rhash_mode;
        return k2_relay_launch(b, check, sms, a.rsmem, st);
    }
    if (a.rslots && a.rfilter && !rec_pair_off() && use_pair(a.mean_len, PAIR_MAX_MEAN_LEN_HOTSET)) {
        // short trials with relay records: k2_pair over the relay's records
        // and its per-occurrence-terms filter (fewer gathers, no financial
        // terms or dependent overflow load per occurrence)
        const size_t rsm = k2_hotset_fixed_smem(a.n_sel) + (size_t)a.rfilter_words * 4u;
        if (rsm <= (size_t)k2_max_dynamic_smem()) {
            K2Args b = a;
            b.filter = a.rfilter;
            b.filter_words = a.rfilter_words;
            b.nbits = a.rnbits;
            b.hash_mode = a.rhash_mode;
            switch (b.hash_mode * 2 + (check ? 1 : 0)) {
                case 0: k2_pair<0, false, false, true><<<grid, block, rsm, st>>>(b); break;
                case 1: k2_pair<0, true, false, true><<<grid, block, rsm, st>>>(b); break;
                case 2: k2_pair<1, false, false, true><<<grid, block, rsm, st>>>(b); break;
                case 3: k2_pair<1, true, false, true><<<grid, block, rsm, st>>>(b); break;
                case 4: k2_pair<2, false, false, true><<<grid, block, rsm, st>>>(b); break;
                default: k2_pair<2, true, false, true><<<grid, block, rsm, st>>>(b); break;
            }
            ARE_LAUNCHED();
            return ARE_OK;
        }
    }
    if (a.precombined)
        launch_hotset<true>(a, sel, grid, block, smem_bytes, st);
    else
        launch_hotset<false>(a, sel, grid, block, smem_bytes, st);
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
