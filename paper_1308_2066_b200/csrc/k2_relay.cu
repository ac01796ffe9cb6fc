// K2-R -- the relay kernel: the hot-set simulation with the in-order fold
// moved off the streaming warps.
//
// Same contract and float64 sequence as k2_hotset (k2_trials.cu; reference
// run_trials, pkg/src/aggrisk/engine/_kernel.pyx:61-118): for trial t and
// each occurrence e in trial order
//     comb = 0.0 + f_{j1}(x) + f_{j2}(x) + ...        (selection order)
//     c   += clamp(comb - occ_ret, 0, occ_lim)
//     out[t] = clamp(c - agg_ret, 0, agg_lim)
// where f_j(x) = share_j * clamp(rate_j * x - ret_j, 0, lim_j) is evaluated
// once per table entry by K1 (k1_relay_slots: a pure function of the entry,
// same _rn operations), so K2 still gathers every (event, ELT) entry of a hot
// event and sums them in selection order, but no longer re-evaluates the
// financial terms per occurrence.
//
// One persistent CTA of 1024 threads per SM:
//   * warps 0..30 ("producers") each own trials first + b*31 + w, +31*grid,
//     ...: they stream the trial's ids (32-id coalesced rows, two 192-id
//     chunks in flight), test each id against the shared-memory filter,
//     append the hot ones in trial order to a per-warp queue, and per 32
//     queued events gather one 16-byte record per lane (one LDG.128:
//     the event's first partial sum and its second entry, or a tagged
//     pointer to its entries for the rare events with 3+; common.cuh RSlot)
//     and compute the event's occurrence value.  The 32 values go to the
//     warp's ring in shared memory -- one STS per lane -- instead of being
//     folded;
//   * warp 31 ("fold") folds: lane l consumes producer l's ring, adding each
//     batch's 32 values to its trial's running sum strictly in order (+0.0 for
//     lanes past a trial's last event: c >= +0, so that is exact), and writes
//     out[t] at the batch that ends the trial.  One warp instruction advances
//     31 trials' chains, where k2_hotset spent 16 LDS.128 + 32 dependent DADD
//     of a whole warp on every batch.
// Producer and fold synchronise through two mbarriers per ring slot (full:
// the producer's 32 lanes arrive after storing; empty: the fold lane arrives
// after reading), release/acquire at CTA scope without a fence; a ring holds
// KR_NB batches.
#include "k2_trials.cuh"

namespace are {

// Build-time variants (A/B experiments; the defaults are the measured choice).
#ifndef ARE_KR_NF
#define ARE_KR_NF 1        // fold warps
#endif
#ifndef ARE_KR_NB
#define ARE_KR_NB 2        // ring slots (batches) per producer
#endif
#ifndef ARE_KR_ROWDRAIN
#define ARE_KR_ROWDRAIN 0  // drain the queue after every row (64-entry queue) instead of every two
#endif
#ifndef ARE_KR_TEX
#define ARE_KR_TEX 0       // 1: gather the records through the texture pipe (tex1Dfetch) instead of LDG
#endif
#ifndef ARE_KR_TMAF
#define ARE_KR_TMAF 1      // the filter enters shared memory by TMA bulk copies (one thread, no register staging)
#endif
#ifndef ARE_KR_NOALLOC
#define ARE_KR_NOALLOC 1   // record gathers (load path) bypass L1 allocation
#endif
#ifndef ARE_KR_FOLD_TRYWAIT
#define ARE_KR_FOLD_TRYWAIT 0  // the fold polls with try_wait (zero suspend hint) instead of test_wait
#endif
#ifndef ARE_KR_FOLD_SLEEP
#define ARE_KR_FOLD_SLEEP 32  // ns the fold warp sleeps when no producer has a batch ready
#endif
#ifndef ARE_KR_BOUNDS
#define ARE_KR_BOUNDS 0  // debug build: packed-array and queue-capacity checks set bits 2/4 of the plan's error word
#endif
#ifndef ARE_KR_EXP
#define ARE_KR_EXP 0       // timing experiments only (results are wrong when != 0)
#endif
static constexpr int KR_NF = ARE_KR_NF;
static constexpr int KR_NP = (K2R_THREADS / 32 - KR_NF) / KR_NF * KR_NF;  // producer warps
static constexpr int KR_PF = KR_NP / KR_NF;                                // producers per fold warp
#ifndef ARE_KR_RPD
#define ARE_KR_RPD (ARE_KR_ROWDRAIN ? 1 : 3)  // uint32 stream: rows appended between drain checks
#endif
#ifndef ARE_KR_RPD_PK
#define ARE_KR_RPD_PK 3  // packed stream (6 rows per step): rows between drain checks
#endif
#ifndef ARE_KR_ROWS
#define ARE_KR_ROWS 6  // uint32 stream: 32-id rows per chunk (two chunks in flight; 4 rows: E=250 2.51 vs 2.43 ms)
#endif
static constexpr int KR_RPD = ARE_KR_RPD, KR_RPD_PK = ARE_KR_RPD_PK;
static constexpr int KR_ROWS = ARE_KR_ROWS, KR_CH = 32 * ARE_KR_ROWS;
#ifndef ARE_KR_AHEAD
#define ARE_KR_AHEAD 2  // uint32 stream: chunks loaded ahead of the one being filtered (2-4)
#endif
#ifndef ARE_KR_PKB
#define ARE_KR_PKB 1  // packed stream: 96-id blocks per chunk (two chunks in flight; 2 blocks: 1.726 vs 1.716 ms)
#endif
static constexpr int KR_PKB = ARE_KR_PKB;
#ifndef ARE_KR_PK_AHEAD
#define ARE_KR_PK_AHEAD 3  // packed stream: chunks loaded ahead of the one being filtered (2-4; 2: 1.715 vs 1.687 ms)
#endif
// per-producer hot queue: < 32 pending after a drain + 32 per row appended before the next
constexpr int kr_qcap(int rows) { return 31 + 32 * rows <= 64 ? 64 : (31 + 32 * rows <= 128 ? 128 : 256); }
static constexpr int KR_QCAP = kr_qcap(KR_RPD > KR_RPD_PK ? KR_RPD : KR_RPD_PK);
static constexpr int KR_NB = ARE_KR_NB;                     // batches per ring
static constexpr int KR_RSTRIDE = KR_NB * 32 + 2;  // doubles per ring (+16 B: the fold's 32 lanes hit distinct banks)

size_t k2_relay_fixed_smem() {
    return (size_t)KR_NP * KR_QCAP * sizeof(uint32_t) + (size_t)KR_NP * KR_RSTRIDE * sizeof(double) +
           (size_t)2 * 32 * KR_NB * sizeof(uint64_t) + (size_t)32 * KR_NB * sizeof(uint32_t) + 16;
}

// A gathered relay record kept exactly as loaded (four doubles; count and
// overflow index decoded where used), so the loop-carried pending batch can
// live in the load's own destination registers (no copy of an in-flight load).
// A gathered relay record kept exactly as loaded (RSlot's two doubles,
// decoded where the value is computed, one batch later), so the loop-carried
// pending batch lives in the load's own destination registers.
struct RRaw {
    double a, b;
};
__device__ __forceinline__ RRaw ld_rslot(const RSlot *p, uint64_t policy) {
    RRaw r;
#if ARE_KR_NOALLOC == 2  // A/B: L2-only load (.cg)
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.a), "=d"(r.b) : "l"(p), "l"(policy));
#elif ARE_KR_NOALLOC == 3  // A/B: allocate, evict first
    asm volatile("ld.global.nc.L1::evict_first.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.a), "=d"(r.b) : "l"(p), "l"(policy));
#elif ARE_KR_NOALLOC
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.a), "=d"(r.b) : "l"(p), "l"(policy));
#else
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(r.a), "=d"(r.b) : "l"(p), "l"(policy));
#endif
    return r;
}
// mbarrier helpers (shared::cta).  arrive has release and test/try_wait
// acquire semantics at CTA scope; neither waits for the thread's in-flight
// global loads (a fence would: MEMBAR.CTA stalls until the id stream's
// outstanding LDGs return).
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint32_t a, uint32_t parity) {
    uint32_t r;
#if ARE_KR_FOLD_TRYWAIT
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(a), "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(r)
        : "r"(a), "r"(parity)
        : "memory");
#endif
    return r != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}

template <int HASH>
__device__ __forceinline__ uint32_t relay_hash(uint32_t e, uint32_t nbits) {
    if (HASH == 0) return e;
    if (HASH == 1) return min(e, e - nbits);
    return e % nbits;
}

// The fold warp: lane l < KR_NP consumes producer l's batches.  Batch h of
// a producer sits in ring slot h % KR_NB; full[slot] completes its phase
// h / KR_NB when the producer's 32 lanes have stored it, empty[slot] when the
// fold lane has read it.
__device__ __forceinline__ void relay_fold(const K2Args &a, int fw, const double *s_ring, uint32_t full0,
                                           uint32_t empty0, const uint32_t *s_end) {
    const int lane = threadIdx.x & 31;
    const int64_t W = (int64_t)gridDim.x * KR_NP;
    const int me = fw * KR_PF + (lane < KR_PF ? lane : 0);  // the producer this lane folds for
    int64_t t = lane < KR_PF ? a.first + (int64_t)blockIdx.x * KR_NP + me : a.last;
    const double *ring = s_ring + me * KR_RSTRIDE;
    const uint32_t full = full0 + me * KR_NB * 8, empty = empty0 + me * KR_NB * 8;
    const double agg_ret = a.agg_ret, agg_lim = a.agg_lim;
    double c = 0.0;
    uint32_t head = 0;
    while (__any_sync(0xffffffffu, t < a.last)) {
        const uint32_t slot = head & (KR_NB - 1);
        bool ready = false;
        if (t < a.last) ready = mbar_test(full + slot * 8, (head / KR_NB) & 1);
        if (!__any_sync(0xffffffffu, ready)) {
            if (ARE_KR_FOLD_SLEEP) __nanosleep(ARE_KR_FOLD_SLEEP);
            continue;
        }
        if (ready) {
            const double2 *r2 = reinterpret_cast<const double2 *>(ring + slot * 32);
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                double2 w[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) w[i] = r2[4 * g + i];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    c = __dadd_rn(c, w[i].x);
                    c = __dadd_rn(c, w[i].y);
                }
            }
            const uint32_t end = s_end[me * KR_NB + slot];
            mbar_arrive(empty + slot * 8);  // the slot's values are in registers
            ++head;
            if (end) {
                a.out[t - a.out_base] = clamp_ref(__dsub_rn(c, agg_ret), agg_lim);
                c = 0.0;
                t += W;
            }
        }
    }
}

template <int HASH, bool CHECK, bool PK>
__global__ void __launch_bounds__(K2R_THREADS, 1) k2_relay(const K2Args a) {
    static_assert(!(PK && CHECK), "packed ids are validated ids");
    extern __shared__ __align__(16) unsigned char smem[];
    // the filter at offset 0 (its LDS addresses need no base register)
    uint32_t *s_filter = reinterpret_cast<uint32_t *>(smem);
    uint32_t *s_q = s_filter + a.filter_words;
    double *s_ring = reinterpret_cast<double *>(s_q + KR_NP * KR_QCAP);
    uint64_t *s_bar = reinterpret_cast<uint64_t *>(s_ring + KR_NP * KR_RSTRIDE);  // full[32][NB], empty[32][NB]
    uint32_t *s_end = reinterpret_cast<uint32_t *>(s_bar + 2 * 32 * KR_NB);
    const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(s_bar);
    const uint32_t empty0 = full0 + 32 * KR_NB * 8;
    {
#if ARE_KR_TMAF
        // one thread hands the whole filter to the TMA unit in 16 KB bulk
        // copies completing on one mbarrier (no LDG/STS round trips through
        // registers)
        const uint32_t fbar = (uint32_t)__cvta_generic_to_shared(s_end + 32 * KR_NB);
        if (threadIdx.x == 0) {
            const uint32_t bytes = a.filter_words * 4u, dst = (uint32_t)__cvta_generic_to_shared(s_filter);
            mbar_init(fbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fbar), "r"(bytes) : "memory");
            for (uint32_t off = 0; off < bytes; off += 16384u) {
                const uint32_t n = min(16384u, bytes - off);
                asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst + off),
                             "l"(reinterpret_cast<const unsigned char *>(a.filter) + off), "r"(n), "r"(fbar)
                             : "memory");
            }
        }
#else
        const uint4 *src = reinterpret_cast<const uint4 *>(a.filter);
        uint4 *dst = reinterpret_cast<uint4 *>(s_filter);
        const int n4 = (int)(a.filter_words >> 2);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) dst[i] = src[i];
#endif
        if (threadIdx.x < KR_NP * KR_NB) {
            mbar_init(full0 + threadIdx.x * 8, 32);  // the producer's 32 lanes
            mbar_init(empty0 + threadIdx.x * 8, 1);  // its fold lane
        }
    }
    __syncthreads();
#if ARE_KR_TMAF
    mbar_wait((uint32_t)__cvta_generic_to_shared(s_end + 32 * KR_NB), 0);
#endif

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp >= KR_NP) {
        if (warp < KR_NP + KR_NF) relay_fold(a, warp - KR_NP, s_ring, full0, empty0, s_end);
        return;
    }
    const uint32_t my_full = full0 + warp * KR_NB * 8, my_empty = empty0 + warp * KR_NB * 8;

    uint32_t *q = s_q + warp * KR_QCAP;
    const uint32_t q_saddr = (uint32_t)__cvta_generic_to_shared(q);
    double *ring = s_ring + warp * KR_RSTRIDE;
    const uint32_t lt = lanemask_lt();
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t nbits = a.nbits, last_id = a.row_len - 1;
    const double occ_ret = a.occ_ret, occ_lim = a.occ_lim;
    const uint32_t *const ids = a.ids;
    const int64_t W = (int64_t)gridDim.x * KR_NP;
    uint32_t emax = 0;
    const uint32_t pad = cold_pad(s_filter, a.filter_words, nbits, a.row_len);
    uint32_t seq = 0;  // batches published (uniform)

    // publish one batch of 32 occurrence values (lanes past the batch: +0.0)
    auto push = [&](double v, uint32_t end) {
        const uint32_t slot = seq & (KR_NB - 1), use = seq / KR_NB;
        if (use) mbar_wait(my_empty + slot * 8, (use - 1) & 1);  // the fold has read the slot's last batch
        ring[slot * 32 + lane] = v;
        if (lane == 0) s_end[warp * KR_NB + slot] = end;
        mbar_arrive(my_full + slot * 8);
        ++seq;
    };
    // occurrence value of this lane's gathered event (slot 0 -- empty -- for
    // lanes past the batch: comb = +0.0, v = clamp(-occ_ret) = +-0)
    auto value = [&](const RRaw &s) -> double {
        double comb;
        if (!rslot_complex(s.a)) {
            comb = __dadd_rn(s.a, s.b);  // one or two entries (RSlot)
        } else {
            comb = s.b;
            const uint32_t cnt = rslot_cnt(s.a), o = rslot_ovf(s.a);
#pragma unroll 1
            for (uint32_t i = 1; i < cnt; ++i) comb = __dadd_rn(comb, a.rovf[o + i - 1]);
        }
        return clamp_ref(__dsub_rn(comb, occ_ret), occ_lim);
    };
    auto gather = [&](uint32_t qh, uint32_t n) -> RRaw {
        const uint32_t e = q[(qh + lane) & (KR_QCAP - 1)];
#if ARE_KR_EXP == 4  // timing experiment: every gather from a 512 KB window
        return ld_rslot(a.rslots + ((uint32_t)lane < n ? (e & 0x3FFFu) : 0u), pol_keep);
#endif
#if ARE_KR_EXP == 7  // timing experiment: every gather from one 128-byte line (L1 hits)
        return ld_rslot(a.rslots + ((uint32_t)lane < n ? (e & 7u) : 0u), pol_keep);
#endif
#if ARE_KR_EXP == 8  // timing experiment: every gather from a 16 KB window (L1-resident)
        return ld_rslot(a.rslots + ((uint32_t)lane < n ? (e & 1023u) : 0u), pol_keep);
#endif
#if ARE_KR_TEX
        // through the texture pipe (the host runs this kernel only with a
        // texture object over the records): one 16-byte texel per record
        const int i = (int)((uint32_t)lane < n ? e : 0u);
        RRaw r;
        asm volatile("{\n\t.reg .b32 a0, a1, a2, a3;\n\t"
                     "tex.1d.v4.u32.s32 {a0, a1, a2, a3}, [%2, {%3}];\n\t"
                     "mov.b64 %0, {a0, a1};\n\tmov.b64 %1, {a2, a3};\n\t}"
                     : "=d"(r.a), "=d"(r.b)
                     : "l"(a.rtex), "r"(i));
        return r;
#else
        return ld_rslot(a.rslots + ((uint32_t)lane < n ? e : 0u), pol_keep);
#endif
    };

    // One row = 32 ids of a trial in trial order, one per lane.  append_row
    // queues a row's hot ids in order (ballot + predicated STS); drain turns
    // every full 32-event batch of the queue into a gather (this batch) and a
    // value + push (the previous batch, whose gather has had a batch of
    // filtering to land).
    uint32_t qh = 0, qt = 0;
    bool pending = false;
    RRaw ps{};
    auto append_row = [&](uint32_t e, uint32_t w) {
        const bool hot = (w >> (relay_hash<HASH>(e, nbits) & 31)) & 1u;
#if ARE_KR_EXP == 1  // timing experiment: filter only
        emax += hot;
        return;
#endif
        const uint32_t b = ballot_full(hot);
        st_shared_if(q_saddr + (((qt + __popc(b & lt)) & (KR_QCAP - 1)) << 2), e, hot);
        qt += __popc(b);
#if ARE_KR_BOUNDS  // debug build: the ring never holds more than KR_QCAP entries
        if (qt - qh > (uint32_t)KR_QCAP) atomicOr(a.err, 4u);
#endif
    };
    auto drain = [&]() {
        __syncwarp();
        while (qt - qh >= 32u) {
#if ARE_KR_EXP == 2  // timing experiment: filter + append, no batches
            qh += 32u;
            continue;
#endif
            // the pending batch's value first, then the new gather into
            // the same registers: no register copy of an in-flight load
            const double v = value(ps);
#if ARE_KR_EXP == 5  // timing experiment: gather, no value, no push
            emax ^= (uint32_t)__double2loint(ps.a) ^ (uint32_t)__double2hiint(ps.b);
            ps = gather(qh, 32u);
            qh += 32u;
            continue;
#endif
#if ARE_KR_EXP == 6  // timing experiment: value of the queued ids (no gather), no push
            {
                const double v6 = value(ps);
                if (v6 == 12345.0) emax++;
                const uint32_t e6 = q[(qh + lane) & (KR_QCAP - 1)];
                ps = RRaw{(double)e6, 0.0};
                qh += 32u;
                continue;
            }
#endif
#if ARE_KR_EXP == 3  // timing experiment: no push
            ps = gather(qh, 32u);
            if (v == 12345.0) emax++;
            pending = true;
            qh += 32u;
            continue;
#endif
            ps = gather(qh, 32u);
            if (pending) push(v, 0u);
            pending = true;
            qh += 32u;
        }
    };
    // the trial's final partial batch, then its end marker
    auto flush = [&]() {
        const uint32_t n = qt - qh;
        const double v = value(ps);
        if (n) {
            ps = gather(qh, n);
            if (pending) push(v, 0u);
            push(value(ps), 1u);
        } else {
            push(pending ? v : 0.0, 1u);
        }
        qh = qt = 0;
        pending = false;
    };

    int64_t t = a.first + (int64_t)blockIdx.x * KR_NP + warp;
    uint32_t len = 0, rel = 0;
    int nchunks = 0;
    int64_t nlo = 0, nhi = 0;  // the bounds of the warp's next trial
    if constexpr (!PK) {
        // A trial's ids are streamed as KR_CH-id chunks (6 rows) aligned to 128-byte lines
        // (`skew` positions before the trial; `rel` wraps below zero there, so one
        // unsigned compare bounds both ends).  The next trial's first two chunks
        // are requested before the current trial's final batch is flushed, so
        // their latency overlaps that batch's gather.
        const uint32_t *p = ids;
        uint32_t r0[KR_ROWS], r1[KR_ROWS], r2[KR_ROWS];
#if ARE_KR_AHEAD >= 3
        uint32_t r3[KR_ROWS];
#endif
#if ARE_KR_AHEAD >= 4
        uint32_t r4[KR_ROWS];
#endif
        auto begin = [&](int64_t lo, int64_t hi) {
            const int64_t rlo = lo - a.id_base;
            len = (uint32_t)(hi - lo);
            const uint32_t skew = (uint32_t)((reinterpret_cast<uintptr_t>(ids + rlo) >> 2) & 31);
            p = ids + (rlo - skew) + lane;
            rel = (uint32_t)lane - skew;
            nchunks = (int)((len + skew + KR_CH - 1) / KR_CH);
#pragma unroll
            for (int k = 0; k < KR_ROWS; ++k) r0[k] = ld_stream_if(p + 32 * k, rel + 32 * k, len, pol_stream, pad);
#pragma unroll
            for (int k = 0; k < KR_ROWS; ++k) r1[k] = ld_stream_if(p + KR_CH + 32 * k, rel + KR_CH + 32 * k, len, pol_stream, pad);
#if ARE_KR_AHEAD >= 3
#pragma unroll
            for (int k = 0; k < KR_ROWS; ++k)
                r2[k] = ld_stream_if(p + 2 * KR_CH + 32 * k, rel + 2 * KR_CH + 32 * k, len, pol_stream, pad);
#endif
#if ARE_KR_AHEAD >= 4
#pragma unroll
            for (int k = 0; k < KR_ROWS; ++k)
                r3[k] = ld_stream_if(p + 3 * KR_CH + 32 * k, rel + 3 * KR_CH + 32 * k, len, pol_stream, pad);
#endif
        };
        if (t < a.last) begin(a.offsets[t - a.t_base], a.offsets[t - a.t_base + 1]);
        for (; t < a.last; t += W) {
            const int64_t tn = t + W;
            if (tn < a.last) {  // next trial's bounds, in flight during this trial
                nlo = a.offsets[tn - a.t_base];
                nhi = a.offsets[tn - a.t_base + 1];
            }
            auto step = [&](uint32_t (&cur)[KR_ROWS], uint32_t (&fut)[KR_ROWS]) {
                const uint32_t rel0 = rel - (uint32_t)lane + (uint32_t)(ARE_KR_AHEAD * KR_CH);  // start of the chunk loaded now, trial-relative
                if ((int32_t)rel0 >= 0 && rel0 + (uint32_t)KR_CH <= len) {
#pragma unroll
                    for (int k = 0; k < KR_ROWS; ++k) fut[k] = ld_stream_u32(p + ARE_KR_AHEAD * KR_CH + 32 * k, pol_stream);
                } else {
#pragma unroll
                    for (int k = 0; k < KR_ROWS; ++k) fut[k] = ld_stream_if(p + ARE_KR_AHEAD * KR_CH + 32 * k, rel + ARE_KR_AHEAD * KR_CH + 32 * k, len,
                                              pol_stream, pad);
                }
                uint32_t ev[KR_ROWS], word[KR_ROWS];
#pragma unroll
                for (int k = 0; k < KR_ROWS; ++k) {
                    uint32_t e = cur[k];
                    if (CHECK) {
                        emax = max(emax, e);
                        e = min(e, last_id);
                    }
                    ev[k] = e;
                    word[k] = s_filter[relay_hash<HASH>(e, nbits) >> 5];
                }
#pragma unroll
                for (int k = 0; k < KR_ROWS; ++k) {
                    append_row(ev[k], word[k]);
                    if ((k + 1) % KR_RPD == 0 || k == KR_ROWS - 1) drain();
                }
                p += KR_CH;
                rel += KR_CH;
            };
#if ARE_KR_AHEAD == 4
            for (int ch = 0; ch < nchunks; ch += 5) {
                step(r0, r4);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
                if (ch + 3 >= nchunks) break;
                step(r3, r2);
                if (ch + 4 >= nchunks) break;
                step(r4, r3);
            }
#elif ARE_KR_AHEAD == 3
            for (int ch = 0; ch < nchunks; ch += 4) {
                step(r0, r3);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
                if (ch + 3 >= nchunks) break;
                step(r3, r2);
            }
#else
            for (int ch = 0; ch < nchunks; ch += 3) {
                step(r0, r2);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
            }
#endif
            if (tn < a.last) begin(nlo, nhi);  // the next trial's first chunks, in flight during the flush
            flush();
        }
    } else {
        // Packed resident ids (are_yet_pack_device): three 21-bit ids per
        // 64-bit word, 96-id blocks of 32 words, word l of a block holding
        // block positions l, l+32, l+64 -- so one LDG.64 per lane brings three
        // 32-id rows that are each in lane order, and the in-order append is
        // unchanged.  A chunk is KR_PKB blocks (one: 96 ids, 3 rows, one drain
        // check); two chunks are in flight while one is filtered.  2/3 of the
        // id sectors of the uint32 stream.
        const unsigned long long *pp = a.pids;
        unsigned long long r0[KR_PKB], r1[KR_PKB], r2[KR_PKB];
#if ARE_KR_PK_AHEAD >= 3
        unsigned long long r3[KR_PKB];
#endif
#if ARE_KR_PK_AHEAD >= 4
        unsigned long long r4[KR_PKB];
#endif
        int32_t bleft = 0;  // the trial's blocks from the current chunk on
        auto ldw = [&](const unsigned long long *w, bool ok) -> unsigned long long {
            unsigned long long r = 0;
#if ARE_KR_BOUNDS  // debug build: every packed word read lies inside the packed array
            if (ok && (uint64_t)(w - a.pids) >= (uint64_t)packed_id_words(a.n_ids)) atomicOr(a.err, 2u);
#endif
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t"
                "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%2], %3;\n\t}"
                : "+l"(r)
                : "r"((uint32_t)ok), "l"(w), "l"(pol_stream));
            return r;
        };
        auto begin = [&](int64_t lo, int64_t hi) {
            const uint64_t rlo = (uint64_t)(lo - a.id_base);
            const uint64_t b0 = rlo / 96u;
            const uint32_t skew = (uint32_t)(rlo - b0 * 96u);
            len = (uint32_t)(hi - lo);
            pp = a.pids + b0 * 32u + lane;
            rel = (uint32_t)lane - skew;
            bleft = (int32_t)((len + skew + 95u) / 96u);
            nchunks = (bleft + KR_PKB - 1) / KR_PKB;
#pragma unroll
            for (int j = 0; j < KR_PKB; ++j) r0[j] = ldw(pp + 32 * j, j < bleft);
#pragma unroll
            for (int j = 0; j < KR_PKB; ++j) r1[j] = ldw(pp + 32 * KR_PKB + 32 * j, KR_PKB + j < bleft);
#if ARE_KR_PK_AHEAD >= 3
#pragma unroll
            for (int j = 0; j < KR_PKB; ++j) r2[j] = ldw(pp + 64 * KR_PKB + 32 * j, 2 * KR_PKB + j < bleft);
#endif
#if ARE_KR_PK_AHEAD >= 4
#pragma unroll
            for (int j = 0; j < KR_PKB; ++j) r3[j] = ldw(pp + 96 * KR_PKB + 32 * j, 3 * KR_PKB + j < bleft);
#endif
        };
        if (t < a.last) begin(a.offsets[t - a.t_base], a.offsets[t - a.t_base + 1]);
        for (; t < a.last; t += W) {
            const int64_t tn = t + W;
            if (tn < a.last) {
                nlo = a.offsets[tn - a.t_base];
                nhi = a.offsets[tn - a.t_base + 1];
            }
            auto step = [&](unsigned long long (&cur)[KR_PKB], unsigned long long (&fut)[KR_PKB]) {
#pragma unroll
                for (int j = 0; j < KR_PKB; ++j)
                    fut[j] = ldw(pp + 32 * ARE_KR_PK_AHEAD * KR_PKB + 32 * j, ARE_KR_PK_AHEAD * KR_PKB + j < bleft);
                uint32_t ev[3 * KR_PKB], word[3 * KR_PKB];
#pragma unroll
                for (int j = 0; j < KR_PKB; ++j) {
                    const uint32_t lo32 = (uint32_t)cur[j], hi32 = (uint32_t)(cur[j] >> 32);
                    const uint32_t x[3] = {lo32 & 0x1FFFFFu, __funnelshift_r(lo32, hi32, 21) & 0x1FFFFFu, hi32 >> 10};
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const uint32_t e = rel + (uint32_t)(96 * j + 32 * k) < len ? x[k] : pad;
                        ev[3 * j + k] = e;
                        word[3 * j + k] = s_filter[relay_hash<HASH>(e, nbits) >> 5];
                    }
                }
#pragma unroll
                for (int k = 0; k < 3 * KR_PKB; ++k) {
                    append_row(ev[k], word[k]);
                    if ((k + 1) % KR_RPD_PK == 0 || k == 3 * KR_PKB - 1) drain();
                }
                pp += 32 * KR_PKB;
                rel += 96 * KR_PKB;
                bleft -= KR_PKB;
            };
#if ARE_KR_PK_AHEAD == 4
            for (int ch = 0; ch < nchunks; ch += 5) {
                step(r0, r4);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
                if (ch + 3 >= nchunks) break;
                step(r3, r2);
                if (ch + 4 >= nchunks) break;
                step(r4, r3);
            }
#elif ARE_KR_PK_AHEAD == 3
            for (int ch = 0; ch < nchunks; ch += 4) {
                step(r0, r3);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
                if (ch + 3 >= nchunks) break;
                step(r3, r2);
            }
#else
            for (int ch = 0; ch < nchunks; ch += 3) {
                step(r0, r2);
                if (ch + 1 >= nchunks) break;
                step(r1, r0);
                if (ch + 2 >= nchunks) break;
                step(r2, r1);
            }
#endif
            if (tn < a.last) begin(nlo, nhi);
            flush();
        }
    }
#if ARE_KR_EXP
    if (emax == 0xFFFFFFFFu) a.out[0] = 1.0;
#endif
    if (CHECK && __any_sync(0xffffffffu, emax > last_id) && lane == 0) atomicOr(a.err, 1u);
}

bool k2_relay_needs_texture() { return ARE_KR_TEX != 0; }

template <int HASH, bool CHECK, bool PK>
static int relay_attr() {
    ARE_CUDA(cudaFuncSetAttribute(k2_relay<HASH, CHECK, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize, k2_max_dynamic_smem()));
    return ARE_OK;
}

int k2_relay_prepare() {
    int rc;
    if ((rc = relay_attr<0, false, false>()) || (rc = relay_attr<0, true, false>()) || (rc = relay_attr<1, false, false>()) ||
        (rc = relay_attr<1, true, false>()) || (rc = relay_attr<2, false, false>()) || (rc = relay_attr<2, true, false>()) ||
        (rc = relay_attr<0, false, true>()) || (rc = relay_attr<1, false, true>()) || (rc = relay_attr<2, false, true>()))
        return rc;
    return ARE_OK;
}

int k2_relay_launch(const K2Args &a, bool check, int sms, size_t smem_bytes, cudaStream_t st) {
    if (a.last <= a.first) return ARE_OK;
    const int64_t trials = a.last - a.first;
    int64_t g = (trials + KR_NP - 1) / KR_NP;
    if (g > sms) g = sms;  // persistent: one CTA per SM (the filter fills shared memory)
    const dim3 grid((unsigned)g), block(K2R_THREADS);
    if (a.pids && !check) {  // packed resident ids (validated by construction)
        switch (a.hash_mode) {
            case 0: k2_relay<0, false, true><<<grid, block, smem_bytes, st>>>(a); break;
            case 1: k2_relay<1, false, true><<<grid, block, smem_bytes, st>>>(a); break;
            default: k2_relay<2, false, true><<<grid, block, smem_bytes, st>>>(a); break;
        }
        ARE_LAUNCHED();
        return ARE_OK;
    }
    const int sel = a.hash_mode * 2 + (check ? 1 : 0);
    switch (sel) {
        case 0: k2_relay<0, false, false><<<grid, block, smem_bytes, st>>>(a); break;
        case 1: k2_relay<0, true, false><<<grid, block, smem_bytes, st>>>(a); break;
        case 2: k2_relay<1, false, false><<<grid, block, smem_bytes, st>>>(a); break;
        case 3: k2_relay<1, true, false><<<grid, block, smem_bytes, st>>>(a); break;
        case 4: k2_relay<2, false, false><<<grid, block, smem_bytes, st>>>(a); break;
        default: k2_relay<2, true, false><<<grid, block, smem_bytes, st>>>(a); break;
    }
    ARE_LAUNCHED();
    return ARE_OK;
}

// Packed resident ids: word b*32 + l of block b holds positions 96b + l,
// 96b + 32 + l, 96b + 64 + l in bits [0,21), [21,42), [42,63) (zero past
// n_ids).  Ids >= 2^21 cannot be packed: they set *err (the caller validated
// the YET, so this is a contract check).
__global__ void k1_pack_ids(const uint32_t *__restrict__ ids, int64_t n_ids, unsigned long long *__restrict__ pk,
                            int64_t n_words, unsigned int *err) {
    bool bad = false;
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = (w >> 5) * 96 + (w & 31);
        unsigned long long v = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int64_t i = base + 32 * k;
            const uint32_t e = i < n_ids ? __ldcs(ids + i) : 0u;
            bad |= e > 0x1FFFFFu;
            v |= (unsigned long long)(e & 0x1FFFFFu) << (21 * k);
        }
        __stcs(pk + w, v);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0 && err) atomicOr(err, 1u);
}

int k1_pack_ids_launch(const uint32_t *ids, int64_t n_ids, unsigned long long *pk, unsigned int *err, int sms,
                       cudaStream_t st) {
    const int64_t n_words = packed_id_words(n_ids);
    if (n_words == 0) return ARE_OK;
    int64_t g = (n_words + 255) / 256;
    if (g > (int64_t)sms * 8) g = (int64_t)sms * 8;
    k1_pack_ids<<<(unsigned)g, 256, 0, st>>>(ids, n_ids, pk, n_words, err);
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
