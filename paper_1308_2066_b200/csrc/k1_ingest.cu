// K1 -- ELT ingestion and hot-set build.
//
// Replaces TableSet.from_elts / selection_arrays (reference
// pkg/src/aggrisk/tables.py:95-117, :133-153).  Two stages:
//
//  (1) dense direct-access tables on the device: float64 (n_tables, row_len),
//      row-major, slot 0 unused -- the reference's `stacked` layout
//      (tables.py:107-115), built either from the caller's dense array or by
//      scattering the sparse ELT records on the device;
//  (2) per (selection, financial terms) a hot-set "plan": one 16-byte Slot per
//      event id holding the first non-zero loss of the event in selection
//      order plus the count of non-zero losses, an overflow array with the
//      remaining losses (selection order), and a bit filter over event ids
//      that K2 keeps in shared memory.  Events absent from every selected
//      table contribute exactly +-0 to the trial sum ("Zero-skip
//      exactness"), so K2 only touches the records of hot events.
//
// All passes are deterministic (no order-dependent atomics on data).
#include "k1_ingest.cuh"
#include "k2_trials.cuh"

namespace are {

static unsigned grid_for(int64_t n, int threads, int sms, int per_sm = 8);

// ---- (1) dense tables ----------------------------------------------------

// blockIdx.y = table; scatter table y's records into its dense row.
__global__ void k1_scatter_records(const uint32_t *__restrict__ ids,
                                   const double *__restrict__ losses,
                                   const int64_t *__restrict__ table_offsets,
                                   int64_t row_len, double *__restrict__ stacked) {
    const int64_t tab = blockIdx.y;
    const int64_t lo = table_offsets[tab], hi = table_offsets[tab + 1];
    double *row = stacked + tab * row_len;
    for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x)
        row[ids[i]] = losses[i];
}

// ---- (2) hot-set plan ----------------------------------------------------

// One thread per event id: walk the selected rows in selection order
// (the accumulation order of _kernel.pyx:69-76), record the first non-zero
// loss and the non-zero count.  "Non-zero" is !(x == 0.0): NaN and inf are
// kept as entries and flow through the same arithmetic as the reference.
__global__ void k1_slots(const double *__restrict__ stacked, int64_t row_len,
                         const int64_t *__restrict__ rows, int n_sel,
                         Slot *__restrict__ slots, uint32_t *__restrict__ extra,
                         unsigned long long *__restrict__ counters) {
    __shared__ int64_t srows[ARE_MAX_TABLES];
    __shared__ unsigned long long s_hot, s_ent;
    for (int s = threadIdx.x; s < n_sel; s += blockDim.x) srows[s] = rows[s] * row_len;
    if (threadIdx.x == 0) { s_hot = 0; s_ent = 0; }
    __syncthreads();
    unsigned long long hot = 0, ent = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t n = 0, j0 = 0;
        double x0 = 0.0;
        for (int s = 0; s < n_sel; ++s) {
            double x = stacked[srows[s] + e];
            if (!(x == 0.0)) {
                if (n == 0) { x0 = x; j0 = (uint32_t)s; }
                ++n;
            }
        }
        Slot sl;
        sl.x = x0;
        sl.meta = j0 | (n << 16);
        sl.ovf = 0;
        slots[e] = sl;
        extra[e] = n > 1 ? n - 1 : 0;
        hot += n > 0;
        ent += n;
    }
    // warp then block reduction of the two counters
    for (int o = 16; o; o >>= 1) {
        hot += __shfl_xor_sync(0xffffffffu, hot, o);
        ent += __shfl_xor_sync(0xffffffffu, ent, o);
    }
    if ((threadIdx.x & 31) == 0) { atomicAdd(&s_hot, hot); atomicAdd(&s_ent, ent); }
    __syncthreads();
    if (threadIdx.x == 0) { atomicAdd(&counters[0], s_hot); atomicAdd(&counters[1], s_ent); }
}

// Entries 2..n of every multi-table event, written at its scanned offset.
__global__ void k1_overflow(const double *__restrict__ stacked, int64_t row_len,
                            const int64_t *__restrict__ rows, int n_sel,
                            const uint32_t *__restrict__ extra,
                            const uint32_t *__restrict__ ovf_off,
                            Slot *__restrict__ slots, Entry *__restrict__ ovf) {
    __shared__ int64_t srows[ARE_MAX_TABLES];
    for (int s = threadIdx.x; s < n_sel; s += blockDim.x) srows[s] = rows[s] * row_len;
    __syncthreads();
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (extra[e] == 0) continue;
        uint32_t w = ovf_off[e];
        slots[e].ovf = w;
        bool first = true;
        for (int s = 0; s < n_sel; ++s) {
            double x = stacked[srows[s] + e];
            if (!(x == 0.0)) {
                if (first) { first = false; continue; }
                Entry en;
                en.x = x;
                en.j = (uint32_t)s;
                en.pad = 0;
                ovf[w++] = en;
            }
        }
    }
}

// Hot filter: bit b is set iff some event e with e mod nbits == b is hot.
// Exact (one event per bit) when nbits >= row_len.  One warp builds one word.
__global__ void k1_filter(const Slot *__restrict__ slots, int64_t row_len, int64_t nbits,
                          int64_t nwords, uint32_t *__restrict__ words) {
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = w * 32 + lane;
        bool hot = false;
        if (b < nbits)
            for (int64_t e = b; e < row_len; e += nbits) hot |= (slots[e].meta >> 16) != 0;
        const uint32_t word = __ballot_sync(0xffffffffu, hot);
        if (lane == 0) words[w] = word;
    }
}

// Pre-combination: fold every hot event's entries
// into its combined loss comb = 0.0 + sum_j fin_j(x_j) (selection order, the
// same _rn operations K2 performs), stored in the record's x with count 1.
// K2 then skips the financial terms; results stay bit-identical.
__global__ void k1_precombine(Slot *__restrict__ slots, const Entry *__restrict__ ovf, const Fin *__restrict__ fin,
                              int64_t row_len) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        Slot s = slots[e];
        const uint32_t cnt = s.meta >> 16;
        if (!cnt) continue;
        double comb = __dadd_rn(0.0, fin_term(fin[s.meta & 0xFFFFu], s.x));
        for (uint32_t i = 1; i < cnt; ++i) {
            const Entry en = ovf[s.ovf + i - 1];
            comb = __dadd_rn(comb, fin_term(fin[en.j], en.x));
        }
        s.x = comb;
        s.meta = 1u << 16;
        slots[e] = s;
    }
}

int k1_precombine_plan(PlanBuffers &pb, const Fin *d_fin, int64_t row_len, int sms, cudaStream_t st) {
    k1_precombine<<<grid_for(row_len, 256, sms), 256, 0, st>>>(pb.slots, pb.ovf, d_fin, row_len);
    ARE_LAUNCHED();
    return ARE_OK;
}

// Relay records (k2_relay.cu): the financial terms applied once per entry, in
// the same _rn operations K2 would use, and the first partial sum 0.0 + f
// taken here, so K2 adds f_{j2}, f_{j3}, ... in selection order exactly as
// the reference's comb loop does (_kernel.pyx:69-76).
__global__ void k1_relay_slots(const Slot *__restrict__ slots, const Entry *__restrict__ ovf,
                               const Fin *__restrict__ fin, int64_t row_len, RSlot *__restrict__ rs,
                               bool precombined) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        const Slot s = slots[e];
        const uint32_t cnt = s.meta >> 16;
        RSlot r;
        r.a = 0.0;
        r.b = 0.0;
        if (cnt && precombined) {
            // the record already holds comb = 0.0 + sum_j fin_j(x_j) (k1_precombine;
            // never -0.0): comb + (+0.0) is comb, a NaN comb takes the tagged form
            if (!(s.x != s.x)) {
                r.a = s.x;
            } else {
                r.a = __longlong_as_double((long long)(RSLOT_COMPLEX | (1ull << 32)));
                r.b = s.x;
            }
        } else if (cnt) {
            const double x0 = __dadd_rn(0.0, fin_term(fin[s.meta & 0xFFFFu], s.x));
            const double f1 = cnt >= 2 ? fin_term(fin[ovf[s.ovf].j], ovf[s.ovf].x) : 0.0;
            if (cnt <= 2 && !(x0 != x0) && !(f1 != f1)) {
                r.a = x0;
                r.b = f1;
            } else {  // complex: entries 2..cnt from the relay overflow array
                r.a = __longlong_as_double((long long)(RSLOT_COMPLEX | ((unsigned long long)cnt << 32) | s.ovf));
                r.b = x0;
            }
        }
        rs[e] = r;
    }
}

// Fused-layer records: the financial terms applied once per entry (the same
// _rn operations K2-L used to apply per occurrence), so K2-L gathers one
// 32-byte record per hot event and no dependent overflow load for the
// second entry.
__global__ void k1_layer_records(const Slot *__restrict__ slots, const Entry *__restrict__ ovf,
                                 const Fin *__restrict__ fin, int64_t row_len, LRec *__restrict__ out) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < row_len;
         e += (int64_t)gridDim.x * blockDim.x) {
        const Slot s = slots[e];
        const uint32_t cnt = s.meta >> 16;
        LRec r;
        r.fa = 0.0;
        r.fb = 0.0;
        r.x0 = s.x;
        r.ovf = s.ovf;
        uint32_t j0 = 0, j1 = 0;
        if (cnt) {
            j0 = s.meta & 0xFFFFu;
            r.fa = __dadd_rn(0.0, fin_term(fin[j0], s.x));
        }
        if (cnt >= 2) {
            const Entry en = ovf[s.ovf];
            j1 = en.j;
            r.fb = fin_term(fin[j1], en.x);
        }
        r.meta = (j0 & 0xFFu) | ((j1 & 0xFFu) << 8) | (cnt << 16);
        out[e] = r;
    }
}

int k1_build_layer_records(const PlanBuffers &pb, const Fin *d_fin, int64_t row_len, LRec **out, int sms,
                           cudaStream_t st) {
    if (cudaMalloc(out, row_len * sizeof(LRec)) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(ARE_ENOMEM, "device allocation failed while building the fused-layer records");
    }
    k1_layer_records<<<grid_for(row_len, 256, sms), 256, 0, st>>>(pb.slots, pb.ovf, d_fin, row_len, *out);
    ARE_LAUNCHED();
    return ARE_OK;
}

// comb of one relay record, in the reference's order (K2 and the filter)
__device__ __forceinline__ double relay_comb(const RSlot &r, const double *__restrict__ rovf) {
    if (!rslot_complex(r.a)) return __dadd_rn(r.a, r.b);
    double comb = r.b;
    const uint32_t cnt = rslot_cnt(r.a), o = rslot_ovf(r.a);
    for (uint32_t i = 1; i < cnt; ++i) comb = __dadd_rn(comb, rovf[o + i - 1]);
    return comb;
}

__global__ void k1_relay_ovf(const Entry *__restrict__ ovf, const Fin *__restrict__ fin, int64_t n,
                             double *__restrict__ rovf) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Entry en = ovf[i];
        rovf[i] = fin_term(fin[en.j], en.x);
    }
}

int k1_build_relay(const PlanBuffers &pb, const Fin *d_fin, int64_t row_len, int64_t filter_bits, RelayBuffers &rb,
                   int sms, cudaStream_t st, bool precombined) {
    const int64_t n_ovf = std::max<int64_t>(pb.overflow_entries, 1);
    if (cudaMalloc(&rb.rslots, row_len * sizeof(RSlot)) != cudaSuccess ||
        cudaMalloc(&rb.rovf, n_ovf * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        rb.release();
        return fail(ARE_ENOMEM, "device allocation failed while building the relay records");
    }
    k1_relay_slots<<<grid_for(row_len, 256, sms), 256, 0, st>>>(pb.slots, pb.ovf, d_fin, row_len, rb.rslots,
                                                                precombined);
    ARE_LAUNCHED();
    if (pb.overflow_entries && !precombined) {
        k1_relay_ovf<<<grid_for(pb.overflow_entries, 256, sms), 256, 0, st>>>(pb.ovf, d_fin, pb.overflow_entries,
                                                                               rb.rovf);
        ARE_LAUNCHED();
    }
    rb.filter_words = (filter_bits + 31) / 32;  // the per-terms filters (k1_relay_filter)
    if (k2_relay_needs_texture() && row_len <= (int64_t)1 << 27) {  // linear textures hold up to 2^27 texels
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = rb.rslots;
        rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
        rd.res.linear.sizeInBytes = (size_t)row_len * sizeof(RSlot);
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        if (cudaCreateTextureObject(&rb.tex, &rd, &td, nullptr) != cudaSuccess) {
            cudaGetLastError();
            rb.tex = 0;
        }
    }
    return ARE_OK;
}

// Contributing events: an event whose
// occurrence value v = clamp(comb - occ_ret, 0, occ_lim) is +-0 adds +-0 to a
// trial sum that is never -0, so skipping it is exact, like skipping an event
// absent from every table.  comb is evaluated from the relay record in the
// same _rn sequence K2 uses.  One warp per filter word; bit b covers the events
// e = b, b + nbits, ... (the relay kernel's hash).
__global__ void k1_relay_filter_kernel(const RSlot *__restrict__ rs, const double *__restrict__ rovf, int64_t row_len,
                                       int64_t nbits, int64_t nwords, double occ_ret, double occ_lim,
                                       uint32_t *__restrict__ words) {
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = w * 32 + lane;
        bool hot = false;
        if (b < nbits)
            for (int64_t e = b; e < row_len; e += nbits) {
                const RSlot r = rs[e];
                if (!__double_as_longlong(r.a) && !__double_as_longlong(r.b)) continue;  // comb = +0.0
                const double comb = relay_comb(r, rovf);
                double v = __dsub_rn(comb, occ_ret);
                if (v < 0.0) v = 0.0;
                if (v > occ_lim) v = occ_lim;
                hot |= !(v == 0.0);
            }
        const uint32_t word = __ballot_sync(0xffffffffu, hot);
        if (lane == 0) words[w] = word;
    }
}

int k1_relay_filter(const RelayBuffers &rb, int64_t row_len, int64_t nbits, double occ_ret, double occ_lim,
                    uint32_t *words, int sms, cudaStream_t st) {
    const int64_t nwords = (nbits + 31) / 32;
    ARE_CUDA(cudaMemsetAsync(words, 0, (nwords + 4) * sizeof(uint32_t), st));
    k1_relay_filter_kernel<<<grid_for(nwords * 32, 256, sms), 256, 0, st>>>(rb.rslots, rb.rovf, row_len, nbits, nwords,
                                                                             occ_ret, occ_lim, words);
    ARE_LAUNCHED();
    return ARE_OK;
}

// ---- exclusive scan of uint32 counts (3 passes, deterministic) ------------
static constexpr int SCAN_THREADS = 1024;
static constexpr int SCAN_ITEMS = 4;
static constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *warp_tot, uint64_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += n;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
        uint64_t ti = t;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t n = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= o) ti += n;
        }
        warp_tot[lane] = ti - t;
        if (lane == 31) *total = ti;
    }
    __syncthreads();
    return warp_tot[warp] + inc - v;
}

__global__ void k1_scan_tiles(const uint32_t *__restrict__ in, int64_t n, uint64_t *__restrict__ tile_sums) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t total;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    uint64_t v = 0;
    for (int i = 0; i < SCAN_ITEMS; ++i) v += base + i < n ? in[base + i] : 0;
    block_excl_scan(v, warp_tot, &total);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Single block: exclusive scan of the tile sums in place; grand total at [ntiles].
__global__ void k1_scan_tile_sums(uint64_t *__restrict__ tile_sums, int64_t ntiles) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t total;
    uint64_t carry = 0;
    for (int64_t base = 0; base < ntiles; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        uint64_t v = i < ntiles ? tile_sums[i] : 0;
        uint64_t ex = block_excl_scan(v, warp_tot, &total);
        if (i < ntiles) tile_sums[i] = carry + ex;
        carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) tile_sums[ntiles] = carry;
}

__global__ void k1_scan_apply(const uint32_t *__restrict__ in, int64_t n,
                              const uint64_t *__restrict__ tile_sums, uint32_t *__restrict__ out) {
    __shared__ uint64_t warp_tot[32];
    __shared__ uint64_t total;
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    uint64_t s = 0;
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    uint64_t run = tile_sums[blockIdx.x] + block_excl_scan(s, warp_tot, &total);
    for (int i = 0; i < SCAN_ITEMS; ++i) {
        if (base + i < n) out[base + i] = (uint32_t)run;
        run += v[i];
    }
}

int scan_exclusive_u32(const uint32_t *d_in, uint32_t *d_out, int64_t n, uint64_t *d_tiles,
                       uint64_t *h_total, cudaStream_t st) {
    const int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles == 0) { *h_total = 0; return ARE_OK; }
    k1_scan_tiles<<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(d_in, n, d_tiles);
    ARE_LAUNCHED();
    k1_scan_tile_sums<<<1, SCAN_THREADS, 0, st>>>(d_tiles, ntiles);
    ARE_LAUNCHED();
    k1_scan_apply<<<(unsigned)ntiles, SCAN_THREADS, 0, st>>>(d_in, n, d_tiles, d_out);
    ARE_LAUNCHED();
    ARE_CUDA(cudaMemcpyAsync(h_total, d_tiles + ntiles, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    ARE_CUDA(cudaStreamSynchronize(st));
    return ARE_OK;
}

// ---- host drivers --------------------------------------------------------

static unsigned grid_for(int64_t n, int threads, int sms, int per_sm) {
    int64_t g = (n + threads - 1) / threads;
    int64_t cap = (int64_t)sms * per_sm;
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

int k1_scatter(const uint32_t *d_ids, const double *d_losses, const int64_t *d_table_offsets,
               int64_t n_tables, int64_t max_records, int64_t row_len, double *d_stacked,
               int sms, cudaStream_t st) {
    if (n_tables == 0 || max_records == 0) return ARE_OK;
    dim3 grid(grid_for(max_records, 256, sms, 4), (unsigned)n_tables);
    k1_scatter_records<<<grid, 256, 0, st>>>(d_ids, d_losses, d_table_offsets, row_len, d_stacked);
    ARE_LAUNCHED();
    return ARE_OK;
}

int k1_build_plan(const double *d_stacked, int64_t row_len, const int64_t *d_rows, int n_sel,
                  int64_t filter_bits, PlanBuffers &pb, int sms, cudaStream_t st) {
    // counters
    unsigned long long *d_cnt = nullptr;
    uint32_t *d_extra = nullptr, *d_off = nullptr;
    uint64_t *d_tiles = nullptr;
    const int64_t ntiles = (row_len + SCAN_TILE - 1) / SCAN_TILE;
    int rc = ARE_OK;
    unsigned long long h_cnt[2] = {0, 0};
    uint64_t total_extra = 0;
    const int64_t nwords = (filter_bits + 31) / 32;
    auto cleanup = [&]() {
        cudaFree(d_cnt); cudaFree(d_extra); cudaFree(d_off); cudaFree(d_tiles);
    };
    if (cudaMalloc(&d_cnt, 2 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMalloc(&d_extra, row_len * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&d_off, row_len * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&d_tiles, (ntiles + 1) * sizeof(uint64_t)) != cudaSuccess ||
        cudaMalloc(&pb.slots, row_len * sizeof(Slot)) != cudaSuccess ||
        cudaMalloc(&pb.filter, (nwords + 4) * sizeof(uint32_t)) != cudaSuccess) {
        cleanup();
        return fail(ARE_ENOMEM, "device allocation failed while building the hot set");
    }
    cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), st);
    cudaMemsetAsync(pb.filter, 0, (nwords + 4) * sizeof(uint32_t), st);
    k1_slots<<<grid_for(row_len, 256, sms), 256, 0, st>>>(d_stacked, row_len, d_rows, n_sel,
                                                           pb.slots, d_extra, d_cnt);
    g_launches.fetch_add(1);
    if ((rc = cudaGetLastError()) != cudaSuccess) { cleanup(); return cuda_fail((cudaError_t)rc, "k1_slots"); }
    rc = scan_exclusive_u32(d_extra, d_off, row_len, d_tiles, &total_extra, st);
    if (rc != ARE_OK) { cleanup(); return rc; }
    if (total_extra >= (1ull << 32)) { cleanup(); return fail(ARE_EINVAL, "hot set exceeds 2^32 overflow entries"); }
    pb.overflow_entries = (int64_t)total_extra;
    if (total_extra) {
        if (cudaMalloc(&pb.ovf, total_extra * sizeof(Entry)) != cudaSuccess) {
            cleanup();
            return fail(ARE_ENOMEM, "device allocation failed for the overflow entries");
        }
        k1_overflow<<<grid_for(row_len, 256, sms), 256, 0, st>>>(d_stacked, row_len, d_rows, n_sel,
                                                                  d_extra, d_off, pb.slots, pb.ovf);
        g_launches.fetch_add(1);
        if ((rc = cudaGetLastError()) != cudaSuccess) { cleanup(); return cuda_fail((cudaError_t)rc, "k1_overflow"); }
    }
    k1_filter<<<grid_for(nwords * 32, 256, sms), 256, 0, st>>>(pb.slots, row_len, filter_bits, nwords, pb.filter);
    g_launches.fetch_add(1);
    if ((rc = cudaGetLastError()) != cudaSuccess) { cleanup(); return cuda_fail((cudaError_t)rc, "k1_filter"); }
    cudaMemcpyAsync(h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    cleanup();
    if (e != cudaSuccess) return cuda_fail(e, "hot-set build");
    pb.hot_events = (int64_t)h_cnt[0];
    pb.entries = (int64_t)h_cnt[1];
    pb.filter_words = nwords;
    return ARE_OK;
}

// One thread per (event, selection position), events fastest: the reads of
// each selected row are coalesced, the writes land in 8-byte slots of
// consecutive event lines.
__global__ void k1_event_major_kernel(const double *__restrict__ stacked, int64_t row_len,
                                      const int64_t *__restrict__ rows, int n_sel, int stride,
                                      double *__restrict__ em) {
    const int64_t total = row_len * (int64_t)n_sel;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / row_len, e = i - s * row_len;
        em[e * stride + s] = stacked[rows[s] * row_len + e];
    }
}

int k1_event_major(const double *d_stacked, int64_t row_len, const int64_t *d_rows, int n_sel, int stride,
                   double *d_em, int sms, cudaStream_t st) {
    ARE_CUDA(cudaMemsetAsync(d_em, 0, (size_t)row_len * stride * sizeof(double), st));
    const int threads = 256;
    const int64_t total = row_len * (int64_t)n_sel;
    int64_t g = (total + threads - 1) / threads;
    if (g > (int64_t)sms * 16) g = (int64_t)sms * 16;
    k1_event_major_kernel<<<(unsigned)g, threads, 0, st>>>(d_stacked, row_len, d_rows, n_sel, stride, d_em);
    ARE_LAUNCHED();
    return ARE_OK;
}

}  // namespace are
