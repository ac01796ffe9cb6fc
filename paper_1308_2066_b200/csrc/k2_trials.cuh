#pragma once
#include "common.cuh"

namespace are {

// Arguments of one K2 launch.  Indices are absolute (reference numbering):
// occurrence i lives at ids[i - id_base], trial t's offsets at
// offsets[t - t_base], and its result goes to out[t - out_base].
struct K2Args {
    const uint32_t *ids;
    int64_t id_base;
    int64_t n_ids;
    const int64_t *offsets;
    int64_t t_base;
    int64_t first, last;
    double *out;
    int64_t out_base;
    // hot set
    const uint32_t *filter;
    int64_t filter_words;  // multiple of 4
    uint32_t nbits;
    int32_t hash_mode;     // 0: e, 1: e - nbits once, 2: e % nbits
    const Slot *slots;
    const Entry *ovf;
    uint32_t row_len;
    // terms
    const Fin *fin;
    int32_t n_sel;
    int32_t fin_bytes;     // n_sel * sizeof(Fin)
    double occ_ret, occ_lim, agg_ret, agg_lim;
    // dense variant
    const double *stacked;
    const int64_t *rows;
    unsigned int *err;
    int32_t precombined;   // records hold comb (k1_precombine): skip the financial terms
    // dense variant, event-major copy of the selected rows (k1_event_major):
    // em[e * em_stride + s] = stacked[rows[s]][e], em_stride even; null = row-major
    const double *em;
    int32_t em_stride;
    // mean occurrences per trial of the launch (host estimate): short trials
    // run the paired kernel (k2_pair), long ones k2_hotset
    double mean_len;
    // fraction of catalog events in at least one selected table (plan): the
    // relay kernel pays off on mid-length trials only when enough ids are hot
    double hot_frac;
    // relay kernel (k2_relay.cu): its records, fin-applied overflow values
    // and its own filter (its fixed shared memory differs from k2_hotset's)
    const RSlot *rslots = nullptr;
    const double *rovf = nullptr;
    const uint32_t *rfilter = nullptr;
    int64_t rfilter_words = 0;
    uint32_t rnbits = 0;
    int32_t rhash_mode = 0;
    size_t rsmem = 0;
    unsigned long long rtex = 0;  // texture object over rslots (uint4 texels), 0: none
    // packed resident ids (are_yet_pack_device), indexed like `ids`; the relay
    // kernel streams them instead of `ids` when the ids are validated
    const unsigned long long *pids = nullptr;
};

// Threads per CTA of the hot-set kernel (one persistent CTA per SM).
constexpr int K2_THREADS = 1024;
// Threads per CTA of the relay kernel: 31 producer warps + 1 fold warp.
#ifndef ARE_KR_THREADS
#define ARE_KR_THREADS 1024
#endif
constexpr int K2R_THREADS = ARE_KR_THREADS;

// Fused multi-layer kernel (k2_layers.cu): 16 warps per CTA, up to 16 layers
// per launch over one ELT pool of up to 64 tables.
constexpr int K2L_THREADS = 512;
constexpr int K2L_MAX_LAYERS = 16;
constexpr int K2L_MAX_POOL = 64;

struct LayerTerm {
    double occ_ret, occ_lim, agg_ret, agg_lim;
};
struct K2Layers {
    int32_t n_layers;
    int64_t out_stride;      // out[l * out_stride + t]
    const uint64_t *masks;   // pool-row bitmask per layer
    const LayerTerm *terms;  // per layer
    const double *occ_table = nullptr;  // pre-combined: occ[e * 16 + l] (k1_layer_occ)
    const LRec *lrec = nullptr;         // exact fused layers: per-event records (k1_layer_records)
};

// An event id whose filter bit is clear, used for the stream positions
// outside a trial (they must not count as hits: event 0 shares its bit with
// event nbits under HASH 1/2).  Searches the first 1024 bits; 0 if none
// (then only speed suffers).  Warp-uniform result.
__device__ __forceinline__ uint32_t cold_pad(const uint32_t *s_filter, int64_t filter_words, uint32_t nbits,
                                             uint32_t row_len) {
    const int lane = threadIdx.x & 31;
    const uint32_t w = lane < filter_words ? s_filter[lane] : 0xFFFFFFFFu;
    const uint32_t lim = min(nbits, row_len);
    uint32_t cand = 0xFFFFFFFFu;
    if (~w) cand = (uint32_t)lane * 32 + (__ffs(~w) - 1);
    if (cand >= lim) cand = 0xFFFFFFFFu;
    cand = __reduce_min_sync(0xffffffffu, cand);
    return cand == 0xFFFFFFFFu ? 0u : cand;
}

// Largest dynamic shared-memory carve-out requested by K2 (sm_100: 227 KB).
inline int k2_max_dynamic_smem() { return 227 * 1024; }
size_t k2_hotset_fixed_smem(int n_sel);
bool k2_relay_needs_texture();
// 64-bit words of the packed id layout for n ids (whole 96-id blocks)
__host__ __device__ inline int64_t packed_id_words(int64_t n) { return (n + 95) / 96 * 32; }
int k1_pack_ids_launch(const uint32_t *ids, int64_t n_ids, unsigned long long *pk, unsigned int *err, int sms,
                       cudaStream_t st);  // the relay build gathers through a texture object
int k2_prepare(int device);
int k2_launch(const K2Args &a, int variant, int sms, size_t smem_bytes, cudaStream_t st);
size_t k2_relay_fixed_smem();
int k2_relay_prepare();
int k2_relay_launch(const K2Args &a, bool check, int sms, size_t smem_bytes, cudaStream_t st);
size_t k2_layers_fixed_smem(int n_sel);
int k2_layers_prepare();
int k2_layers_launch(const K2Args &a, const K2Layers &L, bool check, int sms, size_t smem_bytes, cudaStream_t st);
// pre-combined fused layers (k2_layers_pre.cu)
int k1_layer_occ_build(const K2Args &a, const K2Layers &L, double *d_occ, int sms, cudaStream_t st);
int k2_layers_pre_prepare();
int k2_layers_pre_launch(const K2Args &a, const K2Layers &L, bool check, int sms, cudaStream_t st);

}  // namespace are
