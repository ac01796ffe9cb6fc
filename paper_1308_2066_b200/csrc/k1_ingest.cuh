#pragma once
#include "common.cuh"

namespace are {

struct PlanBuffers {
    Slot *slots = nullptr;       // row_len records
    Entry *ovf = nullptr;        // overflow entries
    uint32_t *filter = nullptr;  // filter_words (+4 pad) words
    int64_t filter_words = 0;
    int64_t hot_events = 0;
    int64_t entries = 0;
    int64_t overflow_entries = 0;
};

// Relay-kernel buffers of a plan (k1_build_relay / k2_relay.cu).
struct RelayBuffers {
    RSlot *rslots = nullptr;     // row_len records
    double *rovf = nullptr;      // fin-applied overflow values (same indexing as PlanBuffers::ovf)
    int64_t filter_words = 0;    // words of each per-terms filter (k1_relay_filter)
    cudaTextureObject_t tex = 0; // rslots as uint4 texels (gathers through the texture pipe)
    void release() {
        if (tex) cudaDestroyTextureObject(tex);
        tex = 0;
        cudaFree(rslots);
        cudaFree(rovf);
        rslots = nullptr;
        rovf = nullptr;
    }
};

int k1_build_layer_records(const PlanBuffers &pb, const Fin *d_fin, int64_t row_len, LRec **out, int sms,
                           cudaStream_t st);
int k1_build_relay(const PlanBuffers &pb, const Fin *d_fin, int64_t row_len, int64_t filter_bits, RelayBuffers &rb,
                   int sms, cudaStream_t st, bool precombined = false);

// The relay filter for one pair of occurrence terms: bit b set iff some
// event e with hash(e) == b has an occurrence value that is not +-0 under
// (occ_ret, occ_lim); words must hold (nbits + 31) / 32 (+4 pad) words.
int k1_relay_filter(const RelayBuffers &rb, int64_t row_len, int64_t nbits, double occ_ret, double occ_lim,
                    uint32_t *words, int sms, cudaStream_t st);

int k1_scatter(const uint32_t *d_ids, const double *d_losses, const int64_t *d_table_offsets,
               int64_t n_tables, int64_t max_records, int64_t row_len, double *d_stacked,
               int sms, cudaStream_t st);

int k1_build_plan(const double *d_stacked, int64_t row_len, const int64_t *d_rows, int n_sel,
                  int64_t filter_bits, PlanBuffers &pb, int sms, cudaStream_t st);

int k1_precombine_plan(PlanBuffers &pb, const Fin *d_fin, int64_t row_len, int sms, cudaStream_t st);

// Event-major copy of the selected rows for the dense kernel:
// em[e * stride + s] = stacked[rows[s] * row_len + e] (s < n_sel; pad = 0).
int k1_event_major(const double *d_stacked, int64_t row_len, const int64_t *d_rows, int n_sel, int stride,
                   double *d_em, int sms, cudaStream_t st);

int scan_exclusive_u32(const uint32_t *d_in, uint32_t *d_out, int64_t n, uint64_t *d_tiles,
                       uint64_t *h_total, cudaStream_t st);

}  // namespace are
