/*
 * aggrisk_b200.h -- C ABI of the B200 aggregate-analysis engine
 * (libaggrisk_b200.so, built from paper_1308_2066_b200/csrc/).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary
 * (`void *stream` is a cudaStream_t, 0 = the legacy default stream).
 * Every entry point returns an `are_status` and records a thread-local
 * message readable through are_last_error().
 *
 * The reference seam this library replaces is the backend module's
 * `run_trials` (reference: pkg/src/aggrisk/engine/_kernel.pyx:17-30, chosen
 * by _backend_module at pkg/src/aggrisk/engine/__init__.py:147-148 and
 * called from _run_layer.task :179-191 and analyse_trial :313-319), together
 * with the table build it consumes (TableSet.from_elts, tables.py:95-117)
 * and the order statistics downstream of it (metrics.py:29-115).  The
 * one-to-one mapping is given per function below; INTEGRATION.md shows the
 * ctypes binding a maintainer adds on the reference side.
 *
 * Ownership: the caller owns every host buffer and every device buffer it
 * passes in; the library only borrows them for the duration of the call.
 * Handles (are_tables_t, are_plan_t) own device memory and are freed with
 * their *_free call.  Handles are immutable after construction and may be
 * used from several host threads at once (the reference kernel is
 * re-entrant; so is this library).
 */
#ifndef AGGRISK_B200_H
#define AGGRISK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    ARE_OK = 0,
    ARE_EINVAL = 1,      /* reference raises ValueError           */
    ARE_ERANGE = 2,      /* reference raises EventOutOfRangeError */
    ARE_ECUDA = 3,       /* CUDA runtime failure (no device, launch error ...) */
    ARE_ENOMEM = 4,      /* device or pinned-host allocation failed */
    ARE_EINDEX = 5       /* reference raises IndexError (bad selection row) */
} are_status;

#define ARE_MAX_TABLES 256 /* reference: _kernel.pyx:14 (MAX_TABLES) */

/* K2 variant selector for are_simulate_* */
#define ARE_VARIANT_AUTO 0   /* hot-set kernel when zero-skip is exact and the plan
                                is not dense-overlap (>= 3.5 entries per catalog
                                event, 4-32 rows), else dense */
#define ARE_VARIANT_HOTSET 1 /* force the hot-set kernel (fails if not exact)      */
#define ARE_VARIANT_DENSE 2  /* force the dense direct-access kernel              */
/* OR-able flag: the caller guarantees every event id of the YET is < row_len
 * (validated once, e.g. by validate_portfolio); K2 then skips its per-id
 * range check.  Without it an out-of-catalog id raises ARE_ERANGE. */
#define ARE_FLAG_IDS_VALIDATED 0x100
/* OR-able field for are_simulate_device: the persistent K2 grid leaves k SMs
 * (0..255) free, so work queued on another stream (a pipelined caller's K3
 * of the previous batch, its YLT exchange) runs beside it instead of after. */
#define ARE_SPARE_SMS(k) ((int32_t)(k) << 12)

typedef struct are_tables_s *are_tables_t;
typedef struct are_plan_s *are_plan_t;
typedef struct are_layer_table_s *are_layer_table_t;
typedef struct are_yet_s *are_yet_t;

typedef struct {
    int64_t n_sel;            /* selected tables (accumulation order)            */
    int64_t row_len;          /* catalog_size + 1                                 */
    int64_t hot_events;       /* events with >= 1 non-zero loss in the selection  */
    int64_t entries;          /* non-zero (event, table) pairs                    */
    int64_t overflow_entries; /* entries beyond the first per event               */
    int64_t filter_bits;      /* bits of the shared-memory hot filter             */
    int64_t device_bytes;     /* device memory owned by the plan                  */
    int32_t zero_skip_exact;  /* every fin_j(+-0) == +-0 (hot-set kernel usable)  */
    int32_t smem_bytes;       /* dynamic shared memory of the hot-set kernel      */
    int64_t relay_filter_bits; /* bits of the relay kernel's per-terms filter (0: no relay records yet) */
    int32_t relay;            /* 1 when long-trial launches run k2_relay (records built on first use) */
    int32_t relay_smem_bytes; /* dynamic shared memory of k2_relay               */
} are_plan_info_t;

/* ---- library / device ------------------------------------------------ */
const char *are_last_error(void);
int are_version(void);
int are_device_count(int *n);
int are_select_device(int ordinal);
int are_device_sm_count(int *n);
/* Number of kernels this library launched in the calling process. */
int64_t are_launch_count(void);
/* Pin / unpin a caller-owned host buffer (cudaHostRegister) so the host
 * entry points copy from it without staging. */
int are_host_register(void *ptr, int64_t bytes);
int are_host_unregister(void *ptr);
/* 1 when `ptr` is page-locked host memory the copy engines can read directly. */
int are_host_is_pinned(const void *ptr);

/* ---- K1: ELT ingestion (replaces TableSet.from_elts, tables.py:95-117) -- */
/* Dense stacked float64 (n_tables, row_len), row-major, as TableSet.stacked. */
int are_tables_from_dense(const double *stacked, int64_t n_tables, int64_t row_len,
                          are_tables_t *out);
/* Sparse ELT records: table i owns ids/losses[table_offsets[i] .. [i+1]).
 * Ids must lie in [1, row_len-1] (else ARE_ERANGE, tables.py:111-114) and be
 * unique within a table. */
int are_tables_from_records(const uint32_t *ids, const double *losses,
                            const int64_t *table_offsets, int64_t n_tables,
                            int64_t row_len, are_tables_t *out);
int are_tables_info(are_tables_t t, int64_t *n_tables, int64_t *row_len,
                    int64_t *device_bytes);
/* Copy dense row `row` (row_len doubles) back to the host. */
int are_tables_read_row(are_tables_t t, int64_t row, double *host_out);
int are_tables_free(are_tables_t t);

/* ---- selection + financial terms (TableSet.selection_arrays, tables.py:133-153) */
int are_plan_build(are_tables_t t, const int64_t *rows, int64_t n_sel,
                   const double *fin_rate, const double *fin_ret,
                   const double *fin_lim, const double *fin_share,
                   are_plan_t *out);
/* Plan over an ELT pool for the fused multi-layer kernel (its filter is sized
 * for that kernel's shared-memory layout).  rows = the pool, in pool order. */
int are_plan_build_pool(are_tables_t t, const int64_t *rows, int64_t n_sel,
                        const double *fin_rate, const double *fin_ret,
                        const double *fin_lim, const double *fin_share,
                        are_plan_t *out);
/* Pre-combined plan: K1 folds each event's losses through
 * the financial terms once (comb = 0.0 + sum_j fin_j(x_j), selection order),
 * so K2 reads one value per hot event.  A different unit of work from the
 * per-lookup path -- reported separately, never as the headline. */
int are_plan_build_precombined(are_tables_t t, const int64_t *rows, int64_t n_sel,
                               const double *fin_rate, const double *fin_ret,
                               const double *fin_lim, const double *fin_share,
                               are_plan_t *out);
int are_plan_info(are_plan_t p, are_plan_info_t *info);
int are_plan_free(are_plan_t p);

/* ---- K2: per-trial simulation (replaces run_trials, _kernel.pyx:17-119) --
 * Trials [first, last) of a YET whose offsets are int64 (length T+1) and
 * whose event ids are uint32.  out[t] (float64) is written for t in range.
 *
 * Device form: d_event_ids[i] is occurrence i, d_offsets[t] is offset t,
 * d_out[t] is trial t (pointers may be offset by the caller as usual).
 * Launches on `stream`; does not synchronise.  Event ids >= row_len set a
 * device error flag that the next are_check_errors() reports (ARE_ERANGE). */
int are_simulate_device(are_plan_t p, const uint32_t *d_event_ids, int64_t n_occ,
                        const int64_t *d_offsets, int64_t n_trials,
                        int64_t first, int64_t last,
                        double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                        double *d_out, void *stream, int32_t variant);
int are_check_errors(are_plan_t p, void *stream);

/* Packed resident ids (a device data layout for a YET kept in HBM across
 * calls, as the reference's pricing sessions keep theirs, service.py:169-188):
 * three 21-bit ids per 64-bit word, 96-id blocks of 32 words, word l of block
 * b holding occurrences 96b+l, 96b+32+l, 96b+64+l (bits 0-20, 21-41, 42-62;
 * zero past n_occ).  are_packed_id_words(n) = words to allocate (2/3 of the
 * uint32 bytes).  are_yet_pack_device builds it on `stream` from validated
 * ids; an id >= 2^21 ORs 1 into *d_flag (nullable).
 * are_simulate_device_packed = are_simulate_device reading d_packed instead
 * of d_event_ids when the relay kernel runs with ARE_FLAG_IDS_VALIDATED and
 * the plan's catalogue is below 2^21 (otherwise it reads d_event_ids);
 * results are bit-identical either way. */
int64_t are_packed_id_words(int64_t n_occ);
int are_yet_pack_device(int32_t device, const uint32_t *d_event_ids, int64_t n_occ,
                        uint64_t *d_packed, uint32_t *d_flag, void *stream);
int are_simulate_device_packed(are_plan_t p, const uint32_t *d_event_ids, const uint64_t *d_packed,
                               int64_t n_occ, const int64_t *d_offsets, int64_t n_trials,
                               int64_t first, int64_t last,
                               double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                               double *d_out, void *stream, int32_t variant);

/* Fused multi-layer K2 (replaces the per-layer loop of
 * run_aggregate_analysis_with_stats, engine/__init__.py:242-253).  `p` is a
 * pool plan (are_plan_build_pool, <= 64 tables); layer l selects the pool rows
 * in bit mask masks[l] (its selection order must be increasing pool order) and
 * has terms layer_terms[4l..4l+3] = (occ_ret, occ_lim, agg_ret, agg_lim).
 * n_layers <= 16.  Writes d_out[l * out_stride + t] for t in [first, last).
 * Each layer's result is bit-identical to a single-layer run. */
int are_simulate_layers_device(are_plan_t p, int32_t n_layers, const uint64_t *masks,
                               const double *layer_terms,
                               const uint32_t *d_event_ids, int64_t n_occ,
                               const int64_t *d_offsets, int64_t n_trials,
                               int64_t first, int64_t last,
                               double *d_out, int64_t out_stride, void *stream, int32_t flags);

/* Pre-combined fused layers (SURVEY 8(f) rows 2 + 4; a separately reported
 * work unit): are_layer_table_build evaluates, once per (pool plan, masks,
 * layer terms), every hot event's occurrence value in every layer -- the
 * float64 sequence of are_simulate_layers_device -- into a device table of
 * 16 doubles per event id; are_simulate_layers_precombined then streams the
 * ids and folds one table line per candidate event.  Bit-identical results.
 * The plan must outlive the table.  Same arguments and errors as
 * are_simulate_layers_device. */
int are_layer_table_build(are_plan_t p, int32_t n_layers, const uint64_t *masks,
                          const double *layer_terms, void *stream, are_layer_table_t *out);
int are_layer_table_free(are_layer_table_t t);
int are_simulate_layers_precombined(are_layer_table_t t, const uint32_t *d_event_ids, int64_t n_occ,
                                    const int64_t *d_offsets, int64_t n_trials,
                                    int64_t first, int64_t last,
                                    double *d_out, int64_t out_stride, void *stream, int32_t flags);

/* Host form: host ids/offsets/out; the library streams trial chunks to the
 * device (overlapping copies with K2) and returns when `out` is filled.
 * *lookups = n_sel * (offsets[last] - offsets[first]) exactly as the
 * reference counts them (_kernel.pyx:77). */
int are_simulate_host(are_plan_t p, const uint32_t *event_ids, int64_t n_occ,
                      const int64_t *offsets, int64_t n_trials,
                      int64_t first, int64_t last,
                      double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                      double *out, int64_t *lookups, int32_t variant);

/* Drop-in for the reference run_trials with its exact argument list
 * (_kernel.pyx:17-30).  `chunk` and `scratch` keep their reference meaning
 * for validation only (chunk > 0 requires scratch_len >= chunk,
 * _kernel.pyx:51-52); results do not depend on them.  Uploads `stacked`
 * on every call -- use the tables/plan handles to keep it resident. */
int are_run_trials(const uint32_t *event_ids, int64_t n_occ,
                   const int64_t *offsets, int64_t n_offsets,
                   const double *stacked, int64_t n_tables, int64_t row_len,
                   const int64_t *rows, int64_t n_sel,
                   const double *fin_rate, const double *fin_ret,
                   const double *fin_lim, const double *fin_share,
                   double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                   int64_t chunk, int64_t first_trial, int64_t last_trial,
                   double *out, int64_t scratch_len, int64_t *lookups);

/* ---- K0: YET validation (replaces the YET half of validate_portfolio,
 * model.py:371-395).  Scans ids [0, n_ids) of d_ids, the n_trials trials of
 * d_offsets (absolute occurrence indices; trial k of the slice is trial
 * t_base + k) and, when d_ts is non-null, their timestamps (d_ts[i - ts_base]
 * is occurrence i).  Slices may be validated piecewise and the reports merged. */
typedef struct {
    uint32_t min_id, max_id;   /* over the scanned ids                         */
    int64_t bad_trials;        /* trials with length outside [1, max_len]      */
    int64_t first_bad_trial;   /* lowest such trial index, -1 if none          */
    int64_t unsorted;          /* timestamp drops strictly inside a trial      */
    int64_t ts_nan;            /* NaN timestamps (numpy min/max propagate NaN) */
    double ts_min, ts_max;     /* over the non-NaN timestamps                  */
    int32_t ts_checked;
} are_yet_report_t;
int are_validate_yet_device(const uint32_t *d_ids, int64_t n_ids,
                            const int64_t *d_offsets, int64_t n_trials, int64_t t_base,
                            const double *d_ts, int64_t ts_base, int64_t max_len,
                            are_yet_report_t *out, void *stream);

/* ---- K3: order statistics (replaces pml/tvar/ep_curve, metrics.py:29-115) --
 * For each return period rp[r]: k = n - floor(n / rp) (metrics.py:40),
 * pml[r] = k-th smallest loss, tvar[r] = mean of the top n-k+1 losses.
 * Requires 1 < rp <= n (ARE_EINVAL otherwise, metrics.py:36-39). */
int are_order_stats_device(const double *d_losses, int64_t n,
                           const double *rps, int64_t n_rp,
                           double *pml_out, double *tvar_out, void *stream);
int are_order_stats_host(const double *losses, int64_t n,
                         const double *rps, int64_t n_rp,
                         double *pml_out, double *tvar_out);
/* Asynchronous form for pipelined callers (no host synchronisation): 1..8
 * return periods; d_res (device, 16 doubles) receives pml[r] at r and
 * tvar[r] at 8 + r, stream-ordered on `stream`; at most max_ctas CTAs
 * (0: the full grid; 1-2 fit beside a K2 launched with ARE_FLAG_SPARE_SM).
 * Calls must be ordered on one stream per device. */
int are_order_stats_async(const double *d_losses, int64_t n, const double *rps, int64_t n_rp, double *d_res,
                          int32_t max_ctas, void *stream);
/* are_order_stats_device plus the table's mean and maximum from the same
 * tail pass: mean_max_out[0] = sum / n (double-double sum), mean_max_out[1] =
 * max (NaN if any loss is NaN), as the pricing service reports them
 * (service.py:237-238). */
int are_order_stats_summary_device(const double *d_losses, int64_t n,
                                   const double *rps, int64_t n_rp,
                                   double *pml_out, double *tvar_out,
                                   double *mean_max_out, void *stream);
/* PML only, for many return periods at once (ep_curve, metrics.py:97-115):
 * one device radix sort of the order-preserving keys, then one gather. */
int are_pml_many_device(const double *d_losses, int64_t n,
                        const double *rps, int64_t n_rp,
                        double *pml_out, void *stream);
/* portfolio_rollup (metrics.py:118-133): d_out[t] = ((y0[t] + y1[t]) + ...). */
int are_rollup_device(const double *const *d_ylts, int64_t n_layers, int64_t n,
                      double *d_out, void *stream);


/* ---- multi-GPU group ----------------------
 * Replaces the reference's worker pool over trial ranges
 * (pkg/src/aggrisk/engine/__init__.py:193-200, _split_by_events :151-159):
 * a request with worker_count > 1 becomes ONE call covering every GPU of the
 * group.  The caller computes the trial -> GPU partition with the reference
 * rule (split_by_events(offsets, G)) and passes it as `bounds` (G + 1 trial
 * cut points); shard s lives on group member s.  Tables are replicated
 * (are_tables_replicate) and planned per GPU; plans[s] must live on shard
 * s's GPU.  Every trial is computed by one warp on one GPU, so the YLT is
 * bit-identical for any group size.  Handles are thread-safe; one layer run
 * at a time per YET handle (internal mutex). */
/* Group = CUDA devices 0..n_gpus-1 (n_gpus <= 0: every visible device). */
int are_init(int n_gpus);
/* Group of explicit ordinals (a device may repeat: several shards on one GPU). */
int are_init_devices(const int *ordinals, int32_t n);
int are_shutdown(void);
int are_group_size(int32_t *n);
int are_group_device(int32_t member, int *ordinal);
int are_tables_device(are_tables_t t, int *device);
int are_plan_device(are_plan_t p, int *device);
/* Copy a table set into another GPU's memory (peer copy). */
int are_tables_replicate(are_tables_t t, int device, are_tables_t *out);
/* Host YET -> HBM, one shard per group member (uploaded concurrently, pinned
 * staging for pageable inputs), validated on the device by K0: ids, trial
 * lengths in [1, max_len] and, when `timestamps` is non-null, the timestamp
 * checks of validate_portfolio (model.py:371-395).  The merged report is
 * read with are_yet_report. */
int are_yet_upload(const uint32_t *ids, int64_t n_occ, const int64_t *offsets, int64_t n_trials,
                   const double *timestamps, const int64_t *bounds, int32_t n_shards, int64_t max_len,
                   are_yet_t *out);
int are_yet_report(are_yet_t y, are_yet_report_t *out);
int are_yet_shards(are_yet_t y, int32_t *n_shards, int64_t *bounds, int *devices);
int are_yet_free(are_yet_t y);
/* K2 over trials [first, last) on every shard's GPU at once (the reference's
 * _run_layer, engine/__init__.py:162-201); out_host[t] for t in range,
 * *lookups = n_sel * occurrences.  With n_rp > 0 (whole table only) the
 * YLT is gathered into the first member's HBM and K3 evaluates pml/tvar
 * there (metrics.py:29-63): with peer access every shard's K2 stores its
 * trials straight into that table (the gather fused into the simulation),
 * else the slices are peer-copied.  out_host may be NULL. */
int are_run_layer(are_yet_t y, const are_plan_t *plans, int32_t n_plans,
                  double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                  int64_t first, int64_t last, double *out_host, int64_t *lookups, int32_t variant,
                  const double *rps, int64_t n_rp, double *pml_out, double *tvar_out);
/* Host-YET form: shard s streams its trials to its GPU over that GPU's own
 * PCIe link (are_simulate_host per shard, concurrently). */
int are_run_layer_host(const uint32_t *ids, int64_t n_occ, const int64_t *offsets, int64_t n_trials,
                       const int64_t *bounds, int32_t n_shards, const are_plan_t *plans,
                       double occ_ret, double occ_lim, double agg_ret, double agg_lim,
                       int64_t first, int64_t last, double *out, int64_t *lookups, int32_t variant);

#ifdef __cplusplus
}
#endif
#endif /* AGGRISK_B200_H */
