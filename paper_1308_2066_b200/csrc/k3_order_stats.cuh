#pragma once
#include "common.cuh"

namespace are {

int order_stat_k(int64_t n, double rp, int64_t *k);
// PML/TVaR per return period; with `summary` (2 doubles) also the mean and
// the maximum of the table from the same tail pass.
int k3_order_stats(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                   double *tvar_out, int sms, cudaStream_t st, double *summary = nullptr);
// Asynchronous form for pipelined callers: <= 8 return periods, results
// written to the device buffer d_res (pml[r] at r, tvar[r] at 8 + r) on
// `st`, at most `max_ctas` CTAs (0: the full grid), no host sync.  Calls must
// be ordered on one stream per device (one shared workspace).
int k3_order_stats_async(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *d_res, int sms,
                         int max_ctas, cudaStream_t st);
// PML only, for many return periods at once (EP curves): one device sort of
// the order-preserving keys, then one gather of every rank.
int k3_pml_sorted(const double *d_x, int64_t n, const double *rps, int64_t n_rp, double *pml_out, int sms,
                  cudaStream_t st);
int k3_rollup_launch(const double *const *d_ylts_host_array, int64_t n_layers, int64_t n, double *d_out,
                     int sms, cudaStream_t st);

}  // namespace are
