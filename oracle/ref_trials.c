/*
 * oracle/ref_trials.c -- CPU restatement of the reference hot loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path; it is linked only by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs.  The product (paper_1308_2066_b200)
 * never loads it.
 *
 * Restates /root/reference/pkg/src/aggrisk/engine/_kernel.pyx:17-119
 * (`run_trials`) operation for operation:
 *   - per occurrence: comb = sum over selected tables, in selection order,
 *     of share * clamp(rate * x - ret, 0, lim)              (_kernel.pyx:66-77)
 *   - occurrence terms: clamp(comb - occ_ret, 0, occ_lim)   (_kernel.pyx:78-83)
 *   - c += occ, trial order, starting from 0.0              (_kernel.pyx:83)
 *   - aggregate terms on the trial total                    (_kernel.pyx:113-118)
 * Clamps are two `if`s (NaN passes through), exactly as the reference.
 * The chunked branch (_kernel.pyx:84-112) stages blocks through scratch; its
 * arithmetic is identical, and it is kept so the chunk parameter has the
 * reference meaning.  Build with -O3 -ffp-contract=off, the reference's own
 * flags (pkg/setup.py:9), so no FMA contraction changes the rounding.
 *
 * Parity pinning: tests/test_oracle.py checks this file against golden
 * vectors written by tests/golden/make_golden.py from the reference package
 * itself (worked example, 1000 random oracle instances, seed-31 digest).
 */
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_MAX_TABLES 256 /* _kernel.pyx:14 */

static inline double clamp_like_reference(double v, double hi)
{
    if (v < 0.0) v = 0.0;
    if (v > hi) v = hi;
    return v;
}

static inline double combined_loss(const double *const *tab, uint32_t e, int64_t n_tab,
                                   const double *rate, const double *ret,
                                   const double *lim, const double *share)
{
    double comb = 0.0;
    for (int64_t j = 0; j < n_tab; ++j) {
        double l = rate[j] * tab[j][e] - ret[j];
        l = clamp_like_reference(l, lim[j]);
        comb += share[j] * l;
    }
    return comb;
}

/* Returns the lookup count (n_sel * occurrences), or -1 on a bad argument
 * (the reference raises ValueError for the same conditions, _kernel.pyx:49-52). */
long long oracle_run_trials(const uint32_t *event_ids, const int64_t *offsets,
                            const double *stacked, int64_t row_len,
                            const int64_t *rows, int64_t n_tab,
                            const double *fin_rate, const double *fin_ret,
                            const double *fin_lim, const double *fin_share,
                            double occ_ret, double occ_lim,
                            double agg_ret, double agg_lim,
                            int64_t chunk, int64_t first_trial, int64_t last_trial,
                            double *out, double *scratch, int64_t scratch_len)
{
    const double *tab[ORACLE_MAX_TABLES];
    long long lookups = 0;
    if (n_tab > ORACLE_MAX_TABLES) return -1;
    if (chunk > 0 && scratch_len < chunk) return -1;
    for (int64_t j = 0; j < n_tab; ++j) tab[j] = stacked + rows[j] * row_len;

    for (int64_t t = first_trial; t < last_trial; ++t) {
        const int64_t lo = offsets[t], hi = offsets[t + 1];
        double c = 0.0;
        if (chunk <= 0) {
            for (int64_t i = lo; i < hi; ++i) {
                double comb = combined_loss(tab, event_ids[i], n_tab,
                                            fin_rate, fin_ret, fin_lim, fin_share);
                lookups += n_tab;
                c += clamp_like_reference(comb - occ_ret, occ_lim);
            }
        } else {
            for (int64_t i = lo; i < hi; i += chunk) {
                int64_t blk = hi - i < chunk ? hi - i : chunk;
                for (int64_t b = 0; b < blk; ++b)
                    scratch[b] = combined_loss(tab, event_ids[i + b], n_tab,
                                               fin_rate, fin_ret, fin_lim, fin_share);
                lookups += blk * n_tab;
                for (int64_t b = 0; b < blk; ++b)
                    scratch[b] = clamp_like_reference(scratch[b] - occ_ret, occ_lim);
                for (int64_t b = 0; b < blk; ++b) c += scratch[b];
            }
        }
        out[t] = clamp_like_reference(c - agg_ret, agg_lim);
    }
    return lookups;
}

/* Scalar term helpers (engine/__init__.py:109-121), exported so the tests can
 * run the reference's term KATs through the same compiled arithmetic. */
double oracle_financial_terms(double loss, double rate, double ret, double lim, double share)
{
    return share * clamp_like_reference(rate * loss - ret, lim);
}

double oracle_occurrence_terms(double loss, double occ_ret, double occ_lim)
{
    return clamp_like_reference(loss - occ_ret, occ_lim);
}
