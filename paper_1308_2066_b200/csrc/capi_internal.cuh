// Internal definitions shared by the C-ABI translation units (capi.cu,
// capi_group.cu).  Not part of the public header include/aggrisk_b200.h.
#pragma once
#include <atomic>
#include <mutex>

#include "common.cuh"
#include "k1_ingest.cuh"
#include "k2_trials.cuh"

namespace are {

struct DeviceInfo {
    int sms = 0;
    int smem_optin = 0;
    bool ready = false;
};
// Sets `dev` current on the calling thread and prepares it once (kernel
// attributes); callers that must not leak the switch hold a DeviceGuard.
int use_device(int dev, DeviceInfo **out);

// Restores the calling thread's current device when the scope ends: every
// entry point that switches devices holds one, so a call on a plan or table
// of another GPU never changes the caller's (e.g. torch's) current device.
struct DeviceGuard {
    int prev = -1;
    DeviceGuard() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};

// Host -> host copy on several threads (pageable -> pinned staging).
void parallel_copy(void *dst, const void *src, size_t bytes);
// 1 when `p` is page-locked host memory (cached per registered range).
bool is_pinned(const void *p);

}  // namespace are

struct are_tables_s {
    int device = 0;
    int64_t n_tables = 0, row_len = 0;
    double *d = nullptr;
    std::atomic<int> refs{1};
};

struct are_plan_s {
    int device = 0;
    are_tables_s *tab = nullptr;
    int64_t n_sel = 0;
    int64_t *d_rows = nullptr;
    are::Fin *d_fin = nullptr;
    are::PlanBuffers pb;
    int64_t nbits = 0;
    int hash_mode = 0;
    bool zero_skip = false;
    bool slot0_hot = false;
    bool pool = false;
    bool precombined = false;
    unsigned int *d_err = nullptr;
    size_t smem = 0;
    // event-major copy of the selected rows for the dense kernel (built on
    // its first use; n_sel <= EM_MAX_SEL)
    std::mutex em_mu;
    double *d_em = nullptr;
    int32_t em_stride = 0;
    bool em_tried = false;
    // relay-kernel records and filter (k1_build_relay), built on first use
    std::mutex relay_mu;
    are::RelayBuffers rb;
    are::LRec *d_lrec = nullptr;  // fused-layer records (pool plans), built on first layered launch
    int64_t rnbits = 0;
    int rhash_mode = 0;
    size_t rsmem = 0;
    bool relay_tried = false;
    // per occurrence terms: the filter of the events whose occurrence value
    // is not +-0 (k1_relay_filter); a few recent terms kept, LRU
    struct OccFilter {
        uint64_t ret_bits = 0, lim_bits = 0, stamp = 0;
        uint32_t *d = nullptr;
    };
    static constexpr int OCC_FILTERS = 4;
    OccFilter occf[OCC_FILTERS];
    uint64_t occ_clock = 0;
};


namespace are {
int simulate_range(are_plan_s *p, const uint32_t *ids, int64_t id_base, int64_t n_ids, const int64_t *off,
                   int64_t t_base, int64_t first, int64_t last, double mean_len, double occ_ret, double occ_lim,
                   double agg_ret, double agg_lim, double *out, int64_t out_base, unsigned int *d_err,
                   cudaStream_t st, int32_t variant);
}  // namespace are
