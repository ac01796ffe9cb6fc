// Multi-GPU C ABI (include/aggrisk_b200.h, "multi-GPU group"): the device
// group, the sharded HBM-resident year event table and the one-call layer run
// that covers every GPU.
//
// The reference turns `worker_count` into contiguous, occurrence-balanced
// trial ranges (_split_by_events, pkg/src/aggrisk/engine/__init__.py:151-159)
// and runs them on a thread pool (:193-200).  Here the same ranges (computed
// by the caller with that exact rule and passed down as `bounds`) are the
// trial -> GPU partition: shard s of a YET lives in the HBM of group GPU s,
// the tables are replicated, K2 runs on every GPU at once, and each GPU's
// YLT slice lands in its own disjoint range of the caller's output (there is
// nothing to reduce: every trial is computed by one warp on one GPU, so the
// YLT is bit-identical for any number of GPUs).  When order statistics are
// requested the slices are gathered into the first GPU's memory with peer
// copies (NVLink / NVSwitch) and K3 runs there.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.cuh"
#include "k3_order_stats.cuh"

namespace are {

struct Group {
    std::mutex mu;
    std::vector<int> devices;            // group member s -> CUDA ordinal (may repeat: shards sharing a GPU)
};
static Group g_group;

static int group_members(std::vector<int> &devs) {
    std::lock_guard<std::mutex> g(g_group.mu);
    if (g_group.devices.empty()) return fail(ARE_EINVAL, "multi-GPU group not initialised (call are_init)");
    devs = g_group.devices;
    return ARE_OK;
}

static void group_clear() { g_group.devices.clear(); }

// Runs fn(s) for every shard on its own host thread (the shards' uploads and
// host-side staging are independent); returns the first non-OK status.  The
// thread-local error message of a failing shard is carried to the caller.
template <class F>
static int for_each_shard(int n, F fn) {
    if (n == 1) return fn(0);
    std::vector<int> rc(n, ARE_OK);
    std::vector<std::string> msg(n);
    std::vector<std::thread> th;
    th.reserve(n);
    try {
        for (int s = 0; s < n; ++s)
            th.emplace_back([&, s] {
                rc[s] = fn(s);
                if (rc[s]) msg[s] = are_last_error();
            });
    } catch (...) {  // no threads: run the rest here
        for (int s = (int)th.size(); s < n; ++s) {
            rc[s] = fn(s);
            if (rc[s]) msg[s] = are_last_error();
        }
    }
    for (auto &t : th) t.join();
    for (int s = 0; s < n; ++s)
        if (rc[s]) return fail(rc[s], "shard " + std::to_string(s) + ": " + msg[s]);
    return ARE_OK;
}

}  // namespace are

using namespace are;

// One shard of a sharded YET: trials [t0, t1) and their occurrences
// [o0, o1) in the HBM of `device`.
struct YetShard {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t t0 = 0, t1 = 0, o0 = 0, o1 = 0;
    uint32_t *d_ids = nullptr;    // occurrences o0 .. o1 (+4 zero ids of padding)
    int64_t *d_off = nullptr;     // offsets t0 .. t1 (absolute occurrence indices)
    double *d_out = nullptr;      // the shard's YLT slice
    unsigned int *d_err = nullptr;
    cudaEvent_t done = nullptr;   // the shard's K2 has finished (fused gather)
    are_yet_report_t rep{};
};

struct are_yet_s {
    std::mutex mu;  // one layer run at a time per table (the slices are per handle)
    int64_t n_trials = 0, n_occ = 0;
    std::vector<int64_t> offsets;  // host copy (lookup counts, ranges)
    std::vector<int64_t> bounds;
    std::vector<YetShard> shards;
    double *d_full = nullptr;  // gathered YLT on shard 0's device (K3), allocated on first use
    int ts_checked = 0;
};

static void yet_release(are_yet_s *y) {
    if (!y) return;
    DeviceGuard dg;
    for (auto &sh : y->shards) {
        cudaSetDevice(sh.device);
        cudaFree(sh.d_ids);
        cudaFree(sh.d_off);
        cudaFree(sh.d_out);
        cudaFree(sh.d_err);
        if (sh.stream) cudaStreamDestroy(sh.stream);
        if (sh.done) cudaEventDestroy(sh.done);
    }
    if (!y->shards.empty() && y->d_full) {
        cudaSetDevice(y->shards[0].device);
        cudaFree(y->d_full);
    }
    delete y;
}

// Host -> device copy of `bytes` from a possibly pageable host range: pinned
// sources go straight to the copy engine; pageable ones are staged through
// two pinned buffers filled by host threads while the other drains.
static int upload(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (!bytes) return ARE_OK;
    if (is_pinned(src)) {
        ARE_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        ARE_CUDA(cudaStreamSynchronize(st));
        return ARE_OK;
    }
    constexpr size_t CH = 64u << 20;
    void *buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int rc = ARE_OK;
    for (int i = 0; i < 2 && rc == ARE_OK; ++i) {
        cudaError_t e = cudaHostAlloc(&buf[i], std::min(CH, bytes), cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) rc = cuda_fail(e, "pinned staging buffer");
    }
    for (size_t a = 0, i = 0; rc == ARE_OK && a < bytes; a += CH, ++i) {
        const size_t n = std::min(CH, bytes - a);
        const int b = (int)(i & 1);
        cudaError_t e = cudaEventSynchronize(ev[b]);  // buffer b drained by its last copy
        if (e == cudaSuccess) {
            parallel_copy(buf[b], (const char *)src + a, n);
            e = cudaMemcpyAsync((char *)dst + a, buf[b], n, cudaMemcpyHostToDevice, st);
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev[b], st);
        if (e != cudaSuccess) rc = cuda_fail(e, "staged upload");
    }
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == ARE_OK) rc = cuda_fail(cudaGetLastError(), "upload");
    for (int i = 0; i < 2; ++i) {
        if (buf[i]) cudaFreeHost(buf[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
    }
    return rc;
}

extern "C" {

int are_init_devices(const int *ordinals, int32_t n) {
    if (n < 1 || !ordinals) return fail(ARE_EINVAL, "a group needs at least one device");
    int count = 0;
    ARE_CUDA(cudaGetDeviceCount(&count));
    for (int i = 0; i < n; ++i)
        if (ordinals[i] < 0 || ordinals[i] >= count) return fail(ARE_EINVAL, "bad device ordinal in group");
    DeviceGuard dg;
    std::lock_guard<std::mutex> g(g_group.mu);
    group_clear();
    for (int i = 0; i < n; ++i) {
        DeviceInfo *di;
        const int rc = use_device(ordinals[i], &di);
        if (rc) {
            group_clear();
            return rc;
        }
        g_group.devices.push_back(ordinals[i]);
    }
    // peer access from the first member (K3's gather target) to the others
    for (int i = 1; i < n; ++i) {
        if (ordinals[i] == ordinals[0]) continue;
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, ordinals[0], ordinals[i]);
        if (ok) {
            cudaSetDevice(ordinals[0]);
            const cudaError_t e = cudaDeviceEnablePeerAccess(ordinals[i], 0);
            if (e != cudaSuccess) cudaGetLastError();  // already enabled is fine
        }
    }
    return ARE_OK;
}

int are_init(int n_gpus) {
    int count = 0;
    ARE_CUDA(cudaGetDeviceCount(&count));
    if (count < 1) return fail(ARE_ECUDA, "no CUDA device visible");
    if (n_gpus <= 0 || n_gpus > count) n_gpus = count;
    std::vector<int> d(n_gpus);
    for (int i = 0; i < n_gpus; ++i) d[i] = i;
    return are_init_devices(d.data(), n_gpus);
}

int are_shutdown(void) {
    DeviceGuard dg;
    std::lock_guard<std::mutex> g(g_group.mu);
    group_clear();
    return ARE_OK;
}

int are_group_size(int32_t *n) {
    std::lock_guard<std::mutex> g(g_group.mu);
    *n = (int32_t)g_group.devices.size();
    return ARE_OK;
}

int are_group_device(int32_t member, int *ordinal) {
    std::lock_guard<std::mutex> g(g_group.mu);
    if (member < 0 || member >= (int32_t)g_group.devices.size()) return fail(ARE_EINVAL, "bad group member");
    *ordinal = g_group.devices[member];
    return ARE_OK;
}

int are_tables_device(are_tables_t t, int *device) {
    if (!t || !device) return fail(ARE_EINVAL, "null tables handle");
    *device = t->device;
    return ARE_OK;
}

int are_plan_device(are_plan_t p, int *device) {
    if (!p || !device) return fail(ARE_EINVAL, "null plan handle");
    *device = p->device;
    return ARE_OK;
}

int are_tables_replicate(are_tables_t t, int device, are_tables_t *out) {
    if (!t || !out) return fail(ARE_EINVAL, "null tables handle");
    DeviceGuard dg;
    DeviceInfo *di;
    int rc = use_device(device, &di);
    if (rc) return rc;
    auto *r = new are_tables_s();
    r->device = device;
    r->n_tables = t->n_tables;
    r->row_len = t->row_len;
    const size_t bytes = (size_t)std::max<int64_t>(t->n_tables, 1) * t->row_len * sizeof(double);
    cudaError_t e = cudaMalloc(&r->d, bytes);
    if (e == cudaSuccess) e = cudaMemcpyPeer(r->d, device, t->d, t->device, bytes);
    if (e != cudaSuccess) {
        cudaFree(r->d);
        delete r;
        return cuda_fail(e, "replicate tables");
    }
    *out = r;
    return ARE_OK;
}

int are_yet_upload(const uint32_t *ids, int64_t n_occ, const int64_t *offsets, int64_t n_trials,
                   const double *timestamps, const int64_t *bounds, int32_t n_shards, int64_t max_len,
                   are_yet_t *out) {
    if (!out || !offsets || n_trials < 0 || n_occ < 0) return fail(ARE_EINVAL, "bad year event table");
    *out = nullptr;
    if (offsets[n_trials] > n_occ) return fail(ARE_EINVAL, "offsets exceed the occurrence count");
    std::vector<int> devs;
    int rc = group_members(devs);
    if (rc) return rc;
    if (n_shards < 1 || n_shards > (int32_t)devs.size())
        return fail(ARE_EINVAL, "need 1..group size shards, got " + std::to_string(n_shards));
    if (bounds[0] != 0 || bounds[n_shards] != n_trials) return fail(ARE_EINVAL, "shard bounds must span every trial");
    for (int s = 0; s < n_shards; ++s)
        if (bounds[s + 1] < bounds[s]) return fail(ARE_EINVAL, "shard bounds must be non-decreasing");
    auto *y = new are_yet_s();
    y->n_trials = n_trials;
    y->n_occ = offsets[n_trials];
    y->offsets.assign(offsets, offsets + n_trials + 1);
    y->bounds.assign(bounds, bounds + n_shards + 1);
    y->shards.resize(n_shards);
    y->ts_checked = timestamps ? 1 : 0;
    for (int s = 0; s < n_shards; ++s) {
        YetShard &sh = y->shards[s];
        sh.device = devs[s];
        sh.t0 = bounds[s];
        sh.t1 = bounds[s + 1];
        sh.o0 = offsets[sh.t0];
        sh.o1 = offsets[sh.t1];
    }
    rc = for_each_shard(n_shards, [&](int s) -> int {
        YetShard &sh = y->shards[s];
        DeviceGuard g;
        DeviceInfo *di;
        int r = use_device(sh.device, &di);
        if (r) return r;
        ARE_CUDA(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));  // owned by the shard
        ARE_CUDA(cudaEventCreateWithFlags(&sh.done, cudaEventDisableTiming));
        const int64_t nid = sh.o1 - sh.o0, nt = sh.t1 - sh.t0;
        ARE_CUDA(cudaMalloc(&sh.d_ids, (nid + 4) * sizeof(uint32_t)));
        ARE_CUDA(cudaMalloc(&sh.d_off, (nt + 1) * sizeof(int64_t)));
        ARE_CUDA(cudaMalloc(&sh.d_out, std::max<int64_t>(nt, 1) * sizeof(double)));
        ARE_CUDA(cudaMalloc(&sh.d_err, sizeof(unsigned int)));
        ARE_CUDA(cudaMemsetAsync(sh.d_ids + nid, 0, 4 * sizeof(uint32_t), sh.stream));
        ARE_CUDA(cudaMemsetAsync(sh.d_err, 0, sizeof(unsigned int), sh.stream));
        if ((r = upload(sh.d_ids, ids + sh.o0, nid * sizeof(uint32_t), sh.stream))) return r;
        if ((r = upload(sh.d_off, offsets + sh.t0, (nt + 1) * sizeof(int64_t), sh.stream))) return r;
        // K0 over the shard: ids range, trial lengths, and the timestamps
        // (uploaded for the scan and dropped) when the caller has them
        double *d_ts = nullptr;
        if (timestamps && nid) {
            ARE_CUDA(cudaMalloc(&d_ts, nid * sizeof(double)));
            if ((r = upload(d_ts, timestamps + sh.o0, nid * sizeof(double), sh.stream))) {
                cudaFree(d_ts);
                return r;
            }
        }
        r = are_validate_yet_device(sh.d_ids, nid, sh.d_off, nt, sh.t0, d_ts, sh.o0, max_len, &sh.rep, sh.stream);
        if (d_ts) cudaFree(d_ts);
        return r;
    });
    if (rc) {
        yet_release(y);
        return rc;
    }
    *out = y;
    return ARE_OK;
}

int are_yet_report(are_yet_t y, are_yet_report_t *out) {
    if (!y || !out) return fail(ARE_EINVAL, "null yet handle");
    are_yet_report_t r{};
    r.min_id = 0xFFFFFFFFu;
    r.max_id = 0;
    r.first_bad_trial = -1;
    bool have_ts = false;
    for (const auto &sh : y->shards) {
        const are_yet_report_t &q = sh.rep;
        if (sh.o1 > sh.o0) {
            r.min_id = std::min(r.min_id, q.min_id);
            r.max_id = std::max(r.max_id, q.max_id);
        }
        r.bad_trials += q.bad_trials;
        if (q.bad_trials && (r.first_bad_trial < 0 || q.first_bad_trial < r.first_bad_trial))
            r.first_bad_trial = q.first_bad_trial;
        r.unsorted += q.unsorted;
        r.ts_nan += q.ts_nan;
        if (q.ts_checked && (sh.o1 - sh.o0) > q.ts_nan) {  // the shard has non-NaN timestamps
            r.ts_min = have_ts ? std::min(r.ts_min, q.ts_min) : q.ts_min;
            r.ts_max = have_ts ? std::max(r.ts_max, q.ts_max) : q.ts_max;
            have_ts = true;
        }
    }
    if (y->n_occ == 0) r.min_id = r.max_id = 0;
    r.ts_checked = y->ts_checked;
    *out = r;
    return ARE_OK;
}

int are_yet_shards(are_yet_t y, int32_t *n_shards, int64_t *bounds, int *devices) {
    if (!y || !n_shards) return fail(ARE_EINVAL, "null yet handle");
    *n_shards = (int32_t)y->shards.size();
    if (bounds) std::copy(y->bounds.begin(), y->bounds.end(), bounds);
    if (devices)
        for (size_t s = 0; s < y->shards.size(); ++s) devices[s] = y->shards[s].device;
    return ARE_OK;
}

int are_yet_free(are_yet_t y) {
    yet_release(y);
    return ARE_OK;
}

// Can kernels on `from` store into `to`'s memory?  Enables peer access once
// per pair (a process-wide setting; idempotent).
static bool peer_store_ok(int from, int to) {
    static std::mutex mu;
    static int state[64][64];  // 0 unknown, 1 ok, 2 no
    if (from < 0 || to < 0 || from >= 64 || to >= 64) return false;
    std::lock_guard<std::mutex> g(mu);
    if (!state[from][to]) {
        int can = 0;
        DeviceGuard dg;
        if (cudaDeviceCanAccessPeer(&can, from, to) == cudaSuccess && can) {
            cudaSetDevice(from);
            const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            state[from][to] = (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) ? 1 : 2;
            if (state[from][to] == 2) cudaGetLastError();
        } else {
            cudaGetLastError();
            state[from][to] = 2;
        }
    }
    return state[from][to] == 1;
}

int are_run_layer(are_yet_t y, const are_plan_t *plans, int32_t n_plans, double occ_ret, double occ_lim,
                  double agg_ret, double agg_lim, int64_t first, int64_t last, double *out_host, int64_t *lookups,
                  int32_t variant, const double *rps, int64_t n_rp, double *pml_out, double *tvar_out) {
    if (!y || !plans) return fail(ARE_EINVAL, "null handle");
    if (n_plans != (int32_t)y->shards.size()) return fail(ARE_EINVAL, "one plan per shard required");
    if (first < 0 || last < first || last > y->n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    const int64_t n_sel = plans[0]->n_sel;
    for (int s = 0; s < n_plans; ++s) {
        if (!plans[s]) return fail(ARE_EINVAL, "null plan handle");
        if (plans[s]->device != y->shards[s].device)
            return fail(ARE_EINVAL, "plan " + std::to_string(s) + " lives on another GPU than its shard");
        if (plans[s]->n_sel != n_sel) return fail(ARE_EINVAL, "plans select different table counts");
    }
    if (lookups) *lookups = n_sel * (y->offsets[last] - y->offsets[first]);
    if (n_rp > 0 && (first != 0 || last != y->n_trials))
        return fail(ARE_EINVAL, "order statistics need the whole year loss table");
    if (last == first) return ARE_OK;
    DeviceGuard dg;
    std::lock_guard<std::mutex> guard(y->mu);
    const double mean_len = (double)(y->offsets[last] - y->offsets[first]) / (double)(last - first);
    int rc = ARE_OK;
    YetShard &s0 = y->shards[0];
    // With return periods the YLT is gathered on shard 0's GPU for K3.  When
    // every shard's GPU can store into that GPU's memory (peer access over
    // NVLink, or the same device), the gather is fused into K2: each trial's
    // fold writes its loss straight into the gathered table, so the exchange
    // overlaps the simulation trial by trial and no copy follows it.
    bool fused = false;
    if (n_rp > 0) {
        ARE_CUDA(cudaSetDevice(s0.device));
        if (!y->d_full) ARE_CUDA(cudaMalloc(&y->d_full, y->n_trials * sizeof(double)));
        static const bool no_fuse = [] {  // ARE_GROUP_NO_FUSE=1: the peer-copy gather (A/B, tests)
            const char *e = getenv("ARE_GROUP_NO_FUSE");
            return e && e[0] == '1';
        }();
        fused = !no_fuse;
        for (auto &sh : y->shards)
            if (sh.t1 > sh.t0 && sh.device != s0.device && !peer_store_ok(sh.device, s0.device)) fused = false;
    }
    // K2 on every GPU (asynchronous launches), each into its slice (or, fused,
    // into the gathered table)
    for (auto &sh : y->shards) {
        const int64_t a = std::max(first, sh.t0), b = std::min(last, sh.t1);
        if (a >= b) continue;
        const int s = (int)(&sh - y->shards.data());
        if ((rc = simulate_range(plans[s], sh.d_ids, sh.o0, sh.o1 - sh.o0, sh.d_off, sh.t0, a, b, mean_len, occ_ret,
                                 occ_lim, agg_ret, agg_lim, fused ? y->d_full : sh.d_out, fused ? 0 : sh.t0,
                                 sh.d_err, sh.stream, variant)))
            return rc;
        ARE_CUDA(cudaSetDevice(sh.device));
        ARE_CUDA(cudaEventRecord(sh.done, sh.stream));
    }
    if (fused) {
        // shard 0's stream waits for every K2 (cross-device events), then one
        // copy of the gathered table to the caller and K3 on it
        ARE_CUDA(cudaSetDevice(s0.device));
        for (auto &sh : y->shards)
            if (sh.t1 > sh.t0 && &sh != &s0) ARE_CUDA(cudaStreamWaitEvent(s0.stream, sh.done, 0));
        if (out_host)
            ARE_CUDA(cudaMemcpyAsync(out_host + first, y->d_full + first, (last - first) * sizeof(double),
                                     cudaMemcpyDeviceToHost, s0.stream));
        unsigned int bad = 0;
        for (auto &sh : y->shards) {
            ARE_CUDA(cudaSetDevice(sh.device));
            unsigned int h = 0;
            ARE_CUDA(cudaMemcpyAsync(&h, sh.d_err, sizeof h, cudaMemcpyDeviceToHost, sh.stream));
            ARE_CUDA(cudaStreamSynchronize(sh.stream));
            if (h) ARE_CUDA(cudaMemsetAsync(sh.d_err, 0, sizeof(unsigned int), sh.stream));
            bad |= h;
        }
        if (bad) return fail(ARE_ERANGE, "event id outside the catalog in the year event table");
        DeviceInfo *di;
        if ((rc = use_device(s0.device, &di))) return rc;
        return k3_order_stats(y->d_full, y->n_trials, rps, n_rp, pml_out, tvar_out, di->sms, s0.stream);
    }
    for (auto &sh : y->shards) {
        const int64_t a = std::max(first, sh.t0), b = std::min(last, sh.t1);
        if (a >= b || !out_host) continue;
        ARE_CUDA(cudaSetDevice(sh.device));
        ARE_CUDA(cudaMemcpyAsync(out_host + a, sh.d_out + (a - sh.t0), (b - a) * sizeof(double),
                                 cudaMemcpyDeviceToHost, sh.stream));
    }
    unsigned int bad = 0;
    for (auto &sh : y->shards) {
        ARE_CUDA(cudaSetDevice(sh.device));
        unsigned int h = 0;
        ARE_CUDA(cudaMemcpyAsync(&h, sh.d_err, sizeof h, cudaMemcpyDeviceToHost, sh.stream));
        ARE_CUDA(cudaStreamSynchronize(sh.stream));
        if (h) ARE_CUDA(cudaMemsetAsync(sh.d_err, 0, sizeof(unsigned int), sh.stream));
        bad |= h;
    }
    if (bad) return fail(ARE_ERANGE, "event id outside the catalog in the year event table");
    if (n_rp <= 0) return ARE_OK;
    // no peer stores: gather the slices into the first GPU's memory with
    // peer copies, then K3 there
    ARE_CUDA(cudaSetDevice(s0.device));
    for (auto &sh : y->shards) {
        if (sh.t1 == sh.t0) continue;
        ARE_CUDA(cudaMemcpyPeerAsync(y->d_full + sh.t0, s0.device, sh.d_out, sh.device,
                                     (sh.t1 - sh.t0) * sizeof(double), s0.stream));
    }
    DeviceInfo *di;
    if ((rc = use_device(s0.device, &di))) return rc;
    return k3_order_stats(y->d_full, y->n_trials, rps, n_rp, pml_out, tvar_out, di->sms, s0.stream);
}

int are_run_layer_host(const uint32_t *ids, int64_t n_occ, const int64_t *offsets, int64_t n_trials,
                       const int64_t *bounds, int32_t n_shards, const are_plan_t *plans, double occ_ret,
                       double occ_lim, double agg_ret, double agg_lim, int64_t first, int64_t last, double *out,
                       int64_t *lookups, int32_t variant) {
    if (!plans || !bounds || n_shards < 1) return fail(ARE_EINVAL, "need at least one shard and its plan");
    if (first < 0 || last < first || last > n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    if (bounds[0] != 0 || bounds[n_shards] != n_trials) return fail(ARE_EINVAL, "shard bounds must span every trial");
    for (int s = 0; s < n_shards; ++s)
        if (!plans[s] || bounds[s + 1] < bounds[s]) return fail(ARE_EINVAL, "bad shard bounds or plan");
    if (lookups) *lookups = plans[0]->n_sel * (offsets[last] - offsets[first]);
    // every GPU streams its own trial range over its own PCIe link; the
    // per-device workspace keeps their staging independent
    return for_each_shard(n_shards, [&](int s) -> int {
        const int64_t a = std::max(first, bounds[s]), b = std::min(last, bounds[s + 1]);
        if (a >= b) return ARE_OK;
        int64_t lk = 0;
        return are_simulate_host(plans[s], ids, n_occ, offsets, n_trials, a, b, occ_ret, occ_lim, agg_ret, agg_lim,
                                 out, &lk, variant);
    });
}

}  // extern "C"
