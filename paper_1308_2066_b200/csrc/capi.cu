// extern "C" surface of libaggrisk_b200.so (include/aggrisk_b200.h) and the
// host-side orchestration around K1/K2/K3: device handles, the chunked
// host->device streaming pipeline for host-resident YETs, and argument
// validation with the reference's error behaviour.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "k1_ingest.cuh"
#include "k2_trials.cuh"
#include "k3_order_stats.cuh"
#include "capi_internal.cuh"

namespace are {

static thread_local std::string t_err;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { t_err = msg; }
int fail(int code, const std::string &msg) {
    t_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char *what) {
    t_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? ARE_ENOMEM : ARE_ECUDA;
}

// ---- per-device facts ------------------------------------------------------
static std::mutex g_dev_mu;
static DeviceInfo g_dev[64];

int use_device(int dev, DeviceInfo **out) {
    if (dev < 0 || dev >= 64) return fail(ARE_EINVAL, "bad device ordinal");
    ARE_CUDA(cudaSetDevice(dev));
    std::lock_guard<std::mutex> g(g_dev_mu);
    DeviceInfo &d = g_dev[dev];
    if (!d.ready) {
        int major = 0;
        ARE_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
        if (major < 10)
            return fail(ARE_ECUDA, "paper_1308_2066_b200 requires an sm_100 (B200) device");
        ARE_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev));
        ARE_CUDA(cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        int rc = k2_prepare(dev);
        if (rc) return rc;
        d.ready = true;
    }
    *out = &d;
    return ARE_OK;
}

static int current_device(int *dev) {
    ARE_CUDA(cudaGetDevice(dev));
    return ARE_OK;
}

}  // namespace are

using namespace are;

static void tables_release(are_tables_s *t) {
    DeviceGuard dg;
    if (t && t->refs.fetch_sub(1) == 1) {
        cudaSetDevice(t->device);
        cudaFree(t->d);
        delete t;
    }
}

// ---- host streaming workspace (one per device, grown on demand) -----------
namespace are {
struct Workspace {
    std::mutex mu;
    bool init = false;
    cudaStream_t copy = nullptr, comp = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    uint32_t *d_ids[2] = {nullptr, nullptr};
    int64_t *d_off[2] = {nullptr, nullptr};
    uint32_t *h_ids[2] = {nullptr, nullptr};  // pinned bounce buffers (pageable inputs)
    int64_t *h_off[2] = {nullptr, nullptr};
    int64_t cap_ids = 0, cap_off = 0;
    double *d_out = nullptr;
    int64_t cap_out = 0;
    unsigned int *d_err = nullptr;
    double *d_k3 = nullptr;  // are_order_stats_host's device copy of the YLT
    int64_t cap_k3 = 0;
};
static Workspace g_ws[64];
static constexpr int64_t CHUNK_OCC = 32ll << 20;  // 32 Mi occurrences (128 MiB of ids) per chunk

// Host -> pinned staging copy on several threads: one thread copies pageable
// memory at ~10-14 GB/s, well below the PCIe rate the copy engine drains it at.
void parallel_copy(void *dst, const void *src, size_t bytes) {
    constexpr size_t MIN_PIECE = 8u << 20;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t n = std::min<size_t>(std::min<size_t>(hw, 16), std::max<size_t>(1, bytes / MIN_PIECE));
    if (n <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t piece = (bytes / n + 63) & ~size_t(63);
    std::vector<std::thread> pool;
    pool.reserve(n - 1);
    size_t done = std::min(bytes, piece);  // [0, done) is this thread's; [launched, bytes) still to copy
    size_t launched = done;
    try {
        for (size_t i = 1; i < n && launched < bytes; ++i) {
            const size_t a = launched, b = std::min(bytes, a + piece);
            pool.emplace_back([=] { std::memcpy((char *)dst + a, (const char *)src + a, b - a); });
            launched = b;
        }
    } catch (...) {  // no threads available: copy the rest here (never throw across the C ABI)
    }
    std::memcpy(dst, src, done);
    if (launched < bytes) std::memcpy((char *)dst + launched, (const char *)src + launched, bytes - launched);
    for (auto &t : pool) t.join();
}

static int ws_reserve(Workspace &w, int64_t ids, int64_t offs, int64_t outs, bool bounce) {
    if (!w.init) {
        ARE_CUDA(cudaStreamCreateWithFlags(&w.copy, cudaStreamNonBlocking));
        ARE_CUDA(cudaStreamCreateWithFlags(&w.comp, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            ARE_CUDA(cudaEventCreateWithFlags(&w.copied[i], cudaEventDisableTiming));
            ARE_CUDA(cudaEventCreateWithFlags(&w.consumed[i], cudaEventDisableTiming));
        }
        ARE_CUDA(cudaMalloc(&w.d_err, sizeof(unsigned int)));
        w.init = true;
    }
    if (ids > w.cap_ids || offs > w.cap_off || (bounce && !w.h_ids[0])) {
        ids = std::max(ids, w.cap_ids);
        offs = std::max(offs, w.cap_off);
        for (int i = 0; i < 2; ++i) {
            cudaFree(w.d_ids[i]);
            cudaFree(w.d_off[i]);
            w.d_ids[i] = nullptr;
            w.d_off[i] = nullptr;
            if (w.h_ids[i]) cudaFreeHost(w.h_ids[i]);
            if (w.h_off[i]) cudaFreeHost(w.h_off[i]);
            w.h_ids[i] = nullptr;
            w.h_off[i] = nullptr;
        }
        for (int i = 0; i < 2; ++i) {
            ARE_CUDA(cudaMalloc(&w.d_ids[i], (ids + 4) * sizeof(uint32_t)));
            ARE_CUDA(cudaMalloc(&w.d_off[i], offs * sizeof(int64_t)));
            if (bounce) {
                ARE_CUDA(cudaHostAlloc(&w.h_ids[i], (ids + 4) * sizeof(uint32_t), cudaHostAllocDefault));
                ARE_CUDA(cudaHostAlloc(&w.h_off[i], offs * sizeof(int64_t), cudaHostAllocDefault));
            }
        }
        w.cap_ids = ids;
        w.cap_off = offs;
    }
    if (outs > w.cap_out) {
        cudaFree(w.d_out);
        w.d_out = nullptr;
        ARE_CUDA(cudaMalloc(&w.d_out, outs * sizeof(double)));
        w.cap_out = outs;
    }
    return ARE_OK;
}

// Page-locked pointers seen before: the e2e path asks on every call, and a
// driver query per call can wait behind other clients of the driver (NVML
// sampling).  Only positive answers are cached: a stale entry (freed, then
// reused as pageable memory) would still copy correctly, cudaMemcpyAsync
// accepts pageable memory.
static std::mutex g_pin_mu;
static const void *g_pinned[64];
static int g_pinned_next = 0;
bool is_pinned(const void *p) {
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        for (const void *q : g_pinned)
            if (q == p) return true;
    }
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeHost) return false;
    std::lock_guard<std::mutex> g(g_pin_mu);
    g_pinned[g_pinned_next] = p;
    g_pinned_next = (g_pinned_next + 1) % 64;
    return true;
}

// Exactness precondition of the hot-set kernel (DESIGN.md "Zero-skip
// exactness"): a zero table entry must contribute +-0 through the financial
// terms.  Evaluated in the reference's float64 arithmetic.
static bool fin_zero_ok(const Fin &f) {
    for (double z : {0.0, -0.0}) {
        double l = f.rate * z - f.ret;
        if (l < 0.0) l = 0.0;
        if (l > f.lim) l = f.lim;
        const double v = f.share * l;
        if (!(v == 0.0)) return false;
    }
    return true;
}
static bool occ_zero_ok(double occ_ret, double occ_lim) {
    double o = 0.0 - occ_ret;
    if (o < 0.0) o = 0.0;
    if (o > occ_lim) o = occ_lim;
    return o == 0.0;
}

// AUTO also picks the dense kernel for dense-overlap plans, where the hot set
// gathers several scattered entries per occurrence and the cooperative
// event-major kernel reads one line instead.  Measured, ms per 100k trials x
// 1000 events, hot set vs dense (scripts/time_density.py): catalog 50k with
// 15 ELTs (6 entries per catalog event) 4.08 vs 2.06; 6 ELTs (2.4) 1.80 vs
// 2.00; 3 ELTs 1.03 vs 1.27; catalog 200k, 15 ELTs (1.5) 1.33 vs 2.06;
// catalog 2M, 15 ELTs (0.15) 0.28 vs 2.47.  Pre-combined plans read one value
// per event on the hot set and always keep it.
static constexpr double DENSE_MIN_ENTRIES_PER_EVENT = 3.5;
static constexpr int64_t EM_MAX_SEL = 32, EM_MIN_SEL = 4;  // the event-major copy (ensure_event_major)
static constexpr int64_t EM_MIN_BYTES = 64ll << 20;
static bool dense_overlap(const are_plan_s *p) {
    return !p->precombined && p->n_sel >= EM_MIN_SEL && p->n_sel <= EM_MAX_SEL &&
           (double)p->pb.entries >= DENSE_MIN_ENTRIES_PER_EVENT * (double)p->tab->row_len;
}

static int choose_variant(const are_plan_s *p, double occ_ret, double occ_lim, int variant, int *out) {
    const int flags = variant & ~0xFF;
    variant &= 0xFF;
    const bool exact = p->zero_skip && !p->slot0_hot && occ_zero_ok(occ_ret, occ_lim);
    if (variant == ARE_VARIANT_AUTO) {
        *out = (exact && !dense_overlap(p) ? ARE_VARIANT_HOTSET : ARE_VARIANT_DENSE) | flags;
        return ARE_OK;
    }
    if (variant == ARE_VARIANT_HOTSET && !exact)
        return fail(ARE_EINVAL, "hot-set kernel requested but a zero loss does not map to zero under these terms");
    if (variant != ARE_VARIANT_HOTSET && variant != ARE_VARIANT_DENSE) return fail(ARE_EINVAL, "unknown K2 variant");
    *out = variant | flags;
    return ARE_OK;
}

// The dense kernel's event-major table: built once per plan on first use.
// Measured, ms per 100k trials x 1000 events (event-major vs row-major):
// 15 rows over catalogs 2M / 200k / 50k: 4.3 vs 19.1 / 4.3 vs 5.4 / 4.3 vs
// 5.4; 6 rows over 50k: 2.0 vs 2.5; 3 rows over 50k: 1.7 vs 1.5 -- so the
// copy is used from 4 selected rows on, or whenever the rows exceed what L2
// keeps.  If it cannot be allocated the row-major dense kernel runs instead.
static int ensure_event_major(are_plan_s *p, int sms, cudaStream_t st) {
    std::lock_guard<std::mutex> g(p->em_mu);
    if (p->em_tried) return ARE_OK;
    p->em_tried = true;
    const int64_t bytes_rows = p->n_sel * p->tab->row_len * (int64_t)sizeof(double);
    if (p->n_sel > EM_MAX_SEL || (p->n_sel < EM_MIN_SEL && bytes_rows < EM_MIN_BYTES)) return ARE_OK;
    const int stride = (int)((p->n_sel + 1) & ~1);
    const size_t bytes = (size_t)p->tab->row_len * stride * sizeof(double);
    double *d = nullptr;
    if (cudaMalloc(&d, bytes) != cudaSuccess) {
        cudaGetLastError();
        return ARE_OK;
    }
    int rc = k1_event_major(p->tab->d, p->tab->row_len, p->d_rows, (int)p->n_sel, stride, d, sms, st);
    // other streams may use the plan next: the table must be complete
    if (rc == ARE_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "event-major table");
    if (rc) {
        cudaFree(d);
        return rc;
    }
    p->d_em = d;
    p->em_stride = stride;
    return ARE_OK;
}

// The relay kernel's records and filter: built once per plan on its first
// hot-set launch (exact plans only; pooled and pre-combined plans keep their
// own kernels).  ARE_K2_RELAY=0 keeps k2_hotset (A/B).  If the records
// cannot be allocated k2_hotset runs instead.
static bool relay_off() {
    static const bool off = [] {
        const char *e = getenv("ARE_K2_RELAY");
        return e && e[0] == '0';
    }();
    return off;
}
static uint64_t dbits(double x) {
    uint64_t b;
    std::memcpy(&b, &x, sizeof b);
    return b;
}
// Builds the plan's relay records on first use and returns (in *filter) the
// filter of the events that contribute under (occ_ret, occ_lim), built once
// per distinct pair of terms (null: run k2_hotset).
static int ensure_relay(are_plan_s *p, const DeviceInfo *di, double occ_ret, double occ_lim, cudaStream_t st,
                        const uint32_t **filter) {
    *filter = nullptr;
    if (p->pool || relay_off()) return ARE_OK;
    std::lock_guard<std::mutex> g(p->relay_mu);
    if (!p->relay_tried) {
        p->relay_tried = true;
        const int64_t fixed = (int64_t)k2_relay_fixed_smem();
        const int64_t avail = std::min<int64_t>(di->smem_optin, k2_max_dynamic_smem()) - fixed - 64;
        const int64_t max_bits = (avail / 16) * 128;
        const int64_t want = ((p->tab->row_len + 127) / 128) * 128;
        int64_t nbits = std::max<int64_t>(std::min(want, max_bits), 128);
        RelayBuffers rb;
        int rc = k1_build_relay(p->pb, p->d_fin, p->tab->row_len, nbits, rb, di->sms, st, p->precombined);
        // other streams may use the plan next: the records must be complete
        if (rc == ARE_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "relay records");
        if (rc) {
            rb.release();
            if (rc == ARE_ENOMEM) return ARE_OK;
            return rc;
        }
        p->rnbits = nbits;
        p->rhash_mode = nbits >= p->tab->row_len ? 0 : (p->tab->row_len <= 2 * nbits ? 1 : 2);
        p->rsmem = (size_t)fixed + (size_t)(nbits / 8);
        p->rb = rb;
    }
    if (!p->rb.rslots) return ARE_OK;
    const uint64_t kr = dbits(occ_ret), kl = dbits(occ_lim);
    are_plan_s::OccFilter *slot = nullptr;
    for (auto &f : p->occf)
        if (f.d && f.ret_bits == kr && f.lim_bits == kl) {
            f.stamp = ++p->occ_clock;
            *filter = f.d;
            return ARE_OK;
        }
    for (auto &f : p->occf)
        if (!slot || !f.d || (slot->d && f.stamp < slot->stamp)) slot = &f;
    const int64_t nwords = (p->rnbits + 31) / 32;
    if (slot->d) {
        // an earlier launch on any stream may still read the evicted filter
        ARE_CUDA(cudaDeviceSynchronize());
    } else if (cudaMalloc(&slot->d, (nwords + 4) * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        slot->d = nullptr;
        return ARE_OK;  // k2_hotset runs instead
    }
    int rc = k1_relay_filter(p->rb, p->tab->row_len, p->rnbits, occ_ret, occ_lim, slot->d, di->sms, st);
    if (rc == ARE_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = cuda_fail(cudaGetLastError(), "relay filter");
    if (rc) {
        cudaFree(slot->d);
        slot->d = nullptr;
        return rc;
    }
    slot->ret_bits = kr;
    slot->lim_bits = kl;
    slot->stamp = ++p->occ_clock;
    *filter = slot->d;
    return ARE_OK;
}

static void fill_args(const are_plan_s *p, K2Args &a, double occ_ret, double occ_lim, double agg_ret,
                      double agg_lim) {
    a.filter = p->pb.filter;
    a.filter_words = p->pb.filter_words;
    a.nbits = (uint32_t)p->nbits;
    a.hash_mode = p->hash_mode;
    a.slots = p->pb.slots;
    a.ovf = p->pb.ovf;
    a.row_len = (uint32_t)p->tab->row_len;
    a.fin = p->d_fin;
    a.n_sel = (int32_t)p->n_sel;
    a.fin_bytes = (int32_t)(p->n_sel * sizeof(Fin));
    a.occ_ret = occ_ret;
    a.occ_lim = occ_lim;
    a.agg_ret = agg_ret;
    a.agg_lim = agg_lim;
    a.stacked = p->tab->d;
    a.rows = p->d_rows;
    a.precombined = p->precombined ? 1 : 0;
    a.em = p->d_em;
    a.em_stride = p->em_stride;
    a.rslots = nullptr;  // set with the terms' filter (ensure_relay)
    a.rovf = p->rb.rovf;
    a.rfilter = nullptr;
    a.rfilter_words = p->rb.filter_words;
    a.rnbits = (uint32_t)p->rnbits;
    a.rhash_mode = p->rhash_mode;
    a.rsmem = p->rsmem;
    a.rtex = p->rb.tex;
    a.hot_frac = p->tab->row_len > 0 ? (double)p->pb.hot_events / (double)p->tab->row_len : 0.0;
}

// K2 over trials [first, last) of ids/offsets indexed from id_base/t_base
// (ids[i - id_base] is occurrence i, off[t - t_base] is offset t) into
// out[t - out_base]; launches on `st`, no synchronisation.  Shared by the
// single-device entry points and the multi-GPU group (capi_group.cu).
int simulate_range(are_plan_s *p, const uint32_t *ids, int64_t id_base, int64_t n_ids, const int64_t *off,
                   int64_t t_base, int64_t first, int64_t last, double mean_len, double occ_ret, double occ_lim,
                   double agg_ret, double agg_lim, double *out, int64_t out_base, unsigned int *d_err,
                   cudaStream_t st, int32_t variant) {
    int v, rc;
    if ((rc = choose_variant(p, occ_ret, occ_lim, variant, &v))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(p->device, &di))) return rc;
    if ((v & 0xFF) == ARE_VARIANT_DENSE && (rc = ensure_event_major(p, di->sms, st))) return rc;
    const uint32_t *rfilter = nullptr;
    if ((v & 0xFF) == ARE_VARIANT_HOTSET && (rc = ensure_relay(p, di, occ_ret, occ_lim, st, &rfilter))) return rc;
    K2Args a{};
    fill_args(p, a, occ_ret, occ_lim, agg_ret, agg_lim);
    if (rfilter) {
        a.rslots = p->rb.rslots;
        a.rfilter = rfilter;
    }
    a.mean_len = mean_len;
    a.ids = ids;
    a.id_base = id_base;
    a.n_ids = n_ids;
    a.offsets = off;
    a.t_base = t_base;
    a.first = first;
    a.last = last;
    a.out = out;
    a.out_base = out_base;
    a.err = d_err ? d_err : p->d_err;
    return k2_launch(a, v, di->sms, p->smem, st);
}

}  // namespace are

extern "C" {

const char *are_last_error(void) { return t_err.c_str(); }
int are_version(void) { return 1; }
int64_t are_launch_count(void) { return g_launches.load(); }

int are_device_count(int *n) {
    ARE_CUDA(cudaGetDeviceCount(n));
    return ARE_OK;
}

int are_select_device(int ordinal) {
    DeviceInfo *d;
    return use_device(ordinal, &d);
}

int are_device_sm_count(int *n) {
    int dev;
    int rc = current_device(&dev);
    if (rc) return rc;
    DeviceInfo *d;
    if ((rc = use_device(dev, &d))) return rc;
    *n = d->sms;
    return ARE_OK;
}

int are_host_register(void *ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) return ARE_OK;
    cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
    if (e == cudaErrorHostMemoryAlreadyRegistered) {
        cudaGetLastError();
        return ARE_OK;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaHostRegister");
    return ARE_OK;
}

int are_host_is_pinned(const void *ptr) { return is_pinned(ptr) ? 1 : 0; }

int are_host_unregister(void *ptr) {
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        for (const void *&q : g_pinned)
            if (q == ptr) q = nullptr;
    }
    cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess && e != cudaErrorHostMemoryNotRegistered) return cuda_fail(e, "cudaHostUnregister");
    cudaGetLastError();
    return ARE_OK;
}

// ---- K1 -------------------------------------------------------------------
int are_tables_from_dense(const double *stacked, int64_t n_tables, int64_t row_len, are_tables_t *out) {
    if (n_tables < 0 || row_len < 1 || (n_tables > 0 && !stacked)) return fail(ARE_EINVAL, "bad table shape");
    if (row_len > 0xFFFFFFFFll) return fail(ARE_EINVAL, "catalog exceeds uint32 event ids");
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    auto *t = new are_tables_s();
    t->device = dev;
    t->n_tables = n_tables;
    t->row_len = row_len;
    const size_t bytes = (size_t)std::max<int64_t>(n_tables, 1) * row_len * sizeof(double);
    cudaError_t e = cudaMalloc(&t->d, bytes);
    if (e != cudaSuccess) {
        delete t;
        return cuda_fail(e, "cudaMalloc(tables)");
    }
    if (n_tables > 0) e = cudaMemcpy(t->d, stacked, (size_t)n_tables * row_len * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(t->d);
        delete t;
        return cuda_fail(e, "upload tables");
    }
    *out = t;
    return ARE_OK;
}

int are_tables_from_records(const uint32_t *ids, const double *losses, const int64_t *table_offsets,
                            int64_t n_tables, int64_t row_len, are_tables_t *out) {
    if (n_tables < 0 || row_len < 1 || !table_offsets) return fail(ARE_EINVAL, "bad table shape");
    if (row_len > 0xFFFFFFFFll) return fail(ARE_EINVAL, "catalog exceeds uint32 event ids");
    const int64_t total = table_offsets[n_tables];
    int64_t max_rec = 0;
    for (int64_t i = 0; i < n_tables; ++i) {
        const int64_t lo = table_offsets[i], hi = table_offsets[i + 1];
        if (hi < lo) return fail(ARE_EINVAL, "table offsets must be non-decreasing");
        max_rec = std::max(max_rec, hi - lo);
        for (int64_t r = lo; r < hi; ++r)
            if (ids[r] < 1 || (int64_t)ids[r] >= row_len)
                return fail(ARE_ERANGE, "elt[" + std::to_string(i) + "] holds event ids outside [1, " +
                                            std::to_string(row_len - 1) + "]");
    }
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    auto *t = new are_tables_s();
    t->device = dev;
    t->n_tables = n_tables;
    t->row_len = row_len;
    uint32_t *d_ids = nullptr;
    double *d_loss = nullptr;
    int64_t *d_toff = nullptr;
    cudaStream_t st = nullptr;
    auto cleanup = [&]() {
        cudaFree(d_ids);
        cudaFree(d_loss);
        cudaFree(d_toff);
        if (st) cudaStreamDestroy(st);
    };
    const size_t bytes = (size_t)std::max<int64_t>(n_tables, 1) * row_len * sizeof(double);
    cudaError_t e;
    if ((e = cudaMalloc(&t->d, bytes)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaMalloc(&d_ids, std::max<int64_t>(total, 1) * sizeof(uint32_t))) != cudaSuccess ||
        (e = cudaMalloc(&d_loss, std::max<int64_t>(total, 1) * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&d_toff, (n_tables + 1) * sizeof(int64_t))) != cudaSuccess) {
        cleanup();
        cudaFree(t->d);
        delete t;
        return cuda_fail(e, "allocate table build buffers");
    }
    cudaMemsetAsync(t->d, 0, bytes, st);
    if (total) {
        cudaMemcpyAsync(d_ids, ids, total * sizeof(uint32_t), cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_loss, losses, total * sizeof(double), cudaMemcpyHostToDevice, st);
    }
    cudaMemcpyAsync(d_toff, table_offsets, (n_tables + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    rc = k1_scatter(d_ids, d_loss, d_toff, n_tables, max_rec, row_len, t->d, di->sms, st);
    if (rc == ARE_OK) {
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "table scatter");
    }
    cleanup();
    if (rc) {
        cudaFree(t->d);
        delete t;
        return rc;
    }
    *out = t;
    return ARE_OK;
}

int are_tables_info(are_tables_t t, int64_t *n_tables, int64_t *row_len, int64_t *device_bytes) {
    if (!t) return fail(ARE_EINVAL, "null tables handle");
    if (n_tables) *n_tables = t->n_tables;
    if (row_len) *row_len = t->row_len;
    if (device_bytes) *device_bytes = std::max<int64_t>(t->n_tables, 1) * t->row_len * (int64_t)sizeof(double);
    return ARE_OK;
}

int are_tables_read_row(are_tables_t t, int64_t row, double *host_out) {
    DeviceGuard dg;
    if (!t) return fail(ARE_EINVAL, "null tables handle");
    if (row < 0 || row >= t->n_tables) return fail(ARE_EINDEX, "table row out of range");
    ARE_CUDA(cudaSetDevice(t->device));
    ARE_CUDA(cudaMemcpy(host_out, t->d + row * t->row_len, t->row_len * sizeof(double), cudaMemcpyDeviceToHost));
    return ARE_OK;
}

int are_tables_free(are_tables_t t) {
    tables_release(t);
    return ARE_OK;
}

// ---- plan -------------------------------------------------------------------
static int plan_build(are_tables_t t, const int64_t *rows, int64_t n_sel, const double *fin_rate,
                      const double *fin_ret, const double *fin_lim, const double *fin_share, bool pool,
                      bool precombine, are_plan_t *out) {
    DeviceGuard dg;
    if (!t) return fail(ARE_EINVAL, "null tables handle");
    if (n_sel < 1) return fail(ARE_EINVAL, "table selection is empty");
    if (n_sel > ARE_MAX_TABLES)
        return fail(ARE_EINVAL, "kernel supports at most 256 tables per layer, got " + std::to_string(n_sel));
    for (int64_t s = 0; s < n_sel; ++s)
        if (rows[s] < 0 || rows[s] >= t->n_tables) return fail(ARE_EINDEX, "table selection out of range");
    DeviceInfo *di;
    int rc;
    if ((rc = use_device(t->device, &di))) return rc;
    auto *p = new are_plan_s();
    p->pool = pool;
    p->device = t->device;
    p->tab = t;
    t->refs.fetch_add(1);
    p->n_sel = n_sel;
    std::vector<Fin> hf(n_sel);
    p->zero_skip = true;
    for (int64_t s = 0; s < n_sel; ++s) {
        hf[s] = Fin{fin_rate[s], fin_ret[s], fin_lim[s], fin_share[s]};
        p->zero_skip = p->zero_skip && fin_zero_ok(hf[s]);
    }
    if (pool && n_sel > K2L_MAX_POOL)
        return fail(ARE_EINVAL, "a layer pool holds at most 64 tables, got " + std::to_string(n_sel));
    // filter size: whatever shared memory the K2 kernel leaves free
    const int64_t fixed = (int64_t)(pool ? k2_layers_fixed_smem((int)n_sel) : k2_hotset_fixed_smem((int)n_sel));
    int64_t avail = std::min<int64_t>(di->smem_optin, k2_max_dynamic_smem()) - fixed - 64;
    int64_t max_bits = (avail / 16) * 128;
    int64_t want = ((t->row_len + 127) / 128) * 128;
    p->nbits = std::min(want, max_bits);
    if (p->nbits < 128) p->nbits = 128;
    p->hash_mode = p->nbits >= t->row_len ? 0 : (t->row_len <= 2 * p->nbits ? 1 : 2);
    p->smem = (size_t)fixed + (size_t)(p->nbits / 8);
    cudaStream_t st = nullptr;
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaMalloc(&p->d_rows, n_sel * sizeof(int64_t))) != cudaSuccess ||
        (e = cudaMalloc(&p->d_fin, n_sel * sizeof(Fin))) != cudaSuccess ||
        (e = cudaMalloc(&p->d_err, sizeof(unsigned int))) != cudaSuccess) {
        if (st) cudaStreamDestroy(st);
        are_plan_free(p);
        return cuda_fail(e, "allocate plan");
    }
    cudaMemcpyAsync(p->d_rows, rows, n_sel * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(p->d_fin, hf.data(), n_sel * sizeof(Fin), cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(p->d_err, 0, sizeof(unsigned int), st);
    rc = k1_build_plan(t->d, t->row_len, p->d_rows, (int)n_sel, p->nbits, p->pb, di->sms, st);
    if (rc == ARE_OK && precombine) {
        rc = k1_precombine_plan(p->pb, p->d_fin, t->row_len, di->sms, st);
        p->precombined = true;
    }
    Slot slot0{};
    if (rc == ARE_OK) {
        cudaError_t ce = cudaMemcpyAsync(&slot0, p->pb.slots, sizeof(Slot), cudaMemcpyDeviceToHost, st);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "read slot 0");
    }
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (rc) {
        are_plan_free(p);
        return rc;
    }
    // K2 reads out-of-trial lanes as event 0; that is only a no-op when the
    // unused slot 0 (tables.py:5-7) holds no loss.  A caller-supplied dense
    // table with a loss in column 0 is served by the dense kernel instead.
    p->slot0_hot = (slot0.meta >> 16) != 0;
    *out = p;
    return ARE_OK;
}

int are_plan_build(are_tables_t t, const int64_t *rows, int64_t n_sel, const double *fin_rate,
                   const double *fin_ret, const double *fin_lim, const double *fin_share, are_plan_t *out) {
    DeviceGuard dg;
    return plan_build(t, rows, n_sel, fin_rate, fin_ret, fin_lim, fin_share, false, false, out);
}

int are_plan_build_precombined(are_tables_t t, const int64_t *rows, int64_t n_sel, const double *fin_rate,
                               const double *fin_ret, const double *fin_lim, const double *fin_share,
                               are_plan_t *out) {
    DeviceGuard dg;
    return plan_build(t, rows, n_sel, fin_rate, fin_ret, fin_lim, fin_share, false, true, out);
}

int are_plan_build_pool(are_tables_t t, const int64_t *rows, int64_t n_sel, const double *fin_rate,
                        const double *fin_ret, const double *fin_lim, const double *fin_share, are_plan_t *out) {
    DeviceGuard dg;
    return plan_build(t, rows, n_sel, fin_rate, fin_ret, fin_lim, fin_share, true, false, out);
}

int are_plan_info(are_plan_t p, are_plan_info_t *info) {
    if (!p || !info) return fail(ARE_EINVAL, "null plan handle");
    info->n_sel = p->n_sel;
    info->row_len = p->tab->row_len;
    info->hot_events = p->pb.hot_events;
    info->entries = p->pb.entries;
    info->overflow_entries = p->pb.overflow_entries;
    info->filter_bits = p->nbits;
    info->device_bytes = p->tab->row_len * (int64_t)sizeof(Slot) + p->pb.overflow_entries * (int64_t)sizeof(Entry) +
                         (p->pb.filter_words + 4) * 4 + p->n_sel * (int64_t)(sizeof(Fin) + sizeof(int64_t));
    info->zero_skip_exact = (p->zero_skip && !p->slot0_hot) ? 1 : 0;
    info->smem_bytes = (int32_t)p->smem;
    std::lock_guard<std::mutex> g(p->relay_mu);
    info->relay = p->rb.rslots && (p->rb.tex || !k2_relay_needs_texture()) ? 1 : 0;
    info->relay_filter_bits = p->rb.rslots ? p->rnbits : 0;
    info->relay_smem_bytes = p->rb.rslots ? (int32_t)p->rsmem : 0;
    return ARE_OK;
}

int are_plan_free(are_plan_t p) {
    DeviceGuard dg;
    if (!p) return ARE_OK;
    cudaSetDevice(p->device);
    cudaFree(p->d_rows);
    cudaFree(p->d_em);
    cudaFree(p->d_fin);
    cudaFree(p->d_err);
    cudaFree(p->pb.slots);
    cudaFree(p->pb.ovf);
    cudaFree(p->pb.filter);
    p->rb.release();
    cudaFree(p->d_lrec);
    for (auto &f : p->occf) cudaFree(f.d);
    tables_release(p->tab);
    delete p;
    return ARE_OK;
}

// ---- K2 -------------------------------------------------------------------
static int simulate_device(are_plan_t p, const uint32_t *d_event_ids, const uint64_t *d_packed, int64_t n_occ,
                           const int64_t *d_offsets, int64_t n_trials, int64_t first, int64_t last, double occ_ret,
                           double occ_lim, double agg_ret, double agg_lim, double *d_out, void *stream,
                           int32_t variant) {
    DeviceGuard dg;
    if (!p) return fail(ARE_EINVAL, "null plan handle");
    if (first < 0 || last < first || last > n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    int v, rc;
    if ((rc = choose_variant(p, occ_ret, occ_lim, variant, &v))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(p->device, &di))) return rc;
    if ((v & 0xFF) == ARE_VARIANT_DENSE && (rc = ensure_event_major(p, di->sms, (cudaStream_t)stream))) return rc;
    const uint32_t *rfilter = nullptr;
    if ((v & 0xFF) == ARE_VARIANT_HOTSET && (rc = ensure_relay(p, di, occ_ret, occ_lim, (cudaStream_t)stream, &rfilter))) return rc;
    K2Args a{};
    a.mean_len = n_trials > 0 ? (double)n_occ / (double)n_trials : 0.0;
    a.ids = d_event_ids;
    a.id_base = 0;
    a.n_ids = n_occ;
    a.offsets = d_offsets;
    a.t_base = 0;
    a.first = first;
    a.last = last;
    a.out = d_out;
    a.out_base = 0;
    a.err = p->d_err;
    fill_args(p, a, occ_ret, occ_lim, agg_ret, agg_lim);
    if (rfilter) {
        a.rslots = p->rb.rslots;
        a.rfilter = rfilter;
        // packed ids: only for ids the caller validated against this plan
        if (d_packed && (variant & ARE_FLAG_IDS_VALIDATED) && p->tab->row_len <= (1u << 21))
            a.pids = reinterpret_cast<const unsigned long long *>(d_packed);
    }
    // ARE_SPARE_SMS(k): the persistent grid leaves k SMs to concurrent work
    // on another stream (a pipelined caller's K3 / exchange)
    const int spare = (v >> 12) & 0xFF;
    const int sms = std::max(1, di->sms - spare);
    return k2_launch(a, v, sms, p->smem, (cudaStream_t)stream);
}

int are_simulate_device(are_plan_t p, const uint32_t *d_event_ids, int64_t n_occ, const int64_t *d_offsets,
                        int64_t n_trials, int64_t first, int64_t last, double occ_ret, double occ_lim,
                        double agg_ret, double agg_lim, double *d_out, void *stream, int32_t variant) {
    return simulate_device(p, d_event_ids, nullptr, n_occ, d_offsets, n_trials, first, last, occ_ret, occ_lim, agg_ret,
                           agg_lim, d_out, stream, variant);
}

int are_simulate_device_packed(are_plan_t p, const uint32_t *d_event_ids, const uint64_t *d_packed, int64_t n_occ,
                               const int64_t *d_offsets, int64_t n_trials, int64_t first, int64_t last,
                               double occ_ret, double occ_lim, double agg_ret, double agg_lim, double *d_out,
                               void *stream, int32_t variant) {
    if (!d_packed) return fail(ARE_EINVAL, "null packed id buffer");
    return simulate_device(p, d_event_ids, d_packed, n_occ, d_offsets, n_trials, first, last, occ_ret, occ_lim,
                           agg_ret, agg_lim, d_out, stream, variant);
}

int64_t are_packed_id_words(int64_t n_occ) { return n_occ < 0 ? -1 : packed_id_words(n_occ); }

int are_yet_pack_device(int32_t device, const uint32_t *d_event_ids, int64_t n_occ, uint64_t *d_packed,
                        uint32_t *d_flag, void *stream) {
    DeviceGuard dg;
    if (n_occ < 0 || (n_occ > 0 && (!d_event_ids || !d_packed))) return fail(ARE_EINVAL, "bad packed id arguments");
    int rc;
    DeviceInfo *di;
    if ((rc = use_device(device, &di))) return rc;
    return k1_pack_ids_launch(d_event_ids, n_occ, reinterpret_cast<unsigned long long *>(d_packed), d_flag, di->sms,
                              (cudaStream_t)stream);
}

}  // extern "C"

namespace are {
// Checks shared by both fused-layer entry points; fills the per-layer terms.
static int layer_terms_check(const are_plan_s *p, int32_t n_layers, const uint64_t *masks, const double *layer_terms,
                             std::vector<LayerTerm> &lt) {
    if (!p) return fail(ARE_EINVAL, "null plan handle");
    if (!p->pool) return fail(ARE_EINVAL, "the fused layer kernel needs a pool plan (are_plan_build_pool)");
    if (n_layers < 1 || n_layers > K2L_MAX_LAYERS) return fail(ARE_EINVAL, "1..16 layers per fused launch");
    if (!(p->zero_skip && !p->slot0_hot)) return fail(ARE_EINVAL, "pool terms are not zero-exact; run layers singly");
    const uint64_t valid = p->n_sel >= 64 ? ~0ull : ((1ull << p->n_sel) - 1);
    lt.resize(n_layers);
    for (int l = 0; l < n_layers; ++l) {
        if (masks[l] & ~valid) return fail(ARE_EINDEX, "layer mask names a table outside the pool");
        lt[l] = LayerTerm{layer_terms[4 * l], layer_terms[4 * l + 1], layer_terms[4 * l + 2], layer_terms[4 * l + 3]};
        if (!occ_zero_ok(lt[l].occ_ret, lt[l].occ_lim))
            return fail(ARE_EINVAL, "layer occurrence terms are not zero-exact; run layers singly");
    }
    return ARE_OK;
}

static void layer_args(const are_plan_s *p, K2Args &a, const uint32_t *d_event_ids, int64_t n_occ,
                       const int64_t *d_offsets, int64_t first, int64_t last, double *d_out) {
    a.ids = d_event_ids;
    a.id_base = 0;
    a.n_ids = n_occ;
    a.offsets = d_offsets;
    a.t_base = 0;
    a.first = first;
    a.last = last;
    a.out = d_out;
    a.out_base = 0;
    a.err = p->d_err;
    fill_args(p, a, 0.0, 0.0, 0.0, 0.0);
}
}  // namespace are

// A layer set's per-event occurrence table over one pool plan (pre-combined
// fused layers).  The plan must outlive it.
struct are_layer_table_s {
    are_plan_s *plan = nullptr;
    int32_t n_layers = 0;
    uint64_t *d_masks = nullptr;
    LayerTerm *d_terms = nullptr;
    double *d_occ = nullptr;
};

extern "C" {

int are_simulate_layers_device(are_plan_t p, int32_t n_layers, const uint64_t *masks, const double *layer_terms,
                               const uint32_t *d_event_ids, int64_t n_occ, const int64_t *d_offsets, int64_t n_trials,
                               int64_t first, int64_t last, double *d_out, int64_t out_stride, void *stream,
                               int32_t flags) {
    DeviceGuard dg;
    std::vector<LayerTerm> lt;
    int rc;
    if ((rc = layer_terms_check(p, n_layers, masks, layer_terms, lt))) return rc;
    if (first < 0 || last < first || last > n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    DeviceInfo *di;
    if ((rc = use_device(p->device, &di))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    {  // the plan's fused-layer records, once (other streams may use them next)
        std::lock_guard<std::mutex> g(p->relay_mu);
        if (!p->d_lrec) {
            if ((rc = k1_build_layer_records(p->pb, p->d_fin, p->tab->row_len, &p->d_lrec, di->sms, st))) return rc;
            if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail(cudaGetLastError(), "fused-layer records");
        }
    }
    uint64_t *d_masks = nullptr;
    LayerTerm *d_terms = nullptr;
    ARE_CUDA(cudaMallocAsync((void **)&d_masks, sizeof(uint64_t) * n_layers, st));
    ARE_CUDA(cudaMallocAsync((void **)&d_terms, sizeof(LayerTerm) * n_layers, st));
    ARE_CUDA(cudaMemcpyAsync(d_masks, masks, sizeof(uint64_t) * n_layers, cudaMemcpyHostToDevice, st));
    ARE_CUDA(cudaMemcpyAsync(d_terms, lt.data(), sizeof(LayerTerm) * n_layers, cudaMemcpyHostToDevice, st));
    K2Args a{};
    layer_args(p, a, d_event_ids, n_occ, d_offsets, first, last, d_out);
    K2Layers L{n_layers, out_stride, d_masks, d_terms};
    L.lrec = p->d_lrec;
    rc = k2_layers_launch(a, L, !(flags & ARE_FLAG_IDS_VALIDATED), di->sms, p->smem, st);
    cudaFreeAsync(d_masks, st);
    cudaFreeAsync(d_terms, st);
    return rc;
}

int are_layer_table_build(are_plan_t p, int32_t n_layers, const uint64_t *masks, const double *layer_terms,
                          void *stream, are_layer_table_t *out) {
    DeviceGuard dg;
    if (!out) return fail(ARE_EINVAL, "null output handle");
    *out = nullptr;
    std::vector<LayerTerm> lt;
    int rc;
    if ((rc = layer_terms_check(p, n_layers, masks, layer_terms, lt))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(p->device, &di))) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    auto *t = new are_layer_table_s();
    t->plan = p;
    t->n_layers = n_layers;
    const int64_t row_len = p->tab->row_len;
    cudaError_t e;
    if ((e = cudaMalloc(&t->d_masks, sizeof(uint64_t) * n_layers)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_terms, sizeof(LayerTerm) * n_layers)) != cudaSuccess ||
        (e = cudaMalloc(&t->d_occ, sizeof(double) * K2L_MAX_LAYERS * row_len)) != cudaSuccess) {
        are_layer_table_free(t);
        return cuda_fail(e, "allocate layer table");
    }
    if ((e = cudaMemcpyAsync(t->d_masks, masks, sizeof(uint64_t) * n_layers, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(t->d_terms, lt.data(), sizeof(LayerTerm) * n_layers, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess) {
        are_layer_table_free(t);
        return cuda_fail(e, "upload layer terms");
    }
    K2Args a{};
    fill_args(p, a, 0.0, 0.0, 0.0, 0.0);
    K2Layers L{n_layers, 0, t->d_masks, t->d_terms, nullptr};
    if ((rc = k1_layer_occ_build(a, L, t->d_occ, di->sms, st)) ||
        (rc = (cudaStreamSynchronize(st) == cudaSuccess ? ARE_OK : cuda_fail(cudaGetLastError(), "layer table")))) {
        are_layer_table_free(t);
        return rc;
    }
    *out = t;
    return ARE_OK;
}

int are_layer_table_free(are_layer_table_t t) {
    DeviceGuard dg;
    if (!t) return ARE_OK;
    cudaFree(t->d_masks);
    cudaFree(t->d_terms);
    cudaFree(t->d_occ);
    delete t;
    return ARE_OK;
}

int are_simulate_layers_precombined(are_layer_table_t t, const uint32_t *d_event_ids, int64_t n_occ,
                                    const int64_t *d_offsets, int64_t n_trials, int64_t first, int64_t last,
                                    double *d_out, int64_t out_stride, void *stream, int32_t flags) {
    DeviceGuard dg;
    if (!t) return fail(ARE_EINVAL, "null layer table handle");
    if (first < 0 || last < first || last > n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    are_plan_s *p = t->plan;
    DeviceInfo *di;
    int rc;
    if ((rc = use_device(p->device, &di))) return rc;
    K2Args a{};
    layer_args(p, a, d_event_ids, n_occ, d_offsets, first, last, d_out);
    K2Layers L{t->n_layers, out_stride, t->d_masks, t->d_terms, t->d_occ};
    return k2_layers_pre_launch(a, L, !(flags & ARE_FLAG_IDS_VALIDATED), di->sms, (cudaStream_t)stream);
}

int are_check_errors(are_plan_t p, void *stream) {
    DeviceGuard dg;
    if (!p) return fail(ARE_EINVAL, "null plan handle");
    ARE_CUDA(cudaSetDevice(p->device));
    unsigned int h = 0;
    cudaStream_t st = (cudaStream_t)stream;
    ARE_CUDA(cudaMemcpyAsync(&h, p->d_err, sizeof(h), cudaMemcpyDeviceToHost, st));
    ARE_CUDA(cudaStreamSynchronize(st));
    if (h) {
        ARE_CUDA(cudaMemsetAsync(p->d_err, 0, sizeof(unsigned int), st));
        ARE_CUDA(cudaStreamSynchronize(st));
        return fail(ARE_ERANGE, "event id outside the catalog in the year event table");
    }
    return ARE_OK;
}

int are_simulate_host(are_plan_t p, const uint32_t *event_ids, int64_t n_occ, const int64_t *offsets,
                      int64_t n_trials, int64_t first, int64_t last, double occ_ret, double occ_lim,
                      double agg_ret, double agg_lim, double *out, int64_t *lookups, int32_t variant) {
    DeviceGuard dg;
    if (!p) return fail(ARE_EINVAL, "null plan handle");
    if (first < 0 || last < first || last > n_trials) return fail(ARE_EINVAL, "trial range out of bounds");
    if (offsets[n_trials] > n_occ) return fail(ARE_EINVAL, "offsets exceed the occurrence count");
    int v, rc;
    if ((rc = choose_variant(p, occ_ret, occ_lim, variant, &v))) return rc;
    if (lookups) *lookups = p->n_sel * (offsets[last] - offsets[first]);
    if (last == first) return ARE_OK;
    DeviceInfo *di;
    if ((rc = use_device(p->device, &di))) return rc;
    Workspace &w = g_ws[p->device];
    std::lock_guard<std::mutex> guard(w.mu);

    // trial chunks of <= CHUNK_OCC occurrences (at least one trial each)
    std::vector<int64_t> cuts{first};
    int64_t max_ids = 0, max_offs = 0;
    while (cuts.back() < last) {
        const int64_t ta = cuts.back();
        const int64_t limit = offsets[ta] + CHUNK_OCC;
        int64_t tb = std::upper_bound(offsets + ta + 1, offsets + last + 1, limit) - offsets - 1;
        if (tb <= ta) tb = ta + 1;
        cuts.push_back(tb);
        max_ids = std::max<int64_t>(max_ids, offsets[tb] - (offsets[ta] & ~(int64_t)3));
        max_offs = std::max(max_offs, tb - ta + 1);
    }
    const bool pinned = is_pinned(event_ids) && is_pinned(offsets);
    if ((rc = ws_reserve(w, max_ids, max_offs, last - first, !pinned))) return rc;
    ARE_CUDA(cudaMemsetAsync(w.d_err, 0, sizeof(unsigned int), w.comp));
    ARE_CUDA(cudaEventRecord(w.consumed[0], w.comp));
    ARE_CUDA(cudaEventRecord(w.consumed[1], w.comp));

    if ((v & 0xFF) == ARE_VARIANT_DENSE && (rc = ensure_event_major(p, di->sms, w.comp))) return rc;
    const uint32_t *rfilter = nullptr;
    if ((v & 0xFF) == ARE_VARIANT_HOTSET && (rc = ensure_relay(p, di, occ_ret, occ_lim, w.comp, &rfilter))) return rc;
    K2Args a{};
    fill_args(p, a, occ_ret, occ_lim, agg_ret, agg_lim);
    if (rfilter) {
        a.rslots = p->rb.rslots;
        a.rfilter = rfilter;
    }
    a.mean_len = (double)(offsets[last] - offsets[first]) / (double)(last - first);
    a.out = w.d_out;
    a.out_base = first;
    a.err = w.d_err;
    const size_t nchunks = cuts.size() - 1;
    for (size_t c = 0; c < nchunks; ++c) {
        const int b = (int)(c & 1);
        const int64_t ta = cuts[c], tb = cuts[c + 1];
        const int64_t oa = offsets[ta] & ~(int64_t)3, ob = offsets[tb];
        const int64_t nid = ob - oa, noff = tb - ta + 1;
        ARE_CUDA(cudaStreamWaitEvent(w.copy, w.consumed[b], 0));
        if (pinned) {
            ARE_CUDA(cudaMemcpyAsync(w.d_ids[b], event_ids + oa, nid * sizeof(uint32_t), cudaMemcpyHostToDevice, w.copy));
            ARE_CUDA(cudaMemcpyAsync(w.d_off[b], offsets + ta, noff * sizeof(int64_t), cudaMemcpyHostToDevice, w.copy));
        } else {
            // the bounce buffer b is free once the copy that last used it finished
            ARE_CUDA(cudaEventSynchronize(w.copied[b]));
            parallel_copy(w.h_ids[b], event_ids + oa, nid * sizeof(uint32_t));
            std::memcpy(w.h_off[b], offsets + ta, noff * sizeof(int64_t));
            ARE_CUDA(cudaMemcpyAsync(w.d_ids[b], w.h_ids[b], nid * sizeof(uint32_t), cudaMemcpyHostToDevice, w.copy));
            ARE_CUDA(cudaMemcpyAsync(w.d_off[b], w.h_off[b], noff * sizeof(int64_t), cudaMemcpyHostToDevice, w.copy));
        }
        ARE_CUDA(cudaEventRecord(w.copied[b], w.copy));
        ARE_CUDA(cudaStreamWaitEvent(w.comp, w.copied[b], 0));
        a.ids = w.d_ids[b];
        a.id_base = oa;
        a.n_ids = nid;
        a.offsets = w.d_off[b];
        a.t_base = ta;
        a.first = ta;
        a.last = tb;
        if ((rc = k2_launch(a, v, di->sms, p->smem, w.comp))) return rc;
        ARE_CUDA(cudaEventRecord(w.consumed[b], w.comp));
    }
    unsigned int herr = 0;
    ARE_CUDA(cudaMemcpyAsync(&herr, w.d_err, sizeof(herr), cudaMemcpyDeviceToHost, w.comp));
    ARE_CUDA(cudaMemcpyAsync(out + first, w.d_out, (last - first) * sizeof(double), cudaMemcpyDeviceToHost, w.comp));
    ARE_CUDA(cudaStreamSynchronize(w.comp));
    ARE_CUDA(cudaStreamSynchronize(w.copy));
    if (herr) return fail(ARE_ERANGE, "event id outside the catalog in the year event table");
    return ARE_OK;
}

int are_run_trials(const uint32_t *event_ids, int64_t n_occ, const int64_t *offsets, int64_t n_offsets,
                   const double *stacked, int64_t n_tables, int64_t row_len, const int64_t *rows, int64_t n_sel,
                   const double *fin_rate, const double *fin_ret, const double *fin_lim, const double *fin_share,
                   double occ_ret, double occ_lim, double agg_ret, double agg_lim, int64_t chunk,
                   int64_t first_trial, int64_t last_trial, double *out, int64_t scratch_len, int64_t *lookups) {
    if (n_sel > ARE_MAX_TABLES)
        return fail(ARE_EINVAL, "kernel supports at most 256 tables per layer, got " + std::to_string(n_sel));
    if (chunk > 0 && scratch_len < chunk) return fail(ARE_EINVAL, "scratch smaller than chunk size");
    if (n_offsets < 1) return fail(ARE_EINVAL, "offsets must hold at least one boundary");
    if (lookups) *lookups = 0;
    if (last_trial <= first_trial) return ARE_OK;
    are_tables_t t = nullptr;
    are_plan_t p = nullptr;
    int rc = are_tables_from_dense(stacked, n_tables, row_len, &t);
    if (rc) return rc;
    rc = are_plan_build(t, rows, n_sel, fin_rate, fin_ret, fin_lim, fin_share, &p);
    if (rc == ARE_OK)
        rc = are_simulate_host(p, event_ids, n_occ, offsets, n_offsets - 1, first_trial, last_trial, occ_ret,
                               occ_lim, agg_ret, agg_lim, out, lookups, ARE_VARIANT_AUTO);
    are_plan_free(p);
    are_tables_free(t);
    return rc;
}

// ---- K3 -------------------------------------------------------------------
int are_order_stats_device(const double *d_losses, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                           double *tvar_out, void *stream) {
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    return k3_order_stats(d_losses, n, rps, n_rp, pml_out, tvar_out, di->sms, (cudaStream_t)stream);
}

int are_order_stats_async(const double *d_losses, int64_t n, const double *rps, int64_t n_rp, double *d_res,
                          int32_t max_ctas, void *stream) {
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    return k3_order_stats_async(d_losses, n, rps, n_rp, d_res, di->sms, max_ctas, (cudaStream_t)stream);
}

int are_order_stats_summary_device(const double *d_losses, int64_t n, const double *rps, int64_t n_rp,
                                   double *pml_out, double *tvar_out, double *mean_max_out, void *stream) {
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    if (!mean_max_out) return fail(ARE_EINVAL, "null summary output");
    return k3_order_stats(d_losses, n, rps, n_rp, pml_out, tvar_out, di->sms, (cudaStream_t)stream, mean_max_out);
}

int are_pml_many_device(const double *d_losses, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                        void *stream) {
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    return k3_pml_sorted(d_losses, n, rps, n_rp, pml_out, di->sms, (cudaStream_t)stream);
}

int are_order_stats_host(const double *losses, int64_t n, const double *rps, int64_t n_rp, double *pml_out,
                         double *tvar_out) {
    if (n <= 0) return fail(ARE_EINVAL, "empty year loss table");
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    // the device's cached workspace: its stream and a YLT buffer kept across
    // calls (no stream or allocation churn on the per-request path; creating
    // and destroying them per call stalled for 0.1-0.8 s on the bench boxes)
    Workspace &w = g_ws[dev];
    std::lock_guard<std::mutex> guard(w.mu);
    if ((rc = ws_reserve(w, 0, 0, 0, false))) return rc;
    if (n > w.cap_k3) {
        cudaFree(w.d_k3);
        w.d_k3 = nullptr;
        w.cap_k3 = 0;
        ARE_CUDA(cudaMalloc(&w.d_k3, n * sizeof(double)));
        w.cap_k3 = n;
    }
    ARE_CUDA(cudaMemcpyAsync(w.d_k3, losses, n * sizeof(double), cudaMemcpyHostToDevice, w.comp));
    return k3_order_stats(w.d_k3, n, rps, n_rp, pml_out, tvar_out, di->sms, w.comp);
}

int are_rollup_device(const double *const *d_ylts, int64_t n_layers, int64_t n, double *d_out, void *stream) {
    int dev, rc;
    if ((rc = current_device(&dev))) return rc;
    DeviceInfo *di;
    if ((rc = use_device(dev, &di))) return rc;
    return k3_rollup_launch(d_ylts, n_layers, n, d_out, di->sms, (cudaStream_t)stream);
}

}  // extern "C"
