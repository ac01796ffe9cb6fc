// Shared definitions for the aggrisk B200 library (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <string>

#include "aggrisk_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1308_2066_b200 is written for sm_100a (B200) only"
#endif

namespace are {

// ---- error plumbing -----------------------------------------------------
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
extern std::atomic<int64_t> g_launches;

#define ARE_CUDA(call)                                                       \
    do {                                                                     \
        cudaError_t _e = (call);                                             \
        if (_e != cudaSuccess) return ::are::cuda_fail(_e, #call);           \
    } while (0)

#define ARE_LAUNCHED()                                                       \
    do {                                                                     \
        ::are::g_launches.fetch_add(1, std::memory_order_relaxed);           \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return ::are::cuda_fail(_e, "kernel launch"); \
    } while (0)

// ---- device-side data layout ------------
// One 16-byte record per catalog slot (event id).  `meta` packs the
// selection position of the first non-zero loss (bits 0..15) and the number
// of non-zero losses n (bits 16..31; n == 0 means absent from every selected
// table).  Losses 2..n live in the overflow array at `ovf`.
struct __align__(16) Slot {
    double x;       // first non-zero loss (float64, exact copy of the table)
    uint32_t meta;  // j0 | n << 16
    uint32_t ovf;   // offset of entries 2..n in the overflow array
};

struct __align__(16) Entry {
    double x;
    uint32_t j;     // selection position
    uint32_t pad;
};

// Relay-kernel record (k2_relay.cu), one per event id, 16 bytes (one
// 128-bit load): the event's selected entries with the financial terms
// already applied by K1, f_j(x_j) = share_j * clamp(rate_j * x_j - ret_j, 0,
// lim_j) in selection order j1 < j2 < ...
//   simple event (at most 2 entries, none NaN):
//       a = 0.0 + f_{j1}   (the first partial sum of comb; +0.0 when absent)
//       b = f_{j2}, or +0.0 when the event has one entry or none
//     comb = a + b is then exactly the reference's sum: for one entry the
//     extra +0.0 leaves a (never -0.0, being 0.0 + f) unchanged;
//   complex event (3+ entries, or a NaN among the first two):
//       a = a quiet NaN whose payload holds cnt (bits 32..50) and the index
//           in the relay overflow array of entry 2 (bits 0..31)
//       b = 0.0 + f_{j1}
//     comb = b + ovf[i] + ovf[i + 1] + ... (cnt - 1 overflow entries).
struct __align__(16) RSlot {
    double a, b;
};
static constexpr unsigned long long RSLOT_COMPLEX = 0x7FF8000000000000ull;  // the NaN tag of a complex record
__device__ __forceinline__ bool rslot_complex(double a) { return a != a; }
__device__ __forceinline__ uint32_t rslot_cnt(double a) {
    return (uint32_t)((unsigned long long)__double_as_longlong(a) >> 32) & 0x7FFFFu;
}
__device__ __forceinline__ uint32_t rslot_ovf(double a) { return (uint32_t)__double2loint(a); }

// Fused-layer record (k2_layers.cu), one per event id, 32 bytes: the
// event's first two pool entries with the financial terms applied by K1 --
// fa = 0.0 + f_{j0}(x0) (the first partial sum), fb = f_{j1}(x1) -- their pool
// positions and count (meta = j0 | j1 << 8 | cnt << 16), the raw first loss
// x0 and the overflow offset of entries 2..cnt (for the general path).
struct __align__(32) LRec {
    double fa, fb, x0;
    uint32_t meta, ovf;
};

// Financial terms of one selected table (FinancialTerms, model.py:46-66).
struct __align__(32) Fin {
    double rate, ret, lim, share;
};

// Reference arithmetic, no contraction (pkg/setup.py:9 -ffp-contract=off):
// every product and sum rounds separately, and clamps are two `if`s so NaN
// passes through (_kernel.pyx:72-75, :79-82, :114-117).
__device__ __forceinline__ double clamp_ref(double v, double hi) {
    if (v < 0.0) v = 0.0;
    if (v > hi) v = hi;
    return v;
}
__device__ __forceinline__ double fin_term(const Fin &f, double x) {
    double l = __dsub_rn(__dmul_rn(f.rate, x), f.ret);
    return __dmul_rn(f.share, clamp_ref(l, f.lim));
}
// Financial terms as four shared-memory arrays (structure of arrays: rate[n],
// ret[n], lim[n], share[n]).  A warp whose lanes evaluate different tables
// reads four 8-byte words per lane from four <= n-word rows, which the
// shared-memory crossbar serves in one or two wavefronts each; the 32-byte
// Fin struct read as two LDS.128 by lanes with different j costs ~9 wavefronts
// each (ncu, profiles/r02_k2_lsu.md).
__device__ __forceinline__ void fin_soa_store(double *s, int n, const Fin *g) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const Fin f = g[i];
        s[i] = f.rate;
        s[n + i] = f.ret;
        s[2 * n + i] = f.lim;
        s[3 * n + i] = f.share;
    }
}
__device__ __forceinline__ double fin_term_soa(const double *s, int n, uint32_t j, double x) {
    double l = __dsub_rn(__dmul_rn(s[j], x), s[n + j]);
    return __dmul_rn(s[3 * n + j], clamp_ref(l, s[2 * n + j]));
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Streaming 16-byte load for the YET id stream: read once, keep it out of L1
// and mark it evict-first in L2 so it does not displace the hot-set records.
__device__ __forceinline__ uint4 ld_stream_u4(const uint32_t *p, uint64_t policy) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(policy));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p, uint64_t policy) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(policy));
    return r;
}
// Predicated streaming load: returns p[0] when rel < len, else `pad` (no access).
__device__ __forceinline__ uint32_t ld_stream_if(const uint32_t *p, uint32_t rel, uint32_t len, uint64_t policy,
                                                 uint32_t pad = 0) {
    uint32_t r = pad;
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "setp.lt.u32 q, %1, %2;\n\t"
        "@q ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%3], %4;\n\t}"
        : "+r"(r)
        : "r"(rel), "r"(len), "l"(p), "l"(policy));
    return r;
}
// Bulk L2 prefetch (cp.async.bulk.prefetch, TMA unit): `bytes` (multiple of
// 16) from a 16-byte aligned global address into L2, no registers or shared
// memory held while it is in flight.
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Hot-set record load: 16 B, L2 evict-last (the records are the L2-resident
// working set; K2).
__device__ __forceinline__ Slot ld_slot(const Slot *p, uint64_t policy) {
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(policy));
    Slot s;
    s.x = __hiloint2double((int)r.y, (int)r.x);
    s.meta = r.z;
    s.ovf = r.w;
    return s;
}

// Read-only float64 gather with an L2 cache policy (resident tables).
__device__ __forceinline__ double ld_nc_f64(const double *p, uint64_t policy) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy));
    return v;
}

// Predicated 32-bit shared store (keeps queue appends branch-free).
__device__ __forceinline__ void st_shared_if(uint32_t saddr, uint32_t v, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}"
                 :: "r"(saddr), "r"(v), "r"((uint32_t)pred) : "memory");
}
__device__ __forceinline__ uint32_t ballot_full(bool pred) {
    uint32_t b;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tvote.sync.ballot.b32 %0, q, 0xffffffff;\n\t}"
                 : "=r"(b) : "r"((uint32_t)pred));
    return b;
}

// Order-preserving map float64 -> uint64 (NaN sorts last, as numpy does).
__device__ __forceinline__ uint64_t order_key(double v) {
    if (v != v) return 0xFFFFFFFFFFFFFFFFull;
    uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_value(uint64_t k) {
    if (k == 0xFFFFFFFFFFFFFFFFull) return __longlong_as_double(0x7FF8000000000000ll);
    uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double((long long)b);
}

}  // namespace are
