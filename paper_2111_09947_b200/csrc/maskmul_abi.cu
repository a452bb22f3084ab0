// C ABI of the B200 masked SpGEMM (declared in include/maskmul_b200.h).
//
// Host orchestration of one multiply, replacing the body of the reference's
// masked_multiply_with_stats (pkg/src/maskmul/multiply.py:349-403):
//   validate (_Prepared :175-233) -> k_analyze (flops_per_row, bins, bounds)
//   -> one summary readback -> k_bin_scatter -> per-bin kernels
//   -> scan -> nnz readback | compaction (1P) or exact numeric (2P).
// Workspace comes from the device's stream-ordered memory pool
// (cudaMallocAsync), so repeated multiplies allocate nothing from the OS.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "../../include/maskmul_b200.h"
#include "analyze.cuh"
#include "common.cuh"
#include "pull_inner.cuh"
#include "push_hash.cuh"
#include "push_hash_items.cuh"
#include "push_rank.cuh"
#include "push_heap.cuh"
#include "push_single.cuh"
#include "push_msa_sparse.cuh"
#include "push_dense.cuh"
#include "push_f64_defer.cuh"
#include "scan_compact.cuh"
#include "graph_ops.cuh"
#include "graph_prep.cuh"

using namespace mm;

namespace {

thread_local std::string g_last_error;
thread_local long long g_launches = 0;   // kernels launched by this thread (profiling)
thread_local long long* g_pinned = nullptr;  // 4 pinned words for small synchronous readbacks

// Pinned host scratch for the free-standing calls' readbacks (allocated once
// per thread: cudaMallocHost per call costs more than the work it reads).
long long* pinned_scratch() {
    if (!g_pinned && cudaMallocHost((void**)&g_pinned, 4 * sizeof(long long)) != cudaSuccess) g_pinned = nullptr;
    return g_pinned;
}

// MM_HOST_TRACE=1: host-side timestamps of one multiply's steps (stderr).
bool host_trace() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("MM_HOST_TRACE");
        on = e && *e && *e != '0';
    }
    return on == 1;
}
thread_local std::chrono::steady_clock::time_point g_t0;
thread_local char g_trace[512];
thread_local int g_trace_len = 0;
void trace(const char* what) {
    if (!host_trace()) return;
    const auto now = std::chrono::steady_clock::now();
    if (what[0] == '^') {
        g_t0 = now;
        g_trace_len = 0;
        what++;
    }
    const double us = std::chrono::duration<double, std::micro>(now - g_t0).count();
    g_trace_len += snprintf(g_trace + g_trace_len, sizeof(g_trace) - g_trace_len, " %s=%.1f", what, us);
    if (what[0] == '$') {
        fprintf(stderr, "[mm trace]%s\n", g_trace);
        g_trace_len = 0;
    }
}

bool debug_launches() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("MM_DEBUG_LAUNCH");
        on = e && *e && *e != '0';
    }
    return on == 1;
}

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail(MM_ERR_CUDA, std::string(#call) + " (maskmul_abi.cu:" + std::to_string(__LINE__) + \
                                         "): " + cudaGetErrorString(_e));                 \
    } while (0)

// Small synchronous readback of n int64 words through the pinned scratch.
int read_i64s(const void* dptr, int64_t* out, int n, cudaStream_t st) {
    long long* h = pinned_scratch();
    if (!h) return fail(MM_ERR_CUDA, "cudaMallocHost failed");
    cudaError_t e = cudaMemcpyAsync(h, dptr, n * sizeof(long long), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return fail(MM_ERR_CUDA, std::string("readback: ") + cudaGetErrorString(e));
    for (int q = 0; q < n; q++) out[q] = h[q];
    return MM_OK;
}

int read_i64(const void* dptr, int64_t* out, cudaStream_t st) { return read_i64s(dptr, out, 1, st); }

// Scoped device selection for every extern "C" entry: the call runs on the
// device that owns its handle / stream / operands and the caller's current
// device is restored on return (torch keeps its own notion of the current
// device, which the library must not change behind its back).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        // An error some earlier runtime call of this thread left unread (the
        // caller's, or another library's) is not this call's: the launches below
        // check cudaGetLastError() and would report it as their own.
        const cudaError_t stale = cudaGetLastError();
        if (stale != cudaSuccess && debug_launches())
            fprintf(stderr, "[mm] stale CUDA error at entry: %s\n", cudaGetErrorString(stale));
        int cur = -1;
        if (dev < 0 || cudaGetDevice(&cur) != cudaSuccess || cur == dev) return;
        if (cudaSetDevice(dev) == cudaSuccess) prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Device of a device pointer (-1 when it is not device memory / unknown).
int pointer_device(const void* ptr) {
    if (!ptr) return -1;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged ? at.device : -1;
}

// Device a free-standing call runs on: the stream's device for a created
// stream, else the device holding its first operand (the legacy default
// stream belongs to whichever device is current).
int call_device(void* stream, const void* operand) {
    int d = -1;
    if (stream && cudaStreamGetDevice((cudaStream_t)stream, &d) == cudaSuccess) return d;
    cudaGetLastError();
    return pointer_device(operand);
}

}  // namespace

struct mm_handle {
    int device = 0;
    int num_sms = 148;
    Summary* h_summary = nullptr;   // pinned
    long long* h_scalar = nullptr;  // pinned
    // ---- state between begin and end ----
    bool active = false;
    cudaStream_t stream = nullptr;
    mm_plan_t plan{};
    Prob prob{};
    AnalyzeParams ap{};
    int kind = 0;        // 0 plus-pair, 1 int64 plus-times, 2 float64 plus-times (ordered)
    int out_f64 = 0;
    int64_t nrows = 0, ncols = 0;
    std::vector<void*> allocs;
    Summary* d_summary = nullptr;
    int64_t* row_flops = nullptr;
    int64_t* bound = nullptr;
    int64_t* bound_ptr = nullptr;      // 1P complement bound offsets (nrows+1)
    const int64_t* bound_off = nullptr;
    uint8_t* row_bin = nullptr;
    int8_t* row_cap_lg = nullptr;
    int32_t* rows_list = nullptr;
    int32_t* cursors = nullptr;        // 3 * NBINS fetch counters (scatter, symbolic, numeric)
    int64_t* scan_scratch = nullptr;
    int64_t* row_nnz = nullptr;
    int64_t* row_nnz2 = nullptr;
    int64_t* c_row_ptr = nullptr;
    int32_t* tmp_idx = nullptr;
    void* tmp_val = nullptr;
    int64_t total_nnz = 0;
    int bin_off[NBINS + 1] = {0};
    Summary sum{};
    mm_stats_t stats{};
    int bound_flag = 0;
    // ---- tuning (mm_set_tuning) ----
    long long tier_flops0 = TIER_FLOPS0, tier_flops1 = TIER_FLOPS1;   // defaults: analyze.cuh
    long long tier_flops1_hash = TIER_FLOPS1_HASH;
    int capc_lg = CAPC_LG, load_shift = 2, load_shift_wide = 1;
    int rank_budget[3] = {6144, 24576, 49152};
    int auto_mca_nm = 0;
    int direct_lg[3] = {9, 10, 12};    // plain shared hash tables per tier: at least 2^direct_lg slots (0 = bin size)
    int64_t tiny_rows = 1 << 15, tiny_nnz = 1 << 20;   // single-pass path for small plain 1P multiplies
    bool direct_on = true;                              // direct path for ordered float64 (see begin_impl)
    int64_t* user_row_ptr = nullptr;                    // mm_multiply: C's row pointer, written by the scan
    bool slice_cursors = true;                          // sliced hub rows resume each B row per slice
    bool split_slices = true;                           // 1P plain sliced rows: (row, slice) work items
    int32_t* early_idx = nullptr;                       // mm_multiply, small plain 1P: C's arrays, compacted
    void* early_val = nullptr;                          //   before the single host sync
    bool compacted = false;
    bool blen_on = true;                                // analysis gathers int32 row lengths of B (k_row_len)
    int64_t mask_nnz = 0;
    int64_t b_nnz = 0;
    // k-blocked passes of the 16-warp plain hash bins (one-phase, int64 / plus-pair counts):
    // when B's index array exceeds this many bytes, the bin's launch is repeated over
    // blocks of B of about this size, so the rows in flight share an L2-resident block
    // (0 = off)
    int64_t kblock_bytes = 0;
    int64_t kblock_min_flops = 1 << 20;   // lighter rows are not cut into passes
    // ---- fused tail (fused_tail.cuh): one-launch small plain 1P multiplies ----
    unsigned* d_done = nullptr;          // device ticket counter, zero between multiplies
    TailResult* h_tail = nullptr;        // mapped pinned host memory the last block writes
    unsigned long long tail_seq = 0;
    cudaStream_t tail_stream = nullptr;  // stream of the last fused multiply (the host does not wait for its kernel to retire)
    int64_t fused_rows = 1 << 13, fused_nnz = 1 << 17;   // one block does the tail: small problems only (0 disables)
    // ---- concurrent bin launches ----
    static constexpr int NAUX = 3;
    cudaStream_t aux[NAUX] = {};
    cudaEvent_t fork_ev = nullptr, join_ev[NAUX] = {};
    // ---- profiling ----
    bool prof = false;
    cudaEvent_t ev[6] = {};
    long long launch_base = 0, launches = 0;
};

namespace {

template <typename T>
int dalloc(mm_handle* h, T** p, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    void* q = nullptr;
    CU(cudaMallocAsync(&q, bytes, h->stream));
    h->allocs.push_back(q);
    *p = (T*)q;
    return MM_OK;
}

void release(mm_handle* h) {
    for (void* q : h->allocs) cudaFreeAsync(q, h->stream);
    h->allocs.clear();
    h->active = false;
}

// ---- scan ----
// Scratch (int64 elements) a scan of n items needs: partials and their
// exclusive scan per level.
int64_t scan_scratch_elems(int64_t n) {
    int64_t total = 0;
    while (n > 0) {
        const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
        total += 2 * (nb + 1);
        if (nb <= 1) break;
        n = nb;
    }
    return total;
}

// out_incl[0..n) = inclusive scan of in (n >= 1); scratch holds
// scan_scratch_elems(n) elements.  zero_prev: also out_incl[-1] = 0.
// bounds_off/flag: one-phase bound check of `in`; total: grand total.
int scan_impl(const int64_t* in, int64_t n, int64_t* out_incl, cudaStream_t st, int64_t* scratch,
              int zero_prev, const int64_t* bounds_off, int* flag, long long* total) {
    const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
    int64_t* partials = scratch;
    int64_t* pscan = scratch + (nb + 1);
    ++g_launches;
    k_scan_tile<<<(unsigned)nb, SCAN_THREADS, 0, st>>>(in, n, out_incl, partials, zero_prev, bounds_off, flag,
                                                       total);
    if (nb > 1) {
        // exclusive offsets per tile: pscan[0] = 0, pscan[1..nb] = incl(partials)
        int rc = scan_impl(partials, nb, pscan + 1, st, scratch + 2 * (nb + 1), 1, nullptr, nullptr, nullptr);
        if (rc) return rc;
        ++g_launches;
        k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out_incl, n, pscan, total);
    }
    CU(cudaGetLastError());
    return MM_OK;
}

// out[0] = 0, out[1..n] = inclusive scan of counts.  scratch: caller-owned
// (scan_scratch_elems(n) elements) or nullptr (allocated from the pool).
int exclusive_scan(const int64_t* counts, int64_t n, int64_t* out, cudaStream_t st, int64_t* scratch = nullptr,
                   const int64_t* bounds_off = nullptr, int* flag = nullptr, long long* total = nullptr) {
    if (n <= 0) {
        CU(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
        if (total) CU(cudaMemsetAsync(total, 0, sizeof(long long), st));
        return MM_OK;
    }
    int64_t* own = nullptr;
    if (!scratch) {
        CU(cudaMallocAsync((void**)&own, scan_scratch_elems(n) * sizeof(int64_t), st));
        scratch = own;
    }
    int rc = scan_impl(counts, n, out + 1, st, scratch, 1, bounds_off, flag, total);
    if (own) cudaFreeAsync(own, st);
    return rc;
}

int validate(const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
             const mm_matrix_t* b, const mm_matrix_t* bt) {
    if (!plan || !mask || !a || !b) return fail(MM_ERR_INPUT, "null argument");
    if (plan->algorithm < MM_ALGO_MSA || plan->algorithm > MM_ALGO_AUTO)
        return fail(MM_ERR_PLAN, "unknown algorithm");
    if (plan->phases != 1 && plan->phases != 2) return fail(MM_ERR_PLAN, "phases must be 1 or 2");
    if (plan->semiring != MM_SR_ARITHMETIC && plan->semiring != MM_SR_PLUS_PAIR)
        return fail(MM_ERR_PLAN, "unknown semiring");
    if (plan->dtype != MM_DTYPE_INT64 && plan->dtype != MM_DTYPE_FLOAT64)
        return fail(MM_ERR_PLAN, "dtype must be int64 or float64");
    if (plan->n_inspect < -1 || plan->n_inspect > 1) return fail(MM_ERR_PLAN, "n_inspect must be 0, 1 or inf");
    if (plan->complemented && plan->algorithm == MM_ALGO_MCA)
        return fail(MM_ERR_PLAN, "the mask-compressed accumulator does not support complemented masks");
    if (plan->complemented && plan->algorithm == MM_ALGO_INNER)
        return fail(MM_ERR_PLAN, "the inner-product algorithm does not support complemented masks");
    if (mask->nrows != a->nrows || mask->ncols != b->ncols || a->ncols != b->nrows)
        return fail(MM_ERR_INPUT, "dimension mismatch: mask (" + std::to_string(mask->nrows) + ", " +
                                      std::to_string(mask->ncols) + "), A (" + std::to_string(a->nrows) +
                                      ", " + std::to_string(a->ncols) + "), B (" +
                                      std::to_string(b->nrows) + ", " + std::to_string(b->ncols) + ")");
    if (a->nrows < 0 || a->nrows >= (1ll << 31) || b->ncols >= (1ll << 31) || a->ncols >= (1ll << 31))
        return fail(MM_ERR_INPUT, "dimensions must be < 2^31");
    // The product loops count one batch of A entries' products (distinct
    // rows of B, canonical A) in 32-bit ints: nnz(B) < 2^31 bounds every such
    // sum (product_loop.cuh flat_products / ordered_products_f64).
    if (a->nnz < 0 || b->nnz < 0 || mask->nnz < 0 || b->nnz >= (1ll << 31) || a->nnz >= (1ll << 31) ||
        mask->nnz >= (1ll << 31))
        return fail(MM_ERR_INPUT, "nnz of A, B and the mask must be in [0, 2^31)");
    if ((a->nnz && (!a->ptr || !a->idx)) || !a->ptr || !b->ptr || !mask->ptr)
        return fail(MM_ERR_INPUT, "missing index arrays");
    // inner reads B only through B^T (B may be its row pointer alone, as the
    // reference's _Prepared holds B as CSC for inner, multiply.py:205-210)
    if (plan->semiring == MM_SR_ARITHMETIC &&
        ((a->nnz && !a->values) || (plan->algorithm != MM_ALGO_INNER && b->nnz && !b->values)))
        return fail(MM_ERR_INPUT, "plus-times needs operand values");
    if (plan->algorithm == MM_ALGO_INNER) {
        if (!bt || !bt->ptr) return fail(MM_ERR_INPUT, "the inner-product algorithm needs B in CSC form");
        if (bt->nrows != b->nrows || bt->ncols != b->ncols)
            return fail(MM_ERR_INPUT, "B^T (CSC) shape differs from B");
        if (plan->semiring == MM_SR_ARITHMETIC && bt->nnz && !bt->values)
            return fail(MM_ERR_INPUT, "plus-times needs B^T values");
    }
    return MM_OK;
}

// Resident blocks per SM of a kernel at a launch shape.  The dynamic
// shared-memory attribute and the occupancy query are host API calls worth a
// few microseconds each, so results are cached per (kernel, threads, smem).
struct OccEntry {
    int device;
    const void* fn;
    int threads;
    size_t smem;
    int occ;
};
std::vector<OccEntry> g_occ_cache;
struct SmemAttr {
    int device;
    const void* fn;
    size_t bytes;
};
std::vector<SmemAttr> g_smem_attr;
std::mutex g_attr_mu;

// Keyed by device as well: cudaFuncSetAttribute applies to the current
// device's context only, so a thread that multiplies on two GPUs sets it on each.
// The caches are process-wide (one mutex): the attribute belongs to the
// context, not the thread — a per-thread record let a second thread lower the
// limit under a thread that had raised it, whose next launch was then refused.
int kernel_occupancy(const void* fn, int threads, size_t smem, int* occ) {
    int dev = 0;
    CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(g_attr_mu);
    for (const OccEntry& e : g_occ_cache)
        if (e.device == dev && e.fn == fn && e.threads == threads && e.smem == smem) { *occ = e.occ; return MM_OK; }
    size_t have_i = g_smem_attr.size();
    for (size_t q = 0; q < g_smem_attr.size(); q++)
        if (g_smem_attr[q].device == dev && g_smem_attr[q].fn == fn) have_i = q;
    if (have_i == g_smem_attr.size()) g_smem_attr.push_back({dev, fn, 0});
    if (smem > g_smem_attr[have_i].bytes) {
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        g_smem_attr[have_i].bytes = smem;
    }
    int o = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, smem));
    g_occ_cache.push_back({dev, fn, threads, smem, o});
    *occ = o;
    return MM_OK;
}

// A refused launch reported with the shape it was refused at and the kernel's
// shared-memory attributes (static bytes, the dynamic limit in force).
int check_launch(const void* fn, int grid, int threads, size_t smem, int line) {
    const cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return MM_OK;
    cudaFuncAttributes fa{};
    const cudaError_t ea = cudaFuncGetAttributes(&fa, fn);
    cudaGetLastError();
    std::string msg = std::string("kernel launch (maskmul_abi.cu:") + std::to_string(line) + "): " +
                      cudaGetErrorString(e) + " [grid " + std::to_string(grid) + " threads " +
                      std::to_string(threads) + " dynamic smem " + std::to_string(smem);
    if (ea == cudaSuccess)
        msg += " static smem " + std::to_string(fa.sharedSizeBytes) + " dynamic limit " +
               std::to_string(fa.maxDynamicSharedSizeBytes) + " regs " + std::to_string(fa.numRegs);
    return fail(MM_ERR_CUDA, msg + "]");
}
#define CHECK_LAUNCH(fn, grid, threads, smem)                                                    \
    do {                                                                                         \
        int _rc = check_launch((const void*)(fn), (grid), (threads), (smem), __LINE__);          \
        if (_rc) return _rc;                                                                     \
    } while (0)

typedef void (*HashKernel)(Prob, Out, Work, const int8_t*, int, unsigned char*);

template <int KIND, int MODE, bool NUM>
HashKernel pick_hash_unordered(int tier, int* gw) {
    switch (tier) {
        case 0: *gw = 1; return k_push_hash<1, true, KIND, MODE, NUM>;
        case 1: *gw = 4; return k_push_hash<4, true, KIND, MODE, NUM>;
        case 2: *gw = 16; return k_push_hash<16, true, KIND, MODE, NUM>;
        default: *gw = 32; return k_push_hash<32, false, KIND, MODE, NUM>;
    }
}

template <int MODE>
HashKernel pick_hash_ordered(int tier, int* gw) {
    // shared tiers: groups split ordered rows by column; the global tier
    // keeps one warp per row (its rows are there for their table size, not
    // their work)
    if (tier == 3) { *gw = 1; return k_push_hash<1, false, 2, MODE, true>; }
    return pick_hash_unordered<2, MODE, true>(tier, gw);
}

template <int MODE>
HashKernel pick_hash_mode(int kind, int tier, bool numeric, int* gw) {
    if (!numeric) return pick_hash_unordered<0, MODE, false>(tier, gw);
    if (kind == 0) return pick_hash_unordered<0, MODE, true>(tier, gw);
    if (kind == 1) return pick_hash_unordered<1, MODE, true>(tier, gw);
    return pick_hash_ordered<MODE>(tier, gw);
}

HashKernel pick_hash(int kind, int mode, int tier, bool numeric, int* gw) {
    if (mode == MODE_PLAIN) return pick_hash_mode<MODE_PLAIN>(kind, tier, numeric, gw);
    if (mode == MODE_CTAB) return pick_hash_mode<MODE_CTAB>(kind, tier, numeric, gw);
    return pick_hash_mode<MODE_CSRCH>(kind, tier, numeric, gw);
}

typedef void (*DenseKernel)(Prob, Out, Work, int);

template <bool COMP, int GW>
DenseKernel pick_dense_gw(int kind, bool numeric) {
    if (!numeric) return k_push_dense<GW, 0, false, COMP>;
    if (kind == 0) return k_push_dense<GW, 0, true, COMP>;
    if (kind == 1) return k_push_dense<GW, 1, true, COMP>;
    return k_push_dense<GW, 2, true, COMP>;
}

template <bool COMP>
DenseKernel pick_dense(int kind, bool numeric, int gw) {
    if (gw == 1) return pick_dense_gw<COMP, 1>(kind, numeric);
    if (gw == 4) return pick_dense_gw<COMP, 4>(kind, numeric);
    return pick_dense_gw<COMP, 8>(kind, numeric);
}

typedef void (*RankKernel)(Prob, Out, Work, int, int, unsigned char*);

template <int KIND, bool MSA, bool NUM>
RankKernel pick_rank_unordered(int tier, int* gw) {
    switch (tier) {
        case 0: *gw = 1; return k_push_rank<1, true, KIND, MSA, NUM>;
#ifndef MM_RANK_T1_GW
#define MM_RANK_T1_GW 4
#endif
        case 1: *gw = MM_RANK_T1_GW; return k_push_rank<MM_RANK_T1_GW, true, KIND, MSA, NUM>;
#ifndef MM_RANK_T2_GW
#define MM_RANK_T2_GW 8
#endif
        case 2: *gw = MM_RANK_T2_GW; return k_push_rank<MM_RANK_T2_GW, true, KIND, MSA, NUM>;
        default: *gw = 32; return k_push_rank<32, false, KIND, MSA, NUM>;
    }
}

template <bool MSA>
RankKernel pick_rank(int kind, int tier, bool numeric, int* gw) {
    if (!numeric || kind == 0) return numeric ? pick_rank_unordered<0, MSA, true>(tier, gw)
                                              : pick_rank_unordered<0, MSA, false>(tier, gw);
    if (kind == 1) return pick_rank_unordered<1, MSA, true>(tier, gw);
    // ordered float64: groups split rows by column in the shared tiers, one
    // warp per row in the global tier (see pick_hash_ordered)
    if (tier == 3) { *gw = 1; return k_push_rank<1, false, 2, MSA, true>; }
    return pick_rank_unordered<2, MSA, true>(tier, gw);
}

// Launch every non-empty bin.  numeric=false: symbolic counts into out.row_nnz.
int launch_bins_on(mm_handle* h, bool numeric, const Out& out, const int* order, int norder);

// Launch every non-empty bin.  Bins run concurrently on NAUX auxiliary
// streams forked from / joined to the caller's stream, heaviest first, so the
// tail of one bin's kernel overlaps the next bin's blocks.
int launch_bins(mm_handle* h, bool numeric, const Out& out) {
    int order[NBINS], n = 0;
    for (int b = 1; b < NBINS; b++)
        if (h->sum.bin_count[b]) order[n++] = b;
    std::sort(order, order + n, [&](int x, int y) { return h->sum.bin_flops[x] > h->sum.bin_flops[y]; });
    return launch_bins_on(h, numeric, out, order, n);
}

// Sliced hub rows of a one-phase plain multiply as (row, slice) items
// (push_hash_items.cuh): item list, the items kernel, the join.
int launch_slice_items(mm_handle* h, const Out& out, const Work& wk, int kind, int cap_lg, size_t smem,
                       cudaStream_t st) {
    if (ITEM_GW != 16)   // the caller sized the 16-warp tier's block: one table, this kernel's batch and queues
        smem = ((size_t)1 << cap_lg) * (kind == 0 ? 8 : 16) + batch_bytes_rt(ITEM_GW, kind) +
               (size_t)ITEM_GW * 64 * (kind == 1 ? 24 : 8);
    const int64_t slice = (int64_t)MM_SLICE_EIGHTHS << (cap_lg - 3);
    const int64_t max_items = (int64_t)wk.count + (h->mask_nnz + slice - 1) / slice;
    if (max_items >= (1ll << 31)) return fail(MM_ERR_INTERNAL, "too many slice items");
    int32_t* buf = nullptr;
    const size_t words = (size_t)(wk.count + 1) + 3 * (size_t)max_items + 2;
    CU(cudaMallocAsync((void**)&buf, words * sizeof(int32_t), st));
    h->allocs.push_back(buf);
    int32_t* row_base = buf;
    int32_t* item_q = row_base + wk.count + 1;
    int32_t* item_s = item_q + max_items;
    int32_t* slice_cnt = item_s + max_items;
    int32_t* ctl = slice_cnt + max_items;   // [0] items, [1] fetch cursor
    CU(cudaMemsetAsync(ctl, 0, 2 * sizeof(int32_t), st));
    ++g_launches;
    k_slice_items<<<1, 1024, 0, st>>>(h->prob, wk, slice, row_base, item_q, item_s, ctl, max_items);
    CU(cudaGetLastError());
    void (*kern)(Prob, Out, Work, const int32_t*, const int32_t*, const int32_t*, int32_t*, int64_t, int,
                 const int32_t*, int32_t*) = kind == 0 ? k_push_hash_items<0> : k_push_hash_items<1>;
    int occ = 0, rc;
    if ((rc = kernel_occupancy((const void*)kern, ITEM_GW * 32, smem, &occ))) return rc;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(max_items, (int64_t)std::max(occ, 1) * h->num_sms));
    ++g_launches;
    if (debug_launches())
        fprintf(stderr, "[mm] sliced items rows %d max_items %lld cap_lg %d smem %zu grid %d occ %d\n", wk.count,
                (long long)max_items, cap_lg, smem, grid, occ);
    kern<<<grid, ITEM_GW * 32, smem, st>>>(h->prob, out, wk, item_q, item_s, ctl, ctl + 1, slice, cap_lg, row_base,
                                           slice_cnt);
    CU(cudaGetLastError());
    ++g_launches;
    k_slice_join<<<wk.count, 512, 0, st>>>(wk, out.off, h->prob.m_ptr, slice, row_base, slice_cnt, out.idx,
                                          (unsigned long long*)out.val, out.row_nnz);
    CU(cudaGetLastError());
    return MM_OK;
}

int launch_bins_on(mm_handle* h, bool numeric, const Out& out, const int* order, int norder) {
    cudaStream_t main_st = h->stream;
    // small multiplies: forking costs more host time than the overlap saves
    const bool concurrent = norder > 1 && h->sum.gen_flops >= (1ull << 22);
    if (concurrent) {
        if (!h->fork_ev) {
            CU(cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming));
            for (int q = 0; q < mm_handle::NAUX; q++) {
                CU(cudaStreamCreateWithFlags(&h->aux[q], cudaStreamNonBlocking));
                CU(cudaEventCreateWithFlags(&h->join_ev[q], cudaEventDisableTiming));
            }
        }
        CU(cudaEventRecord(h->fork_ev, main_st));
        for (int q = 0; q < mm_handle::NAUX && q < norder; q++) CU(cudaStreamWaitEvent(h->aux[q], h->fork_ev, 0));
    }
    int rc = MM_OK;
    int32_t* cursors = h->cursors + (numeric ? 2 * NBINS : NBINS);
    for (int oi = 0; oi < norder; oi++) {
        const int b = order[oi];
        const int cnt = h->sum.bin_count[b];
        cudaStream_t st = concurrent ? h->aux[oi % mm_handle::NAUX] : main_st;
        Work wk{h->rows_list + h->bin_off[b], cnt, cursors + b};
        // a lane per mask entry needs many rows to fill the GPU; small bins
        // run the warp-per-row kernel (same results)
        if (b == BIN_PULL_LANE && cnt >= 16384) {
            const int kind = numeric ? h->kind : 0;
            void (*kern)(Prob, Out, Work);
            if (!numeric) kern = k_pull_lane<0, false>;
            else if (kind == 0) kern = k_pull_lane<0, true>;
            else if (kind == 1) kern = k_pull_lane<1, true>;
            else kern = k_pull_lane<2, true>;
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, 0, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + 255) / 256, std::max(occ, 1) * h->num_sms));
            ++g_launches;
            kern<<<grid, 256, 0, st>>>(h->prob, out, wk);
            CU(cudaGetLastError());
            continue;
        }
        if (b == BIN_PULL || b == BIN_PULL_LANE) {
            int kind = numeric ? h->kind : 0;
            int stage = std::min(std::max(h->sum.max_na, 2), 512);
            stage += stage & 1;
            size_t esz = kind == 0 ? 4 : 12;
            size_t smem = (size_t)8 * stage * esz;
            void (*kern)(Prob, Out, Work, int);
            if (!numeric) kern = k_pull_inner<0, false>;
            else if (kind == 0) kern = k_pull_inner<0, true>;
            else if (kind == 1) kern = k_pull_inner<1, true>;
            else kern = k_pull_inner<2, true>;
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
            int grid = std::max(1, std::min((cnt + 7) / 8, std::max(occ, 1) * h->num_sms));
            ++g_launches;
            kern<<<grid, 256, smem, st>>>(h->prob, out, wk, stage);
            CU(cudaGetLastError());
            continue;
        }
        if (is_hash_bin(b)) {
            int mode = hash_bin_mode(b), tier = hash_bin_tier(b);
            int kind = numeric ? h->kind : 0;
            int gw = 1;
            // plain tier-3 rows (int64 / plus-pair): sliced over the 16-warp
            // tier's largest shared table (hash_row), their own launch
            // (decided by the multiply's kind, not the pass's: the symbolic pass of an
            // ordered float64 multiply runs as kind 0, but its rows were binned — and
            // their tables sized — for the global tier)
            const bool sliced = tier == 3 && mode == MODE_PLAIN && h->kind != 2;
            HashKernel kern = pick_hash(kind, mode, sliced ? 2 : tier, numeric, &gw);
            bool smem_table = tier < 3 || sliced;
            int threads = gw == 32 ? 1024 : (gw == 16 ? 512 : 256);
            int groups = threads / (32 * gw);
            int cap_lg = std::max(h->sum.bin_cap_lg[b], 5);
            // plain masks in shared memory: room for collision-free direct tables
            const int ltier = sliced ? 2 : tier;
            if (mode == MODE_PLAIN && smem_table && kind != 2 && h->direct_lg[ltier] > cap_lg)
                cap_lg = std::min(h->direct_lg[ltier], tier_cap_lg(kind == 0, ltier));
            size_t ebytes = kind == 0 ? 8 : 16;
            size_t table = ((size_t)1 << cap_lg) * ebytes;
            size_t batch = batch_bytes_rt(gw, kind);
            size_t queue = kind == 2 ? 0 : (size_t)64 * (kind == 1 ? 24 : 8);
            size_t smem = (smem_table ? groups * table : 0) + groups * batch + (threads / 32) * queue;
            if (smem > 227 * 1024) return fail(MM_ERR_INTERNAL, "hash tier table exceeds shared memory");
            if (sliced && numeric && h->split_slices && h->plan.phases == 1 && !h->plan.complemented) {
                if ((rc = launch_slice_items(h, out, wk, kind, cap_lg, smem, st))) return rc;
                continue;
            }
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, threads, smem, &occ))) return rc;
            int grid = std::max(1, std::min((cnt + groups - 1) / groups, std::max(occ, 1) * h->num_sms));
            unsigned char* gslab = nullptr;
            Prob pq = h->prob;
            if (!smem_table) {
                size_t bytes = (size_t)grid * groups * table;
                CU(cudaMallocAsync((void**)&gslab, bytes, st));
                h->allocs.push_back(gslab);
            } else if (sliced && h->slice_cursors) {
                // per-group slice cursors (one int64 per A entry of the row,
                // at most 1 GiB in all; wider rows search every slice)
                const int64_t per_group = ((int64_t)1 << 30) / (8 * (int64_t)grid * groups);
                pq.cursor_stride = std::min<int64_t>(std::max(h->sum.max_na, 1), per_group);
                CU(cudaMallocAsync((void**)&gslab, (size_t)grid * groups * pq.cursor_stride * 8, st));
                h->allocs.push_back(gslab);
            }
            // k-blocked passes (push_hash.cuh): B's index array against L2
            int passes = 1;
            if (numeric && kind == 0 && mode == MODE_PLAIN && tier == 2 && !sliced && h->plan.phases == 1 &&
                !h->plan.complemented && h->kblock_bytes > 0 && 4 * h->b_nnz > h->kblock_bytes + h->kblock_bytes / 2)
                passes = (int)std::min<int64_t>(64, (4 * h->b_nnz + h->kblock_bytes - 1) / h->kblock_bytes);
            if (debug_launches())
                fprintf(stderr, "[mm] hash bin %d rows %d gw %d threads %d cap_lg %d smem %zu grid %d occ %d passes %d\n",
                        b, cnt, gw, threads, cap_lg, smem, grid, occ, passes);
            Work wk_heavy = wk;
            if (passes > 1) {
                // the passes before the last fetch only the rows they cut
                int32_t* list = nullptr;
                CU(cudaMallocAsync((void**)&list, ((size_t)cnt + 1) * sizeof(int32_t), st));
                h->allocs.push_back(list);
                CU(cudaMemsetAsync(list, 0xff, (size_t)cnt * sizeof(int32_t), st));
                CU(cudaMemsetAsync(list + cnt, 0, sizeof(int32_t), st));
                ++g_launches;
                const int sg = std::max(1, std::min((cnt + 255) / 256, h->num_sms * 8));
                k_kb_select<<<sg, 256, 0, st>>>(h->prob, wk, (int64_t)MM_SLICE_EIGHTHS << (cap_lg - 3),
                                                h->kblock_min_flops, list, list + cnt);
                CU(cudaGetLastError());
                wk_heavy.rows = list;
            }
            for (int ps = 0; ps < passes; ps++) {
                if (passes > 1) {
                    pq.kb_pass = ps == 0 ? 1 : (ps == passes - 1 ? 3 : 2);
                    pq.kb_min_flops = h->kblock_min_flops;
                    pq.kb_lo = h->b_nnz / passes * ps;
                    pq.kb_hi = h->b_nnz / passes * (ps + 1);
                    if (ps) CU(cudaMemsetAsync(wk.cursor, 0, sizeof(int32_t), st));   // the bin's row fetch restarts
                }
                ++g_launches;
                kern<<<grid, threads, smem, st>>>(pq, out, ps + 1 < passes ? wk_heavy : wk, h->row_cap_lg, cap_lg, gslab);
                CHECK_LAUNCH(kern, grid, threads, smem);
            }
            continue;
        }
        if (is_msa_bin(b) || is_mca_bin(b)) {
            const bool msa = is_msa_bin(b);
            const int tier = b - (msa ? BIN_MSA0 : BIN_MCA0);
            const int kind = numeric ? h->kind : 0;
            int gw = 1;
            RankKernel kern = msa ? pick_rank<true>(kind, tier, numeric, &gw) : pick_rank<false>(kind, tier, numeric, &gw);
            const bool smem_region = tier < 3;
            const int threads = gw == 32 ? 1024 : (gw == 16 ? 512 : 256);
            const int groups = threads / (32 * gw);
            const int words_max = std::max(h->sum.bin_words[b], 1);
            const int nm_max = std::max(h->sum.bin_nmmax[b], 1);
            size_t rb = rank_region_bytes_rt(kind, msa, words_max, nm_max);
            rb = (rb + 15) & ~(size_t)15;
            const size_t batch = batch_bytes_rt(gw, kind);
            const size_t smem = (smem_region ? groups * rb : 0) + groups * batch;
            if (smem > 227 * 1024) return fail(MM_ERR_INTERNAL, "rank tier region exceeds shared memory");
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, threads, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + groups - 1) / groups, std::max(occ, 1) * h->num_sms));
            unsigned char* gslab = nullptr;
            if (!smem_region) {
                CU(cudaMallocAsync((void**)&gslab, (size_t)grid * groups * rb, st));
                h->allocs.push_back(gslab);
            }
            ++g_launches;
            if (debug_launches())
                fprintf(stderr, "[mm] rank bin %d rows %d gw %d threads %d words %d nm %d smem %zu grid %d occ %d\n", b,
                        cnt, gw, threads, words_max, nm_max, smem, grid, occ);
            kern<<<grid, threads, smem, st>>>(h->prob, out, wk, words_max, nm_max, gslab);
            CHECK_LAUNCH(kern, grid, threads, smem);
            continue;
        }
        if (b == BIN_MSAW) {
            // windowed MSA (hub rows): one 16-warp group per block, per-group
            // slice cursors in a global slab
            const int kind = numeric ? h->kind : 0;
            void (*kern)(Prob, Out, Work, unsigned char*) = nullptr;
            if (!numeric) kern = k_push_msaw<0, false>;
            else if (kind == 0) kern = k_push_msaw<0, true>;
            else if (kind == 1) kern = k_push_msaw<1, true>;
            else return fail(MM_ERR_INTERNAL, "windowed MSA bin with ordered float64 rows");
            const size_t smem = ((msaw_region_bytes(kind) + 15) & ~(size_t)15) + batch_bytes_rt(MSAW_GW, kind);
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, MSAW_GW * 32, smem, &occ))) return rc;
            const int grid = std::max(1, std::min(cnt, std::max(occ, 1) * h->num_sms));
            Prob pq = h->prob;
            unsigned char* gslab = nullptr;
            if (h->slice_cursors) {
                const int64_t per_group = ((int64_t)1 << 30) / (8 * (int64_t)grid);
                pq.cursor_stride = std::min<int64_t>(std::max(h->sum.max_na, 1), per_group);
                CU(cudaMallocAsync((void**)&gslab, (size_t)grid * pq.cursor_stride * 8, st));
                h->allocs.push_back(gslab);
            }
            ++g_launches;
            if (debug_launches())
                fprintf(stderr, "[mm] msa-window bin rows %d smem %zu grid %d occ %d\n", cnt, smem, grid, occ);
            kern<<<grid, MSAW_GW * 32, smem, st>>>(pq, out, wk, gslab);
            CU(cudaGetLastError());
            continue;
        }
        if (b == BIN_F64D) {
            // ordered float64, deferred hits: symbolic runs the plain
            // order-free hash kernel (counts only)
            if (!numeric || h->kind != 2) {
                int gw = 1;
                HashKernel kern = pick_hash(0, MODE_PLAIN, 0, false, &gw);
                if (numeric) return fail(MM_ERR_INTERNAL, "deferred float64 bin without float64 values");
                const int cap_lg = std::max(h->sum.bin_cap_lg[b], 5);
                const size_t smem = 8 * (((size_t)8 << cap_lg) + batch_bytes_rt(1, 0)) + 8 * (size_t)64 * 8;
                int occ = 0;
                if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
                const int grid = std::max(1, std::min((cnt + 7) / 8, std::max(occ, 1) * h->num_sms));
                ++g_launches;
                kern<<<grid, 256, smem, st>>>(h->prob, out, wk, h->row_cap_lg, cap_lg, nullptr);
                CU(cudaGetLastError());
                continue;
            }
            const int nm_max = std::max(h->sum.bin_nmmax[b], 1);
            const size_t smem = 8 * defer_warp_bytes(nm_max);
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)k_push_f64_defer<true>, 256, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + 7) / 8, std::max(occ, 1) * h->num_sms));
            ++g_launches;
            if (debug_launches())
                fprintf(stderr, "[mm] f64-defer bin rows %d nm_max %d smem %zu grid %d occ %d\n", cnt, nm_max, smem,
                        grid, occ);
            k_push_f64_defer<true><<<grid, 256, smem, st>>>(h->prob, out, wk, nm_max, 0ll, Tail{});
            CU(cudaGetLastError());
            continue;
        }
        if (b == BIN_HEAP0 + 3) {
            // complemented heap rows with > 32 A entries: iterator state in a
            // per-warp global slab sized by the bin's widest A row
            const int kind = numeric ? h->kind : 0;
            void (*kern)(Prob, Out, Work, int, unsigned char*) = nullptr;
            if (!numeric) kern = k_push_heap_comp<0, false>;
            else if (kind == 0) kern = k_push_heap_comp<0, true>;
            else if (kind == 1) kern = k_push_heap_comp<1, true>;
            else kern = k_push_heap_comp<2, true>;
            const int na_max = std::max(h->sum.bin_words[b], 1);
            const size_t per_block = 8 * heap_iter_bytes(na_max);
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, 0, &occ))) return rc;
            int grid = std::max(1, std::min((cnt + 7) / 8, std::max(occ, 1) * h->num_sms));
            grid = (int)std::max<size_t>(1, std::min<size_t>(grid, ((size_t)1 << 30) / per_block));
            unsigned char* gslab = nullptr;
            CU(cudaMallocAsync((void**)&gslab, (size_t)grid * per_block, st));
            h->allocs.push_back(gslab);
            ++g_launches;
            kern<<<grid, 256, 0, st>>>(h->prob, out, wk, na_max, gslab);
            CU(cudaGetLastError());
            continue;
        }
        if (is_heap_bin(b)) {
            const int sub = b - BIN_HEAP0;
            const bool comp_rows = sub == 2;
            const int kind = numeric ? h->kind : 0;
            const int nm_max = std::max(h->sum.bin_nmmax[b], 1);
            void (*kern)(Prob, Out, Work, int, int, unsigned char*) = nullptr;
            if (comp_rows) {
                if (!numeric) kern = k_push_heap<0, false, true>;
                else if (kind == 0) kern = k_push_heap<0, true, true>;
                else if (kind == 1) kern = k_push_heap<1, true, true>;
                else kern = k_push_heap<2, true, true>;
            } else {
                if (!numeric) kern = k_push_heap<0, false, false>;
                else if (kind == 0) kern = k_push_heap<0, true, false>;
                else if (kind == 1) kern = k_push_heap<1, true, false>;
                else kern = k_push_heap<2, true, false>;
            }
            const size_t wbytes = comp_rows ? 0 : (((size_t)(kind == 0 ? 4 : 12) * nm_max + 15) & ~(size_t)15);
            const bool in_smem = sub == 0;
            const size_t smem = in_smem ? 8 * wbytes : 0;
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + 7) / 8, std::max(occ, 1) * h->num_sms));
            unsigned char* gslab = nullptr;
            if (!in_smem && !comp_rows) {
                CU(cudaMallocAsync((void**)&gslab, (size_t)grid * 8 * wbytes, st));
                h->allocs.push_back(gslab);
            }
            ++g_launches;
            kern<<<grid, 256, smem, st>>>(h->prob, out, wk, nm_max, h->plan.n_inspect, gslab);
            CU(cudaGetLastError());
            continue;
        }
        if (is_msad_bin(b) || is_msadc_bin(b)) {
            const bool comp = is_msadc_bin(b);
            const int tier = b - (comp ? BIN_MSADC0 : BIN_MSAD0);
            const int kind = numeric ? h->kind : 0;
            void (*kern)(Prob, Out, Work, int) = nullptr;
            const int gw = tier == 0 ? 1 : (tier == 1 ? MM_RANK_T1_GW : MM_RANK_T2_GW);
            if (comp) kern = pick_dense<true>(kind, numeric, gw);
            else kern = pick_dense<false>(kind, numeric, gw);
            const int groups = 256 / (32 * gw);
            const int words_max = std::max(h->sum.bin_words[b], 1);
            const size_t rb = (dense_region_bytes(kind, words_max) + 15) & ~(size_t)15;
            const size_t batch = batch_bytes_rt(gw, kind);
            const size_t smem = groups * (rb + batch);
            if (smem > 227 * 1024) return fail(MM_ERR_INTERNAL, "dense MSA window exceeds shared memory");
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + groups - 1) / groups, std::max(occ, 1) * h->num_sms));
            if (debug_launches())
                fprintf(stderr, "[mm] dense-msa bin %d rows %d gw %d words %d smem %zu grid %d occ %d\n", b, cnt, gw,
                        words_max, smem, grid, occ);
            ++g_launches;
            kern<<<grid, 256, smem, st>>>(h->prob, out, wk, words_max);
            CU(cudaGetLastError());
            continue;
        }
        if (is_msas_bin(b)) {
            const int tier = b - BIN_MSAS0;
            const int kind = numeric ? h->kind : 0;
            void (*kern)(Prob, Out, Work, int, int, int) = nullptr;
            int gw = kind == 2 ? 1 : (tier == 0 ? 1 : (tier == 1 ? 4 : 8));
            if (!numeric || kind == 0) {
                if (gw == 1) kern = numeric ? k_push_msas<1, 0, true> : k_push_msas<1, 0, false>;
                else if (gw == 4) kern = numeric ? k_push_msas<4, 0, true> : k_push_msas<4, 0, false>;
                else kern = numeric ? k_push_msas<8, 0, true> : k_push_msas<8, 0, false>;
            } else if (kind == 1) {
                kern = gw == 1 ? k_push_msas<1, 1, true> : (gw == 4 ? k_push_msas<4, 1, true> : k_push_msas<8, 1, true>);
            } else {
                kern = k_push_msas<1, 2, true>;
            }
            const int groups = 256 / (32 * gw);
            const int d_max = std::max(h->sum.bin_words[b], 1);
            const int blk_max = std::max(h->sum.bin_cap_lg[b], 1);
            const int nm_max = std::max(h->sum.bin_nmmax[b], 1);
            size_t rb = (size_t)(kind == 0 ? 0 : 8) * nm_max + 4 * (size_t)nm_max + 2 * (size_t)((d_max + 1) & ~1) +
                        192 * (size_t)blk_max;
            rb = (rb + 15) & ~(size_t)15;
            const size_t batch = batch_bytes_rt(gw, kind);
            const size_t smem = groups * (rb + batch);
            if (smem > 227 * 1024) return fail(MM_ERR_INTERNAL, "sparse MSA region exceeds shared memory");
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + groups - 1) / groups, std::max(occ, 1) * h->num_sms));
            if (debug_launches())
                fprintf(stderr, "[mm] sparse-msa bin %d rows %d gw %d dir %d blk %d nm %d smem %zu grid %d occ %d\n",
                        b, cnt, gw, d_max, blk_max, nm_max, smem, grid, occ);
            ++g_launches;
            kern<<<grid, 256, smem, st>>>(h->prob, out, wk, d_max, blk_max, nm_max);
            CU(cudaGetLastError());
            continue;
        }
        if (b == BIN_SINGLE) {
            const int kind = numeric ? h->kind : 0;
            const bool comp = h->plan.complemented != 0;
            void (*kern)(Prob, Out, Work, int) = nullptr;
            if (!numeric) kern = comp ? k_push_single<0, false, true> : k_push_single<0, false, false>;
            else if (kind == 0) kern = comp ? k_push_single<0, true, true> : k_push_single<0, true, false>;
            else if (kind == 1) kern = comp ? k_push_single<1, true, true> : k_push_single<1, true, false>;
            else kern = comp ? k_push_single<2, true, true> : k_push_single<2, true, false>;
            const int words_max = std::max(h->sum.bin_words[b], 1);
            // two 4-warp groups per block while the bitmaps fit, else one group
            const size_t smem = 2 * 4 * (size_t)words_max;
            if (smem > 227 * 1024) return fail(MM_ERR_INTERNAL, "single-entry bitmap exceeds shared memory");
            int occ = 0;
            if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
            const int grid = std::max(1, std::min((cnt + 1) / 2, std::max(occ, 1) * h->num_sms));
            ++g_launches;
            kern<<<grid, 256, smem, st>>>(h->prob, out, wk, words_max);
            CU(cudaGetLastError());
            continue;
        }
        return fail(MM_ERR_INTERNAL, "unhandled bin " + std::to_string(b));
    }
    if (concurrent) {
        for (int q = 0; q < mm_handle::NAUX && q < norder; q++) {
            CU(cudaEventRecord(h->join_ev[q], h->aux[q]));
            CU(cudaStreamWaitEvent(main_st, h->join_ev[q], 0));
        }
    }
    return MM_OK;
}

void mark(mm_handle* h, int k) {
    if (h->prof) cudaEventRecord(h->ev[k], h->stream);
}

int sync_read(mm_handle* h, void* dst, const void* src, size_t bytes) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return MM_OK;
}

// Fused tail (fused_tail.cuh): arguments of one multiply, and the host's wait
// for the last block's counters in mapped memory (a spin on the sequence
// word; past 2 ms the stream is synchronised, which also surfaces faults).
Tail make_tail(mm_handle* h) {
    Tail t{};
    t.done = h->d_done;
    t.nrows = h->nrows;
    t.row_nnz = h->row_nnz;
    t.slot_off = h->bound_off;
    t.tmp_idx = h->tmp_idx;
    t.tmp_val = h->tmp_val;
    t.c_row_ptr = h->c_row_ptr;
    t.c_idx = h->early_idx;
    t.c_val = h->early_val;
    t.summary = h->d_summary;
    t.host = h->h_tail;
    t.seq = ++h->tail_seq;
    return t;
}

int wait_tail(mm_handle* h, cudaStream_t st, unsigned long long seq) {
    volatile unsigned long long* p = &h->h_tail->seq;
    h->tail_stream = st;
    const auto t0 = std::chrono::steady_clock::now();
    int spins = 0;
    while (*p != seq) {
        if ((++spins & 63) == 0 &&
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() > 2000.0) {
            CU(cudaStreamSynchronize(st));
            if (*p != seq) return fail(MM_ERR_INTERNAL, "fused tail did not report");
            break;
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    // the rest of the multiply reads the counters from the pinned summary
    const TailResult r = *h->h_tail;
#ifdef MM_TAIL_DEBUG
    if (host_trace())
        fprintf(stderr, "[mm tail] A %.1f B %.1f C1 %.1f C2 %.1f us, report %.1f us, fence %.1f us, spins %d\n",
                (r.dbg[4] - r.dbg[0]) * 1e-3, (r.dbg[5] - r.dbg[4]) * 1e-3, (r.dbg[6] - r.dbg[5]) * 1e-3,
                (r.dbg[1] - r.dbg[6]) * 1e-3, (r.dbg[2] - r.dbg[1]) * 1e-3, (r.dbg[3] - r.dbg[2]) * 1e-3, spins);
#endif
    std::memset(h->h_summary, 0, sizeof(Summary));
    h->h_summary->gen_flops = r.gen_flops;
    h->h_summary->evaluated = r.evaluated;
    h->h_summary->total_nnz = r.total_nnz;
    h->h_summary->bin_count[BIN_EMPTY] = r.empty_rows;
    h->h_summary->pad = r.overflow;
    h->h_summary->flag = r.bound_flag;
    return MM_OK;
}

bool use_fused_tail(const mm_handle* h, int64_t m, int64_t mask_nnz) {
    return h->d_done && h->h_tail && h->fused_rows > 0 && m <= h->fused_rows && mask_nnz <= h->fused_nnz;
}

// mm_multiply on a small plain one-phase problem: C's arrays are known before
// nnz(C) is, so the compaction (thread per row: every row fits one slot range)
// is queued right behind the scan and the summary readback is the only sync.
// A row the single pass could not take (fallback) only leaves stale C entries,
// which the fallback's own compaction overwrites.
int early_compact(mm_handle* h, cudaStream_t st) {
    const int64_t m = h->nrows;
    if (!h->early_idx || m <= 0 || m > h->tiny_rows) return MM_OK;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)h->num_sms * 8));
    ++g_launches;
    if (h->out_f64)
        k_compact_rowwise<double><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                        (const double*)h->tmp_val, h->c_row_ptr, h->early_idx,
                                                        (double*)h->early_val, nullptr);
    else
        k_compact_rowwise<long long><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                           (const long long*)h->tmp_val, h->c_row_ptr, h->early_idx,
                                                           (long long*)h->early_val, nullptr);
    CU(cudaGetLastError());
    h->compacted = true;
    return MM_OK;
}

int begin_impl(mm_handle* h, const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
               const mm_matrix_t* b, const mm_matrix_t* bt, cudaStream_t st, bool symbolic_only,
               int64_t* counts_out, int64_t* out_nnz) {
    trace("^begin");
    int rc = validate(plan, mask, a, b, bt);
    if (rc) return rc;
    if (h->active) release(h);
    if (h->tail_stream && h->tail_stream != st) {
        // the previous fused multiply returned before its kernel retired: its
        // ticket reset must land before another stream's multiply starts
        CU(cudaStreamSynchronize(h->tail_stream));
    }
    h->tail_stream = nullptr;
    h->stream = st;
    h->compacted = false;
    h->launch_base = g_launches;
    mark(h, 0);
    h->plan = *plan;
    h->nrows = mask->nrows;
    h->ncols = mask->ncols;
    const bool comp = plan->complemented != 0;
    const bool pair = plan->semiring == MM_SR_PLUS_PAIR;
    h->kind = pair ? 0 : (plan->dtype == MM_DTYPE_FLOAT64 ? 2 : 1);
    h->out_f64 = plan->dtype == MM_DTYPE_FLOAT64;
    Prob& p = h->prob;
    p.a_ptr = a->ptr; p.a_idx = a->idx; p.a_val = a->values;
    p.b_ptr = b->ptr; p.b_idx = b->idx; p.b_val = b->values;
    p.m_ptr = mask->ptr; p.m_idx = mask->idx;
    const bool use_bt = bt && bt->ptr && (plan->algorithm == MM_ALGO_INNER || plan->algorithm == MM_ALGO_AUTO);
    p.bt_ptr = use_bt ? bt->ptr : nullptr;
    p.bt_idx = use_bt ? bt->idx : nullptr;
    p.bt_val = use_bt ? bt->values : nullptr;
    p.nrows = h->nrows;
    p.ncols = h->ncols;
    AnalyzeParams& ap = h->ap;
    switch (plan->algorithm) {
        case MM_ALGO_INNER: ap.family = FAM_PULL; break;
        case MM_ALGO_AUTO: ap.family = FAM_AUTO; break;
        case MM_ALGO_MSA: ap.family = FAM_MSA; break;
        case MM_ALGO_MCA: ap.family = FAM_MCA; break;
        case MM_ALGO_HEAP:
        case MM_ALGO_HEAPDOT: ap.family = FAM_HEAP; break;
        default: ap.family = FAM_HASH; break;   // hash; heap forms: see classify_row
    }
    ap.tier_flops0 = h->tier_flops0;
    ap.tier_flops1 = h->tier_flops1;
    ap.tier_flops1_hash = h->tier_flops1_hash;
    ap.capc_lg = h->capc_lg;
    ap.load_shift = h->load_shift;
    ap.load_shift_wide = h->load_shift_wide;
    for (int t = 0; t < 3; t++) ap.rank_budget[t] = h->rank_budget[t];
    ap.auto_mca_nm = h->auto_mca_nm;
    ap.comp = comp;
    ap.ordered = h->kind == 2;
    ap.pair = pair;
    ap.vbytes = pair ? 0 : 8;
    ap.has_bt = use_bt;
    ap.done = nullptr;
    ap.b_len = nullptr;
    const int64_t m = h->nrows;

    // One pool allocation carves every per-multiply array; summary and fetch
    // cursors sit together at the front so a single memset clears both.
    const bool need_bound = comp && plan->phases == 1 && !symbolic_only;
    const bool plain_1p = !comp && plan->phases == 1 && !symbolic_only;
    h->mask_nnz = mask->nnz;
    h->b_nnz = b->nnz;
    const int64_t scan_elems = scan_scratch_elems(m);
    size_t off = 0;
    auto carve = [&](size_t bytes) { size_t at = off; off += (bytes + 255) & ~(size_t)255; return at; };
    const size_t zero_bytes = sizeof(Summary) + (3 * NBINS + 4) * sizeof(int32_t);   // + long-row count
    const size_t o_sum = carve(zero_bytes);
    const size_t o_long = carve(m * sizeof(int32_t));
    const size_t o_flops = carve(m * sizeof(int64_t));
    const size_t o_nnz = carve(m * sizeof(int64_t));
    const size_t o_ptr = carve((m + 1) * sizeof(int64_t));
    const size_t o_bound = need_bound ? carve(m * sizeof(int64_t)) : 0;
    const size_t o_bptr = need_bound ? carve((m + 1) * sizeof(int64_t)) : 0;
    const size_t o_scan = carve(scan_elems * sizeof(int64_t));
    const size_t o_rows = carve(m * sizeof(int32_t));
    const size_t o_bin = carve(m);
    const size_t o_cap = carve(m);
    // int32 row lengths of B for the analysis (one 4-byte gather per A entry
    // instead of two 8-byte offsets): pays when A has several entries per row of B
    const bool use_blen = h->blen_on && a->nnz >= 4 * b->nrows && a->nnz >= (1 << 20);
    const size_t o_blen = use_blen ? carve((size_t)b->nrows * sizeof(int32_t)) : 0;
    const size_t o_tidx = plain_1p ? carve(mask->nnz * sizeof(int32_t)) : 0;
    const size_t o_tval = plain_1p ? carve(mask->nnz * 8) : 0;
    unsigned char* slab = nullptr;
    if ((rc = dalloc(h, &slab, off))) return rc;
    h->d_summary = (Summary*)(slab + o_sum);
    h->cursors = (int32_t*)(slab + o_sum + sizeof(Summary));
    int* long_n = (int*)(h->cursors + 3 * NBINS);
    int32_t* long_rows = (int32_t*)(slab + o_long);
    h->row_flops = (int64_t*)(slab + o_flops);
    h->row_nnz = (int64_t*)(slab + o_nnz);
    // mm_multiply hands in the caller's row pointer: the scan writes it directly
    h->c_row_ptr = h->user_row_ptr ? h->user_row_ptr : (int64_t*)(slab + o_ptr);
    h->bound = need_bound ? (int64_t*)(slab + o_bound) : nullptr;
    h->bound_ptr = need_bound ? (int64_t*)(slab + o_bptr) : nullptr;
    h->scan_scratch = (int64_t*)(slab + o_scan);
    h->rows_list = (int32_t*)(slab + o_rows);
    h->row_bin = (uint8_t*)(slab + o_bin);
    h->row_cap_lg = (int8_t*)(slab + o_cap);
    h->tmp_idx = plain_1p ? (int32_t*)(slab + o_tidx) : nullptr;
    h->tmp_val = plain_1p ? (void*)(slab + o_tval) : nullptr;
    p.row_flops = h->row_flops;
    trace("slab");
    CU(cudaMemsetAsync(h->d_summary, 0, zero_bytes, st));

    auto run_analysis = [&]() -> int {
        if (m <= 0) return MM_OK;
        if (use_blen && !ap.b_len) {
            int32_t* blen = (int32_t*)(slab + o_blen);
            const int bg = (int)std::max<int64_t>(1, std::min<int64_t>((b->nrows + 255) / 256, (int64_t)h->num_sms * 8));
            ++g_launches;
            k_row_len<<<bg, 256, 0, st>>>(b->nrows, b->ptr, blen);
            CU(cudaGetLastError());
            ap.b_len = blen;
        }
        int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)h->num_sms * 8));
        int64_t* zero_nnz = symbolic_only ? nullptr : h->row_nnz;
        ++g_launches;
        if (ap.b_len)
            k_analyze<true><<<grid, 256, 0, st>>>(p, ap, h->row_flops, h->bound, h->row_bin, h->row_cap_lg,
                                                  h->d_summary, zero_nnz, long_rows, long_n);
        else
            k_analyze<false><<<grid, 256, 0, st>>>(p, ap, h->row_flops, h->bound, h->row_bin, h->row_cap_lg,
                                                   h->d_summary, zero_nnz, long_rows, long_n);
        CU(cudaGetLastError());
        if (a->nnz > LONG_ROW || (ap.has_bt && mask->nnz > LONG_ROW)) {   // a long row is possible
            ++g_launches;
            if (ap.b_len)
                k_analyze_long<true><<<h->num_sms * 2, 256, 0, st>>>(p, ap, h->row_flops, h->bound, h->row_bin,
                                                                      h->row_cap_lg, h->d_summary, zero_nnz,
                                                                      long_rows, long_n);
            else
                k_analyze_long<false><<<h->num_sms * 2, 256, 0, st>>>(p, ap, h->row_flops, h->bound, h->row_bin,
                                                                       h->row_cap_lg, h->d_summary, zero_nnz,
                                                                       long_rows, long_n);
            CU(cudaGetLastError());
        }
        return MM_OK;
    };
    // ---- direct path for ordered float64 plain one-phase multiplies: no
    // analysis pass — the deferred-hit kernel takes every row, sums the
    // generated flops itself, and leaves rows it cannot take (mask row over
    // 128 entries, products over the 1-warp tier bound) marked; one host
    // sync.  Marked rows then run on the binned path below.
    // with B^T (auto), only when the average pull cost per mask entry does not
    // undercut push by 3x (the per-row push/pull model needs the analysis)
    const double est_push = (double)a->nnz * ((double)b->nnz / (double)std::max<int64_t>(b->nrows, 1));
    const double est_pull = (double)mask->nnz * ((double)b->nnz / (double)std::max<int64_t>(b->ncols, 1) +
                                                 (double)a->nnz / (double)std::max<int64_t>(m, 1));
    // ... and only when the mask is neither nearly empty (under a quarter of
    // the rows can have an entry: the analysis never launches the others,
    // the direct kernel would walk their A rows to count products) nor mostly
    // wider than the kernel's 128-entry rows (batched BC's backward steps)
    const bool mask_fits = 4 * mask->nnz >= m && mask->nnz <= 64 * m;
    const bool direct = plain_1p && h->kind == 2 && m > 0 && h->direct_on && (!use_bt || 3.0 * est_pull >= est_push) &&
                        plan->algorithm == MM_ALGO_AUTO && mask_fits;
    bool have_summary = false;
    if (direct) {
        h->bound_off = mask->ptr;   // bounds = mask row lengths (multiply.py:233)
        Out o{};
        o.off = h->bound_off;
        o.idx = h->tmp_idx;
        o.val = h->tmp_val;
        o.row_nnz = h->row_nnz;
        o.evaluated = &h->d_summary->evaluated;
        o.out_f64 = 1;
        o.overflow = &h->d_summary->pad;
        o.gen_flops = &h->d_summary->gen_flops;
        o.empty_rows = &h->d_summary->bin_count[BIN_EMPTY];
        // mask rows up to 128 entries (wider ones fall back): 8 warps x 6 KB,
        // four blocks per SM
        const int nm_max = 128;
        const size_t smem = 8 * defer_warp_bytes(nm_max);
        int occ = 0;
        if ((rc = kernel_occupancy((const void*)k_push_f64_defer<true>, 256, smem, &occ))) return rc;
        const int grid = std::max(1, std::min((int)((m + 7) / 8), std::max(occ, 1) * h->num_sms));
        Work wk{nullptr, (int32_t)m, h->cursors + 2 * NBINS};
        ++g_launches;
        if (use_fused_tail(h, m, mask->nnz)) {
            // one launch: the last block scans, compacts and reports (fused_tail.cuh)
            const size_t fsmem = std::max(smem, tail_smem_bytes());
            if ((rc = kernel_occupancy((const void*)k_push_f64_defer<true, true>, 256, fsmem, &occ))) return rc;
            const int fgrid = std::max(1, std::min((int)((m + 7) / 8), std::max(occ, 1) * h->num_sms));
            const Tail tail = make_tail(h);
            k_push_f64_defer<true, true><<<fgrid, 256, fsmem, st>>>(h->prob, o, wk, nm_max, (long long)h->tier_flops0,
                                                                  tail);
            CU(cudaGetLastError());
            trace("direct1");
            if ((rc = wait_tail(h, st, tail.seq))) return rc;
            h->compacted = h->early_idx != nullptr && !h->h_summary->pad;
        } else {
            k_push_f64_defer<true><<<grid, 256, smem, st>>>(h->prob, o, wk, nm_max, (long long)h->tier_flops0, Tail{});
            CU(cudaGetLastError());
            if ((rc = exclusive_scan(h->row_nnz, m, h->c_row_ptr, st, h->scan_scratch, h->bound_off,
                                     &h->d_summary->flag, &h->d_summary->total_nnz)))
                return rc;
            trace("direct");
            if ((rc = early_compact(h, st))) return rc;
            if ((rc = sync_read(h, h->h_summary, h->d_summary, sizeof(Summary)))) return rc;
        }
        if (!h->h_summary->pad) {
            h->sum = *h->h_summary;
            mark(h, 1);
            mark(h, 2);
            mark(h, 3);
            h->stats = mm_stats_t{};
            h->stats.generated_flops = (int64_t)h->sum.gen_flops;
            h->stats.rows_empty = h->sum.bin_count[BIN_EMPTY];
            h->stats.rows_push = m - h->stats.rows_empty;
            h->total_nnz = h->sum.total_nnz;
            h->stats.evaluated_multiplies = (int64_t)h->sum.evaluated;
            h->bound_flag = h->sum.flag;
            for (int b = 0; b < NBINS; b++) h->sum.bin_count[b] = 0;   // profile: every row in one launch
            h->sum.bin_count[BIN_F64D] = (int)m;
            mark(h, 4);
            *out_nnz = h->total_nnz;
            h->active = true;
            return MM_OK;
        }
        h->compacted = false;
        // rows the direct pass could not take (row_nnz = -1) go through the
        // binned path; its rows stay done (the analysis skips them, their
        // flops / evaluated / empty counts are already in the summary)
        CU(cudaMemsetAsync(&h->d_summary->flag, 0, 2 * sizeof(int), st));          // flag, pad
        CU(cudaMemsetAsync(h->cursors, 0, (3 * NBINS + 4) * sizeof(int32_t), st));  // fetch cursors, long rows
        ap.done = h->row_nnz;
    }
    // ---- the smallest plain one-phase problems: ONE launch (k_tiny_hash: the
    // 1-warp hash kernel over every row, flops summed by the kernel, then the
    // fused tail: scan, compaction, counters into mapped host memory).
    const bool tiny_ok = !direct && plain_1p && m > 0 && m <= h->tiny_rows && mask->nnz <= h->tiny_nnz &&
                         a->nnz <= h->tiny_nnz && (plan->algorithm == MM_ALGO_AUTO || plan->algorithm == MM_ALGO_HASH);
    bool fused_overflow = false;
    if (tiny_ok && use_fused_tail(h, m, mask->nnz) && a->nnz <= h->fused_nnz) {
        h->bound_off = mask->ptr;   // bounds = mask row lengths (multiply.py:233)
        Out o{};
        o.off = h->bound_off;
        o.idx = h->tmp_idx;
        o.val = h->tmp_val;
        o.row_nnz = h->row_nnz;
        o.evaluated = &h->d_summary->evaluated;
        o.out_f64 = h->out_f64;
        o.overflow = &h->d_summary->pad;
        o.gen_flops = &h->d_summary->gen_flops;
        o.empty_rows = &h->d_summary->bin_count[BIN_EMPTY];
        void (*kern)(Prob, Out, Work, int, Tail) =
            h->kind == 0 ? k_tiny_hash<0> : (h->kind == 1 ? k_tiny_hash<1> : k_tiny_hash<2>);
        const int cap_lg = h->kind == 0 ? 10 : 9;
        const size_t ebytes = h->kind == 0 ? 8 : 16;
        const size_t queue = h->kind == 2 ? 0 : (size_t)64 * (h->kind == 1 ? 24 : 8);
        const size_t smem = std::max(8 * (((size_t)1 << cap_lg) * ebytes + batch_bytes_rt(1, h->kind)) + 8 * queue,
                                     tail_smem_bytes());
        int occ = 0;
        if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
        const int grid = std::max(1, std::min((int)((m + 7) / 8), std::max(occ, 1) * h->num_sms));
        Work wk{nullptr, (int32_t)m, h->cursors + 2 * NBINS};
        const Tail tail = make_tail(h);
        ++g_launches;
        kern<<<grid, 256, smem, st>>>(h->prob, o, wk, cap_lg, tail);
        CU(cudaGetLastError());
        trace("tiny1");
        if ((rc = wait_tail(h, st, tail.seq))) return rc;
        if (!h->h_summary->pad) {
            h->compacted = h->early_idx != nullptr;
            h->sum = *h->h_summary;
            mark(h, 1);
            mark(h, 2);
            mark(h, 3);
            h->stats = mm_stats_t{};
            h->stats.generated_flops = (int64_t)h->sum.gen_flops;
            h->stats.rows_empty = h->sum.bin_count[BIN_EMPTY];
            h->stats.rows_push = m - h->stats.rows_empty;
            h->total_nnz = h->sum.total_nnz;
            h->stats.evaluated_multiplies = (int64_t)h->sum.evaluated;
            h->bound_flag = h->sum.flag;
            // profile: every non-empty row ran the 1-warp plain hash kernel
            h->sum.bin_count[hash_bin(MODE_PLAIN, 0, 0)] = (int)h->stats.rows_push;
            h->sum.bin_flops[hash_bin(MODE_PLAIN, 0, 0)] = h->sum.gen_flops;
            trace("sync2");
            mark(h, 4);
            *out_nnz = h->total_nnz;
            h->active = true;
            return MM_OK;
        }
        // a mask row over half the fixed table: the whole multiply runs the binned path
        fused_overflow = true;
        CU(cudaMemsetAsync(h->d_summary, 0, zero_bytes, st));
    }
    if ((rc = run_analysis())) return rc;
    // ---- small plain one-phase problems: one pass over every row with a
    // fixed single-warp table, one host sync (no binning round trip).  A row
    // whose mask does not fit sets the overflow flag and the multiply falls
    // back to the binned path below (the analysis summary is already there).
    // (a hash accumulator: only the plans that name one, or leave the choice)
    const bool tiny = tiny_ok && !fused_overflow;
    if (tiny) {
        h->bound_off = mask->ptr;   // bounds = mask row lengths (multiply.py:233)
        Out o{};
        o.off = h->bound_off;
        o.idx = h->tmp_idx;
        o.val = h->tmp_val;
        o.row_nnz = h->row_nnz;
        o.evaluated = &h->d_summary->evaluated;
        o.out_f64 = h->out_f64;
        o.overflow = &h->d_summary->pad;
        int gw = 1;
        HashKernel kern = pick_hash(h->kind, MODE_PLAIN, 0, true, &gw);
        const int cap_lg = h->kind == 0 ? 10 : 9;
        const size_t ebytes = h->kind == 0 ? 8 : 16;
        const size_t queue = h->kind == 2 ? 0 : (size_t)64 * (h->kind == 1 ? 24 : 8);
        const size_t smem = 8 * (((size_t)1 << cap_lg) * ebytes + batch_bytes_rt(1, h->kind)) + 8 * queue;
        int occ = 0;
        if ((rc = kernel_occupancy((const void*)kern, 256, smem, &occ))) return rc;
        const int grid = std::max(1, std::min((int)((m + 7) / 8), std::max(occ, 1) * h->num_sms));
        Work wk{nullptr, (int32_t)m, h->cursors + 2 * NBINS};
        ++g_launches;
        kern<<<grid, 256, smem, st>>>(h->prob, o, wk, nullptr, cap_lg, nullptr);
        CU(cudaGetLastError());
        if ((rc = exclusive_scan(h->row_nnz, m, h->c_row_ptr, st, h->scan_scratch, h->bound_off,
                                 &h->d_summary->flag, &h->d_summary->total_nnz)))
            return rc;
        trace("tiny");
        if ((rc = early_compact(h, st))) return rc;
        if ((rc = sync_read(h, h->h_summary, h->d_summary, sizeof(Summary)))) return rc;
        have_summary = true;
        if (!h->h_summary->pad) {
            h->sum = *h->h_summary;
            mark(h, 1);
            mark(h, 2);
            mark(h, 3);
            h->stats = mm_stats_t{};
            h->stats.generated_flops = (int64_t)h->sum.gen_flops;
            h->stats.rows_empty = h->sum.bin_count[BIN_EMPTY];
            h->stats.rows_push = m - h->stats.rows_empty;
            h->total_nnz = h->sum.total_nnz;
            h->stats.evaluated_multiplies = (int64_t)h->sum.evaluated;
            h->bound_flag = h->sum.flag;
            // profile: every non-empty row ran the 1-warp plain hash kernel
            for (int b = 1; b < NBINS; b++) {
                h->sum.bin_flops[hash_bin(MODE_PLAIN, 0, 0)] += b == hash_bin(MODE_PLAIN, 0, 0) ? 0 : h->sum.bin_flops[b];
                h->sum.bin_count[hash_bin(MODE_PLAIN, 0, 0)] += b == hash_bin(MODE_PLAIN, 0, 0) ? 0 : h->sum.bin_count[b];
                if (b != hash_bin(MODE_PLAIN, 0, 0)) h->sum.bin_count[b] = 0, h->sum.bin_flops[b] = 0;
            }
            trace("sync2");
            mark(h, 4);
            *out_nnz = h->total_nnz;
            h->active = true;
            return MM_OK;
        }
        h->compacted = false;
        // fallback: forget what the single pass accumulated
        CU(cudaMemsetAsync(&h->d_summary->evaluated, 0, sizeof(h->d_summary->evaluated), st));
        CU(cudaMemsetAsync(h->cursors + 2 * NBINS, 0, NBINS * sizeof(int32_t), st));
        h->h_summary->evaluated = 0;
    }
    if (m > 0) {
        // the scatter reads the bin counts from the device summary, so it is
        // queued before the host waits for that summary (one launch gap fewer)
        int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)h->num_sms * 8);
        ++g_launches;
        k_bin_scatter<<<grid, 256, 0, st>>>(m, h->row_bin, h->d_summary, h->cursors, h->rows_list);
        CU(cudaGetLastError());
    }
    trace("launched");
    if (!have_summary && (rc = sync_read(h, h->h_summary, h->d_summary, sizeof(Summary)))) return rc;
    trace("sync1");
    h->sum = *h->h_summary;
    mark(h, 1);
    h->bin_off[0] = 0;
    for (int b = 0; b < NBINS; b++) h->bin_off[b + 1] = h->bin_off[b] + (b == 0 ? 0 : h->sum.bin_count[b]);
    h->stats = mm_stats_t{};
    h->stats.generated_flops = (int64_t)h->sum.gen_flops;
    h->stats.rows_empty = h->sum.bin_count[BIN_EMPTY];
    h->stats.rows_pull = h->sum.bin_count[BIN_PULL] + h->sum.bin_count[BIN_PULL_LANE];
    h->stats.rows_push = m - h->stats.rows_empty - h->stats.rows_pull;
    mark(h, 2);

    if (symbolic_only || plan->phases == 2) {
        Out o{};
        o.row_nnz = symbolic_only ? counts_out : h->row_nnz;
        if ((rc = launch_bins(h, false, o))) return rc;
        mark(h, 3);
        if (symbolic_only) {
            CU(cudaStreamSynchronize(st));
            return MM_OK;
        }
        if ((rc = exclusive_scan(h->row_nnz, m, h->c_row_ptr, st, h->scan_scratch, nullptr, nullptr,
                                 &h->d_summary->total_nnz)))
            return rc;
        if ((rc = sync_read(h, h->h_scalar, &h->d_summary->total_nnz, sizeof(long long)))) return rc;
        h->total_nnz = *h->h_scalar;
        mark(h, 4);
        *out_nnz = h->total_nnz;
        h->active = true;
        return MM_OK;
    }

    // ---- one-phase: bounded numeric into slots, then exact row pointer ----
    if (comp) {
        if ((rc = exclusive_scan(h->bound, m, h->bound_ptr, st, h->scan_scratch))) return rc;
        h->bound_off = h->bound_ptr;
        const int64_t tmp_total = (int64_t)h->sum.bound_total;
        if ((rc = dalloc(h, &h->tmp_idx, tmp_total))) return rc;
        unsigned char* tv = nullptr;
        if ((rc = dalloc(h, &tv, (size_t)tmp_total * 8))) return rc;
        h->tmp_val = tv;
    } else {
        h->bound_off = mask->ptr;   // bounds = mask row lengths (multiply.py:233)
    }
    Out o{};
    o.off = h->bound_off;
    o.idx = h->tmp_idx;
    o.val = h->tmp_val;
    o.row_nnz = h->row_nnz;
    o.evaluated = &h->d_summary->evaluated;
    o.out_f64 = h->out_f64;
    if ((rc = launch_bins(h, true, o))) return rc;
    trace("bins");
    mark(h, 3);
    // the bound assertion (multiply.py:390) is folded into the scan and rides
    // on the nnz readback below
    if ((rc = exclusive_scan(h->row_nnz, m, h->c_row_ptr, st, h->scan_scratch, h->bound_off,
                             &h->d_summary->flag, &h->d_summary->total_nnz)))
        return rc;
    if ((rc = sync_read(h, h->h_summary, h->d_summary, sizeof(Summary)))) return rc;
    h->total_nnz = h->h_summary->total_nnz;
    h->stats.evaluated_multiplies = (int64_t)h->h_summary->evaluated;
    h->bound_flag = h->h_summary->flag;
    trace("sync2");
    mark(h, 4);
    *out_nnz = h->total_nnz;
    h->active = true;
    return MM_OK;
}

int end_impl(mm_handle* h, int64_t* c_row_ptr, int32_t* c_col_idx, void* c_values, mm_stats_t* stats) {
    if (!h->active) return fail(MM_ERR_INPUT, "mm_multiply_end without a successful mm_multiply_begin");
    trace("end");
    cudaStream_t st = h->stream;
    const int64_t m = h->nrows;
    int rc;
    if (h->total_nnz > 0 && (!c_col_idx || !c_values))
        return fail(MM_ERR_INPUT, "output arrays required for a non-empty result");
    if (c_row_ptr && c_row_ptr != h->c_row_ptr)
        CU(cudaMemcpyAsync(c_row_ptr, h->c_row_ptr, (m + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    int* flag = &h->d_summary->flag;
    if (h->plan.phases == 1 && h->compacted) {
        mark(h, 5);   // compacted before the summary readback (early_compact)
    } else if (h->plan.phases == 1) {
        if (m > 0 && h->total_nnz <= 2 * m) {
            // sparse outputs: a thread per row
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)h->num_sms * 8));
            ++g_launches;
            if (h->out_f64)
                k_compact_rowwise<double><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                                (const double*)h->tmp_val, h->c_row_ptr,
                                                                c_col_idx, (double*)c_values, nullptr);
            else
                k_compact_rowwise<long long><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                                   (const long long*)h->tmp_val, h->c_row_ptr,
                                                                   c_col_idx, (long long*)c_values, nullptr);
            CU(cudaGetLastError());
        } else if (m > 0) {
            int64_t want = std::max<int64_t>((h->total_nnz + 2047) / 2048, (m + 255) / 256);
            int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)h->num_sms * 16));
            ++g_launches;
            if (h->out_f64)
                k_compact<double><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                        (const double*)h->tmp_val, h->c_row_ptr,
                                                        c_col_idx, (double*)c_values, nullptr);
            else
                k_compact<long long><<<grid, 256, 0, st>>>(m, h->bound_off, h->row_nnz, h->tmp_idx,
                                                           (const long long*)h->tmp_val, h->c_row_ptr,
                                                           c_col_idx, (long long*)c_values, nullptr);
            CU(cudaGetLastError());
        }
        mark(h, 5);
        // no sync: counters and the bound flag came back with the nnz readback
    } else {
        if ((rc = dalloc(h, &h->row_nnz2, m))) { release(h); return rc; }
        if (m > 0) CU(cudaMemsetAsync(h->row_nnz2, 0, m * sizeof(int64_t), st));
        Out o{};
        o.off = h->c_row_ptr;
        o.idx = c_col_idx;
        o.val = c_values;
        o.row_nnz = h->row_nnz2;
        o.evaluated = &h->d_summary->evaluated;
        o.out_f64 = h->out_f64;
        if ((rc = launch_bins(h, true, o))) { release(h); return rc; }
        if (m > 0) {
            int grid = (int)std::min<int64_t>((m + 255) / 256, (int64_t)h->num_sms * 8);
            ++g_launches;
            k_check_equal<<<grid, 256, 0, st>>>(m, h->row_nnz, h->row_nnz2, flag);
        }
        mark(h, 5);
        if ((rc = sync_read(h, h->h_summary, h->d_summary, sizeof(Summary)))) { release(h); return rc; }
        h->stats.evaluated_multiplies = (int64_t)h->h_summary->evaluated;
    }
    trace("$done");
    int bad = h->plan.phases == 1 ? h->bound_flag : h->h_summary->flag;
    h->launches = g_launches - h->launch_base;
    h->stats.output_nnz = h->total_nnz;
    if (stats) *stats = h->stats;
    release(h);
    if (bad)
        return fail(MM_ERR_INTERNAL, h->plan.phases == 1 ? "one-phase row bound violated"
                                                         : "symbolic phase disagreed with numeric row sizes");
    return MM_OK;
}

}  // namespace

extern "C" {

int mm_abi_version(void) { return MM_ABI_VERSION; }

const char* mm_last_error(void) { return g_last_error.c_str(); }

int mm_create(int device, mm_handle_t** out) {
    if (!out) return fail(MM_ERR_INPUT, "null handle pointer");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return fail(MM_ERR_CUDA, cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(MM_ERR_INPUT, "no CUDA device " + std::to_string(device));
    DeviceGuard dg(device);
    mm_handle* h = new mm_handle();
    h->device = device;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (cudaMallocHost((void**)&h->h_summary, sizeof(Summary)) != cudaSuccess ||
        cudaMallocHost((void**)&h->h_scalar, sizeof(long long)) != cudaSuccess) {
        delete h;
        return fail(MM_ERR_CUDA, "cudaMallocHost failed");
    }
    // fused tail: a device ticket counter and the mapped host words its last
    // block writes; without them (no mapped memory) the separate kernels run
    if (cudaHostAlloc((void**)&h->h_tail, sizeof(TailResult), cudaHostAllocMapped) == cudaSuccess) {
        std::memset(h->h_tail, 0, sizeof(TailResult));
        if (cudaMalloc((void**)&h->d_done, sizeof(unsigned)) != cudaSuccess ||
            cudaMemset(h->d_done, 0, sizeof(unsigned)) != cudaSuccess) {
            cudaGetLastError();
            if (h->d_done) cudaFree(h->d_done);
            h->d_done = nullptr;
        }
    } else {
        cudaGetLastError();
        h->h_tail = nullptr;
    }
    *out = h;
    return MM_OK;
}

int mm_destroy(mm_handle_t* h) {
    if (!h) return MM_OK;
    DeviceGuard dg(h->device);
    if (h->active) release(h);
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->tail_stream) cudaStreamSynchronize(h->tail_stream);
    cudaFreeHost(h->h_summary);
    cudaFreeHost(h->h_scalar);
    if (h->h_tail) cudaFreeHost(h->h_tail);
    if (h->d_done) cudaFree(h->d_done);
    for (auto& e : h->ev) if (e) cudaEventDestroy(e);
    if (h->fork_ev) {
        cudaEventDestroy(h->fork_ev);
        for (int q = 0; q < mm_handle::NAUX; q++) {
            cudaEventDestroy(h->join_ev[q]);
            cudaStreamDestroy(h->aux[q]);
        }
    }
    delete h;
    return MM_OK;
}

int mm_multiply_begin(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                      const mm_matrix_t* b, const mm_matrix_t* b_csc, void* stream, int64_t* out_nnz) {
    if (!h || !out_nnz) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(h->device);
    int rc = begin_impl(h, plan, mask, a, b, b_csc, (cudaStream_t)stream, false, nullptr, out_nnz);
    if (rc) release(h);
    return rc;
}

int mm_multiply(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                const mm_matrix_t* b, const mm_matrix_t* b_csc, void* stream, int64_t* c_row_ptr, int32_t* c_col_idx,
                void* c_values, int64_t capacity, int64_t* out_nnz, mm_stats_t* stats) {
    if (!h || !out_nnz || !c_row_ptr) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(h->device);
    h->user_row_ptr = c_row_ptr;
    const bool early = plan && mask && !plan->complemented && plan->phases == 1 && capacity >= mask->nnz &&
                       c_col_idx && c_values;
    h->early_idx = early ? c_col_idx : nullptr;
    h->early_val = early ? c_values : nullptr;
    int rc = begin_impl(h, plan, mask, a, b, b_csc, (cudaStream_t)stream, false, nullptr, out_nnz);
    h->user_row_ptr = nullptr;
    h->early_idx = nullptr;
    h->early_val = nullptr;
    if (rc) {
        release(h);
        return rc;
    }
    if (*out_nnz > capacity) return fail(MM_ERR_CAPACITY, "output capacity " + std::to_string(capacity) +
                                                              " below nnz(C) = " + std::to_string(*out_nnz));
    return end_impl(h, c_row_ptr, c_col_idx, c_values, stats);
}

int mm_multiply_end(mm_handle_t* h, int64_t* c_row_ptr, int32_t* c_col_idx, void* c_values, mm_stats_t* stats) {
    if (!h) return fail(MM_ERR_INPUT, "null handle");
    DeviceGuard dg(h->device);
    return end_impl(h, c_row_ptr, c_col_idx, c_values, stats);
}

int mm_profile_enable(mm_handle_t* h, int on) {
    if (!h) return fail(MM_ERR_INPUT, "null handle");
    DeviceGuard dg(h->device);
    if (on && !h->ev[0]) {
        for (auto& e : h->ev) CU(cudaEventCreate(&e));
    }
    h->prof = on != 0;
    return MM_OK;
}

int mm_profile_read(mm_handle_t* h, float* ms, int n, int64_t* launches) {
    if (!h) return fail(MM_ERR_INPUT, "null handle");
    if (launches) *launches = h->launches;
    if (!h->prof || !ms) return MM_OK;
    DeviceGuard dg(h->device);
    CU(cudaEventSynchronize(h->ev[5]));
    static const int from[6] = {0, 1, 2, 3, 4, 0};
    static const int to[6] = {1, 2, 3, 4, 5, 5};
    for (int q = 0; q < n && q < 6; q++) {
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, h->ev[from[q]], h->ev[to[q]]));
        ms[q] = t;
    }
    return MM_OK;
}

int mm_set_tuning(mm_handle_t* h, const int64_t* params, int n) {
    if (!h) return fail(MM_ERR_INPUT, "null handle");
    if (n > 0 && params[0] > 0) h->tier_flops0 = params[0];
    if (n > 1 && params[1] > 0) h->tier_flops1 = h->tier_flops1_hash = params[1];   // params[22] sets the hash one apart
    if (n > 2 && params[2] > 0) h->capc_lg = (int)params[2];
    if (n > 3 && params[3] > 0 && params[3] <= 4) h->load_shift = (int)params[3];
    for (int t = 0; t < 3; t++)
        if (n > 4 + t && params[4 + t] > 0) h->rank_budget[t] = (int)params[4 + t];
    if (n > 7 && params[7] >= 0) h->auto_mca_nm = (int)params[7];
    for (int t = 0; t < 3; t++)
        if (n > 8 + t && params[8 + t] >= 0 && params[8 + t] <= 14) h->direct_lg[t] = (int)params[8 + t];
    if (n > 11 && params[11] > 0 && params[11] <= 4) h->load_shift_wide = (int)params[11];
    if (n > 12 && params[12] >= 0) h->tiny_rows = params[12];   // 0 disables the single-pass path
    if (n > 13 && params[13] >= 0) h->tiny_nnz = params[13];
    if (n > 14 && params[14] >= 0) h->direct_on = params[14] != 0;
    if (n > 15 && params[15] >= 0) h->slice_cursors = params[15] != 0;
    if (n > 16 && params[16] >= 0) h->split_slices = params[16] != 0;
    if (n > 17 && params[17] >= 0) h->fused_rows = params[17];  // 0 disables the one-launch path (fused_tail.cuh)
    if (n > 18 && params[18] >= 0) h->fused_nnz = params[18];
    if (n > 19 && params[19] >= 0) h->blen_on = params[19] != 0;
    if (n > 20 && params[20] >= 0) h->kblock_bytes = params[20];
    if (n > 21 && params[21] >= 0) h->kblock_min_flops = params[21];
    if (n > 22 && params[22] > 0) h->tier_flops1_hash = params[22];
    return MM_OK;
}

int mm_profile_bins(mm_handle_t* h, int64_t* rows, int64_t* flops, int n) {
    if (!h) return fail(MM_ERR_INPUT, "null handle");
    for (int b = 0; b < n && b < NBINS; b++) {
        if (rows) rows[b] = h->sum.bin_count[b];
        if (flops) flops[b] = (int64_t)h->sum.bin_flops[b];
    }
    return NBINS;
}

int mm_symbolic(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                const mm_matrix_t* b, const mm_matrix_t* b_csc, void* stream, int64_t* counts) {
    if (!h || !counts) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(h->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (mask && mask->nrows > 0) {
        cudaError_t e = cudaMemsetAsync(counts, 0, mask->nrows * sizeof(int64_t), st);
        if (e != cudaSuccess) return fail(MM_ERR_CUDA, cudaGetErrorString(e));
    }
    int64_t dummy = 0;
    int rc = begin_impl(h, plan, mask, a, b, b_csc, st, true, counts, &dummy);
    release(h);
    if (!rc) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(MM_ERR_CUDA, cudaGetErrorString(e));
    }
    return rc;
}

int mm_row_flops(const mm_matrix_t* a, const mm_matrix_t* b, int64_t* row_flops, int64_t* total, void* stream) {
    if (!a || !b || !row_flops) return fail(MM_ERR_INPUT, "null argument");
    if (a->ncols != b->nrows) return fail(MM_ERR_INPUT, "dimension mismatch");
    DeviceGuard dg(call_device(stream, a->ptr));
    cudaStream_t st = (cudaStream_t)stream;
    Prob p{};
    p.a_ptr = a->ptr; p.a_idx = a->idx; p.b_ptr = b->ptr; p.b_idx = b->idx;
    // reuse the analysis kernel with a dummy all-rows mask view: only flops matter
    p.m_ptr = a->ptr; p.m_idx = a->idx;
    p.nrows = a->nrows; p.ncols = b->ncols;
    AnalyzeParams ap{};
    ap.family = FAM_HASH;
    Summary* s = nullptr;
    uint8_t* rb = nullptr;
    int8_t* rc_lg = nullptr;
    int32_t* long_rows = nullptr;
    CU(cudaMallocAsync((void**)&s, sizeof(Summary) + 16, st));
    CU(cudaMallocAsync((void**)&long_rows, std::max<int64_t>(a->nrows, 1) * sizeof(int32_t), st));
    int* long_n = (int*)(s + 1);
    CU(cudaMallocAsync((void**)&rb, std::max<int64_t>(a->nrows, 1), st));
    CU(cudaMallocAsync((void**)&rc_lg, std::max<int64_t>(a->nrows, 1), st));
    CU(cudaMemsetAsync(s, 0, sizeof(Summary) + 16, st));
    if (a->nrows > 0) {
        int grid = (int)std::min<int64_t>((a->nrows + 255) / 256, 148 * 8);
        ++g_launches;
        k_analyze<false><<<grid, 256, 0, st>>>(p, ap, row_flops, nullptr, rb, rc_lg, s, nullptr, long_rows, long_n);
        ++g_launches;
        k_analyze_long<false><<<296, 256, 0, st>>>(p, ap, row_flops, nullptr, rb, rc_lg, s, nullptr, long_rows, long_n);
    }
    if (total) CU(cudaMemcpyAsync(total, &s->gen_flops, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    cudaFreeAsync(s, st);
    cudaFreeAsync(rb, st);
    cudaFreeAsync(rc_lg, st);
    cudaFreeAsync(long_rows, st);
    CU(cudaGetLastError());
    return MM_OK;
}

// w_i = flops_i + nnz(M_i): the work estimate behind the multi-GPU cuts and
// the per-row cost model (SURVEY §8(b) mm_row_work, §8(e)).
__global__ void k_add_row_lengths(int64_t n, const int64_t* ptr, int64_t* w) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        w[i] += ptr[i + 1] - ptr[i];
}

int mm_row_work(const mm_matrix_t* a, const mm_matrix_t* b, const mm_matrix_t* mask, int64_t* row_flops,
                int64_t* row_work, void* stream) {
    if (!a || !b || !mask || !row_work) return fail(MM_ERR_INPUT, "null argument");
    if (mask->nrows != a->nrows) return fail(MM_ERR_INPUT, "mask and A row counts differ");
    DeviceGuard dg(call_device(stream, a->ptr));
    cudaStream_t st = (cudaStream_t)stream;
    int rc = mm_row_flops(a, b, row_work, nullptr, stream);
    if (rc) return rc;
    if (row_flops && a->nrows > 0)
        CU(cudaMemcpyAsync(row_flops, row_work, a->nrows * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    if (a->nrows > 0) {
        ++g_launches;
        k_add_row_lengths<<<(int)std::min<int64_t>((a->nrows + 255) / 256, 148 * 8), 256, 0, st>>>(
            a->nrows, mask->ptr, row_work);
        CU(cudaGetLastError());
    }
    return MM_OK;
}

int mm_workspace_bytes(const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                       const mm_matrix_t* b, size_t* bytes) {
    if (!plan || !mask || !a || !b || !bytes) return fail(MM_ERR_INPUT, "null argument");
    const int64_t m = mask->nrows;
    const bool comp = plan->complemented != 0;
    auto r = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t t = r(sizeof(Summary) + (3 * NBINS + 4) * sizeof(int32_t)) + r(m * 4) /* long rows */ +
               3 * r(m * 8) + r((m + 1) * 8) + r(scan_scratch_elems(m) * 8) + r(m * 4) + 2 * r(m);
    if (comp && plan->phases == 1) t += r(m * 8) + r((m + 1) * 8);
    if (!comp && plan->phases == 1) t += r(mask->nnz * 4) + r(mask->nnz * 8);
    if (plan->phases == 2) t += r(m * 8);
    *bytes = t;
    return MM_OK;
}

int mm_exclusive_scan(const int64_t* counts, int64_t n, int64_t* out, void* stream) {
    if (!out || (n > 0 && !counts)) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(call_device(stream, out));
    return exclusive_scan(counts, n, out, (cudaStream_t)stream);
}

int mm_compact_rows(int64_t nrows, const int64_t* bounds_off, const int64_t* row_nnz, const int32_t* tmp_idx,
                    const void* tmp_val, const int64_t* out_ptr, int32_t* out_idx, void* out_val, int dtype,
                    void* stream) {
    if (nrows <= 0) return MM_OK;
    DeviceGuard dg(call_device(stream, out_ptr));
    cudaStream_t st = (cudaStream_t)stream;
    int* flag = nullptr;
    CU(cudaMallocAsync((void**)&flag, sizeof(int), st));
    CU(cudaMemsetAsync(flag, 0, sizeof(int), st));
    int grid = (int)std::min<int64_t>((nrows + 255) / 256, 148 * 16);
    ++g_launches;
    if (dtype == MM_DTYPE_FLOAT64)
        k_compact<double><<<grid, 256, 0, st>>>(nrows, bounds_off, row_nnz, tmp_idx, (const double*)tmp_val,
                                                out_ptr, out_idx, (double*)out_val, flag);
    else
        k_compact<long long><<<grid, 256, 0, st>>>(nrows, bounds_off, row_nnz, tmp_idx,
                                                   (const long long*)tmp_val, out_ptr, out_idx,
                                                   (long long*)out_val, flag);
    int hflag = 0;
    CU(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    cudaFreeAsync(flag, st);
    if (hflag) return fail(MM_ERR_INTERNAL, "one-phase row bound violated");
    return MM_OK;
}

int mm_filter_min(const mm_matrix_t* c, int64_t thr, int64_t* out_row_ptr, int32_t* out_idx,
                  int64_t* out_nnz, void* stream) {
    if (!c || !out_row_ptr || !out_nnz) return fail(MM_ERR_INPUT, "null argument");
    if (c->nnz > 0 && (!c->values || !c->idx || !out_idx)) return fail(MM_ERR_INPUT, "values and output indices required");
    DeviceGuard dg(call_device(stream, out_row_ptr));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t m = c->nrows;
    int64_t* counts = nullptr;
    long long* hnz = pinned_scratch();
    if (!hnz) return fail(MM_ERR_CUDA, "cudaMallocHost failed");
    CU(cudaMallocAsync((void**)&counts, std::max<int64_t>(m, 1) * sizeof(int64_t), st));
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 7) / 8, 148 * 16));
    if (m > 0) {
        ++g_launches;
        k_filter_min<false><<<grid, 256, 0, st>>>(m, c->ptr, c->idx, (const long long*)c->values, thr, counts,
                                                  nullptr, nullptr);
    }
    int rc = exclusive_scan(counts, m, out_row_ptr, st);
    if (rc) { cudaFreeAsync(counts, st); return rc; }
    if (m > 0) {
        ++g_launches;
        k_filter_min<true><<<grid, 256, 0, st>>>(m, c->ptr, c->idx, (const long long*)c->values, thr, nullptr,
                                                 out_row_ptr, out_idx);
    }
    CU(cudaMemcpyAsync(hnz, out_row_ptr + m, sizeof(long long), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    *out_nnz = *hnz;
    cudaFreeAsync(counts, st);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_reduce_sum(const void* values, int64_t n, int dtype, void* out, void* stream) {
    if (!out) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(call_device(stream, out));
    cudaStream_t st = (cudaStream_t)stream;
    const int nparts = 592;
    void* partials = nullptr;
    CU(cudaMallocAsync(&partials, nparts * 8, st));
    if (dtype == MM_DTYPE_FLOAT64) {
        ++g_launches;
        k_reduce_partial<double><<<nparts, 256, 0, st>>>((const double*)values, n, (double*)partials);
        ++g_launches;
        k_reduce_final<double><<<1, 256, 0, st>>>((const double*)partials, nparts, (double*)out);
    } else {
        ++g_launches;
        k_reduce_partial<long long><<<nparts, 256, 0, st>>>((const long long*)values, n, (long long*)partials);
        ++g_launches;
        k_reduce_final<long long><<<1, 256, 0, st>>>((const long long*)partials, nparts, (long long*)out);
    }
    cudaFreeAsync(partials, st);
    CU(cudaGetLastError());
    return MM_OK;
}

// ---- element-wise graph building blocks (graph_ops.cuh) ----

static int warp_grid(int64_t rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, (int64_t)148 * 16));
}

int mm_lookup_rows(const mm_matrix_t* x, const mm_matrix_t* y, int dtype, void* out, uint8_t* found,
                   void* stream) {
    if (!x || !y || (x->nnz > 0 && !out)) return fail(MM_ERR_INPUT, "null argument");
    if (x->nrows != y->nrows || x->ncols != y->ncols) return fail(MM_ERR_INPUT, "lookup_rows: shape mismatch");
    if (x->nnz == 0 || x->nrows == 0) return MM_OK;
    if (y->nnz > 0 && !y->values) return fail(MM_ERR_INPUT, "lookup_rows: Y needs values");
    DeviceGuard dg(call_device(stream, x->ptr));
    cudaStream_t st = (cudaStream_t)stream;
    ++g_launches;
    if (dtype == MM_DTYPE_FLOAT64)
        k_lookup<LK_VALUE, double><<<warp_grid(x->nrows), 256, 0, st>>>(
            x->nrows, x->ptr, x->idx, nullptr, y->ptr, y->idx, (const double*)y->values, nullptr, nullptr, nullptr,
            (double*)out, found);
    else
        k_lookup<LK_VALUE, long long><<<warp_grid(x->nrows), 256, 0, st>>>(
            x->nrows, x->ptr, x->idx, nullptr, y->ptr, y->idx, (const long long*)y->values, nullptr, nullptr,
            nullptr, (long long*)out, found);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_bc_dependency_weights(const mm_matrix_t* sigma, const mm_matrix_t* delta, const mm_matrix_t* paths,
                             double* w, void* stream) {
    if (!sigma || !delta || !paths || (sigma->nnz > 0 && !w)) return fail(MM_ERR_INPUT, "null argument");
    if (sigma->nrows != delta->nrows || sigma->nrows != paths->nrows)
        return fail(MM_ERR_INPUT, "bc weights: row count mismatch");
    if (sigma->nnz == 0) return MM_OK;
    DeviceGuard dg(call_device(stream, sigma->ptr));
    ++g_launches;
    k_lookup<LK_BC_WEIGHT, double><<<warp_grid(sigma->nrows), 256, 0, (cudaStream_t)stream>>>(
        sigma->nrows, sigma->ptr, sigma->idx, nullptr, delta->ptr, delta->idx, (const double*)delta->values,
        paths->ptr, paths->idx, (const double*)paths->values, w, nullptr);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_bc_scale_by(const mm_matrix_t* x, const mm_matrix_t* paths, double* out, void* stream) {
    if (!x || !paths || (x->nnz > 0 && (!out || !x->values))) return fail(MM_ERR_INPUT, "null argument");
    if (x->nrows != paths->nrows) return fail(MM_ERR_INPUT, "bc scale: row count mismatch");
    if (x->nnz == 0) return MM_OK;
    DeviceGuard dg(call_device(stream, x->ptr));
    ++g_launches;
    k_lookup<LK_SCALE, double><<<warp_grid(x->nrows), 256, 0, (cudaStream_t)stream>>>(
        x->nrows, x->ptr, x->idx, (const double*)x->values, paths->ptr, paths->idx, (const double*)paths->values,
        nullptr, nullptr, nullptr, out, nullptr);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_ewise_add_begin(const mm_matrix_t* a, const mm_matrix_t* b, int64_t* c_row_ptr, int64_t* nnz, void* stream) {
    if (!a || !b || !c_row_ptr || !nnz) return fail(MM_ERR_INPUT, "null argument");
    if (a->nrows != b->nrows || a->ncols != b->ncols)
        return fail(MM_ERR_INPUT, "shape mismatch (" + std::to_string(a->nrows) + ", " + std::to_string(a->ncols) +
                                      ") vs (" + std::to_string(b->nrows) + ", " + std::to_string(b->ncols) + ")");
    DeviceGuard dg(call_device(stream, c_row_ptr));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t m = a->nrows;
    int64_t* counts = nullptr;
    long long* total = nullptr;
    CU(cudaMallocAsync((void**)&counts, (std::max<int64_t>(m, 1) + 2) * sizeof(int64_t), st));
    total = (long long*)(counts + std::max<int64_t>(m, 1));
    if (m > 0) {
        ++g_launches;
        k_ewise_count<<<warp_grid(m), 256, 0, st>>>(m, a->ptr, a->idx, b->ptr, b->idx, counts);
    }
    int rc = exclusive_scan(counts, m, c_row_ptr, st, nullptr, nullptr, nullptr, total);
    if (!rc) rc = read_i64(total, nnz, st);
    cudaFreeAsync(counts, st);
    return rc;
}

int mm_ewise_add_end(const mm_matrix_t* a, const mm_matrix_t* b, int dtype, const int64_t* c_row_ptr,
                     int32_t* c_idx, void* c_val, void* stream) {
    if (!a || !b || !c_row_ptr) return fail(MM_ERR_INPUT, "null argument");
    if (a->nrows != b->nrows || a->ncols != b->ncols) return fail(MM_ERR_INPUT, "shape mismatch");
    if ((a->nnz && !a->values) || (b->nnz && !b->values)) return fail(MM_ERR_INPUT, "ewise_add needs values");
    if ((a->nnz || b->nnz) && (!c_idx || !c_val)) return fail(MM_ERR_INPUT, "output arrays required");
    const int64_t m = a->nrows;
    if (m == 0 || (a->nnz == 0 && b->nnz == 0)) return MM_OK;
    DeviceGuard dg(call_device(stream, c_row_ptr));
    cudaStream_t st = (cudaStream_t)stream;
    ++g_launches;
    if (dtype == MM_DTYPE_FLOAT64)
        k_ewise_fill<double><<<warp_grid(m), 256, 0, st>>>(m, a->ptr, a->idx, (const double*)a->values, b->ptr,
                                                           b->idx, (const double*)b->values, c_row_ptr, c_idx,
                                                           (double*)c_val);
    else
        k_ewise_fill<long long><<<warp_grid(m), 256, 0, st>>>(m, a->ptr, a->idx, (const long long*)a->values,
                                                              b->ptr, b->idx, (const long long*)b->values,
                                                              c_row_ptr, c_idx, (long long*)c_val);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_bc_accumulate(const mm_matrix_t* delta, const int32_t* src_col, double* scores, void* stream) {
    if (!delta || !scores || (delta->nnz > 0 && !delta->values)) return fail(MM_ERR_INPUT, "null argument");
    const int64_t m = delta->nrows;
    if (m == 0) return MM_OK;
    DeviceGuard dg(call_device(stream, scores));
    ++g_launches;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, (int64_t)148 * 16));
    k_bc_accumulate<<<grid, 256, 0, (cudaStream_t)stream>>>(m, delta->ptr, delta->idx, (const double*)delta->values,
                                                             src_col, scores);
    CU(cudaGetLastError());
    return MM_OK;
}

// ---- device input preparation (graph_prep.cuh) ----

int mm_expand_rows(int64_t nrows, const int64_t* ptr, int32_t* rows, void* stream) {
    if (nrows <= 0) return MM_OK;
    if (!ptr || !rows) return fail(MM_ERR_INPUT, "null argument");
    DeviceGuard dg(call_device(stream, rows));
    ++g_launches;
    k_expand_rows<<<warp_grid(nrows), 256, 0, (cudaStream_t)stream>>>(nrows, ptr, rows);
    CU(cudaGetLastError());
    return MM_OK;
}


// Sort every segment [ptr[s], ptr[s+1]) of keys (and 8-byte vals) ascending.
static int segmented_sort(int64_t nseg, const int64_t* ptr, int32_t* keys, unsigned long long* vals,
                          cudaStream_t st) {
    if (nseg <= 0) return MM_OK;
    int32_t* big = nullptr;
    unsigned long long* mx = nullptr;
    CU(cudaMallocAsync((void**)&big, nseg * sizeof(int32_t) + 16, st));
    CU(cudaMallocAsync((void**)&mx, 2 * sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(mx, 0, 2 * sizeof(unsigned long long), st));
    int* nbig = (int*)(mx + 1);
    ++g_launches;
    if (vals) k_seg_sort_warp<true><<<warp_grid(nseg), 256, 0, st>>>(nseg, ptr, keys, vals, big, nbig);
    else k_seg_sort_warp<false><<<warp_grid(nseg), 256, 0, st>>>(nseg, ptr, keys, vals, big, nbig);
    ++g_launches;
    k_max_degree<<<(int)std::min<int64_t>((nseg + 255) / 256, 148 * 8), 256, 0, st>>>(nseg, ptr, mx);
    int64_t hv[2] = {0, 0};
    if (int rc = read_i64s(mx, hv, 2, st)) {
        cudaFreeAsync(big, st);
        cudaFreeAsync(mx, st);
        return rc;
    }
    const int64_t maxlen = hv[0];
    const int nb = (int)(hv[1] & 0xffffffff);
    if (nb > 0) {
        int64_t P = 1;
        while (P < maxlen) P <<= 1;
        const int64_t cap = P > PREP_TILE ? P : 0;
        const int grid = (int)std::min<int64_t>(nb, 148 * 2);
        int32_t* sk = nullptr;
        unsigned long long* sv = nullptr;
        if (cap) {
            CU(cudaMallocAsync((void**)&sk, (size_t)grid * cap * sizeof(int32_t), st));
            if (vals) CU(cudaMallocAsync((void**)&sv, (size_t)grid * cap * sizeof(unsigned long long), st));
        }
        ++g_launches;
        if (vals) k_seg_sort_block<true><<<grid, PREP_THREADS, 0, st>>>(ptr, keys, vals, big, nbig, sk, sv, cap);
        else k_seg_sort_block<false><<<grid, PREP_THREADS, 0, st>>>(ptr, keys, vals, big, nbig, sk, sv, cap);
        if (sk) cudaFreeAsync(sk, st);
        if (sv) cudaFreeAsync(sv, st);
    }
    cudaFreeAsync(big, st);
    cudaFreeAsync(mx, st);
    CU(cudaGetLastError());
    return MM_OK;
}

int mm_csr_from_coo(int64_t nrows, int64_t ncols, const void* rows, const void* cols, int idx64, int64_t nnz,
                    const int32_t* map, int flags, const void* vals, int64_t* out_ptr, int32_t* out_idx,
                    void* out_vals, int64_t* out_nnz, void* stream) {
    if (!out_ptr || !out_nnz || (nnz > 0 && (!rows || !cols || !out_idx))) return fail(MM_ERR_INPUT, "null argument");
    if (nrows < 0 || ncols < 0 || nrows >= (1ll << 31) || ncols >= (1ll << 31))
        return fail(MM_ERR_INPUT, "dimensions must be in [0, 2^31)");
    const bool dedup = flags & MM_COO_DEDUP;
    if ((flags & MM_COO_SYMMETRIC) && nrows != ncols) return fail(MM_ERR_INPUT, "symmetrising needs a square matrix");
    if (dedup && vals) return fail(MM_ERR_INPUT, "duplicate merging is pattern-only");
    DeviceGuard dg(call_device(stream, out_ptr));
    cudaStream_t st = (cudaStream_t)stream;
    CooView v{rows, cols, idx64, map, (flags & MM_COO_SYMMETRIC) ? 1 : 0, (flags & MM_COO_NO_DIAG) ? 1 : 0,
              (flags & MM_COO_LOWER) ? 1 : 0, nnz};
    const int64_t cap = nnz * (v.sym ? 2 : 1);
    int64_t* counts = nullptr;
    int64_t* tptr = nullptr;
    CU(cudaMallocAsync((void**)&counts, (nrows + 2) * sizeof(int64_t), st));
    CU(cudaMallocAsync((void**)&tptr, (nrows + 2) * sizeof(int64_t), st));
    CU(cudaMemsetAsync(counts, 0, (nrows + 1) * sizeof(int64_t), st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nnz + 255) / 256, 148 * 16));
    if (nnz > 0) {
        ++g_launches;
        k_coo_count<<<grid, 256, 0, st>>>(v, counts);
    }
    int64_t* dst_ptr = dedup ? tptr : out_ptr;
    int rc = exclusive_scan(counts, nrows, dst_ptr, st);
    int32_t* kidx = out_idx;
    if (!rc && dedup) {
        if (cudaMallocAsync((void**)&kidx, std::max<int64_t>(cap, 1) * sizeof(int32_t), st) != cudaSuccess)
            rc = fail(MM_ERR_CUDA, "cudaMallocAsync failed");
    }
    if (!rc && nnz > 0) {
        // cursors start at the row offsets (counts is reused as the cursor array)
        cudaMemcpyAsync(counts, dst_ptr, nrows * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
        ++g_launches;
        k_coo_scatter<<<grid, 256, 0, st>>>(v, (const unsigned long long*)vals, (unsigned long long*)counts, kidx,
                                            (unsigned long long*)out_vals);
        rc = segmented_sort(nrows, dst_ptr, kidx, (unsigned long long*)(vals ? out_vals : nullptr), st);
    }
    if (!rc && dedup) {
        if (nrows > 0) {
            ++g_launches;
            k_unique_count<<<warp_grid(nrows), 256, 0, st>>>(nrows, tptr, kidx, counts);
        }
        rc = exclusive_scan(counts, nrows, out_ptr, st);
        if (!rc && nrows > 0) {
            ++g_launches;
            k_unique_compact<<<warp_grid(nrows), 256, 0, st>>>(nrows, tptr, kidx, out_ptr, out_idx);
        }
    }
    if (!rc) rc = read_i64(out_ptr + nrows, out_nnz, st);
    if (dedup && kidx && kidx != out_idx) cudaFreeAsync(kidx, st);
    cudaFreeAsync(counts, st);
    cudaFreeAsync(tptr, st);
    if (!rc) CU(cudaGetLastError());
    return rc;
}

int mm_degree_order(const mm_matrix_t* g, int32_t* perm, int32_t* new_label, void* stream) {
    if (!g || !g->ptr || !perm || !new_label) return fail(MM_ERR_INPUT, "null argument");
    if (g->nrows != g->ncols) return fail(MM_ERR_INPUT, "degree_sort_relabel requires a square matrix");
    const int64_t n = g->nrows;
    if (n == 0) return MM_OK;
    DeviceGuard dg(call_device(stream, perm));
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long* mx = nullptr;
    CU(cudaMallocAsync((void**)&mx, sizeof(unsigned long long), st));
    CU(cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
    ++g_launches;
    k_max_degree<<<grid, 256, 0, st>>>(n, g->ptr, mx);
    int64_t maxdeg = 0;
    int rc = read_i64(mx, &maxdeg, st);
    cudaFreeAsync(mx, st);
    if (rc) return rc;
    int64_t* hist = nullptr;
    int64_t* bptr = nullptr;
    CU(cudaMallocAsync((void**)&hist, (maxdeg + 2) * sizeof(int64_t), st));
    CU(cudaMallocAsync((void**)&bptr, (maxdeg + 3) * sizeof(int64_t), st));
    CU(cudaMemsetAsync(hist, 0, (maxdeg + 1) * sizeof(int64_t), st));
    ++g_launches;
    k_degree_hist<<<grid, 256, 0, st>>>(n, g->ptr, maxdeg, hist);
    rc = exclusive_scan(hist, maxdeg + 1, bptr, st);
    if (!rc) {
        cudaMemcpyAsync(hist, bptr, (maxdeg + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st);
        ++g_launches;
        k_degree_scatter<<<grid, 256, 0, st>>>(n, g->ptr, maxdeg, (unsigned long long*)hist, perm);
        rc = segmented_sort(maxdeg + 1, bptr, perm, nullptr, st);   // ids ascending inside a degree
    }
    if (!rc) {
        ++g_launches;
        k_invert_perm<<<grid, 256, 0, st>>>(n, perm, new_label);
    }
    cudaFreeAsync(hist, st);
    cudaFreeAsync(bptr, st);
    if (!rc) CU(cudaGetLastError());
    return rc;
}

}  // extern "C"


