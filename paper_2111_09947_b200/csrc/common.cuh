// Shared device helpers for the masked-SpGEMM kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mm {

constexpr unsigned FULL = 0xffffffffu;
constexpr int32_t EMPTY_KEY = -1;

// Problem view passed by value to every kernel.  Device pointers; B is CSR
// (push), bt is B stored column-major (pull).  Offsets int64, indices int32.
struct Prob {
    const int64_t* a_ptr;
    const int32_t* a_idx;
    const void* a_val;
    const int64_t* b_ptr;
    const int32_t* b_idx;
    const void* b_val;
    const int64_t* m_ptr;
    const int32_t* m_idx;
    const int64_t* bt_ptr;
    const int32_t* bt_idx;
    const void* bt_val;
    const int64_t* row_flops;
    int64_t cursor_stride;   // sliced hub rows: int64 slice cursors per group (entries), 0 = none
    // k-blocked passes of a hash bin (B larger than L2): this launch takes only the A
    // entries whose B row starts in entries [kb_lo, kb_hi) of B; kb_pass 0 = off,
    // 1 = first pass (stores the partial counts), 2 = middle (adds), 3 = last (adds, gathers)
    int64_t kb_lo, kb_hi;
    int64_t kb_min_flops;   // rows under this many products run whole in the last pass
    int kb_pass;
    int64_t nrows;
    int64_t ncols;
};

// Where a kernel writes its rows.  off[i] = slot offset of row i (1P bound
// offsets, or the exact 2P row pointer); idx/val may be null in symbolic mode.
struct Out {
    const int64_t* off;
    int32_t* idx;
    void* val;
    int64_t* row_nnz;
    unsigned long long* evaluated;
    int out_f64;  // 1: values are float64, 0: int64
    int* overflow;  // small-problem path: set when a row does not fit the fixed table (host falls back)
    unsigned long long* gen_flops;   // direct path (no analysis pass): generated flops summed by the kernel
    int* empty_rows;                 // direct path: rows with no product or an empty mask row
};

// A bin of rows handled by one kernel family/tier, fetched dynamically.
struct Work {
    const int32_t* rows;
    int32_t count;
    int32_t* cursor;   // zero-initialised fetch counter
};

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int ceil_log2_i64(int64_t x) {
    if (x <= 1) return 0;
    return 64 - __clzll((unsigned long long)(x - 1));
}

// Fibonacci hash of a column index into a 2^lg table (lg >= 1).
constexpr uint32_t FIB_MULT = 0x9E3779B1u;
__device__ __forceinline__ uint32_t fib_hash(int32_t j, int lg) {
    return ((uint32_t)j * FIB_MULT) >> (32 - lg);
}

// Named barrier for a group of `nthreads` (multiple of 32) threads; id 1..15.
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    if (nthreads == 32) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
    }
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
    return __shfl_sync(FULL, v, src);
}

__device__ __forceinline__ int64_t shfl64(int64_t v, int src) {
    return (int64_t)__shfl_sync(FULL, (long long)v, src);
}

__device__ __forceinline__ long long shfl_up64(long long v, int d) {
    return __shfl_up_sync(FULL, v, d);
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int u = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += u;
    }
    return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

// Smallest l in [0,32) with incl[l] > q, given a non-decreasing inclusive
// scan `incl` held one value per lane and q < incl[31].  All lanes call.
__device__ __forceinline__ int owner_of(int incl, int q) {
    int l = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1) {
        int v = __shfl_sync(FULL, incl, l + step - 1);
        if (v <= q) l += step;
    }
    return l;
}

// first position in idx[lo, hi) whose value is >= key
__device__ __forceinline__ int64_t lower_bound_range(const int32_t* __restrict__ idx, int64_t lo, int64_t hi,
                                                     int32_t key) {
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (idx[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// first position in idx[lo, hi) whose value is >= key, galloping from lo:
// O(log(distance)) loads, one when the answer is lo (sliced hub rows walk
// every B row slice by slice, each slice starting where the previous ended).
__device__ __forceinline__ int64_t gallop_lower_bound(const int32_t* __restrict__ idx, int64_t lo, int64_t hi,
                                                      int32_t key) {
    if (lo >= hi || idx[lo] >= key) return lo;
    int64_t step = 1;
    int64_t prev = lo;   // idx[prev] < key
    for (;;) {
        const int64_t q = prev + step;
        if (q >= hi) return lower_bound_range(idx, prev + 1, hi, key);
        if (idx[q] >= key) return lower_bound_range(idx, prev + 1, q, key);
        prev = q;
        step <<= 1;
    }
}

// lower_bound over a sorted int32 array.
__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t n, int32_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool contains_sorted(const int32_t* a, int64_t n, int32_t key) {
    int64_t p = lower_bound_i32(a, n, key);
    return p < n && a[p] == key;
}

}  // namespace mm
