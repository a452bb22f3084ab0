// Exclusive scan (row-pointer build), 1P compaction and reductions.
//
// Reference: np.cumsum into out_ptr (multiply.py:366-367, 380-381, 391-392),
// compact_rows (_kernels.py:586-594), the one-phase bound assertion
// (multiply.py:390) and the triangle-count reduction (graphs.py:96).
#pragma once
#include "common.cuh"

namespace mm {

constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_ITEMS = 4;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// Block-local inclusive scan of `in` (n items) written to out[0..n);
// each block's total goes to partials[blockIdx.x].  Folded side jobs (so a
// small scan is one launch): out[-1] = 0 when zero_prev (exclusive form),
// the one-phase bound assertion (multiply.py:390) when bounds_off is given,
// and the grand total into *total when the scan is a single tile.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_tile(const int64_t* in, int64_t n,
                                                            int64_t* out, int64_t* partials,
                                                            int zero_prev, const int64_t* bounds_off,
                                                            int* flag, long long* total) {
    __shared__ long long s_warp[32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    if (zero_prev && blockIdx.x == 0 && threadIdx.x == 0) out[-1] = 0;
    long long v[SCAN_ITEMS];
    long long run = 0;
    bool over = false;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; q++) {
        int64_t idx = base + q;
        // counts are never negative, except the -1 with which the direct float64
        // pass marks the rows it leaves to the binned pass: those scan as 0, so the
        // offsets stay monotone and inside C for the compaction queued behind the
        // scan (its stale rows are rewritten after the binned pass)
        long long x = idx < n ? in[idx] : 0;
        x = x > 0 ? x : 0;
        if (bounds_off && idx < n) over |= x > bounds_off[idx + 1] - bounds_off[idx];
        run += x;
        v[q] = run;
    }
    if (bounds_off && __any_sync(FULL, over) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        long long u = __shfl_up_sync(FULL, x, d);
        if (lane >= d) x += u;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long y = s_warp[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            long long u = __shfl_up_sync(FULL, y, d);
            if (lane >= d) y += u;
        }
        s_warp[lane] = y;
    }
    __syncthreads();
    long long prefix = (x - run) + (warp > 0 ? s_warp[warp - 1] : 0);
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; q++) {
        int64_t idx = base + q;
        if (idx < n) out[idx] = v[q] + prefix;
    }
    if (threadIdx.x == SCAN_THREADS - 1) {
        partials[blockIdx.x] = s_warp[31];
        if (total && gridDim.x == 1) *total = s_warp[31];
    }
}

// out[i] += offsets[block of i] (offsets = exclusive scan of the partials);
// the last element's final value also goes to *total when given.
__global__ void k_scan_add(int64_t* out, int64_t n, const int64_t* offsets, long long* total) {
    int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx < n) {
        const int64_t v = out[idx] + offsets[idx / SCAN_TILE];
        out[idx] = v;
        if (total && idx == n - 1) *total = v;
    }
}

__global__ void k_set_zero_i64(int64_t* p) { *p = 0; }

// compact_rows (_kernels.py:586-594), element-parallel: a warp owns 256
// consecutive OUTPUT entries, finds the row of each by a binary search of
// out_ptr restricted to the warp's row span, and copies from the row's slot
// range.  Work is proportional to nnz(C) whatever the row-length skew.  The
// one-phase bound assertion (multiply.py:390) is checked row-parallel: a row
// that overran its slot range raises flag (MM_ERR_INTERNAL at the ABI).
// Last r in [lo, hi] with ptr[r] <= e (ptr non-decreasing, ptr[lo] <= e),
// by a 32-ary search: each round the warp probes 32 evenly spaced rows, so a
// million rows take 4 dependent loads instead of 20.  All lanes call.
__device__ __forceinline__ int64_t warp_upper_row(const int64_t* ptr, int64_t lo, int64_t hi, int64_t e, int lane) {
    while (hi - lo >= 32) {
        const int64_t step = (hi - lo) >> 5;         // probes lo + step .. lo + 32 step <= hi
        const int64_t probe = lo + (int64_t)(lane + 1) * step;
        const bool le = __ldg(ptr + probe) <= e;
        const unsigned bal = __ballot_sync(FULL, le);
        if (bal == 0) {
            hi = lo + step - 1;
        } else {
            const int top = 31 - __clz(bal);            // probes are monotone: bal is a prefix
            lo = lo + (int64_t)(top + 1) * step;
            if (top < 31) hi = lo + step - 1;
        }
    }
    const int64_t probe = lo + lane;
    const bool le = probe <= hi && __ldg(ptr + probe) <= e;
    const unsigned bal = __ballot_sync(FULL, le);
    return lo + (31 - __clz(bal));
}

template <typename T>
__global__ void __launch_bounds__(256) k_compact(int64_t nrows, const int64_t* bounds_off,
                                                 const int64_t* row_nnz, const int32_t* tmp_idx,
                                                 const T* tmp_val, const int64_t* out_ptr,
                                                 int32_t* out_idx, T* out_val, int* flag) {
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    if (flag)
        for (int64_t i = gtid; i < nrows; i += nthreads)
            if (row_nnz[i] > bounds_off[i + 1] - bounds_off[i]) atomicExch(flag, 1);
    const int64_t total = out_ptr[nrows];
    const int64_t warp = gtid >> 5;
    const int64_t nwarps = nthreads >> 5;
    constexpr int PER = 128;
    // A warp owns 128-entry tiles: a 32-ary search of the row pointer finds the
    // row of the tile's first entry; the tile's rows are then read as ONE
    // coalesced load of the next 32 row ends, and only a tile that spans more
    // rows (runs of empty rows) searches for its last row.
    const int64_t tiles = (total + PER - 1) / PER;
    for (int64_t t = warp; t < tiles; t += nwarps) {
        // every row before r_lo ends at or before the tile's first entry
        int64_t r_lo = warp_upper_row(out_ptr, 0, nrows, t * PER, lane);
        const int64_t e0 = t * PER;
        const int64_t e1 = e0 + PER < total ? e0 + PER : total;
        const int64_t r = r_lo + lane;
        const int64_t end = r < nrows ? __ldg(out_ptr + r + 1) : INT64_MAX;
        if (shfl64(end, 31) > e1 - 1) {
            // the tile lies within rows r_lo .. r_lo + 31: owner by a shuffle search
            const int64_t boff = r < nrows ? __ldg(bounds_off + r) - __ldg(out_ptr + r) : 0;
#pragma unroll
            for (int u = 0; u < PER / 32; u++) {
                const int64_t e = e0 + u * 32 + lane;
                int l = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const int64_t v = shfl64(end, l + step - 1);
                    if (v <= e) l += step;
                }
                const int64_t src = shfl64(boff, l) + e;
                if (e < e1) {
                    out_idx[e] = tmp_idx[src];
                    out_val[e] = tmp_val[src];
                }
            }
        } else {
            // a run of more than 32 rows (empty rows among them): search per entry
            const int64_t r_hi = warp_upper_row(out_ptr, r_lo, nrows, e1 - 1, lane);
#pragma unroll 4
            for (int u = 0; u < PER / 32; u++) {
                const int64_t e = e0 + u * 32 + lane;
                if (e < e1) {
                    int64_t lo = r_lo, hi = r_hi;
                    while (lo < hi) {
                        const int64_t mid = (lo + hi + 1) >> 1;
                        if (__ldg(out_ptr + mid) <= e) lo = mid; else hi = mid - 1;
                    }
                    const int64_t src = bounds_off[lo] + (e - out_ptr[lo]);
                    out_idx[e] = tmp_idx[src];
                    out_val[e] = tmp_val[src];
                }
            }
        }
    }
}

// compact_rows, row-parallel: for outputs much sparser than the rows (cfg3:
// 4,075 entries over 262,144 rows) the element-parallel form's row searches
// are a chain of dependent loads per tile; a thread per row reads the row
// counts coalesced and copies its few entries.
template <typename T>
__global__ void __launch_bounds__(256) k_compact_rowwise(int64_t nrows, const int64_t* bounds_off,
                                                         const int64_t* row_nnz, const int32_t* tmp_idx,
                                                         const T* tmp_val, const int64_t* out_ptr,
                                                         int32_t* out_idx, T* out_val, int* flag) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += nthreads) {
        const int64_t n = row_nnz[i];
        if (n == 0) continue;
        const int64_t src = bounds_off[i], dst = out_ptr[i];
        if (flag && n > bounds_off[i + 1] - src) atomicExch(flag, 1);
        for (int64_t q = 0; q < n; q++) {
            out_idx[dst + q] = tmp_idx[src + q];
            out_val[dst + q] = tmp_val[src + q];
        }
    }
}

// 1P check: no row overran its slot range (multiply.py:390).
__global__ void k_check_bounds(int64_t n, const int64_t* row_nnz, const int64_t* bounds_off, int* flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (row_nnz[i] > bounds_off[i + 1] - bounds_off[i]) atomicExch(flag, 1);
}

// 2P check: symbolic counts must equal the numeric row sizes (multiply.py:375).
__global__ void k_check_equal(int64_t n, const int64_t* a, const int64_t* b, int* flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (a[i] != b[i]) atomicExch(flag, 1);
}

// Deterministic two-pass sum: per-block partials in a fixed grid, then one
// block folds them in order.
template <typename T>
__global__ void __launch_bounds__(256) k_reduce_partial(const T* v, int64_t n, T* partials) {
    __shared__ T s[256];
    T acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        acc += v[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 128; d > 0; d >>= 1) {
        if (threadIdx.x < d) s[threadIdx.x] += s[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) partials[blockIdx.x] = s[0];
}

template <typename T>
__global__ void __launch_bounds__(256) k_reduce_final(const T* partials, int nparts, T* out) {
    __shared__ T s[256];
    T acc = 0;
    for (int q = threadIdx.x; q < nparts; q += blockDim.x) acc += partials[q];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int d = 128; d > 0; d >>= 1) {
        if (threadIdx.x < d) s[threadIdx.x] += s[threadIdx.x + d];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}
}  // namespace mm

namespace mm {

// k-truss prune step (graphs.py:111-117): keep the entries of C whose value
// is >= thr.  Pass 1 counts survivors per row (warp per row), pass 2 copies
// them in order into the scanned offsets; the kept pattern stays canonical.
template <bool WRITE>
__global__ void __launch_bounds__(256) k_filter_min(int64_t nrows, const int64_t* ptr, const int32_t* idx,
                                                    const long long* val, long long thr, int64_t* counts,
                                                    const int64_t* out_ptr, int32_t* out_idx) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t s0 = ptr[i], s1 = ptr[i + 1];
        int64_t run = WRITE ? out_ptr[i] : 0;
        for (int64_t b = s0; b < s1; b += 32) {
            const int64_t s = b + lane;
            const bool keep = s < s1 && val[s] >= thr;
            const unsigned bal = __ballot_sync(FULL, keep);
            if (WRITE && keep) out_idx[run + __popc(bal & lanemask_lt())] = idx[s];
            run += __popc(bal);
        }
        if (!WRITE && lane == 0) counts[i] = run;
    }
}

}  // namespace mm
