// Sparse element-wise kernels used by the graph drivers around the masked
// multiply (betweenness centrality, graphs.py:121-200):
//   * lookup_rows (_kernels.py:597-612): values of Y at X's pattern, and the
//     two BC forms fused with their element-wise arithmetic
//     (graphs.py:181-185: w = (1 + delta) / paths on sigma_t's pattern, and
//     contrib = wq * paths on wq's pattern);
//   * ewise_add (sparse.py:360-370): union of two canonical CSR matrices,
//     values added where both hold an entry (count, then fill at exact
//     offsets);
//   * the per-batch score update (graphs.py:188-197): scores[r] += the
//     delta row in column order, then minus the source's own entry.
// One warp per row; rows are canonical (strictly increasing columns), so a
// lane finds its partner entry by binary search in the other row.
#pragma once
#include "common.cuh"

namespace mm {

enum LookupOp : int { LK_VALUE = 0, LK_BC_WEIGHT = 1, LK_SCALE = 2 };

// Per X entry t (row i, column j):
//   LK_VALUE:     out[t] = Y[i,j] (0 when absent), found[t] = present
//   LK_BC_WEIGHT: out[t] = (1 + Y[i,j]) / Z[i,j]       (absent -> 0)
//   LK_SCALE:     out[t] = xv[t] * Y[i,j]               (absent -> 0)
template <int OP, typename T>
__global__ void __launch_bounds__(256) k_lookup(int64_t nrows, const int64_t* __restrict__ x_ptr,
                                                const int32_t* __restrict__ x_idx, const T* __restrict__ x_val,
                                                const int64_t* __restrict__ y_ptr, const int32_t* __restrict__ y_idx,
                                                const T* __restrict__ y_val, const int64_t* __restrict__ z_ptr,
                                                const int32_t* __restrict__ z_idx, const T* __restrict__ z_val,
                                                T* __restrict__ out, uint8_t* __restrict__ found) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t xs = x_ptr[i], xe = x_ptr[i + 1];
        if (xs == xe) continue;
        const int64_t ys = y_ptr[i], ye = y_ptr[i + 1];
        for (int64_t t = xs + lane; t < xe; t += 32) {
            const int32_t j = x_idx[t];
            const int64_t p = lower_bound_range(y_idx, ys, ye, j);
            const bool hit = p < ye && y_idx[p] == j;
            const T y = hit ? y_val[p] : T(0);
            if (OP == LK_VALUE) {
                out[t] = y;
                if (found) found[t] = hit;
            } else if (OP == LK_BC_WEIGHT) {
                const int64_t zs = z_ptr[i], ze = z_ptr[i + 1];
                const int64_t q = lower_bound_range(z_idx, zs, ze, j);
                const T z = (q < ze && z_idx[q] == j) ? z_val[q] : T(0);
                out[t] = (T(1) + y) / z;
            } else {
                out[t] = x_val[t] * y;
            }
        }
    }
}

// Union sizes: counts[i] = |A_i| + |B_i| - |A_i and B_i|.
__global__ void __launch_bounds__(256) k_ewise_count(int64_t nrows, const int64_t* __restrict__ a_ptr,
                                                     const int32_t* __restrict__ a_idx,
                                                     const int64_t* __restrict__ b_ptr,
                                                     const int32_t* __restrict__ b_idx, int64_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t as = a_ptr[i], ae = a_ptr[i + 1], bs = b_ptr[i], be = b_ptr[i + 1];
        int both = 0;
        if (as < ae && bs < be)
            for (int64_t t = as + lane; t < ae; t += 32) {
                const int32_t j = a_idx[t];
                const int64_t p = lower_bound_range(b_idx, bs, be, j);
                both += p < be && b_idx[p] == j;
            }
        both = __reduce_add_sync(FULL, both);
        if (lane == 0) counts[i] = (ae - as) + (be - bs) - both;
    }
}

// Union fill at c_ptr offsets.  The output position of an entry is its rank
// in its own row plus the number of the other row's entries below it, minus
// the coinciding pairs below it (counted once, not twice).  A coinciding pair
// is written by A's lane with value a + b — the reference's dedup add of the
// lexsorted concatenation [A; B] (sparse.py:368-370, :203-211).
template <typename T>
__global__ void __launch_bounds__(256) k_ewise_fill(int64_t nrows, const int64_t* __restrict__ a_ptr,
                                                    const int32_t* __restrict__ a_idx, const T* __restrict__ a_val,
                                                    const int64_t* __restrict__ b_ptr,
                                                    const int32_t* __restrict__ b_idx, const T* __restrict__ b_val,
                                                    const int64_t* __restrict__ c_ptr, int32_t* __restrict__ c_idx,
                                                    T* __restrict__ c_val) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t as = a_ptr[i], ae = a_ptr[i + 1], bs = b_ptr[i], be = b_ptr[i + 1];
        const int64_t cs = c_ptr[i];
        int64_t matched = 0;   // coinciding pairs among A's entries already placed
        for (int64_t t0 = as; t0 < ae; t0 += 32) {
            const int64_t t = t0 + lane;
            const bool live = t < ae;
            int32_t j = 0;
            int64_t p = bs;
            bool hit = false;
            if (live) {
                j = a_idx[t];
                p = lower_bound_range(b_idx, bs, be, j);
                hit = p < be && b_idx[p] == j;
            }
            const unsigned hits = __ballot_sync(FULL, hit);
            if (live) {
                const int64_t pos = (t - as) + (p - bs) - (matched + __popc(hits & lanemask_lt()));
                c_idx[cs + pos] = j;
                c_val[cs + pos] = hit ? a_val[t] + b_val[p] : a_val[t];
            }
            matched += __popc(hits);
        }
        matched = 0;           // coinciding pairs among B's entries already passed
        for (int64_t s0 = bs; s0 < be; s0 += 32) {
            const int64_t s = s0 + lane;
            const bool live = s < be;
            int32_t j = 0;
            int64_t p = as;
            bool hit = false;
            if (live) {
                j = b_idx[s];
                p = lower_bound_range(a_idx, as, ae, j);
                hit = p < ae && a_idx[p] == j;
            }
            const unsigned hits = __ballot_sync(FULL, hit);
            if (live && !hit) {
                const int64_t pos = (s - bs) + (p - as) - (matched + __popc(hits & lanemask_lt()));
                c_idx[cs + pos] = j;
                c_val[cs + pos] = b_val[s];
            }
            matched += __popc(hits);
        }
    }
}

// scores[r] += delta[r, :] in column order (np.add.at over delta.triples(),
// graphs.py:188-189), then scores[r] -= delta[r, src_col[r]] for a source
// row (absent -> 0; graphs.py:192-197).  One thread per row keeps the
// reference's sequential summation order exactly.
__global__ void __launch_bounds__(256) k_bc_accumulate(int64_t nrows, const int64_t* __restrict__ d_ptr,
                                                       const int32_t* __restrict__ d_idx,
                                                       const double* __restrict__ d_val,
                                                       const int32_t* __restrict__ src_col,
                                                       double* __restrict__ scores) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = d_ptr[r], e = d_ptr[r + 1];
        const int32_t own = src_col ? src_col[r] : -1;
        if (s == e && own < 0) continue;
        double acc = scores[r];
        for (int64_t t = s; t < e; t++) acc += d_val[t];
        if (own >= 0) {
            const int64_t p = lower_bound_range(d_idx, s, e, own);
            acc -= (p < e && d_idx[p] == own) ? d_val[p] : 0.0;
        }
        scores[r] = acc;
    }
}

}  // namespace mm
