// Sliced hub rows as independent work items (plain mask, one-phase numeric).
//
// Reference semantics: hash_numeric (_kernels.py:130-218) for rows whose mask
// does not fit the largest shared table; the output stays in mask order
// (:208-216).
//
// hash_row (push_hash.cuh) walks a hub row's slices one after another in one
// 16-warp group, so a hub row is one long work item: R-MAT's largest rows
// leave most SMs idle at the end of the sliced launch (cfg5: SM active cycles
// 63 % of the elapsed ones, profiles/r2/r2_base_cfg5_sliced_details.csv).
// Here every (row, slice) pair is its own item, fetched dynamically by any
// group on any SM.  In the one-phase plain form each row owns nm slots at its
// mask offset, so slice s writes its hits at slot (s * slice) of its row and
// counts them; k_slice_join then closes the gaps (segments moved left in slice
// order) and sets the row's count.  Results are identical to hash_row's: the
// same slices, the same table, the same products per slot.
#pragma once
#include "push_hash.cuh"

namespace mm {

#ifndef MM_ITEM_GW
#define MM_ITEM_GW 32
#endif
constexpr int ITEM_GW = MM_ITEM_GW;   // 32 warps: one 1024-thread block per SM at 64 registers (16: cfg5 349.6 vs 334.4 ms)

// One block: block-wide exclusive scan of x over 1024 threads; returns the
// thread's offset and the total in *tot.
__device__ __forceinline__ int32_t block_excl_scan_1024(int32_t x, int32_t* s_tot, int32_t* tot) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t v = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += y;
    }
    if (lane == 31) s_tot[w] = v;
    __syncthreads();
    if (w == 0) {
        int32_t t = s_tot[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int32_t y = __shfl_up_sync(FULL, t, d);
            if (lane >= d) t += y;
        }
        s_tot[lane] = t;   // inclusive warp totals
    }
    __syncthreads();
    const int32_t before = (w ? s_tot[w - 1] : 0) + v - x;
    *tot = s_tot[31];
    __syncthreads();
    return before;
}

// Items of the bin's rows in row order: row q (position in wk.rows) owns
// items [row_base[q], row_base[q] + ceil(nm / slice)).  One block of 1024.
__global__ void __launch_bounds__(1024) k_slice_items(Prob p, Work wk, int64_t slice, int32_t* row_base,
                                                      int32_t* item_q, int32_t* item_s, int32_t* n_items,
                                                      int64_t max_items) {
    __shared__ int32_t s_tot[32];
    int32_t running = 0;
    for (int32_t q0 = 0; q0 < wk.count; q0 += 1024) {
        const int32_t q = q0 + (int32_t)threadIdx.x;
        int32_t ns = 0;
        if (q < wk.count) {
            const int64_t i = wk.rows[q];
            const int64_t nm = p.m_ptr[i + 1] - p.m_ptr[i];
            ns = (int32_t)((nm + slice - 1) / slice);
            if (ns < 1) ns = 1;
        }
        int32_t tot;
        const int32_t b = running + block_excl_scan_1024(ns, s_tot, &tot);
        if (q < wk.count) {
            row_base[q] = b;
            for (int32_t s = 0; s < ns && b + s < max_items; s++) {
                item_q[b + s] = q;
                item_s[b + s] = s;
            }
        }
        running += tot;
    }
    if (threadIdx.x == 0) {
        row_base[wk.count] = running;
        *n_items = running <= max_items ? running : -1;   // -1: the host bound was wrong (never expected)
    }
}

// Groups of ITEM_GW warps fetch (row, slice) items; table in shared memory.
template <int KIND>
__global__ void __launch_bounds__(ITEM_GW * 32, ITEM_GW == 32 ? 1 : MM_HASH16_MINB)
k_push_hash_items(Prob p, Out o, Work wk, const int32_t* item_q, const int32_t* item_s, const int32_t* n_items,
                  int32_t* item_cursor, int64_t slice, int cap_lg_max, const int32_t* row_base,
                  int32_t* slice_cnt) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_item;
    __shared__ int s_warp[32];
    constexpr int GW = ITEM_GW, GT = GW * 32;
    const int gt = threadIdx.x;
    const int bar_id = 1;
    const int cap_max = 1 << cap_lg_max;
    constexpr size_t BATCH_BYTES = batch_bytes<GW, KIND>();
    unsigned char* base = smem;
    unsigned char* bbase = smem + (size_t)cap_max * HashEntry<KIND>::bytes;
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    unsigned char* wq = bbase + BATCH_BYTES + (size_t)(threadIdx.x >> 5) * queue_bytes<KIND>();
    Table<KIND> tb;
    tb.bind(base, cap_max);
    __shared__ uint32_t s_dummy[GT];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
    for (int e = gt; e < cap_max; e += GT) {   // hash_part keeps it clean from here on
        tb.keys[e] = EMPTY_KEY;
        tb.cnt[e] = 0;
        if (KIND == 1) tb.val[e] = 0ull;
    }
    group_bar(bar_id, GT);
    const int32_t total = *n_items;
    unsigned long long evaluated = 0;
    for (;;) {
        if (gt == 0) s_item = atomicAdd(item_cursor, 1);
        group_bar(bar_id, GT);
        const int t = s_item;
        group_bar(bar_id, GT);
        if (t >= total) break;
        const int32_t q = item_q[t], s = item_s[t];
        RowInfo ri;
        ri.i = wk.rows[q];
        ri.as = p.a_ptr[ri.i];
        ri.ae = p.a_ptr[ri.i + 1];
        ri.ms = p.m_ptr[ri.i];
        ri.me = p.m_ptr[ri.i + 1];
        const int64_t s0 = ri.ms + (int64_t)s * slice;
        const int64_t s1 = s0 + slice < ri.me ? s0 + slice : ri.me;
        const int32_t c_lo = s == 0 ? INT32_MIN : p.m_idx[s0];
        const int32_t c_hi = s1 < ri.me ? p.m_idx[s1] : INT32_MAX;
        int cnt = 0;
        if (ri.ae > ri.as && s1 > s0)
            cnt = hash_part<GW, KIND, MODE_PLAIN, true, true>(p, o, tb, ri, s0, s1, c_lo, c_hi,
                                                              o.off[ri.i] + (s0 - ri.ms), cap_lg_max, cap_lg_max,
                                                              gt, bar_id, s_warp, bsm, wq, dummy_s, evaluated);
        if (gt == 0) slice_cnt[row_base[q] + s] = cnt;
    }
    long long e = warp_sum_ll((long long)evaluated);
    if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
}

// One block per row of the bin: slice s's hits sit at slot s * slice of the
// row; move them left in slice order so the row is contiguous (mask order).
// A chunk is read completely before it is written, and a write lands below
// every slot not read yet, so the move is safe in place.
__global__ void __launch_bounds__(512) k_slice_join(Work wk, const int64_t* off, const int64_t* m_ptr, int64_t slice,
                                                    const int32_t* row_base, const int32_t* slice_cnt, int32_t* idx,
                                                    unsigned long long* val, int64_t* row_nnz) {
    const int32_t q = blockIdx.x;
    if (q >= wk.count) return;
    const int64_t i = wk.rows[q];
    const int32_t b0 = row_base[q], ns = row_base[q + 1] - b0;
    const int64_t o = off[i];
    int64_t dst = slice_cnt[b0];
    for (int32_t s = 1; s < ns; s++) {
        const int32_t c = slice_cnt[b0 + s];
        const int64_t src = (int64_t)s * slice;
        if (dst != src) {
            for (int32_t c0 = 0; c0 < c; c0 += 512) {
                const int32_t e = c0 + (int32_t)threadIdx.x;
                int32_t x = 0;
                unsigned long long v = 0;
                if (e < c) {
                    x = idx[o + src + e];
                    v = val[o + src + e];
                }
                __syncthreads();
                if (e < c) {
                    idx[o + dst + e] = x;
                    val[o + dst + e] = v;
                }
                __syncthreads();
            }
        }
        dst += c;
    }
    if (threadIdx.x == 0) row_nnz[i] = dst;
}

}  // namespace mm
