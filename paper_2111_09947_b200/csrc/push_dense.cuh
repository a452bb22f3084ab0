// Push path, dense MSA over the mask row's column window: the paper's MSA
// accumulator (reference _kernels.py:48-87 — a dense state array per column,
// the mask marked ALLOWED, products accumulated only into allowed columns,
// gathered in mask order) restricted to the window [first, last] mask column
// of the row, so it lives in shared memory.
//
// Layout per group: [val: 8 B per column if KIND != 0][cnt: 4 B per column]
// for 32*words_max columns plus one guard column.  A column's cnt is DENIED
// (INT_MIN) unless it is in the current row's mask; a mask column holds its
// product count (plus-pair value) or a 0/1 "set" flag (plus-times).  The
// array is DENIED everywhere between rows: a row marks its mask columns and
// restores them after its gather, O(nm) per row instead of O(window).
//
// Per product: one clamp (columns outside the window land on the guard, which
// is always DENIED), one shared load, one compare, and for the ~10 % of
// products that survive the mask, one shared atomic.  Chosen (msa / auto)
// when the window fits the tier's budget; otherwise the rank-compressed MSA
// of push_rank.cuh.
//
// COMP: the complemented-mask MSA (_kernels.py:36-40,66-77) for outputs
// narrow enough that every column fits (ncols columns, e.g. the 512 source
// columns of a betweenness-centrality batch): the array is ALLOWED (0) between
// rows, a row marks its mask columns DENIED, products land on any other
// column, and the gather walks the columns in order (the reference sorts the
// inserted keys, :69) before restoring the array.
#pragma once
#include "common.cuh"
#include "product_loop.cuh"
#include "push_rank.cuh"

namespace mm {

constexpr int32_t DENIED = (int32_t)0x80000000;

__host__ __device__ constexpr size_t dense_region_bytes(int kind, int64_t words) {
    return (size_t)(kind == 0 ? 4 : 12) * (size_t)(32 * words + 1);
}

template <int KIND, bool NUMERIC>
struct DenseProber {
    uint32_t cnt_s, val_s;
    int32_t lo;
    uint32_t guard;     // index of the guard column
    uint32_t dummy_s;   // this lane's scratch word (MM_RED_ALL)
    const void* b_val;
    unsigned evaluated;
    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
        uint32_t off[U];
        int32_t v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            off[u] = min((uint32_t)(j[u] - lo), guard);   // EMPTY_KEY and out-of-window -> guard
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[u]) : "r"(cnt_s + (off[u] << 2)));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (KIND == 0) {
                // plus-pair: the evaluated count is the sum of the counts, taken at the gather
                if (NUMERIC)
#ifndef MM_RED_PRED
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t.reg .u32 ad;\n\t"
                        "setp.ge.s32 ph, %0, 0;\n\t"
                        "selp.u32 ad, %1, %2, ph;\n\t"
                        "red.shared.add.u32 [ad], 1;\n\t}" ::"r"(v[u]),
                        "r"(cnt_s + (off[u] << 2)), "r"(dummy_s)
                        : "memory");
#else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ge.s32 ph, %0, 0;\n\t"
                        "@ph red.shared.add.u32 [%1], 1;\n\t}" ::"r"(v[u]),
                        "r"(cnt_s + (off[u] << 2))
                        : "memory");
#endif
                else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ge.s32 ph, %0, 0;\n\t"
                        "@ph st.shared.u32 [%1], 1;\n\t}" ::"r"(v[u]),
                        "r"(cnt_s + (off[u] << 2))
                        : "memory");
            } else if (v[u] >= 0) {
                evaluated++;
                if (NUMERIC) {
                    const long long prod = a[u] * ((const long long*)b_val)[s[u]];
                    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(val_s + (off[u] << 3)), "l"(prod) : "memory");
                }
                asm volatile("st.shared.u32 [%0], 1;" ::"r"(cnt_s + (off[u] << 2)) : "memory");
            }
        }
    }
    __device__ __forceinline__ void drain() {}
};

// Window locator for the ordered float64 path: slot = column offset.
struct DenseWindow {
    const int32_t* cnt;
    int32_t lo;
    uint32_t span;
    __device__ __forceinline__ int rank(int32_t j) const {
        const uint32_t off = (uint32_t)(j - lo);
        if (off > span) return -1;
        return cnt[off] >= 0 ? (int)off : -1;
    }
};

// Complement gather: warp w owns columns [w ncols/GW, (w+1) ncols/GW); set
// columns are emitted in column order and reset to ALLOWED, then the row's
// mask columns are restored to ALLOWED.
template <int GW, int KIND, bool NUMERIC>
__device__ __forceinline__ void dense_gather_comp(const Prob& p, const Out& o, int32_t* cnt, unsigned long long* val,
                                                  const RowInfo& ri, int gt, int bar_id, int* s_warp, int64_t w0,
                                                  unsigned long long& evaluated) {
    constexpr int GT = GW * 32;
    const int lane = gt & 31, wg = gt >> 5;
    const int c_lo = (int)(p.ncols * wg / GW), c_hi = (int)(p.ncols * (wg + 1) / GW);
    int mine = 0;
    for (int c = c_lo + lane; c < c_hi; c += 32) {
        const int v = cnt[c];
        mine += v > 0;
        if (KIND == 0 && NUMERIC && v > 0) evaluated += (unsigned)v;
    }
    mine = (int)warp_sum_ll(mine);
    int before = 0, total = mine;
    if (GW > 1) {
        if (lane == 0) s_warp[wg] = mine;
        group_bar(bar_id, GT);
        total = 0;
#pragma unroll
        for (int q = 0; q < GW; q++) {
            const int c = s_warp[q];
            if (q < wg) before += c;
            total += c;
        }
    }
    int run = before;
    for (int cb = c_lo; cb < c_hi; cb += 32) {
        const int c = cb + lane;
        const int v = c < c_hi ? cnt[c] : 0;
        const bool set = v > 0;
        const unsigned bal = __ballot_sync(FULL, set);
        if (set) {
            if (NUMERIC) {
                const int64_t d = w0 + run + __popc(bal & lanemask_lt());
                o.idx[d] = c;
                if (KIND == 0) {
                    if (o.out_f64) ((double*)o.val)[d] = (double)v;
                    else ((long long*)o.val)[d] = v;
                } else {
                    ((unsigned long long*)o.val)[d] = val[c];
                }
            }
            cnt[c] = 0;
            if (KIND != 0) val[c] = 0ull;
        }
        run += __popc(bal);
    }
    if (gt == 0) o.row_nnz[ri.i] = total;
    group_bar(bar_id, GT);
    for (int64_t t = ri.ms + gt; t < ri.me; t += GT) cnt[p.m_idx[t]] = 0;
    group_bar(bar_id, GT);
}

template <int GW, int KIND, bool NUMERIC, bool COMP>
__device__ __forceinline__ void dense_row(const Prob& p, const Out& o, int32_t* cnt, unsigned long long* val,
                                          int words_max, uint32_t dummy_s, const RowInfo& ri, int gt, int bar_id, int* s_warp,
                                          BatchSmem bsm, unsigned long long& evaluated) {
    constexpr int GT = GW * 32;
    const int lane = gt & 31;
    const int wg = gt >> 5;
    const int64_t i = ri.i, as = ri.as, ae = ri.ae, ms = ri.ms, me = ri.me;
    const int nm = (int)(me - ms);
    const int32_t lo = COMP ? 0 : p.m_idx[ms];
    const int32_t hi = COMP ? (int32_t)(p.ncols - 1) : p.m_idx[me - 1];

    // 1. mark the mask columns (plain: the window is DENIED everywhere else;
    //    complement: ALLOWED everywhere else)
    for (int r = gt; r < nm; r += GT) {
        const int32_t off = p.m_idx[ms + r] - lo;
        if (COMP) {
            cnt[off] = DENIED;
        } else {
            cnt[off] = 0;
            if (KIND != 0) val[off] = 0ull;
        }
    }
    group_bar(bar_id, GT);

    // 2. products
    if (KIND == 2) {
        // groups split the row by output column (see ordered_products_f64):
        // plain by mask rank (the ranks warp wg gathers), complement by column
        int32_t c_lo = INT32_MIN, c_hi = INT32_MAX;
        bool idle = false;
        if (GW > 1) {
            if (COMP) {
                c_lo = wg == 0 ? INT32_MIN : (int32_t)(p.ncols * wg / GW);
                c_hi = wg == GW - 1 ? INT32_MAX : (int32_t)(p.ncols * (wg + 1) / GW);
                idle = wg > 0 && wg < GW - 1 && c_lo == c_hi;
            } else {
                const int r0 = (int)(((long long)nm * wg) / GW), r1 = (int)(((long long)nm * (wg + 1)) / GW);
                idle = r0 == r1;
                c_lo = wg == 0 ? INT32_MIN : p.m_idx[ms + r0];
                c_hi = r1 < nm ? p.m_idx[ms + r1] : INT32_MAX;
            }
        }
        DenseWindow win{cnt, lo, (uint32_t)(hi - lo)};
        RankLocatorF64<DenseWindow> loc{win, cnt, (double*)val};
        if (!idle) evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane, c_lo, c_hi);
    } else {
        DenseProber<KIND, NUMERIC> pr;
        pr.cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
        pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(val);
        pr.lo = lo;
        pr.guard = 32u * (uint32_t)words_max;
        pr.dummy_s = dummy_s;
        pr.b_val = p.b_val;
        pr.evaluated = 0u;
        flat_products<GW, KIND>(p, pr, as, ae, gt, bar_id, s_warp, bsm);
        evaluated += pr.evaluated;
    }
    group_bar(bar_id, GT);

    // 3. gather in mask order (warp w owns mask entries [w nm/GW, (w+1) nm/GW)),
    //    restoring DENIED behind it; complement: in column order
    const int64_t w0 = NUMERIC ? o.off[i] : 0;
    if (COMP) {
        dense_gather_comp<GW, KIND, NUMERIC>(p, o, cnt, val, ri, gt, bar_id, s_warp, w0, evaluated);
        return;
    }
    const int r_lo = (int)(((long long)nm * wg) / GW), r_hi = (int)(((long long)nm * (wg + 1)) / GW);
    int mine = 0;
    for (int r = r_lo + lane; r < r_hi; r += 32) {
        const int c = cnt[p.m_idx[ms + r] - lo];
        mine += c > 0;
        if (KIND == 0 && NUMERIC) evaluated += (unsigned)c;
    }
    mine = (int)warp_sum_ll(mine);
    int before = 0, total = mine;
    if (GW > 1) {
        if (lane == 0) s_warp[wg] = mine;
        group_bar(bar_id, GT);
        total = 0;
#pragma unroll
        for (int q = 0; q < GW; q++) {
            const int c = s_warp[q];
            if (q < wg) before += c;
            total += c;
        }
    }
    int run = before;
    for (int rb0 = r_lo; rb0 < r_hi; rb0 += 32) {
        const int r = rb0 + lane;
        int32_t j = 0, off = 0, c = 0;
        if (r < r_hi) {
            j = p.m_idx[ms + r];
            off = j - lo;
            c = cnt[off];
        }
        const bool set = c > 0;
        const unsigned bal = __ballot_sync(FULL, set);
        if (NUMERIC && set) {
            const int64_t d = w0 + run + __popc(bal & lanemask_lt());
            o.idx[d] = j;
            if (KIND == 0) {
                if (o.out_f64) ((double*)o.val)[d] = (double)c;
                else ((long long*)o.val)[d] = c;
            } else {
                ((unsigned long long*)o.val)[d] = val[off];
            }
        }
        if (r < r_hi) cnt[off] = DENIED;
        run += __popc(bal);
    }
    if (gt == 0) o.row_nnz[i] = total;
    group_bar(bar_id, GT);
}

#ifndef MM_DENSE_MINB
#define MM_DENSE_MINB 5
#endif
template <int GW, int KIND, bool NUMERIC, bool COMP = false>
__global__ void __launch_bounds__(256, GW <= 8 ? MM_DENSE_MINB : 1)
k_push_dense(Prob p, Out o, Work wk, int words_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[16];
    __shared__ int s_warp[32];
    constexpr int GT = GW * 32;
    const int groups = blockDim.x / GT;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int bar_id = 1 + g;
    const int ncol = 32 * words_max + 1;
    const size_t rbytes = (dense_region_bytes(KIND, words_max) + 15) & ~(size_t)15;
    unsigned char* region = smem + (size_t)g * rbytes;
    unsigned long long* val = KIND == 0 ? nullptr : (unsigned long long*)region;
    int32_t* cnt = (int32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)ncol));
    unsigned char* bbase = smem + (size_t)groups * rbytes + (size_t)g * batch_bytes<GW, KIND>();
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    __shared__ uint32_t s_dummy[256];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
    for (int c = gt; c < ncol; c += GT) {
        // complement: ALLOWED columns with zero values, the guard DENIED
        cnt[c] = COMP && c < ncol - 1 ? 0 : DENIED;
        if (COMP && KIND != 0) val[c] = 0ull;
    }
    group_bar(bar_id, GT);
    unsigned long long evaluated = 0;
#ifdef MM_STAGE_TMA
    stage_init();
#endif
    RowFetcher<GW> rf;
    if (wk.count < 4 * (int)(gridDim.x * (blockDim.x / (32 * GW)))) rf.per = 1;   // few rows: one per fetch
    RowInfo ri;
    while (rf.next(p, wk, gt, bar_id, s_row + g, ri))
        dense_row<GW, KIND, NUMERIC, COMP>(p, o, cnt, val, words_max, dummy_s, ri, gt, bar_id, s_warp + g * GW, bsm,
                                           evaluated);
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

}  // namespace mm
