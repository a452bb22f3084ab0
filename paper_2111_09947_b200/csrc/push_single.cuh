// Push path for rows with a single A entry: C_i = a_i1 * B_k filtered by M_i
// (or by not-M_i).  Chosen by algorithm="auto" only.
//
// With one A entry there is nothing to accumulate: every product lands on a
// distinct column, B_k is sorted, so the row of C is B_k's entries that the
// mask allows, in order.  The multi-source BFS step of the benchmark (cfg4,
// C = not(V) (.) (F^T A), one source per row of F^T) is exactly this shape.
// A group of 4 warps owns a row: the mask row is marked in a shared-memory
// bitmap over its column window (one atomicOr per mask entry), every B_k
// entry is tested with one shared load, and survivors are compacted with a
// ballot prefix.  Semantics: the reference kernels on a one-entry A row
// (_kernels.py:48-87 with nins <= |B_k|, complement sorted == B_k order).
#pragma once
#include "common.cuh"
#include "product_loop.cuh"

namespace mm {

constexpr int SINGLE_GW = 4;

template <int KIND, bool NUMERIC, bool COMP>
__global__ void __launch_bounds__(256) k_push_single(Prob p, Out o, Work wk, int words_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[2];
    __shared__ int s_warp[2 * SINGLE_GW];
    constexpr int GT = SINGLE_GW * 32;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int lane = gt & 31;
    const int bar_id = 1 + g;
    uint32_t* bits = (uint32_t*)(smem + (size_t)g * 4 * words_max);
    for (int w = gt; w < words_max; w += GT) bits[w] = 0u;
    unsigned long long evaluated = 0;
    for (;;) {
        if (gt == 0) s_row[g] = atomicAdd(wk.cursor, 1);
        group_bar(bar_id, GT);
        const int r = s_row[g];
        group_bar(bar_id, GT);
        if (r >= wk.count) break;
        const int64_t i = wk.rows[r];
        const int64_t t = p.a_ptr[i];
        const int32_t k = p.a_idx[t];
        const int64_t bs = p.b_ptr[k], be = p.b_ptr[k + 1];
        const int64_t ms = p.m_ptr[i], me = p.m_ptr[i + 1];
        const int32_t lo = me > ms ? p.m_idx[ms] : 0;
        const uint32_t span = me > ms ? (uint32_t)(p.m_idx[me - 1] - lo) : 0u;
        for (int64_t q = ms + gt; q < me; q += GT) {
            const uint32_t off = (uint32_t)(p.m_idx[q] - lo);
            atomicOr(bits + (off >> 5), 1u << (off & 31u));
        }
        group_bar(bar_id, GT);
        long long a_i = 0;
        double a_d = 0.0;
        if (KIND == 1) a_i = ((const long long*)p.a_val)[t];
        if (KIND == 2) a_d = ((const double*)p.a_val)[t];
        const int64_t w0 = NUMERIC ? o.off[i] : 0;
        int running = 0;
        for (int64_t base = bs; base < be; base += GT) {
            const int64_t s = base + gt;
            bool keep = false;
            int32_t j = 0;
            if (s < be) {
                j = p.b_idx[s];
                const uint32_t off = (uint32_t)(j - lo);
                const bool in_mask = me > ms && off <= span && ((bits[off >> 5] >> (off & 31u)) & 1u);
                keep = COMP ? !in_mask : in_mask;
            }
            int tot;
            const int pos = group_prefix<SINGLE_GW>(keep, &tot, s_warp + g * SINGLE_GW, bar_id, gt);
            if (keep) {
                evaluated++;
                if (NUMERIC) {
                    const int64_t d = w0 + running + pos;
                    o.idx[d] = j;
                    if (KIND == 0) {
                        if (o.out_f64) ((double*)o.val)[d] = 1.0;
                        else ((long long*)o.val)[d] = 1;
                    } else if (KIND == 1) {
                        ((long long*)o.val)[d] = a_i * ((const long long*)p.b_val)[s];
                    } else {
                        ((double*)o.val)[d] = a_d * ((const double*)p.b_val)[s];
                    }
                }
            }
            running += tot;
        }
        if (gt == 0) o.row_nnz[i] = running;
        group_bar(bar_id, GT);
        for (int64_t q = ms + gt; q < me; q += GT) bits[((uint32_t)(p.m_idx[q] - lo)) >> 5] = 0u;
        group_bar(bar_id, GT);
    }
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if (lane == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

}  // namespace mm
