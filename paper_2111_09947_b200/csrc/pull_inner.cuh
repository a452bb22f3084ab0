// Pull path: one sparse dot product per mask nonzero (B stored column-major).
//
// Reference: inner_numeric / inner_symbolic (_kernels.py:519-579) — for each
// mask entry (i, j) a two-pointer merge of A_i with column j of B, summing in
// ascending k, emitting only if some k matched; symbolic stops at the first
// hit (:571-573).  Non-complemented masks only (multiply.py:70-72).
//
// GPU form: a warp owns a row; A_i is staged in shared memory (when it fits)
// and the warp walks column j of B 32 entries at a time, each lane
// binary-searching its row index k in A_i.  Hits are gathered with
// __ballot_sync; float64 products are folded in lane (= ascending k) order
// with __shfl_sync so the sum is bit-identical to the reference's merge.
#pragma once
#include "common.cuh"

namespace mm {

template <int KIND, bool NUMERIC>
__global__ void __launch_bounds__(256) k_pull_inner(Prob p, Out o, Work wk, int stage_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const size_t esz = KIND == 0 ? 4 : 12;
    unsigned char* wbase = smem + (size_t)warp * stage_max * esz;
    int32_t* s_idx = (int32_t*)wbase;
    unsigned long long* s_val = (unsigned long long*)(wbase + (size_t)stage_max * 4);
    // keep the 8-byte values 8-byte aligned: stage_max is a multiple of 2
    unsigned long long evaluated = 0;
    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(wk.cursor, 1);
        r = __shfl_sync(FULL, r, 0);
        if (r >= wk.count) break;
        const int64_t i = wk.rows[r];
        const int64_t as = p.a_ptr[i], ae = p.a_ptr[i + 1], na = ae - as;
        const int64_t ms = p.m_ptr[i], me = p.m_ptr[i + 1];
        const bool staged = na <= stage_max;
        if (staged) {
            for (int64_t t = lane; t < na; t += 32) {
                s_idx[t] = p.a_idx[as + t];
                if (KIND != 0) s_val[t] = ((const unsigned long long*)p.a_val)[as + t];
            }
            __syncwarp();
        }
        const int32_t* A = staged ? s_idx : p.a_idx + as;
        const unsigned long long* AV =
            staged ? s_val : (KIND != 0 ? (const unsigned long long*)p.a_val + as : nullptr);
        const int32_t a_last = A[na - 1];
        const int64_t w = NUMERIC ? o.off[i] : 0;
        int n_out = 0;
        for (int64_t t = ms; t < me; t++) {
            const int32_t j = p.m_idx[t];
            const int64_t bs = p.bt_ptr[j], be = p.bt_ptr[j + 1];
            bool hit_any = false;
            long long cnt = 0;
            long long acc_i = 0;
            double acc_d = 0.0;
            for (int64_t s0 = bs; s0 < be; s0 += 32) {
                const int64_t s = s0 + lane;
                const int32_t k = s < be ? p.bt_idx[s] : 0x7fffffff;
                int64_t pos = 0;
                bool hit = false;
                if (s < be && k <= a_last) {
                    pos = lower_bound_i32(A, na, k);
                    hit = pos < na && A[pos] == k;
                }
                unsigned bal = __ballot_sync(FULL, hit);
                if (bal) {
                    cnt += __popc(bal);
                    if (KIND == 1 && NUMERIC) {
                        long long prod = hit ? (long long)AV[pos] * ((const long long*)p.bt_val)[s] : 0;
                        acc_i += warp_sum_ll(prod);
                    } else if (KIND == 2 && NUMERIC) {
                        double prod = hit ? __longlong_as_double((long long)AV[pos]) *
                                                ((const double*)p.bt_val)[s]
                                          : 0.0;
                        unsigned b = bal;
                        while (b) {
                            int src = __ffs(b) - 1;
                            b &= b - 1;
                            double pb = __shfl_sync(FULL, prod, src);
                            acc_d = hit_any ? acc_d + pb : pb;
                            hit_any = true;
                        }
                    }
                    hit_any = true;
                    if (!NUMERIC) break;
                }
                if (__shfl_sync(FULL, k, 31) >= a_last) break;
            }
            evaluated += cnt;
            if (hit_any) {
                if (NUMERIC && lane == 0) {
                    int64_t d = w + n_out;
                    o.idx[d] = j;
                    if (KIND == 0) {
                        if (o.out_f64) ((double*)o.val)[d] = (double)cnt;
                        else ((long long*)o.val)[d] = cnt;
                    } else if (KIND == 1) {
                        ((long long*)o.val)[d] = acc_i;
                    } else {
                        ((double*)o.val)[d] = acc_d;
                    }
                }
                n_out++;
            }
        }
        if (lane == 0) o.row_nnz[i] = n_out;
        __syncwarp();
    }
    if (NUMERIC && lane == 0 && evaluated) atomicAdd(o.evaluated, evaluated);
}

}  // namespace mm
