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

namespace mm {

// Pull path for rows with short masks (<= 32 entries) and short A rows /
// B columns (cfg3's d1 / d4 shape): one LANE per mask entry instead of one
// warp.  A warp takes 32 rows of the bin, packs whole rows into 32-entry
// windows (a row never straddles two windows), and every lane runs the
// reference's two-pointer merge of A_i with column j of B^T on its own
// (_kernels.py:535-548: ascending k, first product stored), so float64 sums
// are bit-identical.  Output positions come from a ballot of the hits
// restricted to the lanes of the same row, in mask order.
template <int KIND, bool NUMERIC>
__global__ void __launch_bounds__(256) k_pull_lane(Prob p, Out o, Work wk) {
    const int lane = threadIdx.x & 31;
    unsigned long long evaluated = 0;
    for (;;) {
        int base = 0;
        if (lane == 0) base = atomicAdd(wk.cursor, 32);
        base = __shfl_sync(FULL, base, 0);
        if (base >= wk.count) break;
        const int nr = wk.count - base < 32 ? wk.count - base : 32;
        int64_t ri = 0, as = 0, ae = 0, ms = 0;
        int nm = 0;
        if (lane < nr) {
            ri = wk.rows[base + lane];
            as = p.a_ptr[ri];
            ae = p.a_ptr[ri + 1];
            ms = p.m_ptr[ri];
            nm = (int)(p.m_ptr[ri + 1] - ms);
        }
        const int incl = warp_incl_scan(nm, lane);
        const int total = __shfl_sync(FULL, incl, 31);
        const int excl = incl - nm;
        int w0 = 0;
        while (w0 < total) {
            // the window ends at the last row that ends within w0 + 32
            const unsigned fit = __ballot_sync(FULL, lane < nr && incl > w0 && incl <= w0 + 32);
            const int wend = fit ? __shfl_sync(FULL, incl, 31 - __clz(fit)) : w0;
            if (wend == w0) break;   // unreachable: the bin holds rows of <= 32 mask entries
            const int e = w0 + lane;
            const bool live = e < wend;
            const int r = owner_of(incl, live ? e : wend - 1);
            const int64_t i = shfl64(ri, r);
            const int64_t a0 = shfl64(as, r), a1 = shfl64(ae, r), m0 = shfl64(ms, r);
            const int r_ex = __shfl_sync(FULL, excl, r), r_in = __shfl_sync(FULL, incl, r);
            bool hit = false;
            long long cnt = 0, acc_i = 0;
            double acc_d = 0.0;
            int32_t j = 0;
            if (live) {
                j = p.m_idx[m0 + (e - r_ex)];
                int64_t ia = a0, ib = p.bt_ptr[j];
                const int64_t be = p.bt_ptr[j + 1];
                int32_t ka = ia < a1 ? p.a_idx[ia] : 0x7fffffff;
                int32_t kb = ib < be ? p.bt_idx[ib] : 0x7fffffff;
                while (ia < a1 && ib < be) {
                    if (ka == kb) {
                        if (NUMERIC) {
                            if (KIND == 1) {
                                acc_i += ((const long long*)p.a_val)[ia] * ((const long long*)p.bt_val)[ib];
                            } else if (KIND == 2) {
                                const double prod = ((const double*)p.a_val)[ia] * ((const double*)p.bt_val)[ib];
                                acc_d = hit ? acc_d + prod : prod;
                            }
                        }
                        hit = true;
                        cnt++;
                        if (!NUMERIC) break;
                        ++ia;
                        ++ib;
                        ka = ia < a1 ? p.a_idx[ia] : 0x7fffffff;
                        kb = ib < be ? p.bt_idx[ib] : 0x7fffffff;
                    } else if (ka < kb) {
                        ++ia;
                        ka = ia < a1 ? p.a_idx[ia] : 0x7fffffff;
                    } else {
                        ++ib;
                        kb = ib < be ? p.bt_idx[ib] : 0x7fffffff;
                    }
                }
            }
            evaluated += cnt;
            const unsigned hits = __ballot_sync(FULL, hit);
            const int lo = r_ex - w0, len = r_in - r_ex;
            const unsigned rowmask = (len >= 32 ? 0xffffffffu : ((1u << len) - 1u)) << lo;
            if (NUMERIC && hit) {
                const int64_t d = o.off[i] + __popc(hits & rowmask & lanemask_lt());
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
            if (live && e == r_ex) o.row_nnz[i] = __popc(hits & rowmask);
            w0 = wend;
        }
    }
    if (NUMERIC) {
        const long long ev = warp_sum_ll((long long)evaluated);
        if (lane == 0 && ev) atomicAdd(o.evaluated, (unsigned long long)ev);
    }
}

}  // namespace mm
