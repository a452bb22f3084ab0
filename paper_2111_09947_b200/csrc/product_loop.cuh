// Product enumeration of one output row, shared by every push accumulator.
//
// Row-wise Gustavson (the reference's outer loops, e.g. _kernels.py:48-51):
// for t in A_i, for s in B_{a_idx[t]}: product (j = b_idx[s], a_val[t]*b_val[s]).
// The accumulator policy (hash table, windowed bitmap, rank search) only sees
// `put(j, a, s)` calls; this header decides how the product space is spread
// over the lanes of a group of GW warps.
#pragma once
#include "common.cuh"
#ifdef MM_STAGE_TMA
#include "stage_tma.cuh"
#endif

namespace mm {

// Group-wide exclusive prefix count of `flag`; returns the prefix, writes the
// group total to *total.  Uses s_warp[GW] scratch for GW > 1.
template <int GW>
__device__ __forceinline__ int group_prefix(bool flag, int* total, int* s_warp, int bar_id, int gt) {
    unsigned bal = __ballot_sync(FULL, flag);
    int lane = gt & 31;
    int in_warp = __popc(bal & lanemask_lt());
    if (GW == 1) {
        *total = __popc(bal);
        return in_warp;
    } else {
        int w = gt >> 5;
        if (lane == 0) s_warp[w] = __popc(bal);
        group_bar(bar_id, GW * 32);
        int before = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < GW; q++) {
            int c = s_warp[q];
            if (q < w) before += c;
            tot += c;
        }
        group_bar(bar_id, GW * 32);
        *total = tot;
        return before + in_warp;
    }
}

// Group-wide inclusive scan of an int (one value per thread); *total = sum.
template <int GW>
__device__ __forceinline__ int group_incl_scan(int v, int* total, int* s_warp, int bar_id, int gt) {
    const int lane = gt & 31;
    int x = warp_incl_scan(v, lane);
    if (GW == 1) {
        *total = __shfl_sync(FULL, x, 31);
        return x;
    } else {
        const int w = gt >> 5;
        if (lane == 31) s_warp[w] = x;
        group_bar(bar_id, GW * 32);
        int before = 0, tot = 0;
#pragma unroll
        for (int q = 0; q < GW; q++) {
            const int c = s_warp[q];
            if (q < w) before += c;
            tot += c;
        }
        group_bar(bar_id, GW * 32);
        *total = tot;
        return x + before;
    }
}

// Offsets of one row (A and mask).
struct RowInfo {
    int64_t i, as, ae, ms, me;
};

// Dynamic row fetch for a group of GW warps.  Single-warp groups take
// ROWS_PER_FETCH rows per global atomic and preload their offsets, one per
// lane, so the fetch latency of small rows is paid once per batch (small
// batches keep the tail balanced).
#ifndef MM_ROWS_PER_FETCH
#define MM_ROWS_PER_FETCH 4
#endif
// ENDMARK: the row list may be shorter than wk.count and then ends with -1
// (k_kb_select's compacted list, push_hash.cuh)
template <int GW, bool ENDMARK = false>
struct RowFetcher {
    int n = 0, q = 0;
    int per = MM_ROWS_PER_FETCH;   // rows per fetch (1-warp groups); 1 when rows are few per warp
    int64_t li = 0, las = 0, lae = 0, lms = 0, lme = 0;
    __device__ __forceinline__ bool next(const Prob& p, const Work& wk, int gt, int bar_id, int* s_row,
                                         RowInfo& ri) {
        const int lane = gt & 31;
        if (GW == 1) {
            if (q >= n) {
                int b = 0;
                if (lane == 0) b = atomicAdd(wk.cursor, per);
                b = __shfl_sync(FULL, b, 0);
                if (b >= wk.count) return false;
                n = wk.count - b < per ? wk.count - b : per;
                q = 0;
                if (lane < n) {
                    li = wk.rows ? wk.rows[b + lane] : b + lane;   // rows == nullptr: every row in order
                    las = p.a_ptr[li];
                    lae = p.a_ptr[li + 1];
                    lms = p.m_ptr[li];
                    lme = p.m_ptr[li + 1];
                }
            }
            ri.i = shfl64(li, q);
            ri.as = shfl64(las, q);
            ri.ae = shfl64(lae, q);
            ri.ms = shfl64(lms, q);
            ri.me = shfl64(lme, q);
            q++;
            return true;
        } else {
            if (gt == 0) *s_row = atomicAdd(wk.cursor, 1);
            group_bar(bar_id, GW * 32);
            const int r = *s_row;
            group_bar(bar_id, GW * 32);
            if (r >= wk.count) return false;
            ri.i = wk.rows ? wk.rows[r] : r;
            if (ENDMARK && ri.i < 0) return false;
            ri.as = p.a_ptr[ri.i];
            ri.ae = p.a_ptr[ri.i + 1];
            ri.ms = p.m_ptr[ri.i];
            ri.me = p.m_ptr[ri.i + 1];
            return true;
        }
    }
};

// Shared-memory staging of one batch of A entries: base of the B row (made
// relative to the batch's product index), the carried A word (int64 plus-times:
// the A value; KIND 3, ordered float64 with deferred hits: the A position),
// and the inclusive product end.  Bytes per group.
__host__ __device__ constexpr bool carries_a(int kind) { return kind == 1 || kind == 3; }
__host__ __device__ constexpr size_t batch_bytes_rt(int gw, int kind) {
    return kind == 2 ? 0 : (size_t)gw * 32 * ((carries_a(kind) ? 16 : 8) + 4);
}
template <int GW, int KIND>
__host__ __device__ constexpr size_t batch_bytes() {
    return batch_bytes_rt(GW, KIND);
}

struct BatchSmem {
    int32_t* incl;
    long long* base;
    long long* av;
};

template <int GW, int KIND>
__device__ __forceinline__ BatchSmem bind_batch(unsigned char* bbase) {
    constexpr int GT = GW * 32;
    BatchSmem bsm;
    bsm.base = (long long*)bbase;
    bsm.av = bsm.base + GT;
    bsm.incl = (int32_t*)(bbase + (size_t)GT * (carries_a(KIND) ? 16 : 8));
    return bsm;
}

// The last, partial chunk of a long B segment: V predicated loads per lane.
template <int V, class PR>
__device__ __forceinline__ void tail_chunk(const Prob& p, PR& pr, const int32_t* bp, int c, int n0, long long a0,
                                           long long b0, int lane32) {
    int32_t jj[V];
    long long aa[V], ss[V];
#pragma unroll
    for (int u = 0; u < V; u++) {
        const int o = c + 32 * u + lane32;
        jj[u] = o < n0 ? __ldg(bp + o) : EMPTY_KEY;
        aa[u] = a0;
        ss[u] = b0 + o;
    }
    pr.template put_batch<V>(jj, aa, ss);
}

// Order-free accumulation (plus-pair counts, int64 sums) over the row's
// flattened product space, batch by batch (NB = GT entries of A_i):
//   1. thread gt loads A entry tb0+gt (base of its B row, length); a
//      group-wide scan gives every product q of the batch the B slot
//      base[l] + q of the entry l with incl[l-1] <= q < incl[l];
//   2. warp w owns the contiguous product range [w P/GW, (w+1) P/GW)
//      (equal work per warp) and walks the entries overlapping it,
//      32 at a time, one per lane:
//        portions >= 32 products: warp-wide chunks of 32*U loads
//        (U independent loads in flight per lane), no search;
//        shorter portions: flattened into 32-wide windows, the owning
//        lane found by a shuffle binary search.
//   Every lane calls pr.put(j, a, s) with j = EMPTY_KEY when it has no
//   product (the policy may use warp collectives).
//   [c_lo, c_hi): only products with a column in this range (a sub-range of
//   each sorted B row, by binary search); the default is every product.
//
//   KIND 3 carries the A position t in the `a` word instead of a value.
//   SEARCH (plain masks): an A entry whose B row is much longer than the
//   mask part [srch_m, srch_m + srch_nm) makes nm·log2(len) probes instead
//   of len — each mask column is binary-searched in B_k, and only the columns
//   found are handed to pr (the same products the scan would keep: the
//   evaluated set, counts and sums are unchanged).  R-MAT hubs: a 10^5-entry
//   B row meets mask rows of a few hundred columns (cfg5).
#ifndef MM_SEARCH_RATIO
#define MM_SEARCH_RATIO 1   // search when len > RATIO/DEN * nm * ceil(log2(len + 1))
#endif
#ifndef MM_SEARCH_DEN
#define MM_SEARCH_DEN 1
#endif
#ifndef MM_SEARCH_U
#define MM_SEARCH_U 2
#endif
//   cur (column-range mode over consecutive ranges of one row): cur[t - as]
//   holds where A entry t's B row reached at the end of the previous range,
//   so a range starts there (no search) and ends by a galloping search.
template <int GW, int KIND, class PR, bool SEARCH = false>
__device__ __forceinline__ void flat_products(const Prob& p, PR& pr, int64_t as, int64_t ae, int gt,
                                              int bar_id, int* s_warp, BatchSmem bsm,
                                              int32_t c_lo = INT32_MIN, int32_t c_hi = INT32_MAX,
                                              const int32_t* srch_m = nullptr, int64_t srch_nm = 0,
                                              int64_t* cur = nullptr) {
    constexpr int GT = GW * 32;
#ifndef MM_PRODUCT_UNROLL
#define MM_PRODUCT_UNROLL 4
#endif
#ifndef MM_WIDE_UNROLL
#define MM_WIDE_UNROLL 8   // 16/32-warp groups: more loads in flight (cfg5 424 -> 406 ms)
#endif
    constexpr int U = GW >= 16 ? MM_WIDE_UNROLL : MM_PRODUCT_UNROLL;   // independent B loads in flight per lane
    constexpr int CH = 32 * U;
    constexpr int NB = GT;
    constexpr bool CARRY = carries_a(KIND);
    const int lane32 = gt & 31;
    for (int64_t tb0 = as; tb0 < ae; tb0 += NB) {
        const int64_t t = tb0 + gt;
        long long base = 0, av = 0;
        int len = 0;
        if (t < ae) {
            const int32_t k = p.a_idx[t];
            base = p.b_ptr[k];
            int64_t end = p.b_ptr[k + 1];
            if (cur) {
                if (c_lo != INT32_MIN) base = cur[t - as];
                if (c_hi != INT32_MAX) {
                    end = gallop_lower_bound(p.b_idx, base, end, c_hi);
                    cur[t - as] = end;
                }
            } else {
                if (c_lo != INT32_MIN) base = lower_bound_range(p.b_idx, base, end, c_lo);
                if (c_hi != INT32_MAX) end = lower_bound_range(p.b_idx, base, end, c_hi);
            }
            len = (int)(end - base);
            if (KIND == 1) av = ((const long long*)p.a_val)[t];
            if (KIND == 3) av = t;
        }
        bool srch = false;
        if (SEARCH && len > 0) {
            const int lg = 32 - __clz(len);          // ceil(log2(len + 1))
            srch = (long long)len * MM_SEARCH_DEN > srch_nm * lg * MM_SEARCH_RATIO;
        }
        const int flen = srch ? 0 : len;             // scanned products of this entry
        int tot;
        const int incl = group_incl_scan<GW>(flen, &tot, s_warp, bar_id, gt);
        int q_lo = 0, q_hi = tot;
        int l_lo = 0, l_end = NB;
        if (GW > 1) {
            bsm.incl[gt] = incl;
            bsm.base[gt] = base - (incl - flen);
            if (CARRY) bsm.av[gt] = av;
            group_bar(bar_id, GT);
            const int wg = gt >> 5;
            q_lo = (int)(((long long)tot * wg) / GW);
            q_hi = (int)(((long long)tot * (wg + 1)) / GW);
            int lo = 0, hi = NB - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (bsm.incl[mid] <= q_lo) lo = mid + 1; else hi = mid;
            }
            l_lo = lo;
            hi = NB - 1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (bsm.incl[mid] < q_hi) lo = mid + 1; else hi = mid;
            }
            l_end = lo + 1;
        }
        for (int l0 = l_lo; l0 < l_end && q_lo < q_hi; l0 += 32) {
            const int l = l0 + lane32;
            long long sb = 0, sa = 0;
            int plen = 0;
            if (GW == 1) {
                sb = base;
                plen = flen;
                sa = av;
            } else if (l < l_end) {
                const int e_in = bsm.incl[l];
                const int e_ex = l > 0 ? bsm.incl[l - 1] : 0;
                const int a0 = e_ex > q_lo ? e_ex : q_lo;
                const int a1 = e_in < q_hi ? e_in : q_hi;
                plen = a1 > a0 ? a1 - a0 : 0;
                sb = bsm.base[l] + a0;
                if (CARRY) sa = bsm.av[l];
            }
            unsigned longm = __ballot_sync(FULL, plen >= 32);
            while (longm) {
                const int src = __ffs(longm) - 1;
                longm &= longm - 1;
                const long long b0 = shfl64(sb, src);
                const int n0 = __shfl_sync(FULL, plen, src);
                const long long a0 = CARRY ? shfl64(sa, src) : 0;
#ifdef MM_STAGE_TMA
                if (n0 >= MM_STAGE_MIN && stage_available()) {
                    stage_segment(p, pr, b0, n0, a0, lane32);
                    continue;
                }
#endif
                const int32_t* bp = p.b_idx + b0;
                int c = 0;
                for (; c + CH <= n0; c += CH) {   // full chunks: no bounds predicates
                    int32_t jj[U];
                    long long aa[U], ss[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int o = c + 32 * u + lane32;
                        jj[u] = __ldg(bp + o);
                        aa[u] = a0;
                        ss[u] = b0 + o;
                    }
                    pr.template put_batch<U>(jj, aa, ss);
                }
                if (n0 - c > 32 * U / 2) {        // tail: as many loads as it needs
                    tail_chunk<U>(p, pr, bp, c, n0, a0, b0, lane32);
                } else if (n0 - c > 32) {
                    tail_chunk<U / 2>(p, pr, bp, c, n0, a0, b0, lane32);
                } else if (c < n0) {
                    tail_chunk<1>(p, pr, bp, c, n0, a0, b0, lane32);
                }
            }
            const int slen = plen < 32 ? plen : 0;
            const int sincl = warp_incl_scan(slen, lane32);
            const int stot = __shfl_sync(FULL, sincl, 31);
            if (stot > 0) {
#ifndef MM_OWNER_BALLOT
                const int sexcl = sincl - slen;
                for (int w0 = 0; w0 < stot; w0 += 64) {
                    int32_t jj[2];
                    long long ss[2], aa[2];
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const int q = w0 + 32 * u + lane32;
                        const int own = owner_of(sincl, q < stot ? q : stot - 1);
                        ss[u] = shfl64(sb, own) + (q - __shfl_sync(FULL, sexcl, own));
                        aa[u] = CARRY ? shfl64(sa, own) : 0;
                        jj[u] = q < stot ? __ldg(p.b_idx + ss[u]) : EMPTY_KEY;
                    }
                    pr.template put_batch<2>(jj, aa, ss);
                }
#else
                // Owner of each flattened product without a search: the
                // non-empty short segments are compacted into lanes 0..ns-1
                // (segment c starts at product c_ex, B slot = c_rel + q).  In
                // the 32-product window at wb, c0 = the segment holding product
                // wb (a ballot), and the segments starting inside the window
                // set bit (start - wb) of S (one REDUX); the owner of product
                // wb + lane is c0 + popc(S & bits[0..lane]).
                const int sexcl = sincl - slen;
                const unsigned nz = __ballot_sync(FULL, slen > 0);
                const int ns = __popc(nz);
                const int src = lane32 < ns ? (int)__fns(nz, 0, lane32 + 1) : 0;
                const long long c_rel = shfl64(sb - sexcl, src);
                const int ex = __shfl_sync(FULL, sexcl, src);
                const int c_ex = lane32 < ns ? ex : 0x7fffffff;
                const long long c_a = CARRY ? shfl64(sa, src) : 0;
                const unsigned upto = 0xffffffffu >> (31 - lane32);
                for (int w0 = 0; w0 < stot; w0 += 64) {
                    int32_t jj[2];
                    long long ss[2], aa[2];
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        const int wb = w0 + 32 * u;
                        const int c0 = __popc(__ballot_sync(FULL, c_ex <= wb)) - 1;
                        const unsigned starts =
                            __reduce_or_sync(FULL, (c_ex > wb && c_ex < wb + 32) ? 1u << (c_ex - wb) : 0u);
                        const int own = c0 + __popc(starts & upto);
                        const int q = wb + lane32;
                        ss[u] = shfl64(c_rel, own) + q;
                        aa[u] = CARRY ? shfl64(c_a, own) : 0;
                        jj[u] = q < stot ? __ldg(p.b_idx + ss[u]) : EMPTY_KEY;
                    }
                    pr.template put_batch<2>(jj, aa, ss);
                }
#endif
            }
            if (GW == 1) break;
        }
        pr.drain();
        if (GW > 1) group_bar(bar_id, GT);
        if (SEARCH) {
            int ntot;
            const int sincl = group_incl_scan<GW>(srch ? 1 : 0, &ntot, s_warp, bar_id, gt);
            if (ntot > 0) {                           // group-uniform
                if (srch) {
                    bsm.base[sincl - 1] = base;
                    bsm.incl[sincl - 1] = len;
                    if (CARRY) bsm.av[sincl - 1] = av;
                }
                if (GW > 1) group_bar(bar_id, GT); else __syncwarp();
                // SU interleaved branch-free lower bounds per lane: their
                // dependent load chains overlap
                constexpr int SU = MM_SEARCH_U;
                const long long total = (long long)ntot * srch_nm;
                for (long long w0 = 0; w0 < total; w0 += (long long)GT * SU) {
                    int32_t jj[SU];
                    long long aa[SU], ss[SU];
                    const int32_t* bb[SU];
                    int nn[SU];
#pragma unroll
                    for (int u = 0; u < SU; u++) {
                        const long long idx = w0 + (long long)u * GT + gt;
                        jj[u] = EMPTY_KEY;
                        aa[u] = 0;
                        ss[u] = 0;
                        bb[u] = p.b_idx;
                        nn[u] = 0;
                        if (idx < total) {
                            const int item = (int)(idx / srch_nm);
                            jj[u] = srch_m[idx - (long long)item * srch_nm];
                            ss[u] = bsm.base[item];
                            bb[u] = p.b_idx + ss[u];
                            nn[u] = bsm.incl[item];
                            if (CARRY) aa[u] = bsm.av[item];
                        }
                    }
                    const int32_t* b0[SU];
#pragma unroll
                    for (int u = 0; u < SU; u++) b0[u] = bb[u];
                    bool more = true;
                    while (more) {
                        more = false;
#pragma unroll
                        for (int u = 0; u < SU; u++) {
                            if (nn[u] > 1) {
                                const int half = nn[u] >> 1;
                                // last entry <= j (the B row is strictly increasing)
                                bb[u] = __ldg(bb[u] + half) <= jj[u] ? bb[u] + half : bb[u];
                                nn[u] -= half;
                                more |= nn[u] > 1;
                            }
                        }
                    }
#pragma unroll
                    for (int u = 0; u < SU; u++) {
                        // nn == 1: bb = the last entry <= j (or the first entry); nn == 0: no product
                        const bool hit = nn[u] == 1 && __ldg(bb[u]) == jj[u];
                        ss[u] += bb[u] - b0[u];
                        if (!hit) jj[u] = EMPTY_KEY;
                    }
                    pr.template put_batch<SU>(jj, aa, ss);
                }
                pr.drain();
                if (GW > 1) group_bar(bar_id, GT); else __syncwarp();
            }
        }
    }
}

// Ordered float64 accumulation for one warp.  The reference folds a slot's
// products in ascending k, the first product stored rather than added to 0.0
// (_kernels.py:48-65); every GPU float64 path keeps that order, so results are
// bit-identical to the reference's MSA/Hash/MCA/Inner.
//
// The warp walks the row's product space flattened in (k, s) order, 32
// consecutive products per window (owner A entry of each lane found by a
// shuffle binary search), so short B rows do not idle lanes.  Windows are
// processed in order; inside a window, lanes whose products land on the same
// slot (two k's hitting one column) fold one after another in lane order
// (__match_any_sync ranks them), everyone else folds at once.
// loc.locate(j) -> slot or -1 (masked out); loc.fold(slot, prod); loc.mark(slot).
//
// Groups of several warps split a heavy row by OUTPUT COLUMN: a warp takes
// only the products with column in [c_lo, c_hi) (each B row is sorted, so
// its share of B_k is a sub-range found by two binary searches).  Every slot
// then belongs to exactly one warp, which still folds it in ascending k: the
// parallelism is across slots, the order inside a slot is untouched.
template <bool NUMERIC, class LOC>
__device__ __forceinline__ unsigned ordered_products_f64(const Prob& p, LOC& loc, int64_t as, int64_t ae,
                                                         int lane, int32_t c_lo = INT32_MIN,
                                                         int32_t c_hi = INT32_MAX) {
    const bool split = c_lo != INT32_MIN || c_hi != INT32_MAX;
    const double* av_p = (const double*)p.a_val;
    const double* bv_p = (const double*)p.b_val;
    unsigned evaluated = 0;
    for (int64_t tb0 = as; tb0 < ae; tb0 += 32) {
        const int64_t t = tb0 + lane;
        int64_t bs = 0;
        int len = 0;
        double av = 0.0;
        if (t < ae) {
            const int32_t k = p.a_idx[t];
            bs = p.b_ptr[k];
            int64_t be = p.b_ptr[k + 1];
            if (split) {
                if (c_lo != INT32_MIN) bs = lower_bound_range(p.b_idx, bs, be, c_lo);
                if (c_hi != INT32_MAX) be = lower_bound_range(p.b_idx, bs, be, c_hi);
            }
            len = (int)(be - bs);
            av = av_p[t];
        }
        const int incl = warp_incl_scan(len, lane);
        const int tot = __shfl_sync(FULL, incl, 31);
        const int excl = incl - len;
        for (int w0 = 0; w0 < tot; w0 += 32) {
            const int q = w0 + lane;
            const int own = owner_of(incl, q < tot ? q : tot - 1);
            const int64_t s = shfl64(bs, own) + (q - __shfl_sync(FULL, excl, own));
            const double a = __shfl_sync(FULL, av, own);
            const int h = q < tot ? loc.locate(p.b_idx[s]) : -1;
            const bool hit = h >= 0;
            evaluated += hit;
            const unsigned hm = __ballot_sync(FULL, hit);
            if (!hm) continue;
            if (NUMERIC) {
                const double prod = hit ? a * bv_p[s] : 0.0;
                const unsigned same = __match_any_sync(FULL, hit ? h : -2 - lane);
                const int myrank = __popc(same & lanemask_lt());
                const int rounds = __reduce_max_sync(FULL, hit ? myrank : 0);
                for (int r = 0; r <= rounds; r++) {
                    if (hit && myrank == r) loc.fold(h, prod);
                    __syncwarp();
                }
            } else if (hit) {
                loc.mark(h);
            }
            __syncwarp();
        }
    }
    return evaluated;
}

}  // namespace mm
