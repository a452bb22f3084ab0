// Push path, ordered float64 rows with deferred hits (plain masks, one warp
// per row, short mask rows).
//
// Reference order (_kernels.py:48-65, 166-190, 292-305): a slot's products
// fold in ascending k, the first product stored rather than added to 0.0.
// The in-order window walk (product_loop.cuh ordered_products_f64) keeps that
// order by construction but pays ~160 instructions per 32 products (owner
// search, rank search, one window at a time).  Masked rows of sparse
// products hit the mask rarely (cfg3: 4,079 of 67 M products at d16), so
// here the ORDER is restored after the fact:
//
//   1. the mask row M_i is copied to shared memory and summarised by a
//      16384-bit filter (word (j phi) >> 23, bit (j phi) mod 32 set for every mask column j);
//   2. products are enumerated with few instructions: the lanes of an A
//      entry (32 / nextpow2(entries) of them for short A rows) walk its B row
//      (4 independent loads per step) — no owner search — and B rows of 64+
//      entries are walked warp-wide, coalesced; each column
//      is tested against the filter (one shared load); a filter hit is
//      resolved by binary search in the mask row (its mask rank = the
//      output slot), and a true hit appends (rank, t, a_t * b_s) to the
//      warp's hit list (warp-aggregated; B values read only for hits);
//   3. the hits fold into their rank slots in ascending t (each hit's order
//      among the hits of its slot, then rounds: order 0 stores) — the
//      reference's ascending-k order, bit for bit;
//   4. the distinct hit slots are the row's entries, emitted in rank order =
//      mask order (_kernels.py:78-85, 308-313); the filter words are reset.
//
// A row with more hits than the list holds is redone with the in-order walk
// over the same slots, so results never depend on the list capacity.
#pragma once
#include "analyze.cuh"
#include "common.cuh"
#include "fused_tail.cuh"
#include "product_loop.cuh"

namespace mm {

#ifndef MM_DEFER_CAP
#define MM_DEFER_CAP 128   // hits per warp list
#endif
constexpr int DEFER_CAP = MM_DEFER_CAP;
constexpr int DEFER_FILTER_LG = 14;   // filter bits (log2)
constexpr int DEFER_LONG = 64;        // B rows walked warp-wide from this length

// Per-warp shared bytes for mask rows of up to nm_max entries: filter,
// mask copy, slot values and flags, hit list (rank, t, value).
__host__ __device__ constexpr size_t defer_warp_bytes(int nm_max) {
    return ((size_t)1 << (DEFER_FILTER_LG - 3)) + (((size_t)nm_max * 4 + 15) & ~(size_t)15) +
           (size_t)nm_max * 8 + (((size_t)nm_max * 4 + 15) & ~(size_t)15) + (size_t)DEFER_CAP * 16;
}

struct DeferWarp {
    uint32_t* filter;   // 2^DEFER_FILTER_LG bits
    int32_t* mrow;      // mask row copy
    double* vals;       // slot values by mask rank
    int32_t* cnt;       // slot flags by mask rank
    double* h_val;
    int32_t* h_rank;
    int32_t* h_t;
    __device__ __forceinline__ void bind(unsigned char* base, int nm_max) {
        filter = (uint32_t*)base;
        mrow = (int32_t*)(base + ((size_t)1 << (DEFER_FILTER_LG - 3)));
        vals = (double*)((unsigned char*)mrow + (((size_t)nm_max * 4 + 15) & ~(size_t)15));
        cnt = (int32_t*)(vals + nm_max);
        h_val = (double*)((unsigned char*)cnt + (((size_t)nm_max * 4 + 15) & ~(size_t)15));
        h_rank = (int32_t*)(h_val + DEFER_CAP);
        h_t = h_rank + DEFER_CAP;
    }
};

// Filter bit of column j: word (j phi) >> 23 of the 512, bit (j phi) mod 32
// (the funnel-shift amount, so the test needs no second shift).
__device__ __forceinline__ uint32_t defer_bit(int32_t j) {
    const uint32_t h = (uint32_t)j * FIB_MULT;
    return ((h >> (32 - DEFER_FILTER_LG + 5)) << 5) | (h & 31u);
}

// rank of j in the sorted mask row m[0..nm) or -1 (branch-free lower bound)
__device__ __forceinline__ int defer_rank(const int32_t* m, int nm, int32_t j) {
    int lo = 0, n = nm;
    while (n > 1) {
        const int half = n >> 1;
        lo = m[lo + half] <= j ? lo + half : lo;
        n -= half;
    }
    return (nm > 0 && m[lo] == j) ? lo : -1;
}

// In-order fallback locator (ordered_products_f64) over the same slots.
struct DeferLocatorF64 {
    DeferWarp w;
    int nm;
    __device__ __forceinline__ int locate(int32_t j) {
        const uint32_t b = defer_bit(j);
        if (!((w.filter[b >> 5] >> (b & 31)) & 1u)) return -1;
        return defer_rank(w.mrow, nm, j);
    }
    __device__ __forceinline__ void fold(int h, double prod) {
        if (w.cnt[h] == 0) {
            w.vals[h] = prod;
            w.cnt[h] = 1;
        } else {
            w.vals[h] += prod;
        }
    }
    __device__ __forceinline__ void mark(int h) { w.cnt[h] = 1; }
};

// Products of one warp-step: j[u] (EMPTY_KEY = none) from A position t, B
// position s0 + u * stride.  Filter test (one shared load: the word holding
// bit h = (j phi) >> 20, tested by a wrapping funnel shift), rank search on
// a filter hit, append.
template <int U>
__device__ __forceinline__ void defer_probe(const Prob& p, const DeferWarp& w, uint32_t filter_s, int nm,
                                            const int32_t* j, int64_t t, int64_t s0, int stride, int64_t as,
                                            int& count, unsigned& evaluated) {
    bool maybe[U];
    bool any = false;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint32_t h = (uint32_t)j[u] * FIB_MULT;
        uint32_t word, rot;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(word) : "r"(filter_s + ((h >> (32 - DEFER_FILTER_LG + 5)) << 2)));
        asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(rot) : "r"(word), "r"(h));
        maybe[u] = (rot & 1u) && j[u] >= 0;
        any |= maybe[u];
    }
    if (!__any_sync(FULL, any)) return;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int r = maybe[u] ? defer_rank(w.mrow, nm, j[u]) : -1;
        const bool hit = r >= 0;
        const unsigned bal = __ballot_sync(FULL, hit);
        if (bal) {
            const int pos = count + __popc(bal & lanemask_lt());
            if (hit) {
                evaluated++;
                if (pos < DEFER_CAP) {
                    w.h_rank[pos] = r;
                    w.h_t[pos] = (int32_t)(t - as);
                    w.h_val[pos] = ((const double*)p.a_val)[t] * ((const double*)p.b_val)[s0 + u * stride];
                }
            }
            count += __popc(bal);
        }
    }
}

// Short B rows: the L lanes of an A entry take positions sub, sub + L, ...
// of its row (len entries), 4 per step; L is a compile-time stride, so every
// load is one LDG with an immediate offset.
template <int L>
__device__ __forceinline__ void defer_walk(const Prob& p, const DeferWarp& w, uint32_t filter_s, int nm, int64_t bs,
                                           int sub, int len, int steps, int64_t t, int64_t as, int& count,
                                           unsigned& evaluated) {
    const int32_t* bp = p.b_idx + bs + sub;
    int rem = len - sub;            // positions left for this lane (from the current step)
    for (int o = 0; o < steps; o += 4 * L) {
        int32_t jj[4];
#pragma unroll
        for (int u = 0; u < 4; u++) jj[u] = u * L < rem ? __ldg(bp + u * L) : EMPTY_KEY;
        defer_probe<4>(p, w, filter_s, nm, jj, t, bs + sub + o, L, as, count, evaluated);
        bp += 4 * L;
        rem -= 4 * L;
    }
}

// Fold the warp's hit list (n hits) into the rank slots in ascending t per
// slot, then emit the row straight from the list: the distinct slots are the
// row's output entries, in rank (= mask) order.  Returns the entry count;
// only the slots used are touched, so nothing proportional to nm remains.
template <bool NUMERIC>
__device__ __forceinline__ int defer_fold_emit(int n, const DeferWarp& w, const Out& o, int64_t w0, int lane) {
    constexpr int PER = DEFER_CAP / 32;
    int slot[PER], order[PER];
    double v[PER];
    int maxr = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int e = q * 32 + lane;
        slot[q] = -1;
        order[q] = 0;
        v[q] = 0.0;
        if (e < n) {
            slot[q] = w.h_rank[e];
            v[q] = w.h_val[e];
            const int t = w.h_t[e];
            int r = 0;
            for (int f = 0; f < n; f++) r += (w.h_rank[f] == slot[q]) & (w.h_t[f] < t);
            order[q] = r;
            maxr = max(maxr, r);
        }
    }
    maxr = __reduce_max_sync(FULL, maxr);
    if (NUMERIC) {
        for (int r = 0; r <= maxr; r++) {
#pragma unroll
            for (int q = 0; q < PER; q++) {
                if (slot[q] >= 0 && order[q] == r) {
                    if (r == 0) w.vals[slot[q]] = v[q];
                    else w.vals[slot[q]] += v[q];
                }
            }
            __syncwarp();
        }
    }
    // output position of a slot = distinct slots below it = order-0 hits below it
    __syncwarp();
#pragma unroll
    for (int q = 0; q < PER; q++)
        if (q * 32 + lane < n) w.h_t[q * 32 + lane] = order[q];   // reuse: h_t := order
    __syncwarp();
    int distinct = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const bool first = slot[q] >= 0 && order[q] == 0;
        distinct += first;
        if (NUMERIC && first) {
            int pos = 0;
            for (int f = 0; f < n; f++) pos += (w.h_t[f] == 0) & (w.h_rank[f] < slot[q]);
            o.idx[w0 + pos] = w.mrow[slot[q]];
            ((double*)o.val)[w0 + pos] = w.vals[slot[q]];
        }
    }
    return (int)warp_sum_ll(distinct);
}

// One warp per row of one bin (rows fetched dynamically); nm_max: the bin's
// largest mask row (<= F64D_MAX_NM).
// Direct mode (flops_cap > 0; wk.rows == nullptr: every row, no analysis
// pass before it): the kernel also sums generated_flops and the empty rows
// into o.gen_flops / o.empty_rows, and a row whose mask exceeds nm_max or
// whose products exceed flops_cap raises o.overflow (the host then runs the
// binned path instead).
//
// TAIL: the last block also runs the fused tail (fused_tail.cuh: scan,
// compaction and the counters written to mapped host memory).
constexpr int64_t DIRECT_MAX_NA = 1024;

template <bool NUMERIC, bool TAIL = false>
__global__ void __launch_bounds__(256, 4) k_push_f64_defer(Prob p, Out o, Work wk, int nm_max, long long flops_cap,
                                                           Tail tail) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    DeferWarp w;
    w.bind(smem + (size_t)warp * defer_warp_bytes(nm_max), nm_max);
    for (int e = lane; e < (1 << (DEFER_FILTER_LG - 5)); e += 32) w.filter[e] = 0u;
    for (int e = lane; e < nm_max; e += 32) w.cnt[e] = 0;
    __syncwarp();
    const uint32_t filter_s = (uint32_t)__cvta_generic_to_shared(w.filter);
    unsigned long long evaluated = 0, gen = 0;
    int empty = 0;
    RowFetcher<1> rf;
    // few rows per warp: one row per fetch, so no warp serialises several
    // rows' latency chains while others idle
    if (wk.count < 4 * (int)(gridDim.x * (blockDim.x >> 5))) rf.per = 1;
    RowInfo ri;
    while (rf.next(p, wk, lane, 0, nullptr, ri)) {
        const int64_t ms = ri.ms;
        const int nm = (int)(ri.me - ms);
        // direct mode: wide mask rows, and rows with so many A entries that one
        // warp would walk them for milliseconds just to count their products
        // (R-MAT hubs under a nearly empty mask: a batched-BC backward step),
        // go to the binned pass, whose analysis takes a block per long row
        if (flops_cap && (nm > nm_max || ri.ae - ri.as > DIRECT_MAX_NA)) {
            if (lane == 0) {
                atomicExch(o.overflow, 1);
                o.row_nnz[ri.i] = -1;   // left to the binned pass
            }
            continue;
        }
        long long rf_lane = 0;   // direct mode: this lane's share of the row's products
        // 1. mask copy + filter
        for (int r = lane; r < nm; r += 32) {
            const int32_t j = p.m_idx[ms + r];
            w.mrow[r] = j;
            const uint32_t b = defer_bit(j);
            atomicOr(&w.filter[b >> 5], 1u << (b & 31));
        }
        __syncwarp();
        // 2. products -> hit list
        int nh = 0;
        unsigned ev = 0;
        for (int64_t tb0 = ri.as; tb0 < ri.ae; tb0 += 32) {
            // a batch of cnt <= 32 A entries; with cnt <= 16 every entry gets
            // L = 32 / nextpow2(cnt) lanes, lane sub of an entry taking its B
            // row's positions sub, sub + L, ... (the lanes stay busy)
            const int cnt = ri.ae - tb0 < 32 ? (int)(ri.ae - tb0) : 32;
            const int glg = 32 - __clz(cnt - 1);          // ceil(log2(cnt)), cnt >= 1
            const int entry = lane & ((1 << glg) - 1);
            const int sub = lane >> glg;
            const int L = 32 >> glg;
            const int64_t t = tb0 + entry;
            int64_t bs = 0;
            int len = 0;
            if (entry < cnt) {
                const int32_t k = p.a_idx[t];
                bs = p.b_ptr[k];
                len = (int)(p.b_ptr[k + 1] - bs);
            }
            if (sub == 0) rf_lane += len;
            // direct mode: an empty mask row (never launched by the binned path)
            // only has its flops counted
            if (nm == 0) continue;
            // long B rows: the warp walks them, coalesced, 4 loads in flight
            unsigned longm = __ballot_sync(FULL, sub == 0 && len >= DEFER_LONG);
            while (longm) {
                const int src = __ffs(longm) - 1;
                longm &= longm - 1;
                const int64_t b0 = shfl64(bs, src);
                const int n0 = __shfl_sync(FULL, len, src);
                const int64_t t0 = tb0 + src;
                const int32_t* bp = p.b_idx + b0 + lane;
                for (int c = 0; c < n0; c += 128) {
                    int32_t jj[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) jj[u] = c + 32 * u + lane < n0 ? __ldg(bp + c + 32 * u) : EMPTY_KEY;
                    defer_probe<4>(p, w, filter_s, nm, jj, t0, b0 + c + lane, 32, ri.as, nh, ev);
                }
            }
            // short B rows: the entry's lanes walk its row
            const int mine = len < DEFER_LONG ? len : 0;
            const int steps = __reduce_max_sync(FULL, mine);
            switch (L) {
                case 1: defer_walk<1>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
                case 2: defer_walk<2>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
                case 4: defer_walk<4>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
                case 8: defer_walk<8>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
                case 16: defer_walk<16>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
                default: defer_walk<32>(p, w, filter_s, nm, bs, sub, mine, steps, t, ri.as, nh, ev); break;
            }
        }
        __syncwarp();
        // 3. ordered fold and emit from the hit list, or (list overflow) the
        // in-order walk into the slots and a gather in mask order
        if (flops_cap) {
            const long long rflops = warp_sum_ll(rf_lane);
            if (rflops <= flops_cap) {   // rows left to the binned pass are counted there
                gen += rflops;
                empty += (rflops == 0 || nm == 0);
            }
            if (rflops > flops_cap) {
                if (lane == 0) {
                    atomicExch(o.overflow, 1);
                    o.row_nnz[ri.i] = -1;   // left to the binned pass
                }
                for (int r = lane; r < nm; r += 32) w.filter[defer_bit(w.mrow[r]) >> 5] = 0u;
                __syncwarp();
                continue;
            }
        }
        const int64_t w0 = NUMERIC ? o.off[ri.i] : 0;
        int running = 0;
        if (nh <= DEFER_CAP) {
            evaluated += ev;
            if (nh) running = defer_fold_emit<NUMERIC>(nh, w, o, w0, lane);
        } else {
            DeferLocatorF64 loc{w, nm};
            evaluated += ordered_products_f64<NUMERIC>(p, loc, ri.as, ri.ae, lane);
            __syncwarp();
            for (int rb = 0; rb < nm; rb += 32) {
                const int r = rb + lane;
                const bool set = r < nm && w.cnt[r] > 0;
                const unsigned bal = __ballot_sync(FULL, set);
                if (NUMERIC && set) {
                    const int64_t d = w0 + running + __popc(bal & lanemask_lt());
                    o.idx[d] = w.mrow[r];
                    ((double*)o.val)[d] = w.vals[r];
                }
                running += __popc(bal);
            }
            __syncwarp();
            for (int r = lane; r < nm; r += 32) w.cnt[r] = 0;
        }
        if (lane == 0) o.row_nnz[ri.i] = running;
        // reset the filter words of the mask row
        for (int r = lane; r < nm; r += 32) w.filter[defer_bit(w.mrow[r]) >> 5] = 0u;
        __syncwarp();
    }
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if (lane == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
    if (flops_cap && lane == 0) {
        if (gen) atomicAdd(o.gen_flops, gen);
        if (empty) atomicAdd(o.empty_rows, empty);
    }
    if (TAIL) fused_tail(tail, (int*)smem);
}

}  // namespace mm
