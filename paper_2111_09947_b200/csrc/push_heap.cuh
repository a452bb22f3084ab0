// Push path, heap accumulator: a warp-cooperative k-way merge of B rows.
//
// Reference: heap_numeric / heap_symbolic with _heap_push / _heap_pop /
// _heap_insert (_kernels.py:351-512) — a binary min-heap of B-row iterators
// keyed by their current column; popped columns are matched against the mask
// cursor (advanced monotonically), equal columns combined, the complement form
// keeps columns NOT in the mask; NInspect in {0, 1, inf} lets an iterator skip
// entries that cannot match before it is (re)inserted (Alg. 5).
//
// GPU form: one warp per row; up to 32 iterators at a time, one per lane
// (one per A entry of the batch).  The heap's pop-min becomes a single
// __reduce_min_sync over the lane heads; every lane whose head equals the
// minimum contributes (a __ballot_sync gives them in ascending-k order, so a
// float64 slot folds exactly like the reference MSA order) and advances.
// Plain masks: the mask cursor advances 32 entries per step with a ballot;
// results land in mask-rank slots, so batches of 32 iterators accumulate
// into the same slots.  Complement rows with at most 32 A entries emit their
// sorted columns directly; longer complement rows run on the hash kernels.
// NInspect: 1 skips, on advance, B entries below the mask cursor; inf skips
// every entry absent from the mask row (binary search), 0 inspects nothing.
// Outputs are identical for all three; only the work differs.
#pragma once
#include "analyze.cuh"
#include "common.cuh"

namespace mm {

constexpr uint32_t HEAP_DONE = 0x7fffffffu;

// first mask position >= c, starting at cursor (warp-uniform result)
__device__ __forceinline__ int64_t mask_advance(const int32_t* m, int64_t cur, int64_t nm, int32_t c, int lane) {
    for (;;) {
        const int64_t q = cur + lane;
        const bool below = q < nm && m[q] < c;
        const unsigned bal = __ballot_sync(FULL, below);
        const int n = __popc(bal);
        cur += n;
        if (n < 32) return cur;
    }
}

template <int KIND, bool NUMERIC, bool COMP>
__global__ void __launch_bounds__(256) k_push_heap(Prob p, Out o, Work wk, int nm_max, int ninspect,
                                                   unsigned char* gslab) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const size_t wbytes = COMP ? 0 : (((size_t)(KIND == 0 ? 4 : 12) * nm_max + 15) & ~(size_t)15);
    unsigned char* region = gslab ? gslab + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * wbytes
                                  : smem + (size_t)warp * wbytes;
    unsigned long long* sval = (unsigned long long*)region;
    int32_t* scnt = (int32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)nm_max));
    unsigned long long evaluated = 0;
    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(wk.cursor, 1);
        r = __shfl_sync(FULL, r, 0);
        if (r >= wk.count) break;
        const int64_t i = wk.rows[r];
        const int64_t as = p.a_ptr[i], ae = p.a_ptr[i + 1];
        const int64_t ms = p.m_ptr[i], me = p.m_ptr[i + 1], nm = me - ms;
        const int32_t* m = p.m_idx + ms;
        const int64_t w0 = NUMERIC ? o.off[i] : 0;
        int64_t n_out = 0;
        if (!COMP) {
            for (int64_t q = lane; q < nm; q += 32) {
                scnt[q] = 0;
                if (KIND == 1) sval[q] = 0ull;
            }
            __syncwarp();
        }
        for (int64_t tb0 = as; tb0 < ae; tb0 += 32) {
            const int64_t t = tb0 + lane;
            int64_t pos = 0, end = 0;
            long long a_i = 0;
            double a_d = 0.0;
            if (t < ae) {
                const int32_t k = p.a_idx[t];
                pos = p.b_ptr[k];
                end = p.b_ptr[k + 1];
                if (KIND == 1) a_i = ((const long long*)p.a_val)[t];
                if (KIND == 2) a_d = ((const double*)p.a_val)[t];
            }
            int64_t mcur = 0;
            // NInspect = inf (HeapDot): an iterator only ever sits on mask columns
            if (!COMP && ninspect < 0)
                while (pos < end && !contains_sorted(m, nm, p.b_idx[pos])) pos++;
            uint32_t head = pos < end ? (uint32_t)p.b_idx[pos] : HEAP_DONE;
            for (;;) {
                const uint32_t c = __reduce_min_sync(FULL, head);
                if (c == HEAP_DONE) break;
                const bool mine = head == c;
                bool hit;
                mcur = mask_advance(m, mcur, nm, (int32_t)c, lane);
                if (!COMP) {
                    if (mcur >= nm) break;              // mask exhausted (_kernels.py:459-460)
                    hit = m[mcur] == (int32_t)c;
                } else {
                    hit = !(mcur < nm && m[mcur] == (int32_t)c);
                }
                const unsigned who = __ballot_sync(FULL, mine);
                if (hit) {
                    evaluated += lane == 0 ? __popc(who) : 0;
                    if (!COMP) {
                        if (KIND == 0) {
                            if (lane == 0) scnt[mcur] += NUMERIC ? __popc(who) : 1;
                        } else if (KIND == 1) {
                            long long prod = (mine && NUMERIC) ? a_i * ((const long long*)p.b_val)[pos] : 0;
#pragma unroll
                            for (int d = 16; d > 0; d >>= 1) prod += __shfl_xor_sync(FULL, prod, d);
                            if (lane == 0) {
                                sval[mcur] += (unsigned long long)prod;
                                scnt[mcur] = 1;
                            }
                        } else {
                            const double prod = (mine && NUMERIC) ? a_d * ((const double*)p.b_val)[pos] : 0.0;
                            unsigned b = who;
                            double acc = 0.0;
                            int first = scnt[mcur] == 0;
                            if (!first) acc = __longlong_as_double((long long)sval[mcur]);
                            while (b) {
                                const int src = __ffs(b) - 1;
                                b &= b - 1;
                                const double pb = __shfl_sync(FULL, prod, src);
                                acc = first ? pb : acc + pb;
                                first = 0;
                            }
                            if (lane == 0) {
                                sval[mcur] = (unsigned long long)__double_as_longlong(acc);
                                scnt[mcur] = 1;
                            }
                        }
                    } else {
                        // complement, single batch: columns arrive sorted
                        if (NUMERIC) {
                            if (KIND == 2) {
                                const double prod = mine ? a_d * ((const double*)p.b_val)[pos] : 0.0;
                                unsigned b = who;
                                double acc = 0.0;
                                bool first = true;
                                while (b) {
                                    const int src = __ffs(b) - 1;
                                    b &= b - 1;
                                    const double pb = __shfl_sync(FULL, prod, src);
                                    acc = first ? pb : acc + pb;
                                    first = false;
                                }
                                if (lane == 0) {
                                    o.idx[w0 + n_out] = (int32_t)c;
                                    ((double*)o.val)[w0 + n_out] = acc;
                                }
                            } else {
                                long long prod = 0;
                                if (mine) prod = KIND == 1 ? a_i * ((const long long*)p.b_val)[pos] : 1;
#pragma unroll
                                for (int d = 16; d > 0; d >>= 1) prod += __shfl_xor_sync(FULL, prod, d);
                                if (lane == 0) {
                                    o.idx[w0 + n_out] = (int32_t)c;
                                    if (KIND == 0 && o.out_f64) ((double*)o.val)[w0 + n_out] = (double)prod;
                                    else ((long long*)o.val)[w0 + n_out] = prod;
                                }
                            }
                        }
                        n_out++;
                    }
                }
                __syncwarp();
                if (mine) {
                    pos++;
                    if (!COMP && ninspect != 0) {
                        // Alg. 5 inspection: skip entries that cannot match any more
                        if (ninspect > 0) {
                            const int32_t floor_c = mcur < nm ? m[mcur] : 0x7fffffff;
                            while (pos < end && p.b_idx[pos] < floor_c) pos++;
                        } else {
                            while (pos < end && !contains_sorted(m, nm, p.b_idx[pos])) pos++;
                        }
                    }
                    head = pos < end ? (uint32_t)p.b_idx[pos] : HEAP_DONE;
                }
            }
        }
        if (!COMP) {
            // gather the mask-rank slots in mask order
            int64_t running = 0;
            for (int64_t base = 0; base < nm; base += 32) {
                const int64_t q = base + lane;
                const bool set = q < nm && scnt[q] > 0;
                const unsigned bal = __ballot_sync(FULL, set);
                if (NUMERIC && set) {
                    const int64_t d = w0 + running + __popc(bal & lanemask_lt());
                    o.idx[d] = m[q];
                    if (KIND == 0) {
                        if (o.out_f64) ((double*)o.val)[d] = (double)scnt[q];
                        else ((long long*)o.val)[d] = scnt[q];
                    } else {
                        ((unsigned long long*)o.val)[d] = sval[q];
                    }
                }
                running += __popc(bal);
            }
            n_out = running;
        }
        if (lane == 0) o.row_nnz[i] = n_out;
        __syncwarp();
    }
    if (NUMERIC && lane == 0 && evaluated) atomicAdd(o.evaluated, evaluated);
}

}  // namespace mm

namespace mm {

// Complemented heap rows with more than 32 A entries: every A entry of the
// row is an iterator (the reference pushes them all into one heap,
// _kernels.py:444-447, NInspect forced to 0 for the complement, :437).
// Lane l owns iterators q = l + 32u (u < K = ceil(na / 32)), their state in
// the warp's slab: head column, remaining length, B position.  The lane keeps
// the minimum head of its iterators; the warp-wide minimum is the heap's pop
// (__reduce_min_sync), the mask cursor advances to it, and every iterator
// sitting on that column contributes and advances.  Contributions fold in
// ascending A position (u-major, then lane: ascending k, the MSA order, so a
// float64 slot is bit-identical to MSA); the output arrives column-sorted.
// Per-iterator bytes in the slab: 4 (head) + 4 (remaining) + 8 (position).
__host__ __device__ constexpr size_t heap_iter_bytes(int64_t na_max) {
    return (size_t)16 * (size_t)((na_max + 31) & ~31ll);
}

template <int KIND, bool NUMERIC>
__global__ void __launch_bounds__(256) k_push_heap_comp(Prob p, Out o, Work wk, int na_max, unsigned char* gslab) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t cap = (na_max + 31) & ~31;
    unsigned char* slab = gslab + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * heap_iter_bytes(na_max);
    uint32_t* s_head = (uint32_t*)slab;
    uint32_t* s_rem = s_head + cap;
    int64_t* s_pos = (int64_t*)(s_rem + cap);
    unsigned long long evaluated = 0;
    for (;;) {
        int r = 0;
        if (lane == 0) r = atomicAdd(wk.cursor, 1);
        r = __shfl_sync(FULL, r, 0);
        if (r >= wk.count) break;
        const int64_t i = wk.rows[r];
        const int64_t as = p.a_ptr[i], ae = p.a_ptr[i + 1];
        const int64_t ms = p.m_ptr[i], nm = p.m_ptr[i + 1] - ms;
        const int32_t* m = p.m_idx + ms;
        const int64_t w0 = NUMERIC ? o.off[i] : 0;
        const int na = (int)(ae - as);
        const int K = (na + 31) >> 5;
        // load every iterator; lane minimum
        uint32_t lmin = HEAP_DONE;
        for (int u = 0; u < K; u++) {
            const int q = u * 32 + lane;
            uint32_t head = HEAP_DONE;
            if (q < na) {
                const int32_t k = p.a_idx[as + q];
                const int64_t b0 = p.b_ptr[k], b1 = p.b_ptr[k + 1];
                s_pos[q] = b0;
                s_rem[q] = (uint32_t)(b1 - b0);
                head = b1 > b0 ? (uint32_t)p.b_idx[b0] : HEAP_DONE;
                s_head[q] = head;
            }
            lmin = min(lmin, head);
        }
        __syncwarp();
        int64_t mcur = 0, n_out = 0;
        for (;;) {
            const uint32_t c = __reduce_min_sync(FULL, lmin);
            if (c == HEAP_DONE) break;
            mcur = mask_advance(m, mcur, nm, (int32_t)c, lane);
            const bool hit = !(mcur < nm && m[mcur] == (int32_t)c);
            const bool mine = lmin == c;
            long long isum = 0;
            double acc = 0.0;
            bool first = true;
            int contrib = 0;
            uint32_t nmin = HEAP_DONE;
            if (KIND == 2) {
                // ascending A position: u-major, lanes in order inside u
                for (int u = 0; u < K; u++) {
                    const int q = u * 32 + lane;
                    const bool on = mine && q < na && s_head[q] == c;
                    unsigned b = __ballot_sync(FULL, on);
                    double prod = 0.0;
                    if (on && hit && NUMERIC) prod = ((const double*)p.a_val)[as + q] * ((const double*)p.b_val)[s_pos[q]];
                    while (b) {
                        const int src = __ffs(b) - 1;
                        b &= b - 1;
                        const double pb = __shfl_sync(FULL, prod, src);
                        acc = first ? pb : acc + pb;
                        first = false;
                        contrib++;
                    }
                }
            }
            if (mine) {
                // advance every iterator of this lane on column c
                for (int u = 0; u < K; u++) {
                    const int q = u * 32 + lane;
                    if (q >= na) break;
                    uint32_t head = s_head[q];
                    if (head == c) {
                        const int64_t pos = s_pos[q];
                        if (KIND != 2) {
                            contrib++;
                            if (NUMERIC && hit)
                                isum += KIND == 1 ? ((const long long*)p.a_val)[as + q] * ((const long long*)p.b_val)[pos] : 1;
                        }
                        const uint32_t rem = s_rem[q] - 1;
                        s_rem[q] = rem;
                        s_pos[q] = pos + 1;
                        head = rem ? (uint32_t)p.b_idx[pos + 1] : HEAP_DONE;
                        s_head[q] = head;
                    }
                    nmin = min(nmin, head);
                }
                lmin = nmin;
            }
            __syncwarp();
            if (hit) {
                if (KIND == 2) {
                    if (lane == 0) {
                        evaluated += contrib;
                        if (NUMERIC) {
                            o.idx[w0 + n_out] = (int32_t)c;
                            ((double*)o.val)[w0 + n_out] = acc;
                        }
                    }
                } else {
                    const long long cnt = warp_sum_ll(contrib);
                    const long long sum = warp_sum_ll(isum);
                    if (lane == 0) {
                        evaluated += cnt;
                        if (NUMERIC) {
                            o.idx[w0 + n_out] = (int32_t)c;
                            if (KIND == 0 && o.out_f64) ((double*)o.val)[w0 + n_out] = (double)sum;
                            else ((long long*)o.val)[w0 + n_out] = sum;
                        }
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
