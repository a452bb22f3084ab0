// Push path, hash accumulator: row-wise Gustavson with a table keyed on the
// mask row.
//
// Reference semantics: hash_numeric / hash_symbolic (_kernels.py:130-268) —
// per-row open addressing with linear probing, mask keys marked first
// (:156-162), products probed (:169-171), absent keys discarded (plain,
// :173-174) or claimed (complement, :175-180), complement output sorted
// (:198), plain output in mask order (:208-216).  Every product that survives
// the mask is counted in `evaluated` (the lazy-thunk rule).
//
// GPU form: a group of GW warps owns one row at a time and a table of
// 2^cap_lg (key:int32, cnt:int32[, val:8B]) entries in shared memory
// (tiers 0-2) or in a per-group global slab (tier 3).  The row's products are
// enumerated as a flattened (k, s) space per batch of 32 A entries, so every
// lane does useful work regardless of B row lengths; probes are smem atomics.
//
// KIND: 0 = plus-pair (cnt is the value), 1 = int64 plus-times (atomic add,
// order-free and exact), 2 = float64 plus-times (single warp, products folded
// in ascending k exactly like the reference: bit-identical to MSA/Hash/MCA).
// MODE: MODE_PLAIN, MODE_CTAB (complement, mask marked in the table),
// MODE_CSRCH (complement, mask membership by binary search).
#pragma once
#include "analyze.cuh"
#include "common.cuh"
#include "fused_tail.cuh"
#include "product_loop.cuh"

namespace mm {

template <int KIND>
struct HashEntry {
    static constexpr int bytes = KIND == 0 ? 8 : 16;
};

// Per-warp deferred-probe queue (WarpProber): 64 entries of (j, slot[, s, a]).
template <int KIND>
__host__ __device__ constexpr size_t queue_bytes() {
    return KIND == 2 ? 0 : (size_t)64 * (KIND == 1 ? 24 : 8);
}

// Pointers into one group's table region.
template <int KIND>
struct Table {
    int32_t* keys;
    int32_t* cnt;
    unsigned long long* val;   // KIND != 0: 8-byte payload (int64 bits or double bits)
    __device__ __forceinline__ void bind(unsigned char* base, int cap_max) {
        if (KIND == 0) {
            keys = (int32_t*)base;
            cnt = keys + cap_max;
            val = nullptr;
        } else {
            val = (unsigned long long*)base;
            keys = (int32_t*)(val + cap_max);
            cnt = keys + cap_max;
        }
    }
};

// Find the slot of key j (present or absent).  Returns slot index whose key is
// j, or the EMPTY slot where the probe sequence ended (negated - 1).
__device__ __forceinline__ int probe_find(const int32_t* keys, int32_t j, int lg, uint32_t mask,
                                          uint32_t mult = FIB_MULT) {
    uint32_t h = ((uint32_t)j * mult) >> (32 - lg);
    for (;;) {
        int32_t k = keys[h];
        if (k == j) return (int)h;
        if (k == EMPTY_KEY) return -(int)h - 1;
        h = (h + 1) & mask;
    }
}

// Find-or-insert (complement modes).  Returns the slot holding j.
__device__ __forceinline__ int probe_insert(int32_t* keys, int32_t j, int lg, uint32_t mask) {
    uint32_t h = fib_hash(j, lg);
    for (;;) {
        int32_t k = keys[h];
        if (k == j) return (int)h;
        if (k == EMPTY_KEY) {
            int32_t old = atomicCAS(&keys[h], EMPTY_KEY, j);
            if (old == EMPTY_KEY || old == j) return (int)h;
        }
        h = (h + 1) & mask;
    }
}

// Locate the slot a product with column j accumulates into, or -1 if the
// mask discards it (plain: j absent; complement: j in the mask).
template <int MODE, int KIND>
__device__ __forceinline__ int hash_locate_t(Table<KIND>& tb, int32_t j, int lg, uint32_t cmask,
                                             const int32_t* mrow, int64_t nm) {
    if (MODE == MODE_PLAIN) {
        const int h = probe_find(tb.keys, j, lg, cmask);
        return h < 0 ? -1 : h;
    }
    if (MODE == MODE_CSRCH && contains_sorted(mrow, nm, j)) return -1;
    const int h = probe_insert(tb.keys, j, lg, cmask);
    return tb.cnt[h] < 0 ? -1 : h;
}

// Order-free accumulation of one surviving product into slot h.
template <int KIND, bool NUMERIC>
__device__ __forceinline__ void hash_accumulate(Table<KIND>& tb, int h, long long a,
                                                const void* b_val, int64_t s) {
    if (KIND == 0) {
        if (NUMERIC) atomicAdd(&tb.cnt[h], 1);
        else tb.cnt[h] = 1;
    } else {
        if (NUMERIC) {
            const long long prod = a * ((const long long*)b_val)[s];
            atomicAdd(&tb.val[h], (unsigned long long)prod);
        }
        tb.cnt[h] = 1;
    }
}

// Table access for the plain-mask prober.  Shared-memory tables are addressed
// with 32-bit shared-window addresses (ld/red.shared), so the hot loop carries
// no generic-to-shared conversions; tier-3 tables live in global memory.
template <bool SMEM>
struct TabIO;

template <>
struct TabIO<true> {
    uint32_t keys, cnt, val;
    __device__ __forceinline__ void bind(const int32_t* k, int32_t* c, unsigned long long* v) {
        keys = (uint32_t)__cvta_generic_to_shared(k);
        cnt = (uint32_t)__cvta_generic_to_shared(c);
        val = v ? (uint32_t)__cvta_generic_to_shared(v) : 0u;
    }
    __device__ __forceinline__ int32_t key(uint32_t h) const {
        int32_t x;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(x) : "r"(keys + (h << 2)));
        return x;
    }
    __device__ __forceinline__ void inc(uint32_t h) const {
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(cnt + (h << 2)) : "memory");
    }
    __device__ __forceinline__ void set(uint32_t h) const {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(cnt + (h << 2)), "r"(1) : "memory");
    }
    __device__ __forceinline__ void add64(uint32_t h, unsigned long long x) const {
        asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(val + (h << 3)), "l"(x) : "memory");
    }
};

template <>
struct TabIO<false> {
    const int32_t* keys;
    int32_t* cnt;
    unsigned long long* val;
    __device__ __forceinline__ void bind(const int32_t* k, int32_t* c, unsigned long long* v) {
        keys = k;
        cnt = c;
        val = v;
    }
    __device__ __forceinline__ int32_t key(uint32_t h) const {
        return *(volatile const int32_t*)(keys + h);
    }
    __device__ __forceinline__ void inc(uint32_t h) const { atomicAdd(cnt + h, 1); }
    __device__ __forceinline__ void set(uint32_t h) const { cnt[h] = 1; }
    __device__ __forceinline__ void add64(uint32_t h, unsigned long long x) const { atomicAdd(val + h, x); }
};

// Warp-level prober for the plain mask: every lane probes its product's first
// slot; hits accumulate at once, misses on an EMPTY slot are dropped, and the
// products whose first slot holds another key are queued in shared memory and
// resolved 32 at a time.  A probe continuation is rare per product but almost
// certain somewhere in a warp of 32, so deferring it keeps the common path
// branch-free and the continuation loop dense.  Complement modes (which insert)
// use the direct per-lane path.
template <int KIND, int MODE, bool NUMERIC, bool SMEM>
struct WarpProber {
    Table<KIND> tb;
    TabIO<SMEM> io;
    int lg;
    uint32_t cmask;
    const int32_t* mrow;
    int64_t nm;
    const void* b_val;
    int32_t* qj;
    int32_t* qh;
    long long* qs;
    long long* qa;
    int qn;
    int lane;
    unsigned evaluated;

    __device__ __forceinline__ void accumulate(uint32_t h, long long a, long long s) {
        if (KIND == 0) {
            if (NUMERIC) io.inc(h);
            else io.set(h);
        } else {
            if (NUMERIC) {
                const long long prod = a * ((const long long*)b_val)[s];
                io.add64(h, (unsigned long long)prod);
            }
            io.set(h);
        }
    }

    __device__ __forceinline__ void flush(int c) {
        const int base = qn - c;
        bool act = lane < c;
        int32_t j = 0;
        uint32_t h = 0;
        long long s = 0, a = 0;
        if (act) {
            j = qj[base + lane];
            h = (uint32_t)qh[base + lane];
            if (KIND == 1) {
                s = qs[base + lane];
                a = qa[base + lane];
            }
        }
        __syncwarp();
        qn = base;
        while (act) {
            const int32_t k = io.key(h);
            if (k == j) {
                evaluated++;
                accumulate(h, a, s);
                break;
            }
            if (k == EMPTY_KEY) break;
            h = (h + 1) & cmask;
        }
        __syncwarp();
    }

    // Called by all 32 lanes; lanes without a product pass j = EMPTY_KEY.
    __device__ __forceinline__ void put(int32_t j, long long a, long long s) {
        const bool valid = j != EMPTY_KEY;
        if (MODE != MODE_PLAIN) {
            if (valid) {
                const int h = hash_locate_t<MODE, KIND>(tb, j, lg, cmask, mrow, nm);
                if (h >= 0) {
                    evaluated++;
                    accumulate((uint32_t)h, a, s);
                }
            }
            return;
        }
        const uint32_t h = fib_hash(j, lg);
        const int32_t k = io.key(h);
        const bool hit = valid && k == j;
        const bool pend = valid && k != j && k != EMPTY_KEY;
        if (hit) {
            evaluated++;
            accumulate(h, a, s);
        }
        const unsigned pm = __ballot_sync(FULL, pend);
        if (pm) {
            if (pend) {
                const int pos = qn + __popc(pm & lanemask_lt());
                qj[pos] = j;
                qh[pos] = (int32_t)((h + 1) & cmask);
                if (KIND == 1) {
                    qs[pos] = s;
                    qa[pos] = a;
                }
            }
            qn += __popc(pm);
            if (qn >= 32) {
                __syncwarp();
                flush(32);
            }
        }
    }

    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
#pragma unroll
        for (int u = 0; u < U; u++) put(j[u], a[u], s[u]);
    }

    __device__ __forceinline__ void drain() {
        if (qn) {
            __syncwarp();
            flush(qn);
        }
    }
};

// Collision-free multipliers tried for small plain masks (odd constants).
__device__ __forceinline__ uint32_t direct_mult(int t) {
    switch (t) {
        case 0: return FIB_MULT;
        case 1: return 0x85EBCA77u;
        case 2: return 0xC2B2AE3Du;
        case 3: return 0x27D4EB2Fu;
        case 4: return 0x165667B1u;
        case 5: return 0xD3A2646Du;
        case 6: return 0xFD7046C5u;
        default: return 0xB55A4F09u;
    }
}
constexpr int DIRECT_TRIES = 8;

constexpr int CUCKOO_TRIES = 4;
constexpr int CUCKOO_MAXIT = 64;

// Where the mask keys of a plain row sit.  hm = 0: linear probing from the
// Fibonacci hash; hm = 1 (direct): every key in its home slot
// (j * m1) >> (32 - lg); hm = 2 (two-choice cuckoo): every key in one of its
// two candidate slots, (j * m1) >> (33 - lg) in the lower half of the table
// or half + (j * m2) >> (33 - lg) in the upper half.
struct Placement {
    int hm;
    int lg;
    uint32_t m1, m2;
    __device__ __forceinline__ uint32_t h1(int32_t j) const {
        return hm == 2 ? ((uint32_t)j * m1) >> (33 - lg) : ((uint32_t)j * m1) >> (32 - lg);
    }
    __device__ __forceinline__ uint32_t h2(int32_t j) const {
        return (1u << (lg - 1)) + (((uint32_t)j * m2) >> (33 - lg));
    }
    // slot of a key known to be in the table
    __device__ __forceinline__ int slot(const int32_t* keys, int32_t j) const {
        if (hm == 1) return (int)h1(j);
        if (hm == 2) {
            const uint32_t a = h1(j);
            return keys[a] == j ? (int)a : (int)h2(j);
        }
        return probe_find(keys, j, lg, (1u << lg) - 1u, m1);
    }
};

// Plain mask with every key at a fixed candidate slot (direct: one, cuckoo:
// two): membership is one or two independent shared loads and compares, with
// no probe sequence and nothing to defer.
template <int KIND, bool NUMERIC, int WAYS>
struct DirectProber {
    uint32_t keys_s, cnt_s, val_s;
    uint32_t mult, mult2;
    int shift;            // 32 - lg (direct) or 33 - lg (cuckoo, per half)
    uint32_t half;        // cuckoo: first slot of the upper half
    uint32_t dummy_s;     // this lane's scratch word
    const void* b_val;
    unsigned evaluated;
    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
        uint32_t h[U];
        int32_t k[U];
        uint32_t hb[U];
        int32_t kb[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            h[u] = ((uint32_t)j[u] * mult) >> shift;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(k[u]) : "r"(keys_s + (h[u] << 2)));
            if (WAYS == 2) {
                hb[u] = half + (((uint32_t)j[u] * mult2) >> shift);
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(kb[u]) : "r"(keys_s + (hb[u] << 2)));
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            bool hit = k[u] == j[u];
            if (WAYS == 2) {
                if (!hit) h[u] = hb[u];
                hit |= kb[u] == j[u];
            }
            hit &= j[u] >= 0;   // padding lanes carry EMPTY_KEY
            if (KIND == 0) {
                // plus-pair: evaluated = sum of the counts, taken at the gather
                if (NUMERIC)
#ifndef MM_RED_PRED
                    // every lane issues the RED (a miss counts into its own
                    // dummy word): no branch around the atomic
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t.reg .u32 ad;\n\t"
                        "setp.ne.u32 ph, %0, 0;\n\t"
                        "selp.u32 ad, %1, %2, ph;\n\t"
                        "red.shared.add.u32 [ad], 1;\n\t}" ::"r"((uint32_t)hit),
                        "r"(cnt_s + (h[u] << 2)), "r"(dummy_s)
                        : "memory");
#else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ne.u32 ph, %0, 0;\n\t"
                        "@ph red.shared.add.u32 [%1], 1;\n\t}" ::"r"((uint32_t)hit),
                        "r"(cnt_s + (h[u] << 2))
                        : "memory");
#endif
                else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ne.u32 ph, %0, 0;\n\t"
                        "@ph st.shared.u32 [%1], 1;\n\t}" ::"r"((uint32_t)hit),
                        "r"(cnt_s + (h[u] << 2))
                        : "memory");
            } else if (hit) {
                evaluated++;
                if (NUMERIC) {
                    const long long prod = a[u] * ((const long long*)b_val)[s[u]];
                    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(val_s + (h[u] << 3)), "l"(prod) : "memory");
                }
                asm volatile("st.shared.u32 [%0], 1;" ::"r"(cnt_s + (h[u] << 2)) : "memory");
            }
        }
    }
    __device__ __forceinline__ void drain() {}
};

// Slot locator for the ordered float64 path (single warp).
template <int MODE>
struct HashLocatorF64 {
    int32_t* keys;
    int32_t* cnt;
    double* vals;
    int lg;
    uint32_t cmask;
    const int32_t* mrow;
    int64_t nm;
    __device__ __forceinline__ int locate(int32_t j) {
        if (MODE == MODE_PLAIN) {
            const int h = probe_find(keys, j, lg, cmask);
            return h < 0 ? -1 : h;
        }
        if (MODE == MODE_CSRCH && contains_sorted(mrow, nm, j)) return -1;
        const int h = probe_insert(keys, j, lg, cmask);
        return cnt[h] < 0 ? -1 : h;
    }
    __device__ __forceinline__ void fold(int h, double prod) {
        if (cnt[h] == 0) {
            vals[h] = prod;
            cnt[h] = 1;
        } else {
            vals[h] += prod;
        }
    }
    __device__ __forceinline__ void mark(int h) { cnt[h] = 1; }
};

// ---------------------------------------------------------------------------
// The row processor.
// ---------------------------------------------------------------------------
// One part of a row: the mask entries [ms, me) and the products whose column
// lies in [c_lo, c_hi) (the whole row unless the row is sliced, see
// hash_row).  Writes its results at w_base (NUMERIC) and returns their count.
#ifndef MM_SEARCH_ON
#define MM_SEARCH_ON 1   // mask-driven binary search of long B rows (plain hash rows)
#endif
template <int GW, int KIND, int MODE, bool NUMERIC, bool SMEM>
__device__ __forceinline__ int hash_part(const Prob& p, const Out& o, Table<KIND> tb, const RowInfo& ri,
                                         int64_t ms, int64_t me, int32_t c_lo, int32_t c_hi, int64_t w_base,
                                         int cap_lg, int cap_lg_max, int gt, int bar_id, int* s_warp,
                                         BatchSmem bsm, unsigned char* wq, uint32_t dummy_s,
                                         unsigned long long& evaluated, int64_t* cur = nullptr, int kb = 0) {
    constexpr int GT = GW * 32;
    // Plain masks in shared memory keep the table clean between rows (each
    // row cleans what it touched) and first look for a multiplier that puts
    // every mask key in its home slot of the full 2^cap_lg_max table.
    constexpr bool CLEAN = MODE == MODE_PLAIN && SMEM && KIND != 2;
    const int lane = gt & 31;
    const int wg = gt >> 5;
    const int64_t as = ri.as, ae = ri.ae;
    const int64_t nm = me - ms;
    Placement pl{0, cap_lg, FIB_MULT, 0u};
    // group-wide OR of a per-thread flag
    auto group_any = [&](bool v) {
        bool any = __any_sync(FULL, v);
        if (GW > 1) {
            if (lane == 0) s_warp[wg] = any;
            group_bar(bar_id, GT);
            any = false;
#pragma unroll
            for (int w = 0; w < GW; w++) any |= s_warp[w] != 0;
            group_bar(bar_id, GT);
        }
        return any;
    };
    if (CLEAN && nm * nm <= (1ll << (cap_lg_max + 2))) {
        // direct: a multiplier without collisions over the whole 2^cap_lg_max table
        const int sh = 32 - cap_lg_max;
        for (int t = 0; t < DIRECT_TRIES && pl.hm == 0; t++) {
            const uint32_t m = direct_mult(t);
            bool clash = false;
            for (int64_t q = ms + gt; q < me; q += GT) {
                const int32_t j = p.m_idx[q];
                clash |= atomicCAS(&tb.keys[((uint32_t)j * m) >> sh], EMPTY_KEY, j) != EMPTY_KEY;
            }
            if (!group_any(clash)) {
                pl = Placement{1, cap_lg_max, m, 0u};
            } else {
                for (int64_t q = ms + gt; q < me; q += GT) {
                    const int32_t j = p.m_idx[q];
                    const uint32_t h = ((uint32_t)j * m) >> sh;
                    if (tb.keys[h] == j) tb.keys[h] = EMPTY_KEY;
                }
                group_bar(bar_id, GT);
            }
        }
    }
    if (CLEAN && pl.hm == 0 && cap_lg >= 4) {
        // two-choice cuckoo in the row's table (load <= 1/2 by construction):
        // atomicExch insertion, each displaced key moved to its other slot
        const uint32_t half = 1u << (cap_lg - 1);
        for (int t = 0; t < CUCKOO_TRIES && pl.hm == 0; t++) {
            const Placement c{2, cap_lg, direct_mult(2 * t), direct_mult(2 * t + 1)};
            bool lost = false;
            for (int64_t q = ms + gt; q < me; q += GT) {
                int32_t cur = p.m_idx[q];
                uint32_t h = c.h1(cur);
                int it = 0;
                for (; it < CUCKOO_MAXIT; it++) {
                    const int32_t old = atomicExch(&tb.keys[h], cur);
                    if (old == EMPTY_KEY) break;
                    cur = old;
                    h = h < half ? c.h2(cur) : c.h1(cur);
                }
                lost |= it == CUCKOO_MAXIT;
            }
            if (!group_any(lost)) {
                pl = c;
            } else {
                for (int e = gt; e < (1 << cap_lg); e += GT) tb.keys[e] = EMPTY_KEY;
                group_bar(bar_id, GT);
            }
        }
    }
    if (pl.hm == 1) cap_lg = cap_lg_max;
    if (CLEAN) __syncwarp();
    const int cap = 1 << cap_lg;
    const uint32_t cmask = (uint32_t)cap - 1;
    pl.lg = cap_lg;
    // 1. clear the table (CLEAN: already clean)
    if (!CLEAN) {
        for (int e = gt; e < cap; e += GT) {
            tb.keys[e] = EMPTY_KEY;
            tb.cnt[e] = 0;
            if (KIND == 1) tb.val[e] = 0ull;
        }
        group_bar(bar_id, GT);
    }
    // 2. mark the mask row (plain: ALLOWED; table complement: NOT-ALLOWED = -1)
    if (MODE != MODE_CSRCH && pl.hm == 0) {
        for (int64_t t = ms + gt; t < me; t += GT) {
            int32_t j = p.m_idx[t];
            uint32_t h = fib_hash(j, cap_lg);
            for (;;) {
                int32_t old = atomicCAS(&tb.keys[h], EMPTY_KEY, j);
                if (old == EMPTY_KEY) break;
                h = (h + 1) & cmask;
            }
            if (MODE == MODE_CTAB) tb.cnt[h] = -1;
        }
        group_bar(bar_id, GT);
    }

    // 3. products
    if (KIND == 2) {
        // ordered float64 in a group: warp wg folds its own output columns —
        // a slice of the mask row (plain) or of [0, ncols) (complement)
        int32_t c_lo = INT32_MIN, c_hi = INT32_MAX;
        bool idle = false;
        if (GW > 1) {
            if (MODE == MODE_PLAIN) {
                const int64_t r0 = nm * wg / GW, r1 = nm * (wg + 1) / GW;
                idle = r0 == r1;
                c_lo = wg == 0 ? INT32_MIN : p.m_idx[ms + r0];
                c_hi = r1 < nm ? p.m_idx[ms + r1] : INT32_MAX;
            } else {
                c_lo = wg == 0 ? INT32_MIN : (int32_t)(p.ncols * wg / GW);
                c_hi = wg == GW - 1 ? INT32_MAX : (int32_t)(p.ncols * (wg + 1) / GW);
                idle = c_lo != INT32_MIN && c_hi != INT32_MAX && c_lo == c_hi;
            }
        }
        HashLocatorF64<MODE> loc{tb.keys, tb.cnt, (double*)tb.val, cap_lg, cmask, p.m_idx + ms, me - ms};
        if (!idle) evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane, c_lo, c_hi);
    } else if (CLEAN && pl.hm == 1) {
        DirectProber<KIND, NUMERIC, 1> pr;
        pr.keys_s = (uint32_t)__cvta_generic_to_shared(tb.keys);
        pr.cnt_s = (uint32_t)__cvta_generic_to_shared(tb.cnt);
        pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(tb.val);
        pr.mult = pl.m1;
        pr.mult2 = 0u;
        pr.shift = 32 - cap_lg;
        pr.half = 0u;
        pr.dummy_s = dummy_s;
        pr.b_val = p.b_val;
        pr.evaluated = 0;
        flat_products<GW, KIND, decltype(pr), MODE == MODE_PLAIN && MM_SEARCH_ON>(p, pr, as, ae, gt, bar_id, s_warp, bsm, c_lo, c_hi,
                                                                               p.m_idx + ms, nm, cur);
        evaluated += pr.evaluated;
    } else if (CLEAN && pl.hm == 2) {
        DirectProber<KIND, NUMERIC, 2> pr;
        pr.keys_s = (uint32_t)__cvta_generic_to_shared(tb.keys);
        pr.cnt_s = (uint32_t)__cvta_generic_to_shared(tb.cnt);
        pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(tb.val);
        pr.mult = pl.m1;
        pr.mult2 = pl.m2;
        pr.shift = 33 - cap_lg;
        pr.half = 1u << (cap_lg - 1);
        pr.dummy_s = dummy_s;
        pr.b_val = p.b_val;
        pr.evaluated = 0;
        flat_products<GW, KIND, decltype(pr), MODE == MODE_PLAIN && MM_SEARCH_ON>(p, pr, as, ae, gt, bar_id, s_warp, bsm, c_lo, c_hi,
                                                                               p.m_idx + ms, nm, cur);
        evaluated += pr.evaluated;
    } else {
        WarpProber<KIND, MODE, NUMERIC, SMEM> pr;
        pr.tb = tb;
        pr.io.bind(tb.keys, tb.cnt, tb.val);
        pr.lg = cap_lg;
        pr.cmask = cmask;
        pr.mrow = p.m_idx + ms;
        pr.nm = me - ms;
        pr.b_val = p.b_val;
        pr.qj = (int32_t*)wq;
        pr.qh = pr.qj + 64;
        pr.qs = (long long*)(pr.qh + 64);
        pr.qa = pr.qs + 64;
        pr.qn = 0;
        pr.lane = lane;
        pr.evaluated = 0;
        flat_products<GW, KIND, decltype(pr), MODE == MODE_PLAIN && MM_SEARCH_ON>(p, pr, as, ae, gt, bar_id, s_warp, bsm, c_lo, c_hi,
                                                                               p.m_idx + ms, nm, cur);
        evaluated += pr.evaluated;
    }
    group_bar(bar_id, GT);

    // 4. gather
    const int64_t w = w_base;
    int running = 0;
    if (MODE == MODE_PLAIN) {
        // mask order, like the reference's gather (_kernels.py:78-85,208-216)
        for (int64_t base = ms; base < me; base += GT) {
            int64_t t = base + gt;
            bool set = false;
            int32_t j = 0;
            int h = 0;
            long long c = 0;
            if (t < me) {
                j = p.m_idx[t];
                h = CLEAN ? pl.slot(tb.keys, j) : probe_find(tb.keys, j, cap_lg, cmask);
                c = tb.cnt[h];
                if (CLEAN && KIND == 0 && NUMERIC && pl.hm != 0) evaluated += (unsigned)tb.cnt[h];
                if (CLEAN && KIND == 0 && NUMERIC && kb) {
                    // k-blocked passes: the row's partial counts wait in its own
                    // (mask-shaped) value slots; the last pass reads a chunk's slots
                    // before the prefix barrier and writes at or below them
                    long long* acc = (long long*)o.val + w + (t - ms);
                    if (kb == 1) *acc = c;
                    else if (kb == 2) { if (c) *acc += c; }
                    else c += *acc;
                }
                set = c > 0;
            }
            if (CLEAN && KIND == 0 && NUMERIC && (kb == 1 || kb == 2)) continue;
            int tot;
            int pos = group_prefix<GW>(set, &tot, s_warp, bar_id, gt);
            if (NUMERIC && set) {
                int64_t d = w + running + pos;
                o.idx[d] = j;
                if (KIND == 0) {
                    if (o.out_f64) ((double*)o.val)[d] = (double)c;
                    else ((long long*)o.val)[d] = c;
                } else {
                    ((unsigned long long*)o.val)[d] = tb.val[h];
                }
            }
            running += tot;
        }
    } else {
        // complement: emit inserted keys in column order (_kernels.py:69,198)
        // count, then bitonic-sort the table by key with invalid slots last
        int mine = 0;
        for (int e = gt; e < cap; e += GT) {
            bool v = tb.keys[e] != EMPTY_KEY && tb.cnt[e] > 0;
            mine += v;
            if (NUMERIC && !v) tb.keys[e] = 0x7fffffff;
        }
        int tot;
        // reuse group_prefix as a reduction: every thread contributes `mine`
        {
            int acc = mine;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(FULL, acc, d);
            if (GW == 1) {
                tot = acc;
            } else {
                if (lane == 0) s_warp[wg] = acc;
                group_bar(bar_id, GT);
                tot = 0;
#pragma unroll
                for (int q = 0; q < GW; q++) tot += s_warp[q];
            }
            group_bar(bar_id, GT);
        }
        if (NUMERIC && tot > 0) {
            for (int kk = 2; kk <= cap; kk <<= 1) {
                for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                    for (int e = gt; e < cap; e += GT) {
                        int prt = e ^ jj;
                        if (prt > e) {
                            bool up = (e & kk) == 0;
                            int32_t ke = tb.keys[e], kp = tb.keys[prt];
                            if ((ke > kp) == up) {
                                tb.keys[e] = kp;
                                tb.keys[prt] = ke;
                                int32_t c = tb.cnt[e];
                                tb.cnt[e] = tb.cnt[prt];
                                tb.cnt[prt] = c;
                                if (KIND != 0) {
                                    unsigned long long v = tb.val[e];
                                    tb.val[e] = tb.val[prt];
                                    tb.val[prt] = v;
                                }
                            }
                        }
                    }
                    group_bar(bar_id, GT);
                }
            }
            for (int e = gt; e < tot; e += GT) {
                int64_t d = w + e;
                o.idx[d] = tb.keys[e];
                if (KIND == 0) {
                    if (o.out_f64) ((double*)o.val)[d] = (double)tb.cnt[e];
                    else ((long long*)o.val)[d] = tb.cnt[e];
                } else {
                    ((unsigned long long*)o.val)[d] = tb.val[e];
                }
            }
        }
        running = tot;
    }
    group_bar(bar_id, GT);
    if (CLEAN) {
        // leave the table clean: the key slots of a direct / cuckoo row, else the row's whole table
        if (pl.hm != 0) {
            for (int64_t q = ms + gt; q < me; q += GT) {
                const int h = pl.slot(tb.keys, p.m_idx[q]);
                tb.keys[h] = EMPTY_KEY;
                tb.cnt[h] = 0;
                if (KIND == 1) tb.val[h] = 0ull;
            }
        } else {
            for (int e = gt; e < cap; e += GT) {
                tb.keys[e] = EMPTY_KEY;
                tb.cnt[e] = 0;
                if (KIND == 1) tb.val[e] = 0ull;
            }
        }
        group_bar(bar_id, GT);
    }
    return running;
}

// Rows of a bin that the k-blocked passes cut (not sliced, at least min_flops
// products), compacted to the front of `list` (filled with -1 beforehand: the row
// fetch stops at the first); the same rule as k_push_hash's.
__global__ void __launch_bounds__(256) k_kb_select(Prob p, Work wk, int64_t slice, int64_t min_flops,
                                                   int32_t* list, int32_t* count) {
    const int lane = threadIdx.x & 31;
    for (int base = blockIdx.x * blockDim.x; base < wk.count; base += gridDim.x * blockDim.x) {
        const int q = base + threadIdx.x;
        int32_t i = -1;
        bool take = false;
        if (q < wk.count) {
            i = wk.rows[q];
            take = p.m_ptr[i + 1] - p.m_ptr[i] <= slice && p.row_flops[i] >= min_flops;
        }
        const unsigned pick = __ballot_sync(FULL, take);
        int start = 0;
        if (lane == 0 && pick) start = atomicAdd(count, __popc(pick));
        start = __shfl_sync(FULL, start, 0);
        if (take) list[start + __popc(pick & ((1u << lane) - 1))] = i;
    }
}

// First A entry of [as, ae) whose B row starts at or after entry `bound` of B
// (A's columns ascend, so B's row starts do): the cut of a k-blocked pass.
__device__ __forceinline__ int64_t kb_lower(const Prob& p, int64_t as, int64_t ae, int64_t bound) {
    while (as < ae) {
        const int64_t mid = (as + ae) >> 1;
        if (p.b_ptr[p.a_idx[mid]] < bound) as = mid + 1;
        else ae = mid;
    }
    return as;
}

// A row.  Plain rows whose mask does not fit the largest shared table
// (cfg5 hubs: up to 163,558 mask entries; the bin's tier-3 launch, see
// maskmul_abi.cu) are processed in slices of 3/8 of the table's slots of
// consecutive mask entries: each slice keeps only the
// products whose column falls in its column range (a sub-range of every
// sorted B row, found by binary search), so the table stays in shared memory
// instead of an L2/DRAM-resident global table.  Slices run in column order
// and append to the row's output, which therefore stays in mask order.
template <int GW, int KIND, int MODE, bool NUMERIC, bool SMEM>
__device__ __forceinline__ void hash_row(const Prob& p, const Out& o, Table<KIND> tb, const RowInfo& ri,
                                         int cap_lg, int cap_lg_max, int gt, int bar_id, int* s_warp,
                                         BatchSmem bsm, unsigned char* wq, uint32_t dummy_s,
                                         unsigned long long& evaluated, int64_t* cur = nullptr, int kb = 0) {
    constexpr bool CLEAN = MODE == MODE_PLAIN && SMEM && KIND != 2;
    const int64_t nm = ri.me - ri.ms;
    const int64_t w = NUMERIC ? o.off[ri.i] : 0;
    int64_t total = 0;
#ifndef MM_SLICE_EIGHTHS
#define MM_SLICE_EIGHTHS 3
#endif
    // load 3/8 of the table: two-choice cuckoo placement succeeds
    const int64_t slice = (int64_t)MM_SLICE_EIGHTHS << (cap_lg_max - 3);
    if (!CLEAN || nm <= slice) {
        total = hash_part<GW, KIND, MODE, NUMERIC, SMEM>(p, o, tb, ri, ri.ms, ri.me, INT32_MIN, INT32_MAX, w,
                                                         cap_lg, cap_lg_max, gt, bar_id, s_warp, bsm, wq,
                                                         dummy_s, evaluated, nullptr, kb);
        if (kb == 1 || kb == 2) return;   // partial counts only
    } else {
        for (int64_t s0 = ri.ms; s0 < ri.me; s0 += slice) {
            const int64_t s1 = s0 + slice < ri.me ? s0 + slice : ri.me;
            const int32_t c_lo = s0 == ri.ms ? INT32_MIN : p.m_idx[s0];
            const int32_t c_hi = s1 < ri.me ? p.m_idx[s1] : INT32_MAX;
            // slice cursors: each A entry's B row resumes where the previous slice ended
            total += hash_part<GW, KIND, MODE, NUMERIC, SMEM>(p, o, tb, ri, s0, s1, c_lo, c_hi, w + total,
                                                              cap_lg_max, cap_lg_max, gt, bar_id, s_warp, bsm,
                                                              wq, dummy_s, evaluated,
                                                              ri.ae - ri.as <= p.cursor_stride ? cur : nullptr);
        }
    }
    if (gt == 0) o.row_nnz[ri.i] = total;
}

// ---------------------------------------------------------------------------
// Kernel: groups of GW warps fetch rows of one bin dynamically.
// SMEM: table in dynamic shared memory (groups_per_block * 2^cap_lg_max entries)
// otherwise in `gslab` (one slab of 2^cap_lg_max entries per group).
// ---------------------------------------------------------------------------
#ifndef MM_HASH_MINB
#define MM_HASH_MINB 4   // <= 64 registers: 4 blocks of 256 threads per SM (5 spills; measured on cfg2)
#endif
template <int GW, bool SMEM, int KIND, int MODE, bool NUMERIC>
#ifndef MM_HASH16_MINB
#define MM_HASH16_MINB 2
#endif
__global__ void __launch_bounds__(GW == 32 ? 1024 : (GW == 16 ? 512 : 256), GW <= 8 ? MM_HASH_MINB : (GW == 16 ? MM_HASH16_MINB : 1))
k_push_hash(Prob p, Out o, Work wk, const int8_t* row_cap_lg, int cap_lg_max,
            unsigned char* gslab) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[16];
    __shared__ int s_warp[32];
    constexpr int GT = GW * 32;
    const int groups = blockDim.x / GT;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int bar_id = 1 + g;
    const int cap_max = 1 << cap_lg_max;
    constexpr size_t BATCH_BYTES = batch_bytes<GW, KIND>();
    unsigned char* base = SMEM ? smem + (size_t)g * cap_max * HashEntry<KIND>::bytes
                               : gslab + ((size_t)blockIdx.x * groups + g) * (size_t)cap_max *
                                             HashEntry<KIND>::bytes;
    unsigned char* bbase = smem + (SMEM ? (size_t)groups * cap_max * HashEntry<KIND>::bytes : 0) +
                           (size_t)g * BATCH_BYTES;
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    unsigned char* wq = smem + (SMEM ? (size_t)groups * cap_max * HashEntry<KIND>::bytes : 0) +
                        (size_t)groups * BATCH_BYTES + (size_t)(threadIdx.x >> 5) * queue_bytes<KIND>();
#ifdef MM_STAGE_TMA
    stage_init();
#endif
    Table<KIND> tb;
    tb.bind(base, cap_max);
    // shared-memory tables: gslab, when given, holds the sliced rows' cursors
    int64_t* cursors = SMEM && gslab && p.cursor_stride
                           ? (int64_t*)gslab + ((size_t)blockIdx.x * groups + g) * (size_t)p.cursor_stride
                           : nullptr;
    __shared__ uint32_t s_dummy[(GW == 32 ? 32 : (GW == 16 ? 16 : 8)) * 32];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
    if (MODE == MODE_PLAIN && SMEM && KIND != 2) {   // hash_row keeps it clean from here on
        for (int e = gt; e < cap_max; e += GT) {
            tb.keys[e] = EMPTY_KEY;
            tb.cnt[e] = 0;
            if (KIND == 1) tb.val[e] = 0ull;
        }
        group_bar(bar_id, GT);
    }
    unsigned long long evaluated = 0;
    RowFetcher<GW, GW == 16 && MODE == MODE_PLAIN && SMEM && KIND == 0 && NUMERIC> rf;
    if (wk.count < 4 * (int)(gridDim.x * groups)) rf.per = 1;   // few rows per group: one per fetch
    RowInfo ri;
    while (rf.next(p, wk, gt, bar_id, s_row + g, ri)) {
        if (!row_cap_lg) {
            // small-problem path (no analysis pass before it): every row with
            // the full table; a plain mask row over half of it is left to the
            // host's fallback to the binned path
            if (ri.me - ri.ms > (1 << (cap_lg_max - 1))) {
                if (gt == 0) {
                    atomicExch(o.overflow, 1);
                    o.row_nnz[ri.i] = 0;
                }
                continue;
            }
            if (ri.ae == ri.as || ri.me == ri.ms) {   // no products / empty mask row
                if (gt == 0) o.row_nnz[ri.i] = 0;
                continue;
            }
        }
        int kb = 0;
        if (GW == 16 && MODE == MODE_PLAIN && SMEM && KIND == 0 && NUMERIC && p.kb_pass) {
            // k-blocked passes (launch_bins_on): this launch folds only the A entries whose
            // B row lies in the pass's block of B, so the rows in flight share an
            // L2-resident part of B.  A row cut into slices, or too light to pay for the
            // passes' table set-ups, runs whole in the last pass.
            kb = p.kb_pass;
            if (ri.me - ri.ms > ((int64_t)MM_SLICE_EIGHTHS << (cap_lg_max - 3)) || p.row_flops[ri.i] < p.kb_min_flops) {
                if (kb != 3) continue;
                kb = 0;
            } else {
                if (kb != 1) ri.as = kb_lower(p, ri.as, ri.ae, p.kb_lo);
                if (kb != 3) ri.ae = kb_lower(p, ri.as, ri.ae, p.kb_hi);
                if (kb == 2 && ri.as == ri.ae) continue;
            }
        }
        hash_row<GW, KIND, MODE, NUMERIC, SMEM>(p, o, tb, ri, row_cap_lg ? row_cap_lg[ri.i] : cap_lg_max,
                                                cap_lg_max, gt, bar_id, s_warp + g * GW, bsm, wq, dummy_s,
                                                evaluated, cursors, kb);
    }
    if (NUMERIC) {
        long long e = warp_sum_ll((long long)evaluated);
        if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

// ---------------------------------------------------------------------------
// Small plain one-phase multiplies in ONE launch: the 1-warp plain hash kernel
// over every row (no analysis pass: the warp sums the row's products itself,
// as flops_per_row does, multiply.py:103-108) followed by the fused tail
// (fused_tail.cuh).  A mask row over half the fixed table raises o.overflow
// and the host runs the binned path instead.
// ---------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(256, MM_HASH_MINB)
k_tiny_hash(Prob p, Out o, Work wk, int cap_lg_max, Tail tail) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int GW = 1, GT = 32;
    const int groups = blockDim.x / GT;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int cap_max = 1 << cap_lg_max;
    constexpr size_t BATCH_BYTES = batch_bytes<GW, KIND>();
    unsigned char* base = smem + (size_t)g * cap_max * HashEntry<KIND>::bytes;
    unsigned char* bbase = smem + (size_t)groups * cap_max * HashEntry<KIND>::bytes + (size_t)g * BATCH_BYTES;
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    unsigned char* wq = smem + (size_t)groups * cap_max * HashEntry<KIND>::bytes + (size_t)groups * BATCH_BYTES +
                        (size_t)g * queue_bytes<KIND>();
    Table<KIND> tb;
    tb.bind(base, cap_max);
    __shared__ uint32_t s_dummy[256];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
    if (KIND != 2) {   // hash_row keeps the table clean from here on
        for (int e = gt; e < cap_max; e += GT) {
            tb.keys[e] = EMPTY_KEY;
            tb.cnt[e] = 0;
            if (KIND == 1) tb.val[e] = 0ull;
        }
        __syncwarp();
    }
    unsigned long long evaluated = 0, gen = 0;
    int empty = 0;
    RowFetcher<GW> rf;
    if (wk.count < 4 * (int)(gridDim.x * groups)) rf.per = 1;
    RowInfo ri;
    while (rf.next(p, wk, gt, 0, nullptr, ri)) {
        long long f = 0;
        for (int64_t t = ri.as + gt; t < ri.ae; t += 32) {
            const int32_t k = p.a_idx[t];
            f += p.b_ptr[k + 1] - p.b_ptr[k];
        }
        f = warp_sum_ll(f);
        gen += (unsigned long long)f;
        if (f == 0 || ri.me == ri.ms) {   // no products / empty mask row (_kernels.py:143-145)
            empty++;
            if (gt == 0) o.row_nnz[ri.i] = 0;
            continue;
        }
        if (ri.me - ri.ms > (1 << (cap_lg_max - 1))) {
            if (gt == 0) {
                atomicExch(o.overflow, 1);
                o.row_nnz[ri.i] = 0;
            }
            continue;
        }
        hash_row<GW, KIND, MODE_PLAIN, true, true>(p, o, tb, ri, cap_lg_max, cap_lg_max, gt, 0, nullptr, bsm, wq,
                                                   dummy_s, evaluated, nullptr);
    }
    const long long e = warp_sum_ll((long long)evaluated);
    if (gt == 0) {
        if (e) atomicAdd(o.evaluated, (unsigned long long)e);
        if (gen) atomicAdd(o.gen_flops, gen);
        if (empty) atomicAdd(o.empty_rows, empty);
    }
    fused_tail(tail, (int*)smem);
}

}  // namespace mm
