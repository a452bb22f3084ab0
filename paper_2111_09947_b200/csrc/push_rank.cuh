// Push path, rank-slot accumulators: MSA (windowed bitmap) and MCA (rank search).
//
// Both keep one value slot per mask entry (slot r = the r-th column of M_i),
// so the output row is produced in mask order without any lookup — the
// plain-mask gather of the reference (_kernels.py:78-85, 308-313).
//
// MSA — reference msa_numeric / msa_symbolic (_kernels.py:30-123): a dense
// state per column.  GPU form: a bitmap over the mask row's column window
// [lo, hi] (1 bit per column, 32 columns per word) plus, per word, the mask
// rank of its first set bit.  A product with column j tests bit j-lo; when set,
// its slot is prefix[word] + popc(word & below(j)).  One shared load per
// product, no probing, no divergence but the hit.
//
// MCA — reference mca_numeric / mca_symbolic (_kernels.py:275-344): arrays of
// length nnz(M_i) indexed by mask rank, position found by merging B_k against
// M_i.  GPU form: the mask row staged in shared memory, the rank of each
// product found by a branch-free binary search.
//
// Plain masks only (MCA rejects complement, multiply.py:67-69; the MSA
// complement form runs through the hash kernels).
#pragma once
#include "analyze.cuh"
#include "common.cuh"
#include "product_loop.cuh"

#include <type_traits>

namespace mm {

template <int KIND>
struct RankSlots {
    int32_t* cnt;
    unsigned long long* val;
};

// One product's accumulation into slot r (order-free kinds).
template <int KIND, bool NUMERIC>
__device__ __forceinline__ void rank_accumulate(RankSlots<KIND>& sl, int r, long long a,
                                                const void* b_val, long long s) {
    if (KIND == 0) {
        if (NUMERIC) atomicAdd(sl.cnt + r, 1);
        else sl.cnt[r] = 1;
    } else {
        if (NUMERIC) {
            const long long prod = a * ((const long long*)b_val)[s];
            atomicAdd(sl.val + r, (unsigned long long)prod);
        }
        sl.cnt[r] = 1;
    }
}

// --- MSA bitmap probe ------------------------------------------------------
template <class PreT>
struct MsaBits {
    const uint32_t* bits;
    const PreT* pre;
    int32_t lo;
    uint32_t span;   // hi - lo
    // slot of column j, or -1
    __device__ __forceinline__ int rank(int32_t j) const {
        const uint32_t off = (uint32_t)(j - lo);
        if (off > span) return -1;
        const uint32_t w = off >> 5;
        const uint32_t word = bits[w];
        const uint32_t b = off & 31u;
        if (!((word >> b) & 1u)) return -1;
        return (int)pre[w] + __popc(word & ((1u << b) - 1u));
    }
};

// Shared tiers pack 16 columns and the 16-bit mask rank of the word's first
// set bit into one 32-bit word: (rank << 16) | bits.  One shared load gives
// both the membership bit and the rank base.
struct MsaPacked {
    const uint32_t* words;
    int32_t lo;
    uint32_t span;
    __device__ __forceinline__ int rank(int32_t j) const {
        const uint32_t off = (uint32_t)(j - lo);
        if (off > span) return -1;
        const uint32_t word = words[off >> 4];
        const uint32_t b = off & 15u;
        if (!((word >> b) & 1u)) return -1;
        return (int)(word >> 16) + __popc(word & ((1u << b) - 1u));
    }
};

// --- MCA rank search -------------------------------------------------------
template <bool SMEM>
struct McaRow {
    const int32_t* m;   // mask row (shared when SMEM, else the group's global slab)
    int nm;
    int steps;          // ceil(log2(nm + 1))
    uint32_t m_s;       // 32-bit shared address of m (SMEM)
    __device__ __forceinline__ McaRow(const int32_t* m_, int nm_, int steps_) : m(m_), nm(nm_), steps(steps_) {
        m_s = SMEM ? (uint32_t)__cvta_generic_to_shared(m_) : 0u;
    }
    __device__ __forceinline__ int32_t at(int r) const {
        if (SMEM) {
            int32_t v;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(m_s + 4u * (uint32_t)r));
            return v;
        }
        return m[r];
    }
    __device__ __forceinline__ int rank(int32_t j) const {
        // branch-free lower bound with a fixed step count: every probe index
        // is clamped into the row (the select discards out-of-range probes)
        if (nm == 0) return -1;
        int pos = 0;
        for (int st = steps - 1; st >= 0; st--) {
            const int q = pos + (1 << st);
            const int32_t v = at(min(q, nm) - 1);
            pos = (q <= nm && v < j) ? q : pos;
        }
        const int32_t v = at(min(pos, nm - 1));
        return (pos < nm && v == j) ? pos : -1;
    }
};

// Branch-free MSA probe for the order-free kinds: every step predicated,
// 32-bit shared-window addresses, no divergence (the lazy rule holds: the
// B value of a product is loaded only when its column survives the mask).
template <int KIND, bool NUMERIC>
struct MsaProber {
    uint32_t bits_s, cnt_s, val_s;     // bits_s: packed (rank << 16 | 16 column bits) words
    int32_t lo;                        // window start, a multiple of 16
    uint32_t guard;                    // offset of the all-zero guard word (multiple of 16)
    uint32_t dummy_s;                  // this lane's scratch word (MM_RED_ALL)
    const void* b_val;
    unsigned evaluated;
    // U products at once, stage by stage, so the shared loads of the U
    // products are in flight together (ILP) instead of one dependency chain
    // after another.
    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
#ifdef MM_EXPERIMENT_NOPROBE
        // profiling-only build (tools/): enumerate and load products, skip the accumulator
#pragma unroll
        for (int u = 0; u < U; u++) evaluated += (j[u] != EMPTY_KEY);
        return;
#endif
        // word = (rank of the group's first mask column << 16) | column bits.
        // t = word << (31 - c) moves column c's bit to the sign and drops both
        // the columns above c and the rank half, so hit = (t < 0) and the slot
        // is rank + popc(t) - 1 (the -1 is folded into the slot base).
        // Offsets outside the window (and EMPTY_KEY) clamp onto the guard word.
        uint32_t word[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t off = min((uint32_t)(j[u] - lo), guard);
            uint32_t addr;   // bits_s + 4 * (off >> 4) as SHF + LEA (ptxas otherwise emits SHF, LOP3, IADD)
            asm("{\n\t.reg .u32 q;\n\tshr.u32 q, %1, 4;\n\tmad.lo.u32 %0, q, 4, %2;\n\t}"
                : "=r"(addr) : "r"(off), "r"(bits_s));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(word[u]) : "r"(addr));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            // shift 31 - (j & 15) = (~j | 16) mod 32: one LOP3 + a wrapping funnel shift
            uint32_t t;
            asm("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(t) : "r"(0u), "r"(word[u]), "r"(~(uint32_t)j[u] | 16u));
            const uint32_t slot = (word[u] >> 16) + __popc(t);     // rank + 1
            const bool hit = (int32_t)t < 0;
            if (KIND == 0) {
                // plus-pair: the evaluated count is the sum of the slot counts,
                // taken when the row is gathered
                if (NUMERIC)
#ifndef MM_RED_PRED
                    // every lane issues the RED: a miss counts into its own
                    // dummy word, so ptxas needs no branch around the atomic
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t.reg .u32 ad;\n\t"
                        "setp.lt.s32 ph, %0, 0;\n\t"
                        "selp.u32 ad, %1, %2, ph;\n\t"
                        "red.shared.add.u32 [ad], 1;\n\t}" ::"r"(t),
                        "r"(cnt_s - 4u + (slot << 2)), "r"(dummy_s)
                        : "memory");
#else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.lt.s32 ph, %0, 0;\n\t"
                        "@ph red.shared.add.u32 [%1], 1;\n\t}" ::"r"(t),
                        "r"(cnt_s - 4u + (slot << 2))
                        : "memory");
#endif
                else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.lt.s32 ph, %0, 0;\n\t"
                        "@ph st.shared.u32 [%1], 1;\n\t}" ::"r"(t),
                        "r"(cnt_s - 4u + (slot << 2))
                        : "memory");
            } else if (hit) {
                evaluated++;
                if (NUMERIC) {
                    const long long prod = a[u] * ((const long long*)b_val)[s[u]];
                    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(val_s - 8u + (slot << 3)), "l"(prod) : "memory");
                }
                asm volatile("st.shared.u32 [%0], 1;" ::"r"(cnt_s - 4u + (slot << 2)) : "memory");
            }
        }
    }
    __device__ __forceinline__ void drain() {}
};

template <int KIND, bool NUMERIC, class R>
struct RankProber {
    R r;
    RankSlots<KIND> sl;
    const void* b_val;
    unsigned evaluated;
    __device__ __forceinline__ void put(int32_t j, long long a, long long s) {
        if (j == EMPTY_KEY) return;
        const int k = r.rank(j);
        if (k >= 0) {
            evaluated++;
            rank_accumulate<KIND, NUMERIC>(sl, k, a, b_val, s);
        }
    }
    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
#pragma unroll
        for (int u = 0; u < U; u++) put(j[u], a[u], s[u]);
    }
    __device__ __forceinline__ void drain() {}
};

template <class R>
struct RankLocatorF64 {
    R r;
    int32_t* cnt;
    double* vals;
    __device__ __forceinline__ int locate(int32_t j) { return r.rank(j); }
    __device__ __forceinline__ void fold(int k, double prod) {
        if (cnt[k] == 0) {
            vals[k] = prod;
            cnt[k] = 1;
        } else {
            vals[k] += prod;
        }
    }
    __device__ __forceinline__ void mark(int k) { cnt[k] = 1; }
};

// Per-group region: [val: 8*NM if KIND != 0][cnt: 4*NM]
//   MSA shared tiers: [packed words 4*(2W' + 4)]  (16 columns + 16-bit rank each;
//                      window start aligned down to 16 columns, plus an all-zero guard word)
//   MSA global tier:  [bits 4*W'][pre 4*W' + 16]   MCA: [mask 4*NM]
// W = 32-column words spanned by the mask window, W' = W rounded up to even.
__host__ __device__ constexpr size_t rank_region_bytes_rt(int kind, bool msa, int64_t words, int64_t nm) {
    return (size_t)(kind == 0 ? 0 : 8) * nm + 4 * (size_t)nm +
           (msa ? 8 * (size_t)(((words + 1) & ~1ll) + 2) : 4 * (size_t)nm);
}
template <int KIND>
__host__ __device__ constexpr size_t rank_region_bytes(bool msa, bool, int64_t words, int64_t nm) {
    return rank_region_bytes_rt(KIND, msa, words, nm);
}
__host__ __device__ constexpr int msa_words16(int words_max) { return 2 * (((words_max + 1) & ~1) + 2); }

template <int GW, int KIND, bool MSA, bool NUMERIC, bool SMEM>
__device__ __forceinline__ void rank_row(const Prob& p, const Out& o, unsigned char* region, int nm_max,
                                         int words_max, uint32_t dummy_s,
                                         const RowInfo& ri, int gt, int bar_id, int* s_warp, BatchSmem bsm,
                                         unsigned long long& evaluated) {
    constexpr int GT = GW * 32;
    const int lane = gt & 31;
    const int64_t i = ri.i, as = ri.as, ae = ri.ae, ms = ri.ms, me = ri.me;
    const int nm = (int)(me - ms);
    RankSlots<KIND> sl;
    sl.val = KIND == 0 ? nullptr : (unsigned long long*)region;
    sl.cnt = (int32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)nm_max));
    unsigned char* aux = (unsigned char*)(sl.cnt + nm_max);
    const int32_t lo = MSA && SMEM ? p.m_idx[ms] & ~15 : p.m_idx[ms];
    const int32_t hi = p.m_idx[me - 1];
    uint32_t* bits = (uint32_t*)aux;          // all-zero on entry (cleared by the previous row)
    int32_t* pre = (int32_t*)(aux + 4 * (size_t)(((words_max + 1) & ~1) + 2));   // global tier only
    int32_t* mrow = (int32_t*)aux;

    // 1. clear slots, 2. mark the mask row
    for (int r = gt; r < nm; r += GT) {
        sl.cnt[r] = 0;
        if (KIND == 1) sl.val[r] = 0ull;
    }
    group_bar(bar_id, GT);
    for (int r = gt; r < nm; r += GT) {
        const int32_t j = p.m_idx[ms + r];
        if (MSA && SMEM) {
            const uint32_t off = (uint32_t)(j - lo);
            const uint32_t w = off >> 4;
            const bool first = r == 0 || (((uint32_t)(p.m_idx[ms + r - 1] - lo)) >> 4) != w;
            atomicOr(bits + w, (1u << (off & 15u)) | (first ? (uint32_t)r << 16 : 0u));
        } else if (MSA) {
            const uint32_t off = (uint32_t)(j - lo);
            const uint32_t w = off >> 5;
            atomicOr(bits + w, 1u << (off & 31u));
            if (r == 0 || (((uint32_t)(p.m_idx[ms + r - 1] - lo)) >> 5) != w) pre[w] = r;
        } else {
            mrow[r] = j;
        }
    }
    group_bar(bar_id, GT);

    // 3. products
    // ordered float64 in a group: warp wg folds the columns of mask ranks
    // [wg nm/GW, (wg+1) nm/GW) — the same ranks it gathers in step 4
    int32_t c_lo = INT32_MIN, c_hi = INT32_MAX;
    bool idle = false;
    if (KIND == 2 && GW > 1) {
        const int wg = gt >> 5;
        const int r0 = (int)(((long long)nm * wg) / GW), r1 = (int)(((long long)nm * (wg + 1)) / GW);
        idle = r0 == r1;
        c_lo = wg == 0 ? INT32_MIN : p.m_idx[ms + r0];
        c_hi = r1 < nm ? p.m_idx[ms + r1] : INT32_MAX;
    }
    if (MSA) {
        if (KIND == 2) {
            if (idle) {
            } else if (SMEM) {
                MsaPacked rb{bits, lo, (uint32_t)(hi - lo)};
                RankLocatorF64<MsaPacked> loc{rb, sl.cnt, (double*)sl.val};
                evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane, c_lo, c_hi);
            } else {
                MsaBits<int32_t> rb{bits, pre, lo, (uint32_t)(hi - lo)};
                RankLocatorF64<MsaBits<int32_t>> loc{rb, sl.cnt, (double*)sl.val};
                evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane, c_lo, c_hi);
            }
        } else {
          if (!SMEM) {
            MsaBits<int32_t> rb{bits, pre, lo, (uint32_t)(hi - lo)};
            RankProber<KIND, NUMERIC, MsaBits<int32_t>> pr{rb, sl, p.b_val, 0u};
            flat_products<GW, KIND>(p, pr, as, ae, gt, bar_id, s_warp, bsm);
            evaluated += pr.evaluated;
          } else {
            MsaProber<KIND, NUMERIC> pr;
            pr.bits_s = (uint32_t)__cvta_generic_to_shared(bits);
            pr.cnt_s = (uint32_t)__cvta_generic_to_shared(sl.cnt);
            pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(sl.val);
            pr.lo = lo;
            pr.guard = (((uint32_t)(hi - lo) >> 4) + 1) << 4;
            pr.dummy_s = dummy_s;
            pr.b_val = p.b_val;
            pr.evaluated = 0u;
            flat_products<GW, KIND>(p, pr, as, ae, gt, bar_id, s_warp, bsm);
            evaluated += pr.evaluated;
          }
        }
    } else {
        int steps = 0;
        while ((1 << steps) <= nm) steps++;
        McaRow<SMEM> rb(mrow, nm, steps);
        if (KIND == 2) {
            RankLocatorF64<McaRow<SMEM>> loc{rb, sl.cnt, (double*)sl.val};
            if (!idle) evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane, c_lo, c_hi);
        } else {
            RankProber<KIND, NUMERIC, McaRow<SMEM>> pr{rb, sl, p.b_val, 0u};
            flat_products<GW, KIND>(p, pr, as, ae, gt, bar_id, s_warp, bsm);
            evaluated += pr.evaluated;
        }
    }
    group_bar(bar_id, GT);

    // 4. gather in mask order: warp w owns ranks [w nm/GW, (w+1) nm/GW)
    const int64_t w0 = NUMERIC ? o.off[i] : 0;
    const int wg = gt >> 5;
    const int r_lo = (int)(((long long)nm * wg) / GW), r_hi = (int)(((long long)nm * (wg + 1)) / GW);
    int mine = 0;
    for (int r = r_lo + lane; r < r_hi; r += 32) {
        mine += sl.cnt[r] > 0;
        if (MSA && SMEM && KIND == 0 && NUMERIC) evaluated += (unsigned)sl.cnt[r];
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
    if (NUMERIC) {
        int run = before;
        for (int rb0 = r_lo; rb0 < r_hi; rb0 += 32) {
            const int r = rb0 + lane;
            const bool set = r < r_hi && sl.cnt[r] > 0;
            const unsigned bal = __ballot_sync(FULL, set);
            if (set) {
                const int64_t d = w0 + run + __popc(bal & lanemask_lt());
                o.idx[d] = p.m_idx[ms + r];
                if (KIND == 0) {
                    if (o.out_f64) ((double*)o.val)[d] = (double)sl.cnt[r];
                    else ((long long*)o.val)[d] = sl.cnt[r];
                } else {
                    ((unsigned long long*)o.val)[d] = sl.val[r];
                }
            }
            run += __popc(bal);
        }
    }
    if (gt == 0) o.row_nnz[i] = total;
    // 5. leave the bitmap all-zero for the next row (only the touched words)
    if (MSA)
        for (int r = gt; r < nm; r += GT) bits[((uint32_t)(p.m_idx[ms + r] - lo)) >> (SMEM ? 4 : 5)] = 0u;
    group_bar(bar_id, GT);
}

// Groups of GW warps fetch rows of one bin.  SMEM: the per-group region lives
// in dynamic shared memory, otherwise in one global slab per group (tier 3).
template <int GW, bool SMEM, int KIND, bool MSA, bool NUMERIC>
#ifndef MM_RANK_MINB
#define MM_RANK_MINB 5   // <= 51 registers: 5 blocks of 256 threads per SM (measured best on cfg2)
#endif
__global__ void __launch_bounds__(GW == 32 ? 1024 : (GW == 16 ? 512 : 256), GW <= 8 ? MM_RANK_MINB : 1)
k_push_rank(Prob p, Out o, Work wk, int words_max, int nm_max, unsigned char* gslab) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[16];
    __shared__ int s_warp[32];
    constexpr int GT = GW * 32;
    const int groups = blockDim.x / GT;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int bar_id = 1 + g;
    const size_t rbytes = (rank_region_bytes<KIND>(MSA, SMEM, words_max, nm_max) + 15) & ~(size_t)15;
    unsigned char* region = SMEM ? smem + (size_t)g * rbytes : gslab + ((size_t)blockIdx.x * groups + g) * rbytes;
    unsigned char* bbase = smem + (SMEM ? (size_t)groups * rbytes : 0) + (size_t)g * batch_bytes<GW, KIND>();
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    __shared__ uint32_t s_dummy[(GW == 32 ? 32 : (GW == 16 ? 16 : 8)) * 32];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
#ifdef MM_STAGE_TMA
    stage_init();
#endif
    unsigned long long evaluated = 0;
    if (MSA) {
        uint32_t* bits = (uint32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)nm_max) + 4 * (size_t)nm_max);
        for (int w = gt; w < (SMEM ? msa_words16(words_max) : words_max); w += GT) bits[w] = 0u;
    }
    RowFetcher<GW> rf;
    if (wk.count < 4 * (int)(gridDim.x * (blockDim.x / (32 * GW)))) rf.per = 1;   // few rows: one per fetch
    RowInfo ri;
    while (rf.next(p, wk, gt, bar_id, s_row + g, ri))
        rank_row<GW, KIND, MSA, NUMERIC, SMEM>(p, o, region, nm_max, words_max, dummy_s, ri, gt, bar_id,
                                               s_warp + g * GW, bsm, evaluated);
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

}  // namespace mm

namespace mm {

// ---------------------------------------------------------------------------
// Windowed MSA for hub rows (plain masks, order-free kinds): the mask row is
// cut into column windows whose packed bitmap (16 columns + 16-bit rank per
// word) and rank slots fit a fixed shared-memory region; each window keeps
// only the products whose column falls inside it (each B row's sub-range,
// resumed from a per-A-entry cursor), so a 163,558-entry mask row runs in
// ~30 windows with the one-load MSA probe.  Reference semantics: MSA
// (_kernels.py:30-87) restricted to a column range per pass; windows run in
// column order and append, so C stays in mask order.
// ---------------------------------------------------------------------------
constexpr int MSAW_GW = 16;
constexpr int MSAW_WORDS = 8192;   // packed words per window (131,072 columns)
constexpr int MSAW_SLOTS = 6144;   // mask entries per window

__host__ __device__ constexpr size_t msaw_region_bytes(int kind) {
    return (size_t)(kind == 0 ? 0 : 8) * MSAW_SLOTS + 4 * (size_t)MSAW_SLOTS + 4 * (size_t)(MSAW_WORDS + 4);
}

template <int KIND, bool NUMERIC>
__global__ void __launch_bounds__(MSAW_GW * 32, 2) k_push_msaw(Prob p, Out o, Work wk, unsigned char* gslab) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[1];
    __shared__ int s_warp[MSAW_GW];
    __shared__ int s_r1;
    constexpr int GT = MSAW_GW * 32;
    const int gt = threadIdx.x;
    const int bar_id = 1;
    unsigned char* region = smem;
    unsigned long long* val = (unsigned long long*)region;                     // KIND 1
    int32_t* cnt = (int32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)MSAW_SLOTS));
    uint32_t* words = (uint32_t*)(cnt + MSAW_SLOTS);
    BatchSmem bsm = bind_batch<MSAW_GW, KIND>(smem + ((msaw_region_bytes(KIND) + 15) & ~(size_t)15));
    __shared__ uint32_t s_dummy[GT];
    const uint32_t dummy_s = (uint32_t)__cvta_generic_to_shared(s_dummy + threadIdx.x);
    int64_t* cur = gslab && p.cursor_stride ? (int64_t*)gslab + (size_t)blockIdx.x * (size_t)p.cursor_stride : nullptr;
    for (int w = gt; w < MSAW_WORDS + 4; w += GT) words[w] = 0u;
    group_bar(bar_id, GT);
    unsigned long long evaluated = 0;
    RowFetcher<MSAW_GW> rf;
    RowInfo ri;
    while (rf.next(p, wk, gt, bar_id, s_row, ri)) {
        const int64_t ms = ri.ms, nm = ri.me - ri.ms;
        const int64_t w0 = NUMERIC ? o.off[ri.i] : 0;
        int64_t* rcur = ri.ae - ri.as <= p.cursor_stride ? cur : nullptr;
        int64_t total = 0;
        for (int64_t r0 = 0; r0 < nm;) {
            const int32_t lo = p.m_idx[ms + r0] & ~15;
            if (gt == 0) {
                // the window: mask entries with column < lo + 16 * (MSAW_WORDS - 1), at most MSAW_SLOTS
                const int64_t cap = nm - r0 < MSAW_SLOTS ? nm - r0 : MSAW_SLOTS;
                const int64_t lim = (int64_t)lo + 16ll * (MSAW_WORDS - 1);
                int64_t n = cap;
                if ((int64_t)p.m_idx[ms + r0 + cap - 1] >= lim)
                    n = lower_bound_range(p.m_idx, ms + r0, ms + r0 + cap, (int32_t)lim) - (ms + r0);
                s_r1 = (int)(n > 0 ? n : 1);
            }
            group_bar(bar_id, GT);
            const int ns = s_r1;
            group_bar(bar_id, GT);
            const int64_t r1 = r0 + ns;
            const int32_t hi = p.m_idx[ms + r1 - 1];
            // 1. clear slots, 2. mark the window's mask entries
            for (int r = gt; r < ns; r += GT) {
                cnt[r] = 0;
                if (KIND == 1) val[r] = 0ull;
            }
            group_bar(bar_id, GT);
            for (int r = gt; r < ns; r += GT) {
                const int32_t j = p.m_idx[ms + r0 + r];
                const uint32_t off = (uint32_t)(j - lo);
                const uint32_t w = off >> 4;
                const bool first = r == 0 || (((uint32_t)(p.m_idx[ms + r0 + r - 1] - lo)) >> 4) != w;
                atomicOr(words + w, (1u << (off & 15u)) | (first ? (uint32_t)r << 16 : 0u));
            }
            group_bar(bar_id, GT);
            // 3. products whose column lies in the window's range
            const int32_t c_lo = r0 == 0 ? INT32_MIN : p.m_idx[ms + r0];
            const int32_t c_hi = r1 < nm ? p.m_idx[ms + r1] : INT32_MAX;
            MsaProber<KIND, NUMERIC> pr;
            pr.bits_s = (uint32_t)__cvta_generic_to_shared(words);
            pr.cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
            pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(val);
            pr.lo = lo;
            pr.guard = (((uint32_t)(hi - lo) >> 4) + 1) << 4;
            pr.dummy_s = dummy_s;
            pr.b_val = p.b_val;
            pr.evaluated = 0u;
            flat_products<MSAW_GW, KIND>(p, pr, ri.as, ri.ae, gt, bar_id, s_warp, bsm, c_lo, c_hi, nullptr, 0,
                                         rcur);
            evaluated += pr.evaluated;
            group_bar(bar_id, GT);
            // 4. gather the window in mask order, appended to the row
            int running = 0;
            for (int rb = 0; rb < ns; rb += GT) {
                const int r = rb + gt;
                const bool set = r < ns && cnt[r] > 0;
                if (KIND == 0 && NUMERIC && set) evaluated += (unsigned)cnt[r];
                int tot;
                const int pos = group_prefix<MSAW_GW>(set, &tot, s_warp, bar_id, gt);
                if (NUMERIC && set) {
                    const int64_t d = w0 + total + running + pos;
                    o.idx[d] = p.m_idx[ms + r0 + r];
                    if (KIND == 0) {
                        if (o.out_f64) ((double*)o.val)[d] = (double)cnt[r];
                        else ((long long*)o.val)[d] = cnt[r];
                    } else {
                        ((unsigned long long*)o.val)[d] = val[r];
                    }
                }
                running += tot;
            }
            total += running;
            // 5. leave the bitmap all-zero
            for (int r = gt; r < ns; r += GT) words[((uint32_t)(p.m_idx[ms + r0 + r] - lo)) >> 4] = 0u;
            group_bar(bar_id, GT);
            r0 = r1;
        }
        if (gt == 0) o.row_nnz[ri.i] = total;
    }
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

}  // namespace mm
