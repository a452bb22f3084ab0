// Push path, MSA with a sparse (two-level) window bitmap.
//
// Same accumulator as the MSA tiers of push_rank.cuh — a bitmap over the mask
// row's columns plus mask-rank slots (reference msa_numeric, _kernels.py:30-87)
// — for rows whose mask is narrow but spread over a wide column window, where
// a dense bitmap would not fit in shared memory.  The window is cut into
// 1024-column blocks; a u16 directory maps each block to a compact block of
// 32 bitmap words (+ u16 rank prefixes) holding only the blocks the mask
// touches.  A product costs two dependent shared loads (directory, word) and
// a bit test; a hit adds the prefix load, popc and one shared reduction.
// Plain masks only (see DESIGN.md §4 for the complement forms).
#pragma once
#include "common.cuh"
#include "product_loop.cuh"

namespace mm {

constexpr uint32_t SPARSE_NONE = 0xFFFFu;

template <int KIND>
__host__ __device__ constexpr size_t sparse_region_bytes(int64_t d_max, int64_t blk_max, int64_t nm) {
    return (size_t)(KIND == 0 ? 0 : 8) * nm + 4 * (size_t)nm + 2 * (size_t)((d_max + 1) & ~1ll) +
           4 * 32 * (size_t)blk_max + 2 * 32 * (size_t)blk_max;
}

// slot of column j (generic form, used by the ordered float64 path)
struct SparseBits {
    const uint16_t* dir;
    const uint32_t* words;
    const uint16_t* pre;
    int32_t lo;
    uint32_t span;
    __device__ __forceinline__ int rank(int32_t j) const {
        const uint32_t off = (uint32_t)(j - lo);
        if (off > span) return -1;
        const uint32_t d = dir[off >> 10];
        if (d == SPARSE_NONE) return -1;
        const uint32_t wi = (d << 5) | ((off >> 5) & 31u);
        const uint32_t word = words[wi];
        const uint32_t b = off & 31u;
        if (!((word >> b) & 1u)) return -1;
        return (int)pre[wi] + __popc(word & ((1u << b) - 1u));
    }
};

template <int KIND, bool NUMERIC>
struct SparseProber {
    uint32_t dir_s, words_s, pre_s, cnt_s, val_s;
    int32_t lo;
    uint32_t span;
    const void* b_val;
    unsigned evaluated;
    template <int U>
    __device__ __forceinline__ void put_batch(const int32_t* j, const long long* a, const long long* s) {
        uint32_t off[U], d[U], wi[U], word[U], pre[U], hit[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            off[u] = (uint32_t)(j[u] - lo);
            d[u] = SPARSE_NONE;
            word[u] = 0u;
            pre[u] = 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            asm volatile(
                "{\n\t.reg .pred pin;\n\t"
                "setp.le.u32 pin, %1, %2;\n\t"
                "@pin ld.shared.u16 %0, [%3];\n\t}"
                : "+r"(d[u])
                : "r"(off[u]), "r"(span), "r"(dir_s + ((off[u] >> 10) << 1)));
#pragma unroll
        for (int u = 0; u < U; u++) {
            wi[u] = (d[u] << 5) | ((off[u] >> 5) & 31u);
            asm volatile(
                "{\n\t.reg .pred pv;\n\t"
                "setp.ne.u32 pv, %1, 65535;\n\t"
                "@pv ld.shared.u32 %0, [%2];\n\t}"
                : "+r"(word[u])
                : "r"(d[u]), "r"(words_s + (wi[u] << 2)));
        }
#pragma unroll
        for (int u = 0; u < U; u++) hit[u] = (word[u] >> (off[u] & 31u)) & 1u;
#pragma unroll
        for (int u = 0; u < U; u++)
            asm volatile(
                "{\n\t.reg .pred ph;\n\t"
                "setp.ne.u32 ph, %1, 0;\n\t"
                "@ph ld.shared.u16 %0, [%2];\n\t}"
                : "+r"(pre[u])
                : "r"(hit[u]), "r"(pre_s + (wi[u] << 1)));
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t rank = pre[u] + __popc(word[u] & ((1u << (off[u] & 31u)) - 1u));
            evaluated += hit[u];
            if (KIND == 0) {
                if (NUMERIC)
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ne.u32 ph, %0, 0;\n\t"
                        "@ph red.shared.add.u32 [%1], 1;\n\t}" ::"r"(hit[u]),
                        "r"(cnt_s + (rank << 2))
                        : "memory");
                else
                    asm volatile(
                        "{\n\t.reg .pred ph;\n\t"
                        "setp.ne.u32 ph, %0, 0;\n\t"
                        "@ph st.shared.u32 [%1], 1;\n\t}" ::"r"(hit[u]),
                        "r"(cnt_s + (rank << 2))
                        : "memory");
            } else if (hit[u]) {
                if (NUMERIC) {
                    const long long prod = a[u] * ((const long long*)b_val)[s[u]];
                    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(val_s + (rank << 3)), "l"(prod) : "memory");
                }
                asm volatile("st.shared.u32 [%0], 1;" ::"r"(cnt_s + (rank << 2)) : "memory");
            }
        }
    }
    __device__ __forceinline__ void drain() {}
};

template <class R>
struct SparseLocatorF64 {
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

template <int GW, int KIND, bool NUMERIC>
__device__ __forceinline__ void msas_row(const Prob& p, const Out& o, unsigned char* region, int nm_max,
                                         int d_max, int blk_max, const RowInfo& ri, int gt, int bar_id,
                                         int* s_warp, BatchSmem bsm, unsigned long long& evaluated) {
    constexpr int GT = GW * 32;
    const int lane = gt & 31;
    const int wg = gt >> 5;
    const int64_t i = ri.i, as = ri.as, ae = ri.ae, ms = ri.ms, me = ri.me;
    const int nm = (int)(me - ms);
    unsigned long long* val = KIND == 0 ? nullptr : (unsigned long long*)region;
    int32_t* cnt = (int32_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)nm_max));
    uint16_t* dir = (uint16_t*)(cnt + nm_max);
    uint32_t* words = (uint32_t*)(dir + ((d_max + 1) & ~1));
    uint16_t* pre = (uint16_t*)(words + 32 * (size_t)blk_max);
    const int32_t lo = p.m_idx[ms];
    const int32_t hi = p.m_idx[me - 1];
    const int32_t* m = p.m_idx + ms;

    // 1. clear slots; 2. directory of the touched 1024-column blocks (mask
    // entries are sorted, so compact block ids follow a scan of block starts)
    for (int r = gt; r < nm; r += GT) {
        cnt[r] = 0;
        if (KIND == 1) val[r] = 0ull;
    }
    int running = 0;
    for (int base = 0; base < nm; base += GT) {
        const int r = base + gt;
        uint32_t off = 0;
        bool first = false;
        if (r < nm) {
            off = (uint32_t)(m[r] - lo);
            first = r == 0 || ((uint32_t)(m[r - 1] - lo) >> 10) != (off >> 10);
        }
        int tot;
        const int pos = group_prefix<GW>(first, &tot, s_warp, bar_id, gt);
        if (first) dir[off >> 10] = (uint16_t)(running + pos);
        running += tot;
    }
    group_bar(bar_id, GT);
    for (int r = gt; r < nm; r += GT) {
        const uint32_t off = (uint32_t)(m[r] - lo);
        const uint32_t wi = ((uint32_t)dir[off >> 10] << 5) | ((off >> 5) & 31u);
        atomicOr(words + wi, 1u << (off & 31u));
        if (r == 0 || ((uint32_t)(m[r - 1] - lo) >> 5) != (off >> 5)) pre[wi] = (uint16_t)r;
    }
    group_bar(bar_id, GT);

    // 3. products
    SparseBits sb{dir, words, pre, lo, (uint32_t)(hi - lo)};
    if (KIND == 2) {
        SparseLocatorF64<SparseBits> loc{sb, cnt, (double*)val};
        evaluated += ordered_products_f64<NUMERIC>(p, loc, as, ae, lane);
    } else {
        SparseProber<KIND, NUMERIC> pr;
        pr.dir_s = (uint32_t)__cvta_generic_to_shared(dir);
        pr.words_s = (uint32_t)__cvta_generic_to_shared(words);
        pr.pre_s = (uint32_t)__cvta_generic_to_shared(pre);
        pr.cnt_s = (uint32_t)__cvta_generic_to_shared(cnt);
        pr.val_s = KIND == 0 ? 0u : (uint32_t)__cvta_generic_to_shared(val);
        pr.lo = lo;
        pr.span = (uint32_t)(hi - lo);
        pr.b_val = p.b_val;
        pr.evaluated = 0u;
        flat_products<GW, KIND>(p, pr, as, ae, gt, bar_id, s_warp, bsm);
        evaluated += pr.evaluated;
    }
    group_bar(bar_id, GT);

    // 4. gather in mask order (warp w owns ranks [w nm/GW, (w+1) nm/GW))
    const int64_t w0 = NUMERIC ? o.off[i] : 0;
    const int r_lo = (int)(((long long)nm * wg) / GW), r_hi = (int)(((long long)nm * (wg + 1)) / GW);
    int mine = 0;
    for (int r = r_lo + lane; r < r_hi; r += 32) mine += cnt[r] > 0;
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
            const bool set = r < r_hi && cnt[r] > 0;
            const unsigned bal = __ballot_sync(FULL, set);
            if (set) {
                const int64_t d = w0 + run + __popc(bal & lanemask_lt());
                o.idx[d] = m[r];
                if (KIND == 0) {
                    if (o.out_f64) ((double*)o.val)[d] = (double)cnt[r];
                    else ((long long*)o.val)[d] = cnt[r];
                } else {
                    ((unsigned long long*)o.val)[d] = val[r];
                }
            }
            run += __popc(bal);
        }
    }
    if (gt == 0) o.row_nnz[i] = total;
    // 5. leave words zero and the directory empty for the next row
    group_bar(bar_id, GT);
    for (int r = gt; r < nm; r += GT) {
        const uint32_t off = (uint32_t)(m[r] - lo);
        words[((uint32_t)dir[off >> 10] << 5) | ((off >> 5) & 31u)] = 0u;
    }
    group_bar(bar_id, GT);
    for (int r = gt; r < nm; r += GT) dir[((uint32_t)(m[r] - lo)) >> 10] = (uint16_t)SPARSE_NONE;
    group_bar(bar_id, GT);
}

template <int GW, int KIND, bool NUMERIC>
__global__ void __launch_bounds__(256) k_push_msas(Prob p, Out o, Work wk, int d_max, int blk_max, int nm_max) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int s_row[8];
    __shared__ int s_warp[8];
    constexpr int GT = GW * 32;
    const int groups = blockDim.x / GT;
    const int g = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int bar_id = 1 + g;
    const size_t rbytes = (sparse_region_bytes<KIND>(d_max, blk_max, nm_max) + 15) & ~(size_t)15;
    unsigned char* region = smem + (size_t)g * rbytes;
    unsigned char* bbase = smem + (size_t)groups * rbytes + (size_t)g * batch_bytes<GW, KIND>();
    BatchSmem bsm = bind_batch<GW, KIND>(bbase);
    {
        uint16_t* dir = (uint16_t*)(region + (KIND == 0 ? 0 : 8 * (size_t)nm_max) + 4 * (size_t)nm_max);
        uint32_t* words = (uint32_t*)(dir + ((d_max + 1) & ~1));
        for (int q = gt; q < d_max; q += GT) dir[q] = (uint16_t)SPARSE_NONE;
        for (int q = gt; q < 32 * blk_max; q += GT) words[q] = 0u;
    }
    unsigned long long evaluated = 0;
#ifdef MM_STAGE_TMA
    stage_init();
#endif
    RowFetcher<GW> rf;
    if (wk.count < 4 * (int)(gridDim.x * (blockDim.x / (32 * GW)))) rf.per = 1;   // few rows: one per fetch
    RowInfo ri;
    while (rf.next(p, wk, gt, bar_id, s_row + g, ri))
        msas_row<GW, KIND, NUMERIC>(p, o, region, nm_max, d_max, blk_max, ri, gt, bar_id, s_warp + g * GW, bsm,
                                    evaluated);
    if (NUMERIC) {
        const long long e = warp_sum_ll((long long)evaluated);
        if ((threadIdx.x & 31) == 0 && e) atomicAdd(o.evaluated, (unsigned long long)e);
    }
}

}  // namespace mm
