// Row analysis, binning and row-list construction.
//
// Reference: flops_per_row (multiply.py:103-108), the per-row hash capacity
// rule (multiply.py:220-226), one_phase_bounds (multiply.py:230-233) and the
// empty-row short-circuits of every kernel (_kernels.py:42-44,143-145,284-286,
// 441-443).  On the GPU the same per-row quantities decide which kernel tier
// computes the row: a row's tier depends only on the row itself, so results
// are independent of how rows are partitioned across launches or devices.
#pragma once
#include "common.cuh"

namespace mm {

// Kernel families (the paper's accumulators) + the pull path.
enum Family : int { FAM_HASH = 0, FAM_MSA = 1, FAM_MCA = 2, FAM_HEAP = 3, FAM_PULL = 4, FAM_AUTO = 5 };

// Hash-family modes.
enum Mode : int { MODE_PLAIN = 0, MODE_CTAB = 1, MODE_CSRCH = 2 };

// Bins.  0 = nothing to compute (row_nnz = 0).  Hash bins: 7 per mode =
// tiers 0..2 x {small table (<= 2^CAPC_LG slots), large table} + the
// global-memory tier 3; the table class keeps the shared-memory footprint of
// a launch (and so its occupancy) sized for the rows it actually holds.
constexpr int CAPC_LG = 9;
enum Bin : int {
    BIN_EMPTY = 0,
    BIN_HASH0 = 1,    // + mode*7 + (tier < 3 ? tier*2 + class : 6)
    BIN_PULL = 22,
    BIN_MSA0 = 23,    // + tier (0..3)
    BIN_MCA0 = 27,    // + tier
    BIN_HEAP0 = 31,   // + tier
    BIN_SINGLE = 35,  // one A entry: filtered, scaled copy of B_k (auto)
    BIN_MSAS0 = 36,   // + tier (0..2): MSA with a sparse two-level window bitmap
    BIN_MSAD0 = 39,   // + tier (0..2): MSA with a dense per-column window (push_dense.cuh)
    BIN_MSADC0 = 42,  // + tier (0..2): complemented MSA over every column (narrow outputs)
    BIN_PULL_LANE = 45,  // pull, one lane per mask entry (short masks, short A rows and B columns)
    BIN_F64D = 46,       // ordered float64, plain hash with deferred hits (push_f64_defer.cuh)
    BIN_MSAW = 47,       // MSA plan, plain order-free rows too wide for the shared tiers: windowed MSA (push_rank.cuh)
    NBINS = 48
};
__host__ __device__ constexpr bool is_msadc_bin(int b) { return b >= BIN_MSADC0 && b < BIN_MSADC0 + 3; }
__host__ __device__ constexpr bool is_msas_bin(int b) { return b >= BIN_MSAS0 && b < BIN_MSAS0 + 3; }
__host__ __device__ constexpr bool is_msad_bin(int b) { return b >= BIN_MSAD0 && b < BIN_MSAD0 + 3; }
__host__ __device__ constexpr bool is_msa_bin(int b) { return b >= BIN_MSA0 && b < BIN_MSA0 + 4; }
__host__ __device__ constexpr bool is_mca_bin(int b) { return b >= BIN_MCA0 && b < BIN_MCA0 + 4; }
__host__ __device__ constexpr bool is_heap_bin(int b) { return b >= BIN_HEAP0 && b < BIN_HEAP0 + 4; }

__host__ __device__ constexpr int hash_bin(int mode, int tier, int cls) {
    return BIN_HASH0 + mode * 7 + (tier < 3 ? tier * 2 + cls : 6);
}
__host__ __device__ constexpr bool is_hash_bin(int b) { return b >= BIN_HASH0 && b < BIN_HASH0 + 21; }
__host__ __device__ constexpr int hash_bin_mode(int b) { return (b - BIN_HASH0) / 7; }
__host__ __device__ constexpr int hash_bin_tier(int b) {
    return ((b - BIN_HASH0) % 7) == 6 ? 3 : ((b - BIN_HASH0) % 7) / 2;
}

// Hash tiers: group width (warps) and the largest table (log2 entries) each
// tier keeps in shared memory.  Tier 3 keeps its table in global memory.
__host__ __device__ constexpr int tier_gw(int t) { return t == 0 ? 1 : (t == 1 ? 4 : (t == 2 ? 16 : 32)); }
__host__ __device__ constexpr int tier_cap_lg_pair(int t) { return t == 0 ? 10 : (t == 1 ? 13 : (t == 2 ? 14 : 30)); }
__host__ __device__ constexpr int tier_cap_lg_val(int t) { return t == 0 ? 10 : (t == 1 ? 12 : (t == 2 ? 13 : 30)); }
constexpr int64_t TIER_FLOPS0 = 8192;
constexpr int64_t TIER_FLOPS1 = 65536;
// Plain order-free hash rows stay in the 4-warp tier up to 8x more products (when their table
// fits it): cfg5 334.4 -> 316.8 ms at 2^19 (326.8 at 2^17, 325.6 at 2^20, 540 at 2^22), while the
// MSA tiers of cfg2 lose 11 % past 2^17 — hence a boundary of its own.
constexpr int64_t TIER_FLOPS1_HASH = 524288;

struct Summary {
    unsigned long long gen_flops;
    unsigned long long bound_total;
    unsigned long long evaluated;
    long long total_nnz;
    unsigned long long bin_flops[NBINS];
    int bin_count[NBINS];
    int bin_cap_lg[NBINS];
    int bin_words[NBINS];    // MSA: largest mask window (32-column words) in the bin
    int bin_nmmax[NBINS];    // MSA / MCA / heap: largest mask row in the bin
    int max_na;
    int max_nm;
    int flag;
    int pad;
};

struct AnalyzeParams {
    long long tier_flops0;   // rows with <= this many products: 1-warp tier
    long long tier_flops1;   // ... 4-warp tier; above: 16-warp tier
    long long tier_flops1_hash;   // the same boundary for plain order-free hash rows (see TIER_FLOPS1_HASH)
    int capc_lg;             // table-size class boundary (log2 slots)
    int load_shift;          // preferred table size = keys << load_shift
    int load_shift_wide;     // same for plain rows of the 16-warp tier
    int rank_budget[3];      // MSA / MCA shared bytes per group allowed in tiers 0..2
    int auto_mca_nm;         // AUTO: 1-warp rows whose MSA window is too wide use MCA if nm <= this
    int family;      // Family
    int comp;        // complemented mask
    int ordered;     // fp64 plus-times: single-warp ordered accumulation
    int pair;        // plus-pair (4-byte table values)
    int vbytes;      // value bytes read per operand entry (0 plus-pair, 8 otherwise)
    int has_bt;      // B^T (CSC) available
    const int64_t* done;   // rows with done[i] >= 0 were computed already (direct pass): skipped
    const int32_t* b_len;  // nnz(B_k*) per row of B (k_row_len), or null: the analysis gathers one
                           // 4-byte length per A entry instead of two 8-byte offsets (half the sectors)
};

// Row lengths of B as int32 (nnz(B) < 2^31 is validated).
__global__ void __launch_bounds__(256) k_row_len(int64_t nrows, const int64_t* ptr, int32_t* len) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
        len[i] = (int32_t)(ptr[i + 1] - ptr[i]);
}

template <bool BLEN>
__device__ __forceinline__ long long b_row_len(const Prob& p, const AnalyzeParams& ap, int32_t k) {
    return BLEN ? (long long)__ldg(ap.b_len + k) : (long long)(p.b_ptr[k + 1] - p.b_ptr[k]);
}

__host__ __device__ __forceinline__ int tier_cap_lg(int pair, int tier) {
    return pair ? tier_cap_lg_pair(tier) : tier_cap_lg_val(tier);
}

// Shared-memory bytes per row of the rank-slot accumulators.
__host__ __device__ constexpr int64_t msa_bytes(int64_t words, int64_t nm, int kind) {
    return 8 * words + 16 + (kind == 0 ? 4 : 12) * nm;   // shared tiers: 16 columns + 16-bit rank per word
}
// sparse window: u16 directory per 1024 columns + 32 words (+u16 prefixes) per touched block
__host__ __device__ constexpr int64_t msas_dir(int64_t words) { return ((words - 1) >> 5) + 1; }
__host__ __device__ constexpr int64_t msas_blocks(int64_t words, int64_t nm) {
    return nm < msas_dir(words) ? nm : msas_dir(words);
}
__host__ __device__ constexpr int64_t msas_bytes(int64_t words, int64_t nm, int kind) {
    return 2 * msas_dir(words) + 192 * msas_blocks(words, nm) + (kind == 0 ? 4 : 12) * nm;
}
// dense window: a state per column of the window plus a guard column
__host__ __device__ constexpr int64_t msad_bytes(int64_t words, int kind) {
    // budget accounting: the state (+ value) per window column; the guard
    // column on top is not charged (a 512-column window fits the 1-warp tier)
    return (kind == 0 ? 4 : 12) * (32 * words);
}
__host__ __device__ constexpr int64_t mca_bytes(int64_t nm, int kind) {
    return (kind == 0 ? 8 : 16) * nm;
}

// Largest mask row of the deferred-hit float64 bin (its table: 2^8..2^9 slots).
constexpr int64_t F64D_MAX_NM = 256;

// The symbolic pass of that bin runs the plain tier-0 hash kernel: its table size.
__device__ __forceinline__ int f64d_bin(int64_t nm, int* cap_lg_out) {
    const int lg = ceil_log2_i64(4 * nm);
    *cap_lg_out = lg < 5 ? 5 : lg;
    return BIN_F64D;
}

// Chooses the bin for a row and the table size (log2) the row will use.
// words = 32-column words spanned by the mask row (MSA window).
__device__ __forceinline__ int classify_row(const AnalyzeParams& ap, int64_t na, int64_t nm,
                                            int64_t flops, int64_t ncols, int64_t pull_cols,
                                            int64_t words, int* cap_lg_out, int64_t* aux_out) {
    *cap_lg_out = 0;
    *aux_out = words;
    if (flops == 0 || (!ap.comp && nm == 0)) return BIN_EMPTY;
    const int kind = ap.pair ? 0 : (ap.ordered ? 2 : 1);
    const int tf = flops <= ap.tier_flops0 ? 0 : (flops <= ap.tier_flops1 ? 1 : 2);
    // budget tier of the single-warp-only kernels (dense / sparse MSA) for
    // ordered float64; the rank and hash families split heavy ordered rows
    // over a group by output column (ordered_products_f64)
    const int tr = ap.ordered ? 0 : tf;
    int fam = ap.family;
    // one A entry, many products, a wide mask window: the bitmap filter (cfg4 shape)
    if (fam == FAM_AUTO && na == 1 && words >= 256 && 4 * words <= 98304) return BIN_SINGLE;
    if (fam == FAM_AUTO) {
        fam = FAM_HASH;
        if (!ap.comp) {
            // per-row byte cost model: push vs pull
            int64_t w = 4 + ap.vbytes;
            int64_t push = 16 * na + flops * w;
            int64_t pull = 16 * nm + (nm * na + pull_cols) * w;
            // ordered float64 rows push through the deferred-hit kernel at a
            // fraction of the in-order walk's cost: pull must win by 2.5x
            // (cfg3: d1 rows pull, d4 / d16 / d64 rows push)
            if (ap.has_bt && (ap.ordered ? (5 * pull) >> 1 : pull) < push) fam = FAM_PULL;
            // ordered float64 single-warp rows with short masks: the deferred-hit
            // kernel (mask filter, hits folded in k order afterwards)
            else if (ap.ordered && tf == 0 && nm <= F64D_MAX_NM) return f64d_bin(nm, cap_lg_out);
            // ordered float64 rows (one warp, k order): the rank search beats
            // both the bitmap and the hash for short mask rows
            else if (ap.ordered && nm <= 512 && msad_bytes(words, kind) > ap.rank_budget[tf]) fam = FAM_MCA;
            // push: the bitmap accumulator when the mask window is compact
            else if (msa_bytes(words, nm, kind) <= ap.rank_budget[tr]) fam = FAM_MSA;
            else if (tr == 0 && nm <= ap.auto_mca_nm) fam = FAM_MCA;
        }
    }
    if (fam == FAM_PULL) {
        // short masks, A rows and B^T columns: a lane per mask entry runs the merge
        if (nm <= 32 && na <= 128 && pull_cols <= 32 * nm) return BIN_PULL_LANE;
        return BIN_PULL;
    }
    if (fam == FAM_HEAP) {
        // plain: mask-rank slots in shared memory (tier 0) or global (tier 1);
        // complement rows with <= 32 A entries: sorted single-batch merge (2),
        // more A entries: the multi-iterator merge (3)
        if (!ap.comp) {
            const int64_t bytes = (kind == 0 ? 4 : 12) * nm;
            return BIN_HEAP0 + (bytes <= ap.rank_budget[0] ? 0 : 1);
        }
        if (na <= 32) return BIN_HEAP0 + 2;
        // wider complement rows: every A entry an iterator (k_push_heap_comp);
        // the bin keeps its largest A row in bin_words
        *aux_out = na;
        return BIN_HEAP0 + 3;
    }
    const bool single_ok = !ap.ordered || tf == 0;
    if (!ap.comp && fam == FAM_MSA && single_ok && msa_bytes(words, nm, kind) > ap.rank_budget[tr] &&
        msas_bytes(words, nm, kind) <= ap.rank_budget[tr] && nm < 65536) {
        // narrow mask over a wide window: sparse two-level bitmap
        *cap_lg_out = (int)msas_blocks(words, nm);   // per-bin maximum of touched blocks
        *aux_out = msas_dir(words);                   // per-bin maximum directory length
        return BIN_MSAS0 + tr;
    }
    // the dense window when it fits: one load and one compare per product
    if (!ap.comp && fam == FAM_MSA && msad_bytes(words, kind) <= ap.rank_budget[ap.ordered ? tf : tr])
        return BIN_MSAD0 + (ap.ordered ? tf : tr);
    // complemented MSA / auto with an output narrow enough for a state per column
    if (ap.comp && (ap.family == FAM_MSA || ap.family == FAM_AUTO) &&
        msad_bytes((ncols + 31) >> 5, kind) <= ap.rank_budget[tf]) {
        *aux_out = (ncols + 31) >> 5;
        return BIN_MSADC0 + tf;
    }
    if (!ap.comp && (fam == FAM_MSA || fam == FAM_MCA)) {
        const int64_t bytes = fam == FAM_MSA ? msa_bytes(words, nm, kind) : mca_bytes(nm, kind);
        const int tier = bytes <= ap.rank_budget[tf] ? tf : 3;
        // MSA rows past the shared tiers: shared-memory windows, not a global bitmap
        if (fam == FAM_MSA && tier == 3 && !ap.ordered) return BIN_MSAW;
        return (fam == FAM_MSA ? BIN_MSA0 : BIN_MCA0) + tier;
    }
    // hash family (and the complement forms of MSA / heap)
    int64_t fc = flops < ncols ? flops : ncols;
    int mode;
    int64_t keys;
    if (!ap.comp) {
        mode = MODE_PLAIN;
        keys = nm;
    } else {
        int lgm = 1;
        while ((1ll << lgm) <= nm) lgm++;
        // membership by binary search when it is cheaper than marking the mask
        if (fc * lgm <= nm) {
            mode = MODE_CSRCH;
            keys = fc;
        } else {
            mode = MODE_CTAB;
            keys = nm + fc;
        }
    }
    int need = ceil_log2_i64(2 * keys);
    if (need < 5) need = 5;
    int tier;
    {
        int tc = 3;
        for (int t = 0; t < 3; t++) {
            if (need <= tier_cap_lg(ap.pair, t)) { tc = t; break; }
        }
        // a binary search per product is a chain of dependent loads: spread
        // the row's products over more lanes much earlier than for probing
        const int tfh = mode == MODE_PLAIN && !ap.ordered
                            ? (flops <= ap.tier_flops0 ? 0 : (flops <= ap.tier_flops1_hash ? 1 : 2)) : tf;
        const int tfm = mode == MODE_CSRCH ? (flops <= 64 ? 0 : (flops <= 1024 ? 1 : 2)) : tfh;
        tier = tc > tfm ? tc : tfm;
    }
    // wide plain rows (16-warp tier) hold their keys by two-choice cuckoo
    // placement, which needs only load <= 1/2: smaller tables, more blocks
    const int ls = tier == 2 && mode == MODE_PLAIN ? ap.load_shift_wide : ap.load_shift;
    int want = ceil_log2_i64(keys << ls);
    if (want < 5) want = 5;
    // plain rows past the shared tiers: sliced over the largest shared table
    // (hash_row), not a global table
    const bool sliced = tier == 3 && mode == MODE_PLAIN && !ap.ordered;
    int lim = tier_cap_lg(ap.pair, sliced ? 2 : tier);
    const int used = want < lim ? want : lim;
    *cap_lg_out = used;
    return hash_bin(mode, tier, used > ap.capc_lg ? 1 : 0);
}

// Rows with more A entries than this (or, when the cost model needs B^T
// column lengths, more mask entries) are analysed by k_analyze_long, a block
// per row: hub rows (cfg5: 163,558 entries) would otherwise hold one warp for
// milliseconds while the rest of the grid idles.
constexpr int64_t LONG_ROW = 2048;

// One warp per row.  Computes row_flops, 1P complement bounds, bin + table size.
// Long rows are appended to long_rows[] (count in long_rows_n) instead.
template <bool BLEN>
__global__ void __launch_bounds__(256) k_analyze(Prob p, AnalyzeParams ap, int64_t* row_flops,
                                                 int64_t* bound, uint8_t* row_bin, int8_t* row_cap_lg,
                                                 Summary* s, int64_t* row_nnz, int32_t* long_rows,
                                                 int* long_rows_n) {
    __shared__ int s_count[NBINS];
    __shared__ int s_cap[NBINS];
    __shared__ unsigned long long s_bflops[NBINS];
    __shared__ int s_words[NBINS], s_nmx[NBINS];
    __shared__ unsigned long long s_flops, s_bound;
    __shared__ int s_na, s_nm;
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) { s_count[b] = 0; s_cap[b] = 0; s_bflops[b] = 0; s_words[b] = 0; s_nmx[b] = 0; }
    if (threadIdx.x == 0) { s_flops = 0; s_bound = 0; s_na = 0; s_nm = 0; }
    __syncthreads();
    // A warp takes 32 consecutive rows, one per lane: short rows (<= 32 A
    // entries / mask entries) are summed by their own lane with unrolled,
    // independent loads; longer ones by the whole warp.  Classification runs
    // lane-parallel; bin counters use warp-aggregated shared atomics.
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const bool want_pull = (ap.family == FAM_AUTO || ap.family == FAM_PULL) && ap.has_bt && !ap.comp;
    unsigned long long my_flops = 0, my_bound = 0;
    for (int64_t r0 = warp * 32; r0 < p.nrows; r0 += nwarps * 32) {
        const int64_t i = r0 + lane;
        bool live = i < p.nrows;
        if (live && ap.done && ap.done[i] >= 0) {   // computed by the direct pass
            live = false;
            row_bin[i] = (uint8_t)BIN_EMPTY;
        }
        int64_t as = 0, ae = 0, ms = 0, me = 0;
        if (live) {
            as = p.a_ptr[i];
            ae = p.a_ptr[i + 1];
            ms = p.m_ptr[i];
            me = p.m_ptr[i + 1];
            if (ae - as > LONG_ROW || (want_pull && me - ms > LONG_ROW)) {
                long_rows[atomicAdd(long_rows_n, 1)] = (int32_t)i;
                live = false;
                as = ae = ms = me = 0;
            }
        }
        long long f = 0;
        if (ae - as <= 32) {
            int64_t t = as;
            for (; t + 4 <= ae; t += 4) {
                const int32_t k0 = p.a_idx[t], k1 = p.a_idx[t + 1], k2 = p.a_idx[t + 2], k3 = p.a_idx[t + 3];
                f += b_row_len<BLEN>(p, ap, k0) + b_row_len<BLEN>(p, ap, k1) + b_row_len<BLEN>(p, ap, k2) + b_row_len<BLEN>(p, ap, k3);
            }
            for (; t < ae; t++) {
                const int32_t k = p.a_idx[t];
                f += b_row_len<BLEN>(p, ap, k);
            }
        }
        unsigned longm = __ballot_sync(FULL, ae - as > 32);
        while (longm) {
            const int src = __ffs(longm) - 1;
            longm &= longm - 1;
            const int64_t s0 = shfl64(as, src), s1 = shfl64(ae, src);
            long long g = 0;
            for (int64_t t = s0 + lane; t < s1; t += 32) {
                const int32_t k = p.a_idx[t];
                g += b_row_len<BLEN>(p, ap, k);
            }
            g = warp_sum_ll(g);
            if (lane == src) f = g;
        }
        const int64_t nm = me - ms;
        long long pull_cols = 0;
        if (want_pull) {
            if (f > 0 && nm > 0 && nm <= 32)
                for (int64_t t = ms; t < me; t++) {
                    const int32_t j = p.m_idx[t];
                    pull_cols += p.bt_ptr[j + 1] - p.bt_ptr[j];
                }
            unsigned lm = __ballot_sync(FULL, f > 0 && nm > 32);
            while (lm) {
                const int src = __ffs(lm) - 1;
                lm &= lm - 1;
                const int64_t s0 = shfl64(ms, src), s1 = shfl64(me, src);
                long long g = 0;
                for (int64_t t = s0 + lane; t < s1; t += 32) {
                    const int32_t j = p.m_idx[t];
                    g += p.bt_ptr[j + 1] - p.bt_ptr[j];
                }
                g = warp_sum_ll(g);
                if (lane == src) pull_cols = g;
            }
        }
        int b = -1, cap_lg = 0;
        int64_t words = 0;
        if (live) {
            const int64_t na = ae - as;
            row_flops[i] = f;
            if (bound) {
                const int64_t bd = f < p.ncols ? f : p.ncols;
                bound[i] = bd;
                my_bound += bd;
            }
            words = nm > 0 ? (((int64_t)p.m_idx[me - 1] - p.m_idx[ms]) >> 5) + 1 : 0;
            b = classify_row(ap, na, nm, f, p.ncols, pull_cols, words, &cap_lg, &words);
            row_bin[i] = (uint8_t)b;
            row_cap_lg[i] = (int8_t)cap_lg;
            // rows no kernel visits still need a count of 0
            if (row_nnz && b == BIN_EMPTY) row_nnz[i] = 0;
            my_flops += f;
        }
        // per-bin sums and maxima, aggregated over the warp's rows of each bin
        // (one shared atomic per distinct bin instead of one per row)
        unsigned todo = __ballot_sync(FULL, live);
        while (todo) {
            const int leader = __ffs(todo) - 1;
            const int bl = __shfl_sync(FULL, b, leader);
            const bool in = live && b == bl;
            const unsigned peers = __ballot_sync(FULL, in);
            todo &= ~peers;
            const long long fs = warp_sum_ll(in ? f : 0);
            const int capm = __reduce_max_sync(FULL, in ? cap_lg : 0);
            const int wm = __reduce_max_sync(FULL, in ? (int)(words < 0x7fffffff ? words : 0x7fffffff) : 0);
            const int nmm = __reduce_max_sync(FULL, in ? (int)(nm < 0x7fffffff ? nm : 0x7fffffff) : 0);
            if (lane == leader) {
                atomicAdd(&s_count[bl], __popc(peers));
                atomicAdd(&s_bflops[bl], (unsigned long long)fs);
                if (capm) atomicMax(&s_cap[bl], capm);
                if (bl != BIN_EMPTY) {
                    atomicMax(&s_words[bl], wm);
                    atomicMax(&s_nmx[bl], nmm);
                }
            }
        }
        const int na_max = __reduce_max_sync(FULL, live ? (int)min(ae - as, (int64_t)0x7fffffff) : 0);
        const int nm_max = __reduce_max_sync(FULL, live ? (int)min(nm, (int64_t)0x7fffffff) : 0);
        if (lane == 0) {
            atomicMax(&s_na, na_max);
            atomicMax(&s_nm, nm_max);
        }
    }
    my_flops = (unsigned long long)warp_sum_ll((long long)my_flops);
    my_bound = (unsigned long long)warp_sum_ll((long long)my_bound);
    if (lane == 0) {
        atomicAdd(&s_flops, my_flops);
        atomicAdd(&s_bound, my_bound);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < NBINS; b += blockDim.x) {
        if (s_count[b]) {
            atomicAdd(&s->bin_count[b], s_count[b]);
            atomicAdd(&s->bin_flops[b], s_bflops[b]);
            atomicMax(&s->bin_cap_lg[b], s_cap[b]);
            atomicMax(&s->bin_words[b], s_words[b]);
            atomicMax(&s->bin_nmmax[b], s_nmx[b]);
        }
    }
    if (threadIdx.x == 0) {
        atomicAdd(&s->gen_flops, s_flops);
        atomicAdd(&s->bound_total, s_bound);
        atomicMax(&s->max_na, s_na);
        atomicMax(&s->max_nm, s_nm);
    }
}

// Long rows (see LONG_ROW): one block per row, same quantities and the same
// classification as k_analyze, folded into the summary with global atomics.
// Runs after k_analyze on the same stream; grid-strides over the list.
template <bool BLEN>
__global__ void __launch_bounds__(256) k_analyze_long(Prob p, AnalyzeParams ap, int64_t* row_flops,
                                                      int64_t* bound, uint8_t* row_bin, int8_t* row_cap_lg,
                                                      Summary* s, int64_t* row_nnz, const int32_t* long_rows,
                                                      const int* long_rows_n) {
    __shared__ long long s_red[8];
    const int n_long = *long_rows_n;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool want_pull = (ap.family == FAM_AUTO || ap.family == FAM_PULL) && ap.has_bt && !ap.comp;
    for (int q = blockIdx.x; q < n_long; q += gridDim.x) {
        const int64_t i = long_rows[q];
        const int64_t as = p.a_ptr[i], ae = p.a_ptr[i + 1], ms = p.m_ptr[i], me = p.m_ptr[i + 1];
        long long f = 0;
        int64_t t = as + threadIdx.x;
        for (; t + 3 * 256 < ae; t += 4 * 256) {
            const int32_t k0 = p.a_idx[t], k1 = p.a_idx[t + 256], k2 = p.a_idx[t + 512], k3 = p.a_idx[t + 768];
            f += b_row_len<BLEN>(p, ap, k0) + b_row_len<BLEN>(p, ap, k1) + b_row_len<BLEN>(p, ap, k2) + b_row_len<BLEN>(p, ap, k3);
        }
        for (; t < ae; t += 256) {
            const int32_t k = p.a_idx[t];
            f += b_row_len<BLEN>(p, ap, k);
        }
        f = warp_sum_ll(f);
        if (lane == 0) s_red[wid] = f;
        __syncthreads();
        f = 0;
        for (int w = 0; w < 8; w++) f += s_red[w];
        __syncthreads();
        const int64_t nm = me - ms;
        long long pull_cols = 0;
        if (want_pull && f > 0 && nm > 0) {
            for (int64_t u = ms + threadIdx.x; u < me; u += 256) {
                const int32_t j = p.m_idx[u];
                pull_cols += p.bt_ptr[j + 1] - p.bt_ptr[j];
            }
            pull_cols = warp_sum_ll(pull_cols);
            if (lane == 0) s_red[wid] = pull_cols;
            __syncthreads();
            pull_cols = 0;
            for (int w = 0; w < 8; w++) pull_cols += s_red[w];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const int64_t na = ae - as;
            row_flops[i] = f;
            unsigned long long bd = 0;
            if (bound) {
                bd = f < p.ncols ? f : p.ncols;
                bound[i] = bd;
            }
            int64_t words = nm > 0 ? (((int64_t)p.m_idx[me - 1] - p.m_idx[ms]) >> 5) + 1 : 0;
            int cap_lg = 0;
            const int b = classify_row(ap, na, nm, f, p.ncols, pull_cols, words, &cap_lg, &words);
            row_bin[i] = (uint8_t)b;
            row_cap_lg[i] = (int8_t)cap_lg;
            if (row_nnz && b == BIN_EMPTY) row_nnz[i] = 0;
            atomicAdd(&s->bin_count[b], 1);
            atomicAdd(&s->bin_flops[b], (unsigned long long)f);
            if (cap_lg) atomicMax(&s->bin_cap_lg[b], cap_lg);
            if (b != BIN_EMPTY) {
                atomicMax(&s->bin_words[b], (int)(words < 0x7fffffff ? words : 0x7fffffff));
                atomicMax(&s->bin_nmmax[b], (int)(nm < 0x7fffffff ? nm : 0x7fffffff));
            }
            atomicAdd(&s->gen_flops, (unsigned long long)f);
            atomicAdd(&s->bound_total, bd);
            atomicMax(&s->max_na, (int)(na < 0x7fffffff ? na : 0x7fffffff));
            atomicMax(&s->max_nm, (int)(nm < 0x7fffffff ? nm : 0x7fffffff));
        }
    }
}


// Scatter row ids into per-bin lists (warp-aggregated atomics).
// Bin offsets come from the analysis summary (same rule as the host:
// off[0] = 0, off[b+1] = off[b] + (b == BIN_EMPTY ? 0 : count[b])).
__global__ void __launch_bounds__(256) k_bin_scatter(int64_t nrows, const uint8_t* row_bin,
                                                     const Summary* s, int32_t* bin_cursor,
                                                     int32_t* rows_out) {
    __shared__ int32_t bin_off[NBINS + 1];
    if (threadIdx.x == 0) {
        int run = 0;
        bin_off[0] = 0;
        for (int b = 0; b < NBINS; b++) {
            run += b == BIN_EMPTY ? 0 : s->bin_count[b];
            bin_off[b + 1] = run;
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < nrows;
         base += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = base + threadIdx.x;
        int b = i < nrows ? row_bin[i] : 0;
        unsigned peers = __match_any_sync(FULL, b);
        int leader = __ffs(peers) - 1;
        int rank = __popc(peers & lanemask_lt());
        int start = 0;
        if (lane == leader && b != 0) start = atomicAdd(&bin_cursor[b], __popc(peers));
        start = __shfl_sync(FULL, start, leader);
        if (b != 0) rows_out[bin_off[b] + start + rank] = (int32_t)i;
    }
}

}  // namespace mm
