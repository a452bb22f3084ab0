// Device-side input preparation: the canonicalisation the
// reference does on the host before every masked multiply it times —
//   from_arrays / _canonical_from_sorted_triples (sparse.py:190-244): COO ->
//       canonical CSR (rows sorted, duplicates merged),
//   simple_undirected_graph (sparse.py:344-357): symmetrise, drop self-loops,
//       merge duplicates,
//   degree_sort_relabel + permute_symmetric (sparse.py:318-341): relabel by
//       non-increasing degree, ties by index,
//   tril_strict (sparse.py:285-291) and to_csc / transpose (sparse.py:257-283).
// Building blocks: an atomic-cursor scatter of (row, col[, value]) into row
// segments, then a segmented sort of every row (keys = columns, optional
// 8-byte payload), then duplicate removal.  The scatter order inside a row is
// arbitrary, the sort makes the result canonical and deterministic (keys are
// unique after dedup, and unique per row for transposes).
#pragma once
#include "common.cuh"

namespace mm {

constexpr int PREP_TILE = 4096;          // keys sorted in shared memory by one block
constexpr int PREP_THREADS = 512;

// Emission rule shared by count and scatter: entry e of a COO list (or of a
// CSR whose rows are expanded) becomes (r, c) and, when sym, (c, r); map
// relabels both endpoints; nodiag drops r == c; lower keeps c < r.
struct CooView {
    const void* rows;     // int32 or int64 row of each entry
    const void* cols;     // int32 or int64 column of each entry
    int idx64;            // 1: rows/cols are int64
    const int32_t* map;   // optional relabelling (new id of old id)
    int sym, nodiag, lower;
    int64_t nnz;
};

__device__ __forceinline__ void coo_entry(const CooView& v, int64_t e, int32_t& r, int32_t& c) {
    if (v.idx64) {
        r = (int32_t)((const int64_t*)v.rows)[e];
        c = (int32_t)((const int64_t*)v.cols)[e];
    } else {
        r = ((const int32_t*)v.rows)[e];
        c = ((const int32_t*)v.cols)[e];
    }
    if (v.map) {
        r = v.map[r];
        c = v.map[c];
    }
}

__device__ __forceinline__ bool coo_keep(const CooView& v, int32_t r, int32_t c) {
    return !(v.nodiag && r == c) && !(v.lower && c >= r);
}

__global__ void __launch_bounds__(256) k_coo_count(CooView v, int64_t* counts) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < v.nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t r, c;
        coo_entry(v, e, r, c);
        if (coo_keep(v, r, c)) atomicAdd((unsigned long long*)(counts + r), 1ull);
        if (v.sym && coo_keep(v, c, r)) atomicAdd((unsigned long long*)(counts + c), 1ull);
    }
}

// cursor[r] starts at ptr[r]; vals/out_val optional (8-byte payload).
__global__ void __launch_bounds__(256) k_coo_scatter(CooView v, const unsigned long long* vals,
                                                     unsigned long long* cursor, int32_t* out_idx,
                                                     unsigned long long* out_val) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < v.nnz; e += (int64_t)gridDim.x * blockDim.x) {
        int32_t r, c;
        coo_entry(v, e, r, c);
        if (coo_keep(v, r, c)) {
            const unsigned long long q = atomicAdd(cursor + r, 1ull);
            out_idx[q] = c;
            if (out_val) out_val[q] = vals[e];
        }
        if (v.sym && coo_keep(v, c, r)) {
            const unsigned long long q = atomicAdd(cursor + c, 1ull);
            out_idx[q] = r;
            if (out_val) out_val[q] = vals[e];
        }
    }
}

// Row id of every CSR entry (expands row_ptr; warp per row).
__global__ void __launch_bounds__(256) k_expand_rows(int64_t nrows, const int64_t* ptr, int32_t* rows) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps)
        for (int64_t t = ptr[i] + lane; t < ptr[i + 1]; t += 32) rows[t] = (int32_t)i;
}

// --- segmented sort ---------------------------------------------------------
// Segments of <= 32 keys: one warp, a register bitonic network over the
// lanes.  Longer segments are appended to `big` and sorted by
// k_seg_sort_block.
template <bool PAYLOAD>
__global__ void __launch_bounds__(256) k_seg_sort_warp(int64_t nseg, const int64_t* ptr, int32_t* keys,
                                                       unsigned long long* vals, int32_t* big, int* nbig) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = warp; s < nseg; s += nwarps) {
        const int64_t b = ptr[s], e = ptr[s + 1];
        const int64_t len = e - b;
        if (len <= 1) continue;
        if (len > 32) {
            if (lane == 0) big[atomicAdd(nbig, 1)] = (int32_t)s;
            continue;
        }
        int32_t k = lane < len ? keys[b + lane] : INT32_MAX;
        unsigned long long v = PAYLOAD && lane < len ? vals[b + lane] : 0ull;
#pragma unroll
        for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
            for (int j = size >> 1; j > 0; j >>= 1) {
                const int32_t ok = __shfl_xor_sync(FULL, k, j);
                const unsigned long long ov = PAYLOAD ? __shfl_xor_sync(FULL, v, j) : 0ull;
                const bool up = (lane & size) == 0;
                const bool lower = (lane & j) == 0;
                // lower lane keeps min when ascending
                const bool take = lower == up ? ok < k : ok > k;
                if (take) {
                    k = ok;
                    if (PAYLOAD) v = ov;
                }
            }
        }
        if (lane < len) {
            keys[b + lane] = k;
            if (PAYLOAD) vals[b + lane] = v;
        }
    }
}

// One block sorts one long segment: a bitonic sort over the segment padded to
// a power of two P.  Stages with stride < PREP_TILE run on shared-memory
// tiles, larger strides run in place in a global scratch copy.  PAYLOAD:
// an 8-byte value travels with each key.
template <bool PAYLOAD>
__device__ void block_bitonic_tiles(int32_t* gk, unsigned long long* gv, int64_t P, int size_from, int32_t* sk,
                                    unsigned long long* sv) {
    // every tile of PREP_TILE elements: finish all stages with stride < TILE
    // for sizes size_from .. min(P, TILE) (size_from = 2: full local sort),
    // or, for size > TILE, the tail strides TILE/2 .. 1 of that size
    for (int64_t t0 = 0; t0 < P; t0 += PREP_TILE) {
        for (int q = threadIdx.x; q < PREP_TILE; q += blockDim.x) {
            sk[q] = gk[t0 + q];
            if (PAYLOAD) sv[q] = gv[t0 + q];
        }
        __syncthreads();
        const int64_t lo_size = size_from, hi_size = size_from > PREP_TILE ? size_from : (P < PREP_TILE ? P : PREP_TILE);
        for (int64_t size = lo_size; size <= hi_size; size <<= 1) {
            for (int64_t j = (size > PREP_TILE ? PREP_TILE : size) >> 1; j > 0; j >>= 1) {
                for (int q = threadIdx.x; q < PREP_TILE / 2; q += blockDim.x) {
                    const int i = (int)(2 * q - (q & (j - 1)));   // lower index of the pair (bit j clear)
                    const int m = i + (int)j;
                    const bool up = (((t0 + i) & size) == 0);
                    const int32_t a = sk[i], b = sk[m];
                    if ((a > b) == up) {
                        sk[i] = b;
                        sk[m] = a;
                        if (PAYLOAD) {
                            const unsigned long long va = sv[i];
                            sv[i] = sv[m];
                            sv[m] = va;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int q = threadIdx.x; q < PREP_TILE; q += blockDim.x) {
            gk[t0 + q] = sk[q];
            if (PAYLOAD) gv[t0 + q] = sv[q];
        }
        __syncthreads();
    }
}

template <bool PAYLOAD>
__global__ void __launch_bounds__(PREP_THREADS) k_seg_sort_block(const int64_t* ptr, int32_t* keys,
                                                                 unsigned long long* vals, const int32_t* big,
                                                                 const int* nbig, int32_t* scratch_k,
                                                                 unsigned long long* scratch_v, int64_t scratch_cap) {
    __shared__ int32_t sk[PREP_TILE];
    __shared__ unsigned long long sv[PAYLOAD ? PREP_TILE : 1];
    const int n = *nbig;
    for (int q = blockIdx.x; q < n; q += gridDim.x) {
        const int64_t s = big[q];
        const int64_t b = ptr[s], e = ptr[s + 1], len = e - b;
        int64_t P = 1;
        while (P < len) P <<= 1;
        if (P <= PREP_TILE) {
            // whole segment in shared memory
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                sk[i] = i < len ? keys[b + i] : INT32_MAX;
                if (PAYLOAD) sv[i] = i < len ? vals[b + i] : 0ull;
            }
            __syncthreads();
            for (int size = 2; size <= P; size <<= 1)
                for (int j = size >> 1; j > 0; j >>= 1) {
                    for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
                        const int i = 2 * t - (t & (j - 1));
                        const int m = i + j;
                        const bool up = (i & size) == 0;
                        const int32_t x = sk[i], y = sk[m];
                        if ((x > y) == up) {
                            sk[i] = y;
                            sk[m] = x;
                            if (PAYLOAD) {
                                const unsigned long long vx = sv[i];
                                sv[i] = sv[m];
                                sv[m] = vx;
                            }
                        }
                    }
                    __syncthreads();
                }
            for (int i = threadIdx.x; i < len; i += blockDim.x) {
                keys[b + i] = sk[i];
                if (PAYLOAD) vals[b + i] = sv[i];
            }
            __syncthreads();
            continue;
        }
        // long segment: padded copy in this block's scratch slice
        int32_t* gk = scratch_k + (int64_t)blockIdx.x * scratch_cap;
        unsigned long long* gv = PAYLOAD ? scratch_v + (int64_t)blockIdx.x * scratch_cap : nullptr;
        for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
            gk[i] = i < len ? keys[b + i] : INT32_MAX;
            if (PAYLOAD) gv[i] = i < len ? vals[b + i] : 0ull;
        }
        __syncthreads();
        block_bitonic_tiles<PAYLOAD>(gk, gv, P, 2, sk, sv);        // every tile sorted (alternating directions)
        for (int64_t size = 2 * PREP_TILE; size <= P; size <<= 1) {
            for (int64_t j = size >> 1; j >= PREP_TILE; j >>= 1) {   // global strides
                for (int64_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
                    const int64_t i = 2 * t - (t & (j - 1));
                    const int64_t m = i + j;
                    const bool up = (i & size) == 0;
                    const int32_t x = gk[i], y = gk[m];
                    if ((x > y) == up) {
                        gk[i] = y;
                        gk[m] = x;
                        if (PAYLOAD) {
                            const unsigned long long vx = gv[i];
                            gv[i] = gv[m];
                            gv[m] = vx;
                        }
                    }
                }
                __syncthreads();
            }
            block_bitonic_tiles<PAYLOAD>(gk, gv, P, (int)size, sk, sv);   // strides < TILE of this size
        }
        for (int64_t i = threadIdx.x; i < len; i += blockDim.x) {
            keys[b + i] = gk[i];
            if (PAYLOAD) vals[b + i] = gv[i];
        }
        __syncthreads();
    }
}

// Distinct keys per (sorted) row; keep_first marks survivors for compaction.
__global__ void __launch_bounds__(256) k_unique_count(int64_t nrows, const int64_t* ptr, const int32_t* keys,
                                                      int64_t* counts) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t b = ptr[i], e = ptr[i + 1];
        long long c = 0;
        for (int64_t t = b + lane; t < e; t += 32) c += (t == b || keys[t] != keys[t - 1]);
        c = warp_sum_ll(c);
        if (lane == 0) counts[i] = c;
    }
}

__global__ void __launch_bounds__(256) k_unique_compact(int64_t nrows, const int64_t* ptr, const int32_t* keys,
                                                        const int64_t* out_ptr, int32_t* out_idx) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < nrows; i += nwarps) {
        const int64_t b = ptr[i], e = ptr[i + 1];
        int64_t run = out_ptr[i];
        for (int64_t t0 = b; t0 < e; t0 += 32) {
            const int64_t t = t0 + lane;
            const bool keep = t < e && (t == b || keys[t] != keys[t - 1]);
            const unsigned bal = __ballot_sync(FULL, keep);
            if (keep) out_idx[run + __popc(bal & lanemask_lt())] = keys[t];
            run += __popc(bal);
        }
    }
}

// Degree relabelling, step 1: histogram of degrees (bucket = maxdeg - deg, so
// buckets run from the highest degree down).
__global__ void __launch_bounds__(256) k_degree_hist(int64_t n, const int64_t* ptr, int64_t maxdeg, int64_t* hist) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)(hist + (maxdeg - (ptr[v + 1] - ptr[v]))), 1ull);
}

// step 2: vertices scattered into their degree bucket (any order inside it;
// the segmented sort by id then gives non-increasing degree, ties by index —
// np.lexsort((arange(n), -deg)), sparse.py:338).
__global__ void __launch_bounds__(256) k_degree_scatter(int64_t n, const int64_t* ptr, int64_t maxdeg,
                                                        unsigned long long* cursor, int32_t* perm) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        perm[atomicAdd(cursor + (maxdeg - (ptr[v + 1] - ptr[v])), 1ull)] = (int32_t)v;
}

// step 3: new_label[perm[i]] = i.
__global__ void __launch_bounds__(256) k_invert_perm(int64_t n, const int32_t* perm, int32_t* new_label) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        new_label[perm[i]] = (int32_t)i;
}

__global__ void __launch_bounds__(256) k_max_degree(int64_t n, const int64_t* ptr, unsigned long long* out) {
    unsigned long long m = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = (unsigned long long)(ptr[v + 1] - ptr[v]);
        m = d > m ? d : m;
    }
    m = __reduce_max_sync(FULL, (unsigned)min(m, 0xffffffffull));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace mm
