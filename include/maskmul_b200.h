/*
 * maskmul_b200 — C ABI of the B200-native masked SpGEMM
 *
 *     C = M (.) (A B)        and        C = (not M) (.) (A B)
 *
 * over the plus-times / plus-pair semirings with int64 or float64 values.
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (arxiv 2111.09947, package `maskmul`) has no native FFI: its driver
 * `masked_multiply_with_stats` (pkg/src/maskmul/multiply.py:349-403) calls
 * numba-compiled row-chunk kernels (pkg/src/maskmul/_kernels.py:30-594)
 * through the internal signature
 *     <algo>_numeric(lo, hi, a_ptr, a_idx, a_val, b_ptr, b_idx, b_val,
 *                    m_ptr, m_idx, comp, sr, one, <scratch>, out_off,
 *                    out_idx, out_val, row_nnz) -> evaluated
 * Each entry point below names the reference function it replaces.  All
 * pointers in mm_matrix_t are DEVICE pointers (cudaMalloc / torch CUDA
 * tensors); every call is ordered on the caller's stream (cudaStream_t passed
 * as void*).  No torch types cross this boundary.
 *
 * Status codes mirror the reference's error classes and CLI exit codes
 * (cli.py:387-410): 0 ok, 1 PlanError, 2 SparseError (shape / input),
 * 3 internal bound violation (the reference's assertions at
 * multiply.py:375,390), 4 CUDA error.  mm_last_error() returns a thread-local
 * message for the last non-zero status.
 *
 * Threads: a handle (mm_create) serves one multiply at a time — give every
 * host thread its own (the Python host keeps one per device and thread).
 * Different handles may be used concurrently from different threads; what the
 * library shares between them (its record of each kernel's occupancy and
 * dynamic shared-memory limit, which belong to the CUDA context) sits behind
 * one mutex.  Every entry runs on its handle's / operands' device and
 * restores the caller's current device; an error some earlier CUDA call of
 * the thread left unread is dropped at entry, not reported as this call's.
 */
#ifndef MASKMUL_B200_H
#define MASKMUL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MM_ABI_VERSION 1

/* algorithms: multiply.py:35 ALGORITHMS, plus MM_ALGO_AUTO (per-row push/pull cost model) */
enum {
    MM_ALGO_MSA = 0,
    MM_ALGO_HASH = 1,
    MM_ALGO_MCA = 2,
    MM_ALGO_HEAP = 3,
    MM_ALGO_HEAPDOT = 4,
    MM_ALGO_INNER = 5,
    MM_ALGO_AUTO = 6
};

enum { MM_OK = 0, MM_ERR_PLAN = 1, MM_ERR_INPUT = 2, MM_ERR_INTERNAL = 3, MM_ERR_CUDA = 4, MM_ERR_CAPACITY = 5 };

/* semiring.py:23-24 kernel_id */
enum { MM_SR_ARITHMETIC = 0, MM_SR_PLUS_PAIR = 1 };
enum { MM_DTYPE_INT64 = 0, MM_DTYPE_FLOAT64 = 1 };

/* A sparse matrix on the device.  CSR: ptr = row_ptr[nrows+1], idx = col_idx[nnz].
 * CSC (the pull path's B^T, sparse.py:257-266): ptr = col_ptr[ncols+1],
 * idx = row_idx[nnz].  Offsets are int64 like the reference (sparse.py:9);
 * indices are int32 (all dimensions < 2^31).  values may be NULL for masks
 * and for plus-pair operands (the reference never reads them, _kernels.py:56). */
typedef struct {
    int64_t nrows;
    int64_t ncols;
    int64_t nnz;
    const int64_t* ptr;
    const int32_t* idx;
    const void* values;
} mm_matrix_t;

/* MultiplyPlan (multiply.py:46-81).  workers/grain have no GPU meaning. */
typedef struct {
    int32_t algorithm;     /* MM_ALGO_* */
    int32_t phases;        /* 1 = one-phase (bounded + compact), 2 = symbolic + exact */
    int32_t complemented;  /* plan.complemented OR mask.complemented (multiply.py:181) */
    int32_t semiring;      /* MM_SR_* */
    int32_t dtype;         /* MM_DTYPE_* */
    int32_t n_inspect;     /* heap: -1 = inf, 0, 1 (multiply.py:227-228) */
} mm_plan_t;

/* MultiplyStats (multiply.py:84-100) */
typedef struct {
    int64_t generated_flops;      /* sum over A nonzeros of nnz(B_k*) */
    int64_t evaluated_multiplies; /* products computed after mask filtering */
    int64_t output_nnz;
    int64_t rows_push;            /* rows computed by push kernels */
    int64_t rows_pull;            /* rows computed by the pull (inner) kernel */
    int64_t rows_empty;           /* rows skipped (empty mask row / zero flops) */
} mm_stats_t;

typedef struct mm_handle mm_handle_t;

int mm_abi_version(void);
const char* mm_last_error(void);

/* One handle per device; owns the stream-ordered workspace pool and the
 * state carried between mm_multiply_begin and mm_multiply_end. */
int mm_create(int device, mm_handle_t** out);
int mm_destroy(mm_handle_t* h);

/*
 * Two-call protocol for masked_multiply_with_stats (multiply.py:349-403):
 *
 *   mm_multiply_begin: validation (_Prepared, multiply.py:175-233), per-row
 *     work estimate (flops_per_row, :103-108), row binning, then
 *       1P: bounded numeric into workspace slots (:377-387) and the exact
 *           row-pointer scan (:391-393);
 *       2P: symbolic phase + exclusive scan (:358-368).
 *     Writes nnz(C) to *out_nnz (one small device->host readback).
 *   The caller allocates c_col_idx[nnz] (int32) and c_values[nnz] (dtype).
 *   mm_multiply_end: 1P compaction (compact_rows, _kernels.py:586-594) or 2P
 *     numeric into the exact slots (:369-376); copies row_ptr[nrows+1] and
 *     fills *stats.  Returns MM_ERR_INTERNAL if the reference's assertions
 *     (multiply.py:375,390) would fail.
 *
 * b: B as CSR (required: push kernels and flops_per_row read it; for
 *   MM_ALGO_INNER only its row pointer is read — idx / values may be NULL,
 *   as the reference's _Prepared holds B only as CSC for inner,
 *   multiply.py:205-210).
 * b_csc: B^T storage (CSC) for the pull path; required when
 *   plan->algorithm is MM_ALGO_INNER, optional for MM_ALGO_AUTO (without it
 *   AUTO runs push only), ignored otherwise.
 * mask: pattern only (values ignored); complement via plan->complemented.
 */
int mm_multiply_begin(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask,
                      const mm_matrix_t* a, const mm_matrix_t* b, const mm_matrix_t* b_csc,
                      void* stream, int64_t* out_nnz);
int mm_multiply_end(mm_handle_t* h, int64_t* c_row_ptr, int32_t* c_col_idx, void* c_values,
                    mm_stats_t* stats);

/* One-call form of the two calls above for callers that can bound nnz(C) in
 * advance (a plain mask: nnz(C) <= nnz(M), the one-phase bound of
 * multiply.py:233): c_col_idx / c_values hold `capacity` entries, c_row_ptr
 * nrows + 1 (written by the row-pointer scan itself); one host sync (the
 * nnz readback), compaction queued right after it.  If nnz(C) > capacity it
 * returns MM_ERR_CAPACITY with *out_nnz set and the handle still holding
 * the multiply: allocate nnz(C) entries and finish with mm_multiply_end.
 * Like every entry point the results are ordered on `stream`: the smallest
 * plain one-phase multiplies run as ONE launch whose last block reports the
 * counters through mapped host memory, and the call may return as soon as
 * they arrive, before that launch has retired — use C on `stream`, or
 * synchronise it first (the handle itself waits when the next multiply names
 * another stream). */
int mm_multiply(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                const mm_matrix_t* b, const mm_matrix_t* b_csc, void* stream, int64_t* c_row_ptr,
                int32_t* c_col_idx, void* c_values, int64_t capacity, int64_t* out_nnz, mm_stats_t* stats);

/* Per-phase device timing (CUDA events recorded on the caller's stream) of
 * every later multiply on this handle; off by default.  mm_profile_read
 * waits for the last multiply and returns ms[0..5] = {analyze + bin summary,
 * bin scatter, numeric (1P) or symbolic (2P) kernels, row-pointer scan and
 * nnz readback, compaction (1P) or numeric (2P), whole multiply} and the
 * number of kernels the library launched for it. */
int mm_profile_enable(mm_handle_t* h, int on);
int mm_profile_read(mm_handle_t* h, float* ms, int n, int64_t* launches);
/* Kernel-tier tuning of this handle (0 keeps a value): params[0] = max
 * products of a row in the 1-warp tier (default 8192), params[1] = max in the
 * 4-warp tier (65536), params[2] = log2 table-size class boundary (9),
 * params[3] = preferred table size as keys << params[3] (2, i.e. load 1/4),
 * params[4..6] = shared bytes per row allowed for the MSA / MCA rank-slot
 * accumulators in the 1-, 4- and 16-warp tiers (6144, 24576, 49152),
 * params[7] = AUTO: 1-warp rows whose MSA window does not fit use MCA when
 * their mask row has at most this many entries (0; negative keeps),
 * params[8..10] = log2 of the smallest plain shared-memory hash table in the
 * 1-, 4- and 16-warp tiers, which leaves room for a collision-free
 * (direct-mapped) table (9, 10, 12; 0 = bin size; negative keeps),
 * params[11] = params[3] for plain rows of the 16-warp tier (1),
 * params[12] / params[13] = row / nnz limits of the single-pass small-problem
 * path (32768 / 2^20; 0 disables it), params[14] = 0 disables the direct
 * path of ordered float64 plain one-phase multiplies (no analysis pass),
 * params[15] = 0 disables the slice cursors of sliced hub rows,
 * params[16] = 0 runs one-phase plain sliced hub rows slice after slice in one
 * group instead of as (row, slice) work items,
 * params[17] / params[18] = row / nnz limits of the one-launch path for the
 * smallest plain one-phase multiplies (8192 / 2^17; 0 disables it): the row
 * kernel's last block scans, compacts and reports through mapped host memory,
 * params[19] = 0 makes the analysis gather B's 8-byte row offsets instead of
 * the int32 row lengths it otherwise derives first,
 * params[20] = k-blocked passes of the 16-warp plain hash bins of one-phase
 * plus-pair multiplies: bytes of B's index array per block of B's rows (0 =
 * off, the default: measured slower on cfg5), params[21] = rows
 * under this many products are not cut into passes (2^20), params[22] =
 * params[1] for plain order-free hash rows (524288; params[1] sets both). */
int mm_set_tuning(mm_handle_t* h, const int64_t* params, int n);
/* Rows and generated flops per kernel bin of the last multiply (bin ids in
 * DESIGN.md §4); returns the number of bins. */
int mm_profile_bins(mm_handle_t* h, int64_t* rows, int64_t* flops, int n);

/* symbolic_phase (multiply.py:411-419): exact per-row output counts into the
 * device array counts[mask->nrows] (int64).  Synchronous on `stream`. */
int mm_symbolic(mm_handle_t* h, const mm_plan_t* plan, const mm_matrix_t* mask,
                const mm_matrix_t* a, const mm_matrix_t* b, const mm_matrix_t* b_csc,
                void* stream, int64_t* counts);

/* ---- building blocks (stream-ordered, device pointers) ---- */

/* flops_per_row (multiply.py:103-108): row_flops[i] = sum_{k in A_i} nnz(B_k*);
 * *total (device int64) receives the sum (generated_flops, :353). */
int mm_row_flops(const mm_matrix_t* a, const mm_matrix_t* b, int64_t* row_flops, int64_t* total,
                 void* stream);

/* Work estimate per row, w_i = flops_i + nnz(M_i) (the multi-GPU row cuts and
 * the per-row cost model; SURVEY §8(b) "mm_row_work").  row_flops (optional)
 * also receives flops_i. */
int mm_row_work(const mm_matrix_t* a, const mm_matrix_t* b, const mm_matrix_t* mask, int64_t* row_flops,
                int64_t* row_work, void* stream);

/* Device workspace one multiply draws from the stream-ordered pool (the
 * library allocates it itself with cudaMallocAsync and returns it at
 * mm_multiply_end).  Complemented one-phase plans add 12 bytes per bound
 * slot, sum_i min(flops_i, ncols) (known after mm_row_flops), not included. */
int mm_workspace_bytes(const mm_plan_t* plan, const mm_matrix_t* mask, const mm_matrix_t* a,
                       const mm_matrix_t* b, size_t* bytes);

/* np.cumsum into a row pointer (multiply.py:366-367,391-392):
 * out[0] = 0, out[i+1] = out[i] + counts[i]; n+1 outputs. */
int mm_exclusive_scan(const int64_t* counts, int64_t n, int64_t* out, void* stream);

/* compact_rows (_kernels.py:586-594) with int32 indices. */
int mm_compact_rows(int64_t nrows, const int64_t* bounds_off, const int64_t* row_nnz,
                    const int32_t* tmp_idx, const void* tmp_val, const int64_t* out_ptr,
                    int32_t* out_idx, void* out_val, int dtype, void* stream);

/* k-truss prune step (graphs.py:111-117): the pattern of C's entries with
 * int64 value >= thr, as CSR (out_row_ptr[nrows+1], out_idx[capacity nnz(C)]);
 * *out_nnz (host) receives the kept count.  Synchronous on `stream`. */
int mm_filter_min(const mm_matrix_t* c, int64_t thr, int64_t* out_row_ptr, int32_t* out_idx,
                  int64_t* out_nnz, void* stream);

/* sum of values[0..n) into *out (device, int64 or float64) — the triangle
 * count reduction of triangle_count (graphs.py:96). */
int mm_reduce_sum(const void* values, int64_t n, int dtype, void* out, void* stream);

/* ---- element-wise building blocks of the graph drivers (graphs.py:121-200) ---- */

/* lookup_rows (_kernels.py:597-612): for every stored entry t of X (row i,
 * column j), out[t] = Y[i, j] and found[t] = 1 when Y holds that entry, else
 * out[t] = 0 and found[t] = 0 (graphs._values_at, graphs.py:121-129).  X and
 * Y canonical, same shape; dtype MM_DTYPE_* of Y's values; found may be NULL. */
int mm_lookup_rows(const mm_matrix_t* x, const mm_matrix_t* y, int dtype, void* out, uint8_t* found,
                   void* stream);

/* Betweenness-centrality dependency weights on sigma_t's pattern
 * (graphs.py:181-184): w[t] = (1 + delta[i,j]) / paths[i,j], absent delta
 * entries reading 0.  float64. */
int mm_bc_dependency_weights(const mm_matrix_t* sigma_t, const mm_matrix_t* delta, const mm_matrix_t* paths,
                             double* w, void* stream);

/* out[t] = x.values[t] * paths[i,j] on x's pattern (graphs.py:186). float64. */
int mm_bc_scale_by(const mm_matrix_t* x, const mm_matrix_t* paths, double* out, void* stream);

/* ewise_add (sparse.py:360-370), two calls like the multiply: begin writes
 * the union's row pointer into c_row_ptr[nrows+1] (device) and its nnz into
 * *nnz (host; synchronous on `stream`); end fills c_idx / c_val (device,
 * nnz entries), values added where both operands hold an entry. */
int mm_ewise_add_begin(const mm_matrix_t* a, const mm_matrix_t* b, int64_t* c_row_ptr, int64_t* nnz,
                       void* stream);
int mm_ewise_add_end(const mm_matrix_t* a, const mm_matrix_t* b, int dtype, const int64_t* c_row_ptr,
                     int32_t* c_idx, void* c_val, void* stream);

/* BC score update for one source batch (graphs.py:188-197): for every row r,
 * scores[r] += delta[r, :] summed in column order, then, when src_col[r] >= 0
 * (r is the batch's source in column src_col[r]), scores[r] -= delta[r,
 * src_col[r]] (0 when absent).  src_col may be NULL (no sources). */
int mm_bc_accumulate(const mm_matrix_t* delta, const int32_t* src_col, double* scores, void* stream);

/* ---- device input preparation (graph_prep.cuh) ---- */

/* flags of mm_csr_from_coo */
enum { MM_COO_SYMMETRIC = 1, MM_COO_NO_DIAG = 2, MM_COO_LOWER = 4, MM_COO_DEDUP = 8 };

/* from_arrays / _canonical_from_sorted_triples (sparse.py:190-244) on the
 * device: COO (rows, cols: int64 when idx64 else int32; nnz entries) -> CSR
 * with rows sorted by column.  map (optional, int32[n]) relabels both
 * endpoints first (permute_symmetric, sparse.py:318-325).  MM_COO_SYMMETRIC
 * also emits (c, r); MM_COO_NO_DIAG drops r == c; MM_COO_LOWER keeps c < r
 * (tril_strict, sparse.py:285-291); MM_COO_DEDUP merges duplicates
 * (pattern only: simple_undirected_graph, sparse.py:344-357).  vals
 * (optional 8-byte payload per entry, not with DEDUP) travel with the columns
 * into out_vals.  out_idx / out_vals need capacity nnz (2 nnz when
 * symmetrising); *out_nnz (host) receives the entry count.  Synchronous. */
int mm_csr_from_coo(int64_t nrows, int64_t ncols, const void* rows, const void* cols, int idx64, int64_t nnz,
                    const int32_t* map, int flags, const void* vals, int64_t* out_ptr, int32_t* out_idx,
                    void* out_vals, int64_t* out_nnz, void* stream);

/* Row id of every CSR entry: rows[t] = i for ptr[i] <= t < ptr[i+1]. */
int mm_expand_rows(int64_t nrows, const int64_t* ptr, int32_t* rows, void* stream);

/* degree_sort_relabel's permutation (sparse.py:328-341): perm[new] = old in
 * non-increasing degree order, ties by index; new_label[old] = new.
 * Synchronous (reads the maximum degree back). */
int mm_degree_order(const mm_matrix_t* g, int32_t* perm, int32_t* new_label, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MASKMUL_B200_H */
