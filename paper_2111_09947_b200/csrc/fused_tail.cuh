// Fused tail of the single-pass kernels for small plain one-phase multiplies.
//
// Reference: the 1P assembly (multiply.py:381-399): exclusive scan of the row
// counts, compaction of the bounded slots into C, counters handed back.  On a
// small problem those steps cost more host time (three launches, a D2H copy
// and a stream synchronisation) than device time, so the row kernel does them
// itself: the last block to finish (a device counter) scans row_nnz into C's
// row pointer, copies every row's slots into C, and writes the multiply's
// counters straight into mapped pinned host memory, where the host spins on a
// sequence word instead of synchronising the stream.  One launch, no readback.
//
// One block does the whole tail, so the host uses it only below a row / nnz
// limit (mm_handle::fused_rows / fused_nnz); larger problems keep the
// separate scan and compaction kernels.
#pragma once
#include "analyze.cuh"
#include "common.cuh"

namespace mm {

// What the host reads back (mapped pinned memory, written by the last block).
struct TailResult {
    unsigned long long seq;   // written last, after a system-wide fence
    unsigned long long gen_flops;
    unsigned long long evaluated;
    long long total_nnz;
    int empty_rows;
    int overflow;             // a row the single pass could not take: the host runs the binned path
    int bound_flag;
    int pad;
    unsigned long long dbg[8];   // MM_TAIL_DEBUG: %globaltimer at tail entry / after the rows / after the fence
};

// Kernel argument (by value).  done == nullptr: no tail.
struct Tail {
    unsigned* done;            // persistent device counter, zero between multiplies (the tail resets it)
    long long nrows;
    const int64_t* row_nnz;
    const int64_t* slot_off;   // 1P slot offsets = the mask's row pointer (multiply.py:233)
    const int32_t* tmp_idx;
    const void* tmp_val;
    int64_t* c_row_ptr;        // nrows + 1
    int32_t* c_idx;            // null: scan only (mm_multiply_end compacts)
    void* c_val;
    Summary* summary;          // device counters the row kernel accumulated
    TailResult* host;
    unsigned long long seq;
};

// Called by every thread of every block at the very end of the row kernel
// (256 threads per block).  scratch: the block's dynamic shared memory (the
// row work is over), room for 3 * (TAIL_ROWS + TAIL_ROWS / 32) ints.
constexpr int TAIL_ROWS = 4096;   // rows per pass: 3 padded int arrays (tail_smem_bytes)
__host__ __device__ constexpr size_t tail_smem_bytes() { return (size_t)3 * (TAIL_ROWS + TAIL_ROWS / 32) * sizeof(int); }

__device__ __forceinline__ void fused_tail(const Tail& t, int* scratch) {
    __shared__ int s_last;
    __shared__ long long s_warp[8];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();   // this block's row_nnz / slot writes and counter atomics before the ticket
        s_last = atomicAdd(t.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    // (every other block's writes were fenced before its ticket; this block
    // reads them from L2 with ld.cg, past its own L1)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#ifdef MM_TAIL_DEBUG
    unsigned long long tg0 = 0, tg1 = 0, tga = 0, tgb = 0, tgc = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
#endif
    const long long m = t.nrows;
    long long carry = 0;
    int over = 0;
    // shared arrays of a pass, padded one word per 32 so a thread's contiguous
    // rows (stride `per` words between lanes) do not collide on a bank
    constexpr int PADDED = TAIL_ROWS + TAIL_ROWS / 32;
    int* pre = scratch;               // row count, then the row's exclusive prefix
    int* srcs = scratch + PADDED;     // the row's slot offset
    int* list = scratch + 2 * PADDED; // rows of the pass with output, in row order
    const int32_t* __restrict__ tmp_idx = t.tmp_idx;
    const long long* __restrict__ tmp_val = (const long long*)t.tmp_val;
    int32_t* __restrict__ c_idx = t.c_idx;
    long long* __restrict__ c_val = (long long*)t.c_val;
#define MM_TAIL_AT(q) ((q) + ((q) >> 5))
    for (long long r0 = 0; r0 < m; r0 += TAIL_ROWS) {
        const int cnt = (int)(m - r0 < TAIL_ROWS ? m - r0 : TAIL_ROWS);
        // A. row counts and slot offsets, coalesced, into shared memory (rows
        //    left to the binned pass carry -1: their sizes are redone there)
#pragma unroll 8
        for (int q = tid; q < cnt; q += 256) {
            const long long n = __ldcg(t.row_nnz + r0 + q);
            const long long so = t.slot_off[r0 + q];
            pre[MM_TAIL_AT(q)] = n > 0 ? (int)n : 0;
            srcs[MM_TAIL_AT(q)] = (int)so;
        }
        __syncthreads();
#ifdef MM_TAIL_DEBUG
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tga));
#endif
        // B. thread-contiguous sums and non-empty row counts (one packed block
        //    scan: nnz(C) <= nnz(M) < 2^31 on this path), exclusive prefixes
        //    in place, the non-empty rows listed
        const int per = (cnt + 255) / 256;
        const int q0 = tid * per < cnt ? tid * per : cnt;
        const int q1 = q0 + per < cnt ? q0 + per : cnt;
        long long mine = 0;
        for (int q = q0; q < q1; q++) {
            const int n = pre[MM_TAIL_AT(q)];
            mine += (long long)n + (n > 0 ? (1ll << 32) : 0ll);
        }
        long long incl = mine;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const long long u = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += u;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        long long before = 0, both = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const long long c = s_warp[q];
            if (q < wid) before += c;
            both += c;
        }
        const long long excl = before + incl - mine;
        const int total = (int)(both & 0xffffffffll), nz_total = (int)(both >> 32);
        int run = (int)(excl & 0xffffffffll), lpos = (int)(excl >> 32);
        for (int q = q0; q < q1; q++) {
            const int n = pre[MM_TAIL_AT(q)];
            pre[MM_TAIL_AT(q)] = run;
            run += n;
            if (n > 0) list[lpos++] = q;
        }
        __syncthreads();
#ifdef MM_TAIL_DEBUG
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tgb));
#endif
        // C. C's row pointer (coalesced stores, no loads) ...
        for (int q = tid; q < cnt; q += 256) t.c_row_ptr[r0 + q] = carry + pre[MM_TAIL_AT(q)];
#ifdef MM_TAIL_DEBUG
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tgc));
#endif
        // ... and the compaction: a thread per non-empty row, the first entry
        // of four rows in flight together
        for (int l0 = 0; l0 < nz_total; l0 += 4 * 256) {
            int nn[4], ss[4];
            long long dd[4];
            int32_t j0[4];
            long long v0[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int l = l0 + u * 256 + tid;
                nn[u] = 0;
                ss[u] = 0;
                dd[u] = 0;
                if (l < nz_total) {
                    const int q = list[l];
                    const int p = pre[MM_TAIL_AT(q)];
                    nn[u] = (q + 1 < cnt ? pre[MM_TAIL_AT(q + 1)] : total) - p;
                    ss[u] = srcs[MM_TAIL_AT(q)];
                    dd[u] = carry + p;
                    // the 1P bound assertion (multiply.py:390): slots = the mask row
                    const int lim = (q + 1 < cnt ? srcs[MM_TAIL_AT(q + 1)] : (int)t.slot_off[r0 + cnt]) - ss[u];
                    if (nn[u] > lim) {
                        over = 1;
                        nn[u] = 0;
                    }
                }
            }
            if (c_idx) {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (nn[u] > 0) {
                        j0[u] = __ldcg(tmp_idx + ss[u]);
                        v0[u] = __ldcg(tmp_val + ss[u]);
                    }
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (nn[u] > 0) {
                        c_idx[dd[u]] = j0[u];
                        c_val[dd[u]] = v0[u];
                        for (int e = 1; e < nn[u]; e++) {
                            c_idx[dd[u] + e] = __ldcg(tmp_idx + ss[u] + e);
                            c_val[dd[u] + e] = __ldcg(tmp_val + ss[u] + e);
                        }
                    }
            }
        }
        carry += total;
        __syncthreads();
    }
#undef MM_TAIL_AT
    over = __syncthreads_or(over);
#ifdef MM_TAIL_DEBUG
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg1));
#endif
    if (tid == 0) {
        t.c_row_ptr[m] = carry;
        TailResult* r = t.host;
        r->gen_flops = __ldcg(&t.summary->gen_flops);
        r->evaluated = __ldcg(&t.summary->evaluated);
        r->total_nnz = carry;
        r->empty_rows = __ldcg(&t.summary->bin_count[BIN_EMPTY]);
        r->overflow = __ldcg(&t.summary->pad);
        r->bound_flag = over;
        *t.done = 0u;   // every other block has left: ready for the next multiply
#ifdef MM_TAIL_DEBUG
        r->dbg[0] = tg0;
        r->dbg[1] = tg1;
        r->dbg[4] = tga;
        r->dbg[5] = tgb;
        r->dbg[6] = tgc;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
        r->dbg[2] = tg0;
#endif
        __threadfence_system();
#ifdef MM_TAIL_DEBUG
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tg0));
        r->dbg[3] = tg0;
        __threadfence_system();
#endif
        *(volatile unsigned long long*)&r->seq = t.seq;
    }
}

}  // namespace mm
