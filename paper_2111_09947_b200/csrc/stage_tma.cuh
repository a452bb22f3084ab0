// EXPERIMENT (build flag MM_STAGE_TMA, tools/build_variants.sh): long B-row
// segments of the order-free product loop staged into shared memory by
// 1-D bulk copies (cp.async.bulk = TMA, UBLKCP in SASS) with mbarrier
// completion, double-buffered per warp, instead of 16 coalesced LDGs per
// lane per 512 products.  The copy source is rounded down to 16 bytes (the
// 0-3 leading entries are skipped when reading: the head fix-up) and the
// size up to 16 bytes, so a copy may read up to 12 bytes past a segment
// (inside the same B array but for the last row; torch's caching allocator
// rounds allocations to 512 bytes).  Only blocks of <= 8 warps stage.
// Kept as an experiment, not in the product build: see DESIGN.md §7b.
#pragma once
#include "common.cuh"

namespace mm {

#ifndef MM_STAGE_PIECE
#define MM_STAGE_PIECE 512   // entries per staged piece (2 KB)
#endif
#ifndef MM_STAGE_MIN
#define MM_STAGE_MIN 256     // stage segments of at least this many products
#endif
constexpr int STAGE_P = MM_STAGE_PIECE;
constexpr int STAGE_BUF = STAGE_P + 8;   // + head (<= 3) + tail rounding, multiple of 4 entries

struct StageWarp {
    int32_t* buf;       // 2 buffers of STAGE_BUF entries (16-byte aligned)
    uint32_t mbar_s;    // 2 mbarriers (shared addresses), 8 bytes apart
    uint32_t* phase;    // per-warp parity bits of the two barriers
};

__device__ __forceinline__ unsigned char* stage_smem() {
    __shared__ __align__(16) unsigned char s_stage[8 * (2 * STAGE_BUF * 4 + 16 + 16)];
    return s_stage;
}

__device__ __forceinline__ bool stage_available() { return blockDim.x <= 256; }

__device__ __forceinline__ StageWarp stage_warp() {
    const int w = threadIdx.x >> 5;
    unsigned char* base = stage_smem() + (size_t)w * (2 * STAGE_BUF * 4 + 16 + 16);
    StageWarp s;
    s.buf = (int32_t*)base;
    s.mbar_s = (uint32_t)__cvta_generic_to_shared(base + 2 * STAGE_BUF * 4);
    s.phase = (uint32_t*)(base + 2 * STAGE_BUF * 4 + 16);
    return s;
}

// Once per block at kernel start (every thread calls).
__device__ __forceinline__ void stage_init() {
    if (!stage_available()) return;
    if ((threadIdx.x & 31) == 0) {
        StageWarp s = stage_warp();
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s.mbar_s));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s.mbar_s + 8));
        *s.phase = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
}

// lane 0: bulk-copy entries [src, src + n) of a 4-byte array to buffer b;
// returns (on every lane) the head offset of the first entry in the buffer.
__device__ __forceinline__ int stage_issue(const StageWarp& s, int b, const int32_t* src, int n, int lane) {
    const uintptr_t a = (uintptr_t)src;
    const uintptr_t a16 = a & ~(uintptr_t)15;
    const int head = (int)((a - a16) >> 2);
    if (lane == 0) {
        const uint32_t bytes = (uint32_t)(((head + n) * 4 + 15) & ~15);
        const uint32_t mb = s.mbar_s + 8u * b;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s.buf + b * STAGE_BUF);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // earlier generic reads of the buffer
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(a16), "r"(bytes), "r"(mb)
                     : "memory");
    }
    return head;
}

__device__ __forceinline__ void stage_wait(const StageWarp& s, int b, uint32_t parity) {
    const uint32_t mb = s.mbar_s + 8u * b;
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(mb), "r"(parity)
            : "memory");
    }
}

// The whole segment B[b0, b0 + n0): pieces of STAGE_P entries, piece i+1 in
// flight while piece i is probed (put_batch<4> over 128-entry chunks).
template <class PR>
__device__ __forceinline__ void stage_segment(const Prob& p, PR& pr, int64_t b0, int n0, long long a0, int lane) {
    const StageWarp s = stage_warp();
    uint32_t ph = *s.phase;
    __syncwarp();
    const int np = (n0 + STAGE_P - 1) / STAGE_P;
    int head_cur = stage_issue(s, 0, p.b_idx + b0, min(n0, STAGE_P), lane);
    for (int i = 0; i < np; i++) {
        const int b = i & 1;
        int head_next = 0;
        if (i + 1 < np)
            head_next = stage_issue(s, b ^ 1, p.b_idx + b0 + (int64_t)(i + 1) * STAGE_P,
                                    min(n0 - (i + 1) * STAGE_P, STAGE_P), lane);
        stage_wait(s, b, (ph >> b) & 1u);
        ph ^= 1u << b;
        const int n = min(n0 - i * STAGE_P, STAGE_P);
        const int32_t* sb = s.buf + b * STAGE_BUF + head_cur;
        const int64_t base = b0 + (int64_t)i * STAGE_P;
        for (int c = 0; c < n; c += 128) {
            int32_t jj[4];
            long long aa[4], ss[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int o = c + 32 * u + lane;
                jj[u] = o < n ? sb[o] : EMPTY_KEY;
                aa[u] = a0;
                ss[u] = base + o;
            }
            pr.template put_batch<4>(jj, aa, ss);
        }
        __syncwarp();
        head_cur = head_next;
    }
    if (lane == 0) *s.phase = ph;
    __syncwarp();
}

}  // namespace mm
