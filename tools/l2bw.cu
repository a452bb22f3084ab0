// L2-resident read bandwidth on one B200 (roofline denominator for kernels
// whose B-row re-reads hit in L2).  Two patterns over a buffer that fits in
// L2 (after a warm-up pass):
//   stream  — coalesced 16-byte loads, grid-stride (ideal L2 -> SM rate)
//   gather  — 4-byte loads where each group of 8 lanes reads one random
//             32-byte sector (the flattened short-B-row product reads)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_stream(const int4* __restrict__ p, size_t n16, int reps, int* out) {
    int acc = 0;
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
            int4 v = __ldcg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x12345678) out[0] = acc;
}

__global__ void k_gather(const int* __restrict__ p, size_t nsect, long long iters, int* out) {
    int acc = 0;
    const unsigned lane = threadIdx.x & 31;
    unsigned long long x = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) / 8 * 0x9E3779B97F4A7C15ull + 1;
    for (long long it = 0; it < iters; it += 8) {
        int v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {                          // 8 independent loads in flight
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;          // same x for the 8 lanes of a sector group
            const size_t sect = (size_t)((x >> 20) & (nsect - 1));   // nsect: power of two
            v[u] = __ldcg(p + sect * 8 + (lane & 7));
        }
#pragma unroll
        for (int u = 0; u < 8; u++) acc ^= v[u];
    }
    if (acc == 0x12345678) out[0] = acc;
}

int main() {
    int* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t mb : {16, 32, 64}) {
        size_t bytes = mb << 20;
        void* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        int grid = 148 * 8, block = 256;
        k_stream<<<grid, block>>>((const int4*)buf, bytes / 16, 1, out);
        int reps = 40;
        cudaEventRecord(a);
        k_stream<<<grid, block>>>((const int4*)buf, bytes / 16, reps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("stream %3zu MB: %.2f TB/s\n", mb, bytes * (double)reps / (ms * 1e-3) / 1e12);
        long long iters = 4096;
        k_gather<<<grid, block>>>((const int*)buf, bytes / 32, 64, out);
        cudaEventRecord(a);
        k_gather<<<grid, block>>>((const int*)buf, bytes / 32, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double useful = (double)grid * block * iters * 4;
        printf("gather %3zu MB: %.2f TB/s useful (4 B per lane, 32 B sectors)\n", mb, useful / (ms * 1e-3) / 1e12);
        cudaFree(buf);
    }
    return 0;
}
