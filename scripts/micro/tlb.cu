// Microbenchmark: random 128-byte segment reads (one warp each) from a buffer of
// B bytes -- does the span of the buffer (TLB reach) matter?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_seg(const uint32_t *buf, uint64_t nwords, const uint64_t *offs, uint32_t nseg, uint32_t *out) {
    uint32_t acc = 0;
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nseg; s += (gridDim.x * blockDim.x) >> 5) {
        acc += __ldg(buf + offs[s] + lane);
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_rows(const uint4 *buf, const uint64_t *offs, uint32_t nrow, uint32_t rowvec, uint32_t *out) {
    // one CTA per row: stream rowvec x 16 B
    uint32_t acc = 0;
    for (uint32_t r = blockIdx.x; r < nrow; r += gridDim.x) {
        const uint4 *p = buf + offs[r];
        for (uint32_t x = threadIdx.x; x < rowvec; x += blockDim.x) { uint4 v = __ldg(p + x); acc += v.x ^ v.w; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}
int main() {
    const uint64_t maxB = 8ull << 30;
    uint32_t *buf; cudaMalloc(&buf, maxB); cudaMemset(buf, 1, maxB);
    uint32_t *out; cudaMalloc(&out, 4);
    const uint32_t nseg = 102400;
    uint64_t *offs, *h = new uint64_t[nseg]; cudaMalloc(&offs, 8ull * nseg);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint64_t B : {64ull << 20, 256ull << 20, 1ull << 30, 4ull << 30, 8ull << 30}) {
        uint64_t x = 88172645463325252ull;
        for (uint32_t i = 0; i < nseg; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (x % (B / 4 - 64)) & ~31ull; }
        cudaMemcpy(offs, h, 8ull * nseg, cudaMemcpyHostToDevice);
        float best = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(a); k_seg<<<148 * 4, 512>>>(buf, B / 4, offs, nseg, out); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        // rows: 2400 random rows of 10 KB
        const uint32_t nrow = 2400, rowvec = 640;
        for (uint32_t i = 0; i < nrow; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = x % (B / 16 - rowvec); }
        cudaMemcpy(offs, h, 8ull * nrow, cudaMemcpyHostToDevice);
        float bestr = 1e9;
        for (int rep = 0; rep < 5; rep++) {
            cudaEventRecord(a); k_rows<<<148 * 2, 512>>>((const uint4 *)buf, offs, nrow, rowvec, out); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (ms < bestr) bestr = ms;
        }
        printf("span %6llu MB: 102400 random 128B segments %.1f us (%.2f TB/s of sectors);  2400 random 10KB rows %.1f us (%.2f TB/s)\n",
               (unsigned long long)(B >> 20), best * 1e3, nseg * 128.0 / (best * 1e-3) / 1e12, bestr * 1e3, nrow * 10240.0 / (bestr * 1e-3) / 1e12);
    }
    return 0;
}
