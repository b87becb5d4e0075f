// Microbenchmark: HBM read bandwidth vs. size (8 independent 16-byte loads per
// thread in flight, L2 flushed before every run, CUDA-event timed) -- the
// achievable rate for the per-step byte volumes of the SNN step (10-100 MB).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int U>
__global__ void k_read(const uint4 *buf, uint64_t n, uint32_t *out) {
    uint32_t acc = 0;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t x0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x0 < n; x0 += T * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) { const uint64_t x = x0 + T * u; v[u] = x < n ? __ldg(buf + x) : make_uint4(0, 0, 0, 0); }
#pragma unroll
        for (int u = 0; u < U; u++) acc += v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
int main() {
    const uint64_t B = 4ull << 30;
    uint4 *buf; cudaMalloc(&buf, B); cudaMemset(buf, 1, B);
    uint32_t *out; cudaMalloc(&out, 4);
    char *fl; cudaMalloc(&fl, 512ull << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (uint64_t mb : {8ull, 16ull, 32ull, 64ull, 128ull, 256ull, 1024ull, 4000ull}) {
        const uint64_t n = (mb << 20) / 16;
        for (int grid : {148 * 2, 148 * 4}) {
            float best = 1e9, tot = 0;
            for (int rep = 0; rep < 6; rep++) {
                cudaMemset(fl, rep, 512ull << 20);
                cudaEventRecord(a); k_read<8><<<grid, 512>>>(buf + (rep * 1234567ull) % (B / 16 - n), n, out); cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b); if (rep) { tot += ms; if (ms < best) best = ms; }
            }
            printf("%6llu MB grid %4d: mean %8.2f us (%.2f TB/s) best %.2f us\n", (unsigned long long)mb, grid, tot / 5 * 1e3,
                   (mb << 20) / (tot / 5 * 1e-3) / 1e12, best * 1e3);
            fflush(stdout);
        }
    }
    // empty kernel: launch + event overhead
    float tot = 0;
    for (int rep = 0; rep < 6; rep++) { cudaEventRecord(a); k_read<8><<<148, 512>>>(buf, 0, out); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (rep) tot += ms; }
    printf("empty kernel: %.2f us\n", tot / 5 * 1e3);
    return 0;
}
