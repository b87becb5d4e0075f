// Microbenchmark: the forced-flush access pattern of cfg3 -- ~2470 random rows
// of 2530 sorted uint32 targets (+ fp32 weights) out of a 4 GB id array, each
// target probed in a 16 KB shared bitmap -- as a pure streaming floor.
//   mode 0: ids only, LDG.128, U chunks in flight per thread
//   mode 1: ids + weights
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
constexpr int kRowLen = 2528;            // multiple of 4
template <int U, int MODE>
__global__ void __launch_bounds__(1024, 1) k_stream(const uint4 *ids, const uint4 *w, const uint64_t *rows, int nrows,
                                                    const uint32_t *bitmap, uint32_t nbw, uint32_t *out) {
    __shared__ uint32_t bm[4096];
    for (uint32_t x = threadIdx.x; x < nbw; x += blockDim.x) bm[x] = bitmap[x];
    __syncthreads();
    const int r0 = (int)((long long)nrows * blockIdx.x / gridDim.x), r1 = (int)((long long)nrows * (blockIdx.x + 1) / gridDim.x);
    const int chunks_per_row = kRowLen / 4;
    const int T = (r1 - r0) * chunks_per_row;
    uint32_t hits = 0;
    float acc = 0.f;
    for (int c0 = threadIdx.x; c0 < T; c0 += blockDim.x * U) {
        uint4 v[U], ww[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int c = c0 + u * blockDim.x;
            if (c < T) {
                const int r = r0 + c / chunks_per_row, k = c % chunks_per_row;
                v[u] = __ldg(ids + rows[r] / 4 + k);
                if (MODE == 1) ww[u] = __ldg(w + rows[r] / 4 + k);
            } else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t j[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int e = 0; e < 4; e++) hits += (bm[(j[e] >> 5) & 4095] >> (j[e] & 31)) & 1u;
            if (MODE == 1) acc += ww[u].x ^ ww[u].w ? 1.f : 0.f;
        }
    }
    if (hits == 0xdeadbeef || acc == 1234.5f) out[0] = hits;
    atomicAdd(out + 1, hits);
}
__global__ void k_fill(uint32_t *p, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = (uint32_t)((i * 2654435761ull) % 126491);
}
template <int U, int MODE>
float run(const uint4 *ids, const uint4 *w, uint64_t *d_rows, std::vector<std::vector<uint64_t>> &sets, const uint32_t *bm,
          uint32_t *out, int grid) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int nrows = (int)sets[0].size();
    float tot = 0;
    for (size_t s = 0; s < sets.size(); s++) {
        cudaMemcpy(d_rows, sets[s].data(), 8 * nrows, cudaMemcpyHostToDevice);
        cudaEventRecord(a);
        k_stream<U, MODE><<<grid, 1024>>>(ids, w, d_rows, nrows, bm, 3953, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (s > 2) tot += ms;
    }
    return tot / (sets.size() - 3) * 1e3f;
}
int main() {
    const uint64_t n = 1000000000ull;
    uint32_t *ids, *w, *bm, *out; uint64_t *d_rows;
    cudaMalloc(&ids, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&bm, 4 * 4096); cudaMalloc(&out, 8); cudaMalloc(&d_rows, 8 * 10000);
    k_fill<<<4096, 256>>>(ids, n); k_fill<<<4096, 256>>>(w, n);
    std::vector<uint32_t> hb(4096); std::mt19937 g(1);
    for (auto &x : hb) x = (g() & g() & g());                   // ~12.5% bits set
    cudaMemcpy(bm, hb.data(), 4 * 4096, cudaMemcpyHostToDevice);
    int grid = 148;
    for (uint64_t span : {4000000000ull, 1000000000ull, 250000000ull, 64000000ull, 16000000ull}) {
        std::vector<std::vector<uint64_t>> sets(23, std::vector<uint64_t>(2470));
        for (auto &s : sets) for (auto &r : s) r = ((uint64_t)g() * 977ull % ((span / 4) - 4096)) & ~3ull;
        printf("span %5.0f MB: ids U=4 %.2f us, ids+w U=4 %.2f us\n", span / 1e6,
               run<4, 0>((uint4 *)ids, (uint4 *)w, d_rows, sets, bm, out, grid),
               run<4, 1>((uint4 *)ids, (uint4 *)w, d_rows, sets, bm, out, grid));
    }
    {   // contiguous rows (one block)
        std::vector<std::vector<uint64_t>> sets(23, std::vector<uint64_t>(2470));
        uint64_t b = 0;
        for (auto &s : sets) { for (size_t i = 0; i < s.size(); i++) s[i] = b + i * kRowLen; b += 2470ull * kRowLen; }
        printf("contiguous: ids U=4 %.2f us, ids+w U=4 %.2f us\n",
               run<4, 0>((uint4 *)ids, (uint4 *)w, d_rows, sets, bm, out, grid),
               run<4, 1>((uint4 *)ids, (uint4 *)w, d_rows, sets, bm, out, grid));
    }
    {   // empty launch
        std::vector<std::vector<uint64_t>> sets(23, std::vector<uint64_t>(1, 0));
        printf("1 row (launch floor): %.2f us\n", run<4, 0>((uint4 *)ids, (uint4 *)w, d_rows, sets, bm, out, grid));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
