// Microbenchmark: the forced-flush access pattern -- ~2400 random rows of 10 KB
// (ids) + 10 KB (weights) out of an 8 GB graph, L2 flushed between runs --
// read by (a) LDG.128 CTA-per-row, (b) LDG.128 warp-per-2KB-piece, (c) TMA
// bulk copies of 2 KB / 8 KB pieces into a shared ring; vs one contiguous 48 MB read.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void k_rows(const uint4 *buf, const uint64_t *offs, uint32_t nrow, uint32_t rowvec, uint64_t half, uint32_t *out) {
    uint32_t acc = 0;
    for (uint32_t r = blockIdx.x; r < nrow; r += gridDim.x) {
        const uint4 *p = buf + offs[r], *q = p + half;
        for (uint32_t x = threadIdx.x; x < rowvec; x += blockDim.x) { uint4 v = __ldg(p + x), w = __ldg(q + x); acc += v.x ^ w.w; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_pieces(const uint4 *buf, const uint64_t *offs, uint32_t nrow, uint32_t rowvec, uint64_t half, uint32_t *out) {
    // warp per 128-vector piece (2 KB), 4 vectors per lane
    uint32_t acc = 0;
    const uint32_t lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t ppr = (rowvec + 127) / 128;
    for (uint32_t p = gw; p < nrow * ppr; p += nw) {
        const uint32_t r = p / ppr, c0 = (p % ppr) * 128;
        const uint4 *a = buf + offs[r], *b = a + half;
        uint4 v[4], w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) { uint32_t c = c0 + lane + 32 * q; if (c < rowvec) { v[q] = __ldg(a + c); w[q] = __ldg(b + c); } else { v[q] = w[q] = make_uint4(0,0,0,0); } }
#pragma unroll
        for (int q = 0; q < 4; q++) acc += v[q].x ^ w[q].w;
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int PIECE>
__global__ void k_tma(const uint4 *buf, const uint64_t *offs, uint32_t nrow, uint32_t rowvec, uint64_t half, uint32_t *out, uint32_t nst) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + 64;
    unsigned char *stg = sm + 1024;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ncons = blockDim.x / 32 - 1;
    const uint32_t ppr = (rowvec + PIECE - 1) / PIECE;
    const uint32_t np = nrow * ppr;
    const uint32_t pb = (uint32_t)((uint64_t)np * blockIdx.x / gridDim.x), pe = (uint32_t)((uint64_t)np * (blockIdx.x + 1) / gridDim.x);
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < nst; s++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + s)), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(empty + s)), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t acc = 0;
    if (warp == ncons) {
        if (lane == 0)
            for (uint32_t p = pb; p < pe; p++) {
                const uint32_t g = p - pb, s = g % nst;
                uint32_t ok = 0;
                while (!ok) asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }" : "=r"(ok) : "r"(smem_u32(empty + s)), "r"(((g / nst) & 1) ^ 1) : "memory");
                const uint32_t r = p / ppr, c0 = (p % ppr) * PIECE, n = min((uint32_t)PIECE, rowvec - c0);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(full + s)), "r"(32 * n) : "memory");
                const uint4 *a = buf + offs[r] + c0;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(stg + s * 32 * PIECE)), "l"(a), "r"(16 * n), "r"(smem_u32(full + s)) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(stg + s * 32 * PIECE + 16 * PIECE)), "l"(a + half), "r"(16 * n), "r"(smem_u32(full + s)) : "memory");
            }
    } else {
        for (uint32_t p = pb + warp; p < pe; p += ncons) {
            const uint32_t g = p - pb, s = g % nst;
            uint32_t ok = 0;
            while (!ok) asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }" : "=r"(ok) : "r"(smem_u32(full + s)), "r"((g / nst) & 1) : "memory");
            const uint4 *st = (const uint4 *)(stg + s * 32 * PIECE);
            for (uint32_t c = lane; c < PIECE; c += 32) { uint4 v = st[c], w = st[PIECE + c]; acc += v.x ^ w.w; }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)) : "memory");
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}
__global__ void k_flat(const uint4 *buf, uint64_t n, uint32_t *out) {
    uint32_t acc = 0;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) { uint4 v = __ldg(buf + x); acc += v.x; }
    if (acc == 0x12345678u) out[0] = acc;
}
int main() {
    const uint64_t B = 8ull << 30, half = B / 32;     // ids in the first half, weights in the second (in uint4)
    uint4 *buf; cudaMalloc(&buf, B); cudaMemset(buf, 1, B);
    uint32_t *out; cudaMalloc(&out, 4);
    char *fl; cudaMalloc(&fl, 512ull << 20);
    const uint32_t nrow = 2400, rowvec = 640;
    uint64_t *offs; cudaMalloc(&offs, 8ull * nrow);
    std::vector<uint64_t> h(nrow);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaFuncSetAttribute(k_tma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_tma<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    uint64_t x = 88172645463325252ull;
    uint64_t span = half;      // rows drawn from the first `span` uint4 of each half
    auto run = [&](const char *name, auto launch) {
        float tot = 0; int n = 0;
        for (int rep = 0; rep < 6; rep++) {
            for (uint32_t i = 0; i < nrow; i++) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; h[i] = (x % (span - rowvec)) & ~7ull; }
            cudaMemcpy(offs, h.data(), 8ull * nrow, cudaMemcpyHostToDevice);
            cudaMemset(fl, rep, 512ull << 20);
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (rep) { tot += ms; n++; }
        }
        const double us = tot / n * 1e3;
        printf("%-34s %8.2f us  %.2f TB/s\n", name, us, 2.0 * nrow * rowvec * 16 / (us * 1e-6) / 1e12);
        fflush(stdout);
    };
    run("CTA/row 512thr x148x2", [&] { k_rows<<<296, 512>>>(buf, offs, nrow, rowvec, half, out); });
    run("CTA/row 1024thr x148", [&] { k_rows<<<148, 1024>>>(buf, offs, nrow, rowvec, half, out); });
    run("warp/piece 4/lane 1024x148", [&] { k_pieces<<<148, 1024>>>(buf, offs, nrow, rowvec, half, out); });
    run("warp/piece 4/lane 512x296", [&] { k_pieces<<<296, 512>>>(buf, offs, nrow, rowvec, half, out); });
    // (nst a multiple of the 16 consumer warps: each slot is consumed by one warp, in phase order)
    for (uint32_t nst : {16u, 32u, 48u}) {
        char nm[64]; snprintf(nm, 64, "TMA 4KB pieces x%u stages", nst);
        run(nm, [&] { k_tma<128><<<148, 544, 1024 + nst * 4096>>>(buf, offs, nrow, rowvec, half, out, nst); });
    }
    for (uint64_t mb : {64ull, 256ull, 1024ull, 4096ull}) {
        span = (mb << 20) / 16;
        char nm[64]; snprintf(nm, 64, "warp/piece span %llu MB", (unsigned long long)mb);
        run(nm, [&] { k_pieces<<<148, 1024>>>(buf, offs, nrow, rowvec, half, out); });
    }
    span = half;
    run("flat 49 MB contiguous", [&] { k_flat<<<148 * 4, 512>>>(buf + 12345678, 2ull * nrow * rowvec, out); });
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
