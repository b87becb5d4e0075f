// Microbenchmark: the delivery access pattern -- 110K random (row, slice)
// segments of ~20 synapses -- read as two separate arrays (u32 ids + f32
// weights, SoA) vs one interleaved array of (id, weight) pairs (AoS).
// A CTA per "slice" strides its segments' elements 512 wide, 8 in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int kT = 512, kU = 8;
__global__ void k_soa(const uint32_t *idx, const float *w, const uint64_t *seg, const uint32_t *len, int nseg_per_cta,
                      uint32_t *out) {
    __shared__ uint32_t s_start[1025];
    const uint64_t *sg = seg + (size_t)blockIdx.x * nseg_per_cta;
    // flatten: prefix of lengths (serial by thread 0 for simplicity)
    for (int i = threadIdx.x; i <= nseg_per_cta; i += blockDim.x) s_start[i] = len[blockIdx.x * (nseg_per_cta + 1) + i];
    __syncthreads();
    const uint32_t T = s_start[nseg_per_cta];
    uint32_t acc = 0;
    for (uint32_t x0 = 0; x0 < T; x0 += kT * kU) {
        uint32_t j[kU]; float ww[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint32_t x = min(x0 + u * kT + threadIdx.x, T - 1);
            int lo = 0, hi = nseg_per_cta;
            while (hi - lo > 1) { int m = (lo + hi) / 2; if (s_start[m] <= x) lo = m; else hi = m; }
            const uint64_t c = sg[lo] + (x - s_start[lo]);
            j[u] = __ldg(idx + c); ww[u] = __ldg(w + c);
        }
#pragma unroll
        for (int u = 0; u < kU; u++) acc += j[u] ^ __float_as_uint(ww[u]);
    }
    if (acc == 0x12345u) out[0] = acc;
}
__global__ void k_aos(const uint2 *iw, const uint64_t *seg, const uint32_t *len, int nseg_per_cta, uint32_t *out) {
    __shared__ uint32_t s_start[1025];
    const uint64_t *sg = seg + (size_t)blockIdx.x * nseg_per_cta;
    for (int i = threadIdx.x; i <= nseg_per_cta; i += blockDim.x) s_start[i] = len[blockIdx.x * (nseg_per_cta + 1) + i];
    __syncthreads();
    const uint32_t T = s_start[nseg_per_cta];
    uint32_t acc = 0;
    for (uint32_t x0 = 0; x0 < T; x0 += kT * kU) {
        uint2 v[kU];
#pragma unroll
        for (int u = 0; u < kU; u++) {
            const uint32_t x = min(x0 + u * kT + threadIdx.x, T - 1);
            int lo = 0, hi = nseg_per_cta;
            while (hi - lo > 1) { int m = (lo + hi) / 2; if (s_start[m] <= x) lo = m; else hi = m; }
            const uint64_t c = sg[lo] + (x - s_start[lo]);
            v[u] = __ldg(iw + c);
        }
#pragma unroll
        for (int u = 0; u < kU; u++) acc += v[u].x ^ v[u].y;
    }
    if (acc == 0x12345u) out[0] = acc;
}
int main() {
    const uint64_t S = 1000000000ull;   // 1e9 synapses (cfg3)
    uint32_t *idx; float *w; uint2 *iw;
    cudaMalloc(&idx, 4 * S); cudaMalloc(&w, 4 * S); cudaMalloc(&iw, 8 * S);
    cudaMemset(idx, 1, 4 * S); cudaMemset(w, 1, 4 * S); cudaMemset(iw, 1, 8 * S);
    const int ncta = 155, nsc = 663;   // slices x arriving rows
    const int nseg = ncta * nsc;
    uint64_t *hseg = new uint64_t[nseg]; uint32_t *hlen = new uint32_t[ncta * (nsc + 1)];
    uint64_t x = 88172645463325252ull;
    for (int r = 0; r < nsc; r++) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const uint64_t row = (x % (S / 3162 - 1)) * 3162;     // random row of 3162 synapses
        for (int k = 0; k < ncta; k++) { hseg[k * nsc + r] = row + k * 20; hlen[k * (nsc + 1) + r] = 20 * r; }
    }
    for (int k = 0; k < ncta; k++) hlen[k * (nsc + 1) + nsc] = 20 * nsc;
    uint64_t *seg; uint32_t *len, *out;
    cudaMalloc(&seg, 8ull * nseg); cudaMalloc(&len, 4ull * ncta * (nsc + 1)); cudaMalloc(&out, 4);
    cudaMemcpy(seg, hseg, 8ull * nseg, cudaMemcpyHostToDevice); cudaMemcpy(len, hlen, 4ull * ncta * (nsc + 1), cudaMemcpyHostToDevice);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 3; rep++) {
        float t1, t2;
        cudaEventRecord(a); k_soa<<<ncta, kT>>>(idx, w, seg, len, nsc, out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&t1, a, b);
        cudaEventRecord(a); k_aos<<<ncta, kT>>>(iw, seg, len, nsc, out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&t2, a, b);
        printf("110K segments x 20 synapses: SoA (ids, weights) %.1f us, AoS (id, weight) pairs %.1f us\n", t1 * 1e3, t2 * 1e3);
    }
    return 0;
}
