// build.cu -- on-GPU construction of the neuron-domain-sliced CSR graph
// (Sec. III P:185 "constructed only once", Fig. 1
// P:180 pivots, Sec. III-B P:348 slices, Sec. IV-B P:391 GPU setup).
//
// Row i lists, ascending, every target j in this rank's range [tgt_lo, tgt_hi)
// kept by the Bernoulli draw of reading R22/R23.  Pivots are NOT binary-searched
// here (the oracle does that): the count pass produces per-(row, slice)
// counts whose exclusive prefix IS the pivot row -- an independent route to the
// same table, so the two cross-check each other.
#include <cub/cub.cuh>

#include "common.cuh"
#include "philox.cuh"

namespace snn {

constexpr int kBuildThreads = 256;

// Decision for 4 consecutive candidates j0..j0+3 of source row i.
// Returns a 4-bit mask (bit e = candidate j0+e kept).
__device__ __forceinline__ uint32_t decide4(const NetDev &net, const uint64_t *thr_tab,
                                            const uint8_t *autapse_tab, int sp, uint32_t i,
                                            uint32_t j0, uint32_t jend) {
    uint32_t mask = 0;
    int cached_dp = -1;
    uint32_t cached_q = 0xffffffffu;
    u32x4 r{0, 0, 0, 0};
    int dp = find_pop(net, j0 < net.N ? j0 : net.N - 1);
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const uint32_t j = j0 + e;
        if (j >= jend) break;
        while (dp + 1 < (int)net.npop && j >= net.pop[dp + 1].base) dp++;
        const uint64_t thr = thr_tab[sp * kMaxPops + dp];
        if (thr == 0) continue;                       // no projection sp -> dp (or p == 0)
        if (j == i && !autapse_tab[sp * kMaxPops + dp]) continue;
        const uint32_t jl = j - net.pop[dp].base;
        const uint32_t qd = jl >> 2;
        if (dp != cached_dp || qd != cached_q) {
            r = philox4x32_10(i, qd, 1u, (uint32_t)dp, net.key0, net.key1);
            cached_dp = dp;
            cached_q = qd;
        }
        if ((uint64_t)lane_of(r, jl & 3u) < thr) mask |= 1u << e;
    }
    return mask;
}

// Pass 1: per (row, slice) counts -> piv[i][k+1]; piv[i][0] = 0.  The CTA of
// row i walks the row's candidates 1024 at a time (4 per thread, one Philox
// draw); a thread adds its kept count to its slice's shared counter, so there
// is no barrier per slice.
__global__ void __launch_bounds__(kBuildThreads)
k_count(NetDev net, BuildTabs tabs, uint32_t *piv, uint32_t row0, uint32_t nrows) {
    extern __shared__ uint32_t cnt_s[];           // [nslices]
    const uint32_t i = row0 + blockIdx.x;
    if (i >= row0 + nrows) return;
    const int sp = find_pop(net, i);
    const uint32_t P = net.nslices + 1;
    uint32_t *prow = piv + (size_t)i * P;
    bool any = false;
    for (int d = 0; d < (int)net.npop; d++) any |= tabs.thr[sp * kMaxPops + d] != 0;
    for (uint32_t k = threadIdx.x; k < net.nslices; k += kBuildThreads) cnt_s[k] = 0;
    __syncthreads();
    if (any) {
        for (uint32_t j0 = net.tgt_lo + 4 * threadIdx.x; j0 < net.tgt_hi; j0 += 4 * kBuildThreads) {
            const uint32_t m = decide4(net, tabs.thr, tabs.autapse, sp, i, j0, net.tgt_hi);
            if (m) atomicAdd(&cnt_s[(j0 - net.tgt_lo) >> net.log2C], (uint32_t)__popc(m));   // C >= 32: one slice
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) prow[0] = 0;
    for (uint32_t k = threadIdx.x; k < net.nslices; k += kBuildThreads) prow[k + 1] = cnt_s[k];
}

// Pass 2: per row, counts -> exclusive prefix (the pivots); row length out.
__global__ void k_pivot_scan(NetDev net, uint32_t *piv, int64_t *len, uint32_t nrows) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= nrows) return;
    const uint32_t P = net.nslices + 1;
    uint32_t *prow = piv + (size_t)warp * P;
    uint32_t carry = 0;
    for (uint32_t b = 1; b < P; b += 32) {
        const uint32_t k = b + lane;
        uint32_t v = k < P ? prow[k] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (k < P) prow[k] = carry + v;
        carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) len[warp] = carry;
}

// Pass 3: fill targets (sorted by construction) and initial weights.  The CTA
// of row i walks the row's candidates 4096 at a time (16 per thread, four
// Philox draws); one block scan of the kept counts orders the writes.
constexpr int kFillPer = 16;                      // candidates per thread and pass
__global__ void __launch_bounds__(kBuildThreads)
k_fill(NetDev net, BuildTabs tabs, const uint32_t *piv, const int64_t *row_ptr, uint32_t *idx,
       float *w) {
    typedef cub::BlockScan<uint32_t, kBuildThreads> Scan;
    __shared__ typename Scan::TempStorage tmp;
    const uint32_t i = blockIdx.x;
    const int sp = find_pop(net, i);
    const uint32_t P = net.nslices + 1;
    const uint32_t *prow = piv + (size_t)i * P;
    if (prow[net.nslices] == 0) return;
    int64_t pos = row_ptr[i];
    for (uint32_t jb = net.tgt_lo; jb < net.tgt_hi; jb += kFillPer * kBuildThreads) {
        const uint32_t j0 = jb + kFillPer * threadIdx.x;
        uint32_t m = 0;                           // bit e: candidate j0 + e kept
#pragma unroll
        for (int q = 0; q < kFillPer / 4; q++)
            if (j0 + 4 * q < net.tgt_hi)
                m |= decide4(net, tabs.thr, tabs.autapse, sp, i, j0 + 4 * q, net.tgt_hi) << (4 * q);
        uint32_t off, tot;
        Scan(tmp).ExclusiveSum((uint32_t)__popc(m), off, tot);
        while (m) {
            const int e = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t j = j0 + e;
            const int dp = find_pop(net, j);
            idx[pos + off] = j;
            w[pos + off] = tabs.weight[sp * kMaxPops + dp];
            off++;
        }
        pos += tot;
        __syncthreads();
    }
}

// Plastic segment [lo, hi) of each PF_PRE_PLASTIC row: the targets inside the
// STDP projection's destination population (rows are sorted, so it is one
// contiguous run, found by binary search).
__global__ void k_segments(NetDev net, const int64_t *row_ptr, const uint32_t *idx, uint2 *seg) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    const int sp = find_pop(net, i);
    uint2 s = make_uint2(0, 0);
    if (net.pop[sp].stdp >= 0) {
        const PopDev &dp = net.pop[net.stdp[net.pop[sp].stdp].dst_pop];
        const int64_t b = row_ptr[i], e = row_ptr[i + 1];
        auto lb = [&](uint32_t v) {
            int64_t a = b, c = e;
            while (a < c) {
                const int64_t m = (a + c) >> 1;
                if (idx[m] < v) a = m + 1; else c = m;
            }
            return (uint32_t)(a - b);
        };
        s.x = lb(dp.base);
        s.y = lb(dp.base + dp.n);
    }
    seg[i] = s;
}

// Initial state: V0 = v_reset + (v_th - v_reset) * u, u = (x >> 8) 2^-24 with
// x = Philox(i, 0, 3, 0).x; all else 0; tlu = -1 (R4).
__global__ void k_init_state(NetDev net, StateDev st) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    const PopDev &p = net.pop[find_pop(net, i)];
    float v = 0.0f;
    if (p.kind != POP_POISSON) {
        const u32x4 r = philox4x32_10(i, 0u, 3u, 0u, net.key0, net.key1);
        const float u = __fmul_rn(__uint2float_rn(r.x >> 8), 0x1p-24f);
        const float span = __fsub_rn(p.v_th, p.v_reset);
        v = __fadd_rn(p.v_reset, __fmul_rn(span, u));
    }
    st.V[i] = v;
    st.ge[i] = 0.0f;
    st.gi[i] = 0.0f;
    st.xpost[i] = 0.0f;
    st.ref[i] = 0;
    st.in_e[i] = 0;
    st.in_i[i] = 0;
    st.hist[i] = 0ull;
    if (net.H > 64) st.hist_hi[i] = 0ull;
    st.nspk[i] = 0u;
    st.xpre[i] = 0.0f;
    st.tlu[i] = -1;
}

// ---------------------------------------------------------------- launchers
cudaError_t build_count(const NetDev &net, const BuildTabs &tabs, uint32_t *piv, cudaStream_t s) {
    const size_t smem = 4ull * (net.nslices > 0 ? net.nslices : 1);
    if (smem > 48 * 1024) {
        if (smem > 227 * 1024) return cudaErrorInvalidValue;       // > 58K slices per rank
        const cudaError_t e = cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const uint32_t chunk = 1u << 20;
    for (uint32_t r0 = 0; r0 < net.N; r0 += chunk) {
        const uint32_t nr = min(chunk, net.N - r0);
        k_count<<<nr, kBuildThreads, smem, s>>>(net, tabs, piv, r0, nr);
    }
    return cudaGetLastError();
}

cudaError_t build_scan(const NetDev &net, uint32_t *piv, int64_t *len, int64_t *row_ptr,
                       void *tmp, size_t *tmp_bytes, cudaStream_t s) {
    if (tmp == nullptr) {
        return cub::DeviceScan::ExclusiveSum(nullptr, *tmp_bytes, len, row_ptr, (int)net.N + 1, s);
    }
    k_pivot_scan<<<(net.N * 32 + 255) / 256, 256, 0, s>>>(net, piv, len, net.N);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // len[N] = 0 was set by the caller; row_ptr = exclusive scan over N+1 entries
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, len, row_ptr, (int)net.N + 1, s);
}

cudaError_t build_fill(const NetDev &net, const BuildTabs &tabs, const uint32_t *piv,
                       const int64_t *row_ptr, uint32_t *idx, float *w, cudaStream_t s) {
    k_fill<<<net.N, kBuildThreads, 0, s>>>(net, tabs, piv, row_ptr, idx, w);
    return cudaGetLastError();
}

// Compressed indices: a target's offset in its slice,
// (j - tgt_lo) mod C -- every (row, slice) segment indexes only C neurons.
__global__ void k_idx16(NetDev net, const uint32_t *idx, uint16_t *idx16, int64_t S) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < S; c += (int64_t)gridDim.x * blockDim.x)
        idx16[c] = (uint16_t)((idx[c] - net.tgt_lo) & (net.C - 1u));
}

cudaError_t build_idx16(const NetDev &net, const uint32_t *idx, uint16_t *idx16, int64_t S, cudaStream_t s) {
    if (S > 0) k_idx16<<<1184, 256, 0, s>>>(net, idx, idx16, S);
    return cudaGetLastError();
}

cudaError_t build_segments(const NetDev &net, const int64_t *row_ptr, const uint32_t *idx,
                           uint2 *seg, cudaStream_t s) {
    k_segments<<<(net.N + 255) / 256, 256, 0, s>>>(net, row_ptr, idx, seg);
    return cudaGetLastError();
}

cudaError_t init_state(const NetDev &net, const StateDev &st, cudaStream_t s) {
    k_init_state<<<(net.N + 255) / 256, 256, 0, s>>>(net, st);
    return cudaGetLastError();
}

}  // namespace snn
