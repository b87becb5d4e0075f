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
#include <cstdlib>

#include "common.cuh"
#include "philox.cuh"

namespace snn {

constexpr int kGeoThreads = 128;

// Exact geometric skipping (R32): the kept candidates of row i
// in destination population d are reached by gaps g >= 1 with P(g > k) =
// gap[k-1] / 2^32 = floor((1-p)^k 2^32) / 2^32, drawn from the counter-based
// stream Philox(i, n >> 2, 4, d)[n & 3] -- the law of independent Bernoulli(p)
// trials with one draw per synapse instead of one per candidate pair.  The
// candidates are d's neurons ascending without i itself (no autapse, R21).
// A draw beyond the table advances kGapTab and keeps nothing (memoryless).
// Calls f(j) for every kept target j < hi, ascending; stops at hi.
template <typename F>
__device__ __forceinline__ void geo_row(const NetDev &net, const BuildTabs &tabs, uint32_t i, int sp,
                                        uint32_t hi, F &&f) {
    for (int d = 0; d < (int)net.npop; d++) {
        const int slot = tabs.gap_slot[sp * kMaxPops + d];
        if (slot < 0) continue;
        const PopDev &dp = net.pop[d];
        if (dp.base >= hi) break;
        const uint32_t *tab = tabs.gap + (size_t)slot * kGapTab;
        const bool excl = !tabs.autapse[sp * kMaxPops + d] && i >= dp.base && i < dp.base + dp.n;
        const uint32_t il = i - dp.base;
        const int64_t M = (int64_t)dp.n - (excl ? 1 : 0);
        int64_t c = -1;
        u32x4 r = {0, 0, 0, 0};
        for (uint32_t n = 0;; n++) {
            if ((n & 3u) == 0) r = philox4x32_10(i, n >> 2, 4u, (uint32_t)d, net.key0, net.key1);
            const uint32_t x = lane_of(r, n & 3u);
            uint32_t lo = 0, up = kGapTab;        // entries > x (the table is non-increasing)
            while (lo < up) {
                const uint32_t mid = (lo + up) >> 1;
                if (__ldg(tab + mid) > x) lo = mid + 1; else up = mid;
            }
            // g = 1 + #{k : gap[k-1] > x}; lo == kGapTab: beyond the table -> advance kGapTab, keep nothing
            const bool beyond = lo == (uint32_t)kGapTab;
            c += beyond ? (int64_t)kGapTab : (int64_t)lo + 1;
            if (c >= M) break;
            if (beyond) continue;
            const uint32_t jl = (uint32_t)c + ((excl && (uint32_t)c >= il) ? 1u : 0u);
            const uint32_t j = dp.base + jl;
            if (j >= hi) return;
            f(j, d);
        }
    }
}

// ---- warp-cooperative rows: the same draws as geo_row, a warp
// per row.  Lane l of an iteration draws n = n0 + 4 l .. n0 + 4 l + 3 (one
// Philox call, counter (i, n0 / 4 + l, 4, d)); the gap of a draw comes from
// the inverse CDF, g - 1 = #{k in [1, kGapTab] : gap[k-1] > x}, estimated as
// ceil(log(x 2^-32) / log(1 - p)) - 1 and corrected against the table (exact:
// the table decides); a warp prefix sum of the gaps gives every draw's
// candidate position.  Kept targets in [lo, hi) are passed, ascending, to
// emit(lane's j[4], mask, rank of its first one among the row's kept targets,
// d) once per iteration (every lane; uniform call).
__device__ __forceinline__ uint32_t geo_gap_count(const uint32_t *__restrict__ tab, float inv_l2q, uint32_t x) {
    // #{k in [1, kGapTab] : tab[k-1] > x} (tab non-increasing)
    int k;
    if (x == 0u) {
        k = kGapTab;
    } else {
        const float e = __log2f((float)x) - 32.0f;          // log2(x 2^-32) < 0
        const float ks = ceilf(e * inv_l2q) - 1.0f;         // inv_l2q = 1 / log2(1 - p) < 0
        k = ks < 0.0f ? 0 : ks > (float)kGapTab ? kGapTab : (int)ks;
    }
    // correct: want tab[k-1] > x (or k == 0) and (k == kGapTab or tab[k] <= x)
    int steps = 0;
    while (k < kGapTab && __ldg(tab + k) > x && steps < 4) { k++; steps++; }
    while (k > 0 && __ldg(tab + k - 1) <= x && steps < 4) { k--; steps++; }
    if (steps >= 4) {                                         // (far off: x tiny) -- binary search
        uint32_t lo = 0, up = kGapTab;
        while (lo < up) {
            const uint32_t mid = (lo + up) >> 1;
            if (__ldg(tab + mid) > x) lo = mid + 1; else up = mid;
        }
        k = (int)lo;
    }
    return (uint32_t)k;
}

template <typename F>
__device__ __forceinline__ void geo_row_warp(const NetDev &net, const BuildTabs &tabs, uint32_t i, int sp, uint32_t lo,
                                             uint32_t hi, F &&emit) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t kept_before = 0;                         // kept synapses of the row so far
    for (int d = 0; d < (int)net.npop; d++) {
        const int slot = tabs.gap_slot[sp * kMaxPops + d];
        if (slot < 0) continue;
        const PopDev &dp = net.pop[d];
        if (dp.base >= hi) break;
        const uint32_t *tab = tabs.gap + (size_t)slot * kGapTab;
        const float inv_l2q = tabs.inv_l2q[sp * kMaxPops + d];
        const bool excl = !tabs.autapse[sp * kMaxPops + d] && i >= dp.base && i < dp.base + dp.n;
        const uint32_t il = i - dp.base;
        const int64_t M = (int64_t)dp.n - (excl ? 1 : 0);
        int64_t c0 = -1;                              // candidate position of the last draw so far
        for (uint32_t n0 = 0;; n0 += 128) {
            const u32x4 r = philox4x32_10(i, (n0 >> 2) + lane, 4u, (uint32_t)d, net.key0, net.key1);
            uint32_t g[4], keep = 0, kk[4];
            int64_t gs = 0;
            // the inverse-CDF estimates of the lane's four gaps and both table
            // entries that confirm them, loaded together; a draw whose estimate
            // the table does not confirm takes the corrected search (rare)
            {
                uint32_t t0[4], t1[4];
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const uint32_t x = lane_of(r, (uint32_t)e);
                    int k = kGapTab;
                    if (x != 0u) {
                        const float ks = ceilf((__log2f((float)x) - 32.0f) * inv_l2q) - 1.0f;
                        k = ks < 0.0f ? 0 : ks > (float)kGapTab ? kGapTab : (int)ks;
                    }
                    kk[e] = (uint32_t)k;
                    t0[e] = k > 0 ? __ldg(tab + k - 1) : 0xffffffffu;        // want tab[k-1] > x (or k == 0)
                    t1[e] = k < kGapTab ? __ldg(tab + k) : 0u;               // want tab[k] <= x (or k == kGapTab)
                }
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    const uint32_t x = lane_of(r, (uint32_t)e);
                    const bool ok = (kk[e] == 0u || t0[e] > x) && t1[e] <= x;
                    if (!ok) kk[e] = geo_gap_count(tab, inv_l2q, x);
                }
            }
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const uint32_t k = kk[e];
                const bool beyond = k == (uint32_t)kGapTab;   // advance kGapTab, keep nothing
                g[e] = beyond ? (uint32_t)kGapTab : k + 1;
                keep |= (beyond ? 0u : 1u) << e;
                gs += g[e];
            }
            // warp exclusive prefix of the lanes' gap sums (64-bit: rows beyond 2^32 candidates never occur,
            // but the sum of 128 gaps stays < 2^20)
            uint32_t inc = (uint32_t)gs;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= (uint32_t)o) inc += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            int64_t c = c0 + (int64_t)(inc - (uint32_t)gs);
            uint32_t jv[4], mask = 0;
            bool stop = false;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                c += g[e];
                jv[e] = 0;
                if (c >= M) { stop = true; continue; }
                if (!((keep >> e) & 1u)) continue;
                const uint32_t jl = (uint32_t)c + ((excl && (uint32_t)c >= il) ? 1u : 0u);
                const uint32_t j = dp.base + jl;
                if (j >= hi) { stop = true; continue; }         // (and every later one: the row ends)
                if (j < lo) continue;
                jv[e] = j;
                mask |= 1u << e;
            }
            // (a stop condition is monotone in n: every later draw is stopped too)
            const uint32_t nk = __popc(mask);
            uint32_t kin = nk;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, kin, o);
                if (lane >= (uint32_t)o) kin += y;
            }
            emit(jv, mask, kept_before + kin - nk, d);
            kept_before += __shfl_sync(0xffffffffu, kin, 31);
            if (__any_sync(0xffffffffu, stop)) break;    // (a stop is monotone in n: every later draw stops too)
            c0 += tot;
        }
    }
}

constexpr int kGeoWarpThreads = 256;   // 8 rows per CTA

// Pass 1 (warp per row): the pivots directly -- piv[i][k] = #kept targets
// below B_k = tgt_lo + kC (Fig. 1) -- and the row length.  Targets ascend, so
// after an iteration whose last kept target lies in slice kl, the pivots
// k <= kl not yet written are final: each is the row's kept count before the
// iteration plus the iteration's kept targets below B_k (a warp reduction);
// lane k - k0 holds pivot k and they are stored together, coalesced.
__global__ void __launch_bounds__(kGeoWarpThreads, 4)
k_count_warp(NetDev net, BuildTabs tabs, uint32_t *piv, int64_t *len) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= net.N) return;                           // (warp-uniform)
    const int sp = find_pop(net, i);
    uint32_t *prow = piv + (size_t)i * (net.nslices + 1);
    const uint32_t C = net.C;
    uint32_t next = 0;                                // first pivot not yet written (warp-uniform)
    uint32_t total = 0;
    geo_row_warp(net, tabs, i, sp, net.tgt_lo, net.tgt_hi, [&](const uint32_t (&jv)[4], uint32_t mask, uint32_t q0, int) {
        // the iteration's last kept target (every lane: the warp maximum)
        uint32_t jmax = 0;
        bool any = false;
#pragma unroll
        for (int e = 0; e < 4; e++)
            if ((mask >> e) & 1u) { jmax = jv[e]; any = true; }
        const uint32_t kb = __ballot_sync(0xffffffffu, any);
        const uint32_t nk_it = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(mask));
        const uint32_t before = __shfl_sync(0xffffffffu, q0, 0);       // kept before this iteration
        if (kb) {
            jmax = __shfl_sync(0xffffffffu, jmax, 31 - __clz(kb));      // (the highest lane with a kept target)
            const uint32_t kl = (jmax - net.tgt_lo) / C;                // its slice: pivots next .. kl are final
            for (uint32_t k0 = next; k0 <= kl; k0 += 32) {
                uint32_t val = 0;
                const uint32_t kend = min(kl + 1, k0 + 32u);
                for (uint32_t k = k0; k < kend; k++) {                  // (warp-uniform loop)
                    const uint32_t Bk = net.tgt_lo + k * C;
                    uint32_t below = 0;
#pragma unroll
                    for (int e = 0; e < 4; e++) below += (((mask >> e) & 1u) && jv[e] < Bk) ? 1u : 0u;
                    below = __reduce_add_sync(0xffffffffu, below);
                    if (lane == k - k0) val = before + below;
                }
                if (k0 + lane < kend) prow[k0 + lane] = val;
            }
            next = kl + 1;
        }
        total = before + nk_it;
    });
    // slices after the last kept target: the row length
    for (uint32_t k = next + lane; k <= net.nslices; k += 32) prow[k] = total;
    if (lane == 0) len[i] = total;
}

// Pass 3 (warp per row): targets (sorted by construction) and initial weights;
// an iteration's kept targets are staged in shared memory by rank, then
// written out coalesced.
__global__ void __launch_bounds__(kGeoWarpThreads, 4)
k_fill_warp(NetDev net, BuildTabs tabs, const int64_t *row_ptr, uint32_t *idx, float *w) {
    __shared__ uint32_t stage[kGeoWarpThreads / 32][128];
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= net.N) return;
    uint32_t *buf = stage[threadIdx.x >> 5];
    const int sp = find_pop(net, i);
    const int64_t base = row_ptr[i];
    geo_row_warp(net, tabs, i, sp, net.tgt_lo, net.tgt_hi, [&](const uint32_t (&jv)[4], uint32_t mask, uint32_t q0, int d) {
        const float wd = tabs.weight[sp * kMaxPops + d];
        const uint32_t before = __shfl_sync(0xffffffffu, q0, 0);
        uint32_t q = q0 - before;
#pragma unroll
        for (int e = 0; e < 4; e++) {
            if (!((mask >> e) & 1u)) continue;
            buf[q++] = jv[e];
        }
        const uint32_t n = __shfl_sync(0xffffffffu, q, 31);             // (lane 31's rank end = the count)
        __syncwarp();
        for (uint32_t x = lane; x < n; x += 32) {
            idx[base + before + x] = buf[x];
            w[base + before + x] = wd;
        }
        __syncwarp();
    });
}

// Pass 1: per (row, slice) counts -> piv[i][k+1]; piv[i][0] = 0 (thread per row;
// the targets come ascending, so the slices are written in order).
__global__ void __launch_bounds__(kGeoThreads)
k_count(NetDev net, BuildTabs tabs, uint32_t *piv) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    const int sp = find_pop(net, i);
    uint32_t *prow = piv + (size_t)i * (net.nslices + 1);
    prow[0] = 0;
    uint32_t k = 0, cnt = 0;                      // current slice and its count
    geo_row(net, tabs, i, sp, net.tgt_hi, [&](uint32_t j, int) {
        if (j < net.tgt_lo) return;
        const uint32_t kj = (j - net.tgt_lo) / net.C;
        while (k < kj) {
            prow[k + 1] = cnt;
            cnt = 0;
            k++;
        }
        cnt++;
    });
    for (; k < net.nslices; k++) {
        prow[k + 1] = cnt;
        cnt = 0;
    }
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

// Pass 3: fill targets (sorted by construction) and initial weights.
__global__ void __launch_bounds__(kGeoThreads)
k_fill(NetDev net, BuildTabs tabs, const int64_t *row_ptr, uint32_t *idx, float *w) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    const int sp = find_pop(net, i);
    int64_t pos = row_ptr[i];
    geo_row(net, tabs, i, sp, net.tgt_hi, [&](uint32_t j, int d) {
        if (j < net.tgt_lo) return;
        idx[pos] = j;
        w[pos] = tabs.weight[sp * kMaxPops + d];
        pos++;
    });
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
    for (int b = 0; b < 4; b++) st.fpos[(size_t)b * st.fstride + i] = 0xfeu;
    for (int b = 0; b < 12; b++) st.fpot[(size_t)b * st.fstride + i] = 0.0f;
    st.nspk[i] = 0u;
    st.xpre[i] = 0.0f;
    st.tlu[i] = -1;
}

// ---------------------------------------------------------------- launchers
// (SNN_BUILD_THREAD_PER_ROW: the round-1 thread-per-row builder, for comparison)
static bool build_thread_per_row() { return getenv("SNN_BUILD_THREAD_PER_ROW") != nullptr; }

// Load the construction kernels' modules (lazy loading would otherwise load
// each on its first launch, inside the device-timed construction), the CUB
// scan's included by one scan of a single element.
cudaError_t build_preload(cudaStream_t s) {
    cudaFuncAttributes a;
    cudaError_t e;
    const void *ks[] = {(const void *)k_count_warp, (const void *)k_fill_warp, (const void *)k_count,
                        (const void *)k_fill, (const void *)k_pivot_scan, (const void *)k_segments};
    for (const void *k : ks)
        if ((e = cudaFuncGetAttributes(&a, k)) != cudaSuccess) return e;
    int64_t *buf = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    if ((e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, buf, buf, 1, s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&buf, 2 * sizeof(int64_t), s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync(&tmp, tmp_bytes + 16, s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(buf, 0, 2 * sizeof(int64_t), s)) != cudaSuccess) return e;
    if ((e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, buf, buf + 1, 1, s)) != cudaSuccess) return e;
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(buf, s);
    return cudaStreamSynchronize(s);
}

cudaError_t build_count(const NetDev &net, const BuildTabs &tabs, uint32_t *piv, int64_t *len, cudaStream_t s) {
    if (build_thread_per_row()) {
        k_count<<<(net.N + kGeoThreads - 1) / kGeoThreads, kGeoThreads, 0, s>>>(net, tabs, piv);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        k_pivot_scan<<<(net.N * 32 + 255) / 256, 256, 0, s>>>(net, piv, len, net.N);
    } else {
        const uint32_t per = kGeoWarpThreads / 32;
        k_count_warp<<<(net.N + per - 1) / per, kGeoWarpThreads, 0, s>>>(net, tabs, piv, len);
    }
    return cudaGetLastError();
}

cudaError_t build_scan(const NetDev &net, uint32_t *piv, int64_t *len, int64_t *row_ptr,
                       void *tmp, size_t *tmp_bytes, cudaStream_t s) {
    (void)piv;
    if (tmp == nullptr) {
        return cub::DeviceScan::ExclusiveSum(nullptr, *tmp_bytes, len, row_ptr, (int)net.N + 1, s);
    }
    // len[N] = 0 was set by the caller; row_ptr = exclusive scan over N+1 entries
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, len, row_ptr, (int)net.N + 1, s);
}

cudaError_t build_fill(const NetDev &net, const BuildTabs &tabs, const uint32_t *piv,
                       const int64_t *row_ptr, uint32_t *idx, float *w, cudaStream_t s) {
    (void)piv;
    if (build_thread_per_row()) {
        k_fill<<<(net.N + kGeoThreads - 1) / kGeoThreads, kGeoThreads, 0, s>>>(net, tabs, row_ptr, idx, w);
    } else {
        const uint32_t per = kGeoWarpThreads / 32;
        k_fill_warp<<<(net.N + per - 1) / per, kGeoWarpThreads, 0, s>>>(net, tabs, row_ptr, idx, w);
    }
    return cudaGetLastError();
}

// Compressed indices: (j - tgt_lo) mod 2^16.  Every
// (row, slice) segment indexes only C <= 2^16 neurons, so the delivery reads
// the slice offset as (v - (kC mod 2^16)) mod 2^16; the STDP stream rebuilds j
// from the row's crossings of multiples of 2^16 (k_b64).
__global__ void k_idx16(NetDev net, const uint32_t *idx, uint16_t *idx16, int64_t S) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < S; c += (int64_t)gridDim.x * blockDim.x)
        idx16[c] = (uint16_t)((idx[c] - net.tgt_lo) & 0xffffu);
}

// b64[i][m - 1] = #targets j of row i with j - tgt_lo < m 2^16 (lower bound), m = 1..4.
__global__ void k_b64(NetDev net, const int64_t *row_ptr, const uint32_t *idx, uint32_t *b64) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    const int64_t b = row_ptr[i], e = row_ptr[i + 1];
    uint32_t r[4];
#pragma unroll
    for (int m = 1; m <= 4; m++) {
        const uint64_t v = (uint64_t)net.tgt_lo + ((uint64_t)m << 16);
        int64_t a = b, c = e;
        while (a < c) {
            const int64_t mid = (a + c) >> 1;
            if ((uint64_t)idx[mid] < v) a = mid + 1; else c = mid;
        }
        r[m - 1] = (uint32_t)(a - b);
    }
    reinterpret_cast<uint4 *>(b64)[i] = make_uint4(r[0], r[1], r[2], r[3]);
}

cudaError_t build_idx16(const NetDev &net, const uint32_t *idx, uint16_t *idx16, int64_t S, cudaStream_t s) {
    if (S > 0) k_idx16<<<1184, 256, 0, s>>>(net, idx, idx16, S);
    return cudaGetLastError();
}

cudaError_t build_b64(const NetDev &net, const int64_t *row_ptr, const uint32_t *idx, uint32_t *b64, cudaStream_t s) {
    k_b64<<<(net.N + 255) / 256, 256, 0, s>>>(net, row_ptr, idx, b64);
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
