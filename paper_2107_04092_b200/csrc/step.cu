// step.cu -- the per-step hot path:
//   k_neuron   (a1) neuron + Poisson update, firing bits -> bitmask ring, history push
//   k_worklist (a2) arrivals A(t) and plastic row visits A(t) u F(t)
//   k_stdp     (a3) lazy + event-driven STDP over 64-bit histories (Fig. 2c)
//   k_deliver  (a4) neuron-domain-sliced delivery with shared-memory atomics (Fig. 3b)
//
// Floating point: every fp32 op is written with an explicit __f*_rn intrinsic so
// that no FMA contraction happens (R19); integer accumulators are
// int32 fixed point with F fraction bits (R18).
#include "common.cuh"
#include "philox.cuh"

namespace snn {

// ------------------------------------------------------------------- (a1)
// One thread per neuron; warps cover 32 consecutive ids = one ring word.
// P:36 "Update neurons, note which ones fire"; P:192 history push.
__global__ void __launch_bounds__(256)
k_neuron(NetDev net, StateDev st, uint32_t lo, uint32_t hi) {
    const int64_t t = st.ctr->t;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st.ctr->nA = 0;
        st.ctr->nV = 0;
    }
    const uint32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x;
    bool fired = false;
    if (i < hi) {
        const PopDev &p = net.pop[find_pop(net, i)];
        if (p.kind == POP_POISSON) {
            const u32x4 r = philox4x32_10(i, (uint32_t)t, 2u, 0u, net.key0, net.key1);
            fired = (uint64_t)r.x < p.thr;
        } else if (p.kind == POP_LIF_DELTA) {
            // App. B: I = in 2^-F; in = 0; if ref>0 {ref--} else {V = V k_m; V = V + I}
            const int32_t q = st.in_e[i];
            const float I = __fmul_rn(__int2float_rn(q), net.inv_scale);
            if (q != 0) st.in_e[i] = 0;
            int32_t ref = st.ref[i];
            float V = st.V[i];
            if (ref > 0) {
                ref--;
            } else {
                V = __fadd_rn(__fmul_rn(V, p.k_m), I);
            }
            if (ref == 0 && V >= p.v_th) {
                fired = true;
                V = p.v_reset;
                ref = p.n_ref;
            }
            st.V[i] = V;
            st.ref[i] = ref;
        } else {  // POP_LIF_CUBA
            const int32_t qe = st.in_e[i], qi = st.in_i[i];
            float ge = __fadd_rn(st.ge[i], __fmul_rn(__int2float_rn(qe), net.inv_scale));
            float gi = __fadd_rn(st.gi[i], __fmul_rn(__int2float_rn(qi), net.inv_scale));
            if (qe != 0) st.in_e[i] = 0;
            if (qi != 0) st.in_i[i] = 0;
            int32_t ref = st.ref[i];
            float V = st.V[i];
            if (ref > 0) {
                ref--;
            } else {
                const float t1 = __fsub_rn(p.v_rest, V);
                const float t2 = __fadd_rn(t1, ge);
                const float t3 = __fadd_rn(t2, gi);
                V = __fadd_rn(V, __fmul_rn(p.a_m, t3));
            }
            ge = __fmul_rn(ge, p.d_e);
            gi = __fmul_rn(gi, p.d_i);
            if (ref == 0 && V >= p.v_th) {
                fired = true;
                V = p.v_reset;
                ref = p.n_ref;
            }
            st.V[i] = V;
            st.ref[i] = ref;
            st.ge[i] = ge;
            st.gi[i] = gi;
        }
        if (p.flags & PF_POST_PLASTIC) {
            st.hist[i] = (st.hist[i] << 1) | (uint64_t)fired;
            // x_post = x_post * d- (+1 on a post spike): the per-neuron trace of R7
            const float x = __fmul_rn(st.xpost[i], p.d_minus);
            st.xpost[i] = fired ? __fadd_rn(x, 1.0f) : x;
        }
        if (fired) st.nspk[i] += 1u;
    }
    const uint32_t word = __ballot_sync(0xffffffffu, fired);
    if ((threadIdx.x & 31) == 0 && i < hi)
        st.ring[(size_t)(t & (kRingSlots - 1)) * net.nwords + (i >> 5)] = word;
}

// ------------------------------------------------------------------- (a2)
// Blocks [0, nbA): arrivals A(t) = neurons whose spike of step t-D arrives now
// (hist[delay]).  Blocks [nbA, ...): plastic source rows, visited when
// they are arrivals or their age reached H (forced flush, R3).
__global__ void __launch_bounds__(256)
k_worklist(NetDev net, StateDev st, uint32_t nbA, uint32_t pl_lo, uint32_t pl_hi) {
    const int64_t t = st.ctr->t;
    const uint32_t lane = threadIdx.x & 31;
    const bool have_slot = t >= (int64_t)net.D;
    const uint32_t *slot = st.ring + (size_t)((t - net.D) & (kRingSlots - 1)) * net.nwords;
    if (blockIdx.x < nbA) {
        const uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x;
        uint32_t bits = (have_slot && wi < net.nwords) ? slot[wi] : 0u;
        const uint32_t cnt = __popc(bits);
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t base = 0;
        if (lane == 31 && total) base = atomicAdd(&st.ctr->nA, total);
        base = __shfl_sync(0xffffffffu, base, 31);
        uint32_t pos = base + incl - cnt;
        unsigned long long ev = 0;
        while (bits) {
            const uint32_t b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t id = (wi << 5) + b;
            st.arr_list[pos++] = id;
            ev += (unsigned long long)(st.row_ptr[id + 1] - st.row_ptr[id]);
        }
        ev = __reduce_add_sync(0xffffffffu, (uint32_t)ev);   // per-warp events < 2^32
        if (lane == 0 && total) {
            atomicAdd(&st.ctr->metric[0], ev);
            atomicAdd(&st.ctr->metric[1], (unsigned long long)total);
        }
    } else {
        const uint32_t i = pl_lo + (blockIdx.x - nbA) * blockDim.x + threadIdx.x;
        bool visit = false;
        uint32_t tag = 0;
        if (i < pl_hi && (net.pop[find_pop(net, i)].flags & PF_PRE_PLASTIC)) {
            const bool arr = have_slot && ((slot[i >> 5] >> (i & 31)) & 1u);
            const int64_t age = t - (int64_t)st.tlu[i];
            visit = arr || age >= kHistBits;
            tag = i | (arr ? kArrBit : 0u);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, visit);
        if (m) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&st.ctr->nV, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (visit) st.visit_list[base + __popc(m & ((1u << lane) - 1u))] = tag;
        }
    }
}

// ------------------------------------------------------------------- (a3)
// Lazy + event-driven STDP (Fig. 2c; Sec. III-A), with the
// additive trace rule of R7 in its closed form.  One CTA per visited plastic row
// (grid-stride over the visit list).  For each plastic synapse (i -> j):
//   m = hist[j] & window(age)        post spikes in steps (tlu, t]   (R2)
//   for set bits p, oldest first (63 - clz):
//       w = min(w + A+ * (x_pre * D+[age - p]), w_max)
//   if the row's spike arrives now:  w = max(w - A- * x_post[j], 0)
// then once per row: x_pre = x_pre * D+[age] + arr; tlu = t.
// Weights are touched only where the window holds a post spike (with x_pre > 0)
// or on an arrival -- a flush of a row with an empty window reads only idx.
template <bool kFixedT>
__global__ void __launch_bounds__(256)
k_stdp(NetDev net, StateDev st, int64_t t_fixed, uint32_t n_fixed) {
    const int64_t t = kFixedT ? t_fixed : st.ctr->t;
    const uint32_t nV = kFixedT ? n_fixed : st.ctr->nV;
    unsigned long long n_w = 0;
    for (uint32_t r = blockIdx.x; r < nV; r += gridDim.x) {
        const uint32_t tag = st.visit_list[r];
        const uint32_t i = tag & ~kArrBit;
        const bool arr = (tag & kArrBit) != 0;
        const PopDev &sp = net.pop[find_pop(net, i)];
        const StdpDev &sd = net.stdp[sp.stdp];
        const int age = (int)(t - (int64_t)st.tlu[i]);     // 1..64
        const float xp = st.xpre[i];
        const uint2 sg = st.seg[i];
        const int64_t base = st.row_ptr[i];
        const uint64_t wmask = age >= 64 ? ~0ull : ((1ull << age) - 1ull);
        const bool pot = xp != 0.0f;          // potentiation adds A+ x_pre d^n = 0 otherwise
        const int64_t c0 = base + sg.x, c1 = base + sg.y;
        for (int64_t c = (c0 & ~3ll) + 4 * (int64_t)threadIdx.x; c < c1; c += 4 * (int64_t)blockDim.x) {
            const uint4 j4 = *reinterpret_cast<const uint4 *>(st.idx + c);
            const uint32_t jj[4] = {j4.x, j4.y, j4.z, j4.w};
            uint64_t m[4];
            bool need[4];
            bool any = false;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const bool in = (c + e >= c0) && (c + e < c1);
                m[e] = in ? (st.hist[jj[e]] & wmask) : 0ull;
                need[e] = in && ((pot && m[e] != 0ull) || arr);
                any |= need[e];
            }
            if (!any) continue;
            const bool full = (c >= c0) && (c + 3 < c1);
            float wv[4];
            if (full) {
                const float4 w4 = *reinterpret_cast<const float4 *>(st.w + c);
                wv[0] = w4.x; wv[1] = w4.y; wv[2] = w4.z; wv[3] = w4.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; e++) wv[e] = need[e] ? st.w[c + e] : 0.0f;
            }
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (!need[e]) continue;
                float w = wv[e];
                uint64_t mm = pot ? m[e] : 0ull;
                while (mm) {
                    const int p = 63 - __clzll((long long)mm);
                    mm &= ~(1ull << p);
                    const float x = __fmul_rn(xp, sd.dplus[age - p]);
                    const float nw = __fadd_rn(w, __fmul_rn(sd.a_plus, x));
                    w = nw < sd.w_max ? nw : sd.w_max;
                }
                if (arr) {
                    const float nw = __fsub_rn(w, __fmul_rn(sd.a_minus, st.xpost[jj[e]]));
                    w = nw > 0.0f ? nw : 0.0f;
                }
                wv[e] = w;
                n_w++;
            }
            if (full) {
                *reinterpret_cast<float4 *>(st.w + c) = make_float4(wv[0], wv[1], wv[2], wv[3]);
            } else {
#pragma unroll
                for (int e = 0; e < 4; e++)
                    if (need[e]) st.w[c + e] = wv[e];
            }
        }
        __syncthreads();   // every thread has read xpre/tlu/seg of row i
        if (threadIdx.x == 0) {
            atomicAdd(&st.ctr->metric[3], (unsigned long long)(sg.y - sg.x));
            if (!arr) atomicAdd(&st.ctr->metric[5], 1ull);
            const float x = __fmul_rn(xp, sd.dplus[age]);
            st.xpre[i] = arr ? __fadd_rn(x, 1.0f) : x;
            st.tlu[i] = (int32_t)t;
        }
    }
    n_w = __reduce_add_sync(0xffffffffu, (uint32_t)n_w);
    if ((threadIdx.x & 31) == 0 && n_w) atomicAdd(&st.ctr->metric[4], n_w);
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&st.ctr->metric[2], (unsigned long long)nV);
}

// Read-out flush list (R11): every plastic row not updated at t_last.
__global__ void k_flush_list(NetDev net, StateDev st, int64_t t_last, uint32_t pl_lo, uint32_t pl_hi,
                             uint32_t *count) {
    const uint32_t i = pl_lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pl_hi) return;
    if ((net.pop[find_pop(net, i)].flags & PF_PRE_PLASTIC) && (int64_t)st.tlu[i] < t_last) {
        const uint32_t pos = atomicAdd(count, 1u);
        st.visit_list[pos] = i;
    }
}

// ------------------------------------------------------------------- (a4)
// Shared-memory sliced delivery (Fig. 3b, Sec. III-B).
// CTA (slice k, split s): zero acc[nrcpt][C] in smem; every warp takes 32
// arrivals at a time, reads their (row_ptr, pivot pair) for slice k, flattens
// the 32 segments [piv[a][k], piv[a][k+1]) into one index space and walks it
// 32 lanes wide, adding q(w) = RNE(w 2^F) with native int32 shared atomics
// (ATOMS.ADD); finally one coalesced pass adds the non-zero accumulators to the
// global input arrays (RED.ADD.S32; several CTAs may share a slice).
// The last CTA to finish advances the step counter.
constexpr int kDeliverThreads = 512;

__global__ void __launch_bounds__(kDeliverThreads)
k_deliver(NetDev net, StateDev st) {
    extern __shared__ int32_t acc[];
    const uint32_t k = blockIdx.x;
    const uint32_t nsplit = gridDim.y, split = blockIdx.y;
    const uint32_t C = net.C;
    const uint32_t slo = net.tgt_lo + (k << net.log2C);
    const uint32_t shi = min(slo + C, net.tgt_hi);
    const uint32_t width = shi > slo ? shi - slo : 0;
    for (uint32_t x = threadIdx.x; x < net.nrcpt * C; x += blockDim.x) acc[x] = 0;
    __syncthreads();

    const uint32_t nA = st.ctr->nA;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    const uint32_t P = net.nslices + 1;
    const float scale = net.scale;
    unsigned long long nseg = 0;
    const uint32_t nA_eff = k < net.nslices ? nA : 0u;
    for (uint32_t b = (split * nwarps + warp) * 32; b < nA_eff; b += nsplit * nwarps * 32) {
        uint32_t len = 0;
        int64_t start = 0;
        int sp = 0;
        if (b + lane < nA) {
            const uint32_t a = st.arr_list[b + lane];
            const uint32_t *pv = st.piv + (size_t)a * P + k;
            const uint32_t p0 = pv[0], p1 = pv[1];
            len = p1 - p0;
            if (len) {
                start = st.row_ptr[a] + p0;
                sp = find_pop(net, a);
            }
        }
        nseg += len != 0;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - len;
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t e = e0 + lane;
            // owner = number of lanes whose segment ends at or before e
            uint32_t own = 0;
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, own + s - 1);
                if (v <= e) own += s;
            }
            own = min(own, 31u);
            const int64_t ostart = __shfl_sync(0xffffffffu, start, own);
            const uint32_t oexcl = __shfl_sync(0xffffffffu, excl, own);
            const int osp = __shfl_sync(0xffffffffu, sp, own);
            if (e < total) {
                const int64_t c = ostart + (e - oexcl);
                const uint32_t j = __ldg(st.idx + c);
                const float wv = st.w[c];
                int r = net.pop[osp].rcpt_uniform;
                if (r < 0) r = net.rcpt[osp][find_pop(net, j)];
                const int32_t qv = __float2int_rn(__fmul_rn(wv, scale));
                atomicAdd(&acc[r * C + (j - slo)], qv);
            }
        }
    }
    __syncthreads();
    for (uint32_t r = 0; r < net.nrcpt; r++) {
        int32_t *dst = r == 0 ? st.in_e : st.in_i;
        for (uint32_t x = threadIdx.x; x < width; x += blockDim.x) {
            const int32_t v = acc[r * C + x];
            if (v != 0) atomicAdd(dst + slo + x, v);
        }
    }
    nseg = __reduce_add_sync(0xffffffffu, (uint32_t)nseg);
    if (lane == 0 && nseg) atomicAdd(&st.ctr->metric[6], nseg);
    // step completion ticket
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nblk = gridDim.x * gridDim.y;
        const uint32_t tk = atomicAdd(&st.ctr->ticket, 1u);
        if (tk == nblk - 1) {
            st.ctr->ticket = 0;
            st.ctr->t = st.ctr->t + 1;
        }
    }
}

// History reconstruction from the bitmask ring (read-out of SNN_FIELD_HIST):
// bit s of hist[i] = spike of i at step t_last - s.
__global__ void k_hist_from_ring(NetDev net, const uint32_t *ring, int64_t t_last, uint64_t *out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= net.N) return;
    uint64_t h = 0;
    for (int s = kHistBits - 1; s >= 0; s--) {
        h <<= 1;
        const int64_t u = t_last - s;
        if (u >= 0) h |= (ring[(size_t)(u & (kRingSlots - 1)) * net.nwords + (i >> 5)] >> (i & 31)) & 1u;
    }
    out[i] = h;
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_neuron(const NetDev &net, const StateDev &st, uint32_t lo, uint32_t hi, cudaStream_t s) {
    const uint32_t n = hi - lo;
    k_neuron<<<(n + 255) / 256, 256, 0, s>>>(net, st, lo, hi);
    return cudaGetLastError();
}

cudaError_t launch_worklist(const NetDev &net, const StateDev &st, uint32_t pl_lo, uint32_t pl_hi,
                            cudaStream_t s) {
    const uint32_t nbA = (net.nwords + 255) / 256;
    const uint32_t nbV = (pl_hi - pl_lo + 255) / 256;
    k_worklist<<<nbA + nbV, 256, 0, s>>>(net, st, nbA, pl_lo, pl_hi);
    return cudaGetLastError();
}

cudaError_t launch_stdp(const NetDev &net, const StateDev &st, uint32_t grid, cudaStream_t s) {
    k_stdp<false><<<grid, 256, 0, s>>>(net, st, 0, 0);
    return cudaGetLastError();
}

cudaError_t launch_stdp_fixed(const NetDev &net, const StateDev &st, int64_t t, uint32_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_stdp<true><<<min(n, 148u * 16u), 256, 0, s>>>(net, st, t, n);
    return cudaGetLastError();
}

cudaError_t launch_flush_list(const NetDev &net, const StateDev &st, int64_t t_last, uint32_t pl_lo,
                              uint32_t pl_hi, uint32_t *count, cudaStream_t s) {
    if (pl_hi <= pl_lo) return cudaSuccess;
    k_flush_list<<<(pl_hi - pl_lo + 255) / 256, 256, 0, s>>>(net, st, t_last, pl_lo, pl_hi, count);
    return cudaGetLastError();
}

size_t deliver_smem_bytes(const NetDev &net) { return (size_t)net.nrcpt * net.C * sizeof(int32_t); }

cudaError_t deliver_configure(const NetDev &net) {
    return cudaFuncSetAttribute(k_deliver, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)deliver_smem_bytes(net));
}

cudaError_t launch_deliver(const NetDev &net, const StateDev &st, uint32_t splits, cudaStream_t s) {
    dim3 grid(net.nslices > 0 ? net.nslices : 1, splits);
    k_deliver<<<grid, kDeliverThreads, deliver_smem_bytes(net), s>>>(net, st);
    return cudaGetLastError();
}

cudaError_t launch_hist_from_ring(const NetDev &net, const uint32_t *ring, int64_t t_last, uint64_t *out,
                                  cudaStream_t s) {
    k_hist_from_ring<<<(net.N + 255) / 256, 256, 0, s>>>(net, ring, t_last, out);
    return cudaGetLastError();
}

}  // namespace snn
