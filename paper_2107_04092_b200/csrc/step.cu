// step.cu -- the per-step hot path, two kernels per step:
//
//   k_front  (a1)+(a2)  neuron / Poisson update, firing bits -> bitmask ring,
//                       64-bit history push, and the step's work lists:
//                       plastic row visits A(t) u F(t) (arrivals + forced
//                       flushes, R3) and static arrivals, compacted per CTA
//                       into that CTA's own list region (no global atomics);
//                       also finalises the per-row STDP state (x_pre, tlu) of
//                       rows visited at t-1.
//   k_slice  (a3)+(a4)  one CTA group per neuron slice (Fig. 3b):
//                       stages the slice's 64-bit histories and post traces in
//                       shared memory, runs lazy + event-driven STDP (Fig. 2c,
//                       P:233-246) on every visited row's segment in the slice
//                       and delivers every arriving row's segment into int32
//                       shared-memory accumulators (native ATOMS.ADD), then adds
//                       them to the global input arrays in one coalesced pass.
//
// Floating point: every fp32 op is an explicit __f*_rn intrinsic, so there is no
// FMA contraction (R19); accumulators are int32 fixed point (R18).
#include "common.cuh"
#include "philox.cuh"

namespace snn {

__device__ __forceinline__ uint32_t ring_bit(const uint32_t *ring, uint32_t nwords, int64_t step, uint32_t i) {
    return (ring[(size_t)(step & (kRingSlots - 1)) * nwords + (i >> 5)] >> (i & 31)) & 1u;
}

// x_pre after a row update: x_pre * D+[age] (+1 on a pre spike), R7 closed form.
__device__ __forceinline__ float xpre_after(const StdpDev &sd, float xp, int age, bool arr) {
    const float x = __fmul_rn(xp, sd.dplus[age]);
    return arr ? __fadd_rn(x, 1.0f) : x;
}

// Block-wide compaction of up to two predicates into this CTA's list regions.
// Returns each thread's slot for (a, b); writes the per-CTA counts to *counts.
struct Compact2 {
    uint32_t wa[kFrontThreads / 32], wb[kFrontThreads / 32];
};
__device__ __forceinline__ void compact2(Compact2 &sm, bool a, bool b, uint32_t &slot_a, uint32_t &slot_b,
                                         uint32_t &tot_a, uint32_t &tot_b) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ba = __ballot_sync(0xffffffffu, a), bb = __ballot_sync(0xffffffffu, b);
    if (lane == 0) {
        sm.wa[warp] = __popc(ba);
        sm.wb[warp] = __popc(bb);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint32_t va = lane < nw ? sm.wa[lane] : 0u, vb = lane < nw ? sm.wb[lane] : 0u;
        uint32_t ia = va, ib = vb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o);
            if (lane >= o) {
                ia += xa;
                ib += xb;
            }
        }
        if (lane < nw) {
            sm.wa[lane] = ia - va;
            sm.wb[lane] = ib - vb;
        }
        tot_a = __shfl_sync(0xffffffffu, ia, 31);
        tot_b = __shfl_sync(0xffffffffu, ib, 31);
    }
    __syncthreads();
    const uint32_t lm = (1u << lane) - 1u;
    slot_a = sm.wa[warp] + __popc(ba & lm);
    slot_b = sm.wb[warp] + __popc(bb & lm);
}

// ------------------------------------------------------------------ k_front
// One thread per neuron i (it also owns source row i); warps cover 32
// consecutive ids = one ring word.  P:36 "Update neurons, note which ones fire".
__global__ void __launch_bounds__(kFrontThreads)
k_front(NetDev net, StateDev st) {
    __shared__ Compact2 cs;
    const int64_t t = st.ctr->t;
    const uint32_t par = (uint32_t)(t & 1);
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    const bool valid = i < net.N;
    const int pi = valid ? find_pop(net, i) : 0;
    const PopDev &p = net.pop[pi];
    bool fired = false;
    // ---- (1) neuron dynamics (App. B op order)
    if (valid) {
        if (p.kind == POP_POISSON) {
            const u32x4 r = philox4x32_10(i, (uint32_t)t, 2u, 0u, net.key0, net.key1);
            fired = (uint64_t)r.x < p.thr;
        } else if (p.kind == POP_LIF_DELTA) {
            const int32_t q = st.in_e[i];
            const float I = __fmul_rn(__int2float_rn(q), net.inv_scale);
            if (q != 0) st.in_e[i] = 0;
            int32_t ref = st.ref[i];
            float V = st.V[i];
            const float V0 = V;
            const int32_t ref0 = ref;
            if (ref > 0) ref--;
            else V = __fadd_rn(__fmul_rn(V, p.k_m), I);
            if (ref == 0 && V >= p.v_th) {
                fired = true;
                V = p.v_reset;
                ref = p.n_ref;
            }
            if (__float_as_uint(V) != __float_as_uint(V0)) st.V[i] = V;
            if (ref != ref0) st.ref[i] = ref;
        } else {  // POP_LIF_CUBA
            const int32_t qe = st.in_e[i], qi = st.in_i[i];
            float ge = __fadd_rn(st.ge[i], __fmul_rn(__int2float_rn(qe), net.inv_scale));
            float gi = __fadd_rn(st.gi[i], __fmul_rn(__int2float_rn(qi), net.inv_scale));
            if (qe != 0) st.in_e[i] = 0;
            if (qi != 0) st.in_i[i] = 0;
            int32_t ref = st.ref[i];
            const int32_t ref0 = ref;
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
            if (ref != ref0) st.ref[i] = ref;
            st.ge[i] = ge;
            st.gi[i] = gi;
        }
        if (p.flags & PF_POST_PLASTIC) {
            st.hist[i] = (st.hist[i] << 1) | (uint64_t)fired;
            const float x = __fmul_rn(st.xpost[i], p.d_minus);   // x_post decay (+1 on a post spike), R7
            st.xpost[i] = fired ? __fadd_rn(x, 1.0f) : x;
        }
        if (fired) st.nspk[i] += 1u;
    }
    const uint32_t fword = __ballot_sync(0xffffffffu, fired);
    if (lane == 0 && valid) st.ring[(size_t)(t & (kRingSlots - 1)) * net.nwords + (i >> 5)] = fword;

    // ---- (2) arrival of row i at step t: its spike of step t - D (hist[delay])
    bool arr = false;
    if (valid) {
        if (net.D == 0) arr = fired;
        else if (t >= (int64_t)net.D) arr = ring_bit(st.ring, net.nwords, t - net.D, i);
    }
    const bool plastic_row = valid && (p.flags & PF_PRE_PLASTIC);
    bool visit = false;
    RowDesc d;
    if (plastic_row) {
        const StdpDev &sd = net.stdp[p.stdp];
        int32_t tl = st.tlu[i];
        float xp = st.xpre[i];
        // finalise a visit of step t-1 (its synapses were updated by k_slice(t-1))
        if (t >= 1 && ((st.vmask[par ^ 1u][i >> 5] >> (i & 31)) & 1u)) {
            const bool arr_prev = (t - 1 >= (int64_t)net.D) && ring_bit(st.ring, net.nwords, t - 1 - net.D, i);
            xp = xpre_after(sd, xp, (int)(t - 1 - tl), arr_prev);
            tl = (int32_t)(t - 1);
            st.xpre[i] = xp;
            st.tlu[i] = tl;
        }
        const int age = (int)(t - tl);
        visit = arr || age >= kHistBits;    // forced flush at maximum age (R3)
        if (visit) {
            const uint2 sg = st.seg[i];
            d.start = st.row_ptr[i];
            d.row = i;
            d.meta = (uint32_t)age | (arr ? kMetaArr : 0u) | kMetaPlastic | ((uint32_t)(p.rcpt_uniform & 3) << 8) |
                     ((uint32_t)p.stdp << 12);
            d.xp = xp;
            d.s0 = sg.x;
            d.s1 = sg.y;
            d.pad = 0;
        }
    }
    const uint32_t vword = __ballot_sync(0xffffffffu, visit);
    if (net.nstdp && lane == 0 && valid) st.vmask[par][i >> 5] = vword;
    const bool sarr = arr && !plastic_row;          // static arrivals (rows without STDP)
    uint32_t sv, sa, nv, na;
    compact2(cs, visit, sarr, sv, sa, nv, na);
    const size_t region = (size_t)blockIdx.x * kFrontThreads;
    if (visit) st.vdesc[par][region + sv] = d;
    if (sarr) {
        RowDesc a;
        a.start = st.row_ptr[i];
        a.row = i;
        a.meta = kMetaArr | ((uint32_t)(p.rcpt_uniform & 3) << 8);
        a.xp = 0.0f;
        a.s0 = a.s1 = 0;
        a.pad = 0;
        st.adesc[par][region + sa] = a;
    }
    // per-CTA counts (arrivals and flushes for the metrics)
    const uint32_t na_all = __syncthreads_count(arr);
    const uint32_t nflush = __syncthreads_count(visit && !arr);
    if (threadIdx.x == 0) st.cnt[par][blockIdx.x] = make_uint4(nv, na, na_all, nflush);
}

// ------------------------------------------------------------------ k_slice
constexpr int kSliceThreads = 512;
constexpr int kSliceWarps = kSliceThreads / 32;
constexpr int kMaxPieces = 512;     // piece table entries per round

// Map a flattened row index r (over the per-CTA regions) to its descriptor.
__device__ __forceinline__ RowDesc fetch_row(const uint32_t *pre_v, const uint32_t *pre_a, uint32_t nblk, uint32_t nV,
                                             const RowDesc *V, const RowDesc *A, uint32_t r) {
    const uint32_t *pre = r < nV ? pre_v : pre_a;
    const uint32_t x = r < nV ? r : r - nV;
    uint32_t lo = 0, hi = nblk;          // largest b with pre[b] <= x
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (pre[mid] <= x) lo = mid; else hi = mid;
    }
    const size_t idx = (size_t)lo * kFrontThreads + (x - pre[lo]);
    return r < nV ? V[idx] : A[idx];
}

// One plastic synapse update (Fig. 2c with the closed-form skip-ahead of R7):
// potentiation for every post spike in the window, oldest first (P:284
// "__clz"), then the depression of an arriving pre spike.
__device__ __forceinline__ float stdp_update(const StdpDev &sd, float w, uint64_t m, float xp, int age, bool arr,
                                             float xpost) {
    while (m) {
        const int pb = 63 - __clzll((long long)m);
        m &= ~(1ull << pb);
        const float x = __fmul_rn(xp, sd.dplus[age - pb]);
        const float nw = __fadd_rn(w, __fmul_rn(sd.a_plus, x));
        w = nw < sd.w_max ? nw : sd.w_max;
    }
    if (arr) {
        const float nw = __fsub_rn(w, __fmul_rn(sd.a_minus, xpost));
        w = nw > 0.0f ? nw : 0.0f;
    }
    return w;
}

// ---- TMA bulk copy + mbarrier helpers (sm_90+ async proxy; SASS UBLKCP / SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}

// A piece = one (row, slice) segment (or a part of a long one): the 16-byte
// aligned span [cb, cb + 4*n4) of the CSR arrays staged by one bulk copy each
// for the target ids and the weights.
struct __align__(16) Piece {
    int64_t cb;          // aligned CSR offset of the span
    uint32_t lohi;       // valid elements [lo, hi) relative to cb (16 + 16 bit)
    uint32_t prange;     // plastic elements [p0, p1) relative to cb (16 + 16 bit)
    uint32_t meta;       // RowDesc meta; bits 16-19 = source population
    float xp;
    uint32_t n4;         // 4-element chunks staged
    uint32_t pad;
};

// One CTA = (slice k, split s).  Round structure:
//   1. all threads: each takes one of this CTA's rows (per-CTA list regions,
//      k_front) -> descriptor + pivot pair (Fig. 1 / P:348) -> the pieces of its
//      segment, block-compacted into the shared piece table;
//   2. every warp runs its own TMA pipeline over pieces warp, warp+16, ...:
//      kStages bulk copies in flight, each piece processed from shared memory
//      32 lanes wide (STDP update, changed weights stored back, delivery by
//      int32 shared atomics).
template <int kStages>
__global__ void __launch_bounds__(kSliceThreads, 2)
k_slice(NetDev net, StateDev st, int64_t t_fixed, uint32_t slot_elems) {
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t C = net.C;
    const uint32_t nblk = st.nblk;
    // t_fixed < 0: step t = ctr->t with the lists of parity t & 1;
    // t_fixed >= 0: read-out flush at t_fixed, no delivery.
    const bool deliver = t_fixed < 0;
    const int64_t t = deliver ? st.ctr->t : t_fixed;
    const uint32_t par = (uint32_t)(t & 1);
    const RowDesc *Vl = deliver ? st.vdesc[par] : st.rdesc;
    const RowDesc *Al = st.adesc[par];
    const uint4 *cnt = deliver ? st.cnt[par] : st.rcnt;

    // shared memory carve-up (all offsets 16-byte multiples)
    const uint32_t npre = (nblk + 1 + 3) & ~3u;
    unsigned char *p = smem;
    uint64_t *bars = reinterpret_cast<uint64_t *>(p);            p += 16 * kSliceWarps * kStages / 2 * 1;  // [warps][stages]
    Piece *pieces = reinterpret_cast<Piece *>(p);                p += sizeof(Piece) * kMaxPieces;
    uint32_t *slots = reinterpret_cast<uint32_t *>(p);           p += 8ull * slot_elems * kSliceWarps * kStages;
    int32_t *acc = reinterpret_cast<int32_t *>(p);               p += 4ull * net.nrcpt * C;
    uint64_t *hist_s = reinterpret_cast<uint64_t *>(p);          p += net.nstdp ? 8ull * C : 0;
    float *xpost_s = reinterpret_cast<float *>(p);               p += net.nstdp ? 4ull * C : 0;
    uint32_t *pre_v = reinterpret_cast<uint32_t *>(p);           p += 4ull * npre;
    uint32_t *pre_a = reinterpret_cast<uint32_t *>(p);          p += 4ull * npre;
    float *dplus_s = reinterpret_cast<float *>(p);              // [nstdp][65]

    const uint32_t k = blockIdx.x;
    const uint32_t nsplit = gridDim.y, split = blockIdx.y;
    const uint32_t slo = net.tgt_lo + (k << net.log2C);
    const uint32_t shi = min(slo + C, net.tgt_hi);
    const uint32_t width = shi > slo ? shi - slo : 0u;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    __shared__ uint32_t wsum[2][kSliceWarps];
    __shared__ uint32_t s_round[2];
    // ---- barriers
    if (threadIdx.x < kSliceWarps * kStages) mbar_init(&bars[threadIdx.x], 1);
    // ---- per-CTA list regions -> exclusive prefix sums (visits, static arrivals)
    {
        const uint32_t per = (nblk + kSliceThreads - 1) / kSliceThreads;
        const uint32_t b0 = threadIdx.x * per;
        uint32_t sv = 0, sa = 0;
        for (uint32_t b = b0; b < min(b0 + per, nblk); b++) {
            const uint4 c4 = cnt[b];
            sv += c4.x;
            sa += deliver ? c4.y : 0u;
        }
        uint32_t iv = sv, ia = sa;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xv = __shfl_up_sync(0xffffffffu, iv, o), xa = __shfl_up_sync(0xffffffffu, ia, o);
            if (lane >= o) {
                iv += xv;
                ia += xa;
            }
        }
        if (lane == 31) {
            wsum[0][warp] = iv;
            wsum[1][warp] = ia;
        }
        __syncthreads();
        uint32_t ov = 0, oa = 0;
        for (uint32_t w2 = 0; w2 < warp; w2++) {
            ov += wsum[0][w2];
            oa += wsum[1][w2];
        }
        uint32_t rv = ov + iv - sv, ra = oa + ia - sa;
        for (uint32_t b = b0; b < min(b0 + per, nblk); b++) {
            pre_v[b] = rv;
            pre_a[b] = ra;
            const uint4 c4 = cnt[b];
            rv += c4.x;
            ra += deliver ? c4.y : 0u;
        }
        if (threadIdx.x == kSliceThreads - 1) {
            pre_v[nblk] = rv;
            pre_a[nblk] = ra;
        }
    }
    for (uint32_t x = threadIdx.x; x < net.nstdp * (kHistBits + 1); x += blockDim.x)
        dplus_s[x] = net.stdp[x / (kHistBits + 1)].dplus[x % (kHistBits + 1)];
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // ---- stage: zero accumulators, load the slice's histories / post traces
    if (deliver)
        for (uint32_t x = threadIdx.x; x < net.nrcpt * C; x += blockDim.x) acc[x] = 0;
    bool post_plastic = false;
    for (uint32_t q = 0; q < net.npop; q++) {
        const PopDev &pp = net.pop[q];
        if ((pp.flags & PF_POST_PLASTIC) && pp.base < shi && pp.base + pp.n > slo) post_plastic = true;
    }
    __syncthreads();
    const uint32_t nV = pre_v[nblk];
    const uint32_t nA = pre_a[nblk];
    if (post_plastic && nV > 0) {
        for (uint32_t x = threadIdx.x; x < width; x += blockDim.x) {
            hist_s[x] = st.hist[slo + x];
            xpost_s[x] = st.xpost[slo + x];
        }
    }
    // (the first __syncthreads of the round loop publishes the staging)

    const uint32_t P = net.nslices + 1;
    const float scale = net.scale;
    uint32_t n_syn = 0, n_w = 0, n_ev = 0, n_seg = 0, n_el = 0;
    const uint32_t total = nV + nA;
    const uint32_t r_begin = (uint32_t)(((uint64_t)total * split) / nsplit);
    const uint32_t r_end = (uint32_t)(((uint64_t)total * (split + 1)) / nsplit);
    uint64_t *mybars = bars + warp * kStages;
    uint32_t *myslots = slots + (size_t)warp * kStages * 2 * slot_elems;
    uint32_t uses = 0;     // pieces this warp has consumed so far (barrier phase tracking)
    for (uint32_t r0 = r_begin; r0 < r_end;) {
        // ---- 1. rows -> pieces
        const uint32_t r = r0 + threadIdx.x;
        uint32_t np = 0, chunks = 0;
        int64_t cb0 = 0;
        uint32_t lo = 0, hi = 0, cp0 = 0, cp1 = 0, meta = 0;
        uint32_t c_syn = 0, c_ev = 0;
        float xp = 0.0f;
        if (r < r_end) {
            const RowDesc d = fetch_row(pre_v, pre_a, nblk, nV, Vl, Al, r);
            const uint32_t *pv = st.piv + (size_t)d.row * P + k;
            const uint32_t q0 = pv[0], q1 = pv[1];
            const bool arr = (d.meta & kMetaArr) != 0;
            uint32_t ps0 = 0, ps1 = 0;
            if (d.meta & kMetaPlastic) {
                ps0 = min(max(d.s0, q0), q1) - q0;
                ps1 = max(min(d.s1, q1), q0) - q0;
            }
            xp = d.xp;
            const bool pot = xp != 0.0f;       // potentiation adds A+ x_pre D+[n] = 0 otherwise
            const bool active = q1 > q0 && (arr || (pot && ps1 > ps0));   // a flush that changes no weight is skipped
            if (active) {
                const int64_t rs = d.start + q0;
                const int64_t cs = rs + (arr ? 0 : ps0);
                const int64_t ce = rs + (arr ? (q1 - q0) : ps1);
                cb0 = cs & ~3ll;
                lo = (uint32_t)(cs - cb0);
                hi = (uint32_t)(ce - cb0);
                cp0 = (uint32_t)(rs + ps0 - cb0 < 0 ? 0 : rs + ps0 - cb0);
                cp1 = (uint32_t)(rs + ps1 - cb0 < 0 ? 0 : rs + ps1 - cb0);
                chunks = (hi + 3) >> 2;
                np = (chunks * 4 + slot_elems - 1) / slot_elems;
                meta = d.meta & 0xffffu;
                if (((d.meta >> 8) & 3u) == 3u) meta |= (uint32_t)find_pop(net, d.row) << 16;
                c_syn = ps1 - ps0;
                c_ev = arr ? (q1 - q0) : 0u;
            }
        }
        // block exclusive scan of np; rows whose pieces overflow the table wait
        uint32_t inc = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += x;
        }
        __syncthreads();                       // previous round fully consumed
        if (lane == 31) wsum[0][warp] = inc;
        __syncthreads();
        uint32_t off = 0;
        for (uint32_t w2 = 0; w2 < warp; w2++) off += wsum[0][w2];
        const uint32_t excl = off + inc - np;
        const bool fits = excl + np <= kMaxPieces;
        if (fits && np) {
            n_syn += c_syn;
            n_ev += c_ev;
            n_el += hi - lo;
            n_seg += 1;
            const uint32_t per = slot_elems / 4;   // chunks per piece
            for (uint32_t q = 0; q < np; q++) {
                Piece pc;
                pc.cb = cb0 + 4ll * per * q;
                const uint32_t base = 4 * per * q;
                const uint32_t n4 = min(per, chunks - per * q);
                const uint32_t vlo = lo > base ? lo - base : 0u;
                const uint32_t vhi = min(hi - base, 4 * n4);
                const uint32_t plo = cp0 > base ? min(cp0 - base, 4 * n4) : 0u;
                const uint32_t phi = cp1 > base ? min(cp1 - base, 4 * n4) : 0u;
                pc.lohi = vlo | (vhi << 16);
                pc.prange = plo | (phi << 16);
                pc.meta = meta;
                pc.xp = xp;
                pc.n4 = n4;
                pc.pad = 0;
                pieces[excl + q] = pc;
            }
        }
        // rows consumed this round: the prefix of rows whose pieces fit
        if (threadIdx.x == 0) s_round[0] = 0;
        const uint32_t fitcount = __syncthreads_count(fits && r < r_end);
        if (fits && np) atomicMax(&s_round[0], excl + np);
        __syncthreads();
        const uint32_t npieces = s_round[0];
        r0 += fitcount;

        // ---- 2. per-warp TMA pipeline over pieces warp, warp + 16, ...
        auto issue = [&](uint32_t pi, uint32_t stage) {
            const Piece &pc = pieces[pi];
            uint32_t *dst = myslots + stage * 2 * slot_elems;
            const uint32_t bytes = pc.n4 * 16u;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&mybars[stage], 2 * bytes);
            bulk_g2s(dst, st.idx + pc.cb, bytes, &mybars[stage]);
            bulk_g2s(dst + slot_elems, st.w + pc.cb, bytes, &mybars[stage]);
        };
        const uint32_t mine = warp < npieces ? (npieces - warp + kSliceWarps - 1) / kSliceWarps : 0u;
        if (lane == 0)
            for (uint32_t q = 0; q < min(mine, (uint32_t)kStages); q++) issue(warp + q * kSliceWarps, (uses + q) % kStages);
        __syncwarp();
        for (uint32_t q = 0; q < mine; q++) {
            const uint32_t pi = warp + q * kSliceWarps;
            const uint32_t stage = (uses + q) % kStages;
            const uint32_t phase = ((uses + q) / kStages) & 1u;
            mbar_wait(&mybars[stage], phase);
            const Piece pc = pieces[pi];
            const uint32_t *jv = myslots + stage * 2 * slot_elems;
            const float *wv = reinterpret_cast<const float *>(jv + slot_elems);
            const uint32_t vlo = pc.lohi & 0xffffu, vhi = pc.lohi >> 16;
            const uint32_t plo = pc.prange & 0xffffu, phi = pc.prange >> 16;
            const int age = (int)(pc.meta & 0x7fu);
            const uint64_t wmask = age >= 64 ? ~0ull : ((1ull << age) - 1ull);
            const float xp = pc.xp;
            const uint32_t si = (pc.meta >> 12) & 0xfu;
            const float a_plus = net.stdp[si].a_plus, a_minus = net.stdp[si].a_minus, w_max = net.stdp[si].w_max;
            const float *dp = dplus_s + si * (kHistBits + 1);
            float *wg = st.w + pc.cb;
            if (!(pc.meta & kMetaArr)) {
                // forced flush (R3): only the plastic span, potentiation only
                for (uint32_t x = vlo + lane; x < vhi; x += 32) {
                    uint64_t m = hist_s[jv[x] - slo] & wmask;       // post spikes in (tlu, t], R2
                    if (m) {
                        float w = wv[x];
                        do {                                         // oldest first, "__clz"
                            const int pb = 63 - __clzll((long long)m);
                            m &= ~(1ull << pb);
                            const float nw = __fadd_rn(w, __fmul_rn(a_plus, __fmul_rn(xp, dp[age - pb])));
                            w = nw < w_max ? nw : w_max;
                        } while (m);
                        wg[x] = w;
                        n_w++;
                    }
                }
            } else {
                // arrival: STDP on the plastic span (posts, then the pre spike at t),
                // then delivery of every element of the segment
                const bool pot = xp != 0.0f;
                const int rc = (int)((pc.meta >> 8) & 3u);
                int32_t *accr = acc + (rc == 3 ? 0 : rc) * C;
                for (uint32_t x = vlo + lane; x < vhi; x += 32) {
                    const uint32_t j = jv[x];
                    const uint32_t jl = j - slo;
                    float w = wv[x];
                    if (x >= plo && x < phi) {
                        uint64_t m = pot ? (hist_s[jl] & wmask) : 0ull;
                        while (m) {
                            const int pb = 63 - __clzll((long long)m);
                            m &= ~(1ull << pb);
                            const float nw = __fadd_rn(w, __fmul_rn(a_plus, __fmul_rn(xp, dp[age - pb])));
                            w = nw < w_max ? nw : w_max;
                        }
                        const float nw = __fsub_rn(w, __fmul_rn(a_minus, xpost_s[jl]));
                        w = nw > 0.0f ? nw : 0.0f;
                        wg[x] = w;
                        n_w++;
                    }
                    if (deliver) {
                        int32_t *a = accr;
                        if (rc == 3) a = acc + net.rcpt[(pc.meta >> 16) & 0xfu][find_pop(net, j)] * C;
                        atomicAdd(a + jl, __float2int_rn(__fmul_rn(w, scale)));
                    }
                }
            }
            __syncwarp();
            const uint32_t nq = q + kStages;
            if (lane == 0 && nq < mine) issue(warp + nq * kSliceWarps, stage);
            __syncwarp();
        }
        uses += mine;
    }
    // ---- write-back (one coalesced pass; several CTAs may share a slice)
    __syncthreads();
    if (deliver) {
        for (uint32_t rr = 0; rr < net.nrcpt; rr++) {
            int32_t *dst = rr == 0 ? st.in_e : st.in_i;
            for (uint32_t x = threadIdx.x; x < width; x += blockDim.x) {
                const int32_t v = acc[rr * C + x];
                if (v != 0) atomicAdd(dst + slo + x, v);
            }
        }
    }
    // ---- counters
    n_syn = __reduce_add_sync(0xffffffffu, n_syn);
    n_w = __reduce_add_sync(0xffffffffu, n_w);
    n_ev = __reduce_add_sync(0xffffffffu, n_ev);
    n_seg = __reduce_add_sync(0xffffffffu, n_seg);
    n_el = __reduce_add_sync(0xffffffffu, n_el);
    if (lane == 0) {
        if (n_el) atomicAdd(&st.ctr->metric[7], (unsigned long long)n_el);
        if (n_syn) atomicAdd(&st.ctr->metric[3], (unsigned long long)n_syn);
        if (n_w) atomicAdd(&st.ctr->metric[4], (unsigned long long)n_w);
        if (n_ev) atomicAdd(&st.ctr->metric[0], (unsigned long long)n_ev);
        if (n_seg) atomicAdd(&st.ctr->metric[6], (unsigned long long)n_seg);
    }
    if (!deliver) return;
    // ---- step completion: the last CTA books the list counts and advances t
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nb = gridDim.x * gridDim.y;
        const uint32_t tk = atomicAdd(&st.ctr->ticket, 1u);
        if (tk == nb - 1) {
            unsigned long long spikes = 0, flushes = 0;
            for (uint32_t b = 0; b < nblk; b++) {
                const uint4 c4 = cnt[b];
                spikes += c4.z;
                flushes += c4.w;
            }
            st.ctr->metric[1] += spikes;
            st.ctr->metric[2] += nV;
            st.ctr->metric[5] += flushes;
            st.ctr->ticket = 0;
            __threadfence();
            st.ctr->t = t + 1;
        }
    }
}

// ----------------------------------------------------------- read-out (R11)
// (1) finalise the visits of step t_last (pending x_pre / tlu updates) and
//     clear their mask; (2) list every plastic row with tlu < t_last.
__global__ void __launch_bounds__(kFrontThreads)
k_readout_prepare(NetDev net, StateDev st, int64_t t_last) {
    __shared__ Compact2 cs;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    const bool valid = i < net.N;
    const PopDev &p = net.pop[valid ? find_pop(net, i) : 0];
    const uint32_t par = (uint32_t)(t_last & 1);
    bool stale = false;
    RowDesc d;
    if (valid && (p.flags & PF_PRE_PLASTIC)) {
        const StdpDev &sd = net.stdp[p.stdp];
        int32_t tl = st.tlu[i];
        float xp = st.xpre[i];
        if ((st.vmask[par][i >> 5] >> (i & 31)) & 1u) {
            const bool arr_prev = (t_last >= (int64_t)net.D) && ring_bit(st.ring, net.nwords, t_last - net.D, i);
            xp = xpre_after(sd, xp, (int)(t_last - tl), arr_prev);
            tl = (int32_t)t_last;
            st.xpre[i] = xp;
            st.tlu[i] = tl;
        }
        if (tl < t_last) {
            stale = true;
            const uint2 sg = st.seg[i];
            d.start = st.row_ptr[i];
            d.row = i;
            d.meta = (uint32_t)(t_last - tl) | kMetaPlastic | ((uint32_t)p.stdp << 12);
            d.xp = xp;
            d.s0 = sg.x;
            d.s1 = sg.y;
            d.pad = 0;
        }
    }
    __syncwarp();
    if (valid && lane == 0 && net.nstdp) st.vmask[par][i >> 5] = 0u;
    uint32_t s0, s1, n0, n1;
    compact2(cs, stale, false, s0, s1, n0, n1);
    if (stale) st.rdesc[(size_t)blockIdx.x * kFrontThreads + s0] = d;
    if (threadIdx.x == 0) st.rcnt[blockIdx.x] = make_uint4(n0, 0u, 0u, 0u);
}

// (3) after k_slice ran the flush on the listed rows: their x_pre / tlu.
__global__ void __launch_bounds__(kFrontThreads)
k_readout_finish(NetDev net, StateDev st, int64_t t_last) {
    if (threadIdx.x >= st.rcnt[blockIdx.x].x) return;
    const RowDesc d = st.rdesc[(size_t)blockIdx.x * kFrontThreads + threadIdx.x];
    const StdpDev &sd = net.stdp[(d.meta >> 12) & 0xfu];
    st.xpre[d.row] = xpre_after(sd, d.xp, (int)(d.meta & 0x7fu), false);
    st.tlu[d.row] = (int32_t)t_last;
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
        if (u >= 0) h |= ring_bit(ring, net.nwords, u, i);
    }
    out[i] = h;
}

// ---------------------------------------------------------------- launchers
uint32_t front_blocks(const NetDev &net) { return (net.N + kFrontThreads - 1) / kFrontThreads; }

cudaError_t launch_front(const NetDev &net, const StateDev &st, cudaStream_t s) {
    k_front<<<front_blocks(net), kFrontThreads, 0, s>>>(net, st);
    return cudaGetLastError();
}

constexpr int kStagesDefault = 4;

size_t slice_smem_bytes(const NetDev &net, uint32_t slot_elems) {
    const size_t nblk = front_blocks(net);
    size_t b = 16ull * kSliceWarps * kStagesDefault / 2;          // mbarriers
    b += sizeof(Piece) * kMaxPieces;
    b += 8ull * slot_elems * kSliceWarps * kStagesDefault;         // staged ids + weights
    b += 4ull * net.nrcpt * net.C;
    if (net.nstdp) b += 12ull * net.C;
    b += 8 * ((nblk + 1 + 3) & ~(size_t)3);
    b += 4ull * 4 * (kHistBits + 1);                               // D+ tables
    return b;
}

cudaError_t slice_configure(const NetDev &net, uint32_t slot_elems) {
    return cudaFuncSetAttribute(k_slice<kStagesDefault>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)slice_smem_bytes(net, slot_elems));
}

static cudaError_t launch_slice(const NetDev &net, const StateDev &st, int64_t t_fixed, uint32_t splits,
                                uint32_t slot_elems, cudaStream_t s) {
    dim3 grid(net.nslices > 0 ? net.nslices : 1, splits);
    k_slice<kStagesDefault><<<grid, kSliceThreads, slice_smem_bytes(net, slot_elems), s>>>(net, st, t_fixed,
                                                                                        slot_elems);
    return cudaGetLastError();
}

cudaError_t launch_step_slice(const NetDev &net, const StateDev &st, uint32_t splits, uint32_t slot_elems,
                              cudaStream_t s) {
    return launch_slice(net, st, -1, splits, slot_elems, s);
}

cudaError_t launch_readout(const NetDev &net, const StateDev &st, int64_t t_last, uint32_t splits,
                           uint32_t slot_elems, cudaStream_t s) {
    k_readout_prepare<<<front_blocks(net), kFrontThreads, 0, s>>>(net, st, t_last);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if ((e = launch_slice(net, st, t_last, splits, slot_elems, s)) != cudaSuccess) return e;
    k_readout_finish<<<front_blocks(net), kFrontThreads, 0, s>>>(net, st, t_last);
    return cudaGetLastError();
}

cudaError_t launch_hist_from_ring(const NetDev &net, const uint32_t *ring, int64_t t_last, uint64_t *out,
                                  cudaStream_t s) {
    k_hist_from_ring<<<(net.N + 255) / 256, 256, 0, s>>>(net, ring, t_last, out);
    return cudaGetLastError();
}

}  // namespace snn
