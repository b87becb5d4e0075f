// step.cu -- the per-step hot path, three kernels per step:
//
//   k_front    (a1)+(a2)  neuron / Poisson update, firing bits -> bitmask ring,
//                         64-bit history push, "fired in the last 64
//                         steps" bitmap of post-synaptic neurons, and the work
//                         lists: plastic row visits A(t) u F(t) (arrivals +
//                         forced flushes, R3) and arrivals A(t), compacted per
//                         CTA and appended to global lists (one atomic per CTA
//                         and list: the lists' order is irrelevant, every row
//                         is processed independently and sums are integer);
//                         also finalises the per-row STDP state (x_pre, tlu) of
//                         rows visited at t-1.
//   k_stdp     (a3)       lazy + event-driven STDP (Fig. 2c) over the
//                         visited rows: one warp streams a row's plastic span
//                         with 16-byte loads; the shared-memory bitmap filters
//                         the targets whose 64-bit history can hold a post spike,
//                         only those histories are gathered.
//   k_deliver  (a4)       neuron-domain-sliced delivery (Fig. 3b, P:313-331,
//                         P:348-355): one CTA per slice accumulates every
//                         arriving spike's segment in int32 shared memory with
//                         native atomics (ATOMS.ADD), then one coalesced
//                         write-back; a warp per 32 spikes, lanes over targets.
//
// Floating point: every fp32 op is an explicit __f*_rn intrinsic, so there is no
// FMA contraction (R19); accumulators are int32 fixed point (R18).
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>

#include "common.cuh"
#include "philox.cuh"

namespace snn {

// Programmatic dependent launch (PDL): the next kernel of the step is launched
// early and parks at pdl_wait() until this grid has completed and flushed;
// pdl_launch() lets the dependent grid start.  No-ops without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t ring_bit(const uint32_t *ring, uint32_t stride, int64_t step, uint32_t i) {
    return (ring[(size_t)(step & (kRingSlots - 1)) * stride + (i >> 5)] >> (i & 31)) & 1u;
}

// x_pre after a row update: x_pre * D+[age] (+1 on a pre spike), R7 closed form.
__device__ __forceinline__ float xpre_after(const StdpDev &sd, float xp, int age, bool arr) {
    const float x = __fmul_rn(xp, sd.dplus[age]);
    return arr ? __fadd_rn(x, 1.0f) : x;
}

// Block-wide compaction of up to three predicates into global lists: the CTA
// books its totals with one atomic per list on lens[0..2] (the lists' lengths)
// and returns each thread's slot for (a, b[, c]) and the CTA totals.
struct Compact2 {
    uint32_t wa[kFrontThreads / 32], wb[kFrontThreads / 32], wc[kFrontThreads / 32];
    uint32_t tot[3], base[3];
};
__device__ __forceinline__ void compact3(Compact2 &sm, uint32_t *len_a, uint32_t *len_b, uint32_t *len_c, bool a,
                                         bool b, bool c, uint32_t &slot_a,
                                         uint32_t &slot_b, uint32_t &slot_c, uint32_t &tot_a, uint32_t &tot_b,
                                         uint32_t &tot_c) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ba = __ballot_sync(0xffffffffu, a), bb = __ballot_sync(0xffffffffu, b),
                   bc = __ballot_sync(0xffffffffu, c);
    if (lane == 0) {
        sm.wa[warp] = __popc(ba);
        sm.wb[warp] = __popc(bb);
        sm.wc[warp] = __popc(bc);
    }
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint32_t va = lane < nw ? sm.wa[lane] : 0u, vb = lane < nw ? sm.wb[lane] : 0u, vc = lane < nw ? sm.wc[lane] : 0u;
        uint32_t ia = va, ib = vb, ic = vc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t xa = __shfl_up_sync(0xffffffffu, ia, o), xb = __shfl_up_sync(0xffffffffu, ib, o),
                           xc = __shfl_up_sync(0xffffffffu, ic, o);
            if (lane >= o) {
                ia += xa;
                ib += xb;
                ic += xc;
            }
        }
        if (lane < nw) {
            sm.wa[lane] = ia - va;
            sm.wb[lane] = ib - vb;
            sm.wc[lane] = ic - vc;
        }
        if (lane == 31) {                     // lanes >= nw add 0: lane 31 holds the totals
            sm.tot[0] = ia;
            sm.tot[1] = ib;
            sm.tot[2] = ic;
            sm.base[0] = ia ? atomicAdd(len_a, ia) : 0u;
            sm.base[1] = ib ? atomicAdd(len_b, ib) : 0u;
            sm.base[2] = ic ? atomicAdd(len_c, ic) : 0u;
        }
    }
    __syncthreads();
    const uint32_t lm = (1u << lane) - 1u;
    slot_a = sm.base[0] + sm.wa[warp] + __popc(ba & lm);
    slot_b = sm.base[1] + sm.wb[warp] + __popc(bb & lm);
    slot_c = sm.base[2] + sm.wc[warp] + __popc(bc & lm);
    tot_a = sm.tot[0];
    tot_b = sm.tot[1];
    tot_c = sm.tot[2];
}

// ------------------------------------------------------------------ k_front
// One thread per neuron i (it also owns source row i); warps cover 32
// consecutive ids = one ring word.  P:36 "Update neurons, note which ones fire".
// One neuron's update at step t (App. B op order, "Update neurons, note
// which ones fire"): Poisson draw or Euler LIF step (consuming the fixed-point
// input delivered at t-1), then for post-synaptic STDP targets the history
// push, the window's spike position / flush factors (buffers t & 3) and
// the x_post trace.  Returns `fired`; `recent`: a spike in the last H steps.
// Shared by k_front and k_deliver's epilogue (the fused step), so both compute
// exactly the same operations.
// The update is split into its loads (neuron_load: every state word the step
// reads, issued together before any store, so a thread waits for one memory
// round trip instead of a chain of them) and its arithmetic + stores
// (neuron_step).
struct NeuronIn {
    int32_t qe, qi, ref;
    float V, ge, gi, xq;
    uint64_t h0, hh0;
};
__device__ __forceinline__ void neuron_load(const NetDev &net, const StateDev &st, uint32_t i, const PopDev &p,
                                            NeuronIn &n) {
    n.qe = n.qi = n.ref = 0;
    n.V = n.ge = n.gi = n.xq = 0.0f;
    n.h0 = n.hh0 = 0ull;
    if (p.kind == POP_LIF_DELTA) {
        n.qe = st.in_e[i];
        n.ref = st.ref[i];
        n.V = st.V[i];
    } else if (p.kind == POP_LIF_CUBA) {
        n.qe = st.in_e[i];
        n.qi = st.in_i[i];
        n.ref = st.ref[i];
        n.V = st.V[i];
        n.ge = st.ge[i];
        n.gi = st.gi[i];
    }
    if (p.flags & PF_POST_PLASTIC) {
        n.h0 = st.hist[i];
        if (net.H > kHistBits) n.hh0 = st.hist_hi[i];
        n.xq = st.xpost[i];
    }
}
__device__ __forceinline__ bool neuron_step(const NetDev &net, const StateDev &st, uint32_t i, const PopDev &p,
                                            int64_t t, bool &recent, const NeuronIn &n) {
    bool fired = false;
    recent = false;
    if (p.kind == POP_POISSON) {
        const u32x4 r = philox4x32_10(i, (uint32_t)t, 2u, 0u, net.key0, net.key1);
        fired = (uint64_t)r.x < p.thr;
    } else if (p.kind == POP_LIF_DELTA) {
        const int32_t q = n.qe;
        const float I = __fmul_rn(__int2float_rn(q), net.inv_scale);
        if (q != 0) st.in_e[i] = 0;
        int32_t ref = n.ref;
        float V = n.V;
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
        const int32_t qe = n.qe, qi = n.qi;
        float ge = __fadd_rn(n.ge, __fmul_rn(__int2float_rn(qe), net.inv_scale));
        float gi = __fadd_rn(n.gi, __fmul_rn(__int2float_rn(qi), net.inv_scale));
        if (qe != 0) st.in_e[i] = 0;
        if (qi != 0) st.in_i[i] = 0;
        int32_t ref = n.ref;
        const int32_t ref0 = ref;
        float V = n.V;
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
        const uint64_t h0 = n.h0;
        const uint64_t h = (h0 << 1) | (uint64_t)fired;
        st.hist[i] = h;
        uint64_t hh = 0ull;
        if (net.H > kHistBits) {                 // H = 128: second word, bits 64..127
            hh = (n.hh0 << 1) | (h0 >> 63);
            st.hist_hi[i] = hh;
        }
        recent = (h | hh) != 0ull;
        // the window's spike position (k_stdp_ev's shared table): 0xfe no
        // spike in the last H steps, 0xff several, else the bit of the only one
        {
            const uint32_t n1 = __popcll(h) + __popcll(hh);
            st.fpos[(size_t)(t & 3) * st.fstride + i] = n1 == 0 ? (uint8_t)0xfeu
                       : n1 > 1 ? (uint8_t)0xffu
                                : (uint8_t)(h ? 63 - __clzll((long long)h) : 127 - __clzll((long long)hh));
        }
        // potentiation factors of a forced flush for this target, oldest
        // spike first (k_flush: w = min(w + A+ (x_pre f), w_max)), for a flush
        // of age H - k (flushed k steps early, R36): f_k = sum over its spikes
        // s <= H - 1 - k of D+[H - k - s] (buffer 4k + (t & 3); k <= 1, or 2 with
        // the 3-step deadline).  k_flush(t) runs beside k_front(t+1), so it
        // reads these step-t buffers, never the live history words
        if (recent) {
            const float *dpl = net.stdp[p.post_stdp].dplus;
            const int H = (int)net.H;
            float f = 0.0f, f1 = 0.0f, f2 = 0.0f;
            for (uint64_t m = hh; m; ) {
                const int b = 63 - __clzll((long long)m);
                m &= ~(1ull << b);
                f = __fadd_rn(f, dpl[H - 64 - b]);
                if (64 + b <= H - 2) f1 = __fadd_rn(f1, dpl[H - 1 - 64 - b]);
                if (64 + b <= H - 3) f2 = __fadd_rn(f2, dpl[H - 2 - 64 - b]);
            }
            for (uint64_t m = h; m; ) {
                const int b = 63 - __clzll((long long)m);
                m &= ~(1ull << b);
                f = __fadd_rn(f, dpl[H - b]);
                if (b <= H - 2) f1 = __fadd_rn(f1, dpl[H - 1 - b]);
                if (b <= H - 3) f2 = __fadd_rn(f2, dpl[H - 2 - b]);
            }
            st.fpot[(size_t)(t & 3) * st.fstride + i] = f;
            st.fpot[(size_t)(4 + (t & 3)) * st.fstride + i] = f1;
            if (net.fl_lag >= 3) st.fpot[(size_t)(8 + (t & 3)) * st.fstride + i] = f2;
        }
        const float x = __fmul_rn(n.xq, p.d_minus);   // x_post decay (+1 on a post spike), R7
        st.xpost[i] = fired ? __fadd_rn(x, 1.0f) : x;
    }
    if (fired) atomicAdd(st.nspk + i, 1u);          // (fire and forget: no round trip)
    return fired;
}
__device__ __forceinline__ bool neuron_update(const NetDev &net, const StateDev &st, uint32_t i, const PopDev &p,
                                              int64_t t, bool &recent) {
    NeuronIn n;
    neuron_load(net, st, i, p, n);
    return neuron_step(net, st, i, p, t, recent, n);
}

// kPart (world > 1 with D = 0, where the arrivals of t include the other
// ranks' spikes of t): 1 = the neuron update and ring words only, 2 = the
// lists only, after the exchange put every rank's words of t in the ring;
// 3 = the fused step's front (the neurons without inputs, >= R, and every
// row's lists; k_deliver(t-1)'s epilogue updated [0, R) and wrote their ring
// words); 0 = all (every other case).  The step comes from the front's own
// counter in the fused step (use_tf: ctr->tf, advanced by the last CTA), where
// k_front(t) runs beside k_deliver(t), which advances ctr->t; else ctr->t.
template <bool kAhead, int kPart>
__global__ void __launch_bounds__(kFrontThreads, 2048 / kFrontThreads)   // two CTAs per SM: <= 32 registers
k_front(NetDev net, StateDev st, uint32_t use_tf) {
    __shared__ Compact2 cs;
    const unsigned long long t_entry = st.kspan ? gtimer() : 0ull;
    pdl_wait();            // k_deliver(t-1): inputs, step counter
    pdl_launch();
    trace_mark(st.trace, 0, 0);
    const int64_t t = use_tf ? *(volatile const int64_t *)&st.ctr->tf : st.ctr->t;
    constexpr int kSpan = (kPart == 2 || kPart == 4) ? 4 : 0;     // (span slot 4: the second front kernel)
    if (st.kspan) kspan_begin(st.kspan, t, kSpan, t_entry, gtimer());
    const uint32_t par = (uint32_t)(t & 1);
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t lane = threadIdx.x & 31;
    const bool valid = i < net.N;
    const int pi = valid ? find_pop(net, i) : 0;
    const PopDev &p = net.pop[pi];
    bool fired = false, recent = false;
    // this rank updates its own target range and every neuron without inputs
    // (Poisson: counter-based, identical on all ranks); the spike bits of the
    // other input neurons arrive by the exchange
    const bool owned = i >= net.R || (i >= net.tgt_lo && i < net.tgt_hi);
    const bool upd = kPart == 4 ? (valid && i < net.R)
                                : (kPart != 2 && valid && owned && (kPart != 3 || i >= net.R));
    // ---- (0) every load of the step's reads that does not depend on this
    //      step's arithmetic, issued together before any store: the neuron's
    //      state, the ring words of its arrivals, the row's STDP state
    NeuronIn nin;
    if (upd) neuron_load(net, st, i, p, nin);
    const bool plastic_row = valid && (p.flags & PF_PRE_PLASTIC);
    const bool lists = kPart != 1 && kPart != 4;
    uint32_t rw_arr = 0u, rw_arr1 = 0u, rw_arr2 = 0u, rw_prev = 0u, vm_prev = 0u;
    int32_t tl0 = 0;
    float xp0 = 0.0f;
    if (lists && valid) {
        const uint32_t *ring = st.ring + (i >> 5);
        const uint32_t rs = net.ring_stride;
        auto word = [&](int64_t step) { return ring[(size_t)(step & (kRingSlots - 1)) * rs]; };
        if (net.D != 0 && t >= (int64_t)net.D) rw_arr = word(t - net.D);
        if (kAhead && t + 1 >= (int64_t)net.D) rw_arr1 = word(t + 1 - net.D);
        if (kAhead && net.D != 2 && t + 2 >= (int64_t)net.D) rw_arr2 = word(t + 2 - net.D);
        if (plastic_row) {
            tl0 = st.tlu[i];
            xp0 = st.xpre[i];
            if (t >= 1) vm_prev = st.vmask[par ^ 1u][i >> 5];
            if (t - 1 >= (int64_t)net.D) rw_prev = word(t - 1 - net.D);
        }
    }
    // ---- (1) neuron dynamics (App. B op order); kPart 3 (the fused / split
    //      step): the input neurons [0, R) were updated elsewhere (k_deliver(t-1)'s
    //      epilogue / kPart 4); kPart 4: only those, and the stateless Poisson
    //      draws of the neurons >= R sharing R's ring word
    if (upd) {
        fired = neuron_step(net, st, i, p, t, recent, nin);
    } else if (kPart == 4 && valid && p.kind == POP_POISSON) {
        const u32x4 r = philox4x32_10(i, (uint32_t)t, 2u, 0u, net.key0, net.key1);
        fired = (uint64_t)r.x < p.thr;
    }
    const uint32_t fword = __ballot_sync(0xffffffffu, fired);
    const uint32_t rword = __ballot_sync(0xffffffffu, recent);
    // ring word of ids [i, i + 32): written by the rank owning its input
    // neurons (the word straddling R by the last rank), by all if it has none
    const bool wown = i >= net.R ? true : (i + 32 <= net.R ? (i >= net.tgt_lo && i + 32 <= net.tgt_hi)
                                                           : (i >= net.tgt_lo && net.tgt_hi == net.R));
    if (kPart != 2 && lane == 0 && valid && wown && (kPart != 3 || i >= net.R) && (kPart != 4 || i < net.R)) {
        // (kPart 3 / 4: i = the warp's first neuron -- R's word belongs to kPart 4)
        st.ring[(size_t)(t & (kRingSlots - 1)) * net.ring_stride + (i >> 5)] = fword;
        if (net.nstdp) st.recent[(size_t)(t & 3) * st.rstride + (i >> 5)] = rword;
        // this rank's share of the step's input-neuron words, for the exchange
        const uint32_t w = i >> 5, w0 = net.rank_lo[net.rank] >> 5;
        if (net.xchg && i < net.R && w >= w0 && w < w0 + net.wmax) st.sendbuf[w - w0] = fword;
    }

    if (kPart == 1 || kPart == 4) {              // (the list part, kPart 2 / 3, advances ctr->tf)
        trace_mark(st.trace, 0, 3);
        kspan_end(st.kspan, t, kSpan);
        return;
    }

    // ---- (2) arrival of row i at step t: its spike of step t - D (hist[delay])
    bool arr = false, arr1 = false, arr2 = false;
    if (valid) {
        const uint32_t b = i & 31;
        if (net.D == 0) arr = kPart == 2 ? ring_bit(st.ring, net.ring_stride, t, i) != 0u : fired;
        else arr = (rw_arr >> b) & 1u;
        // kAhead (D >= 2): the arrivals of t + 1 and t + 2 are spikes of steps <= t - 1
        if (kAhead) arr1 = (rw_arr1 >> b) & 1u;
        if (kAhead && t + 2 >= (int64_t)net.D) {
            // (D = 2: the spike of this step -- this thread's own `fired` where it
            // updated neuron i, the other CTAs of this grid write the ring slot)
            const bool own = owned && (kPart != 3 || i >= net.R);
            arr2 = net.D == 2 ? (own ? fired : ring_bit(st.ring, net.ring_stride, t, i) != 0u) : ((rw_arr2 >> b) & 1u);
        }
    }
    bool visit = false, flush = false;
    RowDesc d, a;
    if (plastic_row) {
        const StdpDev &sd = net.stdp[p.stdp];
        int32_t tl = tl0;
        float xp = xp0;
        // finalise a visit of step t-1 (its synapses were updated at t-1)
        if (t >= 1 && ((vm_prev >> (i & 31)) & 1u)) {
            const bool arr_prev = (rw_prev >> (i & 31)) & 1u;
            xp = xpre_after(sd, xp, (int)(t - 1 - tl), arr_prev);
            tl = (int32_t)(t - 1);
            st.xpre[i] = xp;
            st.tlu[i] = tl;
        }
        const int age = (int)(t - tl);
        const int H = (int)net.H;
        if (kAhead) {
            // forced flush (R3) of the split step graph: k_flush(t) runs beside
            // the delivery (and arrival STDP) of steps t and t+1, so a row it
            // flushes must not arrive at t + 1.  A row of age H arriving at t + 1
            // waits for that arrival (age H there); a row of age H - 1 arriving at
            // t + 2 is flushed one step early (age H - 1) -- then no row of age H
            // arrives at t + 1 (D >= 2: known one step ahead).  Exact by R4.
            // With the 3-step deadline (fl_lag 3, D >= 3): a row of age >= H - 2
            // is flushed unless it arrives at t, t+1 or t+2 (then that arrival,
            // age <= H, replays it) -- no row flushed at t arrives before t + 3.
            if (net.fl_lag >= 3) flush = !arr && !arr1 && !arr2 && age >= H - 2;
            else flush = !arr && !arr1 && (age >= H || (age == H - 1 && arr2));
            visit = arr || flush;
        } else {
            // forced flush (R3): at age H, or -- batched schedule (R33) -- every
            // flush_period steps for the rows of age >= H - flush_period
            const uint32_t K = net.flush_period;
            visit = arr || (K == 0 ? age >= H : ((uint32_t)(t % K) == K - 1 && age >= (int)(H - K)));
            if (net.plast_mode == 2u) visit = true;   // SNN_PLAST_NAIVE: every row every step (Fig. 2a schedule)
            flush = visit && !arr;
        }
        if (visit && (!kAhead || flush)) {
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
        if (kAhead && arr1) {
            // the row's STDP state at t + 1 for the arrival (delivery of t + 1):
            // after this step's visit, if any (its x_pre / tlu are finalised by
            // k_front(t+1), identically)
            const float xp1 = visit ? xpre_after(sd, xp, age, arr) : xp;
            const int32_t tl1 = visit ? (int32_t)t : tl;
            const uint2 sg = st.seg[i];
            a.meta = (uint32_t)(t + 1 - tl1) | kMetaPlastic | ((uint32_t)p.stdp << 12);
            a.xp = xp1;
            a.s0 = sg.x;
            a.s1 = sg.y;
        }
    }
    // (the arriving row's CSR start: loaded before the list compaction, so the
    // load and the compaction's atomics share one round trip)
    if (kAhead ? arr1 : arr) a.start = st.row_ptr[i];
    const uint32_t vword = __ballot_sync(0xffffffffu, visit);
    if (net.nstdp && lane == 0 && valid) st.vmask[par][i >> 5] = vword;
    uint32_t sp, sa, sf, np, na, nf;
    if (kAhead) {
        // forced flushes of t -> k_flush(t); arrivals of t + 1 -> k_deliver(t+1)
        // (which runs the plastic arrivals' STDP, Fig. 2c, before delivering)
        compact3(cs, st.ctr->lst[t & 7], st.ctr->lst[(t + 1) & 7] + 1, st.ctr->lst[t & 7] + 2, false, arr1, flush,
                 sp, sa, sf, np, na, nf);
        if (flush) st.vdesc[t & 3][(size_t)st.nblk * kFrontThreads - 1 - sf] = d;
        if (arr1) {
            a.row = i;
            if (!plastic_row) a.meta = 0u;
            a.meta |= kMetaArr | ((uint32_t)(p.rcpt_uniform & 3) << 8);
            if (p.rcpt_uniform < 0) a.meta |= (uint32_t)pi << 16;
            if (!plastic_row) {
                a.xp = 0.0f;
                a.s0 = a.s1 = 0;
            }
            a.pad = 0;
            st.adesc[(t + 1) & 1][sa] = a;
        }
        np = __syncthreads_count(visit && arr);      // (metrics: plastic arrivals visited at t)
        na = 0;                                      // (arrivals are counted by k_deliver)
    } else {
        // plastic visits -> k_stdp: the arrivals from the front of the list, the
        // forced flushes from its back (so k_stdp can share each kind evenly);
        // every arrival -> k_deliver
        const bool parr = visit && arr;
        compact3(cs, st.ctr->lst[t & 7], st.ctr->lst[t & 7] + 1, st.ctr->lst[t & 7] + 2, parr, arr, flush, sp, sa, sf,
                 np, na, nf);
        if (parr) st.vdesc[t & 3][sp] = d;
        if (flush) st.vdesc[t & 3][(size_t)st.nblk * kFrontThreads - 1 - sf] = d;
        if (arr) {                                       // every arriving row is delivered
            a.row = i;
            a.meta = kMetaArr | ((uint32_t)(p.rcpt_uniform & 3) << 8);
            if (p.rcpt_uniform < 0) a.meta |= (uint32_t)pi << 16;
            a.xp = 0.0f;
            a.s0 = a.s1 = 0;
            a.pad = 0;
            st.adesc[par][sa] = a;
        }
    }
    if (threadIdx.x == 0) {
        // slot (t + 2) & 7 was last used by step t - 6 (long consumed): reset it
        // for the lists of t + 2 (kAhead: its arrivals are appended by k_front(t+1))
        if (blockIdx.x == 0) *reinterpret_cast<uint4 *>(st.ctr->lst[(t + 2) & 7]) = make_uint4(0u, 0u, 0u, 0u);
        // metrics (fire-and-forget reductions): spikes arriving, plastic rows
        // visited (arrivals + forced flushes), forced flushes
        if (na) atomicAdd(&st.ctr->metric[1], (unsigned long long)na);
        if (np + nf) atomicAdd(&st.ctr->metric[2], (unsigned long long)(np + nf));
        if (nf) atomicAdd(&st.ctr->metric[5], (unsigned long long)nf);
    }
    trace_mark(st.trace, 0, 3);
    kspan_end(st.kspan, t, kSpan);
    if (use_tf) {
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(&st.ctr->fr_ticket, 1u) == gridDim.x - 1) {   // the last CTA: next step
            st.ctr->fr_ticket = 0;
            st.ctr->tf = t + 1;
        }
    }
}

// ---------------------------------------------------- CTA row-table helpers
// Block-wide inclusive scan of one u32 per thread (kThreads <= 1024).
template <int kThreads>
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t *wsum, uint32_t &total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t off = 0, tot = 0;
    for (int w2 = 0; w2 < kThreads / 32; w2++) {
        const uint32_t x = wsum[w2];
        if (w2 < (int)warp) off += x;
        tot += x;
    }
    total = tot;
    return off + inc;
}

// ------------------------------------------------------------------ k_stdp
// Shared / predicated global loads written out in PTX so that the compiler
// neither re-derives the shared window per access nor branches around a load.
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint64_t ldg_u64_if(const uint64_t *p, uint32_t pred) {
    uint64_t v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.b64 %0, 0;\n @q ld.global.nc.u64 %0, [%1];\n}\n"
                 : "=l"(v) : "l"(p), "r"(pred));
    return v;
}
__device__ __forceinline__ float ldg_f32_if(const float *p, uint32_t pred) {
    float v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.b32 %0, 0f00000000;\n @q ld.global.nc.f32 %0, [%1];\n}\n"
                 : "=f"(v) : "l"(p), "r"(pred));
    return v;
}
// p[j] if pred, else 0 (one wide multiply-add for the address)
__device__ __forceinline__ float ldg_f32_idx_if(const float *p, uint32_t j, uint32_t pred) {
    float v;
    asm volatile("{\n .reg .pred q;\n .reg .u64 a;\n setp.ne.u32 q, %3, 0;\n mov.b32 %0, 0f00000000;\n"
                 " mad.wide.u32 a, %2, 4, %1;\n @q ld.global.nc.f32 %0, [a];\n}\n"
                 : "=f"(v) : "l"(p), "r"(j), "r"(pred));
    return v;
}
__device__ __forceinline__ uint32_t ldg_u8_if(const uint8_t *p, uint32_t pred) {
    uint32_t v;
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n mov.b32 %0, 255;\n @q ld.global.nc.u8 %0, [%1];\n}\n"
                 : "=r"(v) : "l"(p), "r"(pred));
    return v;
}
__device__ __forceinline__ void stg_f32_if(float *p, float v, uint32_t pred) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}\n"
                 :: "l"(p), "f"(v), "r"(pred) : "memory");
}

// ---- TMA bulk copies and mbarriers (producer / consumer stage ring)
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
                     " selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(a), "r"(parity), "r"(0x989680u) : "memory");   // suspend-time hint (ns)
}
// global -> shared bulk copy (16-byte aligned, size a multiple of 16), completes on mbar
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ uint4 lds_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Fig. 2b (SNN_PLAST_LAZY, ablation): the same updates as stdp_synapse, found
// by replaying every step of the window instead of jumping between set bits.
__device__ __noinline__ float stdp_synapse_lazy(float w, uint64_t m, bool arr, float xq, float xp, int age,
                                                uint32_t dp, float a_plus, float a_minus, float w_max,
                                                uint64_t mhi) {
    for (int s = age - 1; s >= 0; s--) {             // steps t - s, oldest first
        const uint64_t bit = s >= 64 ? (mhi >> (s - 64)) & 1ull : (m >> s) & 1ull;
        if (bit) {
            const float nw = __fadd_rn(w, __fmul_rn(a_plus, __fmul_rn(xp, lds_f32(dp + 4u * (uint32_t)(age - s)))));
            w = nw < w_max ? nw : w_max;
        }
    }
    const float dw = __fsub_rn(w, __fmul_rn(a_minus, xq));
    return arr ? (dw > 0.0f ? dw : 0.0f) : w;
}

// Window of a row of age `age`: history bits [0, age) = post spikes in steps
// (tlu, t] (R2); bits 64..127 live in the second word (H = 128).
__device__ __forceinline__ uint64_t window_lo(uint64_t lo, int age) { return age >= 64 ? lo : lo & ((1ull << age) - 1ull); }
__device__ __forceinline__ uint64_t window_hi(uint64_t hi, int age) {
    return age <= 64 ? 0ull : (age >= 128 ? hi : hi & ((1ull << (age - 64)) - 1ull));
}

// One plastic synapse (Fig. 2c, R7): potentiation by the post spikes in
// (mhi:m), oldest first ("__clz") with the closed-form skip-ahead
// w = min(w + A+ (x_pre D+[age - p]), w_max), then, on an arrival, the
// depression w = max(w - A- x_post, 0).  dp = shared address of the D+ table.
__device__ __forceinline__ float stdp_synapse(float w, uint64_t m, bool arr, float xq, float xp, int age,
                                              uint32_t dp, float a_plus, float a_minus, float w_max,
                                              uint64_t mhi = 0ull) {
    while (mhi) {                         // steps t-127 .. t-64 (H = 128)
        const int pb = 127 - __clzll((long long)mhi);
        mhi &= ~(1ull << (pb - 64));
        const float nw = __fadd_rn(w, __fmul_rn(a_plus, __fmul_rn(xp, lds_f32(dp + 4u * (uint32_t)(age - pb)))));
        w = nw < w_max ? nw : w_max;
    }
    while (m) {
        const int pb = 63 - __clzll((long long)m);
        m &= ~(1ull << pb);
        const float nw = __fadd_rn(w, __fmul_rn(a_plus, __fmul_rn(xp, lds_f32(dp + 4u * (uint32_t)(age - pb)))));
        w = nw < w_max ? nw : w_max;
    }
    const float dw = __fsub_rn(w, __fmul_rn(a_minus, xq));
    return arr ? (dw > 0.0f ? dw : 0.0f) : w;
}

// k_stdp launch shape: one CTA per SM; 4 consumer groups of 4 warps take the
// stages round-robin (so the gathers of one group overlap the filtering of the
// others) + 1 TMA producer warp; 6 stages in the ring.
#ifndef SNN_STDP_GROUPS
#define SNN_STDP_GROUPS 4
#endif
#ifndef SNN_STDP_CH
#define SNN_STDP_CH 4
#endif
constexpr int kStdpGroups = SNN_STDP_GROUPS;
constexpr int kStdpGroupWarps = 4;
constexpr int kStdpGroupThr = kStdpGroupWarps * 32;
constexpr int kStdpConsWarps = kStdpGroups * kStdpGroupWarps;
constexpr int kStdpCons = kStdpConsWarps * 32;     // consumer threads
constexpr int kStdpThreads = kStdpCons + 32;       // + the producer warp
constexpr int kStdpWarps = kStdpThreads / 32;
constexpr int kStdpChPerThr = SNN_STDP_CH;         // 16-byte chunks (16 synapses) per consumer thread and stage
constexpr int kStdpStageCh = kStdpChPerThr * kStdpGroupThr;   // 512 chunks per stage: 8 KB ids + 8 KB weights
#ifndef SNN_STDP_STAGES
#define SNN_STDP_STAGES 6
#endif
// 96 KB in flight per SM: measured on cfg3 (us/step) 4: 50.3, 5: 47.5, 6: 46.0,
// 7: 46.3, 8: 46.3, 10: 50.8 -- the rest of the 256 KB stays L1 for the gathers
constexpr int kStdpStages = SNN_STDP_STAGES;
#ifndef SNN_STDP_ROWS
#define SNN_STDP_ROWS 128
#endif
#ifndef SNN_STDP_LIST
#define SNN_STDP_LIST 128
#endif
constexpr int kStdpRows = SNN_STDP_ROWS;            // row table per round
constexpr uint32_t kStdpList = SNN_STDP_LIST;       // per-warp list of the synapses to update (a stage
                                                    // lists more in several passes)

struct __align__(16) StdpRow {   // one visited row of this CTA (shared memory)
    int64_t cb;      // 16-byte aligned CSR offset of its plastic span
    float xp;        // x_pre at tlu
    uint32_t meta;
    uint32_t lo, hi; // valid elements [lo, hi) relative to cb
    uint32_t first;  // flattened index of its first 16-byte chunk
    uint32_t nch;    // chunks
};

struct StdpSmem {                       // static part of k_stdp's shared memory
    uint64_t full[kStdpStages], empty[kStdpStages], bmap;
    StdpRow rows[kStdpRows];
    uint32_t incl[kStdpRows];
    uint32_t wsum[kStdpWarps];
    float dplus[4 * (kMaxHist + 1)];
    float4 par[4];                      // per projection: a_plus, a_minus, w_max
    uint32_t list[kStdpConsWarps][kStdpList];   // (element p in stage << 9) | (rec << 8) | row slot
};

// Lazy + event-driven STDP over the visited rows (Fig. 2c).  For each plastic
// synapse (i -> j):
//   m = hist[j] & window(age)        post spikes in steps (tlu, t]   (R2)
//   for set bits p, oldest first:    w = min(w + A+ (x_pre D+[age-p]), w_max)
//   on an arrival:                   w = max(w - A- x_post[j], 0)
// One CTA per SM takes a contiguous share of the visited rows.  A producer
// thread streams the rows' plastic spans (target ids and weights) into a ring
// of shared-memory stages with TMA bulk copies (cp.async.bulk, mbarrier
// complete_tx), so the bytes in flight do not depend on the consumers.  A
// consumer group filters a stage (16 synapses per thread): forced-flush
// synapses whose target fired in the last 64 steps (shared bitmap probe) and
// every synapse of an arriving row go to its warp's list; the list is then
// drained four entries per lane (history / x_post gathers, Fig. 2c, store of
// the changed weights) and the stage released to the producer.
// kGeneric: the step-by-step list drain of the lazy schedule (and the read-out
// flush) -- the default step kernel does not carry it.
template <bool kLazy, bool kH128, bool kGeneric>
__global__ void __launch_bounds__(kStdpThreads, 1)
k_stdp(NetDev net, StateDev st, int64_t t_fixed, uint32_t pp_lo, uint32_t pp_hi) {
    extern __shared__ __align__(16) unsigned char smem[];
    const unsigned long long t_entry = st.kspan ? gtimer() : 0ull;
    StdpSmem &sm = *reinterpret_cast<StdpSmem *>(smem);
    unsigned char *stage_base = smem + ((sizeof(StdpSmem) + 127) & ~(size_t)127);   // [stages][ids 8K | w 8K]
    uint32_t *recent_s = reinterpret_cast<uint32_t *>(stage_base + (size_t)kStdpStages * kStdpStageCh * 32);  // bitmap
    const bool readout = t_fixed >= 0;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool producer = warp == kStdpConsWarps;
    const uint32_t w_lo = (pp_lo >> 7) << 2, w_hi = (pp_hi + 31) >> 5;     // 16-byte aligned start
    const uint32_t full_a = smem_u32(sm.full), empty_a = smem_u32(sm.empty), bmap_a = smem_u32(&sm.bmap);
    const uint32_t stage_a = smem_u32(stage_base);
    // ---- prologue independent of k_front(t): barriers, STDP constants
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStdpStages; s++) {
            mbar_init(full_a + 8 * s, 1);
            mbar_init(empty_a + 8 * s, kStdpGroupWarps);
        }
        mbar_init(bmap_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t x = threadIdx.x; x < net.nstdp * (kMaxHist + 1); x += kStdpThreads)
        sm.dplus[x] = st.stdp[x / (kMaxHist + 1)].dplus[x % (kMaxHist + 1)];
    if (threadIdx.x < net.nstdp)
        sm.par[threadIdx.x] = make_float4(st.stdp[threadIdx.x].a_plus, st.stdp[threadIdx.x].a_minus,
                                          st.stdp[threadIdx.x].w_max, 0.0f);
    // the step counter was advanced by k_deliver(t-1), which completed before
    // k_front(t) triggered this launch: read it before waiting for k_front(t)
    const int64_t t = readout ? t_fixed : *(volatile const int64_t *)&st.ctr->t;
    pdl_wait();            // k_front(t): lists, histories, bitmap
    pdl_launch();          // k_deliver may start its tabulation (k_front is complete)
    if (!readout) trace_mark(st.trace, 1, 0);
    if (!readout && st.kspan) kspan_begin(st.kspan, t, 1, t_entry, gtimer());
    const uint32_t par = (uint32_t)(t & 1);
    const RowDesc *Vl = readout ? st.rdesc : st.vdesc[t & 3];
    const uint32_t *lens = readout ? st.ctr->rlst : st.ctr->lst[t & 7];
    // (k_front(t) complete).  The event schedule's forced flushes are k_flush's
    const uint32_t nA = lens[0], nF = (readout || !kGeneric) ? 0u : lens[2];
    const size_t cap_back = (size_t)st.nblk * kFrontThreads - 1;   // forced flushes: from the back
    const uint32_t bm_bytes = 16u * ((w_hi - w_lo + 3) >> 2);
    if (threadIdx.x == 0) {   // bitmap of recently fired post neurons (one bulk copy; the barrier's initialiser)
        mbar_expect_tx(bmap_a, bm_bytes);
        bulk_g2s(smem_u32(recent_s), st.recent + (size_t)(t & 3) * st.rstride + w_lo, bm_bytes, bmap_a);
    }
    __syncthreads();       // barrier init visible
    // even shares of each kind: plastic arrivals (front of the list; read-out
    // rows) and forced flushes (back); this CTA's rows: [0, nAb) arrivals, then flushes
    const uint32_t a_begin = (uint32_t)(((uint64_t)nA * blockIdx.x) / gridDim.x);
    const uint32_t a_end = (uint32_t)(((uint64_t)nA * (blockIdx.x + 1)) / gridDim.x);
    const uint32_t f_begin = (uint32_t)(((uint64_t)nF * blockIdx.x) / gridDim.x);
    const uint32_t f_end = (uint32_t)(((uint64_t)nF * (blockIdx.x + 1)) / gridDim.x);
    const uint32_t nAb = a_end - a_begin;
    const uint32_t r_begin = 0, r_end = nAb + (f_end - f_begin);
    const uint32_t rs_addr = smem_u32(recent_s) - 4u * w_lo;     // bitmap word of neuron j: + 4 (j >> 5)
    const uint32_t dp_addr = smem_u32(sm.dplus);
    if (!readout) trace_mark(st.trace, 1, 1);
    uint32_t n_syn = 0, n_w = 0, n_rw = 0;
    unsigned long long dbg_wait = 0, dbg_busy = 0, dbg_n = 0, dbg_first = 0;   // (SNN_FLAG_TRACE only)
    unsigned long long dbg_filt = 0, dbg_arr = 0;
    uint32_t g0 = 0;             // global stage index of the round's first stage (ring position)
    bool bm_ready = false;
    const uint64_t *__restrict__ ghist = st.hist;
    const uint64_t *__restrict__ ghist_hi = st.hist_hi;
    // compile-time variants: H = 128 (second history word), SNN_PLAST_LAZY (Fig. 2b)
    constexpr uint32_t hi_on = kH128 ? 1u : 0u;
    constexpr bool lazy = kLazy;
    const float *__restrict__ gxpost = st.xpost;
    float *__restrict__ gw = st.w;
    for (uint32_t r0 = r_begin; r0 < r_end; r0 += kStdpRows) {
        // ---- tabulate up to kStdpRows rows (one per thread), chunk prefix
        const uint32_t r = r0 + threadIdx.x;
        uint32_t nch = 0;
        StdpRow rw;
        rw.cb = 0;
        rw.lo = rw.hi = 0;
        rw.xp = 0.0f;
        rw.meta = 0;
        if (threadIdx.x < kStdpRows && r < r_end) {
            const RowDesc d = Vl[r < nAb ? (size_t)(a_begin + r) : cap_back - (f_begin + (r - nAb))];
            const bool arr = (d.meta & kMetaArr) != 0;
            const int64_t cs = d.start + d.s0, ce = d.start + d.s1;
            // a flush with x_pre == 0 changes no weight (potentiation adds 0)
            if (cs < ce && (arr || d.xp != 0.0f || lazy)) {
                rw.cb = cs & ~3ll;
                rw.lo = (uint32_t)(cs - rw.cb);
                rw.hi = (uint32_t)(ce - rw.cb);
                rw.xp = d.xp;
                rw.meta = d.meta;
                nch = (rw.hi + 3) >> 2;
                n_syn += (uint32_t)(ce - cs);
            }
        }
        uint32_t T = 0;
        const uint32_t inc = block_incl_scan<kStdpThreads>(nch, sm.wsum, T);
        if (threadIdx.x < kStdpRows) {
            rw.first = inc - nch;
            rw.nch = nch;
            sm.rows[threadIdx.x] = rw;
            sm.incl[threadIdx.x] = inc;
        }
        __syncthreads();
        if (!readout) trace_mark(st.trace, 1, 2);
        const uint32_t nst = (T + kStdpStageCh - 1) / kStdpStageCh;
        if (producer) {
            // ---- TMA producer: stage s covers flattened chunks [s C, s C + C)
            if (lane == 0) {
                uint32_t pr = 0;
                for (uint32_t s = 0; s < nst; s++) {
                    const uint32_t g = g0 + s, slot = g % kStdpStages;
                    const unsigned long long tw0 = st.trace ? clock64() : 0ull;
                    mbar_wait(empty_a + 8 * slot, ((g / kStdpStages) & 1u) ^ 1u);
                    if (st.trace) { dbg_wait += clock64() - tw0; dbg_n++; }
                    const uint32_t a = s * kStdpStageCh, b = min(a + kStdpStageCh, T);
                    const uint32_t fb = full_a + 8 * slot;
                    mbar_expect_tx(fb, 32u * (b - a));
                    const uint32_t dst = stage_a + slot * (kStdpStageCh * 32);
                    for (uint32_t c = a; c < b;) {
                        while (c >= sm.incl[pr]) pr++;
                        const StdpRow &rr = sm.rows[pr];
                        const uint32_t e = min(b, sm.incl[pr]);
                        const int64_t gc = rr.cb + 4ll * (c - rr.first);     // element offset
                        const uint32_t bytes = 16u * (e - c);
                        bulk_g2s(dst + 16u * (c - a), st.idx + gc, bytes, fb);
                        bulk_g2s(dst + kStdpStageCh * 16 + 16u * (c - a), gw + gc, bytes, fb);
                        c = e;
                    }
                }
            }
        } else {
            // ---- consumer group grp takes the stages g = grp (mod 4); thread gt
            //      of the group takes chunks gt + 128 u of the stage
            const uint32_t grp = warp / kStdpGroupWarps, gt = threadIdx.x % kStdpGroupThr;
            if (!bm_ready) {
                mbar_wait(bmap_a, 0);
                bm_ready = true;
            }
            uint32_t o = 0, o_end = sm.incl[0];
            uint4 cur = lds_v4(smem_u32(&sm.rows[0]) + 16);     // lo, hi, first, nch
            uint2 cm = make_uint2(sm.rows[0].meta, __float_as_uint(sm.rows[0].xp));
            uint32_t *list = sm.list[warp];
            const uint32_t list_a = smem_u32(list);
            for (uint32_t g = g0 + ((grp + kStdpGroups - g0 % kStdpGroups) % kStdpGroups); g < g0 + nst;
                 g += kStdpGroups) {
                const uint32_t slot = g % kStdpStages;
                const uint32_t a = (g - g0) * kStdpStageCh;
                const uint32_t sa = stage_a + slot * (kStdpStageCh * 32);
                uint32_t hm = 0, rm = 0, slots = 0;   // 16-bit masks: list the synapse / target may hold a post spike
                uint32_t am = 0;                      // 16-bit mask: synapses of arriving rows (updated in place)
                const unsigned long long tw0 = st.trace ? clock64() : 0ull;
                mbar_wait(full_a + 8 * slot, (g / kStdpStages) & 1u);
                const unsigned long long tw1 = st.trace ? clock64() : 0ull;
                if (st.trace) { dbg_wait += tw1 - tw0; dbg_n++; if (!dbg_first) dbg_first = gtimer(); }
#pragma unroll
                for (int u = 0; u < kStdpChPerThr; u++) {
                    const uint32_t c = a + gt + kStdpGroupThr * u;
                    if (c < T) {
                        if (c >= o_end) {
                            while (c >= o_end) o_end = sm.incl[++o];
                            cur = lds_v4(smem_u32(&sm.rows[o]) + 16);
                            cm = make_uint2(sm.rows[o].meta, __float_as_uint(sm.rows[o].xp));
                        }
                        const uint4 j4 = lds_v4(sa + 16u * (gt + kStdpGroupThr * u));
                        const uint32_t x0 = 4u * (c - cur.z);
                        const bool arr = (cm.x & kMetaArr) != 0;
                        const bool pot = __uint_as_float(cm.y) != 0.0f;
                        const uint32_t jj[4] = {j4.x, j4.y, j4.z, j4.w};
                        uint32_t bits = 0, inm = 0xfu;
                        if (x0 < cur.x || x0 + 4 > cur.y) {      // a row's first / last chunk
                            inm = 0;
#pragma unroll
                            for (int e = 0; e < 4; e++) inm |= (uint32_t)(x0 + e >= cur.x && x0 + e < cur.y) << e;
                        }
#pragma unroll
                        for (int e = 0; e < 4; e++) {
                            const uint32_t j = ((inm >> e) & 1u) ? jj[e] : pp_lo;
                            bits |= ((lds_u32(rs_addr + ((j >> 5) << 2)) >> (j & 31)) & 1u) << e;
                        }
                        // event (Fig. 2c): only targets that fired in the window; lazy
                        // (Fig. 2b): every synapse, its history always read
                        const uint32_t rec = lazy ? inm : (pot ? (bits & inm) : 0u);
                        const uint32_t sel = arr ? 0u : rec;
                        hm |= sel << (4 * u);
                        am |= (arr ? inm : 0u) << (4 * u);
                        rm |= rec << (4 * u);
                        slots |= o << (8 * u);
                    }
                }
                n_rw += __popc(am) + __popc(hm);     // 8(d): weights read + written (arrival / window hit)
                const unsigned long long tf1 = st.trace ? clock64() : 0ull;
                if (st.trace) dbg_filt += tf1 - tw1;
                // ---- arrivals (every synapse: history window + depression, Fig. 2c):
                //      in place, two chunks (8 synapses) of gathers in flight per lane
                if (__any_sync(0xffffffffu, am != 0u)) {
#pragma unroll 1
                    for (int hf = 0; hf < kStdpChPerThr / 2; hf++) {
                        uint64_t hh[8], hh2[8];
                        float xq[8];
                        uint32_t jv[8];
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const int u = 2 * hf + (q >> 2);
                            const uint32_t bit = 4 * u + (q & 3);
                            const uint32_t on = (am >> bit) & 1u;
                            jv[q] = on ? lds_u32(sa + 16u * (gt + kStdpGroupThr * u) + 4u * (q & 3)) : 0u;
                            hh[q] = ldg_u64_if(ghist + jv[q], on & (rm >> bit));
                            hh2[q] = ldg_u64_if(ghist_hi + jv[q], on & (rm >> bit) & hi_on);
                            xq[q] = ldg_f32_if(gxpost + jv[q], on);
                        }
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const int u = 2 * hf + (q >> 2);
                            const uint32_t bit = 4 * u + (q & 3);
                            if (!((am >> bit) & 1u)) continue;
                            const StdpRow &rr = sm.rows[(slots >> (8 * u)) & 0xffu];
                            const uint32_t meta = rr.meta;
                            const int age = (int)(meta & kMetaAge);
                            const uint32_t si = (meta >> 12) & 0x3u;
                            const float4 pr = sm.par[si];
                            const uint32_t ch = gt + kStdpGroupThr * u;             // chunk in the stage
                            const float w0v = lds_f32(sa + kStdpStageCh * 16 + 16u * ch + 4u * (q & 3));
                            const uint32_t dp = dp_addr + si * 4u * (kMaxHist + 1);
                            const float w = lazy ? stdp_synapse_lazy(w0v, window_lo(hh[q], age), true, xq[q], rr.xp, age,
                                                                     dp, pr.x, pr.y, pr.z, window_hi(hh2[q], age))
                                                 : stdp_synapse(w0v, window_lo(hh[q], age), true, xq[q], rr.xp, age,
                                                                dp, pr.x, pr.y, pr.z, window_hi(hh2[q], age));   // (tlu, t], R2
                            const uint32_t chg = __float_as_uint(w) != __float_as_uint(w0v) ? 1u : 0u;
                            const int64_t off = rr.cb + 4ll * ((int64_t)(a + ch) - (int64_t)rr.first) + (q & 3);
                            stg_f32_if(gw + off, w, chg);
                            n_w += chg;
                        }
                    }
                }
                const unsigned long long ta1 = st.trace ? clock64() : 0ull;
                if (st.trace) dbg_arr += ta1 - tf1;
                if constexpr (kGeneric) {
                    // ---- list the selected synapses (warp-exclusive prefix of the counts)
                    const uint32_t k = __popc(hm);
                    uint32_t ex = k;
    #pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, ex, d);
                        if (lane >= (uint32_t)d) ex += y;
                    }
                    const uint32_t ntot = __shfl_sync(0xffffffffu, ex, 31);
                    ex -= k;
                    for (uint32_t base = 0; base < ntot; base += kStdpList) {
                    uint32_t n = ntot - base < kStdpList ? ntot - base : kStdpList;
                    {
                        uint32_t m = hm, e = ex;
                        while (m) {
                            const uint32_t bpos = __ffs(m) - 1u;
                            m &= m - 1u;
                            const uint32_t u = bpos >> 2;
                            const uint32_t p = 4u * (gt + kStdpGroupThr * u) + (bpos & 3u);     // element in the stage
                            if (e - base < kStdpList)
                                sts_u32(list_a + 4u * (e - base),
                                        (p << 9) | (((rm >> bpos) & 1u) << 8) | ((slots >> (8 * u)) & 0xffu));
                            e++;
                        }
                    }
                    __syncwarp();
                    // ---- drain the list, four entries per lane in flight
                    for (uint32_t b = 0; b < n; b += 128) {
                        uint32_t ent[4];
                        uint32_t jv[4];
                        float wv[4];
                        uint64_t hh[4], hh2[4];
                        float xq[4];
    #pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const uint32_t q = b + 32 * u + lane;
                            const bool ok = q < n;
                            ent[u] = ok ? lds_u32(list_a + 4u * q) : 0u;
                            const uint32_t p = ent[u] >> 9;
                            jv[u] = lds_u32(sa + 4u * p);
                            wv[u] = lds_f32(sa + kStdpStageCh * 16 + 4u * p);
                            const bool arr = ok && (sm.rows[ent[u] & 0xffu].meta & kMetaArr) != 0;
                            hh[u] = ldg_u64_if(ghist + jv[u], ok && ((ent[u] >> 8) & 1u) ? 1u : 0u);
                            hh2[u] = ldg_u64_if(ghist_hi + jv[u], ok && ((ent[u] >> 8) & 1u) ? hi_on : 0u);
                            xq[u] = ldg_f32_if(gxpost + jv[u], arr ? 1u : 0u);
                        }
    #pragma unroll
                        for (int u = 0; u < 4; u++) {
                            if (b + 32 * u + lane >= n) continue;
                            const StdpRow &rr = sm.rows[ent[u] & 0xffu];
                            const uint32_t meta = rr.meta;
                            const bool arr = (meta & kMetaArr) != 0;
                            const int age = (int)(meta & kMetaAge);
                            const uint32_t si = (meta >> 12) & 0x3u;
                            const float4 pr = sm.par[si];
                            const uint32_t dp = dp_addr + si * 4u * (kMaxHist + 1);
                            const float w = lazy ? stdp_synapse_lazy(wv[u], window_lo(hh[u], age), arr, xq[u], rr.xp, age,
                                                                     dp, pr.x, pr.y, pr.z, window_hi(hh2[u], age))
                                                 : stdp_synapse(wv[u], window_lo(hh[u], age), arr, xq[u], rr.xp, age,
                                                                dp, pr.x, pr.y, pr.z, window_hi(hh2[u], age));   // (tlu, t], R2
                            const uint32_t chg = __float_as_uint(w) != __float_as_uint(wv[u]) ? 1u : 0u;
                            const int64_t off = rr.cb + 4ll * ((int64_t)a - (int64_t)rr.first) + (ent[u] >> 9);
                            stg_f32_if(gw + off, w, chg);
                            n_w += chg;
                        }
                    }
                    __syncwarp();                              // list reused by the next pass
                    }
                }
                if (st.trace) dbg_busy += clock64() - tw1;
                if (lane == 0) mbar_arrive(empty_a + 8 * slot);   // stage and list free
            }
        }
        g0 += nst;
        __syncthreads();                           // row table reused next round
    }
    if (threadIdx.x == 0 && !bm_ready) mbar_wait(bmap_a, 0);   // (no rows) the bitmap copy has landed
    n_syn = __reduce_add_sync(0xffffffffu, n_syn);
    n_w = __reduce_add_sync(0xffffffffu, n_w);
    n_rw = __reduce_add_sync(0xffffffffu, n_rw);
    if (lane == 0) {
        if (n_syn) atomicAdd(&st.ctr->metric[3], (unsigned long long)n_syn);
        if (n_w) atomicAdd(&st.ctr->metric[4], (unsigned long long)n_w);
        if (n_rw) atomicAdd(&st.ctr->metric[8], (unsigned long long)n_rw);
    }
    if (st.trace && !readout && lane == 0 && (warp == 0 || warp == kStdpConsWarps)) {
        // debug: consumer warp 0 / the producer: cycles waiting on full / empty
        // stages, cycles busy on stages, stages, time of the first stage
        unsigned long long *tr = st.trace + ((size_t)3 * kTraceCtas + blockIdx.x) * 4;
        if (warp == 0) { tr[0] = dbg_wait; tr[1] = dbg_busy; tr[2] = dbg_n; tr[3] = dbg_first; }
        else st.trace[((size_t)3 * kTraceCtas + 2048 + blockIdx.x) * 4] = dbg_wait;
        if (warp == 0) { st.trace[((size_t)3 * kTraceCtas + 1024 + blockIdx.x) * 4] = dbg_filt;
                         st.trace[((size_t)3 * kTraceCtas + 1024 + blockIdx.x) * 4 + 1] = dbg_arr; }
    }
    if (!readout) {
        __syncthreads();
        trace_mark(st.trace, 1, 3);
        kspan_end(st.kspan, t, 1);
    }
}

// --------------------------------------------------------------- k_stdp_ev
// Lazy + event-driven STDP of the event schedule (Fig. 2c) over the
// step's visited plastic rows: the plastic arrivals A(t) and the forced flushes
// F(t) (R3).
//  * kMode 2 (k_flush, the ahead step, engine.cu): the forced flushes of t,
//    after k_deliver(t) -- which ran the plastic arrivals' STDP itself
//    (deliver_stdp) -- so that k_deliver(t) follows k_front(t) directly.  It
//    reads step t's tables (fpos / fpot / recent: four buffers by t & 3; lists
//    by t & 7) and no delivery of t reads a flushed row (a forced flush is a
//    row that does not arrive at t).
//  * kMode 0: both kinds between k_front(t) and k_deliver(t) (the step without
//    the ahead list: D < 2).
// Both stream their share of the rows' plastic spans as 16-byte chunks (4
// synapses): thread x takes chunks x + kT u, coalesced 16-byte loads of ids and
// weights, the next iteration's loads issued before the current one's gathers.
// A synapse i -> j is filtered by the bit of j in the shared-memory copy of the
// `recent` bitmap (j fired in the last H steps); only then is the one-byte
// spike position fpos[j] gathered (0xff: several spikes) -- the paper's regime
// has 0-1 post spikes per window:
//  * forced flush (age H): every flush of the step shares the window
//    (t - H, t], so w = min(w + A+ (x_pre_i D+[H - p]), w_max) for j's one
//    spike at bit p (the closed-form skip-ahead of P:284); several spikes: by
//    the gathered fpot[j] = sum of D+[H - s] (potentiations only, so the
//    sequential clamps are one clamp of the sum);
//  * arrival: potentiation by the spikes in the window (tlu, t] (one: p < age;
//    several: the gathered history, oldest first with __clz), then the
//    pre spike's depression by x_post[j] (gathered).
// Only weights that change are stored.
#ifndef SNN_FL_GRID
#define SNN_FL_GRID 1        // k_flush CTAs per SM
#endif
constexpr int kEvRowsMax = 256;              // row table per round
constexpr int kEvU = 2;                      // chunks per thread and iteration

struct __align__(16) EvRow {
    int64_t cb;      // 16-byte aligned CSR offset of the plastic span
    uint32_t lo, hi; // valid elements [lo, hi) relative to cb
    float xp;        // x_pre at tlu
    uint32_t meta;   // age, arrival bit, STDP projection (RowDesc::meta)
    uint32_t first;  // flattened index of its first chunk
    uint32_t pad;
};
struct EvSmem {
    uint64_t bmap;                   // mbarrier of the bitmap's bulk copy
    EvRow rows[kEvRowsMax];
    uint32_t incl[kEvRowsMax + 1];   // inclusive prefix of the rows' chunk counts
    uint32_t wsum[32];
    float4 par[4];                   // per projection: a_plus, a_minus, w_max
    float dplus[4 * (kMaxHist + 1)];
};

// bitmap words [pp_lo / 128 * 4, ceil(pp_hi / 32)): 16-byte aligned, whole 16-byte units
__host__ __device__ inline uint32_t ev_bm_lo(uint32_t pp_lo) { return (pp_lo >> 7) << 2; }
__host__ __device__ inline uint32_t ev_bm_bytes(uint32_t pp_lo, uint32_t pp_hi) {
    return 16u * ((((pp_hi + 31) >> 5) - ev_bm_lo(pp_lo) + 3) >> 2);
}
size_t ev_smem_bytes(uint32_t pp_lo, uint32_t pp_hi) {
    return ((sizeof(EvSmem) + 15) & ~(size_t)15) + ev_bm_bytes(pp_lo, pp_hi);
}

// One iteration's loads: chunk c (c < T) of the CTA's flattened rows; r walks
// forward (a thread's chunks increase).
struct EvLoad {
    uint4 j, w;
    uint32_t r, x0;   // row slot, element offset of the chunk in the row (rel. cb)
};

__device__ __forceinline__ void ev_load(const EvSmem &sm, const uint32_t *__restrict__ idx,
                                        const float *__restrict__ w, uint32_t c, uint32_t T, uint32_t &cur,
                                        EvLoad &L) {
    if (c < T) {
        while (c >= sm.incl[cur]) cur++;
        const EvRow &er = sm.rows[cur];
        L.r = cur;
        L.x0 = 4u * (c - er.first);
        const int64_t off = er.cb + L.x0;
        L.j = __ldg(reinterpret_cast<const uint4 *>(idx + off));
        L.w = __ldg(reinterpret_cast<const uint4 *>(w + off));
    } else {
        L.r = 0xffffffffu;
        L.x0 = 0;
        L.j = make_uint4(0, 0, 0, 0);
        L.w = make_uint4(0, 0, 0, 0);
    }
}

// A flush of age < H whose target fired several times in the H window: the
// window's spikes from the history word (potentiation only, no pre spike).
template <bool kH128>
__device__ __noinline__ float flush_hist(const uint64_t *hist, const uint64_t *hist_hi, uint32_t j, float w, float xp,
                                         uint32_t age, uint32_t dp, float4 pr) {
    return stdp_synapse(w, window_lo(__ldg(hist + j), (int)age), false, 0.0f, xp, (int)age, dp, pr.x, pr.y, pr.z,
                        kH128 ? window_hi(__ldg(hist_hi + j), (int)age) : 0ull);
}

// Per-iteration counters (metrics, 8(d) bytes).
struct EvCount {
    uint32_t syn = 0, fsyn = 0, w = 0, rw = 0, frw = 0;
};

// The U chunks of one iteration, in phases so that each phase's gathers of all
// U x 4 synapses are in flight together: (1) span mask and bitmap filter, (2)
// fpos (+ x_post for arrivals), (3) fpot / history where several spikes, (4)
// the updates and the stores of changed weights.
template <bool kH128, int U, bool kArr, bool kFl>
__device__ __forceinline__ void ev_process(const EvSmem &sm, const StateDev &st, const EvLoad (&L)[U],
                                           uint32_t bm_addr, const uint8_t *__restrict__ fpos,
                                           const float *__restrict__ fpot, uint32_t dp_addr, uint32_t H,
                                           EvCount &n) {
    uint32_t inm[U], hm[U];
    bool arr[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        inm[u] = 0;
        hm[u] = 0;
        arr[u] = false;
        if (L[u].r == 0xffffffffu) continue;
        const EvRow &er = sm.rows[L[u].r];
        arr[u] = kArr && (!kFl || (er.meta & kMetaArr) != 0);
        uint32_t m = 0xfu;
        if (L[u].x0 < er.lo || L[u].x0 + 4 > er.hi) {                // a row's first / last chunk
            m = 0;
#pragma unroll
            for (int e = 0; e < 4; e++) m |= (uint32_t)(L[u].x0 + e >= er.lo && L[u].x0 + e < er.hi) << e;
        }
        inm[u] = m;
        const uint32_t jj[4] = {L[u].j.x, L[u].j.y, L[u].j.z, L[u].j.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {       // (outside the span: a neighbour's target, maybe no post neuron)
            const uint32_t j = ((m >> e) & 1u) ? jj[e] : (bm_addr & 0u);
            const uint32_t bit = ((m >> e) & 1u) ? (lds_u32(bm_addr + ((j >> 5) << 2)) >> (j & 31)) & 1u : 0u;
            hm[u] |= bit << e;
        }
        n.rw += __popc(arr[u] ? m : hm[u]);
        if (!arr[u]) n.frw += __popc(hm[u]);
    }
    uint32_t pos[U][4];
    float xq[U][4];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint32_t jj[4] = {L[u].j.x, L[u].j.y, L[u].j.z, L[u].j.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            pos[u][e] = ldg_u8_if(fpos + jj[e], (hm[u] >> e) & 1u);          // 0xff where not gathered
            xq[u][e] = kArr ? ldg_f32_if(st.xpost + jj[e], arr[u] ? (inm[u] >> e) & 1u : 0u) : 0.0f;
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        if (!inm[u]) continue;
        const EvRow &er = sm.rows[L[u].r];
        const uint32_t si = (er.meta >> 12) & 0x3u;
        const float4 pr = sm.par[si];
        const uint32_t dp = dp_addr + si * 4u * (kMaxHist + 1);
        const uint32_t jj[4] = {L[u].j.x, L[u].j.y, L[u].j.z, L[u].j.w};
        const float wv[4] = {__uint_as_float(L[u].w.x), __uint_as_float(L[u].w.y), __uint_as_float(L[u].w.z),
                             __uint_as_float(L[u].w.w)};
        float *wp = st.w + er.cb + L[u].x0;
        if (kFl && !arr[u]) {
            // ---- forced flush (age H, or H - 1 when flushed a step early,
            //      k_front): the window's spike at bit p < age adds
            //      A+ (x_pre D+[age - p]); several spikes at age H: the fpot
            //      factor (gathered); several at age H - 1: the history word
            if (!hm[u]) continue;
            const uint32_t age = er.meta & kMetaAge;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const bool hit = (hm[u] >> e) & 1u;
                const uint32_t p = pos[u][e];
                float w = wv[e];
                if (hit && (p < age || (p == 0xffu && age == H))) {
                    const float f = p < age ? lds_f32(dp + 4u * (age - p)) : __ldg(fpot + jj[e]);
                    const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(er.xp, f)));
                    w = nw < pr.z ? nw : pr.z;
                } else if (hit && p == 0xffu) {
                    w = flush_hist<kH128>(st.hist, st.hist_hi, jj[e], w, er.xp, age, dp, pr);
                }
                const uint32_t chg = (hit && __float_as_uint(w) != __float_as_uint(wv[e])) ? 1u : 0u;
                stg_f32_if(wp + e, w, chg);
                n.w += chg;
            }
        } else if (kArr) {
            // ---- arrival (Fig. 2c): every synapse.  Potentiation by the spikes
            //      in the window (tlu, t] (one: bit p < age, closed form; several:
            //      the history word, oldest first with __clz), then the pre spike's
            //      depression by x_post[j]
            const uint32_t age = er.meta & kMetaAge;
#pragma unroll
            for (int e = 0; e < 4; e++) {
                if (!((inm[u] >> e) & 1u)) continue;
                float w = wv[e];
                const uint32_t p = ((hm[u] >> e) & 1u) ? pos[u][e] : 0xfeu;
                if (p == 0xffu) {
                    w = stdp_synapse(w, window_lo(__ldg(st.hist + jj[e]), (int)age), true, xq[u][e], er.xp, (int)age,
                                     dp, pr.x, pr.y, pr.z,
                                     kH128 ? window_hi(__ldg(st.hist_hi + jj[e]), (int)age) : 0ull);
                } else {
                    if (p < age) {                     // the window's only post spike
                        const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(er.xp, lds_f32(dp + 4u * (age - p)))));
                        w = nw < pr.z ? nw : pr.z;
                    }
                    const float dw = __fsub_rn(w, __fmul_rn(pr.y, xq[u][e]));
                    w = dw > 0.0f ? dw : 0.0f;
                }
                const uint32_t chg = __float_as_uint(w) != __float_as_uint(wv[e]) ? 1u : 0u;
                stg_f32_if(wp + e, w, chg);
                n.w += chg;
            }
        }
    }
}

// The CTA's rows -- [0, nAb) from the front of the visit list at a_begin, then
// nFb from its back at f_back downwards -- flattened into one chunk stream, in
// rounds of kRows rows.  The bitmap copy (mbarrier bmap_a) is awaited once,
// after the first round's table.
template <bool kH128, int kT, int kMode>
__device__ __forceinline__ void ev_rows(EvSmem &sm, const StateDev &st, const RowDesc *Vl, uint32_t a_begin,
                                        uint32_t nAb, size_t f_back, uint32_t r_end, uint32_t bm_addr,
                                        uint32_t bmap_a, const uint8_t *fpos, const float *fpot, uint32_t dp_addr,
                                        uint32_t H, EvCount &n) {
    constexpr int kRows = kT < kEvRowsMax ? kT : kEvRowsMax;
    bool bm_ready = false;
    for (uint32_t r0 = 0; r0 < r_end; r0 += kRows) {
        const uint32_t nrows = min(r_end - r0, (uint32_t)kRows);
        uint32_t nch = 0;
        EvRow er;
        if (threadIdx.x < nrows) {
            const uint32_t r = r0 + threadIdx.x;
            const RowDesc d = Vl[r < nAb ? (size_t)(a_begin + r) : f_back - (r - nAb)];
            const bool arr = (d.meta & kMetaArr) != 0;
            const int64_t cs = d.start + d.s0, ce = d.start + d.s1;
            er.cb = cs & ~3ll;
            er.lo = (uint32_t)(cs - er.cb);
            er.hi = (uint32_t)(ce - er.cb);
            er.xp = d.xp;
            er.meta = d.meta;
            er.pad = 0;
            // a flush with x_pre == 0 changes no weight (potentiation adds A+ 0, R31)
            if (cs < ce && (arr || d.xp != 0.0f)) {
                nch = (er.hi + 3) >> 2;
                n.syn += (uint32_t)(ce - cs);
                if (!arr) n.fsyn += (uint32_t)(ce - cs);
            }
        }
        uint32_t T = 0;
        const uint32_t inc = block_incl_scan<kT>(nch, sm.wsum, T);
        if (threadIdx.x < nrows) {
            er.first = inc - nch;
            sm.rows[threadIdx.x] = er;
            sm.incl[threadIdx.x] = inc;
        }
        if (threadIdx.x == 0) sm.incl[nrows] = 0xffffffffu;      // (the walk never passes the last row)
        __syncthreads();
        if (!bm_ready) {
            mbar_wait(bmap_a, 0);
            bm_ready = true;
        }
        uint32_t cur = 0;
        constexpr bool kArr = kMode != 2, kFl = kMode != 1;
        if constexpr (kMode == 2) {
            // forced flushes (the long stream): the next iteration's loads are
            // issued before the current one's gathers
            EvLoad L[kEvU], Ln[kEvU];
#pragma unroll
            for (int u = 0; u < kEvU; u++) ev_load(sm, st.idx, st.w, kT * u + threadIdx.x, T, cur, L[u]);
            for (uint32_t c0 = 0; c0 < T; c0 += kT * kEvU) {
#pragma unroll
                for (int u = 0; u < kEvU; u++)
                    ev_load(sm, st.idx, st.w, c0 + kT * (kEvU + u) + threadIdx.x, T, cur, Ln[u]);
                ev_process<kH128, kEvU, kArr, kFl>(sm, st, L, bm_addr, fpos, fpot, dp_addr, H, n);
#pragma unroll
                for (int u = 0; u < kEvU; u++) L[u] = Ln[u];
            }
        } else {
            for (uint32_t c0 = 0; c0 < T; c0 += kT * kEvU) {
                EvLoad L[kEvU];
#pragma unroll
                for (int u = 0; u < kEvU; u++) ev_load(sm, st.idx, st.w, c0 + kT * u + threadIdx.x, T, cur, L[u]);
                ev_process<kH128, kEvU, kArr, kFl>(sm, st, L, bm_addr, fpos, fpot, dp_addr, H, n);
            }
        }
        __syncthreads();                           // row table reused next round
    }
    if (!bm_ready && threadIdx.x == 0) mbar_wait(bmap_a, 0);   // (no rows) the copy has landed
}

// kMode: 0 arrivals + forced flushes, 1 arrivals (k_stdp_arr), 2 forced flushes (k_flush)
template <bool kH128, int kMode, int kT>
__global__ void __launch_bounds__(kT, 65536 / (kT * 64))
k_stdp_ev(NetDev net, StateDev st, uint32_t pp_lo, uint32_t pp_hi) {
    extern __shared__ __align__(16) unsigned char smem[];
    const unsigned long long t_entry = st.kspan ? gtimer() : 0ull;
    EvSmem &sm = *reinterpret_cast<EvSmem *>(smem);
    uint32_t *bm_s = reinterpret_cast<uint32_t *>(smem + ((sizeof(EvSmem) + 15) & ~(size_t)15));
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t bmap_a = smem_u32(&sm.bmap);
    // ---- prologue independent of k_front(t): barrier, STDP constants
    if (threadIdx.x == 0) {
        mbar_init(bmap_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (uint32_t x = threadIdx.x; x < net.nstdp * (kMaxHist + 1); x += kT)
        sm.dplus[x] = st.stdp[x / (kMaxHist + 1)].dplus[x % (kMaxHist + 1)];
    if (threadIdx.x < net.nstdp)
        sm.par[threadIdx.x] = make_float4(st.stdp[threadIdx.x].a_plus, st.stdp[threadIdx.x].a_minus,
                                          st.stdp[threadIdx.x].w_max, 0.0f);
    // kMode 0 / 1: after k_front(t); kMode 2 (flushes on a side branch): its
    // step from the flush sequence counter (advanced by its last CTA)
    pdl_wait();            // k_front(t): lists, bitmap, fpos / fpot
    const int64_t t = kMode == 2 ? *(volatile const int64_t *)&st.ctr->tfl : *(volatile const int64_t *)&st.ctr->t;
    pdl_launch();          // the next kernel may start its prologue
    trace_mark(st.trace, kMode == 2 ? 3 : 1, 0);
    if (st.kspan) kspan_begin(st.kspan, t, kMode == 2 ? 3 : 1, t_entry, gtimer());
    const uint32_t par = (uint32_t)(t & 1);
    const uint32_t wlo = ev_bm_lo(pp_lo), bm_bytes = ev_bm_bytes(pp_lo, pp_hi);
    __syncthreads();       // barrier init visible
    if (threadIdx.x == 0) {    // bitmap of recently fired post neurons (one bulk copy)
        mbar_expect_tx(bmap_a, bm_bytes);
        bulk_g2s(smem_u32(bm_s), st.recent + (size_t)(t & 3) * st.rstride + wlo, bm_bytes, bmap_a);
    }
    const RowDesc *Vl = st.vdesc[t & 3];
    const uint32_t *lens = st.ctr->lst[t & 7];
    const uint32_t nA = kMode == 2 ? 0u : lens[0], nF = kMode == 1 ? 0u : lens[2];
    const size_t cap_back = (size_t)st.nblk * kFrontThreads - 1;      // forced flushes: from the back
    const uint32_t a_begin = (uint32_t)(((uint64_t)nA * blockIdx.x) / gridDim.x);
    const uint32_t a_end = (uint32_t)(((uint64_t)nA * (blockIdx.x + 1)) / gridDim.x);
    const uint32_t f_begin = (uint32_t)(((uint64_t)nF * blockIdx.x) / gridDim.x);
    const uint32_t f_end = (uint32_t)(((uint64_t)nF * (blockIdx.x + 1)) / gridDim.x);
    const uint32_t bm_addr = smem_u32(bm_s) - 4u * wlo;          // bitmap word of neuron j: + 4 (j >> 5)
    const uint32_t dp_addr = smem_u32(sm.dplus);
    const uint8_t *fpos = st.fpos + (size_t)(t & 3) * st.fstride;
    const float *fpot = st.fpot + (size_t)(t & 3) * st.fstride;
    EvCount n;
    // (experiments: net.debug 2 = no arrivals, 4 = no flushes)
    const uint32_t nAb = (net.debug & 2u) ? 0u : a_end - a_begin, nFb = (net.debug & 4u) ? 0u : f_end - f_begin;
    ev_rows<kH128, kT, kMode>(sm, st, Vl, a_begin, nAb, cap_back - f_begin, nAb + nFb, bm_addr, bmap_a, fpos, fpot,
                       dp_addr, net.H, n);
    n.syn = __reduce_add_sync(0xffffffffu, n.syn);
    n.w = __reduce_add_sync(0xffffffffu, n.w);
    n.rw = __reduce_add_sync(0xffffffffu, n.rw);
    n.fsyn = __reduce_add_sync(0xffffffffu, n.fsyn);
    n.frw = __reduce_add_sync(0xffffffffu, n.frw);
    if (lane == 0) {
        if (n.syn) atomicAdd(&st.ctr->metric[3], (unsigned long long)n.syn);
        if (n.w) atomicAdd(&st.ctr->metric[4], (unsigned long long)n.w);
        if (n.rw) atomicAdd(&st.ctr->metric[8], (unsigned long long)n.rw);
        if (n.fsyn) atomicAdd(&st.ctr->metric[9], (unsigned long long)n.fsyn);
        if (n.frw) atomicAdd(&st.ctr->metric[10], (unsigned long long)n.frw);
    }
    if (st.trace) {
        __syncthreads();
        trace_mark(st.trace, kMode == 2 ? 3 : 1, 3);
    }
    kspan_end(st.kspan, t, kMode == 2 ? 3 : 1);
    if (kMode == 2) {
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(&st.ctr->fticket, 1u) == gridDim.x - 1) {   // the last CTA: next step
            st.ctr->fticket = 0;
            st.ctr->tfl = t + 1;
        }
    }
}

// ------------------------------------------------------------------ k_flush
// The forced flushes F(t) of the ahead step (R3).  A forced flush changes w_ij
// only where the target j fired in the row's window (0-1 spikes per
// window, most targets none), so the kernel is a stream whose only memory
// round trip is the stream itself: everything a synapse needs besides its id
// and weight is in shared memory --
//  * kStaged: the post population's one-byte spike positions fpos (k_front:
//    0xfe none in the H window, 0xff several, else the bit of the only one),
//    TMA bulk copies (cfg3: 126 KB);
//  * else (a post population too large for shared memory): the `recent`
//    bitmap (1 bit per neuron) and fpos gathered (L2) for the set bits.
// Work unit: a piece = 32 kFlQ 16-byte chunks (128 kFlQ synapses) of one row's
// plastic span; warp w takes the CTA's pieces w, w + 32, ... with the row's
// state in registers; lane l loads chunks l + 32 q (q < kFlQ) -- ids and
// weights, all 2 kFlQ 16-byte loads in flight together (the other warps'
// pieces cover the latency).  A synapse i -> j whose target's only spike is at
// bit p < age (age H, or H - 1 when flushed a step early, k_front's rule)
// becomes w = min(w + A+ (x_pre D+[age - p]), w_max) -- the closed-form
// skip-ahead of P:284 -- stored in place; several spikes: the fpot[j] factor
// (age H: sum of D+[H - s] over them, potentiations only, so the sequential
// clamps are one clamp of the sum) or the history word (age H - 1).
// Its inputs are k_front(t)'s (lists, fpos / fpot / bitmap, the rows' x_pre)
// and no k_deliver(t) access touches a flushed row (a forced flush is a row
// that does not arrive at t, and k_deliver(t) updates only arriving rows), so
// the whole kernel runs before its dependency wait: its CTAs start as
// k_deliver(t)'s retire; the wait at the end only orders k_front(t+1) after
// k_deliver(t) (PDL chain).
// 8(d) bytes: 4 B per visited synapse (its id) + 8 B per hit (weight read and
// written) + 16 B per row.
#ifndef SNN_FL_Q
#define SNN_FL_Q 4
#endif
#ifndef SNN_FL_T
#define SNN_FL_T 1024
#endif
#ifndef SNN_FL_BF
#define SNN_FL_BF 1              // 1: branch-free filter + update (staged table), 0: per-element branches
#endif
#ifndef SNN_FL_STAGED
#define SNN_FL_STAGED 1          // 0: always the bitmap filter (smaller shared memory)
#endif
constexpr int kFlT = SNN_FL_T;
constexpr int kFlWarps = kFlT / 32;
constexpr int kFlRows = 256;
constexpr int kFlQ = SNN_FL_Q;          // chunks per lane and piece
constexpr int kFlPieceCh = 32 * kFlQ;   // chunks per piece
constexpr bool kFlBF = SNN_FL_BF != 0;

struct FlSmem {
    uint64_t bmap;                      // mbarrier of the table's bulk copies
    EvRow rows[kFlRows];                // EvRow::first = the row's first piece
    uint32_t incl[kFlRows + 1];         // inclusive prefix of the rows' piece counts
    uint32_t wsum[kFlWarps];
    float4 par[4];
    float dplus[4 * (kMaxHist + 1)];
    uint4 bnd[kFlRows];                 // (kI16) the row's 2^16 crossings relative to cb (0xffffffff: none)
};

// The row of piece p (warp-uniform): the first r >= cur with incl[r] > p,
// 32 rows per probe (incl[nrows] = 0xffffffff)
__device__ __forceinline__ uint32_t fl_row_of(const uint32_t *incl, uint32_t cur, uint32_t nrows, uint32_t p,
                                              uint32_t lane) {
    for (;;) {
        const uint32_t b = __ballot_sync(0xffffffffu, p >= incl[min(cur + lane, nrows)]);
        cur += __popc(b);
        if (b != 0xffffffffu) return cur;
    }
}

// table: fpos bytes [pp_lo & ~15, pp_hi) (16-byte units), else the bitmap
__host__ __device__ inline uint32_t fl_tab_bytes(uint32_t pp_lo, uint32_t pp_hi, bool staged) {
    return staged ? ((pp_hi - (pp_lo & ~15u) + 15u) & ~15u) : ev_bm_bytes(pp_lo, pp_hi);
}
bool flush_staged(uint32_t pp_lo, uint32_t pp_hi) {
    return SNN_FL_STAGED && ((sizeof(FlSmem) + 15) & ~(size_t)15) + fl_tab_bytes(pp_lo, pp_hi, true) <= 227u * 1024u;
}
size_t flush_smem_bytes(uint32_t pp_lo, uint32_t pp_hi) {
    return ((sizeof(FlSmem) + 15) & ~(size_t)15) + fl_tab_bytes(pp_lo, pp_hi, flush_staged(pp_lo, pp_hi));
}

// kI16 (SNN_FLAG_IDX16, SURVEY 8(f1) on the STDP stream): the ids streamed
// as 16-bit (j - tgt_lo) mod 2^16 (2 instead of 4 B per visited synapse); j is
// rebuilt from the row's crossings of multiples of 2^16 (st.b64, at most four
// inside a plastic span), a chunk = 8 synapses.
template <bool kH128, bool kStaged, bool kI16>
__global__ void __launch_bounds__(kFlT, kFlT >= 1024 ? 1 : 1024 / kFlT)
k_flush(NetDev net, StateDev st, uint32_t pp_lo, uint32_t pp_hi) {
    extern __shared__ __align__(16) unsigned char smem[];
    const unsigned long long t_entry = st.kspan ? gtimer() : 0ull;
    FlSmem &sm = *reinterpret_cast<FlSmem *>(smem);
    unsigned char *tab = smem + ((sizeof(FlSmem) + 15) & ~(size_t)15);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bmap_a = smem_u32(&sm.bmap);
    pdl_launch();          // k_front(t+1) may be scheduled (it waits for this grid)
    // the step of the flushes: k_flush runs once per step, in order (one
    // stream); the previous launch's last CTA advanced the counter
    const int64_t t = *(volatile const int64_t *)&st.ctr->tfl;
    trace_mark(st.trace, 3, 0);
    if (st.kspan) kspan_begin(st.kspan, t, 3, t_entry, t_entry);
    const uint8_t *__restrict__ fpos = st.fpos + (size_t)(t & 3) * st.fstride;
    const float *__restrict__ fpot = st.fpot + (size_t)(t & 3) * st.fstride;
    const uint32_t f_lo = pp_lo & ~15u, wlo = ev_bm_lo(pp_lo);
    const uint32_t tab_bytes = fl_tab_bytes(pp_lo, pp_hi, kStaged);
    if (threadIdx.x == 0) {
        mbar_init(bmap_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(bmap_a, tab_bytes);
        const unsigned char *src = kStaged ? (const unsigned char *)(fpos + f_lo)
                                           : (const unsigned char *)(st.recent + (size_t)(t & 3) * st.rstride + wlo);
        for (uint32_t off = 0; off < tab_bytes; off += 32768u)      // (bulk copies of at most 32 KB)
            bulk_g2s(smem_u32(tab) + off, src + off, min(32768u, tab_bytes - off), bmap_a);
    }
    // (entry 0 of each table is 0: a flush never reads D+[0] (n = age - pos
    // >= 1), so the branch-free update selects it for a target without a
    // spike in the window -- w + A+ (x_pre 0) = w, bit for bit)
    for (uint32_t x = threadIdx.x; x < net.nstdp * (kMaxHist + 1); x += kFlT)
        sm.dplus[x] = (kFlBF && x % (kMaxHist + 1) == 0) ? 0.0f : st.stdp[x / (kMaxHist + 1)].dplus[x % (kMaxHist + 1)];
    if (threadIdx.x < net.nstdp)
        sm.par[threadIdx.x] = make_float4(st.stdp[threadIdx.x].a_plus, st.stdp[threadIdx.x].a_minus,
                                          st.stdp[threadIdx.x].w_max, 0.0f);
    const RowDesc *Vl = st.vdesc[t & 3];
    const uint32_t nF = st.ctr->lst[t & 7][2];
    const size_t cap_back = (size_t)st.nblk * kFrontThreads - 1;      // forced flushes: from the back
    const uint32_t f_begin = (uint32_t)(((uint64_t)nF * blockIdx.x) / gridDim.x);
    const uint32_t f_end = (uint32_t)(((uint64_t)nF * (blockIdx.x + 1)) / gridDim.x);
    // kStaged: fpos of neuron j at + j; else the bitmap word of j at + 4 (j >> 5)
    const uint32_t tab_a = kStaged ? smem_u32(tab) - f_lo : smem_u32(tab) - 4u * wlo;
    const uint32_t dp_addr = smem_u32(sm.dplus);
    const uint32_t *__restrict__ gidx = st.idx;
    float *__restrict__ gw = st.w;
    const uint32_t H = net.H;
    uint32_t n_syn = 0, n_w = 0, n_hit = 0;
    bool tab_ready = false;
    const uint32_t nrows_all = f_end - f_begin;
    for (uint32_t r0 = 0; r0 < nrows_all; r0 += (kFlRows < kFlT ? kFlRows : kFlT)) {
        // ---- row table: plastic spans as pieces (x_pre = 0: no change, R31)
        const uint32_t nrows = min(nrows_all - r0, (uint32_t)(kFlRows < kFlT ? kFlRows : kFlT));
        uint32_t npc = 0;
        EvRow er;
        if (threadIdx.x < nrows) {
            const RowDesc d = Vl[cap_back - (f_begin + r0 + threadIdx.x)];
            const int64_t cs = d.start + d.s0, ce = d.start + d.s1;
            er.cb = kI16 ? cs & ~7ll : cs & ~3ll;
            er.lo = (uint32_t)(cs - er.cb);
            er.hi = (uint32_t)(ce - er.cb);
            er.xp = d.xp;
            er.meta = d.meta;
            er.pad = 0;
            if (cs < ce && d.xp != 0.0f) {
                npc = kI16 ? (((er.hi + 7) >> 3) + 63) / 64 : (((er.hi + 3) >> 2) + kFlPieceCh - 1) / kFlPieceCh;
                n_syn += (uint32_t)(ce - cs);
            }
            if (kI16) {        // the row's 2^16 crossings, relative to cb
                const uint4 b = reinterpret_cast<const uint4 *>(st.b64)[d.row];
                const int64_t off = er.cb - d.start;     // row-relative index of cb (<= s0)
                auto rel = [&](uint32_t v) { return (int64_t)v <= off ? 0u : (uint32_t)((int64_t)v - off); };
                sm.bnd[threadIdx.x] = make_uint4(rel(b.x), rel(b.y), rel(b.z), rel(b.w));
            }
        }
        // (warp-level prefix + one pass over the warp totals)
        uint32_t inc = npc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (lane == 31) sm.wsum[warp] = inc;
        __syncthreads();                             // (also: the barrier's init, the constants)
        uint32_t wpre = 0, P = 0;
        {
            const uint32_t v = lane < (uint32_t)kFlWarps ? sm.wsum[lane] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            wpre = __shfl_sync(0xffffffffu, x - v, warp);
            P = __shfl_sync(0xffffffffu, x, 31);
        }
        inc += wpre;
        if (threadIdx.x < nrows) {
            er.first = inc - npc;
            sm.rows[threadIdx.x] = er;
            sm.incl[threadIdx.x] = inc;
        }
        if (threadIdx.x == 0) sm.incl[nrows] = 0xffffffffu;
        __syncthreads();
        if (!tab_ready) {
            trace_mark(st.trace, 3, 1);
            mbar_wait(bmap_a, 0);
            tab_ready = true;
            trace_mark(st.trace, 3, 2);
        }
        // ---- the warp's pieces: p = warp + 32 i
        uint32_t cur = 0;
        if constexpr (kI16) {
        for (uint32_t p = warp; p < P; p += kFlWarps) {
            cur = fl_row_of(sm.incl, cur, nrows, p, lane);
            const EvRow &rr = sm.rows[cur];
            const uint32_t c0 = (p - rr.first) * 64u;            // chunks of 8 synapses, 64 per piece
            const uint32_t lo = rr.lo, hi = rr.hi, nch = (hi + 7) >> 3;
            const int64_t cb = rr.cb;
            const uint4 bnd = sm.bnd[cur];
            uint4 J[2], Wa[2], Wb[2];
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t c = c0 + lane + 32u * q;
                const bool ok = c < nch;
                J[q] = ok ? __ldg(reinterpret_cast<const uint4 *>(st.idx16 + cb + 8ll * c)) : make_uint4(0, 0, 0, 0);
                Wa[q] = ok ? __ldg(reinterpret_cast<const uint4 *>(gw + cb + 8ll * c)) : make_uint4(0, 0, 0, 0);
                Wb[q] = ok ? __ldg(reinterpret_cast<const uint4 *>(gw + cb + 8ll * c + 4)) : make_uint4(0, 0, 0, 0);
            }
            const uint32_t age = rr.meta & kMetaAge, si = (rr.meta >> 12) & 0x3u;
            const float4 pr = sm.par[si];
            const float xp = rr.xp;
            const uint32_t dp = dp_addr + si * 4u * (kMaxHist + 1);
            if constexpr (kFlBF && kStaged) {      // (the branch-free form of the 32-bit stream's loop)
                const float *__restrict__ fpf = fpot + (size_t)4 * (H - age) * st.fstride;
                float F[2][8];
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    const uint32_t x0 = 8u * (c0 + lane + 32u * q);
                    const uint32_t h0 = (uint32_t)(bnd.x <= x0) + (uint32_t)(bnd.y <= x0) + (uint32_t)(bnd.z <= x0) +
                                        (uint32_t)(bnd.w <= x0);
                    const bool cross = (bnd.x > x0 && bnd.x < x0 + 8) || (bnd.y > x0 && bnd.y < x0 + 8) ||
                                       (bnd.z > x0 && bnd.z < x0 + 8) || (bnd.w > x0 && bnd.w < x0 + 8);
                    const uint32_t vw[4] = {J[q].x, J[q].y, J[q].z, J[q].w};
                    const bool full = __all_sync(0xffffffffu, x0 >= lo && x0 + 8u <= hi);
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const bool in = full || x0 + e - lo < hi - lo;
                        uint32_t hh = h0;
                        if (cross)
                            hh = (uint32_t)(bnd.x <= x0 + e) + (uint32_t)(bnd.y <= x0 + e) + (uint32_t)(bnd.z <= x0 + e) +
                                 (uint32_t)(bnd.w <= x0 + e);
                        const uint32_t v = (vw[e >> 1] >> (16 * (e & 1))) & 0xffffu;
                        const uint32_t j = in ? net.tgt_lo + (hh << 16) + v : pp_lo;
                        const uint32_t p8 = lds_u8(tab_a + j);
                        const uint32_t pos = in ? p8 : 0xfeu;
                        const uint32_t n = pos < age ? age - pos : 0u;
                        const float f1 = lds_f32(dp + 4u * n);
                        const float fm = ldg_f32_idx_if(fpf, j, pos == 0xffu);
                        F[q][e] = pos == 0xffu ? fm : f1;
                    }
                }
#pragma unroll
                for (int q = 0; q < 2; q++) {
                    const uint32_t x0 = 8u * (c0 + lane + 32u * q);
                    const uint32_t wb[8] = {Wa[q].x, Wa[q].y, Wa[q].z, Wa[q].w, Wb[q].x, Wb[q].y, Wb[q].z, Wb[q].w};
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const float w0 = __uint_as_float(wb[e]);
                        const float nw = __fadd_rn(w0, __fmul_rn(pr.x, __fmul_rn(xp, F[q][e])));
                        const float w = nw < pr.z ? nw : pr.z;
                        const bool ch = __float_as_uint(w) != __float_as_uint(w0);
                        stg_f32_if(gw + cb + x0 + e, w, ch);
                        n_w += ch ? 1u : 0u;
                    }
                }
                continue;
            }
#pragma unroll
            for (int q = 0; q < 2; q++) {
                const uint32_t x0 = 8u * (c0 + lane + 32u * q);
                const bool edge = x0 < lo || x0 + 8 > hi;       // a row's first / last chunk (or past it)
                // j = tgt_lo + 2^16 (crossings <= x) + v; per element only if one falls inside the chunk
                const uint32_t h0 = (uint32_t)(bnd.x <= x0) + (uint32_t)(bnd.y <= x0) + (uint32_t)(bnd.z <= x0) +
                                    (uint32_t)(bnd.w <= x0);
                const bool cross = (bnd.x > x0 && bnd.x < x0 + 8) || (bnd.y > x0 && bnd.y < x0 + 8) ||
                                   (bnd.z > x0 && bnd.z < x0 + 8) || (bnd.w > x0 && bnd.w < x0 + 8);
                const uint32_t vw[4] = {J[q].x, J[q].y, J[q].z, J[q].w};
                const uint32_t wb[8] = {Wa[q].x, Wa[q].y, Wa[q].z, Wa[q].w, Wb[q].x, Wb[q].y, Wb[q].z, Wb[q].w};
#pragma unroll
                for (int e = 0; e < 8; e++) {
                    const bool in = !edge || (x0 + e >= lo && x0 + e < hi);
                    uint32_t hh = h0;
                    if (cross)
                        hh = (uint32_t)(bnd.x <= x0 + e) + (uint32_t)(bnd.y <= x0 + e) + (uint32_t)(bnd.z <= x0 + e) +
                             (uint32_t)(bnd.w <= x0 + e);
                    const uint32_t v = (vw[e >> 1] >> (16 * (e & 1))) & 0xffffu;
                    const uint32_t j = in ? net.tgt_lo + (hh << 16) + v : pp_lo;
                    uint32_t pos;
                    if (kStaged) {
                        pos = in ? lds_u8(tab_a + j) : 0xfeu;
                    } else {
                        const uint32_t b = (lds_u32(tab_a + ((j >> 5) << 2)) >> (j & 31)) & 1u;
                        pos = (in && b) ? ldg_u8_if(fpos + j, 1u) : 0xfeu;
                    }
                    const float w0 = __uint_as_float(wb[e]);
                    float w = w0;
                    if (pos < age) {
                        const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(xp, lds_f32(dp + 4u * (age - pos)))));
                        w = nw < pr.z ? nw : pr.z;
                    } else if (pos == 0xffu) {
                        const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(xp, __ldg(fpot + (size_t)4 * (H - age) * st.fstride + j))));
                        w = nw < pr.z ? nw : pr.z;
                    }
                    n_hit += pos != 0xfeu ? 1u : 0u;
                    if (__float_as_uint(w) != __float_as_uint(w0)) {
                        gw[cb + x0 + e] = w;
                        n_w++;
                    }
                }
            }
        }
        } else {
        for (uint32_t p = warp; p < P; p += kFlWarps) {
            cur = fl_row_of(sm.incl, cur, nrows, p, lane);
            const EvRow &rr = sm.rows[cur];
            const uint32_t c0 = (p - rr.first) * kFlPieceCh;
            const uint32_t lo = rr.lo, hi = rr.hi, nch = (hi + 3) >> 2;
            const int64_t cb = rr.cb;
            uint4 J[kFlQ], Wt[kFlQ];
#pragma unroll
            for (int q = 0; q < kFlQ; q++) {
                const uint32_t c = c0 + lane + 32u * q;
                const bool ok = c < nch;
                J[q] = ok ? __ldg(reinterpret_cast<const uint4 *>(gidx + cb + 4ll * c))
                          : make_uint4(pp_lo, pp_lo, pp_lo, pp_lo);
                Wt[q] = ok ? __ldg(reinterpret_cast<const uint4 *>(gw + cb + 4ll * c)) : make_uint4(0, 0, 0, 0);
            }
            const uint32_t age = rr.meta & kMetaAge, si = (rr.meta >> 12) & 0x3u;
            const float4 pr = sm.par[si];
            const float xp = rr.xp;
            const uint32_t dp = dp_addr + si * 4u * (kMaxHist + 1);
            if constexpr (kFlBF && kStaged) {
                // (1) every element's factor f: D+[age - pos] for one spike in the
                // window, the step's flush factor for several (fpot, k_front), 0
                // for none -- no branch; the several-spike loads of the whole
                // piece are issued together
                const float *__restrict__ fpf = fpot + (size_t)4 * (H - age) * st.fstride;
                float F[kFlQ][4];
#pragma unroll
                for (int q = 0; q < kFlQ; q++) {
                    const uint32_t x0 = 4u * (c0 + lane + 32u * q);
                    const uint32_t jj[4] = {J[q].x, J[q].y, J[q].z, J[q].w};
                    // (warp-uniform: no lane holds a span edge -> no per-element bounds)
                    const bool full = __all_sync(0xffffffffu, x0 >= lo && x0 + 4u <= hi);
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const bool in = full || x0 + e - lo < hi - lo;   // inside [lo, hi)
                        const uint32_t j = in ? jj[e] : pp_lo;          // (pp_lo: inside the table)
                        const uint32_t p8 = lds_u8(tab_a + j);
                        const uint32_t pos = in ? p8 : 0xfeu;
                        const uint32_t n = pos < age ? age - pos : 0u;
                        const float f1 = lds_f32(dp + 4u * n);
                        const float fm = ldg_f32_idx_if(fpf, j, pos == 0xffu);
                        F[q][e] = pos == 0xffu ? fm : f1;
                    }
                }
                // (2) w = min(w + A+ (x_pre f), w_max) (= w where f = 0), stored if changed
#pragma unroll
                for (int q = 0; q < kFlQ; q++) {
                    const uint32_t x0 = 4u * (c0 + lane + 32u * q);
                    const uint32_t wb[4] = {Wt[q].x, Wt[q].y, Wt[q].z, Wt[q].w};
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        const float w0 = __uint_as_float(wb[e]);
                        const float nw = __fadd_rn(w0, __fmul_rn(pr.x, __fmul_rn(xp, F[q][e])));
                        const float w = nw < pr.z ? nw : pr.z;
                        const bool ch = __float_as_uint(w) != __float_as_uint(w0);
                        stg_f32_if(gw + cb + x0 + e, w, ch);
                        n_w += ch ? 1u : 0u;
                    }
                }
                continue;
            }
#pragma unroll
            for (int q = 0; q < kFlQ; q++) {
                const uint32_t x0 = 4u * (c0 + lane + 32u * q);
                const bool edge = x0 < lo || x0 + 4 > hi;       // a row's first / last chunk (or past it)
                const uint32_t jj[4] = {J[q].x, J[q].y, J[q].z, J[q].w};
                const uint32_t wb[4] = {Wt[q].x, Wt[q].y, Wt[q].z, Wt[q].w};
#pragma unroll
                for (int e = 0; e < 4; e++) {
                    // (outside the span: a neighbour's target, maybe outside the table)
                    const bool in = !edge || (x0 + e >= lo && x0 + e < hi);
                    const uint32_t j = in ? jj[e] : pp_lo;
                    uint32_t pos;
                    if (kStaged) {
                        pos = in ? lds_u8(tab_a + j) : 0xfeu;
                    } else {
                        const uint32_t b = (lds_u32(tab_a + ((j >> 5) << 2)) >> (j & 31)) & 1u;
                        pos = (in && b) ? ldg_u8_if(fpos + j, 1u) : 0xfeu;
                    }
                    const float w0 = __uint_as_float(wb[e]);
                    float w = w0;
                    if (pos < age) {
                        const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(xp, lds_f32(dp + 4u * (age - pos)))));
                        w = nw < pr.z ? nw : pr.z;
                    } else if (pos == 0xffu) {
                        // several spikes: the step's factor for age H or H - 1 (k_front)
                        const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(xp, __ldg(fpot + (size_t)4 * (H - age) * st.fstride + j))));
                        w = nw < pr.z ? nw : pr.z;
                    }
                    n_hit += pos != 0xfeu ? 1u : 0u;
                    if (__float_as_uint(w) != __float_as_uint(w0)) {
                        gw[cb + x0 + e] = w;
                        n_w++;
                    }
                }
            }
        }
        }                                          // (the 32-bit id stream)
        __syncthreads();                           // row table reused next round
    }
    if (!tab_ready && threadIdx.x == 0) mbar_wait(bmap_a, 0);   // (no rows) the copy has landed
    // (the branch-free stream counts no window hits separately: a hit changes
    // its weight unless it is already at w_max, so the weights read and
    // written there are counted by the stores)
    n_hit = __reduce_add_sync(0xffffffffu, (kFlBF && kStaged) ? n_w : n_hit);
    n_syn = __reduce_add_sync(0xffffffffu, n_syn);
    n_w = __reduce_add_sync(0xffffffffu, n_w);
    if (lane == 0) {
        if (n_syn) {
            atomicAdd(&st.ctr->metric[3], (unsigned long long)n_syn);
            atomicAdd(&st.ctr->metric[9], (unsigned long long)n_syn);
        }
        if (n_w) {
            atomicAdd(&st.ctr->metric[4], (unsigned long long)n_w);
            atomicAdd(&st.ctr->metric[11], (unsigned long long)n_w);
        }
        if (n_hit) {
            atomicAdd(&st.ctr->metric[8], (unsigned long long)n_hit);
            atomicAdd(&st.ctr->metric[10], (unsigned long long)n_hit);
        }
    }
    pdl_wait();            // k_deliver(t) complete: k_front(t+1), which waits for this grid, reads its inputs
    if (st.trace) {
        __syncthreads();
        trace_mark(st.trace, 3, 3);
    }
    kspan_end(st.kspan, t, 3);
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&st.ctr->fticket, 1u) == gridDim.x - 1) {   // the last CTA: next step
        st.ctr->fticket = 0;
        st.ctr->tfl = t + 1;
    }
}

// --------------------------------------------------------------- k_deliver
constexpr int kDelThreads = 512;
constexpr int kDelWarps = kDelThreads / 32;
constexpr int kDelRows = 1024;     // row table per round (two rows per thread)
constexpr int kDelWin = 32 * kDelThreads;   // flattened elements per owner window (one bitmap word per thread)
#ifndef SNN_DEL_U
#define SNN_DEL_U 3
#endif
#ifndef SNN_DEL_MINB
#define SNN_DEL_MINB 2
#endif
constexpr int kDelU = SNN_DEL_U;   // elements in flight per thread
#ifndef SNN_DEL_PRE
#define SNN_DEL_PRE 1              // kAhead: the static segments delivered before the dependency wait
#endif


// Block-wide inclusive scan of a packed pair (low 32 bits: elements, high 32:
// segments) per thread.
__device__ __forceinline__ unsigned long long block_incl_scan64(unsigned long long v, unsigned long long *wsum,
                                                                unsigned long long &total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned long long off = 0, tot = 0;
#pragma unroll
    for (int w2 = 0; w2 < kDelWarps; w2++) {
        const unsigned long long x = wsum[w2];
        if (w2 < (int)warp) off += x;
        tot += x;
    }
    total = tot;
    return off + inc;
}

// Delivery helpers: 32-bit shared addresses, read-only global loads.
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint64_t lds_u64(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void red_shared_add(uint32_t addr, int32_t v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ldg_nc_u32(uint64_t a) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
}
__device__ __forceinline__ float ldg_nc_f32(uint64_t a) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(a));
    return v;
}

// Plastic arrivals inside the delivery (kPl, the split step graph): the
// (row, slice) segment's plastic part [pl.x, pl.y) (flattened) is updated by
// Fig. 2c before it is delivered (plasticity before delivery) -- its
// window (tlu, t] from the target's one-byte spike position (0xff: several
// spikes -> the history word, oldest first with __clz), then the pre
// spike's depression by x_post[j]; the slice's x_post / fpos are staged in
// shared memory.  The changed weight is stored and the new one delivered.
// Per-segment STDP tables of k_deliver (namespace-scope shared memory: fixed
// addresses, no registers to hold them)
__shared__ uint2 g_del_pl[kDelRows];            // segment g: plastic part, flattened [x, y)
__shared__ uint2 g_del_row[kDelRows];           // segment g: (x_pre at tlu, meta: age, projection)
__shared__ float g_del_dp[4 * (kMaxHist + 1)];  // D+ tables
__shared__ float4 g_del_par[4];                 // per projection: a_plus, a_minus, w_max
struct DelStdp {
    uint32_t xq_a;             // shared, by slice offset jl = j - slo: x_post (f32) at + 4 jl, the history
                               // words at + 4 C + 8 jl (bits 64..127 at + 12 C + 8 jl, H = 128), the
                               // spike positions (u8) at + fp_off + jl
    uint32_t n_syn, n_w;       // metrics
};
template <bool kH128>
__host__ __device__ constexpr uint32_t del_fpos_off(uint32_t C) { return 4u * C + (kH128 ? 16u : 8u) * C; }

// (several post spikes in the H window: rare in the paper's regime, P:399;
// the slice's history words are staged in shared memory)
template <bool kH128>
__device__ __noinline__ float deliver_stdp_hist(uint32_t h_a, uint32_t C, float w, float xq, float xp, uint32_t age,
                                                uint32_t dp, float4 pr) {
    return stdp_synapse(w, window_lo(lds_u64(h_a), (int)age), true, xq, xp, (int)age, dp, pr.x, pr.y, pr.z,
                        kH128 ? window_hi(lds_u64(h_a + 8u * C), (int)age) : 0ull);
}

template <bool kH128>
__device__ __forceinline__ float deliver_stdp(const StateDev &st, uint32_t xq_a, uint32_t C, uint32_t jl, uint32_t j,
                                              float w0, uint32_t g) {
    const uint2 rw = g_del_row[g];                         // (x_pre bits, meta)
    const float xp = __uint_as_float(rw.x);
    const uint32_t age = rw.y & kMetaAge, si = (rw.y >> 12) & 0x3u;
    const uint32_t pos = lds_u8(xq_a + del_fpos_off<kH128>(C) + jl);
    const float xq = lds_f32(xq_a + 4u * jl);
    const uint32_t dp = smem_u32(g_del_dp) + si * 4u * (kMaxHist + 1);
    const float4 pr = g_del_par[si];
    float w = w0;
    if (pos == 0xffu) {
        w = deliver_stdp_hist<kH128>(xq_a + 4u * C + 8u * jl, C, w, xq, xp, age, dp, pr);
    } else {
        if (pos < age) {                     // the window's only post spike (0xfe: none)
            const float nw = __fadd_rn(w, __fmul_rn(pr.x, __fmul_rn(xp, lds_f32(dp + 4u * (age - pos)))));
            w = nw < pr.z ? nw : pr.z;
        }
        const float dw = __fsub_rn(w, __fmul_rn(pr.y, xq));
        w = dw > 0.0f ? dw : 0.0f;
    }
    return w;
}

// Owner-window pass (k_deliver): thread x takes elements w0 + x + 512 u of the
// window.  Segment of element x: bw.y + popc(start bits <= x) (s_bw word).
// s_ptr holds per segment the byte address of idx[c] for flattened element 0.
__device__ __forceinline__ uint32_t ldg_nc_u16(uint64_t a) {
    uint16_t v;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(a));
    return v;
}

// kIdx16 (SNN_FLAG_IDX16): s_ptr addresses the 16-bit
// slice-local offsets (2 B per element, the weight at 2 a + dw) and the target
// is already local to the slice; else the 32-bit ids (4 B, weight at a + dw).
template <bool kMulti, bool kCheck, bool kIdx16, bool kPl, bool kH128>
__device__ __forceinline__ void deliver_pass(const NetDev &net, const StateDev &st, uint32_t x0, uint32_t wlen,
                                             uint32_t w0, uint32_t bw_a, uint32_t ptr_a, uint32_t rc_a,
                                             uint32_t acc_a, uint64_t dw, float scale, uint32_t slo, DelStdp &ps) {
    uint32_t jj[kDelU], rr[kDelU], gg[kDelU];
    float ww[kDelU];
    const uint32_t slo16 = (slo - net.tgt_lo) & 0xffffu;   // (kIdx16: the slice's first offset mod 2^16)
#pragma unroll
    for (int u = 0; u < kDelU; u++) {
        // ragged pass: a thread past the end re-reads the last element (no
        // branch around the loads, so they stay in flight together) and skips
        // its atomic below
        const uint32_t x = kCheck ? min(x0 + u * kDelThreads + threadIdx.x, wlen - 1u)
                                  : x0 + u * kDelThreads + threadIdx.x;
        const uint2 bw = lds_u2(bw_a + ((x >> 5) << 3));
        const uint32_t gi = bw.y + __popc(bw.x & (0xffffffffu >> (31u - (x & 31u))));
        gg[u] = gi;
        if (kIdx16) {
            const uint64_t a = lds_u64(ptr_a + (gi << 3)) + 2ull * (w0 + x);
            jj[u] = (ldg_nc_u16(a) - slo16) & 0xffffu;          // the slice offset j - slo
            ww[u] = ldg_nc_f32(2ull * a + dw);
        } else {
            const uint64_t a = lds_u64(ptr_a + (gi << 3)) + 4ull * (w0 + x);
            jj[u] = ldg_nc_u32(a);
            ww[u] = ldg_nc_f32(a + dw);
        }
        rr[u] = kMulti ? lds_u8(rc_a + gi) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kDelU; u++) {
        const uint32_t x = x0 + u * kDelThreads + threadIdx.x;
        if (!kCheck || x < wlen) {
            uint32_t r2 = rr[u];
            float wv = ww[u];
            if (kPl) {
                const uint2 pl = g_del_pl[gg[u]];
                if (w0 + x >= pl.x && w0 + x < pl.y) {
                    const uint32_t jl = kIdx16 ? jj[u] : jj[u] - slo;
                    const float wn = deliver_stdp<kH128>(st, ps.xq_a, net.C, jl, slo + jl, wv, gg[u]);
                    ps.n_syn++;
                    if (__float_as_uint(wn) != __float_as_uint(wv)) {
                        const uint64_t a = lds_u64(ptr_a + (gg[u] << 3));
                        float *wp = reinterpret_cast<float *>(kIdx16 ? 2ull * (a + 2ull * (w0 + x)) + dw
                                                                     : a + 4ull * (w0 + x) + dw);
                        *wp = wn;
                        ps.n_w++;
                        wv = wn;
                    }
                }
            }
            if (kMulti && r2 >= 3u) r2 = (uint32_t)net.rcpt[r2 >> 2][find_pop(net, kIdx16 ? slo + jj[u] : jj[u])];
            red_shared_add(acc_a + ((r2 * net.C + jj[u]) << 2), __float2int_rn(__fmul_rn(wv, scale)));
        }
    }
}

template <bool kMulti, bool kIdx16, bool kPl, bool kH128>
__device__ __forceinline__ void deliver_window(const NetDev &net, const StateDev &st, uint32_t xa, uint32_t wlen,
                                               uint32_t w0, uint32_t bw_a, uint32_t ptr_a, uint32_t rc_a, uint32_t acc_a,
                                               uint64_t dw, float scale, uint32_t slo, DelStdp &ps) {
    for (uint32_t x0 = xa; x0 < wlen; x0 += kDelThreads * kDelU) {      // (window elements [xa, wlen))
        if (x0 + kDelThreads * kDelU <= wlen)
            deliver_pass<kMulti, false, kIdx16, kPl, kH128>(net, st, x0, wlen, w0, bw_a, ptr_a, rc_a, acc_a, dw,
                                                            scale, slo, ps);
        else
            deliver_pass<kMulti, true, kIdx16, kPl, kH128>(net, st, x0, wlen, w0, bw_a, ptr_a, rc_a, acc_a, dw,
                                                           scale, slo, ps);
    }
}

// k_deliver's dependency wait: kAhead, k_front(t) (x_post, histories; inputs
// consumed); else k_stdp(t) (or k_front(t), already waited)
__device__ __forceinline__ void del_wait(const StateDev &st, unsigned long long &t_wait) {
    pdl_wait();
    pdl_launch();
    if (st.kspan) t_wait = gtimer();
    trace_mark(st.trace, 2, 1);
}

// One CTA per (slice k, split s) (Fig. 3b).  The CTA tabulates the
// non-empty (row, slice) segments of its share of the arriving rows
// (descriptor + pivot pair) in shared memory and concatenates them into
// one flattened element range.  A bitmap marks the first element of every
// segment, so the segment of element e is a popcount (no search, no loop);
// the threads then stride the range 512 wide -- consecutive threads read
// consecutive synapses -- and each element adds q(w) = RNE(w 2^F) to the slice
// accumulator with a shared atomic.
// kMulti: two receptor accumulators (a receptor code per segment); kIdx16:
// SNN_FLAG_IDX16; kAhead: the arrival list of step t was written by
// k_front(t-1) (D >= 2), so the CTA tabulates it while k_front(t) still runs
// and waits for k_front(t) only before the elements; with STDP it also runs the
// plastic arrivals' update (kPl = kAhead && STDP, see deliver_stdp) --
// compile-time variants, so a kernel carries only its path.
template <bool kMulti, bool kIdx16, bool kAhead, bool kH128>
__global__ void __launch_bounds__(kDelThreads, SNN_DEL_MINB)
k_deliver(NetDev net, StateDev st, uint32_t epi) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t wsum[kDelWarps];
    __shared__ unsigned long long wsum64[kDelWarps];
    __shared__ uint64_t s_ptr[kDelRows];     // segment g: byte address of idx[c] of flattened element 0
    __shared__ uint8_t s_rc[kDelRows];       // segment g: receptor code
    __shared__ uint2 s_bw[kDelWin / 32];     // window word: (segment-start bits, segments begun before it - 1)
    constexpr bool kPlT = kAhead;            // (runtime: net.nstdp != 0)
    const uint32_t C = net.C;
    int32_t *acc = reinterpret_cast<int32_t *>(smem);                           // [nrcpt][C]
    const uint32_t k = blockIdx.x;
    const uint32_t nsplit = gridDim.y, split = blockIdx.y;
    const uint32_t slo = net.tgt_lo + k * C;
    const uint32_t shi = min(slo + C, net.tgt_hi);
    const uint32_t width = shi > slo ? shi - slo : 0u;
    const uint32_t lane = threadIdx.x & 31;
    const unsigned long long t_entry = st.kspan ? gtimer() : 0ull;
    unsigned long long t_wait = 0ull;
    const bool pl_on = kAhead && net.nstdp != 0;
    trace_mark(st.trace, 2, 0);

    // prologue: reads only the arrival list -- kAhead: k_front(t-1)'s, complete
    // before k_front(t) triggered this launch; else k_front(t)'s, complete before
    // k_stdp(t) triggered it (without STDP the primary IS k_front(t), so wait)
    if (!kAhead && net.nstdp == 0) pdl_wait();
    // the step and every slot's arrival count in one round trip
    const int64_t t = st.ctr->t;
    const uint32_t par = (uint32_t)(t & 1);
    const RowDesc *Al = st.adesc[par];
    const uint32_t nAs = st.ctr->lst[t & 7][1];
    const uint32_t nA = k < net.nslices ? nAs : 0u;
    for (uint32_t x = threadIdx.x; x < net.nrcpt * C; x += kDelThreads) acc[x] = 0;
    DelStdp ps;
    ps.n_syn = ps.n_w = 0;
    ps.xq_a = 0;
    if (kPlT && pl_on) {
        for (uint32_t x = threadIdx.x; x < net.nstdp * (kMaxHist + 1); x += kDelThreads)
            g_del_dp[x] = st.stdp[x / (kMaxHist + 1)].dplus[x % (kMaxHist + 1)];
        if (threadIdx.x < net.nstdp)
            g_del_par[threadIdx.x] = make_float4(st.stdp[threadIdx.x].a_plus, st.stdp[threadIdx.x].a_minus,
                                                 st.stdp[threadIdx.x].w_max, 0.0f);
        ps.xq_a = smem_u32(acc + net.nrcpt * C);
    }
    __syncthreads();
    const uint32_t r_begin = (uint32_t)(((uint64_t)nA * split) / nsplit);
    const uint32_t r_end = (uint32_t)(((uint64_t)nA * (split + 1)) / nsplit);
    const uint32_t P = net.nslices + 1;
    const float scale = net.scale;
    const uint32_t bw_a = smem_u32(s_bw), ptr_a = smem_u32(s_ptr), rc_a = smem_u32(s_rc);
    constexpr bool idx16 = kIdx16;
    // accumulator of target j (32-bit ids) / slice offset j - slo (16-bit), receptor r: + 4 (r C + j)
    const uint32_t acc_a = idx16 ? smem_u32(acc) : smem_u32(acc) - 4u * slo;
    // w[c] at idx[c] + dw, or at 2 idx16[c] + dw (bytes)
    const uint64_t dw = idx16 ? (uint64_t)st.w - 2ull * (uint64_t)st.idx16 : (uint64_t)st.w - (uint64_t)st.idx;
    uint32_t n_ev = 0, n_seg = 0;
    bool waited = !kAhead && net.nstdp == 0;    // (that case waited above)
    for (uint32_t r0 = r_begin; r0 < r_end; r0 += kDelRows) {
        // ---- tabulate (two rows per thread): descriptor + pivot pair
        uint32_t len2[2] = {0, 0};
        RowDesc d2[2];
        uint2 pp[2];
#pragma unroll
        for (int q = 0; q < 2; q++) {                 // both rows' loads in flight together
            const uint32_t r = r0 + threadIdx.x * 2 + q;
            if (r < r_end) d2[q] = Al[r];
        }
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const uint32_t r = r0 + threadIdx.x * 2 + q;
            if (r < r_end) {
                const uint32_t *pv = st.piv + (size_t)d2[q].row * P + k;
                pp[q] = make_uint2(pv[0], pv[1]);
            }
        }
        int64_t c0q[2] = {0, 0};                     // CSR offset of the segment's first synapse
        uint32_t rcq[2] = {0, 0};
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const uint32_t r = r0 + threadIdx.x * 2 + q;
            if (r < r_end) {
                len2[q] = pp[q].y - pp[q].x;
                c0q[q] = d2[q].start + pp[q].x;
                rcq[q] = (d2[q].meta >> 8) & 3u;
                if (rcq[q] == 3u) rcq[q] = 3u | (((d2[q].meta >> 16) & 0xfu) << 2);
            }
        }
        // kAhead: the segments without a plastic part (static synapses: weights
        // and ids fixed) come first in the flattened order and are delivered
        // before the dependency wait, while k_front(t) still runs; the plastic
        // ones (STDP of the arrival, Fig. 2c, needs k_front(t)'s post spikes)
        // after it.  Else (D < 2) every segment after the wait.
        bool plq[2] = {false, false};
#pragma unroll
        for (int q = 0; q < 2; q++)
            plq[q] = kAhead && len2[q] != 0 && (net.nstdp != 0) && max(pp[q].x, d2[q].s0) < min(pp[q].y, d2[q].s1);
        const uint32_t ns_s = (len2[0] != 0 && !plq[0]) + (len2[1] != 0 && !plq[1]);
        const uint32_t ns_p = (uint32_t)plq[0] + (uint32_t)plq[1];
        const uint32_t ne_s = (plq[0] ? 0u : len2[0]) + (plq[1] ? 0u : len2[1]);
        const uint32_t ne_p = (plq[0] ? len2[0] : 0u) + (plq[1] ? len2[1] : 0u);
        n_ev += len2[0] + len2[1];
        n_seg += ns_s + ns_p;
        // ---- compact the non-empty segments: flattened start and slot of each
        // (static ones first: slots [0, Ns), elements [0, Ts); then the plastic)
        unsigned long long tot_s = 0, tot_p = 0;
        const unsigned long long inc_s =
            block_incl_scan64(((unsigned long long)ns_s << 32) | ne_s, wsum64, tot_s);
        __syncthreads();                             // (wsum64 reused)
        const unsigned long long inc_p =
            block_incl_scan64(((unsigned long long)ns_p << 32) | ne_p, wsum64, tot_p);
        const uint32_t Ts = (uint32_t)tot_s, Ns = (uint32_t)(tot_s >> 32);
        const uint32_t T = Ts + (uint32_t)tot_p;
        uint32_t es = (uint32_t)inc_s - ne_s, ep = Ts + (uint32_t)inc_p - ne_p;   // next flattened start
        uint32_t gs = (uint32_t)(inc_s >> 32) - ns_s, gp = Ns + (uint32_t)(inc_p >> 32) - ns_p;
        uint32_t est[2];                             // flattened start of the thread's two segments
#pragma unroll
        for (int q = 0; q < 2; q++) {
            if (len2[q] == 0) continue;
            uint32_t &e = plq[q] ? ep : es;
            uint32_t &g = plq[q] ? gp : gs;
            est[q] = e;
            e += len2[q];
            s_rc[g] = (uint8_t)rcq[q];
            s_ptr[g] = idx16 ? (uint64_t)(st.idx16 + c0q[q]) - 2ull * est[q]
                             : (uint64_t)(st.idx + c0q[q]) - 4ull * est[q];
            if (kPlT && pl_on) {
                // the segment's plastic part: row-relative [max(piv, s0), min(piv', s1))
                const uint32_t a0 = max(pp[q].x, d2[q].s0), a1 = min(pp[q].y, d2[q].s1);
                g_del_pl[g] = a0 < a1 ? make_uint2(est[q] + a0 - pp[q].x, est[q] + a1 - pp[q].x) : make_uint2(0u, 0u);
                g_del_row[g] = make_uint2(__float_as_uint(d2[q].xp), d2[q].meta);
            }
            g++;
        }
        for (uint32_t w0 = 0; w0 < T; w0 += kDelWin) {
            const uint32_t wlen = min(T - w0, (uint32_t)kDelWin);
            s_bw[threadIdx.x].x = 0u;
            __syncthreads();                         // also: table written, previous window done
#pragma unroll
            for (int q = 0; q < 2; q++)
                if (len2[q] != 0 && est[q] >= w0 && est[q] - w0 < wlen)
                    atomicOr(&s_bw[(est[q] - w0) >> 5].x, 1u << ((est[q] - w0) & 31));
            // segments begun before the window (the sync of the bitmap, too)
            const uint32_t before = __syncthreads_count(len2[0] != 0 && est[0] < w0) +
                                    __syncthreads_count(len2[1] != 0 && est[1] < w0);
            const uint32_t pc = __popc(s_bw[threadIdx.x].x);
            uint32_t wt = 0;
            const uint32_t winc = block_incl_scan<kDelThreads>(pc, wsum, wt);
            s_bw[threadIdx.x].y = before + winc - pc - 1u;
            __syncthreads();
            // ---- elements: thread x takes w0 + x + 512 u (coalesced); the
            //      static part of the window [0, xs) before the wait (kAhead)
            const uint32_t xs = (kAhead && SNN_DEL_PRE) ? (Ts > w0 ? min(Ts - w0, wlen) : 0u) : 0u;
            if (xs)
                deliver_window<kMulti, kIdx16, false, false>(net, st, 0u, xs, w0, bw_a, ptr_a, rc_a, acc_a, dw, scale,
                                                             slo, ps);
            if (xs < wlen && !waited) {
                del_wait(st, t_wait);
                waited = true;
                if (kPlT && pl_on) {
                    // the slice's x_post, history words and spike positions (k_front(t)) -> shared
                    const uint32_t plo = net.pp_lo > slo ? net.pp_lo : slo, phi = net.pp_hi < shi ? net.pp_hi : shi;
                    const uint8_t *fpos = st.fpos + (size_t)(t & 3) * st.fstride;
                    unsigned char *xs_b = reinterpret_cast<unsigned char *>(acc + net.nrcpt * C);
                    for (uint32_t j = plo + threadIdx.x; j < phi; j += kDelThreads) {
                        const uint32_t jl = j - slo;
                        reinterpret_cast<float *>(xs_b)[jl] = st.xpost[j];
                        reinterpret_cast<uint64_t *>(xs_b + 4u * C)[jl] = st.hist[j];
                        if (kH128) reinterpret_cast<uint64_t *>(xs_b + 12u * C)[jl] = st.hist_hi[j];
                        xs_b[del_fpos_off<kH128>(C) + jl] = fpos[j];
                    }
                    __syncthreads();
                }
            }
            if (xs < wlen) {
                if (kPlT && pl_on)
                    deliver_window<kMulti, kIdx16, kPlT, kH128>(net, st, xs, wlen, w0, bw_a, ptr_a, rc_a, acc_a, dw,
                                                                scale, slo, ps);
                else
                    deliver_window<kMulti, kIdx16, false, false>(net, st, xs, wlen, w0, bw_a, ptr_a, rc_a, acc_a, dw,
                                                                 scale, slo, ps);
            }
            if (w0 + kDelWin < T) __syncthreads();  // bitmap reused by the next window
        }
        __syncthreads();                           // table reused next round
    }
    // (the write-back adds to the inputs k_front(t) consumed: after its completion)
    if (!waited) {
        del_wait(st, t_wait);
        waited = true;
    }
    trace_mark(st.trace, 2, 2);
    // ---- write-back (one coalesced pass; several CTAs may share a slice)
    for (uint32_t rr = 0; rr < net.nrcpt; rr++) {
        int32_t *dst = rr == 0 ? st.in_e : st.in_i;
        for (uint32_t x = threadIdx.x; x < width; x += kDelThreads) {
            const int32_t v = acc[rr * C + x];
            if (v != 0) atomicAdd(dst + slo + x, v);
        }
    }
    n_ev = __reduce_add_sync(0xffffffffu, n_ev);
    n_seg = __reduce_add_sync(0xffffffffu, n_seg);
    if (kPlT && pl_on) {
        ps.n_syn = __reduce_add_sync(0xffffffffu, ps.n_syn);
        ps.n_w = __reduce_add_sync(0xffffffffu, ps.n_w);
    }
    if (lane == 0) {
        if (n_ev) {
            atomicAdd(&st.ctr->metric[0], (unsigned long long)n_ev);
            atomicAdd(&st.ctr->metric[7], (unsigned long long)n_ev);
        }
        if (n_seg) atomicAdd(&st.ctr->metric[6], (unsigned long long)n_seg);
        if (kPlT && ps.n_syn) {
            atomicAdd(&st.ctr->metric[3], (unsigned long long)ps.n_syn);
            atomicAdd(&st.ctr->metric[8], (unsigned long long)ps.n_syn);    // 8(d): every arrival weight r+w
        }
        if (kPlT && ps.n_w) atomicAdd(&st.ctr->metric[4], (unsigned long long)ps.n_w);
    }
    // kAhead: the arriving rows of the step (k_front counts the arrivals of t + 1)
    if (kAhead && k == 0 && split == 0 && threadIdx.x == 0 && nAs) atomicAdd(&st.ctr->metric[1], (unsigned long long)nAs);
    if (kAhead && epi && k < net.nslices) {
        // ---- the fused step (SURVEY 8(a4) fusion lever 2): the last CTA of
        //      the slice to finish its write-back updates the slice's neurons
        //      for step t + 1 (neuron_update, the same operations as k_front)
        //      and writes their ring / recent words -- the input never waits
        //      for a separate neuron kernel.  The Poisson neurons of the word
        //      straddling R get their (stateless) draw here too; k_front(t+1)
        //      updates every other neuron >= R.
        __shared__ uint32_t s_last;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(st.slice_ticket + k, 1u) == nsplit - 1 ? 1u : 0u;
        __syncthreads();
        if (s_last) {
            if (threadIdx.x == 0) st.slice_ticket[k] = 0;
            __threadfence();                       // the other splits' write-backs
            const int64_t t1 = t + 1;
            const uint32_t hi32 = shi == net.R ? min((net.R + 31u) & ~31u, net.N) : shi;
            for (uint32_t x0 = 0; slo + x0 < hi32; x0 += kDelThreads) {
                const uint32_t i = slo + x0 + threadIdx.x;
                bool fired = false, recent = false;
                if (i < shi) {
                    fired = neuron_update(net, st, i, net.pop[find_pop(net, i)], t1, recent);
                } else if (i < hi32) {
                    const PopDev &pp = net.pop[find_pop(net, i)];
                    const u32x4 r = philox4x32_10(i, (uint32_t)t1, 2u, 0u, net.key0, net.key1);
                    fired = (uint64_t)r.x < pp.thr;
                }
                const uint32_t fw = __ballot_sync(0xffffffffu, fired), rw = __ballot_sync(0xffffffffu, recent);
                if (lane == 0 && i < hi32) {
                    st.ring[(size_t)(t1 & (kRingSlots - 1)) * net.ring_stride + (i >> 5)] = fw;
                    if (net.nstdp) st.recent[(size_t)(t1 & 3) * st.rstride + (i >> 5)] = rw;
                }
            }
        }
    }
    if (st.kspan) kspan_begin(st.kspan, t, 2, t_entry, t_wait ? t_wait : gtimer());
    // ---- step completion: the last CTA advances t
    __syncthreads();
    trace_mark(st.trace, 2, 3);
    kspan_end(st.kspan, t, 2);
    // (no fence: nothing the last CTA does depends on the other CTAs' writes,
    // and k_front(t+1) reads them after this grid completes)
    if (threadIdx.x == 0) {
        const uint32_t nb = gridDim.x * gridDim.y;
        if (atomicAdd(&st.ctr->ticket, 1u) == nb - 1) {
            st.ctr->ticket = 0;
            st.ctr->t = t + 1;
        }
    }
}

// ------------------------------------------------------ k_deliver_rowwise
// Fig. 3a (SNN_DELIV_ROWWISE, the ablation baseline): a warp per
// arriving row, lanes over its columns, each delivery an int32 global atomic
// (RED.ADD) into the target's accumulator -- no slicing, no shared memory.
constexpr int kRowThreads = 512;

__global__ void __launch_bounds__(kRowThreads)
k_deliver_rowwise(NetDev net, StateDev st) {
    const uint32_t lane = threadIdx.x & 31;
    if (net.nstdp == 0) pdl_wait();
    const int64_t t = st.ctr->t;
    const uint32_t par = (uint32_t)(t & 1);
    const RowDesc *Al = st.adesc[par];
    const uint32_t nA = st.ctr->lst[t & 7][1];
    pdl_wait();            // k_stdp(t): updated weights of plastic arrivals
    pdl_launch();
    const float scale = net.scale;
    uint32_t n_ev = 0;
    const uint32_t gw = (blockIdx.x * kRowThreads + threadIdx.x) >> 5, nw = (gridDim.x * kRowThreads) >> 5;
    for (uint32_t r = gw; r < nA; r += nw) {
        const RowDesc d = Al[r];
        const int64_t c0 = d.start, c1 = st.row_ptr[d.row + 1];
        uint32_t rc = (d.meta >> 8) & 3u;
        const int src_pop = (int)((d.meta >> 16) & 0xfu);
        n_ev += (uint32_t)(c1 - c0);
        for (int64_t c = c0 + lane; c < c1; c += 32) {
            const uint32_t j = __ldg(st.idx + c);
            const float w = __ldg(st.w + c);
            uint32_t r2 = rc;
            if (r2 == 3u) r2 = (uint32_t)net.rcpt[src_pop][find_pop(net, j)];
            atomicAdd((r2 == 0 ? st.in_e : st.in_i) + j, __float2int_rn(__fmul_rn(w, scale)));
        }
    }
    n_ev = __reduce_add_sync(0xffffffffu, lane == 0 ? n_ev : 0u);
    if (lane == 0 && n_ev) {
        atomicAdd(&st.ctr->metric[0], (unsigned long long)n_ev);
        atomicAdd(&st.ctr->metric[7], (unsigned long long)n_ev);
    }
    // ---- step completion: the last CTA books the list counts and advances t
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(&st.ctr->ticket, 1u) == gridDim.x - 1) {
            st.ctr->ticket = 0;
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
            const bool arr_prev = (t_last >= (int64_t)net.D) && ring_bit(st.ring, net.ring_stride, t_last - net.D, i);
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
    uint32_t s0, s1, s2, n0, n1, n2;
    compact3(cs, st.ctr->rlst, st.ctr->rlst + 1, st.ctr->rlst + 2, stale, false, false, s0, s1, s2, n0, n1,
             n2);   // (rlst zeroed by the launcher)
    if (stale) st.rdesc[s0] = d;
}

// (3) after k_stdp ran the flush on the listed rows: their x_pre / tlu.
__global__ void __launch_bounds__(kFrontThreads)
k_readout_finish(NetDev net, StateDev st, int64_t t_last) {
    const uint32_t n = st.ctr->rlst[0];
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const RowDesc d = st.rdesc[r];
        const StdpDev &sd = net.stdp[(d.meta >> 12) & 0xfu];
        st.xpre[d.row] = xpre_after(sd, d.xp, (int)(d.meta & kMetaAge), false);
        st.tlu[d.row] = (int32_t)t_last;
    }
}

// (4) kAhead: the arrivals of t_last + 1 were listed by k_front(t_last) with
// their rows' state at t_last + 1; after the read-out flush every plastic row
// has tlu = t_last: age 1 and the flushed x_pre.
__global__ void k_readout_ahead(NetDev net, StateDev st, int64_t t_last) {
    const uint32_t n = st.ctr->lst[(t_last + 1) & 7][1];
    RowDesc *A = st.adesc[(t_last + 1) & 1];
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        RowDesc d = A[r];
        if (!(d.meta & kMetaPlastic)) continue;
        d.meta = (d.meta & ~kMetaAge) | (uint32_t)(t_last + 1 - st.tlu[d.row]);
        d.xp = st.xpre[d.row];
        A[r] = d;
    }
}

// Exchange (world > 1): the other ranks' spike words of step tp, gathered in
// `gath` (one share of wmax words per rank), into ring slot tp.  t_fixed < 0:
// tp = the current step (NCCL: unpack right after the all-gather of the step).
__global__ void k_unpack(NetDev net, StateDev st, const uint32_t *gath, int64_t t_fixed) {
    // t_fixed < 0: the exchange's own step counter (one exchange per step, in
    // order; it may run beside the step, after k_deliver advanced ctr->t)
    const int64_t tp = t_fixed >= 0 ? t_fixed : *(volatile const int64_t *)&st.ctr->tx;
    if (t_fixed < 0) {
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(&st.ctr->xticket, 1u) == gridDim.x - 1) {   // the last CTA: next step
            st.ctr->xticket = 0;
            st.ctr->tx = tp + 1;
        }
    }
    if (tp < 0) return;
    const uint32_t nwR = (net.R + 31) >> 5;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwR; w += gridDim.x * blockDim.x) {
        uint32_t r = 0;                        // the rank owning word w (ranges are 32-aligned)
        while (r + 1 < net.world && 32u * w >= net.rank_lo[r + 1]) r++;
        if (r == net.rank) continue;
        st.ring[(size_t)(tp & (kRingSlots - 1)) * net.ring_stride + w] =
            gath[(size_t)r * net.wmax + (w - (net.rank_lo[r] >> 5))];
    }
}

cudaError_t launch_unpack(const NetDev &net, const StateDev &st, const uint32_t *gath, int64_t t_fixed,
                          cudaStream_t s) {
    const uint32_t nwR = (net.R + 31) >> 5;
    const uint32_t blocks = (nwR + 255) / 256 < 296 ? (nwR + 255) / 256 : 296;
    k_unpack<<<blocks > 0 ? blocks : 1, 256, 0, s>>>(net, st, gath, t_fixed);
    return cudaGetLastError();
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
        if (u >= 0) h |= ring_bit(ring, net.ring_stride, u, i);
    }
    out[i] = h;
}

// ---------------------------------------------------------------- launchers
uint32_t front_blocks(const NetDev &net) { return (net.N + kFrontThreads - 1) / kFrontThreads; }

// Launch with the programmatic-stream-serialization attribute (PDL) and, when
// set (g_prio: a step graph with a side branch), a scheduling priority.
static int g_prio = 0;   // 0: none, else the priority of the next launches (set per launch by the engine)
void set_launch_priority(int p) { g_prio = p; }
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    if (g_prio) {
        attr[na].id = cudaLaunchAttributePriority;
        attr[na].val.priority = g_prio;
        na++;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// use_tf: the step from the front's own counter (the fused step graph, where
// k_front(t) runs beside k_deliver(t), which advances ctr->t)
cudaError_t launch_front(const NetDev &net, const StateDev &st, cudaStream_t s, bool pdl, bool ahead, int part,
                         bool use_tf) {
    void (*k)(NetDev, StateDev, uint32_t) = ahead ? (part == 4 ? k_front<true, 4> : part == 3 ? k_front<true, 3>
                                                                                  : k_front<true, 0>)
                                        : part == 1 ? k_front<false, 1> : part == 2 ? k_front<false, 2> : k_front<false, 0>;
    if (part == 4) {             // neurons [0, R) and R's word: 512-thread CTAs (one wave beside k_flush)
        const uint32_t n = std::min((net.R + 31u) & ~31u, net.N);
        return launch_pdl(k, dim3(std::max(1u, (n + 511u) / 512u)), dim3(512), 0, s, pdl, net, st, 0u);
    }
    return launch_pdl(k, dim3(front_blocks(net)), dim3(kFrontThreads), 0, s, pdl, net, st, use_tf ? 1u : 0u);
}

// k_deliver variants by (two receptors, 16-bit ids, ahead list, H = 128)
static void (*const g_deliver[16])(NetDev, StateDev, uint32_t) = {
    k_deliver<false, false, false, false>, k_deliver<false, false, false, true>,
    k_deliver<false, false, true, false>,  k_deliver<false, false, true, true>,
    k_deliver<false, true, false, false>,  k_deliver<false, true, false, true>,
    k_deliver<false, true, true, false>,   k_deliver<false, true, true, true>,
    k_deliver<true, false, false, false>,  k_deliver<true, false, false, true>,
    k_deliver<true, false, true, false>,   k_deliver<true, false, true, true>,
    k_deliver<true, true, false, false>,   k_deliver<true, true, false, true>,
    k_deliver<true, true, true, false>,    k_deliver<true, true, true, true>};

size_t stdp_smem_bytes(const NetDev &net, uint32_t pp_lo, uint32_t pp_hi) {
    (void)net;
    return ((sizeof(StdpSmem) + 127) & ~(size_t)127) + (size_t)kStdpStages * kStdpStageCh * 32 + 16ull * ((((pp_hi + 31) >> 5) - ((pp_lo >> 7) << 2) + 3) >> 2);
}

// accumulators [nrcpt][C]; + the slice's x_post [C] and fpos [C] with the
// plastic arrivals' STDP (kAhead with STDP)
size_t deliver_smem_bytes(const NetDev &net, bool ahead) {
    // + (plastic arrivals) the slice's x_post, history words and spike positions
    return 4ull * net.nrcpt * net.C + (ahead && net.nstdp ? (13ull + (net.H > kHistBits ? 8ull : 0ull)) * net.C + 16 : 0ull);
}

// The dynamic shared-memory limit is an attribute of the kernel function, not
// of a handle: set it once per device to the opt-in maximum (minus the
// kernel's static shared memory), so no handle can lower it under another.
cudaError_t kernels_configure(int device) {
    static std::mutex mu;
    static std::set<int> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(device)) return cudaSuccess;
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (e != cudaSuccess) return e;
    auto set_max = [&](const void *k) -> cudaError_t {
        cudaFuncAttributes a;
        cudaError_t r = cudaFuncGetAttributes(&a, k);
        if (r != cudaSuccess) return r;
        return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
    };
    for (auto k : g_deliver)
        if ((e = set_max((const void *)k)) != cudaSuccess) return e;
    void (*ks[6])(NetDev, StateDev, int64_t, uint32_t, uint32_t) = {
        k_stdp<false, false, false>, k_stdp<false, true, false>, k_stdp<false, false, true>,
        k_stdp<false, true, true>, k_stdp<true, false, true>, k_stdp<true, true, true>};
    for (auto k : ks)
        if ((e = set_max((const void *)k)) != cudaSuccess) return e;
    void (*ke[6])(NetDev, StateDev, uint32_t, uint32_t) = {k_stdp_ev<false, 0, 1024>, k_stdp_ev<true, 0, 1024>,
                                                          k_stdp_ev<false, 1, 512>, k_stdp_ev<true, 1, 512>,
                                                          k_stdp_ev<false, 2, 512>, k_stdp_ev<true, 2, 512>};
    for (auto k : ke)
        if ((e = set_max((const void *)k)) != cudaSuccess) return e;
    void (*kf[8])(NetDev, StateDev, uint32_t, uint32_t) = {
        k_flush<false, false, false>, k_flush<false, true, false>, k_flush<true, false, false>, k_flush<true, true, false>,
        k_flush<false, false, true>, k_flush<false, true, true>, k_flush<true, false, true>, k_flush<true, true, true>};
    for (auto k : kf)
        if ((e = set_max((const void *)k)) != cudaSuccess) return e;
    done.insert(device);
    return cudaSuccess;
}

cudaError_t launch_stdp(const NetDev &net, const StateDev &st, int64_t t_fixed, uint32_t grid, uint32_t pp_lo,
                        uint32_t pp_hi, cudaStream_t s, bool pdl) {
    const bool lazy = net.plast_mode == 1u, h128 = net.H > kHistBits;
    // read-out flush, lazy, naive, batched flushes (rows of several ages): the
    // per-target forced-flush factor assumes age H
    const bool generic = t_fixed >= 0 || net.plast_mode != 0u || net.flush_period != 0u;
    void (*k)(NetDev, StateDev, int64_t, uint32_t, uint32_t) =
        lazy ? (h128 ? k_stdp<true, true, true> : k_stdp<true, false, true>)
             : generic ? (h128 ? k_stdp<false, true, true> : k_stdp<false, false, true>)
                       : (h128 ? k_stdp<false, true, false> : k_stdp<false, false, false>);
    return launch_pdl(k, dim3(grid), dim3(kStdpThreads), stdp_smem_bytes(net, pp_lo, pp_hi), s, pdl, net, st,
                      t_fixed, pp_lo, pp_hi);
}

// mode 0: arrivals + forced flushes (the step without the ahead list), 1: the
// plastic arrivals only (a step whose flushes run on a side branch), 2: the
// forced flushes (k_flush)
uint32_t stdp_ev_threads(int mode) { return mode == 2 ? kFlT : mode == 1 ? 512u : 1024u; }
uint32_t flush_ctas_per_sm() { return SNN_FL_GRID; }
cudaError_t launch_stdp_ev(const NetDev &net, const StateDev &st, uint32_t grid, uint32_t pp_lo, uint32_t pp_hi,
                           cudaStream_t s, bool pdl, int mode) {
    const bool h = net.H > kHistBits;
    if (mode == 2 && getenv("SNN_FLUSH_EV"))    // (experiments: the per-thread-chunk flush stream)
        return launch_pdl(h ? k_stdp_ev<true, 2, 512> : k_stdp_ev<false, 2, 512>, dim3(grid), dim3(512),
                          ev_smem_bytes(pp_lo, pp_hi), s, pdl, net, st, pp_lo, pp_hi);
    if (mode == 2) {
        const bool stg = flush_staged(pp_lo, pp_hi);
        void (*kf[8])(NetDev, StateDev, uint32_t, uint32_t) = {
            k_flush<false, false, false>, k_flush<false, true, false>, k_flush<true, false, false>, k_flush<true, true, false>,
            k_flush<false, false, true>, k_flush<false, true, true>, k_flush<true, false, true>, k_flush<true, true, true>};
        const uint32_t v = (st.b64 ? 4u : 0u) | (h ? 2u : 0u) | (stg ? 1u : 0u);
        return launch_pdl(kf[v], dim3(grid), dim3(kFlT), flush_smem_bytes(pp_lo, pp_hi), s, pdl, net, st, pp_lo, pp_hi);
    }
    void (*k)(NetDev, StateDev, uint32_t, uint32_t) =
        mode == 1 ? (h ? k_stdp_ev<true, 1, 512> : k_stdp_ev<false, 1, 512>)
                  : (h ? k_stdp_ev<true, 0, 1024> : k_stdp_ev<false, 0, 1024>);
    return launch_pdl(k, dim3(grid), dim3(stdp_ev_threads(mode)), ev_smem_bytes(pp_lo, pp_hi), s, pdl, net, st,
                      pp_lo, pp_hi);
}

cudaError_t launch_deliver_rowwise(const NetDev &net, const StateDev &st, uint32_t grid, cudaStream_t s, bool pdl) {
    return launch_pdl(k_deliver_rowwise, dim3(grid), dim3(kRowThreads), 0, s, pdl, net, st);
}

// epi: the fused step's epilogue (the neurons of t + 1 by the slices' last CTAs)
cudaError_t launch_deliver(const NetDev &net, const StateDev &st, uint32_t splits, cudaStream_t s, bool pdl,
                           bool ahead, bool epi) {
    dim3 grid(net.nslices > 0 ? net.nslices : 1, splits);
    const uint32_t v = (net.nrcpt > 1 ? 8u : 0u) | (st.idx16 ? 4u : 0u) | (ahead ? 2u : 0u) | (net.H > kHistBits ? 1u : 0u);
    return launch_pdl(g_deliver[v], grid, dim3(kDelThreads), deliver_smem_bytes(net, ahead), s, pdl, net, st,
                      epi ? 1u : 0u);
}

cudaError_t launch_readout(const NetDev &net, const StateDev &st, int64_t t_last, uint32_t grid, uint32_t pp_lo,
                           uint32_t pp_hi, cudaStream_t s, bool ahead) {
    cudaError_t e = cudaMemsetAsync(st.ctr->rlst, 0, sizeof(st.ctr->rlst), s);
    if (e != cudaSuccess) return e;
    k_readout_prepare<<<front_blocks(net), kFrontThreads, 0, s>>>(net, st, t_last);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if ((e = launch_stdp(net, st, t_last, grid, pp_lo, pp_hi, s, false)) != cudaSuccess) return e;
    k_readout_finish<<<front_blocks(net), kFrontThreads, 0, s>>>(net, st, t_last);
    if (ahead) k_readout_ahead<<<64, 256, 0, s>>>(net, st, t_last);
    return cudaGetLastError();
}

// SNN_FLAG_KTIME: every slot back to (entry, wait) = +inf, (end, ctas) = 0.
__global__ void k_kspan_reset(KSpan *ks, uint32_t n) {
    for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x)
        ks[x] = KSpan{~0ull, ~0ull, 0ull, 0ull};
}

cudaError_t launch_kspan_reset(KSpan *ks, cudaStream_t s) {
    const uint32_t n = kKSpanSlots * kKSpanKernels;
    k_kspan_reset<<<256, 256, 0, s>>>(ks, n);
    return cudaGetLastError();
}

cudaError_t launch_hist_from_ring(const NetDev &net, const uint32_t *ring, int64_t t_last, uint64_t *out,
                                  cudaStream_t s) {
    k_hist_from_ring<<<(net.N + 255) / 256, 256, 0, s>>>(net, ring, t_last, out);
    return cudaGetLastError();
}

}  // namespace snn
