// common.cuh -- device-side tables and state of one simulation handle.
//
// Part of the product path (libsnn.so).  Shares nothing with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace snn {

constexpr int kMaxPops = 16;
constexpr int kMaxRanks = 64;   // world size limit of the target-range partition
constexpr int kHistBits = 64;     // bits per history word
constexpr int kMaxHist = 128;     // H: 64 (one word) or 128 (two words)
constexpr int kRingSlots = 64;    // bitmask ring: slot t % 64 holds step t's spikes
constexpr uint32_t kArrBit = 0x80000000u;

enum PopKind : uint32_t { POP_POISSON = 0, POP_LIF_DELTA = 1, POP_LIF_CUBA = 2 };
enum PopFlags : uint32_t {
    PF_HAS_INPUT = 1u,       // target of at least one projection
    PF_POST_PLASTIC = 2u,    // target of an STDP projection: keeps hist u64 + x_post
    PF_PRE_PLASTIC = 4u      // source of an STDP projection: rows carry tlu / x_pre
};

// Per-population constants, computed once on the host in double and rounded
// to fp32 (R19).
struct PopDev {
    uint32_t base, n, kind, flags;
    uint64_t thr;        // POISSON: floor(rate*dt*2^32) (2^32 = always)
    float k_m;           // LIF_DELTA: fp32(1 - dt/tau_m)
    float a_m;           // LIF_CUBA:  fp32(dt/tau_m)
    float d_e, d_i;      // LIF_CUBA:  fp32(exp(-dt/tau_e)), fp32(exp(-dt/tau_i))
    float v_th, v_reset, v_rest;
    int32_t n_ref;       // refractory steps
    float d_minus;       // PF_POST_PLASTIC: fp32(exp(-dt/tau_-)) of the x_post trace
    int32_t stdp;        // PF_PRE_PLASTIC: index into NetDev::stdp, else -1
    int32_t rcpt_uniform;// receptor used by every projection out of this pop (-1: mixed)
    int32_t post_stdp;   // PF_POST_PLASTIC: the StdpDev whose D+ table its forced-flush factor uses, else -1
};

struct StdpDev {
    uint32_t dst_pop;
    float a_plus, a_minus, w_max;
    float dplus[kMaxHist + 1];    // fp32(exp(-n dt / tau_+)), n = 0..H (closed-form skip-ahead)
};

struct NetDev {
    uint32_t N;          // neurons
    uint32_t R;          // neurons [0, R) may receive synapses (slice domain)
    uint32_t tgt_lo, tgt_hi;  // this rank's target range
    uint32_t C, log2C, nslices;   // slice width and number of local slices
    uint32_t nwords;     // 32-bit words of spike bits per step = ceil(N/32)
    uint32_t ring_stride;// words per ring slot (nwords + exchange padding)
    uint32_t world, rank;        // ranks sharing the target range
    uint32_t xchg;               // the spike-word exchange runs (world > 1, or SNN_FLAG_EXCHANGE)
    uint32_t debug;              // SNN_DEBUG_KERNELS bits (experiments only; 0 in normal runs)
    uint32_t wmax;               // words exchanged per rank and step (the largest share + 1)
    uint32_t rank_lo[kMaxRanks + 1];   // target range of rank r: [rank_lo[r], rank_lo[r + 1]) (C-aligned)
    uint32_t D;          // delay
    uint32_t H;          // history bits: 64 or 128 (forced flush at age H, R3)
    uint32_t flush_period; // 0: flush at age H; K: every K steps the rows of age >= H - K (R33)
    uint32_t fl_lag;     // the ahead step's flush deadline L (2 or 3): k_flush(t) ends before k_deliver(t+L) (R36)
    uint32_t plast_mode; // SNN_PLAST_EVENT / LAZY / NAIVE (ablation)
    uint32_t deliv_mode; // SNN_DELIV_SLICED / ROWWISE (ablation)
    uint32_t npop, nstdp;
    int32_t F;           // fixed-point fraction bits
    float scale, inv_scale;       // 2^F, 2^-F
    uint32_t key0, key1;          // Philox key
    uint32_t nrcpt;      // accumulator arrays in use (1 or 2)
    PopDev pop[kMaxPops];
    int8_t rcpt[kMaxPops][kMaxPops];   // receptor of projection (src, dst), -1 = none
    StdpDev stdp[4];
    // plastic source rows: concatenation of the PF_PRE_PLASTIC populations
    uint32_t n_plastic_rows;
    uint32_t pp_lo, pp_hi;        // neurons [pp_lo, pp_hi) hold the post-synaptic STDP state (hist, x_post)
};

// Tables of the graph builder (per (src pop, dst pop) projection).
constexpr int kGapTab = 4096;          // geometric gap table length (R32)
struct BuildTabs {
    uint64_t thr[kMaxPops * kMaxPops];     // Bernoulli thresholds floor(p 2^32), 0 = none
    uint8_t autapse[kMaxPops * kMaxPops];
    float weight[kMaxPops * kMaxPops];     // initial (final, caller-scaled) weight
    int16_t gap_slot[kMaxPops * kMaxPops]; // projection (src, dst) -> its gap table, -1 = none
    float inv_l2q[kMaxPops * kMaxPops];    // 1 / log2(1 - p): the inverse-CDF estimate of a gap (warp builder)
    const uint32_t *gap;                   // [projections][kGapTab]: floor((1-p)^k 2^32), k = 1..kGapTab
};

#ifndef SNN_FRONT_T
#define SNN_FRONT_T 1024
#endif
constexpr int kFrontThreads = SNN_FRONT_T;   // k_front CTA = one list region

struct Counters {
    int64_t t;               // next step to simulate
    int64_t tfl;             // the step of the next k_flush launch (k_flush runs once per step, in order;
                             // its last CTA advances it)
    uint32_t fticket;        // CTA-completion ticket of k_flush
    uint32_t xticket;        // CTA-completion ticket of k_unpack (world > 1)
    int64_t tx;              // the step of the next NCCL exchange (k_unpack advances it)
    uint32_t ticket;         // CTA-completion ticket of the slice kernel
    uint32_t fr_ticket;      // CTA-completion ticket of k_front
    int64_t tf;              // the step of the next k_front (its last CTA advances it)
    unsigned long long metric[16];
    alignas(16) uint32_t lst[8][4];      // by step t & 7: list lengths (plastic arrivals, arrivals, forced flushes, 0);
                             // several slots: the forced flushes of step t are read by k_flush(t), which runs
                             // beside the next steps' k_deliver / k_front (engine.cu, side branch)
    uint32_t rlst[4];        // read-out flush list length
};

// One row to process, written by the front kernel: forced flushes for k_stdp,
// arrivals for k_deliver (which also runs the STDP of plastic arrivals).
// meta: bits 0-7 age (1..H), bits 8-9 receptor (3 = per target), bit 10
//       plastic row, bit 11 arrival, bits 12-15 STDP projection index, bits 16+
//       source pop (per-target receptor).
struct __align__(16) RowDesc {
    int64_t start;   // CSR offset of the row
    uint32_t row;    // source neuron id
    uint32_t meta;
    float xp;        // x_pre of the row at its last update (tlu)
    uint32_t s0, s1; // plastic segment [s0, s1), row-relative
    uint32_t pad;
};
constexpr uint32_t kMetaArr = 1u << 11;
constexpr uint32_t kMetaAge = 0xffu;
constexpr uint32_t kMetaPlastic = 1u << 10;

struct KSpan;

struct StateDev {
    // neurons (indexed by global id)
    float *V, *ge, *gi, *xpost;
    int32_t *ref, *in_e, *in_i;
    uint64_t *hist;          // bits 0..63 of the spike history (bit s: step t - s)
    uint64_t *hist_hi;       // H = 128: bits 64..127 (else unused)
    // four buffers by step (buffer t & 3 at + (t & 3) * fstride / rstride): k_flush(t) reads step t's
    // while k_front(t+1), k_front(t+2) write theirs
    float *fpot;             // post-plastic j with spikes in its H-bit window, for a flush of age H - k
                             // (k = 0, 1, 2): sum of D+[H - k - s] over its spikes s <= H - 1 - k, buffer 4k + (t & 3)
    uint8_t *fpos;           // post-plastic j: 0xfe no spike in its H-bit window, 0xff several, else the bit of the only one
    uint32_t fstride;        // elements per fpos / fpot buffer
    uint32_t rstride;        // words per `recent` buffer
    uint32_t *nspk;
    uint32_t *ring;          // [kRingSlots][ring_stride]
    // source rows
    float *xpre;
    int32_t *tlu;
    // graph (this rank's target range)
    int64_t *row_ptr;        // [N+1]
    uint32_t *idx;           // [S + pad]
    uint16_t *idx16;         // [S + pad] (j - tgt_lo) mod 2^16 (SNN_FLAG_IDX16), else null
    uint32_t *b64;           // [N][4] a row's element indices where j - tgt_lo reaches m 2^16 (m = 1..4; the
                             // row length if never) -- k_flush's 16-bit id stream (IDX16 + STDP), else null
    float *w;                // [S + pad]
    uint32_t *piv;           // [N][nslices+1], row-relative
    uint2 *seg;              // [N] plastic segment (lo, hi), row-relative
    // work lists (by step parity), appended by k_front CTAs (one atomic per
    // CTA and list, lengths in Counters::lst): plastic visits (arrivals from
    // the front, forced flushes from the back: entry cap - 1 - r) and arrivals
    RowDesc *vdesc[4], *adesc[2];   // visits by t & 3; arrivals by the parity of their step
    RowDesc *rdesc;          // read-out flush rows (length Counters::rlst[0])
    uint32_t nblk;           // k_front CTAs (list capacity nblk * kFrontThreads)
    uint32_t *vmask[2];      // [nwords] rows visited at the step of that parity
    uint32_t *recent;        // [4][rstride] bit i: post-plastic neuron i fired in the last H steps
    uint32_t *sendbuf;       // [wmax] this rank's spike words of the step (world > 1)
    uint32_t *gath;          // [2][world][wmax] all ranks' words (NCCL: slot 0; local group: by step parity)
    Counters *ctr;
    uint32_t *slice_ticket;  // [nslices] CTA-completion tickets of a slice's splits (the fused step's epilogue)
    const StdpDev *stdp;     // device copy of NetDev::stdp (coalesced table loads into shared memory)
    unsigned long long *trace;   // optional (SNN_FLAG_TRACE): per-CTA phase timestamps
    struct KSpan *kspan;         // optional (SNN_FLAG_KTIME): per-step kernel spans, [slot][kernel]
};

// Kernel spans of the graph-replayed step (SNN_FLAG_KTIME): thread 0 of every
// CTA folds its %globaltimer marks into the slot of its step t and kernel k --
// earliest CTA entry, earliest return from the kernel's dependency wait (PDL
// griddepcontrol.wait: the start of its exposed part), latest CTA end.  The
// host folds the slots into per-kernel averages (snn_read_state(KTIME)).
struct KSpan {
    unsigned long long entry, wait, end, ctas;
};
constexpr uint32_t kKSpanSlots = 65536;   // steps between two read-outs
constexpr int kKSpanKernels = 5;          // front, stdp, deliver, (spare), lists (world > 1, D = 0)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long g = 0;
#ifdef __CUDA_ARCH__
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
#endif
    return g;
}
__device__ __forceinline__ void kspan_begin(KSpan *ks, int64_t t, int k, unsigned long long t_entry,
                                            unsigned long long t_wait) {
#ifdef __CUDA_ARCH__
    if (ks && threadIdx.x == 0) {
        KSpan &s = ks[(size_t)(t & (kKSpanSlots - 1)) * kKSpanKernels + k];
        atomicMin(&s.entry, t_entry);
        atomicMin(&s.wait, t_wait);
        atomicAdd(&s.ctas, 1ull);
    }
#endif
}
// (uniform in the launch: every thread calls it; the barrier makes thread 0's
// mark the CTA's end)
__device__ __forceinline__ void kspan_end(KSpan *ks, int64_t t, int k) {
#ifdef __CUDA_ARCH__
    if (ks) {
        __syncthreads();
        if (threadIdx.x == 0) atomicMax(&ks[(size_t)(t & (kKSpanSlots - 1)) * kKSpanKernels + k].end, gtimer());
    }
#endif
}

// Phase trace (debug, SNN_FLAG_TRACE): thread 0 of each CTA stores %globaltimer
// at phase boundaries: trace[(kernel * kTraceCtas + cta) * 4 + phase].
constexpr int kTraceCtas = 4096;
constexpr int kTraceKernels = 4;   // front, stdp (flush), deliver, stdp_arr
__device__ __forceinline__ void trace_mark(unsigned long long *tr, int kernel, int phase) {
#ifdef __CUDA_ARCH__
    if (tr && threadIdx.x == 0) {
        const uint32_t cta = blockIdx.y * gridDim.x + blockIdx.x;
        if (cta < (uint32_t)kTraceCtas) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            tr[((size_t)kernel * kTraceCtas + cta) * 4 + phase] = g;
        }
    }
#endif
}

__host__ __device__ inline int find_pop(const NetDev &net, uint32_t i) {
    int p = 0;
#pragma unroll 1
    for (int k = 1; k < (int)net.npop; k++)
        if (i >= net.pop[k].base) p = k;
    return p;
}

}  // namespace snn
