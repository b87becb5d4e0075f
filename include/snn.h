/*
 * snn.h -- C ABI of libsnn.so, a B200-native (sm_100a) implementation of the
 * clock-driven SNN simulation step accelerated by arXiv 2107.04092 ("Spice").
 *
 * The problem statement followed (PAPER.md line numbers "P:n"):
 *   - a static directed graph, grouped by source and sorted, built once;
 *   - neurons with a 64-bit firing history, LSB = most recent, synapses
 *     with state, one network-wide delay in steps;
 *   - per step: (1) update neurons and note which fire; (2) update
 *     synapses -- lazy + event-driven plasticity over the history bitfields
 *     (Fig. 2c, Sec. III-A); (3) deliver spikes through
 *     an adjacency list partitioned into equal-width neuron slices with
 *     shared-memory atomics (Fig. 3b, Sec. III-B);
 *   - "users can still define custom models" is narrowed to the built-in
 *     population and synapse kinds below.
 *
 * Conventions for every entry point:
 *   - Plain C types only; no C++ type or exception crosses this boundary.
 *   - Every call returns an snn_status (0 = SNN_OK, < 0 = error).  On error a
 *     message is available from snn_last_error(sim) until the next call on that
 *     handle.  CUDA errors map to SNN_E_CUDA, NCCL errors to SNN_E_NCCL.
 *   - Ownership: the handle owns every DEVICE buffer it allocates (through the
 *     dev_alloc/dev_free hooks when given, e.g. PyTorch's caching allocator,
 *     else cudaMalloc) and frees them in snn_destroy.  Parameter structs are
 *     copied at call time.  HOST buffers passed in (host_dst) stay owned by the
 *     caller.
 *   - Lifecycle: CONFIG (add_population / connect allowed) -> FINALIZED by the
 *     first snn_step (graph construction = setup) -> RUNNING.
 *     add_population / connect after that return SNN_E_STATE.
 *   - Threading: a handle is not thread-safe; use one handle per (process, GPU).
 *   - All device work is enqueued on cfg.stream (a borrowed cudaStream_t;
 *     NULL = the legacy default stream).
 *   - world > 1: every rank makes the identical call sequence (collective
 *     semantics, like NCCL).  Rank r owns the target-neuron range given by
 *     snn_read_state(SNN_FIELD_INFO) (tgt_lo, tgt_hi); see DESIGN.md section 7.
 */
#ifndef SNN_H
#define SNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNN_ABI_VERSION 4u

typedef struct snn_sim snn_sim; /* opaque; owned by the library */
typedef int32_t snn_status;

enum {
    SNN_OK = 0,
    SNN_E_INVALID = -1,     /* bad argument: p outside [0,1], n == 0, D > 62,
                               slice width not a multiple of 32 in [32, 32768],
                               fixed-point overflow bound violated, ...      */
    SNN_E_STATE = -2,       /* call not allowed in the handle's lifecycle state */
    SNN_E_OOM = -3,         /* device allocation failed                        */
    SNN_E_CUDA = -4,        /* a CUDA runtime error (text in snn_last_error)   */
    SNN_E_NCCL = -5,        /* an NCCL error                                   */
    SNN_E_UNSUPPORTED = -6  /* valid but not implemented (e.g. 2 STDP
                               projections from one source population, or
                               world > 1 with delay 0)                         */
};

/* population kinds (R9): */
enum {
    SNN_POP_POISSON = 0,    /* Bernoulli(rate*dt) per step from Philox, no inputs */
    SNN_POP_LIF_DELTA = 1,  /* Brunel 2000 model A: delta-current LIF, 1 receptor */
    SNN_POP_LIF_CUBA = 2    /* Vogels-Abbott CUBA: exc/inh exponential currents   */
};
/* synapse kinds: */
enum { SNN_SYN_STATIC = 0, SNN_SYN_STDP = 1 };
/* receptors: */
enum { SNN_RCPT_EXC = 0, SNN_RCPT_INH = 1 };

/* plasticity schedules (the paper's ablation, Fig. 2 / P:362,
   P:399); all three compute the same weights (the naive sweep of Fig. 2a): */
enum {
    SNN_PLAST_EVENT = 0,    /* Fig. 2c: lazy + event-driven (default)            */
    SNN_PLAST_LAZY = 1,     /* Fig. 2b: lazy, every synapse of a visited row is
                               replayed step by step over its window (no bitmap
                               filter, no skipping of empty steps)             */
    SNN_PLAST_NAIVE = 2     /* Fig. 2a schedule: every plastic row is visited
                               (streamed and updated) every step               */
};
/* delivery kernels (Fig. 3): */
enum {
    SNN_DELIV_SLICED = 0,   /* Fig. 3b: neuron-domain slices, shared atomics     */
    SNN_DELIV_ROWWISE = 1   /* Fig. 3a: a warp per arriving row, global atomics  */
};

/* config flags */
enum {
    SNN_FLAG_NO_GRAPH = 1u << 0,     /* launch kernels directly instead of replaying
                                        a captured CUDA graph of the step          */
    SNN_FLAG_PHASE_TIMING = 1u << 1, /* record CUDA events around every phase of
                                        every step (implies NO_GRAPH); read with
                                        SNN_FIELD_PHASE_TIMES                       */
    SNN_FLAG_TRACE = 1u << 2,        /* debug: per-CTA %globaltimer phase marks of
                                        the last step (implies NO_GRAPH); read with
                                        SNN_FIELD_TRACE                             */
    SNN_FLAG_NO_PDL = 1u << 3,       /* no programmatic dependent launch between
                                        the kernels of a step                       */
    SNN_FLAG_KTIME = 1u << 5,        /* kernel spans inside the graph-replayed step:
                                        every CTA folds %globaltimer marks into its
                                        step's slot (entry, end of the dependency
                                        wait, end); read with SNN_FIELD_KTIME      */
    SNN_FLAG_EXCHANGE = 1u << 6,     /* run the spike-word exchange (ncclAllGather +
                                        unpack, on its graph branch) even at world ==
                                        1 -- a one-GPU run of the NCCL data path;
                                        needs nccl_unique_id                          */
    SNN_FLAG_IDX16 = 1u << 4         /* compressed indices:
                                        delivery reads 16-bit slice-local target
                                        offsets (j - slice base) instead of 32-bit
                                        ids -- 6 instead of 8 B per event; the
                                        32-bit ids stay for STDP and read-out      */
};

typedef struct {
    uint32_t abi_version;    /* must be SNN_ABI_VERSION                          */
    uint32_t struct_size;    /* sizeof(snn_config)                                */
    float dt_ms;             /* step length; 0.1 ms in the paper          */
    uint32_t delay_steps;    /* network-wide delay D in steps; D <= 62    */
    uint32_t history_bits;   /* H: 64 or 128 ("64 to 128"):
                                  forced flush at age H; 128 halves the flush work  */
    uint32_t slice_width;    /* C: neurons per slice; multiple of 32
                                in [32, 32768]; 0 = automatic                      */
    int32_t accum_frac_bits; /* F: fixed-point fraction bits of the int32 input
                                accumulators (R18); 0..30, default 20   */
    uint32_t flags;          /* SNN_FLAG_*                                        */
    uint64_t seed;           /* Philox key = (seed & 0xffffffff, seed >> 32)      */
    int32_t device;          /* CUDA device ordinal                               */
    int32_t rank, world;     /* this process' rank and the number of ranks (GPUs) */
    void *stream;            /* cudaStream_t, borrowed                            */
    /* optional device allocator hooks (e.g. torch caching allocator); both NULL
       -> cudaMalloc / cudaFree.  dev_alloc returns NULL on failure.            */
    void *(*dev_alloc)(size_t bytes, void *stream, void *ctx);
    void (*dev_free)(void *ptr, void *stream, void *ctx);
    void *alloc_ctx;
    /* world > 1: the 128-byte ncclUniqueId, identical on all ranks (the caller
       broadcasts it, e.g. with torch.distributed); the library then exchanges
       the spike words with ncclAllGather (libnccl.so.2 is loaded at run time).
       Ignored when world == 1.                                                  */
    const void *nccl_unique_id;
    /* world > 1 without NCCL: a non-zero key shared by the `world` handles of
       one process, which then exchange by device copies on the same GPU (a
       test transport: partitions of one network on one GPU, stepped in
       lockstep by the caller).                                                 */
    uint64_t group_key;
    uint32_t plasticity;     /* SNN_PLAST_* (ablation; results identical)        */
    uint32_t delivery;       /* SNN_DELIV_* (ablation; results identical)        */
    uint32_t flush_period;   /* forced-flush schedule (R3, R33): 0 = a
                                row is flushed when its age reaches H (the
                                paper's); K in [1, H/2] = every K steps, all rows
                                of age >= H - K at once (same results: any
                                schedule with age <= H is exact, R4), so the
                                flushes stream as one bulk pass               */
    uint32_t exchange_window;/* world > 1: steps of spike words gathered per
                                exchange (W; 0 = automatic).  W = 1 when D <= 1;
                                else 1 <= W <= D - 1, and the exchange of a window
                                overlaps the next steps' compute (DESIGN.md
                                section 7)                                      */
} snn_config;

typedef struct {
    uint32_t struct_size;    /* sizeof(snn_pop_params)                            */
    uint32_t kind;           /* SNN_POP_*                                         */
    float rate_hz;           /* POISSON: firing rate                              */
    float tau_m_ms;          /* LIF membrane time constant                        */
    float v_rest_mv;         /* CUBA leak reversal E_l (unused by LIF_DELTA: 0)   */
    float v_reset_mv;        /* reset potential; initial V ~ U[v_reset, v_th)      */
    float v_th_mv;           /* threshold: fire iff V >= v_th (R20)               */
    float tau_ref_ms;        /* refractory period, rounded to steps               */
    float tau_e_ms, tau_i_ms;/* CUBA receptor time constants                      */
} snn_pop_params;

typedef struct {
    uint32_t struct_size;    /* sizeof(snn_syn_params)                            */
    uint32_t kind;           /* SNN_SYN_STATIC | SNN_SYN_STDP                     */
    uint32_t receptor;       /* SNN_RCPT_*; LIF_DELTA targets accept only EXC     */
    uint32_t allow_autapses; /* 0: no i -> i synapse (R21)                        */
    double p;                /* connection probability in [0, 1]: each ordered
                                pair is a synapse independently with probability
                                p, realised by exact geometric skipping over
                                Philox draws (R32)                      */
    float weight;            /* initial weight, FINAL value (caller scales, R10)  */
    float tau_plus_ms, tau_minus_ms; /* STDP trace time constants (R7)            */
    float a_plus, a_minus;   /* STDP amplitudes (additive rule, R7)               */
    float w_max;             /* STDP hard upper bound; lower bound is 0           */
} snn_syn_params;

/* fields for snn_read_state (element type / count in brackets).  Neuron
 * fields cover the population pop_id; pop_id = UINT32_MAX means all N neurons.
 * Synapse fields are in CSR order of this rank's graph. */
enum {
    SNN_FIELD_V = 0,            /* [f32 / n]   membrane potential               */
    SNN_FIELD_REFRACTORY = 1,   /* [i32 / n]   remaining refractory steps       */
    SNN_FIELD_G_EXC = 2,        /* [f32 / n]   CUBA exc current                 */
    SNN_FIELD_G_INH = 3,        /* [f32 / n]   CUBA inh current                 */
    SNN_FIELD_INPUT_EXC = 4,    /* [i32 / n]   pending fixed-point input, exc   */
    SNN_FIELD_INPUT_INH = 5,    /* [i32 / n]   pending fixed-point input, inh   */
    SNN_FIELD_HIST = 6,         /* [u64 / n]   64-bit firing history of
                                   every neuron, rebuilt from the bitmask ring   */
    SNN_FIELD_SPIKE_COUNT = 7,  /* [u32 / n]   spikes since start               */
    SNN_FIELD_XPOST = 8,        /* [f32 / n]   post-synaptic trace per neuron   */
    SNN_FIELD_XPRE_ROW = 9,     /* [f32 / n]   pre-synaptic trace per source row (after flush) */
    SNN_FIELD_TLU = 10,         /* [i32 / n]   timeOfLastUpdate per row (after flush) */
    SNN_FIELD_ROW_PTR = 11,     /* [i64 / N+1] CSR row offsets                  */
    SNN_FIELD_IDX = 12,         /* [u32 / S]   CSR target ids                   */
    SNN_FIELD_WEIGHTS = 13,     /* [f32 / S]   weights, after the read-out flush (R11) */
    SNN_FIELD_PIVOTS = 14,      /* [u32 / N*(nslices+1)] row-relative pivots    */
    SNN_FIELD_STEP = 15,        /* [i64 / 1]   number of steps simulated        */
    SNN_FIELD_METRICS = 16,     /* [u64 / 16]  see SNN_METRIC_*                 */
    SNN_FIELD_SPIKE_RING = 17,  /* [u32 / 64*ceil(N/32)] bitmask ring; slot t%64
                                   holds the spikes of step t                    */
    SNN_FIELD_PHASE_TIMES = 18, /* [f64 / 8]  ms per phase (SNN_PHASE_*), summed
                                   over steps run with SNN_FLAG_PHASE_TIMING     */
    SNN_FIELD_INFO = 19,        /* [i64 / 8]  N, S, nslices, C, R, tgt_lo, tgt_hi,
                                   (delivery splits << 32) | STDP grid          */
    SNN_FIELD_TRACE = 20,       /* [u64 / 4*4096*4] debug phase marks (ns) of the
                                   last step: [kernel][cta][phase], kernels
                                   front / stdp / deliver                        */
    SNN_FIELD_IDX16 = 21,       /* [u16 / S]   slice-local target offsets
                                   (j - tgt_lo) mod 2^16 (SNN_FLAG_IDX16 only)   */
    SNN_FIELD_HIST_DEV = 22,    /* [u64 / n]   the device history word, bits 0-63
                                   (bit s: spike at step t - s), that k_stdp
                                   reads; maintained for neurons post-synaptic
                                   to STDP (0 elsewhere)                         */
    SNN_FIELD_HIST_DEV_HI = 23, /* [u64 / n]   bits 64-127 (history_bits = 128)  */
    SNN_FIELD_FPOT = 24,        /* [f32 / n]   post-plastic neuron with spikes in
                                   its H-bit window: the forced-flush factor, the
                                   sum over those spikes s (oldest first) of
                                   D+[H - s] = fp32(exp(-(H - s) dt / tau_+))
                                   (stale elsewhere)                             */
    SNN_FIELD_RECENT = 25,      /* [u32 / ceil(N/32)] bit j: post-plastic neuron
                                   j fired in the last H steps                   */
    SNN_FIELD_KTIME = 26,       /* [u64 / 20] per kernel k (front, stdp, deliver,
                                   spare, lists): [4k] sum over steps of (last CTA end -
                                   first CTA entry) ns, [4k+1] sum of (last end -
                                   first return from the dependency wait) ns,
                                   [4k+2] steps, [4k+3] CTAs; cumulative
                                   (SNN_FLAG_KTIME; read at least every 65,536
                                   steps)                                       */
    SNN_FIELD_FPOS = 27,        /* [u8 / n]    post-plastic neuron: 0xfe no spike
                                   in its H-bit window, 0xff several, else the
                                   bit index of the only one                     */
    SNN_FIELD_COUNT = 28
};

/* SNN_FIELD_METRICS layout (device counters, cumulative over steps) */
enum {
    SNN_METRIC_EVENTS = 0,       /* delivered (arriving spike, target) pairs (R24) */
    SNN_METRIC_SPIKES = 1,       /* arriving spikes (rows delivered)               */
    SNN_METRIC_STDP_ROWS = 2,    /* plastic rows visited (arrivals + flushes)      */
    SNN_METRIC_STDP_SYN = 3,     /* plastic synapses visited                       */
    SNN_METRIC_STDP_WSTORE = 4,  /* plastic synapses whose weight changed (stored) */
    SNN_METRIC_FLUSH_ROWS = 5,   /* rows visited by a forced flush (R3)            */
    SNN_METRIC_SEGMENTS = 6,     /* non-empty (row, slice) segments processed      */
    SNN_METRIC_ELEMS = 7,        /* synapse entries read by the delivery kernel    */
    SNN_METRIC_STDP_WRW = 8,     /* visited plastic synapses whose weight the method
                                    must read and write: every
                                    synapse of an arriving row, and forced-flush
                                    synapses whose target fired in the window     */
    SNN_METRIC_FLUSH_SYN = 9,    /* of STDP_SYN: forced-flush synapses (event schedule) */
    SNN_METRIC_FLUSH_WRW = 10    /* of STDP_WRW: their window hits (the staged flush
                                    stream counts the hits that changed their weight:
                                    all but those already at w_max)               */
};

/* SNN_FIELD_PHASE_TIMES layout: the kernels of a step */
enum {
    SNN_PHASE_FRONT = 0,    /* neuron update + firing bits + work lists       */
    SNN_PHASE_STDP = 1,     /* lazy + event-driven STDP                       */
    SNN_PHASE_DELIVERY = 2, /* sliced shared-atomic delivery                  */
    SNN_PHASE_EXCHANGE = 3, /* spike-bitmask all-gather (world > 1)           */
    SNN_PHASE_TOTAL = 4,
    SNN_PHASE_BUILD = 5     /* graph construction on the GPU (count, scan, fill,
                               segments), device time of the last finalize; not
                               part of a step            */
};

/* Creates a simulation handle bound to cfg->device / cfg->stream.
 * out receives the handle (NULL on failure).  Errors: SNN_E_INVALID (bad cfg),
 * SNN_E_CUDA, SNN_E_NCCL (world > 1 communicator setup). */
snn_status snn_create(const snn_config *cfg, snn_sim **out);

/* Appends a population of n neurons; ids are contiguous in call order
 * (list populations that receive synapses first, so slices span only them).
 * pop_id receives its index.  Errors: SNN_E_INVALID (n == 0, bad kind or
 * parameters), SNN_E_STATE (after finalize). */
snn_status snn_add_population(snn_sim *sim, uint32_t n, const snn_pop_params *params,
                              uint32_t *pop_id);

/* Declares the projection src_pop -> dst_pop: every ordered pair (i, j) is a
 * synapse with probability p (geometric skipping over the counter-based Philox
 * stream (i, n >> 2, 4, dst_pop), R32), one projection per pair of
 * populations.  Errors: SNN_E_INVALID (p outside [0,1], POISSON target, bad
 * receptor, duplicate projection, STDP weight outside [0, w_max]),
 * SNN_E_UNSUPPORTED (second STDP projection from one source population),
 * SNN_E_STATE. */
snn_status snn_connect(snn_sim *sim, uint32_t src_pop, uint32_t dst_pop,
                       const snn_syn_params *params);

/* Enqueues n_steps simulation steps on cfg->stream (asynchronous).  The first
 * call finalizes: it builds the sliced CSR graph and the initial state on the
 * device (setup).  n_steps == 0 only finalizes.  Errors: SNN_E_INVALID
 * (fixed-point overflow bound, empty network), SNN_E_OOM, SNN_E_CUDA,
 * SNN_E_NCCL. */
snn_status snn_step(snn_sim *sim, uint32_t n_steps);

/* Copies a state field (SNN_FIELD_*) of population pop_id (UINT32_MAX = all
 * neurons; ignored for synapse / global fields) into the caller's HOST buffer
 * host_dst of dst_bytes bytes, synchronising cfg->stream.  If host_dst is
 * NULL, only *needed (bytes required) is written.  Reading WEIGHTS, XPRE_ROW
 * or TLU first brings every stale plastic row up to the current step without a
 * pre spike (read-out flush, R11), which does not change future results.
 * Errors: SNN_E_INVALID (unknown field / pop, dst_bytes too small),
 * SNN_E_STATE (before finalize), SNN_E_CUDA. */
snn_status snn_read_state(snn_sim *sim, uint32_t field, uint32_t pop_id, void *host_dst,
                          size_t dst_bytes, size_t *needed);

/* Like snn_read_state, for elements [first, first + count) of the field (pop
 * fields: relative to the population's first neuron; SPIKE_RING: slot-major,
 * ceil(N/32) words per slot).  Sampled checks of networks with 2^32+ synapses
 * read a few rows instead of the whole array.  Errors: SNN_E_INVALID (range
 * outside the field, dst_bytes < count * element size, NULL host_dst), and
 * those of snn_read_state. */
snn_status snn_read_state_range(snn_sim *sim, uint32_t field, uint32_t pop_id, uint64_t first, uint64_t count,
                                void *host_dst, size_t dst_bytes);

/* Releases every device buffer, graph, event and communicator of the handle. */
void snn_destroy(snn_sim *sim);

/* The message of the last failed call on sim (or of the last failed
 * snn_create when sim is NULL).  Valid until the next call on the handle. */
const char *snn_last_error(const snn_sim *sim);

/* The ABI version the library was built with (SNN_ABI_VERSION). */
uint32_t snn_abi_version(void);

/* Host-only helper (no device work): the target range [*lo, *hi) of `rank`
 * among `world` ranks for n_targets neurons with inputs and slice width C --
 * C-aligned equal shares, the last one truncated (the
 * partition of the neuron domain of P:48 / P:348).  Errors: SNN_E_INVALID
 * (world == 0, rank >= world, C not a multiple of 32, NULL outputs). */
snn_status snn_partition(uint32_t n_targets, uint32_t slice_width, uint32_t world, uint32_t rank, uint32_t *lo,
                         uint32_t *hi);

/* The partition the library uses: rank `rank`'s range
 * [*lo, *hi) of [0, n_targets), contiguous and C-aligned, with boundaries at
 * the slice prefixes closest to r / world of the total expected work
 * (`slice_cost[k]` >= 0: the expected per-step bytes of slice k = targets
 * [kC, (k+1)C), host memory, owned by the caller; the engine uses the
 * SURVEY 8(d) byte model).  Ranks may get unequal neuron counts -- e.g. the
 * plastic (E) targets, whose forced flushes dominate, are spread over more
 * ranks.  Every rank computes every range identically (deterministic, host
 * only).  Errors: SNN_E_INVALID (world == 0, rank >= world, C not a positive
 * multiple of 32, nslices * C < n_targets, a negative or NaN cost, NULL
 * pointers). */
snn_status snn_partition_weighted(const double *slice_cost, uint32_t nslices, uint32_t n_targets,
                                  uint32_t slice_width, uint32_t world, uint32_t rank, uint32_t *lo, uint32_t *hi);

#ifdef __cplusplus
}
#endif
#endif /* SNN_H */
