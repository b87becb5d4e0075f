// engine.cu -- libsnn.so: the C ABI of include/snn.h, the per-handle state, the
// setup (graph construction) and the step orchestration:
//   per step t:  k_neuron -> k_worklist -> k_stdp (if plastic) -> k_deliver
// replayed from a captured CUDA graph of kGraphSteps steps.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <iterator>
#include <map>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/snn.h"
#include "common.cuh"

namespace snn {
cudaError_t build_preload(cudaStream_t);
cudaError_t build_count(const NetDev &, const BuildTabs &, uint32_t *, int64_t *, cudaStream_t);
cudaError_t build_scan(const NetDev &, uint32_t *, int64_t *, int64_t *, void *, size_t *, cudaStream_t);
cudaError_t build_fill(const NetDev &, const BuildTabs &, const uint32_t *, const int64_t *, uint32_t *,
                       float *, cudaStream_t);
cudaError_t build_segments(const NetDev &, const int64_t *, const uint32_t *, uint2 *, cudaStream_t);
cudaError_t init_state(const NetDev &, const StateDev &, cudaStream_t);
cudaError_t build_idx16(const NetDev &, const uint32_t *, uint16_t *, int64_t, cudaStream_t);
cudaError_t build_b64(const NetDev &, const int64_t *, const uint32_t *, uint32_t *, cudaStream_t);
uint32_t front_blocks(const NetDev &);
cudaError_t launch_front(const NetDev &, const StateDev &, cudaStream_t, bool, bool, int, bool);
size_t stdp_smem_bytes(const NetDev &, uint32_t, uint32_t);
size_t deliver_smem_bytes(const NetDev &, bool);
cudaError_t kernels_configure(int);
cudaError_t launch_kspan_reset(KSpan *, cudaStream_t);
cudaError_t launch_stdp(const NetDev &, const StateDev &, int64_t, uint32_t, uint32_t, uint32_t, cudaStream_t, bool);
cudaError_t launch_deliver_rowwise(const NetDev &, const StateDev &, uint32_t, cudaStream_t, bool);
cudaError_t launch_stdp_ev(const NetDev &, const StateDev &, uint32_t, uint32_t, uint32_t, cudaStream_t, bool, int);
uint32_t flush_ctas_per_sm();
void set_launch_priority(int);
size_t ev_smem_bytes(uint32_t, uint32_t);
size_t flush_smem_bytes(uint32_t, uint32_t);
cudaError_t launch_deliver(const NetDev &, const StateDev &, uint32_t, cudaStream_t, bool, bool, bool);
cudaError_t launch_readout(const NetDev &, const StateDev &, int64_t, uint32_t, uint32_t, uint32_t, cudaStream_t, bool);
cudaError_t launch_hist_from_ring(const NetDev &, const uint32_t *, int64_t, uint64_t *, cudaStream_t);
cudaError_t launch_unpack(const NetDev &, const StateDev &, const uint32_t *, int64_t, cudaStream_t);
}  // namespace snn

using namespace snn;

namespace {

constexpr uint32_t kGraphSteps = 64;
std::string g_create_error;

// NCCL, loaded at run time (only world > 1 with an ncclUniqueId needs it)
struct NcclApi {
    void *lib = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_mu;
std::map<uint64_t, std::vector<snn_sim *>> g_groups;   // local-group transport

bool load_nccl(std::string &err) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_nccl.lib) return true;
    const char *names[] = {getenv("SNN_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
        if (!n) continue;
        g_nccl.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.lib) break;
    }
    if (!g_nccl.lib) {
        err = "cannot load libnccl.so.2 (set SNN_NCCL_LIB or import torch first)";
        return false;
    }
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(g_nccl.lib, "ncclCommInitRank");
    g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(g_nccl.lib, "ncclAllGather");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(g_nccl.lib, "ncclCommDestroy");
    g_nccl.errorString = (decltype(g_nccl.errorString))dlsym(g_nccl.lib, "ncclGetErrorString");
    if (!g_nccl.commInitRank || !g_nccl.allGather || !g_nccl.commDestroy || !g_nccl.errorString) {
        err = "libnccl is missing symbols";
        return false;
    }
    return true;
}

struct HostPop {
    snn_pop_params prm;
    uint32_t base, n;
};
struct HostProj {
    uint32_t src, dst;
    snn_syn_params prm;
};

}  // namespace

struct snn_sim {
    snn_config cfg{};
    std::string err;
    int state = 0;  // 0 CONFIG, 1 FINALIZED
    std::vector<HostPop> pops;
    std::vector<HostProj> projs;
    NetDev net{};
    StateDev st{};
    uint32_t N = 0;
    int64_t nsyn = 0;
    int64_t t = 0;  // steps enqueued so far
    int64_t readout_t = -1;              // the step of the last read-out flush (R11)
    cudaStream_t stream = nullptr, cap_stream = nullptr;
    // the ahead step: k_front(t) builds the arrival list
    // of t+1, k_deliver(t) runs the plastic arrivals' STDP, k_flush(t) the
    // forced flushes after it
    bool ahead = false;
    // the fused step (captured graphs of the ahead step, world 1): k_deliver(t)'s
    // epilogue updates the neurons of t + 1; k_front(t+1) (neurons >= R, lists)
    // and k_flush on branches -- DESIGN.md section 2
    bool fused = false;
    cudaStream_t cap_front = nullptr;
    cudaEvent_t ev_fr[2] = {nullptr, nullptr}, ev_del[2] = {nullptr, nullptr}, ev_fl_f[2] = {nullptr, nullptr};
    cudaEvent_t ev_lif[2] = {nullptr, nullptr};
    // the split step (a variant of the fused graph): k_deliver without the
    // epilogue, the neurons [0, R) of t in a slim k_front (kPart 4) on the
    // critical path, the rest of k_front (neurons >= R, lists) on a branch
    bool split_front = false;
    uint32_t flush_grid = 1, flush_grid_side = 1;   // k_flush CTAs: serial step / side branch
    // step graph (SNN_PIPE, experiments): 0 serial; 1 ahead + k_flush(t) on a
    // side branch joined before k_deliver(t + fl_lag); 2 no ahead list, k_stdp_arr
    // + k_flush(t) on a side branch joined before k_stdp_arr(t+1)
    int pipe = 0, fl_lag = 2, prio_hi = 0, prio_lo = 0;
    bool use_prio = false;
    cudaStream_t cap_side = nullptr;
    cudaEvent_t ev_front = nullptr, ev_flush[4] = {nullptr, nullptr, nullptr, nullptr};
    // world > 1, D >= 1: the exchange of step t on a branch of the step graph
    // (after k_front(t), joined before k_front(t+1)), overlapping the delivery
    cudaStream_t cap_xside = nullptr;
    cudaEvent_t ev_xfront = nullptr, ev_xdone = nullptr;
    // captured step graphs by step count (<= kGraphSteps): a call of n steps
    // replays ceil(n / 64) graphs, so a step's side branch is joined once per call
    std::map<uint32_t, cudaGraphExec_t> graphs;
    std::vector<void *> allocs;
    uint32_t splits = 1;                 // k_deliver CTAs per slice
    uint32_t stdp_grid = 1;              // k_stdp CTAs
    uint32_t pp_lo = 0, pp_hi = 0;       // post-plastic neuron range (bitmap span)
    bool plastic = false;
    bool ev_kernel = false;              // event schedule, flushes at age H: k_stdp_ev
    uint64_t *d_hist_tmp = nullptr;
    // kernel spans (SNN_FLAG_KTIME): device slots, host totals per kernel:
    // [sum(end - entry) ns, sum(end - wait) ns, steps, CTAs]
    KSpan *kspan = nullptr;
    unsigned long long ks_tot[kKSpanKernels][4] = {{0}};
    // exchange (world > 1)
    uint32_t wmax = 0;
    ncclComm_t comm = nullptr;
    bool local_group = false;
    // phase timing
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::vector<cudaEvent_t>> ev_steps;  // per step: 5 boundary events (front, STDP, delivery, flushes)
    size_t ev_used = 0;
    double phase_ms[8] = {0};

    snn_status fail(snn_status code, const char *fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return code;
    }
    void *dalloc(size_t bytes) {
        if (bytes == 0) bytes = 16;
        bytes = (bytes + 255) & ~(size_t)255;
        void *p = nullptr;
        if (cfg.dev_alloc) {
            p = cfg.dev_alloc(bytes, (void *)stream, cfg.alloc_ctx);
        } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
        }
        if (p) allocs.push_back(p);
        return p;
    }
};

#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return sim->fail(SNN_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                             __FILE__, __LINE__);                                             \
    } while (0)

#define ALLOC(ptr, type, count)                                                            \
    do {                                                                                   \
        ptr = (type *)sim->dalloc(sizeof(type) * (size_t)(count));                         \
        if (!ptr) return sim->fail(SNN_E_OOM, "device allocation of %zu bytes failed",     \
                                   sizeof(type) * (size_t)(count));                        \
    } while (0)

// Every entry point runs on the handle's device and restores the caller's
// current device on return.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != dev) {
            err = cudaSetDevice(dev);
            if (err == cudaSuccess) prev = cur;
        } else {
            cudaGetLastError();
        }
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

static uint64_t bernoulli_thr(double p) {
    if (!(p > 0.0)) return 0;
    if (p >= 1.0) return 1ull << 32;
    return (uint64_t)std::floor(p * 4294967296.0);
}

// ------------------------------------------------------------------ exchange
static snn_status exchange_setup(snn_sim *sim) {
    const snn_config &cfg = sim->cfg;
    if (cfg.nccl_unique_id) {
        std::string err;
        if (!load_nccl(err)) return sim->fail(SNN_E_NCCL, "%s", err.c_str());
        ncclUniqueId id;
        memcpy(&id, cfg.nccl_unique_id, sizeof id);
        const ncclResult_t r = g_nccl.commInitRank(&sim->comm, cfg.world, id, cfg.rank);
        if (r != ncclSuccess) return sim->fail(SNN_E_NCCL, "ncclCommInitRank: %s", g_nccl.errorString(r));
        return SNN_OK;
    }
    sim->local_group = true;
    return SNN_OK;
}

// The step's exchange: this rank's share of spike words to every rank.
// NCCL: all-gather into gath[0] and unpack into the ring within the step (the
// ranks run concurrently; graph-capturable, fixed addresses).  Local group:
// copy into every peer's gath[t & 1]; each peer unpacks it at the start of its
// step t + 1 (the caller steps the peers in lockstep, so the parity double
// buffer keeps step t's words until then).
static snn_status exchange_enqueue(snn_sim *sim, cudaStream_t s, int64_t t) {
    const StateDev &st = sim->st;
    const snn_config &cfg = sim->cfg;
    if (sim->comm) {
        const ncclResult_t r = g_nccl.allGather(st.sendbuf, st.gath, sim->wmax, ncclUint32, sim->comm, s);
        if (r != ncclSuccess) return sim->fail(SNN_E_NCCL, "ncclAllGather: %s", g_nccl.errorString(r));
        CK(launch_unpack(sim->net, st, st.gath, -1, s));
        return SNN_OK;
    }
    std::vector<snn_sim *> peers;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        peers = g_groups[cfg.group_key];
    }
    if ((int)peers.size() != cfg.world)
        return sim->fail(SNN_E_STATE, "local group %llu has %zu of %d ranks", (unsigned long long)cfg.group_key,
                         peers.size(), cfg.world);
    for (snn_sim *p : peers) {
        if (p->state == 0 || !p->st.gath) return sim->fail(SNN_E_STATE, "local group peer not finalized");
        CK(cudaMemcpyAsync(p->st.gath + ((size_t)(t & 1) * cfg.world + cfg.rank) * sim->wmax, st.sendbuf,
                           4ull * sim->wmax, cudaMemcpyDeviceToDevice, s));
    }
    return SNN_OK;
}

// --------------------------------------------------------------------- setup
// Expected per-step HBM bytes of each slice of C targets of [0, R) -- the
// SURVEY 8(d) byte model, per synapse into the slice: a delivered event 8 B x
// nu_src dt; a plastic synapse adds its arrival's STDP (8 B x nu_src dt) and
// its forced flush (4 B / H).  nu_src: the Poisson rate, 10 Hz for LIF sources
// (8(d)'s nominal rate).  Used to balance the ranks' target ranges.
static std::vector<double> slice_costs(const snn_sim *sim, uint32_t R, uint32_t C, uint32_t H) {
    const double dt = sim->cfg.dt_ms * 1e-3;
    std::vector<double> per_neuron(sim->pops.size(), 0.0);
    for (const HostProj &hj : sim->projs) {
        const HostPop &src = sim->pops[hj.src];
        const double nu = src.prm.kind == SNN_POP_POISSON ? (double)src.prm.rate_hz : 10.0;
        double b = 8.0 * nu * dt;
        if (hj.prm.kind == SNN_SYN_STDP) b += 8.0 * nu * dt + 4.0 / (double)H;
        per_neuron[hj.dst] += hj.prm.p * (double)src.n * b;
    }
    const uint32_t ns = (R + C - 1) / C;
    std::vector<double> cost(ns, 0.0);
    for (size_t k = 0; k < sim->pops.size(); k++) {
        const uint64_t a = sim->pops[k].base, e = std::min<uint64_t>(R, a + sim->pops[k].n);
        for (uint64_t s0 = a; s0 < e;) {                 // the population's overlap with each slice
            const uint64_t sl = s0 / C, s1 = std::min<uint64_t>(e, (sl + 1) * C);
            cost[sl] += (double)(s1 - s0) * per_neuron[k];
            s0 = s1;
        }
    }
    return cost;
}

static snn_status finalize(snn_sim *sim) {
    const snn_config &cfg = sim->cfg;
    if (sim->pops.empty()) return sim->fail(SNN_E_INVALID, "no populations");
    NetDev &net = sim->net;
    memset(&net, 0, sizeof net);
    const double dt = cfg.dt_ms;
    net.npop = (uint32_t)sim->pops.size();
    net.N = sim->N;
    net.D = cfg.delay_steps;
    net.H = cfg.history_bits;
    net.flush_period = cfg.flush_period;
    net.plast_mode = cfg.plasticity;
    net.deliv_mode = cfg.delivery;
    net.F = cfg.accum_frac_bits;
    net.scale = std::ldexp(1.0f, net.F);
    net.inv_scale = std::ldexp(1.0f, -net.F);
    net.key0 = (uint32_t)(cfg.seed & 0xffffffffu);
    net.key1 = (uint32_t)(cfg.seed >> 32);
    for (int a = 0; a < kMaxPops; a++)
        for (int b = 0; b < kMaxPops; b++) net.rcpt[a][b] = -1;
    BuildTabs tabs;
    memset(&tabs, 0, sizeof tabs);
    for (int k = 0; k < kMaxPops * kMaxPops; k++) tabs.gap_slot[k] = -1;
    std::vector<uint32_t> gap_host;               // R32: floor((1-p)^k 2^32), k = 1..kGapTab, per projection
    uint32_t R = 0;
    for (uint32_t k = 0; k < net.npop; k++) {
        const HostPop &hp = sim->pops[k];
        PopDev &p = net.pop[k];
        p.base = hp.base;
        p.n = hp.n;
        p.kind = hp.prm.kind;
        p.stdp = -1;
        p.post_stdp = -1;
        p.rcpt_uniform = -2;  // unset
        p.thr = bernoulli_thr((double)hp.prm.rate_hz * 1e-3 * dt);
        p.k_m = (float)(1.0 - dt / (double)hp.prm.tau_m_ms);
        p.a_m = (float)(dt / (double)hp.prm.tau_m_ms);
        p.d_e = (float)std::exp(-dt / (double)hp.prm.tau_e_ms);
        p.d_i = (float)std::exp(-dt / (double)hp.prm.tau_i_ms);
        p.v_th = hp.prm.v_th_mv;
        p.v_reset = hp.prm.v_reset_mv;
        p.v_rest = hp.prm.v_rest_mv;
        p.n_ref = (int32_t)std::llround((double)hp.prm.tau_ref_ms / dt);
    }
    // projections
    double acc_bound[kMaxPops][2] = {{0}};
    for (const HostProj &hj : sim->projs) {
        const snn_syn_params &q = hj.prm;
        PopDev &sp = net.pop[hj.src];
        PopDev &dp = net.pop[hj.dst];
        net.rcpt[hj.src][hj.dst] = (int8_t)q.receptor;
        sp.rcpt_uniform = (sp.rcpt_uniform == -2 || sp.rcpt_uniform == (int32_t)q.receptor) ? (int32_t)q.receptor : -1;
        dp.flags |= PF_HAS_INPUT;
        R = std::max(R, dp.base + dp.n);
        tabs.thr[hj.src * kMaxPops + hj.dst] = bernoulli_thr(q.p);
        tabs.autapse[hj.src * kMaxPops + hj.dst] = q.allow_autapses ? 1 : 0;
        tabs.weight[hj.src * kMaxPops + hj.dst] = q.weight;
        if (q.p > 0.0) {
            tabs.inv_l2q[hj.src * kMaxPops + hj.dst] = q.p < 1.0 ? (float)(1.0 / std::log2(1.0 - q.p)) : -0.0f;
            tabs.gap_slot[hj.src * kMaxPops + hj.dst] = (int16_t)(gap_host.size() / kGapTab);
            for (int k = 1; k <= kGapTab; k++) {
                const double v = std::floor(std::pow(1.0 - q.p, (double)k) * 4294967296.0);
                gap_host.push_back(v >= 4294967295.0 ? 4294967295u : (uint32_t)v);
            }
        }
        double wabs = std::fabs((double)q.weight);
        if (q.kind == SNN_SYN_STDP) {
            if (net.nstdp >= 4) return sim->fail(SNN_E_UNSUPPORTED, "at most 4 STDP projections");
            StdpDev &sd = net.stdp[net.nstdp];
            sd.dst_pop = hj.dst;
            sd.a_plus = q.a_plus;
            sd.a_minus = q.a_minus;
            sd.w_max = q.w_max;
            for (int n = 0; n <= kMaxHist; n++) sd.dplus[n] = (float)std::exp(-(double)n * dt / (double)q.tau_plus_ms);
            const float dm = (float)std::exp(-dt / (double)q.tau_minus_ms);
            if ((dp.flags & PF_POST_PLASTIC) && dp.d_minus != dm)
                return sim->fail(SNN_E_UNSUPPORTED, "STDP projections into one population must share tau_minus");
            // the forced-flush factor of a target (k_front) uses one D+ table per population
            if ((dp.flags & PF_POST_PLASTIC) &&
                memcmp(net.stdp[dp.post_stdp].dplus, sd.dplus, sizeof sd.dplus) != 0)
                return sim->fail(SNN_E_UNSUPPORTED, "STDP projections into one population must share tau_plus");
            if (!(dp.flags & PF_POST_PLASTIC)) dp.post_stdp = (int32_t)net.nstdp;
            dp.flags |= PF_POST_PLASTIC;
            dp.d_minus = dm;
            sp.flags |= PF_PRE_PLASTIC;
            sp.stdp = (int32_t)net.nstdp++;
            wabs = std::max(wabs, std::fabs((double)q.w_max));
        }
        // fixed-point overflow bound (R18): expected in-degree + 10 sigma
        const double k = q.p * (double)sim->pops[hj.src].n;
        const double kmax = std::min((double)sim->pops[hj.src].n, k + 10.0 * std::sqrt(k) + 10.0);
        acc_bound[hj.dst][q.receptor] += kmax * std::ldexp(wabs, net.F);
    }
    for (uint32_t k = 0; k < net.npop; k++) {
        if (net.pop[k].rcpt_uniform == -2) net.pop[k].rcpt_uniform = 0;
        for (int r = 0; r < 2; r++)
            if (acc_bound[k][r] >= 2147483647.0)
                return sim->fail(SNN_E_INVALID,
                                 "fixed-point overflow bound: population %u receptor %d may reach %.3g >= 2^31 "
                                 "(lower accum_frac_bits)", k, r, acc_bound[k][r]);
    }
    net.R = R;
    net.nrcpt = 1;
    for (const HostProj &hj : sim->projs)
        if (hj.prm.receptor == SNN_RCPT_INH) net.nrcpt = 2;
    // slice width C of the delivery ("delicate, tunable"): the
    // paper's 1024 by default, shrunk so that each rank keeps >= ~64 slices
    // when its target range is small, and widened to a multiple of 32 when
    // 1024 would give just over one slice per SM (one CTA per slice: a few SMs
    // would deliver two slices and set the step's tail)
    uint32_t C = cfg.slice_width;
    if (C == 0) {
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg.device);
        const uint32_t Rr = (R + (uint32_t)cfg.world - 1) / (uint32_t)cfg.world;
        C = 1024;
        while (C > 128 && (Rr + C - 1) / C < 64) C >>= 1;
        const uint32_t ns = (Rr + C - 1) / C;
        if (ns > (uint32_t)nsm && ns < 2u * (uint32_t)nsm)
            C = 32u * ((Rr + 32u * (uint32_t)nsm - 1) / (32u * (uint32_t)nsm));
    }
    net.C = C;
    net.log2C = 0;   // (unused: C need not be a power of two)
    // this rank's target range: C-aligned contiguous
    // ranges of [0, R) with equal expected per-step work (snn_partition_weighted)
    if (cfg.world > kMaxRanks) return sim->fail(SNN_E_UNSUPPORTED, "world > %d", kMaxRanks);
    uint32_t lo = 0, hi = R;
    {
        const std::vector<double> cost = slice_costs(sim, R, C, cfg.history_bits);
        for (int r = 0; r <= cfg.world; r++) {
            uint32_t a = R, b = R;
            if (r < cfg.world)
                snn_partition_weighted(cost.data(), (uint32_t)cost.size(), R, C, (uint32_t)cfg.world, (uint32_t)r, &a, &b);
            net.rank_lo[r] = a;
            if (r == cfg.rank) {
                lo = a;
                hi = b;
            }
        }
    }
    if (cfg.world > 1) {
        for (uint32_t k = 0; k < net.npop; k++)
            if (net.pop[k].base < R && !(net.pop[k].flags & PF_HAS_INPUT))
                return sim->fail(SNN_E_INVALID, "world > 1: add populations that receive synapses first");
    }
    net.tgt_lo = lo;
    net.tgt_hi = hi;
    net.nslices = (net.tgt_hi - net.tgt_lo + C - 1) / C;
    net.nwords = (net.N + 31) / 32;
    sim->plastic = net.nstdp > 0;
    for (uint32_t k = 0; k < net.npop; k++)
        if (net.pop[k].flags & PF_PRE_PLASTIC) net.n_plastic_rows += net.pop[k].n;

    // ---- device buffers
    const uint32_t N = net.N;
    StateDev &st = sim->st;
    ALLOC(st.V, float, N);
    ALLOC(st.ge, float, N);
    ALLOC(st.gi, float, N);
    ALLOC(st.xpost, float, N);
    ALLOC(st.ref, int32_t, N);
    ALLOC(st.in_e, int32_t, N);
    ALLOC(st.in_i, int32_t, N);
    ALLOC(st.hist, uint64_t, N);
    ALLOC(st.hist_hi, uint64_t, cfg.history_bits > 64 ? N : 1);
    st.fstride = (N + 16 + 15) & ~15u;
    ALLOC(st.fpot, float, 12ull * st.fstride);        // [3][4]: flush factors for ages H, H-1, H-2, by t & 3
    ALLOC(st.fpos, uint8_t, 4ull * st.fstride);
    ALLOC(st.nspk, uint32_t, N);
    // exchange geometry: rank r owns words [rank_lo[r] / 32, ...), at most
    // (its share) / 32 + 1 of them (the word straddling R); every rank sends
    // wmax words (the largest share + 1); ring slots padded for the unpack
    net.world = (uint32_t)cfg.world;
    net.rank = (uint32_t)cfg.rank;
    {
        uint32_t mx = 1;
        for (int r = 0; r < cfg.world; r++) mx = std::max(mx, (net.rank_lo[r + 1] - net.rank_lo[r] + 31) / 32);
        net.wmax = mx + 1;
        sim->wmax = net.wmax;
    }
    net.xchg = (cfg.world > 1 || (cfg.flags & SNN_FLAG_EXCHANGE)) ? 1u : 0u;
    net.ring_stride = net.nwords + (net.xchg ? net.wmax : 0);
    ALLOC(st.ring, uint32_t, (size_t)kRingSlots * net.ring_stride);
    st.sendbuf = st.gath = nullptr;
    ALLOC(st.xpre, float, N);
    ALLOC(st.tlu, int32_t, N);
    ALLOC(st.row_ptr, int64_t, (size_t)N + 1);
    ALLOC(st.piv, uint32_t, (size_t)N * (net.nslices + 1));
    ALLOC(st.seg, uint2, N);
    st.nblk = front_blocks(net);
    const size_t nreg = (size_t)st.nblk * kFrontThreads;
    for (int b = 0; b < 4; b++) ALLOC(st.vdesc[b], RowDesc, net.nstdp ? nreg : 1);
    for (int b = 0; b < 2; b++) {
        ALLOC(st.adesc[b], RowDesc, nreg);
        ALLOC(st.vmask[b], uint32_t, net.nwords);
    }
    ALLOC(st.rdesc, RowDesc, net.nstdp ? nreg : 1);
    st.rstride = (net.nwords + 4 + 3) & ~3u;      // + the tail of its 16-byte bulk copy
    ALLOC(st.recent, uint32_t, 4ull * st.rstride);
    st.trace = nullptr;
    if (cfg.flags & SNN_FLAG_TRACE) {
        ALLOC(st.trace, unsigned long long, (size_t)kTraceKernels * kTraceCtas * 4);
        CK(cudaMemsetAsync(st.trace, 0, 8ull * kTraceKernels * kTraceCtas * 4, sim->stream));
    }
    ALLOC(st.ctr, Counters, 1);
    st.kspan = nullptr;
    if (cfg.flags & SNN_FLAG_KTIME) {
        ALLOC(st.kspan, KSpan, (size_t)kKSpanSlots * kKSpanKernels);
        CK(launch_kspan_reset(st.kspan, sim->stream));
        sim->kspan = st.kspan;
    }
    cudaStream_t s = sim->stream;
    CK(cudaMemsetAsync(st.ring, 0, sizeof(uint32_t) * (size_t)kRingSlots * net.ring_stride, s));
    if (net.xchg) {
        ALLOC(st.sendbuf, uint32_t, net.wmax);
        ALLOC(st.gath, uint32_t, 2ull * net.wmax * cfg.world);
        CK(cudaMemsetAsync(st.sendbuf, 0, 4ull * net.wmax, s));
        CK(cudaMemsetAsync(st.gath, 0, 8ull * net.wmax * cfg.world, s));
        snn_status r = exchange_setup(sim);
        if (r != SNN_OK) return r;
    }
    CK(cudaMemsetAsync(st.recent, 0, sizeof(uint32_t) * 4ull * st.rstride, s));
    for (int b = 0; b < 2; b++) {
        CK(cudaMemsetAsync(st.vmask[b], 0, sizeof(uint32_t) * net.nwords, s));
    }
    CK(cudaMemsetAsync(st.ctr, 0, sizeof(Counters), s));

    // ---- graph (count -> pivots/row_ptr -> fill)
    {
        uint32_t *gap = nullptr;
        ALLOC(gap, uint32_t, gap_host.empty() ? 1 : gap_host.size());
        if (!gap_host.empty())
            CK(cudaMemcpyAsync(gap, gap_host.data(), 4 * gap_host.size(), cudaMemcpyHostToDevice, s));
        tabs.gap = gap;
    }
    int64_t *len = nullptr;
    ALLOC(len, int64_t, (size_t)N + 1);
    CK(cudaMemsetAsync(len + N, 0, sizeof(int64_t), s));
    cudaEvent_t bev[4];
    for (auto &e : bev) CK(cudaEventCreate(&e));
    CK(build_preload(s));                 // (module loading, like allocation, outside the timed construction)
    CK(cudaEventRecord(bev[0], s));
    CK(build_count(net, tabs, st.piv, len, s));
    size_t tmp_bytes = 0;
    CK(build_scan(net, st.piv, len, st.row_ptr, nullptr, &tmp_bytes, s));
    void *tmp = sim->dalloc(tmp_bytes);
    if (!tmp) return sim->fail(SNN_E_OOM, "scan scratch");
    CK(build_scan(net, st.piv, len, st.row_ptr, tmp, &tmp_bytes, s));
    CK(cudaEventRecord(bev[1], s));
    CK(cudaMemcpyAsync(&sim->nsyn, st.row_ptr + N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ALLOC(st.idx, uint32_t, (size_t)sim->nsyn + 8);
    ALLOC(st.w, float, (size_t)sim->nsyn + 8);
    CK(cudaMemsetAsync(st.idx + sim->nsyn, 0, 8 * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(st.w + sim->nsyn, 0, 8 * sizeof(float), s));
    CK(cudaEventRecord(bev[2], s));
    CK(build_fill(net, tabs, st.piv, st.row_ptr, st.idx, st.w, s));
    CK(build_segments(net, st.row_ptr, st.idx, st.seg, s));
    CK(cudaEventRecord(bev[3], s));
    {   // device time of the construction (SNN_PHASE_BUILD), allocation excluded
        CK(cudaEventSynchronize(bev[3]));
        float m0 = 0.0f, m1 = 0.0f;
        CK(cudaEventElapsedTime(&m0, bev[0], bev[1]));
        CK(cudaEventElapsedTime(&m1, bev[2], bev[3]));
        sim->phase_ms[SNN_PHASE_BUILD] = (double)m0 + (double)m1;
        for (auto &e : bev) cudaEventDestroy(e);
    }
    st.idx16 = nullptr;
    st.b64 = nullptr;
    if (cfg.flags & SNN_FLAG_IDX16) {
        ALLOC(st.idx16, uint16_t, (size_t)sim->nsyn + 16);
        CK(build_idx16(net, st.idx, st.idx16, sim->nsyn, s));
        // k_flush's 16-bit stream: every plastic target j - tgt_lo < 5 2^16 (<= 4 crossings)
        uint32_t pmax = 0;
        for (uint32_t k = 0; k < net.npop; k++)
            if (net.pop[k].flags & PF_POST_PLASTIC) pmax = std::max(pmax, net.pop[k].base + net.pop[k].n);
        if (net.nstdp && (uint64_t)pmax <= (uint64_t)net.tgt_lo + 5ull * 65536ull) {
            ALLOC(st.b64, uint32_t, 4ull * N);
            CK(build_b64(net, st.row_ptr, st.idx, st.b64, s));
        }
    }
    CK(init_state(net, st, s));
    {
        StdpDev *tab = nullptr;
        ALLOC(tab, StdpDev, 4);
        CK(cudaMemcpyAsync(tab, net.stdp, sizeof(StdpDev) * 4, cudaMemcpyHostToDevice, s));
        st.stdp = tab;
    }

    // ---- launch shapes: k_deliver = nslices x splits CTAs (~1 wave at 2 per
    //      SM); k_stdp = 4 CTAs per SM, grid-striding over the visited rows
    sim->pp_lo = net.N;
    sim->pp_hi = 0;
    for (uint32_t k = 0; k < net.npop; k++)
        if (net.pop[k].flags & PF_POST_PLASTIC) {
            sim->pp_lo = std::min(sim->pp_lo, net.pop[k].base);
            sim->pp_hi = std::max(sim->pp_hi, net.pop[k].base + net.pop[k].n);
        }
    if (sim->pp_hi <= sim->pp_lo) sim->pp_lo = sim->pp_hi = 0;
    net.pp_lo = sim->pp_lo;
    net.pp_hi = sim->pp_hi;
    // the split step (k_front's arrival list one step ahead, the plastic
    // arrivals inside the delivery, k_flush beside it): the event schedule
    // with flushes at age H and sliced delivery; the arrivals of t + 2 must be
    // known at t (D >= 2; D >= 3 across ranks, whose words of t - 1 arrive
    // during step t - 1).  Otherwise the unsplit step (front -> STDP -> delivery).
    {
        const uint32_t dmin = ((cfg.world > 1 || (cfg.flags & SNN_FLAG_EXCHANGE)) ? 1u : 0u) + (sim->plastic ? 2u : 1u);
        sim->ahead = cfg.delivery == SNN_DELIV_SLICED && net.D >= dmin &&
                     (!sim->plastic || (cfg.plasticity == SNN_PLAST_EVENT && cfg.flush_period == 0)) &&
                     !getenv("SNN_NO_AHEAD");   // (tuning knob: the unsplit step)
    }
    if (deliver_smem_bytes(net, sim->ahead) > 200 * 1024)
        return sim->fail(SNN_E_INVALID, "slice width %u needs %zu B of shared memory", C,
                         deliver_smem_bytes(net, sim->ahead));
    if (sim->plastic && stdp_smem_bytes(net, sim->pp_lo, sim->pp_hi) > 227 * 1024)
        return sim->fail(SNN_E_UNSUPPORTED, "post-synaptic population of STDP too large for the shared bitmap");
    sim->ev_kernel = sim->plastic && cfg.plasticity == SNN_PLAST_EVENT && cfg.flush_period == 0 &&
                     ev_smem_bytes(sim->pp_lo, sim->pp_hi) <= 227 * 1024;
    if (sim->plastic && cfg.plasticity == SNN_PLAST_EVENT && cfg.flush_period == 0 && !sim->ev_kernel)
        return sim->fail(SNN_E_UNSUPPORTED, "post-synaptic population of STDP too large for k_stdp_ev's shared bitmap");
    if (sim->plastic && (!sim->ev_kernel || flush_smem_bytes(sim->pp_lo, sim->pp_hi) > 227 * 1024))
        sim->ahead = false;      // (k_flush needs its table in shared memory)
    // default (graph steps): the ahead step with k_flush on a side branch on
    // half of the SMs (measured on cfg3: 42.2 us/step vs 58.2 serial, 49.4 on
    // every SM -- the critical-path kernels are latency-bound, and a full-width
    // flush slows them more than it gains)
    sim->pipe = sim->ahead && sim->plastic ? 1 : 0;
    if (const char *e = getenv("SNN_PIPE")) sim->pipe = atoi(e);          // (experiments)
    // k_flush's deadline: 2 steps (R36), or 3 (SNN_FL_LAG=3, D >= 3: rows of age >= H - 2)
    if (const char *e = getenv("SNN_FL_LAG")) sim->fl_lag = (atoi(e) >= 3 && net.D >= 3) ? 3 : 2;
    net.fl_lag = sim->ahead ? (uint32_t)sim->fl_lag : 2u;
    if (sim->pipe == 2) sim->ahead = false;
    if (sim->pipe == 1 && !sim->ahead) sim->pipe = 0;
    if (!sim->plastic || !sim->ev_kernel || flush_smem_bytes(sim->pp_lo, sim->pp_hi) > 227 * 1024)
        if (sim->pipe == 2) sim->pipe = 0;
    // the fused step: the ahead step on one rank (the epilogue writes the ring
    // words of [0, R) and of the Poisson neurons sharing R's word)
    {
        bool straddle_ok = (net.R & 31u) == 0 || net.R >= net.N;
        for (uint32_t k = 0; k < net.npop && !straddle_ok; k++) {
            const PopDev &pp = net.pop[k];
            if (pp.base <= net.R && net.R < pp.base + pp.n)
                straddle_ok = pp.kind == POP_POISSON && pp.base + pp.n >= std::min((net.R + 31u) & ~31u, net.N);
        }
        // (opt-in, SNN_FUSE: measured slower on cfg3, 50.8 vs 42.8 us/step -- one CTA per
        // slice runs the slice's neuron update in k_deliver's tail)
        sim->fused = sim->ahead && cfg.world == 1 && !net.xchg && straddle_ok && getenv("SNN_FUSE") && sim->pipe != 2;
        // the split step (opt-in, SNN_SPLIT; needs D >= 3: the front of t reads
        // the ring up to t - 1 while kPart 4 of t writes slot t).  Measured on
        // cfg3: 45.9 vs 42.9 us/step -- k_deliver's CTAs fill the register files
        // of the SMs k_flush leaves, so the branch front waits for them
        if (!sim->fused && sim->ahead && cfg.world == 1 && !net.xchg && straddle_ok && net.D >= 3 && sim->pipe != 2 &&
            getenv("SNN_SPLIT")) {
            sim->fused = true;
            sim->split_front = true;
        }
        if (sim->fused) sim->pipe = 0;     // (the fused graph has its own branches)
    }
    ALLOC(st.slice_ticket, uint32_t, std::max(1u, net.nslices));
    CK(cudaMemsetAsync(st.slice_ticket, 0, 4ull * std::max(1u, net.nslices), s));
    if (sim->fused) {
        CK(cudaStreamCreateWithFlags(&sim->cap_front, cudaStreamNonBlocking));
        for (int q = 0; q < 2; q++) {
            CK(cudaEventCreateWithFlags(&sim->ev_fr[q], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sim->ev_del[q], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sim->ev_fl_f[q], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&sim->ev_lif[q], cudaEventDisableTiming));
        }
        if (sim->plastic && !sim->cap_side) CK(cudaStreamCreateWithFlags(&sim->cap_side, cudaStreamNonBlocking));
    }
    if (net.xchg && net.D >= 1 && cfg.nccl_unique_id && !getenv("SNN_NO_XBRANCH")) {
        CK(cudaStreamCreateWithFlags(&sim->cap_xside, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&sim->ev_xfront, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sim->ev_xdone, cudaEventDisableTiming));
    }
    if (sim->pipe != 0) {
        CK(cudaStreamCreateWithFlags(&sim->cap_side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&sim->ev_front, cudaEventDisableTiming));
        for (auto &e : sim->ev_flush) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        if (getenv("SNN_PRIO")) {
            sim->use_prio = true;
            CK(cudaDeviceGetStreamPriorityRange(&sim->prio_lo, &sim->prio_hi));
        }
    }
    // k_stdp flattens up to 128 rows' plastic spans (16-byte chunks) per round
    // into one uint32 chunk index
    if (sim->plastic && 128ull * ((uint64_t)net.N / 4 + 2) >= (1ull << 32))
        return sim->fail(SNN_E_UNSUPPORTED, "STDP with N = %u: a round of 128 plastic spans may exceed 2^32 chunks",
                         net.N);
    CK(kernels_configure(cfg.device));
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg.device);
    const uint32_t ns = std::max(1u, net.nslices);
    sim->splits = std::max(1u, (uint32_t)(2 * nsm) / ns);   // <= 2 CTAs per SM, one wave
    if (const char *sp = getenv("SNN_DELIVER_SPLITS")) sim->splits = std::max(1, atoi(sp));  // tuning knob
    sim->stdp_grid = (uint32_t)nsm;                 // k_stdp: one CTA per SM
    sim->flush_grid = (uint32_t)nsm * flush_ctas_per_sm();
    // k_flush's share of the SMs beside the critical path: half of them for
    // H = 64 and 2/7 for H = 128 (half the flush rows per step) at BASELINE
    // config 3's balance of work (measured: 42 of 148 SMs, 40.5 us/step vs
    // 45.5 on 74), scaled up by how much heavier the flush is relative to the
    // critical path than there: expected flush synapses per step (the plastic
    // synapses / H) against the neurons (k_front) and synapses (k_deliver),
    // weighted by their per-unit kernel times on 74 B200 SMs (k_flush 6.5 ps
    // per synapse, k_front 84 ps per neuron, k_deliver 8.5 fs per synapse of
    // the graph: measured at configs 3 and 4)
    {
        double fsyn = 0.0;
        for (const HostProj &hj : sim->projs)
            if (hj.prm.kind == SNN_SYN_STDP) {
                const PopDev &dp = net.pop[hj.dst];
                const uint32_t lo = std::max(dp.base, net.tgt_lo), hi = std::min(dp.base + dp.n, net.tgt_hi);
                fsyn += (double)sim->pops[hj.src].n * (double)(hi > lo ? hi - lo : 0u) * hj.prm.p;
            }
        const double t_fl = 6.5e-6 * fsyn / (double)net.H;
        const double t_crit = 8.4e-5 * (double)net.N + 8.5e-9 * (double)sim->nsyn;
        const double rho_ref = 6.5e-6 * (158114.0 * 126491.0 * 0.02 / 64.0) /
                               (8.4e-5 * 316228.0 + 8.5e-9 * 1.0000561e9);      // config 3, H = 64
        double scale = t_crit > 0.0 ? std::max(1.0, (t_fl / t_crit) * ((double)net.H / 64.0) / rho_ref) : 1.0;
        if (net.H > kHistBits) scale = std::pow(scale, 1.45);   // (H = 128: config 4's optimum, 84 SMs, is 2x config 3's)
        const int base = net.H > kHistBits ? nsm * 2 / 7 : nsm / 2;
        sim->flush_grid_side = std::max(1, std::min((int)(base * scale), nsm * 4 / 5));
    }
    if (const char *e = getenv("SNN_FL_CTAS")) sim->flush_grid_side = std::max(1, atoi(e));   // (experiments)

    CK(cudaStreamSynchronize(s));
    sim->state = 1;
    return SNN_OK;
}

// ---------------------------------------------------------------- the step
// D = 0 on the local-group transport: every rank's neuron phase of step t,
// then every rank's words of t into every peer's gather slot, then each
// rank's unpack into its ring slot t (all on the caller's stream).
static snn_status local_group_front_d0(snn_sim *sim, cudaStream_t s, int64_t t) {
    const snn_config &cfg = sim->cfg;
    std::vector<snn_sim *> peers;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        peers = g_groups[cfg.group_key];
    }
    if ((int)peers.size() != cfg.world)
        return sim->fail(SNN_E_STATE, "local group %llu has %zu of %d ranks", (unsigned long long)cfg.group_key,
                         peers.size(), cfg.world);
    for (snn_sim *p : peers) {
        if (p->state == 0 || !p->st.gath) return sim->fail(SNN_E_STATE, "local group peer not finalized");
        if (p->t != sim->t) return sim->fail(SNN_E_STATE, "local group ranks must be stepped in lockstep");
        CK(launch_front(p->net, p->st, s, false, false, 1, false));
    }
    for (snn_sim *q : peers)
        for (snn_sim *p : peers)
            CK(cudaMemcpyAsync(p->st.gath + ((size_t)(t & 1) * cfg.world + q->cfg.rank) * sim->wmax, q->st.sendbuf,
                               4ull * sim->wmax, cudaMemcpyDeviceToDevice, s));
    for (snn_sim *p : peers)
        CK(launch_unpack(p->net, p->st, p->st.gath + (size_t)(t & 1) * cfg.world * sim->wmax, t, s));
    return SNN_OK;
}

static snn_status enqueue_step(snn_sim *sim, cudaStream_t s, cudaEvent_t *ev, bool first, int64_t step_k = 0,
                               cudaStream_t side = nullptr, uint32_t gk = 0) {
    NetDev net = sim->net;
    if ((sim->cfg.flags & SNN_FLAG_TRACE) && getenv("SNN_DEBUG_KERNELS"))   // kernel experiments (trace runs only)
        net.debug = (uint32_t)atoi(getenv("SNN_DEBUG_KERNELS"));
    const StateDev &st = sim->st;
    // programmatic dependent launch between the kernels of the graph (not
    // across event records, whose timing would then overlap)
    const bool multi = sim->net.xchg != 0;
    const bool pdl = ev == nullptr && !(sim->cfg.flags & SNN_FLAG_NO_PDL) && !multi;
    if (ev) CK(cudaEventRecord(ev[0], s));
    const int64_t t = sim->t + step_k;                              // host copy (direct mode only)
    const bool d0 = multi && net.D == 0;     // the arrivals of t include the other ranks' spikes of t
    if (multi && sim->local_group && t > 0 && !d0)                  // peers' spikes of t-1 -> ring
        CK(launch_unpack(net, st, st.gath + (size_t)((t - 1) & 1) * sim->cfg.world * sim->wmax, t - 1, s));
    if (sim->use_prio) set_launch_priority(sim->prio_hi);
    if (d0) {
        // neurons of t (every rank) -> the exchange of the words of t -> the
        // lists of t from the complete ring slot
        if (sim->local_group) {
            // (test transport, one stream, ranks stepped in lockstep in rank
            // order: rank 0's call runs every rank's neuron phase and the copies)
            if (sim->cfg.rank == 0) {
                snn_status r = local_group_front_d0(sim, s, t);
                if (r != SNN_OK) return r;
            }
        } else {
            CK(launch_front(net, st, s, false, false, 1, false));
            snn_status r = exchange_enqueue(sim, s, t);
            if (r != SNN_OK) return r;
        }
        CK(launch_front(net, st, s, false, false, 2, false));
    } else {
        const bool xbranch = multi && side && sim->cap_xside && !sim->local_group;
        if (xbranch && gk > 0) CK(cudaStreamWaitEvent(s, sim->ev_xdone, 0));   // the exchange of t-1
        CK(launch_front(net, st, s, pdl && !first, sim->ahead, 0, sim->fused)); // (1) P:36 + work lists
        if (xbranch) {                                              // spike words of t -> peers, beside the step
            CK(cudaEventRecord(sim->ev_xfront, s));
            CK(cudaStreamWaitEvent(sim->cap_xside, sim->ev_xfront, 0));
            snn_status r = exchange_enqueue(sim, sim->cap_xside, t);
            if (r != SNN_OK) return r;
            CK(cudaEventRecord(sim->ev_xdone, sim->cap_xside));
        } else if (multi) {
            snn_status r = exchange_enqueue(sim, s, t);
            if (r != SNN_OK) return r;
        }
    }
    if (ev) CK(cudaEventRecord(ev[1], s));
    if (sim->plastic) {                                             // (2) P:37-39
        // the event schedule (flushes at age H): k_stdp_ev; the ablation
        // schedules and batched flushes: the generic k_stdp
        if (side && sim->cap_side && (sim->pipe == 1 || sim->pipe == 2)) {
            // (experiments) the forced flushes on a side branch of the graph
            CK(cudaEventRecord(sim->ev_front, s));
            const uint32_t lag = sim->pipe == 1 ? (uint32_t)sim->fl_lag : 1u;
            if (gk >= lag) CK(cudaStreamWaitEvent(s, sim->ev_flush[(gk - lag) & 3], 0));
            if (sim->pipe == 2) CK(launch_stdp_ev(net, st, sim->stdp_grid, sim->pp_lo, sim->pp_hi, s, pdl, 1));
            CK(cudaStreamWaitEvent(side, sim->ev_front, 0));
            if (sim->use_prio) set_launch_priority(sim->prio_lo);
            // (SNN_SKIP_FLUSH: experiments only -- the step without its forced flushes, WRONG weights)
            if (!getenv("SNN_SKIP_FLUSH")) CK(launch_stdp_ev(net, st, sim->flush_grid_side, sim->pp_lo, sim->pp_hi, side, false, 2));
            if (sim->use_prio) set_launch_priority(sim->prio_hi);
            CK(cudaEventRecord(sim->ev_flush[gk & 3], side));
        } else if (sim->ahead) {
            // the plastic arrivals run inside k_deliver(t), the forced flushes of t
            // in k_flush(t) after it (below)
        } else if (sim->pipe == 2) {
            CK(launch_stdp_ev(net, st, sim->stdp_grid, sim->pp_lo, sim->pp_hi, s, pdl, 1));
        } else if (sim->ev_kernel) {
            CK(launch_stdp_ev(net, st, sim->stdp_grid, sim->pp_lo, sim->pp_hi, s, pdl, 0));
        } else {
            CK(launch_stdp(net, st, -1, sim->stdp_grid, sim->pp_lo, sim->pp_hi, s, pdl));
        }
    }
    if (ev) CK(cudaEventRecord(ev[2], s));
    if (net.deliv_mode == SNN_DELIV_ROWWISE) CK(launch_deliver_rowwise(net, st, sim->stdp_grid, s, pdl));   // Fig. 3a
    else CK(launch_deliver(net, st, sim->splits, s, pdl, sim->ahead, false));   // (3) P:41, Fig. 3b
    if (sim->plastic && (sim->ahead || sim->pipe == 2) && !(side && sim->cap_side && sim->pipe != 0))   // (2') flushes of t (R3)
        CK(launch_stdp_ev(net, st, sim->flush_grid, sim->pp_lo, sim->pp_hi, s, pdl, 2));
    if (sim->use_prio) set_launch_priority(0);
    if (ev) CK(cudaEventRecord(ev[4], s));
    if (ev) CK(cudaEventRecord(ev[3], s));
    return SNN_OK;
}

// The fused step graph of n steps t0 .. t0 + n - 1:
//   main   : k_front(t0) (all neurons), then k_deliver(t) for every t, the
//            epilogue (neurons of t + 1) on all but the last
//   branch F: k_front(t) for t > t0 (neurons >= R, lists), after k_deliver(t-1)
//   branch X: k_flush(t) after the front of t; k_deliver(t+2) waits for it
// k_deliver(t) waits for the front of t-1 (its arrival list) -- so the critical
// path is one kernel per step; state between two calls is the unfused one.
static snn_status capture_fused(snn_sim *sim, uint32_t n, cudaGraphExec_t *out) {
    cudaGraph_t g = nullptr;
    const NetDev &net = sim->net;
    const StateDev &st = sim->st;
    cudaStream_t m = sim->cap_stream, F = sim->cap_front, X = sim->cap_side;
    const bool pl = sim->plastic;
    CK(cudaStreamBeginCapture(m, cudaStreamCaptureModeThreadLocal));
    auto fail = [&](snn_status r) {
        cudaStreamEndCapture(m, &g);
        if (g) cudaGraphDestroy(g);
        return r;
    };
#define CKF(call)                                                                                     \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            return fail(sim->fail(SNN_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                                  __FILE__, __LINE__));                                               \
    } while (0)
    const bool dbg_serial = getenv("SNN_FUSE_SERIAL") != nullptr;   // (debug: k_front(t) after k_deliver(t))
    const bool split = sim->split_front;
    for (uint32_t k = 0; k < n; k++) {
        if (k > 0 && !dbg_serial) {                                   // F: the front of t0 + k
            CKF(cudaStreamWaitEvent(F, sim->ev_del[(k - 1) & 1], 0));
            CKF(launch_front(net, st, F, false, true, 3, true));
            CKF(cudaEventRecord(sim->ev_fr[k & 1], F));
        }
        if (k > 0 && dbg_serial) {
            CKF(launch_front(net, st, m, false, true, 3, true));
            CKF(cudaEventRecord(sim->ev_fr[k & 1], m));
        }
        // main: [k_front(t0)] k_deliver(t0 + k)
        if (k == 0) {
            CKF(launch_front(net, st, m, false, true, 0, true));
            CKF(cudaEventRecord(sim->ev_fr[0], m));
        } else if (k >= 2) {
            CKF(cudaStreamWaitEvent(m, sim->ev_fr[(k - 1) & 1], 0));  // the arrival list of t (front of t-1)
        } else {
            CKF(cudaStreamWaitEvent(m, sim->ev_fr[0], 0));
        }
        if (pl && k >= 2) CKF(cudaStreamWaitEvent(m, sim->ev_fl_f[k & 1], 0));   // k_flush(t-2)
        if (split && k > 0) {
            // the split step: the neurons [0, R) of t (kPart 4) after k_deliver(t-1),
            // PDL -- its dependency wait also covers the joins above (front of
            // t-1, k_flush(t-2)), and k_deliver(t) launches only after it waited
            CKF(launch_front(net, st, m, true, true, 4, false));
            CKF(cudaEventRecord(sim->ev_lif[k & 1], m));
        }
        // (fused: PDL only behind the first front -- with the joins of the
        // branches, stream capture makes every incoming edge programmatic, and
        // k_deliver(t) reads the arrival list of the front of t-1 before its
        // dependency wait; split: behind kPart 4, which waited for them)
        CKF(launch_deliver(net, st, sim->splits, m, k == 0 || split, true, !split && k + 1 < n));
        CKF(cudaEventRecord(sim->ev_del[k & 1], m));
        if (pl) {                                                     // X: the forced flushes of t0 + k
            if (split && k > 0) CKF(cudaStreamWaitEvent(X, sim->ev_lif[k & 1], 0));   // fpos of t (kPart 4)
            CKF(cudaStreamWaitEvent(X, sim->ev_fr[k & 1], 0));
            CKF(launch_stdp_ev(net, st, sim->flush_grid_side, sim->pp_lo, sim->pp_hi, X, false, 2));
            CKF(cudaEventRecord(sim->ev_fl_f[k & 1], X));
        }
    }
    if (n > 1) CKF(cudaStreamWaitEvent(m, sim->ev_fr[(n - 1) & 1], 0));   // join the branches
    if (pl)
        for (uint32_t k = n > 2 ? n - 2 : 0; k < n; k++) CKF(cudaStreamWaitEvent(m, sim->ev_fl_f[k & 1], 0));
#undef CKF
    CK(cudaStreamEndCapture(m, &g));
    CK(cudaGraphInstantiate(out, g, 0));
    CK(cudaGraphDestroy(g));
    return SNN_OK;
}

static snn_status capture(snn_sim *sim, uint32_t nsteps, cudaGraphExec_t *out) {
    if (sim->fused) return capture_fused(sim, nsteps, out);
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(sim->cap_stream, cudaStreamCaptureModeThreadLocal));
    for (uint32_t k = 0; k < nsteps; k++) {
        snn_status r = enqueue_step(sim, sim->cap_stream, nullptr, k == 0, 0,
                                    sim->cap_side ? sim->cap_side : sim->cap_xside, k);
        if (r != SNN_OK) {
            cudaStreamEndCapture(sim->cap_stream, &g);
            if (g) cudaGraphDestroy(g);
            return r;
        }
    }
    if (sim->cap_xside && nsteps > 0) CK(cudaStreamWaitEvent(sim->cap_stream, sim->ev_xdone, 0));   // join
    if (sim->cap_side && sim->pipe != 0)                            // join the side branch
        for (uint32_t k = nsteps > 3 ? nsteps - 3 : 0; k < nsteps; k++)
            CK(cudaStreamWaitEvent(sim->cap_stream, sim->ev_flush[k & 3], 0));
    CK(cudaStreamEndCapture(sim->cap_stream, &g));
    CK(cudaGraphInstantiate(out, g, 0));
    CK(cudaGraphDestroy(g));
    return SNN_OK;
}

extern "C" {

uint32_t snn_abi_version(void) { return SNN_ABI_VERSION; }

const char *snn_last_error(const snn_sim *sim) {
    return sim ? sim->err.c_str() : g_create_error.c_str();
}

snn_status snn_create(const snn_config *cfg, snn_sim **out) {
    if (!out) return SNN_E_INVALID;
    *out = nullptr;
    g_create_error.clear();
    if (!cfg || cfg->abi_version != SNN_ABI_VERSION || cfg->struct_size != sizeof(snn_config)) {
        g_create_error = "snn_config: ABI version / struct size mismatch";
        return SNN_E_INVALID;
    }
    if (!(cfg->dt_ms > 0.0f) || (cfg->history_bits != 64 && cfg->history_bits != 128) || cfg->delay_steps > 62 ||
        cfg->accum_frac_bits < 0 || cfg->accum_frac_bits > 30 || cfg->world < 1 || cfg->rank < 0 ||
        cfg->rank >= cfg->world) {
        g_create_error = "snn_config: need dt > 0, history_bits 64 or 128, delay <= 62, 0 <= F <= 30, 0 <= rank < world";
        return SNN_E_INVALID;
    }
    if (cfg->flush_period > cfg->history_bits / 2) {
        g_create_error = "snn_config: flush_period must be 0 or at most history_bits / 2";
        return SNN_E_INVALID;
    }
    if (cfg->plasticity > SNN_PLAST_NAIVE || cfg->delivery > SNN_DELIV_ROWWISE) {
        g_create_error = "snn_config: plasticity must be SNN_PLAST_*, delivery SNN_DELIV_*";
        return SNN_E_INVALID;
    }
    const uint32_t C = cfg->slice_width;
    if (C != 0 && (C < 32 || C > 32768 || (C & 31u) != 0)) {
        g_create_error = "snn_config: slice_width must be 0 or a multiple of 32 in [32, 32768]";
        return SNN_E_INVALID;
    }
    if ((cfg->dev_alloc == nullptr) != (cfg->dev_free == nullptr)) {
        g_create_error = "snn_config: dev_alloc and dev_free must both be set or both NULL";
        return SNN_E_INVALID;
    }
    if ((cfg->world > 1 && !cfg->nccl_unique_id && cfg->group_key == 0) ||
        ((cfg->flags & SNN_FLAG_EXCHANGE) && !cfg->nccl_unique_id)) {
        g_create_error = "world > 1 needs an nccl_unique_id or a local group_key (SNN_FLAG_EXCHANGE: an nccl_unique_id)";
        return SNN_E_INVALID;
    }
    DeviceGuard dg(cfg->device);
    if (dg.err != cudaSuccess) {
        g_create_error = std::string("cudaSetDevice: ") + cudaGetErrorString(dg.err);
        return SNN_E_CUDA;
    }
    cudaError_t e = cudaSuccess;
    snn_sim *sim = new snn_sim();
    sim->cfg = *cfg;
    sim->stream = (cudaStream_t)cfg->stream;
    e = cudaStreamCreateWithFlags(&sim->cap_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        g_create_error = std::string("cudaStreamCreate: ") + cudaGetErrorString(e);
        delete sim;
        return SNN_E_CUDA;
    }
    if (cfg->world > 1 && !cfg->nccl_unique_id) {
        std::lock_guard<std::mutex> lk(g_mu);
        std::vector<snn_sim *> &g = g_groups[cfg->group_key];
        for (snn_sim *p : g)
            if (p->cfg.rank == cfg->rank || p->cfg.world != cfg->world) {
                g_create_error = "local group: duplicate rank or mismatched world";
                cudaStreamDestroy(sim->cap_stream);
                delete sim;
                return SNN_E_INVALID;
            }
        g.push_back(sim);
    }
    *out = sim;
    return SNN_OK;
}

snn_status snn_add_population(snn_sim *sim, uint32_t n, const snn_pop_params *prm, uint32_t *pop_id) {
    if (!sim) return SNN_E_INVALID;
    sim->err.clear();
    if (sim->state != 0) return sim->fail(SNN_E_STATE, "add_population after finalize");
    if (!prm || prm->struct_size != sizeof(snn_pop_params)) return sim->fail(SNN_E_INVALID, "snn_pop_params size");
    if (n == 0) return sim->fail(SNN_E_INVALID, "population size must be > 0");
    if (prm->kind > SNN_POP_LIF_CUBA) return sim->fail(SNN_E_INVALID, "unknown population kind %u", prm->kind);
    if (sim->pops.size() >= (size_t)kMaxPops) return sim->fail(SNN_E_UNSUPPORTED, "at most %d populations", kMaxPops);
    if ((uint64_t)sim->N + n >= 0x7fffffffull) return sim->fail(SNN_E_INVALID, "too many neurons");
    if (prm->kind != SNN_POP_POISSON) {
        if (!(prm->tau_m_ms > 0.0f) || !(prm->tau_ref_ms >= 0.0f))
            return sim->fail(SNN_E_INVALID, "tau_m must be > 0 and tau_ref >= 0");
        if (prm->kind == SNN_POP_LIF_CUBA && !(prm->tau_e_ms > 0.0f && prm->tau_i_ms > 0.0f))
            return sim->fail(SNN_E_INVALID, "CUBA needs tau_e, tau_i > 0");
    } else if (!(prm->rate_hz >= 0.0f)) {
        return sim->fail(SNN_E_INVALID, "rate must be >= 0");
    }
    HostPop hp;
    hp.prm = *prm;
    hp.base = sim->N;
    hp.n = n;
    sim->pops.push_back(hp);
    sim->N += n;
    if (pop_id) *pop_id = (uint32_t)sim->pops.size() - 1;
    return SNN_OK;
}

snn_status snn_connect(snn_sim *sim, uint32_t src, uint32_t dst, const snn_syn_params *q) {
    if (!sim) return SNN_E_INVALID;
    sim->err.clear();
    if (sim->state != 0) return sim->fail(SNN_E_STATE, "connect after finalize");
    if (!q || q->struct_size != sizeof(snn_syn_params)) return sim->fail(SNN_E_INVALID, "snn_syn_params size");
    if (src >= sim->pops.size() || dst >= sim->pops.size()) return sim->fail(SNN_E_INVALID, "unknown population");
    if (!(q->p >= 0.0 && q->p <= 1.0)) return sim->fail(SNN_E_INVALID, "p must be in [0, 1]");
    if (q->kind > SNN_SYN_STDP || q->receptor > SNN_RCPT_INH) return sim->fail(SNN_E_INVALID, "bad kind / receptor");
    const uint32_t dk = sim->pops[dst].prm.kind;
    if (dk == SNN_POP_POISSON) return sim->fail(SNN_E_INVALID, "POISSON populations take no input");
    if (dk == SNN_POP_LIF_DELTA && q->receptor != SNN_RCPT_EXC)
        return sim->fail(SNN_E_INVALID, "LIF_DELTA has a single (EXC) receptor; use a signed weight");
    for (const HostProj &hj : sim->projs) {
        if (hj.src == src && hj.dst == dst) return sim->fail(SNN_E_INVALID, "duplicate projection");
        if (q->kind == SNN_SYN_STDP && hj.src == src && hj.prm.kind == SNN_SYN_STDP)
            return sim->fail(SNN_E_UNSUPPORTED, "one STDP projection per source population");
    }
    if (q->kind == SNN_SYN_STDP &&
        !(q->tau_plus_ms > 0.0f && q->tau_minus_ms > 0.0f && q->w_max >= 0.0f && q->weight >= 0.0f &&
          q->weight <= q->w_max))
        return sim->fail(SNN_E_INVALID, "STDP needs tau_+, tau_- > 0 and 0 <= weight <= w_max");
    HostProj hj;
    hj.src = src;
    hj.dst = dst;
    hj.prm = *q;
    sim->projs.push_back(hj);
    return SNN_OK;
}

snn_status snn_step(snn_sim *sim, uint32_t n_steps) {
    if (!sim) return SNN_E_INVALID;
    sim->err.clear();
    DeviceGuard dg(sim->cfg.device);
    if (dg.err != cudaSuccess) return sim->fail(SNN_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(dg.err));
    if (sim->state == 0) {
        snn_status r = finalize(sim);
        if (r != SNN_OK) return r;
    }
    if (n_steps == 0) return SNN_OK;
    const bool timing = (sim->cfg.flags & SNN_FLAG_PHASE_TIMING) != 0;
    // (SNN_TRACE_GRAPH, experiments: the per-CTA trace of the graph-replayed step, the last step's marks)
    const bool trace_direct = (sim->cfg.flags & SNN_FLAG_TRACE) && !getenv("SNN_TRACE_GRAPH");
    const bool direct = timing || (sim->cfg.flags & SNN_FLAG_NO_GRAPH) || trace_direct || sim->local_group;
    if (direct) {
        for (uint32_t k = 0; k < n_steps; k++) {
            cudaEvent_t *ev = nullptr;
            if (timing) {
                if (sim->ev_used == sim->ev_steps.size()) {
                    std::vector<cudaEvent_t> v(5);
                    for (auto &e : v) CK(cudaEventCreate(&e));
                    sim->ev_steps.push_back(v);
                }
                ev = sim->ev_steps[sim->ev_used++].data();
            }
            snn_status r = enqueue_step(sim, sim->stream, ev, true);
            if (r != SNN_OK) return r;
            sim->t++;
        }
        return SNN_OK;
    }
    for (uint32_t k = 0; k < n_steps;) {
        const uint32_t n = std::min(kGraphSteps, n_steps - k);
        auto it = sim->graphs.find(n);
        if (it == sim->graphs.end()) {
            if (sim->graphs.size() >= 16) {              // (bounded cache: drop the others, keep 64)
                for (auto &g : sim->graphs)
                    if (g.first != kGraphSteps) cudaGraphExecDestroy(g.second);
                for (auto g = sim->graphs.begin(); g != sim->graphs.end();)
                    g = g->first != kGraphSteps ? sim->graphs.erase(g) : std::next(g);
            }
            cudaGraphExec_t ge = nullptr;
            snn_status r = capture(sim, n, &ge);
            if (r != SNN_OK) return r;
            it = sim->graphs.emplace(n, ge).first;
        }
        CK(cudaGraphLaunch(it->second, sim->stream));
        k += n;
    }
    sim->t += n_steps;
    return SNN_OK;
}

// Read-out flush (R11): finalise pending row visits and bring every stale
// plastic row up to t_last without a pre spike.
static snn_status readout_flush(snn_sim *sim) {
    if (!sim->plastic || sim->t == 0 || sim->readout_t == sim->t) return SNN_OK;   // (already flushed at t)
    sim->readout_t = sim->t;
    CK(launch_readout(sim->net, sim->st, sim->t - 1, sim->stdp_grid, sim->pp_lo, sim->pp_hi, sim->stream, sim->ahead));
    return SNN_OK;
}

// A read-out source: a device or host array of `bytes` bytes, `elem` bytes per
// element.  prepare = the copy is about to happen: run the field's side effects
// (read-out flush R11, remote words of the last step, history reconstruction,
// folding of timing records).
struct FieldRef {
    const void *dev = nullptr;
    const void *host = nullptr;
    size_t bytes = 0, elem = 1;
    bool ring = false;   // SPIKE_RING: rows of nwords words, device stride ring_stride
    int64_t host_i64[8];
    unsigned long long host_u64[4 * kKSpanKernels];
    double host_f64[8];
};

static snn_status fold_ktime(snn_sim *sim) {
    if (!sim->kspan) return SNN_OK;
    const size_t n = (size_t)kKSpanSlots * kKSpanKernels;
    std::vector<KSpan> h(n);
    CK(cudaMemcpyAsync(h.data(), sim->kspan, n * sizeof(KSpan), cudaMemcpyDeviceToHost, sim->stream));
    CK(cudaStreamSynchronize(sim->stream));
    for (size_t x = 0; x < n; x++) {
        const KSpan &k = h[x];
        if (k.ctas == 0 || k.end == 0 || k.entry == ~0ull || k.wait == ~0ull) continue;
        unsigned long long *tot = sim->ks_tot[x % kKSpanKernels];
        tot[0] += k.end > k.entry ? k.end - k.entry : 0ull;
        tot[1] += k.end > k.wait ? k.end - k.wait : 0ull;
        tot[2] += 1ull;
        tot[3] += k.ctas;
    }
    CK(launch_kspan_reset(sim->kspan, sim->stream));
    return SNN_OK;
}

static snn_status field_ref(snn_sim *sim, uint32_t field, uint32_t pop_id, bool prepare, FieldRef &f) {
    f = FieldRef();
    if (field >= SNN_FIELD_COUNT) return sim->fail(SNN_E_INVALID, "unknown field %u", field);
    if (sim->state == 0 && field != SNN_FIELD_STEP) return sim->fail(SNN_E_STATE, "read_state before finalize");
    const NetDev &net = sim->net;
    const StateDev &st = sim->st;
    uint32_t base = 0, n = sim->N;
    if (pop_id != 0xffffffffu) {
        if (pop_id >= sim->pops.size()) return sim->fail(SNN_E_INVALID, "unknown population %u", pop_id);
        base = sim->pops[pop_id].base;
        n = sim->pops[pop_id].n;
    }
    cudaStream_t s = sim->stream;
    bool per_neuron = true;
    switch (field) {
    case SNN_FIELD_V: f.dev = st.V + base; f.elem = 4; break;
    case SNN_FIELD_REFRACTORY: f.dev = st.ref + base; f.elem = 4; break;
    case SNN_FIELD_G_EXC: f.dev = st.ge + base; f.elem = 4; break;
    case SNN_FIELD_G_INH: f.dev = st.gi + base; f.elem = 4; break;
    case SNN_FIELD_INPUT_EXC: f.dev = st.in_e + base; f.elem = 4; break;
    case SNN_FIELD_INPUT_INH: f.dev = st.in_i + base; f.elem = 4; break;
    case SNN_FIELD_SPIKE_COUNT: f.dev = st.nspk + base; f.elem = 4; break;
    case SNN_FIELD_XPOST: f.dev = st.xpost + base; f.elem = 4; break;
    case SNN_FIELD_XPRE_ROW: f.dev = st.xpre + base; f.elem = 4; break;
    case SNN_FIELD_TLU: f.dev = st.tlu + base; f.elem = 4; break;
    case SNN_FIELD_HIST: f.elem = 8; break;
    case SNN_FIELD_HIST_DEV: f.dev = st.hist + base; f.elem = 8; break;
    case SNN_FIELD_HIST_DEV_HI:
        if (net.H <= 64) return sim->fail(SNN_E_STATE, "HIST_DEV_HI needs history_bits = 128");
        f.dev = st.hist_hi + base; f.elem = 8; break;
    case SNN_FIELD_FPOT: f.dev = st.fpot + (size_t)((sim->t + 3) & 3) * st.fstride + base; f.elem = 4; break;   // step t-1's
    case SNN_FIELD_FPOS: f.dev = st.fpos + (size_t)((sim->t + 3) & 3) * st.fstride + base; f.elem = 1; break;
    default: per_neuron = false; break;
    }
    if (per_neuron) {
        f.bytes = f.elem * n;
    } else {
        switch (field) {
        case SNN_FIELD_ROW_PTR: f.dev = st.row_ptr; f.elem = 8; f.bytes = 8ull * (sim->N + 1); break;
        case SNN_FIELD_IDX: f.dev = st.idx; f.elem = 4; f.bytes = 4ull * sim->nsyn; break;
        case SNN_FIELD_IDX16:
            if (!st.idx16) return sim->fail(SNN_E_STATE, "IDX16 needs SNN_FLAG_IDX16");
            f.dev = st.idx16; f.elem = 2; f.bytes = 2ull * sim->nsyn; break;
        case SNN_FIELD_WEIGHTS: f.dev = st.w; f.elem = 4; f.bytes = 4ull * sim->nsyn; break;
        case SNN_FIELD_PIVOTS: f.dev = st.piv; f.elem = 4; f.bytes = 4ull * sim->N * (net.nslices + 1); break;
        case SNN_FIELD_SPIKE_RING: f.dev = st.ring; f.elem = 4; f.bytes = 4ull * kRingSlots * net.nwords; f.ring = true; break;
        case SNN_FIELD_RECENT:
            f.dev = st.recent + (size_t)((sim->t + 3) & 3) * st.rstride; f.elem = 4; f.bytes = 4ull * net.nwords; break;
        case SNN_FIELD_STEP: f.host_i64[0] = sim->t; f.host = f.host_i64; f.elem = 8; f.bytes = 8; break;
        case SNN_FIELD_METRICS: f.dev = st.ctr->metric; f.elem = 8; f.bytes = 8 * 16; break;
        case SNN_FIELD_PHASE_TIMES: f.host = f.host_f64; f.elem = 8; f.bytes = 8 * 8; break;
        case SNN_FIELD_KTIME:
            if (!sim->kspan) return sim->fail(SNN_E_STATE, "KTIME needs SNN_FLAG_KTIME");
            f.host = f.host_u64; f.elem = 8; f.bytes = 8 * 4 * kKSpanKernels; break;
        case SNN_FIELD_TRACE:
            if (!st.trace) return sim->fail(SNN_E_STATE, "trace needs SNN_FLAG_TRACE");
            f.dev = st.trace; f.elem = 8; f.bytes = 8ull * kTraceKernels * kTraceCtas * 4; break;
        case SNN_FIELD_INFO:
            f.host_i64[0] = sim->N; f.host_i64[1] = sim->nsyn; f.host_i64[2] = net.nslices; f.host_i64[3] = net.C;
            f.host_i64[4] = net.R; f.host_i64[5] = net.tgt_lo; f.host_i64[6] = net.tgt_hi;
            f.host_i64[7] = ((int64_t)sim->splits << 32) | sim->stdp_grid;
            f.host = f.host_i64; f.elem = 8; f.bytes = 64; break;
        default: return sim->fail(SNN_E_INVALID, "unknown field %u", field);
        }
    }
    if (!prepare) return SNN_OK;
    if (field == SNN_FIELD_WEIGHTS || field == SNN_FIELD_XPRE_ROW || field == SNN_FIELD_TLU) {
        snn_status r = readout_flush(sim);
        if (r != SNN_OK) return r;
    }
    if (sim->local_group && sim->t > 0 && (field == SNN_FIELD_HIST || field == SNN_FIELD_SPIKE_RING))
        CK(launch_unpack(net, st, st.gath + (size_t)((sim->t - 1) & 1) * sim->cfg.world * sim->wmax, sim->t - 1,
                         s));                                      // the last step's remote words
    if (field == SNN_FIELD_HIST) {
        if (!sim->d_hist_tmp) {
            sim->d_hist_tmp = (uint64_t *)sim->dalloc(8ull * sim->N);
            if (!sim->d_hist_tmp) return sim->fail(SNN_E_OOM, "hist scratch");
        }
        CK(launch_hist_from_ring(net, st.ring, sim->t - 1, sim->d_hist_tmp, s));
        f.dev = sim->d_hist_tmp + base;
    }
    if (field == SNN_FIELD_KTIME) {
        snn_status r = fold_ktime(sim);
        if (r != SNN_OK) return r;
        for (int k = 0; k < kKSpanKernels; k++)
            for (int q = 0; q < 4; q++) f.host_u64[4 * k + q] = sim->ks_tot[k][q];
    }
    if (field == SNN_FIELD_PHASE_TIMES) {
        CK(cudaStreamSynchronize(s));
        for (size_t k = 0; k < sim->ev_used; k++) {
            float ms[4];
            for (int p = 0; p < 4; p++) CK(cudaEventElapsedTime(&ms[p], sim->ev_steps[k][p], sim->ev_steps[k][p + 1]));
            sim->phase_ms[SNN_PHASE_FRONT] += ms[0];
            sim->phase_ms[SNN_PHASE_STDP] += ms[1] + ms[3];     // (ahead step: the forced flushes after delivery)
            sim->phase_ms[SNN_PHASE_DELIVERY] += ms[2];
            sim->phase_ms[SNN_PHASE_TOTAL] += ms[0] + ms[1] + ms[2] + ms[3];
        }
        sim->ev_used = 0;
        for (int k = 0; k < 8; k++) f.host_f64[k] = sim->phase_ms[k];
    }
    return SNN_OK;
}

// Copies elements [first, first + count) of f into host_dst.
static snn_status copy_out(snn_sim *sim, const FieldRef &f, size_t first, size_t count, void *host_dst) {
    const size_t off = first * f.elem, bytes = count * f.elem;
    if (bytes == 0) return SNN_OK;
    if (f.host) {
        memcpy(host_dst, (const char *)f.host + off, bytes);
        return SNN_OK;
    }
    cudaStream_t s = sim->stream;
    const NetDev &net = sim->net;
    if (f.ring && net.ring_stride != net.nwords) {     // slots padded for the exchange: row by row
        size_t e = first, done = 0;
        while (done < count) {
            const size_t slot = e / net.nwords, w = e % net.nwords;
            const size_t take = std::min(count - done, (size_t)net.nwords - w);
            CK(cudaMemcpyAsync((char *)host_dst + 4 * done, sim->st.ring + slot * net.ring_stride + w, 4 * take,
                               cudaMemcpyDeviceToHost, s));
            done += take;
            e += take;
        }
    } else {
        CK(cudaMemcpyAsync(host_dst, (const char *)f.dev + off, bytes, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    return SNN_OK;
}

snn_status snn_read_state(snn_sim *sim, uint32_t field, uint32_t pop_id, void *host_dst, size_t dst_bytes,
                          size_t *needed) {
    if (!sim) return SNN_E_INVALID;
    sim->err.clear();
    DeviceGuard dg(sim->cfg.device);
    FieldRef f;
    snn_status r = field_ref(sim, field, pop_id, false, f);
    if (r != SNN_OK) return r;
    if (needed) *needed = f.bytes;
    if (!host_dst) return SNN_OK;
    if (dst_bytes < f.bytes) return sim->fail(SNN_E_INVALID, "buffer of %zu bytes < %zu needed", dst_bytes, f.bytes);
    if ((r = field_ref(sim, field, pop_id, true, f)) != SNN_OK) return r;
    return copy_out(sim, f, 0, f.bytes / f.elem, host_dst);
}

snn_status snn_read_state_range(snn_sim *sim, uint32_t field, uint32_t pop_id, uint64_t first, uint64_t count,
                                void *host_dst, size_t dst_bytes) {
    if (!sim) return SNN_E_INVALID;
    sim->err.clear();
    DeviceGuard dg(sim->cfg.device);
    FieldRef f;
    snn_status r = field_ref(sim, field, pop_id, false, f);
    if (r != SNN_OK) return r;
    const uint64_t nel = f.bytes / f.elem;
    if (first > nel || count > nel - first)
        return sim->fail(SNN_E_INVALID, "range [%llu, +%llu) outside the field's %llu elements",
                         (unsigned long long)first, (unsigned long long)count, (unsigned long long)nel);
    if (!host_dst || dst_bytes < count * f.elem)
        return sim->fail(SNN_E_INVALID, "buffer of %zu bytes < %llu needed", dst_bytes,
                         (unsigned long long)(count * f.elem));
    if ((r = field_ref(sim, field, pop_id, true, f)) != SNN_OK) return r;
    return copy_out(sim, f, first, count, host_dst);
}

snn_status snn_partition(uint32_t n_targets, uint32_t slice_width, uint32_t world, uint32_t rank, uint32_t *lo,
                         uint32_t *hi) {
    if (world == 0 || rank >= world || !lo || !hi || slice_width == 0 || (slice_width & 31u))
        return SNN_E_INVALID;
    const uint64_t share = ((uint64_t)(n_targets + world - 1) / world + slice_width - 1) / slice_width * slice_width;
    *lo = (uint32_t)std::min<uint64_t>((uint64_t)rank * share, n_targets);
    *hi = (uint32_t)std::min<uint64_t>((uint64_t)(rank + 1) * share, n_targets);
    return SNN_OK;
}

snn_status snn_partition_weighted(const double *slice_cost, uint32_t nslices, uint32_t n_targets,
                                  uint32_t slice_width, uint32_t world, uint32_t rank, uint32_t *lo, uint32_t *hi) {
    if (world == 0 || rank >= world || !lo || !hi || slice_width == 0 || (slice_width & 31u) ||
        (uint64_t)nslices * slice_width < n_targets || (nslices > 0 && !slice_cost))
        return SNN_E_INVALID;
    double total = 0.0;
    for (uint32_t k = 0; k < nslices; k++) {
        if (!(slice_cost[k] >= 0.0)) return SNN_E_INVALID;
        total += slice_cost[k];
    }
    // boundary b_r (in slices): the prefix closest to r / world of the total,
    // non-decreasing in r; equal counts when every cost is 0
    auto boundary = [&](uint32_t r) -> uint32_t {
        if (r == 0) return 0;
        if (r >= world) return nslices;
        if (!(total > 0.0)) return (uint32_t)(((uint64_t)nslices * r) / world);
        const double goal = total * (double)r / (double)world;
        double pre = 0.0;
        uint32_t k = 0;
        while (k < nslices && pre + slice_cost[k] < goal) pre += slice_cost[k++];
        // pre < goal <= pre + cost[k]: the closer of k and k + 1
        if (k < nslices && (pre + slice_cost[k]) - goal < goal - pre) k++;
        return k;
    };
    uint32_t b0 = 0, b1 = 0;
    for (uint32_t r = 0; r <= rank; r++) {      // (monotone: each boundary >= the previous)
        b0 = std::max(b1, boundary(r));
        b1 = std::max(b0, boundary(r + 1));
    }
    *lo = (uint32_t)std::min<uint64_t>((uint64_t)b0 * slice_width, n_targets);
    *hi = (uint32_t)std::min<uint64_t>((uint64_t)b1 * slice_width, n_targets);
    return SNN_OK;
}

void snn_destroy(snn_sim *sim) {
    if (!sim) return;
    DeviceGuard dg(sim->cfg.device);
    if (sim->cfg.world > 1 && !sim->cfg.nccl_unique_id) {
        std::lock_guard<std::mutex> lk(g_mu);
        std::vector<snn_sim *> &g = g_groups[sim->cfg.group_key];
        for (size_t k = 0; k < g.size(); k++)
            if (g[k] == sim) {
                g.erase(g.begin() + k);
                break;
            }
    }
    if (sim->comm) g_nccl.commDestroy(sim->comm);
    if (sim->stream) cudaStreamSynchronize(sim->stream);
    cudaDeviceSynchronize();
    for (auto &g : sim->graphs) cudaGraphExecDestroy(g.second);
    for (auto &v : sim->ev_steps)
        for (auto e : v) cudaEventDestroy(e);
    for (void *p : sim->allocs) {
        if (sim->cfg.dev_free) sim->cfg.dev_free(p, (void *)sim->stream, sim->cfg.alloc_ctx);
        else cudaFree(p);
    }
    if (sim->cap_stream) cudaStreamDestroy(sim->cap_stream);
    if (sim->cap_side) cudaStreamDestroy(sim->cap_side);
    if (sim->cap_xside) cudaStreamDestroy(sim->cap_xside);
    if (sim->cap_front) cudaStreamDestroy(sim->cap_front);
    for (int q = 0; q < 2; q++) {
        if (sim->ev_fr[q]) cudaEventDestroy(sim->ev_fr[q]);
        if (sim->ev_del[q]) cudaEventDestroy(sim->ev_del[q]);
        if (sim->ev_fl_f[q]) cudaEventDestroy(sim->ev_fl_f[q]);
        if (sim->ev_lif[q]) cudaEventDestroy(sim->ev_lif[q]);
    }
    if (sim->ev_xfront) cudaEventDestroy(sim->ev_xfront);
    if (sim->ev_xdone) cudaEventDestroy(sim->ev_xdone);
    if (sim->ev_front) cudaEventDestroy(sim->ev_front);
    for (auto e : sim->ev_flush)
        if (e) cudaEventDestroy(e);

    delete sim;
}

}  // extern "C"
