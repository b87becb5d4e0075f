/*
 * snn_oracle.c -- plain, slow, obviously-correct CPU oracle for one clock-driven
 * SNN simulation step of arXiv 2107.04092 ("Spice").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path
 * (paper_2107_04092_b200/csrc); neither side includes or links the other.
 *
 * What it computes (PAPER.md line numbers, "P:n"):
 *   - the 3-phase step of P:34-42 (Sec. I): (1) update neurons, note firing,
 *     (2) update synapses -- NAIVE plasticity, Fig. 2a: every plastic
 *     synapse, every step, update(syn, n.hist[delay], syn.dst.hist[0]),
 *     (3) deliver spikes -- NAIVE row-wise delivery, Fig. 3a;
 *   - the firing history word, LSB = most recent step, pushed every step;
 *   - pivots by binary search (Fig. 1 caption; Sec. III-B);
 *   - fp32 arithmetic with forward Euler, no FMA contraction
 *     (compiled with -ffp-contract=off), constants computed in double and
 *     rounded to fp32 once (reading R19).
 * Readings of points the paper leaves open (model constants, STDP rule, fixed-point
 * accumulators, Philox counters) are listed in DESIGN.md section 3 and cited below
 * as "R<n>".
 *
 * Parity pins: see tests/test_oracle_*.py.  Long-run rate / weight-histogram
 * statistics are "parity unpinned" in absolute terms (R27).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <stdio.h>

#define OMAX_POP 16
#define OMAX_PROJ 64

enum { O_POISSON = 0, O_LIF_DELTA = 1, O_LIF_CUBA = 2 };
enum { O_STATIC = 0, O_STDP = 1 };

/* ---------------------------------------------------------------- Philox ----
 * Philox4x32-10 (Salmon et al., SC'11 "Parallel random numbers: as easy as
 * 1, 2, 3"), the counter-based generator named by BASELINE.json north_star.
 * Pinned by the Random123 known-answer vectors in tests/golden/philox_kat.txt. */
static void philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; r++) {
        if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void oracle_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    philox4x32_10(ctr, key, out);
}

/* Bernoulli(p) threshold, R22: keep iff u32 < floor(p * 2^32); p >= 1 -> always. */
static uint64_t bern_threshold(double p)
{
    if (p <= 0.0) return 0;
    if (p >= 1.0) return (uint64_t)1 << 32;
    return (uint64_t)floor(p * 4294967296.0);
}

/* ---------------------------------------------------------------- model ---- */
typedef struct {
    int kind;
    uint32_t base, n;
    /* user parameters (ms, mV, Hz) */
    float rate_hz, tau_m, v_rest, v_reset, v_th, tau_ref, tau_e, tau_i;
    /* derived, computed once in double and rounded to fp32 (R19) */
    uint64_t thr;      /* Poisson: floor(rate*dt * 2^32)                     */
    float k_m;         /* delta LIF: fp32(1 - dt/tau_m)                        */
    float a_m;         /* CUBA: fp32(dt/tau_m)                                 */
    float d_e, d_i;    /* CUBA: fp32(exp(-dt/tau_e)), fp32(exp(-dt/tau_i))     */
    int32_t n_ref;     /* round(tau_ref/dt)                                    */
} opop;

typedef struct {
    uint32_t src, dst;
    int kind, receptor, autapses;
    double p;
    uint64_t thr;
    float w, tau_plus, tau_minus, a_plus, a_minus, w_max;
    float d_plus, d_minus;  /* fp32(exp(-dt/tau_+)), fp32(exp(-dt/tau_-)) */
} oproj;

/* Geometric gap table of a projection (R32): gap_tab[k-1] = floor((1-p)^k 2^32),
 * k = 1..OGAP; the gap g >= 1 between kept candidates has P(g > k) =
 * gap_tab[k-1] / 2^32. */
#define OGAP 4096

typedef struct osim {
    uint32_t *gap_tab[OMAX_PROJ];   /* R32: per projection, OGAP entries */
    uint64_t seed;
    uint32_t key[2];
    float dt;
    uint32_t D;          /* network-wide delay in steps              */
    int32_t F;           /* fixed-point fraction bits of the accumulators R18 */
    float inv_scale;     /* 2^-F */
    float scale;         /* 2^F  */
    int npop, nproj;
    opop pop[OMAX_POP];
    oproj proj[OMAX_PROJ];
    int proj_of[OMAX_POP][OMAX_POP];
    uint32_t N;
    int finalized;
    int64_t t;           /* next step to compute */
    /* graph: CSR rows grouped by source, sorted; 1:1 synapse array */
    int64_t *row_ptr;    /* N+1 */
    uint32_t *idx;
    float *w;
    float *xpre, *xpost; /* per-synapse traces, 12 B per plastic synapse */
    int64_t nsyn;
    /* neuron state */
    float *V, *ge, *gi;
    int32_t *ref, *in_e, *in_i;
    uint64_t *hist;
    uint32_t *nspk;
    uint64_t events;     /* delivered (spike, target) pairs, R24 */
    uint64_t stdp_updates;
    int nthreads;
} osim;

static int pop_of(const osim *s, uint32_t j)
{
    for (int d = 0; d < s->npop; d++)
        if (j >= s->pop[d].base && j < s->pop[d].base + s->pop[d].n) return d;
    return -1;
}

osim *oracle_create(uint64_t seed, float dt_ms, uint32_t delay, int32_t frac_bits)
{
    if (delay >= 64 || frac_bits < 0 || frac_bits > 30) return NULL;
    osim *s = (osim *)calloc(1, sizeof(osim));
    s->seed = seed;
    s->key[0] = (uint32_t)(seed & 0xffffffffu);
    s->key[1] = (uint32_t)(seed >> 32);
    s->dt = dt_ms;
    s->D = delay;
    s->F = frac_bits;
    s->scale = ldexpf(1.0f, frac_bits);
    s->inv_scale = ldexpf(1.0f, -frac_bits);
    for (int a = 0; a < OMAX_POP; a++)
        for (int b = 0; b < OMAX_POP; b++) s->proj_of[a][b] = -1;
    s->nthreads = 1;
    return s;
}

void oracle_set_threads(osim *s, int n) { s->nthreads = n < 1 ? 1 : n; }

/* params: rate_hz, tau_m, v_rest, v_reset, v_th, tau_ref, tau_e, tau_i */
int oracle_add_pop(osim *s, int kind, uint32_t n, const float *prm)
{
    if (s->finalized || s->npop >= OMAX_POP || n == 0) return -1;
    if (kind < O_POISSON || kind > O_LIF_CUBA) return -1;
    opop *p = &s->pop[s->npop];
    memset(p, 0, sizeof(*p));
    p->kind = kind;
    p->base = s->N;
    p->n = n;
    p->rate_hz = prm[0]; p->tau_m = prm[1]; p->v_rest = prm[2]; p->v_reset = prm[3];
    p->v_th = prm[4]; p->tau_ref = prm[5]; p->tau_e = prm[6]; p->tau_i = prm[7];
    double dt = (double)s->dt;
    p->thr = bern_threshold((double)p->rate_hz * 1e-3 * dt);
    if (kind != O_POISSON) {
        p->k_m = (float)(1.0 - dt / (double)p->tau_m);
        p->a_m = (float)(dt / (double)p->tau_m);
        p->n_ref = (int32_t)llround((double)p->tau_ref / dt);
        if (kind == O_LIF_CUBA) {
            p->d_e = (float)exp(-dt / (double)p->tau_e);
            p->d_i = (float)exp(-dt / (double)p->tau_i);
        }
    }
    s->N += n;
    return s->npop++;
}

/* f: weight, tau_plus, tau_minus, a_plus, a_minus, w_max */
int oracle_connect(osim *s, uint32_t src, uint32_t dst, int kind, int receptor, double p,
                   const float *f, int autapses)
{
    if (s->finalized || s->nproj >= OMAX_PROJ) return -1;
    if ((int)src >= s->npop || (int)dst >= s->npop || p < 0.0 || p > 1.0) return -1;
    if (s->proj_of[src][dst] >= 0) return -1;
    if (s->pop[dst].kind == O_POISSON) return -1;
    if (s->pop[dst].kind == O_LIF_DELTA && receptor != 0) return -1;
    if (receptor < 0 || receptor > 1) return -1;
    oproj *q = &s->proj[s->nproj];
    memset(q, 0, sizeof(*q));
    q->src = src; q->dst = dst; q->kind = kind; q->receptor = receptor;
    q->autapses = autapses; q->p = p; q->thr = bern_threshold(p);
    /* R32: gap table floor((1-p)^k 2^32), k = 1..OGAP, in double */
    s->gap_tab[s->nproj] = (uint32_t *)malloc(OGAP * sizeof(uint32_t));
    for (int k = 1; k <= OGAP; k++) {
        double v = floor(pow(1.0 - p, (double)k) * 4294967296.0);
        s->gap_tab[s->nproj][k - 1] = v >= 4294967295.0 ? 4294967295u : (uint32_t)v;
    }
    q->w = f[0]; q->tau_plus = f[1]; q->tau_minus = f[2];
    q->a_plus = f[3]; q->a_minus = f[4]; q->w_max = f[5];
    if (kind == O_STDP) {
        q->d_plus = (float)exp(-(double)s->dt / (double)q->tau_plus);
        q->d_minus = (float)exp(-(double)s->dt / (double)q->tau_minus);
    }
    s->proj_of[src][dst] = s->nproj;
    return s->nproj++;
}

/* Row i of the graph (grouped by source, sorted): for each destination
 * population d in ascending id order, the kept candidates are found by exact
 * geometric skipping (R32, R23): the candidates are d's neurons ascending,
 * without i itself unless autapses are allowed (R21); starting before the
 * first, each draw x_n = Philox(i, n>>2, 4, d)[n & 3] (n = 0, 1, ...) advances
 * by the gap g(x) = 1 + #{k in 1..OGAP : gap_tab[k-1] > x} and keeps the
 * candidate reached; a draw below gap_tab[OGAP-1] advances OGAP and keeps
 * nothing (the geometric law is memoryless).  p = 1 keeps every candidate,
 * p = 0 none.  Only targets in [lo, hi) are produced (a rank's column range,
 * DESIGN.md section 7).  Returns the row length; writes at most cap ids. */
int64_t oracle_build_row(const osim *s, uint32_t i, uint32_t lo, uint32_t hi,
                         uint32_t *out, int64_t cap)
{
    int sp = pop_of(s, i);
    if (sp < 0) return -1;
    int64_t len = 0;
    for (int d = 0; d < s->npop; d++) {
        int pj = s->proj_of[sp][d];
        if (pj < 0) continue;
        const oproj *q = &s->proj[pj];
        if (q->p <= 0.0) continue;
        const uint32_t *tab = s->gap_tab[pj];
        const opop *dp = &s->pop[d];
        /* candidate list: d's local indices, i's own left out (no autapse) */
        int excl = !q->autapses && i >= dp->base && i < dp->base + dp->n;
        uint32_t il = i - dp->base;
        int64_t M = (int64_t)dp->n - (excl ? 1 : 0);
        int64_t c = -1;
        for (uint64_t n = 0;; n++) {
            uint32_t ctr[4] = { i, (uint32_t)(n >> 2), 4u, (uint32_t)d };
            uint32_t r[4];
            philox4x32_10(ctr, s->key, r);
            uint32_t x = r[n & 3];
            /* g = 1 + number of k with tab[k-1] > x (tab is non-increasing) */
            int64_t g = 1;
            while (g <= OGAP && tab[g - 1] > x) g++;
            if (g > OGAP) {            /* beyond the table: advance, keep nothing */
                c += OGAP;
                if (c >= M) break;
                continue;
            }
            c += g;
            if (c >= M) break;
            uint32_t jl = (uint32_t)c + ((excl && (uint32_t)c >= il) ? 1u : 0u);
            uint32_t j = dp->base + jl;
            if (j >= hi) break;
            if (j >= lo) {
                if (len < cap) out[len] = j;
                len++;
            }
        }
    }
    return len;
}

/* Pivots by binary search, Fig. 1 caption and P:348: piv[k] = index of
 * the first entry >= lo + k*C, k = 0..nslices (the explicit leading 0 and the
 * row-end value included, R16).  row must be sorted ascending. */
static int64_t lower_bound_u32(const uint32_t *row, int64_t len, uint64_t v)
{
    int64_t a = 0, b = len;
    while (a < b) {
        int64_t m = a + (b - a) / 2;
        if ((uint64_t)row[m] < v) a = m + 1; else b = m;
    }
    return a;
}

void oracle_pivots(const uint32_t *row, int64_t len, uint32_t lo, uint32_t C,
                   uint32_t nslices, int64_t *piv)
{
    for (uint32_t k = 0; k <= nslices; k++)
        piv[k] = lower_bound_u32(row, len, (uint64_t)lo + (uint64_t)k * C);
}

/* Initial state, R: V0 = v_reset + (v_th - v_reset) * u, u = (x >> 8) 2^-24,
 * x = Philox(i, 0, 3, 0)[0]; everything else 0; tlu = -1 implicit (naive). */
static void init_state(osim *s)
{
    for (int d = 0; d < s->npop; d++) {
        const opop *p = &s->pop[d];
        for (uint32_t k = 0; k < p->n; k++) {
            uint32_t i = p->base + k;
            if (p->kind == O_POISSON) { s->V[i] = 0.0f; continue; }
            uint32_t ctr[4] = { i, 0u, 3u, 0u };
            uint32_t r[4];
            philox4x32_10(ctr, s->key, r);
            float u = (float)(r[0] >> 8) * 0x1p-24f;
            float span = p->v_th - p->v_reset;
            float prod = span * u;
            s->V[i] = p->v_reset + prod;
        }
    }
}

int oracle_finalize(osim *s)
{
    if (s->finalized) return -1;
    uint32_t N = s->N;
    s->row_ptr = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
    /* pass 1: row lengths (rows are independent: the threads only share the
     * read-only tables), then their running sum */
    #pragma omp parallel for num_threads(s->nthreads) schedule(dynamic, 256)
    for (int64_t i = 0; i < (int64_t)N; i++)
        s->row_ptr[i + 1] = oracle_build_row(s, (uint32_t)i, 0, N, NULL, 0);
    for (uint32_t i = 0; i < N; i++)
        s->row_ptr[i + 1] += s->row_ptr[i];
    s->nsyn = s->row_ptr[N];
    size_t ns = (size_t)(s->nsyn > 0 ? s->nsyn : 1);
    s->idx = (uint32_t *)malloc(ns * sizeof(uint32_t));
    s->w = (float *)malloc(ns * sizeof(float));
    s->xpre = (float *)calloc(ns, sizeof(float));
    s->xpost = (float *)calloc(ns, sizeof(float));
    /* pass 2: fill */
    #pragma omp parallel for num_threads(s->nthreads) schedule(dynamic, 256)
    for (int64_t ii = 0; ii < (int64_t)N; ii++) {
        uint32_t i = (uint32_t)ii;
        int64_t b = s->row_ptr[i], len = s->row_ptr[i + 1] - b;
        oracle_build_row(s, i, 0, N, s->idx + b, len);
        int sp = pop_of(s, i);
        for (int64_t c = 0; c < len; c++) {
            int dp = pop_of(s, s->idx[b + c]);
            s->w[b + c] = s->proj[s->proj_of[sp][dp]].w;
        }
    }
    s->V = (float *)calloc(N, sizeof(float));
    s->ge = (float *)calloc(N, sizeof(float));
    s->gi = (float *)calloc(N, sizeof(float));
    s->ref = (int32_t *)calloc(N, sizeof(int32_t));
    s->in_e = (int32_t *)calloc(N, sizeof(int32_t));
    s->in_i = (int32_t *)calloc(N, sizeof(int32_t));
    s->hist = (uint64_t *)calloc(N, sizeof(uint64_t));
    s->nspk = (uint32_t *)calloc(N, sizeof(uint32_t));
    init_state(s);
    s->t = 0;
    s->finalized = 1;
    return 0;
}

/* Step (1): neuron update, R9/R20 op order, fp32, Euler. */
static int neuron_update(osim *s, uint32_t i, const opop *p)
{
    int fired = 0;
    if (p->kind == O_POISSON) {
        uint32_t ctr[4] = { i, (uint32_t)s->t, 2u, 0u };
        uint32_t r[4];
        philox4x32_10(ctr, s->key, r);
        fired = (uint64_t)r[0] < p->thr;
    } else if (p->kind == O_LIF_DELTA) {
        float I = (float)s->in_e[i] * s->inv_scale;
        s->in_e[i] = 0;
        if (s->ref[i] > 0) {
            s->ref[i] -= 1;
        } else {
            float v = s->V[i] * p->k_m;
            s->V[i] = v + I;
        }
        if (s->ref[i] == 0 && s->V[i] >= p->v_th) {
            fired = 1;
            s->V[i] = p->v_reset;
            s->ref[i] = p->n_ref;
        }
    } else { /* O_LIF_CUBA */
        float ie = (float)s->in_e[i] * s->inv_scale;
        float ii = (float)s->in_i[i] * s->inv_scale;
        s->ge[i] = s->ge[i] + ie;
        s->gi[i] = s->gi[i] + ii;
        s->in_e[i] = 0;
        s->in_i[i] = 0;
        if (s->ref[i] > 0) {
            s->ref[i] -= 1;
        } else {
            float t1 = p->v_rest - s->V[i];
            float t2 = t1 + s->ge[i];
            float t3 = t2 + s->gi[i];
            float dv = p->a_m * t3;
            s->V[i] = s->V[i] + dv;
        }
        s->ge[i] = s->ge[i] * p->d_e;
        s->gi[i] = s->gi[i] * p->d_i;
        if (s->ref[i] == 0 && s->V[i] >= p->v_th) {
            fired = 1;
            s->V[i] = p->v_reset;
            s->ref[i] = p->n_ref;
        }
    }
    return fired;
}

/* Step (2): naive plasticity, Fig. 2a: every plastic synapse gets
 * update(syn, n.hist[delay], syn.dst.hist[0]).  update() is the additive pair
 * STDP with exponential traces of R7 (one step, post-then-pre order):
 *   x_pre *= d+;  x_post *= d-;
 *   if post: w = min(w + A+ x_pre, w_max); x_post += 1
 *   if pre:  w = max(w - A- x_post, 0);    x_pre  += 1                         */
static void naive_stdp_synapse(const oproj *q, int pre, int post, float *w_, float *xp_, float *xq_)
{
    float xp = *xp_ * q->d_plus;
    float xq = *xq_ * q->d_minus;
    float w = *w_;
    if (post) {
        float dw = q->a_plus * xp;
        float nw = w + dw;
        w = nw < q->w_max ? nw : q->w_max;
        xq = xq + 1.0f;
    }
    if (pre) {
        float dw = q->a_minus * xq;
        float nw = w - dw;
        w = nw > 0.0f ? nw : 0.0f;
        xp = xp + 1.0f;
    }
    *w_ = w;
    *xp_ = xp;
    *xq_ = xq;
}

static void naive_stdp_row(osim *s, uint32_t i, int sp)
{
    int pre = (int)((s->hist[i] >> s->D) & 1u);
    int64_t b = s->row_ptr[i], e = s->row_ptr[i + 1];
    for (int64_t c = b; c < e; c++) {
        uint32_t j = s->idx[c];
        int pj = s->proj_of[sp][pop_of(s, j)];
        const oproj *q = &s->proj[pj];
        if (q->kind != O_STDP) continue;
        int post = (int)(s->hist[j] & 1u);
        naive_stdp_synapse(q, pre, post, &s->w[c], &s->xpre[c], &s->xpost[c]);
    }
}

/* The same per-synapse update, replayed for one synapse of the STDP projection
 * src_pop -> dst_pop over T steps from the initial state (w0, traces 0), with
 * its pre events (pre[t]: the source fired at t - D) and post events (post[t]:
 * the target fired at t) given -- the naive oracle on a sampled synapse of a
 * network too large to run here in full.  Returns the weight, NAN if the
 * projection is not plastic. */
float oracle_synapse_replay(const osim *s, int src_pop, int dst_pop, const uint8_t *pre, const uint8_t *post,
                            int64_t T)
{
    int pj = s->proj_of[src_pop][dst_pop];
    if (pj < 0 || s->proj[pj].kind != O_STDP) return NAN;
    const oproj *q = &s->proj[pj];
    float w = q->w, xp = 0.0f, xq = 0.0f;
    for (int64_t t = 0; t < T; t++) naive_stdp_synapse(q, pre[t] != 0, post[t] != 0, &w, &xp, &xq);
    return w;
}

/* Quantisation of a weight to the int32 fixed-point accumulator, R18:
 * q(w) = round-to-nearest-even(w * 2^F). */
static int32_t quantize(const osim *s, float w)
{
    return (int32_t)lrintf(w * s->scale);
}

static int pop_has_stdp(const osim *s, int sp)
{
    for (int d = 0; d < s->npop; d++) {
        int pj = s->proj_of[sp][d];
        if (pj >= 0 && s->proj[pj].kind == O_STDP) return 1;
    }
    return 0;
}

void oracle_step(osim *s, uint32_t nsteps)
{
    if (!s->finalized) return;
    for (uint32_t it = 0; it < nsteps; it++) {
        /* (1) update neurons, note which ones fire; push history */
        for (int d = 0; d < s->npop; d++) {
            const opop *p = &s->pop[d];
            #pragma omp parallel for num_threads(s->nthreads) schedule(static)
            for (int64_t k = 0; k < (int64_t)p->n; k++) {
                uint32_t i = p->base + (uint32_t)k;
                int f = neuron_update(s, i, p);
                s->hist[i] = (s->hist[i] << 1) | (uint64_t)f;
                s->nspk[i] += (uint32_t)f;
            }
        }
        /* (2) update synapses: naive plasticity over every plastic synapse */
        uint64_t upd = 0;
        for (int sp = 0; sp < s->npop; sp++) {
            if (!pop_has_stdp(s, sp)) continue;
            const opop *p = &s->pop[sp];
            #pragma omp parallel for num_threads(s->nthreads) schedule(dynamic, 64)
            for (int64_t k = 0; k < (int64_t)p->n; k++)
                naive_stdp_row(s, p->base + (uint32_t)k, sp);
            upd += 1;
        }
        s->stdp_updates += upd;
        /* (3) deliver spikes, row-wise (Fig. 3a): every neuron whose
         * spike arrives now, i.e. fired D steps ago (hist[delay]), adds
         * q(w) of each outgoing synapse to the target's receptor accumulator,
         * consumed by the target's neuron update at step t+1 (R5). */
        for (uint32_t i = 0; i < s->N; i++) {
            if (!((s->hist[i] >> s->D) & 1u)) continue;
            int sp = pop_of(s, i);
            for (int64_t c = s->row_ptr[i]; c < s->row_ptr[i + 1]; c++) {
                uint32_t j = s->idx[c];
                const oproj *q = &s->proj[s->proj_of[sp][pop_of(s, j)]];
                int32_t v = quantize(s, s->w[c]);
                if (q->receptor == 0) s->in_e[j] += v; else s->in_i[j] += v;
                s->events++;
            }
        }
        s->t++;
    }
}

/* ------------------------------------------------------------- accessors --- */
uint32_t oracle_n(const osim *s) { return s->N; }
int64_t oracle_nsyn(const osim *s) { return s->nsyn; }
int64_t oracle_t(const osim *s) { return s->t; }
void oracle_set_t(osim *s, int64_t t) { s->t = t; }
uint64_t oracle_events(const osim *s) { return s->events; }
int oracle_pop_of(const osim *s, uint32_t j) { return pop_of(s, j); }

/* field ids: 0 V, 1 ge, 2 gi, 3 ref, 4 in_e, 5 in_i, 6 hist, 7 nspk,
 *            8 row_ptr, 9 idx, 10 w, 11 xpre, 12 xpost */
void *oracle_field(osim *s, int f)
{
    switch (f) {
    case 0: return s->V;      case 1: return s->ge;     case 2: return s->gi;
    case 3: return s->ref;    case 4: return s->in_e;   case 5: return s->in_i;
    case 6: return s->hist;   case 7: return s->nspk;   case 8: return s->row_ptr;
    case 9: return s->idx;    case 10: return s->w;     case 11: return s->xpre;
    case 12: return s->xpost;
    default: return NULL;
    }
}

void oracle_destroy(osim *s)
{
    if (!s) return;
    free(s->row_ptr); free(s->idx); free(s->w); free(s->xpre); free(s->xpost);
    free(s->V); free(s->ge); free(s->gi); free(s->ref); free(s->in_e); free(s->in_i);
    free(s->hist); free(s->nspk);
    for (int k = 0; k < s->nproj; k++) free(s->gap_tab[k]);
    free(s);
}
