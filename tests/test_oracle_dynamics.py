"""Pins of the oracle's neuron dynamics, STDP and delivery against closed forms,
textbook routines and hand-wired spike trains (never against itself)."""
import math

import numpy as np
import pytest

from oracle import oracle as O

F = 20
Q = 2.0 ** F
DT = 0.1


def q(x):
    return int(np.rint(np.float32(x) * np.float32(Q)))


# ------------------------------------------------------------------ LIF (delta)
def _delta(n=1, v_reset=10.0, v_th=20.0, tau_ref=0.0, seed=5):
    o = O.Oracle(seed, DT, 0, F)
    o.add_population(O.LIF_DELTA, n, tau_m=20.0, v_reset=v_reset, v_th=v_th, tau_ref=tau_ref)
    o.finalize()
    return o


def test_delta_lif_free_decay_closed_form():
    """No input: V_n = V_0 (1 - dt/tau)^n (Euler)."""
    o = _delta(4)
    V = o.array("V")
    v0 = V.astype(np.float64).copy()
    assert np.all((v0 >= 10.0) & (v0 < 20.0))       # initial V in [v_reset, v_th)
    for n in range(1, 201):
        o.step(1)
        exact = v0 * (1.0 - DT / 20.0) ** n
        assert np.allclose(V, exact, rtol=2e-5, atol=0)


def test_delta_lif_constant_input_closed_form_and_first_spike():
    """Constant input I per step: V_n = V_inf + (V_0 - V_inf) k^n with
    V_inf = I / (1 - k); the first threshold crossing happens at the step the
    closed form predicts."""
    o = _delta(1, v_th=1e9)               # no firing: follow the trajectory
    V, ine = o.array("V"), o.array("in_e")
    I = 0.5
    k = 1.0 - DT / 20.0
    v0 = float(V[0])
    vinf = I / (1 - k)
    for n in range(1, 300):
        ine[0] = q(I)
        o.step(1)
        exact = vinf + (v0 - vinf) * k ** n
        assert abs(V[0] - exact) <= 3e-5 * abs(exact)
    o2 = _delta(1, v_th=30.0)
    V2, ine2 = o2.array("V"), o2.array("in_e")
    v0 = float(V2[0])
    n_pred = next(n for n in range(1, 10000) if vinf + (v0 - vinf) * k ** n >= 30.0)
    for n in range(1, n_pred + 1):
        ine2[0] = q(I)
        o2.step(1)
        fired = int(o2.array("hist")[0] & 1)
        assert fired == (n == n_pred)
    assert V2[0] == np.float32(10.0)      # reset value exact


def test_refractory_length_exact_and_inputs_discarded():
    """tau_ref = 2 ms -> 20 steps held at V_reset, delta inputs discarded (R20)."""
    o = _delta(1, tau_ref=2.0)
    V, ine, ref = o.array("V"), o.array("in_e"), o.array("ref")
    ine[0] = q(50.0)
    o.step(1)
    assert o.array("hist")[0] & 1
    assert ref[0] == 20
    for s in range(20):
        ine[0] = q(50.0)
        o.step(1)
        assert not (o.array("hist")[0] & 1)
        assert V[0] == np.float32(10.0)
    ine[0] = q(50.0)
    o.step(1)                              # 21st step: integrates and fires again
    assert o.array("hist")[0] & 1


# -------------------------------------------------------------------- CUBA LIF
def test_cuba_exponential_conductance_and_voltage_closed_form():
    """A pulse g0 into the exc receptor: g_n = g0 d^n; V follows the linear
    recurrence V_{n+1} = V_n + a (E_l - V_n + g_n), whose closed form is
    V_n = E_l + (V0-E_l) r^n + a g0 (d^n - r^n)/(d - r), r = 1 - a."""
    o = O.Oracle(9, DT, 0, F)
    o.add_population(O.LIF_CUBA, 1, tau_m=20.0, v_rest=-49.0, v_reset=-60.0, v_th=1e9,
                     tau_ref=5.0, tau_e=5.0, tau_i=10.0)
    o.finalize()
    V, ge, ine = o.array("V"), o.array("ge"), o.array("in_e")
    v0 = float(V[0])
    g0 = 2.0
    a = DT / 20.0
    r = 1 - a
    d = math.exp(-DT / 5.0)
    ine[0] = q(g0)
    for n in range(1, 400):
        o.step(1)
        assert abs(ge[0] - g0 * d ** n) <= 2e-5 * g0 * d ** n + 1e-30
        # V after n updates: uses g_0..g_{n-1}
        exact = -49.0 + (v0 + 49.0) * r ** n + a * g0 * (d ** n - r ** n) / (d - r)
        assert abs(V[0] - exact) <= 2e-5 * abs(exact)


# --------------------------------------------------------------------- Poisson
def test_poisson_rate_and_independence():
    o = O.Oracle(123, DT, 0, F)
    o.add_population(O.POISSON, 2000, rate_hz=16.0)
    o.finalize()
    T = 2000
    counts = np.zeros(2000)
    prev = None
    same = 0
    for t in range(T):
        o.step(1)
        s = (o.array("hist") & 1).astype(bool)
        counts += s
        if prev is not None:
            same += int(np.sum(s & prev))
        prev = s
    p = 16.0 * 1e-3 * DT
    n = 2000 * T
    assert abs(counts.sum() / n - p) < 5 * math.sqrt(p * (1 - p) / n)
    # consecutive steps independent: joint rate ~ p^2
    assert abs(same / (2000 * (T - 1)) - p * p) < 5 * math.sqrt(p * p / (2000 * (T - 1)))


# ------------------------------------------------------------------ STDP (R7)
A_PLUS, A_MINUS, W_MAX, TAU = 0.01, 0.0105, 1.0, 20.0


def _pair(delay=0, w0=0.5, seed=1):
    """Two delta neurons A -> B (p = 1, STDP).  Neither fires unless forced."""
    o = O.Oracle(seed, DT, delay, F)
    a = o.add_population(O.LIF_DELTA, 1, tau_m=20.0, v_reset=0.0, v_th=20.0)
    b = o.add_population(O.LIF_DELTA, 1, tau_m=20.0, v_reset=0.0, v_th=20.0)
    o.connect(a, b, O.STDP, 0, 1.0, w0, tau_plus=TAU, tau_minus=TAU, a_plus=A_PLUS,
              a_minus=A_MINUS, w_max=W_MAX)
    o.finalize()
    return o


def _run(o, fire_at, T):
    """fire_at: {step: [neuron ids]} forced by a large input."""
    ine = o.array("in_e")
    for t in range(T):
        for i in fire_at.get(t, []):
            ine[i] = q(100.0)
        o.step(1)


@pytest.mark.parametrize("delay", [0, 3, 15])
@pytest.mark.parametrize("dlt", [1, 5, 37, 63])
def test_stdp_pre_then_post_potentiation_closed_form(delay, dlt):
    """Pre at u (arrival D steps after the source spike), post at u+dlt:
    dw = A+ exp(-dlt dt / tau+)."""
    o = _pair(delay)
    u = 10 + delay
    _run(o, {10: [0], u + dlt: [1]}, u + dlt + 1)
    dw = float(o.array("w")[0]) - 0.5
    assert abs(dw - A_PLUS * math.exp(-dlt * DT / TAU)) <= 1e-5 * A_PLUS + 1e-7


@pytest.mark.parametrize("dlt", [1, 7, 40])
def test_stdp_post_then_pre_depression_closed_form(dlt):
    o = _pair(0)
    _run(o, {10: [1], 10 + dlt: [0]}, 10 + dlt + 1)
    dw = float(o.array("w")[0]) - 0.5
    assert abs(dw + A_MINUS * math.exp(-dlt * DT / TAU)) <= 1e-5 * A_MINUS + 1e-7


def test_stdp_same_step_is_post_then_pre():
    """Same step: potentiation sees x_pre before the pre increment (0) and the
    depression sees x_post after the post increment (1): dw = -A- (R7)."""
    o = _pair(0)
    _run(o, {10: [0, 1]}, 11)
    assert abs(float(o.array("w")[0]) - (0.5 - A_MINUS)) < 1e-7


def test_stdp_hard_bounds_and_no_spike_no_change():
    o = _pair(0, w0=W_MAX - 1e-4)
    _run(o, {10: [0], 11: [1]}, 12)
    assert o.array("w")[0] == np.float32(W_MAX)
    o = _pair(0, w0=1e-4)
    _run(o, {10: [1], 11: [0]}, 12)
    assert o.array("w")[0] == np.float32(0.0)
    o = _pair(0)
    _run(o, {}, 300)
    assert o.array("w")[0] == np.float32(0.5)


# -------------------------------------------------------------------- delivery
def test_delivery_equals_dense_matvec():
    """Row-wise delivery (Fig. 3a) = the matrix-vector product of the spike
    vector s(t-D) with the quantised weight matrix (a textbook routine)."""
    import workloads as W
    rc = W.brunel(1200, p=0.05, plastic=False, delay=2, seed=4)
    o = O.Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
    rc.apply(o)
    o.finalize()
    N = o.n
    rp, idx, w = o.array("row_ptr"), o.array("idx"), o.array("w")
    Wq = np.zeros((N, N), dtype=np.int64)
    for i in range(N):
        for c in range(rp[i], rp[i + 1]):
            Wq[i, idx[c]] += int(np.rint(np.float64(w[c]) * Q))
    checked = 0
    for t in range(60):
        o.step(1)
        s = ((o.array("hist") >> np.uint64(rc.delay)) & np.uint64(1)).astype(np.int64)
        assert np.array_equal(o.array("in_e").astype(np.int64), s @ Wq)
        checked += int(s.sum())
    assert checked > 0


def test_quantisation_rounds_half_to_even():
    """q(w) = RNE(w 2^F) (R18): ties go to the even integer."""
    for frac, expect in [(2.5, 2), (3.5, 4), (-2.5, -2), (1.25, 1)]:
        o = O.Oracle(1, DT, 0, F)
        a = o.add_population(O.LIF_DELTA, 1, v_reset=0.0, v_th=20.0)
        b = o.add_population(O.LIF_DELTA, 1, v_reset=0.0, v_th=1e9)
        o.connect(a, b, O.STATIC, 0, 1.0, frac / Q)
        o.finalize()
        o.array("in_e")[0] = q(100.0)
        o.step(1)
        assert o.array("in_e")[1] == expect


def test_synapse_replay_equals_the_network_oracle():
    """oracle.synapse_replay (used to check sampled synapses of networks too
    large for the full oracle) reproduces, for every plastic synapse of a small
    Brunel+ network, the weight the network oracle computes over 150 steps
    (same per-synapse update, pre = source fired at t - D, post = target fired
    at t)."""
    import workloads as W
    rc = W.brunel(1500, p=0.1, plastic=True, delay=3, seed=5)
    o = O.Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
    rc.apply(o)
    o.finalize()
    T = 150
    fired = np.zeros((T, o.n), dtype=np.uint8)
    for t in range(T):
        o.step(1)
        fired[t] = (o.array("hist") & 1).astype(np.uint8)
    rp, idx, w = o.array("row_ptr"), o.array("idx"), o.array("w")
    ne, ni = rc.pops[0].n, rc.pops[1].n
    base_p = ne + ni
    pre_shift = np.zeros_like(fired)
    pre_shift[rc.delay:] = fired[:T - rc.delay]
    checked = 0
    rng = np.random.default_rng(1)
    for i in rng.choice(np.arange(base_p, o.n), 40, replace=False):
        for c in range(rp[i], rp[i + 1]):
            j = idx[c]
            if j >= ne:
                continue
            ww = o.synapse_replay(2, 0, pre_shift[:, i], fired[:, j])
            assert ww == w[c], (i, j, ww, w[c])
            checked += 1
    assert checked > 200
    assert np.isnan(o.synapse_replay(0, 0, pre_shift[:, 0], fired[:, 0]))   # E -> E is static


# --------------------------------------------- STDP over several spikes (R7)
def _d(n):
    return math.exp(-n * DT / TAU)


@pytest.mark.parametrize("delay", [0, 4])
def test_stdp_two_pre_then_post_traces_accumulate(delay):
    """All-to-all pair STDP (R7): the pre trace sums every earlier pre spike,
    x_pre(v) = d^(v-u1) + d^(v-u2), so a post at v after pre arrivals at u1 < u2
    gives dw = A+ (d^(v-u1) + d^(v-u2)).  A nearest-neighbour trace (reset to 1
    at a spike) would give A+ d^(v-u2) only."""
    o = _pair(delay)
    u1, u2, v = 10 + delay, 17 + delay, 29 + delay
    _run(o, {u1 - delay: [0], u2 - delay: [0], v: [1]}, v + 1)
    dw = float(o.array("w")[0]) - 0.5
    exp = A_PLUS * (_d(v - u1) + _d(v - u2))
    assert abs(dw - exp) <= 1e-5 * exp
    assert abs(dw - A_PLUS * _d(v - u2)) > 0.1 * A_PLUS * _d(v - u1)     # not nearest-neighbour


def test_stdp_pre_post_pre_triplet():
    """pre at u1, post at v, pre at u2 > v: potentiation at v by x_pre(v) =
    d^(v-u1), depression at u2 by x_post(u2) = d^(u2-v):
    dw = A+ d^(v-u1) - A- d^(u2-v)."""
    o = _pair(0)
    u1, v, u2 = 10, 16, 25
    _run(o, {u1: [0], v: [1], u2: [0]}, u2 + 1)
    dw = float(o.array("w")[0]) - 0.5
    exp = A_PLUS * _d(v - u1) - A_MINUS * _d(u2 - v)
    assert abs(dw - exp) <= 1e-5 * (A_PLUS + A_MINUS)


def test_stdp_post_post_pre_depression_sums_post_trace():
    """posts at v1 < v2, then a pre at u: the potentiations see x_pre = 0 and
    the depression sees x_post(u) = d^(u-v1) + d^(u-v2):
    dw = -A- (d^(u-v1) + d^(u-v2))."""
    o = _pair(0)
    v1, v2, u = 10, 13, 30
    _run(o, {v1: [1], v2: [1], u: [0]}, u + 1)
    dw = float(o.array("w")[0]) - 0.5
    exp = -A_MINUS * (_d(u - v1) + _d(u - v2))
    assert abs(dw - exp) <= 1e-5 * abs(exp)


def test_stdp_pre_pre_post_post_four_pairs():
    """Two pre then two post spikes: every (pre, post) pair contributes,
    dw = A+ sum_{a,b} d^(v_b - u_a) (four terms)."""
    o = _pair(0)
    u1, u2, v1, v2 = 10, 12, 20, 33
    _run(o, {u1: [0], u2: [0], v1: [1], v2: [1]}, v2 + 1)
    dw = float(o.array("w")[0]) - 0.5
    exp = A_PLUS * sum(_d(v - u) for u in (u1, u2) for v in (v1, v2))
    assert abs(dw - exp) <= 1e-5 * exp


def test_stdp_sequential_upper_bound_per_post_spike():
    """The hard bound applies at every post spike (min(w + A+ x_pre, w_max)),
    not once at the end: from w0 = w_max - A+/2, a pre then two posts saturate
    at w_max and stay there."""
    o = _pair(0, w0=W_MAX - A_PLUS / 2)
    _run(o, {10: [0], 11: [1], 12: [1]}, 13)
    assert o.array("w")[0] == np.float32(W_MAX)


# ------------------------------------------------- CUBA refractory (R20)
def test_cuba_refractory_holds_v_while_currents_integrate():
    """R20 (CUBA): for n_ref = round(tau_ref / dt) = 50 steps after a spike V
    is held at V_reset, while the exponential currents keep decaying and keep
    taking input: g_n = sum_k in_k d^(n-k).  The first step after the
    refractory period integrates with the accumulated currents:
    V = V_reset + a (E_l - V_reset + g_e + g_i)."""
    o = O.Oracle(9, DT, 0, F)
    o.add_population(O.LIF_CUBA, 1, tau_m=20.0, v_rest=-49.0, v_reset=-60.0, v_th=-50.0,
                     tau_ref=5.0, tau_e=5.0, tau_i=10.0)
    o.finalize()
    V, ge, gi, ine, ini, ref = (o.array(k) for k in ("V", "ge", "gi", "in_e", "in_i", "ref"))
    de, di, a = math.exp(-DT / 5.0), math.exp(-DT / 10.0), DT / 20.0
    inputs_e = {0: 2000.0, 12: 3.0, 40: 1.5}        # step -> exc input (the first one forces the spike)
    inputs_i = {20: -4.0, 50: -2.0}
    T = 52
    for n in range(T):
        if n in inputs_e:
            ine[0] = q(inputs_e[n])
        if n in inputs_i:
            ini[0] = q(inputs_i[n])
        o.step(1)
        fired = int(o.array("hist")[0] & 1)
        ge_exp = sum(q(x) / Q * de ** (n - k + 1) for k, x in inputs_e.items() if k <= n)
        gi_exp = sum(q(x) / Q * di ** (n - k + 1) for k, x in inputs_i.items() if k <= n)
        assert abs(ge[0] - ge_exp) <= 1e-5 * abs(ge_exp)
        if gi_exp:
            assert abs(gi[0] - gi_exp) <= 1e-5 * abs(gi_exp)
        if n == 0:
            assert fired and ref[0] == 50 and V[0] == np.float32(-60.0)
        elif n <= 50:
            assert not fired and V[0] == np.float32(-60.0), n     # held for exactly 50 steps
            assert ref[0] == 50 - n
        else:
            # first free step: the currents of this step before their decay
            g_e = sum(q(x) / Q * de ** (n - k) for k, x in inputs_e.items() if k <= n)
            g_i = sum(q(x) / Q * di ** (n - k) for k, x in inputs_i.items() if k <= n)
            exp = -60.0 + a * (-49.0 + 60.0 + g_e + g_i)
            assert abs(V[0] - exp) <= 1e-5 * abs(exp)
