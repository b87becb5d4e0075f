"""Pins of the readings of Fig. 2 (R1-R4, R11-R13) with an exact,
order-sensitive integer model on tiny hand-built spike trains (brute force)."""
import random

import pytest

from oracle import replay as R


def _random_net(n, deg, T, p_fire, seed):
    rnd = random.Random(seed)
    rows = [sorted(rnd.sample([j for j in range(n) if j != i], deg)) for i in range(n)]
    spikes = [[rnd.random() < p_fire for _ in range(n)] for _ in range(T)]
    return rows, spikes


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("D", [0, 3, 15])
@pytest.mark.parametrize("p_fire", [0.001, 0.02, 0.3])
def test_naive_equals_lazy_equals_event_with_forced_flush(seed, D, p_fire):
    rows, spikes = _random_net(24, 5, 400, p_fire, seed)
    S_n, calls_n = R.naive(rows, spikes, 400, D, R.exact_model_update)
    S_l, calls_l, _ = R.lazy_or_event(rows, spikes, 400, D, R.exact_model_update, event=False)
    S_e, calls_e, _ = R.lazy_or_event(rows, spikes, 400, D, R.exact_model_update, event=True)
    assert S_l == S_n
    assert S_e == S_n
    # P:399 "both algorithms perform the exact same number of computations"
    assert calls_l == calls_n
    assert calls_e <= calls_n


def test_event_call_partition_spec_example():
    """age = 5, post bits {4, 1}, arrival: calls (pre,post,n) = (F,T,1),(F,T,3),
    (T,F,1) (chronological post flags T,F,F,T,F -- reading R12/R13)."""
    log = []

    def upd(s, pre, post, n):
        log.append((pre, post, n))
        return s

    S = {(0, 0): 0}
    R._event_replay(S, 0, [1], [0, 0b10010], 5, True, upd)
    assert log == [(False, True, 1), (False, True, 3), (True, False, 1)]
    log.clear()
    R._lazy_replay(S, 0, [1], [0, 0b10010], 5, True, upd)
    assert [p for (_, p, _) in log] == [True, False, False, True, False]
    assert [p for (p, _, _) in log] == [False] * 4 + [True]


def test_event_calls_bounded_by_popcount_plus_one_and_sum_age():
    rnd = random.Random(5)
    for _ in range(2000):
        age = rnd.randint(1, 64)
        h = rnd.getrandbits(64)
        log = []

        def upd(s, pre, post, n):
            log.append(n)
            return s

        R._event_replay({(0, 0): 0}, 0, [1], [0, h], age, rnd.random() < 0.5, upd)
        m = h & ((1 << age) - 1)
        assert sum(log) == age
        assert len(log) <= bin(m).count("1") + 1


def test_clamp_reading_without_forced_flush_is_not_exact():
    """SPEC's clamp reading (replay min(age, H), no forced flush) loses post
    spikes older than the window and differs from naive (R3)."""
    rows, spikes = _random_net(24, 5, 600, 0.004, 3)
    S_n, _ = R.naive(rows, spikes, 600, 2, R.exact_model_update)
    S_c, _, _ = R.lazy_or_event(rows, spikes, 600, 2, R.exact_model_update, event=True,
                                forced_flush=False)
    assert S_c != S_n


def test_readout_flush_needed():
    """Without the read-out flush the lazy state is stale (R11)."""
    rows, spikes = _random_net(24, 5, 300, 0.01, 4)
    S_n, _ = R.naive(rows, spikes, 300, 0, R.exact_model_update)
    S_s, _, _ = R.lazy_or_event(rows, spikes, 300, 0, R.exact_model_update, event=True,
                                readout_flush=False)
    assert S_s != S_n


def test_forced_flush_visit_share_low_rate():
    """At ~10 Hz (p = 0.001 per step) forced flushes dominate the row visits
    (SURVEY hard part 5; P:399 'most neurons reach their maximum age')."""
    rows, spikes = _random_net(40, 6, 3000, 0.001, 6)
    _, _, visits = R.lazy_or_event(rows, spikes, 3000, 3, lambda s, a, b, n: s, event=True,
                                   readout_flush=False)
    arrivals = sum(sum(1 for x in st if x) for st in spikes[:3000 - 3])
    assert visits > 5 * arrivals
