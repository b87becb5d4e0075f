"""Tiny pure-Python replays of Fig. 2 (a), (b), (c) -- naive, lazy and
event-driven plasticity -- over an arbitrary per-synapse ``update`` callback.

TEST INFRASTRUCTURE ONLY (see oracle/snn_oracle.c header).  Used on tiny
hand-built spike trains to pin the readings of PAPER.md that the CUDA STDP
kernel relies on (R1-R4, R11):

* Fig. 2a: every step, every synapse: update(syn, pre=n.hist[delay],
  post=syn.dst.hist[0]).
* Fig. 2b: only rows whose spike arrives now; ``age = now -
  timeOfLastUpdate``; replay exactly ``age`` steps, chronologically, steps
  (tlu, now] (R1), pre only on the last one.
* Fig. 2c: iterate only the set bits of the destination history
  window (bits [0, age-1], bit s <=> step now-s), oldest first (``__clz``,
  P:284); each call covers (prev, s] and skips ahead n = prev - s steps; a tail
  call covers what is left (R2).
* Forced flush (R3): a row whose age reaches H (=64) is replayed at that step
  without a pre spike, so no post spike leaves the 64-bit window ("(up to)
  64 update steps", "both algorithms perform the exact same number of
  computations").
* Read-out flush (R11): before state is observed, every stale row is brought
  up to ``now`` without a pre spike (P:267 keeps synapses "in a stale state").

The update callback contract ("numSteps"): update(s, pre, post, n)
advances n-1 silent steps then one step with the given flags.
"""
from __future__ import annotations

MASK64 = (1 << 64) - 1


def exact_model_update(s: int, pre: bool, post: bool, n: int) -> int:
    """Order-sensitive exact integer model s <- s*3^n + pre + 2*post (mod 2^64).
    Unlike a commutative counter it detects any misordered or mis-split call."""
    return (s * pow(3, n, 1 << 64) + int(pre) + 2 * int(post)) & MASK64


def histories(spikes, T):
    """hist[t][i]: 64-bit history of neuron i after the neuron phase of step t
    (LSB = most recent)."""
    n = len(spikes[0]) if spikes else 0
    h = [0] * n
    out = []
    for t in range(T):
        h = [((h[i] << 1) | int(spikes[t][i])) & MASK64 for i in range(n)]
        out.append(list(h))
    return out


def naive(rows, spikes, T, D, update, s0=0):
    """Fig. 2a.  rows: list of target lists per source neuron."""
    H = histories(spikes, T)
    S = {(i, c): s0 for i, r in enumerate(rows) for c in range(len(r))}
    calls = 0
    for t in range(T):
        for i, r in enumerate(rows):
            pre = bool((H[t][i] >> D) & 1)
            for c, j in enumerate(r):
                S[(i, c)] = update(S[(i, c)], pre, bool(H[t][j] & 1), 1)
                calls += 1
    return S, calls


def _lazy_replay(S, i, r, hist_now, age, arr, update):
    calls = 0
    for c, j in enumerate(r):
        s = S[(i, c)]
        for k in range(age - 1, -1, -1):       # chronological: step now-k
            s = update(s, arr and k == 0, bool((hist_now[j] >> k) & 1), 1)
            calls += 1
        S[(i, c)] = s
    return calls


def _event_replay(S, i, r, hist_now, age, arr, update):
    calls = 0
    m_all = MASK64 if age >= 64 else (1 << age) - 1
    for c, j in enumerate(r):
        s = S[(i, c)]
        m = hist_now[j] & m_all
        prev = age                               # steps-ago position before the window
        while m:
            p = m.bit_length() - 1               # oldest set bit (63 - clz)
            s = update(s, arr and p == 0, True, prev - p)
            calls += 1
            prev = p
            m &= ~(1 << p)
        if prev > 0:                             # tail: (prev, 0], pre on the last step
            s = update(s, arr, False, prev)
            calls += 1
        S[(i, c)] = s
    return calls


def lazy_or_event(rows, spikes, T, D, update, event: bool, Hbits: int = 64, s0=0,
                  forced_flush: bool = True, readout_flush: bool = True):
    """Fig. 2b (event=False) / Fig. 2c (event=True) with forced flush at age H."""
    Hh = histories(spikes, T)
    S = {(i, c): s0 for i, r in enumerate(rows) for c in range(len(r))}
    tlu = [-1] * len(rows)
    calls = 0
    visits = 0
    fn = _event_replay if event else _lazy_replay
    for t in range(T):
        for i, r in enumerate(rows):
            arr = bool((Hh[t][i] >> D) & 1)
            age = t - tlu[i]
            if arr or (forced_flush and age == Hbits):
                calls += fn(S, i, r, Hh[t], min(age, Hbits), arr, update)
                visits += 1
                tlu[i] = t
    if readout_flush and T > 0:
        for i, r in enumerate(rows):
            age = (T - 1) - tlu[i]
            if age > 0:
                calls += fn(S, i, r, Hh[T - 1], age, False, update)
                tlu[i] = T - 1
    return S, calls, visits
