"""Pins of the oracle's Philox, connectivity and pivots against things the
paper / mathematics fix (not against the oracle itself)."""
import math
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(fname):
    out = []
    for line in open(os.path.join(GOLD, fname)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line)
    return out


def test_philox_known_answers():
    """Random123 KAT vectors (tests/golden/philox_kat.txt)."""
    for line in _rows("philox_kat.txt"):
        v = [int(x, 16) for x in line.split()]
        assert O.philox(v[0:4], v[4:6]) == v[6:10]


def test_fig1_pivots_worked_example():
    """PAPER.md Fig. 1: the printed pivots for N=9, chunk 3."""
    for line in _rows("fig1_pivots.txt"):
        head, row, piv = [s.split() for s in line.split("|")]
        N, C = int(head[0]), int(head[1])
        ids = [0x7FFFFFFF if x == "inf" else int(x) for x in row]
        nslices = -(-N // C)
        got = O.pivots(ids, 0, C, nslices)
        assert got.tolist() == [int(x) for x in piv]


@settings(max_examples=60, deadline=None)
@given(st.integers(1, 300), st.sampled_from([1, 3, 32, 100, 1024]), st.integers(0, 2**31))
def test_pivots_equal_bruteforce_chunk_counts(n, C, seed):
    """Brute force: pivots[k+1]-pivots[k] = number of entries in chunk k, every
    entry of segment k lies in [kC, (k+1)C) (partition completeness)."""
    rng = np.random.default_rng(seed)
    row = np.sort(rng.choice(n, size=rng.integers(0, n + 1), replace=False)).astype(np.uint32)
    ns = -(-n // C)
    piv = O.pivots(row, 0, C, ns)
    assert piv[0] == 0 and piv[-1] == len(row)
    for k in range(ns):
        seg = row[piv[k]:piv[k + 1]]
        assert np.all((seg >= k * C) & (seg < (k + 1) * C))
        assert len(seg) == sum(1 for x in row if k * C <= x < (k + 1) * C)


def _net(N, p, autapses=False, seed=7):
    o = O.Oracle(seed, 0.1, 0, 20)
    a = o.add_population(O.LIF_DELTA, N, v_reset=10.0, v_th=20.0)
    o.connect(a, a, O.STATIC, 0, p, 0.1, autapses=autapses)
    o.finalize()
    return o


def test_complete_digraph_p1():
    """p = 1, no autapses -> complete digraph (S:61 example: rows [1,2],[0,2],[0,1])."""
    o = _net(3, 1.0)
    rp, idx = o.array("row_ptr"), o.array("idx")
    assert [idx[rp[i]:rp[i + 1]].tolist() for i in range(3)] == [[1, 2], [0, 2], [0, 1]]
    o2 = _net(5, 1.0, autapses=True)
    assert o2.nsyn == 25


def test_empty_graph_p0():
    o = _net(50, 0.0)
    assert o.nsyn == 0


def test_connectivity_statistics_and_invariants():
    """Rows sorted, unique, no autapses (R21); realised synapse count
    within 5 sigma of the binomial mean."""
    N, p = 1500, 0.1
    o = _net(N, p, seed=42)
    rp, idx = o.array("row_ptr"), o.array("idx")
    for i in range(N):
        r = idx[rp[i]:rp[i + 1]]
        assert np.all(np.diff(r.astype(np.int64)) > 0)
        assert i not in r
        assert np.all(r < N)
    mean = p * N * (N - 1)
    sd = np.sqrt(N * (N - 1) * p * (1 - p))
    assert abs(o.nsyn - mean) < 5 * sd
    # in-degree and out-degree both binomial(N-1, p): spread within 5 sigma
    outdeg = np.diff(rp)
    indeg = np.bincount(idx, minlength=N)
    s1 = np.sqrt((N - 1) * p * (1 - p))
    assert abs(outdeg.mean() - (N - 1) * p) < 5 * s1 / np.sqrt(N) + 1e-9
    assert abs(outdeg.std() - s1) < 0.2 * s1
    assert abs(indeg.std() - s1) < 0.2 * s1


def test_build_row_matches_finalized_rows_and_ranges():
    """A single row built on demand (sampled full-size checks) equals the
    finalized row, and a column range [lo,hi) is the row's restriction to it
    (the rank partition of DESIGN.md section 7)."""
    o = _net(700, 0.05, seed=3)
    rp, idx = o.array("row_ptr"), o.array("idx")
    for i in [0, 1, 350, 699]:
        full = idx[rp[i]:rp[i + 1]]
        assert np.array_equal(o.build_row(i), full)
        part = o.build_row(i, 128, 512)
        assert np.array_equal(part, full[(full >= 128) & (full < 512)])


def test_pair_acceptance_frequency_is_p():
    """Independent Bernoulli(p) per (source, target): acceptance frequency
    over 1e6 pairs within 5 sigma of p."""
    o = _net(1000, 0.02, autapses=True, seed=11)
    n = 1000 * 1000
    assert abs(o.nsyn / n - 0.02) < 5 * np.sqrt(0.02 * 0.98 / n)


@pytest.mark.parametrize("N,p,rows,ks", [(40_000, 0.02, 50, (1, 5, 20, 50, 100, 200)),
                                        (4_000_000, 0.0002, 50, (100, 2000, 4096, 5000, 9000))])
def test_geometric_gaps_follow_the_bernoulli_law(N, p, rows, ks):
    """R32: the gaps between kept candidates of a row are geometric -- the law
    of independent Bernoulli(p) trials (P(gap > k) = (1-p)^k) -- checked at
    several k within 5 sigma, including gaps beyond the 4096-entry table (the
    memoryless continuation), and each target position is kept with frequency
    p across rows (no positional bias).  Rows are long against the mean gap
    (the gap cut by a row's end is not observed)."""
    o = O.Oracle(7, 0.1, 0, 20)
    a = o.add_population(O.LIF_DELTA, N, tau_m=20.0, v_reset=10.0, v_th=20.0)
    o.connect(a, a, O.STATIC, 0, p, 0.1, autapses=True)
    gaps = []
    hits = np.zeros(N, dtype=np.int64)
    for i in range(rows):
        r = o.build_row(i).astype(np.int64)
        hits[r] += 1
        gaps.append(np.diff(np.concatenate([[-1], r])))
    g = np.concatenate(gaps)
    n = len(g)
    assert n > 20_000
    for k in ks:
        q = (1 - p) ** k
        assert abs((g > k).mean() - q) < 5 * np.sqrt(q * (1 - q) / n), k
    B = N // 40                                                  # 40 blocks of positions
    f = hits.reshape(40, B).sum(axis=1) / (rows * B)
    assert np.all(np.abs(f - p) < 5 * np.sqrt(p * (1 - p) / (rows * B)))


def test_pair_inclusion_independent_at_every_lag():
    """Independent Bernoulli(p) per pair (R23, realised by R32): for two
    candidates k apart in one row, P(both kept) = p^2 at every lag k -- in
    particular at k = 1, which a gap law off by one (gaps >= 2, or g = 0
    allowed) would empty or double."""
    import workloads as W
    from oracle.oracle import Oracle
    p, n = 0.05, 4000
    rc = W.Recipe("lag", 3, 0.1, 0, 20,
                  [W.Pop("A", W.LIF_DELTA, n, dict(W.BRUNEL_LIF)), W.Pop("B", W.LIF_DELTA, 600, dict(W.BRUNEL_LIF))],
                  [W.Proj(1, 0, W.STATIC, W.EXC, p, 0.1)])
    o = Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits)
    rc.apply(o)
    X = np.zeros((600, n), dtype=bool)
    for r in range(600):
        X[r, o.build_row(n + r)] = True
    for k in (1, 2, 3, 7, 50, 333):
        both = (X[:, :-k] & X[:, k:]).mean()
        m = X[:, :-k].size
        assert abs(both - p * p) < 5 * math.sqrt(p * p * (1 - p * p) / m), (k, both)
    assert abs(X.mean() - p) < 5 * math.sqrt(p * (1 - p) / X.size)
