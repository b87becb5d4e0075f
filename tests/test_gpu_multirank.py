"""The partitioned (multi-GPU) path, run as `world` partitions of one network
on ONE GPU (local-group transport: the spike words of each step are copied
into every partition's gather buffer, exactly what ncclAllGather does across
GPUs).  The partitioned run must equal the single-partition run bit-exactly
(integer accumulation, identical per-synapse arithmetic) -- SURVEY 8(e)."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _run(rc, world, steps, C=0):
    from paper_2107_04092_b200 import Snn
    key = 0x5EED0000 + world
    sims = []
    for r in range(world):
        g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=C, rank=r, world=world,
                group_key=key if world > 1 else 0)
        rc.apply(g)
        sims.append(g)
    for g in sims:
        g.finalize()
    for t in range(steps):
        for g in sims:          # lockstep: every partition finishes step t before step t+1
            g.step(1)
    return sims


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("plastic", [False, True])
def test_partitioned_equals_single(world, plastic):
    rc = W.brunel(9000, p=0.05, plastic=plastic, delay=15, seed=21)
    ref = _run(rc, 1, 200)[0]
    parts = _run(rc, world, 200)
    h_ref = ref.read_state("HIST")
    v_ref = ref.read_state("V")
    ev = 0
    rp_ref, idx_ref = ref.read_state("ROW_PTR"), ref.read_state("IDX")
    w_ref = ref.read_state("WEIGHTS")
    for g in parts:
        info = g.info()
        lo, hi = info["tgt_lo"], info["tgt_hi"]
        assert np.array_equal(g.read_state("HIST"), h_ref)          # every neuron's spikes
        assert np.array_equal(g.read_state("V")[lo:hi], v_ref[lo:hi])  # owned neurons
        ev += g.metrics()["EVENTS"]
        # local CSR = the global rows restricted to [lo, hi); weights bit-exact
        rp, idx, w = g.read_state("ROW_PTR"), g.read_state("IDX"), g.read_state("WEIGHTS")
        for i in list(range(0, info["N"], 97)) + [info["N"] - 1]:
            full = idx_ref[rp_ref[i]:rp_ref[i + 1]]
            sel = (full >= lo) & (full < hi)
            assert np.array_equal(idx[rp[i]:rp[i + 1]], full[sel])
            assert np.array_equal(w[rp[i]:rp[i + 1]], w_ref[rp_ref[i]:rp_ref[i + 1]][sel])
    assert ev == ref.metrics()["EVENTS"]


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_d0_equals_single(world):
    """D = 0 (BASELINE config 5, Vogels-Abbott): the arrivals of step t include
    the other ranks' spikes of step t, so each step runs the neuron phase, the
    exchange of the step's words and then the lists (k_front parts 1 / 2);
    the partitioned run equals the single one bit-exactly (rasters, V, CUBA
    currents, pending inputs of both receptors)."""
    rc = W.vogels(6000, seed=22)
    assert rc.delay == 0
    ref = _run(rc, 1, 300)[0]
    parts = _run(rc, world, 300)
    h_ref, v_ref = ref.read_state("HIST"), ref.read_state("V")
    ge_ref, gi_ref = ref.read_state("G_EXC"), ref.read_state("G_INH")
    ie_ref, ii_ref = ref.read_state("INPUT_EXC"), ref.read_state("INPUT_INH")
    assert int(ref.read_state("SPIKE_COUNT").sum()) > 1000
    ev = 0
    for g in parts:
        info = g.info()
        lo, hi = info["tgt_lo"], info["tgt_hi"]
        assert np.array_equal(g.read_state("HIST"), h_ref)
        for f, r in (("V", v_ref), ("G_EXC", ge_ref), ("G_INH", gi_ref), ("INPUT_EXC", ie_ref),
                     ("INPUT_INH", ii_ref)):
            assert np.array_equal(g.read_state(f)[lo:hi], r[lo:hi]), f
        ev += g.metrics()["EVENTS"]
    assert ev == ref.metrics()["EVENTS"]


@pytest.mark.parametrize("cfg", ["brunel+15", "vogels0"])
def test_nccl_exchange_path_world1_equals_plain(cfg):
    """The NCCL data path on one GPU (SNN_FLAG_EXCHANGE, world 1): the
    communicator from a torch-created ncclUniqueId, ncclAllGather of the step's
    spike words + k_unpack on the exchange branch of the captured step graph
    (D >= 1) or between the two k_front parts (D = 0) -- the run equals the
    plain one bit-exactly (rasters, V, weights)."""
    import torch
    from paper_2107_04092_b200 import Snn, FLAG_EXCHANGE
    rc = W.brunel(9000, p=0.05, plastic=True, delay=15, seed=31) if cfg == "brunel+15" else W.vogels(6000, seed=32)
    uid = bytes(torch.cuda.nccl.unique_id())
    out = []
    for flags, kw in ((0, {}), (FLAG_EXCHANGE, {"nccl_unique_id": uid})):
        g = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, flags=flags, **kw)
        rc.apply(g)
        for _ in range(4):
            g.step(50)
        out.append((g.read_state("HIST"), g.read_state("V"), g.read_state("WEIGHTS"), g.metrics()["EVENTS"]))
        g.close()
    (h0, v0, w0, e0), (h1, v1, w1, e1) = out
    assert np.array_equal(h0, h1) and np.array_equal(v0, v1) and np.array_equal(w0, w1) and e0 == e1
    assert int(h0.astype(bool).sum()) > 100
