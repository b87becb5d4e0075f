"""Seeded synthetic workload recipes shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method: it only lists populations,
projections, model constants and seeds (the input recipe of DESIGN.md section 4),
and hands the same final values to whichever simulator object it is applied to
(the C-ABI binding ``paper_2107_04092_b200.Snn`` or the test oracle
``oracle.Oracle``; both expose ``add_population`` / ``connect``).

Model constants are the readings of DESIGN.md R7-R10, R26 (PAPER.md P:367
names Vogels-Abbott, Brunel and Brunel+ and defers their details; the values
are Vogels & Abbott 2005 / Brette et al. 2007 benchmark 2 (CUBA) and Brunel
2000 model A).  Weight scaling by network size ("We apply a scaling
factor to synaptic weights") follows reading R10: w = w_base * k_base / k with k
the expected in-degree p * |source population|.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

POISSON, LIF_DELTA, LIF_CUBA = 0, 1, 2
STATIC, STDP = 0, 1
EXC, INH = 0, 1


@dataclass
class Pop:
    name: str
    kind: int
    n: int
    params: dict


@dataclass
class Proj:
    src: int
    dst: int
    kind: int
    receptor: int
    p: float
    weight: float
    stdp: dict = field(default_factory=dict)


@dataclass
class Recipe:
    name: str
    seed: int
    dt_ms: float
    delay: int
    frac_bits: int
    pops: List[Pop]
    projs: List[Proj]
    plastic: bool = False

    @property
    def n(self) -> int:
        return sum(p.n for p in self.pops)

    @property
    def expected_synapses(self) -> float:
        return sum(pr.p * self.pops[pr.src].n * self.pops[pr.dst].n for pr in self.projs)

    def apply(self, sim):
        """Issue the recipe's add_population / connect calls on ``sim``."""
        ids = []
        for p in self.pops:
            ids.append(sim.add_population(p.kind, p.n, **p.params))
        for pr in self.projs:
            sim.connect(ids[pr.src], ids[pr.dst], pr.kind, pr.receptor, pr.p, pr.weight, **pr.stdp)
        return ids


# --------------------------------------------------------------- Vogels (CUBA)
VOGELS_LIF = dict(tau_m=20.0, v_rest=-49.0, v_reset=-60.0, v_th=-50.0, tau_ref=5.0,
                  tau_e=5.0, tau_i=10.0)
VOGELS_WE, VOGELS_WI = 1.62, -9.0          # mV at the base in-degrees below
VOGELS_KE, VOGELS_KI = 64.0, 16.0          # N=4000, p=0.02 (Brette 2007)


def vogels(n_total: int = 4000, p: float = 0.02, seed: int = 1, delay: int = 0,
           frac_bits: int = 20) -> Recipe:
    """Vogels-Abbott CUBA network: 80 % E / 20 % I, Erdos-Renyi p (BASELINE.json configs 1, 5)."""
    ne = int(round(0.8 * n_total))
    ni = n_total - ne
    we = VOGELS_WE * VOGELS_KE / (p * ne) if p > 0 else VOGELS_WE
    wi = VOGELS_WI * VOGELS_KI / (p * ni) if p > 0 else VOGELS_WI
    pops = [Pop("E", LIF_CUBA, ne, dict(VOGELS_LIF)), Pop("I", LIF_CUBA, ni, dict(VOGELS_LIF))]
    projs = [Proj(0, 0, STATIC, EXC, p, we), Proj(0, 1, STATIC, EXC, p, we),
             Proj(1, 0, STATIC, INH, p, wi), Proj(1, 1, STATIC, INH, p, wi)]
    return Recipe(f"vogels{n_total}", seed, 0.1, delay, frac_bits, pops, projs)


# ------------------------------------------------------------ Brunel / Brunel+
BRUNEL_LIF = dict(tau_m=20.0, v_rest=0.0, v_reset=10.0, v_th=20.0, tau_ref=2.0)
BRUNEL_J, BRUNEL_KBASE, BRUNEL_G, BRUNEL_NU_P = 0.1, 1000.0, 5.0, 16.0


def brunel(n_total: int = 100_000, p: float = 0.02, plastic: bool = False, seed: int = 1,
           delay: int = 15, frac_bits: int = 20, g: float = BRUNEL_G,
           nu_p: float = BRUNEL_NU_P) -> Recipe:
    """Brunel (2000, model A) E/I delta-LIF network with an explicit Poisson
    population P (|P| = |E| + |I|, reading R26).  With ``plastic`` the P->E
    synapses carry additive STDP (Brunel+, exactly 40 % of all synapses, R8)."""
    ne = int(round(0.4 * n_total))
    ni = int(round(0.1 * n_total))
    npp = n_total - ne - ni
    J = BRUNEL_J * BRUNEL_KBASE / (p * ne) if p > 0 else BRUNEL_J
    w_max = 2.0 * J
    a_plus = 0.01 * w_max
    stdp = dict(tau_plus=20.0, tau_minus=20.0, a_plus=a_plus, a_minus=1.05 * a_plus, w_max=w_max)
    pops = [Pop("E", LIF_DELTA, ne, dict(BRUNEL_LIF)), Pop("I", LIF_DELTA, ni, dict(BRUNEL_LIF)),
            Pop("P", POISSON, npp, dict(rate_hz=nu_p))]
    projs = [Proj(0, 0, STATIC, EXC, p, J), Proj(0, 1, STATIC, EXC, p, J),
             Proj(1, 0, STATIC, EXC, p, -g * J), Proj(1, 1, STATIC, EXC, p, -g * J),
             Proj(2, 0, STDP if plastic else STATIC, EXC, p, J, stdp if plastic else {}),
             Proj(2, 1, STATIC, EXC, p, J)]
    name = ("brunel+" if plastic else "brunel") + str(n_total)
    return Recipe(name, seed, 0.1, delay, frac_bits, pops, projs, plastic=plastic)


# BASELINE.json configs
def config(k: int, seed: int = 1, gpus: int = 1) -> Recipe:
    if k == 1:
        return vogels(4000, seed=seed)
    if k == 2:
        return brunel(100_000, seed=seed)
    if k == 3:
        return brunel(316_228, plastic=True, seed=seed)
    if k == 4:
        return brunel(632_456, plastic=True, seed=seed)
    if k == 5:
        n = {1: 316_228, 2: 447_214, 4: 632_456, 8: 894_427}[gpus]
        return vogels(n, seed=seed)
    raise ValueError(k)
