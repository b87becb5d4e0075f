"""ctypes wrapper around the plain C oracle (oracle/snn_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.  It shares no
code with the CUDA path and never imports paper_2107_04092_b200.

The oracle is the plain definition of what the method computes (PAPER.md
P:34-42 three-phase step; Fig. 2a naive plasticity P:197-210; Fig. 3a row-wise
delivery P:305-310; Fig. 1 binary-search pivots P:180).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "snn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

POISSON, LIF_DELTA, LIF_CUBA = 0, 1, 2
STATIC, STDP = 0, 1

FIELDS = {  # name -> (id, dtype, length kind)
    "V": (0, np.float32, "n"), "ge": (1, np.float32, "n"), "gi": (2, np.float32, "n"),
    "ref": (3, np.int32, "n"), "in_e": (4, np.int32, "n"), "in_i": (5, np.int32, "n"),
    "hist": (6, np.uint64, "n"), "nspk": (7, np.uint32, "n"),
    "row_ptr": (8, np.int64, "n+1"), "idx": (9, np.uint32, "s"), "w": (10, np.float32, "s"),
    "xpre": (11, np.float32, "s"), "xpost": (12, np.float32, "s"),
}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FMA contraction (R19)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-shared", "-fPIC", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        vp, u32, i32, i64, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        P = ctypes.POINTER
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [u64, ctypes.c_float, u32, i32]
        L.oracle_set_threads.argtypes = [vp, ctypes.c_int]
        L.oracle_add_pop.restype = ctypes.c_int
        L.oracle_add_pop.argtypes = [vp, ctypes.c_int, u32, P(ctypes.c_float)]
        L.oracle_connect.restype = ctypes.c_int
        L.oracle_connect.argtypes = [vp, u32, u32, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                     P(ctypes.c_float), ctypes.c_int]
        L.oracle_build_row.restype = i64
        L.oracle_build_row.argtypes = [vp, u32, u32, u32, P(u32), i64]
        L.oracle_pivots.argtypes = [P(u32), i64, u32, u32, u32, P(i64)]
        L.oracle_finalize.restype = ctypes.c_int
        L.oracle_finalize.argtypes = [vp]
        L.oracle_step.argtypes = [vp, u32]
        L.oracle_n.restype = u32
        L.oracle_n.argtypes = [vp]
        L.oracle_nsyn.restype = i64
        L.oracle_nsyn.argtypes = [vp]
        L.oracle_t.restype = i64
        L.oracle_t.argtypes = [vp]
        L.oracle_set_t.argtypes = [vp, i64]
        L.oracle_events.restype = u64
        L.oracle_events.argtypes = [vp]
        L.oracle_pop_of.restype = ctypes.c_int
        L.oracle_pop_of.argtypes = [vp, u32]
        L.oracle_field.restype = vp
        L.oracle_field.argtypes = [vp, ctypes.c_int]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_philox.argtypes = [P(u32), P(u32), P(u32)]
        L.oracle_synapse_replay.restype = ctypes.c_float
        L.oracle_synapse_replay.argtypes = [vp, ctypes.c_int, ctypes.c_int, P(ctypes.c_uint8), P(ctypes.c_uint8), i64]
        _lib = L
    return _lib


def philox(ctr, key):
    """Philox4x32-10 of the oracle (for its own known-answer pin)."""
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox(c, k, o)
    return [int(x) for x in o]


def pivots(row, lo: int, C: int, nslices: int) -> np.ndarray:
    """Binary-search pivots of one sorted row (Fig. 1 caption)."""
    r = np.ascontiguousarray(np.asarray(row, dtype=np.uint32))
    out = np.zeros(nslices + 1, dtype=np.int64)
    lib().oracle_pivots(r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(r), lo, C, nslices,
                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
    return out


class Oracle:
    """One simulated network on the host.  Mirrors the C-ABI call sequence
    (create / add_population / connect / step / read) so tests can drive both
    sides from the same recipe."""

    def __init__(self, seed: int, dt_ms: float = 0.1, delay: int = 0, frac_bits: int = 20,
                 threads: int = 1):
        self._s = lib().oracle_create(seed, dt_ms, delay, frac_bits)
        if not self._s:
            raise ValueError("oracle_create rejected the configuration")
        lib().oracle_set_threads(self._s, threads)
        self.delay = delay
        self.frac_bits = frac_bits
        self.pops = []

    def __del__(self):
        if getattr(self, "_s", None):
            lib().oracle_destroy(self._s)
            self._s = None

    def add_population(self, kind: int, n: int, rate_hz=0.0, tau_m=20.0, v_rest=0.0, v_reset=0.0,
                       v_th=1.0, tau_ref=0.0, tau_e=5.0, tau_i=10.0) -> int:
        prm = (ctypes.c_float * 8)(rate_hz, tau_m, v_rest, v_reset, v_th, tau_ref, tau_e, tau_i)
        pid = lib().oracle_add_pop(self._s, kind, n, prm)
        if pid < 0:
            raise ValueError("oracle_add_pop rejected")
        base = sum(p[1] for p in self.pops)
        self.pops.append((base, n, kind))
        return pid

    def connect(self, src: int, dst: int, kind: int, receptor: int, p: float, weight: float,
                tau_plus=20.0, tau_minus=20.0, a_plus=0.0, a_minus=0.0, w_max=0.0,
                autapses: bool = False) -> int:
        f = (ctypes.c_float * 6)(weight, tau_plus, tau_minus, a_plus, a_minus, w_max)
        r = lib().oracle_connect(self._s, src, dst, kind, receptor, p, f, int(autapses))
        if r < 0:
            raise ValueError("oracle_connect rejected")
        return r

    def build_row(self, i: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
        """One row of the graph without building the rest (for sampled checks)."""
        hi = self.n if hi is None else hi
        L = lib()
        length = L.oracle_build_row(self._s, i, lo, hi, None, 0)
        out = np.zeros(max(length, 1), dtype=np.uint32)
        L.oracle_build_row(self._s, i, lo, hi, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), length)
        return out[:length]

    def synapse_replay(self, src_pop: int, dst_pop: int, pre, post) -> float:
        """Naive STDP (Fig. 2a, R7) of one synapse of the projection src_pop ->
        dst_pop from its initial state, given its pre events (pre[t]: the source
        fired at t - D) and post events (post[t]: the target fired at t)."""
        pre = np.ascontiguousarray(pre, dtype=np.uint8)
        post = np.ascontiguousarray(post, dtype=np.uint8)
        assert pre.shape == post.shape
        P8 = ctypes.POINTER(ctypes.c_uint8)
        return float(lib().oracle_synapse_replay(self._s, src_pop, dst_pop, pre.ctypes.data_as(P8),
                                                  post.ctypes.data_as(P8), len(pre)))

    def set_threads(self, threads: int):
        """Host threads of the following steps (OpenMP-style row / neuron loops)."""
        lib().oracle_set_threads(self._s, threads)

    def finalize(self):
        if lib().oracle_finalize(self._s) != 0:
            raise RuntimeError("oracle_finalize failed")

    def step(self, n: int = 1):
        lib().oracle_step(self._s, n)

    @property
    def n(self) -> int:
        return lib().oracle_n(self._s)

    @property
    def nsyn(self) -> int:
        return lib().oracle_nsyn(self._s)

    @property
    def t(self) -> int:
        return lib().oracle_t(self._s)

    @t.setter
    def t(self, v: int):
        lib().oracle_set_t(self._s, v)

    @property
    def events(self) -> int:
        return lib().oracle_events(self._s)

    def pop_of(self, j: int) -> int:
        return lib().oracle_pop_of(self._s, j)

    def array(self, name: str) -> np.ndarray:
        """A live numpy view on an oracle array (writable: used to load a
        snapshot for the from-shared-state parity runs)."""
        fid, dt, kind = FIELDS[name]
        length = {"n": self.n, "n+1": self.n + 1, "s": self.nsyn}[kind]
        ptr = lib().oracle_field(self._s, fid)
        if not ptr or length == 0:
            return np.zeros(0, dtype=dt)
        buf = (ctypes.c_char * (length * np.dtype(dt).itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dt, count=length)
