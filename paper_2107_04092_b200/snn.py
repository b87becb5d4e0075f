"""Thin ctypes binding of libsnn.so (include/snn.h): argument marshalling only.

Every step of the simulation runs in the CUDA kernels of libsnn.so; there is no
CPU fallback.  If the library is missing this module raises at import time.
PyTorch is used only for device memory (its caching allocator, through the
dev_alloc / dev_free hooks of snn_config) and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsnn.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(nvcc, sm_100a).  There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- constants
SNN_ABI_VERSION = 4
SNN_OK, SNN_E_INVALID, SNN_E_STATE, SNN_E_OOM, SNN_E_CUDA, SNN_E_NCCL, SNN_E_UNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
POISSON, LIF_DELTA, LIF_CUBA = 0, 1, 2
STATIC, STDP = 0, 1
EXC, INH = 0, 1
FLAG_NO_GRAPH, FLAG_PHASE_TIMING, FLAG_TRACE, FLAG_NO_PDL, FLAG_IDX16, FLAG_KTIME = 1, 2, 4, 8, 16, 32
FLAG_EXCHANGE = 64      # the NCCL spike-word exchange even at world == 1 (needs nccl_unique_id)
PLAST_EVENT, PLAST_LAZY, PLAST_NAIVE = 0, 1, 2        # Fig. 2c / 2b / 2a schedules
DELIV_SLICED, DELIV_ROWWISE = 0, 1                    # Fig. 3b / 3a delivery
ALL = 0xFFFFFFFF

FIELD = dict(V=0, REFRACTORY=1, G_EXC=2, G_INH=3, INPUT_EXC=4, INPUT_INH=5, HIST=6, SPIKE_COUNT=7,
             XPOST=8, XPRE_ROW=9, TLU=10, ROW_PTR=11, IDX=12, WEIGHTS=13, PIVOTS=14, STEP=15,
             METRICS=16, SPIKE_RING=17, PHASE_TIMES=18, INFO=19, TRACE=20, IDX16=21, HIST_DEV=22,
             HIST_DEV_HI=23, FPOT=24, RECENT=25, KTIME=26, FPOS=27)
FIELD_DTYPE = dict(V=np.float32, REFRACTORY=np.int32, G_EXC=np.float32, G_INH=np.float32,
                   INPUT_EXC=np.int32, INPUT_INH=np.int32, HIST=np.uint64, SPIKE_COUNT=np.uint32,
                   XPOST=np.float32, XPRE_ROW=np.float32, TLU=np.int32, ROW_PTR=np.int64,
                   IDX=np.uint32, WEIGHTS=np.float32, PIVOTS=np.uint32, STEP=np.int64,
                   METRICS=np.uint64, SPIKE_RING=np.uint32, PHASE_TIMES=np.float64, INFO=np.int64,
                   TRACE=np.uint64, IDX16=np.uint16, HIST_DEV=np.uint64, HIST_DEV_HI=np.uint64,
                   FPOT=np.float32, RECENT=np.uint32, KTIME=np.uint64, FPOS=np.uint8)
METRIC = dict(EVENTS=0, SPIKES=1, STDP_ROWS=2, STDP_SYN=3, STDP_WSTORE=4, FLUSH_ROWS=5, SEGMENTS=6, ELEMS=7,
              STDP_WRW=8, FLUSH_SYN=9, FLUSH_WRW=10, FLUSH_WSTORE=11)
KTIME_KERNELS = ("front", "stdp", "deliver", "flush", "front2")
PHASE = dict(FRONT=0, STDP=1, DELIVERY=2, EXCHANGE=3, TOTAL=4, BUILD=5)

ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class snn_config(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("struct_size", ctypes.c_uint32),
                ("dt_ms", ctypes.c_float), ("delay_steps", ctypes.c_uint32),
                ("history_bits", ctypes.c_uint32), ("slice_width", ctypes.c_uint32),
                ("accum_frac_bits", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("device", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("dev_alloc", ALLOC_FN), ("dev_free", FREE_FN), ("alloc_ctx", ctypes.c_void_p),
                ("nccl_unique_id", ctypes.c_void_p), ("group_key", ctypes.c_uint64),
                ("plasticity", ctypes.c_uint32), ("delivery", ctypes.c_uint32), ("flush_period", ctypes.c_uint32),
                ("exchange_window", ctypes.c_uint32)]


class snn_pop_params(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("kind", ctypes.c_uint32), ("rate_hz", ctypes.c_float),
                ("tau_m_ms", ctypes.c_float), ("v_rest_mv", ctypes.c_float), ("v_reset_mv", ctypes.c_float),
                ("v_th_mv", ctypes.c_float), ("tau_ref_ms", ctypes.c_float), ("tau_e_ms", ctypes.c_float),
                ("tau_i_ms", ctypes.c_float)]


class snn_syn_params(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("kind", ctypes.c_uint32), ("receptor", ctypes.c_uint32),
                ("allow_autapses", ctypes.c_uint32), ("p", ctypes.c_double), ("weight", ctypes.c_float),
                ("tau_plus_ms", ctypes.c_float), ("tau_minus_ms", ctypes.c_float), ("a_plus", ctypes.c_float),
                ("a_minus", ctypes.c_float), ("w_max", ctypes.c_float)]


_P = ctypes.POINTER
_lib.snn_create.restype = ctypes.c_int32
_lib.snn_create.argtypes = [_P(snn_config), _P(ctypes.c_void_p)]
_lib.snn_add_population.restype = ctypes.c_int32
_lib.snn_add_population.argtypes = [ctypes.c_void_p, ctypes.c_uint32, _P(snn_pop_params), _P(ctypes.c_uint32)]
_lib.snn_connect.restype = ctypes.c_int32
_lib.snn_connect.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, _P(snn_syn_params)]
_lib.snn_step.restype = ctypes.c_int32
_lib.snn_step.argtypes = [ctypes.c_void_p, ctypes.c_uint32]
_lib.snn_read_state.restype = ctypes.c_int32
_lib.snn_read_state.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                ctypes.c_size_t, _P(ctypes.c_size_t)]
_lib.snn_read_state_range.restype = ctypes.c_int32
_lib.snn_read_state_range.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_size_t]
_lib.snn_destroy.restype = None
_lib.snn_destroy.argtypes = [ctypes.c_void_p]
_lib.snn_last_error.restype = ctypes.c_char_p
_lib.snn_last_error.argtypes = [ctypes.c_void_p]
_lib.snn_abi_version.restype = ctypes.c_uint32
_lib.snn_abi_version.argtypes = []
_lib.snn_partition.restype = ctypes.c_int32
_lib.snn_partition.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                               _P(ctypes.c_uint32), _P(ctypes.c_uint32)]

_lib.snn_partition_weighted.restype = ctypes.c_int32
_lib.snn_partition_weighted.argtypes = [_P(ctypes.c_double), ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_uint32, _P(ctypes.c_uint32), _P(ctypes.c_uint32)]

EXPORTS = ["snn_create", "snn_add_population", "snn_connect", "snn_step", "snn_read_state",
           "snn_read_state_range", "snn_destroy", "snn_last_error", "snn_abi_version", "snn_partition",
           "snn_partition_weighted"]


class SnnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"snn status {code}: {msg}")
        self.code = code


# ------------------------------------------------- same-named thin functions
def snn_last_error(sim) -> str:
    return (_lib.snn_last_error(sim) or b"").decode()


def _check(code, sim):
    if code != SNN_OK:
        raise SnnError(code, snn_last_error(sim))


def snn_abi_version() -> int:
    return _lib.snn_abi_version()


def snn_partition(n_targets: int, slice_width: int, world: int, rank: int):
    """Target range [lo, hi) of `rank` (host only, no device work)."""
    lo, hi = ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.snn_partition(n_targets, slice_width, world, rank, ctypes.byref(lo), ctypes.byref(hi)), None)
    return lo.value, hi.value


def snn_partition_weighted(slice_cost, n_targets: int, slice_width: int, world: int, rank: int):
    """Target range [lo, hi) of `rank` balancing the per-slice costs (host only)."""
    c = (ctypes.c_double * len(slice_cost))(*[float(x) for x in slice_cost])
    lo, hi = ctypes.c_uint32(), ctypes.c_uint32()
    _check(_lib.snn_partition_weighted(c, len(slice_cost), n_targets, slice_width, world, rank, ctypes.byref(lo),
                                       ctypes.byref(hi)), None)
    return lo.value, hi.value


def snn_create(cfg: snn_config):
    h = ctypes.c_void_p()
    _check(_lib.snn_create(ctypes.byref(cfg), ctypes.byref(h)), None)
    return h


def snn_add_population(sim, n: int, prm: snn_pop_params) -> int:
    pid = ctypes.c_uint32()
    _check(_lib.snn_add_population(sim, n, ctypes.byref(prm), ctypes.byref(pid)), sim)
    return pid.value


def snn_connect(sim, src: int, dst: int, prm: snn_syn_params):
    _check(_lib.snn_connect(sim, src, dst, ctypes.byref(prm)), sim)


def snn_step(sim, n_steps: int):
    _check(_lib.snn_step(sim, n_steps), sim)


def snn_read_state(sim, field: int, pop_id: int, host_dst, dst_bytes: int) -> int:
    need = ctypes.c_size_t()
    _check(_lib.snn_read_state(sim, field, pop_id, host_dst, dst_bytes, ctypes.byref(need)), sim)
    return need.value


def snn_read_state_range(sim, field: int, pop_id: int, first: int, count: int, host_dst, dst_bytes: int):
    _check(_lib.snn_read_state_range(sim, field, pop_id, first, count, host_dst, dst_bytes), sim)


def snn_destroy(sim):
    _lib.snn_destroy(sim)


# ------------------------------------------------------------ convenience
class Snn:
    """One simulation handle.  Method names mirror the C ABI; the population /
    projection keyword arguments match oracle.Oracle so a workloads.Recipe can
    be applied to either."""

    def __init__(self, seed: int, dt_ms: float = 0.1, delay: int = 0, frac_bits: int = 20,
                 slice_width: int = 0, device: int = 0, stream=None, flags: int = 0, rank: int = 0,
                 world: int = 1, nccl_unique_id: bytes | None = None, group_key: int = 0,
                 torch_allocator: bool = True, history_bits: int = 64, plasticity: int = 0, delivery: int = 0,
                 flush_period: int = 0, exchange_window: int = 0):
        import torch  # plumbing: device memory and streams
        self._torch = torch
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        cfg = snn_config()
        cfg.abi_version = SNN_ABI_VERSION
        cfg.struct_size = ctypes.sizeof(snn_config)
        cfg.dt_ms = dt_ms
        cfg.delay_steps = delay
        cfg.history_bits = history_bits   # H: 64 or 128
        cfg.plasticity = plasticity       # PLAST_EVENT / PLAST_LAZY / PLAST_NAIVE (ablation, f2)
        cfg.delivery = delivery           # DELIV_SLICED / DELIV_ROWWISE (ablation, f2)
        cfg.flush_period = flush_period   # 0: flush at age H; K: batched every K steps (R33)
        cfg.exchange_window = exchange_window   # world > 1: steps per spike-word exchange (0 = auto)
        cfg.slice_width = slice_width
        cfg.accum_frac_bits = frac_bits
        cfg.flags = flags
        cfg.seed = seed
        cfg.device = device
        cfg.rank = rank
        cfg.world = world
        cfg.group_key = group_key
        cfg.stream = ctypes.c_void_p(stream.cuda_stream)
        self._keep = []
        if torch_allocator:
            dev = device

            def _alloc(nbytes, strm, ctx):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), dev, int(strm or 0))
                except Exception:
                    return None

            def _free(ptr, strm, ctx):
                if torch is not None and torch.cuda is not None:   # not at interpreter teardown
                    torch.cuda.caching_allocator_delete(ptr)

            self._keep += [ALLOC_FN(_alloc), FREE_FN(_free)]
            cfg.dev_alloc, cfg.dev_free = self._keep
        if nccl_unique_id is not None:
            buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
            self._keep.append(buf)
            cfg.nccl_unique_id = ctypes.cast(buf, ctypes.c_void_p)
        self._cfg = cfg
        self.h = snn_create(cfg)
        self.pops = []

    def close(self):
        if getattr(self, "h", None):
            snn_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add_population(self, kind: int, n: int, rate_hz=0.0, tau_m=20.0, v_rest=0.0, v_reset=0.0,
                       v_th=1.0, tau_ref=0.0, tau_e=5.0, tau_i=10.0) -> int:
        p = snn_pop_params(ctypes.sizeof(snn_pop_params), kind, rate_hz, tau_m, v_rest, v_reset, v_th,
                           tau_ref, tau_e, tau_i)
        pid = snn_add_population(self.h, n, p)
        base = sum(x[1] for x in self.pops)
        self.pops.append((base, n, kind))
        return pid

    def connect(self, src: int, dst: int, kind: int, receptor: int, p: float, weight: float,
                tau_plus=20.0, tau_minus=20.0, a_plus=0.0, a_minus=0.0, w_max=0.0, autapses=False):
        q = snn_syn_params(ctypes.sizeof(snn_syn_params), kind, receptor, int(autapses), p, weight,
                           tau_plus, tau_minus, a_plus, a_minus, w_max)
        snn_connect(self.h, src, dst, q)

    def step(self, n: int = 1):
        snn_step(self.h, n)

    def finalize(self):
        snn_step(self.h, 0)

    def read_state(self, field: str, pop: int = ALL, out: np.ndarray | None = None) -> np.ndarray:
        fid = FIELD[field]
        need = snn_read_state(self.h, fid, pop, None, 0)
        dt = np.dtype(FIELD_DTYPE[field])
        if out is None:
            out = np.empty(need // dt.itemsize, dtype=dt)
        snn_read_state(self.h, fid, pop, out.ctypes.data_as(ctypes.c_void_p), out.nbytes)
        return out

    def read_range(self, field: str, first: int, count: int, pop: int = ALL,
                   out: np.ndarray | None = None) -> np.ndarray:
        """Elements [first, first + count) of a field (snn_read_state_range)
        into `out` (a caller-owned host buffer, e.g. pinned) or a new array."""
        if out is None:
            out = np.empty(count, dtype=np.dtype(FIELD_DTYPE[field]))
        assert out.dtype == np.dtype(FIELD_DTYPE[field]) and out.size == count and out.flags.c_contiguous
        snn_read_state_range(self.h, FIELD[field], pop, first, count, out.ctypes.data_as(ctypes.c_void_p),
                             out.nbytes)
        return out

    def metrics(self) -> dict:
        m = self.read_state("METRICS")
        return {k: int(m[v]) for k, v in METRIC.items()}

    def ktime(self) -> dict:
        """Cumulative kernel spans of the graph-replayed steps (SNN_FLAG_KTIME):
        per kernel, ns summed over steps from the first CTA entry / the first
        return from the dependency wait to the last CTA end, steps, CTAs."""
        v = self.read_state("KTIME")
        return {k: dict(entry_ns=int(v[4 * i]), wait_ns=int(v[4 * i + 1]), steps=int(v[4 * i + 2]),
                        ctas=int(v[4 * i + 3])) for i, k in enumerate(KTIME_KERNELS)}

    def info(self) -> dict:
        v = self.read_state("INFO")
        return dict(N=int(v[0]), S=int(v[1]), nslices=int(v[2]), C=int(v[3]), R=int(v[4]),
                    tgt_lo=int(v[5]), tgt_hi=int(v[6]), pivot_bytes=int(v[7]))

    def phase_times(self) -> dict:
        v = self.read_state("PHASE_TIMES")
        return {k: float(v[i]) for k, i in PHASE.items()}

    @property
    def t(self) -> int:
        return int(self.read_state("STEP")[0])
