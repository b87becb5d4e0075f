"""bench.py -- throughput of the clock-driven SNN step (BASELINE.json metric:
wall-s per bio-second & synaptic events/s; % HBM roofline) on synthetic
Brunel+ / Brunel / Vogels-Abbott networks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--settle S] [--config 3] [--impl ours|reference]

A "step" is one simulation step (dt = 0.1 ms) of the whole hot path: neuron
update, lazy+event-driven STDP, sliced shared-atomic delivery.
Default workload: BASELINE config 3 (Brunel+, 316,228 neurons, ~1e9 synapses,
40 % plastic) -- the only single-GPU config that exercises every 8(a) row.

The timed window is the network's steady state: every run first simulates S
"settle" steps (default 3,000 = 0.3 s of biological time: past the
synchronous first forced flush at t = 63 and the rate transient), then W
warm-up steps, then times exactly K steps (the paper's measure is wall time
over long biological time).  `value` = wall-seconds per biological
second over the K steps (lower is better); synaptic events/s is reported
beside it.  Three handles of the same seed simulate the identical trajectory
(the simulation is deterministic) over the same window:
  A  the device-timed K steps (CUDA events on the simulation stream),
  B  the same K steps with in-graph kernel spans (SNN_FLAG_KTIME): per-kernel
     durations for the roofline, measured inside the graph-replayed step,
  C  the same K steps through the public API with host buffers (e2e).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import glob
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "wall-s per bio-second & synaptic events/s at 1/2/4/8 B200; % HBM roofline"
KERNEL_OF = {"front": "k_front", "stdp": "k_stdp_ev", "flush": "k_flush", "deliver": "k_deliver"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=1000)
    ap.add_argument("--settle", type=int, default=3000,
                    help="steps simulated before the warm-up (steady state; not timed)")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--slice-width", type=int, default=0)
    ap.add_argument("--plasticity", default="event", choices=["event", "lazy", "naive"],
                    help="STDP schedule: Fig. 2c (default) / 2b / 2a (ablation, SURVEY 8(f2))")
    ap.add_argument("--delivery", default="sliced", choices=["sliced", "rowwise"],
                    help="delivery: Fig. 3b (default) / 3a (ablation)")
    ap.add_argument("--flush-period", type=int, default=0,
                    help="forced flushes batched every K steps at ages >= H - K (DESIGN.md R33); 0 = at age H")
    ap.add_argument("--idx16", action="store_true",
                    help="delivery reads 16-bit slice-local target offsets (SURVEY 8(f1), P:405)")
    ap.add_argument("--history-bits", type=int, default=64, choices=[64, 128],
                    help="H: 64 (the paper's default, P:192) or 128 (SURVEY 8(f3), P:399)")
    ap.add_argument("--exchange-window", type=int, default=0, help="world > 1: steps per spike exchange (0 = auto)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ktime", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0, help="oracle threads (0 = all host cores)")
    ap.add_argument("--cpu-budget", type=float, default=30.0, help="seconds of timed oracle steps (cpu_baseline)")
    return ap.parse_args(argv)


def source_sha() -> str:
    """Hash of the CUDA sources: an ncu capture counts for this run only if it
    was taken on the same kernels."""
    h = hashlib.sha256()
    for f in sorted(glob.glob(os.path.join(ROOT, "paper_2107_04092_b200", "csrc", "*.cu*"))):
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel: str, cfg: int, flags: str):
    """DRAM bytes per launch of `kernel` from a committed `ncu --set full`
    summary (profiles/<round>/ncu_<tag>.json, scripts/summarize_ncu.py) taken
    on the same source revision, config and flags -- else None."""
    sha = source_sha()
    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_*.json")), reverse=True):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        meta = d.get("_meta", {})
        if meta.get("source_sha") != sha or meta.get("config") != cfg or meta.get("flags", "") != flags:
            continue
        for name, v in d.items():              # template instances: "void k_stdp<0, 0, 0>"
            if name != "_meta" and name.split("<")[0].split()[-1] == kernel and "dram_bytes" in v:
                return v["dram_bytes"], os.path.relpath(p, ROOT)
    return None, None


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)                    # first sample before the timed region
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ oracle
def run_oracle(cfg: int, seed: int, steps: int, warmup: int, budget_s: float, threads: int = 0,
               budget_1thread: float = 0.0):
    """Time the oracle as it stands (test infrastructure; only this leg of
    bench.py runs it) on the FULL network of the BASELINE config: build the
    graph (untimed), `warmup` untimed steps, then up to `steps` timed steps or
    until `budget_s` seconds -- a bounded sample of the workload.  Per-step
    time x 10,000 = wall-s per bio-second, extrapolated."""
    from oracle.oracle import Oracle
    rc = W.config(cfg, seed=seed)
    cores = threads or os.cpu_count() or 1
    o = Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, threads=cores)
    rc.apply(o)
    t0 = time.perf_counter()
    o.finalize()
    build_s = time.perf_counter() - t0
    o.step(warmup)

    def timed(budget):
        e0 = o.events
        t0 = time.perf_counter()
        done = 0
        while done < steps:
            o.step(1)
            done += 1
            if time.perf_counter() - t0 > budget:
                break
        return done, time.perf_counter() - t0, o.events - e0

    done, dt, ev = timed(budget_s)
    per_step = dt / done
    one = None
    if cores > 1 and budget_1thread > 0:          # the same oracle on one host thread (a shorter sample)
        o.set_threads(1)
        d1, t1, _ = timed(budget_1thread)
        one = dict(value=t1 / d1 / (rc.dt_ms * 1e-3), steps=d1, ms_per_step=1e3 * t1 / d1)
    return dict(value=per_step / (rc.dt_ms * 1e-3), unit="wall-s per bio-second (extrapolated)", cores=cores,
                kind="oracle",
                sample=(f"BASELINE config {cfg} at full size ({rc.name}, {o.nsyn:,} synapses; graph build "
                        f"{build_s:.1f} s untimed): {done} timed steps after {warmup} untimed steps from t = 0 "
                        f"on {cores} host threads, per-step time x 10,000 = 1 bio-second (extrapolated).  The "
                        f"naive STDP sweep (Fig. 2a, every plastic synapse every step) dominates the oracle's "
                        f"step and does not depend on activity; delivery runs at the cold network's rates"),
                events_per_s=ev / dt, steps=done, seconds=dt, synapses=int(o.nsyn), ms_per_step=1e3 * per_step,
                one_thread=one)


# ------------------------------------------------------------------ GPU arm
def main(argv=None):
    a = parse(argv)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    scaling = "strong" if a.config in (2, 3, 4) else "weak"
    if a.impl == "reference":
        if rank != 0:
            return
        r = run_oracle(a.config, a.seed, a.steps, max(a.warmup, 0), budget_s=60.0, threads=a.cpu_threads)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "wall-s per bio-second",
            "n_gpus": a.gpus, "steps": r["steps"], "warmup": a.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": False, "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"BASELINE config {a.config}: {W.config(a.config).name} (oracle, full size)",
                       "settle_steps": 0},
            "events_per_s": r["events_per_s"],
            "cpu_baseline": {"value": r["value"], "unit": r["unit"], "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "wall-s per bio-second", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }))
        return

    import torch
    import torch.distributed as dist
    from paper_2107_04092_b200 import Snn, FLAG_IDX16, FLAG_KTIME
    from paper_2107_04092_b200 import dist as pdist

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    if world > 1:
        # one process per GPU; torch.distributed bootstraps the library's NCCL
        # communicator (the spike exchange runs inside libsnn.so), times reduce
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    rc = W.config(a.config, seed=a.seed, gpus=world)
    stream = torch.cuda.Stream(dev)
    pre_steps = a.settle + a.warmup

    def prepare(s, chunks):
        """The untimed settle + warm-up steps, issued so that the step graphs the
        timed region replays (one per distinct call size in `chunks`, captured
        and instantiated by the library on first use) already exist."""
        sizes = sorted({min(c, 64) for c in chunks if c > 0})
        head = pre_steps - a.warmup - sum(sizes)
        if head > 0:
            s.step(head)
            for c in sizes:
                s.step(c)
        else:
            s.step(pre_steps - a.warmup)
        s.step(a.warmup)

    def make(flags=0):
        if a.idx16:
            flags |= FLAG_IDX16
        uid = pdist.nccl_unique_id() if world > 1 else None
        s = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=a.slice_width, device=dev, stream=stream,
                flags=flags, rank=rank, world=world, nccl_unique_id=uid, history_bits=a.history_bits,
                plasticity=["event", "lazy", "naive"].index(a.plasticity),
                delivery=["sliced", "rowwise"].index(a.delivery), flush_period=a.flush_period,
                exchange_window=a.exchange_window)
        rc.apply(s)
        return s

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def reduce(x, op):
        if world == 1:
            return x
        v = torch.tensor([float(x)], dtype=torch.float64, device=f"cuda:{dev}")
        dist.all_reduce(v, op=op)
        return float(v.item())

    MAX = dist.ReduceOp.MAX if world > 1 else None
    SUM = dist.ReduceOp.SUM if world > 1 else None

    # ------------------------------------------- A: device-timed K steps
    sim = make()
    t0 = time.perf_counter()
    sim.finalize()
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    info = sim.info()
    build_ms = sim.phase_times()["BUILD"]      # device time of count + scan + fill + segments (f4)
    prepare(sim, [a.steps])                    # settle + warm-up (untimed)
    barrier()
    m0 = sim.metrics()
    spk0 = sim.read_state("SPIKE_COUNT").astype(np.int64)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev) as clk:
        barrier()
        ev0.record(stream)
        sim.step(a.steps)
        ev1.record(stream)
        barrier()
    ms = reduce(ev0.elapsed_time(ev1), MAX)                   # max over ranks
    m1 = sim.metrics()
    spk = sim.read_state("SPIKE_COUNT").astype(np.int64) - spk0
    dm = {k: int(reduce(m1[k] - m0[k], SUM)) for k in m1}     # work of all ranks in the window
    dm_local = {k: m1[k] - m0[k] for k in m1}
    sim.close()
    del sim
    t_win = a.steps * rc.dt_ms * 1e-3
    rates = {p.name: float(spk[b:b + p.n].sum()) / p.n / t_win
             for p, b in zip(rc.pops, np.cumsum([0] + [p.n for p in rc.pops])[:-1])}
    sec = ms * 1e-3
    events_per_s = dm["EVENTS"] / sec
    ms_per_step = ms / a.steps
    wall_per_bio = (ms_per_step * 1e-3) / (rc.dt_ms * 1e-3)

    # ------------------------------ B: kernel spans inside the replayed graph
    spans = None
    if not a.no_ktime:
        sk = make(FLAG_KTIME)
        prepare(sk, [a.steps])
        k0 = sk.ktime()                         # folds (and discards) the settle / warm-up steps
        mk0 = sk.metrics()
        barrier()
        ek0, ek1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ek0.record(stream)
        sk.step(a.steps)
        ek1.record(stream)
        barrier()
        k1 = sk.ktime()
        mk1 = sk.metrics()
        ms_k = reduce(ek0.elapsed_time(ek1), MAX)
        same = all(mk1[k] - mk0[k] == dm_local[k] for k in dm_local)
        sk.close()
        del sk
        spans = {"same_window": bool(reduce(0.0 if same else 1.0, MAX) == 0.0),
                 "ms_per_step_instrumented": ms_k / a.steps}
        for k in ("front", "front2", "stdp", "flush", "deliver"):
            st = k1[k]["steps"] - k0[k]["steps"]
            if st <= 0:
                continue
            spans[k] = {"us_from_entry": reduce((k1[k]["entry_ns"] - k0[k]["entry_ns"]) / st * 1e-3, MAX),
                        "us_from_wait": reduce((k1[k]["wait_ns"] - k0[k]["wait_ns"]) / st * 1e-3, MAX),
                        "steps": st, "ctas_per_launch": (k1[k]["ctas"] - k0[k]["ctas"]) / st}

    # --------------------------------- C: end to end through the public API
    e2e = None
    if not a.no_e2e:
        se = make()
        prepare(se, [64, a.steps % 64])
        nw = (info["N"] + 31) // 32
        chunk = 64
        # the steps' rasters land in a pinned host buffer the caller owns
        host = torch.empty(chunk * nw, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        me0 = se.metrics()
        barrier()
        t0 = time.perf_counter()
        done = 0
        d2h = 0
        while done < a.steps:
            n = min(chunk, a.steps - done)
            t_first = pre_steps + done
            se.step(n)
            s0 = t_first % 64                       # ring slots of the chunk's steps (slot t % 64)
            k1n = min(n, 64 - s0)
            se.read_range("SPIKE_RING", s0 * nw, k1n * nw, out=host[:k1n * nw])
            if k1n < n:                              # the chunk wraps around the ring
                se.read_range("SPIKE_RING", 0, (n - k1n) * nw, out=host[k1n * nw:n * nw])
            d2h += 4 * n * nw
            done += n
        t1 = time.perf_counter()
        me1 = se.metrics()
        wall = reduce(t1 - t0, MAX)
        same_e = all(me1[k] - me0[k] == dm_local[k] for k in dm_local)
        se.close()
        del se
        e2e = {"value": wall / (a.steps * rc.dt_ms * 1e-3), "unit": "wall-s per bio-second",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(d2h / a.steps),
               "events_per_s": dm["EVENTS"] / wall, "same_window": bool(reduce(0.0 if same_e else 1.0, MAX) == 0.0),
               "note": "snn_step(n) + snn_read_state_range(SPIKE_RING) of the n steps' rasters into a pinned host "
                       "buffer, n = 64 (host wall clock, max over ranks); an SNN step has no host input (the "
                       "Poisson drive is counter-based on the device), so h2d = 0"}

    # ------------------------------------------------------------ roofline
    nrcpt = 2 if any(pr.receptor == W.INH for pr in rc.projs) else 1
    K = a.steps
    # algorithmic HBM bytes per launch:
    #   k_stdp_ev (k_stdp for the ablation schedules): 4 B target id per
    #              visited plastic synapse + 8 B (weight read and written) per
    #              synapse of an arriving row or whose target fired in the
    #              window + 16 B per visited row; split into the arrivals
    #              ("stdp", critical path) and the forced flushes ("flush",
    #              side branch) when the step graph runs them apart
    #   k_deliver: 8 B per delivered event (id + weight; 6 B with --idx16) +
    #              8 B per (arriving row, slice) pivot pair + 4 B per slice
    #              neuron and receptor written back
    #   k_front:   32 B per LIF neuron, 16 B per Poisson neuron (8(a1))
    n_pois = sum(p.n for p in rc.pops if p.kind == W.POISSON)
    stdp_b = (4 * dm_local["STDP_SYN"] + 8 * dm_local["STDP_WRW"] + 16 * dm_local["STDP_ROWS"]) / K
    flush_b = (4 * dm_local["FLUSH_SYN"] + 8 * dm_local["FLUSH_WRW"] + 16 * dm_local["FLUSH_ROWS"]) / K
    split = bool(spans and "flush" in spans)
    # the ahead step runs the plastic arrivals' STDP inside k_deliver: their
    # weights are read as delivered events and written back where they change
    fused_arr = split and not (spans and "stdp" in spans)
    arr_stores = dm_local["STDP_WSTORE"] - dm_local["FLUSH_WSTORE"]
    kb = {
        "stdp": 0.0 if fused_arr else (stdp_b - flush_b if split else stdp_b),
        "flush": flush_b if split else 0.0,
        "deliver": ((6 if a.idx16 else 8) * dm_local["EVENTS"] + 8 * dm_local["SPIKES"] * info["nslices"]
                    + ((4 * arr_stores + 16 * (dm_local["STDP_ROWS"] - dm_local["FLUSH_ROWS"])) if fused_arr else 0)) / K
                   + 4 * nrcpt * (info["tgt_hi"] - info["tgt_lo"]),
        "front": 32.0 * (info["N"] - n_pois) + 16.0 * n_pois,
    }
    hbm, peak_src = peaks()
    kern = {}
    for k, by in kb.items():
        if by <= 0 or not spans or k not in spans:
            continue
        us = spans[k]["us_from_wait"]
        kern[k] = {"bytes_per_launch": by, "us_per_launch": us, "us_per_launch_from_entry": spans[k]["us_from_entry"],
                   "achieved_gbs": by / (us * 1e-6) / 1e9 if us > 0 else 0.0}
        kern[k]["frac"] = kern[k]["achieved_gbs"] / hbm
        kern[k]["share_of_step"] = us * 1e-3 / ms_per_step
    dom = max(kern, key=lambda k: kern[k]["us_per_launch"]) if kern else None
    flags_s = ",".join(x for x, on in [("idx16", a.idx16), (f"H{a.history_bits}", a.history_bits != 64),
                                       (a.plasticity, a.plasticity != "event"), (a.delivery, a.delivery != "sliced")]
                       if on)
    roof = None
    if dom:
        dk = KERNEL_OF[dom]
        if dom == "deliver" and a.delivery == "rowwise":
            dk = "k_deliver_rowwise"
        if dom == "stdp" and (a.plasticity != "event" or a.flush_period):
            dk = "k_stdp"
        traffic, traffic_src = ncu_traffic(dk, a.config, flags_s)
        sd = [k for k in ("stdp", "flush", "deliver") if k in kern]
        sd_b = sum(kern[k]["bytes_per_launch"] for k in sd)
        sd_us = sum(kern[k]["us_per_launch"] for k in sd)
        step_b = sum(kb.values())
        roof = {"bound": "hbm", "kernel": dk, "achieved": kern[dom]["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                "frac": kern[dom]["achieved_gbs"] / hbm, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram__bytes_read.sum + dram__bytes_write.sum)",
                "traffic_source": traffic_src or "no ncu --set full capture of this source revision / config",
                "algorithmic_bytes_per_launch": kern[dom]["bytes_per_launch"], "peak_source": peak_src,
                "duration": "per launch, from the kernel's first return from its dependency wait (PDL) to its "
                            "last CTA's end, %globaltimer marks inside the graph-replayed timed steps "
                            "(SNN_FLAG_KTIME, run B on the identical window); CUDA events bracket the window",
                "kernels": kern,
                "stdp_plus_delivery": {"bytes_per_step": sd_b, "us_per_step": sd_us,
                                       "achieved_gbs": sd_b / (sd_us * 1e-6) / 1e9 if sd_us else 0.0,
                                       "frac": sd_b / (sd_us * 1e-6) / 1e9 / hbm if sd_us else 0.0},
                "step": {"bytes": step_b, "achieved_gbs": step_b / (ms_per_step * 1e-3) / 1e9,
                         "frac": step_b / (ms_per_step * 1e-3) / 1e9 / hbm}}

    out = {
        "metric": METRIC, "value": wall_per_bio, "unit": "wall-s per bio-second", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32 (int32 fixed-point accumulators)",
        "data": "synthetic",
        "config": {"workload": f"BASELINE config {a.config}: {rc.name}", "neurons": info["N"],
                   "synapses": int(reduce(info["S"], SUM)), "plastic": rc.plastic, "dt_ms": rc.dt_ms,
                   "delay_steps": rc.delay, "settle_steps": a.settle, "timed_steps_from": pre_steps,
                   "history_bits": a.history_bits, "flush_period": a.flush_period, "plasticity": a.plasticity,
                   "delivery": a.delivery, "index_bits": 16 if a.idx16 else 32, "slice_width": info["C"],
                   "slices": info["nslices"], "seed": a.seed,
                   "parallelism": f"target-range partition x{world}, NCCL spike-word all-gather" if world > 1
                   else "1 GPU",
                   "l2": "inputs larger than L2: %.1f GB of graph, each step touches the rows of that step's spikes"
                         % (info["S"] * 8 / 1e9)},
        "events_per_s": events_per_s,
        "setup": {"wall_s": setup_s, "build_ms": build_ms,
                  "synapses_per_ms": info["S"] / build_ms if build_ms > 0 else None,
                  "note": "GPU construction (geometric-skip count, scan, fill, plastic spans), device-timed, "
                          "allocation excluded; the paper quotes ~200M synapses/ms on its GPU (P:391, context)"},
        "rates_hz": rates,
        "per_step": {k.lower(): v / a.steps for k, v in dm.items()},
        # launches of the library's kernels per step: one per kernel with an in-graph span
        # (k_front, its second part, k_stdp_ev / k_stdp, k_flush, k_deliver), + k_unpack per exchange
        "gpu_launches": a.steps * (len([k for k in ("front", "front2", "stdp", "flush", "deliver")
                                        if spans and k in spans]) or (3 if rc.plastic else 2))
                        + (a.steps if world > 1 else 0),
        "roofline": roof,
        "kernel_spans": spans,
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    if not a.no_cpu_baseline and rank == 0 and world == 1:
        r = run_oracle(a.config, a.seed, 1000, 1, budget_s=a.cpu_budget, threads=a.cpu_threads,
                       budget_1thread=a.cpu_budget / 2)
        out["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        out["cpu_baseline"]["ms_per_step"] = r["ms_per_step"]
        if r.get("one_thread"):
            out["cpu_baseline"]["one_thread"] = dict(r["one_thread"], unit=r["unit"], cores=1)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
