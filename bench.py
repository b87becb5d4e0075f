"""bench.py -- throughput of the clock-driven SNN step (BASELINE.json metric:
wall-s per bio-second & synaptic events/s; % HBM roofline) on synthetic
Brunel+ / Brunel / Vogels-Abbott networks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one simulation step (dt = 0.1 ms) of the whole hot path: neuron
update, lazy+event-driven STDP, sliced shared-atomic delivery.
Default workload: BASELINE config 3 (Brunel+, 316,228 neurons, ~1e9 synapses,
40 % plastic) -- the only single-GPU config that exercises every 8(a) row.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--warmup", type=int, default=1000)
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
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--phase-steps", type=int, default=0, help="steps of the per-phase timing pass (0 = --steps)")
    return ap.parse_args()


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the newest committed ncu --set full
    summary (profiles/<round>/ncu_<tag>.json, written by scripts/summarize_ncu.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_v*.json")),
                   key=lambda p: (os.path.basename(os.path.dirname(p)), int(os.path.basename(p)[5:-5])))
    for p in reversed(files):
        try:
            d = json.load(open(p))
        except Exception:
            continue
        for name, v in d.items():              # template instances: "k_stdp<false, ...>"
            if name.split("<")[0].split()[-1] == kernel and "dram_bytes" in v:
                return v["dram_bytes"], os.path.relpath(p, ROOT)
    return None, None


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
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


def cpu_sample_recipe(cfg: int, seed: int):
    """Bounded oracle sample of the same workload family."""
    if cfg in (3, 4):
        return W.brunel(31_623, plastic=True, seed=seed), "Brunel+ scaled to N=31,623 (same composition, p=0.02, ~1e7 synapses, 40% plastic)"
    if cfg == 2:
        return W.brunel(31_623, plastic=False, seed=seed), "Brunel scaled to N=31,623 (same composition, p=0.02, ~1e7 synapses)"
    if cfg == 5:
        return W.vogels(31_623, seed=seed), "Vogels CUBA scaled to N=31,623 (p=0.02, ~2e7 synapses)"
    return W.config(1, seed=seed), "Vogels CUBA 4,000 (the full config 1)"


def run_oracle(cfg: int, seed: int, steps: int, warmup: int, budget_s: float = 20.0):
    """Time the oracle as it stands (test infrastructure; only this leg of bench.py runs it)."""
    from oracle.oracle import Oracle
    rc, sample = cpu_sample_recipe(cfg, seed)
    cores = os.cpu_count() or 1
    o = Oracle(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, threads=cores)
    rc.apply(o)
    o.finalize()
    o.step(warmup)
    e0 = o.events
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        o.step(1)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    ev = o.events - e0
    return dict(value=ev / dt, unit="events/s", cores=cores, kind="oracle",
                sample=f"{sample}; {done} timed steps after {warmup} warm-up steps",
                wall_s_per_bio_s=(dt / done) / (rc.dt_ms * 1e-3), steps=done, seconds=dt,
                synapses=int(o.nsyn))


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    if a.impl == "reference":
        if rank != 0:
            return
        r = run_oracle(a.config, a.seed, a.steps, max(a.warmup, 0), budget_s=60.0)
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "events/s",
            "n_gpus": a.gpus, "steps": r["steps"], "warmup": a.warmup,
            "ms_per_step": 1e3 * r["seconds"] / r["steps"], "higher_is_better": True,
            "scaling": "strong" if a.config in (2, 3, 4) else "weak",      # (as the GPU arm's line)
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"BASELINE config {a.config} (oracle sample: {r['sample']})"},
            "wall_s_per_bio_s": r["wall_s_per_bio_s"],
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch
    import torch.distributed as dist
    from paper_2107_04092_b200 import Snn, FLAG_PHASE_TIMING, FLAG_IDX16
    from paper_2107_04092_b200 import dist as pdist

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    if world > 1:
        # one process per GPU; torch.distributed bootstraps the library's NCCL
        # communicator (the spike exchange runs inside libsnn.so), times reduce
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    rc = W.config(a.config, seed=a.seed, gpus=world)
    stream = torch.cuda.Stream(dev)

    def make(flags=0):
        if a.idx16:
            flags |= FLAG_IDX16
        uid = pdist.nccl_unique_id() if world > 1 else None
        s = Snn(rc.seed, rc.dt_ms, rc.delay, rc.frac_bits, slice_width=a.slice_width, device=dev, stream=stream,
                flags=flags, rank=rank, world=world, nccl_unique_id=uid, history_bits=a.history_bits,
                plasticity=["event", "lazy", "naive"].index(a.plasticity),
                delivery=["sliced", "rowwise"].index(a.delivery), flush_period=a.flush_period)
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

    # ---------------------------------------------------------- device-timed
    sim = make()
    t0 = time.perf_counter()
    sim.finalize()
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    info = sim.info()
    build_ms = sim.phase_times()["BUILD"]      # device time of count + scan + fill + segments (f4)
    with ClockSampler(dev) as clk:
        sim.step(a.warmup)
        barrier()
        m0 = sim.metrics()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        sim.step(a.steps)
        ev1.record(stream)
        barrier()
    ms = reduce(ev0.elapsed_time(ev1), MAX)                   # max over ranks
    m1 = sim.metrics()
    dm = {k: int(reduce(m1[k] - m0[k], SUM)) for k in m1}     # work of all ranks
    spikes = sim.read_state("SPIKE_COUNT")
    t_total = (a.warmup + a.steps) * rc.dt_ms * 1e-3
    rates = {p.name: float(spikes[b:b + p.n].sum()) / p.n / t_total
             for p, b in zip(rc.pops, np.cumsum([0] + [p.n for p in rc.pops])[:-1])}
    sec = ms * 1e-3
    events_per_s = dm["EVENTS"] / sec
    ms_per_step = ms / a.steps
    wall_per_bio = (ms_per_step * 1e-3) / (rc.dt_ms * 1e-3)

    # --------------------------------------------------- e2e through the C ABI
    e2e = None
    if not a.no_e2e:
        chunk = 64
        # the step rasters land in a pinned host buffer (the caller owns host_dst)
        ring = torch.empty(64 * ((info["N"] + 31) // 32), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        m0e = sim.metrics()
        barrier()
        t0 = time.perf_counter()
        done = 0
        while done < a.steps:
            n = min(chunk, a.steps - done)
            sim.step(n)
            sim.read_state("SPIKE_RING", out=ring)     # D2H of the step rasters into a host buffer
            done += n
        t1 = time.perf_counter()
        m1e = sim.metrics()
        wall = reduce(t1 - t0, MAX)
        evs = reduce(m1e["EVENTS"] - m0e["EVENTS"], SUM)
        e2e = {"value": evs / wall, "unit": "events/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(ring.nbytes / chunk),
               "wall_s_per_bio_s": wall / (a.steps * rc.dt_ms * 1e-3),
               "note": "snn_step(64) + snn_read_state(SPIKE_RING) into a pinned host buffer per 64 steps; an SNN "
                       "step has no host input (Poisson drive is counter-based on device), so h2d = 0"}
    sim.close()
    del sim
    torch.cuda.synchronize()

    # ------------------------------------------- per-phase timing (roofline)
    psteps = a.phase_steps or a.steps
    sp = make(FLAG_PHASE_TIMING)
    sp.step(a.warmup)
    sp.phase_times()   # drain warm-up events
    base = sp.phase_times()
    mp0 = sp.metrics()
    sp.step(psteps)
    ph = sp.phase_times()
    mp1 = sp.metrics()
    ph = {k: reduce(ph[k] - base[k], MAX) for k in ph}
    d = {k: int(reduce(mp1[k] - mp0[k], SUM)) for k in mp1}
    sp.close()
    nrcpt = 2 if any(pr.receptor == W.INH for pr in rc.projs) else 1
    # algorithmic HBM bytes per kernel:
    #   k_stdp:    4 B target id per visited plastic synapse, 8 B where the weight
    #              is read and written, 16 B per visited row (x_pre, tlu, row_ptr, seg)
    #   k_deliver: 8 B per delivered event (id + weight; 6 B with --idx16), 8 B per (arriving row,
    #              slice) pivot pair, 4 B per slice neuron and receptor written back
    kb = {
        "STDP": 4 * d["STDP_SYN"] + 8 * d["STDP_WTOUCH"] + 16 * d["STDP_ROWS"],
        "DELIVERY": (6 if a.idx16 else 8) * d["EVENTS"] + 8 * d["SPIKES"] * info["nslices"]
                    + 4 * nrcpt * info["R"] * psteps,
    }
    hbm, peak_src = peaks()
    kern = {}
    for k2, by in kb.items():
        ms_k = ph[k2]
        kern[k2] = {"bytes_per_step": by / psteps, "ms_per_step": ms_k / psteps,
                    "achieved_gbs": by / (ms_k * 1e-3) / 1e9 if ms_k > 0 else 0.0}
    dom = max(kern, key=lambda k2: kern[k2]["ms_per_step"])
    achieved = kern[dom]["achieved_gbs"]
    dom_kernel = {"STDP": "k_stdp", "DELIVERY": "k_deliver_rowwise" if a.delivery == "rowwise" else "k_deliver"}[dom]
    traffic, traffic_src = ncu_traffic(dom_kernel)
    shares = {k: ph[k] / ph["TOTAL"] for k in ("FRONT", "STDP", "DELIVERY")} if ph["TOTAL"] else {}
    sd_bytes, sd_ms = kb["STDP"] + kb["DELIVERY"], ph["STDP"] + ph["DELIVERY"]
    # level (i) of SURVEY 8(d): the whole step -- STDP + delivery bytes plus the
    # neuron update (~32 B per LIF neuron, 16 B per Poisson neuron, 8(a1)) over
    # the graph-replayed step time
    n_pois = sum(p.n for p in rc.pops if p.kind == W.POISSON)
    front_bytes_step = 32.0 * (info["N"] - n_pois) + 16.0 * n_pois
    step_bytes = sd_bytes / psteps + front_bytes_step
    split_group = info["pivot_bytes"]

    out = {
        "metric": METRIC, "value": events_per_s, "unit": "events/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if a.config in (2, 3, 4) else "weak",
        "vs_baseline": None, "dtype": "f32 (int32 fixed-point accumulators)", "data": "synthetic",
        "config": {"workload": f"BASELINE config {a.config}: {rc.name}", "neurons": info["N"],
                   "synapses": info["S"], "plastic": rc.plastic, "dt_ms": rc.dt_ms, "delay_steps": rc.delay,
                   "history_bits": a.history_bits, "flush_period": a.flush_period, "plasticity": a.plasticity,
                   "delivery": a.delivery, "index_bits": 16 if a.idx16 else 32, "slice_width": info["C"], "slices": info["nslices"], "seed": a.seed,
                   "parallelism": f"target-range partition x{world}, NCCL spike-word all-gather" if world > 1 else "1 GPU",
                   "l2": "inputs larger than L2: %.1f GB of graph, each step touches the rows of that step's spikes"
                         % (info["S"] * 8 / 1e9)},
        "wall_s_per_bio_s": wall_per_bio,
        "setup_s": setup_s,
        "setup": {"wall_s": setup_s, "build_ms": build_ms,
                  "synapses_per_ms": info["S"] / build_ms if build_ms > 0 else None,
                  "note": "GPU construction (Philox-Bernoulli count, scan, fill, plastic spans), device-timed, "
                          "allocation excluded; the paper quotes ~200M synapses/ms on its GPU (P:391, context)"},
        "rates_hz": rates,
        "per_step": {k.lower(): v / a.steps for k, v in dm.items()},
        "gpu_launches": a.steps * (3 if rc.plastic else 2),
        "roofline": {"bound": "hbm", "kernel": dom_kernel,
                     "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read + write)",
                     "traffic_source": traffic_src, "algorithmic_bytes_per_launch": kern[dom]["bytes_per_step"],
                     "peak_source": peak_src, "kernels": kern,
                     "stdp_plus_delivery": {"achieved_gbs": sd_bytes / (sd_ms * 1e-3) / 1e9 if sd_ms else 0.0,
                                            "frac": sd_bytes / (sd_ms * 1e-3) / 1e9 / hbm if sd_ms else 0.0},
                     "step": {"bytes": step_bytes, "achieved_gbs": step_bytes / (ms_per_step * 1e-3) / 1e9,
                              "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / hbm},
                     "phase_ms_per_step": {k: ph[k] / psteps for k in ph}, "phase_share": shares,
                     "deliver_splits": split_group >> 32, "stdp_grid": split_group & 0xffffffff},
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    if not a.no_cpu_baseline and rank == 0 and world == 1:
        r = run_oracle(a.config, a.seed, 2000, 50, budget_s=15.0)
        out["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        out["cpu_baseline"]["wall_s_per_bio_s"] = r["wall_s_per_bio_s"]
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
