#!/usr/bin/env python
"""bench.py -- throughput of the ensemble-SSA hot path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

A step is one pass of the whole hot path over one
batch: BASELINE.json configs[2] (the paper's HIV model, Table 1 / PAPER.md:62-93,
2^18 trajectories over 100 days, grid dt = 1 day, seed 3) per GPU.  Multi-GPU
is weak scaling: rank r simulates the aligned id shard r of 2^18 * N
trajectories (ssa_run_shard), the per-GPU moment roots are all-gathered with
NCCL and merged in fixed rank order (ssa_merge_roots).

Metric: SSA events/s (applied events of the whole job / max-over-ranks device
time); trajectories/s alongside.  `roofline` reports the issue-slot roofline of
the dominant kernel (K1, the SSA event loop) against an algorithmic
instruction count per event.  `cpu_baseline` times the CPU
oracle (test infrastructure, rank 0 only) on a bounded sample of the same
workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic.json")
FP64_PER_SMSP_CLK = 0.497   # DADD/DMUL/DFMA issue rate per SMSP per clock, profiles/r1h_pipe_peaks.txt


def profiled_activity(workload: str, kernel: str):
    """ncu's issue-slot and FP64-pipe activity of `kernel` (smsp__issue_active,
    sm__pipe_fp64_cycles_active) from the committed capture named in profiles/traffic.json."""
    if not os.path.exists(TRAFFIC_FILE):
        return None
    e = json.load(open(TRAFFIC_FILE)).get(workload, {}).get(kernel, {})
    if "issue_active" not in e:
        return None
    return {"issue_active": e["issue_active"], "fp64_pipe_active": e.get("fp64_pipe_active"),
            "source": e.get("activity_source")}


def lsu_wavefronts_per_event(workload: str):
    """Shared-memory (LSU data pipe) wavefronts per applied event of K2 from the committed ncu
    capture named in profiles/traffic.json (None when absent)."""
    if not os.path.exists(TRAFFIC_FILE):
        return None
    return json.load(open(TRAFFIC_FILE)).get(workload, {}).get("ssa_k2", {}).get("lsu_wavefronts_per_event")


def measured_traffic(workload: str, kernel: str, default_size: bool):
    """DRAM read+write bytes per launch of `kernel` from the committed ncu pass (profiles/traffic.json),
    for the default-size workload only (other sizes: None)."""
    if not default_size or not os.path.exists(TRAFFIC_FILE):
        return None
    e = json.load(open(TRAFFIC_FILE)).get(workload, {}).get(kernel)
    return None if e is None else int(e["read"] + e["write"])


# ---------------------------------------------------------------- helpers
def alg_instr_per_event(net, path: int) -> float:
    """Algorithmic thread-instructions per applied event of the thread path
    (DESIGN.md §7): what a minimal implementation of a2-a8 must issue."""
    philox = 40          # 10 rounds x (2 wide multiplies + 2 three-input xors)
    u53 = 6              # 2 x (shift/or + 2 exact adds)
    plog = 21            # bits -> exponent, bucket index and fold (6), 2 table loads, r (1), 5-term Horner,
                         # r^2 and ln(1+r) (2), e -> double, recombination (4) (R11)
    tau = 9              # IEEE divide (~8) + add
    props = 0
    for r in net.reactions:
        fac = sum(0 if m == 1 else (3 if m == 2 else 14) for _, m in r.reactants)
        props += fac + max(len(r.reactants) - 1, 0) + (1 if r.reactants else 0)
        # a modified rate k^ = max(0, k + d x_m) is a function of x_m alone: it is
        # evaluated when x_m changes (rare; HIV: F only grows by V4 -> F + V4), not per event
    R = net.R
    prefix = max(R - 1, 0)
    select = 2 * max(R - 1, 0)   # compare + predicated add per prefix entry
    update = 4
    rest = 1 + 2 + 5 + 3          # r = u2 a0, grid check, hash, counter/loop
    return philox + u53 + plog + tau + props + prefix + select + update + rest


def alg_fp64_per_event(net) -> float:
    """Algorithmic FP64-pipe instructions per applied event of the thread path:
    u53 (1 exact add each) 2, plog (r 1, Horner 5, r^2 and ln(1+r) 2, recombination 4) 12,
    tau (divide 8 + add) 9, per reaction the factor ops (C(x,2): add + 2 multiplies; C(x,3): 7),
    the products and k*h, prefix R-1 adds, selection R-1 compares, r = u2 a0, the grid compare,
    and the update's count adds (mean |nu_j| over reactions)."""
    props = 0
    for r in net.reactions:
        props += sum(0 if m == 1 else (3 if m == 2 else 7) for _, m in r.reactants)
        props += max(len(r.reactants) - 1, 0) + (1 if r.reactants else 0)
    R = net.R
    upd = 0
    for r in net.reactions:
        nu = {}
        for sp, m in r.reactants:
            nu[sp] = nu.get(sp, 0) - m
        for sp, m in r.products:
            nu[sp] = nu.get(sp, 0) + m
        upd += sum(1 for v in nu.values() if v != 0)
    upd /= max(R, 1)
    return 2 + 12 + 9 + props + 2 * max(R - 1, 0) + 1 + 1 + upd


def alg_warp_instr_per_event(net, lanes: int = 32) -> float:
    """Algorithmic WARP-instructions per applied event of the warp paths (K2,
    DESIGN.md §7), `lanes` = 32 (one trajectory per warp, order warp32) or 16
    (two per warp, order warp16s), P = ceil(R/lanes) propensities per lane.
    Per warp iteration: lane sum (P loads + P adds), log2(lanes)-step scan (2
    shuffles + add), 3 broadcasts, tau (IEEE divide 9 + add), grid check,
    selection, update and dependency recompute (one lane-parallel pass each),
    Philox 40 + u53 6 + plog 21 (-3 shared with tau) amortised over `lanes` events, loop; divided by the
    32/lanes trajectories a warp advances per iteration.  Selection: warp32 --
    r, each lane re-sums its P propensities from v_{l-1} with a compare each
    (2P), vprev shuffle, ballot/ffs/broadcast (2P + 5); warp16s -- r, ballot +
    ffs for lane*, broadcast of v_{lane*-1}, one load, a 4-step scan of lane*'s
    propensities, add, compare, ballot + ffs (22)."""
    P = max(1, -(-net.R // lanes))
    steps = 5 if lanes == 32 else 4
    select = (2 * P + 5) if lanes == 32 else (1 + 2 + 2 + 1 + 3 * 4 + 1 + 1 + 2)
    per_iter = 2 * P + 3 * steps + 6 + 10 + 2 + select + 5 + 15 + 64 / lanes + 3
    return per_iter / (32 // lanes)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], stdout=subprocess.PIPE,
                                     stderr=subprocess.DEVNULL, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for name, v in zip(names, s[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        power = [float(s[3]) for s in self.samples if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "power_w_max": max(power) if power else None,
                "samples": len(self.samples)}


def _oracle_worker(args):
    net_cfg, ids, seed, t_end, dt = args
    import inputs
    from oracle import oracle as O
    cfg = inputs.config(net_cfg)
    r = O.run(O.OracleModel(cfg.network), ids, seed, t_end, dt, 0, keep=True)
    return int(r.summaries["events"].sum()), len(ids)


def sample_ids(cfg_index: int, n_traj: int):
    """The CPU sample: n_traj ids drawn uniformly from the config's whole id range
    (inputs.dump_ids' generator), so early die-outs appear at their ensemble rate."""
    import inputs
    cfg = inputs.config(cfg_index)
    return [int(v) for v in inputs.dump_ids(cfg.n_trajectories, n_traj, cfg.seed + 0xC0)]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg_index: int, n_traj: int, cores: int, t_end=None):
    """Time the unmodified CPU oracle on `n_traj` trajectories of the config
    (sample_ids), spread over `cores` worker processes.  Returns (events,
    trajectories, seconds)."""
    import multiprocessing as mp

    import inputs
    cfg = inputs.config(cfg_index)
    t_end = t_end or cfg.t_end
    ids = sample_ids(cfg_index, n_traj)
    parts = [ids[i::cores] for i in range(cores) if ids[i::cores]]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(parts)) as pool:
        outs = pool.map(_oracle_worker, [(cfg_index, p, cfg.seed, t_end, cfg.dt) for p in parts])
    dt = time.perf_counter() - t0
    return sum(o[0] for o in outs), sum(o[1] for o in outs), dt


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle, as it stands, on this host's cores."""
    if rank != 0:
        return 0
    import inputs
    from oracle import oracle as O
    O.build()
    cfg = inputs.config(args.config)
    cores = host_cores()
    per_step = 3 * max(cores, 8)  # three ~0.4 s HIV trajectories per core per step (~15-20 s of CPU work)
    for _ in range(args.warmup):
        oracle_sample(args.config, per_step, cores)
    ev = tr = 0
    secs = 0.0
    for _ in range(args.steps):
        e, t, s = oracle_sample(args.config, per_step, cores)
        ev += e; tr += t; secs += s
    value = ev / secs
    line = {
        "impl": "reference", "metric": "ssa_events_per_s", "value": value, "unit": "events/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{args.config}-{cfg.name}", "t_end": cfg.t_end, "sample_dt": cfg.dt,
                   "seed": cfg.seed, "trajectories_per_step": per_step, "parallelism": "cpu-processes"},
        "trajectories_per_s": tr / secs,
        "cpu_baseline": {"value": value, "unit": "events/s", "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} full {cfg.name} trajectories per step (ids drawn uniformly from "
                                   f"the {cfg.n_trajectories}-id ensemble) over {cores} processes"},
        "e2e": {"value": value, "unit": "events/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- sweep workload
def run_sweep_bench(args, rank, world):
    """The paper's delta_t sensitivity sweep (Fig. 4 panels 2-4)
    as one ssa_run_sweep: 3 points x (config-2 trajectories / 3) over config 2's
    horizon, on one GPU.  Device time by CUDA events on the run's stream."""
    if world != 1:
        print(json.dumps({"error": "the sweep workload runs on one GPU"}))
        return 1
    import torch

    import inputs
    from paper_1007_1768_b200 import build as B
    B.build()
    from paper_1007_1768_b200 import ssa as S
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    net, rates = inputs.hiv_delta_t_sweep()
    cfg = inputs.config(2)
    n_per = (args.n_per_gpu or cfg.n_trajectories) // len(rates)
    t_end = args.t_end or cfg.t_end
    m = S.Model(net)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        S.run_sweep(m, rates, n_per, t_end, cfg.dt, cfg.seed, stream=stream.cuda_stream)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    events, launches = 0, 0
    with ClockSampler(0) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            l2.zero_()
            r = S.run_sweep(m, rates, n_per, t_end, cfg.dt, cfg.seed, stream=stream.cuda_stream)
            events += r.events
            launches += r.kernel_launches
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    line = {"metric": "ssa_events_per_s", "value": events / (ms / 1e3), "unit": "events/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "fig4-delta-t-sweep", "model": net.name, "points": [float(v) for v in rates[:, 5]],
                       "swept_reaction": 6, "n_trajectories_per_point": n_per, "t_end": t_end, "sample_dt": cfg.dt,
                       "seed": cfg.seed, "path": "thread", "l2": "flushed between steps (256 MiB write)"},
            "trajectories_per_s": len(rates) * n_per * args.steps / (ms / 1e3),
            "events_per_step": events / args.steps, "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- union-time workload
def union_roofline(ms, recorded_bytes, points, S):
    """The union reduction against HBM: its algorithmic bytes are the recorded
    event rows read once (t 8 B, reaction 4 B, U pre-event counts 4 B each) plus the output
    points written once (time and count 8 B each, mean and variance 8 B per species)."""
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    peak = float(peaks.get("hbm_gbs", 7700.0))
    alg = recorded_bytes + points * (16 + 16 * S)
    gbs = alg / (ms / 1e3) / 1e9 if ms > 0 else None
    return {"ms": ms, "recorded_bytes": recorded_bytes, "output_bytes": points * (16 + 16 * S),
            "bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak if gbs else None,
            "peak_basis": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200 nominal"}


def run_union_bench(args, rank, world):
    """Selective memory at union times (NEXT 2): 16 HIV trajectories (Fig. 4,
    "multiple trajectories (16x)") over config 2's horizon,
    Avg-XY with k_x = 16 (SPEC.md's default k_x = k).  Device time of the whole
    call (CUDA events inside the library: counting run, recording run, sort,
    scans, X-groups); the reduction's own time and bytes are reported too."""
    if world != 1:
        print(json.dumps({"error": "the union workload runs on one GPU"}))
        return 1
    import torch

    import inputs
    from paper_1007_1768_b200 import build as B
    B.build()
    from paper_1007_1768_b200 import ssa as S
    torch.cuda.set_device(0)
    cfg = inputs.config(2)
    n = args.n_per_gpu or 16
    t_end = args.t_end or cfg.t_end
    m = S.Model(inputs.hiv("B") if args.variant == "B" else cfg.network)
    first = S.run_union(m, n, t_end, cfg.seed, args.kx)           # sizes the output (untimed)
    cap = len(first.times)
    for _ in range(max(args.warmup - 1, 0)):
        S.run_union(m, n, t_end, cfg.seed, args.kx, capacity=cap)
    dev_ms, red_ms, red_b, events, launches = [], [], 0, 0, 0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            u = S.run_union(m, n, t_end, cfg.seed, args.kx, capacity=cap)
            dev_ms.append(u.result.device_ms)
            red_ms.append(u.result.reduce_ms)
            red_b = u.result.reduce_bytes
            events += u.result.events
            launches += u.result.kernel_launches
    ms = sum(dev_ms)
    line = {"metric": "ssa_events_per_s", "value": events / (ms / 1e3), "unit": "events/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+i64", "data": "synthetic",
            "config": {"workload": "union-time-selective-memory", "model": m.network.name, "n_trajectories": n,
                       "t_end": t_end, "thin_kx": args.kx, "seed": cfg.seed, "output_points": cap,
                       "timing": "device time of each call (CUDA events in the library)"},
            "events_per_step": events / args.steps, "gpu_launches": launches,
            "union_reduction": union_roofline(statistics.mean(red_ms), red_b, cap, m.network.S),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- full-trajectory output workload
def run_traj_bench(args, rank, world):
    """Stride-sampled full trajectories (NEXT 4): the paper's output
    experiment, "a 1:10 sampling (outputting 1 simulation point every 10)"
    (PAPER.md:175), for 16 HIV trajectories over config 2's horizon.  Device
    time of each call (simulation + sort/gather + the device-to-host copy of
    the points, CUDA events in the library)."""
    if world != 1:
        print(json.dumps({"error": "the trajectories workload runs on one GPU"}))
        return 1
    import torch

    import inputs
    from paper_1007_1768_b200 import build as B
    B.build()
    from paper_1007_1768_b200 import ssa as S
    torch.cuda.set_device(0)
    cfg = inputs.config(2)
    n = args.n_per_gpu or 16
    t_end = args.t_end or cfg.t_end
    m = S.Model(cfg.network)
    first = S.run_trajectories(m, n, t_end, cfg.seed, 10)
    cap = len(first.time)
    for _ in range(max(args.warmup - 1, 0)):
        S.run_trajectories(m, n, t_end, cfg.seed, 10, capacity=cap)
    dev_ms, events, d2h, red_ms, launches = [], 0, 0, [], 0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            u = S.run_trajectories(m, n, t_end, cfg.seed, 10, capacity=cap)
            dev_ms.append(u.result.device_ms)
            red_ms.append(u.result.reduce_ms)
            d2h = u.result.d2h_bytes
            events += u.result.events
            launches += u.result.kernel_launches
    ms = sum(dev_ms)
    line = {"metric": "ssa_events_per_s", "value": events / (ms / 1e3), "unit": "events/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "full-trajectories-1:10", "model": cfg.network.name, "n_trajectories": n,
                       "t_end": t_end, "stride": 10, "seed": cfg.seed, "points": cap,
                       "timing": "device time of each call incl. the D2H of the points (CUDA events in the library)"},
            "points_per_s": cap * args.steps / (ms / 1e3), "output_bytes_per_step": d2h,
            "sort_gather_ms": statistics.mean(red_ms), "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


def run_dump_bench(args, rank, world):
    """Raw-trajectory dump (a11; north_star: "achieved HBM GB/s for the raw-trajectory dump"):
    config 2 (HIV, 2^18 trajectories, 100 d) with 65,536 dumped ids (R24) into page-locked host
    arrays.  The K1 dump variant writes each dumped trajectory's grid states, event counts and
    last-event times to HBM as it crosses grid points; the library copies them to the host after
    the run (timed separately with CUDA events: `dump_ms`)."""
    if world != 1:
        print(json.dumps({"error": "the dump workload runs on one GPU"}))
        return 1
    import torch

    import inputs
    from paper_1007_1768_b200 import build as B
    B.build()
    from paper_1007_1768_b200 import ssa as S
    torch.cuda.set_device(0)
    cfg = inputs.config(2)
    n = args.n_per_gpu or cfg.n_trajectories
    t_end = args.t_end or cfg.t_end
    n_dump = min(65536, n)
    ids = inputs.dump_ids(n, n_dump, cfg.seed)
    m = S.Model(cfg.network)
    base = [S.run(m, n, t_end, cfg.dt, cfg.seed) for _ in range(2)][-1]    # K1 without the dump
    for _ in range(args.warmup):
        S.run(m, n, t_end, cfg.dt, cfg.seed, dump_ids=ids, dump_pinned=True)
    dev_ms, ssa_ms, dump_ms, events, dbytes, launches = [], [], [], 0, 0, 0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            r = S.run(m, n, t_end, cfg.dt, cfg.seed, dump_ids=ids, dump_pinned=True)
            dev_ms.append(r.device_ms + r.dump_ms)
            ssa_ms.append(r.ssa_ms)
            dump_ms.append(r.dump_ms)
            events += r.events
            dbytes = r.dump_bytes
            launches += r.kernel_launches
    ms = sum(dev_ms)
    k1 = statistics.mean(ssa_ms)
    dm = statistics.mean(dump_ms)
    line = {"metric": "ssa_events_per_s", "value": events / (ms / 1e3), "unit": "events/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2-hiv-100d-dump65536", "model": cfg.network.name, "n_trajectories": n,
                       "n_dump": n_dump, "t_end": t_end, "sample_dt": cfg.dt, "seed": cfg.seed,
                       "timing": "device time of each call incl. the D2H of the dump (CUDA events in the library)"},
            "dump": {"bytes_per_step": dbytes, "d2h_ms": dm, "d2h_GBps": dbytes / (dm / 1e3) / 1e9 if dm > 0 else None,
                     "host_memory": "page-locked",
                     "written_in_loop_GBps": dbytes / (k1 / 1e3) / 1e9,
                     "note": "the dump is written by K1 while it simulates (grid crossings of the dumped "
                             "ids), so its HBM write rate is set by the event loop, not by bandwidth",
                     "k1_ms_with_dump": k1, "k1_ms_without_dump": base.ssa_ms,
                     "k1_overhead": k1 / base.ssa_ms - 1.0},
            "gpu_launches": launches, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n-per-gpu", type=int, default=0, help="override trajectories per GPU (profiling)")
    ap.add_argument("--t-end", type=float, default=0.0, help="override horizon (profiling)")
    ap.add_argument("--path", type=int, default=0)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--tail-lanes", type=int, default=0, help="K1 tail compaction threshold (0 default, -1 off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dump", action="store_true", help="config 4: skip the raw-trajectory dump")
    ap.add_argument("--variant", default="A", choices=["A", "B"],
                    help="HIV configs: B = the gated time-triggered mutation (SPEC.md:424, NEXT 3)")
    ap.add_argument("--workload", default="config", choices=["config", "sweep", "union", "trajectories", "dump"],
                    help="sweep: the Fig. 4 delta_t sensitivity sweep (ssa_run_sweep, 1 GPU); union: selective "
                         "memory at union times over 16 HIV trajectories (ssa_run_union, Fig. 4's ensemble)")
    ap.add_argument("--kx", type=int, default=16, help="union workload: X-reduction factor k_x")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "sweep":
        return run_sweep_bench(args, rank, world)
    if args.workload == "union":
        return run_union_bench(args, rank, world)
    if args.workload == "trajectories":
        return run_traj_bench(args, rank, world)
    if args.workload == "dump":
        return run_dump_bench(args, rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist

    import inputs
    from paper_1007_1768_b200 import build as B
    B.build()
    from paper_1007_1768_b200 import dist as D
    from paper_1007_1768_b200 import ssa as S

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = inputs.config(args.config)
    net = cfg.network
    if args.variant == "B":
        if net.name != "hiv":
            raise SystemExit("--variant B applies to the HIV configs (2, 4)")
        net = inputs.hiv("B")
    # config 4 (box scale, 2^24 trajectories over 8 GPUs): one GPU runs one W=8 shard, 2^21
    # trajectories, and weak scaling keeps that per GPU (N = 8: the full 2^24)
    default_per_gpu = cfg.n_trajectories // 8 if args.config == 4 else cfg.n_trajectories
    n_per = args.n_per_gpu or default_per_gpu
    n_total = n_per * world
    t_end = args.t_end or cfg.t_end
    dt = cfg.dt
    G = S.grid_size(t_end, dt)
    model = S.Model(net)
    path = args.path or cfg.path
    opts = dict(block=args.block, blocks_per_sm=args.blocks_per_sm, tail_lanes=args.tail_lanes)

    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    # config 4 dumps its 65,536 chosen trajectories raw (BASELINE configs[4], R24): each
    # rank dumps the ones in its shard into page-locked host memory, gathered in rank order
    dump_ids = None
    if args.config == 4 and not args.no_dump:
        all_dump = inputs.dump_ids(cfg.n_trajectories, cfg.n_dump, cfg.seed)
        dump_ids = all_dump[all_dump < n_total]
    # rank r owns the aligned id shard r; roots all-gathered over NCCL, merged in rank order
    ens = D.ShardedEnsemble.for_model(model, n_total, t_end, dt, cfg.seed, dev, path=path, stream=sh,
                                      dump_ids=dump_ids, dump_pinned=dump_ids is not None, **opts)
    cells = ens.cells
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    dump_stats = []

    def step():
        l2.zero_()                                               # flush L2 between steps
        res = ens.step()
        if dump_ids is not None:
            loc = res.local
            g = D.gather_dump(loc.dump if loc is not None else None, dev)   # rank order, on rank 0
            dump_stats.append((loc.dump_bytes if loc is not None else 0, loc.dump_ms if loc is not None else 0.0,
                               0 if g is None else len(g.ids)))
        return res

    # JIT + warm-up (untimed)
    jit0 = time.perf_counter()
    model.prepare(local_rank, path)
    jit_s = time.perf_counter() - jit0
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region: K steps, barrier + sync on both sides, device time via events
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    events = 0
    ssa_ms = []
    red_ms, red_bytes = [], 0
    launches = 0
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            res = step()                       # job-wide StepResult, the same on every rank
            events += res.events
            loc = res.local                    # this rank's ssa_run_shard result
            if loc is not None:
                ssa_ms.append(loc.ssa_ms)
                red_ms.append(loc.reduce_ms)
                red_bytes = loc.reduce_bytes
                launches += loc.kernel_launches
            launches += 2      # merge + finalize of ssa_merge_roots
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms, launches = D.max_and_sum([ms, launches], dev)   # max-over-ranks time, launches summed over ranks
    events, launches = int(events), int(launches)
    value = events / (ms / 1e3)
    traj_per_s = n_total * args.steps / (ms / 1e3)

    # end to end through the public API with host buffers (copies inside the timed region)
    e2e = None
    if not args.no_e2e:
        e2e_steps = args.steps                 # the same number of steps as `value`
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_events = 0
        h2d = d2h = 0
        for _ in range(e2e_steps):
            if world == 1:
                r = S.run(model, n_per, t_end, dt, cfg.seed, path=path, stream=sh, **opts)
                e2e_events += r.events
                h2d, d2h = r.h2d_bytes, r.d2h_bytes
            else:
                res = step()
                e2e_events += res.events               # job-wide
                merged = ens.out.cpu()                 # D2H of this step's mean/var/M2/n grids
                h2d = res.local.h2d_bytes if res.local is not None else 0
                d2h = merged.numel() * merged.element_size()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        wall, _ = D.max_and_sum([wall, 0], dev)
        e2e = {"value": e2e_events / wall, "unit": "events/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "note": "ssa_run with host result buffers; wall clock incl. per-run model upload and D2H"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # roofline of the dominant kernel (K1): issue slots
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    props = torch.cuda.get_device_properties(dev)
    n_sm = props.multi_processor_count
    per_rank_events = events / world / args.steps
    k1_ms = statistics.mean(ssa_ms) if ssa_ms else float("nan")
    if path == 1:
        I = alg_instr_per_event(net, path)                                # thread-instructions per event
        achieved = per_rank_events * I / 32.0 / (k1_ms / 1e3) / 1e9      # G warp-instr/s
    else:
        I = alg_warp_instr_per_event(net, 16 if path == 3 else 32)        # warp-instructions per event
        achieved = per_rank_events * I / (k1_ms / 1e3) / 1e9
    peak = n_sm * 4 * sm_max * 1e6 / 1e9                                  # G warp-instr/s
    workload = f"config{args.config}-{cfg.name}" + ("-variantB" if args.variant == "B" else "")
    default_size = not args.n_per_gpu and not args.t_end and args.config != 4
    kname = "ssa_k1" if path == 1 else "ssa_k2"
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s", "frac": achieved / peak,
                "traffic": measured_traffic(workload, kname, default_size),
                "traffic_source": "profiles/traffic.json (ncu dram__bytes_read+write per launch)",
                "ncu_activity": profiled_activity(workload, kname), "kernel": "ssa_k1" if path == 1 else ("ssa_k2" if path == 2 else "ssa_k2 (half-warp)"),
                ("alg_thread_instr_per_event" if path == 1 else "alg_warp_instr_per_event"): I, "kernel_ms": k1_ms,
                "peak_basis": f"{n_sm} SMs x 4 issue slots/clk x {sm_max:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)"}
    if path == 1:
        # round 1 counted plog at 35 (its division-based log): the same achieved rate on that count
        roofline["frac_at_round1_count"] = per_rank_events * (I + 14) / 32.0 / (k1_ms / 1e3) / 1e9 / peak
        # the co-bound: the FP64 pipe issues 0.497 warp-instructions per clock per SMSP
        # (measured, profiles/r1h_pipe_peaks.txt), and about half of K1's work is FP64
        F = alg_fp64_per_event(net)
        f_ach = per_rank_events * F / 32.0 / (k1_ms / 1e3) / 1e9
        f_peak = n_sm * 4 * FP64_PER_SMSP_CLK * sm_max * 1e6 / 1e9
        roofline["fp64_pipe"] = {"achieved": f_ach, "peak": f_peak, "unit": "Gwarp-inst/s", "frac": f_ach / f_peak,
                                 "alg_fp64_thread_instr_per_event": F,
                                 "peak_basis": f"{n_sm} SMs x 4 SMSPs x {FP64_PER_SMSP_CLK} FP64 warp-inst/clk "
                                               f"(scripts/pipe_peaks.cu) x {sm_max:.0f} MHz"}

    if path != 1:
        # K2's co-bound: the shared-memory (LSU data) pipe, one wavefront per clock per SM; K2's
        # propensity rows, state, model tables and shuffles all pass through it.
        # Wavefronts per applied event from the committed ncu capture of the same kernel.
        W = lsu_wavefronts_per_event(workload)
        if W:
            l_ach = per_rank_events * W / (k1_ms / 1e3) / 1e9
            l_peak = n_sm * sm_max * 1e6 / 1e9
            roofline["lsu_pipe"] = {"achieved": l_ach, "peak": l_peak, "unit": "Gwavefronts/s",
                                    "frac": l_ach / l_peak, "wavefronts_per_event": W,
                                    "peak_basis": f"{n_sm} SMs x 1 shared-memory wavefront/clk x {sm_max:.0f} MHz",
                                    "source": "profiles/traffic.json (ncu l1tex__data_pipe_lsu_wavefronts_mem_shared "
                                              "per applied event)"}

    # secondary: the chunk reduction (K3) reads the staged grid samples once -- HBM bound
    hbm_peak = float(peaks.get("hbm_gbs", 7700.0))
    r_ms = statistics.mean(red_ms) if red_ms else float("nan")
    r_gbs = red_bytes / (r_ms / 1e3) / 1e9 if red_ms and r_ms > 0 else None
    roofline_reduce = {"bound": "hbm", "achieved": r_gbs, "peak": hbm_peak, "unit": "GB/s",
                       "frac": (r_gbs / hbm_peak) if r_gbs else None,
                       "traffic": measured_traffic(workload, "ssa_tree_leaf", default_size), "kernel": "ssa_tree_leaf",
                       "bytes_per_launch": red_bytes, "kernel_ms": r_ms,
                       "peak_basis": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200 nominal"}

    clocks = clk.summary()
    dump_block = None
    if dump_ids is not None and dump_stats:
        timed = dump_stats[args.warmup:args.warmup + args.steps]
        b = statistics.mean(x[0] for x in timed)
        dms = statistics.mean(x[1] for x in timed)
        dump_block = {"n_dump_per_gpu": int(len(dump_ids) // world), "n_dump_gathered": int(timed[-1][2]),
                      "bytes_per_step_per_gpu": int(b), "d2h_ms": dms,
                      "d2h_GBps": b / (dms / 1e3) / 1e9 if dms > 0 else None,
                      "written_in_loop_GBps": b / (k1_ms / 1e3) / 1e9 if k1_ms == k1_ms else None,
                      "host_memory": "page-locked", "gather": "rank order (contiguous shards = id order)",
                      "note": "K1's dump variant writes each dumped trajectory's grid states, event counts and "
                              "last-event times while it simulates; the library copies them to the host after "
                              "the run (d2h_ms, CUDA events)"}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cores = host_cores()
        n_cpu = 3 * max(cores, 8)
        ce, ct, cs = oracle_sample(args.config, n_cpu, cores, t_end)
        cpu = {"value": ce / cs, "unit": "events/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{n_cpu} full trajectories of {cfg.name} (ids drawn uniformly from the "
                         f"{cfg.n_trajectories}-id ensemble) over {cores} processes, {cs:.1f} s wall",
               "trajectories_per_s": ct / cs}

    line = {
        "metric": "ssa_events_per_s", "value": value, "unit": "events/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config{args.config}-{cfg.name}" + ("-variantB" if args.variant == "B" else ""),
                   "model": net.name, "species": net.S,
                   "reactions": net.R, "n_trajectories_per_gpu": n_per, "global_batch": n_total, "t_end": t_end,
                   "sample_dt": dt, "grid_points": G, "seed": cfg.seed, "path": {1: "thread", 2: "warp", 3: "halfwarp"}[path],
                   "parallelism": f"dp{world}", "l2": "flushed between steps (256 MiB write)"},
        "trajectories_per_s": traj_per_s,
        "events_per_step": events / args.steps,
        "roofline": roofline,
        "roofline_reduce": roofline_reduce,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "dump": dump_block,
        "gpu_launches": launches,
        "clocks": clocks,
        "jit_s": jit_s,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
