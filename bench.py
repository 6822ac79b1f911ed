#!/usr/bin/env python
"""Benchmark: time-to-price and path-steps/s of the nested-MC pricers on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--mode parity|fast]
    python bench.py --impl reference ...      # the reference CPU pricer, same metric

A step is one full pricing run of the configured BASELINE.json workload
through the public API: rule build over every exercise date (CMC: sample +
label + AdaBoost per date; I&Z: probe solves + regression per date) plus the
final pricing run.  ``value`` is nominal path-steps (paths x remaining exercise
dates, the reference's unit) of the whole job per second of device time; the
default workload is config 5 (the BASELINE scaling sweep, CMC max-call d=10),
sharded over N GPUs (strong scaling).  Multi-GPU runs are one process per GPU
under torch.distributed (NCCL); rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = 1827  # master_seed = 1827 for every config

CONFIGS = {
    "c1": dict(name="c1-iz-put-d1", method="iz", d=1, payoff="put", s0=40.0, strike=40.0, r=0.06, sigma=0.2,
               delta=0.0, rho=None, maturity=1.0, n_dates=10, j_points=1, n_inner=2000, solver="bisection",
               bracket=(20.0, 40.0), tol=1e-4, n_paths=1 << 18, mode="parity"),
    "c2": dict(name="c2-iz-geoput-d5", method="iz", d=5, payoff="geoput", s0=100.0, strike=100.0, r=0.03,
               sigma=0.4, delta=0.0, rho=None, maturity=1.0, n_dates=10, j_points=64, n_inner=5000,
               solver="bisection", bracket=(50.0, 100.0), tol=1e-4, n_paths=1 << 20, mode="parity"),
    "c3": dict(name="c3-cmc-maxcall-d5", method="cmc", d=5, payoff="maxcall", s0=100.0, strike=100.0, r=0.05,
               sigma=0.2, delta=0.10, rho=None, maturity=3.0, n_dates=9, n_train=5000, n_label=500, rounds=150,
               n_paths=1 << 20, sampler="forward", mode="fast"),
    "c4": dict(name="c4-cmc-basketput-d40", method="cmc", d=40, payoff="basketput", s0=100.0, strike=100.0,
               r=0.05, sigma="u[0.2,0.4]", delta=0.0, rho=0.3, maturity=1.0, n_dates=20, n_train=20000,
               n_label=1000, rounds=200, n_paths=1 << 22, sampler="forward", mode="fast"),
    "c5": dict(name="c5-cmc-maxcall-d10", method="cmc", d=10, payoff="maxcall", s0=100.0, strike=100.0, r=0.05,
               sigma=0.2, delta=0.10, rho=None, maturity=3.0, n_dates=9, n_train=10000, n_label=2000, rounds=100,
               n_paths=1 << 24, sampler="bridge", mode="parity"),
}

# ALGORITHMIC fp64 operations per executed asset-step of the parity pipeline
# (SURVEY.md section 8(d)): AS241 central ~33 DP + divide + the 15% tail share
# (log + sqrt), 53-bit uniform 2, GBM step 3, exp 17 -> ~70 DP instructions.
# This is the work the roofline counts, independent of this build's SASS.
DP_OPS_PER_ASSET_STEP = 70.0
# What the walker actually executes on the fp64 pipe (ncu: DADD+DMUL+DFMA+DSETP
# thread instructions / executed asset-steps on the C5 label launch of the
# log-price walker, profiles/r02f/walk_log_c5_sass_mix.txt; the price stepper
# of the other parity configs executes 80.7): reported beside the algorithmic
# count, it is fewer because the log-price state needs no per-step exponential.
DP_OPS_EXECUTED_NCU = 66.3
DP_OPS_EXECUTED_NCU_PRICE_STEPPER = 80.7
# DRAM bytes per walker launch from the same capture (dram__bytes_read+write,
# profiles/r02f/walk_log_c5_summary.txt): label launch 959.7 KB, pricing 80.4 KB
WALK_DRAM_BYTES_PER_LAUNCH = (959.7e3 + 80.4e3) / 2
FP64_LANES_PER_SM = 64
N_SMS = 148
# fast mode (fp32 Box-Muller) walker: issue-bound (ncu issue slots 68%, ALU
# 46%, XU 23% on the C5 label launch).  ALGORITHMIC thread instructions per
# asset-step: 3 MUFU + ~8 FP32 + ~15 INT (Philox,
# 1/4 call per normal) + ~5 other = 31; peak = 4 schedulers x 32 lanes per SM
# per clock.  The d = 10 walker executes 72.8 (ncu, profiles/r01d_walk_c5_fast.txt).
FAST_INST_PER_ASSET_STEP = 31.0
FAST_INST_EXECUTED_NCU_D10 = 72.8
# d = 40 walker with the column-constant prefix step and the lean Box-Muller / ex2 arithmetic
# (C4 label launch of date 1, profiles/r02h/walk_c4_fast_lines.txt; 74.0 with the triangular product)
FAST_INST_EXECUTED_NCU_D40 = 35.2
ISSUE_LANES_PER_SM = 128


def sigma_of(cfg):
    if cfg["sigma"] == "u[0.2,0.4]":
        return np.random.default_rng(SEED).uniform(0.2, 0.4, cfg["d"])
    return cfg["sigma"]


def nominal_path_steps(cfg, iterations=None) -> float:
    nd = cfg["n_dates"]
    final = cfg["n_paths"] * nd
    if cfg["method"] == "cmc":
        build = sum(cfg["n_train"] * cfg["n_label"] * (nd - m) for m in range(1, nd))
    else:
        if iterations is None:
            iterations = math.ceil(math.log2((cfg["bracket"][1] - cfg["bracket"][0]) / cfg["tol"]))
        items = cfg["j_points"] * (1 if cfg["payoff"] == "geoput" else cfg["d"])
        build = sum(items * iterations * cfg["n_inner"] * (nd - m) for m in range(1, nd))
    return float(build + final)


# ------------------------------------------------------------------ clocks ----
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ engine ----
def build_objects(cfg, E):
    kind = {"maxcall": E.PayoffKind.MAX_CALL, "put": E.PayoffKind.PUT_1D, "geoput": E.PayoffKind.GEO_PUT,
            "basketput": E.PayoffKind.BASKET_PUT}[cfg["payoff"]]
    params = E.MarketParams(d=cfg["d"], s0=cfg["s0"], r=cfg["r"], sigma=sigma_of(cfg), delta=cfg["delta"],
                            rho=cfg["rho"])
    spec = E.BermudanSpec(cfg["strike"], cfg["maturity"], cfg["n_dates"], kind)
    return params, spec


def engine_step(cfg, E, params, spec, mode):
    if cfg["method"] == "cmc":
        rule, rep = E.build_cmc_rule(params, spec, E.CmcBuildConfig(cfg["n_train"], cfg["n_label"], cfg["rounds"]),
                                     seed=SEED, sampler=cfg["sampler"], mode=mode)
        est = E.price(params, spec, E.CmcScoreRule(rule), cfg["n_paths"], SEED, mode=mode)
        return est, rep, None
    b, rep = E.build_iz_boundary(params, spec, cfg["j_points"], cfg["n_inner"], seed=SEED, solver=cfg["solver"],
                                 bracket=cfg["bracket"], tol=cfg["tol"], mode=mode)
    est = E.price(params, spec, E.IzRule(b), cfg["n_paths"], SEED, mode=mode, unconverged_points=rep.unconverged_points)
    return est, rep, float(np.mean(rep.iteration_counts)) if rep.iteration_counts else None


def run_engine(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo: host-staged collectives (lets several ranks share one GPU in tests)
            dist.init_process_group("gloo")
    import paper_0805_1827_b200 as E
    from paper_0805_1827_b200 import _native as N

    mode = args.mode or cfg["mode"]
    params, spec = build_objects(cfg, E)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        engine_step(cfg, E, params, spec, mode)
    barrier()

    # (1) device time: CUDA events on the launch stream, clocks sampled, every
    #     library launch bracketed by events (kernel shares, roofline)
    N.profile_reset()
    N.profile_enable(True)
    times, ests = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            est, rep, iters = engine_step(cfg, E, params, spec, mode)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            ests.append(est)
            barrier()
    N.profile_enable(False)
    prof = N.profile_read()
    # (2) end to end: wall clock around the public API call (numpy / Python
    #     objects in, PriceEstimate out), host<->device staging counted
    N.profile_reset()
    walls = []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        w0 = time.perf_counter()
        engine_step(cfg, E, params, spec, mode)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - w0)
        barrier()
    h2d, d2h = N.transfer_read()
    alt = None
    if cfg["method"] == "cmc" and mode == "parity" and not args.no_fast_line:
        # the same workload in fast mode (fp32 Box-Muller stepping, fixed-point AdaBoost), for reference
        engine_step(cfg, E, params, spec, "fast")
        ts = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            est_f, _, _ = engine_step(cfg, E, params, spec, "fast")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms_f = float(np.mean(ts))
        alt = {"mode": "fast", "dtype": "f32-step/f64-sum", "ms_per_step": ms_f,
               "value": nominal_path_steps(cfg) / (ms_f / 1e3), "price": est_f.price, "ci95": est_f.ci95}
    ms = float(np.mean(times))
    wall = float(np.mean(walls))
    if world > 1:
        t = torch.tensor([ms, wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, wall = float(t[0]), float(t[1])
    work = nominal_path_steps(cfg, iters)
    value = work / (ms / 1e3)
    clocks = clk.summary()

    # roofline of the dominant kernel: the walker (labels + pricing + probe walks)
    walk_ms, walk_launches, walk_steps = prof["walk"]
    iz_ms, iz_launches, iz_steps = prof["iz"]
    kern_ms, kern_steps, kern_launches = walk_ms + iz_ms, walk_steps + iz_steps, walk_launches + iz_launches
    sm_mhz = clocks["sm_mhz"] or 1965.0
    peak = FP64_LANES_PER_SM * N_SMS * sm_mhz * 1e6 / 1e12  # T fp64 lane-ops/s at the sampled clock
    if mode == "fast":
        peak = ISSUE_LANES_PER_SM * N_SMS * sm_mhz * 1e6 / 1e12  # T thread-instructions/s issue peak
    ops = DP_OPS_PER_ASSET_STEP if mode == "parity" else FAST_INST_PER_ASSET_STEP
    log_walker = cfg["method"] == "cmc" and cfg.get("payoff") == "maxcall" and not cfg.get("rho")
    executed = ((DP_OPS_EXECUTED_NCU if log_walker else DP_OPS_EXECUTED_NCU_PRICE_STEPPER) if mode == "parity"
                else (FAST_INST_EXECUTED_NCU_D40 if cfg["d"] == 40 else FAST_INST_EXECUTED_NCU_D10))
    achieved = (kern_steps * cfg["d"] * ops) / (kern_ms / 1e3) / 1e12 if kern_ms > 0 else None
    total_launches = sum(v[1] for v in prof.values())
    total_kernel_ms = sum(v[0] for v in prof.values())

    line = None
    if rank == 0:
        est = ests[-1]
        line = {
            "metric": "path-steps/sec (nominal, whole job) & time-to-price",
            "value": value, "unit": "path-steps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "time_to_price_s": ms / 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if mode == "parity" else "f32-step/f64-sum",
            "data": "synthetic (BASELINE.json config, master_seed 1827)",
            "config": {"workload": cfg["name"], "method": cfg["method"], "d": cfg["d"], "n_dates": cfg["n_dates"],
                       **({"n_train": cfg["n_train"], "n_label": cfg["n_label"], "boost_rounds": cfg["rounds"],
                           "sampler": cfg["sampler"]} if cfg["method"] == "cmc" else
                          {"j_points": cfg["j_points"], "n_inner": cfg["n_inner"], "solver": cfg["solver"]}),
                       "n_paths": cfg["n_paths"], "mode": mode, "nominal_path_steps": work,
                       "l2": "flushed (256 MB write) before every timed step", "parallelism": f"dp{world}"},
            "price": est.price, "ci95": est.ci95,
            "e2e": {"value": work / wall, "unit": "path-steps/s", "h2d_bytes_per_step": h2d // max(args.steps, 1),
                    "d2h_bytes_per_step": d2h // max(args.steps, 1),
                    "note": "public API (numpy in/out) wall clock incl. host staging"},
            "value_basis": "CUDA events on the launch stream around the public-API call (host gaps included); "
                           "kernel_ms_total_per_step is the sum of the library's own kernel times",
            "gpu_launches": total_launches // max(args.steps, 1),
            "kernel_ms_per_step": {k: v[0] / max(args.steps, 1) for k, v in prof.items() if v[1]},
            "kernel_ms_total_per_step": total_kernel_ms / max(args.steps, 1),
            "roofline": {"bound": "fp64-pipe" if mode == "parity" else "issue", "achieved": achieved,
                         "peak": peak if achieved is not None else None,
                         "unit": "TFLOP/s" if mode == "parity" else "T thread-instructions/s",
                         "frac": achieved / peak if achieved is not None else None,
                         "asset_steps_per_s": kern_steps * cfg["d"] / (kern_ms / 1e3) if kern_ms > 0 else None,
                         "traffic": WALK_DRAM_BYTES_PER_LAUNCH, "traffic_unit": "bytes/launch (ncu, r02f capture of the C5 walker)",
                         "kernel": "walk_units+iz_probes",
                         "work": (f"{ops:g} algorithmic " + ("fp64 ops" if mode == "parity" else "thread-instructions")
                                  + " per asset-step (SURVEY.md 8(d)) x executed asset-steps "
                                  f"({kern_steps // max(args.steps, 1)} path-steps x d per step)"),
                         "executed_per_asset_step_ncu": executed,
                         "pipe_utilisation": (achieved * executed / ops / peak) if achieved is not None else None,
                         "kernel_ms_per_step": kern_ms / max(args.steps, 1),
                         "launches_per_step": kern_launches / max(args.steps, 1),
                         **({"note": "geometric-put probes: only pass 0 of each date's bisection simulates paths "
                                     "(and is counted); the other passes replay its record (draw cache), so the "
                                     "fp64 fraction understates the probe kernel by construction"}
                            if cfg["method"] == "iz" and cfg.get("payoff") == "geoput" and mode == "parity" else {}),
                         "peak_source": "of NOMINAL peak: 148 SM x " + ("64 fp64 lanes" if mode == "parity" else
                                                                "4 schedulers x 32 lanes") + " x sampled SM clock "
                                        "(MEASURED_PEAKS.json has no fp64 / issue figure)"},
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, full=args.cpu_baseline == "full")
        if alt is not None:
            line["fast_mode"] = alt
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


# --------------------------------------------------------------- reference ----
def reference_sample(cfg) -> dict:
    """A bounded (~10-30 s on 8 cores) sample of the workload for the reference CPU pricer."""
    s = dict(cfg)
    if cfg["method"] == "cmc":
        s.update(n_train=max(cfg["n_train"] // 20, 250), n_paths=1 << 20)
    else:
        s.update(n_paths=min(cfg["n_paths"], 1 << 20))
    return s


def reference_step(sample, B, engine):
    kind = {"maxcall": B.PayoffKind.MAX_CALL, "put": B.PayoffKind.PUT_1D}.get(sample["payoff"])
    if kind is None:
        raise NotImplementedError(f"the reference has no {sample['payoff']} payoff")
    params = B.MarketParams(d=sample["d"], s0=sample["s0"], r=sample["r"], sigma=sigma_of(sample),
                            delta=sample["delta"], rho=sample["rho"])
    spec = B.BermudanSpec(sample["strike"], sample["maturity"], sample["n_dates"], kind)
    if sample["method"] == "cmc":
        rule, _ = B.build_cmc_rule(params, spec, B.CmcBuildConfig(sample["n_train"], sample["n_label"],
                                                                  sample["rounds"]), seed=SEED, engine=engine)
        return B.price(params, spec, B.CmcScoreRule(rule), sample["n_paths"], SEED, engine=engine), None
    # the reference's own solver (fixed point, boundary_iz.py:223-247); its nominal work uses its iteration count
    b, rep = B.build_iz_boundary(params, spec, sample["j_points"], sample["n_inner"], seed=SEED, engine=engine)
    return B.price(params, spec, B.IzRule(b), sample["n_paths"], SEED, engine=engine), float(np.mean(rep.iteration_counts))


RESTATED_SCALE = {"c4": 0.01}  # training points and final paths of the restated C4 run (label paths stay full)


def restated_baseline(cfg) -> dict:
    """configs the reference cannot express (C2,
    C4) are timed on the C restatement over every host core (oracle/restated.py),
    labelled "restated, not reference"; C4 at a stated scale factor."""
    from oracle import restated as RS
    key = [k for k, v in CONFIGS.items() if v["name"] == cfg["name"]][0]
    r = RS.time_config(cfg, scale=RESTATED_SCALE.get(key, 1.0), seed=SEED)
    return {"value": r["value"], "unit": "path-steps/s", "cores": r["threads"], "kind": "port",
            "sample": f"restated, not reference (the reference has no {cfg['payoff']} payoff, market.py:40-47): "
                      f"oracle/restated.py C walker on {r['threads']} threads, {r['sample']}, "
                      f"{r['path_steps']:.3g} nominal path-steps in {r['seconds']:.1f} s",
            "seconds_per_run": r["seconds"]}


def cpu_baseline(cfg, steps: int = 1, full: bool = True) -> dict:
    if cfg["payoff"] not in ("maxcall", "put"):
        return restated_baseline(cfg)
    try:
        from oracle import reference as R
        from oracle.oracle import cpu_count
        B = R.bermuda()
    except ImportError as exc:
        return {"value": None, "unit": "path-steps/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}
    sample = dict(cfg) if full else reference_sample(cfg)
    cores = cpu_count()
    engine = B.Engine(workers=cores, pool="process")
    t = []
    iters = None
    for _ in range(steps):
        t0 = time.perf_counter()
        _, iters = reference_step(sample, B, engine)
        t.append(time.perf_counter() - t0)
    work = nominal_path_steps(sample, iters)
    return {"value": work / float(np.mean(t)), "unit": "path-steps/s", "cores": cores, "kind": "reference",
            "sample": ((f"the FULL {sample['name']} config, one run: " if full else f"{sample['name']} sample: ") +
                       f"n_train={sample.get('n_train')} n_paths={sample['n_paths']} "
                       f"({work:.3g} nominal path-steps), unmodified reference (oracle/_ref, Cython walker, "
                       f"Engine(workers={cores}, pool='process')), {np.mean(t):.1f} s per run"),
            "seconds_per_run": float(np.mean(t))}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    try:
        from oracle import reference as R
        from oracle.oracle import cpu_count
        B = R.bermuda()
    except ImportError as exc:
        return {"impl": "reference", "unavailable": f"reference build missing: {exc}"}
    sample = reference_sample(cfg)
    if sample["payoff"] not in ("maxcall", "put"):
        # no reference implementation: the restated C port over every host core
        for _ in range(args.warmup if args.warmup <= 1 else 1):
            restated_baseline(cfg)
        runs = [restated_baseline(cfg) for _ in range(max(1, min(args.steps, 3)))]
        value = float(np.mean([r["value"] for r in runs]))
        cb = dict(runs[-1], value=value)
        return {"metric": "path-steps/sec (nominal, whole job) & time-to-price", "value": value,
                "unit": "path-steps/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": len(runs),
                "warmup": args.warmup, "ms_per_step": float(np.mean([r["seconds_per_run"] for r in runs])) * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (BASELINE.json config, master_seed 1827)",
                "config": {"workload": cfg["name"], "parallelism": f"cpu{cb['cores']}",
                           "scale": RESTATED_SCALE.get(args.config, 1.0)},
                "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": value, "unit": "path-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    cores = cpu_count()
    engine = B.Engine(workers=cores, pool="process")
    for _ in range(args.warmup):
        reference_step(sample, B, engine)
    t, iters = [], None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _, iters = reference_step(sample, B, engine)
        t.append(time.perf_counter() - t0)
    work = nominal_path_steps(sample, iters)
    ms = float(np.mean(t)) * 1e3
    value = work / (ms / 1e3)
    return {"metric": "path-steps/sec (nominal, whole job) & time-to-price", "value": value, "unit": "path-steps/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE.json config, master_seed 1827)",
            "config": {"workload": cfg["name"], "sample_n_train": sample.get("n_train"),
                       "sample_n_paths": sample["n_paths"], "nominal_path_steps": work,
                       "parallelism": f"cpu{cores}"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "path-steps/s", "cores": cores, "kind": "reference",
                             "sample": f"{cfg['name']} scaled to n_train={sample.get('n_train')}, "
                                       f"n_paths={sample['n_paths']}; unmodified reference (oracle/_ref)"},
            "e2e": {"value": value, "unit": "path-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("engine", "reference"), default="engine")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--mode", choices=("parity", "fast"), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-baseline", choices=("full", "sample"), default="full",
                    help="time the reference CPU pricer on the full config (default) or the bounded sample")
    ap.add_argument("--no-fast-line", action="store_true", help="skip the fast-mode companion measurement")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl")
    ap.add_argument("--scale", type=float, default=1.0, help="scale n_train / n_paths (tests only)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.scale != 1.0:
        for key in ("n_train", "n_paths", "j_points"):
            if key in cfg:
                cfg[key] = max(1, int(cfg[key] * args.scale))
    line = run_reference(args, cfg) if args.impl == "reference" else run_engine(args, cfg)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
