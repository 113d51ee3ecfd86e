#!/usr/bin/env python3
"""Benchmark of the SMC-in-MPC hot path on B200 (contract: see DESIGN.md section 8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl smcatm|reference]
                    [--config 2] [--no-cpu-baseline]

A step is one MPC update of the workload BASELINE.json's metric is quoted on,
configs[4] (c5: 16 aircraft, L = 2^20 particles, S = 64 wind samples, H = 6,
K = 101 SMC rounds): fresh population, K rounds of rollout + MH + reduce +
systematic resampling + proposal, final selection and the plant step --
every row of SURVEY.md 8(a).  `value` is aircraft-step rollouts per second
over the whole job (device time, inputs resident); `e2e` is the same metric
through the public C ABI call mpc_step() with pinned host buffers,
host<->device copies inside the timed region.  N > 1 (torchrun): the same
2^20 particles sharded over the N GPUs, NCCL exchange each round (strong
scaling).  --config 2|3|4|6|7 selects the other
workloads (c2-c4, the paper's Table-1 workload, the 20-aircraft latency
target).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "aircraft-step rollouts/sec (MPC-step latency reported alongside)"
UNIT = "aircraft-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="smcatm", choices=["smcatm", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--rounds", type=int, default=0,
                    help="SMC rounds per MPC step (0: the config's K; other values are for quick A/B only)")
    ap.add_argument("--phase-steps", type=int, default=2,
                    help="steps of the second (per-kernel timed) pass")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--traffic", default="c3", choices=["c3", "mixed", "congested"],
                    help="traffic stream of --loop")
    ap.add_argument("--mh", type=int, default=-1, choices=[-1, 0, 1, 2],
                    help="move: 0 paper Alg.1, 1 joint MH (R1), 2 per-aircraft MH (R46); -1 = the config's")
    ap.add_argument("--wind-grid", default="",
                    help="N_x,N_y,N_z wind grid points (P:454; default the paper's 2,2,2)")
    ap.add_argument("--warm", type=float, default=0.0,
                    help="warm-start fraction of the population from the previous winner (R45)")
    ap.add_argument("--lfinal", type=int, default=0,
                    help="shrink the population linearly to this many particles by the last round (P:1225)")
    ap.add_argument("--loop-config", type=int, default=3, help="solver configuration of --loop")
    ap.add_argument("--loop", type=int, default=0,
                    help="run the rolling-window MPC loop of c3's traffic for this many steps instead")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4) if len(r) > 5 + j and "Active" in r[5 + j]
                          and "Not" not in r[5 + j]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic(cfgname):
    """dram bytes per K2 launch from the committed ncu --set full capture (profiles/)."""
    p = os.path.join(ROOT, "profiles", "k2_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfgname)
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(scn, cfg, seconds=8.0):
    """The FP64 oracle, as it stands, on this host's cores: evaluation (Alg.1 l.9-18)
    of a bounded particle sample of the same workload (one SMC round's rollouts),
    repeated for ~`seconds` at nproc threads and at one thread; plus c1 (the parity
    config) run in full through the oracle's Alg.1.  Returns the baseline dict."""
    import oracle as O
    from paper_1506_02869_b200 import scenarios as sc
    P = O.Problem(scn)
    nproc = os.cpu_count() or 1
    S = cfg.S or 8                                          # paper schedule: S_0 = 8
    Ha = int(sum(scn["H"] - e for e in scn["first_step"]))

    def rate(nthreads, Lp, budget):
        ctrl = P.init_population(Lp, cfg.seed)
        done, k, t0 = 0, 0, time.perf_counter()
        while True:
            P.evaluate(ctrl, S, k + 1, cfg.seed, nthreads=nthreads)
            done += Lp * S * Ha
            k += 1
            el = time.perf_counter() - t0
            if el >= budget:
                return done / el, k, el

    Lp = min(cfg.L, 2048)
    v, reps, el = rate(nproc, Lp, seconds)
    v1, reps1, el1 = rate(1, min(cfg.L, 128), seconds / 2)
    scn1, cfg1 = sc.config(1)
    t0 = time.perf_counter()
    O.Problem(scn1).run_smc(L=cfg1.L, S=cfg1.S, K=cfg1.K, seed=cfg1.seed, sigma=cfg1.sigma, nthreads=nproc)
    c1_s = time.perf_counter() - t0
    return {"value": v, "unit": UNIT, "cores": nproc, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"oracle evaluate of {Lp} particles x S={S} x {Ha} aircraft-steps (one round's rollouts), "
                      f"{reps} reps, {el:.1f}s, {nproc} threads",
            "value_1thread": v1, "sample_1thread": f"{min(cfg.L, 128)} particles x S={S}, {reps1} reps, {el1:.1f}s",
            "c1_full_mpc_step_s": c1_s,
            "c1_full": f"c1 (2 aircraft, L={cfg1.L}, S={cfg1.S}, H={scn1['H']}, K={cfg1.K}) whole Alg.1 + MH solve, "
                       f"{nproc} threads"}


def workload_str(scn, cfg, args):
    return (f"{cfg.name}: {scn['n']} aircraft ({int((scn['kind'] == 0).sum())} arr / "
            f"{int((scn['kind'] == 1).sum())} dep), L={cfg.L}"
            + (f"->{args.lfinal}" if args.lfinal else "")
            + (", S_k=floor(3+5e^(0.05k))" if cfg.sched_paper else f", S={cfg.S}")
            + f", H={scn['H']}, K={cfg.K} rounds, "
            + {0: "paper Alg.1 (no MH)", 1: "MH on", 2: "per-aircraft MH"}[int(cfg.mh)]
            + (f", wind grid {'x'.join(str(v) for v in scn['wind_n'])}" if args.wind_grid else ""))


def run_reference(args):
    """--impl reference: the FP64 oracle timed on the host cores (rank 0 only)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1506_02869_b200 import roofline, scenarios as sc
    scn, cfg = sc.config(args.config)
    import oracle as O
    P = O.Problem(scn)
    nthreads = os.cpu_count() or 1
    Lp = min(cfg.L, 2048)
    S = cfg.S or 8
    ctrl = P.init_population(Lp, cfg.seed)
    Ha = int(sum(scn["H"] - e for e in scn["first_step"]))
    per_step = Lp * S * Ha
    for w in range(args.warmup):
        P.evaluate(ctrl, S, 1, cfg.seed, nthreads=nthreads)
    ts = []
    for s in range(args.steps):
        t0 = time.perf_counter()
        P.evaluate(ctrl, S, 1 + s, cfg.seed, nthreads=nthreads)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    value = per_step * args.steps / tot
    steps_full = roofline.aircraft_steps(scn, cfg.L, roofline.samples_list(cfg), cfg.mh)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_str(scn, cfg, args),
                   "sample": f"each step: one evaluation round (Alg.1 l.9-18) of {Lp} of the {cfg.L} particles"},
        "mpc_step_latency_ms_extrapolated": 1000 * steps_full / value,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"oracle evaluate of {Lp} particles x S={S} x {Ha} aircraft-steps per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_loop(args):
    """Rolling-window MPC loop: per-step latency vs number of active aircraft
    (SURVEY 8(d) c3 'full MPC receding-horizon loop') and the closed-loop audit (N2):
    landings / exits, realised separation, fuel.  --traffic picks c3's stream (16 arr /
    8 dep) or the paper's mixed (10 + 10) / congested (24 arrivals) shapes."""
    from paper_1506_02869_b200 import mpc_loop, scenarios as sc
    # the loop runs c3's solver unless --loop-config names another configuration
    base, cfg = sc.config(args.loop_config)
    if args.mh >= 0:
        cfg = dataclasses.replace(cfg, mh=args.mh)
    if args.traffic == "mixed":
        tr, desc = sc.paper_mixed(), "paper mixed: 10 arrivals / 10 departures"
    elif args.traffic == "congested":
        tr, desc = sc.paper_congested(), "paper congested: 24 arrivals"
    else:
        tr, desc = sc.traffic(16, 8, seed=1003, arr_every=2, dep_every=8), "c3 traffic: 16 arrivals / 8 departures"
    recs, done, fuel, aud = mpc_loop.run(base, tr, L=cfg.L, S=cfg.S, K=cfg.K, sigma=cfg.sigma, seed=cfg.seed,
                                         n_steps=args.loop, max_aircraft=32, return_audit=True,
                                         warm_fraction=args.warm, L_final=args.lfinal, mh=int(cfg.mh))
    lat = [r.latency_ms for r in recs]
    print(json.dumps({"mode": "mpc_loop", "config": f"{desc}, {cfg.name} solver: L={cfg.L}, S={cfg.S}, K={cfg.K}, mh={int(cfg.mh)}"
                      + (f", warm start {args.warm}" if args.warm else "") + (f", L_final {args.lfinal}" if args.lfinal else ""),
                      "steps": len(recs),
                      "per_step": [{"step": r.step, "window": r.window, "active": r.active,
                                    "latency_ms": round(r.latency_ms, 2), "infeasible": r.infeasible} for r in recs],
                      "max_latency_ms": max(lat) if lat else None, "dt_s": float(base["dt"]),
                      "audit": {"aircraft": aud.n_aircraft, "landed": aud.landed, "exited": aud.exited,
                                "unfinished": aud.unfinished, "separation_violations": aud.sep_violations,
                                "min_separation_m": aud.min_sep_m, "fuel_total_kg": aud.fuel_total_kg},
                      "completed": {str(k): v for k, v in done.items()}}), flush=True)
    return 0


def run_pipe_micro():
    """The pipe microbenchmarks (tools/micro/pipes.cu, built by __graft_entry__.build()) on this
    GPU in this run; [] if the binary is absent."""
    exe = os.path.join(ROOT, "tools", "micro", "pipes")
    if not os.path.exists(exe):
        return []
    try:
        out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
        return [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    except Exception:
        return []


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.loop:
        return run_loop(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1506_02869_b200 import roofline, scenarios as sc, smcatm

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    scn, cfg = sc.config(args.config)
    if args.mh >= 0:
        cfg = dataclasses.replace(cfg, mh=args.mh)
    if args.rounds:
        cfg = dataclasses.replace(cfg, K=args.rounds)
    if args.wind_grid:
        scn["wind_n"] = tuple(int(v) for v in args.wind_grid.split(","))
    stream = torch.cuda.Stream(device=local)
    # N > 1: the config's L particles sharded over the N GPUs (NCCL exchange each round):
    # strong scaling -- the whole job is one MPC problem of fixed size
    L_glob = cfg.L
    L_loc = smcatm.shard_range(L_glob, world, rank)
    L_loc = L_loc[1] - L_loc[0]
    micro = run_pipe_micro() if rank == 0 else []

    def make_solver(profile):
        # profile=True brackets every kernel with CUDA events on the library's stream (graph
        # event nodes, ~5 us each between dependent kernels): used only for the per-kernel pass
        return smcatm.Solver(scn, L=L_glob, S=cfg.S, K=cfg.K, sigma=cfg.sigma, seed=cfg.seed,
                             anneal=cfg.anneal, mh=cfg.mh, sched_paper=cfg.sched_paper, device=local, stream=stream,
                             profile=profile, use_graph=not args.no_graph, rank=rank, world_size=world,
                             L_final=args.lfinal)

    sol = make_solver(False)
    S_list = roofline.samples_list(cfg)
    ac_steps = roofline.aircraft_steps(scn, L_glob, S_list, cfg.mh, args.lfinal)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            sol.solve()
        barrier()
        n0 = sol.launches
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        with ClockSampler(local) as clk:
            barrier()
            for s in range(args.steps):
                flush.fill_(s & 0xFF)                       # L2 flush between timed steps (outside events)
                evs[s][0].record(stream)
                sol.solve()
                evs[s][1].record(stream)
            barrier()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        launches = sol.launches - n0
        # per-kernel pass: 1 warm-up + phase_steps steps with CUDA events around every launch on
        # the launching stream (smc_phase_times) -> K2's average launch duration for the roofline
        psteps = max(1, min(args.phase_steps, args.steps))
        psol = make_solver(True)
        psol.solve()
        barrier()
        psol.phase_times()                                  # reset phase accumulators
        pevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(psteps)]
        for s in range(psteps):
            flush.fill_(s & 0xFF)
            pevs[s][0].record(stream)
            psol.solve()
            pevs[s][1].record(stream)
        barrier()
        phases = psol.phase_times()
        pstep_ms = [a.elapsed_time(b) for a, b in pevs]
        del psol
    tot_ms = sum(step_ms)
    t_local = torch.tensor([tot_ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    tmax_ms = float(t_local.item())
    value = ac_steps * args.steps / (tmax_ms / 1000.0)

    # ---- e2e: public C ABI mpc_step with pinned host buffers, copies inside the timed region
    n = scn["n"]
    meas = torch.from_numpy(np.ascontiguousarray(scn["x0"], dtype=np.float64)).pin_memory()
    applied = torch.empty((n, 3), dtype=torch.float32).pin_memory()
    nxt = torch.empty((n, 6), dtype=torch.float64).pin_memory()
    flags = torch.empty((n,), dtype=torch.int32).pin_memory()
    e2e_ms = []
    with torch.cuda.stream(stream):
        if args.e2e_steps > 0:
            sol.mpc_step_ptr(meas.data_ptr(), applied.data_ptr(), nxt.data_ptr(), flags.data_ptr())   # warm
        barrier()
        sol.io_bytes()                                      # reset the library's copy counters
        for s in range(args.e2e_steps):
            flush.fill_(s & 0xFF)
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            sol.mpc_step_ptr(meas.data_ptr(), applied.data_ptr(), nxt.data_ptr(), flags.data_ptr())
            b.record(stream)
            b.synchronize()
            e2e_ms.append(a.elapsed_time(b))
        sol.phase_times()
        io_h2d, io_d2h = sol.io_bytes()
    e2e_t = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = ac_steps * args.e2e_steps / (float(e2e_t.item()) / 1000.0) if e2e_ms else None
    # bytes the library copied per e2e step (counted in libsmcatm: measured states, per-aircraft
    # constants, MPC index up; winner index, next states, applied controls, flags down)
    h2d = io_h2d // max(1, args.e2e_steps)
    d2h = io_d2h // max(1, args.e2e_steps)

    sol.close()                      # every rank tears its communicator down at the same point
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (K2 rollout + MH): max over the pipes of the algorithmic
    # op count / the pipe's measured peak (roofline.py), against K2's measured time
    peaks, peak_src = load_peaks()
    clocks = clk.summary()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    pipe_pk, pipe_src = roofline.load_pipe_peaks(ROOT, micro)
    k2_ms, k2_n = phases["rollout"]
    rounds = [(st * psteps * L_loc / L_glob, C, S) for st, C, S in
              roofline.round_list(scn, L_glob, S_list, cfg.mh, args.lfinal)]
    rf = roofline.k2_roofline(scn, rounds, k2_ms / 1000.0, sm_mhz, pipe_pk)
    bind = rf["binding_pipe"]
    peak_ops = pipe_pk[bind] * roofline.SMS * sm_mhz * 1e6
    achieved = rf["ops"][bind] / (k2_ms / 1000.0) if k2_ms > 0 else 0.0
    all_ms = sum(v[0] for v in phases.values())
    # Table 1's workload (config 6) is the one with a printed number: 56 s per MPC update on
    # a GTX 580, i.e. ac_steps / 56 aircraft-steps/s
    vs_baseline = value / (ac_steps / 56.0) if (cfg.name == "table1" and world == 1 and not args.lfinal
                                                   and not args.wind_grid) else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tmax_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": vs_baseline, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_str(scn, cfg, args),
                   "parallelism": (f"{L_glob} particles sharded over {world} GPUs ({L_loc} on rank 0; per round NCCL "
                                   "all-reduce of column maxima + all-gather of per-rank weight totals, parent rows "
                                   "read in place from their owner over NVLink (CUDA IPC peer mappings))"
                                   if world > 1 else "single GPU"),
                   "l2": "flushed between timed steps (256 MiB write, outside the events)",
                   "cuda_graph": not args.no_graph,
                   "aircraft_steps_per_step": ac_steps},
        "mpc_step_latency_ms": tmax_ms / args.steps,
        "step_ms": step_ms,
        "e2e": ({"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                 "mpc_step_latency_ms": sum(e2e_ms) / len(e2e_ms)} if e2e_ms else None),
        "gpu_launches": launches,
        "phase_ms_per_step": {k: v[0] / psteps for k, v in phases.items()},
        "phase_pass": {"what": f"second pass: 1 warm-up + {psteps} steps with CUDA events around every kernel "
                               "launch (its event nodes lengthen the step, so value is timed without them)",
                       "ms_per_step": sum(pstep_ms) / len(pstep_ms)},
        "roofline": {"kernel": "k_rollout (K2: rollout + MH)", "bound": "alu", "pipe": bind,
                     "achieved": achieved / 1e9, "peak": peak_ops / 1e9,
                     "unit": f"Gop/s on the {bind} pipe (algorithmic ops, roofline.py)",
                     "frac": rf["frac"], "traffic": load_traffic(cfg.name),
                     "t_roof_ms_per_pipe": {p: 1e3 * t / psteps for p, t in rf["t_pipe_s"].items()},
                     "k2_ms_per_step": k2_ms / psteps,
                     "peak_source": f"{pipe_pk[bind]:.2f} ops/SM/clk ({pipe_src}) x 148 SMs x sm_max_mhz {sm_mhz} "
                                    f"({peak_src})",
                     "pipe_peaks_per_sm_clk": pipe_pk,
                     "ops_per_aircraft_step": {f"C={c}": {p: round(float(v), 2) for p, v in
                                                          roofline.pipe_ops(scn, c, cfg.S or 8).items()}
                                               for c in (1, 2)},
                     "k2_share_of_step": k2_ms / all_ms if all_ms else None},
        "clocks": clocks,
    }
    # resample/propose phase vs HBM
    rs_ms = phases["resample"][0] + phases["propose"][0]
    if rs_ms > 0:
        rb = roofline.resample_bytes(scn["n"], L_loc, scn["H"]) * (cfg.K - 1) * psteps
        line["roofline_resample"] = {"bound": "hbm", "achieved": rb / (rs_ms / 1000.0) / 1e9,
                                     "peak": float(peaks.get("hbm_gbs", 6650.0)), "unit": "GB/s",
                                     "frac": rb / (rs_ms / 1000.0) / 1e9 / float(peaks.get("hbm_gbs", 6650.0))}
    if micro:
        line["pipe_micro"] = micro
    if not args.no_cpu_baseline and world == 1:      # the oracle on the host cores: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(scn, cfg)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
