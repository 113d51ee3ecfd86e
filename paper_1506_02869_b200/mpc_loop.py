"""Rolling-window MPC loop around libsmcatm.

Host bookkeeping only: which aircraft are in the planning window, their entry
step inside the horizon (first_step), the measured states carried from one
MPC update to the next, and completion (landed / exited flags returned by the
plant step).  Every per-particle computation runs in the CUDA kernels behind
``mpc_step``.

An aircraft is *activated* once its entry step falls inside the horizon
[k, k+H] and is optimised from the point it enters (first_step =
entry - k, R20); it is deactivated after the plant step reports it
landed (Eq. TO_init) or, for a departure, beyond D_TMA (R19).
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np

from . import smcatm

PER_AC = ["theta_F", "z_tf", "v_D", "beta_f", "S", "cd0", "cd2", "eta", "m_empty", "T_min", "T_max", "v_min",
          "v_max", "gamma_max", "phi_max", "z_min", "z_max"]


@dataclasses.dataclass
class StepRecord:
    step: int
    active: int
    window: int
    latency_ms: float
    best_lambda: float
    infeasible: bool


@dataclasses.dataclass
class Audit:
    """Closed-loop solution quality of one run."""
    n_aircraft: int
    landed: int
    exited: int
    unfinished: int
    sep_violations: int            # (step, pair) with Eq. avoidance failed in the realised states
    min_sep_m: float               # smallest horizontal distance of a vertically overlapping pair
    fuel_total_kg: float
    fuel_kg: dict                  # aircraft -> fuel burnt so far
    completion: dict               # aircraft -> (MPC step, "landed" | "exited")


def audit(base: dict, traffic: dict, plant_log, done: dict, fuel: dict) -> Audit:
    """Post-hoc audit of the realised (plant) trajectories.  plant_log[k] maps every
    aircraft the plant advanced at MPC step k to its state after the step.  A pair
    is in conflict when Eq. avoidance fails: horizontal distance
    < 2 P_r and altitude difference < 2 P_h."""
    two_r, two_h = 2.0 * float(base["P_r"]), 2.0 * float(base["P_h"])
    viol, min_sep = 0, float("inf")
    for states in plant_log:
        ids = sorted(states)
        for u in range(len(ids)):
            for w in range(u + 1, len(ids)):
                a, b = states[ids[u]], states[ids[w]]
                dxy = float(np.hypot(a[0] - b[0], a[1] - b[1]))
                if abs(a[2] - b[2]) < two_h:
                    min_sep = min(min_sep, dxy)
                    if dxy < two_r:
                        viol += 1
    n_tot = len(traffic["kind"])
    landed = sum(1 for v in done.values() if v[1] == "landed")
    exited = sum(1 for v in done.values() if v[1] == "exited")
    return Audit(n_tot, landed, exited, n_tot - landed - exited, viol, min_sep,
                 float(sum(fuel.values())), dict(fuel), dict(done))


def window_scenario(base: dict, traffic: dict, ids, k: int, states: dict) -> dict:
    """Planning problem of MPC step k for the aircraft `ids` of `traffic`."""
    H = int(base["H"])
    scn = {key: val for key, val in base.items() if key not in ("n", "kind", "first_step", "x0", *PER_AC)}
    scn["n"] = len(ids)
    scn["id"] = np.array(ids, np.int64)           # persistent identity for warm starts (R45)
    scn["kind"] = np.array([traffic["kind"][a] for a in ids], np.int32)
    scn["first_step"] = np.array([min(H, max(0, int(traffic["entry"][a]) - k)) for a in ids], np.int32)
    scn["x0"] = np.array([states.get(a, traffic["x0"][a]) for a in ids], np.float64).reshape(-1, 6)
    for key in PER_AC:
        scn[key] = np.array([traffic[key][a] for a in ids], np.float64)
    return scn


def run(base: dict, traffic: dict, L: int, S: int, K: int, sigma, seed: int, n_steps: int,
        max_aircraft: int = 32, use_graph: bool = True, log=None, return_audit: bool = False, **solver_kw):
    """Run the receding-horizon loop for n_steps MPC updates; returns per-step records
    and per-aircraft outcomes (completion step and mode, fuel burnt), plus the
    closed-loop Audit when return_audit.  solver_kw go to smcatm.Solver."""
    H = int(base["H"])
    n_tot = len(traffic["kind"])
    states, done = {}, {}
    records = []
    plant_log = []
    solver = None
    for k in range(n_steps):
        ids = [a for a in range(n_tot) if a not in done and int(traffic["entry"][a]) <= k + H]
        if not ids:
            if all(int(traffic["entry"][a]) <= k for a in range(n_tot)):
                break
            continue
        scn = window_scenario(base, traffic, ids, k, states)
        if solver is None:
            solver = smcatm.Solver(scn, L=L, S=S, K=K, sigma=sigma, seed=seed, max_aircraft=max_aircraft,
                                   max_horizon=H, use_graph=use_graph, **solver_kw)
        else:
            solver.set_scenario(scn)
        solver.mpc_index = k
        t0 = time.perf_counter()
        ok = True
        try:
            applied, nxt, flags = solver.mpc_step(scn["x0"])
        except smcatm.SmcError as e:
            if e.status != smcatm.SMC_EINFEASIBLE:
                raise
            ok = False
        dt_ms = 1000.0 * (time.perf_counter() - t0)
        lam = float("-inf")
        if ok:
            _, lam, _ = solver.best_controls(allow_infeasible=True)
            plant_log.append({})
            for j, a in enumerate(ids):
                if scn["first_step"][j] != 0:
                    continue
                states[a] = nxt[j].copy()
                plant_log[-1][a] = states[a]
                if flags[j] & 1:
                    done[a] = (k + 1, "landed")
                elif flags[j] & 2:
                    done[a] = (k + 1, "exited")
        active = int((scn["first_step"] == 0).sum())
        records.append(StepRecord(k, active, len(ids), dt_ms, lam, not ok))
        if log:
            log(f"step {k:3d}: window {len(ids):2d} active {active:2d} {dt_ms:8.1f} ms "
                f"lambda {lam:9.3f}{' INFEASIBLE' if not ok else ''}")
        if not ok:
            break
    fuel = {a: float(traffic["x0"][a][5] - states[a][5]) for a in states}
    if solver is not None:
        solver.close()
    if return_audit:
        return records, done, fuel, audit(base, traffic, plant_log, done, fuel)
    return records, done, fuel
