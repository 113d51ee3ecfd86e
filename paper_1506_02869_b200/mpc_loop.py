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


def window_scenario(base: dict, traffic: dict, ids, k: int, states: dict) -> dict:
    """Planning problem of MPC step k for the aircraft `ids` of `traffic`."""
    H = int(base["H"])
    scn = {key: val for key, val in base.items() if key not in ("n", "kind", "first_step", "x0", *PER_AC)}
    scn["n"] = len(ids)
    scn["kind"] = np.array([traffic["kind"][a] for a in ids], np.int32)
    scn["first_step"] = np.array([min(H, max(0, int(traffic["entry"][a]) - k)) for a in ids], np.int32)
    scn["x0"] = np.array([states.get(a, traffic["x0"][a]) for a in ids], np.float64).reshape(-1, 6)
    for key in PER_AC:
        scn[key] = np.array([traffic[key][a] for a in ids], np.float64)
    return scn


def run(base: dict, traffic: dict, L: int, S: int, K: int, sigma, seed: int, n_steps: int,
        max_aircraft: int = 32, use_graph: bool = True, log=None):
    """Run the receding-horizon loop for n_steps MPC updates; returns per-step records
    and per-aircraft outcomes (completion step and mode, fuel burnt)."""
    H = int(base["H"])
    n_tot = len(traffic["kind"])
    states, done = {}, {}
    records = []
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
                                   max_horizon=H, use_graph=use_graph)
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
            for j, a in enumerate(ids):
                if scn["first_step"][j] != 0:
                    continue
                states[a] = nxt[j].copy()
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
    return records, done, fuel
