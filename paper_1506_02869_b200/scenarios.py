"""Seeded synthetic, Gatwick-shaped inputs shared by the CUDA path and the oracle.

This module holds NO arithmetic of the method (no dynamics, costs, wind
covariance, popdense, resampling ...): it only draws initial aircraft states,
goals and constants, and returns them as a plain dict of numpy arrays.  Both
``paper_1506_02869_b200.smcatm`` (the product binding) and ``oracle`` (test
infrastructure) consume the same dict.  The recipe is DESIGN.md section 5.

Geometry: single E-W runway at the origin, TMA = 30 km circle, x East,
y North.  Aircraft type: A320-class constants (values in DESIGN.md).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

DEG = math.pi / 180.0

# A320-class type (S, C_D0, C_D2 from SPEC S:46; bounds and eta invented, labelled in DESIGN.md)
A320 = dict(S=122.6, cd0=0.024, cd2=0.0375, eta=1.0e-5,
            T_min=0.0, T_max=1.2e5, v_min=70.0, v_max=180.0,
            gamma_max=6.0 * DEG, phi_max=30.0 * DEG, z_min=0.0, z_max=12000.0)

DEP_BEARINGS = [45.0, 90.0, 135.0, -45.0, -90.0, -135.0]
ARR_SECTORS = [(20.0, 70.0), (-70.0, -20.0), (95.0, 140.0)]
LAYERS = [2500.0, 3200.0, 3900.0, 4600.0]


@dataclasses.dataclass
class SmcConfig:
    name: str
    L: int            # particles
    S: int            # wind samples per particle per round (BASELINE "J")
    K: int            # SMC rounds = J_max + 1
    sigma: tuple      # perturbation std (T [N], phi [rad], gamma [rad])
    anneal: float = 0.98
    mh: bool = True
    sched_paper: bool = False
    seed: int = 0x5EED0000


def base_scenario(H: int = 6, dt: float = 10.0) -> dict:
    """Constants shared by every config."""
    return dict(
        H=H, dt=dt, g=9.81, density_mode=0, rho_const=1.225,
        P_runway=4000.0, P_beta=6.0 * DEG, P_chi=15.0 * DEG, P_vs=80.0, P_r=2500.0, P_h=300.0,
        alpha_dep=[0.4, 0.1, 0.25, 0.25],          # Table coeff
        alpha_arr=[0.25, 0.65, 0.1],               # heading, altitude, fuel (P:598-600 by meaning)
        noise_w=0.0, A_c=4000.0, centres=np.zeros((0, 3)),
        pop_nx=0, pop_ny=0, pop_x0=0.0, pop_y0=0.0, pop_dx=1000.0,
        wind_lo=[-30000.0, -30000.0, 0.0], wind_hi=[30000.0, 30000.0, 12000.0],
        wind_n=(2, 2, 2),             # grid points per axis; the paper uses 2x2x2
        sigma_lo=1.5, sigma_hi=4.0,
        beta_w=1.6e-6, gamma_w=1.5e-5, lambda_t=6.0e-6,   # P:451 (lambda read as s^-1)
        nominal=[0.0, 0.0], turb_sigma=0.0, tma_radius=30000.0,
    )


def _finish(scn: dict, ac: list) -> dict:
    n = len(ac)
    scn["n"] = n
    scn["kind"] = np.array([a["kind"] for a in ac], dtype=np.int32)
    scn["first_step"] = np.array([a.get("first_step", 0) for a in ac], dtype=np.int32)
    scn["x0"] = np.array([a["x0"] for a in ac], dtype=np.float64).reshape(n, 6)
    for k in ["theta_F", "z_tf", "v_D", "beta_f", "m_empty"]:
        scn[k] = np.array([a[k] for a in ac], dtype=np.float64)
    for k, v in A320.items():
        scn[k] = np.full(n, v, dtype=np.float64)
    return scn


def _arrival(rng, a: int, n_arr: int, H: int) -> dict:
    sec = ARR_SECTORS[a % 3]
    slot = a // 3
    per_sector = max(1, (n_arr + 2) // 3)
    frac = (slot + 0.5) / per_sector
    ang = (sec[0] + (sec[1] - sec[0]) * frac + rng.uniform(-2.0, 2.0)) * DEG
    r = 30000.0
    x, y = r * math.cos(ang), r * math.sin(ang)
    z = LAYERS[a % 4]
    v = rng.uniform(120.0, 140.0)
    chi = math.atan2(-y, -x) + rng.uniform(-15.0, 15.0) * DEG
    m0 = 64000.0
    return dict(kind=0, x0=[x, y, z, v, chi, m0], theta_F=0.0, z_tf=0.0, v_D=0.0,
                beta_f=3.0 * DEG, m_empty=m0 - 3800.0)


def _departure_snapshot(d: int) -> dict:
    th = DEP_BEARINGS[d % 6] * DEG
    r = 2000.0 + 3000.0 * d
    m0 = 73500.0
    return dict(kind=1, x0=[r * math.cos(th), r * math.sin(th), 400.0 + 700.0 * d, 100.0, th, m0],
                theta_F=th, z_tf=6000.0, v_D=150.0, beta_f=0.0, m_empty=58000.0)


def _departure_release(d: int) -> dict:
    th = DEP_BEARINGS[d % 6] * DEG
    m0 = 73500.0
    return dict(kind=1, x0=[-1500.0, 0.0, 400.0, 85.0, math.pi, m0],
                theta_F=th, z_tf=6000.0, v_D=150.0, beta_f=0.0, m_empty=58000.0)


def snapshot(n_arr: int, n_dep: int, seed: int, H: int = 6, dt: float = 10.0) -> dict:
    """All-active, initially separated snapshot."""
    rng = np.random.default_rng(seed)
    scn = base_scenario(H, dt)
    ac = [_arrival(rng, a, n_arr, H) for a in range(n_arr)]
    ac += [_departure_snapshot(d) for d in range(n_dep)]
    return _finish(scn, ac)


def population_centres(seed: int, n: int = 20) -> np.ndarray:
    """20 synthetic population centres (positions are figure-only):
    radius U[1.5, 4] km (P:1114 'greater than 1.5km'), uniform in the 3-40 km annulus."""
    rng = np.random.default_rng(seed)
    out = np.zeros((n, 3))
    for c in range(n):
        rad = math.sqrt(rng.uniform(3.0 ** 2, 40.0 ** 2)) * 1000.0
        ang = rng.uniform(-math.pi, math.pi)
        out[c] = [rad * math.cos(ang), rad * math.sin(ang), rng.uniform(1.5, 4.0) * 1000.0]
    return out


def config(num: int, noise_w: float = 0.1):
    """Return (scenario dict, SmcConfig) for BASELINE.json configs[num-1]."""
    seed = 1000 + num
    sig = (0.05 * (A320["T_max"] - A320["T_min"]), 2.0 * DEG, 0.5 * DEG)
    if num == 1:
        rng = np.random.default_rng(seed)
        scn = base_scenario(H=20, dt=10.0)
        ac = [_arrival(rng, 0, 1, 20), _departure_release(0)]
        scn = _finish(scn, ac)
        return scn, SmcConfig("c1", L=256, S=4, K=10, sigma=sig, seed=0x5EED0001)
    if num == 2:
        scn = snapshot(4, 4, seed)
        scn["nominal"] = [8.0, 0.0]
        scn["turb_sigma"] = 1.0
        return scn, SmcConfig("c2", L=16384, S=16, K=101, sigma=sig, seed=0x5EED0002)
    if num == 3:
        scn = snapshot(16, 8, seed)
        return scn, SmcConfig("c3", L=65536, S=32, K=101, sigma=sig, seed=0x5EED0003)
    if num == 4:
        scn = snapshot(6, 6, seed, dt=20.0)
        scn["noise_w"] = noise_w
        scn["centres"] = population_centres(seed)
        scn.update(pop_nx=81, pop_ny=81, pop_x0=-40000.0, pop_y0=-40000.0, pop_dx=1000.0)
        # one low-fuel-reserve arrival (R34): m0 = m_empty + 400 kg
        scn["x0"][0, 5] = scn["m_empty"][0] + 400.0
        return scn, SmcConfig("c4", L=32768, S=16, K=101, sigma=sig, seed=0x5EED0004)
    if num == 5:
        scn = snapshot(8, 8, seed)
        return scn, SmcConfig("c5", L=1 << 20, S=64, K=101, sigma=sig, seed=0x5EED0005)
    if num == 6:
        # Table 1's timing workload: 10 aircraft all active over the
        # whole H = 6 horizon, L = 10 240, paper Alg.1 (no MH, S_k = floor(3 + 5 e^{0.05k}),
        # J_max = 100).  Not a BASELINE.json config: a like-for-like latency line.
        scn = snapshot(5, 5, seed)
        return scn, SmcConfig("table1", L=10240, S=8, K=101, sigma=sig, mh=False, sched_paper=True,
                              seed=0x5EED0006)
    if num == 7:
        # BASELINE.json's latency target: a 20-aircraft MPC step (10 arrivals / 10 departures,
        # all active -- the paper's mixed traffic at its densest) with c2's solver,
        # against the 10 s re-planning interval.  Not a BASELINE.json config.
        scn = snapshot(10, 10, seed)
        scn["nominal"] = [8.0, 0.0]
        scn["turb_sigma"] = 1.0
        return scn, SmcConfig("n20", L=16384, S=16, K=101, sigma=sig, seed=0x5EED0007)
    raise ValueError(num)


def small(n_arr=2, n_dep=2, H=6, seed=7, **over):
    """Small parity scenario (several tiles, ragged lanes) with optional overrides."""
    scn = snapshot(n_arr, n_dep, seed, H=H)
    scn.update(over)
    return scn


def random_controls(scn: dict, L: int, seed: int, spread: float = 1.0) -> np.ndarray:
    """Seeded float32 control population [L][n][H][3] inside (or, with
    spread > 1, partly outside) the envelope -- a test input, not the method's init."""
    rng = np.random.default_rng(seed)
    n, H = scn["n"], scn["H"]
    out = np.zeros((L, n, H, 3), dtype=np.float32)
    for i in range(n):
        Tl, Th = scn["T_min"][i], scn["T_max"][i]
        mid, half = 0.5 * (Tl + Th), 0.5 * (Th - Tl) * spread
        out[:, i, :, 0] = rng.uniform(mid - half, mid + half, (L, H))
        out[:, i, :, 1] = rng.uniform(-1, 1, (L, H)) * scn["phi_max"][i] * spread
        out[:, i, :, 2] = rng.uniform(-1, 1, (L, H)) * scn["gamma_max"][i] * spread
    return out


def paper_mixed(seed: int = 2001) -> dict:
    """The paper's mixed closed-loop scenario shape: 10 arrivals + 10 departures
    (P:607-616), arrivals every 2 MPC steps, departures every 6."""
    return traffic(10, 10, seed, arr_every=2, dep_every=6)


def paper_congested(seed: int = 2002) -> dict:
    """The paper's congested shape: 24 arrivals, no departures."""
    return traffic(24, 0, seed, arr_every=2, dep_every=6)


def traffic(n_arr: int, n_dep: int, seed: int, arr_every: int = 2, dep_every: int = 6, jitter: int = 1) -> dict:
    """Arrival/departure stream for the rolling-window MPC loop:
    entries at fixed, evenly spread MPC steps with a small seeded jitter;
    arrivals enter on the TMA boundary, departures are released at the
    runway end at 400 m heading West."""
    rng = np.random.default_rng(seed)
    ac, entry = [], []
    for a in range(n_arr):
        ac.append(_arrival(rng, a, n_arr, 6))
        entry.append(arr_every * a + int(rng.integers(0, jitter + 1)))
    for d in range(n_dep):
        ac.append(_departure_release(d))
        entry.append(dep_every * d + 3)
    out = _finish({}, ac)
    out["entry"] = np.array(entry, np.int32)
    return out
