"""Algorithmic work model of the hot path.

K2 (rollout + MH) is bound by the FP32 / integer / MUFU pipes -- there is no
dense contraction (no tensor cores) and its HBM traffic is ~12H bytes per
(particle, candidate, aircraft) against S*H aircraft-steps of arithmetic.
Its roofline is therefore an ALU roofline: the ALGORITHMIC operation count
per aircraft-step, counted from the equations (not from SASS), expressed in
FP32-lane-equivalent operations, against the SM array's FP32 lane rate.

One MUFU (transcendental: sin, cos, lg2, ex2, rcp, rsqrt) counts as 8 FP32
lane-ops, the ratio of the FP32 (128/clk/SM) to the MUFU (16/clk/SM) pipe.

K4-K6 (reduce, scans, gather/propose) are HBM-bound; their algorithmic
bytes per (aircraft, particle) per round are 8 + 36 H.
"""
from __future__ import annotations

import math

import numpy as np

MUFU_W = 8.0          # FP32-lane-op equivalent of one MUFU op
SMS = 148
FP32_LANES_PER_SM_CLK = 128

# --- per aircraft-step, per candidate (counted from Eq. hor, Eq. TO_init)
DYN_FP, DYN_MUFU = 30, 7          # rho(z) ISA, q, C_L, D, sin/cos chi, 6 state updates, fuel
WIND_INTERP_FP = 37               # clamp/normalise 3 coords, 2 x trilinear (7 lerps)
CHECKS = 10                       # envelope, mass, finiteness
THETA_FP, THETA_MUFU = 12, 1      # atan2(y, x)
DEP_FP = 8                        # A, B, C deviations
ARR_FP, ARR_MUFU = 32, 4          # rho_h, arc s, beta = atan2, landing test, D, E
NOISE_FP = 20                     # bilinear popdense, J_noise
PAIR_OPS = 7                      # one unordered pair: dx dy dz, d^2, 2 compares, and
# --- per (particle, sample, step): the shared 2x2x2 wind field
WINDGEN_INT = 4 * 10 * 8          # 4 Philox4x32-10 calls
WINDGEN_FP, WINDGEN_MUFU = 48 + 32 + 72, 32   # Box-Muller x8, AR(1) x16, Qhat Z (2 x 36 FMA)
# --- per (particle, candidate, sample, aircraft): horizon-end utility and weight
END_FP, END_MUFU = 20, 1
# --- per (particle, sample, aircraft, 2 steps): gusts (R15)
GUST_INT, GUST_FP, GUST_MUFU = 80, 12, 8


def ops_per_aircraft_step(scn: dict, C: int) -> float:
    """FP32-lane-equivalent algorithmic ops per aircraft-step (all-active horizon)."""
    n, H = int(scn["n"]), int(scn["H"])
    n_arr = int((scn["kind"] == 0).sum())
    f_arr = n_arr / n
    per = DYN_FP + MUFU_W * DYN_MUFU + WIND_INTERP_FP + CHECKS + THETA_FP + MUFU_W * THETA_MUFU
    per += (1 - f_arr) * DEP_FP + f_arr * (ARR_FP + MUFU_W * ARR_MUFU)
    if float(scn["noise_w"]) > 0 and int(scn["pop_nx"]) > 0:
        per += NOISE_FP
    per += PAIR_OPS * (n - 1) / 2.0
    G = int(np.prod(scn.get("wind_n", (2, 2, 2)))) if "wind_n" in scn else 8
    if G == 8:
        per += (WINDGEN_INT + WINDGEN_FP + MUFU_W * WINDGEN_MUFU) / (n * C)
    else:
        # dense grid: ceil(2G/4) Philox calls, G Box-Muller pairs (6 FP + 4 MUFU each),
        # 2G AR(1) updates (2 FP), W = Qhat Z over the lower triangle (2 x G(G+1)/2 FMA = 2 ops),
        # plus the cell index per candidate step (9 FP)
        nblk = (2 * G + 3) // 4
        gen = nblk * 80 + G * 6 + MUFU_W * G * 4 + 2 * G * 2 + 2 * G * (G + 1)
        per += gen / (n * C) + 9
    per += (END_FP + MUFU_W * END_MUFU) / H
    if float(scn["turb_sigma"]) > 0:
        per += (GUST_INT + GUST_FP + MUFU_W * GUST_MUFU) / (2.0 * C)
    return per


def sample_schedule(k: int) -> int:
    """S_k of SMC_SCHED_PAPER: floor(3 + 5 e^{0.05 k}), as the library counts it."""
    return int(math.floor(3.0 + 5.0 * math.exp(0.05 * k)))


def samples_list(cfg) -> list:
    return [sample_schedule(k) for k in range(cfg.K)] if cfg.sched_paper else [cfg.S] * cfg.K


def particles_of(L: int, L_final: int, K: int, k: int) -> int:
    """Particle count of round k (smc_config.n_particles_final, include/smcatm.h)."""
    if not L_final or L_final >= L or K < 2:
        return L
    return L - ((L - L_final) * min(k, K - 1)) // (K - 1)


def aircraft_steps(scn: dict, L: int, S_list, mh: bool = True, L_final: int = 0) -> int:
    """L_k * C_k * S_k * sum_i H_a,i summed over rounds (C_0 = 1, C_k = 2 with MH)."""
    Ha = int(sum(int(scn["H"]) - int(e) for e in scn["first_step"]))
    tot = 0
    K = len(S_list)
    for k, S in enumerate(S_list):
        C = 1 if (k == 0 or not mh) else 2
        tot += particles_of(L, L_final, K, k) * C * S * Ha
    return tot


def peak_alu_ops(sm_mhz: float) -> float:
    """FP32 lane-ops per second of the SM array at sm_mhz."""
    return SMS * FP32_LANES_PER_SM_CLK * sm_mhz * 1e6


def resample_bytes(n: int, L: int, H: int) -> int:
    """Algorithmic HBM bytes of one reduce + resample + propose phase."""
    return n * L * (8 + 36 * H)
