"""Algorithmic work model of the hot path, per pipe.

K2 (rollout + MH) has no dense contraction (no tensor cores) and reads ~12H
bytes of controls per (particle, candidate, aircraft) against S*H aircraft-
steps of arithmetic, so it is bound by the SM's compute pipes.  Its roofline
is the time the ALGORITHMIC operations -- counted from the equations of the
paper (Eq. hor, Eq. cov / AR(1), Eq. TO_init, the envelope, Eq. avoidance,
the utilities), not from SASS -- need on the busiest pipe:

    T_roof = max_p  ops_p x aircraft-steps / peak_p

with the pipe peaks MEASURED on the B200 (tools/micro/pipes.cu; run inside
bench.py, committed as profiles/r02_pipe_micro.jsonl), per SM per clock:

    fma  FFMA/FADD/FMUL (FFMA2 = 2 lane-ops)          124.5
         IMAD.WIDE.U32 occupies the same pipe at 4 FMA slots (FFMA +
         IMAD.WIDE + LOP3 1:1:1 runs at 74.3 ops/clk = 128 / (4 + 1) x 3)
    alu  LOP3, IADD3, FMNMX, FSETP, FSEL, SHF, I2F       63.8
    xu   MUFU ex2/lg2/sin/cos/rcp/rsqrt and FRND          16.0
    shfl                                                  31.9

A pipe count is the minimum the equations need: e.g. the trilinear
interpolation of the 2x2x2 field is counted in its 7-coefficient polynomial
form, the lower-triangular 8x8 factor as 36 FMA per component, atan2 as
its degree-15 odd polynomial on the MUFU reciprocal.  Work shared by several
aircraft-steps is divided among them: the wind field of a (particle, sample,
step) is shared by the N aircraft and, under common random numbers, by both
MH candidates; the airframe states z, v, chi, m of Eq. hor do not depend on
the wind (it enters only dx/dt, dy/dt), so their integration, the envelope
and the departures' altitude / speed terms are shared by the S samples of a
(particle, candidate, aircraft, step).

K4-K6 (scans, gather/propose) are HBM-bound; their algorithmic bytes per
(aircraft, particle) per round are 8 + 36 H.
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

SMS = 148
PIPES = ("fma", "alu", "xu", "shfl")
IMADW_FMA_SLOTS = 4.0

# measured per SM per clock (profiles/r02_pipe_micro.jsonl, B200, 1965 MHz)
DEFAULT_PEAK_PER_CLK = {"fma": 124.45, "alu": 63.78, "xu": 15.98, "shfl": 31.93}


def _v(fma=0.0, alu=0.0, xu=0.0, imadw=0.0, shfl=0.0):
    return np.array([fma, alu, xu, imadw, shfl], dtype=np.float64)


# --- airframe, per (particle, candidate, aircraft, step) -- shared by the S samples (Eq. hor, P:246-255;
# R12): rho(z): 1 FMA + max + lg2 + mul + ex2; q = c v^2 rho: 3; m g / q: rcp + 2; D = q (cd0 + cd2 (1 +
# tan^2) (mg/q)^2): 5; sin/cos chi + wrap (2 FMA, FRND); z, v, chi, m updates: 9 FMA + rcp m + rcp v; the
# air-relative ground velocity v cos g (cos chi, sin chi): 3; envelope and mass at the new state:
# 5 compares; the control bounds: 4 compares
AIRFRAME = _v(fma=2 + 3 + 2 + 5 + 2 + 9 + 3, alu=1 + 5 + 4, xu=2 + 1 + 2 + 1 + 2)
# --- ground track per aircraft-step (one sample, one candidate): x, y (wind added, 2 FMA each), fuel
TRACK = _v(fma=4 + 1)
# trilinear wind at the aircraft: 3 normalised coordinates, 4 shared products, 7 FMA per component,
# nominal + gust
WIND_INTERP = _v(fma=3 + 4 + 14 + 2)
# theta = atan2(y, x): rcp, 11 FMA (polynomial), max/min, 2 selects, sign
THETA = _v(fma=12, alu=5, xu=1)
# arrival: rho_h (rsqrt), arc s (rcp), beta = atan2(z, s) (right half-plane), heading wrap, landing sector
# (3 position compares per sample; speed and heading: 2 compares per airframe step), deviation D
# (chi_hat = pi + 2 theta, wrap) and E
ARR = _v(fma=2 + 1 + 2 + 10 + 1 + 2 + 2 + 2 + 1 + 2, alu=1 + 3 + 3 + 1, xu=1 + 1 + 1 + 1 + 1)
ARR_AIRFRAME = _v(alu=2)
# departure: A = |wrap(theta - theta_F)| per sample; B = |z_tf - z|, C = |v - v_D| per airframe step
# (a departure never lands: both are sample-independent)
DEP = _v(fma=4, xu=1)
DEP_AIRFRAME = _v(fma=4)
# noise (bilinear 1 km grid): q(z), cell index, 3 lerps, J_noise
NOISE = _v(fma=14, alu=11)
# one unordered pair of Eq. avoidance: dx dy dz d^2 (5), 2 compares + and + or, one exchange
PAIR = _v(fma=5, alu=4, shfl=1)
# --- per (particle, sample, step), shared by n aircraft x C candidates: the 2x2x2 field
# 4 Philox4x32-10 (20 IMAD.WIDE + 20 LOP3 + counter), 8 Box-Muller pairs (per pair: 2 SHF + 2 I2F, 2 FMA
# scale, lg2 + mul, rsqrt + mul, sin + cos (+2 range FMUL), 2 FMA), AR(1) 16 x (FMUL + FFMA), Qhat Z 2 x 36
WINDGEN = _v(fma=8 * 8 + 32 + 72, alu=4 * 21 + 8 * 4, xu=8 * 4, imadw=4 * 20)
# --- per (particle, sample, aircraft, 2 steps), shared by C candidates: gusts (R15)
GUST = _v(fma=2 * 8 + 2 * 2, alu=21 + 2 * 4, xu=2 * 4, imadw=20)
# --- per (particle, candidate, sample, aircraft): utility J_T, log2 and the weight
END = _v(fma=13, alu=8, xu=1)


def _pipes(v):
    """[fma, alu, xu, imadw, shfl] -> pipe loads {fma, alu, xu, shfl} (IMAD.WIDE on the FMA pipe)."""
    return {"fma": v[0] + IMADW_FMA_SLOTS * v[3], "alu": v[1], "xu": v[2], "shfl": v[4]}


def ops_vector(scn: dict, C: int, S: int = 16) -> np.ndarray:
    """Algorithmic ops per aircraft-step [fma, alu, xu, imadw, shfl] (all-active horizon)."""
    n, H = int(scn["n"]), int(scn["H"])
    f_arr = float((np.asarray(scn["kind"]) == 0).sum()) / n
    Sd = max(S, 1)
    v = TRACK + WIND_INTERP + THETA + AIRFRAME / Sd
    v = v + f_arr * (ARR + ARR_AIRFRAME / Sd) + (1 - f_arr) * (DEP + DEP_AIRFRAME / Sd)
    if float(scn["noise_w"]) > 0 and int(scn["pop_nx"]) > 0:
        v = v + NOISE
    v = v + PAIR * (n - 1) / 2.0
    G = int(np.prod(scn.get("wind_n", (2, 2, 2))))
    if G == 8:
        v = v + WINDGEN / (n * C)
    else:
        # dense grid (R48): ceil(2G/4) Philox calls, G Box-Muller pairs, 2G AR(1) updates,
        # Qhat Z over the lower triangle (2 x G(G+1)/2 FMA); per candidate step the grid cell (3
        # normalised coordinates, 3 floor/min) and the 7-lerp trilinear per component (28 FMA)
        nblk = (2 * G + 3) // 4
        gen = _v(fma=G * 8 + 2 * G * 2 + G * (G + 1), alu=nblk * 21 + G * 4, xu=G * 4, imadw=nblk * 20)
        v = v - WIND_INTERP + _v(fma=3 + 28 + 2, alu=9) + gen / (n * C)
    v = v + END / H
    if float(scn["turb_sigma"]) > 0:
        v = v + GUST / (2.0 * C)
    return v


def pipe_ops(scn: dict, C: int, S: int = 16) -> dict:
    return _pipes(ops_vector(scn, C, S))


def load_pipe_peaks(root: str, fresh: list | None = None) -> tuple:
    """Per-SM-per-clock pipe peaks: this run's microbenchmark lines if given, else the committed
    profiles/r02_pipe_micro.jsonl, else the defaults above.  Returns (peaks, source)."""
    lines, src = fresh, "measured in this run (tools/micro/pipes.cu)"
    if not lines:
        p = os.path.join(root, "profiles", "r02_pipe_micro.jsonl")
        try:
            lines = [json.loads(x) for x in open(p) if x.startswith("{")]
            src = "measured, profiles/r02_pipe_micro.jsonl"
        except Exception:
            return dict(DEFAULT_PEAK_PER_CLK), "defaults (measured values copied in roofline.py)"
    by = {d.get("op"): d.get("per_sm_per_clk") for d in lines if "op" in d}
    pk = dict(DEFAULT_PEAK_PER_CLK)
    if by.get("FFMA"):
        pk["fma"] = max(by["FFMA"], by.get("FFMA2") or 0.0)
    alu = [by[k] for k in ("LOP3", "IADD3", "FMNMX") if by.get(k)]
    if alu:
        pk["alu"] = min(alu)
    xu = [by[k] for k in ("MUFU.EX2", "MUFU.LG2", "MUFU.SIN", "MUFU.RSQ") if by.get(k)]
    if xu:
        pk["xu"] = min(xu)
    if by.get("SHFL"):
        pk["shfl"] = by["SHFL"]
    return pk, src


def k2_roofline(scn: dict, rounds: list, seconds: float, sm_mhz: float, peaks_per_clk: dict) -> dict:
    """rounds: [(aircraft-steps, C, S)] of the timed K2 launches; seconds: their measured time.
    Returns the per-pipe roofline times, the binding pipe and frac = T_roof / T_measured."""
    load = {p: 0.0 for p in PIPES}
    for steps, C, S in rounds:
        for p, v in pipe_ops(scn, C, S).items():
            load[p] += v * steps
    t = {p: load[p] / (peaks_per_clk[p] * SMS * sm_mhz * 1e6) for p in PIPES}
    bind = max(t, key=t.get)
    return {"t_pipe_s": t, "binding_pipe": bind, "t_roof_s": t[bind],
            "frac": t[bind] / seconds if seconds > 0 else None,
            "ops": load}


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


def round_list(scn: dict, L: int, S_list, mh: bool = True, L_final: int = 0) -> list:
    """[(aircraft-steps, C, S)] per round of one MPC step."""
    Ha = int(sum(int(scn["H"]) - int(e) for e in scn["first_step"]))
    K = len(S_list)
    out = []
    for k, S in enumerate(S_list):
        C = 1 if (k == 0 or not mh) else 2
        out.append((particles_of(L, L_final, K, k) * C * S * Ha, C, S))
    return out


def resample_bytes(n: int, L: int, H: int) -> int:
    """Algorithmic HBM bytes of one reduce + resample + propose phase."""
    return n * L * (8 + 36 * H)
