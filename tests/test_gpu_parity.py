"""GPU (libsmcatm, sm_100a) vs FP64 oracle parity, through the C ABI.

Tolerances (SURVEY 8(c) parity metric): rollout
quantities |gpu - ora| <= 1e-4 |ora| + atol (positions 0.1 m, speed 1e-3 m/s,
heading 1e-4 rad, mass/fuel 1e-2 kg, utilities 1e-4); log2 weights, element
by element, |d ell| <= 1e-4 (|ell| + S); MH decisions, ancestors, integer
totals, selection: bit-exact.

Discrete decisions (violation, landing) are compared exactly.  The oracle
reports a conjunction-aware margin for each (R30); where it is below
EPS = 1e-5 FP32 and FP64 may legitimately take either side, so:
  * rollouts dumped by the debug hook are re-run by the oracle in decision-
    replay mode (it takes the GPU's decision only for those events) and every
    continuous quantity is then compared;
  * production launches (weights only) exclude the (particle, aircraft)
    entries whose margin is below EPS.
Replayed decisions and excluded entries are counted (parity_log, printed in
the pytest summary) and must stay below 1e-3 of the units compared.
"""
import math

import numpy as np
import pytest

import oracle as O
import parity_log
from paper_1506_02869_b200 import scenarios as sc

pytestmark = pytest.mark.gpu

EPS = 1e-5
RATE = 1e-3            # bound on replayed / excluded units


@pytest.fixture(scope="module")
def smc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_02869_b200 import smcatm
    smcatm.load()
    return smcatm


def _solver(smc, scn, L=64, S=4, K=3, seed=0x5EED0001, **kw):
    sig = (0.05 * 1.2e5, 2 * math.pi / 180, 0.5 * math.pi / 180)
    return smc.Solver(scn, L=L, S=S, K=K, sigma=sig, seed=seed, **kw)


def _in_domain(traj):
    """[n][H+1] mask: steps up to which the oracle state stays where FP32 and FP64
    evaluate Eq. hor alike (finite, airspeed above 20 m/s -- the turn rate g tan(phi)/v
    and the induced drag blow up as v -> 0, P:250-255 -- and inside 1000 km)."""
    v = traj[..., 3]
    ok = np.isfinite(traj).all(-1) & (v > 20.0) & (np.abs(traj[..., :3]) < 1e6).all(-1)
    return np.logical_and.accumulate(ok, axis=1)


def _compare_rollouts(smc, scn, L, S, k, seed, ctrl, l0=0, name=None):
    """Per-(particle, sample, aircraft) states, fuel, utilities and decisions of the
    debug rollout vs the oracle run in decision-replay mode (R30)."""
    sol = _solver(smc, scn, L=max(L, 1), S=S, seed=seed)
    P = O.Problem(scn)
    g = sol.debug_rollout(ctrl, S, k, l0=l0, traj=True)
    n = scn["n"]
    replayed = units = 0
    tol = np.array([0.1, 0.1, 0.1, 1e-3, 1e-4, 1e-2])
    for l in range(L):
        for s in range(S):
            r = P.rollout(ctrl[l].astype(np.float64), l0 + l, s, k, seed,
                          replay=(g["landed"][l, s], g["viol"][l, s].astype(np.int32), EPS))
            units += n
            replayed += int(np.count_nonzero(r["replayed"]))
            assert np.array_equal(g["viol"][l, s].astype(bool), r["viol"].astype(bool)), (l, s, r["margin"])
            assert np.array_equal(g["landed"][l, s], r["landed_step"]), (l, s)
            tg, to = g["traj"][l, s].astype(np.float64), r["traj"]
            dom = _in_domain(to)
            dif = np.abs(tg - to)
            # the GPU keeps the heading wrapped to [-pi, pi], the oracle does not (R32): compare modulo 2 pi
            dif[..., 4] = np.abs(np.remainder(tg[..., 4] - to[..., 4] + np.pi, 2 * np.pi) - np.pi)
            err = dif - (1e-4 * np.abs(np.where(np.arange(6) == 4, np.pi, to)) + tol)
            err[~dom] = -1.0
            assert np.all(err <= 0), (l, s, np.unravel_index(np.argmax(err), err.shape), tg, to)
            full = dom.all(1)                      # aircraft whose whole rollout stayed in the domain
            assert np.allclose(g["fuel"][l, s][full], r["fuel"][full], rtol=1e-4, atol=1e-2), (l, s)
            assert np.allclose(g["J"][l, s][full], r["J"][full], rtol=0, atol=1e-4), (l, s, g["J"][l, s], r["J"])
            assert np.allclose(g["comp"][l, s][full], r["comp"][full], rtol=0, atol=1e-4), (l, s)
    parity_log.record(name or f"rollout n={n}", units, replayed=replayed)
    assert replayed <= RATE * units, (replayed, units)
    sol.close()
    return units, replayed


def _check_ell(ell_g, ell_o, margin, S, name, lam_g=None):
    """Element-by-element log2 weights: finiteness exact and |d ell| <= 1e-4 (|ell| + S)
    wherever the oracle's decision margin is at least EPS; the rest is excluded and
    counted.  lam_g (optional): the GPU's lambda per particle, checked against the
    oracle's sum over aircraft where no entry of the particle is excluded."""
    ell_g = np.asarray(ell_g, np.float64)
    amb = margin < EPS
    ok = ~amb
    fin_g, fin_o = np.isfinite(ell_g), np.isfinite(ell_o)
    bad = ok & (fin_g != fin_o)
    assert not bad.any(), (name, np.argwhere(bad)[:5], ell_g[bad][:5], ell_o[bad][:5], margin[bad][:5])
    both = ok & fin_g & fin_o
    err = np.abs(ell_g - ell_o) - 1e-4 * (np.abs(ell_o) + S)
    err[~both] = -1.0
    assert np.all(err <= 0), (name, np.unravel_index(np.argmax(err), err.shape), err.max())
    if lam_g is not None:
        rows = ~amb.any(1)
        lam_o = np.where(fin_o.all(1), np.where(fin_o, ell_o, 0.0).sum(1), -np.inf)
        lg = np.asarray(lam_g)[rows]
        lo = lam_o[rows]
        assert np.array_equal(np.isfinite(lg), np.isfinite(lo)), name
        f = np.isfinite(lo)
        n = ell_o.shape[1]
        assert np.all(np.abs(lg[f] - lo[f]) <= 1e-4 * (np.abs(lo[f]) + n * S)), name
    parity_log.record(name, ell_o.size, excluded=int(amb.sum()))
    assert amb.sum() <= RATE * ell_o.size + 0, (name, int(amb.sum()), ell_o.size)


def _near_trim_controls(scn, L, seed):
    """Float32 controls near trim with noise: mostly feasible, some violations."""
    rng = np.random.default_rng(seed)
    n, H = scn["n"], scn["H"]
    c = np.zeros((L, n, H, 3), np.float32)
    c[..., 0] = rng.uniform(20000, 70000, (L, n, H))
    c[..., 1] = rng.uniform(-0.45, 0.45, (L, n, H))
    c[..., 2] = rng.uniform(-0.08, 0.08, (L, n, H))
    return c


def _ring_scenario(n):
    """All-active snapshot of n aircraft (half arrivals): every separation-ring
    instance R in {6, 10, 12, 14, 20, 24, 28} of K2 is reached by some n."""
    scn = sc.snapshot((n + 1) // 2, n // 2, seed=40 + n)
    scn["nominal"] = [5.0, -3.0]
    scn["turb_sigma"] = 1.0
    return scn


ROLLOUT_CASES = ["c1", "c2", "n3_partial", "n12_noise", "n24", "n1", "n6", "n14", "n20", "n28", "dense332_n3",
                 "dense444_c2", "dense442_n1", "dense_n20"]


def _rollout_case(case):
    if case == "c1":
        scn, cfg = sc.config(1)
        return scn, 400, 4, cfg.seed
    if case == "c2":
        scn, cfg = sc.config(2)
        return scn, 300, 4, cfg.seed
    if case == "n3_partial":
        scn = sc.small(2, 1, H=7, seed=5)
        scn["first_step"] = np.array([0, 3, 7], np.int32)
        return scn, 400, 3, 99
    if case == "n12_noise":
        scn, cfg = sc.config(4, noise_w=0.2)
        return scn, 200, 2, cfg.seed
    if case == "n24":
        scn, cfg = sc.config(3)
        return scn, 60, 2, cfg.seed
    if case in ("n6", "n14", "n28"):
        n = int(case[1:])
        return _ring_scenario(n), max(40, 1200 // n), 2, 0x5EED0100 + n
    if case == "n20":                       # the 20-aircraft latency config (--config 7, R = 20)
        scn, cfg = sc.config(7)
        return scn, 60, 2, cfg.seed
    if case == "dense332_n3":               # denser wind grids (N3): 18 points, W = 4
        scn = sc.small(2, 1, H=7, seed=5)
        scn.update(wind_n=(3, 3, 2), sigma_lo=3.0, sigma_hi=6.0)
        return scn, 300, 3, 99
    if case == "dense444_c2":               # 64 points, W = 8
        scn, cfg = sc.config(2)
        scn.update(wind_n=(4, 4, 4), sigma_lo=3.0, sigma_hi=6.0)
        return scn, 150, 3, cfg.seed
    if case == "dense442_n1":               # one aircraft: segment padded to W = 4
        scn = sc.small(1, 0, H=6, seed=3)
        scn.update(wind_n=(4, 4, 2), sigma_lo=3.0, sigma_hi=6.0)
        return scn, 1000, 2, 5
    if case == "dense_n20":                 # 5x3x2 grid, 20 aircraft (W = 32)
        scn = sc.snapshot(12, 8, seed=21)
        scn.update(wind_n=(5, 3, 2), sigma_lo=3.0, sigma_hi=6.0)
        return scn, 60, 2, 31
    scn = sc.small(1, 0, H=6, seed=3)       # n1
    return scn, 1000, 2, 5


@pytest.mark.parametrize("case", ROLLOUT_CASES)
def test_rollout_parity(smc, case):
    scn, L, S, seed = _rollout_case(case)
    ctrl = _near_trim_controls(scn, L, seed=11)
    _compare_rollouts(smc, scn, L, S, k=2, seed=seed, ctrl=ctrl, l0=1000, name=f"rollout {case}")


def test_rollout_landing_exercised(smc):
    """Arrivals set up to land mid-horizon (near-trimmed 3 deg descent along the
    runway axis): landing step and frozen state agree with the oracle."""
    scn = sc.small(1, 1, H=8, seed=2)
    DEG = math.pi / 180
    scn["x0"][0] = [7000.0, 300.0, 7000 * math.tan(3 * DEG), 76.0, math.pi, 64000.0]
    scn["x0"][1] = [-20000.0, -20000.0, 5000.0, 140.0, -2.3, 70000.0]
    P = O.Problem(scn)
    rng = np.random.default_rng(1)
    L = 256
    ctrl = np.zeros((L, 2, 8, 3), np.float32)
    for l in range(L):
        st = scn["x0"][0].copy()
        for t in range(8):
            _, D = P.lift_drag(0, st, 0.0)
            g = -3 * DEG + rng.uniform(-0.005, 0.005)
            ctrl[l, 0, t] = [D + st[5] * 9.81 * math.sin(g) + rng.uniform(-2000, 2000), rng.uniform(-0.01, 0.01), g]
            st = P.step(0, st, ctrl[l, 0, t].astype(np.float64))
    ctrl[:, 1, :, 0] = 50000.0
    landed_o = sum(P.rollout(ctrl[l].astype(np.float64), l, 0, 0, 7)["landed_step"][0] > 0 for l in range(L))
    assert landed_o > L // 4
    _compare_rollouts(smc, scn, L, 4, k=0, seed=7, ctrl=ctrl, name="rollout landing")


@pytest.mark.parametrize("two", [False, True])
def test_landing_hoisted_parity(smc, two):
    """An arrival set up to land in the first step of an 8-step horizon (a near-trimmed 3 deg
    descent along the runway axis, every landing condition met with a margin) among 6 aircraft,
    through the production kernels that integrate the airframe
    once per particle: the landing sector's speed / heading conditions come from the airframe
    pass, the position conditions per sample, and a landed sample stops accumulating -- weights
    element by element against the oracle (single-candidate kernel, or two=True the two-chain
    kernel)."""
    scn = sc.small(3, 3, H=8, seed=2)
    DEG = math.pi / 180
    # 4.5 km out on the axis: the 4 km circle is crossed with a margin in the first step
    scn["x0"][0] = [4500.0, 150.0, 4500.0 * math.tan(3 * DEG), 76.0, math.pi, 64000.0]
    scn["first_step"] = np.array([0, 0, 0, 8, 0, 0], np.int32)     # the departure on the runway never enters
    P = O.Problem(scn)
    rng = np.random.default_rng(11)
    L, H = 384, 8
    ctrl = _near_trim_controls(scn, L, seed=11)
    for a in range(1):
        for l in range(L):
            st = scn["x0"][a].copy()
            for t in range(H):
                _, D = P.lift_drag(a, st, 0.0)
                g = -3 * DEG + rng.uniform(-0.005, 0.005)
                ctrl[l, a, t] = [D + st[5] * 9.81 * math.sin(g) + rng.uniform(-2000, 2000), rng.uniform(-0.01, 0.01), g]
                st = P.step(a, st, ctrl[l, a, t].astype(np.float64))
    landed = sum(int(P.rollout(ctrl[l].astype(np.float64), l, 0, 4, 7)["landed_step"][0] > 0) for l in range(0, L, 8))
    assert landed > L // 16                                      # landings happen in the sample
    S = 5
    sol = _solver(smc, scn, L=L, S=S, seed=7)
    ell_g = sol.debug_evaluate(ctrl, S, 4, two=two).astype(np.float64)
    ell_o, mg = P.evaluate(ctrl.astype(np.float64), S, 4, 7, margin=True)
    _check_ell(ell_g, ell_o, mg, S, f"landing hoisted two={two}")
    sol.close()


def test_violator_keeps_flying_on_gpu(smc):
    """Alg.1 l.11-13 / Eq. avoidance on the GPU: an aircraft
    that breaks its envelope at step 0 keeps flying and, at step 2, conflicts with a
    neighbour that broke nothing -- both are zeroed, as in the oracle's pin
    (test_oracle_conventions.test_violator_keeps_flying_and_zeroes_a_later_neighbour)."""
    scn = sc.snapshot(0, 2, seed=1)
    scn.update(sigma_lo=0.0, sigma_hi=0.0, nominal=[0.0, 0.0], turb_sigma=0.0)
    scn["x0"][0] = [-8000.0, 0.0, 3000.0, 100.0, 0.0, 73500.0]
    scn["x0"][1] = [0.0, 0.0, 3000.0, 100.0, math.pi, 73500.0]
    P = O.Problem(scn)
    u = np.zeros((1, 2, scn["H"], 3), np.float32)
    for i in range(2):
        st = scn["x0"][i].copy()
        for t in range(scn["H"]):
            _, D = P.lift_drag(i, st, 0.0)
            u[0, i, t] = [D, 0.0, 0.0]
            st = P.step(i, st, u[0, i, t].astype(np.float64))
    u[0, 1, 0, 0] = 1.5 * scn["T_max"][1]
    sol = _solver(smc, scn, L=1, S=1, seed=3)
    g = sol.debug_rollout(u, 1, 0, traj=True)
    r = P.rollout(u[0].astype(np.float64), 0, 0, 0, 3)
    assert g["viol"][0, 0].tolist() == [1, 1] and r["viol"].tolist() == [1, 1]
    gt, ot = g["traj"][0, 0].astype(np.float64), r["traj"]
    keep = [0, 1, 2, 3, 5]
    assert np.allclose(gt[..., keep], ot[..., keep], rtol=1e-5, atol=0.1)
    dchi = np.remainder(gt[..., 4] - ot[..., 4] + np.pi, 2 * np.pi) - np.pi  # heading modulo 2 pi (R32)
    assert np.all(np.abs(dchi) < 1e-4)
    assert g["traj"][0, 0, 1, -1, 0] < g["traj"][0, 0, 1, 1, 0] - 4000.0       # the violator kept flying West
    sol.close()


@pytest.mark.parametrize("case,sp", [("c2", "1"), ("c2", "0"), ("table1", "1"), ("n24", "1"), ("n12_noise", "1"),
                                     ("n24", "0"), ("n6", "1"), ("n14", "1"), ("n20", "1"), ("n28", "1"),
                                     ("n28", "0"), ("c2", "2"), ("table1", "2"), ("n6", "2"), ("n12_noise", "2"),
                                     ("n14", "2"), ("n20", "2"), ("n24", "2"), ("n28", "2"), ("n9_partial", "1"),
                                     ("n9_partial", "2"), ("n9_h20", "1"), ("n9_h20", "2"), ("n9_h32", "1"),
                                     ("n9_h32", "2")])
def test_evaluate_parity(smc, case, sp, monkeypatch):
    """Evaluation of caller controls in the production K2 instances against the oracle,
    element by element: single candidate (round 0 / paper mode) with sample pairs in the
    float2 slots (SMC_K2_SP, default) or one sample per lane, or (sp = "2") the two-candidate
    two-chain kernel with both candidates = the controls; S odd (last pair half used), and
    every separation-ring instance (n = 6, 10, 12, 14, 20, 24, 28)."""
    monkeypatch.setenv("SMC_K2_SP", "1" if sp == "2" else sp)
    if case == "table1":
        scn, cfg = sc.config(6)
        seed = cfg.seed
    elif case == "n24":
        scn, cfg = sc.config(3)
        seed = cfg.seed
    elif case == "n12_noise":
        scn, cfg = sc.config(4, noise_w=0.2)
        seed = cfg.seed
    elif case == "n20":
        scn, cfg = sc.config(7)
        seed = cfg.seed
    elif case in ("n6", "n14", "n28"):
        scn = _ring_scenario(int(case[1:]))
        seed = 0x5EED0200 + int(case[1:])
    elif case in ("n9_h20", "n9_h32"):
        # long horizons (H <= 32, include/smcatm.h): beyond the two-chain kernel's 2 H <= 32 flag
        # bits two-candidate launches take the one-chain kernel; H = 32 fills the sample-pair
        # kernel's flag word
        scn = _ring_scenario(9)
        scn["H"] = int(case[4:])
        seed = 0x5EED0300 + scn["H"]
    elif case == "n9_partial":
        # aircraft entering the horizon late (simulated from their first step): the
        # once-per-particle airframe pass must hold their state until then
        scn = _ring_scenario(9)
        scn["H"] = 8
        scn["first_step"] = np.array([0, 3, 0, 7, 1, 0, 5, 2, 8], np.int32)
        seed = 0x5EED0209
    else:
        scn, cfg = sc.config(2)
        seed = cfg.seed
    n = scn["n"]
    S = 5
    L = max(64, 12000 // (n * S))
    ctrl = _near_trim_controls(scn, L, seed=3)
    sol = _solver(smc, scn, L=L, S=S, seed=seed)
    ell_g = sol.debug_evaluate(ctrl, S, 4, two=sp == "2").astype(np.float64)
    ell_o, mg = O.Problem(scn).evaluate(ctrl.astype(np.float64), S, 4, seed, margin=True)
    _check_ell(ell_g, ell_o, mg, S, f"evaluate {case} sp={sp}")
    sol.close()


@pytest.mark.parametrize("two", [False, True])
def test_stalled_airframe_parity(smc, two):
    """An aircraft that leaves the model's domain: thrust 0 and a climb beyond gamma_max at dt = 20 s
    (c4) drive v through 0 within the horizon.  The oracle propagates the state literally (P:250,
    R42's replacement: violated aircraft keep flying); with gamma = 0.6 the FP32 state overflows and
    K2's once-per-particle airframe replaces it by a far-away sentinel (no conflict, envelope failed),
    with the legal maximum climb it stays finite with v < 0 on both sides.  The stalled aircraft is
    infeasible on both sides and every other aircraft's weight matches the oracle's (no spurious or
    missed conflict).  two: through the two-candidate kernel (both candidates = the controls)."""
    scn, cfg = sc.config(4, noise_w=0.0)
    n, H = scn["n"], scn["H"]
    L, S = 512, 5
    ctrl = _near_trim_controls(scn, L, seed=5)
    stall = np.arange(L) % 4 == 0
    ctrl[stall, 0, :, 0] = 0.0
    ctrl[stall, 0, :, 2] = np.where(np.arange(L)[stall, None] % 8 == 0, 0.6, float(scn["gamma_max"][0]))
    P = O.Problem(scn)
    r6 = P.rollout(ctrl[0].astype(np.float64), 0, 0, 4, cfg.seed)
    r1 = P.rollout(ctrl[4].astype(np.float64), 4, 0, 4, cfg.seed)
    assert np.abs(r6["traj"][0, -1, 3]) > 1e38 and r1["traj"][0, -1, 3] < 0.0     # overflow / reversed flight
    sol = _solver(smc, scn, L=L, S=S, seed=cfg.seed)
    ell_g = sol.debug_evaluate(ctrl, S, 4, two=two).astype(np.float64)
    ell_o, mg = P.evaluate(ctrl.astype(np.float64), S, 4, cfg.seed, margin=True)
    assert not np.isfinite(ell_o[stall, 0]).any() and not np.isfinite(ell_g[stall, 0]).any()
    _check_ell(ell_g, ell_o, mg, S, f"stalled airframe two={two}")
    sol.close()


@pytest.mark.parametrize("case", ["c1", "c2", "n6", "n12_noise", "n12_noise_rect", "n12_noise_big", "n14", "n16", "n20",
                                  "n24", "n28"])
def test_production_rounds_parity(smc, case):
    """Real SMC rounds through smc_iterate -- round 0 (single candidate, sample pairs)
    and rounds 1-2 (both MH candidates, packed FP32) -- on every separation-ring
    instance: each candidate's log2 weight per (particle, aircraft) against the oracle
    evaluating the GPU's own controls, lambda of both candidates, the survivor's weights
    (the candidate its mask bit names) and the MH decisions replayed bit-exactly on the
    GPU's lambdas."""
    if case in ("n6", "n14", "n28"):
        scn = _ring_scenario(int(case[1:]))
        seed = 0x5EED0300 + int(case[1:])
    elif case == "n16":
        scn, cfg = sc.config(5)
        seed = cfg.seed
    elif case == "n20":
        scn, cfg = sc.config(7)
        seed = cfg.seed
    elif case == "n24":
        scn, cfg = sc.config(3)
        seed = cfg.seed
    elif case.startswith("n12_noise"):
        scn, cfg = sc.config(4, noise_w=0.2)
        seed = cfg.seed
        if case == "n12_noise_rect":
            # 13 x 7 grid over part of the airspace: row stride != column count, most aircraft
            # clamped to an edge (the two-chain kernel's padded shared-memory grid)
            scn.update(pop_nx=13, pop_ny=7, pop_x0=-15000.0, pop_y0=-9000.0, pop_dx=2500.0)
        elif case == "n12_noise_big":
            # 121 x 121 grid: larger than the shared-memory staging limit (read from global)
            scn.update(pop_nx=121, pop_ny=121, pop_x0=-42000.0, pop_y0=-42000.0, pop_dx=700.0)
    else:
        scn, cfg = sc.config(int(case[1:]))
        seed = cfg.seed
    n = scn["n"]
    S = 4
    L = max(128, 16000 // (n * S * 2))
    sol = _solver(smc, scn, L=L, S=S, K=4, seed=seed)
    P = O.Problem(scn)
    for k in range(3):
        sol.iterate(1)
        pop = sol.population()
        ell_c, mg_c = P.evaluate(pop["cur"].astype(np.float64), S, k, seed, margin=True)
        if k == 0:
            _check_ell(pop["ell"].T, ell_c, mg_c, S, f"rounds {case} k=0", lam_g=pop["lam"])
            continue
        ell_p, mg_p = P.evaluate(pop["prop"].astype(np.float64), S, k, seed, margin=True)
        lc_g, lp_g = pop["lam_cand"]
        acc = np.array([O.mh_accept(lc_g[l], lp_g[l], l, k, seed) for l in range(L)])
        assert np.array_equal(pop["surv"].astype(bool), acc), case            # MH bit-exact on the GPU's lambdas
        sv = pop["surv"][:, None] == 1
        ell_o = np.where(sv, ell_p, ell_c)
        mg = np.where(sv, mg_p, mg_c)
        # both candidates' lambdas: checked through particles with no excluded entry
        rows_c, rows_p = ~(mg_c < EPS).any(1), ~(mg_p < EPS).any(1)
        for lg, eo, rows in ((lc_g, ell_c, rows_c), (lp_g, ell_p, rows_p)):
            lo = np.where(np.isfinite(eo).all(1), np.where(np.isfinite(eo), eo, 0).sum(1), -np.inf)
            assert np.array_equal(np.isfinite(lg[rows]), np.isfinite(lo[rows])), (case, k)
            f = rows & np.isfinite(lo)
            assert np.all(np.abs(lg[f] - lo[f]) <= 1e-4 * (np.abs(lo[f]) + n * S)), (case, k)
        _check_ell(pop["ell"].T, ell_o, mg, S, f"rounds {case} k={k}", lam_g=pop["lam"])
    sol.close()


def test_mh_bitexact(smc):
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, seed=cfg.seed)
    rng = np.random.default_rng(5)
    L = 20000
    lc = rng.uniform(-80, -10, L)
    d = np.concatenate([rng.uniform(-30, 2, L // 2), rng.normal(0, 1e-9, L // 4), rng.uniform(-1100, -1000, L - L // 2 - L // 4)])
    lp = lc + d
    lc[rng.uniform(size=L) < 0.05] = -np.inf
    lp[rng.uniform(size=L) < 0.05] = -np.inf
    for k in (1, 7, 100):
        acc = sol.debug_mh(lc, lp, k)
        ref = np.array([O.mh_accept(lc[l], lp[l], l, k, cfg.seed) for l in range(L)], np.uint8)
        assert np.array_equal(acc, ref)


def test_mh_aircraft_bitexact(smc):
    """Per-aircraft MH decisions (R46) of the production device function vs the oracle."""
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, seed=cfg.seed)
    rng = np.random.default_rng(6)
    L, N = 6000, 7
    ec = rng.uniform(-40, -2, (L, N)).astype(np.float32)
    ep = (ec + np.concatenate([rng.uniform(-8, 1, (L // 2, N)), rng.normal(0, 1e-6, (L - L // 2, N))])).astype(np.float32)
    ec[rng.uniform(size=(L, N)) < 0.05] = -np.inf
    ep[rng.uniform(size=(L, N)) < 0.05] = -np.inf
    for k in (1, 9):
        mask = sol.debug_mh_aircraft(ec, ep, k)
        for l in range(0, L, 3):
            ref = sum(O.mh_accept_aircraft(float(ec[l, i]), float(ep[l, i]), l, i, k, cfg.seed) << i for i in range(N))
            assert mask[l] == ref, (l, k)


def test_per_aircraft_mh_rounds(smc):
    """mh = 2 (R46) in real rounds: every survivor row is the candidate its mask bit names,
    its log-weight is the oracle's for that candidate (element by element), the decisions
    replay bit-exactly on the GPU's candidate weights, and the final pick is the best
    jointly evaluated candidate."""
    scn, cfg = sc.config(2)
    L, S, K = 512, 3, 4
    sol = _solver(smc, scn, L=L, S=S, K=K, seed=cfg.seed, mh=2)
    P = O.Problem(scn)
    n = scn["n"]
    sol.iterate(1)
    for k in range(1, K):
        sol.iterate(1)
        pop = sol.population()
        mask = pop["surv_mask"]
        ell_c, mg_c = P.evaluate(pop["cur"].astype(np.float64), S, k, cfg.seed, margin=True)
        ell_p, mg_p = P.evaluate(pop["prop"].astype(np.float64), S, k, cfg.seed, margin=True)
        bits = ((mask[:, None] >> np.arange(n)[None, :]) & 1).astype(bool)
        ell_o = np.where(bits, ell_p, ell_c)
        mg = np.where(bits, mg_p, mg_c)
        ell_g = pop["ell"].T.astype(np.float64)
        _check_ell(ell_g, ell_o, mg, S, f"per-aircraft MH k={k}")
        assert np.allclose(pop["lam"], np.where(np.isfinite(ell_g).all(1), ell_g.sum(1), -np.inf), rtol=1e-12)
        # the decisions on the oracle's weights agree wherever neither candidate is ambiguous
        clear = (mg_c >= EPS) & (mg_p >= EPS)
        dec = np.array([[O.mh_accept_aircraft(ell_c[l, i], ell_p[l, i], l, i, k, cfg.seed) for i in range(n)]
                        for l in range(L)])
        both_inf = ~np.isfinite(ell_c) & ~np.isfinite(ell_p)
        near = np.abs(ell_p - ell_c) < 1e-3                # MH on float vs double weights: near-ties may differ
        assert np.all((dec == bits)[clear & ~near] | both_inf[clear & ~near])
        assert 0.02 < bits.mean() < 0.98                 # both outcomes occur
    _, lam_best, idx = sol.best_controls(allow_infeasible=True)
    pop = sol.population()
    lc, lp = pop["lam_cand"]
    both = np.concatenate([lc, lp])
    assert lam_best == np.max(both[np.isfinite(both)])
    sol.close()


@pytest.mark.parametrize("mode", ["mp", "bisect", "bisect2"])
@pytest.mark.parametrize("L", [1, 7, 2048, 2049, 5000, 70001, 300001])
def test_resample_bitexact(smc, L, mode, monkeypatch):
    """Ancestors bit-exact against the oracle, by the merge-path K5, the per-slot bisection
    and K6's production two-level search through K4's every-16th CDF samples (SMC_ANC)."""
    monkeypatch.setenv("SMC_ANC", mode)
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, seed=cfg.seed)
    rng = np.random.default_rng(L)
    N = 5
    ell = rng.normal(-25, 8, (N, L)).astype(np.float32)
    ell[rng.uniform(size=(N, L)) < 0.3] = -np.inf
    ell[3] = -np.inf                                      # infeasible column
    ell[4] = np.float32(-7.25)                            # equal weights
    for k in (0, 5):
        anc, Q = sol.debug_resample(ell, k)
        for i in range(N):
            r = O.resample_column(ell[i].astype(np.float64), i, k, cfg.seed)
            assert Q[i] == r["Q"], (i, k)
            assert np.array_equal(anc[i], r["anc"]), (i, k, np.nonzero(anc[i] != r["anc"])[0][:10])


@pytest.mark.parametrize("scan", ["cluster", "lookback"])
@pytest.mark.parametrize("L", [1, 9, 2049, 16384, 65536])
def test_resample_scan_variants_bitexact(smc, L, scan, monkeypatch):
    """The integer CDF by the 8-CTA cluster scan (DSMEM exchange, default up to 65 536
    particles) and by the decoupled look-back scan: ancestors and totals bit-exact."""
    monkeypatch.setenv("SMC_SCAN", scan)
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, seed=cfg.seed)
    rng = np.random.default_rng(L + 17)
    N = 3
    ell = rng.normal(-25, 8, (N, L)).astype(np.float32)
    ell[rng.uniform(size=(N, L)) < 0.3] = -np.inf
    ell[2] = -np.inf
    anc, Q = sol.debug_resample(ell, 4)
    for i in range(N):
        r = O.resample_column(ell[i].astype(np.float64), i, 4, cfg.seed)
        assert Q[i] == r["Q"] and np.array_equal(anc[i], r["anc"]), i


@pytest.mark.parametrize("mode", ["mp", "bisect", "bisect2"])
@pytest.mark.parametrize("L,M", [(5000, 1), (5000, 777), (5000, 4999), (2049, 1500), (70001, 30000), (1, 1), (3, 1),
                                 (4099, 4099), (17, 5)])
def test_resample_to_fewer_bitexact(smc, L, M, mode, monkeypatch):
    """Shrinking populations: M < L slots drawn from L particles."""
    monkeypatch.setenv("SMC_ANC", mode)
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, seed=cfg.seed)
    rng = np.random.default_rng(L + M)
    N = 3
    ell = rng.normal(-25, 8, (N, L)).astype(np.float32)
    ell[rng.uniform(size=(N, L)) < 0.3] = -np.inf
    ell[2] = np.float32(-3.5)
    for k in (0, 7):
        anc, Q = sol.debug_resample(ell, k, M=M)
        assert anc.shape == (N, M)
        for i in range(N):
            r = O.resample_column(ell[i].astype(np.float64), i, k, cfg.seed, M=M)
            assert Q[i] == r["Q"], (i, k)
            assert np.array_equal(anc[i], r["anc"]), (i, k)


@pytest.mark.parametrize("L,Lf,S,K,mode", [(256, 40, 4, 6, None), (140000, 60000, 2, 3, None),
                                           (256, 40, 4, 6, "mp"), (140000, 60000, 2, 3, "bisect"),
                                           (5000, 3001, 2, 3, "plain")])
def test_shrinking_population_rounds(smc, L, Lf, S, K, mode, monkeypatch):
    """Real rounds with L_k falling linearly to L_final: population
    sizes follow the oracle's schedule, each round's ancestors (read back from
    the next round's x' rows) are the oracle's resampling of the GPU's ell into
    L_{k+1} slots, and the log-weights match the oracle's evaluation.  Both
    ancestor paths: merge-path K5 (default from 2^17 particles) and bisection in
    K6 (two-level through K4's every-16th-prefix samples by default, or plain)."""
    if mode == "plain":                     # bisection over the whole CDF, no 16-entry samples
        monkeypatch.setenv("SMC_ANC", "bisect")
        monkeypatch.setenv("SMC_CDF_SAMPLE", "0")
    elif mode:
        monkeypatch.setenv("SMC_ANC", mode)
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, L=L, S=S, K=K, seed=cfg.seed, L_final=Lf)
    P = O.Problem(scn)
    n = scn["n"]
    prev = None
    for k in range(K):
        sol.iterate(1)
        pop = sol.population()
        Lk = O.particles_of(L, Lf, K, k)
        assert pop["cur"].shape[0] == Lk and pop["ell"].shape == (n, Lk), (k, Lk)
        if prev is not None:
            chosen, ell_prev, kp = prev
            for i in range(n):
                r = O.resample_column(ell_prev[i].astype(np.float64), i, kp, cfg.seed, M=Lk)
                if r["Q"] == 0:
                    continue
                assert np.array_equal(pop["cur"][:, i], chosen[r["anc"], i]), (k, i)
        sub = slice(0, min(Lk, 4000))              # the oracle checks the first 4000 particles
        ell_c, mg_c = P.evaluate(pop["cur"][sub].astype(np.float64), S, k, cfg.seed, margin=True,
                                 ell0=-math.log2(Lk))
        if k > 0:
            ell_p, mg_p = P.evaluate(pop["prop"][sub].astype(np.float64), S, k, cfg.seed, margin=True,
                                     ell0=-math.log2(Lk))
            sv = pop["surv"][sub][:, None] == 1
            ell_o, mg = np.where(sv, ell_p, ell_c), np.where(sv, mg_p, mg_c)
        else:
            ell_o, mg = ell_c, mg_c
        _check_ell(pop["ell"].T[sub], ell_o, mg, S, f"shrinking L={L} k={k}")
        chosen = np.where(pop["surv"][:, None, None, None] == 1, pop["prop"], pop["cur"])
        prev = (chosen, pop["ell"], k)
    sol.close()


def test_propose_parity(smc):
    scn, cfg = sc.config(2)
    L = 500
    sol = _solver(smc, scn, L=L, seed=cfg.seed)
    P = O.Problem(scn)
    surv = _near_trim_controls(scn, L, seed=4)
    rng = np.random.default_rng(3)
    anc = np.sort(rng.integers(0, L, (scn["n"], L)), axis=1).astype(np.int32)
    k = 9
    xp, xs = sol.debug_propose(surv, anc, k)
    sig = np.array(cfg.sigma) * 0.98 ** k
    for j in range(0, L, 7):
        for i in range(scn["n"]):
            parent = surv[anc[i, j], i]
            assert np.array_equal(xp[j, i], parent)
            ref = P.perturb_row(i, parent.astype(np.float64), j, k, cfg.seed, sig)
            assert np.allclose(xs[j, i], ref, rtol=1e-5, atol=1e-4 * np.array([1.0, 1e-4, 1e-4])), (j, i)


def test_init_population_parity(smc):
    scn, cfg = sc.config(2)
    L = 300
    sol = _solver(smc, scn, L=L, seed=cfg.seed)
    pop = sol.population()
    ref = O.Problem(scn).init_population(L, cfg.seed)
    assert np.allclose(pop["cur"], ref, rtol=1e-6, atol=1e-6)


def test_round_replay_bitexact(smc):
    """Real SMC rounds on the GPU (c1), replayed stage by stage through the
    oracle: survivors' log-weights (tolerance), MH decisions on the GPU's
    lambdas, ancestors on the GPU's ell, proposals on the GPU's survivors."""
    scn, cfg = sc.config(1)
    L, S = 256, 4
    sol = _solver(smc, scn, L=L, S=S, K=10, seed=cfg.seed)
    P = O.Problem(scn)
    n = scn["n"]
    for k in range(4):
        before = sol.population() if k > 0 else None
        sol.iterate(1)
        pop = sol.population()
        if k == 0:
            ell_o, mg = P.evaluate(pop["cur"].astype(np.float64), S, 0, cfg.seed, margin=True)
            assert np.all(pop["surv"] == 0)
        else:
            ell_c, mg_c = P.evaluate(pop["cur"].astype(np.float64), S, k, cfg.seed, margin=True)
            ell_p, mg_p = P.evaluate(pop["prop"].astype(np.float64), S, k, cfg.seed, margin=True)
            # MH replay on the GPU's own lambdas is bit-exact
            lc_g, lp_g = pop["lam_cand"]
            acc_ref = np.array([O.mh_accept(lc_g[l], lp_g[l], l, k, cfg.seed) for l in range(L)])
            assert np.array_equal(pop["surv"].astype(bool), acc_ref)
            sv = pop["surv"][:, None] == 1
            ell_o, mg = np.where(sv, ell_p, ell_c), np.where(sv, mg_p, mg_c)
        _check_ell(pop["ell"].T, ell_o, mg, S, f"round replay c1 k={k}", lam_g=pop["lam"])
        # resampling replay: the oracle on the GPU's survivor ell gives the GPU's ancestors
        if k < 3:
            anc_g, _ = sol.debug_resample(pop["ell"], k)
            for i in range(n):
                r = O.resample_column(pop["ell"][i].astype(np.float64), i, k, cfg.seed)
                assert np.array_equal(anc_g[i], r["anc"])


def test_select_and_plant_parity(smc):
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, L=256, S=4, K=6, seed=cfg.seed)
    applied, nxt, flags = sol.mpc_step(scn["x0"])
    pop = sol.population()
    lam = pop["lam"]
    best = O.select(lam)
    assert best >= 0
    P = O.Problem(scn)
    ref_next, ref_flags, _, _ = P.plant_step(scn["x0"], applied.astype(np.float64), cfg.seed, 0)
    assert np.allclose(nxt, ref_next, rtol=1e-12, atol=1e-9)
    assert np.array_equal(flags.astype(np.int32), ref_flags)
    ctrl = pop["prop"][best] if pop["surv"][best] else pop["cur"][best]
    assert np.array_equal(applied, ctrl[:, 0, :])


def test_plant_parity_dense_grid(smc):
    """K8 (FP64 plant) on a 4x3x2 wind grid, two consecutive MPC steps (AR(1) carry)."""
    scn, cfg = sc.config(1)
    scn.update(wind_n=(4, 3, 2), sigma_lo=3.0, sigma_hi=6.0)
    sol = _solver(smc, scn, L=256, S=4, K=4, seed=cfg.seed)
    P = O.Problem(scn)
    Z, zi, x = None, 0, scn["x0"].copy()
    for m in range(2):
        applied, nxt, flags = sol.mpc_step(x)
        ref_next, ref_flags, Z, zi = P.plant_step(x, applied.astype(np.float64), cfg.seed, m, Z, zi)
        assert np.allclose(nxt, ref_next, rtol=1e-12, atol=1e-9), m
        assert np.array_equal(flags.astype(np.int32), ref_flags)
        x = nxt
    sol.close()


def test_graph_replay_matches_direct_launches(smc):
    """The CUDA-graph replay of smc_solve is bit-identical to direct launches,
    across MPC-step indices (the index is read from device memory)."""
    scn, cfg = sc.config(2)
    out = []
    for use_graph in (False, True):
        sol = smc.Solver(scn, L=2048, S=4, K=5, sigma=cfg.sigma, seed=cfg.seed, use_graph=use_graph)
        res = []
        for m in (0, 3, 3):
            sol.mpc_index = m
            sol.solve(advance_plant=False)
            pop = sol.population()
            res.append((pop["cur"].copy(), pop["ell"].copy(), pop["lam"].copy(), sol.best_controls(allow_infeasible=True)[0]))
        out.append(res)
        sol.close()
    for a, b in zip(out[0], out[1]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    assert not np.array_equal(out[0][0][1], out[0][1][1])     # different MPC index, different streams


@pytest.mark.parametrize("num", [2, 3, 4, 5])
def test_full_size_sampled_parity(smc, num):
    """Configs c2-c5 at full size (c5: L = 2^20, N = 16, S = 64) in the bench's
    launch configuration (CUDA graph): two rounds on the GPU; 48 sampled
    survivors of round 1 re-evaluated by the oracle one by one (element by
    element), and 2000 MH decisions replayed bit-exactly on the GPU's lambdas."""
    scn, cfg = sc.config(num)
    sol = smc.Solver(scn, L=cfg.L, S=cfg.S, K=cfg.K, sigma=cfg.sigma, seed=cfg.seed, use_graph=True)
    sol.iterate(2)
    pop = sol.population()
    lc, lp = pop["lam_cand"]
    rng0 = np.random.default_rng(1)
    for l in rng0.choice(cfg.L, 2000, replace=False):
        assert pop["surv"][l] == O.mh_accept(lc[l], lp[l], int(l), 1, cfg.seed)
    P = O.Problem(scn)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(cfg.L, 48, replace=False))
    ctrl = np.stack([(pop["prop"][l] if pop["surv"][l] else pop["cur"][l]) for l in idx]).astype(np.float64)
    ell_o = np.full((len(idx), scn["n"]), -np.log2(cfg.L))
    mg = np.full((len(idx), scn["n"]), np.inf)
    for j, l in enumerate(idx):                # particle l's global index keys its streams
        r_ell = ell_o[j].copy()
        for s in range(cfg.S):
            r = P.rollout(ctrl[j], int(l), s, 1, cfg.seed)
            lmin = r["margin_land"].min()
            mg[j] = np.minimum(mg[j], np.minimum(r["margin"], lmin))
            r_ell = np.where(r["viol"].astype(bool) | (r["J"] <= 0), -np.inf,
                             r_ell + np.log2(np.maximum(r["J"], 1e-300)))
        ell_o[j] = r_ell
    _check_ell(pop["ell"][:, idx].T, ell_o, mg, cfg.S, f"full size c{num}")


def test_mpc_loop_rolling_window(smc):
    """Short rolling-window loop: aircraft enter mid-horizon, the
    plant advances active ones only, and the realised trajectories satisfy the
    envelope (post-hoc audit of the applied controls)."""
    from paper_1506_02869_b200 import mpc_loop
    base, cfg = sc.config(3)
    tr = sc.traffic(3, 2, seed=9, arr_every=3, dep_every=10)
    recs, done, fuel, aud = mpc_loop.run(base, tr, L=2048, S=4, K=8, sigma=cfg.sigma, seed=cfg.seed, n_steps=8,
                                         max_aircraft=8, return_audit=True)
    assert len(recs) >= 6
    assert recs[0].window >= 1 and any(r.active > recs[0].active for r in recs)
    assert all(not r.infeasible for r in recs)
    assert all(f >= 0 for f in fuel.values())
    assert aud.landed + aud.exited + aud.unfinished == aud.n_aircraft == 5
    assert aud.sep_violations == 0 and aud.min_sep_m > 0


def test_paper_literal_mode_replay(smc):
    """Alg.1 exactly as printed (N1): no MH (x* always replaces x') and the
    paper's SampleSchedule floor(3 + 5 e^{0.05 J}).  Replayed against
    the oracle round by round; the oracle's own full run uses the same rules."""
    scn, cfg = sc.config(1)
    L = 2048
    sol = smc.Solver(scn, L=L, S=cfg.S, K=4, sigma=cfg.sigma, seed=cfg.seed, mh=False, sched_paper=True)
    P = O.Problem(scn)
    stats = []
    for k in range(3):
        st = sol.iterate(1, stats=True)[0]
        assert st["n_samples"] == O.sample_schedule(k)
        pop = sol.population()
        if k == 0:
            assert np.all(pop["surv"] == 0)
            ctrl = pop["cur"]
        else:
            assert np.all(pop["surv"] == 1)
            ctrl = pop["prop"]
        ell_o, mg = P.evaluate(ctrl.astype(np.float64), O.sample_schedule(k), k, cfg.seed, margin=True)
        _check_ell(pop["ell"].T, ell_o, mg, O.sample_schedule(k), f"paper-literal k={k}", lam_g=pop["lam"])


@pytest.mark.parametrize("num,vw,mh", [(1, 2, 1), (2, 3, 1), (5, 4, 1), (2, 3, 2)])
@pytest.mark.parametrize("exchange", ["peer", "allgather"])
def test_virtual_ranks_bitexact(smc, num, vw, mh, exchange, monkeypatch):
    """G-invariance on one GPU: the multi-GPU resampling path (per-rank CDFs,
    rank-offset bisection, record merge; parent rows read in place from their
    owner's buffers -- the NVLink peer mode -- or from the all-gathered compacted
    survivor rows) run for vw virtual ranks reproduces the single-rank
    populations bit for bit."""
    monkeypatch.setenv("SMC_P2P", "1" if exchange == "peer" else "0")
    scn, cfg = sc.config(num)
    L = min(cfg.L, 65536 + 123)
    res = []
    for v in (0, vw):
        sol = smc.Solver(scn, L=L, S=min(cfg.S, 4), K=4, sigma=cfg.sigma, seed=cfg.seed, virtual_world=v, mh=mh)
        sol.iterate(3)
        pop = sol.population()
        best = sol.best_controls(allow_infeasible=True)
        res.append((pop, best))
        sol.close()
    (a, ba), (b, bb) = res
    for key in ("cur", "prop", "surv_mask", "ell", "lam"):
        assert np.array_equal(a[key], b[key]), key
    assert np.array_equal(ba[0], bb[0]) and ba[1] == bb[1] and ba[2] == bb[2]


@pytest.mark.parametrize("use_graph", [False, True])
def test_warm_start_init_parity(smc, use_graph):
    """Warm start (R45): after an MPC step, a new window sharing two aircraft (by id)
    starts its first Lw particles from the shifted winner -- particle 0 exactly, the
    rest perturbed -- and everything else from the fresh draw; vs the oracle."""
    from paper_1506_02869_b200 import mpc_loop
    base, cfg = sc.config(3)
    tr = sc.traffic(3, 1, seed=5, arr_every=1, dep_every=1)
    tr["entry"][:] = 0
    scn1 = mpc_loop.window_scenario(base, tr, [0, 1, 2], 10, {})
    scn2 = mpc_loop.window_scenario(base, tr, [1, 2, 3], 11, {})
    L, Lw = 400, 100
    sol = smc.Solver(scn1, L=L, S=4, K=4, sigma=cfg.sigma, seed=cfg.seed, warm_fraction=Lw / L,
                     use_graph=use_graph, max_aircraft=4)
    sol.mpc_step(scn1["x0"])
    u_prev, lam, idx = sol.best_controls(allow_infeasible=True)
    assert idx >= 0
    sol.set_scenario(scn2)
    pop = sol.population()
    P2 = O.Problem(scn2)
    prev = np.zeros((3, scn2["H"], 3))
    prev[0], prev[1] = u_prev[1], u_prev[2]                  # ids 1, 2 were rows 1, 2; id 3 is new
    ref = P2.init_population_warm(L, cfg.seed, prev, [1, 1, 0], Lw, cfg.sigma, mpc=sol.mpc_index)
    g = pop["cur"].astype(np.float64)
    shifted = np.concatenate([u_prev[1:3, 1:], u_prev[1:3, -1:]], axis=1)
    assert np.array_equal(pop["cur"][0, :2], shifted)        # exact copy of the shifted winner
    tol = np.array([1e-4 * cfg.sigma[0], 1e-4 * cfg.sigma[1], 1e-4 * cfg.sigma[2]]) + 1e-6 * np.abs(ref)
    assert np.all(np.abs(g - ref) <= tol), np.unravel_index(np.argmax(np.abs(g - ref) - tol), g.shape)
    # a solve from the warm population runs (and the next window maps again)
    sol.mpc_step(scn2["x0"])
    sol.close()


def test_fuel_estimates_parity(smc):
    """Section-5 fuel estimates (N4) on 300 synthetic traces of ragged
    length -- forward-simulated, circling and degenerate ones -- vs the oracle."""
    scn = sc.snapshot(0, 1, seed=1)
    P = O.Problem(scn)
    rng = np.random.default_rng(8)
    n, max_len, dt, Cf = 300, 40, 60.0, (1.1e-5, 500.0)
    traces = np.zeros((n, max_len, 5))
    lens = rng.integers(1, max_len + 1, n)
    lens[:3] = [1, 2, max_len]
    lens[13] = max_len
    m0 = rng.uniform(55000, 75000, n)
    for j in range(n):
        K = int(lens[j])
        st = np.array([rng.uniform(-2e4, 2e4), rng.uniform(-2e4, 2e4), rng.uniform(500, 8000),
                       rng.uniform(90, 200), rng.uniform(-3, 3)])
        for k in range(K):
            traces[j, k] = st
            if j % 50 == 7:                       # circling: no displacement
                st = st.copy(); st[4] += 0.5
                continue
            st = st + [dt * st[3] * math.cos(st[4]) + rng.normal(0, 60), dt * st[3] * math.sin(st[4]) + rng.normal(0, 60),
                       rng.normal(0, 150), rng.normal(0, 4), rng.normal(0, 0.1)]
            if j % 50 == 11:                      # implausible climb
                st[2] += 1e5
    traces[13, 3, 3] = np.nan                     # a missing airspeed: undefined burn, none booked
    ty = np.array([scn["S"][0], scn["cd0"][0], scn["cd2"][0], Cf[0], Cf[1], scn["gamma_max"][0]])
    out = smc.fuel_estimates(traces, lens, m0, np.tile(ty, (n, 1)), dt, g=scn["g"], density_mode=scn["density_mode"])
    for j in range(n):
        K = int(lens[j])
        m1, w, f1 = P.fuel_estimate1(0, traces[j, :K], dt, m0[j], Cf)
        m2, f2 = P.fuel_estimate2(0, traces[j, :K], dt, m0[j], Cf)
        assert np.allclose(out["m1"][j, :K], m1, rtol=1e-12, atol=0), j
        assert np.allclose(out["m2"][j, :K], m2, rtol=1e-12, atol=0), j
        assert np.allclose(out["wres"][j, :K], w, rtol=1e-10, atol=1e-9, equal_nan=True), j
        assert out["flags"][j] == (f1 | f2), j
        assert out["fuel"][j, 0] == pytest.approx(m0[j] - m1[-1], rel=1e-12, abs=1e-9)
    assert (out["flags"] & 2).any() and (out["flags"] & 1).any()


def test_peer_mapping_ipc(smc, tmp_path):
    """The CUDA IPC export/map that peer mode uses (smc_init with world_size > 1
    maps every peer's workspace this way): a second process maps this
    context's record -- handle of the torch allocation holding the workspace
    plus the workspace's offset in it -- and reads the initial population at
    workspace offset 0 (the x' buffer) byte for byte."""
    import os
    import subprocess
    import sys
    scn, cfg = sc.config(1)
    sol = _solver(smc, scn, L=300, seed=cfg.seed)
    pop = sol.population()
    rec = sol.ipc_record()
    out = tmp_path / "peek.bin"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (f"import sys; sys.path.insert(0, {root!r}); from paper_1506_02869_b200 import smcatm; "
            f"open({str(out)!r}, 'wb').write(smcatm.ipc_peek(bytes.fromhex({rec.hex()!r}), 0, {pop['cur'].nbytes}))")
    subprocess.run([sys.executable, "-c", code], check=True, timeout=300)
    assert out.read_bytes() == pop["cur"].tobytes()
    sol.close()


def test_infeasible_report_names_aircraft_and_round(smc):
    """SMC_EINFEASIBLE names the aircraft that is zero in every particle and
    the first round its column was all zero: aircraft 1 starts below its empty mass, so the
    mass bound fails at every step of every particle from round 0 on."""
    scn, cfg = sc.config(2)
    scn["x0"][1, 5] = scn["m_empty"][1] - 10.0
    sol = _solver(smc, scn, L=2048, S=2, K=3, seed=cfg.seed)
    sol.iterate(3)
    with pytest.raises(smc.SmcError) as e:
        sol.best_controls()
    msg = str(e.value)
    assert "SMC_EINFEASIBLE" in msg and "aircraft 1 " in msg and "since round 0" in msg, msg
    assert "aircraft 0 " not in msg
    with pytest.raises(smc.SmcError) as e2:
        sol.mpc_step(scn["x0"])
    assert "MPC step 0" in str(e2.value) and "aircraft 1 " in str(e2.value), str(e2.value)
    sol.close()
