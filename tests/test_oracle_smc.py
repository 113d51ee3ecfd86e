"""Pins for the oracle's SMC machinery: weight recursion, separation
bookkeeping, MH acceptance (R1), systematic resampling (K96),
final selection, plant step and an end-to-end toy problem
against exhaustive search."""
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_1506_02869_b200 import scenarios as sc

DEG = math.pi / 180.0


def _calm(scn):
    scn = dict(scn)
    scn.update(sigma_lo=0.0, sigma_hi=0.0, nominal=[0.0, 0.0], turb_sigma=0.0)
    return scn


# ---------------------------------------------------------------- weights
def test_weight_recursion_closed_form(ora):
    """Deterministic case (no wind, fixed controls): after S samples
    ell = -log2 L + S log2 J_T (W^{j+1} = W^j J, W^0 = 1/L)."""
    scn = _calm(sc.snapshot(2, 2, seed=3))
    P = ora.Problem(scn)
    ctrl = sc.random_controls(scn, 64, seed=4, spread=0.4).astype(np.float64)
    ell = P.evaluate(ctrl, S=5, k=0, seed=11)
    for l in range(64):
        r = P.rollout(ctrl[l], l, 0, 0, 11)
        for i in range(scn["n"]):
            if r["viol"][i]:
                assert ell[l, i] == -np.inf
            else:
                assert ell[l, i] == pytest.approx(-math.log2(64) + 5 * math.log2(r["J"][i]), abs=1e-12)


def test_zero_weight_absorbs(ora):
    """Any violation in any sample -> weight 0 for the round."""
    scn = sc.snapshot(2, 2, seed=3)
    P = ora.Problem(scn)
    ctrl = sc.random_controls(scn, 128, seed=5, spread=1.2).astype(np.float64)
    ell = P.evaluate(ctrl, S=6, k=0, seed=12)
    for l in range(0, 128, 7):
        any_viol = np.zeros(scn["n"], bool)
        for s in range(6):
            any_viol |= P.rollout(ctrl[l], l, s, 0, 12)["viol"].astype(bool)
        assert np.array_equal(np.isneginf(ell[l]), any_viol)


def test_separation_flags_match_bruteforce(ora):
    """Re-derive every violation flag from the oracle's own trajectories with
    a brute-force O(N^2) pair scan of Eq. avoidance plus the unary bounds:
    every aircraft is in every pair test at every step, violated or not
    (Alg.1 l.11-13; Eq. avoidance "for every time step ... i != j")."""
    scn = sc.snapshot(3, 3, seed=21)
    # crowd the aircraft so that conflicts actually occur
    scn["x0"][:, 0] *= 0.5
    scn["x0"][:, 1] *= 0.5
    scn["x0"][:, 2] = 3000.0 + 150.0 * np.arange(scn["n"])
    scn["kind"][:] = 1                      # departures: no landing removals
    P = ora.Problem(scn)
    n, H = scn["n"], scn["H"]
    ctrl = sc.random_controls(scn, 40, seed=8, spread=0.5).astype(np.float64)
    n_conf = n_late = 0
    for l in range(40):
        r = P.rollout(ctrl[l], l, 0, 0, 5)
        tr = r["traj"]
        viol = np.zeros(n, bool)
        for j in range(1, H + 1):
            before = viol.copy()
            for i in range(n):
                u = ctrl[l, i, j - 1]
                st = tr[i, j]
                bad = (abs(u[2]) > scn["gamma_max"][i] or not abs(u[1]) < scn["phi_max"][i]
                       or u[0] < scn["T_min"][i] or u[0] > scn["T_max"][i]
                       or not scn["z_min"][i] <= st[2] <= scn["z_max"][i]
                       or not scn["v_min"][i] <= st[3] <= scn["v_max"][i]
                       or st[5] < scn["m_empty"][i])
                if bad:
                    viol[i] = True
            for i in range(n):
                for q in range(i + 1, n):
                    d2 = (tr[i, j, 0] - tr[q, j, 0]) ** 2 + (tr[i, j, 1] - tr[q, j, 1]) ** 2
                    if d2 < (2 * 2500.0) ** 2 and abs(tr[i, j, 2] - tr[q, j, 2]) < 600.0:
                        n_late += int(before[i] != before[q])     # one side already violated earlier
                        viol[i] = viol[q] = True
                        n_conf += 1
        assert np.array_equal(viol, r["viol"].astype(bool)), l
    assert n_conf > 0 and not np.all(viol)
    assert n_late > 0          # conflicts of an earlier violator with a clean aircraft are exercised


def test_head_on_conflict_step(ora):
    """Hand-built crossing: two departures 20 km apart flying at each other at
    140 m/s, trimmed, same altitude -> first conflict when the gap < 5 km,
    i.e. at j = 6 (20000 - 2*140*10*j < 5000 first holds for j = 6);
    with |dz| = 600 m = 2 P_h they never conflict (inclusive bound)."""
    for dz, expect in [(0.0, True), (600.0, False)]:
        scn = _calm(sc.snapshot(0, 2, seed=1, H=8))
        scn["density_mode"] = 1
        scn["x0"][0] = [-10000.0, 0.0, 3000.0, 140.0, 0.0, 70000.0]
        scn["x0"][1] = [10000.0, 0.0, 3000.0 + dz, 140.0, math.pi, 70000.0]
        P = ora.Problem(scn)
        u = np.zeros((2, 8, 3))
        # trim each step so v stays 140 (the drag does not depend on x, y)
        st = [scn["x0"][0].copy(), scn["x0"][1].copy()]
        for t in range(8):
            for i in range(2):
                _, D = P.lift_drag(i, st[i], 0.0)
                u[i, t, 0] = D
                st[i] = P.step(i, st[i], u[i, t])
        r = P.rollout(u, 0, 0, 0, 1)
        gap = abs(r["traj"][0, :, 0] - r["traj"][1, :, 0])
        assert bool(r["viol"][0]) == expect and bool(r["viol"][1]) == expect
        if expect:
            first = int(np.argmax(gap < 5000.0))
            assert first == 6
            # after the conflict both keep flying their controls (Alg.1 l.11-13)
            assert r["traj"][0, 8, 0] > r["traj"][0, 7, 0] > r["traj"][0, 6, 0]


def test_landing_freezes_and_bonus(ora):
    """An arrival that lands mid-horizon is frozen and scores perfect remaining
    steps: its mean deviations only include steps up to landing."""
    scn = _calm(sc.snapshot(1, 0, seed=2, H=6))
    scn["density_mode"] = 1
    scn["x0"][0] = [6000.0, 0.0, 6000 * math.tan(3 * DEG), 75.0, math.pi, 64000.0]
    P = ora.Problem(scn)
    u = np.zeros((1, 6, 3))
    u[0, :, 2] = -3 * DEG
    st = scn["x0"][0].copy()
    for t in range(6):
        _, D = P.lift_drag(0, st, 0.0)
        u[0, t, 0] = D + st[5] * 9.81 * math.sin(-3 * DEG)
        st = P.step(0, st, u[0, t])
    r = P.rollout(u, 0, 0, 0, 1)
    j = r["landed_step"][0]
    assert 1 <= j < 6 and not r["viol"][0]
    tr = r["traj"][0]
    assert np.all(tr[j + 1:] == tr[j])
    # heading term: flying exactly West on the axis -> zero heading deviation every step
    assert r["comp"][0, 0] == pytest.approx(1.0, abs=1e-9)


def test_first_step_partial_horizon(ora):
    """An aircraft entering at step e is simulated on [e, H) only and
    its means are over H - e steps (R20); e = H contributes nothing."""
    scn = _calm(sc.snapshot(0, 2, seed=2, H=6))
    scn["first_step"] = np.array([0, 6], np.int32)
    P = ora.Problem(scn)
    u = np.zeros((2, 6, 3)); u[..., 0] = 40000.0
    r = P.rollout(u, 0, 0, 0, 1)
    assert np.all(r["traj"][1] == scn["x0"][1])
    assert r["J"][1] == 1.0 and r["viol"][1] == 0
    scn["first_step"] = np.array([0, 3], np.int32)
    P = ora.Problem(scn)
    r = P.rollout(u, 0, 0, 0, 1)
    assert np.all(r["traj"][1, :4] == scn["x0"][1])
    assert np.any(r["traj"][1, 4] != scn["x0"][1])


# ---------------------------------------------------------------- MH
def test_mh_rules(ora):
    seed = 0x5EED0001
    assert ora.mh_accept(-np.inf, -np.inf, 0, 1, seed)
    assert ora.mh_accept(-np.inf, -3.0, 0, 1, seed)
    assert not ora.mh_accept(-3.0, -np.inf, 0, 1, seed)
    for l in range(50):
        assert ora.mh_accept(-10.0, -10.0, l, 3, seed)          # delta = 0
        assert ora.mh_accept(-10.0, -2.0, l, 3, seed)
        assert not ora.mh_accept(-10.0, -10.0 - 1100.0, l, 3, seed)


def test_mh_decision_is_u53_below_2_pow_delta(ora):
    """accept iff u53 < 2^delta with u53 = (r64 >> 11) 2^-53 of the MH stream (R1);
    2^delta from Python's pow (skipping draws within 1e-15 of the threshold)."""
    seed = 99
    n = 0
    for l in range(300):
        u = (ora.r64(5, l, 4, seed) >> 11) * 2.0 ** -53
        for delta in [-0.5, -1.0, -2.0, -0.125, -7.0, -1e-9]:
            thr = 2.0 ** delta
            if abs(u - thr) < 1e-15:
                continue
            assert ora.mh_accept(-10.0, -10.0 + delta, l, 4, seed) == (u < thr)
            n += 1
    assert n > 1700


def test_mh_acceptance_frequency(ora):
    """E[accept] = min(1, 2^delta) over independent particles."""
    seed = 0xABCD
    for delta, p in [(-1.0, 0.5), (-3.0, 0.125), (-0.2, 2 ** -0.2)]:
        acc = np.array([ora.mh_accept(-5.0, -5.0 + delta, l, 2, seed) for l in range(20000)])
        assert acc.mean() == pytest.approx(p, abs=4 * math.sqrt(p * (1 - p) / acc.size))


# ---------------------------------------------------------------- resampling
def _textbook_systematic(q, R, Q):
    """Kitagawa/systematic resampling with the single offset u = R/Q (exact
    rationals): slot j takes the first l whose normalised CDF exceeds (j+u)/L."""
    L = len(q)
    cdf, acc = [], 0
    for v in q:
        acc += v
        cdf.append(Fraction(acc, Q))
    out = []
    for j in range(L):
        pos = (j + Fraction(R, Q)) / L
        out.append(next(l for l in range(L) if cdf[l] > pos))
    return out


def test_resample_matches_textbook_systematic(ora):
    rng = np.random.default_rng(10)
    for trial in range(60):
        L = int(rng.integers(1, 40))
        ell = rng.uniform(-40, 0, L)
        ell[rng.uniform(size=L) < 0.2] = -np.inf
        if trial % 7 == 0:
            ell[:] = -np.inf
        r = ora.resample_column(ell, i=trial % 5, k=trial, seed=0x77)
        q = [int(v) for v in r["q"]]
        assert sum(q) == r["Q"]
        assert r["anc"].tolist() == _textbook_systematic(q, r["R"], r["Q"])


def test_resample_invariants(ora):
    rng = np.random.default_rng(11)
    for trial in range(40):
        L = int(rng.integers(50, 3000))
        ell = rng.normal(-20, 6, L)
        ell[rng.uniform(size=L) < 0.3] = -np.inf
        r = ora.resample_column(ell, i=3, k=trial, seed=0x1234)
        anc, q, Q = r["anc"], r["q"].astype(object), r["Q"]
        counts = np.bincount(anc, minlength=L)
        assert counts.sum() == L                                     # particle count preserved
        assert np.all(np.diff(anc) >= 0)                              # monotone
        assert np.all(counts[np.array(q) == 0] == 0)                 # zero weight never chosen
        for l in range(L):                                           # {floor, ceil} of L q/Q
            e = Fraction(int(q[l]) * L, Q)
            assert math.floor(e) <= counts[l] <= math.ceil(e)


def test_resample_special_columns(ora):
    L = 16
    r = ora.resample_column(np.full(L, -3.0), 0, 0, 5)
    assert r["anc"].tolist() == list(range(L))                      # equal weights
    ell = np.full(L, -np.inf); ell[11] = -2.0
    r = ora.resample_column(ell, 0, 0, 5)
    assert np.all(r["anc"] == 11)                                    # degenerate column
    r = ora.resample_column(np.full(L, -np.inf), 0, 0, 5)
    assert r["infeasible"] and r["anc"].tolist() == list(range(L))  # uniform fallback (R25)
    # weights (0.5, 0.25, 0.25, 0): counts (2,1,1,0) for every offset
    ell = np.array([0.0, -1.0, -1.0, -np.inf])
    for k in range(40):
        r = ora.resample_column(ell, 1, k, 9)
        assert np.bincount(r["anc"], minlength=4).tolist() == [2, 1, 1, 0]


# ---------------------------------------------------------------- selection
def test_select(ora):
    lam = np.array([math.log2(0.9) + -np.inf, math.log2(0.1) + math.log2(0.1)])
    assert ora.select(lam) == 1                                       # (0.9, 0) loses to (0.1, 0.1)
    assert ora.select(np.array([-3.0, -1.0, -1.0, -2.0])) == 1        # ties -> lowest l (R27)
    assert ora.select(np.full(5, -np.inf)) == -1                       # infeasible


# ---------------------------------------------------------------- plant
def test_plant_step_matches_model(ora):
    scn = _calm(sc.snapshot(2, 2, seed=4))
    scn["first_step"] = np.array([0, 0, 0, 2], np.int32)
    P = ora.Problem(scn)
    u0 = np.array([[40000, 0.1, -0.02], [30000, -0.1, 0.0], [50000, 0.0, 0.03], [1, 1, 1]], float)
    nxt, flags, Z, zi = P.plant_step(scn["x0"], u0, 7, 0)
    for i in range(3):
        assert np.allclose(nxt[i], P.step(i, scn["x0"][i], u0[i]), rtol=0, atol=0)
    assert np.all(nxt[3] == scn["x0"][3])                           # not yet entered
    assert zi == 1


def test_plant_flags(ora):
    scn = _calm(sc.snapshot(1, 1, seed=4))
    scn["density_mode"] = 1
    scn["x0"][0] = [2500.0, 0.0, 2500 * math.tan(3 * DEG), 75.0, math.pi, 64000.0]
    scn["x0"][1] = [29500.0 * math.cos(0.3), 29500.0 * math.sin(0.3), 5000.0, 150.0, 0.3, 70000.0]
    P = ora.Problem(scn)
    u0 = np.array([[20000.0, 0.0, -3 * DEG], [50000.0, 0.0, 0.0]])
    nxt, flags, _, _ = P.plant_step(scn["x0"], u0, 7, 3)
    assert flags[0] & 1 and flags[1] & 2


# ---------------------------------------------------------------- end to end
@pytest.mark.slow
def test_toy_smc_vs_exhaustive_grid(ora):
    """1 aircraft, H = 1, deterministic (no wind): SMC's best utility within 2%
    of an exhaustive 30^3 grid over the control box."""
    scn = _calm(sc.snapshot(0, 1, seed=5, H=1))
    P = ora.Problem(scn)
    n = 30
    T = np.linspace(0.0, 1.2e5, n)
    ph = np.linspace(-30 * DEG, 30 * DEG, n + 2)[1:-1]
    ga = np.linspace(-6 * DEG, 6 * DEG, n)
    grid = np.array(np.meshgrid(T, ph, ga, indexing="ij")).reshape(3, -1).T
    ell = P.evaluate(grid.reshape(-1, 1, 1, 3), S=1, k=0, seed=1, ell0=0.0)
    best_grid = 2.0 ** ell.max()
    res = P.run_smc(L=1024, S=1, K=12, seed=3, sigma=(6000.0, 2 * DEG, 0.5 * DEG))
    assert res["rc"] == 0
    best_smc = 2.0 ** (res["best_lambda"] + math.log2(1024))
    assert best_smc >= 0.98 * best_grid


def _textbook_systematic_m(q, R, Q, M):
    """Systematic resampling into M slots with offset u = R/Q (exact rationals)."""
    cdf, acc = [], 0
    for v in q:
        acc += v
        cdf.append(Fraction(acc, Q))
    return [next(l for l in range(len(q)) if cdf[l] > (j + Fraction(R, Q)) / M) for j in range(M)]


def test_resample_to_fewer_particles(ora):
    """Shrinking populations: M < L slots, same systematic definition;
    counts lie in {floor(M q/Q), ceil(M q/Q)} and sum to M."""
    rng = np.random.default_rng(12)
    for trial in range(40):
        L = int(rng.integers(2, 60))
        M = int(rng.integers(1, L + 1))
        ell = rng.uniform(-30, 0, L)
        ell[rng.uniform(size=L) < 0.2] = -np.inf
        r = ora.resample_column(ell, i=trial % 4, k=trial, seed=0x99, M=M)
        q = [int(v) for v in r["q"]]
        assert r["anc"].tolist() == _textbook_systematic_m(q, r["R"], r["Q"], M)
        counts = np.bincount(r["anc"], minlength=L)
        assert counts.sum() == M
        for l in range(L):
            e = Fraction(q[l] * M, r["Q"])
            assert math.floor(e) <= counts[l] <= math.ceil(e)


def test_particle_schedule(ora):
    """Linear particle count from L to L_final over K rounds (integer arithmetic)."""
    assert [ora.particles_of(1000, 400, 4, k) for k in range(4)] == [1000, 800, 600, 400]
    assert ora.particles_of(1000, 0, 10, 5) == 1000
    assert all(ora.particles_of(16384, 4096, 101, k) >= ora.particles_of(16384, 4096, 101, k + 1) for k in range(100))
    res = ora.Problem(sc.config(1)[0]).run_smc(L=256, S=4, K=6, seed=1, sigma=(6000.0, 0.03, 0.008), L_final=64)
    assert res["rc"] in (0, 2)


def test_warm_start_init(ora):
    """R45: shifted previous winner seeds the first Lw particles; everything else is
    the fresh uniform draw."""
    import numpy as np
    from paper_1506_02869_b200 import scenarios as sc
    scn = sc.small(n_arr=2, n_dep=1, H=6)
    P = ora.Problem(scn)
    n, H, L, seed = scn["n"], scn["H"], 300, 77
    fresh = P.init_population(L, seed, mpc=3)
    prev = np.zeros((n, H, 3))
    for i in range(n):
        for t in range(H):
            prev[i, t] = [5e4 + 100 * t + i, 0.01 * t, -0.001 * t]
    sig = (2000.0, 0.02, 0.005)
    # no warm particles / no previous rows: identical to the fresh population
    assert np.array_equal(P.init_population_warm(L, seed, prev, [1] * n, 0, sig, mpc=3), fresh)
    assert np.array_equal(P.init_population_warm(L, seed, prev, [0] * n, 100, sig, mpc=3), fresh)
    has = [1, 0, 1]
    w = P.init_population_warm(L, seed, prev, has, 100, sig, mpc=3)
    shifted = np.concatenate([prev[:, 1:], prev[:, -1:]], axis=1)
    for i in range(n):
        if has[i]:
            assert np.array_equal(w[0, i], shifted[i])                 # particle 0: exact shifted winner
        else:
            assert np.array_equal(w[:, i], fresh[:, i])                # new aircraft: fresh rows
    assert np.array_equal(w[100:], fresh[100:])                        # beyond Lw: fresh
    z = (w[1:100][:, [0, 2]] - shifted[[0, 2]][None]) / np.array(sig)  # standardised perturbations
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05
    wc = P.init_population_warm(L, seed, prev, has, 100, (1e6, 10.0, 10.0), mpc=3, clamp=True)
    for i in (0, 2):
        assert np.all(wc[:, i, :, 0] <= scn["T_max"][i]) and np.all(wc[:, i, :, 0] >= scn["T_min"][i])
        assert np.all(np.abs(wc[:, i, :, 1]) <= scn["phi_max"][i]) and np.all(np.abs(wc[:, i, :, 2]) <= scn["gamma_max"][i])


def test_mh_accept_aircraft_rules(ora):
    """R46: the joint rules (R1) on one aircraft's weights; acceptance frequency 2^Delta."""
    import numpy as np
    inf = float("inf")
    assert ora.mh_accept_aircraft(-inf, -inf, 3, 1, 2, 9)
    assert not ora.mh_accept_aircraft(-5.0, -inf, 3, 1, 2, 9)
    assert ora.mh_accept_aircraft(-5.0, -5.0, 3, 1, 2, 9)
    acc = np.mean([ora.mh_accept_aircraft(-3.0, -4.0, l, 2, 5, 11) for l in range(20000)])
    assert abs(acc - 0.5) < 0.02
    # aircraft index enters the counter: decisions of different aircraft are not copies
    a = [ora.mh_accept_aircraft(-3.0, -4.0, l, 0, 5, 11) for l in range(2000)]
    b = [ora.mh_accept_aircraft(-3.0, -4.0, l, 1, 5, 11) for l in range(2000)]
    assert a != b
    # aircraft 0 uses the joint stream's counter: same decision as the joint rule on equal values
    assert all(ora.mh_accept_aircraft(-3.0, -3.7, l, 0, 4, 13) == ora.mh_accept(-3.0, -3.7, l, 4, 13)
               for l in range(500))


def test_per_aircraft_mh_single_aircraft_reduces_to_joint(ora):
    """With one aircraft the per-aircraft move is the joint move (same decisions, same
    survivors): identical round statistics; its final pick over both candidates can
    only be at least as good."""
    import numpy as np
    from paper_1506_02869_b200 import scenarios as sc
    scn = sc.small(n_arr=1, n_dep=0, H=6, seed=3)
    P = ora.Problem(scn)
    sig = (0.05 * 1.2e5, 0.035, 0.0087)
    r1 = P.run_smc(128, 3, 5, 77, sig, mh=1)
    r2 = P.run_smc(128, 3, 5, 77, sig, mh=2)
    assert np.array_equal(r1["stats"], r2["stats"])
    assert r2["best_lambda"] >= r1["best_lambda"]


# ---------------------------------------------------------------- init and perturbation
def _ks_uniform(x):
    x = np.sort(x)
    n = len(x)
    i = np.arange(1, n + 1)
    return max(np.max(i / n - x), np.max(x - (i - 1) / n))


def test_init_population_uniform_in_bounds(ora):
    """Alg.1 l.5 draws every control uniformly over the envelope of P:240:
    T in [T_min, T_max], phi in [-phi_max, phi_max], gamma in [-gamma_max, gamma_max].
    Each component, scaled to [0, 1], passes a Kolmogorov-Smirnov test (alpha ~ 1e-3);
    components, aircraft and steps are uncorrelated."""
    scn = sc.snapshot(2, 2, seed=3)
    P = ora.Problem(scn)
    L = 3000
    c = P.init_population(L, 0x5EED0042)
    lo = np.array([scn["T_min"][0], -scn["phi_max"][0], -scn["gamma_max"][0]])
    hi = np.array([scn["T_max"][0], scn["phi_max"][0], scn["gamma_max"][0]])
    assert np.all(c > lo) and np.all(c < hi)
    u = (c - lo) / (hi - lo)
    n = u[..., 0].size
    for q in range(3):
        assert _ks_uniform(u[..., q].ravel()) < 1.95 / math.sqrt(n), q
    flat = u.reshape(L, -1)
    cc = np.corrcoef(flat[:, :24].T)
    assert np.max(np.abs(cc - np.eye(24))) < 0.08


def test_perturbation_residuals_are_standard_normal(ora):
    """Alg.1 l.23: x* = x' + Gaussian white noise with the per-component
    sigma.  The standardised residuals (x* - x')/sigma are N(0, 1) in every component
    (mean, variance, KS against the normal CDF), independent across steps and
    aircraft; sigma = 0 returns the parent exactly; without the clamp option nothing is
    clipped (an out-of-envelope proposal is a constraint violation, R16), with it every
    component lands in the envelope."""
    scn = sc.snapshot(2, 1, seed=3)
    P = ora.Problem(scn)
    sig = np.array([6000.0, 0.035, 0.0087])
    parent = np.tile(np.array([60000.0, 0.1, -0.02]), (scn["H"], 1))
    z = []
    for l in range(600):
        for i in range(scn["n"]):
            x = P.perturb_row(i, parent, l, 7, 0x77, sig)
            z.append((x - parent) / sig)
    z = np.array(z)                                    # [600 n][H][3]
    from math import erf
    for q in range(3):
        v = z[..., q].ravel()
        assert abs(v.mean()) < 4 / math.sqrt(v.size) and v.var() == pytest.approx(1.0, rel=0.06)
        cdf = np.array([0.5 * (1 + erf(s / math.sqrt(2))) for s in np.sort(v)])
        i = np.arange(1, v.size + 1)
        assert max(np.max(i / v.size - cdf), np.max(cdf - (i - 1) / v.size)) < 1.95 / math.sqrt(v.size)
    flat = z.reshape(z.shape[0], -1)
    cc = np.corrcoef(flat.T)
    assert np.max(np.abs(cc - np.eye(cc.shape[0]))) < 0.15
    assert np.array_equal(P.perturb_row(0, parent, 3, 7, 0x77, (0.0, 0.0, 0.0)), parent)
    big = P.perturb_row(0, parent, 3, 7, 0x77, (1e6, 10.0, 10.0))
    assert np.any(big[:, 0] > scn["T_max"][0]) or np.any(big[:, 0] < scn["T_min"][0])
    cl = P.perturb_row(0, parent, 3, 7, 0x77, (1e6, 10.0, 10.0), clamp=True)
    assert np.all((cl[:, 0] >= scn["T_min"][0]) & (cl[:, 0] <= scn["T_max"][0]))
    assert np.all(np.abs(cl[:, 1]) <= scn["phi_max"][0]) and np.all(np.abs(cl[:, 2]) <= scn["gamma_max"][0])


def test_proposal_spread_anneals(ora):
    """The proposal spread of round k is sigma * anneal^k (R16): with a single
    particle per aircraft and a calm, deterministic scenario, the paper-literal run
    (mh = 0) reproduces the oracle's own perturbation with sigma 0.98^k for the
    proposal of round k -- its selected controls after K = 3 rounds equal
    perturb(perturb(init, k = 0, sigma), k = 1, 0.98 sigma)."""
    scn = _calm(sc.snapshot(0, 1, seed=5, H=3))
    P = ora.Problem(scn)
    sig = (3000.0, 0.02, 0.004)
    res = P.run_smc(L=1, S=1, K=3, seed=0x32, sigma=sig, mh=False, anneal=0.98)
    assert res["rc"] == 0
    x = P.init_population(1, 0x32)[0, 0]
    x = P.perturb_row(0, x, 0, 0, 0x32, sig)
    x1 = P.perturb_row(0, x, 0, 1, 0x32, tuple(0.98 * s for s in sig))
    assert np.allclose(res["best_ctrl"][0], x1, rtol=0, atol=1e-9)
    x1_flat = P.perturb_row(0, x, 0, 1, 0x32, sig)           # without annealing: a different row
    assert not np.allclose(res["best_ctrl"][0], x1_flat, rtol=0, atol=1e-6)
