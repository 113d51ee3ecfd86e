"""Pins for the oracle's bookkeeping conventions where the paper gives a rule in
prose only: the rolling-window partial horizon (R20, "optimised from the
point they enter"), the post-landing bonus (R18, "best possible cost, 1,
for all remaining steps"), constraint handling after a violation (Alg.1
l.11-13 and Eq. avoidance: the violator keeps flying and
stays in every pair test) -- and the MH move (R1, north_star; not in the
paper), whose common random numbers and acceptance rule are pinned against
the paper's own Alg.1 move.  Each is pinned by an invariant or a closed form
computed here from first principles (no oracle cost helper is called for the
expected value); the R18/R20/constraint cases fly in calm air so that every
rollout is deterministic."""
import math

import numpy as np
import pytest

from paper_1506_02869_b200 import scenarios as sc

DEG = math.pi / 180.0


def _calm(scn):
    scn.update(sigma_lo=0.0, sigma_hi=0.0, nominal=[0.0, 0.0], turb_sigma=0.0)
    return scn


def _dep(x, y, z, v, chi, first_step=0):
    return dict(kind=1, x0=[x, y, z, v, chi, 73500.0], theta_F=chi, z_tf=6000.0, v_D=150.0, beta_f=0.0,
                m_empty=58000.0, first_step=first_step)


def _scenario(ac, H, dt=10.0):
    return _calm(sc._finish(sc.base_scenario(H=H, dt=dt), ac))


def _cruise_controls(ora, scn, i, H, climb=1.0 * DEG, bank=0.0):
    """Controls that keep aircraft i in the envelope: thrust = drag + weight component."""
    P = ora.Problem(scn)
    u = np.zeros((H, 3))
    st = np.asarray(scn["x0"][i], dtype=np.float64).copy()
    for t in range(H):
        _, D = P.lift_drag(i, st, bank)
        u[t] = [D + st[5] * 9.81 * math.sin(climb), bank, climb]
        st = P.step(i, st, u[t])
    return u


# ---------------------------------------------------------------- R20
@pytest.mark.parametrize("e", [1, 2, 4])
def test_partial_horizon_equals_shorter_horizon(ora, e):
    """An aircraft entering at step e of an H-step window (R20) scores exactly
    what the same aircraft scores over an (H - e)-step window entered at step 0
    with the same controls: its means run over H_a = H - e predicted states
    and its fuel normaliser over H_a steps (no term sees the absolute step)."""
    H = 6
    a = _dep(-12000.0, -9000.0, 1500.0, 110.0, 0.3)
    b = _dep(9000.0, 8000.0, 2500.0, 120.0, 2.0)
    full = _scenario([a, dict(b, first_step=e)], H)
    ub = _cruise_controls(ora, _scenario([b], H - e), 0, H - e, climb=2.0 * DEG, bank=5.0 * DEG)
    u = np.zeros((2, H, 3))
    u[0] = _cruise_controls(ora, _scenario([a], H), 0, H)
    u[1, e:] = ub
    u[1, :e] = ub[0]                          # before entry: never applied
    r = ora.Problem(full).rollout(u, 0, 0, 0, 1)
    short = _scenario([b], H - e)
    rs = ora.Problem(short).rollout(ub[None], 0, 0, 0, 1)
    assert r["viol"][1] == 0 and rs["viol"][0] == 0
    assert r["J"][1] == pytest.approx(rs["J"][0], abs=1e-12)
    assert np.allclose(r["comp"][1], rs["comp"][0], atol=1e-12)
    assert r["fuel"][1] == pytest.approx(rs["fuel"][0], rel=1e-12)
    assert np.allclose(r["traj"][1, e:], rs["traj"][0], rtol=1e-12, atol=1e-9)


# ---------------------------------------------------------------- constraint handling (Alg.1 l.11-13)
def test_violator_keeps_flying_and_zeroes_a_later_neighbour(ora):
    """Alg.1 simulates every agent to H and only then tests the constraints
    (l.11-13); Eq. avoidance holds "for every time step ... for all
    i != j" and a failing pair zeroes both aircraft.  B breaks its
    envelope at step 0 (thrust above T_max) and keeps flying its own controls:
    its trajectory equals its trajectory flown alone.  At step 1 the pair is
    still 6 km apart; at step 2 B, now only a violator, comes within 2 P_r of A
    at the same altitude -- and A, which broke no bound of its own, is zeroed."""
    H = 6
    A = _dep(-8000.0, 0.0, 3000.0, 100.0, 0.0)         # flies East, trimmed
    B = _dep(0.0, 0.0, 3000.0, 100.0, math.pi)         # flies West
    both = _scenario([A, B], H)
    uA = _cruise_controls(ora, _scenario([A], H), 0, H, climb=0.0)
    uB = _cruise_controls(ora, _scenario([B], H), 0, H, climb=0.0)
    uB[0, 0] = 1.5 * both["T_max"][1]                  # envelope violation at step 0 only
    r = ora.Problem(both).rollout(np.stack([uA, uB]), 0, 0, 0, 1)
    ra = ora.Problem(_scenario([A], H)).rollout(uA[None], 0, 0, 0, 1)
    rb = ora.Problem(_scenario([B], H)).rollout(uB[None], 0, 0, 0, 1)
    # the simulation does not depend on the constraint outcomes
    assert np.array_equal(r["traj"][0], ra["traj"][0]) and np.array_equal(r["traj"][1], rb["traj"][0])
    assert ra["viol"][0] == 0 and rb["viol"][0] == 1
    gap = np.hypot(r["traj"][0, :, 0] - r["traj"][1, :, 0], r["traj"][0, :, 1] - r["traj"][1, :, 1])
    assert gap[1] > 2 * both["P_r"] and gap[2] < 2 * both["P_r"]   # first conflict after B's violating step
    assert r["viol"][0] == 1 and r["viol"][1] == 1
    # A's continuous outcome is untouched; only its weight is zeroed
    assert r["J"][0] == ra["J"][0] and np.array_equal(r["comp"][0], ra["comp"][0])


def test_violated_aircraft_conflicts_on_its_violating_step(ora):
    """A pair conflict on the violating step itself zeroes both (Eq. avoidance,
    P:303-309)."""
    H = 4
    A = _dep(-1200.0, 0.0, 3000.0, 100.0, 0.0)
    B = _dep(0.0, 0.0, 3000.0, 100.0, 0.0)
    both = _scenario([A, B], H)
    uA = _cruise_controls(ora, _scenario([A], H), 0, H, climb=0.0)
    uB = _cruise_controls(ora, _scenario([B], H), 0, H, climb=0.0)
    uB[0, 0] = 1.5 * both["T_max"][1]
    r = ora.Problem(both).rollout(np.stack([uA, uB]), 0, 0, 0, 1)
    assert r["viol"][0] == 1 and r["viol"][1] == 1


def test_violator_far_from_everyone_zeroes_only_itself(ora):
    """Per-aircraft weights: a violator that never comes near the
    others zeroes itself only; the others' outcomes equal their outcomes with
    the violator absent."""
    H = 6
    A = _dep(-12000.0, -9000.0, 1500.0, 110.0, 0.3)
    B = _dep(9000.0, 8000.0, 5500.0, 120.0, 2.0)
    uA = _cruise_controls(ora, _scenario([A], H), 0, H)
    uB = _cruise_controls(ora, _scenario([B], H), 0, H)
    uB[2, 2] = 2.0 * DEG * 4                          # |gamma| > gamma_max at step 2
    r = ora.Problem(_scenario([A, B], H)).rollout(np.stack([uA, uB]), 0, 0, 0, 1)
    ra = ora.Problem(_scenario([A], H)).rollout(uA[None], 0, 0, 0, 1)
    assert r["viol"].tolist() == [0, 1]
    assert r["J"][0] == ra["J"][0] and np.array_equal(r["traj"][0], ra["traj"][0])


# ---------------------------------------------------------------- R18
def test_post_landing_steps_score_best_cost(ora):
    """R18 closed form.  An arrival on the extended runway axis (y = 0) flying
    West on a 2 deg glide with beta_f = 1 deg lands at step j < H.  On the axis
    the heading target is West (chi_hat = pi + 2 atan2(0, x) = pi) and the arc
    length is x, so beta_t = atan2(z_t, x_t).  Steps after landing add zero
    deviation and no fuel, and every mean divides by H:
      heading  = 1 - sum_{t<=j} |wrap(chi_t - pi)| / (H pi)
      altitude = 1 - sum_{t<=j} |beta_t - beta_f| / (H max(beta_f, pi/2 - beta_f))
      fuel     = 1 - sum_{t<j} dt eta T_t / (dt H T_max eta)."""
    H, dt = 8, 10.0
    glide = 2.0 * DEG
    x0 = 5200.0
    arr = dict(kind=0, x0=[x0, 0.0, x0 * math.tan(glide), 75.0, math.pi, 64000.0], theta_F=0.0, z_tf=0.0,
               v_D=0.0, beta_f=1.0 * DEG, m_empty=60200.0)
    scn = _scenario([arr], H, dt)
    scn["density_mode"] = 1
    P = ora.Problem(scn)
    u = np.zeros((1, H, 3))
    u[0, :, 2] = -glide
    st = np.asarray(scn["x0"][0], dtype=np.float64).copy()
    for t in range(H):
        _, D = P.lift_drag(0, st, 0.0)
        u[0, t, 0] = D + st[5] * 9.81 * math.sin(-glide)
        st = P.step(0, st, u[0, t])
    r = P.rollout(u, 0, 0, 0, 1)
    j = int(r["landed_step"][0])
    assert 1 <= j < H and r["viol"][0] == 0
    tr = r["traj"][0]
    bf = 1.0 * DEG
    head = 1.0 - sum(abs(math.remainder(tr[t, 4] - math.pi, 2 * math.pi)) for t in range(1, j + 1)) / (H * math.pi)
    alt = 1.0 - sum(abs(math.atan2(tr[t, 2], tr[t, 0]) - bf) for t in range(1, j + 1)) / (
        H * max(bf, math.pi / 2 - bf))
    eta, Tmax = scn["eta"][0], scn["T_max"][0]
    fuel = 1.0 - sum(dt * eta * u[0, t, 0] for t in range(j)) / (dt * H * Tmax * eta)
    assert r["comp"][0, 0] == pytest.approx(head, abs=1e-9)
    assert r["comp"][0, 1] == pytest.approx(alt, abs=1e-9)
    assert r["comp"][0, 2] == pytest.approx(fuel, abs=1e-9)
    a = scn["alpha_arr"]
    assert r["J"][0] == pytest.approx(a[0] * head + a[1] * alt + a[2] * fuel, abs=1e-9)


# ---------------------------------------------------------------- R1
def _windy():
    scn = sc.snapshot(2, 2, seed=7)
    scn["nominal"] = [6.0, -2.0]
    scn["turb_sigma"] = 1.0
    return scn


def test_mh_zero_proposal_spread_always_accepts(ora):
    """R1 uses common random numbers: x' and x* are evaluated under the SAME
    wind and gust draws.  With sigma = 0 the proposal equals the resampled
    particle, so lambda* = lambda' exactly and every decision accepts
    (Delta = 0) -- in a windy scenario, where independent draws would make
    the two evaluations differ and reject about half the time."""
    P = ora.Problem(_windy())
    r = P.run_smc(L=96, S=3, K=5, seed=0x5EED0101, sigma=(0.0, 0.0, 0.0))
    assert r["rc"] == 0
    assert np.all(r["stats"][1:, 1] == 1.0)


def test_mh_with_zero_spread_reduces_to_paper_algorithm(ora):
    """With sigma = 0 the MH move (R1) and the paper's unconditional move
    (Alg.1 l.23, mh = 0) produce identical rounds: same best lambda every
    round and the same selected controls."""
    P = ora.Problem(_windy())
    a = P.run_smc(L=96, S=3, K=5, seed=0x5EED0102, sigma=(0.0, 0.0, 0.0), mh=True)
    b = P.run_smc(L=96, S=3, K=5, seed=0x5EED0102, sigma=(0.0, 0.0, 0.0), mh=False)
    assert np.array_equal(a["stats"][:, 0], b["stats"][:, 0])
    assert np.array_equal(a["best_ctrl"], b["best_ctrl"]) and a["best_index"] == b["best_index"]


def test_mh_rejects_only_worse_proposals(ora):
    """R1 never rejects an improving proposal: a spread large enough to push
    proposals out of the envelope (weight 0) gives acceptance strictly below 1,
    and every rejection is of a proposal with lower lambda (re-derived here
    from the oracle's own evaluations of both candidates)."""
    scn = _windy()
    P = ora.Problem(scn)
    L, S, k, seed = 128, 3, 1, 0x5EED0103
    cur = P.init_population(L, seed)
    sig = (0.3 * (scn["T_max"][0] - scn["T_min"][0]), 12 * DEG, 4 * DEG)
    prop = np.stack([np.stack([P.perturb_row(i, cur[l, i], l, k, seed, sig) for i in range(scn["n"])])
                     for l in range(L)])
    ec = P.evaluate(cur, S, k, seed)
    ep = P.evaluate(prop, S, k, seed)
    lc = np.where(np.isfinite(ec).all(1), ec.sum(1), -np.inf)
    lp = np.where(np.isfinite(ep).all(1), ep.sum(1), -np.inf)
    acc = np.array([ora.mh_accept(lc[l], lp[l], l, k, seed) for l in range(L)])
    assert 0 < acc.sum() < L
    assert np.all(lp[~acc] < lc[~acc])
