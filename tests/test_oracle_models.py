"""Pins for the oracle's models: dynamics (Eq. hor), wind (Eq. cov + AR(1)),
constraints, flow field / descent angle (Eq. flow) and objectives.

Each check pins the oracle to the paper or to mathematics: closed forms of the
difference equations, library factorisations, numerically integrated curves,
brute force on hand-built scenarios and the paper's printed anchors.
"""
import math

import numpy as np
import pytest

from paper_1506_02869_b200 import scenarios as sc

DEG = math.pi / 180.0


def _calm(scn):
    """No wind at all: zero random field, no nominal wind, no gusts."""
    scn = dict(scn)
    scn.update(sigma_lo=0.0, sigma_hi=0.0, nominal=[0.0, 0.0], turb_sigma=0.0)
    return scn


@pytest.fixture(scope="module")
def one_dep(ora):
    scn = _calm(sc.snapshot(0, 1, seed=1))
    scn["density_mode"] = 1
    return ora.Problem(scn)


# ---------------------------------------------------------------- dynamics
def test_lift_at_zero_bank(ora, one_dep):
    """L = m g = 588 600 N at phi = 0, m = 60 000 kg."""
    L, D = one_dep.lift_drag(0, [0, 0, 1000, 100, 0, 60000], 0.0)
    assert L == pytest.approx(588600.0, rel=1e-15)
    L2, D2 = one_dep.lift_drag(0, [0, 0, 1000, 100, 0, 60000], 0.3)
    L3, D3 = one_dep.lift_drag(0, [0, 0, 1000, 100, 0, 60000], -0.3)
    assert (L2, D2) == (L3, D3)                                  # even in phi
    assert L2 == pytest.approx(588600.0 / math.cos(0.3), rel=1e-15)


def test_drag_hand_value(ora, one_dep):
    """Parabolic polar at rho=1.225, v=100, S=122.6, CD0=0.024, CD2=0.0375,
    m=60000, phi=0: q = 750925 N, C_L = 588600/750925,
    D = q (0.024 + 0.0375 C_L^2) = 35 323.3599... N (exact rational evaluation)."""
    q = 0.5 * 1.225 * 100.0 ** 2 * 122.6
    assert q == 750925.0
    _, D = one_dep.lift_drag(0, [0, 0, 0, 100, 0, 60000], 0.0)
    assert D == pytest.approx(35323.359902786564, rel=1e-12)


def test_trimmed_level_flight(ora, one_dep):
    """gamma = phi = 0, T_k = D_k: v constant, x_k = x_0 + k dt v cos(chi),
    y, z unchanged, m_k = m_0 - dt eta sum_k T_k (Eq. hor)."""
    st = np.array([1000.0, -2000.0, 3000.0, 130.0, 0.7, 65000.0])
    x0 = st.copy()
    fuel = 0.0
    for k in range(1, 8):
        _, D = one_dep.lift_drag(0, st, 0.0)
        st = one_dep.step(0, st, [D, 0.0, 0.0])
        fuel += 10.0 * 1.0e-5 * D
        assert st[3] == pytest.approx(130.0, abs=1e-9)
        assert st[0] == pytest.approx(x0[0] + k * 10.0 * 130.0 * math.cos(0.7), abs=1e-7)
        assert st[1] == pytest.approx(x0[1] + k * 10.0 * 130.0 * math.sin(0.7), abs=1e-7)
        assert st[2] == x0[2] and st[4] == x0[4]
        assert st[5] == pytest.approx(x0[5] - fuel, abs=1e-9)


def test_zero_thrust_keeps_mass(ora, one_dep):
    st = one_dep.step(0, [0, 0, 3000, 130, 0.3, 65000], [0.0, 0.1, 0.02])
    assert st[5] == 65000.0


def test_constant_descent(ora, one_dep):
    """gamma = -3 deg, T_k = D_k + m g sin(gamma): v constant, z linear, m exact."""
    g = -3.0 * DEG
    st = np.array([0.0, 0.0, 3000.0, 120.0, 0.0, 64000.0])
    m0 = st[5]
    fuel = 0.0
    for k in range(1, 6):
        _, D = one_dep.lift_drag(0, st, 0.0)
        T = D + st[5] * 9.81 * math.sin(g)
        st = one_dep.step(0, st, [T, 0.0, g])
        fuel += 10.0 * 1e-5 * T
        assert st[3] == pytest.approx(120.0, abs=1e-9)
        assert st[2] == pytest.approx(3000.0 + k * 10.0 * 120.0 * math.sin(g), abs=1e-8)
        assert st[0] == pytest.approx(k * 10.0 * 120.0 * math.cos(g), abs=1e-8)
        assert st[5] == pytest.approx(m0 - fuel, abs=1e-9)


def test_coordinated_turn_rate(ora, one_dep):
    """Level turn at constant v: chi_k = chi_0 + k dt g tan(phi)/v (mass-free)."""
    phi = 25.0 * DEG
    st = np.array([0.0, 0.0, 2000.0, 120.0, 0.1, 64000.0])
    for k in range(1, 6):
        _, D = one_dep.lift_drag(0, st, phi)
        st = one_dep.step(0, st, [D, phi, 0.0])
        assert st[4] == pytest.approx(0.1 + k * 10.0 * 9.81 * math.tan(phi) / 120.0, abs=1e-12)
    assert 10.0 * 9.81 * math.tan(phi) / 120.0 / DEG == pytest.approx(21.84, abs=0.01)


def test_wind_offset_and_ground_speed(ora, one_dep):
    """Eq. hor a,b: the wind adds w dt; |ground - wind| = v cos(gamma)."""
    st = np.array([0.0, 0.0, 2000.0, 110.0, 1.1, 64000.0])
    u = [40000.0, 0.1, 0.05]
    a = one_dep.step(0, st, u, (0.0, 0.0))
    b = one_dep.step(0, st, u, (7.0, -3.0))
    assert b[0] - a[0] == pytest.approx(70.0, abs=1e-9)
    assert b[1] - a[1] == pytest.approx(-30.0, abs=1e-9)
    assert np.all(a[2:] == b[2:])
    gs = math.hypot((b[0] - st[0]) / 10.0 - 7.0, (b[1] - st[1]) / 10.0 + 3.0)
    assert gs == pytest.approx(110.0 * math.cos(0.05), rel=1e-12)


def test_isa_density_mode(ora):
    scn = _calm(sc.snapshot(0, 1, seed=1))
    P = ora.Problem(scn)
    # sea level ISA gives the constant-density drag
    scn2 = dict(scn); scn2["density_mode"] = 1
    P2 = ora.Problem(scn2)
    assert P.lift_drag(0, [0, 0, 0, 100, 0, 60000], 0.0) == P2.lift_drag(0, [0, 0, 0, 100, 0, 60000], 0.0)
    # drag decreases with altitude at fixed v (thinner air, P:255 'standard relations')
    d = [P.lift_drag(0, [0, 0, z, 200, 0, 60000], 0.0)[1] for z in (0, 4000, 8000)]
    assert d[0] > d[1] > d[2]


# ---------------------------------------------------------------- wind model
def test_covariance_and_cholesky(ora):
    scn = sc.base_scenario()
    scn = sc._finish(scn, [sc._departure_snapshot(0)])
    P = ora.Problem(scn)
    R, Q = P.Rhat, P.Qhat
    # Eq. cov at the same point: sigma(z)^2; symmetric; decays with distance
    sig = np.array([1.5, 1.5, 1.5, 1.5, 4.0, 4.0, 4.0, 4.0])
    assert np.allclose(np.diag(R), sig ** 2, rtol=1e-15)
    assert np.allclose(R, R.T, rtol=0, atol=0)
    assert R[0, 1] == pytest.approx(1.5 * 1.5 * math.exp(-1.6e-6 * 60000.0), rel=1e-14)
    assert R[0, 3] == pytest.approx(2.25 * math.exp(-1.6e-6 * 60000.0 * math.sqrt(2)), rel=1e-14)
    assert R[0, 4] == pytest.approx(1.5 * 4.0 * math.exp(-1.5e-5 * 12000.0), rel=1e-14)
    # Qhat Qhat^T = Rhat, lower triangular, equals LAPACK's factor
    assert np.allclose(Q @ Q.T, R, rtol=0, atol=1e-12)
    assert np.all(np.triu(Q, 1) == 0.0)
    assert np.allclose(Q, np.linalg.cholesky(R), rtol=0, atol=1e-12)
    a, b = P.ab
    assert a == pytest.approx(math.exp(-6e-6 * 10.0), rel=1e-15)
    # Q Q^T = (1-a^2) Rhat with Q = b Qhat
    assert np.allclose((b * Q) @ (b * Q).T, (1 - a * a) * R, rtol=0, atol=1e-15)


def test_trilinear_nodes_linear_fields_clamp(ora):
    scn = sc._finish(sc.base_scenario(), [sc._departure_snapshot(0)])
    P = ora.Problem(scn)
    lo, hi = np.array(scn["wind_lo"]), np.array(scn["wind_hi"])
    rng = np.random.default_rng(5)
    W = rng.normal(size=8)
    for n in range(8):
        pos = [hi[a] if (n >> a) & 1 else lo[a] for a in range(3)]
        assert P.trilinear(W, pos) == pytest.approx(W[n], abs=1e-15)
    c = rng.normal(size=4)
    lin = lambda p: c[0] + c[1] * p[0] / 1e4 + c[2] * p[1] / 1e4 + c[3] * p[2] / 1e4
    Wl = [lin([hi[a] if (n >> a) & 1 else lo[a] for a in range(3)]) for n in range(8)]
    for _ in range(50):
        p = rng.uniform(lo, hi)
        assert P.trilinear(Wl, p) == pytest.approx(lin(p), abs=1e-12)
    # outside the box: clamped to the boundary value
    assert P.trilinear(Wl, [1e6, 0.0, 5000.0]) == pytest.approx(lin([hi[0], 0.0, 5000.0]), abs=1e-12)


def test_wind_field_statistics(ora):
    """Stationary N(0, Rhat) field: sample covariance of W(0) over many
    (particle, sample) draws matches Rhat within 5% of max|Rhat|."""
    scn = _calm(sc.snapshot(0, 1, seed=1))
    scn.update(sigma_lo=1.5, sigma_hi=4.0)
    scn["x0"][0] = [-30000.0, -30000.0, 0.0, 130.0, 0.0, 70000.0]      # sits on node 0
    P = ora.Problem(scn)
    # a zero-thrust 1-step rollout exposes the node-0 wind through x1 - x0 - v dt cos
    u = np.zeros((1, P.H, 3))
    vals = []
    for l in range(4000):
        tr = P.rollout(u, l, 0, 0, 77)["traj"][0]
        vals.append((tr[1, 0] - tr[0, 0] - 10 * 130.0) / 10.0)
    vals = np.array(vals)
    assert vals.mean() == pytest.approx(0.0, abs=4 * 1.5 / math.sqrt(len(vals)))
    assert vals.var() == pytest.approx(1.5 ** 2, rel=0.08)


# ---------------------------------------------------------------- constraints
def test_envelope_boundaries(ora, one_dep):
    P = one_dep
    st = [0, 0, 3000, 130, 0, 65000]
    assert not P.unary_violation(0, [60000, 0.1, 0.01], st)
    assert P.unary_violation(0, [60000, 30 * DEG, 0.0], st)          # |phi| < phi_max strict
    assert P.unary_violation(0, [60000, -30 * DEG, 0.0], st)
    assert not P.unary_violation(0, [1.2e5, 0.0, 6 * DEG], st)      # T = T_max, gamma = gamma_max inclusive
    assert P.unary_violation(0, [1.2e5 + 1, 0.0, 0.0], st)
    assert P.unary_violation(0, [-1, 0.0, 0.0], st)
    assert not P.unary_violation(0, [0, 0, 0], [0, 0, 12000, 180, 0, 58000])   # inclusive bounds
    assert P.unary_violation(0, [0, 0, 0], [0, 0, 12000.01, 180, 0, 58000])
    assert P.unary_violation(0, [0, 0, 0], [0, 0, 100, 69.99, 0, 65000])
    assert P.unary_violation(0, [0, 0, 0], [0, 0, 100, 100, 0, 57999.99])      # m >= m_empty
    assert P.unary_violation(0, [0, 0, 0], [0, 0, float("nan"), 100, 0, 65000])


def test_separation_boundaries(ora, one_dep):
    P = one_dep
    a = np.array([0, 0, 3000, 100, 0, 1])
    assert not P.pair_conflict(a, a + [5000, 0, 0, 0, 0, 0])       # exactly 2 P_r
    assert P.pair_conflict(a, a + [4999.9, 0, 0, 0, 0, 0])
    assert P.pair_conflict(a, a)                                     # co-located
    assert not P.pair_conflict(a, a + [0, 0, 600, 0, 0, 0])        # |dz| = 2 P_h
    assert P.pair_conflict(a, a + [3000, 3000, 599, 0, 0, 0])
    rng = np.random.default_rng(6)
    for _ in range(200):
        b = a + np.r_[rng.uniform(-8000, 8000, 2), rng.uniform(-900, 900), 0, 0, 0]
        assert P.pair_conflict(a, b) == P.pair_conflict(b, a)      # symmetric


def test_landing_sector(ora, one_dep):
    P = one_dep
    on = [2000.0, 0.0, 2000.0 * math.tan(3 * DEG), 75.0, math.pi, 64000.0]
    assert P.landed(on)
    assert not P.landed([*on[:4], 0.0, 64000.0])                    # flying away
    assert P.landed([*on[:4], math.pi + 14.9999 * DEG, 64000.0])     # heading bound
    assert not P.landed([*on[:4], math.pi + 15.01 * DEG, 64000.0])
    assert P.landed([*on[:3], 80.0, *on[4:]])                       # v = P_vs inclusive
    assert not P.landed([*on[:3], 80.01, *on[4:]])
    assert not P.landed([-2000.0, 0.0, 100.0, 75.0, math.pi, 64000.0])   # west of runway (R10)
    assert not P.landed([4100.0, 0.0, 100.0, 75.0, math.pi, 64000.0])    # beyond P_runway
    assert not P.landed([2000.0, 0.0, 2000 * math.tan(6.5 * DEG), 75.0, math.pi, 64000.0])  # too high
    # monotone in v_s
    for v in np.linspace(60, 80, 9):
        assert P.landed([*on[:3], v, *on[4:]])


# ---------------------------------------------------------------- flow field
def test_flow_field_special_points(ora):
    w = lambda a: a % (2 * math.pi)
    assert w(ora.flow_heading(5000, 0)) == pytest.approx(math.pi)          # east of runway: head West
    assert w(ora.flow_heading(0, 5000)) == pytest.approx(0.0, abs=1e-12)   # north: head East
    assert w(ora.flow_heading(-5000, 0)) == pytest.approx(math.pi)         # due West: long diversion
    assert w(ora.flow_heading(3000, 3000)) == pytest.approx(1.5 * math.pi)  # x = y > 0: head South


def _follow(ora, x, y, h=5.0):
    """Integrate dx/ds = (cos chi_hat, sin chi_hat) until within 50 m of the origin."""
    s = 0.0
    for _ in range(200000):
        r = math.hypot(x, y)
        if r < 50.0:
            return s + r, ora.flow_heading(x, y)
        c = ora.flow_heading(x, y)
        # midpoint (RK2) step
        xm, ym = x + 0.5 * h * math.cos(c), y + 0.5 * h * math.sin(c)
        cm = ora.flow_heading(xm, ym)
        x, y, s = x + h * math.cos(cm), y + h * math.sin(cm), s + h
    raise AssertionError("did not converge")


@pytest.mark.parametrize("start", [(20000, 5000), (10000, 15000), (-5000, 20000), (8000, -12000), (-15000, -9000)])
def test_flow_field_reaches_runway_heading_west_and_arc_length(ora, start):
    """Following chi_hat reaches the origin on the east side heading West,
    and the distance flown equals the arc length used in beta (R9)."""
    s_num, chi_end = _follow(ora, *start)
    assert ora.angdist(chi_end - math.pi) < 0.05
    assert s_num == pytest.approx(ora.arc_length(*start), rel=2e-3)


def test_beta_limits(ora):
    assert ora.beta(12000, 5000, 0.0) == 0.0
    assert ora.beta(10000, 0, 10000 * math.tan(0.05)) == pytest.approx(0.05, rel=1e-12)
    assert ora.arc_length(10000, 0) == 10000
    assert ora.arc_length(0, 10000) == pytest.approx(10000 * math.pi / 2, rel=1e-12)   # quarter circle x2


# ---------------------------------------------------------------- objectives
def _radial_departure(ora, theta_F, bearing, H=6):
    scn = _calm(sc.snapshot(0, 1, seed=1, H=H))
    scn["x0"][0] = [5000 * math.cos(bearing), 5000 * math.sin(bearing), 1000.0, 150.0, bearing, 70000.0]
    scn["theta_F"][0] = theta_F
    return ora.Problem(scn)


def test_departure_bearing_anchors(ora):
    """on-bearing every step -> J1 = 1; 90 deg off every step -> 0.5."""
    b = 30 * DEG
    P = _radial_departure(ora, b, b)
    u = np.zeros((1, 6, 3))
    u[..., 0] = 38000.0
    r = P.rollout(u, 0, 0, 0, 1)
    assert r["comp"][0, 0] == pytest.approx(1.0, abs=1e-12)
    P = _radial_departure(ora, b + 90 * DEG, b)
    r = P.rollout(u, 0, 0, 0, 1)
    assert r["comp"][0, 0] == pytest.approx(0.5, abs=1e-12)


def test_fuel_term_zero_fuel_and_full_thrust(ora):
    P = _radial_departure(ora, 0.0, 0.0)
    u = np.zeros((1, 6, 3))
    r = P.rollout(u, 0, 0, 0, 1)
    assert r["comp"][0, 1] == 1.0 and r["fuel"][0] == 0.0
    P1 = _radial_departure(ora, 0.0, 0.0, H=1)
    u1 = np.zeros((1, 1, 3)); u1[..., 0] = 1.2e5
    r = P1.rollout(u1, 0, 0, 0, 1)
    assert not r["viol"][0]
    assert r["comp"][0, 1] == pytest.approx(0.0, abs=1e-12)         # T_max over the whole horizon
    assert r["fuel"][0] == pytest.approx(10 * 1e-5 * 1.2e5, rel=1e-14)


def test_noise_term_and_popdense(ora):
    scn = _calm(sc.snapshot(0, 1, seed=1))
    scn["centres"] = np.array([[5000.0, 0.0, 1500.0]])
    scn.update(noise_w=0.2, pop_nx=41, pop_ny=41, pop_x0=-20000.0, pop_y0=-20000.0, pop_dx=1000.0)
    P = ora.Problem(scn)
    assert P.popdense(5000, 0, grid=False) == pytest.approx(0.2659615202676218, rel=1e-14)  # P:1133, c = 1.5 km
    assert P.popdense(5000, 0, grid=True) == pytest.approx(0.2659615202676218, rel=1e-14)   # on a grid node
    assert P.popdense(40000, 40000, grid=False) < 1e-30
    scn2 = dict(scn); scn2["centres"] = np.array([[0.0, 0.0, 300.0]])
    assert ora.Problem(scn2).popdense(0, 0, grid=False) == 1.0      # clipped at 1
    g = P.pop_grid()
    assert g.shape == (41, 41) and g.max() <= 1.0 and g.min() >= 0.0
    # J_noise = 1 above A_c regardless of density: a level departure at
    # 5000 m over the centre has mean noise term 1 -> J = 0.8 J^D + 0.2
    scn3 = dict(scn)
    scn3["x0"] = np.array([[3000.0, 0.0, 5000.0, 150.0, 0.0, 70000.0]])
    P3 = ora.Problem(scn3)
    u = np.zeros((1, 6, 3)); u[..., 0] = 50000.0
    r = P3.rollout(u, 0, 0, 0, 1)
    a = np.array(scn["alpha_dep"])
    JD = float(a @ r["comp"][0])
    assert r["J"][0] == pytest.approx(0.8 * JD + 0.2, abs=1e-12)


def test_costs_in_unit_interval(ora):
    """Every component and total in [0,1]."""
    scn, _ = sc.config(2)
    P = ora.Problem(scn)
    ctrl = sc.random_controls(scn, 300, seed=9, spread=1.3)
    for l in range(300):
        r = P.rollout(ctrl[l], l, 0, 0, 3)
        assert np.all((r["J"] >= 0) & (r["J"] <= 1))
        assert np.all((r["comp"] >= 0) & (r["comp"] <= 1))


# ---------------------------------------------------------------- denser wind grids (N3)
def _grid_nodes(scn, nx, ny, nz):
    lo, hi = np.array(scn["wind_lo"]), np.array(scn["wind_hi"])
    pts = []
    for iz in range(nz):
        for iy in range(ny):
            for ix in range(nx):
                pts.append(lo + (hi - lo) * np.array([ix / (nx - 1), iy / (ny - 1), iz / (nz - 1)]))
    return np.array(pts)


def test_dense_grid_covariance(ora):
    """N_x N_y N_z grid: Rhat entries are Eq. cov at the evenly
    spaced grid points, node n = ix + N_x (iy + N_y iz); Qhat is its Cholesky factor."""
    scn = sc._finish(sc.base_scenario(), [sc._departure_snapshot(0)])
    scn["wind_n"] = (3, 4, 2)
    P = ora.Problem(scn)
    assert P.wind_grid == (3, 4, 2)
    R, Q = P.Rhat, P.Qhat
    assert R.shape == (24, 24)
    pts = _grid_nodes(scn, 3, 4, 2)
    zlo, zhi = scn["wind_lo"][2], scn["wind_hi"][2]
    sig = lambda z: scn["sigma_lo"] + (scn["sigma_hi"] - scn["sigma_lo"]) * (z - zlo) / (zhi - zlo)
    for a in range(24):
        for b in range(24):
            d = pts[a] - pts[b]
            ref = sig(pts[a][2]) * sig(pts[b][2]) * math.exp(-scn["beta_w"] * math.hypot(d[0], d[1])) \
                * math.exp(-scn["gamma_w"] * abs(d[2]))
            assert R[a, b] == pytest.approx(ref, rel=1e-13)
    assert np.allclose(Q, np.linalg.cholesky(R), rtol=0, atol=1e-12)


def test_dense_grid_trilinear(ora):
    """Cell-wise trilinear interpolation on a 4x3x3 grid: node values at nodes, exact
    for any globally trilinear field (a + b x + ... + h x y z), clamped outside."""
    scn = sc._finish(sc.base_scenario(), [sc._departure_snapshot(0)])
    scn["wind_n"] = (4, 3, 3)
    P = ora.Problem(scn)
    pts = _grid_nodes(scn, 4, 3, 3)
    rng = np.random.default_rng(3)
    W = rng.normal(size=len(pts))
    for n in (0, 5, 17, 35):
        assert P.trilinear(W, pts[n]) == pytest.approx(W[n], abs=1e-14)
    c = rng.normal(size=8)
    f = lambda p: (c[0] + c[1] * p[0] / 1e4 + c[2] * p[1] / 1e4 + c[3] * p[2] / 1e4 + c[4] * p[0] * p[1] / 1e8
                   + c[5] * p[0] * p[2] / 1e8 + c[6] * p[1] * p[2] / 1e8 + c[7] * p[0] * p[1] * p[2] / 1e12)
    Wf = np.array([f(p) for p in pts])
    lo, hi = np.array(scn["wind_lo"]), np.array(scn["wind_hi"])
    for _ in range(100):
        p = rng.uniform(lo, hi)
        assert P.trilinear(Wf, p) == pytest.approx(f(p), abs=1e-10)
    # a field that is trilinear per cell only: piecewise values differ from the global fit
    Wk = np.abs(pts[:, 0] - pts[1, 0])                    # kink at the second x-node
    mid = (pts[0] + pts[1]) / 2
    assert P.trilinear(Wk, mid) == pytest.approx(abs(mid[0] - pts[1, 0]), rel=1e-12)
    assert P.trilinear(Wf, [1e7, -1e7, 1e7]) == pytest.approx(f([hi[0], lo[1], hi[2]]), abs=1e-10)


def test_dense_grid_field_statistics(ora):
    """W(0) at an interior grid point of a 3x3x3 grid is N(0, sigma(z)^2): the
    normal -> (component, node) mapping and the Qhat rows."""
    scn = _calm(sc.snapshot(0, 1, seed=1))
    scn.update(sigma_lo=1.5, sigma_hi=4.0, wind_n=(3, 3, 3))
    mid = _grid_nodes(scn, 3, 3, 3)[13]                   # centre node
    scn["x0"][0] = [mid[0], mid[1], mid[2], 130.0, 0.0, 70000.0]
    P = ora.Problem(scn)
    zlo, zhi = scn["wind_lo"][2], scn["wind_hi"][2]
    s_mid = 1.5 + 2.5 * (mid[2] - zlo) / (zhi - zlo)
    u = np.zeros((1, P.H, 3))
    vals = []
    for l in range(4000):
        tr = P.rollout(u, l, 0, 0, 91)["traj"][0]
        vals.append((tr[1, 1] - tr[0, 1]) / 10.0)           # y component: heading 0 -> no airspeed in y
    vals = np.array(vals)
    assert vals.mean() == pytest.approx(0.0, abs=4 * s_mid / math.sqrt(len(vals)))
    assert vals.var() == pytest.approx(s_mid ** 2, rel=0.08)


# ---------------------------------------------------------------- fuel estimators (section 5, N4)
def _fuel_forward(P, i, x0, T, gam, wind, dt, Cf):
    """Forward Euler of Eq. hor with zero bank and eta(v) = Cf1 (1 + v/Cf2)
    (P:709): the trace a recorder would see, and the true mass series."""
    st = np.array(x0, float)
    tr, ms = [st[:5].copy()], [st[5]]
    for k in range(len(T)):
        x, y, z, v, chi, m = st
        _, D = P.lift_drag(i, st, 0.0)
        eta = Cf[0] * (1.0 + v / Cf[1])
        st = np.array([x + dt * (v * math.cos(chi) * math.cos(gam[k]) + wind[0]),
                       y + dt * (v * math.sin(chi) * math.cos(gam[k]) + wind[1]),
                       z + dt * v * math.sin(gam[k]),
                       v + dt * ((T[k] - D) / m - 9.81 * math.sin(gam[k])),
                       chi, m - dt * eta * T[k]])
        tr.append(st[:5].copy())
        ms.append(st[5])
    return np.array(tr), np.array(ms)


def test_fuel_estimate1_roundtrip(ora):
    """Estimate 1 inverts the forward model: a trace simulated with known thrust and a
    constant wind gives back the wind (residuals) and the mass series."""
    scn = sc.snapshot(0, 1, seed=1)
    scn["density_mode"] = 0
    P = ora.Problem(scn)
    rng = np.random.default_rng(2)
    K, dt, Cf = 25, 60.0, (1.1e-5, 500.0)
    T = rng.uniform(3e4, 9e4, K)
    gam = rng.uniform(-0.03, 0.05, K)
    tr, ms = _fuel_forward(P, 0, [-5000.0, 2000.0, 3000.0, 150.0, 0.7, 70000.0], T, gam, (4.5, -2.25), dt, Cf)
    m, w, fl = P.fuel_estimate1(0, tr, dt, ms[0], Cf)
    assert fl == 0
    assert np.allclose(m, ms, rtol=1e-9, atol=0)
    assert np.allclose(w[:-1], [4.5, -2.25], rtol=0, atol=1e-6)
    assert np.all(w[-1] == 0.0)
    # zero thrust: no burn (the estimate sees T = 0 up to rounding; negative burn clamped)
    tr0, ms0 = _fuel_forward(P, 0, [0.0, 0.0, 3000.0, 150.0, 0.0, 70000.0], np.zeros(5), np.zeros(5), (0.0, 0.0), dt, Cf)
    m0, _, _ = P.fuel_estimate1(0, tr0, dt, ms0[0], Cf)
    assert np.allclose(m0, 70000.0, rtol=1e-12)


def test_fuel_estimate2_properties(ora):
    scn = sc.snapshot(0, 1, seed=1)
    P = ora.Problem(scn)
    dt, Cf = 60.0, (1.1e-5, 500.0)
    # straight, level, constant speed, no wind: both estimates reduce to trimmed flight
    v, chi = 160.0, 0.4
    tr = np.array([[k * dt * v * math.cos(chi), k * dt * v * math.sin(chi), 4000.0, v, chi] for k in range(6)])
    m1, _, f1 = P.fuel_estimate1(0, tr, dt, 68000.0, Cf)
    m2, f2 = P.fuel_estimate2(0, tr, dt, 68000.0, Cf)
    assert f1 == 0 and f2 == 0
    assert np.allclose(m2, m1, rtol=1e-12)
    assert m1[-1] < 68000.0                                       # level flight burns fuel against drag
    # circling: same position every sample -> zero-distance intervals flagged, no burn
    circ = np.array([[1000.0, 2000.0, 3000.0, 140.0, 0.3 * k] for k in range(4)])
    m3, f3 = P.fuel_estimate2(0, circ, dt, 68000.0, Cf)
    assert f3 & 2 and np.all(m3 == 68000.0)
    # implausible climb (dz > dt v): gamma clamped to gamma_max and flagged
    bad = np.array([[0.0, 0.0, 0.0, 10.0, 0.0], [600.0, 0.0, 5000.0, 10.0, 0.0]])
    _, _, f4 = P.fuel_estimate1(0, bad, dt, 68000.0, Cf)
    assert f4 & 1


# ---------------------------------------------------------------- ISA density (R12)
@pytest.mark.parametrize("z,rho", [(0.0, 1.2250), (5000.0, 0.73643), (11000.0, 0.36392)])
def test_isa_density_table_values(ora, z, rho):
    """The drag model's density is the ICAO standard atmosphere (troposphere):
    tabulated 1.2250 / 0.73643 / 0.36392 kg m^-3 at 0 / 5 / 11 km.  Exposed through
    the parabolic polar: D = q (C_D0 + C_D2 C_L^2), q = rho v^2 S / 2, C_L = m g / q."""
    scn = _calm(sc.snapshot(0, 1, seed=1))
    P = ora.Problem(scn)
    v, m = 160.0, 62000.0
    _, D = P.lift_drag(0, [0, 0, z, v, 0, m], 0.0)
    q = 0.5 * rho * v * v * scn["S"][0]
    cl = m * scn["g"] / q
    assert D == pytest.approx(q * (scn["cd0"][0] + scn["cd2"][0] * cl * cl), rel=2e-4)


# ---------------------------------------------------------------- AR(1) for t >= 1
def _node0_wind_series(ora, lam, L=3000, H=6):
    """The x wind at grid node 0 for steps t = 0..H-1 of L independent samples.  The
    aircraft flies level at z = 0 heading South-West from the corner (-30 km, -30 km):
    its clamped position is node 0 every step (R14), so w_x(t) = (x_{t+1} - x_t)/dt -
    v_t cos(chi) (Eq. hor a with gamma = 0)."""
    scn = _calm(sc.snapshot(0, 1, seed=1, H=H))
    scn.update(sigma_lo=1.5, sigma_hi=4.0, lambda_t=lam)
    chi = -0.75 * math.pi
    scn["x0"][0] = [-30000.0, -30000.0, 0.0, 130.0, chi, 70000.0]
    P = ora.Problem(scn)
    u = np.zeros((1, H, 3))
    u[..., 0] = 30000.0
    out = np.zeros((L, H))
    for l in range(L):
        tr = P.rollout(u, l, 0, 0, 1234)["traj"][0]
        out[l] = (tr[1:, 0] - tr[:-1, 0]) / scn["dt"] - tr[:-1, 3] * math.cos(chi)
    return out, P


def test_ar1_stationary_variance_and_lag_correlation(ora):
    """W(t) = a W(t-1) + Q v(t), Q = sqrt(1 - a^2) Qhat keeps the field
    stationary: Var W(t) = sigma(z)^2 at every step, Corr(W(t), W(t+1)) = a,
    Corr(W(t), W(t+2)) = a^2, with a = exp(-lambda dt) (R14).  A large lambda
    (a = e^{-0.5}) makes the pin sharp: dropping the innovation (b) decays the
    variance as a^{2t}, dropping the carry (a) zeroes the correlation."""
    lam = 0.05
    w, P = _node0_wind_series(ora, lam)
    a, b = P.ab
    assert a == pytest.approx(math.exp(-lam * 10.0), rel=1e-15) and b == pytest.approx(math.sqrt(1 - a * a), rel=1e-15)
    n = w.shape[0]
    for t in range(w.shape[1]):
        assert w[:, t].var() == pytest.approx(1.5 ** 2, rel=0.09), t
        assert abs(w[:, t].mean()) < 4 * 1.5 / math.sqrt(n)
    c1 = np.mean([np.corrcoef(w[:, t], w[:, t + 1])[0, 1] for t in range(5)])
    c2 = np.mean([np.corrcoef(w[:, t], w[:, t + 2])[0, 1] for t in range(4)])
    assert c1 == pytest.approx(a, abs=0.03)
    assert c2 == pytest.approx(a * a, abs=0.03)


def test_ar1_slow_field_is_nearly_frozen(ora):
    """At the paper's lambda = 6e-6 s^-1 (R14) a = 0.99994: successive steps of a
    sample see almost the same field (the forecast error drifts slowly)."""
    w, P = _node0_wind_series(ora, 6e-6, L=400)
    d = w[:, 1:] - w[:, :-1]
    assert np.sqrt(np.mean(d * d)) < 0.05 * 1.5


# ---------------------------------------------------------------- departure altitude and speed terms
def _level_departure(ora, H, z0, v, climb=0.0, zt=6000.0):
    scn = _calm(sc.snapshot(0, 1, seed=1, H=H))
    scn["density_mode"] = 1
    scn["x0"][0] = [3000.0, 0.0, z0, v, 0.0, 70000.0]
    scn["theta_F"][0] = 0.0
    scn["z_tf"][0] = zt
    P = ora.Problem(scn)
    u = np.zeros((1, H, 3))
    st = scn["x0"][0].copy()
    for t in range(H):                              # trimmed: airspeed constant (Eq. hor d)
        _, D = P.lift_drag(0, st, 0.0)
        u[0, t] = [D + st[5] * 9.81 * math.sin(climb), 0.0, climb]
        st = P.step(0, st, u[0, t])
    return scn, P, u


def test_departure_altitude_term_level_flight_is_one_half(ora):
    """Departure altitude term B with the reachability sup/inf (R21): per
    step j the reachable band is z0 +- j dt v_max sin(gamma_max); a level departure
    below the band-limited target deviates by z_tf - z0 every step, and
    sup_j = z_tf - z0 + r_j, inf_j = z_tf - z0 - r_j give J3 = (mean r)/(2 mean r) = 1/2."""
    H = 6
    scn, P, u = _level_departure(ora, H, 3000.0, 150.0)
    r = P.rollout(u, 0, 0, 0, 1)
    reach = np.array([j * scn["dt"] * scn["v_max"][0] * math.sin(scn["gamma_max"][0]) for j in range(1, H + 1)])
    assert reach.max() < 3000.0                      # the band stays inside [z_min, z_tf]
    supB, infB = P.supinfB()
    assert supB[0] == pytest.approx(3000.0 + reach.mean(), rel=1e-12)
    assert infB[0] == pytest.approx(3000.0 - reach.mean(), rel=1e-12)
    assert r["comp"][0, 2] == pytest.approx(0.5, abs=1e-12)


def test_departure_altitude_term_max_climb_is_one(ora):
    """Climbing at gamma_max with v = v_max every step reaches the top of the reachable
    band, z_j = z0 + j dt v_max sin(gamma_max) = the inf of the deviation: J3 = 1."""
    H = 5
    scn, P, u = _level_departure(ora, H, 3000.0, 180.0, climb=6.0 * DEG)
    r = P.rollout(u, 0, 0, 0, 1)
    assert r["comp"][0, 2] == pytest.approx(1.0, abs=1e-9)


@pytest.mark.parametrize("v,expect", [(150.0, 1.0), (110.0, 0.5), (130.0, 0.75)])
def test_departure_speed_term(ora, v, expect):
    """Speed term C at constant airspeed: J4 = 1 - |v - v_D| / sup_C with
    sup_C = max(v_max - v_D, v_D - v_min) = max(30, 80) = 80 m/s (R21)."""
    scn, P, u = _level_departure(ora, 6, 3000.0, v)
    r = P.rollout(u, 0, 0, 0, 1)
    assert r["comp"][0, 3] == pytest.approx(expect, abs=1e-9)


def test_fuel_estimates_never_gain_weight(ora):
    """"aircraft were restricted from burning negative fuel and gaining weight":
    the mass series of both estimates is non-increasing, also across an interval whose
    burn is undefined (a recorded airspeed missing as NaN gives T = NaN) -- that
    interval burns nothing and the series continues from the same mass (R47)."""
    scn = sc.snapshot(0, 1, seed=1)
    P = ora.Problem(scn)
    dt, Cf = 60.0, (1.1e-5, 500.0)
    rng = np.random.default_rng(4)
    tr = np.zeros((12, 5))
    st = np.array([0.0, 0.0, 3000.0, 150.0, 0.2])
    for k in range(12):
        tr[k] = st
        st = st + [dt * st[3] * math.cos(st[4]), dt * st[3] * math.sin(st[4]), rng.normal(0, 100),
                   rng.normal(0, 15), rng.normal(0, 0.05)]
    tr[5, 3] = float("nan")
    m1, _, _ = P.fuel_estimate1(0, tr, dt, 68000.0, Cf)
    m2, _ = P.fuel_estimate2(0, tr, dt, 68000.0, Cf)
    for m in (m1, m2):
        assert np.all(np.isfinite(m)) and np.all(np.diff(m) <= 0.0)
    assert m1[5] == m1[6] or m1[4] == m1[5]          # the NaN sample's interval burns nothing
