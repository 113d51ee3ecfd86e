"""FP64 CPU oracle for the SMC-in-MPC hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product package ``paper_1506_02869_b200`` never imports it, and the two share
no code: this is a ctypes binding over ``oracle/smc_oracle.c`` (plain C,
FP64), written from PAPER.md (Eele & Maciejowski 2015) and pinned by the
``-m "not gpu"`` tests under ``tests/test_oracle_*.py``.

Parity status: see the header of ``smc_oracle.c``.  The rolling-window
averaging (R20), post-landing bonus (R18), constraint handling after a
violation (Alg.1 l.11-13: the violator keeps flying and stays in
every pair test) and the MH move (R1) are conventions the paper states in
prose; they are pinned by invariants and closed forms in
``tests/test_oracle_conventions.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "smc_oracle.h"))):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = C.CDLL(_LIB)
            _declare(_lib)
    return _lib


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class _Problem(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("H", C.c_int32), ("dt", C.c_double), ("g", C.c_double),
        ("density_mode", C.c_int32), ("rho_const", C.c_double),
        ("kind", _ip), ("first_step", _ip), ("x0", _dp),
        ("theta_F", _dp), ("z_tf", _dp), ("v_D", _dp), ("beta_f", _dp),
        ("S", _dp), ("cd0", _dp), ("cd2", _dp), ("eta", _dp), ("m_empty", _dp),
        ("T_min", _dp), ("T_max", _dp), ("v_min", _dp), ("v_max", _dp),
        ("gamma_max", _dp), ("phi_max", _dp), ("z_min", _dp), ("z_max", _dp),
        ("P_runway", C.c_double), ("P_beta", C.c_double), ("P_chi", C.c_double),
        ("P_vs", C.c_double), ("P_r", C.c_double), ("P_h", C.c_double),
        ("alpha_dep", C.c_double * 4), ("alpha_arr", C.c_double * 3),
        ("noise_w", C.c_double), ("A_c", C.c_double),
        ("n_centres", C.c_int32), ("centres", _dp),
        ("pop_nx", C.c_int32), ("pop_ny", C.c_int32),
        ("pop_x0", C.c_double), ("pop_y0", C.c_double), ("pop_dx", C.c_double),
        ("wind_lo", C.c_double * 3), ("wind_hi", C.c_double * 3),
        ("sigma_lo", C.c_double), ("sigma_hi", C.c_double),
        ("beta_w", C.c_double), ("gamma_w", C.c_double), ("lambda_t", C.c_double),
        ("nominal", C.c_double * 2), ("turb_sigma", C.c_double), ("tma_radius", C.c_double),
        ("wind_n", C.c_int32 * 3),
    ]


class _Derived(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("ng", C.c_int32),
                ("Rhat", C.c_double * 4096), ("Qhat", C.c_double * 4096), ("a", C.c_double),
                ("b", C.c_double), ("supB", C.c_double * 64), ("infB", C.c_double * 64),
                ("pop", _dp)]


class _RollOut(C.Structure):
    _fields_ = [("J", _dp), ("comp", _dp), ("traj", _dp), ("fuel", _dp), ("margin", _dp), ("margin_land", _dp),
                ("viol", _ip), ("landed_step", _ip), ("replayed", _ip)]


class _Replay(C.Structure):
    _fields_ = [("landed_step", _ip), ("viol", _ip), ("eps", C.c_double)]


class _SmcCfg(C.Structure):
    _fields_ = [("L", C.c_uint32), ("S", C.c_uint32), ("K", C.c_uint32),
                ("sched_paper", C.c_uint32), ("mh", C.c_uint32), ("clamp", C.c_uint32),
                ("sigma", C.c_double * 3), ("anneal", C.c_double), ("seed", C.c_uint64),
                ("mpc", C.c_uint32), ("nthreads", C.c_int), ("L_final", C.c_uint32)]


def _declare(L):
    u32, u64, i64, d = C.c_uint32, C.c_uint64, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "ora_philox": (None, [P(u32), P(u32), P(u32)]),
        "ora_u24": (d, [u32]),
        "ora_box_muller": (None, [u32, u32, _dp, _dp]),
        "ora_r64": (u64, [u32, u32, u32, u64, u32]),
        "ora_det_exp2": (d, [d]),
        "ora_det_quant": (u64, [d]),
        "ora_det_coeffs": (_dp, []),
        "ora_sample_schedule": (C.c_int, [C.c_int]),
        "ora_derive": (C.c_int, [P(_Problem), P(_Derived)]),
        "ora_free_derived": (None, [P(_Derived)]),
        "ora_popdense_point": (d, [P(_Problem), d, d]),
        "ora_popdense_grid": (d, [P(_Problem), P(_Derived), d, d]),
        "ora_trilinear": (None, [P(_Problem), P(_Derived), _dp, _dp, _dp]),
        "ora_lift_drag": (None, [P(_Problem), C.c_int, _dp, d, _dp, _dp]),
        "ora_step": (None, [P(_Problem), C.c_int, _dp, _dp, _dp, _dp]),
        "ora_landed": (C.c_int, [P(_Problem), _dp]),
        "ora_unary_violation": (C.c_int, [P(_Problem), C.c_int, _dp, _dp]),
        "ora_pair_conflict": (C.c_int, [P(_Problem), _dp, _dp]),
        "ora_flow_heading": (d, [d, d]),
        "ora_arc_length": (d, [d, d]),
        "ora_beta": (d, [d, d, d]),
        "ora_angdist": (d, [d]),
        "ora_rollout": (None, [P(_Problem), P(_Derived), _dp, u32, u32, u32, u64, u32, P(_RollOut)]),
        "ora_rollout_replay": (None, [P(_Problem), P(_Derived), _dp, u32, u32, u32, u64, u32, P(_Replay),
                                      P(_RollOut)]),
        "ora_evaluate": (None, [P(_Problem), P(_Derived), _dp, u32, u32, u32, u64, u32, _dp, C.c_int]),
        "ora_evaluate_margin": (None, [P(_Problem), P(_Derived), _dp, u32, u32, u32, u64, u32, _dp, _dp, C.c_int]),
        "ora_init_population": (None, [P(_Problem), u32, u64, u32, _dp]),
        "ora_fuel_estimate1": (C.c_int, [P(_Problem), C.c_int, _dp, _dp, C.c_int, d, d, _dp, _dp]),
        "ora_fuel_estimate2": (C.c_int, [P(_Problem), C.c_int, _dp, _dp, C.c_int, d, d, _dp]),
        "ora_init_population_warm": (None, [P(_Problem), u32, u64, u32, _dp, _ip, u32, _dp, C.c_int, _dp]),
        "ora_mh_accept": (C.c_int, [d, d, u32, u32, u64, u32]),
        "ora_mh_accept_aircraft": (C.c_int, [d, d, u32, u32, u32, u64, u32]),
        "ora_resample_column": (C.c_int, [_dp, u32, u32, u32, u64, u32, _ip, P(u64), P(u64), P(u64)]),
        "ora_resample_column_m": (C.c_int, [_dp, u32, u32, u32, u32, u64, u32, _ip, P(u64), P(u64), P(u64)]),
        "ora_particles_of": (u32, [u32, u32, u32, u32]),
        "ora_perturb_row": (None, [P(_Problem), C.c_int, _dp, _dp, u32, u32, u64, u32, _dp, C.c_int]),
        "ora_select": (i64, [_dp, u32]),
        "ora_run_smc": (C.c_int, [P(_Problem), P(_SmcCfg), _dp, _dp, P(i64), _dp]),
        "ora_plant_step": (None, [P(_Problem), P(_Derived), _dp, _dp, u64, u32, _dp, _ip, _dp, _ip]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _ptr(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(x, shape=None):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if shape is not None:
        a = a.reshape(shape)
    return a


PER_AC_F = ["theta_F", "z_tf", "v_D", "beta_f", "S", "cd0", "cd2", "eta", "m_empty",
            "T_min", "T_max", "v_min", "v_max", "gamma_max", "phi_max", "z_min", "z_max"]


class Problem:
    """Oracle view of a scenario dict (see paper_1506_02869_b200.scenarios)."""

    def __init__(self, scn: dict):
        self.scn = scn
        n = int(scn["n"])
        self.n, self.H = n, int(scn["H"])
        keep = {}
        keep["kind"] = np.ascontiguousarray(np.asarray(scn["kind"], dtype=np.int32))
        keep["first_step"] = np.ascontiguousarray(np.asarray(scn["first_step"], dtype=np.int32))
        keep["x0"] = _f64(scn["x0"]).reshape(n, 6)
        for k in PER_AC_F:
            keep[k] = _f64(scn[k]).reshape(n)
        cen = np.asarray(scn.get("centres", np.zeros((0, 3))), dtype=np.float64).reshape(-1, 3)
        keep["centres"] = np.ascontiguousarray(cen)
        self._keep = keep
        p = _Problem()
        p.n, p.H = n, self.H
        p.dt, p.g = float(scn["dt"]), float(scn["g"])
        p.density_mode, p.rho_const = int(scn["density_mode"]), float(scn["rho_const"])
        p.kind = _ptr(keep["kind"], C.c_int32)
        p.first_step = _ptr(keep["first_step"], C.c_int32)
        p.x0 = _ptr(keep["x0"])
        for k in PER_AC_F:
            setattr(p, k, _ptr(keep[k]))
        for k in ["P_runway", "P_beta", "P_chi", "P_vs", "P_r", "P_h", "noise_w", "A_c",
                  "pop_x0", "pop_y0", "pop_dx", "sigma_lo", "sigma_hi", "beta_w", "gamma_w",
                  "lambda_t", "turb_sigma", "tma_radius"]:
            setattr(p, k, float(scn[k]))
        p.alpha_dep[:] = [float(v) for v in scn["alpha_dep"]]
        p.alpha_arr[:] = [float(v) for v in scn["alpha_arr"]]
        p.n_centres = cen.shape[0]
        p.centres = _ptr(keep["centres"])
        p.pop_nx, p.pop_ny = int(scn["pop_nx"]), int(scn["pop_ny"])
        p.wind_lo[:] = [float(v) for v in scn["wind_lo"]]
        p.wind_hi[:] = [float(v) for v in scn["wind_hi"]]
        p.nominal[:] = [float(v) for v in scn["nominal"]]
        p.wind_n[:] = [int(v) for v in scn.get("wind_n", (2, 2, 2))]
        self.p = p
        self.d = _Derived()
        rc = lib().ora_derive(C.byref(self.p), C.byref(self.d))
        if rc != 0:
            raise ValueError(f"ora_derive failed ({rc})")

    def __del__(self):
        try:
            lib().ora_free_derived(C.byref(self.d))
        except Exception:
            pass

    # -- derived constants --------------------------------------------------
    @property
    def Rhat(self):
        g = self.d.ng
        return np.array(self.d.Rhat[: g * g]).reshape(g, g)

    @property
    def Qhat(self):
        g = self.d.ng
        return np.array(self.d.Qhat[: g * g]).reshape(g, g)

    @property
    def wind_grid(self):
        return self.d.nx, self.d.ny, self.d.nz

    @property
    def ab(self):
        return self.d.a, self.d.b

    def supinfB(self):
        return np.array(self.d.supB[: self.n]), np.array(self.d.infB[: self.n])

    def pop_grid(self):
        nx, ny = self.p.pop_nx, self.p.pop_ny
        if nx * ny == 0:
            return np.zeros((0, 0))
        return np.ctypeslib.as_array(self.d.pop, shape=(ny * nx,)).copy().reshape(ny, nx)

    # -- point functions ----------------------------------------------------
    def popdense(self, x, y, grid=True):
        if grid:
            return lib().ora_popdense_grid(C.byref(self.p), C.byref(self.d), float(x), float(y))
        return lib().ora_popdense_point(C.byref(self.p), float(x), float(y))

    def trilinear(self, W, pos):
        W, pos, out = _f64(W, (self.d.ng,)), _f64(pos, (-1,)), np.zeros(1)
        lib().ora_trilinear(C.byref(self.p), C.byref(self.d), _ptr(W), _ptr(pos), _ptr(out))
        return float(out[0])

    def lift_drag(self, i, st, phi):
        st, L_, D_ = _f64(st, (6,)), np.zeros(1), np.zeros(1)
        lib().ora_lift_drag(C.byref(self.p), i, _ptr(st), float(phi), _ptr(L_), _ptr(D_))
        return float(L_[0]), float(D_[0])

    def step(self, i, st, u, wind=(0.0, 0.0)):
        st, u, w, out = _f64(st, (6,)), _f64(u, (3,)), _f64(wind, (2,)), np.zeros(6)
        lib().ora_step(C.byref(self.p), i, _ptr(st), _ptr(u), _ptr(w), _ptr(out))
        return out

    def landed(self, st):
        return bool(lib().ora_landed(C.byref(self.p), _ptr(_f64(st, (6,)))))

    def unary_violation(self, i, u, st):
        return bool(lib().ora_unary_violation(C.byref(self.p), i, _ptr(_f64(u, (3,))), _ptr(_f64(st, (6,)))))

    def pair_conflict(self, a, b):
        return bool(lib().ora_pair_conflict(C.byref(self.p), _ptr(_f64(a, (6,))), _ptr(_f64(b, (6,)))))

    # -- rollout / population ---------------------------------------------
    def rollout(self, u, l, s, k, seed, mpc=0, replay=None):
        """One rollout.  replay = (landed_step[n], viol[n], eps): decisions whose own
        margin is below eps follow the given ones (R30 decision replay)."""
        n, H = self.n, self.H
        u = _f64(u, (n, H, 3))
        res = {"J": np.zeros(n), "comp": np.zeros((n, 4)), "traj": np.zeros((n, H + 1, 6)),
               "fuel": np.zeros(n), "margin": np.zeros(n), "margin_land": np.zeros(n),
               "viol": np.zeros(n, np.int32), "landed_step": np.zeros(n, np.int32),
               "replayed": np.zeros(n, np.int32)}
        o = _RollOut(_ptr(res["J"]), _ptr(res["comp"]), _ptr(res["traj"]), _ptr(res["fuel"]),
                     _ptr(res["margin"]), _ptr(res["margin_land"]), _ptr(res["viol"], C.c_int32),
                     _ptr(res["landed_step"], C.c_int32), _ptr(res["replayed"], C.c_int32))
        if replay is None:
            lib().ora_rollout(C.byref(self.p), C.byref(self.d), _ptr(u), l, s, k, seed, mpc, C.byref(o))
        else:
            ls = np.ascontiguousarray(np.asarray(replay[0], dtype=np.int32).reshape(n))
            vi = np.ascontiguousarray(np.asarray(replay[1], dtype=np.int32).reshape(n))
            rp = _Replay(_ptr(ls, C.c_int32), _ptr(vi, C.c_int32), float(replay[2]))
            lib().ora_rollout_replay(C.byref(self.p), C.byref(self.d), _ptr(u), l, s, k, seed, mpc, C.byref(rp),
                                     C.byref(o))
        return res

    def evaluate(self, ctrl, S, k, seed, mpc=0, ell0=None, nthreads=0, margin=False):
        """ell [L][n] after S samples (Alg.1 l.9-18); with margin=True also the
        per-(particle, aircraft) decision margin [L][n] (R30)."""
        n, H = self.n, self.H
        ctrl = _f64(ctrl).reshape(-1, n, H, 3)
        L = ctrl.shape[0]
        ell = np.full((L, n), -np.log2(L) if ell0 is None else ell0, dtype=np.float64)
        nt = nthreads or (os.cpu_count() or 1)
        if not margin:
            lib().ora_evaluate(C.byref(self.p), C.byref(self.d), _ptr(ctrl), L, S, k, seed, mpc, _ptr(ell), nt)
            return ell
        mg = np.zeros((L, n))
        lib().ora_evaluate_margin(C.byref(self.p), C.byref(self.d), _ptr(ctrl), L, S, k, seed, mpc, _ptr(ell),
                                  _ptr(mg), nt)
        return ell, mg

    def init_population(self, L, seed, mpc=0):
        out = np.zeros((L, self.n, self.H, 3))
        lib().ora_init_population(C.byref(self.p), L, seed, mpc, _ptr(out))
        return out

    def init_population_warm(self, L, seed, prev, has_prev, Lw, sigma, mpc=0, clamp=False):
        """Warm start (R45): prev [n][H][3] previous winner rows mapped to this scenario."""
        out = np.zeros((L, self.n, self.H, 3))
        prev = _f64(prev, (self.n, self.H, 3))
        hp = np.ascontiguousarray(np.asarray(has_prev, dtype=np.int32))
        sig = _f64(sigma, (3,))
        lib().ora_init_population_warm(C.byref(self.p), L, seed, mpc, _ptr(prev),
                                       hp.ctypes.data_as(C.POINTER(C.c_int32)), Lw, _ptr(sig), int(clamp), _ptr(out))
        return out

    def fuel_estimate1(self, i, trace, dt, m1, Cf):
        """Section 5 fuel estimate 1 -> (mass series, wind residuals, flags)."""
        tr = _f64(trace, (-1, 5))
        K = tr.shape[0]
        m, w = np.zeros(K), np.zeros((K, 2))
        fl = lib().ora_fuel_estimate1(C.byref(self.p), i, _ptr(_f64(Cf, (2,))), _ptr(tr), K, float(dt), float(m1),
                                      _ptr(m), _ptr(w))
        return m, w, fl

    def fuel_estimate2(self, i, trace, dt, m1, Cf):
        """Section 5 fuel estimate 2 -> (mass series, flags)."""
        tr = _f64(trace, (-1, 5))
        K = tr.shape[0]
        m = np.zeros(K)
        fl = lib().ora_fuel_estimate2(C.byref(self.p), i, _ptr(_f64(Cf, (2,))), _ptr(tr), K, float(dt), float(m1),
                                      _ptr(m))
        return m, fl

    def perturb_row(self, i, row, l, k, seed, sigma, mpc=0, clamp=False):
        row = _f64(row, (self.H, 3))
        out = np.zeros((self.H, 3))
        sg = _f64(sigma, (3,))
        lib().ora_perturb_row(C.byref(self.p), i, _ptr(row), _ptr(out), l, k, seed, mpc, _ptr(sg), int(clamp))
        return out

    def run_smc(self, L, S, K, seed, sigma, anneal=0.98, mh=True, sched_paper=False, clamp=False,
                mpc=0, nthreads=0, L_final=0):
        cfg = _SmcCfg()
        cfg.L, cfg.S, cfg.K = L, S, K
        cfg.sched_paper, cfg.mh, cfg.clamp = int(sched_paper), int(mh), int(clamp)
        cfg.sigma[:] = [float(v) for v in sigma]
        cfg.anneal, cfg.seed, cfg.mpc = float(anneal), int(seed), int(mpc)
        cfg.nthreads = nthreads or (os.cpu_count() or 1)
        cfg.L_final = int(L_final)
        best = np.zeros((self.n, self.H, 3))
        lam = np.zeros(1)
        idx = C.c_int64(-1)
        stats = np.zeros((K, 4))
        rc = lib().ora_run_smc(C.byref(self.p), C.byref(cfg), _ptr(best), _ptr(lam), C.byref(idx), _ptr(stats))
        return {"rc": rc, "best_ctrl": best, "best_lambda": float(lam[0]), "best_index": int(idx.value),
                "stats": stats}

    def plant_step(self, states, u0, seed, mpc, Zplant=None, zinit=0):
        states = _f64(states, (self.n, 6))
        u0 = _f64(u0, (self.n, 3))
        Z = np.zeros(128) if Zplant is None else _f64(Zplant, (-1,)).copy()
        if Z.size < 128:
            Z = np.concatenate([Z, np.zeros(128 - Z.size)])
        zi = np.array([zinit], dtype=np.int32)
        nxt = np.zeros((self.n, 6))
        flags = np.zeros(self.n, np.int32)
        lib().ora_plant_step(C.byref(self.p), C.byref(self.d), _ptr(states), _ptr(u0), seed, mpc,
                             _ptr(Z), _ptr(zi, C.c_int32), _ptr(nxt), _ptr(flags, C.c_int32))
        return nxt, flags, Z, int(zi[0])


# -- free functions ---------------------------------------------------------
def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (C.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (C.c_uint32 * 4)()
    lib().ora_philox(c, k, o)
    return tuple(o)


def u24(w):
    return lib().ora_u24(int(w) & 0xFFFFFFFF)


def box_muller(w0, w1):
    a, b = C.c_double(), C.c_double()
    lib().ora_box_muller(int(w0) & 0xFFFFFFFF, int(w1) & 0xFFFFFFFF, C.byref(a), C.byref(b))
    return a.value, b.value


def r64(tag, x0, k, seed, mpc=0):
    return lib().ora_r64(tag, x0, k, seed, mpc)


def det_exp2(y):
    return lib().ora_det_exp2(float(y))


def det_quant(d):
    return int(lib().ora_det_quant(float(d)))


def det_coeffs():
    p = lib().ora_det_coeffs()
    return [p[j] for j in range(17)]


def sample_schedule(J):
    return lib().ora_sample_schedule(int(J))


def flow_heading(x, y):
    return lib().ora_flow_heading(float(x), float(y))


def arc_length(x, y):
    return lib().ora_arc_length(float(x), float(y))


def beta(x, y, z):
    return lib().ora_beta(float(x), float(y), float(z))


def angdist(d):
    return lib().ora_angdist(float(d))


def mh_accept(lam_cur, lam_prop, l, k, seed, mpc=0):
    return bool(lib().ora_mh_accept(float(lam_cur), float(lam_prop), l, k, seed, mpc))


def mh_accept_aircraft(ell_cur, ell_prop, l, i, k, seed, mpc=0):
    return bool(lib().ora_mh_accept_aircraft(float(ell_cur), float(ell_prop), l, i, k, seed, mpc))


def resample_column(ell, i, k, seed, mpc=0, M=None):
    ell = _f64(ell, (-1,))
    L = ell.shape[0]
    M = L if M is None else int(M)
    anc = np.zeros(max(M, 1), np.int32)
    q = np.zeros(L, np.uint64)
    Q, R = C.c_uint64(), C.c_uint64()
    inf = lib().ora_resample_column_m(_ptr(ell), L, M, i, k, seed, mpc, _ptr(anc, C.c_int32),
                                      q.ctypes.data_as(C.POINTER(C.c_uint64)), C.byref(Q), C.byref(R))
    anc = anc[:M]
    return {"anc": anc, "q": q, "Q": Q.value, "R": R.value, "infeasible": bool(inf)}


def particles_of(L, L_final, K, k):
    return int(lib().ora_particles_of(int(L), int(L_final), int(K), int(k)))


def select(lam):
    lam = _f64(lam, (-1,))
    return int(lib().ora_select(_ptr(lam), lam.shape[0]))


TAG = {"INIT": 1, "PERTURB": 2, "WIND": 3, "TURB": 4, "MH": 5, "RESAMPLE": 6,
       "PLANT_WIND": 7, "PLANT_TURB": 8}
