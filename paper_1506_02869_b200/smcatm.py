"""Thin ctypes binding over libsmcatm.so (include/smcatm.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the C ABI.  PyTorch provides the device workspace and the
stream.  There is no CPU fallback: if the shared library is missing this
module raises at load time.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsmcatm.so")
# A/B tooling only (tools/gpu_variants.sh): load a variant build of the same library instead
if os.environ.get("SMC_LIB"):
    LIB_PATH = os.environ["SMC_LIB"]
_lib = None

SMC_OK, SMC_EINVAL, SMC_EINFEASIBLE, SMC_ECUDA, SMC_ENCCL, SMC_ENOMEM, SMC_ESTATE = range(7)
_STATUS = {0: "SMC_OK", 1: "SMC_EINVAL", 2: "SMC_EINFEASIBLE", 3: "SMC_ECUDA", 4: "SMC_ENCCL",
           5: "SMC_ENOMEM", 6: "SMC_ESTATE"}


class SmcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class State(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("x", "y", "z", "v", "chi", "m")]


class Control(C.Structure):
    _fields_ = [("thrust", C.c_float), ("bank", C.c_float), ("climb", C.c_float)]


class AircraftType(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("S", "cd0", "cd2", "eta", "m_empty", "T_min", "T_max", "v_min",
                                          "v_max", "gamma_max", "phi_max", "z_min", "z_max")]


class Aircraft(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("type", C.c_uint32), ("first_step", C.c_uint32), ("id", C.c_uint32),
                ("x0", State), ("theta_F", C.c_double), ("z_tf", C.c_double), ("v_D", C.c_double),
                ("beta_f", C.c_double)]


class Scenario(C.Structure):
    _fields_ = [
        ("n_aircraft", C.c_uint32), ("n_types", C.c_uint32),
        ("aircraft", C.POINTER(Aircraft)), ("types", C.POINTER(AircraftType)),
        ("horizon", C.c_uint32), ("density_mode", C.c_int32),
        ("dt", C.c_double), ("g", C.c_double), ("rho_const", C.c_double),
        ("P_runway", C.c_double), ("P_beta", C.c_double), ("P_chi", C.c_double), ("P_vs", C.c_double),
        ("P_r", C.c_double), ("P_h", C.c_double),
        ("alpha_dep", C.c_double * 4), ("alpha_arr", C.c_double * 3),
        ("noise_w", C.c_double), ("A_c", C.c_double),
        ("n_centres", C.c_uint32), ("centres", C.POINTER(C.c_double)),
        ("pop_nx", C.c_uint32), ("pop_ny", C.c_uint32),
        ("pop_x0", C.c_double), ("pop_y0", C.c_double), ("pop_dx", C.c_double),
        ("wind_lo", C.c_double * 3), ("wind_hi", C.c_double * 3),
        ("sigma_lo", C.c_double), ("sigma_hi", C.c_double),
        ("beta_w", C.c_double), ("gamma_w", C.c_double), ("lambda_t", C.c_double),
        ("nominal", C.c_double * 2), ("turb_sigma", C.c_double), ("tma_radius", C.c_double),
        ("wind_n", C.c_uint32 * 3),
    ]


class FuelArgs(C.Structure):
    _fields_ = [("n_traces", C.c_uint32), ("max_len", C.c_uint32), ("len", C.c_void_p), ("trace", C.c_void_p),
                ("m0", C.c_void_p), ("type", C.c_void_p), ("dt", C.c_double), ("g", C.c_double),
                ("density_mode", C.c_int32), ("rho_const", C.c_double), ("m1", C.c_void_p), ("m2", C.c_void_p),
                ("wres", C.c_void_p), ("fuel", C.c_void_p), ("flags", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [
        ("n_particles", C.c_uint32), ("n_samples", C.c_uint32), ("schedule", C.c_uint32),
        ("n_rounds", C.c_uint32), ("mh", C.c_uint32), ("clamp_proposals", C.c_uint32),
        ("sigma", C.c_double * 3), ("anneal", C.c_double), ("seed", C.c_uint64),
        ("device", C.c_int32), ("rank", C.c_int32), ("world_size", C.c_int32),
        ("nccl_unique_id", C.c_void_p), ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("stream", C.c_void_p), ("max_aircraft", C.c_uint32), ("max_horizon", C.c_uint32),
        ("use_graph", C.c_uint32), ("profile", C.c_uint32), ("virtual_world", C.c_uint32),
        ("n_particles_final", C.c_uint32), ("warm_fraction", C.c_double), ("host_coll", C.c_void_p),
    ]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint32), C.c_size_t)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class HostCollectives(C.Structure):
    _fields_ = [("user", C.c_void_p), ("allreduce_max_u32", ALLREDUCE_FN), ("allgather", ALLGATHER_FN)]


def gloo_host_collectives(world: int, rank: int):
    """smc_host_collectives over the default torch.distributed process group (CPU / gloo):
    a test shim for world_size > 1 contexts without NCCL (include/smcatm.h).  Returns the
    structure and the callback objects that must stay alive with it."""
    import torch
    import torch.distributed as dist

    def allreduce(user, buf, count):
        try:
            a = np.ctypeslib.as_array(buf, shape=(count,))
            t = torch.from_numpy(a.astype(np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a[:] = t.numpy().astype(np.uint32)
            return 0
        except Exception:
            return 1

    def allgather(user, send, recv, nbytes):
        try:
            src = np.frombuffer((C.c_char * nbytes).from_address(send), dtype=np.uint8).copy()
            out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(out, torch.from_numpy(src))
            for r in range(world):
                C.memmove(recv + r * nbytes, out[r].numpy().ctypes.data, nbytes)
            return 0
        except Exception:
            return 1

    fa, fg = ALLREDUCE_FN(allreduce), ALLGATHER_FN(allgather)
    hc = HostCollectives(None, fa, fg)
    return hc, (fa, fg)


class RoundStats(C.Structure):
    _fields_ = [("best_lambda", C.c_double), ("accept_rate", C.c_double), ("ess_min", C.c_double),
                ("infeasible_lo", C.c_uint32), ("infeasible_hi", C.c_uint32), ("n_samples", C.c_uint32),
                ("round", C.c_uint32)]


def load():
    """Load libsmcatm.so from the package directory; raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1506_02869_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, v, st = C.POINTER, C.c_void_p, C.c_int
    u32, u64, f32p, f64p = C.c_uint32, C.c_uint64, P(C.c_float), P(C.c_double)
    sig = {
        "smc_workspace_bytes": (C.c_size_t, [P(Config)]),
        "smc_init": (st, [P(Config), P(v)]),
        "smc_set_scenario": (st, [v, P(Scenario)]),
        "smc_iterate": (st, [v, u32, P(RoundStats)]),
        "smc_best_controls": (st, [v, P(Control), f64p, P(C.c_int64)]),
        "mpc_step": (st, [v, P(State), P(Control), P(State), P(u32)]),
        "smc_solve": (st, [v, u32]),
        "smc_phase_times": (st, [v, f64p, P(u64)]),
        "smc_last_error": (C.c_char_p, [v]),
        "smc_destroy": (None, [v]),
        "smc_set_mpc_index": (st, [v, u32]),
        "smc_get_mpc_index": (u32, [v]),
        "smc_launch_count": (u64, [v]),
        "smc_nccl_unique_id": (st, [v]),
        "smc_io_bytes": (None, [v, P(u64), P(u64)]),
        "smc_debug_rollout": (st, [v, f32p, u32, u32, u32, u32, f32p, P(C.c_uint8), f32p, f32p,
                                   P(C.c_int32), f32p]),
        "smc_debug_evaluate": (st, [v, f32p, u32, u32, u32, f32p]),
        "smc_debug_evaluate2": (st, [v, f32p, u32, u32, u32, f32p]),
        "smc_debug_mh": (st, [v, f64p, f64p, u32, u32, P(C.c_uint8)]),
        "smc_debug_resample": (st, [v, f32p, u32, u32, u32, u32, P(C.c_int32), P(u64)]),
        "smc_debug_propose": (st, [v, f32p, P(C.c_int32), u32, u32, f32p, f32p]),
        "smc_debug_population": (st, [v, f32p, f32p, P(C.c_uint32), f32p, f64p, f64p, P(C.c_uint32)]),
        "smc_debug_mh_aircraft": (st, [v, f32p, f32p, u32, u32, u32, P(C.c_uint32)]),
        "smc_shard_range": (None, [u32, C.c_int32, C.c_int32, P(u32), P(u32)]),
        "smc_shard_offsets": (None, [u32, C.c_int32, C.c_int32, P(u64), P(u64), P(u64)]),
        "smc_slot_count": (u64, [u64, u64, u64, u32]),
        "smc_fuel_estimates": (st, [C.POINTER(FuelArgs), v]),
        "smc_ipc_record": (st, [v, v]),
        "smc_ipc_peek": (st, [v, u64, v, C.c_size_t]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = ["smc_workspace_bytes", "smc_init", "smc_set_scenario", "smc_iterate", "smc_best_controls",
            "mpc_step", "smc_solve", "smc_phase_times", "smc_last_error", "smc_destroy", "smc_set_mpc_index", "smc_get_mpc_index",
            "smc_launch_count", "smc_io_bytes", "smc_nccl_unique_id", "smc_debug_rollout", "smc_debug_evaluate", "smc_debug_evaluate2", "smc_debug_mh", "smc_debug_mh_aircraft",
            "smc_debug_resample", "smc_debug_propose", "smc_debug_population", "smc_shard_range",
            "smc_shard_offsets", "smc_slot_count", "smc_fuel_estimates", "smc_ipc_record", "smc_ipc_peek"]


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def pack_scenario(scn: dict):
    """Scenario dict (paper_1506_02869_b200.scenarios) -> (Scenario, keep-alive list)."""
    n = int(scn["n"])
    ac = (Aircraft * n)()
    ty = (AircraftType * n)()
    for i in range(n):
        a = ac[i]
        a.kind = int(scn["kind"][i])
        a.type = i
        a.first_step = int(scn["first_step"][i])
        a.id = int(scn["id"][i]) if "id" in scn else i
        x0 = np.asarray(scn["x0"], dtype=np.float64).reshape(n, 6)[i]
        a.x0 = State(*[float(v) for v in x0])
        a.theta_F, a.z_tf, a.v_D, a.beta_f = (float(scn[k][i]) for k in ("theta_F", "z_tf", "v_D", "beta_f"))
        t = ty[i]
        for k in ("S", "cd0", "cd2", "eta", "m_empty", "T_min", "T_max", "v_min", "v_max", "gamma_max",
                  "phi_max", "z_min", "z_max"):
            setattr(t, k, float(scn[k][i]))
    cen = np.ascontiguousarray(np.asarray(scn.get("centres", np.zeros((0, 3))), dtype=np.float64).reshape(-1, 3))
    s = Scenario()
    s.n_aircraft, s.n_types = n, n
    s.aircraft = C.cast(ac, C.POINTER(Aircraft))
    s.types = C.cast(ty, C.POINTER(AircraftType))
    s.horizon = int(scn["H"])
    s.density_mode = int(scn["density_mode"])
    for k in ("dt", "g", "rho_const", "P_runway", "P_beta", "P_chi", "P_vs", "P_r", "P_h", "noise_w", "A_c",
              "pop_x0", "pop_y0", "pop_dx", "sigma_lo", "sigma_hi", "beta_w", "gamma_w", "lambda_t",
              "turb_sigma", "tma_radius"):
        setattr(s, k, float(scn[k]))
    s.alpha_dep[:] = [float(v) for v in scn["alpha_dep"]]
    s.alpha_arr[:] = [float(v) for v in scn["alpha_arr"]]
    s.n_centres = cen.shape[0]
    s.centres = _p(cen, C.c_double)
    s.pop_nx, s.pop_ny = int(scn["pop_nx"]), int(scn["pop_ny"])
    s.wind_lo[:] = [float(v) for v in scn["wind_lo"]]
    s.wind_hi[:] = [float(v) for v in scn["wind_hi"]]
    s.nominal[:] = [float(v) for v in scn["nominal"]]
    s.wind_n[:] = [int(v) for v in scn.get("wind_n", (2, 2, 2))]
    return s, [ac, ty, cen]


def ipc_peek(record: bytes, offset: int, nbytes: int) -> bytes:
    """Map another process's peer-mode record and copy nbytes from its workspace."""
    lib = load()
    out = C.create_string_buffer(nbytes)
    rc = lib.smc_ipc_peek(C.create_string_buffer(record, 128), int(offset), out, int(nbytes))
    if rc != SMC_OK:
        raise SmcError(rc, "smc_ipc_peek failed")
    return out.raw


class Solver:
    """One libsmcatm context on one GPU (rank)."""

    def __init__(self, scn: dict, L: int, S: int, K: int, sigma, seed: int, anneal: float = 0.98,
                 mh: int = 1, sched_paper: bool = False, clamp: bool = False, device: int = 0,
                 max_aircraft: int | None = None, max_horizon: int | None = None, stream=None,
                 rank: int = 0, world_size: int = 1, use_graph: bool = False, profile: bool = False,
                 virtual_world: int = 0, L_final: int = 0, warm_fraction: float = 0.0,
                 host_collectives: bool = False):
        import torch
        self.lib = load()
        self.torch = torch
        self.device = torch.device("cuda", device)
        # a dedicated stream by default: the legacy default stream cannot be graph-captured
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        cfg = Config()
        cfg.n_particles, cfg.n_samples, cfg.n_rounds = int(L), int(S), int(K)
        cfg.schedule = 1 if sched_paper else 0
        cfg.mh, cfg.clamp_proposals = int(mh), int(clamp)
        cfg.sigma[:] = [float(x) for x in sigma]
        cfg.anneal, cfg.seed = float(anneal), int(seed)
        cfg.device, cfg.rank, cfg.world_size = int(device), int(rank), int(world_size)
        cfg.max_aircraft = int(max_aircraft or scn["n"])
        cfg.max_horizon = int(max_horizon or scn["H"])
        cfg.use_graph = int(use_graph)
        cfg.profile = int(profile)
        cfg.virtual_world = int(virtual_world)
        cfg.n_particles_final = int(L_final)
        cfg.warm_fraction = float(warm_fraction)
        cfg.stream = C.c_void_p(self.stream.cuda_stream)
        if world_size > 1 and host_collectives:
            # test shim: collectives over the CPU process group (no NCCL; e.g. ranks sharing a GPU)
            self._hc, self._hc_keep = gloo_host_collectives(world_size, rank)
            cfg.host_coll = C.cast(C.pointer(self._hc), C.c_void_p)
        elif world_size > 1:
            # rank 0 creates the NCCL id; torch.distributed (any backend) shares it
            import torch.distributed as dist
            buf = (C.c_char * 128)()
            if rank == 0:
                self._check_plain(self.lib.smc_nccl_unique_id(buf), "smc_nccl_unique_id")
            obj = [bytes(buf) if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            self._nccl_id = (C.c_char * 128).from_buffer_copy(obj[0])
            cfg.nccl_unique_id = C.cast(self._nccl_id, C.c_void_p)
        nbytes = self.lib.smc_workspace_bytes(C.byref(cfg))
        if nbytes == 0:
            raise SmcError(SMC_EINVAL, "invalid configuration")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        cfg.workspace = C.c_void_p(self.workspace.data_ptr())
        cfg.workspace_bytes = nbytes
        self.cfg = cfg
        self.ctx = C.c_void_p()
        rc = self.lib.smc_init(C.byref(cfg), C.byref(self.ctx))
        if rc != SMC_OK:
            raise SmcError(rc, "smc_init failed")
        self.L, self.S, self.K = int(L), int(S), int(K)
        self.set_scenario(scn)

    # -- helpers -----------------------------------------------------------
    @staticmethod
    def _check_plain(rc, what):
        if rc != SMC_OK:
            raise SmcError(rc, what)

    def _check(self, rc):
        if rc != SMC_OK:
            raise SmcError(rc, self.lib.smc_last_error(self.ctx).decode())

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            self.lib.smc_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self):
        return int(self.lib.smc_launch_count(self.ctx))

    def io_bytes(self):
        """(h2d, d2h) bytes copied by production calls since the last query."""
        a, b = C.c_uint64(), C.c_uint64()
        self.lib.smc_io_bytes(self.ctx, C.byref(a), C.byref(b))
        return a.value, b.value

    def ipc_record(self) -> bytes:
        """128-byte peer-mode record of this context's workspace (CUDA IPC handle + offset)."""
        buf = C.create_string_buffer(128)
        self._check(self.lib.smc_ipc_record(self.ctx, buf))
        return buf.raw

    @property
    def mpc_index(self):
        return int(self.lib.smc_get_mpc_index(self.ctx))

    @mpc_index.setter
    def mpc_index(self, v):
        self._check(self.lib.smc_set_mpc_index(self.ctx, int(v)))

    # -- API ---------------------------------------------------------------
    def set_scenario(self, scn: dict):
        self.scn = scn
        self.n, self.H = int(scn["n"]), int(scn["H"])
        s, keep = pack_scenario(scn)
        self._check(self.lib.smc_set_scenario(self.ctx, C.byref(s)))

    def iterate(self, n_rounds: int, stats: bool = False):
        st = (RoundStats * n_rounds)() if stats else None
        self._check(self.lib.smc_iterate(self.ctx, int(n_rounds), st))
        if stats:
            return [dict(best_lambda=r.best_lambda, accept_rate=r.accept_rate, ess_min=r.ess_min,
                         infeasible=r.infeasible_lo | (r.infeasible_hi << 32), n_samples=r.n_samples,
                         round=r.round) for r in st]
        return None

    def best_controls(self, allow_infeasible=False):
        out = np.zeros((self.n, self.H, 3), dtype=np.float32)
        lam = C.c_double()
        idx = C.c_int64()
        rc = self.lib.smc_best_controls(self.ctx, out.ctypes.data_as(C.POINTER(Control)), C.byref(lam), C.byref(idx))
        if rc == SMC_EINFEASIBLE and allow_infeasible:
            return out, float("-inf"), -1
        self._check(rc)
        return out, lam.value, idx.value

    def mpc_step(self, measured):
        n = self.n
        m = np.ascontiguousarray(np.asarray(measured, dtype=np.float64).reshape(n, 6))
        applied = np.zeros((n, 3), dtype=np.float32)
        nxt = np.zeros((n, 6), dtype=np.float64)
        flags = np.zeros(n, dtype=np.uint32)
        self._check(self.lib.mpc_step(self.ctx, m.ctypes.data_as(C.POINTER(State)),
                                      applied.ctypes.data_as(C.POINTER(Control)),
                                      nxt.ctypes.data_as(C.POINTER(State)), _p(flags, C.c_uint32)))
        return applied, nxt, flags

    def solve(self, advance_plant: bool = True):
        """Device-resident MPC update (no host copies, no sync)."""
        self._check(self.lib.smc_solve(self.ctx, int(advance_plant)))

    def phase_times(self):
        ms = (C.c_double * 4)()
        n = (C.c_uint64 * 4)()
        self._check(self.lib.smc_phase_times(self.ctx, ms, n))
        names = ("rollout", "resample", "propose", "other")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def mpc_step_ptr(self, measured_ptr: int, applied_ptr: int, next_ptr: int, flags_ptr: int):
        """mpc_step on caller-owned (e.g. pinned) host buffers given by address."""
        rc = self.lib.mpc_step(self.ctx, C.cast(C.c_void_p(measured_ptr), C.POINTER(State)),
                               C.cast(C.c_void_p(applied_ptr), C.POINTER(Control)),
                               C.cast(C.c_void_p(next_ptr), C.POINTER(State)),
                               C.cast(C.c_void_p(flags_ptr), C.POINTER(C.c_uint32)))
        if rc == SMC_EINFEASIBLE:
            return False
        self._check(rc)
        return True

    # -- debug hooks ---------------------------------------------------------
    def debug_rollout(self, controls, S, k, l0=0, traj=False):
        c = np.ascontiguousarray(np.asarray(controls, dtype=np.float32))
        L = c.shape[0]
        n, H = self.n, self.H
        out = {"J": np.zeros((L, S, n), np.float32), "viol": np.zeros((L, S, n), np.uint8),
               "comp": np.zeros((L, S, n, 4), np.float32), "fuel": np.zeros((L, S, n), np.float32),
               "landed": np.zeros((L, S, n), np.int32)}
        tr = np.zeros((L, S, n, H + 1, 6), np.float32) if traj else None
        self._check(self.lib.smc_debug_rollout(self.ctx, _p(c, C.c_float), L, l0, S, k, _p(out["J"], C.c_float),
                                               _p(out["viol"], C.c_uint8), _p(out["comp"], C.c_float),
                                               _p(out["fuel"], C.c_float), _p(out["landed"], C.c_int32),
                                               _p(tr, C.c_float)))
        if traj:
            out["traj"] = tr
        return out

    def debug_evaluate(self, controls, S, k, two=False):
        """smc_debug_evaluate (single-candidate kernel) or, two=True, smc_debug_evaluate2 (the
        two-candidate kernel with both candidates = controls)."""
        c = np.ascontiguousarray(np.asarray(controls, dtype=np.float32))
        L = c.shape[0]
        ell = np.zeros((L, self.n), np.float32)
        fn = self.lib.smc_debug_evaluate2 if two else self.lib.smc_debug_evaluate
        self._check(fn(self.ctx, _p(c, C.c_float), L, S, k, _p(ell, C.c_float)))
        return ell

    def debug_mh(self, lam_cur, lam_prop, k):
        a = np.ascontiguousarray(np.asarray(lam_cur, dtype=np.float64))
        b = np.ascontiguousarray(np.asarray(lam_prop, dtype=np.float64))
        acc = np.zeros(a.shape[0], np.uint8)
        self._check(self.lib.smc_debug_mh(self.ctx, _p(a, C.c_double), _p(b, C.c_double), a.shape[0], k,
                                          _p(acc, C.c_uint8)))
        return acc

    def debug_mh_aircraft(self, ell_cur, ell_prop, k):
        """Per-aircraft MH masks (R46) for injected float log2 weights [L][n]."""
        a = np.ascontiguousarray(np.asarray(ell_cur, dtype=np.float32))
        b = np.ascontiguousarray(np.asarray(ell_prop, dtype=np.float32))
        L, N = a.shape
        mask = np.zeros(L, np.uint32)
        self._check(self.lib.smc_debug_mh_aircraft(self.ctx, _p(a, C.c_float), _p(b, C.c_float), L, N, k,
                                                   _p(mask, C.c_uint32)))
        return mask

    def debug_resample(self, ell, k, M=None):
        e = np.ascontiguousarray(np.asarray(ell, dtype=np.float32))
        N, L = e.shape
        M = L if M is None else int(M)
        anc = np.zeros((N, M), np.int32)
        Q = np.zeros(N, np.uint64)
        self._check(self.lib.smc_debug_resample(self.ctx, _p(e, C.c_float), N, L, M, k, _p(anc, C.c_int32),
                                                _p(Q, C.c_uint64)))
        return anc, Q

    def debug_propose(self, surv_ctrl, anc, k):
        s = np.ascontiguousarray(np.asarray(surv_ctrl, dtype=np.float32))
        a = np.ascontiguousarray(np.asarray(anc, dtype=np.int32))
        xp, xs = np.zeros_like(s), np.zeros_like(s)
        self._check(self.lib.smc_debug_propose(self.ctx, _p(s, C.c_float), _p(a, C.c_int32), s.shape[0], k,
                                               _p(xp, C.c_float), _p(xs, C.c_float)))
        return xp, xs

    def population(self):
        L, n, H = self.L, self.n, self.H
        cur = np.zeros((L, n, H, 3), np.float32)
        prop = np.zeros_like(cur)
        surv = np.zeros(L, np.uint32)
        ell = np.zeros((n, L), np.float32)
        lam = np.zeros(L, np.float64)
        lam2 = np.zeros((2, L), np.float64)
        nev = C.c_uint32()
        self._check(self.lib.smc_debug_population(self.ctx, _p(cur, C.c_float), _p(prop, C.c_float),
                                                  _p(surv, C.c_uint32), _p(ell, C.c_float), _p(lam, C.c_double),
                                                  _p(lam2, C.c_double), C.byref(nev)))
        Lk = nev.value
        # surv: bit 0 of the survivor masks (the joint decision; all bits alike outside mh=2)
        return {"cur": cur[:Lk], "prop": prop[:Lk], "surv": (surv[:Lk] & 1).astype(np.uint8),
                "surv_mask": surv[:Lk],
                "ell": ell.reshape(-1)[:n * Lk].reshape(n, Lk), "lam": lam[:Lk],
                "lam_cand": lam2.reshape(-1)[:2 * Lk].reshape(2, Lk)}


def shard_range(L, world, rank):
    lib = load()
    b, e = C.c_uint32(), C.c_uint32()
    lib.smc_shard_range(int(L), int(world), int(rank), C.byref(b), C.byref(e))
    return b.value, e.value


def shard_offsets(Q_all, rank):
    lib = load()
    Q_all = np.ascontiguousarray(np.asarray(Q_all, dtype=np.uint64))
    world, N = Q_all.shape
    off = np.zeros(N, np.uint64)
    tot = np.zeros(N, np.uint64)
    lib.smc_shard_offsets(N, world, rank, _p(Q_all, C.c_uint64), _p(off, C.c_uint64), _p(tot, C.c_uint64))
    return off, tot


def slot_count(Cv, Q, R, L):
    return int(load().smc_slot_count(int(Cv), int(Q), int(R), int(L)))


def fuel_estimates(traces, lens, m0, types, dt, g=9.81, density_mode=0, rho_const=1.225, device=0):
    """Section-5 fuel estimates 1 and 2 for a batch of recorded traces on
    the GPU (smc_fuel_estimates).  traces [n][max_len][5] (x, y, z, v_s, chi), lens [n],
    m0 [n], types [n][6] (S, cd0, cd2, Cf1, Cf2, gamma_max).  Device memory comes from
    torch; the arithmetic runs in k_fuel.  Returns a dict of numpy arrays."""
    import torch
    lib = load()
    dev = torch.device("cuda", device)
    tr = torch.as_tensor(np.ascontiguousarray(traces, dtype=np.float64), device=dev)
    n, max_len = int(tr.shape[0]), int(tr.shape[1])
    ln = torch.as_tensor(np.ascontiguousarray(lens, dtype=np.uint32).astype(np.int32), device=dev)
    m0_t = torch.as_tensor(np.ascontiguousarray(m0, dtype=np.float64), device=dev)
    ty = torch.as_tensor(np.ascontiguousarray(types, dtype=np.float64).reshape(n, 6), device=dev)
    m1 = torch.zeros((n, max_len), dtype=torch.float64, device=dev)
    m2 = torch.zeros_like(m1)
    w = torch.zeros((n, max_len, 2), dtype=torch.float64, device=dev)
    fuel = torch.zeros((n, 2), dtype=torch.float64, device=dev)
    flags = torch.zeros(n, dtype=torch.int32, device=dev)
    a = FuelArgs(n, max_len, ln.data_ptr(), tr.data_ptr(), m0_t.data_ptr(), ty.data_ptr(), float(dt), float(g),
                 int(density_mode), float(rho_const), m1.data_ptr(), m2.data_ptr(), w.data_ptr(), fuel.data_ptr(),
                 flags.data_ptr())
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = lib.smc_fuel_estimates(C.byref(a), C.c_void_p(stream))
    if rc != SMC_OK:
        raise SmcError(rc, "smc_fuel_estimates failed")
    torch.cuda.synchronize(dev)
    return {"m1": m1.cpu().numpy(), "m2": m2.cpu().numpy(), "wres": w.cpu().numpy(), "fuel": fuel.cpu().numpy(),
            "flags": flags.cpu().numpy().astype(np.uint32)}
