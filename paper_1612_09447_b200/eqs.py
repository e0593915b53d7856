"""Python mirror of the reference `eqsim` hot-path interfaces over the C-ABI.

Every call goes through ``libeqs_b200.so`` (include/eqs_b200.h): host C++
setup/control and sm_100a CUDA kernels. There is no CPU fallback — if the
library or a GPU is missing the constructors raise.

Reference interfaces mirrored (paths relative to /root/reference):
  FemSystem            proj/include/eqs/fem_system.hpp:30-73 (OdeSystem, ode_system.hpp:45-73)
  MatFreeStiffness     proj/include/eqs/matfree.hpp:20-57
  rkc_step / rkc_advance_fixed / euler_step / estimate_spectral_radius
                       proj/include/eqs/integrators.hpp:53-104
  run_scenario         proj/include/eqs/scenario.hpp:86
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EQS_B200_LIB") or os.path.join(_HERE, "libeqs_b200.so")
_lib = None


class EqsError(RuntimeError):
    """Base; subclasses mirror proj/include/eqs/errors.hpp:10-37."""


class ConfigError(EqsError):
    pass


class NumericalError(EqsError):
    pass


class GeometryError(EqsError):
    pass


class InvalidArgument(EqsError, ValueError):
    pass


class ParseError(EqsError):
    pass


class CudaError(EqsError):
    pass


_ERRORS = {1: ConfigError, 2: NumericalError, 3: GeometryError, 4: InvalidArgument, 5: ParseError,
           6: CudaError, 7: EqsError}


class _PcgResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("rel_residual", C.c_double),
                ("initial_rel_residual", C.c_double), ("converged", C.c_int)]


class _SolveStats(C.Structure):
    _fields_ = [(n, C.c_long) for n in ("m_solves", "pcg_iterations", "rho_solves", "rho_pcg_iterations",
                                         "newton_linear_solves", "newton_pcg_iterations", "precond_setups",
                                         "assemblies", "svd_count")] + \
               [(n, C.c_double) for n in ("time_residual", "time_solve", "time_setup", "time_estimator")] + \
               [("applies", C.c_long), ("spe_fallbacks", C.c_long), ("estimator_appends", C.c_long)]


class _RkcOptions(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_stages", C.c_int),
                ("rho_refresh_every", C.c_int)]


class _SdirkOptions(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("newton_tol", C.c_double), ("max_newton", C.c_int)]


class _StepAttempt(C.Structure):
    _fields_ = [("t_start", C.c_double), ("dt", C.c_double), ("accepted", C.c_int), ("stages", C.c_int),
                ("newton_iterations", C.c_int), ("error", C.c_double), ("rho", C.c_double),
                ("dt_next", C.c_double)]


class _StateInfo(C.Structure):
    _fields_ = [("t", C.c_double), ("dt", C.c_double), ("accepted", C.c_long), ("rejected", C.c_long),
                ("stages", C.c_long), ("rho_value", C.c_double), ("rho_age", C.c_long), ("rho_valid", C.c_int)]


class _Sizes(C.Structure):
    _fields_ = [(n, C.c_long) for n in ("n_nodes", "n_tets", "n_dofs", "n_free", "n_fixed", "n_local", "order",
                                         "n_colors", "nnz_mass_free", "nnz_mass_ib", "amg_levels")]


class _Timing(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_long * 8), ("bytes", C.c_double * 8)]


class _RunResult(C.Structure):
    _fields_ = [("exit_code", C.c_int), ("accepted", C.c_long), ("rejected", C.c_long), ("stages", C.c_long),
                ("stats", _SolveStats), ("final_t", C.c_double), ("wall_time", C.c_double), ("n_free", C.c_long)]


def load_library():
    """Load libeqs_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(make -C paper_1612_09447_b200); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.eqs_last_error.restype = C.c_char_p
        L.eqs_destroy.restype = None
        L.eqs_destroy.argtypes = [C.c_void_p]
        L.eqs_launch_count.restype = C.c_long
        L.eqs_comm_close.restype = None
        L.eqs_comm_close.argtypes = [C.c_void_p]
        for fn in ("eqs_eval_rhs", "eqs_eval_residual", "eqs_apply_minv_stiffness", "eqs_lift_full",
                   "eqs_set_state", "eqs_mass_solve", "eqs_rkc_advance_fixed", "eqs_euler_step",
                   "eqs_set_option"):
            getattr(L, fn).argtypes = None
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise _ERRORS.get(rc, EqsError)(load_library().eqs_last_error().decode())


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class StepAttempt:
    """proj/include/eqs/integrators.hpp:32-41"""
    t_start: float
    dt: float
    accepted: bool
    stages: int
    error: float
    rho: float
    dt_next: float
    newton_iterations: int = 0


@dataclass
class PcgResult:
    """proj/include/eqs/pcg.hpp:51-57 (x returned separately)"""
    iterations: int
    rel_residual: float
    initial_rel_residual: float
    converged: bool


def _pcg(r: _PcgResult) -> PcgResult:
    return PcgResult(r.iterations, r.rel_residual, r.initial_rel_residual, bool(r.converged))


class FemSystem:
    """GPU-resident FemSystem (proj/src/fem_system.cpp) built from a reference-schema scenario config.

    The config dict/JSON follows proj/README.md:77-113 (mesh box/file, order,
    materials, excitations, solver, estimator). Vectors are numpy arrays in the
    reference's dof numbering.
    """

    def __init__(self, config, device: int = 0, _handle=None):
        L = load_library()
        if _handle is None:
            text = config if isinstance(config, str) else json.dumps(config)
            h = C.c_void_p()
            _check(L.eqs_create_from_config(text.encode(), C.c_int(device), C.byref(h)))
        else:
            h = _handle
        self._h = h
        s = _Sizes()
        _check(L.eqs_get_sizes(h, C.byref(s)))
        self.n_nodes, self.n_tets, self.n_dofs = s.n_nodes, s.n_tets, s.n_dofs
        self.n_free, self.n_fixed, self.n_local, self.order = s.n_free, s.n_fixed, s.n_local, s.order
        self.nnz_mass_free, self.nnz_mass_ib, self.amg_n_levels = s.nnz_mass_free, s.nnz_mass_ib, s.amg_levels
        info = np.zeros(4, dtype=np.int64)
        _check(L.eqs_partition_info(h, info.ctypes.data_as(C.POINTER(C.c_long))))
        self.rank, self.nranks, self.partition_levels, self.n_own = (int(v) for v in info)

    # --- distributed contexts (node ownership)
    @classmethod
    def distributed(cls, config, device: int, nranks: int, rank: int, nccl_id: bytes):
        """One rank of a multi-GPU run (NCCL); nccl_id from nccl_unique_id() on rank 0."""
        text = config if isinstance(config, str) else json.dumps(config)
        h = C.c_void_p()
        _check(load_library().eqs_create_distributed(text.encode(), C.c_int(device), C.c_int(nranks),
                                                     C.c_int(rank), C.create_string_buffer(nccl_id, 128),
                                                     C.byref(h)))
        return cls(None, _handle=h)

    @classmethod
    def distributed_shm(cls, config, device: int, nranks: int, rank: int, shm_name: str):
        """One rank of a multi-process run whose halos and allreduces are host-staged
        through the POSIX shared-memory segment `shm_name` (same on every rank)."""
        text = config if isinstance(config, str) else json.dumps(config)
        h = C.c_void_p()
        _check(load_library().eqs_create_distributed_shm(text.encode(), C.c_int(device), C.c_int(nranks),
                                                         C.c_int(rank), shm_name.encode(), C.byref(h)))
        return cls(None, _handle=h)

    @classmethod
    def virtual_group(cls, config, nranks: int, device: int = 0):
        """nranks partitions in this process (threads); drive them concurrently, one thread per rank."""
        text = config if isinstance(config, str) else json.dumps(config)
        hs = (C.c_void_p * nranks)()
        _check(load_library().eqs_create_virtual_group(text.encode(), C.c_int(device), C.c_int(nranks), hs))
        return [cls(None, _handle=C.c_void_p(hs[r])) for r in range(nranks)]

    @classmethod
    def partition_host(cls, config, nranks: int, rank: int):
        """Host-only partition plan of one rank (no device)."""
        text = config if isinstance(config, str) else json.dumps(config)
        h = C.c_void_p()
        _check(load_library().eqs_create_partition_host(text.encode(), C.c_int(nranks), C.c_int(rank),
                                                        C.byref(h)))
        return cls(None, _handle=h)

    def partition(self, level: int = 0) -> dict:
        L = load_library()
        info = np.zeros(8, dtype=np.int64)
        _check(L.eqs_partition_level(self._h, C.c_int(level), info.ctypes.data_as(C.POINTER(C.c_long))))
        n_global, n_own, n_ghost = int(info[0]), int(info[1]), int(info[2])
        owner = np.zeros(n_global, dtype=np.int32)
        owned = np.zeros(max(1, n_own), dtype=np.int32)
        ghosts = np.zeros(max(1, n_ghost), dtype=np.int32)
        _check(L.eqs_partition_owner(self._h, C.c_int(level), _ip(owner)))
        _check(L.eqs_partition_owned(self._h, C.c_int(level), _ip(owned)))
        _check(L.eqs_partition_ghosts(self._h, C.c_int(level), _ip(ghosts)))
        sends = {}
        for q in range(self.nranks):
            cnt = C.c_int()
            _check(L.eqs_partition_send(self._h, C.c_int(level), C.c_int(q), None, C.byref(cnt)))
            if cnt.value:
                ids = np.zeros(cnt.value, dtype=np.int32)
                _check(L.eqs_partition_send(self._h, C.c_int(level), C.c_int(q), _ip(ids), C.byref(cnt)))
                sends[q] = ids
        return dict(n_global=n_global, owner=owner, owned=owned[:n_own], ghosts=ghosts[:n_ghost], sends=sends,
                    n_local_tets=int(info[5]), n_local_fixed=int(info[6]), replicated=bool(info[7]))

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.eqs_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def size(self) -> int:
        return self.n_free

    # --- setup artefacts (bit-exact checks)
    def colors(self) -> np.ndarray:
        """color_elements (proj/src/matfree.cpp:11-38), colour per tet."""
        c = np.zeros(self.n_tets, dtype=np.int32)
        _check(load_library().eqs_get_colors(self._h, _ip(c)))
        return c

    def mesh(self):
        nodes = np.zeros((self.n_nodes, 3))
        tets = np.zeros((self.n_tets, 4), dtype=np.int32)
        region = np.zeros(self.n_tets, dtype=np.int32)
        _check(load_library().eqs_get_mesh(self._h, _dp(nodes), _ip(tets), _ip(region)))
        return nodes, tets, region

    def dofs(self):
        ed = np.zeros((self.n_tets, self.n_local), dtype=np.int32)
        fr = np.zeros(self.n_free, dtype=np.int32)
        fx = np.zeros(self.n_fixed, dtype=np.int32)
        _check(load_library().eqs_get_dofs(self._h, _ip(ed), _ip(fr), _ip(fx)))
        return ed, fr, fx

    def mass(self, which: int = 0):
        nnz = self.nnz_mass_free if which == 0 else self.nnz_mass_ib
        rp = np.zeros(self.n_free + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        _check(load_library().eqs_get_mass(self._h, C.c_int(which), _ip(rp), _ip(ci), _dp(v)))
        return rp, ci, v

    def amg_levels(self):
        n = C.c_int()
        rn = np.zeros(64, dtype=np.int64)
        _check(load_library().eqs_amg_levels(self._h, C.byref(n), rn.ctypes.data_as(C.POINTER(C.c_long))))
        return [(int(rn[2 * i]), int(rn[2 * i + 1])) for i in range(n.value)]

    def amg_aggregates(self, level: int) -> np.ndarray:
        rows = self.amg_levels()[level][0]
        a = np.zeros(rows, dtype=np.int32)
        _check(load_library().eqs_amg_aggregates(self._h, C.c_int(level), _ip(a)))
        return a

    def amg_level_csr(self, level: int, which: int = 0):
        """(rows, cols, row_ptr, col_idx, values) of A (0), P (1) or R (2) at a level."""
        L = load_library()
        dims = np.zeros(3, dtype=np.int32)
        _check(L.eqs_amg_level_csr(self._h, C.c_int(level), C.c_int(which), _ip(dims), None, None, None))
        rows, cols, nnz = (int(v) for v in dims)
        rp = np.zeros(rows + 1, dtype=np.int32)
        ci = np.zeros(nnz, dtype=np.int32)
        v = np.zeros(nnz)
        _check(L.eqs_amg_level_csr(self._h, C.c_int(level), C.c_int(which), _ip(dims), _ip(rp), _ip(ci), _dp(v)))
        return rows, cols, rp, ci, v

    # --- MatFreeStiffness (proj/src/matfree.cpp:90-143)
    def kx_apply(self, x_state, v) -> np.ndarray:
        y = np.zeros(self.n_dofs)
        _check(load_library().eqs_kx_apply(self._h, _dp(_f64(x_state)), _dp(_f64(v)), _dp(y)))
        return y

    def kx_residual(self, x_full, b_mass) -> np.ndarray:
        r = np.zeros(self.n_free)
        _check(load_library().eqs_kx_residual(self._h, _dp(_f64(x_full)), _dp(_f64(b_mass)), _dp(r)))
        return r

    # --- OdeSystem
    def eval_residual(self, t: float, x) -> np.ndarray:
        r = np.zeros(self.n_free)
        _check(load_library().eqs_eval_residual(self._h, C.c_double(t), _dp(_f64(x)), _dp(r)))
        return r

    def eval_rhs(self, t: float, x) -> np.ndarray:
        f = np.zeros(self.n_free)
        res = _PcgResult()
        _check(load_library().eqs_eval_rhs(self._h, C.c_double(t), _dp(_f64(x)), _dp(f), C.byref(res)))
        self.last_solve = _pcg(res)
        return f

    def mass_apply(self, v) -> np.ndarray:
        y = np.zeros(self.n_free)
        _check(load_library().eqs_mass_apply(self._h, _dp(_f64(v)), _dp(y)))
        return y

    def mass_solve_sequence(self, B, tol: float = 1e-12, max_iter: int = 500, want_x: bool = False):
        """Solve the rows of B (k x n_free) in order with the configured start-vector
        estimator on the device; returns (iterations[k], device_ms, X or None)."""
        B = np.ascontiguousarray(B, dtype=np.float64)
        k = B.shape[0]
        its = np.zeros(k, dtype=np.int32)
        ms = C.c_double()
        X = np.zeros_like(B) if want_x else None
        _check(load_library().eqs_mass_solve_sequence(
            self._h, _dp(B), C.c_int(k), C.c_double(tol), C.c_int(max_iter), _dp(X) if want_x else None,
            its.ctypes.data_as(C.POINTER(C.c_int)), C.byref(ms)))
        return its, ms.value, X

    def mass_solve(self, b, x0=None, tol: float = 1e-12, max_iter: int = 500):
        x = np.zeros(self.n_free)
        res = _PcgResult()
        x0p = None if x0 is None else _dp(_f64(x0))
        _check(load_library().eqs_mass_solve(self._h, _dp(_f64(b)), x0p, C.c_double(tol), C.c_int(max_iter),
                                             _dp(x), C.byref(res)))
        return x, _pcg(res)

    # --- StartVectorEstimator (proj/include/eqs/start_vector.hpp:52-66)
    def estimator_next(self, b):
        """next(M_II, b) -> (x0, current_rank())."""
        x0 = np.zeros(self.n_free)
        rank = C.c_int(0)
        _check(load_library().eqs_estimator_next(self._h, _dp(_f64(b)), _dp(x0), C.byref(rank)))
        return x0, rank.value

    def estimator_feedback(self, x, iterations: int):
        _check(load_library().eqs_estimator_feedback(self._h, _dp(_f64(x)), C.c_int(int(iterations))))

    def estimator_stats(self) -> dict:
        """StartVectorEstimator::Stats (start_vector.hpp:45-49)."""
        s = self.stats()
        return {"svd_count": s["svd_count"], "appends": s["estimator_appends"], "spe_fallbacks": s["spe_fallbacks"]}

    def apply_minv_stiffness(self, t: float, x_state, v) -> np.ndarray:
        y = np.zeros(self.n_free)
        _check(load_library().eqs_apply_minv_stiffness(self._h, C.c_double(t), _dp(_f64(x_state)),
                                                       _dp(_f64(v)), _dp(y)))
        return y

    def lift_full(self, t: float, x_free) -> np.ndarray:
        y = np.zeros(self.n_dofs)
        _check(load_library().eqs_lift_full(self._h, C.c_double(t), _dp(_f64(x_free)), _dp(y)))
        return y

    def stats(self) -> dict:
        s = _SolveStats()
        _check(load_library().eqs_get_stats(self._h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in _SolveStats._fields_}

    # --- integrator on the device-resident state (proj/src/integrators.cpp)
    def set_state(self, t: float, x, dt: float = 0.0):
        _check(load_library().eqs_set_state(self._h, C.c_double(t), _dp(_f64(x)), C.c_double(dt)))

    def get_state(self, out=None, want_x: bool = True):
        """Owned part of the resident state (all free dofs on a single rank).
        out: optional preallocated float64 array (e.g. pinned host memory) that
        receives x; want_x=False returns (None, info) without the copy."""
        if want_x:
            x = np.zeros(self.n_own) if out is None else out
            if x.dtype != np.float64 or not x.flags.c_contiguous or x.size < self.n_own:
                raise ValueError("get_state: out must be a contiguous float64 array of n_own entries")
        else:
            x = None
        info = _StateInfo()
        _check(load_library().eqs_get_state(self._h, _dp(x) if want_x else None, C.byref(info)))
        return x, {n: getattr(info, n) for n, _ in _StateInfo._fields_}

    def set_rho(self, value: float, valid: bool = True, age: int = 0):
        """Pin the RhoCache of the resident state (integrators.hpp:17-21)."""
        _check(load_library().eqs_set_rho(self._h, C.c_double(value), C.c_int(1 if valid else 0), C.c_long(age)))

    def spectral_radius(self) -> float:
        rho = C.c_double()
        _check(load_library().eqs_spectral_radius(self._h, C.byref(rho)))
        return rho.value

    def rkc_step(self, rtol=1e-2, atol=1e-8, max_stages=200, rho_refresh_every=25) -> StepAttempt:
        o = _RkcOptions(rtol, atol, max_stages, rho_refresh_every)
        a = _StepAttempt()
        _check(load_library().eqs_rkc_step(self._h, C.byref(o), C.byref(a)))
        return StepAttempt(a.t_start, a.dt, bool(a.accepted), a.stages, a.error, a.rho, a.dt_next)

    def rkc_advance_fixed(self, dt: float, s: int, nsteps: int = 1):
        _check(load_library().eqs_rkc_advance_fixed(self._h, C.c_double(dt), C.c_int(s), C.c_int(nsteps)))

    def euler_step(self, dt: float) -> StepAttempt:
        a = _StepAttempt()
        _check(load_library().eqs_euler_step(self._h, C.c_double(dt), C.byref(a)))
        return StepAttempt(a.t_start, a.dt, bool(a.accepted), a.stages, a.error, a.rho, a.dt_next)

    def sdirk_step(self, rtol=1e-2, atol=1e-8, newton_tol=1e-8, max_newton=25) -> StepAttempt:
        """sdirk_step (proj/src/integrators.cpp:297-327) on the resident state."""
        o = _SdirkOptions(rtol, atol, newton_tol, max_newton)
        a = _StepAttempt()
        _check(load_library().eqs_sdirk_step(self._h, C.byref(o), C.byref(a)))
        return StepAttempt(a.t_start, a.dt, bool(a.accepted), a.stages, a.error, a.rho, a.dt_next,
                           a.newton_iterations)

    def shifted_solve(self, t: float, z, gdt: float, rhs, refresh_precond: bool = True) -> np.ndarray:
        """FemSystem::shifted_solve (fem_system.cpp:124-145)."""
        d = np.zeros(self.n_free)
        _check(load_library().eqs_shifted_solve(self._h, C.c_double(t), _dp(_f64(z)), C.c_double(gdt),
                                                _dp(_f64(rhs)), _dp(d), C.c_int(1 if refresh_precond else 0)))
        return d

    def sdirk_advance_fixed(self, dt: float, nsteps: int = 1, newton_tol=1e-8, max_newton=25):
        o = _SdirkOptions(1e-2, 1e-8, newton_tol, max_newton)
        _check(load_library().eqs_sdirk_advance_fixed(self._h, C.c_double(dt), C.c_int(nsteps), C.byref(o)))

    # --- instrumentation / options
    def set_option(self, key: int, value: float):
        _check(load_library().eqs_set_option(self._h, C.c_int(key), C.c_double(value)))

    def timing(self, enable: bool | None = None):
        L = load_library()
        if enable is not None:
            _check(L.eqs_timing_enable(self._h, C.c_int(1 if enable else 0)))
            return None
        t = _Timing()
        _check(L.eqs_timing_get(self._h, C.byref(t)))
        return dict(ms=list(t.ms), launches=list(t.launches), bytes=list(t.bytes))

    def timing_reset(self):
        _check(load_library().eqs_timing_reset(self._h))


class ShmComm:
    """The shared-memory transport on host buffers (no GPU needed): the
    exchange/allreduce protocol of eqs_create_distributed_shm."""

    def __init__(self, shm_name: str, nranks: int, rank: int):
        self._h = C.c_void_p()
        _check(load_library().eqs_comm_open_shm(shm_name.encode(), C.c_int(nranks), C.c_int(rank),
                                                C.byref(self._h)))

    def close(self):
        if self._h:
            load_library().eqs_comm_close(self._h)
            self._h = None

    def barrier(self):
        _check(load_library().eqs_comm_barrier(self._h))

    def allreduce(self, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float64).copy()
        _check(load_library().eqs_comm_allreduce_host(self._h, _dp(a), C.c_int(a.size)))
        return a

    def exchange(self, sends: dict, recv_counts: dict) -> dict:
        """sends: peer -> float64 array; recv_counts: peer -> count. Returns peer -> received array."""
        peers = sorted(set(sends) | set(recv_counts))
        recv = {p: np.zeros(recv_counts.get(p, 0)) for p in peers}
        snd = [np.ascontiguousarray(sends.get(p, np.zeros(0)), dtype=np.float64) for p in peers]
        n = len(peers)
        P = C.POINTER(C.c_double)
        _check(load_library().eqs_comm_exchange_host(
            self._h, C.c_int(n), (C.c_int * n)(*peers), (P * n)(*[_dp(a) for a in snd]),
            (C.c_int * n)(*[a.size for a in snd]), (P * n)(*[_dp(recv[p]) for p in peers]),
            (C.c_int * n)(*[recv[p].size for p in peers])))
        return recv


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load_library().eqs_nccl_unique_id(buf))
    return buf.raw


def run_scenario(config, out_dir: str = "", device: int = 0, x_cap: int = 1 << 26) -> dict:
    """run_scenario (proj/src/scenario.cpp:217-383) on the GPU backend."""
    L = load_library()
    text = config if isinstance(config, str) else json.dumps(config)
    res = _RunResult()
    x = np.zeros(max(1, x_cap)) if x_cap else None
    rc = L.eqs_run_scenario(text.encode(), out_dir.encode(), C.c_int(device), C.byref(res),
                            _dp(x) if x is not None else None, C.c_long(x_cap))
    out = dict(exit_code=res.exit_code, accepted=res.accepted, rejected=res.rejected, stages=res.stages,
               final_t=res.final_t, wall_time=res.wall_time, n_free=res.n_free,
               stats={n: getattr(res.stats, n) for n, _ in _SolveStats._fields_})
    if x is not None and res.n_free <= x_cap:
        out["x"] = x[:res.n_free].copy()
    if rc != 0:
        if res.exit_code == 0:  # failed before the run started (config parse): raise like from_json_text
            _check(rc)
        out["error"] = L.eqs_last_error().decode()  # run failures are reported, never thrown (scenario.hpp:83-85)
    return out
