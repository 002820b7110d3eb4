"""Python mirror of the reference lrsdp API over libcuhallar.so (ctypes).

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/lrsdp/*.hpp):

* ``make_hypercube`` / ``make_cycle`` / ``make_petersen`` / ``load_graph``
  (graph.hpp), ``build_theta_instance`` (instances.hpp:16),
* ``McSpec`` + ``gen_matrix_completion`` + ``matcomp_constraint_count``
  (instances.hpp:24-53), ``PrSpec`` + ``gen_phase_retrieval`` (:60-78),
* ``SdpInstance`` operator callables ``apply_map`` / ``apply_C`` /
  ``apply_adjoint`` / ``C_plus_adjoint`` and ``al_value`` / ``al_gradient`` /
  ``AlFunction.value_and_gradient`` (sdp_instance.hpp),
* ``SolverConfig`` / ``SolveReport`` / ``solve`` (solver.hpp), ``TraceEvent``.

Errors map to the reference exception classes: ``InputError`` (status 64),
``NumericalError`` (3), ``OSError`` (66).  There is no CPU fallback: every
operator and the solve run on the GPU through the C-ABI; importing this module
fails loudly when the shared library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import warnings
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CUHALLAR_LIB") or os.path.join(_HERE, "libcuhallar.so")  # override: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)
_lib.cuhallar_last_error.restype = C.c_char_p
_lib.cuhallar_version.restype = C.c_char_p
_lib.cuhallar_matcomp_constraint_count.restype = C.c_int64

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


class InputError(ValueError):
    """lrsdp::InputError (types.hpp:14-17)."""


class NumericalError(RuntimeError):
    """lrsdp::NumericalError (types.hpp:20-23)."""


class CapacityError(RuntimeError):
    """A device capacity was exceeded (status 71: factor rank above 32, Lanczos
    slots); not a CUDA fault."""


class CudaError(RuntimeError):
    pass


def _check(rc: int):
    if rc == 0:
        return
    msg = _lib.cuhallar_last_error().decode()
    if rc == 64:
        raise InputError(msg)
    if rc == 3:
        raise NumericalError(msg)
    if rc == 66:
        raise OSError(msg)
    if rc == 71:
        raise CapacityError(msg)
    raise CudaError(f"cuhallar error {rc}: {msg}")


class CConfig(C.Structure):
    _fields_ = [
        ("eps", C.c_double), ("beta0", C.c_double), ("beta_growth", C.c_double),
        ("eps0", C.c_double), ("eps_decay", C.c_double), ("eps_floor", C.c_double),
        ("max_outer", C.c_int), ("time_limit", C.c_double), ("seed", C.c_uint64),
        ("eig_tol", C.c_double), ("eig_max_iters", C.c_int), ("eig_block_restart", C.c_int),
        ("aipp_lambda0", C.c_double), ("aipp_rho", C.c_double), ("aipp_max_outer", C.c_int),
        ("aipp_lambda_underflow", C.c_double), ("fista_sigma", C.c_double),
        ("fista_chi", C.c_double), ("fista_mu", C.c_double), ("fista_L0", C.c_double),
        ("fista_max_iters", C.c_int), ("max_fw_steps", C.c_int), ("threads", C.c_int),
        ("trace", C.c_int), ("team_ctas", C.c_int), ("profile", C.c_int),
        ("parity", C.c_int),
    ]


class CReport(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("pval", C.c_double), ("dval", C.c_double),
        ("dval_no_theta", C.c_double), ("rel_pfeas", C.c_double), ("rel_gap", C.c_double),
        ("rel_dfeas", C.c_double), ("rank", C.c_int64), ("outer_iters", C.c_int),
        ("fw_steps", C.c_int), ("aipp_iters", C.c_int64), ("fista_iters", C.c_int64),
        ("eig_products", C.c_int64), ("wall_seconds", C.c_double),
        ("device_seconds", C.c_double), ("tau", C.c_double), ("theta", C.c_double),
        ("trace_dropped", C.c_int64), ("message", C.c_char * 256),
    ]


class CInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("m", C.c_int64), ("identity_constraint", C.c_int64),
        ("field_kind", C.c_int), ("family", C.c_int), ("tau", C.c_double),
        ("norm_b1", C.c_double), ("norm_C1", C.c_double), ("nuclear_norm", C.c_double),
        ("device_bytes", C.c_int64), ("h2d_bytes", C.c_int64), ("team_ctas", C.c_int),
    ]


class CTrace(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("outer_iter", C.c_int), ("beta", C.c_double),
        ("eps_inner", C.c_double), ("gap", C.c_double), ("theta", C.c_double),
        ("rank", C.c_int64), ("al_value", C.c_double), ("fw_alpha", C.c_double),
        ("rel_pfeas", C.c_double), ("rel_gap", C.c_double), ("rel_dfeas", C.c_double),
    ]


_TRACE_FN = C.CFUNCTYPE(None, C.POINTER(CTrace), C.c_void_p)

STATUS = {0: "optimal", 1: "iteration_limit", 2: "time_limit", 3: "numerical_failure"}
TRACE_KIND = {0: "inner_stationary", 1: "inner_rank_step", 2: "outer", 9: "fista_debug",
              10: "parity_jobs"}


def version() -> str:
    return _lib.cuhallar_version().decode()


# ------------------------------------------------------------------ graphs --
@dataclass
class Graph:
    """lrsdp::Graph (graph.hpp:10-15); edges 0-based, i < j, sorted."""
    n_vertices: int
    edges: Optional[np.ndarray] = None  # (E, 2) int64
    _generator: Optional[tuple] = None  # ("hypercube", d) | ("cycle", n) | ("petersen",) | ("file", path, fmt)


def make_hypercube(d: int) -> Graph:
    return Graph(n_vertices=1 << d, _generator=("hypercube", d))


def make_cycle(n: int) -> Graph:
    return Graph(n_vertices=n, _generator=("cycle", n))


def make_petersen() -> Graph:
    return Graph(n_vertices=10, _generator=("petersen",))


_FORMATS = {"edge-list": 0, "matrix-market": 1, "mm": 1, "matrix-market-pattern": 1, "gset": 2}


def load_graph(path: str, fmt: str = "edge-list") -> Graph:
    if fmt not in _FORMATS:
        raise InputError(f"unknown graph format '{fmt}'")
    return Graph(n_vertices=0, _generator=("file", path, _FORMATS[fmt]))


def graph_from_edges(n_vertices: int, edges) -> Graph:
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return Graph(n_vertices=n_vertices, edges=e)


# ---------------------------------------------------------------- instances --
class SdpInstance:
    """Device-resident operator-form SDP (sdp_instance.hpp:22-50)."""

    def __init__(self, handle: C.c_void_p, kind: str):
        self._h = handle
        self.kind = kind
        info = CInfo()
        _check(_lib.cuhallar_instance_get_info(self._h, C.byref(info)))
        self.n = int(info.n)
        self.m = int(info.m)
        self.identity_constraint = None if info.identity_constraint < 0 else int(info.identity_constraint)
        self.field_kind = int(info.field_kind)
        self.tau = float(info.tau)
        self.norm_b1 = float(info.norm_b1)
        self.norm_C1 = float(info.norm_C1)
        self.nuclear_norm = float(info.nuclear_norm)
        self.device_bytes = int(info.device_bytes)

    def info(self) -> dict:
        i = CInfo()
        _check(_lib.cuhallar_instance_get_info(self._h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in CInfo._fields_}

    def __del__(self):
        try:
            if self._h:
                _lib.cuhallar_instance_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def b(self) -> np.ndarray:
        out = np.empty(self.m)
        _check(_lib.cuhallar_instance_get_b(self._h, out.ctypes.data_as(_dp)))
        return out

    def pairs(self):
        cnt = self.m - (1 if self.identity_constraint is not None else 0)
        i = np.empty(cnt, dtype=np.int64)
        j = np.empty(cnt, dtype=np.int64)
        _check(_lib.cuhallar_instance_get_pairs(self._h, i.ctypes.data_as(_i64p), j.ctypes.data_as(_i64p)))
        return i, j

    def pr_data(self):
        """PrInstance::hidden_x (nc) and masks (nc x L) of a phase-retrieval instance."""
        if self.kind != "phaseret":
            raise InputError("pr_data: not a phase-retrieval instance")
        nc = self.n // 2
        L = self.m // nc
        x = np.empty(nc, dtype=np.complex128)
        masks = np.empty(nc * L, dtype=np.complex128)
        _check(_lib.cuhallar_instance_get_phaseret(self._h, x.ctypes.data_as(_dp), masks.ctypes.data_as(_dp)))
        return x, masks.reshape(L, nc).T

    def gauss_data(self):
        """Measurement matrix A (m x n complex, rows a_i) and signal x of a
        Gaussian phase-retrieval instance."""
        if self.kind != "gauss_pr":
            raise InputError("gauss_data: not a Gaussian phase-retrieval instance")
        n = self.n // 2
        are = np.empty((self.m, n))
        aim = np.empty((self.m, n))
        _check(_lib.cuhallar_instance_get_gauss(self._h, are.ctypes.data_as(_dp), aim.ctypes.data_as(_dp)))
        x = np.empty(n, dtype=np.complex128)
        _check(_lib.cuhallar_instance_get_phaseret(self._h, x.ctypes.data_as(_dp), None))
        return are + 1j * aim, x

    # -- operator callables; U is n x s (numpy or torch), results numpy --
    def _dev_factor(self, U):
        import torch
        if isinstance(U, torch.Tensor):
            T = U.detach().to(device="cuda", dtype=torch.float64)
        else:
            T = torch.as_tensor(np.asarray(U, dtype=np.float64), device="cuda")
        if T.dim() == 1:
            T = T[:, None]
        if T.shape[0] != self.n:
            raise InputError(f"factor has {T.shape[0]} rows, instance needs {self.n}")
        if T.shape[1] < 1:
            raise InputError("factor must have >= 1 column")
        return T.t().contiguous(), T.shape[1]  # column-major n x s, ld = n

    def _dev_vec(self, p):
        import torch
        t = torch.as_tensor(np.asarray(p, dtype=np.float64) if not isinstance(p, torch.Tensor) else p,
                            dtype=torch.float64, device="cuda").contiguous()
        if t.numel() != self.m:
            raise InputError(f"multiplier has length {t.numel()}, instance needs {self.m}")
        return t

    @staticmethod
    def _ptr(t):
        return C.cast(C.c_void_p(t.data_ptr()), _dp)

    def _mat_out(self, s):
        import torch
        return torch.empty((s, self.n), dtype=torch.float64, device="cuda")

    def apply_map(self, U) -> np.ndarray:
        import torch
        Ut, s = self._dev_factor(U)
        out = torch.empty(self.m, dtype=torch.float64, device="cuda")
        _check(_lib.cuhallar_apply_map(self._h, self._ptr(Ut), C.c_int64(self.n), C.c_int(s),
                                       self._ptr(out), None))
        return out.cpu().numpy()

    def apply_C(self, U) -> np.ndarray:
        Ut, s = self._dev_factor(U)
        out = self._mat_out(s)
        _check(_lib.cuhallar_apply_C(self._h, self._ptr(Ut), C.c_int64(self.n), C.c_int(s),
                                     self._ptr(out), C.c_int64(self.n), None))
        return out.t().cpu().numpy()

    def apply_adjoint(self, p, U) -> np.ndarray:
        Ut, s = self._dev_factor(U)
        pt = self._dev_vec(p)
        out = self._mat_out(s)
        _check(_lib.cuhallar_apply_adjoint(self._h, self._ptr(pt), self._ptr(Ut), C.c_int64(self.n),
                                           C.c_int(s), self._ptr(out), C.c_int64(self.n), None))
        return out.t().cpu().numpy()

    def C_plus_adjoint(self, q, U) -> np.ndarray:
        Ut, s = self._dev_factor(U)
        qt = self._dev_vec(q)
        out = self._mat_out(s)
        _check(_lib.cuhallar_c_plus_adjoint(self._h, self._ptr(qt), self._ptr(Ut), C.c_int64(self.n),
                                            C.c_int(s), self._ptr(out), C.c_int64(self.n), None))
        return out.t().cpu().numpy()

    def al_value(self, U, p, beta) -> float:
        Ut, s = self._dev_factor(U)
        pt = self._dev_vec(p)
        v = C.c_double()
        _check(_lib.cuhallar_al_value(self._h, self._ptr(Ut), C.c_int64(self.n), C.c_int(s),
                                      self._ptr(pt), C.c_double(beta), C.byref(v), None))
        return v.value

    def al_gradient(self, U, p, beta) -> np.ndarray:
        Ut, s = self._dev_factor(U)
        pt = self._dev_vec(p)
        out = self._mat_out(s)
        _check(_lib.cuhallar_al_gradient(self._h, self._ptr(Ut), C.c_int64(self.n), C.c_int(s),
                                         self._ptr(pt), C.c_double(beta), self._ptr(out),
                                         C.c_int64(self.n), None))
        return out.t().cpu().numpy()

    def al_value_and_gradient(self, U, p, beta):
        Ut, s = self._dev_factor(U)
        pt = self._dev_vec(p)
        out = self._mat_out(s)
        v = C.c_double()
        _check(_lib.cuhallar_al_value_and_gradient(self._h, self._ptr(Ut), C.c_int64(self.n), C.c_int(s),
                                                   self._ptr(pt), C.c_double(beta), C.byref(v),
                                                   self._ptr(out), C.c_int64(self.n), None))
        return v.value, out.t().cpu().numpy()

    # -- sub-solvers (parity testing) --
    def min_eig_gradient(self, U, p, beta, tol=1e-8, max_iters=5000, block_restart=30, seed=0,
                         parity=False):
        U = np.asfortranarray(np.asarray(U, dtype=np.float64).reshape(self.n, -1))
        p = np.ascontiguousarray(p, dtype=np.float64)
        lam, res = C.c_double(), C.c_double()
        mv, conv = C.c_int(), C.c_int()
        v = np.empty(self.n)
        cc = SolverConfig(eig_max_iters=max_iters, eig_block_restart=block_restart, seed=seed,
                          parity=parity)._c()
        _check(_lib.cuhallar_min_eig_gradient_cfg(
            self._h, U.ctypes.data_as(_dp), C.c_int(U.shape[1]), p.ctypes.data_as(_dp), C.c_double(beta),
            C.c_double(tol), C.byref(cc), C.byref(lam),
            v.ctypes.data_as(_dp), C.byref(res), C.byref(mv), C.byref(conv)))
        return dict(lambda_=lam.value, v=v, residual=res.value, matvecs=mv.value, converged=bool(conv.value))

    def last_trace(self, cap=1 << 16) -> list:
        """Raw events of the last traced launch (tuples: kind, outer_iter, beta, eps_inner, gap,
        theta, rank, al_value, fw_alpha, rel_pfeas, rel_gap, rel_dfeas)."""
        buf = (CTrace * cap)()
        k = _lib.cuhallar_last_trace(self._h, buf, cap)
        return [tuple(getattr(buf[i], f) for f, _ in CTrace._fields_) for i in range(k)]

    PROFILE_CATS = ["fista_x~", "fista_value_grad", "fista_y+_map", "fista_grad_y+", "aipp",
                    "lanczos_apply", "lanczos_cgs2", "jacobi", "lanczos_measure", "lanczos_restart",
                    "gradient_operator", "fw_gap", "fw_step", "outer", "other"]

    def last_profile(self) -> dict:
        ns = (C.c_double * 16)()
        cnt = (C.c_int64 * 16)()
        k = _lib.cuhallar_last_profile(self._h, ns, cnt, 16)
        return {self.PROFILE_CATS[i]: (ns[i] * 1e-6, int(cnt[i])) for i in range(min(k, len(self.PROFILE_CATS)))}

    BENCH_KINDS = {"sync": 0, "allreduce": 1, "grad_pass": 2, "map_pass": 3, "lanczos_matvec": 4}

    def bench_pass(self, kind, U, p, beta=1.0, iters=100, team_ctas=0) -> float:
        """ns per pass of one solver phase, timed inside a persistent launch."""
        U = np.asfortranarray(np.asarray(U, dtype=np.float64).reshape(self.n, -1))
        p = np.ascontiguousarray(p, dtype=np.float64)
        ns = C.c_double()
        _check(_lib.cuhallar_bench_pass(self._h, C.c_int(self.BENCH_KINDS.get(kind, kind)),
                                        U.ctypes.data_as(_dp), C.c_int(U.shape[1]), p.ctypes.data_as(_dp),
                                        C.c_double(beta), C.c_int(iters), C.c_int(team_ctas), C.byref(ns)))
        return ns.value

    def aipp(self, p, beta, W, rho, cfg: "SolverConfig" = None):
        W = np.asfortranarray(np.asarray(W, dtype=np.float64).reshape(self.n, -1))
        p = np.ascontiguousarray(p, dtype=np.float64)
        cc = (cfg or SolverConfig())._c()
        Wout = np.empty_like(W, order="F")
        st, pi, fi = C.c_int(), C.c_int(), C.c_int()
        rn, gv, lam = C.c_double(), C.c_double(), C.c_double()
        _check(_lib.cuhallar_aipp(self._h, p.ctypes.data_as(_dp), C.c_double(beta), W.ctypes.data_as(_dp),
                                  C.c_int(W.shape[1]), C.c_double(rho), C.byref(cc),
                                  Wout.ctypes.data_as(_dp), C.byref(st), C.byref(pi), C.byref(fi),
                                  C.byref(rn), C.byref(gv), C.byref(lam)))
        return dict(W=Wout, status=st.value, prox_iters=pi.value, fista_iters=fi.value,
                    R_norm=rn.value, g_value=gv.value, lambda_=lam.value)


def _new(fn, *args, kind="theta") -> SdpInstance:
    h = C.c_void_p()
    _check(fn(*args, C.byref(h)))
    return SdpInstance(h, kind)


def build_theta_instance(g: Graph) -> SdpInstance:
    """build_theta_instance (instances.cpp:63-112)."""
    gen = g._generator
    if gen is not None:
        if gen[0] == "hypercube":
            return _new(_lib.cuhallar_theta_hypercube, C.c_int(gen[1]))
        if gen[0] == "cycle":
            return _new(_lib.cuhallar_theta_cycle, C.c_int(gen[1]))
        if gen[0] == "petersen":
            return _new(_lib.cuhallar_theta_petersen)
        if gen[0] == "file":
            return _new(_lib.cuhallar_theta_file, gen[1].encode(), C.c_int(gen[2]))
    e = np.ascontiguousarray(g.edges, dtype=np.int64).reshape(-1, 2)
    u = np.ascontiguousarray(e[:, 0])
    v = np.ascontiguousarray(e[:, 1])
    return _new(_lib.cuhallar_theta_edges, C.c_int64(g.n_vertices), C.c_int64(len(u)),
                u.ctypes.data_as(_i64p), v.ctypes.data_as(_i64p))


@dataclass
class McSpec:
    """McSpec (instances.hpp:24-34)."""
    n1: int = 0
    n2: int = 0
    r: int = 1
    seed: int = 0
    offset_sample_count: bool = False
    tau_safety: float = 1.2
    # not in the reference: draws_per_dim > 0 selects the paper's sampling rule,
    # draws_per_dim * (n1 + n2) draws with replacement, deduplicated
    draws_per_dim: int = 0


def matcomp_constraint_count(n1, n2, r, offset_sample_count=False) -> int:
    return int(_lib.cuhallar_matcomp_constraint_count(C.c_int64(n1), C.c_int64(n2), C.c_int(r),
                                                      C.c_int(int(offset_sample_count))))


def gen_matrix_completion(spec: McSpec) -> SdpInstance:
    """gen_matrix_completion (instances.cpp:131-234); returns the instance
    (omega via ``inst.pairs()``, ||M||_* via ``inst.nuclear_norm``).  With
    ``spec.draws_per_dim > 0`` the paper's sampling rule replaces the reference's."""
    if spec.draws_per_dim > 0:
        return _new(_lib.cuhallar_gen_matrix_completion_paper, C.c_int64(spec.n1), C.c_int64(spec.n2),
                    C.c_int(spec.r), C.c_uint64(spec.seed),
                    C.c_int64(spec.draws_per_dim * (spec.n1 + spec.n2)), C.c_double(spec.tau_safety),
                    kind="matcomp")
    return _new(_lib.cuhallar_gen_matrix_completion, C.c_int64(spec.n1), C.c_int64(spec.n2), C.c_int(spec.r),
                C.c_uint64(spec.seed), C.c_int(int(spec.offset_sample_count)),
                C.c_double(spec.tau_safety), kind="matcomp")


def matcomp_from_samples(n1: int, n2: int, i, j, b, tau: float) -> SdpInstance:
    """A matrix-completion SdpInstance from host sample arrays (the instance
    gen_matrix_completion builds, instances.cpp:190-234, for data the caller
    holds): (i, j) strictly increasing, b = M(i, j), trace bound tau.  The
    arrays are copied host -> device and the pair CSR is built on the GPU."""
    i = np.ascontiguousarray(i, dtype=np.int64)
    j = np.ascontiguousarray(j, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if not (len(i) == len(j) == len(b)):
        raise InputError("matcomp samples: i, j, b lengths differ")
    return _new(_lib.cuhallar_matcomp_from_samples, C.c_int64(n1), C.c_int64(n2), C.c_int64(len(i)),
                i.ctypes.data_as(_i64p), j.ctypes.data_as(_i64p), b.ctypes.data_as(_dp),
                C.c_double(tau), kind="matcomp")


@dataclass
class PrSpec:
    """PrSpec (instances.hpp:60-70)."""
    n: int = 0
    L: int = 1
    seed: int = 0
    tau_slack: float = 1.1


def gen_phase_retrieval(spec: PrSpec) -> SdpInstance:
    return _new(_lib.cuhallar_gen_phase_retrieval, C.c_int64(spec.n), C.c_int(spec.L),
                C.c_uint64(spec.seed), C.c_double(spec.tau_slack), kind="phaseret")


@dataclass
class GaussPrSpec:
    """Gaussian-measurement phase retrieval (BASELINE configs[2];
    not in the reference): m measurements b_i = |a_i^* x|^2 of an n-dimensional
    complex signal, a_i with i.i.d. CN(0, 1) entries."""
    n: int = 0
    m: int = 0
    seed: int = 0
    tau_slack: float = 1.1


def gen_gauss_phase_retrieval(spec: GaussPrSpec) -> SdpInstance:
    return _new(_lib.cuhallar_gen_gauss_phase_retrieval, C.c_int64(spec.n), C.c_int64(spec.m),
                C.c_uint64(spec.seed), C.c_double(spec.tau_slack), kind="gauss_pr")


# ------------------------------------------------------------------- solver --
@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:12-29) with EigSettings / AippParams / FistaParams."""
    eps: float = 1e-5
    beta0: float = 0.0
    beta_growth: float = 2.0
    eps0: float = 0.0
    eps_decay: float = 0.5
    eps_floor: float = 0.0
    max_outer: int = 500
    time_limit: float = 3600.0
    seed: int = 0
    eig_tol: float = 1e-8
    eig_max_iters: int = 5000
    eig_block_restart: int = 30
    aipp_lambda0: float = 10.0
    aipp_rho: float = 1e-4
    aipp_max_outer: int = 2000
    aipp_lambda_underflow: float = 1e-12
    fista_sigma: float = 0.3
    fista_chi: float = 0.5
    fista_mu: float = 0.5
    fista_L0: float = 1.0
    fista_max_iters: int = 0
    max_fw_steps: int = 500
    deterministic: bool = False
    threads: int = 0
    team_ctas: int = 0
    profile: bool = False
    # parity mode: every reduction in the reference binary's order so the
    # iteration counters match the CPU oracle (pair families, one GPU, slower)
    parity: bool = False

    def _c(self, trace=False) -> CConfig:
        c = CConfig()
        for name, _ in CConfig._fields_:
            if name == "trace":
                # debug (parity mode): CUHALLAR_DEBUG_FISTA=1 adds one "fista_debug" event per
                # FISTA call; CUHALLAR_DEBUG_JOBS=1 also records every job phase (inst.last_trace())
                c.trace = (2 if os.environ.get("CUHALLAR_DEBUG_FISTA") else 1) if trace else 0
                if os.environ.get("CUHALLAR_DEBUG_JOBS"):
                    c.trace = 3
            elif name == "profile":
                c.profile = 1 if self.profile else 0
            elif name == "parity":
                c.parity = 1 if self.parity else 0
            else:
                setattr(c, name, getattr(self, name))
        return c


@dataclass
class TraceEvent:
    kind: str
    outer_iter: int
    beta: float
    eps_inner: float
    gap: float
    theta: float
    rank: int
    al_value: float
    fw_alpha: float
    rel_pfeas: float
    rel_gap: float
    rel_dfeas: float


@dataclass
class SolveReport:
    """SolveReport (solver.hpp:40-61)."""
    status: str
    pval: float
    dval: float
    dval_no_theta: float
    rel_pfeas: float
    rel_gap: float
    rel_dfeas: float
    rank: int
    outer_iters: int
    fw_steps: int
    aipp_iters: int
    fista_iters: int
    eig_products: int
    wall_seconds: float
    device_seconds: float
    message: str
    tau: float
    theta: float
    U: np.ndarray = None
    p: np.ndarray = None
    trace: list = field(default_factory=list)


def solve(inst: SdpInstance, cfg: SolverConfig = None, U0=None, p0=None,
          sink: Optional[Callable[[TraceEvent], None]] = None, fetch: bool = True) -> SolveReport:
    """solve(inst, cfg, sink) / solve(inst, cfg, U0, p0, sink) (solver.hpp:95-101)."""
    cfg = cfg or SolverConfig()
    cc = cfg._c(trace=sink is not None)
    rep = CReport()
    sol = C.c_void_p()
    events = []

    def _cb(ev, _u):  # called while the solve runs (trace.hpp sink semantics)
        e = ev.contents
        te = TraceEvent(TRACE_KIND.get(e.kind, str(e.kind)), e.outer_iter, e.beta, e.eps_inner, e.gap,
                        e.theta, e.rank, e.al_value, e.fw_alpha, e.rel_pfeas, e.rel_gap, e.rel_dfeas)
        events.append(te)
        sink(te)

    cb = _TRACE_FN(_cb) if sink is not None else _TRACE_FN()
    U0p, s0, p0p, _keep = _start_args(inst, U0, p0)
    rc = _lib.cuhallar_solve(inst._h, C.byref(cc), U0p, C.c_int(s0), p0p, C.byref(rep), C.byref(sol),
                             cb, None)
    _check(rc)
    r = _report(inst, rep, sol, fetch)
    if sink is not None:
        r.trace = events
        if rep.trace_dropped > 0:  # the device ring overflowed: the sink missed events
            warnings.warn(f"solve: {rep.trace_dropped} trace events were dropped (device trace ring full)",
                          RuntimeWarning, stacklevel=2)
    return r


def _start_args(inst, U0, p0):
    if U0 is None:
        return None, 0, None, None
    U0a = np.asfortranarray(np.asarray(U0, dtype=np.float64).reshape(inst.n, -1))
    p0a = np.ascontiguousarray(p0 if p0 is not None else np.zeros(inst.m), dtype=np.float64)
    return U0a.ctypes.data_as(_dp), U0a.shape[1], p0a.ctypes.data_as(_dp), (U0a, p0a)


def solve_sharded(insts, cfg: SolverConfig = None, U0=None, p0=None, fetch: bool = True) -> SolveReport:
    """Row-sharded solve: ``insts[r]`` is the same instance built
    on rank r's device (``with torch.cuda.device(r): build(...)``).  Each rank's
    persistent launch owns a block of rows; gathered factor rows travel over
    peer memory and reductions join per-rank partials in rank order.  Ranks may
    share one device (co-resident launches).  Theta and matrix completion only."""
    cfg = cfg or SolverConfig()
    cc = cfg._c()
    rep = CReport()
    sol = C.c_void_p()
    arr = (C.c_void_p * len(insts))(*[i._h for i in insts])
    U0p, s0, p0p, _keep = _start_args(insts[0], U0, p0)
    _check(_lib.cuhallar_solve_sharded(arr, C.c_int(len(insts)), C.byref(cc), U0p, C.c_int(s0), p0p,
                                       C.byref(rep), C.byref(sol)))
    return _report(insts[0], rep, sol, fetch)


class ShardHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 512)]


def shard_export(inst: SdpInstance, team_ctas: int = 0) -> bytes:
    """This rank's IPC handles for the one-process-per-GPU sharded solve."""
    h = ShardHandle()
    _check(_lib.cuhallar_shard_export(inst._h, C.c_int(team_ctas), C.byref(h)))
    return bytes(h.bytes)


def solve_rank(inst: SdpInstance, world: int, rank: int, handles, cfg: SolverConfig = None,
               fetch: bool = False) -> SolveReport:
    """Row-sharded solve, one process per GPU (torchrun): ``handles[q]`` is rank q's
    ``shard_export`` blob (exchanged by any collective); every rank calls this
    concurrently and gets the same report."""
    cfg = cfg or SolverConfig()
    cc = cfg._c()
    arr = (ShardHandle * world)()
    for q, hb in enumerate(handles):
        C.memmove(arr[q].bytes, hb, 512)
    rep = CReport()
    sol = C.c_void_p()
    _check(_lib.cuhallar_solve_rank(inst._h, C.c_int(world), C.c_int(rank), arr, C.byref(cc), None, C.c_int(0),
                                    None, C.byref(rep), C.byref(sol)))
    return _report(inst, rep, sol, fetch)


def _report(inst, rep, sol, fetch) -> SolveReport:
    try:
        r = SolveReport(status=STATUS[rep.status], pval=rep.pval, dval=rep.dval,
                        dval_no_theta=rep.dval_no_theta, rel_pfeas=rep.rel_pfeas, rel_gap=rep.rel_gap,
                        rel_dfeas=rep.rel_dfeas, rank=int(rep.rank), outer_iters=rep.outer_iters,
                        fw_steps=rep.fw_steps, aipp_iters=int(rep.aipp_iters),
                        fista_iters=int(rep.fista_iters), eig_products=int(rep.eig_products),
                        wall_seconds=rep.wall_seconds, device_seconds=rep.device_seconds,
                        message=rep.message.decode(), tau=rep.tau, theta=rep.theta)
        if fetch:
            U = np.empty(inst.n * r.rank)
            _check(_lib.cuhallar_solution_get_U(sol, U.ctypes.data_as(_dp)))
            r.U = U.reshape(r.rank, inst.n).T.copy()
            p = np.empty(inst.m)
            _check(_lib.cuhallar_solution_get_p(sol, p.ctypes.data_as(_dp)))
            r.p = p
    finally:
        _lib.cuhallar_solution_destroy(sol)
    return r
