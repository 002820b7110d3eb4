"""ctypes harness for the HALLaR CPU oracle (oracle/_build/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py — never by the product
package.  Factors cross this boundary column-major (the reference's Eigen
layout, /root/reference/proj/include/lrsdp/types.hpp:9).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_longlong)
_vp = C.c_void_p


class OrcConfig(C.Structure):
    _fields_ = [
        ("eps", C.c_double), ("beta0", C.c_double), ("beta_growth", C.c_double),
        ("eps0", C.c_double), ("eps_decay", C.c_double), ("eps_floor", C.c_double),
        ("max_outer", C.c_int), ("time_limit", C.c_double), ("seed", C.c_ulonglong),
        ("eig_tol", C.c_double), ("eig_max_iters", C.c_int), ("eig_block_restart", C.c_int),
        ("aipp_lambda0", C.c_double), ("aipp_rho", C.c_double), ("aipp_max_outer", C.c_int),
        ("aipp_lambda_underflow", C.c_double), ("fista_sigma", C.c_double),
        ("fista_chi", C.c_double), ("fista_mu", C.c_double), ("fista_L0", C.c_double),
        ("fista_max_iters", C.c_int), ("max_fw_steps", C.c_int), ("threads", C.c_int),
    ]


class OrcReport(C.Structure):
    _fields_ = [
        ("status", C.c_int), ("pval", C.c_double), ("dval", C.c_double),
        ("dval_no_theta", C.c_double), ("rel_pfeas", C.c_double), ("rel_gap", C.c_double),
        ("rel_dfeas", C.c_double), ("rank", C.c_longlong), ("outer_iters", C.c_int),
        ("fw_steps", C.c_int), ("aipp_iters", C.c_longlong), ("fista_iters", C.c_longlong),
        ("eig_products", C.c_longlong), ("wall_seconds", C.c_double), ("tau", C.c_double),
        ("theta", C.c_double), ("message", C.c_char * 256),
    ]


class OrcTrace(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("outer_iter", C.c_int), ("beta", C.c_double),
        ("eps_inner", C.c_double), ("gap", C.c_double), ("theta", C.c_double),
        ("rank", C.c_longlong), ("al_value", C.c_double), ("fw_alpha", C.c_double),
        ("rel_pfeas", C.c_double), ("rel_gap", C.c_double), ("rel_dfeas", C.c_double),
    ]


_TRACE_FN = C.CFUNCTYPE(None, C.POINTER(OrcTrace), C.c_void_p)
STATUS = {0: "optimal", 1: "iteration_limit", 2: "time_limit", 3: "numerical_failure"}


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (g++ only)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.orc_last_error.restype = C.c_char_p
        L.orc_matcomp_count.restype = C.c_longlong
        L.orc_get_pairs.restype = C.c_longlong
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def _ptr(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _colmajor(U):
    U = np.asarray(U, dtype=np.float64)
    if U.ndim == 1:
        U = U[:, None]
    return np.asfortranarray(U)


def default_config(**kw) -> OrcConfig:
    """SolverConfig defaults (reference solver.hpp:12-29, lanczos.hpp:12-19,
    adap_aipp.hpp:8-16, adap_fista.hpp:24-32)."""
    c = OrcConfig(eps=1e-5, beta0=0.0, beta_growth=2.0, eps0=0.0, eps_decay=0.5,
                  eps_floor=0.0, max_outer=500, time_limit=3600.0, seed=0, eig_tol=1e-8,
                  eig_max_iters=5000, eig_block_restart=30, aipp_lambda0=10.0, aipp_rho=1e-4,
                  aipp_max_outer=2000, aipp_lambda_underflow=1e-12, fista_sigma=0.3,
                  fista_chi=0.5, fista_mu=0.5, fista_L0=1.0, fista_max_iters=0,
                  max_fw_steps=500, threads=-1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


@dataclass
class OracleReport:
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
    tau: float
    theta: float
    message: str
    U: np.ndarray = None
    p: np.ndarray = None
    trace: list = field(default_factory=list)


class OracleInstance:
    """One oracle SdpInstance (theta / matcomp / phaseret / dense)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)
        ints = (C.c_longlong * 5)()
        dbls = (C.c_double * 4)()
        lib().orc_info(self._h, ints, dbls)
        self.n, self.m = ints[0], ints[1]
        self.identity_constraint = None if ints[2] < 0 else ints[2]
        self.field_kind = ints[3]
        self.family = ("theta", "matcomp", "phaseret", "dense", "gauss_pr")[ints[4]]
        self.tau, self.norm_b1, self.norm_C1, self.nuclear_norm = dbls[0], dbls[1], dbls[2], dbls[3]

    def __del__(self):
        try:
            lib().orc_free(self._h)
        except Exception:
            pass

    # -- constructors (reference instances.hpp / graph.hpp) --
    @classmethod
    def hypercube(cls, d):
        h = _vp()
        _check(lib().orc_theta_hypercube(C.c_int(d), C.byref(h)))
        return cls(h.value)

    @classmethod
    def cycle(cls, n):
        h = _vp()
        _check(lib().orc_theta_cycle(C.c_int(n), C.byref(h)))
        return cls(h.value)

    @classmethod
    def petersen(cls):
        h = _vp()
        _check(lib().orc_theta_petersen(C.byref(h)))
        return cls(h.value)

    @classmethod
    def theta_edges(cls, n, ei, ej):
        ei = np.ascontiguousarray(ei, dtype=np.int64)
        ej = np.ascontiguousarray(ej, dtype=np.int64)
        h = _vp()
        _check(lib().orc_theta_edges(C.c_longlong(n), C.c_longlong(len(ei)),
                                     ei.ctypes.data_as(_lp), ej.ctypes.data_as(_lp), C.byref(h)))
        return cls(h.value)

    @classmethod
    def matcomp(cls, n1, n2, r, seed=0, offset=False, tau_safety=1.2):
        h = _vp()
        _check(lib().orc_matcomp(C.c_longlong(n1), C.c_longlong(n2), C.c_int(r),
                                 C.c_ulonglong(seed), C.c_int(int(offset)),
                                 C.c_double(tau_safety), C.byref(h)))
        return cls(h.value)

    @classmethod
    def matcomp_paper(cls, n1, n2, r, seed=0, draws_per_dim=40, tau_safety=1.2):
        """The paper's sampling rule (draws_per_dim * (n1 + n2) draws with
        replacement, deduplicated) — SURVEY §8(f) row 2; not in the reference."""
        h = _vp()
        _check(lib().orc_matcomp_paper(C.c_longlong(n1), C.c_longlong(n2), C.c_int(r), C.c_ulonglong(seed),
                                       C.c_longlong(draws_per_dim * (n1 + n2)), C.c_double(tau_safety),
                                       C.byref(h)))
        return cls(h.value)

    @classmethod
    def phaseret(cls, n, L, seed=0, tau_slack=1.1):
        h = _vp()
        _check(lib().orc_phaseret(C.c_longlong(n), C.c_int(L), C.c_ulonglong(seed),
                                  C.c_double(tau_slack), C.byref(h)))
        return cls(h.value)

    @classmethod
    def gauss_pr(cls, A, x, tau_slack=1.1):
        """Gaussian-measurement phase retrieval (not in the
        reference): b_i = |a_i^* x|^2 for the rows a_i of the complex m x n A."""
        A = np.asarray(A, dtype=np.complex128)
        x = np.asarray(x, dtype=np.complex128)
        m, n = A.shape
        are = np.ascontiguousarray(A.real)
        aim = np.ascontiguousarray(A.imag)
        xr = np.ascontiguousarray(x.real)
        xi = np.ascontiguousarray(x.imag)
        h = _vp()
        _check(lib().orc_gauss_pr(C.c_longlong(n), C.c_longlong(m), _ptr(are), _ptr(aim), _ptr(xr), _ptr(xi),
                                  C.c_double(tau_slack), C.byref(h)))
        return cls(h.value)

    @classmethod
    def dense(cls, Cm, As, b, tau=1.0):
        Cm = np.asfortranarray(Cm, dtype=np.float64)
        n = Cm.shape[0]
        m = len(As)
        A = np.concatenate([np.asfortranarray(a, dtype=np.float64).ravel(order="F") for a in As])
        b = _f64(b)
        h = _vp()
        _check(lib().orc_dense(C.c_longlong(n), C.c_longlong(m), _ptr(Cm.ravel(order="F")),
                               _ptr(A), _ptr(b), C.c_double(tau), C.byref(h)))
        return cls(h.value)

    # -- data --
    @property
    def b(self):
        out = np.empty(self.m)
        lib().orc_get_b(self._h, _ptr(out))
        return out

    def pairs(self):
        cnt = lib().orc_get_pairs(self._h, None, None)
        i = np.empty(cnt, dtype=np.int64)
        j = np.empty(cnt, dtype=np.int64)
        lib().orc_get_pairs(self._h, i.ctypes.data_as(_lp), j.ctypes.data_as(_lp))
        return i, j

    def pr_data(self):
        nc = self.n // 2
        L = self.m // nc
        x = np.empty(nc, dtype=np.complex128)
        masks = np.empty(nc * L, dtype=np.complex128)
        lib().orc_get_pr(self._h, x.ctypes.data_as(_dp), masks.ctypes.data_as(_dp))
        return x, masks.reshape(L, nc).T

    # -- operators (reference SdpInstance callables) --
    def apply_map(self, U):
        U = _colmajor(U)
        out = np.empty(self.m)
        _check(lib().orc_apply_map(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(out)))
        return out

    def apply_C(self, U):
        U = _colmajor(U)
        out = np.empty_like(U, order="F")
        _check(lib().orc_apply_C(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(out)))
        return out

    def apply_adjoint(self, p, U):
        U = _colmajor(U)
        p = _f64(p)
        out = np.empty_like(U, order="F")
        _check(lib().orc_apply_adjoint(self._h, _ptr(p), _ptr(U), C.c_longlong(U.shape[1]), _ptr(out)))
        return out

    def C_plus_adjoint(self, q, U):
        U = _colmajor(U)
        q = _f64(q)
        out = np.empty_like(U, order="F")
        _check(lib().orc_apply_C_plus_adjoint(self._h, _ptr(q), _ptr(U), C.c_longlong(U.shape[1]),
                                              _ptr(out)))
        return out

    def al_value(self, U, p, beta):
        U = _colmajor(U)
        p = _f64(p)
        v = C.c_double()
        _check(lib().orc_al_value(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(p),
                                  C.c_double(beta), C.byref(v)))
        return v.value

    def al_gradient(self, U, p, beta):
        U = _colmajor(U)
        p = _f64(p)
        out = np.empty_like(U, order="F")
        _check(lib().orc_al_gradient(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(p),
                                     C.c_double(beta), _ptr(out)))
        return out

    def al_value_and_gradient(self, U, p, beta):
        U = _colmajor(U)
        p = _f64(p)
        v = C.c_double()
        out = np.empty_like(U, order="F")
        _check(lib().orc_al_value_and_gradient(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(p),
                                               C.c_double(beta), C.byref(v), _ptr(out)))
        return v.value, out

    def min_eig_G(self, U, p, beta, tol=1e-8, max_iters=5000, block_restart=30, seed=0):
        U = _colmajor(U)
        p = _f64(p)
        lam, res = C.c_double(), C.c_double()
        mv, conv = C.c_int(), C.c_int()
        v = np.empty(self.n)
        _check(lib().orc_min_eig_G(self._h, _ptr(U), C.c_longlong(U.shape[1]), _ptr(p),
                                   C.c_double(beta), C.c_double(tol), C.c_int(max_iters),
                                   C.c_int(block_restart), C.c_ulonglong(seed), C.byref(lam),
                                   _ptr(v), C.byref(res), C.byref(mv), C.byref(conv)))
        return dict(lambda_=lam.value, v=v, residual=res.value, matvecs=mv.value,
                    converged=bool(conv.value))

    def aipp(self, p, beta, W, rho, cfg=None):
        W = _colmajor(W)
        p = _f64(p)
        cfg = cfg or default_config()
        Wout = np.empty_like(W, order="F")
        st, pi, fi = C.c_int(), C.c_int(), C.c_int()
        rn, gv, lam = C.c_double(), C.c_double(), C.c_double()
        _check(lib().orc_aipp_al(self._h, _ptr(p), C.c_double(beta), _ptr(W),
                                 C.c_longlong(W.shape[1]), C.c_double(rho), C.byref(cfg),
                                 _ptr(Wout), C.byref(st), C.byref(pi), C.byref(fi), C.byref(rn),
                                 C.byref(gv), C.byref(lam)))
        return dict(W=Wout, status=st.value, prox_iters=pi.value, fista_iters=fi.value,
                    R_norm=rn.value, g_value=gv.value, lambda_=lam.value)

    def solve(self, cfg=None, U0=None, p0=None, trace=False, **kw):
        cfg = cfg or default_config(**kw)
        rep = OrcReport()
        events = []

        def _cb(ev, _user):
            e = ev.contents
            events.append({k: getattr(e, k) for k, _ in OrcTrace._fields_})

        cb = _TRACE_FN(_cb) if trace else _TRACE_FN()
        cap = self.n * 600
        Uout = np.zeros(cap)
        pout = np.empty(self.m)
        if U0 is not None:
            U0 = _colmajor(U0)
            p0a = _f64(p0) if p0 is not None else np.zeros(self.m)
            rc = lib().orc_solve(self._h, C.byref(cfg), _ptr(U0), C.c_longlong(U0.shape[1]),
                                 _ptr(p0a), C.byref(rep), _ptr(Uout), C.c_longlong(cap),
                                 _ptr(pout), cb, None)
        else:
            rc = lib().orc_solve(self._h, C.byref(cfg), None, C.c_longlong(0), None, C.byref(rep),
                                 _ptr(Uout), C.c_longlong(cap), _ptr(pout), cb, None)
        _check(rc)
        r = OracleReport(status=STATUS[rep.status], pval=rep.pval, dval=rep.dval,
                         dval_no_theta=rep.dval_no_theta, rel_pfeas=rep.rel_pfeas,
                         rel_gap=rep.rel_gap, rel_dfeas=rep.rel_dfeas, rank=rep.rank,
                         outer_iters=rep.outer_iters, fw_steps=rep.fw_steps,
                         aipp_iters=rep.aipp_iters, fista_iters=rep.fista_iters,
                         eig_products=rep.eig_products, wall_seconds=rep.wall_seconds,
                         tau=rep.tau, theta=rep.theta, message=rep.message.decode())
        r.U = Uout[: self.n * rep.rank].reshape(rep.rank, self.n).T.copy()
        r.p = pout
        r.trace = events
        return r


def matcomp_count(n1, n2, r, offset=False):
    return lib().orc_matcomp_count(C.c_longlong(n1), C.c_longlong(n2), C.c_int(r), C.c_int(int(offset)))


def min_eig_dense(A, tol=1e-8, max_iters=5000, block_restart=30, seed=0):
    A = np.asfortranarray(A, dtype=np.float64)
    n = A.shape[0]
    lam, res = C.c_double(), C.c_double()
    mv, conv = C.c_int(), C.c_int()
    v = np.empty(n)
    _check(lib().orc_min_eig_dense(C.c_longlong(n), _ptr(A.ravel(order="F")), C.c_double(tol),
                                   C.c_int(max_iters), C.c_int(block_restart), C.c_ulonglong(seed),
                                   C.byref(lam), _ptr(v), C.byref(res), C.byref(mv), C.byref(conv)))
    return dict(lambda_=lam.value, v=v, residual=res.value, matvecs=mv.value,
                converged=bool(conv.value))


def jacobi_eigh(H):
    H = np.asfortranarray(H, dtype=np.float64)
    k = H.shape[0]
    ev = np.empty(k)
    evec = np.empty((k, k), order="F")
    lib().orc_jacobi_eigh(C.c_int(k), _ptr(H.ravel(order="F")), _ptr(ev), evec.ctypes.data_as(_dp))
    return ev, evec
