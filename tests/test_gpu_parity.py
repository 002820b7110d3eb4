"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Tolerances: per-kernel relative 1e-12 (the pair kernels
are bit-exact by construction except theta's column-sum term); AL values 1e-10;
final objectives 1e-6 (north_star)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_13719_b200 as H
    return H


def _pairs(H, O, name):
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5)), O.OracleInstance.cycle(5)
    if name == "petersen":
        return H.build_theta_instance(H.make_petersen()), O.OracleInstance.petersen()
    if name.startswith("H"):
        d = int(name[1:])
        return H.build_theta_instance(H.make_hypercube(d)), O.OracleInstance.hypercube(d)
    if name == "mc30":
        return (H.gen_matrix_completion(H.McSpec(30, 70, 2, seed=5)),
                O.OracleInstance.matcomp(30, 70, 2, seed=5))
    if name == "mc100":
        return (H.gen_matrix_completion(H.McSpec(100, 210, 3, seed=0)),
                O.OracleInstance.matcomp(100, 210, 3, seed=0))
    raise KeyError(name)


INSTANCES = ["C5", "petersen", "H6", "H10", "mc30", "mc100"]


def rel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("name", INSTANCES)
def test_instance_identity(H, orc, name):
    inst, ref = _pairs(H, orc, name)
    assert (inst.n, inst.m) == (ref.n, ref.m)
    assert inst.identity_constraint == ref.identity_constraint
    i, j = inst.pairs()
    ri, rj = ref.pairs()
    assert np.array_equal(i, ri) and np.array_equal(j, rj)
    assert np.array_equal(inst.b, ref.b)  # bit-identical right-hand side
    assert inst.tau == pytest.approx(ref.tau, rel=1e-13)
    assert inst.norm_b1 == ref.norm_b1 and inst.norm_C1 == ref.norm_C1


@pytest.mark.parametrize("name", INSTANCES)
@pytest.mark.parametrize("s", [1, 2, 3, 4, 6])
def test_operator_kernels(H, orc, name, s):
    inst, ref = _pairs(H, orc, name)
    rng = np.random.default_rng(100 + s)
    U = rng.standard_normal((inst.n, s))
    p = rng.standard_normal(inst.m)
    # map and the pair adjoint are bit-exact against the reference order
    assert np.array_equal(inst.apply_map(U)[: inst.m - (inst.identity_constraint is not None)],
                          ref.apply_map(U)[: ref.m - (ref.identity_constraint is not None)])
    assert rel(inst.apply_map(U), ref.apply_map(U)) <= 1e-13
    assert rel(inst.apply_C(U), ref.apply_C(U)) <= 1e-13
    assert rel(inst.apply_adjoint(p, U), ref.apply_adjoint(p, U)) <= 1e-13
    assert rel(inst.C_plus_adjoint(p, U), ref.C_plus_adjoint(p, U)) <= 1e-13
    if inst.identity_constraint is None:
        assert np.array_equal(inst.apply_adjoint(p, U), ref.apply_adjoint(p, U))
        assert np.array_equal(inst.C_plus_adjoint(p, U), ref.C_plus_adjoint(p, U))


@pytest.mark.parametrize("name", INSTANCES)
def test_al_functions(H, orc, name):
    inst, ref = _pairs(H, orc, name)
    rng = np.random.default_rng(7)
    for s in (1, 2, 3):
        U = 0.3 * rng.standard_normal((inst.n, s)) / math.sqrt(inst.n)
        p = rng.standard_normal(inst.m)
        beta = 2.5
        assert inst.al_value(U, p, beta) == pytest.approx(ref.al_value(U, p, beta), rel=1e-10, abs=1e-12)
        assert rel(inst.al_gradient(U, p, beta), ref.al_gradient(U, p, beta)) <= 1e-10
        v, g = inst.al_value_and_gradient(U, p, beta)
        rv, rg = ref.al_value_and_gradient(U, p, beta)
        assert v == pytest.approx(rv, rel=1e-10, abs=1e-12)
        assert rel(g, rg) <= 1e-10


def test_adjoint_fuzz(H, orc):
    # test_instances.cpp:27-41 on the device kernels
    inst = H.build_theta_instance(H.make_petersen())
    rng = np.random.default_rng(1002)
    for t in range(20):
        U = rng.standard_normal((inst.n, 1 + t % 3))
        p = rng.standard_normal(inst.m)
        lhs = inst.apply_map(U) @ p
        rhs = float(np.sum(inst.apply_adjoint(p, U) * U))
        assert abs(lhs - rhs) <= 1e-10 * (1 + abs(lhs))


@pytest.mark.parametrize("name", ["C5", "H6", "H10", "mc30"])
def test_lanczos_escape(H, orc, name):
    inst, ref = _pairs(H, orc, name)
    rng = np.random.default_rng(3)
    U = rng.standard_normal((inst.n, 2)); U /= np.linalg.norm(U)
    p = 0.1 * rng.standard_normal(inst.m)
    got = inst.min_eig_gradient(U, p, 3.0, tol=1e-9, seed=0)
    want = ref.min_eig_G(U, p, 3.0, tol=1e-9, seed=0)
    assert got["converged"] == want["converged"]
    assert got["lambda_"] == pytest.approx(want["lambda_"], rel=1e-8, abs=1e-10)
    assert abs(got["matvecs"] - want["matvecs"]) <= 2


@pytest.mark.parametrize("name", ["C5", "H6", "mc30"])
def test_aipp(H, orc, name):
    inst, ref = _pairs(H, orc, name)
    rng = np.random.default_rng(11)
    W = rng.standard_normal((inst.n, 2)); W /= 1.5 * np.linalg.norm(W)
    p = 0.05 * rng.standard_normal(inst.m)
    got = inst.aipp(p, 4.0, W, 1e-3)
    want = ref.aipp(p, 4.0, W, 1e-3)
    assert got["status"] == want["status"]
    assert got["prox_iters"] == want["prox_iters"]
    assert got["fista_iters"] == want["fista_iters"]
    assert got["g_value"] == pytest.approx(want["g_value"], rel=1e-9, abs=1e-12)
    assert rel(got["W"], want["W"]) <= 1e-8


@pytest.mark.parametrize("name,value,tol,relative", [
    ("C5", math.sqrt(5), 1e-4, False), ("petersen", 4.0, 1e-3, False),
    ("H4", 8.0, 1e-4, True), ("H6", 32.0, 1e-4, True), ("H10", 512.0, 1e-4, True)])
def test_solve_theta(H, orc, name, value, tol, relative):
    # acceptance.cpp criteria 1 and 2 on the device, compared with the oracle
    inst, ref = _pairs(H, orc, name)
    rep = H.solve(inst)
    want = ref.solve()
    assert rep.status == "optimal"
    err = abs(-rep.pval - value) / (value if relative else 1.0)
    assert err <= tol
    assert abs(rep.pval - want.pval) <= 1e-6 * max(1.0, abs(want.pval))
    assert max(rep.rel_pfeas, rep.rel_gap, rep.rel_dfeas) <= 1e-5
    assert rep.rank == want.rank
    if name == "H10":
        assert rep.rank == 2


@pytest.mark.parametrize("name", ["mc30", "mc100"])
def test_solve_matcomp(H, orc, name):
    inst, ref = _pairs(H, orc, name)
    rep = H.solve(inst)
    want = ref.solve()
    assert rep.status == "optimal" and rep.rank == want.rank
    assert abs(rep.pval - want.pval) <= 1e-6 * abs(want.pval)
    assert abs(rep.pval - inst.nuclear_norm) / inst.nuclear_norm <= 1e-3


def test_solve_deterministic_and_warm(H, orc):
    inst = H.build_theta_instance(H.make_petersen())
    a = H.solve(inst, H.SolverConfig(eps=1e-4, seed=42))
    b = H.solve(inst, H.SolverConfig(eps=1e-4, seed=42))
    assert a.pval == b.pval and np.array_equal(a.U, b.U) and np.array_equal(a.p, b.p)
    c5 = H.build_theta_instance(H.make_cycle(5))
    r = H.solve(c5)
    again = H.solve(c5, U0=r.U, p0=r.p)
    assert again.status == "optimal" and again.outer_iters == 1


def test_trace_events(H, orc):
    """Fast-mode trace (trace.hpp:12-26) against the oracle's on C5, whose
    counters agree: same event kinds, outer iterations, ranks and penalties,
    values to 1e-9."""
    inst = H.build_theta_instance(H.make_cycle(5))
    ev = []
    rep = H.solve(inst, sink=ev.append)
    outer = [e for e in ev if e.kind == "outer"]
    assert len(outer) == rep.outer_iters and all(e.theta >= 0 for e in outer)
    kinds = {0: "inner_stationary", 1: "inner_rank_step", 2: "outer"}
    o = orc.OracleInstance.cycle(5).solve(trace=True)
    dev = [e for e in ev if e.kind in kinds.values()]
    assert [(e.kind, e.outer_iter, e.rank, e.beta) for e in dev] == \
        [(kinds[e["kind"]], e["outer_iter"], e["rank"], e["beta"]) for e in o.trace]
    for e, f in zip(dev, o.trace):
        assert abs(e.al_value - f["al_value"]) <= 1e-9 * max(1.0, abs(f["al_value"]))
        assert abs(e.rel_pfeas - f["rel_pfeas"]) <= 1e-9


def test_matcomp_paper_rule_instance_and_solve(H, orc):
    # paper sampling rule: device instance identical to the oracle's
    inst = H.gen_matrix_completion(H.McSpec(300, 700, 3, seed=1, draws_per_dim=40))
    ref = orc.OracleInstance.matcomp_paper(300, 700, 3, seed=1, draws_per_dim=40)
    assert (inst.n, inst.m) == (ref.n, ref.m)
    i, j = inst.pairs()
    ri, rj = ref.pairs()
    assert np.array_equal(i, ri) and np.array_equal(j, rj)
    assert np.array_equal(inst.b, ref.b)
    assert inst.tau == pytest.approx(ref.tau, rel=1e-13)
    small = H.gen_matrix_completion(H.McSpec(30, 70, 2, seed=5, draws_per_dim=12))
    small_ref = orc.OracleInstance.matcomp_paper(30, 70, 2, seed=5, draws_per_dim=12)
    rep = H.solve(small)
    want = small_ref.solve()
    assert rep.status == "optimal"
    assert abs(rep.pval - want.pval) <= 1e-6 * abs(want.pval)
