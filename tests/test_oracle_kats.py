"""Pins the CPU oracle against the reference's own known-answer tests.

Every expected value below is taken from the reference test-suite (file:line
cited per test); the reference itself cannot be compiled here (Eigen absent,
SURVEY §8(c)), so these KATs are what anchors the oracle.
"""
import math

import numpy as np
import pytest


def one_dim(O, b=1.0):
    # test_sdp_core.cpp:14-21 — min 2x s.t. x_11 = b
    return O.OracleInstance.dense(np.array([[2.0]]), [np.array([[1.0]])], [b])


def test_al_value_kat(orc):
    # test_sdp_core.cpp:25-31
    inst = one_dim(orc)
    assert inst.al_value(np.array([[0.5]]), np.zeros(1), 2.0) == pytest.approx(1.0625, rel=1e-14)


def test_al_gradient_kat(orc):
    # test_sdp_core.cpp:68-73
    inst = one_dim(orc)
    g = inst.al_gradient(np.array([[0.5]]), np.zeros(1), 2.0)
    assert g[0, 0] == pytest.approx(0.5, rel=1e-14)


def test_gradient_operator_kat(orc):
    # test_sdp_core.cpp:113-119: G.apply_vec(1) = 0.5 with q = p + beta(A(UU')-b)
    inst = one_dim(orc)
    q = np.zeros(1) + 2.0 * (inst.apply_map(np.array([[0.5]])) - inst.b)
    assert inst.C_plus_adjoint(q, np.ones((1, 1)))[0, 0] == pytest.approx(0.5)


def test_al_value_at_zero_is_penalty(orc):
    # test_sdp_core.cpp:33-41
    rng = np.random.default_rng(7)
    n, m = 5, 3
    Cm = rng.standard_normal((n, n)); Cm = Cm + Cm.T
    As = [(lambda a: a + a.T)(rng.standard_normal((n, n))) for _ in range(m)]
    b = rng.standard_normal(m)
    inst = orc.OracleInstance.dense(Cm, As, b)
    for beta in (0.5, 3.0, 100.0):
        v = inst.al_value(np.zeros((n, 2)), np.zeros(m), beta)
        assert v == pytest.approx(0.5 * beta * b @ b, rel=1e-13)


def test_matcomp_counts(orc):
    # test_instances.cpp:147-151
    assert orc.matcomp_count(3000, 7000, 3) == 828931
    assert orc.matcomp_count(3000, 7000, 5) == 2302586
    assert orc.matcomp_count(30, 70, 2) == 1843


def test_theta_structure(orc):
    # test_instances.cpp:85-111
    c5 = orc.OracleInstance.cycle(5)
    assert (c5.n, c5.m, c5.norm_C1, c5.identity_constraint) == (5, 6, 25.0, 5)
    assert c5.b[5] == 1.0
    pet = orc.OracleInstance.petersen()
    assert (pet.n, pet.m) == (10, 16)
    h10 = orc.OracleInstance.hypercube(10)
    assert (h10.n, h10.m) == (1024, 5121)


def test_stable_set_witness(orc):
    # test_instances.cpp:113-123
    c5 = orc.OracleInstance.cycle(5)
    u = np.zeros((5, 1)); u[0, 0] = u[2, 0] = 1 / math.sqrt(2)
    assert np.linalg.norm(c5.apply_map(u) - c5.b) <= 1e-14
    assert float(np.sum(c5.apply_C(u) * u)) == pytest.approx(-2.0, rel=1e-14)


def _theta_dense(n, edges):
    Cm = -np.ones((n, n))
    As = []
    for i, j in zip(*edges):
        A = np.zeros((n, n)); A[i, j] = A[j, i] = 0.5
        As.append(A)
    As.append(np.eye(n))
    return Cm, As


def test_theta_matches_dense_formulation(orc):
    # test_instances.cpp:125-145
    inst = orc.OracleInstance.cycle(5)
    Cm, As = _theta_dense(5, inst.pairs())
    rng = np.random.default_rng(7)
    for _ in range(20):
        U = rng.standard_normal((5, 2)); p = rng.standard_normal(6)
        X = U @ U.T
        want_map = np.array([np.sum(A * X) for A in As])
        assert np.linalg.norm(inst.apply_map(U) - want_map) <= 1e-12
        S = sum(pk * A for pk, A in zip(p, As))
        assert np.linalg.norm(inst.apply_adjoint(p, U) - S @ U) <= 1e-12
        assert np.linalg.norm(inst.apply_C(U) - Cm @ U) <= 1e-12


@pytest.mark.parametrize("maker", ["cycle", "petersen", "matcomp", "phaseret"])
def test_adjoint_fuzz(orc, maker):
    # test_instances.cpp:27-41 — <A(UU'), p> = <(A*p)U, U>; fused == split
    inst = {"cycle": lambda: orc.OracleInstance.cycle(5),
            "petersen": orc.OracleInstance.petersen,
            "matcomp": lambda: orc.OracleInstance.matcomp(30, 70, 2, seed=5),
            "phaseret": lambda: orc.OracleInstance.phaseret(8, 4, seed=11)}[maker]()
    rng = np.random.default_rng(1001)
    for t in range(30):
        U = rng.standard_normal((inst.n, 1 + t % 3)); p = rng.standard_normal(inst.m)
        lhs = inst.apply_map(U) @ p
        rhs = float(np.sum(inst.apply_adjoint(p, U) * U))
        assert abs(lhs - rhs) <= 1e-10 * (1 + abs(lhs))
        fused = inst.C_plus_adjoint(p, U)
        split = inst.apply_C(U) + inst.apply_adjoint(p, U)
        assert np.linalg.norm(fused - split) <= 1e-12 * (1 + np.linalg.norm(split))


def test_matcomp_instance(orc):
    # test_instances.cpp:153-164
    mc = orc.OracleInstance.matcomp(30, 70, 2, seed=5)
    assert (mc.n, mc.m, mc.norm_C1, mc.identity_constraint) == (100, 1843, 50.0, None)
    i, j = mc.pairs()
    key = i * 70 + j
    assert np.all(np.diff(key) > 0) and i.max() < 30 and j.max() < 70
    again = orc.OracleInstance.matcomp(30, 70, 2, seed=5)
    assert np.array_equal(again.b, mc.b)


def test_phaseret_instance(orc):
    # test_instances.cpp:231-309
    pr = orc.OracleInstance.phaseret(8, 4, seed=11)
    assert (pr.n, pr.m, pr.norm_C1, pr.field_kind) == (16, 32, 16.0, 1)
    x, masks = pr.pr_data()
    assert pr.tau == pytest.approx(1.1 * np.sum(np.abs(x) ** 2))
    b = pr.b
    assert b.min() >= 0
    for l in range(4):  # Parseval per mask
        assert b[l * 8:(l + 1) * 8].sum() == pytest.approx(8 * np.sum(np.abs(masks[:, l] * x) ** 2), rel=1e-9)
    # dense measurement vectors a_(l,k) = conj(w^{jk} d_l(j))
    nc = 8
    jk = np.outer(np.arange(nc), np.arange(nc))
    W = np.exp(-2j * np.pi * jk / nc)
    a = [np.conj(W[:, k] * masks[:, l]) for l in range(4) for k in range(nc)]
    rng = np.random.default_rng(12)
    U = rng.standard_normal((16, 2))
    Uc = U[:8] + 1j * U[8:]
    got = pr.apply_map(U)
    want = np.array([sum(abs(np.vdot(ai, Uc[:, c])) ** 2 for c in range(2)) for ai in a])
    assert np.max(np.abs(got - want) / (1 + want)) <= 1e-9
    p = rng.standard_normal(32)
    gadj = pr.apply_adjoint(p, U)
    wadj = sum(pi * np.outer(ai, ai.conj()) @ Uc for pi, ai in zip(p, a))
    assert np.max(np.abs(gadj[:8] - wadj.real)) <= 1e-9
    assert np.max(np.abs(gadj[8:] - wadj.imag)) <= 1e-9
    xe = np.concatenate([x.real, x.imag])[:, None]
    assert np.linalg.norm(pr.apply_map(xe) - b) <= 1e-9 * np.linalg.norm(b)


def test_unit_impulse_measures_mask_modulus(orc):
    # test_instances.cpp:211-229
    pr = orc.OracleInstance.phaseret(4, 1, seed=0)
    _, masks = pr.pr_data()
    xe = np.zeros((8, 1)); xe[0, 0] = 1.0
    assert np.allclose(pr.apply_map(xe), abs(masks[0, 0]) ** 2)


def test_lanczos_kats(orc):
    # test_lanczos.cpp:18-45
    r = orc.min_eig_dense(np.diag([1.0, -2.0]), tol=1e-10)
    assert r["converged"] and r["lambda_"] == pytest.approx(-2.0, rel=1e-10)
    assert abs(abs(r["v"][1]) - 1) <= 1e-10 and abs(r["v"][0]) <= 1e-8
    r = orc.min_eig_dense(np.array([[0.0, 1.0], [1.0, 0.0]]), tol=1e-10)
    assert r["converged"] and r["lambda_"] == pytest.approx(-1.0, rel=1e-10)
    assert r["v"][0] * r["v"][1] < 0


@pytest.mark.parametrize("seed", [10, 20, 30])
def test_lanczos_vs_dense(orc, seed):
    # test_lanczos.cpp:45-59 (random symmetric n=50)
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((50, 50)); A = 0.5 * (A + A.T)
    r = orc.min_eig_dense(A, tol=1e-10, seed=seed)
    assert r["converged"]
    assert abs(r["lambda_"] - np.linalg.eigvalsh(A)[0]) <= 1e-8
    assert np.linalg.norm(A @ r["v"] - r["lambda_"] * r["v"]) <= 1e-9


def test_lanczos_restarts(orc):
    # test_lanczos.cpp:61-71
    rng = np.random.default_rng(3)
    A = rng.standard_normal((120, 120)); A = 0.5 * (A + A.T)
    r = orc.min_eig_dense(A, tol=1e-9, block_restart=8)
    assert r["converged"] and abs(r["lambda_"] - np.linalg.eigvalsh(A)[0]) <= 1e-7


def test_jacobi_eigh(orc):
    rng = np.random.default_rng(0)
    for k in (1, 2, 5, 16, 30, 31):
        H = rng.standard_normal((k, k)); H = H + H.T
        ev, V = orc.jacobi_eigh(H)
        assert np.allclose(ev, np.linalg.eigvalsh(H), atol=1e-12 * max(1, abs(ev).max()))
        assert np.allclose(H @ V, V * ev, atol=1e-11 * max(1, abs(ev).max()))


def test_solve_tiny_sdp(orc):
    # test_solver.cpp:138-147
    r = one_dim(orc, 0.3).solve(eps=1e-6, seed=1)
    assert r.status == "optimal" and r.pval == pytest.approx(0.6, rel=1e-4) and r.rank == 1


@pytest.mark.parametrize("name,value,tol,rel", [
    ("C5", math.sqrt(5), 1e-4, False), ("petersen", 4.0, 1e-3, False),
    ("Q4", 8.0, 1e-4, True), ("Q6", 32.0, 1e-4, True)])
def test_theta_acceptance_c1(orc, name, value, tol, rel):
    # acceptance.cpp:218-246
    inst = {"C5": lambda: orc.OracleInstance.cycle(5), "petersen": orc.OracleInstance.petersen,
            "Q4": lambda: orc.OracleInstance.hypercube(4),
            "Q6": lambda: orc.OracleInstance.hypercube(6)}[name]()
    r = inst.solve()
    err = abs(-r.pval - value) / (value if rel else 1.0)
    assert r.status == "optimal" and err <= tol
    assert max(r.rel_pfeas, r.rel_gap, r.rel_dfeas) <= 1e-5


def test_theta_h10_acceptance_c2(orc):
    # acceptance.cpp:264-274 — H(10,2): theta = 512, rank 2
    r = orc.OracleInstance.hypercube(10).solve()
    assert r.status == "optimal" and abs(-r.pval - 512) / 512 <= 1e-4 and r.rank == 2


@pytest.mark.parametrize("n1,n2,rk", [(30, 70, 2), (100, 210, 3)])
def test_matcomp_acceptance_c3(orc, n1, n2, rk):
    # acceptance.cpp:276-306 (objective vs nuclear norm; rank = r)
    inst = orc.OracleInstance.matcomp(n1, n2, rk, seed=0)
    r = inst.solve()
    assert r.status == "optimal" and r.rank == rk
    assert abs(r.pval - inst.nuclear_norm) / inst.nuclear_norm <= 1e-3
    # recovery of the sampled entries through tau * U U'
    i, j = inst.pairs()
    Y = r.tau * (r.U[:n1] @ r.U[n1:].T)
    assert np.linalg.norm(Y[i, j] - inst.b) / np.linalg.norm(inst.b) <= 1e-3


def test_phaseret_acceptance_c4(orc):
    # acceptance.cpp:308-330 — PR n=64, L=12: overlap >= 0.99, rank <= 3
    inst = orc.OracleInstance.phaseret(64, 12, seed=7)
    r = inst.solve()
    assert r.status == "optimal" and r.rank <= 3
    x, _ = inst.pr_data()
    Uc = r.U[:64] + 1j * r.U[64:]
    w, V = np.linalg.eigh(Uc @ Uc.conj().T)
    xh = V[:, -1]
    ov = abs(np.vdot(xh, x)) ** 2 / (np.vdot(xh, xh).real * np.vdot(x, x).real)
    assert ov >= 0.99


def test_solve_deterministic_and_warm_start(orc):
    # test_solver.cpp:177-199
    inst = orc.OracleInstance.petersen()
    a = inst.solve(eps=1e-4, seed=42)
    b = inst.solve(eps=1e-4, seed=42)
    assert a.pval == b.pval and np.array_equal(a.U, b.U) and np.array_equal(a.p, b.p)
    c5 = orc.OracleInstance.cycle(5)
    r = c5.solve()
    again = c5.solve(U0=r.U, p0=r.p)
    assert again.status == "optimal" and again.outer_iters == 1


def test_thread_count_invariance(orc):
    # test_instances.cpp:358-382 — bitwise identical across worker counts
    inst = orc.OracleInstance.hypercube(8)
    pr = orc.OracleInstance.phaseret(64, 8, seed=4)
    rng = np.random.default_rng(5)
    U = rng.standard_normal((inst.n, 4)); p = rng.standard_normal(inst.m)
    Up = rng.standard_normal((pr.n, 4)); pp = rng.standard_normal(pr.m)
    orc.lib().orc_set_threads(1)
    a = (inst.apply_map(U), inst.apply_adjoint(p, U), pr.apply_map(Up), pr.apply_adjoint(pp, Up))
    orc.lib().orc_set_threads(4)
    b = (inst.apply_map(U), inst.apply_adjoint(p, U), pr.apply_map(Up), pr.apply_adjoint(pp, Up))
    orc.lib().orc_set_threads(0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_matcomp_paper_sampling_rule(orc):
    # SURVEY §0 item 2 / §8(f) row 2 (not in the reference; parity unpinned against it):
    # draws_per_dim * (n1 + n2) draws with replacement, deduplicated and sorted
    n1, n2, d = 300, 700, 40
    inst = orc.OracleInstance.matcomp_paper(n1, n2, 3, seed=1, draws_per_dim=d)
    i, j = inst.pairs()
    draws, N = d * (n1 + n2), n1 * n2
    assert inst.m == len(i) <= draws
    keys = i * n2 + j
    assert np.all(np.diff(keys) > 0)  # sorted, distinct
    expect = N * (1.0 - (1.0 - 1.0 / N) ** draws)  # expected distinct count
    assert abs(inst.m - expect) <= 6 * np.sqrt(expect * np.exp(-draws / N))
    # the paper's 3.2M x 4.8M row: 319,996,871 reported vs this expectation
    N8, D8 = 3_200_000 * 4_800_000, 40 * 8_000_000
    assert abs(N8 * (1.0 - np.exp(-D8 / N8)) - 319_996_871) / 319_996_871 < 1e-5
    # a recoverable small instance solves to ||M||_*
    small = orc.OracleInstance.matcomp_paper(30, 70, 2, seed=5, draws_per_dim=12)
    r = small.solve()
    assert r.status == "optimal"
    assert abs(r.pval - small.nuclear_norm) / small.nuclear_norm <= 1e-3
