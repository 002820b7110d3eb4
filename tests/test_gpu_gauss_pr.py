"""Gaussian-measurement phase retrieval (BASELINE configs[2];
NOT in the reference -- parity is against the dense oracle
oracle/src/families.cpp gauss_pr_instance on the device's own measurement
vectors, the test_instances.cpp:255-297 pattern, and is unpinned against the
reference).  The device map / adjoint are FP64 tensor-core (DMMA) GEMMs, so they
agree with the sequential oracle to rounding (1e-12 relative), not bit for bit."""
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


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(1.0, float(np.max(np.abs(b)))))


@pytest.mark.parametrize("n,m", [(8, 96), (37, 300), (64, 768)])
def test_instance_and_operators_vs_dense_oracle(H, orc, n, m):
    inst = H.gen_gauss_phase_retrieval(H.GaussPrSpec(n, m, seed=3))
    A, x = inst.gauss_data()
    assert A.shape == (m, n) and inst.n == 2 * n and inst.m == m
    # entries are CN(0, 1): mean |a|^2 close to 1
    assert abs(np.mean(np.abs(A) ** 2) - 1.0) < 0.15
    ref = orc.OracleInstance.gauss_pr(A, x, tau_slack=1.1)
    assert rel(inst.b, ref.b) <= 1e-12
    assert inst.tau == pytest.approx(ref.tau, rel=1e-13)
    rng = np.random.default_rng(n)
    for s in (1, 2, 3, 5):
        U = rng.standard_normal((2 * n, s))
        p = rng.standard_normal(m)
        assert rel(inst.apply_map(U), ref.apply_map(U)) <= 1e-12
        assert rel(inst.apply_adjoint(p, U), ref.apply_adjoint(p, U)) <= 1e-12
        assert rel(inst.C_plus_adjoint(p, U), ref.C_plus_adjoint(p, U)) <= 1e-12
        # adjoint identity <A(UU'), p> = <(A* p) U, U>
        lhs = float(inst.apply_map(U) @ p)
        rhs = float(np.sum(inst.apply_adjoint(p, U) * U))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))
        assert rel(inst.al_gradient(U, p, 2.0), ref.al_gradient(U, p, 2.0)) <= 1e-10


def test_solve_recovers_signal(H, orc):
    n, m = 32, 384
    inst = H.gen_gauss_phase_retrieval(H.GaussPrSpec(n, m, seed=1))
    A, x = inst.gauss_data()
    r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0))
    assert r.status == "optimal", r
    u = r.U[:n, 0] + 1j * r.U[n:, 0]
    overlap = abs(np.vdot(u, x)) / np.linalg.norm(u) / np.linalg.norm(x)
    assert overlap >= 0.99
    o = orc.OracleInstance.gauss_pr(A, x).solve(eps=1e-5, seed=0)
    assert o.status == "optimal"
    assert abs(r.pval - o.pval) <= 1e-6 * max(1.0, abs(o.pval))
