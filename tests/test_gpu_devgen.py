"""Device instance generation (csrc/devgen.cu) against the
sequential host generator (CUHALLAR_HOST_GEN=1) and the CPU oracle: identical
constraint index sets, right-hand sides and norms -- bit for bit -- for the
reference's rejection-sampling rule (instances.cpp:138-175, the first m
distinct draws), the paper's draws-with-replacement rule and make_hypercube
(graph.cpp:135-148).  Also the host-buffer instance entry point
cuhallar_matcomp_from_samples (validation, and operators equal to the
generated instance's)."""
import os

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


def _host(fn):
    os.environ["CUHALLAR_HOST_GEN"] = "1"
    try:
        return fn()
    finally:
        del os.environ["CUHALLAR_HOST_GEN"]


def _same(a, b):
    ia, ja = a.pairs()
    ib, jb = b.pairs()
    assert (a.n, a.m) == (b.n, b.m)
    assert np.array_equal(ia, ib) and np.array_equal(ja, jb)
    assert np.array_equal(a.b, b.b)
    assert a.tau == b.tau and a.norm_b1 == b.norm_b1 and a.norm_C1 == b.norm_C1


MC = [(30, 70, 2, 5), (100, 210, 3, 0), (300, 700, 3, 1), (2000, 2000, 3, 0), (3000, 7000, 3, 0)]


@pytest.mark.parametrize("n1,n2,r,seed", MC)
def test_matcomp_device_equals_host(H, n1, n2, r, seed):
    spec = H.McSpec(n1, n2, r, seed=seed)
    dev = H.gen_matrix_completion(spec)
    host = _host(lambda: H.gen_matrix_completion(spec))
    _same(dev, host)
    assert dev.m == H.matcomp_constraint_count(n1, n2, r)


@pytest.mark.parametrize("n1,n2,r,seed", MC[:4])
def test_matcomp_device_equals_oracle(H, orc, n1, n2, r, seed):
    dev = H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=seed))
    ref = orc.OracleInstance.matcomp(n1, n2, r, seed=seed)
    i, j = dev.pairs()
    ri, rj = ref.pairs()
    assert np.array_equal(i, ri) and np.array_equal(j, rj)
    assert np.array_equal(dev.b, ref.b)
    assert dev.tau == pytest.approx(ref.tau, rel=1e-13)
    assert dev.norm_b1 == ref.norm_b1


def test_matcomp_known_counts(H):
    # test_instances.cpp:147-151 / acceptance.cpp:508-527: m for (3000, 7000, r = 3 / 5)
    assert H.gen_matrix_completion(H.McSpec(3000, 7000, 5, seed=0)).m == 2302586


@pytest.mark.parametrize("n1,n2,r,dpd", [(100, 210, 3, 5), (2000, 4000, 3, 40)])
def test_matcomp_paper_rule_device_equals_host(H, orc, n1, n2, r, dpd):
    spec = H.McSpec(n1, n2, r, seed=0, draws_per_dim=dpd)
    dev = H.gen_matrix_completion(spec)
    host = _host(lambda: H.gen_matrix_completion(spec))
    _same(dev, host)
    ref = orc.OracleInstance.matcomp_paper(n1, n2, r, seed=0, draws_per_dim=dpd)
    i, j = dev.pairs()
    ri, rj = ref.pairs()
    assert np.array_equal(i, ri) and np.array_equal(j, rj) and np.array_equal(dev.b, ref.b)


@pytest.mark.parametrize("d", [1, 2, 3, 6, 10, 12, 16])
def test_hypercube_device_equals_host(H, d):
    dev = H.build_theta_instance(H.make_hypercube(d))
    host = _host(lambda: H.build_theta_instance(H.make_hypercube(d)))
    _same(dev, host)


def test_hypercube_device_equals_oracle(H, orc):
    dev = H.build_theta_instance(H.make_hypercube(10))
    ref = orc.OracleInstance.hypercube(10)
    i, j = dev.pairs()
    ri, rj = ref.pairs()
    assert np.array_equal(i, ri) and np.array_equal(j, rj)
    assert np.array_equal(dev.b, ref.b)


def test_matcomp_from_samples_matches_generated(H):
    inst = H.gen_matrix_completion(H.McSpec(300, 700, 3, seed=1))
    i, j = inst.pairs()
    b = inst.b
    inst2 = H.matcomp_from_samples(300, 700, i, j, b, inst.tau)
    _same(inst, inst2)
    rng = np.random.default_rng(3)
    U = rng.standard_normal((inst.n, 3))
    p = rng.standard_normal(inst.m)
    assert np.array_equal(inst.apply_map(U), inst2.apply_map(U))
    assert np.array_equal(inst.C_plus_adjoint(p, U), inst2.C_plus_adjoint(p, U))
    r1 = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0))
    r2 = H.solve(inst2, H.SolverConfig(eps=1e-5, seed=0))
    assert r1.pval == r2.pval and r1.fista_iters == r2.fista_iters


def test_matcomp_from_samples_rejects_bad_input(H):
    i = np.array([0, 0, 1]); j = np.array([0, 2, 1]); b = np.ones(3)
    H.matcomp_from_samples(2, 3, i, j, b, 1.0)  # valid
    with pytest.raises(H.InputError):
        H.matcomp_from_samples(2, 3, np.array([0, 0, 1]), np.array([2, 0, 1]), b, 1.0)  # unsorted
    with pytest.raises(H.InputError):
        H.matcomp_from_samples(2, 3, np.array([0, 0, 2]), np.array([0, 2, 1]), b, 1.0)  # i out of range
    with pytest.raises(H.InputError):
        H.matcomp_from_samples(2, 3, np.array([0, 0, 1]), np.array([0, 0, 1]), b, 1.0)  # duplicate
    with pytest.raises(H.InputError):
        H.matcomp_from_samples(2, 3, i, j, b, 0.0)  # tau
