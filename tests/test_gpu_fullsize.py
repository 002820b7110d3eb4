"""GPU parity at BASELINE.json's full sizes through size-independent
properties (the oracle cannot run these in seconds):

* H(23,2) (n = 8,388,608, m = 96,468,993) and MC(400k x 600k, r = 3)
  (m = 124,339,596): the constraint map A(UU') is bit-identical to a NumPy
  evaluation of the reference formula out_k = sum_c U(i_k,c) U(j_k,c) in
  column order (instances.cpp:27-35), including the trace constraint;
* the adjoint identity <A(UU'), p> = <(A*p)U, U> to 1e-10 relative
  (test_instances.cpp:27-41 at scale);
* fused == split: C_plus_adjoint(q, U) == apply_C(U) + apply_adjoint(q, U) to
  1e-12 (the fused form accumulates onto C U, as the reference does);
* al_gradient (q formed on the fly) == 2 C_plus_adjoint(p + beta (A(UU') - b), U)
  bit for bit;
* the instance itself: edge set of H(23,2) equals make_hypercube's
  (v, v ^ 2^bit) rule; MC sample count equals matcomp_constraint_count.
Both instances take several GB of HBM and tens of seconds to build."""
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


def _map_ref(U, i, j):
    d = U[i, 0] * U[j, 0]
    for c in range(1, U.shape[1]):
        d = d + U[i, c] * U[j, c]
    return d


def _check_operator_properties(inst, U, i, j, trace, rng):
    out = inst.apply_map(U)
    npairs = len(i)
    assert np.array_equal(out[:npairs], _map_ref(U, i, j))
    if trace:
        assert out[-1] == pytest.approx(float(np.sum(U * U)), rel=1e-12)
    p = rng.standard_normal(inst.m)
    adj = inst.apply_adjoint(p, U)
    lhs = float(out @ p)
    rhs = float(np.sum(adj * U))
    assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))
    # al_gradient forms q = p + beta (A(UU') - b) on the fly (row pass with
    # per-entry dots); the same q through the map and C_plus_adjoint must give
    # the bit-identical gradient 2 (C + A*(q))U (sdp_instance.cpp:62-71)
    beta = 3.0
    q = p + beta * (out - inst.b)
    grad = inst.al_gradient(U, p, beta)
    assert np.array_equal(grad, 2.0 * inst.C_plus_adjoint(q, U))
    fused = inst.C_plus_adjoint(p, U)
    split = inst.apply_C(U) + adj
    # the fused form accumulates onto C U (the reference's apply_C_plus_adjoint
    # order), the split form adds C U last: equal to rounding (1e-12, as
    # test_instances.cpp:27-41)
    assert np.max(np.abs(fused - split)) <= 1e-12 * max(1.0, float(np.max(np.abs(split))))


def test_hamming_23_full_size(H):
    inst = H.build_theta_instance(H.make_hypercube(23))
    n = 1 << 23
    assert (inst.n, inst.m) == (n, 96468993)
    i, j = inst.pairs()
    # make_hypercube (graph.cpp:135-148): edges (v, v ^ 2^bit), v < u, sorted
    assert np.all(i < j) and np.all(np.diff(i) >= 0)
    x = i ^ j
    assert np.all((x & (x - 1)) == 0)
    assert np.array_equal(np.bincount(i, minlength=n) + np.bincount(j, minlength=n), np.full(n, 23))
    rng = np.random.default_rng(23)
    U = rng.standard_normal((n, 2)) / np.sqrt(n)
    _check_operator_properties(inst, U, i, j, True, rng)


def test_matcomp_c4_full_size(H):
    spec = H.McSpec(400000, 600000, 3, seed=0)
    inst = H.gen_matrix_completion(spec)
    assert inst.m == H.matcomp_constraint_count(400000, 600000, 3) == 124339596
    i, j = inst.pairs()
    assert np.all(np.diff(i) >= 0) and np.all((np.diff(i) > 0) | (np.diff(j) > 0))  # sorted, distinct
    rng = np.random.default_rng(4)
    U = rng.standard_normal((inst.n, 3)) / np.sqrt(inst.n)
    _check_operator_properties(inst, U, i, j + 400000, False, rng)


def test_matcomp_c4_al_value_row_ordered_map(H):
    """al_value at C4 runs the row-ordered SELL map pass (one gathered row per
    constraint, device.cuh map_pass_sell): r_k is bit-identical to the edge-order
    map, only the partial sums p.r and r.r are formed in another order, so the
    value matches the reference formula (sdp_instance.cpp:50-60) to 1e-12."""
    spec = H.McSpec(400000, 600000, 3, seed=0)
    inst = H.gen_matrix_completion(spec)
    rng = np.random.default_rng(5)
    U = rng.standard_normal((inst.n, 3)) / np.sqrt(inst.n)
    p = rng.standard_normal(inst.m)
    beta = 7.0
    r = inst.apply_map(U) - inst.b
    ref = 0.5 * float(np.sum(U * U)) + float(p @ r) + 0.5 * beta * float(r @ r)
    val = inst.al_value(U, p, beta)
    assert val == pytest.approx(ref, rel=1e-12)


def test_matcomp_solve_row_ordered_map_vs_edge_order(H, monkeypatch):
    """The fast solve with the row-ordered map (default) and with the edge-order
    map (CUHALLAR_NO_SELL_MAP=1, read at instance build) reach the same optimum:
    status, rank and pval within 1e-6 (the two differ only in the order of the
    map's partial sums)."""
    spec = H.McSpec(100000, 150000, 3, seed=0)
    inst = H.gen_matrix_completion(spec)
    rep = H.solve(inst, H.SolverConfig(eps=1e-5))
    monkeypatch.setenv("CUHALLAR_NO_SELL_MAP", "1")
    inst2 = H.gen_matrix_completion(spec)
    rep2 = H.solve(inst2, H.SolverConfig(eps=1e-5))
    assert rep.status == rep2.status == "optimal"
    assert rep.rank == rep2.rank == 3
    assert abs(rep.pval - rep2.pval) <= 1e-6 * abs(rep2.pval)


@pytest.mark.parametrize("d", [18, 23])
def test_hamming_al_value_row_ordered_map(H, d, monkeypatch):
    """Theta on a hypercube (uniform degree, no SELL padding) runs the
    row-ordered SELL map too (upper entries of every slice, the lower prefix
    skipped): al_value equals the reference formula cdot + p.r + beta/2 |r|^2
    (sdp_instance.cpp:50-60) to 1e-12 and the edge-order map's value
    (CUHALLAR_NO_SELL_MAP=1) to 1e-12."""
    inst = H.build_theta_instance(H.make_hypercube(d))
    rng = np.random.default_rng(d)
    U = rng.standard_normal((inst.n, 2)) / np.sqrt(inst.n)
    p = rng.standard_normal(inst.m)
    beta = 5.0
    r = inst.apply_map(U) - inst.b
    ref = float(np.sum(inst.apply_C(U) * U)) + float(p @ r) + 0.5 * beta * float(r @ r)
    val = inst.al_value(U, p, beta)
    assert val == pytest.approx(ref, rel=1e-12)
    del inst
    monkeypatch.setenv("CUHALLAR_NO_SELL_MAP", "1")
    inst2 = H.build_theta_instance(H.make_hypercube(d))
    assert inst2.al_value(U, p, beta) == pytest.approx(val, rel=1e-12)


def test_circulant_theta_al_value_row_ordered_map(H, monkeypatch):
    """A uniform-degree graph that is not a hypercube (circulant, offsets
    1, 5, 77, 1000, 54321: degree 10, lower-entry counts that vary across each
    SELL slice near the wrap-around) takes the row-ordered theta map with the
    lower-prefix skip: al_value equals the reference formula and the
    edge-order map's value to 1e-12."""
    n = 1 << 18
    u = np.arange(n, dtype=np.int64)
    e = []
    for off in (1, 5, 77, 1000, 54321):
        v = (u + off) % n
        e.append(np.stack([np.minimum(u, v), np.maximum(u, v)], axis=1))
    edges = np.unique(np.concatenate(e), axis=0)
    g = H.graph_from_edges(n, edges)
    inst = H.build_theta_instance(g)
    assert inst.m == len(edges) + 1
    rng = np.random.default_rng(11)
    U = rng.standard_normal((n, 2)) / np.sqrt(n)
    p = rng.standard_normal(inst.m)
    beta = 3.0
    r = inst.apply_map(U) - inst.b
    ref = float(np.sum(inst.apply_C(U) * U)) + float(p @ r) + 0.5 * beta * float(r @ r)
    val = inst.al_value(U, p, beta)
    assert val == pytest.approx(ref, rel=1e-12)
    del inst
    monkeypatch.setenv("CUHALLAR_NO_SELL_MAP", "1")
    inst2 = H.build_theta_instance(H.graph_from_edges(n, edges))
    assert inst2.al_value(U, p, beta) == pytest.approx(val, rel=1e-12)
