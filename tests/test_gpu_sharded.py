"""Row-sharded solve on one B200: `world` co-resident persistent
launches on the same device play the ranks, each with its own instance copy
and factor arena, exchanging rows and partial sums through the same
peer-pointer protocol the multi-GPU solve uses over NVLink.  The sharded
solve must reach the reference's answers (KATs, oracle objective within 1e-6)
and be bitwise deterministic for a fixed world size; world = 1 must be the
plain solve bit for bit."""
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


def _make(H, name):
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5))
    if name == "petersen":
        return H.build_theta_instance(H.make_petersen())
    if name.startswith("H"):
        return H.build_theta_instance(H.make_hypercube(int(name[1:])))
    if name == "mc100":
        return H.gen_matrix_completion(H.McSpec(100, 210, 3, seed=0))
    if name == "mc2000":
        return H.gen_matrix_completion(H.McSpec(2000, 2000, 3, seed=0))
    raise KeyError(name)


def _oracle(orc, name):
    if name == "C5":
        return orc.OracleInstance.cycle(5)
    if name == "petersen":
        return orc.OracleInstance.petersen()
    if name.startswith("H"):
        return orc.OracleInstance.hypercube(int(name[1:]))
    if name == "mc100":
        return orc.OracleInstance.matcomp(100, 210, 3, seed=0)
    if name == "mc2000":
        return orc.OracleInstance.matcomp(2000, 2000, 3, seed=0)
    raise KeyError(name)


def test_world1_is_the_plain_solve(H):
    a = H.solve(_make(H, "H6"))
    b = H.solve_sharded([_make(H, "H6")])
    assert a.pval == b.pval and a.fista_iters == b.fista_iters and np.array_equal(a.U, b.U)
    assert np.array_equal(a.p, b.p)


@pytest.mark.parametrize("name,value,relative", [
    ("C5", math.sqrt(5), False), ("petersen", 4.0, False), ("H6", 32.0, True), ("H10", 512.0, True)])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_theta(H, orc, name, value, relative, world):
    insts = [_make(H, name) for _ in range(world)]
    rep = H.solve_sharded(insts)
    single = H.solve(_make(H, name))
    assert rep.status == "optimal"
    err = abs(-rep.pval - value) / (value if relative else 1.0)
    assert err <= 1e-4
    assert abs(rep.pval - single.pval) <= 1e-6 * max(1.0, abs(single.pval))
    # against the CPU oracle's own solve of the same instance (final objective <= 1e-6)
    o = _oracle(orc, name).solve()
    assert o.status == "optimal"
    assert abs(rep.pval - o.pval) <= 1e-6 * max(1.0, abs(o.pval))
    assert max(rep.rel_pfeas, rep.rel_gap, rep.rel_dfeas) <= 1e-5
    assert rep.U.shape == (insts[0].n, rep.rank) and rep.p.shape == (insts[0].m,)
    # the returned (U, p) is a certified point: warm start finishes in one outer iteration
    again = H.solve(_make(H, name), U0=rep.U, p0=rep.p)
    assert again.status == "optimal" and again.outer_iters == 1


@pytest.mark.parametrize("name", ["mc100", "mc2000"])
def test_sharded_matcomp(H, orc, name):
    insts = [_make(H, name) for _ in range(2)]
    rep = H.solve_sharded(insts)
    single = H.solve(_make(H, name))
    assert rep.status == "optimal" and rep.rank == single.rank
    assert abs(rep.pval - single.pval) <= 1e-6 * abs(single.pval)
    assert abs(rep.pval - insts[0].nuclear_norm) / insts[0].nuclear_norm <= 1e-3
    o = _oracle(orc, name).solve()
    assert o.status == "optimal" and o.rank == rep.rank
    assert abs(rep.pval - o.pval) <= 1e-6 * abs(o.pval)


def test_sharded_deterministic(H):
    r1 = H.solve_sharded([_make(H, "petersen") for _ in range(2)], H.SolverConfig(seed=3))
    r2 = H.solve_sharded([_make(H, "petersen") for _ in range(2)], H.SolverConfig(seed=3))
    assert r1.pval == r2.pval and r1.fista_iters == r2.fista_iters
    assert np.array_equal(r1.U, r2.U) and np.array_equal(r1.p, r2.p)


def test_sharded_rejects_phase_retrieval(H):
    insts = [H.gen_phase_retrieval(H.PrSpec(8, 4, seed=1)) for _ in range(2)]
    with pytest.raises(H.InputError):
        H.solve_sharded(insts)


def test_solve_rank_world1_matches_plain_solve(H):
    """The one-process-per-GPU entry points (cuhallar_shard_export /
    cuhallar_solve_rank, used by bench.py under torchrun) at world 1: the IPC
    handle round trip and the rank launch reproduce the plain solve."""
    inst = H.build_theta_instance(H.make_hypercube(6))
    cfg = H.SolverConfig(eps=1e-5, seed=0)
    ref = H.solve(inst, cfg)
    hb = H.shard_export(inst)
    assert isinstance(hb, bytes) and len(hb) == 512
    r = H.solve_rank(inst, 1, 0, [hb], cfg, fetch=True)
    assert r.status == ref.status == "optimal"
    assert abs(r.pval - ref.pval) <= 1e-6 * max(1.0, abs(ref.pval))
    assert r.rank == ref.rank
    with pytest.raises(H.InputError):
        H.solve_rank(inst, 2, 0, [hb], cfg)  # a peer blob is missing
