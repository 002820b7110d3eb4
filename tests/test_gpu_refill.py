"""Lanczos breakdown refills without a cap (lanczos.cpp:127-130): with no
pre-drawn refill vectors (CUHALLAR_LZ_PREDRAW=0) every refill is served by
the launch's host service thread (capi.cu RefillService, solver.cuh
lz_refill); solves must be bit-identical to the pre-drawn path and, in parity
mode, keep the oracle's counters.  Tiny graphs break the Krylov basis down on
every Lanczos call (n < block_restart)."""
import os

import pytest

pytestmark = pytest.mark.gpu

KEYS = ["status", "outer_iters", "fw_steps", "aipp_iters", "fista_iters", "eig_products", "rank"]


@pytest.fixture(scope="module")
def H():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2505_13719_b200 as H
    return H


def _graph(H, name):
    if name == "C5":
        return H.make_cycle(5)
    if name == "petersen":
        return H.make_petersen()
    return H.make_hypercube(int(name[1:]))


@pytest.mark.parametrize("name", ["C5", "petersen", "H4", "H6"])
@pytest.mark.parametrize("parity", [False, True])
def test_refills_from_host_service_bit_identical(H, name, parity):
    cfg = H.SolverConfig(eps=1e-5, seed=0, parity=parity)
    ref = H.solve(H.build_theta_instance(_graph(H, name)), cfg)
    os.environ["CUHALLAR_LZ_PREDRAW"] = "0"
    try:
        got = H.solve(H.build_theta_instance(_graph(H, name)), cfg)
    finally:
        del os.environ["CUHALLAR_LZ_PREDRAW"]
    assert {k: getattr(got, k) for k in KEYS} == {k: getattr(ref, k) for k in KEYS}
    assert got.pval == ref.pval


def test_refills_parity_counters_equal_oracle(H, orc):
    os.environ["CUHALLAR_LZ_PREDRAW"] = "0"
    try:
        got = H.solve(H.build_theta_instance(H.make_cycle(5)), H.SolverConfig(eps=1e-5, seed=0, parity=True))
    finally:
        del os.environ["CUHALLAR_LZ_PREDRAW"]
    o = orc.OracleInstance.cycle(5).solve(eps=1e-5, seed=0)
    assert {k: getattr(got, k) for k in KEYS} == {k: getattr(o, k) for k in KEYS}
    assert got.pval == o.pval
