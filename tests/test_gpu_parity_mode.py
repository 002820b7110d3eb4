"""Parity mode (SolverConfig.parity, csrc/parity.cuh): every reduction in the
reference binary's order (Eigen's LinearVectorized redux, ordered CGS2 dots),
so the device takes the oracle's decisions.  Asserted against the CPU oracle
(oracle/src/algo.cpp, a restatement of solver.cpp / hlr.cpp / adap_aipp.cpp /
adap_fista.cpp / lanczos.cpp): status, rank and all five counters
(outer_iters, fw_steps, aipp_iters, fista_iters, eig_products, SolveReport
solver.hpp:40-61) identical, and pval bit-identical -- on the theta KAT graphs,
the BASELINE configs C1 (MC 2000 x 2000, r = 3) and C2 (H(12,2)), and the
H(13,2) / H(14,2) instances on which the reference algorithm itself ends in
numerical_failure ("fista: curvature estimate diverged", adap_fista.cpp:63-65).
The fast mode is checked too: on matrix completion its counters equal the
oracle's; on hypercubes its trajectory is allowed to differ (both optimal,
objective within 1e-6)."""
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


def _pair(H, O, name):
    if name == "C5":
        return H.build_theta_instance(H.make_cycle(5)), O.OracleInstance.cycle(5)
    if name == "petersen":
        return H.build_theta_instance(H.make_petersen()), O.OracleInstance.petersen()
    if name.startswith("H"):
        d = int(name[1:])
        return H.build_theta_instance(H.make_hypercube(d)), O.OracleInstance.hypercube(d)
    n1, n2, r, seed = {"mc30": (30, 70, 2, 5), "mc100": (100, 210, 3, 0),
                       "mc2000": (2000, 2000, 3, 0)}[name]
    return (H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=seed)),
            O.OracleInstance.matcomp(n1, n2, r, seed=seed))


_ORACLE = {}


def _oracle_solve(O, name, ref):
    if name not in _ORACLE:
        _ORACLE[name] = ref.solve(eps=1e-5, seed=0)
    return _ORACLE[name]


@pytest.mark.parametrize("name", ["C5", "petersen", "H4", "H6", "H8", "H10", "mc30", "mc100",
                                  "mc2000", "H12", "H13", "H14"])
def test_parity_mode_counters_equal_oracle(H, orc, name):
    inst, ref = _pair(H, orc, name)
    o = _oracle_solve(orc, name, ref)
    r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True))
    got = {k: getattr(r, k) for k in KEYS}
    want = {k: getattr(o, k) for k in KEYS}
    assert got == want
    assert r.pval == o.pval  # bit-identical objective
    if name in ("H13", "H14"):
        # the reference algorithm's own outcome on these inputs
        assert r.status == "numerical_failure"


@pytest.mark.parametrize("name", ["mc30", "mc100", "mc2000"])
def test_fast_mode_matcomp_counters_equal_oracle(H, orc, name):
    inst, ref = _pair(H, orc, name)
    o = _oracle_solve(orc, name, ref)
    r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0))
    assert {k: getattr(r, k) for k in KEYS} == {k: getattr(o, k) for k in KEYS}
    assert abs(r.pval - o.pval) <= 1e-6 * max(1.0, abs(o.pval))


@pytest.mark.parametrize("name", ["H10", "H12"])
def test_fast_mode_theta_objective(H, orc, name):
    inst, ref = _pair(H, orc, name)
    o = _oracle_solve(orc, name, ref)
    r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0))
    assert r.status == o.status == "optimal"
    assert abs(r.pval - o.pval) <= 1e-6 * max(1.0, abs(o.pval))


def test_parity_mode_trace_matches_oracle(H, orc):
    """Trace events (trace.hpp:12-26: per HLR step and per outer iteration)
    equal the oracle's, every field bit for bit."""
    kinds = {0: "inner_stationary", 1: "inner_rank_step", 2: "outer"}
    fields = ["outer_iter", "beta", "eps_inner", "gap", "theta", "rank", "al_value", "fw_alpha",
              "rel_pfeas", "rel_gap", "rel_dfeas"]
    for name in ("H8", "mc100"):
        inst, ref = _pair(H, orc, name)
        events = []
        H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True), sink=events.append)
        o = ref.solve(eps=1e-5, seed=0, trace=True)
        dev = [(e.kind,) + tuple(getattr(e, f) for f in fields) for e in events if e.kind in kinds.values()]
        want = [(kinds[e["kind"]],) + tuple(e[f] for f in fields) for e in o.trace]
        assert len(dev) == len(want) > 0
        assert dev == want
