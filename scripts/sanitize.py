"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck):
theta, matrix completion and phase retrieval operators + solves, and a world-2
sharded solve.  `compute-sanitizer --tool memcheck python scripts/sanitize.py`"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2505_13719_b200 as H


def ops(inst, s=2):
    rng = np.random.default_rng(0)
    U = rng.standard_normal((inst.n, s)) / np.sqrt(inst.n)
    p = rng.standard_normal(inst.m)
    inst.apply_map(U)
    inst.C_plus_adjoint(p, U)
    inst.al_value_and_gradient(U, p, 2.0)


for inst in (H.build_theta_instance(H.make_cycle(5)), H.build_theta_instance(H.make_hypercube(6)),
             H.gen_matrix_completion(H.McSpec(30, 70, 2, seed=5)),
             H.gen_phase_retrieval(H.PrSpec(16, 4, seed=1))):
    ops(inst)
    r = H.solve(inst, H.SolverConfig(time_limit=120))
    print(inst.kind, r.status, r.pval, flush=True)
r = H.solve_sharded([H.build_theta_instance(H.make_petersen()) for _ in range(2)])
print("sharded", r.status, r.pval, flush=True)
