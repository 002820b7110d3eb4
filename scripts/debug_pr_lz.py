import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_13719_b200 as H
from oracle import oracle as O
for (n, L, seed) in [(64, 12, 7), (512, 3, 2), (8, 4, 11)]:
    inst = H.gen_phase_retrieval(H.PrSpec(n, L, seed=seed)); ref = O.OracleInstance.phaseret(n, L, seed=seed)
    rng = np.random.default_rng(4)
    U = rng.standard_normal((inst.n, 2)); U /= np.linalg.norm(U)
    p = 0.05 * rng.standard_normal(inst.m)
    for tol in (1e-9, 1e-6):
        got = inst.min_eig_gradient(U, p, 2.0, tol=tol, seed=0)
        want = ref.min_eig_G(U, p, 2.0, tol=tol, seed=0)
        print(n, L, tol, {k: v for k, v in got.items() if k != "v"}, {k: v for k, v in want.items() if k != "v"}, flush=True)
    # one matvec check: G v via C_plus_adjoint with q = p + beta(A(UU')-b)
    q = p + 2.0 * (ref.apply_map(U) - ref.b)
    v = rng.standard_normal(inst.n)
    print("cpa", np.max(np.abs(inst.C_plus_adjoint(q, v[:, None]) - ref.C_plus_adjoint(q, v[:, None]))), flush=True)
