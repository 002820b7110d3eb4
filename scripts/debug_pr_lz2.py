import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_13719_b200 as H
from oracle import oracle as O
n, L, seed = 8, 4, 11
inst = H.gen_phase_retrieval(H.PrSpec(n, L, seed=seed)); ref = O.OracleInstance.phaseret(n, L, seed=seed)
rng = np.random.default_rng(4)
U = rng.standard_normal((inst.n, 2)); U /= np.linalg.norm(U)
p = 0.05 * rng.standard_normal(inst.m)
q = p + 2.0 * (ref.apply_map(U) - ref.b)
G = np.stack([inst.C_plus_adjoint(q, e[:, None])[:, 0] for e in np.eye(inst.n)], 1)
Gr = np.stack([ref.C_plus_adjoint(q, e[:, None])[:, 0] for e in np.eye(inst.n)], 1)
print("dense G diff", np.max(np.abs(G - Gr)), "sym", np.max(np.abs(G - G.T)), "eig", np.linalg.eigvalsh(0.5 * (G + G.T))[:3])
for br, mi in ((2, 2), (2, 3), (3, 3), (4, 4), (4, 5), (8, 8), (8, 9), (16, 16), (16, 17), (16, 40)):
    got = inst.min_eig_gradient(U, p, 2.0, tol=1e-9, max_iters=mi, block_restart=br, seed=0)
    want = ref.min_eig_G(U, p, 2.0, tol=1e-9, max_iters=mi, block_restart=br, seed=0)
    print(br, mi, got["lambda_"], got["residual"], want["residual"], np.max(np.abs(np.abs(got["v"]) - np.abs(want["v"]))), got["matvecs"], got["converged"], "|", want["lambda_"], want["matvecs"], want["converged"])
# gradop check via al_gradient: grad = 2 (C + A*(p + beta r)) U
g = inst.al_gradient(U, p, 2.0); gr = ref.al_gradient(U, p, 2.0)
print("al_gradient diff", np.max(np.abs(g - gr)))
