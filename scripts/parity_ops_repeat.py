"""Bitwise run-to-run determinism of the parity-mode sub-solvers at one size."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

name = sys.argv[1]
inst, ref = pair(name)
rng = np.random.default_rng(1)
for s in (2, 3):
    U = rng.standard_normal((inst.n, s))
    U /= np.linalg.norm(U)
    p = rng.standard_normal(inst.m) * 0.1
    outs = []
    for k in range(6):
        r = inst.min_eig_gradient(U, p, 10.0, tol=1e-9, parity=True)
        outs.append((r["lambda_"], r["matvecs"], r["v"].tobytes()))
    o = ref.min_eig_G(U, p, 10.0, tol=1e-9)
    print("lanczos s=%d" % s, "distinct runs:", len(set(outs)), "lambda", outs[0][0], "oracle", o["lambda_"],
          "matvecs", [x[1] for x in outs], "oracle", o["matvecs"], flush=True)
    cfg = H.SolverConfig(parity=True)
    outs = []
    for k in range(4):
        a = inst.aipp(p, 10.0, U, 1e-3, cfg)
        outs.append((a["status"], a["prox_iters"], a["fista_iters"], a["W"].tobytes(), a["g_value"]))
    from oracle import oracle as O
    oa = ref.aipp(p, 10.0, U, 1e-3)
    print("aipp s=%d" % s, "distinct runs:", len(set(outs)), "fista", [x[2] for x in outs], "oracle",
          oa["fista_iters"], "g", outs[0][4], oa["g_value"], flush=True)
