"""Run one bench_pass launch (after a warm-up launch) for ncu capture.
python scripts/ncu_pass.py H20 grad_pass 2 5   -> 2 hallar_kernel launches; capture with -s 1 -c 1"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2505_13719_b200 as H
name, kind, s, iters = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
if name.startswith("H"):
    inst = H.build_theta_instance(H.make_hypercube(int(name[1:])))
else:
    n1, n2, r = [int(x) for x in name[2:].split("_")]
    inst = H.gen_matrix_completion(H.McSpec(n1, n2, r, seed=0))
rng = np.random.default_rng(0)
U = rng.standard_normal((inst.n, s)); U /= np.linalg.norm(U)
p = rng.standard_normal(inst.m)
print("warm", inst.bench_pass(kind, U, p, beta=10.0, iters=iters))
print("target", inst.bench_pass(kind, U, p, beta=10.0, iters=iters))
