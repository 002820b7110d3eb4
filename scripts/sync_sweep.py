import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_13719_b200 as H
inst = H.build_theta_instance(H.make_hypercube(12))
U = np.ones((inst.n, 2)) / 100.0
p = np.zeros(inst.m)
for ct in (148, 128, 96, 74, 48, 32, 16, 8, 2):
    s = inst.bench_pass("sync", U, p, iters=4000, team_ctas=ct)
    r = inst.bench_pass("allreduce", U, p, iters=4000, team_ctas=ct)
    print(ct, round(s, 1), round(r, 1), flush=True)
