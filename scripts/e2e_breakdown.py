import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_13719_b200 as H
g = H.make_hypercube(12)
inst = H.build_theta_instance(g)
ei, ej = inst.pairs()
cfg = H.SolverConfig(eps=1e-5, seed=0)
H.solve(inst, cfg, fetch=False)
for it in range(6):
    t0 = time.perf_counter()
    gg = H.graph_from_edges(inst.n, np.stack([ei, ej], axis=1))
    t1 = time.perf_counter()
    i2 = H.build_theta_instance(gg)
    t2 = time.perf_counter()
    r = H.solve(i2, cfg, fetch=True)
    t3 = time.perf_counter()
    del i2
    t4 = time.perf_counter()
    print(f"graph {1e3*(t1-t0):.2f} build {1e3*(t2-t1):.2f} solve+fetch {1e3*(t3-t2):.2f} (device {1e3*r.device_seconds:.2f}, wall {1e3*r.wall_seconds:.2f}) del {1e3*(t4-t3):.2f}", flush=True)
