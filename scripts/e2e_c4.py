"""Where the C4 e2e time goes: host samples -> instance (H2D + device CSR/SELL
build) -> first solve (workspace allocation) -> U, p back; vs a second solve on
the same instance.  python scripts/e2e_c4.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_13719_b200 as H

spec = H.McSpec(400000, 600000, 3, seed=0)
inst = H.gen_matrix_completion(spec)
ei, ej = inst.pairs()
hb = inst.b
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
ei, ej, hb = pin(ei), pin(ej), pin(hb)
tau = inst.tau
cfg = H.SolverConfig(eps=1e-5)
del inst
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    i2 = H.matcomp_from_samples(400000, 600000, ei, ej, hb, tau)
    t1 = time.perf_counter()
    r = H.solve(i2, cfg, fetch=False)
    t2 = time.perf_counter()
    r2 = H.solve(i2, cfg, fetch=True)
    t3 = time.perf_counter()
    del i2
    t4 = time.perf_counter()
    print(f"instance {t1-t0:.3f} s | solve#1 {t2-t1:.3f} (device {r.device_seconds:.3f}) | "
          f"solve#2+fetch {t3-t2:.3f} (device {r2.device_seconds:.3f}, wall {r2.wall_seconds:.3f}) | del {t4-t3:.3f}",
          flush=True)
