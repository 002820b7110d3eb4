"""First differing job phase between repeated parity-mode AIPP calls (or vs run 0)."""
import os
import sys

import numpy as np

os.environ["CUHALLAR_DEBUG_JOBS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

inst, ref = pair(sys.argv[1])
s = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(1)
U = rng.standard_normal((inst.n, 2))
U /= np.linalg.norm(U)
p = rng.standard_normal(inst.m) * 0.1
cfg = H.SolverConfig(parity=True)
runs = []
for k in range(8):
    inst.aipp(p, 10.0, U, 1e-3, cfg)
    runs.append([e for e in inst.last_trace() if e[0] == 10])
base = runs[0]
print("phases per run", [len(r) for r in runs])
for k, r in enumerate(runs[1:], 1):
    for i, (a, b) in enumerate(zip(base, r)):
        if a != b:
            print("run", k, "first differing phase", i, "K", a[6])
            print("  run0", a)
            print("  runk", b)
            for j in range(max(0, i - 3), i):
                print("  prev", j, base[j][6], base[j][2:6])
            break
    else:
        print("run", k, "identical")
