"""One parity-mode AIPP call (sanitizer target)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

inst, ref = pair(sys.argv[1])
rng = np.random.default_rng(1)
U = rng.standard_normal((inst.n, 2))
U /= np.linalg.norm(U)
p = rng.standard_normal(inst.m) * 0.1
a = inst.aipp(p, 10.0, U, 1e-3, H.SolverConfig(parity=True))
print(a["fista_iters"], a["g_value"])
