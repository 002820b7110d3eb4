"""Run-to-run determinism of the parity-mode solve: counters of repeated solves."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_13719_b200 as H  # noqa: E402
from parity_compare import pair  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
inst, _ = pair(name)
team = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for k in range(reps):
    r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True, team_ctas=team))
    print(name, k, r.fista_iters, r.aipp_iters, r.eig_products, r.rank, repr(r.pval), flush=True)
